// walk_f32.cu -- production FP32 walk + exit-binning kernel for sm_100a.
//
// One persistent thread per walk slot, register-resident state, lanes refilled
// from a warp-local pool (em_pool.cuh).  The walk is the reference's
// walk-on-ellipsoids chain (S/_kernel.pyx:163-197, S/ = /root/reference/pkg/
// src/exitmeasure/) re-designed for SIMT FP32 issue:
//
//  * RNG: Philox4x32-10 keyed (seed) with counter (draw, rep_lo, pole, rep_hi)
//    -- blocks per lane per 8-step batch, so RNG is warp-uniform work, never
//    a divergent per-lane refill.  2D: a 16-bit azimuth per step (one block
//    per batch); 3D: a 16-bit z and a 16-bit azimuth (Archimedes' projection,
//    two blocks per batch).  No rejection loop (the reference's Marsaglia
//    trials diverge on SIMT).
//  * Step: x <- x + r(x) K^{1/2} u, with r = sd (EM_CHAIN_WOE, the reference
//    chain) or r = a certified lower bound of the largest inscribed
//    K^{1/2}-ellipsoid (EM_CHAIN_MAX; exact for planes, closed form for balls
//    and holes), shrunk by a relative + absolute FP32 margin so no step
//    leaves the closed domain by more than an ulp.
//  * Stop: Euclidean sd <= eps (the reference's shell, S/_kernel.pyx:177-180)
//    as one saturating FFMA that also masks the step; points a rounding step
//    outside count as exits too.
//  * Binning: owner component -> side (S/_kernel.pyx:145-156), then the
//    nearest anchor of that side's family in O(1): circle/square blocks by
//    angle / arc length (S/_kernel.pyx:260-313 without the window scan),
//    unstructured families through a conservative candidate grid.
//  * Accumulation: int64 global atomics on pole-interleaved rows (see
//    em_pool.cuh: concurrent walks spread over all rows, so no hot address).
#include "walk_f32_dev.cuh"

namespace em {
namespace f32 {


// MODE 0: bin exits into the count rows + per-pole step statistics
// MODE 1: write exit points / steps / components (em_run_exits)
// resident 256-thread blocks per SM the register allocation must allow:
// 5 in 2D (<= 51 registers; cfg3 +3%), 4 in 3D (<= 64; 5 costs cfg4 4%),
// measured with tools/ab_bench.sh EM_MIN_BLOCKS
#ifndef EM_MIN_BLOCKS
#define EM_MIN_BLOCKS 0
#endif
#ifndef EM_TAB_WARP
#define EM_TAB_WARP 0
#endif
#define EM_MINB(D) (EM_MIN_BLOCKS > 0 ? EM_MIN_BLOCKS : ((D) == 2 ? 5 : 4))
// 2D rolling disks carry more state per step: fewer resident blocks
#ifndef EM_ROLL2_BLOCKS
#define EM_ROLL2_BLOCKS 4
#endif
#define EM_MINB_K(D, OUTER, CHAIN) \
  ((D) == 2 && (OUTER) == OUTER_BALL && (CHAIN) == EM_CHAIN_TANGENT ? EM_ROLL2_BLOCKS : EM_MINB(D))
// Per-warp exit queue in shared memory: exit point + pole (as int bits in
// .w) and step count, binned 32 at a time.
struct ExitQueue {
  float4 x[kQueue];
  int s[kQueue];
};

template <int D, int OUTER, int NH, int CHAIN, bool IDENT, int MODE, int BINK, int SMEM>
__global__ void __launch_bounds__(256, EM_MINB_K(D, OUTER, CHAIN)) walk_f32_kernel(const F32Params P) {
  const WorkOut& W = P.w;
  constexpr bool SHEAR = Shear<D, OUTER, NH, CHAIN, IDENT>::value;
  __shared__ ExitQueue q_all[kWarps];
  // lane id, lane mask and the queue's shared-window address are made opaque
  // (empty asm) so the compiler keeps them in registers instead of
  // re-deriving them from special registers on every service pass
  int lane = threadIdx.x & 31;
  unsigned eq = 1u << lane, lt = eq - 1u;
  unsigned qb = (unsigned)__cvta_generic_to_shared(&q_all[threadIdx.x >> 5]);
  asm volatile("" : "+r"(lane), "+r"(eq), "+r"(lt), "+r"(qb));
  int qn = 0;  // queued exits of this warp (warp-uniform)
  // idle lanes sit far outside the domain: their distance is negative, so the
  // fast path's stop mask keeps them still without a separate lane flag
  constexpr float kFar = 1.0e4f;
  float x[3] = {kFar, kFar, kFar};
  float px = 0.0f, py = 0.0f, pz = 0.0f;  // this lane's cached pole (start point)
  int cpole = -1;
  unsigned cpid = 0;
  // steps doubles as the RNG draw counter: a walking lane has taken exactly
  // K steps per batch, so its batch index is steps / K
  int steps = 0, pole = 0, rep_off = 0;
  unsigned rep_lo = 0, rep_hi = 0;
  int walking = 0;     // lane flag as an int (bools become PRMT traffic in SASS)
  unsigned live = 0;   // warp mask of lanes holding a walk not yet retired
  WarpPool wp;
  pool_init(wp);
  StepAcc acc;
  acc_init(acc);
  if (MODE == 0 && SMEM != 2) stats_smem_init<SMEM>(W);
  // pole-block scheduler: this block walks replicates [r0, r0 + cnt) of one
  // pole (pole-major block order: concurrent blocks share few rows, which
  // stay L2-resident) into a shared histogram, flushed once at the end
  __shared__ unsigned s_next, s_done;
  __shared__ unsigned long long s_st[3];
  long long bpole = 0, br0 = 0;
  unsigned bcnt = 0;
  if (SMEM == 2) {
    bpole = (long long)blockIdx.x / W.splits;
    br0 = ((long long)blockIdx.x - bpole * W.splits) * W.bc;
    bcnt = (unsigned)(W.n_rep - br0 < W.bc ? W.n_rep - br0 : W.bc);
    unsigned* hist = block_hist();
    for (int i = threadIdx.x; i < W.row_len; i += blockDim.x) hist[i] = 0u;
    if (threadIdx.x == 0) {
      s_next = 0u;
      s_done = 0u;
      s_st[0] = s_st[1] = s_st[2] = 0ULL;
    }
    __syncthreads();
    const float4 p = __ldg(&P.poles[bpole]);
    px = p.x;
    py = p.y;
    pz = p.z;
    cpid = W.pole_ids ? (unsigned)W.pole_ids[bpole] : (unsigned)bpole;
    cpole = (int)bpole;
    acc.pole = (int)bpole;
  }
  constexpr bool TANG = Tangent<D, OUTER, NH, CHAIN, IDENT>::value;
  constexpr bool ROLL = Roll<D, OUTER, NH, CHAIN, IDENT>::value;
  constexpr bool SCALED = SHEAR || TANG;  // axes stored scaled (to_frame)
  // 3D tangent chain: the per-face constant rows, indexed per lane
#if EM_TAB_WARP
  // one copy per warp (warp-synchronous fill: no block barrier)
  __shared__ __align__(16) float ttab_all[(TANG && D == 3) ? 72 * kWarps : 1];
  float* ttab = ttab_all + ((TANG && D == 3) ? 72 * (threadIdx.x >> 5) : 0);
  if (TANG && D == 3) {
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
      for (int k = 0; k < 72; ++k) ttab[k] = P.t3[k / 24][k % 24];
    }
    __syncwarp();
  }
#else
  __shared__ __align__(16) float ttab[(TANG && D == 3) ? 72 : 1];
  if (TANG && D == 3) {
    if (threadIdx.x == 0) {  // constant indices: no dynamic parameter-space indexing
#pragma unroll
      for (int k = 0; k < 72; ++k) ttab[k] = P.t3[k / 24][k % 24];
    }
    __syncthreads();
  }
#endif
  // tangent chain: ~4 steps per walk, so 4-step batches (one Philox block,
  // one 32-bit word per step); elsewhere 8-step batches of 16-bit angles
  constexpr int K = (TANG || ROLL) ? EM_TANG_K : Batch<D>::kSteps;
  constexpr int NB = (TANG || ROLL) ? (EM_TANG_K + 3) / 4 : Batch<D>::kBlocks;
  for (;;) {
    // ---- service: retire finished walks, refill idle lanes ----
    const unsigned need = __ballot_sync(kFull, !walking);
    if (need) {
      const unsigned dm = need & live;  // walks that stopped in the last batch
      const bool done = (dm & eq) != 0u;
      if (MODE == 0) {
        if (dm) {
          if (done) {
            const unsigned slot = qn + __popc(dm & lt);
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(qb + slot * 16u),
                         "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(__int_as_float(pole))
                         : "memory");
            asm volatile("st.shared.s32 [%0], %1;" ::"r"(qb + kQueue * 16u + slot * 4u), "r"(steps)
                         : "memory");
          }
          qn += __popc(dm);
          if (qn >= 32) {  // bin 32 queued exits with every lane active
            __syncwarp();
            const unsigned slot = qn - 32 + lane;
            float ex[3], pw;
            int es;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(ex[0]), "=f"(ex[1]), "=f"(ex[2]), "=f"(pw)
                         : "r"(qb + slot * 16u)
                         : "memory");
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(es) : "r"(qb + kQueue * 16u + slot * 4u)
                         : "memory");
            retire<D, OUTER, NH, BINK, SMEM, SCALED>(P, ex, __float_as_int(pw), es, acc);
            qn -= 32;
            __syncwarp();
          }
        }
      } else if (done) {
        const long long o = (long long)pole * W.n_rep + rep_off;
        EM_DEV_ASSERT(o >= 0 && o < W.total);
        float xf[3];
        to_frame<D, OUTER, SCALED>(P, x, xf);
        double xd[3] = {(double)x[0], (double)x[1], D == 3 ? (double)x[2] : 0.0};
        if (OUTER == OUTER_BALL && P.rot) {
          double t[3] = {0.0, 0.0, 0.0};
          for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) t[i] += (double)P.Q[3 * i + j] * xd[j];
          for (int i = 0; i < D; ++i) xd[i] = t[i];
        } else if (SCALED) {
          for (int i = 0; i < D; ++i) xd[i] *= (double)P.ax[i];
        }
        for (int j = 0; j < D; ++j) W.x_out[o * D + j] = xd[j] + (double)P.frame[j];
        W.steps_out[o] = steps;
        W.comp_out[o] = owner<D, OUTER, NH>(P, xf);
      }
      bool took;
      if (SMEM == 2) {
        // claim replicates from the block's cursor (one shared atomic per warp)
        took = false;
        if (!wp.exhausted) {
          const unsigned n_need = __popc(need);
          unsigned base = 0u;
          if (eq == 1u) base = atomicAdd(&s_next, n_need);
          base = __shfl_sync(kFull, base, 0);
          if (base + n_need >= bcnt) wp.exhausted = 1;
          const unsigned k = base + __popc(need & lt);
          if ((need & eq) && k < bcnt) {
            pole = (int)bpole;
            rep_off = (int)(br0 + k);
            took = true;
          }
        }
      } else {
        took = pool_take_fast(wp, need, W, pole, rep_off, eq, lt);
      }
      if (took) {
        EM_DEV_ASSERT(pole >= 0 && pole < W.n_poles && rep_off >= 0 && rep_off < W.n_rep);
        if (SMEM != 2 && pole != cpole) {
          const float4 p = __ldg(&P.poles[pole]);
          px = p.x;
          py = p.y;
          pz = p.z;
          cpid = W.pole_ids ? (unsigned)W.pole_ids[pole] : (unsigned)pole;
          cpole = pole;
        }
        x[0] = px;
        x[1] = py;
        if (D == 3) x[2] = pz;
        const unsigned long long rep = (unsigned long long)W.rep_start + (unsigned)rep_off;
        rep_lo = (unsigned)rep;
        rep_hi = (unsigned)(rep >> 32);
        steps = 0;
        walking = 1;
      } else if (EM_POST_STOP && !walking) {
        // park a lane left without work: its exit point is already queued,
        // and the batch's own stop test need not agree with the post-batch
        // one to the last rounding (separately scheduled FMA chains), so an
        // idle lane must not sit on a borderline point it could walk from
        x[0] = x[1] = x[2] = kFar;
      }
      live = __ballot_sync(kFull, walking);
      if (wp.exhausted && live == 0) break;
    }
    // ---- a batch of K steps on one or two Philox blocks, branch-free ----
    unsigned wv[4 * NB];
    const unsigned draw = (unsigned)steps / (unsigned)K;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint4 w = philox4x32_10(P.rk, draw * NB + b, rep_lo, cpid, rep_hi);
      wv[4 * b] = w.x;
      wv[4 * b + 1] = w.y;
      wv[4 * b + 2] = w.z;
      wv[4 * b + 3] = w.w;
    }
    if (__all_sync(kFull, steps + K <= P.max_steps)) {
      // fast path: no lane can reach the step budget inside this batch.
      // Bookkeeping on the FMA pipes (the ALU pipe is the busy one): the
      // live mask is a float, FFMA.SAT((e - eps) * 2^k) -- exactly 0 when
      // e <= eps and exactly 1 otherwise, since every representable positive
      // difference scales to >= 1 -- and multiplies the step scale.  No
      // running product is needed: a stopped lane does not move, so every
      // later step of the batch recomputes the same e <= eps (and idle lanes
      // are parked outside the domain, e < 0).
      if (TANG || ROLL) {
        // tangent / rolling chains: the stop tests are compares (the same
        // thresholds the FFMA.SAT masks encode), steps count with predicated
        // integer adds -- as in the packed kernel (walk_f32x2.cu)
        bool go = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          float nx[3];
          if (ROLL && D == 3) go = roll3_go(P, x, wv[k], P.one_bits, nx);
          else if (ROLL) go = roll2_go<NH>(P, x, wv[k], P.one_bits, nx);
          else if (D == 2) go = tang2_go(P, x, wv[k], P.one_bits, nx);
          else go = tang3_go<OUTER>(P, ttab, x, wv[k], P.one_bits, nx);
#pragma unroll
          for (int l = 0; l < D; ++l) x[l] = go ? nx[l] : x[l];
          steps += go;
        }
        walking = go;
        if (EM_POST_STOP) {
          // the stop test of the point the last move landed on (the next
          // batch's first test, evaluated now): a walk that reached the shell
          // on a batch's last step retires at this service pass instead of
          // idling through one more batch (cfg2-cfg5 +9-12%).  Only the
          // predicate of the step functions is live here (the rest is dead
          // code); a lane left without work is parked far outside (service).
          float nx[3];
          bool g2;
          if (ROLL && D == 3) g2 = roll3_go(P, x, 0u, P.one_bits, nx);
          else if (ROLL) g2 = roll2_go<NH>(P, x, 0u, P.one_bits, nx);
          else if (D == 2) g2 = tang2_go(P, x, 0u, P.one_bits, nx);
          else g2 = tang3_go<OUTER>(P, ttab, x, 0u, P.one_bits, nx);
          walking &= g2;
        }
      } else {
        float wm = 0.0f, sf = 0.0f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          float t, r;
          dist<D, OUTER, NH, CHAIN, IDENT>(P, x, t, r);
          wm = t;  // already the saturated 0/1 mask
          step<D, OUTER, IDENT, SHEAR>(P, x, r * wm, D == 3 ? z_of<D>(wv, k, P.one_bits) : 0.0f,
                                       angle_bits<D>(wv, k, P.one_bits));
          sf += wm;
        }
        walking = wm != 0.0f;
        steps += (int)sf;
        if (EM_POST_STOP) {
          float t2, r2;
          dist<D, OUTER, NH, CHAIN, IDENT>(P, x, t2, r2);
          walking &= t2 != 0.0f;
        }
      }
    } else {
      int failed = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        float t = 0.0f, r, nx[3] = {0.0f, 0.0f, 0.0f};
        if (ROLL && D == 3) t = roll3_go(P, x, wv[k], P.one_bits, nx) ? 1.0f : 0.0f;
        else if (ROLL) t = roll2_go<NH>(P, x, wv[k], P.one_bits, nx) ? 1.0f : 0.0f;
        else if (TANG && D == 2) t = tang2_go(P, x, wv[k], P.one_bits, nx) ? 1.0f : 0.0f;
        else if (TANG) t = tang3_go<OUTER>(P, ttab, x, wv[k], P.one_bits, nx) ? 1.0f : 0.0f;
        else dist<D, OUTER, NH, CHAIN, IDENT>(P, x, t, r);
        const int stop = walking & (t <= 0.0f);
        const int over = walking & (stop ^ 1) & (steps >= P.max_steps);
        failed |= over;
        walking &= (stop ^ 1) & (over ^ 1);
        if (TANG || ROLL) {
#pragma unroll
          for (int l = 0; l < D; ++l) x[l] = walking ? nx[l] : x[l];
        } else {
          const float rs = walking ? r : 0.0f;
          step<D, OUTER, IDENT, SHEAR>(P, x, rs, D == 3 ? z_of<D>(wv, k, P.one_bits) : 0.0f,
                                       angle_bits<D>(wv, k, P.one_bits));
        }
        steps += walking;
      }
      // budget overruns: report (smallest key wins), drop from the live set
      // (never binned) and park the lane
      const unsigned fm = __ballot_sync(kFull, failed);
      if (fm) {
        if (failed) {
          atomicMax(W.err_key, ~(unsigned long long)((long long)pole * W.n_rep + rep_off));
          x[0] = x[1] = x[2] = kFar;
        }
        live &= ~fm;
      }
    }
  }
  if (MODE == 0) {
    __syncwarp();
    if (lane < qn) {  // drain the queue
      const ExitQueue& q = q_all[threadIdx.x >> 5];
      const float4 e = q.x[lane];
      const float ex[3] = {e.x, e.y, e.z};
      retire<D, OUTER, NH, BINK, SMEM, SCALED, false>(P, ex, __float_as_int(e.w), q.s[lane], acc);
    }
    if (SMEM == 2) {
      // step statistics: warp reduction, then the block's shared totals
      unsigned long long sm = acc.sum, sq = acc.sq, mx = acc.mx;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sm += __shfl_xor_sync(kFull, sm, o);
        sq += __shfl_xor_sync(kFull, sq, o);
        const unsigned long long t = __shfl_xor_sync(kFull, mx, o);
        mx = t > mx ? t : mx;
      }
      unsigned last = 0u;
      if (eq == 1u) {
        atomicAdd(&s_st[0], sm);
        atomicAdd(&s_st[1], sq);
        atomicMax(&s_st[2], mx);
        __threadfence_block();
        last = atomicAdd(&s_done, 1u) == (unsigned)(blockDim.x / 32 - 1);
      }
      last = __shfl_sync(kFull, last, 0);
      if (last) {
        // the block's last warp flushes the row: one int64 atomic per
        // touched bin, then the pole's statistics
        __threadfence_block();
        const unsigned* hist = block_hist();
        unsigned long long* row = W.counts + bpole * W.row_len;
        for (int i = lane; i < W.row_len; i += 32) {
          const unsigned v = hist[i];
          if (v) atomicAdd(&row[i], (unsigned long long)v);
        }
        if (eq == 1u) {
          atomicAdd(&W.ssum[bpole], s_st[0]);
          atomicAdd(&W.ssq[bpole], s_st[1]);
          atomicMax(&W.smax[bpole], s_st[2]);
        }
      }
    } else {
      acc_flush<SMEM>(acc, W);
      stats_smem_flush<SMEM>(W);
    }
  }
}

// One step of the walk chain from world points (em_debug_step): the same
// device functions as walk_f32_kernel, exposed so tests can check each
// sampler against closed forms (every landing point of a step lies on one
// whitened sphere and follows its Poisson kernel seen from the start point).
template <int D, int OUTER, int NH, int CHAIN, bool IDENT>
__global__ void __launch_bounds__(128) debug_step_kernel(const F32Params P, const double* xin,
                                                         const unsigned* words, long long n,
                                                         double* yout, float* mout) {
  constexpr bool SHEAR = Shear<D, OUTER, NH, CHAIN, IDENT>::value;
  constexpr bool TANG = Tangent<D, OUTER, NH, CHAIN, IDENT>::value;
  constexpr bool ROLL = Roll<D, OUTER, NH, CHAIN, IDENT>::value;
  constexpr bool SCALED = SHEAR || TANG;
  __shared__ __align__(16) float ttab[72];
  if (TANG && D == 3) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < 72; ++k) ttab[k] = P.t3[k / 24][k % 24];
    }
    __syncthreads();
  }
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  // world -> kernel coordinates (capi.cu's to_kernel on the device)
  double v[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < D; ++k) v[k] = xin[j * D + k] - (double)P.frame[k];
  float x[3] = {0.0f, 0.0f, 0.0f};
  for (int k = 0; k < D; ++k) {
    double t = 0.0;
    if (OUTER == OUTER_BALL && P.rot) {
      for (int i = 0; i < D; ++i) t += (double)P.Q[3 * i + k] * v[i];
    } else if (SCALED) {
      t = v[k] / (double)P.ax[k];
    } else {
      t = v[k];
    }
    x[k] = (float)t;
  }
  const unsigned w0 = words[2 * j], w1 = words[2 * j + 1];
  float nx[3] = {x[0], x[1], x[2]}, m = 0.0f;
  if (ROLL && D == 3) {
    m = roll_step3(P, x, w0, P.one_bits, nx);
  } else if (ROLL) {
    m = roll_step2<NH>(P, x, w0, P.one_bits, nx);
  } else if (TANG && D == 2) {
    m = tangent_step(P, x, w0, P.one_bits, nx[0], nx[1]);
  } else if (TANG) {
    m = tangent_step3<OUTER>(P, ttab, x, w0, P.one_bits, nx);
  } else {
    // the batch layout of the woe / max chains: z words, then azimuth words
    const unsigned wv[8] = {w0, w0, w0, w0, D == 3 ? w1 : w0, w1, w1, w1};
    float t, r;
    dist<D, OUTER, NH, CHAIN, IDENT>(P, x, t, r);
    m = t;
    step<D, OUTER, IDENT, SHEAR>(P, nx, r, D == 3 ? z_of<D>(wv, 0, P.one_bits) : 0.0f,
                                 angle_bits<D>(wv, 0, P.one_bits));
  }
  // kernel -> world in double (the exits mode's conversion)
  double xd[3] = {(double)nx[0], (double)nx[1], D == 3 ? (double)nx[2] : 0.0};
  if (OUTER == OUTER_BALL && P.rot) {
    double t[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < D; ++i)
      for (int k = 0; k < D; ++k) t[i] += (double)P.Q[3 * i + k] * xd[k];
    for (int i = 0; i < D; ++i) xd[i] = t[i];
  } else if (SCALED) {
    for (int i = 0; i < D; ++i) xd[i] *= (double)P.ax[i];
  }
  for (int k = 0; k < D; ++k) yout[j * D + k] = xd[k] + (double)P.frame[k];
  mout[j] = m;
}

}  // namespace f32

cudaError_t launch_debug_step(const F32Params& P, int d, int outer, int nh_mode, int chain,
                              bool ident, const double* x, const unsigned* words, long long n,
                              double* y, float* mask, cudaStream_t s) {
  using namespace f32;
  using K = void (*)(F32Params, const double*, const unsigned*, long long, double*, float*);
  K k = nullptr;
  const int nh = nh_mode;  // 0: none, 1: one hole (2D ball), 2: runtime count
#define EM_DBG(D_, O_, NH_, C_, I_) \
  if (d == D_ && outer == O_ && nh == (NH_ < 0 ? 2 : NH_) && chain == C_ && ident == I_) \
    k = debug_step_kernel<D_, O_, NH_, C_, I_>;
  if (ident) {
    EM_DBG(2, OUTER_BALL, 0, EM_CHAIN_WOE, true)
    EM_DBG(3, OUTER_BALL, 0, EM_CHAIN_WOE, true)
    EM_DBG(2, OUTER_BOX, 0, EM_CHAIN_WOE, true)
  } else if (chain == EM_CHAIN_TANGENT) {
    EM_DBG(2, OUTER_BOX, 0, EM_CHAIN_TANGENT, false)
    EM_DBG(3, OUTER_BOX, 0, EM_CHAIN_TANGENT, false)
    EM_DBG(3, OUTER_LBOX, 0, EM_CHAIN_TANGENT, false)
    EM_DBG(3, OUTER_BALL, 0, EM_CHAIN_TANGENT, false)
    EM_DBG(2, OUTER_BALL, 0, EM_CHAIN_TANGENT, false)
    EM_DBG(2, OUTER_BALL, 1, EM_CHAIN_TANGENT, false)
  } else if (chain == EM_CHAIN_MAX) {
    EM_DBG(2, OUTER_BOX, 0, EM_CHAIN_MAX, false)
    EM_DBG(3, OUTER_BOX, 0, EM_CHAIN_MAX, false)
    EM_DBG(3, OUTER_LBOX, 0, EM_CHAIN_MAX, false)
    EM_DBG(3, OUTER_BALL, 0, EM_CHAIN_MAX, false)
    EM_DBG(2, OUTER_BALL, 0, EM_CHAIN_MAX, false)
    EM_DBG(2, OUTER_BALL, 1, EM_CHAIN_MAX, false)
  } else {
    EM_DBG(2, OUTER_BOX, 0, EM_CHAIN_WOE, false)
    EM_DBG(3, OUTER_BOX, 0, EM_CHAIN_WOE, false)
    EM_DBG(3, OUTER_BALL, 0, EM_CHAIN_WOE, false)
    EM_DBG(2, OUTER_BALL, 0, EM_CHAIN_WOE, false)
    EM_DBG(2, OUTER_BALL, 1, EM_CHAIN_WOE, false)
  }
#undef EM_DBG
  if (!k) return cudaErrorInvalidValue;
  k<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(P, x, words, n, y, mask);
  return cudaGetLastError();
}

// Host dispatch over the instantiated (dimension, outer, holes, chain, K=I,
// binner) combinations.  nh_mode: 0 = no holes, 1 = exactly one hole, 2 =
// runtime count.  Specialised binners exist where a BASELINE config needs
// them; everything else takes BIN_ANY.
using F32Kernel = void (*)(F32Params);

// smem: 0 = persistent pole-cycling warps, 1 = the same with per-warp shared
// step-statistics tables (tiny jobs), 2 = the pole-block scheduler with a
// shared-memory histogram per block (capi.cu picks it for long rows; only
// the closed-form / grid binners are instantiated with it)
#define EM_SCHED3(ARGS, BK)                                                          \
  (smem == 2 ? walk_f32_kernel<EM_UNPAREN ARGS, 0, BK, 2>                              \
             : (smem ? walk_f32_kernel<EM_UNPAREN ARGS, 0, BK, 1>                      \
                     : walk_f32_kernel<EM_UNPAREN ARGS, 0, BK, 0>))
#define EM_UNPAREN(...) __VA_ARGS__

template <int D, int OUTER, int NH, int BINK, int SM>
static F32Kernel pick_chain_sm(int mode, int chain, bool ident) {
  using namespace f32;
  if (mode != 0) {
    if (ident) return walk_f32_kernel<D, OUTER, NH, EM_CHAIN_WOE, true, 1, BIN_ANY, 0>;
    if (chain == EM_CHAIN_MAX) return walk_f32_kernel<D, OUTER, NH, EM_CHAIN_MAX, false, 1, BIN_ANY, 0>;
    return walk_f32_kernel<D, OUTER, NH, EM_CHAIN_WOE, false, 1, BIN_ANY, 0>;
  }
  if (ident) return walk_f32_kernel<D, OUTER, NH, EM_CHAIN_WOE, true, 0, BINK, SM>;
  if (chain == EM_CHAIN_MAX) return walk_f32_kernel<D, OUTER, NH, EM_CHAIN_MAX, false, 0, BINK, SM>;
  return walk_f32_kernel<D, OUTER, NH, EM_CHAIN_WOE, false, 0, BINK, SM>;
}

template <int D, int OUTER, int NH, int BINK>
static F32Kernel pick_chain(int mode, int chain, bool ident, int smem) {
  if (smem >= 2) return nullptr;  // the pole-block scheduler: tangent chains only
  return smem ? pick_chain_sm<D, OUTER, NH, BINK, 1>(mode, chain, ident)
              : pick_chain_sm<D, OUTER, NH, BINK, 0>(mode, chain, ident);
}

template <int D, int OUTER, int NH, int B1, int B2>
static F32Kernel pick_bin(int mode, int chain, bool ident, int bink, int smem) {
  if (mode == 0 && bink == B1 && B1 != f32::BIN_ANY) return pick_chain<D, OUTER, NH, B1>(mode, chain, ident, smem);
  if (mode == 0 && bink == B2 && B2 != f32::BIN_ANY) return pick_chain<D, OUTER, NH, B2>(mode, chain, ident, smem);
  return pick_chain<D, OUTER, NH, f32::BIN_ANY>(mode, chain, ident, smem);
}

static F32Kernel pick_f32(int d, int outer, int nh_mode, int mode, int chain, bool ident, int bink,
                          int smem) {
  using namespace f32;
  if (d == 2) {
    if (outer == OUTER_BALL && nh_mode <= 1 && chain == EM_CHAIN_TANGENT && !ident) {
      // rolling disks (capi.cu resolves the chain: no hole or one concentric hole)
      if (nh_mode == 0) {
        if (mode != 0) return walk_f32_kernel<2, OUTER_BALL, 0, EM_CHAIN_TANGENT, false, 1, BIN_ANY, 0>;
        if (bink == BIN_CIRCLE)
          return EM_SCHED3((2, OUTER_BALL, 0, EM_CHAIN_TANGENT, false), BIN_CIRCLE);
        return smem >= 2 ? (F32Kernel) nullptr : smem ? walk_f32_kernel<2, OUTER_BALL, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 1>
                    : walk_f32_kernel<2, OUTER_BALL, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 0>;
      }
      if (mode != 0) return walk_f32_kernel<2, OUTER_BALL, 1, EM_CHAIN_TANGENT, false, 1, BIN_ANY, 0>;
      if (bink == BIN_CIRCLE)
        return EM_SCHED3((2, OUTER_BALL, 1, EM_CHAIN_TANGENT, false), BIN_CIRCLE);
      return smem >= 2 ? (F32Kernel) nullptr : smem ? walk_f32_kernel<2, OUTER_BALL, 1, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 1>
                    : walk_f32_kernel<2, OUTER_BALL, 1, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 0>;
    }
    if (outer == OUTER_BALL) {
      if (nh_mode == 0) return pick_bin<2, OUTER_BALL, 0, BIN_CIRCLE, BIN_ANY>(mode, chain, ident, bink, smem);
      if (nh_mode == 1) return pick_bin<2, OUTER_BALL, 1, BIN_CIRCLE, BIN_ANY>(mode, chain, ident, bink, smem);
      return pick_bin<2, OUTER_BALL, -1, BIN_CIRCLE, BIN_ANY>(mode, chain, ident, bink, smem);
    }
    if (outer == OUTER_BOX) {
      if (nh_mode == 0 && chain == EM_CHAIN_TANGENT && !ident) {
        // the tangent-ball chain exists for this one geometry (capi.cu
        // resolves EM_CHAIN_TANGENT to EM_CHAIN_MAX everywhere else)
        if (mode != 0) return walk_f32_kernel<2, OUTER_BOX, 0, EM_CHAIN_TANGENT, false, 1, BIN_ANY, 0>;
        if (bink == BIN_SQUARE)
          return EM_SCHED3((2, OUTER_BOX, 0, EM_CHAIN_TANGENT, false), BIN_SQUARE);
        if (bink == BIN_GRID)
          return EM_SCHED3((2, OUTER_BOX, 0, EM_CHAIN_TANGENT, false), BIN_GRID);
        return smem >= 2 ? (F32Kernel) nullptr : smem ? walk_f32_kernel<2, OUTER_BOX, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 1>
                    : walk_f32_kernel<2, OUTER_BOX, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 0>;
      }
      if (nh_mode == 0) return pick_bin<2, OUTER_BOX, 0, BIN_SQUARE, BIN_GRID>(mode, chain, ident, bink, smem);
      return pick_bin<2, OUTER_BOX, -1, BIN_ANY, BIN_ANY>(mode, chain, ident, bink, smem);
    }
    return nullptr;
  }
  if (outer == OUTER_BALL) {
    if (nh_mode == 0 && chain == EM_CHAIN_TANGENT && !ident) {
      // rolling balls (capi.cu resolves the chain)
      if (mode != 0) return walk_f32_kernel<3, OUTER_BALL, 0, EM_CHAIN_TANGENT, false, 1, BIN_ANY, 0>;
      if (bink == BIN_GRID)
        return EM_SCHED3((3, OUTER_BALL, 0, EM_CHAIN_TANGENT, false), BIN_GRID);
      return smem >= 2 ? (F32Kernel) nullptr : smem ? walk_f32_kernel<3, OUTER_BALL, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 1>
                    : walk_f32_kernel<3, OUTER_BALL, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 0>;
    }
    if (nh_mode == 0) return pick_bin<3, OUTER_BALL, 0, BIN_GRID, BIN_ANY>(mode, chain, ident, bink, smem);
    return pick_bin<3, OUTER_BALL, -1, BIN_GRID, BIN_ANY>(mode, chain, ident, bink, smem);
  }
  if (nh_mode == 0 && chain == EM_CHAIN_TANGENT && !ident && outer != OUTER_BALL) {
    // 3D box / L-box on tangent balls (capi.cu resolves the chain)
    if (outer == OUTER_BOX) {
      if (mode != 0) return walk_f32_kernel<3, OUTER_BOX, 0, EM_CHAIN_TANGENT, false, 1, BIN_ANY, 0>;
      if (bink == BIN_GRID)
        return EM_SCHED3((3, OUTER_BOX, 0, EM_CHAIN_TANGENT, false), BIN_GRID);
      return smem >= 2 ? (F32Kernel) nullptr : smem ? walk_f32_kernel<3, OUTER_BOX, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 1>
                    : walk_f32_kernel<3, OUTER_BOX, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 0>;
    }
    if (mode != 0) return walk_f32_kernel<3, OUTER_LBOX, 0, EM_CHAIN_TANGENT, false, 1, BIN_ANY, 0>;
    if (bink == BIN_GRID)
      return EM_SCHED3((3, OUTER_LBOX, 0, EM_CHAIN_TANGENT, false), BIN_GRID);
    return smem >= 2 ? (F32Kernel) nullptr : smem ? walk_f32_kernel<3, OUTER_LBOX, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 1>
                    : walk_f32_kernel<3, OUTER_LBOX, 0, EM_CHAIN_TANGENT, false, 0, BIN_ANY, 0>;
  }
  if (outer == OUTER_BOX) {
    if (nh_mode == 0) return pick_bin<3, OUTER_BOX, 0, BIN_GRID, BIN_ANY>(mode, chain, ident, bink, smem);
    return pick_bin<3, OUTER_BOX, -1, BIN_ANY, BIN_ANY>(mode, chain, ident, bink, smem);
  }
  if (nh_mode == 0) return pick_bin<3, OUTER_LBOX, 0, BIN_GRID, BIN_ANY>(mode, chain, ident, bink, smem);
  return pick_bin<3, OUTER_LBOX, -1, BIN_ANY, BIN_ANY>(mode, chain, ident, bink, smem);
}

cudaError_t launch_f32(const F32Params& P, int d, int outer, int nh_mode, int mode, int chain,
                       bool ident, int bink, int grid, int block, cudaStream_t s) {
  if (block != 32 * f32::kWarps) return cudaErrorInvalidConfiguration;
  const int sched = mode == 0 ? P.w.smem_stats : 0;
  F32Kernel k = pick_f32(d, outer, nh_mode, mode, chain, ident, bink, sched);
  if (!k) return cudaErrorInvalidValue;
  size_t smem = 0;
  if (sched == 1) smem = (size_t)f32::kWarps * 3 * P.w.n_poles * 8;
  if (sched == 2) {
    // one block per (pole, replicate range), the row's histogram in shared
    smem = ((size_t)P.w.row_len * 4 + 15) & ~(size_t)15;
    grid = (int)(P.w.n_poles * P.w.splits);
    // the attribute is per (kernel, device context): remember both
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, size_t>> set;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    bool done = false;
    for (auto& e : set)
      if (e.first.first == (const void*)k && e.first.second == dev && e.second >= smem) done = true;
    if (!done) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      set.push_back({{(const void*)k, dev}, smem});
    }
  }
  k<<<grid, block, smem, s>>>(P);
  return cudaGetLastError();
}

// the pole-block scheduler exists for this plan's kernel family
bool f32_has_pole_blocks(int d, int outer, int nh_mode, int chain, bool ident, int bink) {
  return pick_f32(d, outer, nh_mode, 0, chain, ident, bink, 2) != nullptr;
}

cudaError_t f32_blocks_per_sm(int d, int outer, int nh_mode, int chain, bool ident, int bink,
                              int* nb) {
  F32Kernel k = pick_f32(d, outer, nh_mode, 0, chain, ident, bink, 0);
  if (!k) return cudaErrorInvalidValue;
  // per (kernel, device): the query costs microseconds on every plan otherwise
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::pair<const void*, int> key{(const void*)k, dev};
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : cache)
      if (e.first == key) {
        *nb = e.second;
        return cudaSuccess;
      }
  }
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb, k, 32 * f32::kWarps, 0);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    cache.push_back({key, *nb});
  }
  return e;
}

// Compile knobs of this translation unit (em_build_info): every macro that
// changes the FP32 kernel's arithmetic or schedule, as built.
#ifndef EM_X2_BLOCKS
#define EM_X2_BLOCKS 4
#endif
#define EM_STR2(x) #x
#define EM_STR(x) EM_STR2(x)
const char* f32_build_knobs() {
  return "EM_BATCH_STEPS=" EM_STR(EM_BATCH_STEPS) " EM_ANGLE_BITS=" EM_STR(EM_ANGLE_BITS)
         " EM_Z_BITS=" EM_STR(EM_Z_BITS) " EM_TANG_K=" EM_STR(EM_TANG_K)
         " EM_POST_STOP=" EM_STR(EM_POST_STOP) " EM_MIN_BLOCKS=" EM_STR(EM_MIN_BLOCKS)
         " EM_ROLL2_BLOCKS=" EM_STR(EM_ROLL2_BLOCKS) " EM_ROLL2_DYN=" EM_STR(EM_ROLL2_DYN)
         " EM_TAB_WARP=" EM_STR(EM_TAB_WARP) " EM_ROLL2_ONE=" EM_STR(EM_ROLL2_ONE)
         " EM_POLY_SINCOS=" EM_STR(EM_POLY_SINCOS) " EM_X2_BLOCKS=" EM_STR(EM_X2_BLOCKS)
         " EM_DEBUG=" EM_STR(EM_DEBUG);
}

// ---- FP32 point binning (same owner/binner as the walk kernel) ----
template <int D, int OUTER>
__global__ void bin_points_f32_kernel(const F32Params P, const double* pts, long long n,
                                      long long* comp_out, long long* side_out,
                                      long long* bin_out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  float xf[3] = {0.0f, 0.0f, 0.0f}, xw[3] = {0.0f, 0.0f, 0.0f};
  double v[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < D; ++k) {
    xw[k] = (float)pts[j * D + k];
    v[k] = pts[j * D + k] - (double)P.frame[k];
  }
  if (OUTER == OUTER_BALL && P.rot) {  // Q^T v: the frame the hole centres live in
    for (int k = 0; k < D; ++k) {
      double t = 0.0;
      for (int i = 0; i < D; ++i) t += (double)P.Q[3 * i + k] * v[i];
      xf[k] = (float)t;
    }
  } else {
    for (int k = 0; k < D; ++k) xf[k] = (float)v[k];
  }
  const int comp = f32::owner<D, OUTER, -1>(P, xf);
  const int side = P.comp_side[comp];
  comp_out[j] = comp;
  side_out[j] = side;
  bin_out[j] = P.side[side].n_anchors > 0 ? f32::nearest_anchor<D>(side ? P.side[1] : P.side[0], xw) : -1;
}

cudaError_t launch_bin_points_f32(const F32Params& P, int d, int outer, const double* pts,
                                  long long n, long long* comp, long long* side, long long* bin,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const unsigned g = (unsigned)((n + 127) / 128);
  if (d == 2 && outer == OUTER_BALL) bin_points_f32_kernel<2, OUTER_BALL><<<g, 128, 0, s>>>(P, pts, n, comp, side, bin);
  else if (d == 2) bin_points_f32_kernel<2, OUTER_BOX><<<g, 128, 0, s>>>(P, pts, n, comp, side, bin);
  else if (outer == OUTER_BALL) bin_points_f32_kernel<3, OUTER_BALL><<<g, 128, 0, s>>>(P, pts, n, comp, side, bin);
  else if (outer == OUTER_BOX) bin_points_f32_kernel<3, OUTER_BOX><<<g, 128, 0, s>>>(P, pts, n, comp, side, bin);
  else bin_points_f32_kernel<3, OUTER_LBOX><<<g, 128, 0, s>>>(P, pts, n, comp, side, bin);
  return cudaGetLastError();
}

// ---- zero up to 4 output ranges with ONE launch (instead of a memset each) ----
struct ZeroRanges {
  unsigned long long* p[4];
  long long n[4];  // 8-byte words
};

__global__ void zero_ranges_kernel(const ZeroRanges z, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long j = i;
    int r = 0;
    while (j >= z.n[r]) j -= z.n[r++];
    z.p[r][j] = 0ULL;
  }
}

cudaError_t launch_zero_ranges(unsigned long long* const* ptrs, const long long* words, int n,
                               cudaStream_t s) {
  ZeroRanges z{};
  long long total = 0;
  int k = 0;
  for (int i = 0; i < n && k < 4; ++i)
    if (ptrs[i] && words[i] > 0) {
      z.p[k] = ptrs[i];
      z.n[k] = words[i];
      total += words[i];
      ++k;
    }
  if (total == 0) return cudaSuccess;
  const long long blocks = std::min<long long>((total + 255) / 256, 148LL * 8);
  zero_ranges_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, total);
  return cudaGetLastError();
}

// ---- count rows -> float64 in place (em_plan_run_host_f64: the reference's
// float64 raw rows straight from the device; exact below 2^53) ----
__global__ void rows_to_f64_kernel(unsigned long long* rows, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    rows[i] = (unsigned long long)__double_as_longlong((double)(long long)rows[i]);
}

cudaError_t launch_rows_to_f64(unsigned long long* rows, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 8);
  rows_to_f64_kernel<<<(unsigned)blocks, 256, 0, s>>>(rows, n);
  return cudaGetLastError();
}

// ---- fold the step-statistics copies (WorkOut::stat_copies) ----
__global__ void stats_fold_kernel(const unsigned long long* scratch, int copies, long long n_poles,
                                  unsigned long long* stats) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // over 3 n_poles
  if (i >= 3 * n_poles) return;
  const bool is_max = i >= 2 * n_poles;
  unsigned long long v = 0;
  for (int c = 0; c < copies; ++c) {
    const unsigned long long w = scratch[(long long)c * 3 * n_poles + i];
    v = is_max ? (w > v ? w : v) : v + w;
  }
  stats[i] = v;
}

cudaError_t launch_stats_fold(const unsigned long long* scratch, int copies, long long n_poles,
                              unsigned long long* stats, cudaStream_t s) {
  const long long n = 3 * n_poles;
  stats_fold_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(scratch, copies, n_poles, stats);
  return cudaGetLastError();
}

// ---- FP32 issue-rate micro-benchmark (roofline denominator) ----
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters, float a, float b) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fmaf(v[i], a, b);
  }
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

cudaError_t launch_ffma_peak(float* out, int iters, int grid, int block, cudaStream_t s) {
  ffma_peak_kernel<<<grid, block, 0, s>>>(out, iters, 0.999999f, 1e-7f);
  return cudaGetLastError();
}

// Philox4x32-10 known-answer hook (compared with curand in the tests).
__global__ void philox32_kat_kernel(const unsigned* in, unsigned* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned* c = in + 6 * i;
  const PhiloxKey32 k = philox32_schedule(c[4], c[5]);  // KAT only
  const uint4 w = philox4x32_10(k, c[0], c[1], c[2], c[3]);
  out[4 * i] = w.x;
  out[4 * i + 1] = w.y;
  out[4 * i + 2] = w.z;
  out[4 * i + 3] = w.w;
}

cudaError_t launch_philox32_kat(const unsigned* in, unsigned* out, int n, cudaStream_t s) {
  philox32_kat_kernel<<<(n + 127) / 128, 128, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace em
