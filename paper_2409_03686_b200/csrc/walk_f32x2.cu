// walk_f32x2.cu -- two walks per lane with packed FP32 arithmetic (sm_100a).
//
// Blackwell's FFMA2 / FMUL2 / FADD2 (PTX fma/mul/add.f32x2) do two FP32
// operations per lane in ONE issued instruction on a 64-bit register pair, at
// the FMA pipe's full lane rate.  The walk kernel is bound by instructions
// issued, so a lane that carries TWO walks -- their
// coordinates as the halves of one register pair -- runs every add / multiply
// / fma of the step function once for both.  Roots, reciprocals, sin / cos,
// compares, min / max and selects stay one per walk; Philox, the service
// pass and the exit queue are per walk as before.
//
// Same chain, same stop test, same RNG streams (keyed by global pole id and
// replicate index) and the same operation tree as the one-walk-per-lane
// kernel (walk_f32.cu), so a walk does not depend on which kernel or slot
// runs it.  Built for the chains whose step is written over a value type in
// walk_f32_dev.cuh: the 2D ball on rolling disks with no hole or one
// concentric hole (cfg3, the headline; roll2_core), the 2D box on tangent
// balls (cfg2; tang2_core) and the 3D ball on rolling balls (cfg4;
// roll3_core).  The L-box chain reads per-face constants from shared memory
// at a lane-dependent row and stays on the one-walk kernel.
#include "walk_f32_dev.cuh"

// resident 256-thread blocks per SM: 4 (64 registers, a few spilled words in
// the service pass) measured 2.4% faster than 3 (77 registers, no spills) and
// 12% faster than 2 (110 registers: too few warps to cover the MUFU latency)
#ifndef EM_X2_BLOCKS
#define EM_X2_BLOCKS 4
#endif
// the 3D ball's rolling-ball chain on the packed kernel: 3 resident blocks
// (80 registers, no spills; 2 blocks -14%, 4 blocks -1.4%)
#ifndef EM_X2_3D
#define EM_X2_3D 1
#endif
#ifndef EM_X2_BLOCKS3
#define EM_X2_BLOCKS3 3
#endif

namespace em {
namespace f32 {

// walking <=> s2_lo < |x|^2 < s2_hi: the thresholds of the one-walk kernel's
// FFMA.SAT masks (exactly: its scales are powers of two), as two compares
template <int NH>
__device__ __forceinline__ Mask2 walking2(const F32Params& P, float2 s2) {
  Mask2 g = vlt(s2, P.s2_hi);
  if (NH == 1) g = vand(g, vgt(s2, P.s2_lo));
  return g;
}

// CH: 0 = 2D ball, no hole; 1 = 2D ball, one concentric hole (rolling disks);
// 2 = 2D box (tangent balls); 3 = 3D ball, no hole (rolling balls).  One step
// of both walks: candidate points and the walking masks of the CURRENT points.
template <int CH>
__device__ __forceinline__ Mask2 step2(const F32Params& P, float2 x0, float2 x1, float2 x2,
                                       uint2 w, float2& n0, float2& n1, float2& n2) {
  if (CH == 3) {
    float2 s2;
    roll3_core<float2, uint2>(P, x0, x1, x2, w, P.one_bits, s2, n0, n1, n2);
    return vlt(s2, P.s2_hi);
  }
  n2 = x2;
  if (CH == 2) {
    float2 a0, a1;
    tang2_core<float2, uint2>(P, x0, x1, w, P.one_bits, a0, a1, n0, n1);
    return vand(vlt(a0, P.tsb[0]), vlt(a1, P.tsb[1]));
  }
  float2 s2;
  roll2_core<CH == 1 ? 1 : 0, float2, uint2>(P, x0, x1, w, P.one_bits, s2, n0, n1);
  return walking2<CH == 1 ? 1 : 0>(P, s2);
}

// the walking masks alone (post-batch stop test)
template <int CH>
__device__ __forceinline__ Mask2 walking_at(const F32Params& P, float2 x0, float2 x1, float2 x2) {
  if (CH == 3) return vlt(vfma(x2, x2, vfma(x1, x1, vmul(x0, x0))), P.s2_hi);
  if (CH == 2) return vand(vlt(vabs(x0), P.tsb[0]), vlt(vabs(x1), P.tsb[1]));
  return walking2<CH == 1 ? 1 : 0>(P, roll2_s2(x0, x1));
}

// Per-warp exit queue as four word arrays (x, y, pole, steps): a lane's two
// walks keep each AXIS as one register pair, so a slot's (x, y) are not
// adjacent registers and a 128-bit store would cost moves every batch.
template <int D>
struct ExitQueue2 {
  float x[kQueue], y[kQueue];
  int p[kQueue], s[kQueue];
  float z[D == 3 ? kQueue : 1];
};

__device__ __forceinline__ float& comp(float2& v, int t) { return t ? v.y : v.x; }

// Two walks per lane: slot t of a lane owns component t of every float2.
// Scheduling, exit queue, binning and statistics as walk_f32_kernel (MODE 0).
template <int CH, int BINK, int SMEM>
__global__ void __launch_bounds__(256, CH == 3 ? EM_X2_BLOCKS3 : EM_X2_BLOCKS)
    walk_f32x2_kernel(const F32Params P) {
  const WorkOut& W = P.w;
  constexpr int D = CH == 3 ? 3 : 2;
  constexpr int OUTER = CH == 2 ? OUTER_BOX : OUTER_BALL;
  constexpr int NH = CH == 1 ? 1 : 0;
  constexpr bool SCALED = CH == 2;  // box axes stored scaled (to_frame)
  __shared__ ExitQueue2<D> q_all[kWarps];
  int lane = threadIdx.x & 31;
  unsigned eq = 1u << lane, lt = eq - 1u;
  unsigned qb = (unsigned)__cvta_generic_to_shared(&q_all[threadIdx.x >> 5]);
  asm volatile("" : "+r"(lane), "+r"(eq), "+r"(lt), "+r"(qb));
  int qn = 0;
  constexpr float kFar = 1.0e4f;
  // axis 0 / 1 / 2 of both slots
  float2 X0 = make_float2(kFar, kFar), X1 = make_float2(kFar, kFar), X2 = make_float2(kFar, kFar);
  float px = 0.0f, py = 0.0f, pz = 0.0f;  // cached pole (shared by both slots)
  int cpole = -1;
  unsigned ccpid = 0;
  int steps[2] = {0, 0}, pole[2] = {0, 0}, rep_off[2] = {0, 0};
  unsigned rep_lo[2] = {0, 0}, rep_hi[2] = {0, 0}, cpid[2] = {0, 0};
  int walking[2] = {0, 0};
  unsigned live[2] = {0, 0};
  WarpPool wp;
  pool_init(wp);
  StepAcc acc;
  acc_init(acc);
  if (SMEM != 2) stats_smem_init<SMEM>(W);
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
    ccpid = W.pole_ids ? (unsigned)W.pole_ids[bpole] : (unsigned)bpole;
    cpole = (int)bpole;
    acc.pole = (int)bpole;
  }
  // 4-step batches, one 32-bit word per step (5 steps of 23-bit fields from
  // the same block measured +0.3%, 6 of 21 bits -1.4%, 3 steps -4.9%)
  constexpr int K = EM_TANG_K;
  static_assert(EM_TANG_K <= 4, "one Philox block per batch");
  for (;;) {
    // ---- service: retire finished walks, refill idle slots ----
    const unsigned need0 = __ballot_sync(kFull, !walking[0]);
    const unsigned need1 = __ballot_sync(kFull, !walking[1]);
    if (need0 | need1) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const unsigned need = t ? need1 : need0;
        if (need == 0u) continue;
        const unsigned dm = need & live[t];
        const bool done = (dm & eq) != 0u;
        if (dm) {
          if (done) {
            const unsigned slot = qn + __popc(dm & lt);
            const unsigned qa = qb + slot * 4u;
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(qa), "f"(comp(X0, t)) : "memory");
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(qa + kQueue * 4u), "f"(comp(X1, t)) : "memory");
            asm volatile("st.shared.s32 [%0], %1;" ::"r"(qa + kQueue * 8u), "r"(pole[t]) : "memory");
            asm volatile("st.shared.s32 [%0], %1;" ::"r"(qa + kQueue * 12u), "r"(steps[t]) : "memory");
            if (D == 3)
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(qa + kQueue * 16u), "f"(comp(X2, t)) : "memory");
          }
          qn += __popc(dm);
          if (qn >= 32) {
            __syncwarp();
            const unsigned slot = qn - 32 + lane;
            float ex[3] = {0.0f, 0.0f, 0.0f};
            int ep, es;
            const unsigned qa = qb + slot * 4u;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(ex[0]) : "r"(qa) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(ex[1]) : "r"(qa + kQueue * 4u) : "memory");
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(ep) : "r"(qa + kQueue * 8u) : "memory");
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(es) : "r"(qa + kQueue * 12u) : "memory");
            if (D == 3)
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(ex[2]) : "r"(qa + kQueue * 16u) : "memory");
            retire<D, OUTER, NH, BINK, SMEM, SCALED>(P, ex, ep, es, acc);
            qn -= 32;
            __syncwarp();
          }
        }
        bool took;
        if (SMEM == 2) {
          took = false;
          if (!wp.exhausted) {
            const unsigned n_need = __popc(need);
            unsigned base = 0u;
            if (eq == 1u) base = atomicAdd(&s_next, n_need);
            base = __shfl_sync(kFull, base, 0);
            if (base + n_need >= bcnt) wp.exhausted = 1;
            const unsigned k = base + __popc(need & lt);
            if ((need & eq) && k < bcnt) {
              pole[t] = (int)bpole;
              rep_off[t] = (int)(br0 + k);
              took = true;
            }
          }
        } else {
          took = pool_take_fast(wp, need, W, pole[t], rep_off[t], eq, lt);
        }
        if (took) {
          EM_DEV_ASSERT(pole[t] >= 0 && pole[t] < W.n_poles && rep_off[t] >= 0 && rep_off[t] < W.n_rep);
          if (SMEM != 2 && pole[t] != cpole) {
            const float4 p = __ldg(&P.poles[pole[t]]);
            px = p.x;
            py = p.y;
            pz = p.z;
            ccpid = W.pole_ids ? (unsigned)W.pole_ids[pole[t]] : (unsigned)pole[t];
            cpole = pole[t];
          }
          comp(X0, t) = px;
          comp(X1, t) = py;
          if (D == 3) comp(X2, t) = pz;
          cpid[t] = ccpid;
          const unsigned long long rep = (unsigned long long)W.rep_start + (unsigned)rep_off[t];
          rep_lo[t] = (unsigned)rep;
          rep_hi[t] = (unsigned)(rep >> 32);
          steps[t] = 0;
          walking[t] = 1;
        } else if (!walking[t]) {
          comp(X0, t) = comp(X1, t) = kFar;  // park (walk_f32_kernel: EM_POST_STOP)
          if (D == 3) comp(X2, t) = kFar;
        }
        live[t] = __ballot_sync(kFull, walking[t]);
      }
      if (wp.exhausted && (live[0] | live[1]) == 0u) break;
    }
    // ---- a batch of K steps: one Philox block per slot ----
    unsigned wv[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint4 w = philox4x32_10(P.rk, (unsigned)steps[t] / (unsigned)K, rep_lo[t], cpid[t], rep_hi[t]);
      wv[t][0] = w.x;
      wv[t][1] = w.y;
      wv[t][2] = w.z;
      wv[t][3] = w.w;
    }
    float2 x0 = X0, x1 = X1, x2 = X2;
    const int smax = steps[0] > steps[1] ? steps[0] : steps[1];
    if (__all_sync(kFull, smax + K <= P.max_steps)) {
      Mask2 go = {false, false};
#pragma unroll
      for (int k = 0; k < K; ++k) {
        float2 n0, n1, n2;
        go = step2<CH>(P, x0, x1, x2, make_uint2(wv[0][k], wv[1][k]), n0, n1, n2);
        x0 = vsel(go, n0, x0);
        x1 = vsel(go, n1, x1);
        if (D == 3) x2 = vsel(go, n2, x2);
        steps[0] += go.x;
        steps[1] += go.y;
      }
      // post-batch stop test of the landing point (walk_f32_kernel: EM_POST_STOP)
      const Mask2 g2 = walking_at<CH>(P, x0, x1, x2);
      walking[0] = go.x & g2.x;
      walking[1] = go.y & g2.y;
    } else {
      int failed[2] = {0, 0};
#pragma unroll
      for (int k = 0; k < K; ++k) {
        float2 n0, n1, n2;
        const Mask2 gk = step2<CH>(P, x0, x1, x2, make_uint2(wv[0][k], wv[1][k]), n0, n1, n2);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int stop = walking[t] & !(t ? gk.y : gk.x);
          const int over = walking[t] & (stop ^ 1) & (steps[t] >= P.max_steps);
          failed[t] |= over;
          walking[t] &= (stop ^ 1) & (over ^ 1);
          steps[t] += walking[t];
        }
        x0 = make_float2(walking[0] ? n0.x : x0.x, walking[1] ? n0.y : x0.y);
        x1 = make_float2(walking[0] ? n1.x : x1.x, walking[1] ? n1.y : x1.y);
        if (D == 3) x2 = make_float2(walking[0] ? n2.x : x2.x, walking[1] ? n2.y : x2.y);
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const unsigned fm = __ballot_sync(kFull, failed[t]);
        if (fm) {
          if (failed[t]) {
            atomicMax(W.err_key, ~(unsigned long long)((long long)pole[t] * W.n_rep + rep_off[t]));
            if (t == 0) {
              x0.x = x1.x = x2.x = kFar;
            } else {
              x0.y = x1.y = x2.y = kFar;
            }
          }
          live[t] &= ~fm;
        }
      }
    }
    X0 = x0;
    X1 = x1;
    X2 = x2;
  }
  __syncwarp();
  if (lane < qn) {  // drain the queue
    const ExitQueue2<D>& q = q_all[threadIdx.x >> 5];
    const float ex[3] = {q.x[lane], q.y[lane], D == 3 ? q.z[lane] : 0.0f};
    retire<D, OUTER, NH, BINK, SMEM, SCALED, false>(P, ex, q.p[lane], q.s[lane], acc);
  }
  if (SMEM == 2) {
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

}  // namespace f32

using F32Kernel = void (*)(F32Params);

// ch: 0 / 1 = ball without / with one concentric hole, 2 = box
static F32Kernel pick_f32x2(int ch, int bink, int smem) {
  using namespace f32;
#define EM_X2_SCHED(CH_, BK_)                                                     \
  (smem == 2 ? walk_f32x2_kernel<CH_, BK_, 2>                                      \
             : (smem ? walk_f32x2_kernel<CH_, BK_, 1> : walk_f32x2_kernel<CH_, BK_, 0>))
#define EM_X2_ANY(CH_)                                                            \
  (smem == 2 ? (F32Kernel) nullptr                                                 \
             : (smem ? walk_f32x2_kernel<CH_, BIN_ANY, 1> : walk_f32x2_kernel<CH_, BIN_ANY, 0>))
  if (ch == 3) {
    if (bink == BIN_GRID) return EM_X2_SCHED(3, BIN_GRID);
    return EM_X2_ANY(3);
  }
  if (ch == 2) {
    if (bink == BIN_SQUARE) return EM_X2_SCHED(2, BIN_SQUARE);
    if (bink == BIN_GRID) return EM_X2_SCHED(2, BIN_GRID);
    return EM_X2_ANY(2);
  }
  if (bink == BIN_CIRCLE) return ch == 0 ? EM_X2_SCHED(0, BIN_CIRCLE) : EM_X2_SCHED(1, BIN_CIRCLE);
  return ch == 0 ? EM_X2_ANY(0) : EM_X2_ANY(1);
#undef EM_X2_SCHED
#undef EM_X2_ANY
}

static int x2_family(int d, int outer, int nh_mode, int chain, bool ident) {
  if (!EM_ROLL2_GENERIC || chain != EM_CHAIN_TANGENT || ident) return -1;
  if (d == 3) return (EM_X2_3D && outer == OUTER_BALL && nh_mode == 0) ? 3 : -1;
  if (outer == OUTER_BALL && nh_mode <= 1) return nh_mode;
  if (outer == OUTER_BOX && nh_mode == 0) return 2;
  return -1;
}

// The packed kernel exists for this plan's family (counts mode only).
bool f32x2_available(int d, int outer, int nh_mode, int chain, bool ident) {
  return x2_family(d, outer, nh_mode, chain, ident) >= 0;
}

cudaError_t f32x2_blocks_per_sm(int d, int outer, int nh_mode, int bink, int* nb) {
  F32Kernel k = pick_f32x2(d == 3 ? 3 : (outer == OUTER_BOX ? 2 : nh_mode), bink, 0);
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

cudaError_t launch_f32x2(const F32Params& P, int d, int outer, int nh_mode, int bink, int grid,
                         int block, cudaStream_t s) {
  if (block != 32 * f32::kWarps) return cudaErrorInvalidConfiguration;
  const int sched = P.w.smem_stats;
  F32Kernel k = pick_f32x2(d == 3 ? 3 : (outer == OUTER_BOX ? 2 : nh_mode), bink, sched);
  if (!k) return cudaErrorInvalidValue;
  size_t smem = 0;
  if (sched == 1) smem = (size_t)f32::kWarps * 3 * P.w.n_poles * 8;
  if (sched == 2) {
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

}  // namespace em
