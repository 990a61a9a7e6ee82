// walk_ref64.cu -- bit-exact FP64 mirror of the reference walk kernel.
//
// Every expression restates S/_kernel.pyx (S/ = /root/reference/pkg/src/
// exitmeasure/) with the same operand order; this translation unit is built
// with -fmad=false so nvcc never contracts a*b+c into an FMA (the reference is
// compiled by gcc -O2 without FMA), and double sqrt / division are IEEE
// correctly rounded on the GPU.  The only non-IEEE-exact call, atan2, feeds
// nothing but the centre of the +-2 candidate window of a uniform circle block
// (S/_fallback.py:7-9), where an ulp of difference cannot change the winner.
// Result: for identical packed inputs, counts / exits / steps equal the
// reference kernel's bit for bit (tests/test_gpu_parity.py).
//
// Scheduling is the persistent refill of em_pool.cuh; accumulation is int64
// atomics, so the result is independent of the schedule.
#include <cuda_runtime.h>

#include "em_params.cuh"
#include "em_pool.cuh"
#include "em_rng.cuh"

namespace em {
namespace r64 {

__constant__ double kM2PI = 6.283185307179586476925286766559;
constexpr double kInv53 = 1.0 / 9007199254740992.0;
constexpr long long kBigIndex = 1LL << 62;

// One Marsaglia trial of S/_kernel.pyx:57-81 (the reference loops until a
// trial is accepted; the kernel below runs one trial per iteration so a
// rejecting lane does not hold its warp -- same draws, same directions).
// Words 0 and 1 of Philox4x64-10 at key (seed, 0), counter (draw, 0, rep,
// pole) -- exactly philox4x64_10 (em_rng.cuh) on the reference's stream
// layout (S/_kernel.pyx:37-63) -- with the seed's round keys seed + r W0 read
// from the params (constant-bank XOR operands instead of a 64-bit key add per
// round) and round 0's M1 * rep, constant over a walk, passed in.
__device__ __forceinline__ void philox_w01(const unsigned long long* rk0, unsigned long long draw,
                                           unsigned long long h1r, unsigned long long l1r,
                                           unsigned long long pole, unsigned long long& w0,
                                           unsigned long long& w1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const unsigned long long W1 = 0xBB67AE8584CAA73BULL;
  // round 0: c = (draw, 0, rep, pole), k = (seed, 0)
  unsigned long long c0 = h1r ^ rk0[0];
  unsigned long long c1 = l1r;
  unsigned long long c2 = __umul64hi(M0, draw) ^ pole;
  unsigned long long c3 = M0 * draw;
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    const unsigned long long hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const unsigned long long hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const unsigned long long n0 = hi1 ^ c1 ^ rk0[r];
    const unsigned long long n2 = hi0 ^ c3 ^ ((unsigned long long)r * W1);
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  w0 = c0;
  w1 = c1;
}

__device__ __forceinline__ bool direction_trial(int d, const unsigned long long* rk0,
                                                unsigned long long& draw,
                                                unsigned long long h1r, unsigned long long l1r,
                                                unsigned long long pole, double* u) {
  unsigned long long w0, w1;
  philox_w01(rk0, draw, h1r, l1r, pole, w0, w1);
  draw += 1ULL;
  double u0 = (double)(w0 >> 11) * kInv53;
  double u1 = (double)(w1 >> 11) * kInv53;
  double v1 = 2.0 * u0 - 1.0;
  double v2 = 2.0 * u1 - 1.0;
  double s = v1 * v1 + v2 * v2;
  if (d == 2) {
    if (s <= 1.0 && s > 0.0) {
      double rs = sqrt(s);
      u[0] = v1 / rs;
      u[1] = v2 / rs;
      return true;
    }
  } else {
    if (s < 1.0) {
      double f = 2.0 * sqrt(1.0 - s);
      u[0] = v1 * f;
      u[1] = v2 * f;
      u[2] = 1.0 - 2.0 * s;
      return true;
    }
  }
  return false;
}

// S/_kernel.pyx:89-116
__device__ double outer_signed(const Ref64Params& P, const double* x) {
  const double* gf = P.gf;
  const int d = P.d;
  if (P.outer_kind == 0) {
    double dx0 = x[0] - gf[0], dx1 = x[1] - gf[1];
    double t = dx0 * dx0 + dx1 * dx1;
    if (d == 3) {
      double dx2 = x[2] - gf[2];
      t = t + dx2 * dx2;
    }
    return gf[d] - sqrt(t);
  }
  double h = gf[d];
  double q0 = fabs(x[0] - gf[0]) - h;
  double q1 = fabs(x[1] - gf[1]) - h;
  double m = q0;
  if (q1 > m) m = q1;
  double t = (q0 > 0.0 ? q0 : 0.0) * (q0 > 0.0 ? q0 : 0.0) +
             (q1 > 0.0 ? q1 : 0.0) * (q1 > 0.0 ? q1 : 0.0);
  if (d == 3) {
    double q2 = fabs(x[2] - gf[2]) - h;
    if (q2 > m) m = q2;
    t = t + (q2 > 0.0 ? q2 : 0.0) * (q2 > 0.0 ? q2 : 0.0);
  }
  if (m <= 0.0) return -m;
  return -sqrt(t);
}

// S/_kernel.pyx:119-130
__device__ __forceinline__ double hole_dist(const Ref64Params& P, const double* x, int hole) {
  const int d = P.d;
  const int off = d + 1 + hole * (d + 1);
  double dx0 = x[0] - P.gf[off], dx1 = x[1] - P.gf[off + 1];
  double t = dx0 * dx0 + dx1 * dx1;
  if (d == 3) {
    double dx2 = x[2] - P.gf[off + 2];
    t = t + dx2 * dx2;
  }
  return sqrt(t) - P.gf[off + d];
}

// L-box notch extension (same expression as oracle/em_oracle.c)
__device__ __forceinline__ double notch_dist(const Ref64Params& P, const double* x) {
  const int off = (P.d + 1) * (1 + P.n_holes);
  double qx = P.gf[off] - x[0];
  double qy = P.gf[off + 1] - x[1];
  if (qx <= 0.0 && qy <= 0.0) return qx > qy ? qx : qy;
  double ax = qx > 0.0 ? qx : 0.0;
  double ay = qy > 0.0 ? qy : 0.0;
  return sqrt(ax * ax + ay * ay);
}

// S/_kernel.pyx:133-142
__device__ double signed_dist(const Ref64Params& P, const double* x) {
  double sd = outer_signed(P, x);
  for (int h = 0; h < P.n_holes; ++h) {
    double hd = hole_dist(P, x, h);
    if (hd < sd) sd = hd;
  }
  if (P.n_notch) {
    double nd = notch_dist(P, x);
    if (nd < sd) sd = nd;
  }
  return sd;
}

// S/_kernel.pyx:145-156
__device__ int owner_component(const Ref64Params& P, const double* x) {
  double best = fabs(outer_signed(P, x));
  int comp = 0;
  for (int h = 0; h < P.n_holes; ++h) {
    double dd = fabs(hole_dist(P, x, h));
    if (dd < best) {
      best = dd;
      comp = h + 1;
    }
  }
  if (P.n_notch) {
    double dd = fabs(notch_dist(P, x));
    if (dd < best) comp = P.n_holes + 1;
  }
  return comp;
}

// S/_kernel.pyx:204-216
__device__ __forceinline__ void lex_update(const double* x, int d, const double* anchors,
                                           long long g, double& best_d2, long long& best_gi) {
  const double* a = anchors + g * d;
  double dx0 = x[0] - __ldg(a), dx1 = x[1] - __ldg(a + 1);
  double t = dx0 * dx0 + dx1 * dx1;
  if (d == 3) {
    double dx2 = x[2] - __ldg(a + 2);
    t = t + dx2 * dx2;
  }
  if (t < best_d2 || (t == best_d2 && g < best_gi)) {
    best_d2 = t;
    best_gi = g;
  }
}

// S/_kernel.pyx:219-231
__device__ __forceinline__ double square_signed(double cx, double cy, double h, const double* x) {
  double q0 = fabs(x[0] - cx) - h;
  double q1 = fabs(x[1] - cy) - h;
  double m = q0;
  if (q1 > m) m = q1;
  if (m <= 0.0) return -m;
  double t = (q0 > 0.0 ? q0 : 0.0) * (q0 > 0.0 ? q0 : 0.0) +
             (q1 > 0.0 ? q1 : 0.0) * (q1 > 0.0 ? q1 : 0.0);
  return -sqrt(t);
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  if (v < lo) return lo;
  if (v > hi) return hi;
  return v;
}

__device__ __forceinline__ long long wrap(long long k, long long count) {
  k = k % count;
  if (k < 0) k += count;
  return k;
}

// wrap() of k + off for k already in [0, count) and |off| <= 2: one
// conditional add/subtract (same value; the 64-bit modulo is ~60 instructions)
__device__ __forceinline__ long long wrap_near(long long k, long long count) {
  if (count < 3) return wrap(k, count);
  if (k < 0) return k + count;
  if (k >= count) return k - count;
  return k;
}

// S/_kernel.pyx:242-320.  Extension: a block phase p (anchors at spacing*(k+p))
// shifts the centre of the +-2 window by -p; the window still holds the
// minimiser and its ties, so the lexicographic winner is unchanged and equals
// the brute-force rule (S/weights.py:74-87).
__device__ long long assign_anchor(const double* x, int d, const Side64& s) {
  double best_d2 = 1e308;
  long long best_gi = kBigIndex;
  for (int b = 0; b < s.n_blk; ++b) {
    const int kind = s.kind[b];
    const long long start = s.start[b], count = s.count[b];
    const double cx = s.cx[b], cy = s.cy[b], radius = s.radius[b], phase = s.phase[b];
    if (kind == BLK_CIRCLE) {
      double px = x[0] - cx, py = x[1] - cy;
      double ang = atan2(py, px);
      double t = ang * ((double)count / kM2PI);
      if (phase != 0.0) t = t - phase;
      long long k = wrap((long long)floor(t + 0.5), count);
      for (int off = -2; off < 3; ++off)
        lex_update(x, d, s.anchors, start + wrap_near(k + off, count), best_d2, best_gi);
    } else if (kind == BLK_SQUARE) {
      double spacing = 8.0 * radius / (double)count;
      if (fabs(square_signed(cx, cy, radius, x)) <= 0.125 * spacing) {
        double px = x[0] - cx, py = x[1] - cy;
        double dr = fabs(px - radius), dt = fabs(py - radius);
        double dl = fabs(px + radius), db = fabs(py + radius);
        int edge = 0;
        double m = dr, sarc;
        if (dt < m) { m = dt; edge = 1; }
        if (dl < m) { m = dl; edge = 2; }
        if (db < m) { m = db; edge = 3; }
        double cpx = clampd(px, -radius, radius), cpy = clampd(py, -radius, radius);
        if (edge == 0) sarc = cpy + radius;
        else if (edge == 1) sarc = 2.0 * radius + (radius - cpx);
        else if (edge == 2) sarc = 4.0 * radius + (radius - cpy);
        else sarc = 6.0 * radius + (cpx + radius);
        double t = sarc * ((double)count / (8.0 * radius));
        if (phase != 0.0) t = t - phase;
        long long k = wrap((long long)floor(t + 0.5), count);
        for (int off = -2; off < 3; ++off)
          lex_update(x, d, s.anchors, start + wrap_near(k + off, count), best_d2, best_gi);
      } else {
        for (long long idx = 0; idx < count; ++idx)
          lex_update(x, d, s.anchors, start + idx, best_d2, best_gi);
      }
    } else {
      for (long long idx = 0; idx < count; ++idx)
        lex_update(x, d, s.anchors, start + idx, best_d2, best_gi);
    }
  }
  return best_gi;
}

// mode 0: accumulate counts + step statistics (accumulate_chunk / run_accumulate)
// mode 1: write exit points, steps, components (walk_exits_chunk / run_exits)
constexpr int kWarps64 = 8;  // 256-thread blocks

struct ExitQueue64 {
  double x[64][3];
  long long steps[64];
  int pole[64];
};

// Bin one exit exactly as S/_kernel.pyx:445-464 (owner -> side -> anchor) and
// count it; the step statistics go to this lane's per-pole accumulator.
__device__ __forceinline__ void retire64(const Ref64Params& P, const double* xq, int pole,
                                         long long steps, StepAcc& acc) {
  const WorkOut& W = P.w;
  double x[3] = {xq[0], xq[1], xq[2]};
  const int comp = owner_component(P, x);
  const int side = P.comp_side[comp];
  const long long winner = assign_anchor(x, P.d, P.side[side]);
  const long long col = side ? W.col_off1 + winner : winner;
  EM_DEV_ASSERT(winner >= 0 && winner < P.side[side].n_anchors);
  EM_DEV_ASSERT(col >= 0 && col < W.row_len && pole >= 0 && pole < W.n_poles);
  atomicAdd(&W.counts[(long long)pole * W.row_len + col], 1ULL);
  acc_add(acc, W, pole, (unsigned long long)steps);
}

template <int MODE>
__global__ void __launch_bounds__(256, 4) walk_ref64_kernel(const Ref64Params P) {
  const WorkOut& W = P.w;
  const int d = P.d;
  double x[3] = {0.0, 0.0, 0.0};
  double u[3];
  unsigned long long draw = 0, rep = 0, pid = 0;
  unsigned long long h1r = 0, l1r = 0;  // M1 * rep (Philox round 0, fixed per walk)
  long long steps = 0, rep_off = 0;
  int pole = 0;
  bool active = false;
  // 0: evaluate the distance of a new step (stop / budget checks), 1: drawing
  // its direction -- a lane whose Marsaglia trial was rejected stays at 1
  int phase = 0;
  double sd = 0.0;
  // MODE 0: finished walks are queued per warp and binned 32 at a time with
  // every lane active (binning one lane at a time would serialise the warp)
  __shared__ ExitQueue64 q_all[kWarps64];
  ExitQueue64& q = q_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;
  WarpPool wp;
  pool_init(wp);
  StepAcc acc;
  acc_init(acc);
  if (MODE == 0) stats_smem_init(W);
  for (;;) {
    const unsigned need = __ballot_sync(kFull, !active);
    if (need) {
      if (pool_take(wp, need, W, pole, rep_off)) {
        rep = (unsigned long long)(W.rep_start + rep_off);
        h1r = __umul64hi(0xCA5A826395121157ULL, rep);
        l1r = 0xCA5A826395121157ULL * rep;
        pid = W.pole_ids ? (unsigned long long)W.pole_ids[pole] : (unsigned long long)pole;
        for (int j = 0; j < d; ++j) x[j] = P.poles[pole * d + j];
        draw = 0;
        steps = 0;
        phase = 0;
        active = true;
      }
      if (wp.exhausted && __ballot_sync(kFull, active) == 0) break;
    }
    // S/_kernel.pyx:176-197, one direction trial per iteration
    bool stop = false;
    if (active && phase == 0) {
      sd = signed_dist(P, x);
      if (sd <= P.eps) {
        stop = true;
      } else if (steps >= P.max_steps) {
        active = false;
        atomicMax(W.err_key, ~(unsigned long long)((long long)pole * W.n_rep + rep_off));
        if (MODE == 1) {
          const long long o = (long long)pole * W.n_rep + rep_off;
          for (int j = 0; j < d; ++j) W.x_out[o * d + j] = x[j];
          W.steps_out[o] = steps;
          W.comp_out[o] = 0;
        }
      } else {
        phase = 1;
      }
    }
    if (MODE == 0) {
      const unsigned sm = __ballot_sync(kFull, stop);
      if (sm) {
        if (stop) {
          const int slot = qn + __popc(sm & lt);
          for (int j = 0; j < 3; ++j) q.x[slot][j] = j < d ? x[j] : 0.0;
          q.pole[slot] = pole;
          q.steps[slot] = steps;
        }
        qn += __popc(sm);
        if (qn >= 32) {
          __syncwarp();
          const int slot = qn - 32 + lane;
          retire64(P, q.x[slot], q.pole[slot], q.steps[slot], acc);
          qn -= 32;
          __syncwarp();
        }
      }
    } else if (stop) {
      const long long o = (long long)pole * W.n_rep + rep_off;
      EM_DEV_ASSERT(o >= 0 && o < W.total);
      for (int j = 0; j < d; ++j) W.x_out[o * d + j] = x[j];
      W.steps_out[o] = steps;
      W.comp_out[o] = owner_component(P, x);
    }
    if (stop) active = false;
    if (!active || !direction_trial(d, P.rk0, draw, h1r, l1r, pid, u)) continue;
    phase = 0;
    const double* k = P.ks;
    if (d == 2) {
      double y0 = k[0] * u[0] + k[1] * u[1];
      double y1 = k[2] * u[0] + k[3] * u[1];
      x[0] = x[0] + sd * y0;
      x[1] = x[1] + sd * y1;
    } else {
      double y0 = k[0] * u[0] + k[1] * u[1] + k[2] * u[2];
      double y1 = k[3] * u[0] + k[4] * u[1] + k[5] * u[2];
      double y2 = k[6] * u[0] + k[7] * u[1] + k[8] * u[2];
      x[0] = x[0] + sd * y0;
      x[1] = x[1] + sd * y1;
      x[2] = x[2] + sd * y2;
    }
    steps = steps + 1;
  }
  if (MODE == 0) {
    __syncwarp();
    if (lane < qn) retire64(P, q.x[lane], q.pole[lane], q.steps[lane], acc);
    acc_flush(acc, W);
    stats_smem_flush(W);
  }
}

}  // namespace r64

// ---------------------------------------------------------------------------
// IDW weight families (S/_kernel.pyx:323-369), bit-exact.
//
// After the exits kernel (MODE 1) has written every walk's exit point and
// component, idw_prep computes per walk what the reference's scalar loop
// decides first: the anchor it sits on (r < 1e-14), the Voronoi fallback
// winner (no support covers it), or the normaliser `total` -- summed in anchor
// order exactly as the reference does.  idw_scatter then gives each
// (pole, anchor) one thread that walks the pole's walks in replicate order
// and adds w/total (or 1.0) sequentially, restarting a partial sum at every
// CHUNK boundary and folding it into the row in chunk order -- the
// reference driver's per-task zeroed buffers merged in job order
// (S/backend.py:159-198).  With `init` (the chunk API) the sum continues
// in place from the caller's values (S/_kernel.pyx:451-461 writes `out +=`).
// Voronoi sides in a mixed family pair add 1.0 at the winner.

struct IdwSide {
  const double* anchors;
  const double* radii;
  int n, power, wkind;
};

enum : int { IDW_NORMAL = 0, IDW_AT = 1, IDW_WINNER = 2 };

__global__ void idw_prep_kernel(const Ref64Params P, const double* x, const long long* comp,
                                long long n_walks, IdwSide s0, IdwSide s1, int* kind,
                                long long* idx, double* total, int* side_out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n_walks) return;
  const int d = P.d;
  double xw[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < d; ++k) xw[k] = x[j * d + k];
  const int side = P.comp_side[comp[j]];
  side_out[j] = side;
  const IdwSide& S = side ? s1 : s0;
  if (S.wkind == 0) {
    kind[j] = IDW_WINNER;
    idx[j] = r64::assign_anchor(xw, d, P.side[side]);
    total[j] = 0.0;
    return;
  }
  double tot = 0.0;
  for (int i = 0; i < S.n; ++i) {
    const double* a = S.anchors + (long long)i * d;
    double dx0 = xw[0] - a[0], dx1 = xw[1] - a[1];
    double d2 = dx0 * dx0 + dx1 * dx1;
    if (d == 3) {
      double dx2 = xw[2] - a[2];
      d2 = d2 + dx2 * dx2;
    }
    const double r = sqrt(d2);
    if (r < 1e-14) {
      kind[j] = IDW_AT;
      idx[j] = i;
      return;
    }
    double base = S.radii[i] - r;
    if (base > 0.0) {
      base = base / (S.radii[i] * r);
      double w = base;
      for (int q = 0; q < S.power - 1; ++q) w = w * base;
      tot = tot + w;
    }
  }
  if (tot == 0.0) {
    kind[j] = IDW_WINNER;
    idx[j] = r64::assign_anchor(xw, d, P.side[side]);
    total[j] = -1.0;  // marks a fallback (counted in idw_fallbacks)
    return;
  }
  kind[j] = IDW_NORMAL;
  total[j] = tot;
}

__global__ void idw_scatter_kernel(const Ref64Params P, const double* x, long long n_poles,
                                   long long n_rep, long long chunk, IdwSide s0, IdwSide s1,
                                   const int* kind, const long long* idx, const double* total,
                                   const int* side_of, double* out0, double* out1,
                                   const double* init0, const double* init1) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long per_pole = (long long)s0.n + s1.n;
  if (t >= n_poles * per_pole) return;
  const long long pole = t / per_pole;
  int i = (int)(t % per_pole);
  int side = 0;
  if (i >= s0.n) {
    side = 1;
    i -= s0.n;
  }
  const IdwSide& S = side ? s1 : s0;
  double* out = side ? out1 : out0;
  const double* init = side ? init1 : init0;
  const int d = P.d;
  const double* a = S.anchors + (long long)i * d;
  double row = init ? init[pole * S.n + i] : 0.0;
  for (long long c0 = 0; c0 < n_rep; c0 += chunk) {
    const long long c1 = c0 + chunk < n_rep ? c0 + chunk : n_rep;
    double part = 0.0;
    double* acc = init ? &row : &part;
    for (long long r = c0; r < c1; ++r) {
      const long long j = pole * n_rep + r;
      if (side_of[j] != side) continue;
      const int k = kind[j];
      if (k != IDW_NORMAL) {
        if (idx[j] == i) *acc += 1.0;
        continue;
      }
      const double* xw = x + j * d;
      double dx0 = xw[0] - a[0], dx1 = xw[1] - a[1];
      double d2 = dx0 * dx0 + dx1 * dx1;
      if (d == 3) {
        double dx2 = xw[2] - a[2];
        d2 = d2 + dx2 * dx2;
      }
      const double rr = sqrt(d2);
      double base = S.radii[i] - rr;
      if (base > 0.0) {
        base = base / (S.radii[i] * rr);
        double w = base;
        for (int q = 0; q < S.power - 1; ++q) w = w * base;
        *acc += w / total[j];
      }
    }
    if (!init) row += part;
  }
  out[pole * S.n + i] = row;
}

cudaError_t launch_idw(const Ref64Params& P, const double* x, const long long* comp,
                       long long n_poles, long long n_rep, long long chunk,
                       const double* a0, const double* r0, int n0, int pw0, int wk0,
                       const double* a1, const double* r1, int n1, int pw1, int wk1, int* kind,
                       long long* idx, double* total, int* side, double* out0, double* out1,
                       const double* init0, const double* init1, cudaStream_t s) {
  const IdwSide s0{a0, r0, n0, pw0, wk0}, s1{a1, r1, n1, pw1, wk1};
  const long long nw = n_poles * n_rep;
  if (nw > 0)
    idw_prep_kernel<<<(unsigned)((nw + 127) / 128), 128, 0, s>>>(P, x, comp, nw, s0, s1, kind,
                                                                  idx, total, side);
  const long long nt = n_poles * ((long long)n0 + n1);
  if (nt > 0)
    idw_scatter_kernel<<<(unsigned)((nt + 127) / 128), 128, 0, s>>>(
        P, x, n_poles, n_rep, chunk, s0, s1, kind, idx, total, side, out0, out1, init0, init1);
  return cudaGetLastError();
}

// Bin arbitrary points with the exact reference rule: owner component ->
// side -> lexicographic nearest anchor (S/_kernel.pyx:145-156,242-320).  Used
// for cell measures by boundary quadrature (S/weights.py:155-181).
__global__ void bin_points_ref64_kernel(const Ref64Params P, const double* pts, long long n,
                                        long long* comp_out, long long* side_out,
                                        long long* bin_out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int d = P.d;
  double x[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < d; ++k) x[k] = pts[j * d + k];
  const int comp = r64::owner_component(P, x);
  const int side = P.comp_side[comp];
  comp_out[j] = comp;
  side_out[j] = side;
  bin_out[j] = P.side[side].n_anchors > 0 ? r64::assign_anchor(x, d, P.side[side]) : -1;
}

cudaError_t launch_bin_points_ref64(const Ref64Params& P, const double* pts, long long n,
                                    long long* comp, long long* side, long long* bin,
                                    cudaStream_t s) {
  if (n > 0)
    bin_points_ref64_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(P, pts, n, comp, side, bin);
  return cudaGetLastError();
}

cudaError_t launch_ref64(const Ref64Params& P, int mode, int grid, int block, cudaStream_t s) {
  if (mode == 0) {
    const size_t smem = P.w.smem_stats ? (size_t)(block / 32) * 3 * P.w.n_poles * 8 : 0;
    r64::walk_ref64_kernel<0><<<grid, block, smem, s>>>(P);
  } else {
    r64::walk_ref64_kernel<1><<<grid, block, 0, s>>>(P);
  }
  return cudaGetLastError();
}

// Known-answer hook: Philox4x64-10 blocks for golden-vector tests.
__global__ void philox64_kat_kernel(const unsigned long long* in, unsigned long long* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long* c = in + 6 * i;
  u64x4 w = philox4x64_10(c[4], c[5], c[0], c[1], c[2], c[3]);  // (c0..c3, k0, k1)
  out[4 * i] = w.w0;
  out[4 * i + 1] = w.w1;
  out[4 * i + 2] = w.w2;
  out[4 * i + 3] = w.w3;
}

cudaError_t launch_philox64_kat(const unsigned long long* in, unsigned long long* out, int n,
                                cudaStream_t s) {
  philox64_kat_kernel<<<(n + 127) / 128, 128, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace em
