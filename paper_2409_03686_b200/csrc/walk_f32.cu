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
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <utility>
#include <vector>

#include "em_params.cuh"
#include "em_pool.cuh"
#include "em_rng.cuh"

// steps per batch on the tangent chains (one 32-bit word per step, one
// Philox block per 4 steps)
#ifndef EM_TANG_K
#define EM_TANG_K 4
#endif
// test the landing point of a batch's last move before the service pass
#ifndef EM_POST_STOP
#define EM_POST_STOP 1
#endif
#ifndef EM_ROLL2_DYN
#define EM_ROLL2_DYN 0
#endif
// 2D annulus rolling chain: one candidate disk per step (mid-radius choice)
#ifndef EM_ROLL2_ONE
#define EM_ROLL2_ONE 1
#endif
// 2D Moebius samplers: sin / cos of psi in [-pi/2, pi/2) by minimax
// polynomials on the FMA pipe (|error| < 6e-7 / 5e-8, below MUFU.SIN's) instead
// of two MUFU ops: the exit stays on the circle whatever their rounding
#ifndef EM_POLY_SINCOS
#define EM_POLY_SINCOS 0
#endif

namespace em {
namespace f32 {

constexpr float kPi = 3.14159265358979323846f;
constexpr float kInf = __builtin_huge_valf();

// MUFU.SQRT / MUFU.RCP without the denormal-range fix-ups the non-ftz
// approximations carry (an FSETP and two FMULs each); every operand on the
// walk path is a normal number (distances >= ~1e-7, squares >= ~1e-14), so
// flushing subnormals changes nothing.  Non-volatile asm: freely scheduled.
__device__ __forceinline__ float fsqrt(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fdiv(float a, float b) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
  return a * r;
}

// |A v|^2 = v^T K v (A = K^{1/2} symmetric) as a quadratic form: 9 ops in
// 3D (5 in 2D) instead of forming A v and its square norm (12 / 6).
// Kq = (K00, K11, K22, 2 K01, 2 K02, 2 K12).
template <int D>
__device__ __forceinline__ float quad_K(const F32Params& P, float v0, float v1, float v2) {
  const float* q = P.Kq;
  if (D == 2) {
    const float t0 = fmaf(q[3], v1, q[0] * v0);
    return fmaf(v1, q[1] * v1, v0 * t0);
  }
  const float t0 = fmaf(q[4], v2, fmaf(q[3], v1, q[0] * v0));
  const float t1 = fmaf(q[5], v2, q[1] * v1);
  return fmaf(v2, q[2] * v2, fmaf(v1, t1, v0 * t0));
}

// |v|^2 and |Av|^2 of an offset v.  In the rotated ball frame (DIAG, A =
// diag(Ad)) both come from the three squares: 3D 8 ops instead of 12.
template <int D, bool DIAG>
__device__ __forceinline__ void norm_quad(const F32Params& P, float v0, float v1, float v2,
                                          float& s2, float& aa) {
  if (DIAG) {
    const float p0 = v0 * v0, p1 = v1 * v1;
    if (D == 2) {
      s2 = p0 + p1;
      aa = fmaf(P.Kd[0], p0, P.Kd[1] * p1);
    } else {
      const float p2 = v2 * v2;
      s2 = p0 + p1 + p2;
      aa = fmaf(P.Kd[0], p0, fmaf(P.Kd[1], p1, P.Kd[2] * p2));
    }
    return;
  }
  s2 = v0 * v0 + v1 * v1;
  if (D == 3) s2 = fmaf(v2, v2, s2);
  aa = quad_K<D>(P, v0, v1, v2);
}

template <int NH>
__device__ __forceinline__ int n_holes(const F32Params& P) {
  return NH >= 0 ? NH : P.n_holes;
}

// Euclidean signed distance e and the unshrunk step scale r at x (shrunk
// already when FOLD, see dist below).
template <int D, int OUTER, int NH, int CHAIN, bool IDENT>
__device__ __forceinline__ void dist_raw(const F32Params& P, const float* x, float& e, float& r) {
  constexpr bool MAXC = (CHAIN == EM_CHAIN_MAX) && !IDENT;
  constexpr bool FOLD = MAXC && OUTER != OUTER_BALL && NH == 0;
  constexpr bool DIAG = OUTER == OUTER_BALL && !IDENT;  // rotated ball frame
  if (OUTER == OUTER_BALL) {
    // kernel frame: the outer ball is centred at the origin
    const float v0 = x[0], v1 = x[1];
    const float v2 = D == 3 ? x[2] : 0.0f;
    float s2, aa = 0.0f;  // |x|^2, |Ax|^2
    if (MAXC) {
      norm_quad<D, DIAG>(P, v0, v1, v2, s2, aa);
    } else {
      s2 = v0 * v0 + v1 * v1;
      if (D == 3) s2 = fmaf(v2, v2, s2);
    }
    if (MAXC && NH == 0) {
      // stop test on |x|^2 itself (no |x| needed): e > eps <=> |x|^2 <
      // (R - eps)^2, returned already as the FFMA.SAT stop margin (see dist)
      e = fmaf(s2, -P.s2_scale, P.s2_bias);
    } else {
      e = P.oR - fsqrt(s2);
    }
    if (MAXC) {
      // |x + rAu|^2 <= s^2 + 2 r |Av| + r^2 <= R^2  =>  r <= q / (a + sqrt(a^2 + q))
      const float q = P.oR2 - s2;  // R^2 - |x|^2
      r = fdiv(q, fsqrt(aa) + fsqrt(fmaxf(aa + q, 0.0f)));
    } else {
      r = e;
    }
  } else {
    // box / L-box outer: face planes; the maximal ellipsoid touches plane i at
    // (distance to plane) / |A e_i| = distance * g_i
    e = kInf;
    r = kInf;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      // kernel frame: the box is [-bhi_i, bhi_i] (centred), so the distance
      // to the nearer face is one FADD with a free |.| operand
      const float m = P.bhi[i] - fabsf(x[i]);
      e = fminf(e, m);
      if (FOLD) r = fminf(r, fmaf(m, P.gk[i], -P.shrink_abs));
      else if (MAXC) r = fminf(r, m * P.g[i]);
    }
    if (!MAXC) r = e;
    if (OUTER == OUTER_LBOX) {
      // distance to the notch prism; a point a rounding step inside it gets
      // 0, which stops the walk exactly as a negative distance would
      const float qx = P.notch[0] - x[0], qy = P.notch[1] - x[1];
      const float ax = fmaxf(qx, 0.0f), ay = fmaxf(qy, 0.0f);
      const float en = fsqrt(fmaf(ax, ax, ay * ay));
      e = fminf(e, en);
      if (FOLD)  // every term through the same monotone t -> t keep - abs
        r = fminf(r, fmaxf(fmaf(en, P.keep, -P.shrink_abs),
                           fmaxf(fmaf(qx, P.gk[0], -P.shrink_abs), fmaf(qy, P.gk[1], -P.shrink_abs))));
      else if (MAXC)
        r = fminf(r, fmaxf(en, fmaxf(qx * P.g[0], qy * P.g[1])));
      else
        r = e;
    }
  }
  // ball holes
  const int nh = n_holes<NH>(P);
  for (int h = 0; h < nh; ++h) {
    const float v0 = x[0] - P.hc[h][0], v1 = x[1] - P.hc[h][1];
    const float v2 = D == 3 ? x[2] - P.hc[h][2] : 0.0f;
    float s2, aa = 0.0f;  // |v|^2, |Av|^2
    if (MAXC) {
      norm_quad<D, DIAG>(P, v0, v1, v2, s2, aa);
    } else {
      s2 = v0 * v0 + v1 * v1;
      if (D == 3) s2 = fmaf(v2, v2, s2);
    }
    const float s = fsqrt(s2);
    const float rho = P.hr[h];
    const float eh = s - rho;
    e = fminf(e, eh);
    if (MAXC) {
      // min_u |v + rAu|^2 >= s^2 - 2 r |Av| + r^2 m^2 >= rho^2
      const float q = s2 - P.hr2[h];  // |v|^2 - rho^2
      const float rh = fdiv(q, fsqrt(aa) + fsqrt(fmaxf(fmaf(-P.m2, q, aa), 0.0f)));
      r = fminf(r, fmaxf(rh, eh));
    } else {
      r = e;
    }
  }
}

// Euclidean signed distance e and step scale r at x, r already shrunk by the
// FP32 safety margin: r = r_exact * keep - shrink_abs.  Box faces fold the
// margin into their gain (one FFMA per face instead of an FMUL per face plus
// a final FFMA); every other shape applies it once at the end.
// The first output is the lane's 0/1 walking mask t = sat(m): the stop
// margin m is <= 0 exactly when e <= eps and >= 1 otherwise (m = (e - eps)
// 2^k by one FFMA, or the ball's |x|^2 form), so the saturation folds into
// the instruction that computes m.
// Box / L-box on the max chain without holes keeps its axes sheared (see
// F32Params::shear): the stop test and the face bounds come from the sheared
// face distances s_i = sb_i - |xs_i| directly.
template <int D, int OUTER, int NH, int CHAIN, bool IDENT>
struct Shear {
  static constexpr bool value = OUTER != OUTER_BALL && NH == 0 && CHAIN == EM_CHAIN_MAX &&
                                !IDENT && (D == 3 || OUTER == OUTER_BOX);
};

template <int D, int OUTER, int NH, int CHAIN, bool IDENT>
__device__ __forceinline__ void dist(const F32Params& P, const float* x, float& t, float& r) {
  constexpr bool MAXC = (CHAIN == EM_CHAIN_MAX) && !IDENT;
  constexpr bool FOLD = MAXC && OUTER != OUTER_BALL && NH == 0;
  constexpr bool S2STOP = MAXC && OUTER == OUTER_BALL && NH == 0;
  constexpr bool DIAG = OUTER == OUTER_BALL && !IDENT;  // rotated ball frame
  if (OUTER == OUTER_BALL && NH == 1 && MAXC && P.concentric) {
    // annulus / spherical shell: one |v|^2 and one |Av|^2 serve both bounds,
    //   r = min(q_o / D_o, q_h / D_h),  q_o = R^2 - |v|^2,  q_h = |v|^2 - rho^2
    // picked by cross-multiplication, so a single reciprocal replaces two
    // divisions; both stop tests run on |v|^2 against (R - eps)^2 and
    // (rho + eps)^2, so |v| itself is never formed (XU-bound step: 6 MUFU)
    const float v0 = x[0], v1 = x[1];
    const float v2 = D == 3 ? x[2] : 0.0f;
    float s2, aa;  // |v|^2, |Av|^2
    norm_quad<D, DIAG>(P, v0, v1, v2, s2, aa);
    t = fminf(__saturatef(fmaf(s2, -P.s2_scale, P.s2_bias)),
              __saturatef(fmaf(s2, P.h2_scale, P.h2_bias)));
    const float a = fsqrt(aa);
    const float qo = P.oR2 - s2;
    const float Do = a + fsqrt(fmaxf(aa + qo, 0.0f));
    const float qh = s2 - P.hr2[0];
    const float Dh = a + fsqrt(fmaxf(fmaf(-P.m2, qh, aa), 0.0f));
    const bool outer = qo * Dh <= qh * Do;
    r = fmaf(fdiv(outer ? qo : qh, outer ? Do : Dh), P.keep, -P.shrink_abs);
    return;
  }
  if (Shear<D, OUTER, NH, CHAIN, IDENT>::value) {
    // s_i <= 0 exactly when face i is within eps; any positive s_i scales to
    // >= 1 (ss_scale), so sat(t) is the 0/1 walking mask
    const float s0 = P.sb[0] - fabsf(x[0]), s1 = P.sb[1] - fabsf(x[1]);
    const float s2 = D == 3 ? P.sb[2] - fabsf(x[2]) : kInf;
    r = fminf(fmaf(s0, P.sg[0], P.sc[0]), fmaf(s1, P.sg[1], P.sc[1]));
    if (D == 3) r = fminf(r, fmaf(s2, P.sg[2], P.sc[2]));
    if (OUTER == OUTER_LBOX) {
      // notch prism in world units (corner offsets from the frame axes)
      const float qx = fmaf(-P.ax[0], x[0], P.notch[0]), qy = fmaf(-P.ax[1], x[1], P.notch[1]);
      const float nx = fmaxf(qx, 0.0f), ny = fmaxf(qy, 0.0f);
      const float en = fsqrt(fmaf(nx, nx, ny * ny));
      t = fminf(__saturatef(fminf(fminf(s0, s1), s2) * P.ss_scale),
                __saturatef(fmaf(en, P.stop_scale, P.stop_bias)));
      r = fminf(r, fmaxf(fmaf(en, P.keep, -P.shrink_abs),
                         fmaxf(fmaf(qx, P.gk[0], -P.shrink_abs), fmaf(qy, P.gk[1], -P.shrink_abs))));
    } else {
      t = __saturatef(fminf(fminf(s0, s1), s2) * P.ss_scale);
    }
    return;
  }
  float e;
  dist_raw<D, OUTER, NH, CHAIN, IDENT>(P, x, e, r);
  t = __saturatef(S2STOP ? e : fmaf(e, P.stop_scale, P.stop_bias));
  if (!FOLD) r = fmaf(r, P.keep, -P.shrink_abs);
}

// Owner component: argmin of |component distance|, ties to the lowest id
// (S/_kernel.pyx:145-156).
template <int D, int OUTER, int NH>
__device__ __forceinline__ int owner(const F32Params& P, const float* x) {
  if (OUTER == OUTER_BALL && NH == 1 && P.concentric) {
    // concentric shell: |R - r| <= |r - rho| (ties to the outer component)
    // exactly when r >= (R + rho) / 2
    float s2 = x[0] * x[0] + x[1] * x[1];
    if (D == 3) s2 = fmaf(x[2], x[2], s2);
    return s2 >= P.mid2 ? 0 : 1;
  }
  float best;
  if (OUTER == OUTER_BALL) {
    const float v0 = x[0], v1 = x[1];
    const float v2 = D == 3 ? x[2] : 0.0f;
    best = fabsf(P.oR - sqrtf(v0 * v0 + v1 * v1 + v2 * v2));
  } else {
    float m = kInf;
#pragma unroll
    for (int i = 0; i < D; ++i) m = fminf(m, P.bhi[i] - fabsf(x[i]));
    best = fabsf(m);
  }
  int comp = 0;
  const int nh = n_holes<NH>(P);
  for (int h = 0; h < nh; ++h) {
    const float v0 = x[0] - P.hc[h][0], v1 = x[1] - P.hc[h][1];
    const float v2 = D == 3 ? x[2] - P.hc[h][2] : 0.0f;
    const float dd = fabsf(sqrtf(v0 * v0 + v1 * v1 + v2 * v2) - P.hr[h]);
    if (dd < best) {
      best = dd;
      comp = h + 1;
    }
  }
  if (OUTER == OUTER_LBOX) {
    const float qx = P.notch[0] - x[0], qy = P.notch[1] - x[1];
    float en;
    if (qx <= 0.0f && qy <= 0.0f) {
      en = fmaxf(qx, qy);
    } else {
      const float ax = fmaxf(qx, 0.0f), ay = fmaxf(qy, 0.0f);
      en = sqrtf(fmaf(ax, ax, ay * ay));
    }
    if (fabsf(en) < best) comp = nh + 1;
  }
  return comp;
}

// k in [-count, 2 count): wrap without an integer division
__device__ __forceinline__ int wrapi(int k, int count) {
  k = k < 0 ? k + count : k;
  return k >= count ? k - count : k;
}

template <int D>
__device__ __forceinline__ float d2_to(const float4 a, const float* x) {
  const float d0 = x[0] - a.x, d1 = x[1] - a.y;
  float t = fmaf(d0, d0, d1 * d1);
  if (D == 3) {
    const float d2 = x[2] - a.z;
    t = fmaf(d2, d2, t);
  }
  return t;
}

template <int D>
__device__ int brute(const Side32& S, const float* x, int start, int count) {
  float best = kInf;
  int bi = start;
  for (int i = start; i < start + count; ++i) {
    const float t = d2_to<D>(__ldg(&S.anchors[i]), x);
    if (t < best) {
      best = t;
      bi = i;
    }
  }
  return bi;
}

// Cell of one uniform circle block (count <= kBisMax) holding the offset
// (dx, dy) from its centre.  The nearest of equally spaced anchors on a
// circle is the one of nearest angle: a cheap angle (|error| < 8.2e-5 rad,
// far below half a cell) picks a cell k, then exact side tests against its
// two Voronoi boundary rays (cross products with bis[k], bis[k + 1]) move
// it by at most one -- atan2f's work at about half its instructions.
__device__ __forceinline__ int circle_cell(const float2* bis, int count, float scale, float phase,
                                           float dx, float dy) {
  const float ax = fabsf(dx), ay = fabsf(dy);
  const float q = fdiv(fminf(ax, ay), fmaxf(ax, ay));
  const float q2 = q * q;
  float a = q * fmaf(q2, fmaf(q2, fmaf(q2, -0.03899375721812248f, 0.14627520740032196f),
                              -0.3211793601512909f), 0.999214231967926f);
  a = ay > ax ? 1.5707963267948966f - a : a;
  a = dx < 0.0f ? kPi - a : a;
  a = copysignf(a, dy);
  const int k = wrapi((int)floorf(fmaf(a, scale, -phase) + 0.5f), count);
  const int k1 = k + 1 == count ? 0 : k + 1;
  const float2 bl = __ldg(&bis[k]), bh = __ldg(&bis[k1]);
  const float cl = fmaf(bl.x, dy, -bl.y * dx);  // < 0: clockwise of the cell's lower ray
  const float ch = fmaf(bh.x, dy, -bh.y * dx);  // > 0: counter-clockwise of its upper ray
  return cl < 0.0f ? (k == 0 ? count - 1 : k - 1) : (ch > 0.0f ? k1 : k);
}

// Nearest anchor (family-local index) of one side's family.
template <int D>
__device__ int nearest_anchor(const Side32& S, const float* x) {
  if (S.has_grid) {
    const Grid32& G = S.grid;
    const int ix = (int)floorf((x[0] - G.lo[0]) * G.inv_h);
    const int iy = (int)floorf((x[1] - G.lo[1]) * G.inv_h);
    const int iz = D == 3 ? (int)floorf((x[2] - G.lo[2]) * G.inv_h) : 0;
    if (ix >= 0 && iy >= 0 && iz >= 0 && ix < G.n[0] && iy < G.n[1] && iz < G.n[2]) {
      const unsigned w = __ldg(&G.cell[(iz * G.n[1] + iy) * G.n[0] + ix]);
      const unsigned cnt = w & 255u, off = w >> 8;
      if (cnt != 255u) {
        float best = kInf;
        int bi = 0;
        for (unsigned j = 0; j < cnt; ++j) {
          const int a = (int)__ldg(&G.cand[off + j]);
          const float t = d2_to<D>(__ldg(&S.anchors[a]), x);
          if (t < best || (t == best && a < bi)) {
            best = t;
            bi = a;
          }
        }
        return bi;
      }
    }
    return brute<D>(S, x, 0, S.n_anchors);
  }
  float best = kInf;
  int bi = 0;
  for (int b = 0; b < S.n_blk; ++b) {
    int idx;
    const int count = S.count[b];
    if (S.kind[b] == BLK_CIRCLE && S.n_blk == 1 && S.bis) {
      idx = S.start[b] + circle_cell(S.bis, count, S.scale[b], S.phase[b], x[0] - S.cx[b],
                                     x[1] - S.cy[b]);
    } else if (S.kind[b] == BLK_CIRCLE) {
      const float ang = atan2f(x[1] - S.cy[b], x[0] - S.cx[b]);
      const float t = fmaf(ang, S.scale[b], -S.phase[b]);
      idx = S.start[b] + wrapi((int)floorf(t + 0.5f), count);
    } else if (S.kind[b] == BLK_SQUARE) {
      const float h = S.radius[b];
      const float px = x[0] - S.cx[b], py = x[1] - S.cy[b];
      const float dr = fabsf(px - h), dt = fabsf(py - h), dl = fabsf(px + h), db = fabsf(py + h);
      const float cpx = fminf(fmaxf(px, -h), h), cpy = fminf(fmaxf(py, -h), h);
      float s = cpy + h, m = dr;
      if (dt < m) { m = dt; s = 2.0f * h + (h - cpx); }
      if (dl < m) { m = dl; s = 4.0f * h + (h - cpy); }
      if (db < m) { m = db; s = 6.0f * h + (cpx + h); }
      const float t = fmaf(s, S.scale[b], -S.phase[b]);
      idx = S.start[b] + wrapi((int)floorf(t + 0.5f), count);
    } else {
      idx = brute<D>(S, x, S.start[b], count);
    }
    if (S.n_blk == 1) return idx;
    const float t = d2_to<D>(__ldg(&S.anchors[idx]), x);
    if (t < best || (t == best && idx < bi)) {
      best = t;
      bi = idx;
    }
  }
  return bi;
}

// Binner kinds, fixed at compile time per plan (capi.cu picks the kind):
//   BIN_ANY    -- runtime walk over the side's blocks (nearest_anchor above)
//   BIN_CIRCLE -- every used side is ONE uniform circle block: index by angle
//   BIN_SQUARE -- every used side is ONE uniform square block: index by arc
//   BIN_GRID   -- every used side is ONE generic family with a candidate grid
// Side fields are selected branch-free from the two constant-bank copies, so
// nothing is indexed dynamically in parameter space.
enum BinKind { BIN_ANY = 0, BIN_CIRCLE = 1, BIN_SQUARE = 2, BIN_GRID = 3 };

template <class T>
__device__ __forceinline__ T pick(int side, T a, T b) {
  return side ? b : a;
}

template <int D, int BINK>
__device__ __forceinline__ int bin_exit(const F32Params& P, int side, const float* x) {
  const Side32& S0 = P.side[0];
  const Side32& S1 = P.side[1];
  if (BINK == BIN_CIRCLE) {
    const float dx = x[0] - pick(side, S0.cx[0], S1.cx[0]);
    const float dy = x[1] - pick(side, S0.cy[0], S1.cy[0]);
    const float2* bis = pick(side, S0.bis, S1.bis);
    const int count = pick(side, S0.count[0], S1.count[0]);
    if (bis)
      return circle_cell(bis, count, pick(side, S0.scale[0], S1.scale[0]),
                         pick(side, S0.phase[0], S1.phase[0]), dx, dy);
    const float ang = atan2f(dy, dx);
    const float t = fmaf(ang, pick(side, S0.scale[0], S1.scale[0]),
                         -pick(side, S0.phase[0], S1.phase[0]));
    return wrapi((int)floorf(t + 0.5f), count);
  } else if (BINK == BIN_SQUARE) {
    const float h = pick(side, S0.radius[0], S1.radius[0]);
    const float px = x[0] - pick(side, S0.cx[0], S1.cx[0]);
    const float py = x[1] - pick(side, S0.cy[0], S1.cy[0]);
    const float dr = fabsf(px - h), dt = fabsf(py - h), dl = fabsf(px + h), db = fabsf(py + h);
    const float cpx = fminf(fmaxf(px, -h), h), cpy = fminf(fmaxf(py, -h), h);
    float s = cpy + h, m = dr;
    if (dt < m) { m = dt; s = 2.0f * h + (h - cpx); }
    if (dl < m) { m = dl; s = 4.0f * h + (h - cpy); }
    if (db < m) { m = db; s = 6.0f * h + (cpx + h); }
    const float t = fmaf(s, pick(side, S0.scale[0], S1.scale[0]),
                         -pick(side, S0.phase[0], S1.phase[0]));
    return wrapi((int)floorf(t + 0.5f), pick(side, S0.count[0], S1.count[0]));
  } else if (BINK == BIN_GRID) {
    const float4* anchors = pick(side, S0.anchors, S1.anchors);
    const float inv_h = pick(side, S0.grid.inv_h, S1.grid.inv_h);
    const int ix = (int)floorf((x[0] - pick(side, S0.grid.lo[0], S1.grid.lo[0])) * inv_h);
    const int iy = (int)floorf((x[1] - pick(side, S0.grid.lo[1], S1.grid.lo[1])) * inv_h);
    const int iz = D == 3 ? (int)floorf((x[2] - pick(side, S0.grid.lo[2], S1.grid.lo[2])) * inv_h) : 0;
    const int nx = pick(side, S0.grid.n[0], S1.grid.n[0]);
    const int ny = pick(side, S0.grid.n[1], S1.grid.n[1]);
    const int nz = pick(side, S0.grid.n[2], S1.grid.n[2]);
    const int na = pick(side, S0.n_anchors, S1.n_anchors);
    unsigned off = 0, cnt = 255u;
    if (ix >= 0 && iy >= 0 && iz >= 0 && ix < nx && iy < ny && iz < nz) {
      const unsigned w = __ldg(&pick(side, S0.grid.cell, S1.grid.cell)[(iz * ny + iy) * nx + ix]);
      cnt = w & 255u;
      off = w >> 8;
    }
    float best = kInf;
    int bi = 0;
    if (cnt != 255u) {
      // the cell's candidates with their coordinates inline: one 16-byte
      // load per candidate
      const float4* cv = pick(side, S0.grid.candv, S1.grid.candv) + off;
      for (unsigned j = 0; j < cnt; ++j) {
        const float4 c = __ldg(&cv[j]);
        const int a = __float_as_int(c.w);
        const float t = d2_to<D>(c, x);
        if (t < best || (t == best && a < bi)) {
          best = t;
          bi = a;
        }
      }
      return bi;
    }
    for (int j = 0; j < na; ++j) {  // outside the band: brute force
      const float t = d2_to<D>(__ldg(&anchors[j]), x);
      if (t < best) {
        best = t;
        bi = j;
      }
    }
    return bi;
  } else {
    return nearest_anchor<D>(side ? S1 : S0, x);
  }
}

// Steps per service phase and Philox blocks per batch: 2D uses one 32-bit
// word per step (4 steps per block), 3D two words (2 steps per block).
#ifndef EM_BATCH_STEPS
#define EM_BATCH_STEPS 8
#endif
// Random bits per azimuth: 16 (two angles per 32-bit word) or 23.  A uniform
// grid of 2^16 equally spaced angles averages every Fourier mode |k| < 2^16
// exactly, so the mean-value property the step relies on holds to that order
// (DESIGN.md §3.1).
#ifndef EM_ANGLE_BITS
#define EM_ANGLE_BITS 16
#endif
// 3D z = cos(polar angle): 16 bits (two per word: a 3D batch needs two
// Philox blocks instead of three, +7-10% on cfg4/cfg5) or 23.  With 16-bit z
// and 16-bit azimuths a step draws uniformly from 2^32 directions that are
// the centres of 2^32 equal-area cells of the sphere (Archimedes: equal z
// bands have equal area), a midpoint rule whose error for the smooth
// (harmonic) integrands of the mean-value property is O(cell size^2) ~ 1e-9
// -- far below the Monte Carlo error of any run.
#ifndef EM_Z_BITS
#define EM_Z_BITS 16
#endif
template <int D>
struct Batch {
  static constexpr int kSteps = EM_BATCH_STEPS;
  static constexpr int kAngleWords = EM_ANGLE_BITS == 16 ? (kSteps + 1) / 2 : kSteps;
  static constexpr int kZWords = D == 3 ? (EM_Z_BITS == 16 ? (kSteps + 1) / 2 : kSteps) : 0;
  static constexpr int kWords = kZWords + kAngleWords;
  static constexpr int kBlocks = (kWords + 3) / 4;
};

// The angle of step k of a batch, as theta = fmaf(f, kAngScale, kAngBias)
// of the float f built from the batch's words.  16-bit angles: ONE byte
// permute (PRMT) drops a half-word into the low mantissa bytes of 1.0f, so
// f = 1 + k16 / 2^23, and the FFMA maps the 2^16 values onto equally spaced
// angles spanning exactly 2 pi (the offset is irrelevant on the circle).
// (one_bits = 0x3f800000 comes from the params so the compiler keeps it as
// the register/constant operand and the selector as the immediate: with a
// literal it materialises the selector in a register on every step)
template <int D>
__device__ __forceinline__ unsigned angle_bits(const unsigned* wv, int k, unsigned one_bits) {
  if (EM_ANGLE_BITS == 16) {
    const unsigned w = wv[Batch<D>::kZWords + (k >> 1)];
    return __byte_perm(w, one_bits, (k & 1) ? 0x7632u : 0x7610u);
  }
  return one_bits | (wv[Batch<D>::kZWords + k] >> 9);
}

// z of step k in (-1, 1), never +-1, equally spaced: 23 bits from the top of
// word k (-1 + (2m + 1)/2^23), or 16 bits from half a word by the same
// PRMT trick as the angles (f = 1 + m/2^23, m < 2^16: -1 + (2m + 1)/2^16);
// every operation is exact in FP32
template <int D>
__device__ __forceinline__ float z_of(const unsigned* wv, int k, unsigned one_bits) {
  if (EM_Z_BITS == 16) {
    const float f = __uint_as_float(__byte_perm(wv[k >> 1], one_bits, (k & 1) ? 0x7632u : 0x7610u));
    return fmaf(f, 256.0f, -257.0f) + 1.52587890625e-05f;  // + 2^-16
  }
  return sym11_23(wv[k]);
}

// One walk-on-ellipsoids step from x (r from dist()): direction from the RNG
// word(s), y = K^{1/2} u, x += rs y with rs = r shrunk by the FP32 safety
// margin, or rs = 0 for a lane that is not walking (branch-free: the warp
// issues the same instructions whether or not every lane is live).
// Uniform angle on the circle with ONE FFMA from f = 1 + m/2^b in [1,2)
// (the float built by angle_bits): theta = 2 pi f - 3 pi in [-pi, pi).  The
// angles are equally spaced around the circle, so the offset is irrelevant.
#if EM_ANGLE_BITS == 16
// f in [1, 1 + 2^-7): theta = (f - 1) * 2^7 * 2 pi - pi
constexpr float kAngScale = 6.283185307179586f * 128.0f;
constexpr float kAngBias = -(6.283185307179586f * 128.0f) - 3.14159265358979323846f;
#else
// f in [1, 2): theta = 2 pi f - 3 pi
constexpr float kAngScale = 6.283185307179586f;
constexpr float kAngBias = -9.42477796076938f;
#endif
__device__ __forceinline__ float angle_of(unsigned fbits) {
  return fmaf(__uint_as_float(fbits), kAngScale, kAngBias);
}

template <int D, int OUTER, bool IDENT, bool SHEAR>
__device__ __forceinline__ void step(const F32Params& P, float* x, float rs, float z,
                                     unsigned afbits) {
  constexpr bool DIAG = OUTER == OUTER_BALL && !IDENT;
  if (SHEAR) {
    // sheared axes (F32Params::shear)
    if (D == 2) {
      float sn, cs;
      __sincosf(angle_of(afbits), &sn, &cs);
      x[0] = fmaf(rs, cs, x[0]);
      x[1] = fmaf(rs, fmaf(P.shk[0], cs, sn), x[1]);
    } else {
      const float th = angle_of(afbits);
      const float rho = fsqrt(fmaxf(fmaf(-z, z, 1.0f), 0.0f));
      float sn, cs;
      __sincosf(th, &sn, &cs);
      const float rc = rho * cs, rsn = rho * sn;
      x[0] = fmaf(rs, z, x[0]);
      x[1] = fmaf(rs, fmaf(P.shk[0], z, rc), x[1]);
      x[2] = fmaf(rs, fmaf(P.shk[1], rc, fmaf(P.shk[2], z, rsn)), x[2]);
    }
    return;
  }
  float u0, u1, u2 = 0.0f;
  if (D == 3 && DIAG) {
    // rotated ball frame: y = diag(Ad) u, the axis gains folded into rho
    const float th = angle_of(afbits);
    const float rho = fsqrt(fmaxf(fmaf(-z, z, 1.0f), 0.0f));
    float sn, cs;
    __sincosf(th, &sn, &cs);
    x[0] = fmaf(rs, (P.Ad[0] * rho) * cs, x[0]);
    x[1] = fmaf(rs, (P.Ad[1] * rho) * sn, x[1]);
    x[2] = fmaf(rs, P.Ad[2] * z, x[2]);
    return;
  }
  if (D == 2) {
    __sincosf(angle_of(afbits), &u1, &u0);
  } else {
    const float th = angle_of(afbits);
    const float rho = fsqrt(fmaxf(fmaf(-z, z, 1.0f), 0.0f));
    float sn, cs;
    __sincosf(th, &sn, &cs);
    u0 = rho * cs;
    u1 = rho * sn;
    u2 = z;
  }
  float y0 = u0, y1 = u1, y2 = u2;
  if (DIAG) {
    y0 = P.Ad[0] * u0;
    y1 = P.Ad[1] * u1;
  } else if (!IDENT) {
    if (D == 2) {
      y0 = fmaf(P.A[0], u0, P.A[1] * u1);
      y1 = fmaf(P.A[2], u0, P.A[3] * u1);
    } else {
      y0 = fmaf(P.A[0], u0, fmaf(P.A[1], u1, P.A[2] * u2));
      y1 = fmaf(P.A[3], u0, fmaf(P.A[4], u1, P.A[5] * u2));
      y2 = fmaf(P.A[6], u0, fmaf(P.A[7], u1, P.A[8] * u2));
    }
  }
  x[0] = fmaf(rs, y0, x[0]);
  x[1] = fmaf(rs, y1, x[1]);
  if (D == 3) x[2] = fmaf(rs, y2, x[2]);
}

// Walk on tangent balls (EM_CHAIN_TANGENT, 2D box without holes), in the
// stored coordinates xt_i = x_i / R_i (F32Params::tangent).  In whitened
// coordinates z (x = A z) the box is a parallelogram whose face i is
// a_i . z = +-bt_i with unit normal a_i = (row i of A) / R_i, and xt_i =
// a_i . z, so the whitened face distances are m_i = bt_i - |xt_i|.  For the
// nearest face i (sign s = sign xt_i, inward normal n = -s a_i) the foot of
// z is f = z - m n, and the largest ball tangent to face i at f that stays
// inside the parallelogram has radius
//   rho = min(bt_i, (bt_j - xt_j(f)) / (1 - s c), (bt_j + xt_j(f)) / (1 + s c))
// with c = a_i . a_j and xt_j(f) = xt_j + s m c (distances are affine, the
// ball must clear the opposite face and both faces of the other axis; the
// kernel evaluates it mirrored by s, which removes the sign selects).  rho
// >= m always (the centred ball of radius m is one such ball), so the ball
// contains z.  Seen from z at depth m below the tangent point, the exit
// point of Brownian motion from the ball is the Moebius image of a uniform
// point: its angle t from the tangent point has tan(t/2) = m / (2 rho - m)
// tan(psi) with psi uniform in (-pi/2, pi/2).  With N = m sin psi, D =
// (2 rho - m) cos psi, E = N^2 + D^2 the exit lies at depth 2 rho N^2 / E
// below the face and tangential offset 2 rho N D / E from the foot -- on the
// sphere exactly, whatever the rounding of (sin, cos).  Near a face the depth
// contracts quadratically (m -> ~m^2 / 2 rho) instead of by a factor ~2.
__device__ __forceinline__ void psi_sincos(float psi, float* sn, float* cs) {
#if EM_POLY_SINCOS
  const float x2 = psi * psi;
  *sn = psi * fmaf(fmaf(fmaf(-0.00018363844719715416f, x2, 0.008306332863867283f), x2,
                        -0.16664829850196838f), x2, 0.9999966025352478f);
  *cs = fmaf(fmaf(fmaf(fmaf(2.3154105292633176e-05f, x2, -0.0013853712007403374f), x2,
                       0.04166358709335327f), x2, -0.4999990463256836f), x2, 0.9999999403953552f);
#else
  __sincosf(psi, sn, cs);
#endif
}

template <int D, int OUTER, int NH, int CHAIN, bool IDENT>
struct Tangent {
  static constexpr bool value =
      CHAIN == EM_CHAIN_TANGENT && NH == 0 && !IDENT &&
      ((D == 2 && OUTER == OUTER_BOX) || (D == 3 && (OUTER == OUTER_BOX || OUTER == OUTER_LBOX)));
};

// One tangent-ball step from x: the 0/1 walking mask (sat of the Euclidean
// stop margin, as everywhere) and the candidate next point n0, n1.  The
// caller keeps x for lanes that do not walk (stopped, idle: their candidate
// is not meaningful).  word: 32 random bits for psi.
__device__ __forceinline__ float tangent_step(const F32Params& P, const float* x, unsigned word,
                                              unsigned one_bits, float& n0, float& n1) {
  const float a0 = fabsf(x[0]), a1 = fabsf(x[1]);
  const float m0 = P.tbt[0] - a0, m1 = P.tbt[1] - a1;
  const float wm = __saturatef(fminf(P.tsb[0] - a0, P.tsb[1] - a1) * P.ss_scale);
  const bool p0 = m0 <= m1;  // nearest face: axis 0
  const float m = fminf(m0, m1);
  const float xi = p0 ? x[0] : x[1], xj = p0 ? x[1] : x[0];
  const float bti = p0 ? P.tbt[0] : P.tbt[1], btj = p0 ? P.tbt[1] : P.tbt[0];
  // work in the frame mirrored by s = sign xt_i (s xt_j, faces j at -+bt_j
  // swap roles), where the foot is fs = s xt_j + m c and the two face-j
  // limits are (bt_j - fs) / (1 - c) and (bt_j + fs) / (1 + c): no selects
  const float sg = copysignf(1.0f, xi);                    // s
  const float fj = fmaf(m, P.tcd, sg * xj);                // s * foot_j
  float rho = fminf(bti, fminf((btj - fj) * P.tim, (btj + fj) * P.tip));
  rho = fmaf(fmaxf(rho, m), P.tkeep, -P.tsa);
  // psi uniform in [-pi/2, pi/2): the low 23 bits into the mantissa of 1.0f
  // (one LOP3: (word & 0x7fffff) | one_bits)
  const float psi = fmaf(__uint_as_float(one_bits | (word & 0x7fffffu)), kPi, -1.5f * kPi);
  float sn, cs;
  psi_sincos(psi, &sn, &cs);
  const float N = m * sn, Dd = fmaf(2.0f, rho, -m) * cs;
  const float NN = N * N;
  const float g = fdiv(rho + rho, fmaf(Dd, Dd, NN));
  const float dep = g * NN, off = g * N * Dd;              // depth below face i, offset along it
  const float ni = sg * (bti - dep);  // may lie past the centre line: no copysign
  const float nj = sg * fmaf(off, P.tsd, fmaf(-dep, P.tcd, fj));
  n0 = p0 ? ni : nj;
  n1 = p0 ? nj : ni;
  return wm;
}

// 3D box / L-box on tangent balls, same stored coordinates xt_i = a_i . z
// (F32Params::t3 holds the per-face constants, T below is face i's row in
// shared memory).  For the nearest face i (side s, depth m), in the frame
// mirrored by s the foot has coordinates F_l = s xt_l + m C_il (F_i = bt_i)
// and the ball tangent there must clear the other five faces:
//   rho <= min_l min((bt_l - F_l) / (1 - C_il), (bt_l + F_l) / (1 + C_il))
// (l = i: only the opposite face, (bt_i + F_i) / 2 = bt_i).  The L-box adds
// the notch W = {xt_0 >= tn_0, xt_1 >= tn_1}: its two planes are candidate
// tangent faces too (depth d_q = tn_q - xt_q, side s = +1; a ball on the
// far side of either plane misses W), and a ball tangent to a box face must
// lie beyond one of them: rho <= max_q (tn_q - xt_q(f)) / (1 - s C_iq)
// (the centre's distance to the half-space W lies in; a sufficient test).
// Brownian motion from z, on the axis at depth m below the tangent point,
// leaves the ball at polar angle t from that point with |z - y| uniform in
// 1 / |z - y| (3D Poisson kernel), i.e. with V uniform the exit lies at depth
//   dep = (m / den)^2 2 (1 - V) (rho + (rho - m) V),  den = m + 2 (rho - m) V
// below the face (no cancellation as m -> 0) and at tangential distance
// sqrt(dep (2 rho - dep)) along a uniform azimuth.  V and the azimuth take
// 16 bits each of one 32-bit word: 2^32 cells of equal harmonic measure
// (the midpoint rule of the 3D directions).
template <int OUTER>
__device__ __forceinline__ float tangent_step3(const F32Params& P, const float* tab, const float* x,
                                               unsigned word, unsigned one_bits, float* nx) {
  const float a0 = fabsf(x[0]), a1 = fabsf(x[1]), a2 = fabsf(x[2]);
  const float m0 = P.tbt[0] - a0, m1 = P.tbt[1] - a1, m2 = P.tbt[2] - a2;
  float wm = __saturatef(fminf(fminf(P.tsb[0] - a0, P.tsb[1] - a1), P.tsb[2] - a2) * P.ss_scale);
  // nearest face as a running argmin carrying the face's coordinate and the
  // offset of its constant row (selects only, no index arithmetic)
  float m = m0, xi = x[0];
  int off = 0;
  {
    const bool b = m1 < m;
    m = fminf(m, m1);
    xi = b ? x[1] : xi;
    off = b ? 24 : off;
  }
  {
    const bool b = m2 < m;
    m = fminf(m, m2);
    xi = b ? x[2] : xi;
    off = b ? 48 : off;
  }
  float sg = copysignf(1.0f, xi);
  bool notch = false;
  if (OUTER == OUTER_LBOX) {
    // Euclidean distance to the notch prism (world units) for the stop test
    const float qx = fmaf(-P.ax[0], x[0], P.notch[0]), qy = fmaf(-P.ax[1], x[1], P.notch[1]);
    const float ex = fmaxf(qx, 0.0f), ey = fmaxf(qy, 0.0f);
    const float en = fsqrt(fmaf(ex, ex, ey * ey));
    wm = fminf(wm, __saturatef(fmaf(en, P.stop_scale, P.stop_bias)));
    const float d0 = P.tn[0] - x[0], d1 = P.tn[1] - x[1];
    const float dn = fmaxf(d0, d1);
    notch = dn < m;
    off = notch ? (d0 >= d1 ? 0 : 24) : off;
    sg = notch ? 1.0f : sg;
    m = fminf(m, dn);
  }
  const float4* T = reinterpret_cast<const float4*>(tab + off);
  const float4 t0 = T[0], t1 = T[1], t2 = T[2], t3 = T[3], t4 = T[4], t5 = T[5];
  const float C[3] = {t0.x, t0.y, t0.z}, P1[3] = {t0.w, t1.x, t1.y}, P2[3] = {t1.z, t1.w, t2.x};
  const float Bm[3] = {t2.y, t2.z, t2.w}, tim[3] = {t3.x, t3.y, t3.z};
  const float Bp[3] = {t3.w, t4.x, t4.y}, tip[3] = {t4.z, t4.w, t5.x};
  float F[3], rho = kInf;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    F[l] = fmaf(m, C[l], sg * x[l]);
    rho = fminf(rho, fminf(fmaf(-F[l], tim[l], Bm[l]), fmaf(F[l], tip[l], Bp[l])));
  }
  if (OUTER == OUTER_LBOX) {
    const bool pos = sg > 0.0f;
    const float r0 = (P.tn[0] - sg * F[0]) * (pos ? tim[0] : tip[0]);
    const float r1 = (P.tn[1] - sg * F[1]) * (pos ? tim[1] : tip[1]);
    rho = notch ? rho : fminf(rho, fmaxf(r0, r1));
  }
  rho = fmaf(fmaxf(rho, m), P.tkeep, -P.tsa);
  // V2 = 2V = (2k + 1) / 2^16 from the high half-word, azimuth from the low
  const float fv = __uint_as_float(__byte_perm(word, one_bits, 0x7632u));
  const float v2 = fmaf(fv, 256.0f, -256.0f) + 1.52587890625e-05f;
  const float h = rho - m;
  const float g = fdiv(m, fmaf(h, v2, m));
  const float dep = (g * g) * ((2.0f - v2) * fmaf(0.5f * h, v2, rho));
  const float tr = fsqrt(fmaxf(dep * fmaf(2.0f, rho, -dep), 0.0f));
  float sn, cs;
  __sincosf(angle_of(__byte_perm(word, one_bits, 0x7610u)), &sn, &cs);
  const float tc = tr * cs, ts = tr * sn;
#pragma unroll
  for (int l = 0; l < 3; ++l) nx[l] = sg * fmaf(ts, P2[l], fmaf(tc, P1[l], fmaf(-dep, C[l], F[l])));
  return wm;
}

// 3D ball on the tangent chain: walk on ROLLING balls.  In whitened
// coordinates z (x = diag(Ad) z in the rotated frame) the domain is the
// ellipsoid |diag(Ad) z| <= R, inside which every ball of radius rho_b (its
// smallest curvature radius) rolls freely: the ball of that radius
// internally tangent at any boundary point p lies in the domain (Blaschke).
// p is the radial projection of x onto the sphere |x| = R; its inward
// whitened normal is -diag(Ad) x / |Ax|, so with al = 1 - R / |x| and
// be = rho_b / |Ax| the offset from the ball's centre is
//   w = z - c = x (al / Ad + be Ad)          (per axis: one FFMA, one FMUL)
// and z lies in the ball's near half (towards p) iff al |x|^2 + be |Ax|^2 > 0.
// There the step samples the ball's harmonic measure from the off-centre
// point z (distance d = |w| from the centre, axis w / d: the 3D Poisson
// kernel, same depth formula as tangent_step3 with m = rho_b - d, on the
// ball's own axis); elsewhere it is the max chain's centred ball (d = 0, the
// same formula gives the uniform sphere).  Near the boundary z sits close to
// p on the ball's axis, so the depth contracts quadratically (cfg4: 35.6 ->
// ~7 steps per walk).  The orthonormal frame around the axis is Duff et
// al.'s branch-free construction.
__device__ __forceinline__ float rsq(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float roll_step3(const F32Params& P, const float* x, unsigned word,
                                            unsigned one_bits, float* nx) {
  const float p0 = x[0] * x[0], p1 = x[1] * x[1], p2 = x[2] * x[2];
  const float s2 = p0 + p1 + p2;
  const float aa = fmaf(P.Kd[0], p0, fmaf(P.Kd[1], p1, P.Kd[2] * p2));
  const float wm = __saturatef(fmaf(s2, -P.s2_scale, P.s2_bias));
  // clamped: a walk at the exact centre (x = 0) keeps finite terms
  const float iaa = rsq(fmaxf(aa, 1e-30f));
  const float sa = aa * iaa;  // |Ax|
  // max chain: the largest centred whitened ball, r = q / (|Ax| + sqrt(|Ax|^2 + q))
  const float q = P.oR2 - s2;
  const float rm = fmaf(fdiv(q, sa + fsqrt(fmaxf(aa + q, 0.0f))), P.keep, -P.shrink_abs);
  // rolling ball tangent at the radial projection
  const float al = fmaf(-P.oR, rsq(fmaxf(s2, 1e-30f)), 1.0f);
  const float be = P.rho_b * iaa;
  const float w0 = x[0] * fmaf(al, P.ia[0], be * P.Ad[0]);
  const float w1 = x[1] * fmaf(al, P.ia[1], be * P.Ad[1]);
  const float w2 = x[2] * fmaf(al, P.ia[2], be * P.Ad[2]);
  const float d2 = fmaf(w0, w0, fmaf(w1, w1, w2 * w2));
  const bool roll = (d2 < P.rho_b2) & (fmaf(al, s2, be * aa) > 0.0f);
  const float rho = roll ? P.rho_b : rm;
  const float id = rsq(fmaxf(d2, 1e-30f));
  const float d = roll ? d2 * id : 0.0f;
  const float e0 = roll ? w0 * id : 0.0f, e1 = roll ? w1 * id : 0.0f, e2 = roll ? w2 * id : 1.0f;
  const float m = rho - d;
  // V2 = 2V from the high half-word, azimuth from the low one
  const float fv = __uint_as_float(__byte_perm(word, one_bits, 0x7632u));
  const float v2 = fmaf(fv, 256.0f, -256.0f) + 1.52587890625e-05f;
  const float g = fdiv(m, fmaf(d, v2, m));
  const float dep = (g * g) * ((2.0f - v2) * fmaf(0.5f * d, v2, rho));
  const float tr = fsqrt(fmaxf(dep * fmaf(2.0f, rho, -dep), 0.0f));
  float sn, cs;
  __sincosf(angle_of(__byte_perm(word, one_bits, 0x7610u)), &sn, &cs);
  const float tc = tr * cs, ts = tr * sn;
  // Duff et al.: (b1, b2, e) orthonormal, branch-free
  const float sg = copysignf(1.0f, e2);
  const float A = -fdiv(1.0f, sg + e2);
  const float B = e0 * e1 * A;
  const float b10 = fmaf(sg * e0 * e0, A, 1.0f), b11 = sg * B, b12 = -sg * e0;
  const float b20 = B, b21 = fmaf(e1 * e1, A, sg), b22 = -e1;
  const float h = m - dep;
  nx[0] = fmaf(P.Ad[0], fmaf(h, e0, fmaf(tc, b10, ts * b20)), x[0]);
  nx[1] = fmaf(P.Ad[1], fmaf(h, e1, fmaf(tc, b11, ts * b21)), x[1]);
  nx[2] = fmaf(P.Ad[2], fmaf(h, e2, fmaf(tc, b12, ts * b22)), x[2]);
  return wm;
}

// 2D ball / concentric annulus on the tangent chain: the same rolling disks
// for the outer ellipse (radius rho_b, capped so the disk also clears the
// hole), and for the hole the disk of radius rho_h externally tangent at the
// radial projection onto the hole: it misses the (convex) hole whatever its
// radius, and rho_h = (R - rho) / (2 max Ad) keeps it inside the outer
// circle.  The exit from an off-centre point of a disk is the Moebius image
// of a uniform angle (tangent_step's formula with m = radius - d on the
// disk's own axis); the centred max-chain disk is the d = 0 case.
template <int NH>
__device__ __forceinline__ float roll_step2(const F32Params& P, const float* x, unsigned word,
                                            unsigned one_bits, float* nx) {
  const float p0 = x[0] * x[0], p1 = x[1] * x[1];
  const float s2 = p0 + p1;
  const float aa = fmaf(P.Kd[0], p0, P.Kd[1] * p1);
  float wm = __saturatef(fmaf(s2, -P.s2_scale, P.s2_bias));
  if (NH == 1) wm = fminf(wm, __saturatef(fmaf(s2, P.h2_scale, P.h2_bias)));
  // clamped: a walk at the exact centre (x = 0) keeps finite terms.  In the
  // annulus (NH == 1) a walking lane has rho + eps < |x| < R - eps, so every
  // square and root argument below is positive; a lane that is not walking
  // (stopped, parked far outside) may produce NaNs, but its mask is 0 and
  // the caller keeps its point -- no clamps there
  const float iaa = rsq(NH == 1 ? aa : fmaxf(aa, 1e-30f));
  const float sa = aa * iaa;  // |Ax|
  const float ir = rsq(NH == 1 ? s2 : fmaxf(s2, 1e-30f));
  // max chain: the largest centred whitened disk
  float rm;
  if (NH == 0) {
    const float q = P.oR2 - s2;
    rm = fmaf(fdiv(q, sa + fsqrt(fmaxf(aa + q, 0.0f))), P.keep, -P.shrink_abs);
  } else {
    // min(qo / Do, qh / Dh) with one reciprocal: min(qo Dh, qh Do) / (Do Dh)
    const float qo = P.oR2 - s2;
    const float Do = sa + fsqrt(aa + qo);
    const float qh = s2 - P.hr2[0];
    const float Dh = sa + fsqrt(fmaf(-P.m2, qh, aa));
    rm = fmaf(fdiv(fminf(qo * Dh, qh * Do), Do * Dh), P.keep, -P.shrink_abs);
  }
  // rolling disk at the outer ellipse
  float rb = P.rho_b, rb2 = P.rho_b2, rh = P.rho_h, rh2 = P.rho_h2;
  if (NH == 1 && EM_ROLL2_DYN) {
    // radii from the local normal: |diag(Ad) n| = |diag(Ad^2) x| / |Ax|
    const float q4 = fmaf(P.K4[0], p0, P.K4[1] * p1);
    rh = fdiv(P.gap, fmaf(q4 * rsq(q4), iaa, P.amax));
    rb = fminf(P.rb_bl, rh);
    rb2 = rb * rb;
    rh2 = rh * rh;
  }
  float w0, w1, d2, rho;
  bool use;
  if (NH == 1 && EM_ROLL2_ONE && !EM_ROLL2_DYN) {
    // ONE candidate disk per step: the outer rolling disk when |x| lies
    // beyond the annulus' mid radius, else the hole-tangent disk (same
    // offset algebra with the hole's radius and a negative signed radius);
    // z must lie inside it and on its near side, else the centred disk.
    // Any disk containing z inside the domain is a valid step; this choice
    // matches trying the outer disk first and then the hole's (same steps
    // per walk on cfg3), at one disk's cost instead of two.
    const bool outer = s2 > P.mid2;
    const float rc = outer ? rb : rh, rc2 = outer ? rb2 : rh2;
    const float bs = outer ? rb : -rh;  // signed radius: inward from the outer circle
    const float al = fmaf(outer ? -P.oR : -P.hr[0], ir, 1.0f);
    const float be = bs * iaa;
    w0 = x[0] * fmaf(al, P.ia[0], be * P.Ad[0]);
    w1 = x[1] * fmaf(al, P.ia[1], be * P.Ad[1]);
    d2 = fmaf(w0, w0, w1 * w1);
    use = (d2 < rc2) & (fmaf(al, s2, be * aa) * bs > 0.0f);
    rho = use ? rc : rm;
  } else {
  const float al = fmaf(-P.oR, ir, 1.0f);
  const float be = rb * iaa;
  w0 = x[0] * fmaf(al, P.ia[0], be * P.Ad[0]);
  w1 = x[1] * fmaf(al, P.ia[1], be * P.Ad[1]);
  d2 = fmaf(w0, w0, w1 * w1);
  use = (d2 < rb2) & (fmaf(al, s2, be * aa) > 0.0f);
  rho = use ? rb : rm;
  if (NH == 1) {
    // disk tangent to the hole from outside, centre beyond the radial projection
    const float ah = fmaf(-P.hr[0], ir, 1.0f);
    const float bh = rh * iaa;
    const float v0 = x[0] * fmaf(ah, P.ia[0], -bh * P.Ad[0]);
    const float v1 = x[1] * fmaf(ah, P.ia[1], -bh * P.Ad[1]);
    const float dh = fmaf(v0, v0, v1 * v1);
    const bool uh = !use & (dh < rh2) & (fmaf(ah, s2, -bh * aa) < 0.0f);
    w0 = uh ? v0 : w0;
    w1 = uh ? v1 : w1;
    d2 = uh ? dh : d2;
    rho = uh ? rh : rho;
    use |= uh;
  }
  }
  const float id = rsq(fmaxf(d2, 1e-30f));
  const float d = use ? d2 * id : 0.0f;
  const float e0 = use ? w0 * id : 1.0f, e1 = use ? w1 * id : 0.0f;
  const float m = rho - d;
  // Moebius: psi uniform in [-pi/2, pi/2) from the low 23 bits (one LOP3)
  const float psi = fmaf(__uint_as_float(one_bits | (word & 0x7fffffu)), kPi, -1.5f * kPi);
  float sn, cs;
  psi_sincos(psi, &sn, &cs);
  const float N = m * sn, Dd = fmaf(2.0f, rho, -m) * cs;
  const float NN = N * N;
  const float g = fdiv(rho + rho, fmaf(Dd, Dd, NN));
  const float dep = g * NN, off = g * N * Dd;
  const float h = m - dep;
  nx[0] = fmaf(P.Ad[0], fmaf(h, e0, -off * e1), x[0]);
  nx[1] = fmaf(P.Ad[1], fmaf(h, e1, off * e0), x[1]);
  return wm;
}

template <int D, int OUTER, int NH, int CHAIN, bool IDENT>
struct Roll {
  static constexpr bool value = CHAIN == EM_CHAIN_TANGENT && OUTER == OUTER_BALL && !IDENT &&
                                ((D == 3 && NH == 0) || (D == 2 && (NH == 0 || NH == 1)));
};

constexpr int kWarps = 8;   // 256 threads per block
constexpr int kQueue = 64;  // deferred exits per warp (binned 32 at a time)

// Bin one exit (owner component -> side -> nearest anchor), count it, and
// add its step count to this lane's per-pole accumulator.
// Kernel coordinates -> frame coordinates (the frame the owner test reads:
// rotated for balls, whose hole centres are stored rotated; unsheared for
// boxes) and -> world coordinates.
template <int D, int OUTER, bool SHEAR>
__device__ __forceinline__ void to_frame(const F32Params& P, const float* x, float* xf) {
  for (int i = 0; i < 3; ++i) xf[i] = (i < D) ? (SHEAR ? P.ax[i] * x[i] : x[i]) : 0.0f;
}

template <int D, int OUTER>
__device__ __forceinline__ void frame_to_world(const F32Params& P, const float* xf, float* xw) {
  if (OUTER == OUTER_BALL && P.rot) {
    const float* Q = P.Q;
    if (D == 2) {
      xw[0] = fmaf(Q[0], xf[0], fmaf(Q[1], xf[1], P.frame[0]));
      xw[1] = fmaf(Q[3], xf[0], fmaf(Q[4], xf[1], P.frame[1]));
      xw[2] = 0.0f;
    } else {
      xw[0] = fmaf(Q[0], xf[0], fmaf(Q[1], xf[1], fmaf(Q[2], xf[2], P.frame[0])));
      xw[1] = fmaf(Q[3], xf[0], fmaf(Q[4], xf[1], fmaf(Q[5], xf[2], P.frame[1])));
      xw[2] = fmaf(Q[6], xf[0], fmaf(Q[7], xf[1], fmaf(Q[8], xf[2], P.frame[2])));
    }
    return;
  }
  xw[0] = xf[0] + P.frame[0];
  xw[1] = xf[1] + P.frame[1];
  xw[2] = D == 3 ? xf[2] + P.frame[2] : 0.0f;
}

// Pole-block scheduler (SMEM == 2): the block's shared-memory histogram of
// its one pole's count row (dynamic shared memory, row_len u32 words).
__device__ __forceinline__ unsigned* block_hist() {
  return reinterpret_cast<unsigned*>(s_stats);
}

template <int D, int OUTER, int NH, int BINK, int SMEM, bool SHEAR, bool FULL = true>
__device__ __forceinline__ void retire(const F32Params& P, const float* x, int pole, int steps,
                                       StepAcc& acc) {
  const WorkOut& W = P.w;
  float xf[3], xw[3];
  to_frame<D, OUTER, SHEAR>(P, x, xf);
  int side;
  if (OUTER == OUTER_LBOX || NH != 0) side = P.comp_side[owner<D, OUTER, NH>(P, xf)];
  else side = P.comp_side[0];
  frame_to_world<D, OUTER>(P, xf, xw);
  const int a = bin_exit<D, BINK>(P, side, xw);
  const int col = side ? W.col_off1 + a : a;
  EM_DEV_ASSERT(side == 0 || side == 1);
  EM_DEV_ASSERT(a >= 0 && a < (side ? P.side[1].n_anchors : P.side[0].n_anchors));
  EM_DEV_ASSERT(col >= 0 && col < W.row_len && pole >= 0 && pole < W.n_poles);
  if (SMEM == 2) {
    // one pole per block: warp-aggregated shared-memory histogram (all 32
    // lanes bin together in the deferred pass: __match_any_sync groups equal
    // bins, the lowest lane of each group adds the group's count)
    unsigned* hist = block_hist();
    if (FULL) {
      const unsigned peers = __match_any_sync(kFull, col);
      if ((peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0u) atomicAdd(&hist[col], __popc(peers));
    } else {
      atomicAdd(&hist[col], 1u);
    }
    acc.sum += (unsigned long long)steps;
    acc.sq += (unsigned long long)steps * (unsigned long long)steps;
    acc.mx = (unsigned long long)steps > acc.mx ? (unsigned long long)steps : acc.mx;
    return;
  }
  atomicAdd(&W.counts[(long long)pole * W.row_len + col], 1ULL);
  acc_add<SMEM>(acc, W, pole, (unsigned long long)steps);
}

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
      float wm = 0.0f, sf = 0.0f;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (TANG || ROLL) {
          float nx[3];
          if (ROLL && D == 3) wm = roll_step3(P, x, wv[k], P.one_bits, nx);
          else if (ROLL) wm = roll_step2<NH>(P, x, wv[k], P.one_bits, nx);
          else if (D == 2) wm = tangent_step(P, x, wv[k], P.one_bits, nx[0], nx[1]);
          else wm = tangent_step3<OUTER>(P, ttab, x, wv[k], P.one_bits, nx);
          const bool go = wm != 0.0f;
#pragma unroll
          for (int l = 0; l < D; ++l) x[l] = go ? nx[l] : x[l];
        } else {
          float t, r;
          dist<D, OUTER, NH, CHAIN, IDENT>(P, x, t, r);
          wm = t;  // already the saturated 0/1 mask
          step<D, OUTER, IDENT, SHEAR>(P, x, r * wm, D == 3 ? z_of<D>(wv, k, P.one_bits) : 0.0f,
                                       angle_bits<D>(wv, k, P.one_bits));
        }
        sf += wm;
      }
      walking = wm != 0.0f;
      steps += (int)sf;
      if (EM_POST_STOP) {
        // the stop test of the point the last move landed on (the next
        // batch's first test, evaluated now): a walk that reached the shell
        // on a batch's last step retires at this service pass instead of
        // idling through one more batch (cfg2-cfg5 +9-12%).  Only the stop
        // mask of the step functions is live here (the rest is dead code).
        // Same criterion, same moves and draws; the two evaluations of the
        // test may round apart on a point at the shell's edge (separately
        // scheduled FMA chains), so such a walk can end one step earlier --
        // and a lane left without work is parked far outside (service).
        float t2;
        if (TANG || ROLL) {
          float nx[3];
          if (ROLL && D == 3) t2 = roll_step3(P, x, 0u, P.one_bits, nx);
          else if (ROLL) t2 = roll_step2<NH>(P, x, 0u, P.one_bits, nx);
          else if (D == 2) t2 = tangent_step(P, x, 0u, P.one_bits, nx[0], nx[1]);
          else t2 = tangent_step3<OUTER>(P, ttab, x, 0u, P.one_bits, nx);
        } else {
          float r2;
          dist<D, OUTER, NH, CHAIN, IDENT>(P, x, t2, r2);
        }
        walking &= t2 != 0.0f;
      }
    } else {
      int failed = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        float t, r, nx[3] = {0.0f, 0.0f, 0.0f};
        if (ROLL && D == 3) t = roll_step3(P, x, wv[k], P.one_bits, nx);
        else if (ROLL) t = roll_step2<NH>(P, x, wv[k], P.one_bits, nx);
        else if (TANG && D == 2) t = tangent_step(P, x, wv[k], P.one_bits, nx[0], nx[1]);
        else if (TANG) t = tangent_step3<OUTER>(P, ttab, x, wv[k], P.one_bits, nx);
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
#define EM_STR2(x) #x
#define EM_STR(x) EM_STR2(x)
const char* f32_build_knobs() {
  return "EM_BATCH_STEPS=" EM_STR(EM_BATCH_STEPS) " EM_ANGLE_BITS=" EM_STR(EM_ANGLE_BITS)
         " EM_Z_BITS=" EM_STR(EM_Z_BITS) " EM_TANG_K=" EM_STR(EM_TANG_K)
         " EM_POST_STOP=" EM_STR(EM_POST_STOP) " EM_MIN_BLOCKS=" EM_STR(EM_MIN_BLOCKS)
         " EM_ROLL2_BLOCKS=" EM_STR(EM_ROLL2_BLOCKS) " EM_ROLL2_DYN=" EM_STR(EM_ROLL2_DYN)
         " EM_TAB_WARP=" EM_STR(EM_TAB_WARP) " EM_ROLL2_ONE=" EM_STR(EM_ROLL2_ONE)
         " EM_POLY_SINCOS=" EM_STR(EM_POLY_SINCOS)
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
