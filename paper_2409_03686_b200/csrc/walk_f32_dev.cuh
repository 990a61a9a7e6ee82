// walk_f32_dev.cuh -- device functions of the production FP32 walk kernels
// (distance / step / samplers / owner / binners / retire), shared by
// walk_f32.cu (one walk per lane) and walk_f32x2.cu (two walks per lane,
// packed FP32 arithmetic).
#pragma once
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
// is not meaningful).  word: 32 random bits for psi.  Defined below, after
// the one-tree value operations (tang2_core).
__device__ __forceinline__ float tangent_step(const F32Params& P, const float* x, unsigned word,
                                              unsigned one_bits, float& n0, float& n1);

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
// Returns the walking predicate of x (the stop tests as compares: every face
// margin positive, and for the L-box the squared Euclidean distance to the
// notch prism above eps^2 -- no root).
template <int OUTER>
__device__ __forceinline__ bool tang3_go(const F32Params& P, const float* tab, const float* x,
                                         unsigned word, unsigned one_bits, float* nx) {
  const float a0 = fabsf(x[0]), a1 = fabsf(x[1]), a2 = fabsf(x[2]);
  const float m0 = P.tbt[0] - a0, m1 = P.tbt[1] - a1, m2 = P.tbt[2] - a2;
  bool go = (a0 < P.tsb[0]) & (a1 < P.tsb[1]) & (a2 < P.tsb[2]);
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
    go &= fmaf(ex, ex, ey * ey) > P.eps2;
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
  return go;
}

// the same step with the walking mask as a 0/1 float (em_debug_step)
template <int OUTER>
__device__ __forceinline__ float tangent_step3(const F32Params& P, const float* tab, const float* x,
                                               unsigned word, unsigned one_bits, float* nx) {
  return tang3_go<OUTER>(P, tab, x, word, one_bits, nx) ? 1.0f : 0.0f;
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
                                            unsigned one_bits, float* nx);  // below: roll3_core

// 2D ball / concentric annulus on the tangent chain: the same rolling disks
// for the outer ellipse (radius rho_b, capped so the disk also clears the
// hole), and for the hole the disk of radius rho_h externally tangent at the
// radial projection onto the hole: it misses the (convex) hole whatever its
// radius, and rho_h = (R - rho) / (2 max Ad) keeps it inside the outer
// circle.  The exit from an off-centre point of a disk is the Moebius image
// of a uniform angle (tangent_step's formula with m = radius - d on the
// disk's own axis); the centred max-chain disk is the d = 0 case.
template <int NH>
__device__ __forceinline__ float roll_step2_legacy(const F32Params& P, const float* x, unsigned word,
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

// ---- one operation tree for one walk (float) or two walks (float2) ----
// The rolling-disk step is written once over a value type T: float for the
// one-walk-per-lane kernel, float2 for the two-walks-per-lane kernel
// (walk_f32x2.cu), whose adds / multiplies / fmas are Blackwell's packed
// FADD2 / FMUL2 / FFMA2 -- one issued instruction for both walks.  Every
// arithmetic operation is an explicit round-to-nearest intrinsic (no compiler
// contraction), so both instantiations compute the SAME tree and a walk's
// points are bit-identical whichever kernel or slot runs it.
struct Mask2 {
  bool x, y;
};
__device__ __forceinline__ float vmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float vadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float vsub(float a, float b) { return __fadd_rn(a, -b); }
__device__ __forceinline__ float vfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float vneg(float a) { return -a; }
__device__ __forceinline__ float vrsq(float a) { return rsq(a); }
__device__ __forceinline__ float vsqrt(float a) { return fsqrt(a); }
__device__ __forceinline__ float vrcp(float a) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float vmaxs(float a, float s) { return fmaxf(a, s); }
__device__ __forceinline__ bool vlt(float a, float b) { return a < b; }
__device__ __forceinline__ bool vgt(float a, float b) { return a > b; }
__device__ __forceinline__ bool vand(bool a, bool b) { return a & b; }
__device__ __forceinline__ float vsel(bool m, float a, float b) { return m ? a : b; }
__device__ __forceinline__ void vsincos(float a, float& sn, float& cs) { psi_sincos(a, &sn, &cs); }
// 23 low bits of a word into the mantissa of 1.0f (one LOP3)
__device__ __forceinline__ float vbits23(unsigned w, unsigned one_bits) {
  return __uint_as_float(one_bits | (w & 0x7fffffu));
}

__device__ __forceinline__ float2 vbc(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 vneg(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 vmul(float2 a, float s) { return __fmul2_rn(a, vbc(s)); }
__device__ __forceinline__ float2 vadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 vadd(float2 a, float s) { return __fadd2_rn(a, vbc(s)); }
__device__ __forceinline__ float2 vsub(float2 a, float2 b) { return __fadd2_rn(a, vneg(b)); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 vfma(float2 a, float s, float2 c) { return __ffma2_rn(a, vbc(s), c); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float s) { return __ffma2_rn(a, b, vbc(s)); }
__device__ __forceinline__ float2 vfma(float2 a, float s, float t) { return __ffma2_rn(a, vbc(s), vbc(t)); }
__device__ __forceinline__ float2 vrsq(float2 a) { return make_float2(rsq(a.x), rsq(a.y)); }
__device__ __forceinline__ float2 vsqrt(float2 a) { return make_float2(fsqrt(a.x), fsqrt(a.y)); }
__device__ __forceinline__ float2 vrcp(float2 a) { return make_float2(vrcp(a.x), vrcp(a.y)); }
__device__ __forceinline__ float2 vmin(float2 a, float2 b) {
  return make_float2(fminf(a.x, b.x), fminf(a.y, b.y));
}
__device__ __forceinline__ float2 vmaxs(float2 a, float s) {
  return make_float2(fmaxf(a.x, s), fmaxf(a.y, s));
}
__device__ __forceinline__ Mask2 vlt(float2 a, float2 b) { return {a.x < b.x, a.y < b.y}; }
__device__ __forceinline__ Mask2 vlt(float2 a, float s) { return {a.x < s, a.y < s}; }
__device__ __forceinline__ Mask2 vgt(float2 a, float s) { return {a.x > s, a.y > s}; }
__device__ __forceinline__ Mask2 vand(Mask2 a, Mask2 b) { return {a.x && b.x, a.y && b.y}; }
__device__ __forceinline__ float2 vsel(Mask2 m, float2 a, float2 b) {
  return make_float2(m.x ? a.x : b.x, m.y ? a.y : b.y);
}
__device__ __forceinline__ float2 vsel(Mask2 m, float2 a, float s) {
  return make_float2(m.x ? a.x : s, m.y ? a.y : s);
}
__device__ __forceinline__ float2 vsel(Mask2 m, float s, float2 b) {
  return make_float2(m.x ? s : b.x, m.y ? s : b.y);
}
__device__ __forceinline__ float2 vsel(Mask2 m, float s, float t) {
  return make_float2(m.x ? s : t, m.y ? s : t);
}
__device__ __forceinline__ void vsincos(float2 a, float2& sn, float2& cs) {
#if EM_POLY_SINCOS
  const float2 q = vmul(a, a);
  sn = vmul(a, vfma(vfma(vfma(q, -0.00018363844719715416f, 0.008306332863867283f), q,
                         -0.16664829850196838f), q, 0.9999966025352478f));
  cs = vfma(vfma(vfma(vfma(q, 2.3154105292633176e-05f, -0.0013853712007403374f), q,
                      0.04166358709335327f), q, -0.4999990463256836f), q, 0.9999999403953552f);
#else
  __sincosf(a.x, &sn.x, &cs.x);
  __sincosf(a.y, &sn.y, &cs.y);
#endif
}
__device__ __forceinline__ float2 vbits23(uint2 w, unsigned one_bits) {
  return make_float2(__uint_as_float(one_bits | (w.x & 0x7fffffu)),
                     __uint_as_float(one_bits | (w.y & 0x7fffffu)));
}

// |x|^2 as the step and every stop test compute it.  (No add in these trees
// takes a bare product as an operand: where one would, the fma is written out
// -- the packed intrinsics are contracted by the compiler, the scalar _rn
// intrinsics never are, and the two instantiations must round alike.)
template <class T>
__device__ __forceinline__ T roll2_s2(T x0, T x1) {
  return vfma(x1, x1, vmul(x0, x0));
}

// The rolling-disk step (header comment above) from (x0, x1): candidate next
// point (n0, n1) and |x|^2 (the stop tests read it).  T = float / float2,
// WD = unsigned / uint2 (one random word per walk).
template <int NH, class T, class WD>
__device__ __forceinline__ void roll2_core(const F32Params& P, T x0, T x1, WD word,
                                           unsigned one_bits, T& s2_out, T& n0, T& n1) {
  const T p0 = vmul(x0, x0), p1 = vmul(x1, x1);
  const T s2 = vfma(x1, x1, p0);  // roll2_s2
  s2_out = s2;
  const T aa = vfma(p0, P.Kd[0], vmul(p1, P.Kd[1]));
  // clamped: a walk at the exact centre (x = 0) keeps finite terms.  In the
  // annulus (NH == 1) a walking lane has rho + eps < |x| < R - eps, so every
  // square and root argument below is positive; a lane that is not walking
  // (stopped, parked far outside) may produce NaNs, but the caller keeps its
  // point -- no clamps there
  const T iaa = vrsq(NH == 1 ? aa : vmaxs(aa, 1e-30f));
  const T ir = vrsq(NH == 1 ? s2 : vmaxs(s2, 1e-30f));
  // max chain: the largest centred whitened disk, in its difference forms
  //   outer: q / (|Ax| + sqrt(|Ax|^2 + q)) = sqrt(|Ax|^2 + q) - |Ax|,  q = R^2 - |x|^2
  //   hole:  q / (|Ax| + sqrt(|Ax|^2 - m2 q)) = (|Ax| - sqrt(|Ax|^2 - m2 q)) / m2,
  //          q = |x|^2 - rho^2
  // (no reciprocal: two MUFU ops instead of three, five fewer operations than
  // the quotient forms).  The differences cancel near a boundary, but the
  // centred disk is only USED far from both (otherwise z lies in a rolling /
  // hole-tangent disk): there its radius is >= ~the rolling radius and the
  // absolute error of a difference -- bounded by shrink_c, which the plan
  // derives from the MUFU error bounds and max |A| R -- is a ~1e-5 relative
  // shrink.  |Ax| = aa * rsqrt(aa), folded into the fmas.
  T rm;
  const T qo = vfma(s2, -1.0f, P.oR2);
  if (NH == 0) {
    const T ro = vfma(vneg(aa), iaa, vsqrt(vmaxs(vadd(aa, qo), 0.0f)));
    rm = vfma(ro, P.keep, -P.shrink_c);
  } else {
    const T ro = vfma(vneg(aa), iaa, vsqrt(vadd(aa, qo)));
    const T qh = vadd(s2, -P.hr2[0]);
    const T rh_ = vmul(vfma(aa, iaa, vneg(vsqrt(vfma(qh, -P.m2, aa)))), P.im2);
    rm = vfma(vmin(ro, rh_), P.keep, -P.shrink_c);
  }
  const float rb = P.rho_b, rb2 = P.rho_b2, rh = P.rho_h;
  T w0, w1, d2, rho;
  auto use = vlt(s2, s2);  // (type only)
  if (NH == 1) {
    // ONE candidate disk per step: the outer rolling disk when |x| lies
    // beyond the annulus' mid radius, else the hole-tangent disk (same
    // offset algebra with the hole's radius and a negative signed radius);
    // z must lie inside it and on its near side, else the centred disk.
    // Any disk containing z inside the domain is a valid step; this choice
    // matches trying the outer disk first and then the hole's (same steps
    // per walk on cfg3), at one disk's cost instead of two.
    // The choice enters as a 0/1 blend factor, so the four constants it
    // picks are fmas (packed: one instruction for both walks) instead of
    // selects: radius rc = rh + of (rb - rh) -- exact: the plan rounds rb so
    // that fl(rh + rc_d) == rho_b -- side sign sg = 2 of - 1, and minus the
    // tangent circle's radius nr = -hr + of (hr - R).
    const T of = vsel(vgt(s2, P.mid2), 1.0f, 0.0f);
    const T rc = vfma(of, P.rc_d, rh);
    const T sg = vfma(of, 2.0f, -1.0f);  // +1: inward from the outer circle, -1: outward from the hole
    const T al = vfma(vfma(of, P.nr_d, -P.hr[0]), ir, 1.0f);
    const T be = vmul(vmul(rc, iaa), sg);
    w0 = vmul(x0, vfma(al, P.ia[0], vmul(be, P.Ad[0])));
    w1 = vmul(x1, vfma(al, P.ia[1], vmul(be, P.Ad[1])));
    d2 = vfma(w0, w0, vmul(w1, w1));
    use = vand(vlt(d2, vmul(rc, rc)), vgt(vmul(vfma(al, s2, vmul(be, aa)), sg), 0.0f));
    rho = vsel(use, rc, rm);
  } else {
    const T al = vfma(ir, -P.oR, 1.0f);
    const T be = vmul(iaa, rb);
    w0 = vmul(x0, vfma(al, P.ia[0], vmul(be, P.Ad[0])));
    w1 = vmul(x1, vfma(al, P.ia[1], vmul(be, P.Ad[1])));
    d2 = vfma(w0, w0, vmul(w1, w1));
    use = vand(vlt(d2, rb2), vgt(vfma(al, s2, vmul(be, aa)), 0.0f));
    rho = vsel(use, rb, rm);
  }
  // the centred disk is the d = 0 case: 1 / d masked once, axis (1, 0)
  const T id = vsel(use, vrsq(vmaxs(d2, 1e-30f)), 0.0f);
  const T e0 = vsel(use, vmul(w0, id), 1.0f), e1 = vmul(w1, id);
  const T m = vfma(vneg(d2), id, rho);  // rho - d, d = d2 / sqrt(d2)
  // Moebius: psi uniform in [-pi/2, pi/2) from the low 23 bits (one LOP3)
  const T psi = vfma(vbits23(word, one_bits), kPi, -1.5f * kPi);
  T sn, cs;
  vsincos(psi, sn, cs);
  const T N = vmul(m, sn), Dd = vmul(vfma(rho, 2.0f, vneg(m)), cs);
  const T NN = vmul(N, N);
  const T g = vmul(vadd(rho, rho), vrcp(vfma(Dd, Dd, NN)));
  const T off = vmul(vmul(g, N), Dd);
  const T h = vfma(vneg(g), NN, m);  // m - depth
  n0 = vfma(vfma(h, e0, vneg(vmul(off, e1))), P.Ad[0], x0);
  n1 = vfma(vfma(h, e1, vmul(off, e0)), P.Ad[1], x1);
}

// the default-knob chain (one candidate disk, fixed radii) has the generic
// tree above; the measured-and-rejected variants keep their own code
#define EM_ROLL2_GENERIC (EM_ROLL2_ONE && !EM_ROLL2_DYN)

template <int NH>
__device__ __forceinline__ float roll_step2(const F32Params& P, const float* x, unsigned word,
                                            unsigned one_bits, float* nx) {
#if EM_ROLL2_GENERIC
  float s2;
  roll2_core<NH, float, unsigned>(P, x[0], x[1], word, one_bits, s2, nx[0], nx[1]);
  float wm = __saturatef(fmaf(s2, -P.s2_scale, P.s2_bias));
  if (NH == 1) wm = fminf(wm, __saturatef(fmaf(s2, P.h2_scale, P.h2_bias)));
  return wm;
#else
  return roll_step2_legacy<NH>(P, x, word, one_bits, nx);
#endif
}

// ---- 2D box on the tangent-ball chain, same one-tree form ----
__device__ __forceinline__ float vabs(float a) { return fabsf(a); }
__device__ __forceinline__ float2 vabs(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
__device__ __forceinline__ float vsign1(float a) { return copysignf(1.0f, a); }
__device__ __forceinline__ float2 vsign1(float2 a) {
  return make_float2(copysignf(1.0f, a.x), copysignf(1.0f, a.y));
}
__device__ __forceinline__ bool vle(float a, float b) { return a <= b; }
__device__ __forceinline__ Mask2 vle(float2 a, float2 b) { return {a.x <= b.x, a.y <= b.y}; }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float2 vmax(float2 a, float2 b) {
  return make_float2(fmaxf(a.x, b.x), fmaxf(a.y, b.y));
}
__device__ __forceinline__ float2 vmin(float2 a, float s) {
  return make_float2(fminf(a.x, s), fminf(a.y, s));
}

// The tangent-ball step of the whitened parallelogram (comment above
// tangent_step): |xt_0|, |xt_1| out (the stop tests read them), candidate
// next point (n0, n1).
template <class T, class WD>
__device__ __forceinline__ void tang2_core(const F32Params& P, T x0, T x1, WD word,
                                           unsigned one_bits, T& a0, T& a1, T& n0, T& n1) {
  a0 = vabs(x0);
  a1 = vabs(x1);
  const T m0 = vfma(a0, -1.0f, P.tbt[0]), m1 = vfma(a1, -1.0f, P.tbt[1]);
  const auto p0 = vle(m0, m1);  // nearest face: axis 0
  const T m = vmin(m0, m1);
  const T xi = vsel(p0, x0, x1), xj = vsel(p0, x1, x0);
  const T bti = vsel(p0, P.tbt[0], P.tbt[1]), btj = vsel(p0, P.tbt[1], P.tbt[0]);
  // work in the frame mirrored by s = sign xt_i (s xt_j, faces j at -+bt_j
  // swap roles), where the foot is fs = s xt_j + m c and the two face-j
  // limits are (bt_j - fs) / (1 - c) and (bt_j + fs) / (1 + c): no selects
  const T sg = vsign1(xi);
  const T fj = vfma(m, P.tcd, vmul(sg, xj));  // s * foot_j
  T rho = vmin(bti, vmin(vmul(vsub(btj, fj), P.tim), vmul(vadd(btj, fj), P.tip)));
  rho = vfma(vmax(rho, m), P.tkeep, -P.tsa);
  // psi uniform in [-pi/2, pi/2): the low 23 bits into the mantissa of 1.0f
  const T psi = vfma(vbits23(word, one_bits), kPi, -1.5f * kPi);
  T sn, cs;
  vsincos(psi, sn, cs);
  const T N = vmul(m, sn), Dd = vmul(vfma(rho, 2.0f, vneg(m)), cs);
  const T NN = vmul(N, N);
  const T g = vmul(vadd(rho, rho), vrcp(vfma(Dd, Dd, NN)));
  const T dep = vmul(g, NN), off = vmul(vmul(g, N), Dd);  // depth below face i, offset along it
  const T ni = vmul(sg, vfma(vneg(g), NN, bti));  // s (bt_i - depth); may pass the centre line
  const T nj = vmul(sg, vfma(off, P.tsd, vfma(vneg(dep), P.tcd, fj)));
  n0 = vsel(p0, ni, nj);
  n1 = vsel(p0, nj, ni);
}

__device__ __forceinline__ float tangent_step(const F32Params& P, const float* x, unsigned word,
                                              unsigned one_bits, float& n0, float& n1) {
  float a0, a1;
  tang2_core<float, unsigned>(P, x[0], x[1], word, one_bits, a0, a1, n0, n1);
  return __saturatef(fminf(P.tsb[0] - a0, P.tsb[1] - a1) * P.ss_scale);
}

// ---- 3D ball on rolling balls (comment above roll_step3), one-tree form ----
// half-words of the random word into the mantissa of 1.0f (one PRMT each)
__device__ __forceinline__ float vhalf_hi(unsigned w, unsigned one_bits) {
  return __uint_as_float(__byte_perm(w, one_bits, 0x7632u));
}
__device__ __forceinline__ float vhalf_lo(unsigned w, unsigned one_bits) {
  return __uint_as_float(__byte_perm(w, one_bits, 0x7610u));
}
__device__ __forceinline__ float2 vhalf_hi(uint2 w, unsigned one_bits) {
  return make_float2(vhalf_hi(w.x, one_bits), vhalf_hi(w.y, one_bits));
}
__device__ __forceinline__ float2 vhalf_lo(uint2 w, unsigned one_bits) {
  return make_float2(vhalf_lo(w.x, one_bits), vhalf_lo(w.y, one_bits));
}
// sin / cos of an angle in [-pi, pi) (MUFU)
__device__ __forceinline__ void vsincos_full(float a, float& sn, float& cs) { __sincosf(a, &sn, &cs); }
__device__ __forceinline__ void vsincos_full(float2 a, float2& sn, float2& cs) {
  __sincosf(a.x, &sn.x, &cs.x);
  __sincosf(a.y, &sn.y, &cs.y);
}

template <class T, class WD>
__device__ __forceinline__ void roll3_core(const F32Params& P, T x0, T x1, T x2, WD word,
                                           unsigned one_bits, T& s2_out, T& n0, T& n1, T& n2) {
  const T p0 = vmul(x0, x0), p1 = vmul(x1, x1), p2 = vmul(x2, x2);
  const T s2 = vfma(x2, x2, vfma(x1, x1, p0));
  s2_out = s2;
  const T aa = vfma(p0, P.Kd[0], vfma(p1, P.Kd[1], vmul(p2, P.Kd[2])));
  // clamped: a walk at the exact centre (x = 0) keeps finite terms
  const T iaa = vrsq(vmaxs(aa, 1e-30f));
  // max chain: the largest centred whitened ball, sqrt(|Ax|^2 + q) - |Ax|
  // (roll2_core's difference form and margin)
  const T q = vfma(s2, -1.0f, P.oR2);
  const T rm = vfma(vfma(vneg(aa), iaa, vsqrt(vmaxs(vadd(aa, q), 0.0f))), P.keep, -P.shrink_c);
  // rolling ball tangent at the radial projection
  const T al = vfma(vrsq(vmaxs(s2, 1e-30f)), -P.oR, 1.0f);
  const T be = vmul(iaa, P.rho_b);
  const T w0 = vmul(x0, vfma(al, P.ia[0], vmul(be, P.Ad[0])));
  const T w1 = vmul(x1, vfma(al, P.ia[1], vmul(be, P.Ad[1])));
  const T w2 = vmul(x2, vfma(al, P.ia[2], vmul(be, P.Ad[2])));
  const T d2 = vfma(w0, w0, vfma(w1, w1, vmul(w2, w2)));
  const auto roll = vand(vlt(d2, P.rho_b2), vgt(vfma(al, s2, vmul(be, aa)), 0.0f));
  const T rho = vsel(roll, P.rho_b, rm);
  // the centred ball is the d = 0 case: 1 / d masked once, axis (0, 0, 1)
  const T id = vsel(roll, vrsq(vmaxs(d2, 1e-30f)), 0.0f);
  const T d = vmul(d2, id);
  const T e0 = vmul(w0, id), e1 = vmul(w1, id), e2 = vsel(roll, vmul(w2, id), 1.0f);
  const T m = vfma(vneg(d2), id, rho);  // rho - d
  // V2 = 2V from the high half-word, azimuth from the low one
  const T v2 = vadd(vfma(vhalf_hi(word, one_bits), 256.0f, -256.0f), 1.52587890625e-05f);
  const T g = vmul(m, vrcp(vfma(d, v2, m)));
  const T gg = vmul(g, g), tt = vmul(vfma(v2, -1.0f, 2.0f), vfma(vmul(d, 0.5f), v2, rho));
  const T dep = vmul(gg, tt);
  const T tr = vsqrt(vmaxs(vmul(dep, vfma(rho, 2.0f, vneg(dep))), 0.0f));
  T sn, cs;
  vsincos_full(vfma(vhalf_lo(word, one_bits), kAngScale, kAngBias), sn, cs);
  const T tc = vmul(tr, cs), ts = vmul(tr, sn);
  // Duff et al.: (b1, b2, e) orthonormal, branch-free
  const T sg = vsign1(e2);
  const T A = vneg(vrcp(vadd(sg, e2)));
  const T B = vmul(vmul(e0, e1), A);
  const T b10 = vfma(vmul(vmul(sg, e0), e0), A, 1.0f), b11 = vmul(sg, B), b12 = vneg(vmul(sg, e0));
  const T b21 = vfma(vmul(e1, e1), A, sg), b22 = vneg(e1);
  const T h = vfma(vneg(gg), tt, m);  // m - depth
  n0 = vfma(vfma(h, e0, vfma(tc, b10, vmul(ts, B))), P.Ad[0], x0);
  n1 = vfma(vfma(h, e1, vfma(tc, b11, vmul(ts, b21))), P.Ad[1], x1);
  n2 = vfma(vfma(h, e2, vfma(tc, b12, vmul(ts, b22))), P.Ad[2], x2);
}

__device__ __forceinline__ float roll_step3(const F32Params& P, const float* x, unsigned word,
                                            unsigned one_bits, float* nx) {
  float s2;
  roll3_core<float, unsigned>(P, x[0], x[1], x[2], word, one_bits, s2, nx[0], nx[1], nx[2]);
  return __saturatef(fmaf(s2, -P.s2_scale, P.s2_bias));
}

// ---- walking predicates of the tangent / rolling chains (one-walk kernel) ----
// The stop tests as compares on the same thresholds the FFMA.SAT masks encode
// (s2_lo < |x|^2 < s2_hi; |xt_i| < tsb_i), as in the packed kernel.
template <int NH>
__device__ __forceinline__ bool roll2_go(const F32Params& P, const float* x, unsigned word,
                                         unsigned one_bits, float* nx) {
#if EM_ROLL2_GENERIC
  float s2;
  roll2_core<NH, float, unsigned>(P, x[0], x[1], word, one_bits, s2, nx[0], nx[1]);
  return NH == 1 ? (s2 < P.s2_hi) & (s2 > P.s2_lo) : s2 < P.s2_hi;
#else
  return roll_step2_legacy<NH>(P, x, word, one_bits, nx) != 0.0f;
#endif
}
__device__ __forceinline__ bool roll3_go(const F32Params& P, const float* x, unsigned word,
                                         unsigned one_bits, float* nx) {
  float s2;
  roll3_core<float, unsigned>(P, x[0], x[1], x[2], word, one_bits, s2, nx[0], nx[1], nx[2]);
  return s2 < P.s2_hi;
}
__device__ __forceinline__ bool tang2_go(const F32Params& P, const float* x, unsigned word,
                                         unsigned one_bits, float* nx) {
  float a0, a1;
  tang2_core<float, unsigned>(P, x[0], x[1], word, one_bits, a0, a1, nx[0], nx[1]);
  return (a0 < P.tsb[0]) & (a1 < P.tsb[1]);
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

}  // namespace f32
}  // namespace em
