// plan_f32.cu -- host-side constants of the FP32 walk kernel for one
// geometry (F32Params, em_params.cuh), split by what they serve: the kernel
// frame, the rolling balls / disks of the tangent chain on balls, the
// sheared axes of the max chain on boxes, the whitened face tables of the
// tangent chain on boxes / the L-box, the domain (holes, notch, conductivity
// forms), the stop thresholds and the FP32 safety margins.  capi.cu's
// em_plan_create calls build_f32_constants; em_f32_constant exposes single
// constants to the host unit tests (tests/test_plan_constants.py, no GPU).
// Every formula is a closed form of the plan's geometry; DESIGN.md §3.1
// derives each one.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "em_params.cuh"

namespace em {

// Cyclic Jacobi eigendecomposition of a symmetric d x d matrix (d <= 3):
// eigenvalues in lam, eigenvectors as the COLUMNS of v (a = v diag(lam) v^T).
void sym_eig(const double* a_in, int d, double lam[3], double v[3][3]) {
  double a[3][3] = {{0}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) v[i][j] = i == j ? 1.0 : 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) a[i][j] = a_in[i * d + j];
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) off += a[p][q] * a[p][q];
    if (off < 1e-32) break;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) {
        if (a[p][q] == 0.0) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < d; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < d; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < d; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 3; ++i) lam[i] = i < d ? a[i][i] : 0.0;
}

double sym_min_eig(const double* a_in, int d) {
  double lam[3], v[3][3];
  sym_eig(a_in, d, lam, v);
  double m = lam[0];
  for (int i = 1; i < d; ++i) m = std::min(m, lam[i]);
  return m;
}

// Shared state of one build: the geometry, the chain, and the frame the
// kernel stores points in (world = frame + Q x for rotated balls, frame +
// diag(ax) x for scaled box axes).
struct F32Build {
  const em_geometry* g;
  int d, nh, nn, chain;
  bool ident;
  double eps;
  const double* gf;
  F32Params& P;
  double frame[3] = {0.0, 0.0, 0.0};
  double scale = 1.0;
  double roll_S = 0.0;  // rolling chains: bound of |Ax| and of the roots of the centred radius
  double Qd[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
  double Adiag[3] = {1.0, 1.0, 1.0};
  double axd[3] = {1.0, 1.0, 1.0}, shear_g[3] = {1.0, 1.0, 1.0};
  double tcd = 0.0;
  double tah[3][3] = {{0.0}};  // unit whitened face normals a_i (rows of A / R_i)
  F32Build(const em_geometry* g_, int chain_, bool ident_, double eps_, F32Params& P_)
      : g(g_), d((int)g_->gi[0]), nh((int)g_->gi[2]), nn(g_->gi_len >= 4 ? (int)g_->gi[3] : 0),
        chain(chain_), ident(ident_), eps(eps_), gf(g_->gf), P(P_) {}

  // world point -> kernel coordinates
  void to_kernel(const double* w, float* out) const {
    double v[3] = {0.0, 0.0, 0.0};
    for (int j = 0; j < d; ++j) v[j] = w[j] - frame[j];
    for (int j = 0; j < d; ++j) {
      double t = 0.0;
      if (P.rot) {
        for (int i = 0; i < d; ++i) t += Qd[i][j] * v[i];
      } else {
        t = v[j] / axd[j];
      }
      out[j] = (float)t;
    }
  }

  // kernel frame (origin at the ball's / box's centre) and which
  // reformulation of the step the kernel runs: rotated ball frame, sheared
  // box axes, tangent chain
  void frame_and_chain() {
    if (g->gi[1] == 0) {
      for (int j = 0; j < d; ++j) frame[j] = gf[j];
      P.oR = (float)gf[d];
      scale = std::max(scale, gf[d]);
    } else {
      for (int j = 0; j < d; ++j) {
        frame[j] = gf[j];
        P.bhi[j] = (float)gf[d];
      }
      scale = std::max(scale, gf[d]);
    }
    for (int j = 0; j < 3; ++j) P.frame[j] = (float)frame[j];
    // Ball domains: rotate the frame onto the eigenbasis of A = K^{1/2}
    // (A = Q diag(Ad) Q^T).  Box / L-box on the max chain: sheared axes (see
    // F32Params::shear).  Both are exact reformulations of the same step.
    P.rot = (g->gi[1] == 0 && nn == 0 && !ident) ? 1 : 0;
    P.shear = (g->gi[1] == 1 && nh == 0 && chain == EM_CHAIN_MAX && !ident && (d == 3 || nn == 0)) ? 1 : 0;
    P.tangent = chain == EM_CHAIN_TANGENT ? 1 : 0;
    if (P.rot) sym_eig(g->ksqrt, d, Adiag, Qd);
  }

  // tangent chain on balls: rolling balls / disks of the whitened ellipse's
  // smallest curvature radius, and disks tangent to a concentric hole
  void rolling() {
    if (P.rot && P.tangent) {
      // rolling-ball radius: the whitened ellipsoid {z : |diag(Ad) z| <= R}
      // has semi-axes R / Ad_i and smallest curvature radius R min / max^2
      double amin = Adiag[0], amax = Adiag[0];
      for (int i = 1; i < d; ++i) {
        amin = std::min(amin, Adiag[i]);
        amax = std::max(amax, Adiag[i]);
      }
      double rb = gf[d] * amin / (amax * amax);
      if (nh == 1) {
        // annulus: every point y of a disk of radius r tangent at p has
        // | |x_y| - |x_p| | <= 2 r max(Ad), so r = (R - rho) / (2 max Ad)
        // keeps the outer disks off the hole and the hole's disks inside R
        const double lim = (gf[d] - gf[d + 1 + d]) / (2.0 * amax);
        P.rb_bl = (float)(gf[d] * amin / (amax * amax) * (1.0 - 1e-6));
        P.gap = (float)((gf[d] - gf[d + 1 + d]) * (1.0 - 1e-6));
        P.amax = (float)amax;
        for (int i = 0; i < d; ++i) P.K4[i] = (float)(Adiag[i] * Adiag[i] * Adiag[i] * Adiag[i]);
        rb = std::min(rb, lim);
        P.rho_h = (float)(lim * (1.0 - 1e-6));
        P.rho_h2 = (float)((double)P.rho_h * (double)P.rho_h);
      }
      rb *= 1.0 - 1e-6;
      P.rho_b = (float)rb;
      if (nh == 1 && d == 2) {
        // roll2_core blends the radius as fl(rho_h + of rc_d), of in {0, 1}:
        // round rho_b down to a value that sum reproduces exactly
        float dd = P.rho_b - P.rho_h;  // <= 0
        while (P.rho_h + dd > P.rho_b) dd = std::nextafter(dd, -1.0e30f);
        P.rc_d = dd;
        P.rho_b = P.rho_h + dd;
        P.nr_d = (float)gf[d + 1 + d] - (float)gf[d];
      }
      P.rho_b2 = (float)((double)P.rho_b * (double)P.rho_b);
      roll_S = std::max(amax, 1.0) * gf[d];
      for (int i = 0; i < d; ++i) P.ia[i] = (float)(1.0 / Adiag[i]);
    }
  }

  // rotated ball frame: A = Q diag(Ad) Q^T
  void ball_axes() {
    for (int i = 0; i < 3; ++i) {
      P.Ad[i] = (float)Adiag[i];
      P.Kd[i] = (float)(Adiag[i] * Adiag[i]);
      for (int j = 0; j < 3; ++j) P.Q[3 * i + j] = (float)Qd[i][j];
    }
  }

  // max chain on boxes: the sheared axes (F32Params::shear)
  void shear_axes() {
    if (P.shear) {
      const double* A = g->ksqrt;  // d x d, symmetric, rows a_i
      double Rn[3] = {0.0, 0.0, 0.0}, ah[3][3] = {{0.0}};
      for (int i = 0; i < d; ++i) {
        for (int j = 0; j < d; ++j) Rn[i] += A[i * d + j] * A[i * d + j];
        Rn[i] = std::sqrt(Rn[i]);
        for (int j = 0; j < d; ++j) ah[i][j] = A[i * d + j] / Rn[i];
      }
      if (d == 2) {
        // u = (c, s) in the frame where a_0 = R_0 e1: a_1 = R_1 (cos D, sin D)
        const double dD = std::atan2(ah[1][1], ah[1][0]) - std::atan2(ah[0][1], ah[0][0]);
        axd[0] = Rn[0];
        axd[1] = Rn[1] * std::sin(dD);
        P.shk[0] = (float)(std::cos(dD) / std::sin(dD));
      } else {
        // e3 = a_0 / R_0, e1 = the unit part of a_1 orthogonal to e3, e2 = e3 x e1
        double e1[3], e2[3], e3[3];
        for (int j = 0; j < 3; ++j) e3[j] = ah[0][j];
        const double cb = ah[1][0] * e3[0] + ah[1][1] * e3[1] + ah[1][2] * e3[2];
        for (int j = 0; j < 3; ++j) e1[j] = ah[1][j] - cb * e3[j];
        const double sbt = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
        for (int j = 0; j < 3; ++j) e1[j] /= sbt;
        e2[0] = e3[1] * e1[2] - e3[2] * e1[1];
        e2[1] = e3[2] * e1[0] - e3[0] * e1[2];
        e2[2] = e3[0] * e1[1] - e3[1] * e1[0];
        double gm[3] = {0.0, 0.0, 0.0};
        for (int j = 0; j < 3; ++j) {
          gm[0] += ah[2][j] * e1[j];
          gm[1] += ah[2][j] * e2[j];
          gm[2] += ah[2][j] * e3[j];
        }
        axd[0] = Rn[0];
        axd[1] = Rn[1] * sbt;
        axd[2] = Rn[2] * gm[1];
        P.shk[0] = (float)(cb / sbt);
        P.shk[1] = (float)(gm[0] / gm[1]);
        P.shk[2] = (float)(gm[2] / gm[1]);
      }
      for (int i = 0; i < d; ++i) shear_g[i] = std::fabs(axd[i]) / Rn[i];
    }
  }

  // tangent chain on boxes: whitened face normals, stored coordinates
  // xt_i = x_i / R_i
  void tangent_normals() {
    if (P.tangent && g->gi[1] == 1) {  // boxes (balls roll, see below)
      // xt_i = x_i / R_i: the whitened point's coordinate along face normal i
      const double* A = g->ksqrt;
      for (int i = 0; i < d; ++i) {
        double n2 = 0.0;
        for (int j = 0; j < d; ++j) n2 += A[i * d + j] * A[i * d + j];
        axd[i] = std::sqrt(n2);
        for (int j = 0; j < d; ++j) tah[i][j] = A[i * d + j] / axd[i];
      }
      if (d == 2) {
        tcd = tah[0][0] * tah[1][0] + tah[0][1] * tah[1][1];
        P.tcd = (float)tcd;
        P.tsd = (float)std::sqrt(std::max(0.0, 1.0 - tcd * tcd));
        P.tim = (float)(1.0 / (1.0 - tcd));
        P.tip = (float)(1.0 / (1.0 + tcd));
      }
    }
    for (int i = 0; i < 3; ++i) P.ax[i] = (float)axd[i];
  }

  // holes, notch, component sides, K^{1/2}, K's quadratic form, face gains
  void domain() {
    P.concentric = (g->gi[1] == 0 && nh > 0) ? 1 : 0;
    for (int h = 0; h < nh; ++h) {
      const int off = d + 1 + h * (d + 1);
      to_kernel(gf + off, P.hc[h]);
      for (int j = 0; j < d; ++j) {
        if (gf[off + j] != gf[j]) P.concentric = 0;
      }
      P.hr[h] = (float)gf[off + d];
      P.hr2[h] = (float)(gf[off + d] * gf[off + d]);
    }
    if (g->gi[1] == 0 && nh == 1) {  // owner / candidate-disk split of a shell
      const double mid = 0.5 * (gf[d] + gf[d + 1 + d]);
      P.mid2 = (float)(mid * mid);
    }
    if (nn) {
      const int off = (d + 1) * (1 + nh);
      P.notch[0] = (float)(gf[off] - frame[0]);
      P.notch[1] = (float)(gf[off + 1] - frame[1]);
    }
    for (int c = 0; c < 1 + nh + nn; ++c) P.comp_side[c] = g->comp_side[c];
    for (int i = 0; i < d * d; ++i) P.A[i] = (float)g->ksqrt[i];
    {
      double K[3][3] = {{0.0}};
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
          for (int k = 0; k < d; ++k) K[i][j] += g->ksqrt[k * d + i] * g->ksqrt[k * d + j];
      P.Kq[0] = (float)K[0][0];
      P.Kq[1] = (float)K[1][1];
      P.Kq[2] = (float)K[2][2];
      P.Kq[3] = (float)(2.0 * K[0][1]);
      P.Kq[4] = (float)(2.0 * K[0][2]);
      P.Kq[5] = (float)(2.0 * K[1][2]);
    }
    for (int i = 0; i < d; ++i) {
      double n2 = 0.0;
      for (int k = 0; k < d; ++k) n2 += g->ksqrt[k * d + i] * g->ksqrt[k * d + i];
      // 1/|A e_i|, rounded down so the face bound stays a lower bound
      P.g[i] = (float)(1.0 / std::sqrt(n2) * (1.0 - 1e-6));
    }
  }

  // Euclidean stop tests as saturating FFMAs (sat(m) = [e > eps])
  void stops() {
    const double lam = sym_min_eig(g->ksqrt, d);
    P.m2 = (float)(std::max(0.0, lam) * std::max(0.0, lam) * (1.0 - 1e-4));
    P.eps = (float)eps;
    P.eps2 = (float)((double)P.eps * (double)P.eps);
    {
      // scale = 2^k with ulp(eps_f) * 2^k >= 1: every representable e > eps
      // then gives (e - eps) * scale >= 1 (bias = -eps * scale is exact)
      int ex = 0;
      std::frexp((double)P.eps, &ex);  // eps_f in [2^(ex-1), 2^ex)
      const int k = 24 - (ex - 1) + 1;  // ulp(eps_f) = 2^(ex-1-23)
      P.stop_scale = std::ldexp(1.0f, k);
      P.stop_bias = -P.eps * P.stop_scale;
    }
    if (g->gi[1] == 0) P.oR2 = (float)(gf[d] * gf[d]);
    if (g->gi[1] == 0) {
      // ball stop on |x|^2: c = fl32((R - eps)^2); for |x|^2 < c the exact
      // difference c - |x|^2 is >= ulp(c) / 2 (Sterbenz near c, larger
      // below), so a power-of-two scale 2^k >= 2 / ulp(c) maps it to >= 1
      // and the FFMA (exact product, one rounding) keeps its sign
      const double R = gf[d];
      P.oR2 = (float)(R * R);
      const float c = (float)((R - eps) * (R - eps));
      int ex = 0;
      std::frexp((double)c, &ex);  // c in [2^(ex-1), 2^ex)
      const int k = 24 - (ex - 1) + 2;
      P.s2_scale = std::ldexp(1.0f, k);
      P.s2_bias = c * P.s2_scale;
      P.s2_hi = c;
      P.s2_lo = -1.0f;  // no hole: |x|^2 >= 0 always passes
      if (nh >= 1) {
        // concentric hole: the same construction for |x|^2 > (rho + eps)^2
        const double rho = gf[d + 1 + d];
        const float ch = (float)((rho + eps) * (rho + eps));
        std::frexp((double)ch, &ex);
        const int kh = 24 - (ex - 1) + 2;
        P.h2_scale = std::ldexp(1.0f, kh);
        P.h2_bias = -ch * P.h2_scale;
        P.s2_lo = ch;
      }
    }
  }

  // FP32 safety margins of the step scale
  void margins() {
    P.shrink_rel = 4.0e-6f;
    P.shrink_abs = (float)(scale * 1.1920928955078125e-07);
    P.keep = 1.0f - P.shrink_rel;
    // the centred radius of roll2_core as a difference of two terms <= roll_S,
    // each within ~2e-7 relative (rsqrt.approx / sqrt.approx bounds, the
    // rounding of their arguments), times 1 / m2 on the hole's side
    P.im2 = P.m2 > 0.0f ? std::nextafter(1.0f / P.m2, 0.0f) : 0.0f;
    P.shrink_c = P.shrink_abs + (float)(5.0e-7 * roll_S * std::max(1.0, (double)P.im2));
    for (int i = 0; i < 3; ++i)  // rounded down: the folded margin is never smaller
      P.gk[i] = std::nextafter((float)((double)P.g[i] * (double)P.keep), 0.0f);
  }

  // max chain on boxes: stop thresholds and bound gains of the sheared axes
  void shear_thresholds() {
    if (P.shear) {
      // sheared box: kernel box [-bs_i, bs_i]; face i within eps <=> s_i =
      // sb_i - |xs_i| <= 0 with sb_i = bs_i - eps / |ax_i|; bound r_i = m_i /
      // R_i = g_i (s_i + (bs_i - sb_i)), shrunk by keep and by an absolute
      // margin of a few ulps of the kernel box
      double bsmax = 1.0;
      float sbmin = 0.0f;
      for (int i = 0; i < d; ++i) {
        const float bs = (float)(gf[d] / std::fabs(axd[i]));
        bsmax = std::max(bsmax, (double)bs);
        P.sb[i] = (float)((double)bs - eps / std::fabs(axd[i]));
        sbmin = i == 0 ? P.sb[i] : std::min(sbmin, P.sb[i]);
      }
      const double sa = bsmax * 1.1920928955078125e-07;
      for (int i = 0; i < d; ++i) {
        const float bs = (float)(gf[d] / std::fabs(axd[i]));
        const double gk = shear_g[i] * (double)P.keep;
        P.sg[i] = std::nextafter((float)gk, 0.0f);
        const double off = gk * ((double)bs - (double)P.sb[i]) - shear_g[i] * sa;
        float c = (float)off;
        if ((double)c > off) c = std::nextafter(c, -1.0f);
        P.sc[i] = c;
      }
      // every positive s is >= ulp(sb_min) / 2 (Sterbenz near sb, larger
      // below): a power-of-two scale 2^k >= 2 / ulp(sb_min) maps it to >= 1
      // (the tangent chain below uses the same construction)
      int ex = 0;
      std::frexp((double)sbmin, &ex);  // sb in [2^(ex-1), 2^ex), ulp = 2^(ex-24)
      P.ss_scale = std::ldexp(1.0f, 25 - ex + 1);
    }
  }

  // tangent chain on boxes / the L-box: whitened half-widths, stop
  // thresholds, the per-face tables t3 and the notch planes
  void tangent_box() {
    if (P.tangent && g->gi[1] == 1) {  // boxes (balls roll, see below)
      // whitened half-widths and stop thresholds; the ball radius is shrunk
      // by keep and by a few ulps of the whitened box (coordinate rounding)
      float sbmin = 0.0f;
      double btmax = 1.0, gain = 1.0;
      for (int i = 0; i < d; ++i) {
        P.tbt[i] = (float)(gf[d] / axd[i]);
        P.tsb[i] = (float)((double)P.tbt[i] - eps / axd[i]);
        sbmin = i == 0 ? P.tsb[i] : std::min(sbmin, P.tsb[i]);
        btmax = std::max(btmax, (double)P.tbt[i]);
      }
      if (d == 3) {
        // per nearest face i: cosines, tangent frame, face-limit gains (see
        // F32Params::t3); the frame of face i: e1 = the unit part of a_j
        // (j = i + 1) orthogonal to a_i, e2 = a_i x e1
        for (int i = 0; i < 3; ++i) {
          float* T = P.t3[i];
          for (int k = 0; k < 24; ++k) T[k] = 0.0f;
          const int j = (i + 1) % 3;
          double C[3], e1[3], e2[3];
          for (int l = 0; l < 3; ++l)
            C[l] = tah[i][0] * tah[l][0] + tah[i][1] * tah[l][1] + tah[i][2] * tah[l][2];
          C[i] = 1.0;
          for (int k = 0; k < 3; ++k) e1[k] = tah[j][k] - C[j] * tah[i][k];
          const double en = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
          for (int k = 0; k < 3; ++k) e1[k] /= en;
          e2[0] = tah[i][1] * e1[2] - tah[i][2] * e1[1];
          e2[1] = tah[i][2] * e1[0] - tah[i][0] * e1[2];
          e2[2] = tah[i][0] * e1[1] - tah[i][1] * e1[0];
          for (int l = 0; l < 3; ++l) {
            const double bt = (double)P.tbt[l];
            T[l] = (float)C[l];
            if (l != i) {
              T[3 + l] = (float)(tah[l][0] * e1[0] + tah[l][1] * e1[1] + tah[l][2] * e1[2]);
              T[6 + l] = (float)(tah[l][0] * e2[0] + tah[l][1] * e2[1] + tah[l][2] * e2[2]);
              T[9 + l] = (float)(bt / (1.0 - C[l]));
              T[12 + l] = (float)(1.0 / (1.0 - C[l]));
              gain = std::max(gain, 1.0 / (1.0 - std::fabs(C[l])));
            } else {
              T[9 + l] = 3.0e38f;  // no limit from face +bt_i (the tangent face)
              T[12 + l] = 0.0f;
            }
            T[15 + l] = (float)(bt / (1.0 + C[l]));
            T[18 + l] = (float)(1.0 / (1.0 + C[l]));
          }
        }
        if (nn) {
          const int off = (d + 1) * (1 + nh);
          P.tn[0] = (float)((gf[off] - frame[0]) / axd[0]);
          P.tn[1] = (float)((gf[off + 1] - frame[1]) / axd[1]);
        }
      } else {
        gain = std::max(1.0 / (1.0 - std::fabs(tcd)), 1.0);
      }
      int ex = 0;
      std::frexp((double)sbmin, &ex);
      P.ss_scale = std::ldexp(1.0f, 25 - ex + 1);
      P.tkeep = P.keep;
      // a few ulps of the whitened box per coordinate, amplified by the
      // face-limit gains 1 / (1 -+ c)
      P.tsa = (float)(btmax * 2.384185791015625e-07 * (d == 3 ? gain : 1.0));  // 2^-22
    }
  }
};

void* f32_build_new(const em_geometry* g, int chain, bool ident, double eps, int64_t max_steps,
                    F32Params& P) {
  F32Build* b = new F32Build(g, chain, ident, eps, P);
  P.n_holes = b->nh;
  P.has_notch = b->nn;
  b->frame_and_chain();
  b->rolling();
  b->ball_axes();
  b->shear_axes();
  b->tangent_normals();
  b->domain();
  b->stops();
  b->margins();
  b->shear_thresholds();
  b->tangent_box();
  P.one_bits = 0x3f800000u;
  P.max_steps = (int)std::min<int64_t>(max_steps, 2147483647LL);
  return b;
}

void f32_build_to_kernel(const void* b, const double* w, float* out) {
  static_cast<const F32Build*>(b)->to_kernel(w, out);
}

void f32_build_free(void* b) { delete static_cast<F32Build*>(b); }

}  // namespace em

// Host unit-test hook: one named constant of the FP32 kernel for geometry g
// and chain (EM_CHAIN_*, as resolved by the plan: pass the resolved chain),
// computed exactly as em_plan_create does, without a device.  Returns the
// number of floats written (<= n), or -1 for an unknown name.
extern "C" int em_f32_constant(const em_geometry* g, int chain, int ident, double eps,
                               const char* name, float* out, int n) {
  if (!g || !g->gi || !g->gf || !g->ksqrt || !name || !out || g->gi_len < 3) return -1;
  em::F32Params P{};
  em::F32Build b(g, chain, ident != 0, eps, P);
  P.n_holes = b.nh;
  P.has_notch = b.nn;
  b.frame_and_chain();
  b.rolling();
  b.ball_axes();
  b.shear_axes();
  b.tangent_normals();
  b.domain();
  b.stops();
  b.margins();
  b.shear_thresholds();
  b.tangent_box();
  struct Entry {
    const char* key;
    const float* p;
    int len;
  };
  const Entry tab[] = {
      {"t3", &P.t3[0][0], 72},   {"tbt", P.tbt, 3},         {"tsb", P.tsb, 3},
      {"tcd", &P.tcd, 1},        {"tsd", &P.tsd, 1},        {"tim", &P.tim, 1},
      {"tip", &P.tip, 1},        {"tkeep", &P.tkeep, 1},    {"tsa", &P.tsa, 1},
      {"tn", P.tn, 2},           {"rho_b", &P.rho_b, 1},    {"rho_b2", &P.rho_b2, 1},
      {"rho_h", &P.rho_h, 1},    {"rho_h2", &P.rho_h2, 1},  {"mid2", &P.mid2, 1},
      {"Ad", P.Ad, 3},           {"Kd", P.Kd, 3},           {"Q", P.Q, 9},
      {"ia", P.ia, 3},           {"ax", P.ax, 3},           {"g", P.g, 3},
      {"gk", P.gk, 3},           {"m2", &P.m2, 1},          {"sb", P.sb, 3},
      {"sg", P.sg, 3},           {"sc", P.sc, 3},           {"shk", P.shk, 3},
      {"A", P.A, 9},             {"Kq", P.Kq, 6},           {"keep", &P.keep, 1},
      {"shrink_abs", &P.shrink_abs, 1},                     {"ss_scale", &P.ss_scale, 1},
      {"stop_scale", &P.stop_scale, 1},                     {"stop_bias", &P.stop_bias, 1},
      {"s2_scale", &P.s2_scale, 1},                         {"s2_bias", &P.s2_bias, 1},
      {"h2_scale", &P.h2_scale, 1},                         {"h2_bias", &P.h2_bias, 1},
      {"s2_hi", &P.s2_hi, 1},    {"s2_lo", &P.s2_lo, 1},    {"rc_d", &P.rc_d, 1},
      {"nr_d", &P.nr_d, 1},      {"im2", &P.im2, 1},        {"shrink_c", &P.shrink_c, 1},
      {"oR2", &P.oR2, 1},        {"hr", P.hr, 1},           {"hc", &P.hc[0][0], 3},
      {"frame", P.frame, 3},     {"eps", &P.eps, 1},
  };
  for (const Entry& e : tab)
    if (std::strcmp(e.key, name) == 0) {
      const int k = std::min(e.len, n);
      for (int i = 0; i < k; ++i) out[i] = e.p[i];
      return k;
    }
  const int flags[4] = {P.rot, P.shear, P.tangent, P.concentric};
  if (std::strcmp(name, "flags") == 0) {  // rot, shear, tangent, concentric
    const int k = std::min(4, n);
    for (int i = 0; i < k; ++i) out[i] = (float)flags[i];
    return k;
  }
  return -1;
}
