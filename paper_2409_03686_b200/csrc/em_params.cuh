// em_params.cuh -- kernel parameter blocks shared by the REF64 mirror and the
// FP32 production kernels, and the host-side plan that owns their buffers.
#pragma once
#include <stdint.h>

#include "../../include/exitmeasure_b200.h"
#include "em_rng.cuh"

// EM_DEBUG=1 (the debug library, build_native.build(debug=True)) turns on
// device-side bounds checks on every count-row write and work hand-out; a
// failed check prints its location and traps (the launch then fails with a
// CUDA error instead of writing out of bounds).  Off in the production build.
#ifndef EM_DEBUG
#define EM_DEBUG 0
#endif
#if EM_DEBUG
#include <cstdio>
#define EM_DEV_ASSERT(c)                                                      \
  do {                                                                        \
    if (!(c)) {                                                               \
      printf("EM_DEV_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      __trap();                                                               \
    }                                                                         \
  } while (0)
#else
#define EM_DEV_ASSERT(c) \
  do {                   \
  } while (0)
#endif

namespace em {

constexpr int kMaxBlk = 16;         // structured anchor blocks per side
constexpr int kBisMax = 16384;      // circle blocks binned by boundary table
constexpr int kMaxComp = EM_MAX_HOLES + 2;
constexpr int kGfMax = 4 + 4 * EM_MAX_HOLES + 2;

enum BlkKind { BLK_GENERIC = 0, BLK_CIRCLE = 1, BLK_SQUARE = 2 };
enum Outer { OUTER_BALL = 0, OUTER_BOX = 1, OUTER_LBOX = 2 };

// Candidate grid for unstructured anchor families (FP32 path).  cell word =
// offset << 8 | count; count 255 = brute force over the whole family.
struct Grid32 {
  float lo[3];
  float inv_h;
  int n[3];
  const unsigned* cell;
  const unsigned* cand;
  const float4* candv;  // the same lists as coordinates, anchor index in .w (bits)
};

struct Side64 {
  int n_anchors, n_blk, wkind;
  int kind[kMaxBlk];
  long long start[kMaxBlk], count[kMaxBlk];
  double cx[kMaxBlk], cy[kMaxBlk], radius[kMaxBlk], phase[kMaxBlk];
  const double* anchors;
};

struct Side32 {
  int n_anchors, n_blk;
  int kind[kMaxBlk];
  int start[kMaxBlk], count[kMaxBlk];
  float cx[kMaxBlk], cy[kMaxBlk], cz[kMaxBlk], radius[kMaxBlk], phase[kMaxBlk];
  float scale[kMaxBlk];  // circle: count/2pi, square: count/8h
  const float4* anchors;
  // one uniform circle block (BIN_CIRCLE binner, count <= kBisMax): unit
  // directions of the Voronoi boundaries, bis[k] between anchors k-1 and k
  const float2* bis;
  int has_grid;
  Grid32 grid;
};

// Work distribution and outputs common to every walk kernel.
struct WorkOut {
  long long n_poles, rep_start, n_rep, total;  // total = n_poles * n_rep
  long long rb;                                // replicates per chunk
  unsigned long long n_chunks;                 // n_poles * ceil(n_rep / rb)
  double inv_poles;                            // 1/n_poles for chunk -> (block, pole)
  const long long* pole_ids;                   // RNG pole index per row
  unsigned long long* ticket;                  // global chunk counter
  unsigned long long* counts;                  // (n_poles, row_len)
  int row_len, col_off1;                       // side-1 column offset
  int smem_stats;                              // per-block shared stats table (n_poles <= 1024)
  // > 1: ssum/ssq/smax are rows of a (stat_copies, 3, n_poles) scratch, each
  // warp flushes into copy (warp + lane) mod stat_copies, and a second kernel
  // folds the copies (spreads the flush atomics when many warps share a pole)
  int stat_copies;
  // pole-block scheduler (walk_f32_kernel SMEM == 2): block b walks pole
  // b / splits, replicates [(b % splits) * bc, + bc), into a shared-memory
  // histogram of the row flushed once per block
  long long bc, splits;
  unsigned long long *ssum, *ssq, *smax;
  // first failing walk as ~(pole * n_rep + rep) under atomicMax: a zero-filled
  // output block means "no failure" and the smallest key wins
  unsigned long long* err_key;
  // exits mode (em_run_exits / walk_exits_chunk)
  double* x_out;
  long long* steps_out;
  long long* comp_out;
};

struct Ref64Params {
  int d, outer_kind, n_holes, n_notch;
  double gf[kGfMax];
  signed char comp_side[kMaxComp];
  double ks[9];
  double eps;
  long long max_steps;
  unsigned long long seed;
  unsigned long long rk0[10];  // seed + r W0: Philox4x64 round keys (key word 1 is 0)
  const double* poles;  // (n_poles, d)
  Side64 side[2];
  WorkOut w;
};

struct F32Params {
  int n_holes, has_notch;
  int concentric;  // every hole shares the outer ball's centre (annulus, shell)
  // The kernel works in a frame where the outer ball's / box's centre is the
  // origin (saves the per-step x - c); world = frame + offset.
  float frame[3];
  float oR;      // ball outer: radius
  float bhi[3];  // box / L-box outer: half-widths (the box is [-bhi, bhi] in the frame)
  float hc[EM_MAX_HOLES][3], hr[EM_MAX_HOLES];  // hole centres in the frame
  float hr2[EM_MAX_HOLES];                      // hole radii squared
  float notch[2];                               // notch corner in the frame
  signed char comp_side[kMaxComp];
  // Ball domains (rot = 1): the frame is also rotated onto the eigenbasis of
  // A = K^{1/2} (A = Q diag(Ad) Q^T, world = frame + Q x).  Balls are
  // rotation invariant and a uniform direction stays uniform, so the step is
  // y = diag(Ad) u and |Av|^2 = sum Kd_i v_i^2 (3D: 11 -> 5 ops for y, 9 -> 4
  // for the quadratic form).
  int rot;
  float Q[9];       // row-major 3x3 (d x d block used)
  float Ad[3], Kd[3];
  // Box / L-box on the max chain without holes (shear = 1): a uniform
  // direction u is uniform in ANY orthonormal frame, so it is drawn in the
  // frame (e1, e2, e3) where row a_0 of A is R_0 e3 and row a_1 lies in the
  // (e1, e3) plane (2D: u = (c, s) with a_0 = R_0 e1).  With the axes stored
  // sheared, xs_i = x_i / ax_i, the step x += r A u becomes
  //   2D: xs_0 += r c,  xs_1 += r (k c + s)                       (3 FFMA)
  //   3D: xs_0 += r z,  xs_1 += r (rc + k1 z),
  //       xs_2 += r (rs + k2 rc + k3 z)    (rc, rs = rho cos, rho sin; 8 ops)
  // instead of the d x d product and d updates (2D 6 ops, 3D 14).  The face
  // bound of axis i is r_i = m_i / R_i = g_i * (sheared distance), g_i =
  // |ax_i| / R_i; the notch (world axes) keeps its world-unit bounds.
  int shear;
  float ax[3];      // frame coordinate = ax_i * kernel coordinate
  float sb[3];      // stop thresholds: s_i = sb_i - |xs_i| <= 0  <=>  face distance <= eps
  float sg[3];      // bound gain (keep folded in, rounded down): r_i = s_i sg_i + sc_i
  float sc[3];      // bound offset (rounded down)
  float shk[3];     // 2D: k = cot(d_1 - d_0); 3D: k1, k2, k3
  // 2D box on the tangent-ball chain (tangent = 1): axis i stored as
  // xt_i = x_i / R_i (R_i = |row i of A|), i.e. the whitened point's
  // coordinate along the unit face normal: the whitened face distances are
  // bt_i - |xt_i| (ax[] holds R_i for the way back)
  int tangent;
  float tbt[3];     // whitened half-widths bhi / R_i
  float tsb[3];     // stop thresholds bt_i - eps / R_i (<= 0 margin: face within eps)
  float tcd, tsd;   // cos, sin of the angle between the two face normals (sin > 0)
  float tim, tip;   // 1 / (1 - cD), 1 / (1 + cD)
  float tkeep, tsa; // ball radius shrink: rho keep - sa
  // 3D box / L-box on the tangent-ball chain: per nearest face i one row of
  // kTanRow floats (copied to shared memory per block, indexed per lane):
  //   C[3]  = a_i . a_l (whitened face-normal cosines, C[i] = 1)
  //   P1[3], P2[3] = a_l . e1, a_l . e2 (orthonormal tangent frame of face i)
  //   Bm[3] = bt_l / (1 - C_il) (l == i: +huge), tim[3] = 1 / (1 - C_il) (l == i: 0)
  //   Bp[3] = bt_l / (1 + C_il),                 tip[3] = 1 / (1 + C_il)
  // padded to 24 floats (six float4) per row
  float t3[3][24];
  float tn[2];      // L-box: notch planes in stored coordinates, notch_q / R_q
  // 3D ball on the tangent chain (rolling balls, rotated frame A = diag(Ad)):
  // whitened balls of radius rho_b (<= the smallest curvature radius of the
  // whitened ellipsoid, R min(Ad) / max(Ad)^2) roll freely inside it
  float rho_b, rho_b2;
  float rho_h, rho_h2;  // 2D concentric annulus: disks tangent to the hole from outside
  float mid2;           // ((R + rho) / 2)^2: which boundary's disk a step tries (EM_ROLL2_ONE)
  // roll2_core's blends and centred radius: rc_d = rho_b - rho_h with
  // fl(rho_h + rc_d) == rho_b exactly, nr_d = hr - R, im2 = 1 / m2 (rounded
  // down), shrink_c = shrink_abs + the error bound of the difference forms
  float rc_d, nr_d, im2, shrink_c;
  // EM_ROLL2_DYN: per-step radii (R - rho)(1 - 1e-6) / (max Ad + |diag(Ad) n|)
  float rb_bl, gap, amax, K4[3];
  float ia[3];      // 1 / Ad
  float ss_scale;   // stop mask sat(min_i s_i * ss_scale) (power of two)
  float A[9];       // K^{1/2}, row-major
  float Kq[6];      // K = A^T A as (K00, K11, K22, 2 K01, 2 K02, 2 K12): |Av|^2 = v^T K v
  float g[3];       // 1/|A e_i|: face-plane gain of the maximal ellipsoid
  float gk[3];      // g * keep (rounded down): face gain with the relative margin folded in
  float m2;         // sigma_min(A)^2 (hole bound)
  float eps;
  float eps2;  // eps^2 (the L-box notch stop test compares squared distances)
  float stop_scale, stop_bias;   // FFMA.SAT stop test: sat(e * scale + bias) = [e > eps]
  float oR2, s2_scale, s2_bias;  // ball: R^2 and sat(-|x|^2 s + b) = [|x|^2 < (R - eps)^2]
  float h2_scale, h2_bias;       // concentric hole: sat(|x|^2 s + b) = [|x|^2 > (rho + eps)^2]
  // the same two thresholds as plain numbers (the two-walks-per-lane kernel
  // tests them with compares): walking <=> s2_lo < |x|^2 < s2_hi
  float s2_hi, s2_lo;
  float shrink_rel, shrink_abs;  // step safety margins
  float keep;                    // 1 - shrink_rel
  unsigned one_bits;             // 0x3f800000 (1.0f), opaque to the compiler: PRMT operand
  int max_steps;
  unsigned key0, key1;
  PhiloxKey32 rk;   // round keys of (key0, key1), set per run on the host
  const float4* poles;
  Side32 side[2];
  WorkOut w;
};

}  // namespace em
