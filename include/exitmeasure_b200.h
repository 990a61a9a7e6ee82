/*
 * exitmeasure_b200.h -- C ABI of the B200-native exit-measure library
 * (libexitmeasure_b200.so).  Plain pointers and sizes only; host buffers are
 * owned by the caller, device buffers by the library.
 *
 * Reference interface each entry point replaces (S/ = /root/reference/pkg/
 * src/exitmeasure/; the reference binds its kernel through Cython, the
 * ctypes binding that replaces it is paper_2409_03686_b200/_native.py and is
 * shown in INTEGRATION.md):
 *
 *   em_walk_exits_chunk   <- _kernel.walk_exits_chunk   S/_kernel.pyx:376-411
 *   em_accumulate_chunk   <- _kernel.accumulate_chunk   S/_kernel.pyx:414-464
 *   em_plan_* / em_run_accumulate
 *                         <- backend.run_accumulate     S/backend.py:147-199
 *                            (one launch for all (pole, replicate) walks
 *                            instead of a thread pool over 8192-walk chunks)
 *   em_run_exits          <- backend.run_exits          S/backend.py:202-227
 *
 * Two arithmetic paths sit behind the same entry points:
 *   EM_PREC_REF64 -- bit-exact FP64 mirror of the reference kernel: the same
 *                    Philox4x64-10 streams (key (seed,0), counter
 *                    (draw,0,replicate,pole)), Marsaglia directions, operand
 *                    order and lexicographic binning, so counts equal the
 *                    reference's exactly.
 *   EM_PREC_FP32  -- the production kernel: Philox4x32-10 streams keyed by
 *                    (seed, pole, replicate), angle-based directions, FP32
 *                    walk state, persistent lane refill and closed-form /
 *                    grid-accelerated binning.  Statistically equivalent to
 *                    the reference (same exit law), not bit-identical.
 *
 * Return codes: EM_OK, EM_BUDGET (some walk exceeded max_steps; the
 * lexicographically first (pole, replicate) is reported, outputs are then
 * meaningless -- the reference's WalkBudgetError contract, S/backend.py:
 * 189-192), or a negative error with a message from em_last_error().
 * All entry points are reentrant: each calling host thread gets its own
 * stream and workspace (the reference's thread-pool contract,
 * S/backend.py:159-178).
 */
#ifndef EXITMEASURE_B200_H
#define EXITMEASURE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EM_ABI_VERSION 1

#define EM_OK 0
#define EM_BUDGET 1
#define EM_ERR_INVALID (-1)
#define EM_ERR_CUDA (-2)
#define EM_ERR_UNSUPPORTED (-3)
#define EM_ERR_NOMEM (-4)

#define EM_PREC_REF64 0
#define EM_PREC_FP32 1

/* EM_CHAIN_WOE: the reference chain x <- x + sd(x) K^{1/2} u
 *   (S/_kernel.pyx:185-196).
 * EM_CHAIN_MAX: x <- x + r(x) K^{1/2} u with r(x) >= sd(x) a certified lower
 *   bound of the largest K^{1/2}-ellipsoid inscribed in the domain (exact for
 *   faces, closed-form bounds for balls/holes); same stopping rule sd <= eps,
 *   same exit law, fewer steps.  FP32 only. */
#define EM_CHAIN_WOE 0
#define EM_CHAIN_MAX 1
/* EM_CHAIN_TANGENT: walk on tangent balls.  In whitened coordinates (where
 *   K-diffusion is Brownian motion) each step takes a ball inside the domain
 *   that contains the current point and touches the boundary near it, and
 *   jumps to an exact sample of that ball's harmonic measure seen from the
 *   point (2D: the Moebius image of a uniform angle; 3D: the Poisson kernel,
 *   uniform in 1/|z - y|).  Boxes and the L-box: the largest ball tangent to
 *   the nearest face at the foot of the point.  Balls and the concentric
 *   annulus: balls of the whitened ellipse's smallest curvature radius
 *   tangent at the radial projection (they roll freely inside), disks
 *   tangent to the hole from outside, else the max chain's centred ball.
 *   The centred ball is the special case of a point at the centre, so every
 *   step is a valid walk-on-spheres step; near the boundary the depth
 *   contracts quadratically instead of geometrically (steps per walk cfg2
 *   15.7 -> 3.7, cfg3 18.3 -> 5.8, cfg4 35.6 -> 7.0, cfg5 39.1 -> 6.0).
 *   Same stopping rule sd <= eps, same exit law.  FP32 only, K != I; 2D / 3D
 *   boxes and the 3D L-box without holes, the 2D ball with at most one
 *   concentric hole, the 3D ball without holes; elsewhere the plan runs
 *   EM_CHAIN_MAX (em_plan_chain reports the chain in use). */
#define EM_CHAIN_TANGENT 2

#define EM_MAX_HOLES 16

/* Packed geometry: the reference's GeomPack (S/backend.py:50-54,71-83).
 *   gi = [d, outer_kind (0 ball, 1 box), n_holes (, n_notch)]
 *   gf = [outer_center(d), R|h, (hole_center(d), r)*, (nx, ny) if n_notch]
 * The optional 4th gi word is this library's extension for cfg5's L-box: a
 * quadrant prism {x >= nx, y >= ny} removed from a 3D box, boundary
 * component 1 + n_holes. */
typedef struct {
  const int64_t* gi;
  int64_t gi_len;
  const double* gf;
  int64_t gf_len;
  const int8_t* comp_side; /* side (0 gamma0 / 1 gamma1) per component */
  int64_t n_comp;
  const double* ksqrt; /* d x d row-major, normalised (lambda_max = 1) */
} em_geometry;

/* One side's weight family: the reference's SidePack (S/backend.py:57-68).
 * blk rows (kind, start, count): kind 0 generic (brute force / grid),
 * 1 uniform circle, 2 uniform square.  blkf rows (cx, cy, cz, radius|h).
 * blk_phase (NULL = all 0, the reference layout) shifts uniform anchors to
 * spacing * (k + phase) along the curve. */
typedef struct {
  const double* anchors; /* (n_anchors, d) */
  int64_t n_anchors;
  const int64_t* blk;
  const double* blkf;
  int64_t n_blk;
  int32_t wkind; /* 0 voronoi, 1 idw (fractional rows via em_plan_run_raw) */
  int32_t idw_power;
  const double* idw_radii;
  const double* blk_phase;
} em_side;

typedef struct {
  int32_t precision; /* EM_PREC_* */
  int32_t chain;     /* EM_CHAIN_* (EM_PREC_REF64 requires EM_CHAIN_WOE) */
  int32_t device;    /* CUDA ordinal */
  int32_t block;     /* threads per block, 0 = library default */
  int32_t grid;      /* persistent blocks, 0 = library default (SMs x occupancy) */
  int32_t flags;     /* EM_FLAG_* bits, 0 = none */
} em_options;

/* Run EM_CHAIN_TANGENT even when K = I (where it is normally resolved to
 * EM_CHAIN_MAX).  Then the rolling ball of a ball domain is the domain
 * itself, so one step samples the domain's Poisson kernel exactly: the
 * closed-form test of the production samplers (tests/test_gpu_closed_form.py). */
#define EM_FLAG_TANGENT_ON_IDENTITY 1
/* Scheduler of the FP32 tangent-chain kernels (counts are identical under
 * both: every walk's stream is keyed by (seed, pole, replicate) and all
 * accumulation is integer).  Pole-cycling persistent warps add every exit
 * straight into the int64 rows; the pole-block scheduler runs one block per
 * (pole, replicate range) with the row's histogram in shared memory
 * (warp-aggregated __match_any_sync adds, one flush per block).  Default:
 * pole blocks where the rows (n_poles x (n0 + n1) x 8 B) exceed 64 MiB --
 * half the L2 -- and rows are >= 1024 bins, else pole-cycling warps.  The
 * flags force one or the other (A/B measurements). */
#define EM_FLAG_PERSISTENT 2
#define EM_FLAG_POLE_BLOCKS 4
/* FP32 counts on the 2D ball's rolling-disk chain (cfg3) run TWO walks per
 * lane with packed FP32 arithmetic (FFMA2 / FMUL2 / FADD2: one issued
 * instruction per pair of operations; walk_f32x2.cu).  Same walks, same
 * streams, same operation tree: the counts equal the one-walk-per-lane
 * kernel's bit for bit.  This flag forces the one-walk-per-lane kernel
 * (A/B measurements, the equality test). */
#define EM_FLAG_ONE_WALK_PER_LANE 8
/* By default the packed kernel runs where it exists once a run has >= 2e6
 * walks (smaller jobs restart its two slots per lane less evenly and run the
 * one-walk kernel).  This flag runs it at every size (tests). */
#define EM_FLAG_TWO_WALKS_PER_LANE 16

/* Per-run outputs.  Host pointers for em_plan_run / em_run_accumulate,
 * device pointers for em_plan_run_device.  counts is (n_poles, n0 + n1)
 * int64, side-0 columns first. */
typedef struct {
  int64_t* counts;
  int64_t* steps_sum; /* (n_poles,) */
  int64_t* steps_sq;
  int64_t* steps_max;
  int64_t err_pole; /* set when EM_BUDGET (pole position in the plan) */
  int64_t err_rep;
} em_outputs;

typedef struct em_plan em_plan;

int em_abi_version(void);
/* Every compile-time knob the loaded library was built with, as one
 * "key=value ..." string (ABI, arch, debug asserts, the REF64 and FP32 math
 * flags and the FP32 kernel's batch / RNG-resolution / occupancy macros).
 * No reference counterpart: the reference's kernel has no build knobs
 * (R/pkg/setup.py:28-34 fixes its Cython directives). */
const char* em_build_info(void);
const char* em_last_error(void);
int em_device_count(void);
/* sm_count, max SM clock (kHz), compute capability major/minor */
int em_device_info(int device, int* sm_count, int* clock_khz, int* cc_major, int* cc_minor);

/* Drop-in for _kernel.walk_exits_chunk (S/_kernel.pyx:376-411), REF64.
 * x_out (n, d), steps_out (n,), comp_out (n,); *err_rep = first failing
 * replicate or -1. */
int em_walk_exits_chunk(const em_geometry* g, const double* pole_xy, int64_t pole_index,
                        int64_t rep_start, int64_t rep_end, uint64_t seed, double eps,
                        int64_t max_steps, int device, double* x_out, int64_t* steps_out,
                        int64_t* comp_out, int64_t* err_rep);

/* Drop-in for _kernel.accumulate_chunk (S/_kernel.pyx:414-464), REF64.
 * out0/out1 are accumulated in place (+=); stats = (steps_sum, steps_sq,
 * steps_max, idw_fallbacks); *err_rep = first failing replicate or -1. */
int em_accumulate_chunk(const em_geometry* g, const double* pole_xy, int64_t pole_index,
                        int64_t rep_start, int64_t rep_end, uint64_t seed, double eps,
                        int64_t max_steps, const em_side* s0, const em_side* s1, int device,
                        double* out0, double* out1, int64_t* stats, int64_t* err_rep);

/* Batched path (S/backend.py:147-199).  A plan uploads geometry, poles,
 * anchors and the binning accelerators once; runs then keep everything
 * resident in HBM.  pole_ids (NULL = 0..n_poles-1) are the pole indices
 * that key the RNG streams, so a row-sharded multi-GPU run reproduces the
 * single-GPU counts exactly. */
int em_plan_create(const em_geometry* g, const em_side* s0, const em_side* s1,
                   const double* poles, const int64_t* pole_ids, int64_t n_poles,
                   double eps, int64_t max_steps, const em_options* opt, em_plan** out);
int em_plan_destroy(em_plan* p);
/* walks rep in [rep_start, rep_start + n_rep) for every pole; host outputs */
int em_plan_run(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep, em_outputs* out);
/* same, but the whole output block -- counts (n_poles, n0 + n1) | stats
 * (3, n_poles) int64 -- is copied once into a plan-owned page-locked buffer
 * and *block points at it (valid until the next run or destroy): no extra
 * host copy for callers that convert the rows anyway. */
int em_plan_run_host(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                     const int64_t** block, int64_t* err_pole, int64_t* err_rep);
/* same, with the count rows converted to float64 on the device (exact below
 * 2^53): the first n_poles * (n0 + n1) words of *block are doubles -- the
 * reference's float64 raw rows (S/backend.py:137-144) without a host-side
 * conversion; the stats stay int64. */
int em_plan_run_host_f64(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                         const int64_t** block, int64_t* err_pole, int64_t* err_rep);
/* hand the page-locked block of the last em_plan_run_host to the caller
 * (zero-copy results): *block stays valid until em_host_block_free(*block);
 * the plan stages its next run in another block.  (Host-side adapters only:
 * the reference's AccumulateResult owns its arrays, S/backend.py:193-199.) */
int em_plan_detach_block(em_plan* p, int64_t** block);
int em_host_block_free(void* block);
/* same, outputs left in device memory (caller-owned, zeroed by the library)
 * and work ordered on `stream` (cudaStream_t, NULL = the plan's stream).
 * Asynchronous: returns once the work is enqueued; after synchronising,
 * em_plan_check reports a budget overrun of that run (EM_BUDGET) and makes
 * em_plan_last_stats' kernel time available. */
int em_plan_run_device(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                       em_outputs* dev_out, void* stream);
int em_plan_check(em_plan* p, int64_t* err_pole, int64_t* err_rep);
/* device time (ms) of the walk kernel of the last run, CUDA events on the
 * launching stream; walks and steps of that run */
int em_plan_last_stats(const em_plan* p, double* kernel_ms, int64_t* walks, int64_t* steps);
/* number of library kernels launched by the last run (the walk kernel plus
 * any zeroing/packing kernels) */
int em_plan_last_launches(const em_plan* p, int64_t* launches);
int64_t em_plan_n_bins(const em_plan* p, int side);
/* scheduler of the last integer-count run: 0 persistent pole-cycling warps,
 * 1 the same with per-warp shared step-statistics tables (tiny jobs), 2 the
 * pole-block scheduler with per-block shared-memory histograms; -1 none */
int em_plan_last_scheduler(const em_plan* p);
/* walks per lane of the plan's integer-count kernel: 2 where the packed
 * two-walks-per-lane kernel runs (EM_FLAG_ONE_WALK_PER_LANE forces 1) */
int em_plan_walks_per_lane(const em_plan* p);
/* walks per lane of the last integer-count run (1 or 2; 0 before any run) */
int em_plan_last_walks_per_lane(const em_plan* p);
/* the walk chain the plan runs (EM_CHAIN_*): EM_CHAIN_TANGENT falls back to
 * EM_CHAIN_MAX where no tangent-ball step exists for the geometry */
int em_plan_chain(const em_plan* p);
/* the chain a plan over geometry g would run for (precision, chain), without
 * a device: EM_CHAIN_TANGENT resolves to EM_CHAIN_MAX where no tangent-ball
 * step exists; negative EM_ERR_* for an invalid geometry or pair */
int em_resolve_chain(const em_geometry* g, int precision, int chain);

/* Fractional rows (required for IDW weight families; on REF64 valid for
 * Voronoi too): raw0 (n_poles, n0) and raw1 (n_poles, n1) doubles.  On an
 * FP32 plan the walks are the FP32 kernel's and the IDW weights (FP64,
 * S/_kernel.pyx:323-369) are summed over its exits in the same fixed order.  With
 * init0/init1 the sums continue in place from those values in replicate
 * order (the chunk contract, S/_kernel.pyx:451-461); without, every `chunk`
 * replicates (8192 in the reference driver) start a zeroed partial that is
 * folded into the row in chunk order (S/backend.py:159-198), so fractional
 * IDW rows match the reference bit for bit.  stats (3, n_poles). */
int em_plan_run_raw(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep, int64_t chunk,
                    const double* init0, const double* init1, double* raw0, double* raw1,
                    int64_t* stats, int64_t* idw_fallbacks, int64_t* err_pole, int64_t* err_rep);

/* Bin arbitrary points (n, d) with the plan's rule: owner component ->
 * side -> nearest anchor of that side's family (exact lexicographic FP64 on
 * REF64, the walk kernel's FP32 binner otherwise).  Cell measures of
 * unstructured families by boundary quadrature use it (S/weights.py:155-181
 * rejects generic anchors). */
int em_bin_points(em_plan* p, const double* pts, int64_t n, int64_t* comp, int64_t* side,
                  int64_t* bin);

/* One-shot convenience: create, run, destroy. */
int em_run_accumulate(const em_geometry* g, const em_side* s0, const em_side* s1,
                      const double* poles, const int64_t* pole_ids, int64_t n_poles,
                      uint64_t seed, double eps, int64_t max_steps, int64_t n_rep,
                      const em_options* opt, em_outputs* out);

/* Exit points of n_rep walks from every pole of the plan
 * (S/backend.py:202-227 generalised to many poles): x_out (n_poles*n_rep, d)
 * in (pole, replicate) order, steps_out, comp_out likewise. */
int em_run_exits(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                 double* x_out, int64_t* steps_out, int64_t* comp_out, int64_t* err_pole,
                 int64_t* err_rep);

/* Test hook: ONE step of the plan's FP32 walk chain from each of n world
 * points x (n, d) with the random words (n, 2) (the tangent / rolling steps
 * use word 0; the woe / max steps take the azimuth from word 0 -- 3D: z
 * from word 0, azimuth from word 1), through the same device functions as
 * the walk kernel.  y (n, d): the candidate next point in world coordinates;
 * mask (n,): the walk's 0/1 stop mask at x (0 = inside the eps-shell).  No
 * reference counterpart (the reference's step is inline in S/_kernel.pyx:
 * 185-196); it exposes the samplers to closed-form checks. */
int em_debug_step(em_plan* p, const double* x, const uint32_t* words, int64_t n, double* y,
                  float* mask);

/* Host unit-test hook (no device needed): one named closed-form constant of
 * the FP32 kernel for geometry g on chain `chain` (the chain the plan runs)
 * with K = I flag `ident`, as em_plan_create computes it -- e.g. "t3" (the
 * 3 x 24 per-face tables of the tangent chain on 3D boxes), "tbt", "rho_b",
 * "rho_h", "mid2", "Ad", "Q", "shk", "sb", "g", "m2", "stop_scale".  Returns
 * the number of floats written, -1 for an unknown name. */
int em_f32_constant(const em_geometry* g, int chain, int ident, double eps, const char* name,
                    float* out, int n);

/* Micro-benchmark used for the roofline denominator: achieved FP32 FFMA
 * lane-ops/s of an issue-bound kernel on `device` (its own CUDA events). */
int em_fp32_peak(int device, double* flops_per_s, double* ms);

/* Known-answer hooks for the RNG golden tests: n blocks, inputs
 * (c0, c1, c2, c3, k0, k1) per block, outputs 4 words per block. */
int em_philox4x64_blocks(const uint64_t* in6, uint64_t* out4, int n, int device);
int em_philox4x32_blocks(const uint32_t* in6, uint32_t* out4, int n, int device);
/* the CUDA toolkit's curand_Philox4x32_10 on the same inputs (cross-check) */
int em_curand_philox4x32_blocks(const uint32_t* in6, uint32_t* out4, int n, int device);

#ifdef __cplusplus
}
#endif
#endif
