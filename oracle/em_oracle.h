/* em_oracle.h -- C ABI of the CPU parity oracle (test infrastructure only;
 * see em_oracle.c for what it restates and the rule that the product path
 * never links it). */
#ifndef EM_ORACLE_H
#define EM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* One side's packed weight family, the reference's SidePack
 * (S/backend.py:57-68, packed by pack_side :89-126). */
typedef struct {
  const double* anchors;   /* (n_anchors, d) */
  int64_t n_anchors;
  const int64_t* blk;      /* (n_blk, 3): kind, start, count */
  const double* blkf;      /* (n_blk, 4): cx, cy, cz, radius|halfwidth */
  int64_t n_blk;
  int32_t wkind;           /* 0 voronoi, 1 idw */
  int32_t idw_power;
  const double* idw_radii; /* (n_anchors,) when wkind == 1 */
} emo_side;

void emo_philox4x64(uint64_t k0, uint64_t k1, uint64_t c0, uint64_t c1,
                    uint64_t c2, uint64_t c3, uint64_t* out);
double emo_notch_signed(double nx, double ny, const double* x);
double emo_signed_dist(const int64_t* gi, int64_t gi_len, const double* gf,
                       const double* x);
int64_t emo_owner_component(const int64_t* gi, int64_t gi_len, const double* gf,
                            const double* x);
int64_t emo_assign_anchor(const double* x, int d, const emo_side* s);
int64_t emo_walk_exits_chunk(const int64_t* gi, int64_t gi_len, const double* gf,
                             const double* ksqrt, const double* pole_xy,
                             int64_t pole_index, int64_t rep_start, int64_t rep_end,
                             uint64_t seed, double eps, int64_t max_steps,
                             double* x_out, int64_t* steps_out, int64_t* comp_out);
int64_t emo_accumulate_chunk(const int64_t* gi, int64_t gi_len, const double* gf,
                             const int8_t* comp_side, const double* ksqrt,
                             const double* pole_xy, int64_t pole_index,
                             int64_t rep_start, int64_t rep_end, uint64_t seed,
                             double eps, int64_t max_steps, const emo_side* s0,
                             const emo_side* s1, double* out0, double* out1,
                             int64_t* stats);
int64_t emo_run_accumulate(const int64_t* gi, int64_t gi_len, const double* gf,
                           const int8_t* comp_side, const double* ksqrt,
                           const double* poles, int64_t n_poles, uint64_t seed,
                           double eps, int64_t max_steps, int64_t n_rep,
                           const emo_side* s0, const emo_side* s1, double* raw0,
                           double* raw1, int64_t* steps_sum, int64_t* steps_sq,
                           int64_t* steps_max, int64_t* idw_fb, int64_t* err,
                           int nthreads);

#ifdef __cplusplus
}
#endif
#endif
