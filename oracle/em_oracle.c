/*
 * em_oracle.c -- CPU restatement of the reference exit-measure hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker (or the timed CPU baseline).  The
 * product path (paper_2409_03686_b200) never links or calls it and fails
 * loudly when its CUDA library is missing.
 *
 * What it restates (R/ = /root/reference/, S/ = R/pkg/src/exitmeasure/):
 *   - Philox4x64-10 block and stream layout       S/_kernel.pyx:21-54, S/rng.py:19-74
 *   - Marsaglia direction sampling                S/_kernel.pyx:57-81
 *   - ball/box outer + ball-hole signed distance  S/_kernel.pyx:89-142
 *   - owner component                             S/_kernel.pyx:145-156
 *   - walk-on-ellipsoids loop                     S/_kernel.pyx:163-197
 *   - lexicographic nearest-anchor binning        S/_kernel.pyx:204-320
 *   - IDW scatter                                 S/_kernel.pyx:323-369
 *   - walk_exits_chunk / accumulate_chunk         S/_kernel.pyx:376-464
 *   - run_accumulate driver (job order merge)     S/backend.py:147-199
 * Every floating-point expression keeps the reference's operand order; the
 * file must be compiled with -ffp-contract=off (no FMA contraction), as the
 * reference's own build is (gcc -O2, no -march).
 *
 * Extension beyond the reference (BASELINE cfg5, the L-shaped box, which the
 * reference geometry cannot express -- SURVEY.md Appendix A): when the packed
 * geometry carries gi[3] = 1, a quadrant-prism notch {x >= nx, y >= ny} is cut
 * out of the outer box; it is boundary component 1 + n_holes and its signed
 * distance is em_notch_signed below.  Parity for that extension is pinned
 * only by structural invariants (row sums, containment) and cross-checks
 * against the GPU mirror, not by the reference's tests ("parity unpinned").
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "em_oracle.h"

static const double M_2PI_ = 6.283185307179586476925286766559;
static const double INV53 = 1.0 / 9007199254740992.0;

#define PHILOX_M0 0xD2E7470EE14C6C93ULL
#define PHILOX_M1 0xCA5A826395121157ULL
#define PHILOX_W0 0x9E3779B97F4A7C15ULL
#define PHILOX_W1 0xBB67AE8584CAA73BULL
#define BIG_INDEX ((int64_t)1 << 62)

/* S/_kernel.pyx:30-34 -- exact high word of a 64x64 product */
static inline uint64_t mulhi64(uint64_t a, uint64_t b) {
  unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
  return (uint64_t)(p >> 64);
}

/* S/_kernel.pyx:37-54 */
void emo_philox4x64(uint64_t k0, uint64_t k1, uint64_t c0, uint64_t c1,
                    uint64_t c2, uint64_t c3, uint64_t* out) {
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0 = mulhi64(PHILOX_M0, c0), lo0 = PHILOX_M0 * c0;
    uint64_t hi1 = mulhi64(PHILOX_M1, c2), lo1 = PHILOX_M1 * c2;
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += PHILOX_W0;
    k1 += PHILOX_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* S/_kernel.pyx:57-81: one Philox block per rejection trial, counter
 * (draw, 0, rep, pole), key (seed, 0); words 0/1 -> (w >> 11) * 2^-53. */
static void sample_direction(int d, uint64_t seed, uint64_t* draw, uint64_t rep,
                             uint64_t pole, double* u) {
  uint64_t w[4];
  for (;;) {
    emo_philox4x64(seed, 0ULL, *draw, 0ULL, rep, pole, w);
    *draw += 1ULL;
    double u0 = (double)(w[0] >> 11) * INV53;
    double u1 = (double)(w[1] >> 11) * INV53;
    double v1 = 2.0 * u0 - 1.0;
    double v2 = 2.0 * u1 - 1.0;
    double s = v1 * v1 + v2 * v2;
    if (d == 2) {
      if (s <= 1.0 && s > 0.0) {
        double rs = sqrt(s);
        u[0] = v1 / rs;
        u[1] = v2 / rs;
        return;
      }
    } else {
      if (s < 1.0) {
        double f = 2.0 * sqrt(1.0 - s);
        u[0] = v1 * f;
        u[1] = v2 * f;
        u[2] = 1.0 - 2.0 * s;
        return;
      }
    }
  }
}

/* ---- geometry: gi = [d, outer_kind, n_holes(, n_notch)],
 *      gf = [outer_center(d), R|h, (hole_center(d), r)*, (nx, ny)?] ---- */

typedef struct {
  int d, outer_kind, n_holes, n_notch;
  const double* gf;
} geom_t;

static geom_t geom_from(const int64_t* gi, int64_t gi_len, const double* gf) {
  geom_t g;
  g.d = (int)gi[0];
  g.outer_kind = (int)gi[1];
  g.n_holes = (int)gi[2];
  g.n_notch = gi_len >= 4 ? (int)gi[3] : 0;
  g.gf = gf;
  return g;
}

/* S/_kernel.pyx:89-116 */
static double outer_signed(const geom_t* g, const double* x) {
  const double* gf = g->gf;
  int d = g->d;
  if (g->outer_kind == 0) {
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

/* S/_kernel.pyx:119-130 */
static double hole_dist(const geom_t* g, const double* x, int hole) {
  const double* gf = g->gf;
  int d = g->d;
  int off = d + 1 + hole * (d + 1);
  double dx0 = x[0] - gf[off], dx1 = x[1] - gf[off + 1];
  double t = dx0 * dx0 + dx1 * dx1;
  if (d == 3) {
    double dx2 = x[2] - gf[off + 2];
    t = t + dx2 * dx2;
  }
  return sqrt(t) - gf[off + d];
}

/* Extension (cfg5): signed distance to the notch {x >= nx, y >= ny},
 * positive outside the notch (inside the domain). */
double emo_notch_signed(double nx, double ny, const double* x) {
  double qx = nx - x[0];
  double qy = ny - x[1];
  if (qx <= 0.0 && qy <= 0.0) return qx > qy ? qx : qy;
  double ax = qx > 0.0 ? qx : 0.0;
  double ay = qy > 0.0 ? qy : 0.0;
  return sqrt(ax * ax + ay * ay);
}

static double notch_dist(const geom_t* g, const double* x) {
  int off = (g->d + 1) * (1 + g->n_holes);
  return emo_notch_signed(g->gf[off], g->gf[off + 1], x);
}

/* S/_kernel.pyx:133-142 (+ notch extension after the holes) */
static double signed_dist(const geom_t* g, const double* x) {
  double sd = outer_signed(g, x);
  for (int h = 0; h < g->n_holes; ++h) {
    double hd = hole_dist(g, x, h);
    if (hd < sd) sd = hd;
  }
  if (g->n_notch) {
    double nd = notch_dist(g, x);
    if (nd < sd) sd = nd;
  }
  return sd;
}

/* S/_kernel.pyx:145-156 (+ notch as the last component) */
static int owner_component(const geom_t* g, const double* x) {
  double best = fabs(outer_signed(g, x));
  int comp = 0;
  for (int h = 0; h < g->n_holes; ++h) {
    double dd = fabs(hole_dist(g, x, h));
    if (dd < best) {
      best = dd;
      comp = h + 1;
    }
  }
  if (g->n_notch) {
    double dd = fabs(notch_dist(g, x));
    if (dd < best) comp = g->n_holes + 1;
  }
  return comp;
}

/* S/_kernel.pyx:163-197 */
static int run_walk(const geom_t* g, const double* ksqrt, const double* pole_xy,
                    uint64_t pole, uint64_t rep, uint64_t seed, double eps,
                    int64_t max_steps, double* x, int64_t* steps_out) {
  int d = g->d;
  double u[3];
  uint64_t draw = 0;
  int64_t steps = 0;
  for (int j = 0; j < d; ++j) x[j] = pole_xy[j];
  for (;;) {
    double sd = signed_dist(g, x);
    if (sd <= eps) {
      *steps_out = steps;
      return 0;
    }
    if (steps >= max_steps) {
      *steps_out = steps;
      return 1;
    }
    sample_direction(d, seed, &draw, rep, pole, u);
    if (d == 2) {
      double y0 = ksqrt[0] * u[0] + ksqrt[1] * u[1];
      double y1 = ksqrt[2] * u[0] + ksqrt[3] * u[1];
      x[0] = x[0] + sd * y0;
      x[1] = x[1] + sd * y1;
    } else {
      double y0 = ksqrt[0] * u[0] + ksqrt[1] * u[1] + ksqrt[2] * u[2];
      double y1 = ksqrt[3] * u[0] + ksqrt[4] * u[1] + ksqrt[5] * u[2];
      double y2 = ksqrt[6] * u[0] + ksqrt[7] * u[1] + ksqrt[8] * u[2];
      x[0] = x[0] + sd * y0;
      x[1] = x[1] + sd * y1;
      x[2] = x[2] + sd * y2;
    }
    steps = steps + 1;
  }
}

/* ---- nearest-anchor assignment, S/_kernel.pyx:204-320 ---- */

static inline void lex_update(const double* x, int d, const double* anchors,
                              int64_t g, double* best_d2, int64_t* best_gi) {
  const double* a = anchors + g * d;
  double dx0 = x[0] - a[0], dx1 = x[1] - a[1];
  double t = dx0 * dx0 + dx1 * dx1;
  if (d == 3) {
    double dx2 = x[2] - a[2];
    t = t + dx2 * dx2;
  }
  if (t < *best_d2 || (t == *best_d2 && g < *best_gi)) {
    *best_d2 = t;
    *best_gi = g;
  }
}

static double square_signed(double cx, double cy, double h, const double* x) {
  double q0 = fabs(x[0] - cx) - h;
  double q1 = fabs(x[1] - cy) - h;
  double m = q0;
  if (q1 > m) m = q1;
  if (m <= 0.0) return -m;
  double t = (q0 > 0.0 ? q0 : 0.0) * (q0 > 0.0 ? q0 : 0.0) +
             (q1 > 0.0 ? q1 : 0.0) * (q1 > 0.0 ? q1 : 0.0);
  return -sqrt(t);
}

static inline double clampd(double v, double lo, double hi) {
  if (v < lo) return lo;
  if (v > hi) return hi;
  return v;
}

int64_t emo_assign_anchor(const double* x, int d, const emo_side* s) {
  double best_d2 = 1e308;
  int64_t best_gi = BIG_INDEX;
  for (int64_t b = 0; b < s->n_blk; ++b) {
    int64_t kind = s->blk[3 * b], start = s->blk[3 * b + 1], count = s->blk[3 * b + 2];
    double cx = s->blkf[4 * b], cy = s->blkf[4 * b + 1], radius = s->blkf[4 * b + 3];
    if (kind == 1) { /* circle */
      double px = x[0] - cx, py = x[1] - cy;
      double ang = atan2(py, px);
      double t = ang * ((double)count / M_2PI_);
      int64_t k = (int64_t)floor(t + 0.5);
      k = k % count;
      if (k < 0) k += count;
      for (int off = -2; off < 3; ++off) {
        int64_t idx = (k + off) % count;
        if (idx < 0) idx += count;
        lex_update(x, d, s->anchors, start + idx, &best_d2, &best_gi);
      }
    } else if (kind == 2) { /* square */
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
        int64_t k = (int64_t)floor(t + 0.5);
        k = k % count;
        if (k < 0) k += count;
        for (int off = -2; off < 3; ++off) {
          int64_t idx = (k + off) % count;
          if (idx < 0) idx += count;
          lex_update(x, d, s->anchors, start + idx, &best_d2, &best_gi);
        }
      } else {
        for (int64_t idx = 0; idx < count; ++idx)
          lex_update(x, d, s->anchors, start + idx, &best_d2, &best_gi);
      }
    } else { /* generic / sphere: brute force */
      for (int64_t idx = 0; idx < count; ++idx)
        lex_update(x, d, s->anchors, start + idx, &best_d2, &best_gi);
    }
  }
  return best_gi;
}

/* S/_kernel.pyx:323-369 */
static int64_t idw_accumulate(const double* x, int d, const emo_side* s,
                              int64_t winner, double* out) {
  int64_t m = s->n_anchors;
  double total = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    const double* a = s->anchors + i * d;
    double dx0 = x[0] - a[0], dx1 = x[1] - a[1];
    double d2 = dx0 * dx0 + dx1 * dx1;
    if (d == 3) {
      double dx2 = x[2] - a[2];
      d2 = d2 + dx2 * dx2;
    }
    double r = sqrt(d2);
    if (r < 1e-14) {
      out[i] += 1.0;
      return 0;
    }
    double base = s->idw_radii[i] - r;
    if (base > 0.0) {
      base = base / (s->idw_radii[i] * r);
      double w = base;
      for (int q = 0; q < s->idw_power - 1; ++q) w = w * base;
      total = total + w;
    }
  }
  if (total == 0.0) {
    out[winner] += 1.0;
    return 1;
  }
  for (int64_t i = 0; i < m; ++i) {
    const double* a = s->anchors + i * d;
    double dx0 = x[0] - a[0], dx1 = x[1] - a[1];
    double d2 = dx0 * dx0 + dx1 * dx1;
    if (d == 3) {
      double dx2 = x[2] - a[2];
      d2 = d2 + dx2 * dx2;
    }
    double r = sqrt(d2);
    double base = s->idw_radii[i] - r;
    if (base > 0.0) {
      base = base / (s->idw_radii[i] * r);
      double w = base;
      for (int q = 0; q < s->idw_power - 1; ++q) w = w * base;
      out[i] += w / total;
    }
  }
  return 0;
}

/* S/_kernel.pyx:376-411; returns err (first failing replicate) or -1 */
int64_t emo_walk_exits_chunk(const int64_t* gi, int64_t gi_len, const double* gf,
                             const double* ksqrt, const double* pole_xy,
                             int64_t pole_index, int64_t rep_start, int64_t rep_end,
                             uint64_t seed, double eps, int64_t max_steps,
                             double* x_out, int64_t* steps_out, int64_t* comp_out) {
  geom_t g = geom_from(gi, gi_len, gf);
  int d = g.d;
  int64_t n = rep_end - rep_start, err = -1;
  double xw[3];
  int64_t st;
  for (int64_t i = 0; i < n; ++i) {
    int rc = run_walk(&g, ksqrt, pole_xy, (uint64_t)pole_index,
                      (uint64_t)rep_start + (uint64_t)i, seed, eps, max_steps, xw, &st);
    for (int j = 0; j < d; ++j) x_out[i * d + j] = xw[j];
    steps_out[i] = st;
    if (rc != 0) {
      err = rep_start + i;
      break;
    }
    comp_out[i] = owner_component(&g, xw);
  }
  if (err >= 0) memset(comp_out, 0, (size_t)n * sizeof(int64_t));
  return err;
}

/* S/_kernel.pyx:414-464; stats = (steps_sum, steps_sq, steps_max, idw_fb) */
int64_t emo_accumulate_chunk(const int64_t* gi, int64_t gi_len, const double* gf,
                             const int8_t* comp_side, const double* ksqrt,
                             const double* pole_xy, int64_t pole_index,
                             int64_t rep_start, int64_t rep_end, uint64_t seed,
                             double eps, int64_t max_steps, const emo_side* s0,
                             const emo_side* s1, double* out0, double* out1,
                             int64_t* stats) {
  geom_t g = geom_from(gi, gi_len, gf);
  int d = g.d;
  int64_t n = rep_end - rep_start, err = -1;
  int64_t steps_sum = 0, steps_sq = 0, steps_max = 0, idw_fb = 0;
  double xw[3];
  int64_t st;
  for (int64_t i = 0; i < n; ++i) {
    int rc = run_walk(&g, ksqrt, pole_xy, (uint64_t)pole_index,
                      (uint64_t)rep_start + (uint64_t)i, seed, eps, max_steps, xw, &st);
    if (rc != 0) {
      err = rep_start + i;
      break;
    }
    steps_sum += st;
    steps_sq += st * st;
    if (st > steps_max) steps_max = st;
    int comp = owner_component(&g, xw);
    const emo_side* s = comp_side[comp] == 0 ? s0 : s1;
    double* out = comp_side[comp] == 0 ? out0 : out1;
    int64_t winner = emo_assign_anchor(xw, d, s);
    if (s->wkind == 0)
      out[winner] += 1.0;
    else
      idw_fb += idw_accumulate(xw, d, s, winner, out);
  }
  if (err >= 0) {
    stats[0] = stats[1] = stats[2] = stats[3] = 0;
    return err;
  }
  stats[0] = steps_sum;
  stats[1] = steps_sq;
  stats[2] = steps_max;
  stats[3] = idw_fb;
  return -1;
}

typedef struct {
  const int64_t* gi; int64_t gi_len; const double* gf; const int8_t* comp_side;
  const double* ksqrt; const double* poles; int d; uint64_t seed; double eps;
  int64_t max_steps, n_rep, chunk, n_chunks, n_jobs;
  const emo_side *s0, *s1;
  double *b0, *b1;
  int64_t* st;
  int64_t m0, m1;
  _Atomic int64_t next;
} job_ctx;

/* thread-pool worker: claims (pole, chunk) jobs from an atomic counter; every
 * job writes only its private buffers, so the claim order is irrelevant */
static void* job_worker(void* arg) {
  job_ctx* c = (job_ctx*)arg;
  for (;;) {
    int64_t j = atomic_fetch_add(&c->next, 1);
    if (j >= c->n_jobs) break;
    int64_t p = j / c->n_chunks, k = j % c->n_chunks;
    int64_t r0 = k * c->chunk, r1 = r0 + c->chunk < c->n_rep ? r0 + c->chunk : c->n_rep;
    c->st[5 * j + 4] = emo_accumulate_chunk(
        c->gi, c->gi_len, c->gf, c->comp_side, c->ksqrt, c->poles + p * c->d, p, r0, r1,
        c->seed, c->eps, c->max_steps, c->s0, c->s1, c->b0 + j * c->m0,
        c->b1 + j * c->m1, c->st + 5 * j);
  }
  return NULL;
}

/* S/backend.py:147-199: jobs (pole, CHUNK-range) in pole-major order, each
 * with zeroed private buffers, merged in job order (so fractional IDW sums
 * match the reference bit for bit).  Returns 0, or 1 on a budget overrun with
 * the first failing job's (pole, replicate) in err[0], err[1]. */
int64_t emo_run_accumulate(const int64_t* gi, int64_t gi_len, const double* gf,
                           const int8_t* comp_side, const double* ksqrt,
                           const double* poles, int64_t n_poles, uint64_t seed,
                           double eps, int64_t max_steps, int64_t n_rep,
                           const emo_side* s0, const emo_side* s1, double* raw0,
                           double* raw1, int64_t* steps_sum, int64_t* steps_sq,
                           int64_t* steps_max, int64_t* idw_fb, int64_t* err,
                           int nthreads) {
  const int64_t CHUNK = 8192;
  int d = (int)gi[0];
  int64_t n_chunks = (n_rep + CHUNK - 1) / CHUNK;
  int64_t n_jobs = n_poles * n_chunks;
  int64_t m0 = s0->n_anchors, m1 = s1->n_anchors;
  double* b0 = (double*)calloc((size_t)(n_jobs * m0 + 1), sizeof(double));
  double* b1 = (double*)calloc((size_t)(n_jobs * m1 + 1), sizeof(double));
  int64_t* st = (int64_t*)calloc((size_t)(n_jobs * 5 + 1), sizeof(int64_t));
  if (!b0 || !b1 || !st) {
    free(b0); free(b1); free(st);
    return -1;
  }
  if (nthreads < 1) nthreads = 1;
  job_ctx ctx = {gi, gi_len, gf, comp_side, ksqrt, poles, d, seed, eps, max_steps,
                 n_rep, CHUNK, n_chunks, n_jobs, s0, s1, b0, b1, st, m0, m1, 0};
  if (nthreads == 1) {
    job_worker(&ctx);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, job_worker, &ctx);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  int64_t rc = 0;
  *idw_fb = 0;
  for (int64_t p = 0; p < n_poles; ++p) {
    steps_sum[p] = steps_sq[p] = steps_max[p] = 0;
    for (int64_t i = 0; i < m0; ++i) raw0[p * m0 + i] = 0.0;
    for (int64_t i = 0; i < m1; ++i) raw1[p * m1 + i] = 0.0;
  }
  for (int64_t j = 0; j < n_jobs && rc == 0; ++j) {
    int64_t p = j / n_chunks;
    if (st[5 * j + 4] >= 0) {
      err[0] = p;
      err[1] = st[5 * j + 4];
      rc = 1;
      break;
    }
    for (int64_t i = 0; i < m0; ++i) raw0[p * m0 + i] += b0[j * m0 + i];
    for (int64_t i = 0; i < m1; ++i) raw1[p * m1 + i] += b1[j * m1 + i];
    steps_sum[p] += st[5 * j];
    steps_sq[p] += st[5 * j + 1];
    if (st[5 * j + 2] > steps_max[p]) steps_max[p] = st[5 * j + 2];
    *idw_fb += st[5 * j + 3];
  }
  free(b0); free(b1); free(st);
  return rc;
}

double emo_signed_dist(const int64_t* gi, int64_t gi_len, const double* gf,
                       const double* x) {
  geom_t g = geom_from(gi, gi_len, gf);
  return signed_dist(&g, x);
}

int64_t emo_owner_component(const int64_t* gi, int64_t gi_len, const double* gf,
                            const double* x) {
  geom_t g = geom_from(gi, gi_len, gf);
  return owner_component(&g, x);
}
