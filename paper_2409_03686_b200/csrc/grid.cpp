// grid.cpp -- conservative candidate grid for unstructured anchor families.
//
// The reference bins an exit into its nearest anchor by brute force over a
// generic family (S/_kernel.pyx:315-319, S/ = /root/reference/pkg/src/
// exitmeasure/): O(M) per exit, 13-34% of its run time at 512-2048 anchors
// and more than the whole walk at cfg5's 4096+4096.  The FP32
// kernel instead looks up a uniform grid cell and scans only the cell's
// candidate list.  For a cell with centre c and half-diagonal r_c, any anchor
// that can be nearest to some point of the cell satisfies
//     |c - a| <= min_b |c - b| + 2 r_c          (triangle inequality),
// so the list built with that bound (plus a small slack for FP32 rounding of
// the query) always contains the true nearest anchor.  Lists are only built
// in a band around the anchors (where shell exits live); other cells, and
// cells whose list would exceed 254 entries, are flagged for brute force --
// slower, never wrong.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace em {

struct GridHost {
  double lo[3];
  double h;
  int n[3];
  std::vector<uint32_t> cell;  // offset << 8 | count (255 = brute force)
  std::vector<uint32_t> cand;
};

static inline double dist2(const double* a, const double* b, int d) {
  double t = 0.0;
  for (int j = 0; j < d; ++j) {
    const double v = a[j] - b[j];
    t += v * v;
  }
  return t;
}

bool build_grid(const double* anchors, int64_t m, int d, double eps, GridHost& G) {
  if (m <= 0 || (d != 2 && d != 3)) return false;
  // nearest-neighbour spacing (subsampled) sets the cell size and the band
  const int64_t n_probe = std::min<int64_t>(m, 512);
  const int64_t stride = std::max<int64_t>(1, m / n_probe);
  std::vector<double> nn;
  double nn_max = 0.0;
  for (int64_t i = 0; i < m; i += stride) {
    double best = 1e300;
    for (int64_t j = 0; j < m; ++j) {
      if (j == i) continue;
      best = std::min(best, dist2(anchors + i * d, anchors + j * d, d));
    }
    if (best < 1e300) {
      nn.push_back(std::sqrt(best));
      nn_max = std::max(nn_max, std::sqrt(best));
    }
  }
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int j = 0; j < d; ++j) {
    lo[j] = 1e300;
    hi[j] = -1e300;
  }
  for (int64_t i = 0; i < m; ++i)
    for (int j = 0; j < d; ++j) {
      lo[j] = std::min(lo[j], anchors[i * d + j]);
      hi[j] = std::max(hi[j], anchors[i * d + j]);
    }
  double ext = 0.0;
  for (int j = 0; j < d; ++j) ext = std::max(ext, hi[j] - lo[j]);
  if (nn.empty() || nn_max <= 0.0) nn_max = std::max(ext, 1e-3);
  std::sort(nn.begin(), nn.end());
  double spacing = nn.empty() ? nn_max : nn[nn.size() / 2];
  if (spacing <= 0.0) spacing = nn_max;
  const double margin = nn_max + 4.0 * eps + 1e-9 * std::max(ext, 1.0);
  for (int j = 0; j < d; ++j) {
    lo[j] -= margin;
    hi[j] += margin;
  }
  // cell edge: a quarter of the anchor spacing in 3D (about 2.2 candidates
  // per surface cell on cfg5's square families, 6 at half the spacing),
  // half of it in 2D
  double h = (d == 3 ? 0.25 : 0.5) * spacing;
  const double kMaxCells = d == 3 ? double(1 << 23) : double(1 << 22);
  for (;;) {
    double cells = 1.0;
    for (int j = 0; j < d; ++j) cells *= std::ceil((hi[j] - lo[j]) / h);
    if (cells <= kMaxCells) break;
    h *= 1.25;
  }
  int n[3] = {1, 1, 1};
  for (int j = 0; j < d; ++j) n[j] = std::max(1, (int)std::ceil((hi[j] - lo[j]) / h));
  const int64_t n_cells = (int64_t)n[0] * n[1] * n[2];

  // bucket anchors by cell
  auto cell_of = [&](const double* p, int* c) {
    for (int j = 0; j < 3; ++j) c[j] = 0;
    for (int j = 0; j < d; ++j) {
      int v = (int)std::floor((p[j] - lo[j]) / h);
      c[j] = std::min(std::max(v, 0), n[j] - 1);
    }
  };
  std::vector<int64_t> bstart(n_cells + 1, 0);
  std::vector<int32_t> bitem(m);
  std::vector<int64_t> acell(m);
  for (int64_t i = 0; i < m; ++i) {
    int c[3];
    cell_of(anchors + i * d, c);
    acell[i] = ((int64_t)c[2] * n[1] + c[1]) * n[0] + c[0];
    bstart[acell[i] + 1]++;
  }
  for (int64_t c = 0; c < n_cells; ++c) bstart[c + 1] += bstart[c];
  {
    std::vector<int64_t> fill(bstart.begin(), bstart.end() - 1);
    for (int64_t i = 0; i < m; ++i) bitem[fill[acell[i]]++] = (int32_t)i;
  }

  // band: cells within band_r of some anchor get candidate lists
  const double band_r = 1.25 * nn_max + 4.0 * eps;
  const int br = (int)std::ceil(band_r / h) + 1;
  std::vector<uint8_t> band(n_cells, 0);
  for (int64_t i = 0; i < m; ++i) {
    int c[3];
    cell_of(anchors + i * d, c);
    const int zr = d == 3 ? br : 0;
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -br; dy <= br; ++dy)
        for (int dx = -br; dx <= br; ++dx) {
          const int x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
          if (x < 0 || y < 0 || z < 0 || x >= n[0] || y >= n[1] || z >= n[2]) continue;
          band[((int64_t)z * n[1] + y) * n[0] + x] = 1;
        }
  }

  const double rc = 0.5 * h * std::sqrt((double)d);
  const double slack = 0.02 * h;
  G.cell.assign(n_cells, 255u);
  G.cand.clear();
  // band cells are independent: threads take contiguous cell ranges, each
  // writes its lists into a private buffer (cell word = local offset), and
  // the buffers are concatenated in range order -- the same grid as a serial
  // build, whatever the thread count
  const int n_thr = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  constexpr int64_t kChunk = 2048;  // cells per work item (band cells cluster: interleave)
  const int64_t n_items = (n_cells + kChunk - 1) / kChunk;
  std::vector<std::vector<uint32_t>> part(n_items);
  auto work = [&](int t) {
  std::vector<std::pair<double, int32_t>> found;
  for (int64_t it = t; it < n_items; it += n_thr) {
  std::vector<uint32_t>& cand = part[it];
  const int64_t c_lo = it * kChunk, c_hi = std::min<int64_t>(n_cells, c_lo + kChunk);
  for (int64_t ci = c_lo; ci < c_hi; ++ci) {
    if (!band[ci]) continue;
    const int cx = (int)(ci % n[0]), cy = (int)((ci / n[0]) % n[1]), cz = (int)(ci / ((int64_t)n[0] * n[1]));
    double cc[3] = {lo[0] + (cx + 0.5) * h, lo[1] + (cy + 0.5) * h, d == 3 ? lo[2] + (cz + 0.5) * h : 0.0};
    // ring search for the nearest anchor to the cell centre
    double best2 = 1e300;
    int ring = 0;
    const int max_ring = std::max(n[0], std::max(n[1], n[2]));
    for (; ring <= max_ring; ++ring) {
      // cells at Chebyshev distance exactly `ring` are at least (ring - 0.5) h away
      const double lb = (ring - 0.5) * h;
      if (ring > 0 && lb > 0.0 && lb * lb > best2) break;
      const int zr = d == 3 ? ring : 0;
      for (int dz = -zr; dz <= zr; ++dz)
        for (int dy = -ring; dy <= ring; ++dy)
          for (int dx = -ring; dx <= ring; ++dx) {
            if (std::max(std::abs(dx), std::max(std::abs(dy), std::abs(dz))) != ring) continue;
            const int x = cx + dx, y = cy + dy, z = cz + dz;
            if (x < 0 || y < 0 || z < 0 || x >= n[0] || y >= n[1] || z >= n[2]) continue;
            const int64_t b = ((int64_t)z * n[1] + y) * n[0] + x;
            for (int64_t k = bstart[b]; k < bstart[b + 1]; ++k)
              best2 = std::min(best2, dist2(cc, anchors + (int64_t)bitem[k] * d, d));
          }
    }
    const double bound = std::sqrt(best2) + 2.0 * rc + slack;
    const int rr = (int)std::ceil(bound / h + 0.5);
    found.clear();
    const int zr = d == 3 ? rr : 0;
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -rr; dy <= rr; ++dy)
        for (int dx = -rr; dx <= rr; ++dx) {
          const int x = cx + dx, y = cy + dy, z = cz + dz;
          if (x < 0 || y < 0 || z < 0 || x >= n[0] || y >= n[1] || z >= n[2]) continue;
          const int64_t b = ((int64_t)z * n[1] + y) * n[0] + x;
          for (int64_t k = bstart[b]; k < bstart[b + 1]; ++k) {
            const double t = dist2(cc, anchors + (int64_t)bitem[k] * d, d);
            if (t <= bound * bound) found.push_back({t, bitem[k]});
          }
        }
    if (found.empty()) continue;  // brute force
    std::sort(found.begin(), found.end());  // nearest first: early hits
    // prune the triangle bound's list to the anchors whose Voronoi cells can
    // meet the cell: a is never nearest anywhere in the (slack-expanded)
    // cell if a nearer candidate b beats it at every point p of it, i.e. the
    // affine |p - a|^2 - |p - b|^2 = 2 p.(b - a) + |a|^2 - |b|^2 stays
    // positive over the box (its minimum sits at a corner: per axis the
    // lower or upper face by the coefficient's sign).  Exact in double;
    // fewer candidates = fewer iterations of the kernel's divergent scan.
    {
      double blo[3] = {0, 0, 0}, bhi[3] = {0, 0, 0};
      for (int j = 0; j < d; ++j) {
        blo[j] = cc[j] - 0.5 * h - slack;
        bhi[j] = cc[j] + 0.5 * h + slack;
      }
      size_t kept = 0;
      for (size_t i = 0; i < found.size(); ++i) {
        const double* a = anchors + (int64_t)found[i].second * d;
        bool dominated = false;
        for (size_t k = 0; k < kept && k < 16 && !dominated; ++k) {
          const double* b = anchors + (int64_t)found[k].second * d;
          double mn = 0.0;
          for (int j = 0; j < d; ++j) {
            const double coef = 2.0 * (b[j] - a[j]);
            mn += coef * (coef > 0.0 ? blo[j] : bhi[j]) + a[j] * a[j] - b[j] * b[j];
          }
          dominated = mn > 1e-12;
        }
        if (!dominated) found[kept++] = found[i];
      }
      found.resize(kept);
    }
    if (found.size() > 254) continue;  // brute force
    const uint64_t off = cand.size();
    if (off >= (1u << 24)) continue;
    for (auto& f : found) cand.push_back((uint32_t)f.second);
    G.cell[ci] = ((uint32_t)off << 8) | (uint32_t)found.size();
  }
  }
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < n_thr; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  // rebase each range's offsets; lists past 2^24 entries fall back to brute force
  for (int64_t t = 0; t < n_items; ++t) {
    const uint64_t base = G.cand.size();
    const int64_t c_lo = t * kChunk, c_hi = std::min<int64_t>(n_cells, c_lo + kChunk);
    for (int64_t ci = c_lo; ci < c_hi; ++ci) {
      const uint32_t w = G.cell[ci];
      if ((w & 255u) == 255u) continue;
      const uint64_t off = base + (w >> 8);
      G.cell[ci] = off + (w & 255u) <= (1u << 24) ? (uint32_t)((off << 8) | (w & 255u)) : 255u;
    }
    G.cand.insert(G.cand.end(), part[t].begin(), part[t].end());
  }
  if (G.cand.empty()) G.cand.push_back(0);
  for (int j = 0; j < 3; ++j) {
    G.lo[j] = j < d ? lo[j] : 0.0;
    G.n[j] = n[j];
  }
  G.h = h;
  return true;
}

}  // namespace em
