// capi.cu -- C ABI of libexitmeasure_b200.so (declared in
// include/exitmeasure_b200.h): plans, device buffers, launches.
//
// A plan holds one problem (geometry, K^{1/2}, poles, two weight families)
// resident in HBM: poles as float4 / double rows, anchors as float4 / double,
// the candidate grids of unstructured families, and the output rows
// (n_poles x (n0 + n1) int64 counts + three int64 step statistics per pole).
// Each run zeroes the outputs, launches ONE persistent walk kernel and, for
// host outputs, copies the rows back.  Nothing here falls back to the CPU: any
// CUDA failure is returned as EM_ERR_CUDA with the CUDA error string.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "em_params.cuh"

// chunks per resident warp the chunk size aims at on the packed kernel
#ifndef EM_X2_CHUNKS
#define EM_X2_CHUNKS 8.0
#endif
// per-lane step statistics flush three atomics per pole change; spread over
// copies while copies x chunk x poles is below this many walks (measured on
// cfg2: 131072 -> 524288 is +9% on the one-walk kernel, +17% on the packed one)
#ifndef EM_STAT_SPREAD
#define EM_STAT_SPREAD 524288.0
#endif
#ifndef EM_X1_CHUNKS
#define EM_X1_CHUNKS 8.0
#endif

namespace em {
cudaError_t launch_ref64(const Ref64Params& P, int mode, int grid, int block, cudaStream_t s);
cudaError_t launch_f32(const F32Params& P, int d, int outer, int nh_mode, int mode, int chain,
                       bool ident, int bink, int grid, int block, cudaStream_t s);
cudaError_t launch_idw(const Ref64Params& P, const double* x, const long long* comp,
                       long long n_poles, long long n_rep, long long chunk,
                       const double* a0, const double* r0, int n0, int pw0, int wk0,
                       const double* a1, const double* r1, int n1, int pw1, int wk1, int* kind,
                       long long* idx, double* total, int* side, double* out0, double* out1,
                       const double* init0, const double* init1, cudaStream_t s);
cudaError_t launch_bin_points_ref64(const Ref64Params& P, const double* pts, long long n,
                                    long long* comp, long long* side, long long* bin,
                                    cudaStream_t s);
cudaError_t launch_bin_points_f32(const F32Params& P, int d, int outer, const double* pts,
                                  long long n, long long* comp, long long* side, long long* bin,
                                  cudaStream_t s);
cudaError_t launch_ffma_peak(float* out, int iters, int grid, int block, cudaStream_t s);
cudaError_t launch_zero_ranges(unsigned long long* const* ptrs, const long long* words, int n,
                               cudaStream_t s);
cudaError_t launch_rows_to_f64(unsigned long long* rows, long long n, cudaStream_t s);
cudaError_t launch_stats_fold(const unsigned long long* scratch, int copies, long long n_poles,
                              unsigned long long* stats, cudaStream_t s);
cudaError_t f32_blocks_per_sm(int d, int outer, int nh_mode, int chain, bool ident, int bink, int* nb);
bool f32_has_pole_blocks(int d, int outer, int nh_mode, int chain, bool ident, int bink);
// two walks per lane, packed FP32 arithmetic (walk_f32x2.cu)
bool f32x2_available(int d, int outer, int nh_mode, int chain, bool ident);
cudaError_t f32x2_blocks_per_sm(int d, int outer, int nh_mode, int bink, int* nb);
cudaError_t launch_f32x2(const F32Params& P, int d, int outer, int nh_mode, int bink, int grid,
                         int block, cudaStream_t s);
cudaError_t launch_philox64_kat(const unsigned long long* in, unsigned long long* out, int n,
                                cudaStream_t s);
cudaError_t launch_philox32_kat(const unsigned* in, unsigned* out, int n, cudaStream_t s);
const char* f32_build_knobs();
void sym_eig(const double* a_in, int d, double lam[3], double v[3][3]);
double sym_min_eig(const double* a_in, int d);
void* f32_build_new(const em_geometry* g, int chain, bool ident, double eps, int64_t max_steps,
                    F32Params& P);
void f32_build_to_kernel(const void* b, const double* w, float* out);
void f32_build_free(void* b);
cudaError_t launch_debug_step(const F32Params& P, int d, int outer, int nh_mode, int chain,
                              bool ident, const double* x, const unsigned* words, long long n,
                              double* y, float* mask, cudaStream_t s);

struct GridHost {
  double lo[3];
  double h;
  int n[3];
  std::vector<uint32_t> cell;
  std::vector<uint32_t> cand;
};
bool build_grid(const double* anchors, int64_t m, int d, double eps, GridHost& G);

// A candidate grid resident on one device (cell words then candidate lists in
// one allocation), shared by every plan over the same anchors: plans hold a
// reference, so the cache may evict an entry while plans still use it.
struct DeviceGrid {
  double lo[3] = {0, 0, 0};
  double h = 0.0;
  int n[3] = {1, 1, 1};
  int device = -1;
  void* dev = nullptr;
  const uint32_t* cell = nullptr;
  const uint32_t* cand = nullptr;
  const float4* candv = nullptr;  // the candidates' coordinates, index in .w (bits)
  ~DeviceGrid() {
    if (!dev) return;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    cudaFree(dev);
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
  }
};
}  // namespace em

using namespace em;

static thread_local std::string g_last_error = "";

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define EM_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(EM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
  } while (0)

// ---------------------------------------------------------------------------
// plan

// Per-device caching allocator: plans come and go per API call (the one-shot
// run_accumulate creates and destroys one), so device buffers, streams and
// events are recycled instead of paying cudaMalloc/cudaFree (which also
// synchronises the device) on every call.
struct BufCache {
  std::mutex mu;
  std::vector<std::pair<size_t, void*>> free_bufs;  // (capacity, ptr) per device below
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> events;
  std::vector<std::pair<size_t, void*>> free_pinned;
};

static BufCache& cache_of(int dev) {
  static std::mutex mu;
  static std::vector<BufCache*> caches;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)caches.size() <= dev) caches.resize(dev + 1, nullptr);
  if (!caches[dev]) caches[dev] = new BufCache();
  return *caches[dev];
}

static size_t round_cap(size_t n) {
  size_t c = 256;
  while (c < n) c <<= 1;
  return c;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int dev = 0;
  ~DevBuf() { release(); }
  void release() {
    if (!p) return;
    BufCache& c = cache_of(dev);
    std::lock_guard<std::mutex> lk(c.mu);
    c.free_bufs.push_back({bytes, p});
    p = nullptr;
    bytes = 0;
  }
  cudaError_t alloc(size_t n) {
    if (n <= bytes && p) return cudaSuccess;
    release();
    cudaGetDevice(&dev);
    const size_t cap = round_cap(std::max<size_t>(n, 16));
    {
      BufCache& c = cache_of(dev);
      std::lock_guard<std::mutex> lk(c.mu);
      for (size_t i = 0; i < c.free_bufs.size(); ++i)
        if (c.free_bufs[i].first == cap) {
          p = c.free_bufs[i].second;
          bytes = cap;
          c.free_bufs.erase(c.free_bufs.begin() + i);
          return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(&p, cap);
    if (e == cudaSuccess) bytes = cap;
    else p = nullptr;
    return e;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// page-locked host staging, recycled like the device buffers
struct PinBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int dev = 0;
  ~PinBuf() { release(); }
  void release() {
    if (!p) return;
    BufCache& c = cache_of(dev);
    std::lock_guard<std::mutex> lk(c.mu);
    c.free_pinned.push_back({bytes, p});
    p = nullptr;
    bytes = 0;
  }
  cudaError_t alloc(size_t n) {
    if (n <= bytes && p) return cudaSuccess;
    release();
    cudaGetDevice(&dev);
    const size_t cap = round_cap(std::max<size_t>(n, 16));
    {
      BufCache& c = cache_of(dev);
      std::lock_guard<std::mutex> lk(c.mu);
      for (size_t i = 0; i < c.free_pinned.size(); ++i)
        if (c.free_pinned[i].first == cap) {
          p = c.free_pinned[i].second;
          bytes = cap;
          c.free_pinned.erase(c.free_pinned.begin() + i);
          return cudaSuccess;
        }
    }
    cudaError_t e = cudaHostAlloc(&p, cap, cudaHostAllocDefault);
    if (e == cudaSuccess) bytes = cap;
    else p = nullptr;
    return e;
  }
};

static cudaStream_t take_stream(int dev) {
  BufCache& c = cache_of(dev);
  {
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.streams.empty()) {
      cudaStream_t s = c.streams.back();
      c.streams.pop_back();
      return s;
    }
  }
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  return s;
}

static cudaEvent_t take_event(int dev) {
  BufCache& c = cache_of(dev);
  {
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.events.empty()) {
      cudaEvent_t e = c.events.back();
      c.events.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

static void give_back(int dev, cudaStream_t s, cudaEvent_t e0, cudaEvent_t e1) {
  BufCache& c = cache_of(dev);
  std::lock_guard<std::mutex> lk(c.mu);
  if (s) c.streams.push_back(s);
  if (e0) c.events.push_back(e0);
  if (e1) c.events.push_back(e1);
}

struct em_plan {
  int device = 0, precision = EM_PREC_REF64, chain = EM_CHAIN_WOE;
  int d = 2, outer = 0, n_holes = 0, n_notch = 0, nh_mode = 2, bink = 0;
  bool ident = false;
  int64_t n_poles = 0, n0 = 0, n1 = 0;
  int grid = 0, block = 256;
  Ref64Params p64{};
  F32Params p32{};
  // every plan input (poles, pole ids, anchors, candidate grids, IDW radii)
  // lives in one device arena filled by ONE asynchronous H2D from pinned
  // staging on the plan's stream (ev_up marks its completion)
  DevBuf arena;
  PinBuf upin;
  cudaEvent_t ev_up = nullptr;
  const double* radii_dev[2] = {nullptr, nullptr};
  // one output block: counts (n_poles x row) | stats (3 x n_poles) | misc (err, ticket)
  DevBuf counts, stats, misc;
  DevBuf scopies;  // step-statistics copies (WorkOut::stat_copies > 1)
  PinBuf pin;  // host staging of the output block
  bool pin_valid = false;
  unsigned long long *blk_counts = nullptr, *blk_stats = nullptr, *blk_misc = nullptr;
  size_t blk_words = 0;
  DevBuf xo, so, co;           // exits
  DevBuf ikind, iidx, itot, iside, iraw0, iraw1, iinit0, iinit1;
  int wkind[2] = {0, 0}, idw_power[2] = {2, 2};
  int flags = 0;  // em_options.flags
  bool pole_blocks = false;  // the FP32 kernel family has the pole-block scheduler
  bool pack2 = false;        // counts mode runs two walks per lane (walk_f32x2.cu)
  int grid2 = 0;             // its persistent grid
  int last_sched = -1;       // scheduler of the last integer-count launch
  int last_lanes = 0;        // walks per lane of the last integer-count launch
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  int64_t last_walks = 0, last_steps = 0, last_launches = 0, last_n_rep = 0;
  bool last_timed = false;  // ev0 / ev1 bracket the last walk kernel
  cudaStream_t last_stream = nullptr;  // stream of the last run_device
  cudaStream_t last_launch_stream = nullptr;  // stream of the last launch (any entry point)
  std::vector<std::shared_ptr<DeviceGrid>> grids;  // device-resident candidate grids in use
  ~em_plan() {
    // buffers go back to the shared cache: nothing in flight may still use them
    if (stream) cudaStreamSynchronize(stream);
    if (last_timed && ev1) cudaEventSynchronize(ev1);
    give_back(device, stream, ev0, ev1);
    give_back(device, nullptr, ev_up, nullptr);
  }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int sm_count_of(int dev) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 1;
  }
  return cache[dev];
}

// Device-resident cache of candidate grids: a grid is a deterministic
// function of (anchors, d, eps), costs up to ~1 s of host time for 8k
// anchors and tens of MB, so repeated plans over the same bins (one per API
// call) reuse the device copy instead of rebuilding and re-uploading it.
std::shared_ptr<DeviceGrid> cached_device_grid(const double* anchors, int64_t m, int d, double eps,
                                               int device) {
  uint64_t h = 1469598103934665603ULL;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ULL;
  };
  mix(anchors, (size_t)m * d * sizeof(double));
  mix(&m, sizeof(m));
  mix(&d, sizeof(d));
  mix(&eps, sizeof(eps));
  mix(&device, sizeof(device));
  static std::mutex mu;
  static std::vector<std::pair<uint64_t, std::shared_ptr<DeviceGrid>>> lru;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : lru)
    if (e.first == h) return e.second;
  GridHost G;
  if (!build_grid(anchors, m, d, eps, G)) return nullptr;
  auto D = std::make_shared<DeviceGrid>();
  // candidate lists twice: indices (the point binner) and the candidates'
  // FP32 coordinates with the index in .w (the walk kernel's scan: one load
  // per candidate instead of two dependent ones)
  const size_t cb = G.cell.size() * 4, nb = G.cand.size() * 4;
  const size_t vo = (cb + nb + 15) & ~(size_t)15, vb = G.cand.size() * 16;
  std::vector<float> cv(G.cand.size() * 4, 0.0f);
  for (size_t k = 0; k < G.cand.size(); ++k) {
    const uint32_t a = G.cand[k];
    for (int j = 0; j < d; ++j) cv[4 * k + j] = (float)anchors[(size_t)a * d + j];
    std::memcpy(&cv[4 * k + 3], &a, 4);
  }
  D->device = device;
  if (cudaMalloc(&D->dev, vo + vb) != cudaSuccess) {
    D->dev = nullptr;
    cudaGetLastError();
    return nullptr;
  }
  if (cudaMemcpy(D->dev, G.cell.data(), cb, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(static_cast<char*>(D->dev) + cb, G.cand.data(), nb, cudaMemcpyHostToDevice) !=
          cudaSuccess ||
      cudaMemcpy(static_cast<char*>(D->dev) + vo, cv.data(), vb, cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  D->cell = static_cast<const uint32_t*>(D->dev);
  D->cand = reinterpret_cast<const uint32_t*>(static_cast<char*>(D->dev) + cb);
  D->candv = reinterpret_cast<const float4*>(static_cast<char*>(D->dev) + vo);
  for (int j = 0; j < 3; ++j) {
    D->lo[j] = G.lo[j];
    D->n[j] = G.n[j];
  }
  D->h = G.h;
  if (lru.size() >= 8) lru.erase(lru.begin());
  lru.push_back({h, D});
  return D;
}

// The chain a plan runs: EM_CHAIN_TANGENT exists (FP32, K != I) for 2D and
// 3D boxes and the 3D L-box without holes, the 3D ball without holes (rolling
// balls) and the 2D ball with at most one concentric hole (rolling disks,
// hole-tangent disks); elsewhere it runs EM_CHAIN_MAX.  Expects a validated
// geometry and a supported (precision, chain) pair.
int resolve_chain(const em_geometry* g, int precision, int chain, bool on_identity = false) {
  if (precision != EM_PREC_FP32 || chain != EM_CHAIN_TANGENT) return chain;
  const int d = (int)g->gi[0];
  const int64_t nh = g->gi[2], nn = g->gi_len >= 4 ? g->gi[3] : 0;
  bool id = true;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (g->ksqrt[i * d + j] != (i == j ? 1.0 : 0.0)) id = false;
  const bool ok2 = d == 2 && g->gi[1] == 1 && nh == 0 && nn == 0;
  const bool ok3 = d == 3 && g->gi[1] == 1 && nh == 0 && nn <= 1;
  const bool okb = d == 3 && g->gi[1] == 0 && nh == 0 && nn == 0;
  bool conc = nh == 1;
  for (int j = 0; conc && j < d; ++j) conc = g->gf[d + 1 + j] == g->gf[j];
  const bool okd = d == 2 && g->gi[1] == 0 && nn == 0 && (nh == 0 || conc);
  return ((ok2 || ok3 || okb || okd) && (!id || on_identity)) ? EM_CHAIN_TANGENT : EM_CHAIN_MAX;
}

int validate_geometry(const em_geometry* g) {
  if (!g || !g->gi || !g->gf || !g->comp_side || !g->ksqrt)
    return fail(EM_ERR_INVALID, "geometry: null pointer");
  if (g->gi_len < 3) return fail(EM_ERR_INVALID, "geometry: gi needs [d, outer_kind, n_holes]");
  const int64_t d = g->gi[0], ok = g->gi[1], nh = g->gi[2];
  const int64_t nn = g->gi_len >= 4 ? g->gi[3] : 0;
  if (d != 2 && d != 3) return fail(EM_ERR_INVALID, "geometry: dimension must be 2 or 3");
  if (ok != 0 && ok != 1) return fail(EM_ERR_INVALID, "geometry: outer kind must be 0 (ball) or 1 (box)");
  if (nh < 0 || nh > EM_MAX_HOLES) return fail(EM_ERR_UNSUPPORTED, "geometry: too many holes");
  if (nn < 0 || nn > 1) return fail(EM_ERR_INVALID, "geometry: at most one notch");
  if (nn && (d != 3 || ok != 1)) return fail(EM_ERR_INVALID, "geometry: the notch needs a 3D box");
  const int64_t need = (d + 1) * (1 + nh) + 2 * nn;
  if (g->gf_len < need) return fail(EM_ERR_INVALID, "geometry: gf too short");
  if (g->n_comp < 1 + nh + nn) return fail(EM_ERR_INVALID, "geometry: comp_side too short");
  for (int64_t c = 0; c < 1 + nh + nn; ++c)
    if (g->comp_side[c] != 0 && g->comp_side[c] != 1)
      return fail(EM_ERR_INVALID, "geometry: comp_side entries must be 0 or 1");
  return EM_OK;
}

int validate_side(const em_side* s, int d, const char* name, bool used) {
  if (!s) return fail(EM_ERR_INVALID, std::string(name) + ": null");
  if (s->wkind != 0 && s->wkind != 1)
    return fail(EM_ERR_INVALID, std::string(name) + ": weight kind must be 0 (voronoi) or 1 (idw)");
  if (s->wkind == 1 && s->n_anchors > 0 && (!s->idw_radii || s->idw_power < 1 || s->idw_power > 8))
    return fail(EM_ERR_INVALID, std::string(name) + ": IDW needs radii and a power in 1..8");
  if (s->n_anchors < 0 || s->n_blk < 0)
    return fail(EM_ERR_INVALID, std::string(name) + ": negative size");
  if (used && s->n_anchors == 0)
    return fail(EM_ERR_INVALID, std::string(name) +
                                    ": a boundary component maps to this side but it has no "
                                    "anchors (S/estimator.py:130-131)");
  if (s->n_anchors > 0 && (!s->anchors || !s->blk || !s->blkf || s->n_blk < 1))
    return fail(EM_ERR_INVALID, std::string(name) + ": missing anchors or blocks");
  if (s->n_blk > kMaxBlk) return fail(EM_ERR_UNSUPPORTED, std::string(name) + ": too many blocks");
  for (int64_t b = 0; b < (s->n_anchors > 0 ? s->n_blk : 0); ++b) {
    const int64_t kind = s->blk[3 * b], start = s->blk[3 * b + 1], count = s->blk[3 * b + 2];
    if (start < 0 || count < 1 || start + count > s->n_anchors)
      return fail(EM_ERR_INVALID, std::string(name) + ": block outside the anchor array");
    if ((kind == 1 || kind == 2) && d != 2)
      return fail(EM_ERR_INVALID, std::string(name) + ": circle/square blocks are 2D");
  }
  if (s->n_anchors >= (1LL << 31)) return fail(EM_ERR_UNSUPPORTED, "too many anchors");
  return EM_OK;
}

}  // namespace

extern "C" {

int em_abi_version(void) { return EM_ABI_VERSION; }

const char* em_build_info(void) {
  static const std::string info = std::string("abi=") + std::to_string(EM_ABI_VERSION) +
                                  " arch=sm_100a debug=" + std::to_string(EM_DEBUG) +
                                  " ref64=-fmad=false,-prec-div=true,-prec-sqrt=true"
                                  " f32=-fmad=true,-prec-div=false,-prec-sqrt=false " +
                                  f32_build_knobs();
  return info.c_str();
}

const char* em_last_error(void) { return g_last_error.c_str(); }

int em_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int em_device_info(int device, int* sm_count, int* clock_khz, int* cc_major, int* cc_minor) {
  cudaDeviceProp prop;
  EM_CUDA(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
  if (clock_khz) *clock_khz = clk;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return EM_OK;
}

int em_plan_destroy(em_plan* p) {
  if (p) {
    DeviceGuard dg(p->device);
    delete p;
  }
  return EM_OK;
}

int em_plan_create(const em_geometry* g, const em_side* s0, const em_side* s1,
                   const double* poles, const int64_t* pole_ids, int64_t n_poles, double eps,
                   int64_t max_steps, const em_options* opt, em_plan** out) {
  if (!out) return fail(EM_ERR_INVALID, "out is null");
  *out = nullptr;
  int rc = validate_geometry(g);
  if (rc) return rc;
  const int d = (int)g->gi[0];
  const int nh = (int)g->gi[2];
  const int nn = g->gi_len >= 4 ? (int)g->gi[3] : 0;
  bool used[2] = {false, false};
  for (int c = 0; c < 1 + nh + nn; ++c) used[g->comp_side[c]] = true;
  if ((rc = validate_side(s0, d, "side0", used[0]))) return rc;
  if ((rc = validate_side(s1, d, "side1", used[1]))) return rc;
  if (n_poles < 1 || !poles) return fail(EM_ERR_INVALID, "need at least one pole");
  if (!(eps > 0.0)) return fail(EM_ERR_INVALID, "eps must be positive");
  if (max_steps < 1) return fail(EM_ERR_INVALID, "max_steps must be >= 1");
  const em_options dflt{EM_PREC_REF64, EM_CHAIN_WOE, 0, 0, 0, 0};
  const em_options& o = opt ? *opt : dflt;
  if (o.precision != EM_PREC_REF64 && o.precision != EM_PREC_FP32)
    return fail(EM_ERR_INVALID, "unknown precision");
  if (o.chain != EM_CHAIN_WOE && o.chain != EM_CHAIN_MAX && o.chain != EM_CHAIN_TANGENT)
    return fail(EM_ERR_INVALID, "unknown chain");
  if (o.precision == EM_PREC_REF64 && o.chain != EM_CHAIN_WOE)
    return fail(EM_ERR_INVALID, "the REF64 mirror runs the reference chain only");
  if (o.precision == EM_PREC_FP32) {
    // the FP32 kernel's step margins are a few ulps of the domain scale; a
    // shell thinner than 2^-20 x scale (8 ulps) cannot be reached by steps
    // that keep those margins (the walks would stall at the budget): such
    // runs need the FP64 mirror
    const double dscale = std::max(1.0, std::fabs(g->gf[d]));
    if (eps < std::ldexp(dscale, -20))
      return fail(EM_ERR_UNSUPPORTED, "eps " + std::to_string(eps) +
                                          " is below the FP32 kernel's resolution (2^-20 x the "
                                          "domain scale): use precision ref64");
  }
  if (o.precision == EM_PREC_FP32 && o.block > 0 && o.block != 256)
    return fail(EM_ERR_UNSUPPORTED, "the FP32 kernel runs 256-thread blocks");
  int ndev = em_device_count();
  if (o.device < 0 || o.device >= ndev)
    return fail(EM_ERR_CUDA, "no such CUDA device (" + std::to_string(ndev) + " visible)");
  DeviceGuard dg(o.device);

  em_plan* p = new em_plan();
  p->device = o.device;
  p->precision = o.precision;
  p->chain = o.chain;
  const bool on_identity = (o.flags & EM_FLAG_TANGENT_ON_IDENTITY) != 0;
  p->chain = resolve_chain(g, o.precision, o.chain, on_identity);
  p->d = d;
  p->outer = nn ? OUTER_LBOX : (int)g->gi[1];
  p->n_holes = nh;
  p->n_notch = nn;
  p->n_poles = n_poles;
  p->n0 = s0->n_anchors;
  p->n1 = s1->n_anchors;
  p->block = o.block > 0 ? o.block : 256;
  p->flags = o.flags;
  auto bail = [&](int code) {
    delete p;
    return code;
  };
  p->stream = take_stream(o.device);
  p->ev0 = take_event(o.device);
  p->ev1 = take_event(o.device);
  p->ev_up = take_event(o.device);
  if (!p->stream || !p->ev0 || !p->ev1 || !p->ev_up)
    return bail(fail(EM_ERR_CUDA, std::string("stream/event: ") + cudaGetErrorString(cudaGetLastError())));

  bool ident = true;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (g->ksqrt[i * d + j] != (i == j ? 1.0 : 0.0)) ident = false;
  // the forced tangent chain runs its general (K != I) kernels on K = I
  if (on_identity && p->chain == EM_CHAIN_TANGENT) ident = false;
  p->ident = ident;

  const int64_t row = p->n0 + p->n1;
  // input staging: (offset, pointer slot) fixed up once the arena exists
  std::vector<char> stage;
  std::vector<std::pair<size_t, void**>> fixups;
  auto put = [&](const void* src, size_t bytes, void** slot) {
    const size_t off = (stage.size() + 255) & ~(size_t)255;
    stage.resize(off + bytes);
    if (bytes) std::memcpy(stage.data() + off, src, bytes);
    fixups.push_back({off, slot});
  };
  // outputs
  cudaError_t ce;
#define EM_ALLOC(buf, bytes)                                                          \
  if ((ce = (buf).alloc(bytes)) != cudaSuccess)                                       \
    return bail(fail(EM_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(ce)));
  p->blk_words = (size_t)n_poles * row + 3 * (size_t)n_poles + 8;
  EM_ALLOC(p->counts, p->blk_words * 8);
  p->blk_counts = p->counts.as<unsigned long long>();
  p->blk_stats = p->blk_counts + (size_t)n_poles * row;
  p->blk_misc = p->blk_stats + 3 * (size_t)n_poles;

  WorkOut w{};
  w.n_poles = n_poles;
  w.inv_poles = 1.0 / (double)n_poles;
  w.pole_ids = nullptr;  // set from the arena below
  w.ticket = p->blk_misc + 1;
  w.err_key = p->blk_misc;
  w.counts = p->blk_counts;
  w.row_len = (int)row;
  w.col_off1 = (int)p->n0;
  w.ssum = p->blk_stats;
  w.ssq = w.ssum + n_poles;
  w.smax = w.ssq + n_poles;
  w.smem_stats = 0;  // decided per launch (plan_launch)
  w.stat_copies = 1;

  const em_side* sides[2] = {s0, s1};
  // the FP64 side tables (exact binning, IDW weights): the REF64 mirror's,
  // and the FP32 path's IDW post-processing of its exits
  auto fill_sides64 = [&](Ref64Params& P) {
    P.d = d;
    for (int c = 0; c < 1 + nh + nn; ++c) P.comp_side[c] = g->comp_side[c];
    for (int s = 0; s < 2; ++s) {
      const em_side* S = sides[s];
      Side64& D = P.side[s];
      D.n_anchors = (int)S->n_anchors;
      D.n_blk = S->n_anchors > 0 ? (int)S->n_blk : 0;
      D.wkind = S->wkind;
      for (int b = 0; b < D.n_blk; ++b) {
        D.kind[b] = (int)S->blk[3 * b];
        D.start[b] = S->blk[3 * b + 1];
        D.count[b] = S->blk[3 * b + 2];
        D.cx[b] = S->blkf[4 * b];
        D.cy[b] = S->blkf[4 * b + 1];
        D.radius[b] = S->blkf[4 * b + 3];
        D.phase[b] = S->blk_phase ? S->blk_phase[b] : 0.0;
      }
      p->wkind[s] = S->wkind;
      p->idw_power[s] = S->idw_power;
      if (S->n_anchors > 0 && S->wkind == 1)
        put(S->idw_radii, (size_t)S->n_anchors * 8, (void**)&p->radii_dev[s]);
      if (S->n_anchors > 0) put(S->anchors, (size_t)S->n_anchors * d * 8, (void**)&D.anchors);
    }
  };
  if (p->precision == EM_PREC_REF64) {
    Ref64Params& P = p->p64;
    fill_sides64(P);
    P.d = d;
    P.outer_kind = (int)g->gi[1];
    P.n_holes = nh;
    P.n_notch = nn;
    const int64_t ngf = (d + 1) * (1 + nh) + 2 * nn;
    for (int64_t i = 0; i < ngf; ++i) P.gf[i] = g->gf[i];
    for (int i = 0; i < d * d; ++i) P.ks[i] = g->ksqrt[i];
    P.eps = eps;
    P.max_steps = max_steps;
    put(poles, (size_t)n_poles * d * 8, (void**)&P.poles);
    P.w = w;
  } else {
    F32Params& P = p->p32;
    // IDW families: FP32 walks, the FP64 weights of S/_kernel.pyx:323-369 in
    // a fixed (replicate) order on their exits (em_plan_run_raw)
    if (s0->wkind == 1 || s1->wkind == 1) fill_sides64(p->p64);
    // every closed-form constant of the kernel (plan_f32.cu)
    void* fb = f32_build_new(g, p->chain, ident, eps, max_steps, P);
    struct FbFree {
      void* b;
      ~FbFree() { f32_build_free(b); }
    } fb_free{fb};
    auto to_kernel = [&](const double* w, float* out) { f32_build_to_kernel(fb, w, out); };
    std::vector<float> pf(n_poles * 4, 0.0f);
    for (int64_t i = 0; i < n_poles; ++i) to_kernel(poles + i * d, &pf[i * 4]);
    put(pf.data(), (size_t)n_poles * 16, (void**)&P.poles);
    for (int s = 0; s < 2; ++s) {
      const em_side* S = sides[s];
      Side32& D = P.side[s];
      D.n_anchors = (int)S->n_anchors;
      D.n_blk = S->n_anchors > 0 ? (int)S->n_blk : 0;
      D.has_grid = 0;
      for (int b = 0; b < D.n_blk; ++b) {
        D.kind[b] = (int)S->blk[3 * b];
        D.start[b] = (int)S->blk[3 * b + 1];
        D.count[b] = (int)S->blk[3 * b + 2];
        D.cx[b] = (float)S->blkf[4 * b];
        D.cy[b] = (float)S->blkf[4 * b + 1];
        D.cz[b] = (float)S->blkf[4 * b + 2];
        D.radius[b] = (float)S->blkf[4 * b + 3];
        D.phase[b] = (float)(S->blk_phase ? S->blk_phase[b] : 0.0);
        const double cnt = (double)D.count[b];
        if (D.kind[b] == BLK_CIRCLE) D.scale[b] = (float)(cnt / (2.0 * M_PI));
        else if (D.kind[b] == BLK_SQUARE) D.scale[b] = (float)(cnt / (8.0 * S->blkf[4 * b + 3]));
        else D.scale[b] = 0.0f;
      }
      if (S->n_anchors == 0) continue;
      std::vector<float> af(S->n_anchors * 4, 0.0f);
      for (int64_t i = 0; i < S->n_anchors; ++i)
        for (int j = 0; j < d; ++j) af[i * 4 + j] = (float)S->anchors[i * d + j];
      put(af.data(), (size_t)S->n_anchors * 16, (void**)&D.anchors);
      // one uniform circle block: the Voronoi boundaries between consecutive
      // anchors are the bisector rays at (k - 1/2 + phase) 2 pi / count
      D.bis = nullptr;
      if (D.n_blk == 1 && D.kind[0] == BLK_CIRCLE && D.count[0] <= kBisMax) {
        const int cnt = D.count[0];
        const double ph = S->blk_phase ? S->blk_phase[0] : 0.0;
        std::vector<float> bt(2 * (size_t)cnt);
        for (int k = 0; k < cnt; ++k) {
          const double b = (k - 0.5 + ph) * (2.0 * M_PI / cnt);
          bt[2 * k] = (float)std::cos(b);
          bt[2 * k + 1] = (float)std::sin(b);
        }
        put(bt.data(), bt.size() * 4, (void**)&D.bis);
      }
      // one generic block covering the family: accelerate with the grid
      if (D.n_blk == 1 && D.kind[0] == BLK_GENERIC && S->n_anchors > 8) {
        if (auto G = cached_device_grid(S->anchors, S->n_anchors, d, eps, o.device)) {
          D.grid.cell = G->cell;
          D.grid.cand = G->cand;
          D.grid.candv = G->candv;
          D.has_grid = 1;
          for (int j = 0; j < 3; ++j) {
            D.grid.lo[j] = (float)G->lo[j];
            D.grid.n[j] = G->n[j];
          }
          D.grid.inv_h = (float)(1.0 / G->h);
          p->grids.push_back(G);
        }
      }
    }
    P.w = w;
    p->nh_mode = nh == 0 ? 0 : ((nh == 1 && d == 2 && g->gi[1] == 0) ? 1 : 2);
    // binner kind: one structured block per used side -> closed form
    {
      int kinds[2] = {-1, -1};
      bool uniform = true;
      for (int s2 = 0; s2 < 2; ++s2) {
        if (!used[s2]) continue;
        const Side32& D = P.side[s2];
        int k = -1;
        if (D.n_blk == 1 && D.kind[0] == BLK_CIRCLE) k = 1;
        else if (D.n_blk == 1 && D.kind[0] == BLK_SQUARE) k = 2;
        else if (D.has_grid) k = 3;
        kinds[s2] = k;
        if (k < 0) uniform = false;
      }
      int k = -1;
      for (int s2 = 0; s2 < 2; ++s2)
        if (used[s2]) {
          if (k < 0) k = kinds[s2];
          else if (k != kinds[s2]) uniform = false;
        }
      p->bink = (uniform && k > 0) ? k : 0;
    }
  }
  // pole ids last: the WorkOut copy inside the params is the live one
  if (pole_ids)
    put(pole_ids, (size_t)n_poles * 8,
        p->precision == EM_PREC_REF64 ? (void**)&p->p64.w.pole_ids : (void**)&p->p32.w.pole_ids);
  if (!stage.empty()) {
    EM_ALLOC(p->arena, stage.size());
    if ((ce = p->upin.alloc(stage.size())) != cudaSuccess)
      return bail(fail(EM_ERR_NOMEM, std::string("cudaHostAlloc: ") + cudaGetErrorString(ce)));
    std::memcpy(p->upin.p, stage.data(), stage.size());
    if ((ce = cudaMemcpyAsync(p->arena.p, p->upin.p, stage.size(), cudaMemcpyHostToDevice, p->stream)) !=
        cudaSuccess)
      return bail(fail(EM_ERR_CUDA, std::string("upload plan inputs: ") + cudaGetErrorString(ce)));
    for (auto& f : fixups) *f.second = static_cast<char*>(p->arena.p) + f.first;
  }
  if ((ce = cudaEventRecord(p->ev_up, p->stream)) != cudaSuccess)
    return bail(fail(EM_ERR_CUDA, std::string("upload event: ") + cudaGetErrorString(ce)));
#undef EM_ALLOC
  // persistent grid: SMs x resident blocks
  int per_sm = 4;
  if (p->precision == EM_PREC_FP32) {
    int nb = 0;
    if (f32_blocks_per_sm(p->d, p->outer, p->nh_mode, p->chain, p->ident, p->bink, &nb) == cudaSuccess && nb > 0)
      per_sm = nb;
  }
  p->grid = o.grid > 0 ? o.grid : sm_count_of(o.device) * per_sm * (256 / p->block > 0 ? 256 / p->block : 1);
  if (p->precision == EM_PREC_FP32) {
    p->pole_blocks = f32_has_pole_blocks(p->d, p->outer, p->nh_mode, p->chain, p->ident, p->bink);
    int nb2 = 0;
    if (!(o.flags & EM_FLAG_ONE_WALK_PER_LANE) && p->block == 256 &&
        f32x2_available(p->d, p->outer, p->nh_mode, p->chain, p->ident) &&
        f32x2_blocks_per_sm(p->d, p->outer, p->nh_mode, p->bink, &nb2) == cudaSuccess && nb2 > 0) {
      p->pack2 = true;
      p->grid2 = o.grid > 0 ? o.grid : sm_count_of(o.device) * nb2;
    }
  }
  *out = p;
  return EM_OK;
}

// The packed kernel pays off once every slot walks a few walks in a row (two
// slots per lane restart less evenly on tiny jobs: cfg3 at 1e6 walks -12%, at
// 1e7 walks +8%); counts are identical either way.  EM_FLAG_TWO_WALKS_PER_LANE
// forces it (tests of the small-job paths).
static bool use_pack2(const em_plan* p, int64_t total) {
  return (p->flags & EM_FLAG_TWO_WALKS_PER_LANE) || total >= 2000000;
}

static int plan_launch(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep, int mode,
                       unsigned long long* counts, unsigned long long* stats, cudaStream_t s) {
  if (n_rep < 0 || rep_start < 0) return fail(EM_ERR_INVALID, "negative replicate range");
  if (p->precision == EM_PREC_FP32 && n_rep > 2147483647LL)
    return fail(EM_ERR_UNSUPPORTED, "FP32 path: at most 2^31-1 replicates per pole per run");
  const int64_t total = p->n_poles * n_rep;
  if (n_rep > 0 && total / n_rep != p->n_poles) return fail(EM_ERR_INVALID, "walk count overflows");
  if ((double)total > 9.0e15) return fail(EM_ERR_INVALID, "walk count too large");
  // integer-count paths bin to the nearest anchor: an IDW family's
  // fractional rows come only from em_plan_run_raw (never silently Voronoi)
  if (mode == 0 && (p->wkind[0] || p->wkind[1]))
    return fail(EM_ERR_UNSUPPORTED, "IDW weight families need em_plan_run_raw (fractional rows)");
  WorkOut* w = p->precision == EM_PREC_REF64 ? &p->p64.w : &p->p32.w;
  w->rep_start = rep_start;
  w->n_rep = n_rep;
  w->total = total;
  // chunk size: enough chunks for ~8 per resident warp, 32..2048 replicates
  {
    const bool x2 = p->pack2 && mode == 0 && use_pack2(p, total);
    const double warps = (double)(x2 ? p->grid2 : p->grid) * (p->block / 32);
    long long rb = 32;
    while (rb < 2048 && (double)total / (warps * (x2 ? EM_X2_CHUNKS : EM_X1_CHUNKS)) >= (double)(rb * 2)) rb *= 2;
    w->rb = rb;
    w->n_chunks = (unsigned long long)p->n_poles * (unsigned long long)((n_rep + rb - 1) / rb);
    // minimum chunks (tiny jobs: ~1 walk per lane per chunk) mean a pole
    // change (a statistics flush) almost every walk: collect those flushes in
    // per-warp shared tables instead of global atomics (cfg1: 7x); bigger
    // jobs keep the register path (no end-of-kernel burst of table flushes;
    // a 32-pole row shard of cfg2 is 14% faster without the tables)
    w->smem_stats = (p->n_poles <= 128 && rb < 64) ? 1 : 0;
    // every lane flushes its per-pole statistics once per chunk, i.e. ~32
    // atomics per address per rb x n_poles walks; when that product is small
    // (few rows, e.g. a row shard, or few walks per row) the flushes
    // serialise on the 3 n_poles addresses in L2: spread them over copies
    // (folded by a second kernel) so every address sees <= 32 / 2^17 per walk
    // pole-block scheduler (north_star's exit binning): one block per
    // (pole, replicate range) in pole-major order, the row's histogram in
    // shared memory with warp-aggregated adds, one int64 flush per block.
    // Default where the count rows exceed half the 126 MB L2: there the
    // pole-cycling warps' direct atomics miss L2 and re-read / write back
    // DRAM sectors (cfg5: 40 GB of DRAM traffic for 267 MB of rows at full
    // scale; pole blocks: 0.44 GB, at 1% lower walks/s).  L2-resident rows
    // keep the pole-cycling persistent warps (1-4% faster there: no block
    // tails).  Blocks hold ~1/24 of a resident wave's share of the walks, so
    // the last wave's tail stays short.
    w->bc = 0;
    w->splits = 0;
    const int64_t row_len = p->n0 + p->n1;
    const double row_bytes = (double)p->n_poles * (double)row_len * 8.0;
    const bool want_blocks = (p->flags & EM_FLAG_POLE_BLOCKS) ||
                             (!(p->flags & EM_FLAG_PERSISTENT) && row_bytes > 64.0 * 1024 * 1024);
    if (p->precision == EM_PREC_FP32 && mode == 0 && p->pole_blocks && want_blocks &&
        row_len >= 1024 && row_len * 4 <= 160 * 1024 && n_rep >= 4096) {
      long long bc = 1024;
      while (bc < 65536 && (double)total / ((double)p->grid * 24.0) >= (double)(bc * 2)) bc *= 2;
      if (bc > n_rep) bc = n_rep;
      const long long splits = (n_rep + bc - 1) / bc;
      if ((double)p->n_poles * (double)splits < 2147483647.0) {
        w->bc = bc;
        w->splits = splits;
        w->smem_stats = 2;
      }
    }
    w->stat_copies = 1;
    if (p->precision == EM_PREC_FP32 && mode == 0 && w->smem_stats == 0) {
      int c = 1;
      while (c < 64 && (double)c * (double)rb * (double)p->n_poles < EM_STAT_SPREAD) c *= 2;
      w->stat_copies = c;
    }
  }
  w->counts = counts;
  unsigned long long* sdst = stats;
  if (w->stat_copies > 1) {
    const size_t need = (size_t)w->stat_copies * 3 * p->n_poles * 8;
    // growing returns the old buffer to the shared free list: a kernel of an
    // earlier (asynchronous) run may still write it, so wait for that run
    if (p->scopies.p && need > p->scopies.bytes && p->last_launch_stream &&
        cudaStreamSynchronize(p->last_launch_stream) != cudaSuccess)
      return fail(EM_ERR_CUDA, "synchronise before growing the statistics copies");
    if (p->scopies.alloc(need) != cudaSuccess)
      return fail(EM_ERR_NOMEM, "cudaMalloc: statistics copies");
    sdst = p->scopies.as<unsigned long long>();
  }
  w->ssum = sdst;
  w->ssq = sdst + p->n_poles;
  w->smax = sdst + 2 * p->n_poles;
  const int64_t row = p->n0 + p->n1;
  int64_t launches = 0;
  {
    // every output the kernels accumulate into, zeroed by ONE launch:
    // counts | stats | misc (one block on the host path), the statistics
    // copies (the fold then overwrites the caller's stats)
    unsigned long long* zp[4] = {nullptr, nullptr, nullptr, nullptr};
    long long zn[4] = {0, 0, 0, 0};
    if (mode == 0 && counts == p->blk_counts) {
      zp[0] = p->blk_counts;
      zn[0] = (long long)p->blk_words;
    } else {
      if (mode == 0) {
        zp[0] = counts;
        zn[0] = (long long)p->n_poles * row;
        if (w->stat_copies == 1) {
          zp[1] = stats;
          zn[1] = 3 * (long long)p->n_poles;
        }
      }
      zp[2] = p->blk_misc;
      zn[2] = 8;
    }
    if (w->stat_copies > 1) {
      zp[3] = sdst;
      zn[3] = (long long)w->stat_copies * 3 * p->n_poles;
    }
    cudaError_t ze = launch_zero_ranges(zp, zn, 4, s);
    if (ze != cudaSuccess) return fail(EM_ERR_CUDA, std::string("zero outputs: ") + cudaGetErrorString(ze));
    launches = 1;
  }
  p->last_timed = false;
  if (total > 0) {
    const bool x2 = p->pack2 && mode == 0 && use_pack2(p, total);
    const int64_t lanes_needed = x2 ? (total + 63) / 64 * 32 : (total + 31) / 32 * 32;
    int grid = x2 ? p->grid2 : p->grid;
    const int64_t blocks_needed = (lanes_needed + p->block - 1) / p->block;
    if (blocks_needed < grid) grid = (int)std::max<int64_t>(1, blocks_needed);
    EM_CUDA(cudaEventRecord(p->ev0, s));
    cudaError_t e;
    if (s != p->stream) EM_CUDA(cudaStreamWaitEvent(s, p->ev_up, 0));
    if (p->precision == EM_PREC_REF64) {
      p->p64.seed = seed;
      for (int r = 0; r < 10; ++r) p->p64.rk0[r] = seed + (unsigned long long)r * 0x9E3779B97F4A7C15ULL;
      e = launch_ref64(p->p64, mode, grid, p->block, s);
    } else {
      p->p32.key0 = (unsigned)(seed & 0xffffffffULL);
      p->p32.key1 = (unsigned)(seed >> 32);
      p->p32.rk = philox32_schedule(p->p32.key0, p->p32.key1);
      if (x2)
        e = launch_f32x2(p->p32, p->d, p->outer, p->nh_mode, p->bink, grid, p->block, s);
      else
        e = launch_f32(p->p32, p->d, p->outer, p->nh_mode, mode, p->chain, p->ident, p->bink,
                       grid, p->block, s);
    }
    if (e != cudaSuccess) return fail(EM_ERR_CUDA, std::string("walk kernel launch: ") + cudaGetErrorString(e));
    launches += 1;
    if (w->stat_copies > 1) {
      e = launch_stats_fold(sdst, w->stat_copies, p->n_poles, stats, s);
      if (e != cudaSuccess) return fail(EM_ERR_CUDA, std::string("statistics fold: ") + cudaGetErrorString(e));
      launches += 1;
    }
    p->last_timed = true;
    EM_CUDA(cudaEventRecord(p->ev1, s));
  }
  p->last_launches = launches;
  p->last_walks = total;
  if (mode == 0) p->last_sched = w->smem_stats;
  if (mode == 0) p->last_lanes = (p->pack2 && use_pack2(p, total)) ? 2 : 1;
  p->last_launch_stream = s;
  return EM_OK;
}

static int plan_finish(em_plan* p, cudaStream_t s, int64_t n_rep, em_outputs* out,
                       const unsigned long long* host_stats) {
  unsigned long long errv = 0;
  if (p->pin.p && p->pin_valid) {
    EM_CUDA(cudaStreamSynchronize(s));
    errv = reinterpret_cast<const unsigned long long*>(p->pin.p)[p->blk_words - 8];
  } else {
    EM_CUDA(cudaMemcpyAsync(&errv, p->blk_misc, 8, cudaMemcpyDeviceToHost, s));
    EM_CUDA(cudaStreamSynchronize(s));
  }
  const unsigned long long err = errv ? ~errv : ~0ULL;
  float ms = 0.0f;
  if (p->last_timed) {
    EM_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  }
  p->last_ms = ms;
  if (host_stats) {
    int64_t st = 0;
    for (int64_t i = 0; i < p->n_poles; ++i) st += (int64_t)host_stats[i];
    p->last_steps = st;
  }
  if (err != ~0ULL) {
    if (out) {
      out->err_pole = n_rep > 0 ? (int64_t)(err / (unsigned long long)n_rep) : 0;
      out->err_rep = n_rep > 0 ? (int64_t)(err % (unsigned long long)n_rep) : 0;
    }
    return EM_BUDGET;
  }
  if (out) out->err_pole = out->err_rep = -1;
  return EM_OK;
}

// run + one D2H of the whole output block into the plan's pinned staging
static int plan_run_staged(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                           em_outputs* out, bool f64 = false) {
  DeviceGuard dg(p->device);
  int rc = plan_launch(p, seed, rep_start, n_rep, 0, p->blk_counts, p->blk_stats, p->stream);
  if (rc) return rc;
  if (f64) {  // the rows as float64 in place (exact: counts < 2^53), on the device
    cudaError_t e = launch_rows_to_f64(p->blk_counts, p->n_poles * (p->n0 + p->n1), p->stream);
    if (e != cudaSuccess) return fail(EM_ERR_CUDA, std::string("rows to float64: ") + cudaGetErrorString(e));
    p->last_launches += 1;
  }
  cudaError_t ce = p->pin.alloc(p->blk_words * 8);
  if (ce != cudaSuccess) return fail(EM_ERR_NOMEM, std::string("cudaHostAlloc: ") + cudaGetErrorString(ce));
  EM_CUDA(cudaMemcpyAsync(p->pin.p, p->blk_counts, p->blk_words * 8, cudaMemcpyDeviceToHost, p->stream));
  p->pin_valid = true;
  rc = plan_finish(p, p->stream, n_rep, out,
                   reinterpret_cast<const unsigned long long*>(p->pin.p) +
                       (size_t)p->n_poles * (p->n0 + p->n1));
  p->pin_valid = false;
  return rc;
}

int em_plan_run(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep, em_outputs* out) {
  if (!p || !out || !out->counts || !out->steps_sum || !out->steps_sq || !out->steps_max)
    return fail(EM_ERR_INVALID, "plan/outputs null");
  int rc = plan_run_staged(p, seed, rep_start, n_rep, out);
  if (rc < 0) return rc;
  const size_t nc = (size_t)p->n_poles * (p->n0 + p->n1);
  const int64_t* h = reinterpret_cast<const int64_t*>(p->pin.p);
  std::memcpy(out->counts, h, nc * 8);
  std::memcpy(out->steps_sum, h + nc, p->n_poles * 8);
  std::memcpy(out->steps_sq, h + nc + p->n_poles, p->n_poles * 8);
  std::memcpy(out->steps_max, h + nc + 2 * p->n_poles, p->n_poles * 8);
  return rc;
}

int em_plan_run_host(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                     const int64_t** block, int64_t* err_pole, int64_t* err_rep) {
  if (!p || !block) return fail(EM_ERR_INVALID, "plan/block null");
  em_outputs o{};
  int rc = plan_run_staged(p, seed, rep_start, n_rep, &o);
  if (rc < 0) return rc;
  *block = reinterpret_cast<const int64_t*>(p->pin.p);
  if (err_pole) *err_pole = o.err_pole;
  if (err_rep) *err_rep = o.err_rep;
  return rc;
}

namespace {
struct Detached {
  int dev;
  size_t bytes;
};
std::mutex g_detached_mu;
std::unordered_map<void*, Detached> g_detached;
}  // namespace

int em_plan_run_host_f64(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                         const int64_t** block, int64_t* err_pole, int64_t* err_rep) {
  if (!p || !block) return fail(EM_ERR_INVALID, "plan/block null");
  em_outputs o{};
  int rc = plan_run_staged(p, seed, rep_start, n_rep, &o, true);
  if (rc < 0) return rc;
  *block = reinterpret_cast<const int64_t*>(p->pin.p);
  if (err_pole) *err_pole = o.err_pole;
  if (err_rep) *err_rep = o.err_rep;
  return rc;
}

int em_plan_detach_block(em_plan* p, int64_t** block) {
  if (!p || !block) return fail(EM_ERR_INVALID, "plan/block null");
  if (!p->pin.p) return fail(EM_ERR_INVALID, "no staged block to detach");
  {
    std::lock_guard<std::mutex> lk(g_detached_mu);
    g_detached[p->pin.p] = {p->pin.dev, p->pin.bytes};
  }
  *block = static_cast<int64_t*>(p->pin.p);
  p->pin.p = nullptr;
  p->pin.bytes = 0;
  return EM_OK;
}

int em_host_block_free(void* block) {
  if (!block) return EM_OK;
  Detached d;
  {
    std::lock_guard<std::mutex> lk(g_detached_mu);
    auto it = g_detached.find(block);
    if (it == g_detached.end()) return fail(EM_ERR_INVALID, "not a detached block");
    d = it->second;
    g_detached.erase(it);
  }
  BufCache& c = cache_of(d.dev);
  std::lock_guard<std::mutex> lk(c.mu);
  c.free_pinned.push_back({d.bytes, block});
  return EM_OK;
}

int em_plan_run_device(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep,
                       em_outputs* dev_out, void* stream) {
  if (!p || !dev_out || !dev_out->counts || !dev_out->steps_sum)
    return fail(EM_ERR_INVALID, "plan/outputs null");
  DeviceGuard dg(p->device);
  cudaStream_t s = stream ? (cudaStream_t)stream : p->stream;
  // steps_sq / steps_max must follow steps_sum contiguously (one stats block)
  if (dev_out->steps_sq != dev_out->steps_sum + p->n_poles ||
      dev_out->steps_max != dev_out->steps_sum + 2 * p->n_poles)
    return fail(EM_ERR_INVALID, "device stats must be one contiguous (3, n_poles) block");
  int rc = plan_launch(p, seed, rep_start, n_rep, 0,
                       reinterpret_cast<unsigned long long*>(dev_out->counts),
                       reinterpret_cast<unsigned long long*>(dev_out->steps_sum), s);
  if (rc) return rc;
  // asynchronous: nothing waits for the kernel here; em_plan_check reads the
  // budget-error word (and the kernel time) once the caller has synchronised
  p->last_n_rep = n_rep;
  p->last_stream = s;
  return EM_OK;
}

int em_plan_check(em_plan* p, int64_t* err_pole, int64_t* err_rep) {
  if (!p) return fail(EM_ERR_INVALID, "plan null");
  DeviceGuard dg(p->device);
  em_outputs o{};
  int rc = plan_finish(p, p->last_stream ? p->last_stream : p->stream, p->last_n_rep, &o, nullptr);
  if (err_pole) *err_pole = o.err_pole;
  if (err_rep) *err_rep = o.err_rep;
  return rc;
}

int em_plan_last_stats(const em_plan* p, double* kernel_ms, int64_t* walks, int64_t* steps) {
  if (!p) return fail(EM_ERR_INVALID, "plan null");
  if (kernel_ms) *kernel_ms = p->last_ms;
  if (walks) *walks = p->last_walks;
  if (steps) *steps = p->last_steps;
  return EM_OK;
}

int em_plan_chain(const em_plan* p) { return p ? p->chain : -1; }

int em_resolve_chain(const em_geometry* g, int precision, int chain) {
  int rc = validate_geometry(g);
  if (rc) return rc;
  if (precision != EM_PREC_REF64 && precision != EM_PREC_FP32)
    return fail(EM_ERR_INVALID, "unknown precision");
  if (chain != EM_CHAIN_WOE && chain != EM_CHAIN_MAX && chain != EM_CHAIN_TANGENT)
    return fail(EM_ERR_INVALID, "unknown chain");
  if (precision == EM_PREC_REF64 && chain != EM_CHAIN_WOE)
    return fail(EM_ERR_INVALID, "the REF64 mirror runs the reference chain only");
  return resolve_chain(g, precision, chain);
}

int em_plan_last_launches(const em_plan* p, int64_t* launches) {
  if (!p || !launches) return fail(EM_ERR_INVALID, "null");
  *launches = p->last_launches;
  return EM_OK;
}

int em_plan_last_scheduler(const em_plan* p) { return p ? p->last_sched : -1; }
int em_plan_walks_per_lane(const em_plan* p) { return p ? (p->pack2 ? 2 : 1) : -1; }
int em_plan_last_walks_per_lane(const em_plan* p) { return p ? p->last_lanes : -1; }

int64_t em_plan_n_bins(const em_plan* p, int side) {
  if (!p) return -1;
  return side == 0 ? p->n0 : p->n1;
}

int em_run_accumulate(const em_geometry* g, const em_side* s0, const em_side* s1,
                      const double* poles, const int64_t* pole_ids, int64_t n_poles,
                      uint64_t seed, double eps, int64_t max_steps, int64_t n_rep,
                      const em_options* opt, em_outputs* out) {
  em_plan* p = nullptr;
  int rc = em_plan_create(g, s0, s1, poles, pole_ids, n_poles, eps, max_steps, opt, &p);
  if (rc) return rc;
  rc = em_plan_run(p, seed, 0, n_rep, out);
  em_plan_destroy(p);
  return rc;
}

int em_run_exits(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep, double* x_out,
                 int64_t* steps_out, int64_t* comp_out, int64_t* err_pole, int64_t* err_rep) {
  if (!p || !x_out || !steps_out || !comp_out) return fail(EM_ERR_INVALID, "null");
  DeviceGuard dg(p->device);
  const int64_t total = p->n_poles * n_rep;
  cudaError_t ce;
  if ((ce = p->xo.alloc((size_t)std::max<int64_t>(total, 1) * p->d * 8)) != cudaSuccess ||
      (ce = p->so.alloc((size_t)std::max<int64_t>(total, 1) * 8)) != cudaSuccess ||
      (ce = p->co.alloc((size_t)std::max<int64_t>(total, 1) * 8)) != cudaSuccess)
    return fail(EM_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(ce));
  WorkOut* w = p->precision == EM_PREC_REF64 ? &p->p64.w : &p->p32.w;
  w->x_out = p->xo.as<double>();
  w->steps_out = p->so.as<long long>();
  w->comp_out = p->co.as<long long>();
  int rc = plan_launch(p, seed, rep_start, n_rep, 1, p->blk_counts, p->blk_stats, p->stream);
  if (rc) return rc;
  if (total > 0) {
    EM_CUDA(cudaMemcpyAsync(x_out, p->xo.p, total * p->d * 8, cudaMemcpyDeviceToHost, p->stream));
    EM_CUDA(cudaMemcpyAsync(steps_out, p->so.p, total * 8, cudaMemcpyDeviceToHost, p->stream));
    EM_CUDA(cudaMemcpyAsync(comp_out, p->co.p, total * 8, cudaMemcpyDeviceToHost, p->stream));
  }
  em_outputs o{};
  rc = plan_finish(p, p->stream, n_rep, &o, nullptr);
  if (err_pole) *err_pole = o.err_pole;
  if (err_rep) *err_rep = o.err_rep;
  return rc;
}

int em_plan_run_raw(em_plan* p, uint64_t seed, int64_t rep_start, int64_t n_rep, int64_t chunk,
                    const double* init0, const double* init1, double* raw0, double* raw1,
                    int64_t* stats, int64_t* idw_fallbacks, int64_t* err_pole, int64_t* err_rep) {
  if (!p || !raw0 || !raw1 || !stats) return fail(EM_ERR_INVALID, "null");
  if (p->precision == EM_PREC_FP32 && !p->wkind[0] && !p->wkind[1])
    return fail(EM_ERR_UNSUPPORTED, "FP32 raw rows are for IDW families (Voronoi: em_plan_run)");
  if (n_rep < 0 || rep_start < 0) return fail(EM_ERR_INVALID, "negative replicate range");
  DeviceGuard dg(p->device);
  const int64_t total = p->n_poles * n_rep;
  const int d = p->d;
  cudaError_t ce;
  const size_t nw = (size_t)std::max<int64_t>(total, 1);
  if ((ce = p->xo.alloc(nw * d * 8)) != cudaSuccess || (ce = p->so.alloc(nw * 8)) != cudaSuccess ||
      (ce = p->co.alloc(nw * 8)) != cudaSuccess || (ce = p->ikind.alloc(nw * 4)) != cudaSuccess ||
      (ce = p->iidx.alloc(nw * 8)) != cudaSuccess || (ce = p->itot.alloc(nw * 8)) != cudaSuccess ||
      (ce = p->iside.alloc(nw * 4)) != cudaSuccess ||
      (ce = p->iraw0.alloc((size_t)std::max<int64_t>(p->n_poles * p->n0, 1) * 8)) != cudaSuccess ||
      (ce = p->iraw1.alloc((size_t)std::max<int64_t>(p->n_poles * p->n1, 1) * 8)) != cudaSuccess)
    return fail(EM_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(ce));
  WorkOut* w = p->precision == EM_PREC_REF64 ? &p->p64.w : &p->p32.w;
  w->x_out = p->xo.as<double>();
  w->steps_out = p->so.as<long long>();
  w->comp_out = p->co.as<long long>();
  int rc = plan_launch(p, seed, rep_start, n_rep, 1, p->blk_counts, p->blk_stats, p->stream);
  if (rc) return rc;
  const double* d_init0 = nullptr;
  const double* d_init1 = nullptr;
  if (init0 && init1) {
    if ((ce = p->iinit0.alloc((size_t)std::max<int64_t>(p->n_poles * p->n0, 1) * 8)) != cudaSuccess ||
        (ce = p->iinit1.alloc((size_t)std::max<int64_t>(p->n_poles * p->n1, 1) * 8)) != cudaSuccess)
      return fail(EM_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(ce));
    EM_CUDA(cudaMemcpyAsync(p->iinit0.p, init0, p->n_poles * p->n0 * 8, cudaMemcpyHostToDevice, p->stream));
    EM_CUDA(cudaMemcpyAsync(p->iinit1.p, init1, p->n_poles * p->n1 * 8, cudaMemcpyHostToDevice, p->stream));
    d_init0 = p->iinit0.as<double>();
    d_init1 = p->iinit1.as<double>();
  }
  // budget check before binning: outputs are meaningless after a failure
  unsigned long long err = ~0ULL;
  EM_CUDA(cudaMemcpyAsync(&err, p->blk_misc, 8, cudaMemcpyDeviceToHost, p->stream));
  EM_CUDA(cudaStreamSynchronize(p->stream));
  err = err ? ~err : ~0ULL;
  if (err != ~0ULL) {
    if (err_pole) *err_pole = n_rep > 0 ? (int64_t)(err / (unsigned long long)n_rep) : 0;
    if (err_rep) *err_rep = n_rep > 0 ? (int64_t)(err % (unsigned long long)n_rep) : 0;
    return EM_BUDGET;
  }
  const Side64& S0 = p->p64.side[0];
  const Side64& S1 = p->p64.side[1];
  cudaError_t e = launch_idw(p->p64, p->xo.as<double>(), p->co.as<long long>(), p->n_poles, n_rep,
                             chunk > 0 ? chunk : std::max<int64_t>(n_rep, 1),
                             S0.anchors, p->radii_dev[0], (int)p->n0, p->idw_power[0], p->wkind[0],
                             S1.anchors, p->radii_dev[1], (int)p->n1, p->idw_power[1], p->wkind[1],
                             p->ikind.as<int>(), p->iidx.as<long long>(), p->itot.as<double>(),
                             p->iside.as<int>(), p->iraw0.as<double>(), p->iraw1.as<double>(),
                             d_init0, d_init1, p->stream);
  if (e != cudaSuccess) return fail(EM_ERR_CUDA, std::string("idw kernels: ") + cudaGetErrorString(e));
  EM_CUDA(cudaMemcpyAsync(raw0, p->iraw0.p, p->n_poles * p->n0 * 8, cudaMemcpyDeviceToHost, p->stream));
  EM_CUDA(cudaMemcpyAsync(raw1, p->iraw1.p, p->n_poles * p->n1 * 8, cudaMemcpyDeviceToHost, p->stream));
  std::vector<long long> steps(nw);
  std::vector<double> tot(nw);
  if (total > 0) {
    EM_CUDA(cudaMemcpyAsync(steps.data(), p->so.p, total * 8, cudaMemcpyDeviceToHost, p->stream));
    EM_CUDA(cudaMemcpyAsync(tot.data(), p->itot.p, total * 8, cudaMemcpyDeviceToHost, p->stream));
  }
  EM_CUDA(cudaStreamSynchronize(p->stream));
  int64_t fb = 0;
  for (int64_t i = 0; i < p->n_poles; ++i) {
    int64_t ss = 0, sq = 0, sm = 0;
    for (int64_t r = 0; r < n_rep; ++r) {
      const int64_t st = steps[i * n_rep + r];
      ss += st;
      sq += st * st;
      sm = st > sm ? st : sm;
      if (tot[i * n_rep + r] < 0.0) ++fb;
    }
    stats[i] = ss;
    stats[p->n_poles + i] = sq;
    stats[2 * p->n_poles + i] = sm;
  }
  if (idw_fallbacks) *idw_fallbacks = fb;
  if (err_pole) *err_pole = -1;
  if (err_rep) *err_rep = -1;
  p->last_launches += 2;  // + the IDW normaliser and scatter kernels
  return EM_OK;
}

int em_bin_points(em_plan* p, const double* pts, int64_t n, int64_t* comp, int64_t* side,
                  int64_t* bin) {
  if (!p || (n > 0 && (!pts || !comp || !side || !bin))) return fail(EM_ERR_INVALID, "null");
  if (n <= 0) return EM_OK;
  DeviceGuard dg(p->device);
  DevBuf dp, dc, ds, db;
  cudaError_t ce;
  if ((ce = dp.alloc((size_t)n * p->d * 8)) != cudaSuccess || (ce = dc.alloc((size_t)n * 8)) != cudaSuccess ||
      (ce = ds.alloc((size_t)n * 8)) != cudaSuccess || (ce = db.alloc((size_t)n * 8)) != cudaSuccess)
    return fail(EM_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(ce));
  EM_CUDA(cudaMemcpyAsync(dp.p, pts, (size_t)n * p->d * 8, cudaMemcpyHostToDevice, p->stream));
  cudaError_t e = p->precision == EM_PREC_REF64
                      ? launch_bin_points_ref64(p->p64, dp.as<double>(), n, dc.as<long long>(),
                                                ds.as<long long>(), db.as<long long>(), p->stream)
                      : launch_bin_points_f32(p->p32, p->d, p->outer, dp.as<double>(), n,
                                              dc.as<long long>(), ds.as<long long>(),
                                              db.as<long long>(), p->stream);
  if (e != cudaSuccess) return fail(EM_ERR_CUDA, std::string("bin points: ") + cudaGetErrorString(e));
  EM_CUDA(cudaMemcpyAsync(comp, dc.p, (size_t)n * 8, cudaMemcpyDeviceToHost, p->stream));
  EM_CUDA(cudaMemcpyAsync(side, ds.p, (size_t)n * 8, cudaMemcpyDeviceToHost, p->stream));
  EM_CUDA(cudaMemcpyAsync(bin, db.p, (size_t)n * 8, cudaMemcpyDeviceToHost, p->stream));
  EM_CUDA(cudaStreamSynchronize(p->stream));
  return EM_OK;
}

int em_debug_step(em_plan* p, const double* x, const uint32_t* words, int64_t n, double* y,
                  float* mask) {
  if (!p || (n > 0 && (!x || !words || !y || !mask))) return fail(EM_ERR_INVALID, "null");
  if (p->precision != EM_PREC_FP32) return fail(EM_ERR_UNSUPPORTED, "em_debug_step: FP32 plans only");
  if (n <= 0) return EM_OK;
  DeviceGuard dg(p->device);
  DevBuf dx, dw, dy, dm;
  cudaError_t ce;
  if ((ce = dx.alloc((size_t)n * p->d * 8)) != cudaSuccess || (ce = dw.alloc((size_t)n * 8)) != cudaSuccess ||
      (ce = dy.alloc((size_t)n * p->d * 8)) != cudaSuccess || (ce = dm.alloc((size_t)n * 4)) != cudaSuccess)
    return fail(EM_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(ce));
  EM_CUDA(cudaMemcpyAsync(dx.p, x, (size_t)n * p->d * 8, cudaMemcpyHostToDevice, p->stream));
  EM_CUDA(cudaMemcpyAsync(dw.p, words, (size_t)n * 8, cudaMemcpyHostToDevice, p->stream));
  cudaError_t e = launch_debug_step(p->p32, p->d, p->outer, p->nh_mode, p->chain, p->ident,
                                    dx.as<double>(), dw.as<unsigned>(), n, dy.as<double>(),
                                    dm.as<float>(), p->stream);
  if (e == cudaErrorInvalidValue) return fail(EM_ERR_UNSUPPORTED, "em_debug_step: no such kernel family");
  if (e != cudaSuccess) return fail(EM_ERR_CUDA, std::string("debug step: ") + cudaGetErrorString(e));
  EM_CUDA(cudaMemcpyAsync(y, dy.p, (size_t)n * p->d * 8, cudaMemcpyDeviceToHost, p->stream));
  EM_CUDA(cudaMemcpyAsync(mask, dm.p, (size_t)n * 4, cudaMemcpyDeviceToHost, p->stream));
  EM_CUDA(cudaStreamSynchronize(p->stream));
  return EM_OK;
}

// ---- chunk-level drop-ins (the reference's _impl contract) ----

int em_walk_exits_chunk(const em_geometry* g, const double* pole_xy, int64_t pole_index,
                        int64_t rep_start, int64_t rep_end, uint64_t seed, double eps,
                        int64_t max_steps, int device, double* x_out, int64_t* steps_out,
                        int64_t* comp_out, int64_t* err_rep) {
  if (rep_end < rep_start) return fail(EM_ERR_INVALID, "rep_end < rep_start");
  const em_side empty{nullptr, 0, nullptr, nullptr, 0, 0, 2, nullptr, nullptr};
  // exits mode never bins: pretend every component maps to side 0 of an
  // empty family by using a geometry copy whose comp_side is ignored
  em_options o{EM_PREC_REF64, EM_CHAIN_WOE, device, 0, 0, 0};
  em_geometry g2 = *g;
  std::vector<int8_t> cs(std::max<int64_t>(g->n_comp, 1), 0);
  g2.comp_side = cs.data();
  g2.n_comp = (int64_t)cs.size();
  // a dummy one-anchor family keeps validation happy without binning
  const double dummy[3] = {0, 0, 0};
  const int64_t blk[3] = {0, 0, 1};
  const double blkf[4] = {0, 0, 0, 0};
  const em_side one{dummy, 1, blk, blkf, 1, 0, 2, nullptr, nullptr};
  em_plan* p = nullptr;
  const int64_t pid = pole_index;
  int rc = em_plan_create(&g2, &one, &empty, pole_xy, &pid, 1, eps, max_steps, &o, &p);
  if (rc) return rc;
  int64_t ep = -1, er = -1;
  rc = em_run_exits(p, seed, rep_start, rep_end - rep_start, x_out, steps_out, comp_out, &ep, &er);
  em_plan_destroy(p);
  if (err_rep) *err_rep = (rc == EM_BUDGET) ? rep_start + er : -1;
  if (rc == EM_BUDGET) {
    for (int64_t i = 0; i < rep_end - rep_start; ++i) comp_out[i] = 0;
    return EM_OK;
  }
  return rc;
}

int em_accumulate_chunk(const em_geometry* g, const double* pole_xy, int64_t pole_index,
                        int64_t rep_start, int64_t rep_end, uint64_t seed, double eps,
                        int64_t max_steps, const em_side* s0, const em_side* s1, int device,
                        double* out0, double* out1, int64_t* stats, int64_t* err_rep) {
  if (rep_end < rep_start) return fail(EM_ERR_INVALID, "rep_end < rep_start");
  em_options o{EM_PREC_REF64, EM_CHAIN_WOE, device, 0, 0, 0};
  em_plan* p = nullptr;
  const int64_t pid = pole_index;
  int rc = em_plan_create(g, s0, s1, pole_xy, &pid, 1, eps, max_steps, &o, &p);
  if (rc) return rc;
  if (s0->wkind == 1 || s1->wkind == 1) {
    // fractional weights: accumulate in place from out0/out1, walk order
    std::vector<double> r0(std::max<int64_t>(s0->n_anchors, 1)), r1(std::max<int64_t>(s1->n_anchors, 1));
    int64_t st[3] = {0, 0, 0}, fb = 0, ep = -1, er = -1;
    rc = em_plan_run_raw(p, seed, rep_start, rep_end - rep_start, 0, out0, out1, r0.data(),
                         r1.data(), st, &fb, &ep, &er);
    em_plan_destroy(p);
    if (rc == EM_BUDGET) {
      if (stats) stats[0] = stats[1] = stats[2] = stats[3] = 0;
      if (err_rep) *err_rep = rep_start + er;
      return EM_OK;
    }
    if (rc) return rc;
    for (int64_t i = 0; i < s0->n_anchors; ++i) out0[i] = r0[i];
    for (int64_t i = 0; i < s1->n_anchors; ++i) out1[i] = r1[i];
    if (stats) {
      stats[0] = st[0];
      stats[1] = st[1];
      stats[2] = st[2];
      stats[3] = fb;
    }
    if (err_rep) *err_rep = -1;
    return EM_OK;
  }
  const int64_t row = s0->n_anchors + s1->n_anchors;
  std::vector<int64_t> counts(std::max<int64_t>(row, 1));
  int64_t ss = 0, sq = 0, sm = 0;
  em_outputs out{counts.data(), &ss, &sq, &sm, -1, -1};
  rc = em_plan_run(p, seed, rep_start, rep_end - rep_start, &out);
  em_plan_destroy(p);
  if (rc == EM_BUDGET) {
    if (stats) stats[0] = stats[1] = stats[2] = stats[3] = 0;
    if (err_rep) *err_rep = rep_start + out.err_rep;
    return EM_OK;
  }
  if (rc) return rc;
  for (int64_t i = 0; i < s0->n_anchors; ++i) out0[i] += (double)counts[i];
  for (int64_t i = 0; i < s1->n_anchors; ++i) out1[i] += (double)counts[s0->n_anchors + i];
  if (stats) {
    stats[0] = ss;
    stats[1] = sq;
    stats[2] = sm;
    stats[3] = 0;
  }
  if (err_rep) *err_rep = -1;
  return EM_OK;
}

int em_fp32_peak(int device, double* flops_per_s, double* ms_out) {
  DeviceGuard dg(device);
  const int sms = sm_count_of(device);
  float* buf = nullptr;
  EM_CUDA(cudaMalloc(&buf, 1024 * 4));
  cudaEvent_t a, b;
  EM_CUDA(cudaEventCreate(&a));
  EM_CUDA(cudaEventCreate(&b));
  const int grid = sms * 8, block = 256, iters = 1 << 14;
  cudaError_t e = launch_ffma_peak(buf, iters, grid, block, 0);  // warm-up
  if (e != cudaSuccess) return fail(EM_ERR_CUDA, cudaGetErrorString(e));
  EM_CUDA(cudaEventRecord(a, 0));
  e = launch_ffma_peak(buf, iters, grid, block, 0);
  if (e != cudaSuccess) return fail(EM_ERR_CUDA, cudaGetErrorString(e));
  EM_CUDA(cudaEventRecord(b, 0));
  EM_CUDA(cudaEventSynchronize(b));
  float ms = 0.0f;
  EM_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  // one FFMA = one FP32 lane-op in the SURVEY's F_step convention
  const double ops = (double)grid * block * iters * 8.0;
  if (flops_per_s) *flops_per_s = ops / (ms * 1e-3);
  if (ms_out) *ms_out = ms;
  return EM_OK;
}

// known-answer hooks for the RNG golden tests
int em_philox4x64_blocks(const uint64_t* in6, uint64_t* out4, int n, int device) {
  DeviceGuard dg(device);
  unsigned long long *din = nullptr, *dout = nullptr;
  EM_CUDA(cudaMalloc(&din, (size_t)n * 48));
  EM_CUDA(cudaMalloc(&dout, (size_t)n * 32));
  EM_CUDA(cudaMemcpy(din, in6, (size_t)n * 48, cudaMemcpyHostToDevice));
  cudaError_t e = launch_philox64_kat(din, dout, n, 0);
  if (e != cudaSuccess) return fail(EM_ERR_CUDA, cudaGetErrorString(e));
  EM_CUDA(cudaMemcpy(out4, dout, (size_t)n * 32, cudaMemcpyDeviceToHost));
  cudaFree(din);
  cudaFree(dout);
  return EM_OK;
}

int em_philox4x32_blocks(const uint32_t* in6, uint32_t* out4, int n, int device) {
  DeviceGuard dg(device);
  unsigned *din = nullptr, *dout = nullptr;
  EM_CUDA(cudaMalloc(&din, (size_t)n * 24));
  EM_CUDA(cudaMalloc(&dout, (size_t)n * 16));
  EM_CUDA(cudaMemcpy(din, in6, (size_t)n * 24, cudaMemcpyHostToDevice));
  cudaError_t e = launch_philox32_kat(din, dout, n, 0);
  if (e != cudaSuccess) return fail(EM_ERR_CUDA, cudaGetErrorString(e));
  EM_CUDA(cudaMemcpy(out4, dout, (size_t)n * 16, cudaMemcpyDeviceToHost));
  cudaFree(din);
  cudaFree(dout);
  return EM_OK;
}

}  // extern "C"
