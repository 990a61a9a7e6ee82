// em_pool.cuh -- persistent-lane work distribution shared by the walk kernels.
//
// Work unit = a CHUNK: (pole p, replicates [b*RB, b*RB + RB) of that pole),
// chunk id c = b * n_poles + p, so consecutive chunk ids cycle over the poles
// and the walks in flight at any moment are spread over all count rows
// (pole-dependent walk lengths balance out; exit atomics spread over every
// row).  A warp claims one chunk at a time with ONE global atomic and hands
// its replicates to lanes as they finish, so a lane whose walk ended restarts
// immediately instead of idling until the warp's longest walk ends (SURVEY F5:
// lockstep without refill runs at 0.33 lane efficiency).  Because a lane's
// consecutive walks mostly share a pole, per-pole step statistics are summed
// in registers and flushed with one atomic triple per pole change instead of
// three contended atomics per walk.  Results never depend on this schedule:
// every walk's RNG stream is keyed by (seed, pole, replicate) and all
// accumulations are integer.
#pragma once
#include "em_params.cuh"

namespace em {

constexpr unsigned kFull = 0xffffffffu;

struct WarpPool {
  long long rep0;    // first replicate offset of the current chunk
  int pole;          // pole row of the current chunk
  int next, end;     // next / one-past-last replicate index inside the chunk
  int exhausted;     // int, not bool: bools become byte-packed PRMT traffic
};

__device__ __forceinline__ void pool_init(WarpPool& wp) {
  wp.rep0 = 0;
  wp.pole = 0;
  wp.next = 0;
  wp.end = 0;
  wp.exhausted = 0;
}

// Called by all 32 lanes (converged).  Lanes set in need_mask receive
// (pole, replicate offset) and return true, or return false (no work now).
// lane / lt (lanes below this one) may be passed in when the caller keeps
// them in registers.
template <class RepT>
__device__ __forceinline__ bool pool_take(WarpPool& wp, unsigned need_mask, const WorkOut& W,
                                          int& pole, RepT& rep_off, int lane, unsigned lt) {
  const int n_need = __popc(need_mask);
  const int rank = __popc(need_mask & lt);
  const bool me = (need_mask >> lane) & 1u;
  const int avail = wp.end - wp.next;
  bool got = false;
  if (me && rank < avail) {
    pole = wp.pole;
    rep_off = (RepT)(wp.rep0 + wp.next + rank);
    got = true;
  }
  if (avail >= n_need) {
    wp.next += n_need;
    return got;
  }
  wp.next = wp.end;
  if (wp.exhausted) return got;
  unsigned long long c = 0;
  if (lane == 0) c = atomicAdd(W.ticket, 1ULL);
  c = __shfl_sync(kFull, c, 0);
  if (c >= W.n_chunks) {
    wp.exhausted = 1;
    return got;
  }
  // chunk c -> (replicate block b, pole p); exact for c < 2^53
  long long b = (long long)((double)c * W.inv_poles);
  long long p = (long long)c - b * W.n_poles;
  if (p < 0) {
    b -= 1;
    p += W.n_poles;
  } else if (p >= W.n_poles) {
    b += 1;
    p -= W.n_poles;
  }
  const long long r0 = b * W.rb;
  const int valid = (int)(W.n_rep - r0 < W.rb ? W.n_rep - r0 : W.rb);
  const int rem = n_need - avail;
  if (me && rank >= avail && rank - avail < valid) {
    pole = (int)p;
    rep_off = (RepT)(r0 + (rank - avail));
    got = true;
  }
  wp.pole = (int)p;
  wp.rep0 = r0;
  wp.next = rem < valid ? rem : valid;
  wp.end = valid;
  return got;
}

template <class RepT>
__device__ __forceinline__ bool pool_take(WarpPool& wp, unsigned need_mask, const WorkOut& W,
                                          int& pole, RepT& rep_off) {
  const int lane = threadIdx.x & 31;
  return pool_take(wp, need_mask, W, pole, rep_off, lane, (1u << lane) - 1u);
}

// Same contract, shaped for the FP32 kernel's service pass: the common case
// (the current chunk covers every idle lane) is straight-line predicated
// code; only a chunk claim branches.  eq / lt are this lane's bit and the
// bits below it, kept in registers by the caller.
template <class RepT>
__device__ __forceinline__ bool pool_take_fast(WarpPool& wp, unsigned need_mask, const WorkOut& W,
                                               int& pole, RepT& rep_off, unsigned eq, unsigned lt) {
  const int n_need = __popc(need_mask);
  const int rank = __popc(need_mask & lt);
  const int me = (need_mask & eq) != 0u;
  const int avail = wp.end - wp.next;
  int got = me & (rank < avail);
  int np = wp.pole;
  long long r = wp.rep0 + wp.next + rank;
  if (avail < n_need) {  // rare: claim the next chunk for the lanes beyond avail
    wp.next = wp.end;
    if (!wp.exhausted) {
      unsigned long long c = 0;
      if (eq == 1u) c = atomicAdd(W.ticket, 1ULL);
      c = __shfl_sync(kFull, c, 0);
      if (c >= W.n_chunks) {
        wp.exhausted = 1;
      } else {
        long long b = (long long)((double)c * W.inv_poles);
        long long p = (long long)c - b * W.n_poles;
        if (p < 0) {
          b -= 1;
          p += W.n_poles;
        } else if (p >= W.n_poles) {
          b += 1;
          p -= W.n_poles;
        }
        const long long r0 = b * W.rb;
        const int valid = (int)(W.n_rep - r0 < W.rb ? W.n_rep - r0 : W.rb);
        const int rem = n_need - avail;
        if (me && rank >= avail && rank - avail < valid) {
          np = (int)p;
          r = r0 + (rank - avail);
          got = 1;
        }
        wp.pole = (int)p;
        wp.rep0 = r0;
        wp.next = rem < valid ? rem : valid;
        wp.end = valid;
      }
    }
  } else {
    wp.next += n_need;
  }
  if (got) {
    pole = np;
    rep_off = (RepT)r;
  }
  return got != 0;
}

// Per-lane step statistics of the pole the lane is currently walking.
struct StepAcc {
  int pole;
  unsigned long long sum, sq, mx;
};

__device__ __forceinline__ void acc_init(StepAcc& a) {
  a.pole = -1;
  a.sum = a.sq = a.mx = 0;
}

// Per-WARP shared tables of step statistics, (3, n_poles) u64 each, used
// when the job is small (W.smem_stats: few poles, small chunks): then a chunk
// holds ~1 walk per lane, lanes change pole on every walk, and global
// per-pole atomics would serialise on 3 * n_poles addresses.  Warp-private,
// so only __syncwarp is needed (a block barrier in this kernel costs ~20% by
// changing its register allocation); each warp flushes its table at exit.
extern __shared__ unsigned long long s_stats[];

__device__ __forceinline__ unsigned long long* warp_stats(const WorkOut& W) {
  return s_stats + (threadIdx.x >> 5) * 3 * W.n_poles;
}

// SMEM: compile-time choice (the FP32 kernel is instantiated both ways so the
// big-job variant's code generation is untouched); -1 = decide at run time
// from W.smem_stats (the REF64 mirror)
template <int SMEM = -1>
__device__ __forceinline__ void acc_flush(StepAcc& a, const WorkOut& W) {
  if (a.pole >= 0 && a.sum + a.mx > 0) {
    if (SMEM == 1 || (SMEM < 0 && W.smem_stats == 1)) {
      unsigned long long* t = warp_stats(W);
      atomicAdd(&t[a.pole], a.sum);
      atomicAdd(&t[W.n_poles + a.pole], a.sq);
      atomicMax(&t[2 * W.n_poles + a.pole], a.mx);
    } else {
      // W.stat_copies is a power of two; 1 = flush straight into the output
      const long long off =
          (long long)(((threadIdx.x >> 5) + (threadIdx.x & 31) + blockIdx.x * 8) & (W.stat_copies - 1)) *
          3 * W.n_poles;
      atomicAdd(&W.ssum[off + a.pole], a.sum);
      atomicAdd(&W.ssq[off + a.pole], a.sq);
      atomicMax(&W.smax[off + a.pole], a.mx);
    }
  }
  a.sum = a.sq = a.mx = 0;
}

template <int SMEM = -1>
__device__ __forceinline__ void stats_smem_init(const WorkOut& W) {
  if ((SMEM >= 0 && SMEM != 1) || (SMEM < 0 && W.smem_stats != 1)) return;
  unsigned long long* t = warp_stats(W);
  for (int i = threadIdx.x & 31; i < 3 * W.n_poles; i += 32) t[i] = 0;
  __syncwarp();
}

template <int SMEM = -1>
__device__ __forceinline__ void stats_smem_flush(const WorkOut& W) {
  if ((SMEM >= 0 && SMEM != 1) || (SMEM < 0 && W.smem_stats != 1)) return;
  __syncwarp();
  const unsigned long long* t = warp_stats(W);
  const int n = (int)W.n_poles;
  for (int i = threadIdx.x & 31; i < n; i += 32) {
    const unsigned long long sm = t[i], mx = t[2 * n + i];
    if (sm | mx) {
      atomicAdd(&W.ssum[i], sm);
      atomicAdd(&W.ssq[i], t[n + i]);
      atomicMax(&W.smax[i], mx);
    }
  }
}

template <int SMEM = -1>
__device__ __forceinline__ void acc_add(StepAcc& a, const WorkOut& W, int pole,
                                        unsigned long long steps) {
  if (pole != a.pole) {
    acc_flush<SMEM>(a, W);
    a.pole = pole;
  }
  a.sum += steps;
  a.sq += steps * steps;
  a.mx = steps > a.mx ? steps : a.mx;
}

}  // namespace em
