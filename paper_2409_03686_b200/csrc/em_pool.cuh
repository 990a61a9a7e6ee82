// em_pool.cuh -- persistent-lane work distribution shared by the walk kernels.
//
// Walk ids g in [0, n_poles * n_rep) are pole-interleaved (pole = g mod M,
// replicate = g div M), so the walks in flight at any moment are spread over
// every pole: pole-dependent walk lengths balance out and exit atomics spread
// over all M count rows.  Each warp claims CHUNK consecutive ids from one
// global counter at a time (one atomic per CHUNK walks) and hands them to its
// lanes as they finish, so a lane whose walk ended restarts immediately
// instead of idling until the warp's longest walk ends (lockstep
// without refill runs at 0.33 lane efficiency).  Results never depend on this
// schedule: every walk's RNG stream is keyed by (seed, pole, replicate) and
// all accumulations are integer.
#pragma once
#include "em_params.cuh"

namespace em {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kNoWalk = ~0ULL;

struct WarpPool {
  unsigned long long next, end;
  bool exhausted;
};

__device__ __forceinline__ void pool_init(WarpPool& wp) {
  wp.next = 0;
  wp.end = 0;
  wp.exhausted = false;
}

// Called by all 32 lanes (converged).  Lanes set in need_mask receive a walk
// id or kNoWalk.
__device__ __forceinline__ unsigned long long pool_take(WarpPool& wp, unsigned need_mask,
                                                        unsigned long long* ticket,
                                                        unsigned long long total,
                                                        unsigned chunk) {
  const int lane = threadIdx.x & 31;
  const unsigned n_need = __popc(need_mask);
  const unsigned rank = __popc(need_mask & ((1u << lane) - 1u));
  const bool me = (need_mask >> lane) & 1u;
  const unsigned long long avail = wp.end - wp.next;
  unsigned long long my = kNoWalk;
  if (me && rank < avail) my = wp.next + rank;
  if (avail >= n_need) {
    wp.next += n_need;
    return my;
  }
  wp.next = wp.end;
  if (wp.exhausted) return my;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(ticket, (unsigned long long)chunk);
  base = __shfl_sync(kFull, base, 0);
  if (base >= total) {
    wp.exhausted = true;
    return my;
  }
  const unsigned long long end = base + chunk < total ? base + chunk : total;
  const unsigned long long rem = n_need - avail;
  if (me && rank >= avail) {
    const unsigned long long gg = base + (rank - avail);
    my = gg < end ? gg : kNoWalk;
  }
  wp.next = base + rem < end ? base + rem : end;
  wp.end = end;
  return my;
}

// g -> (replicate offset, pole row); exact for g < 2^53.
__device__ __forceinline__ void split_walk(unsigned long long g, long long n_poles,
                                           double inv_poles, long long& rep_off,
                                           long long& pole) {
  long long q = (long long)((double)g * inv_poles);
  long long r = (long long)g - q * n_poles;
  if (r < 0) {
    q -= 1;
    r += n_poles;
  } else if (r >= n_poles) {
    q += 1;
    r -= n_poles;
  }
  rep_off = q;
  pole = r;
}

}  // namespace em
