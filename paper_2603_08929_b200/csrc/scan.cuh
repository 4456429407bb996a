// scan.cuh — block-wide exclusive scans used by the plan/fill kernels.
#pragma once
#include "common.cuh"

namespace bsort {

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= (uint32_t)d) v += o;
  }
  return v;
}

// Exclusive scan over a block of NT threads (NT multiple of 32, <= 1024).  `warp_tot` is
// shared scratch of NT/32 entries.  Returns the exclusive prefix; *total gets the block sum.
// Contains __syncthreads(); every thread of the block must call it.
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_tot, T* total) {
  constexpr int NW = NT / 32;
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < (uint32_t)NW) ? warp_tot[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane < (uint32_t)NW) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == NW - 1) warp_tot[NW] = wi;             // block total (needs NW+1 slots)
  }
  __syncthreads();
  T out = warp_tot[warp] + inc - v;
  if (total) *total = warp_tot[NW];
  return out;
}

}  // namespace bsort
