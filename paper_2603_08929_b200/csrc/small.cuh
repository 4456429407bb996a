// Small-n LSD sort: ONE CTA, ONE launch, the whole sort in shared memory (SURVEY §8 row
// "small-n latency").
//
// Up to 20K keys the multi-launch path (memset, histogram, plan, P scatter passes, copy-back:
// 8-11 dependent launches, ~20 us of device time and ~30 us of host enqueue) is all fixed cost.
// Here one CTA of 512 threads loads the keys into shared memory once and runs every LSD pass
// (the paper's Algorithm 2 counting step per digit, P:174-184, 8 bits at a time) between two
// shared buffers, then stores the result once:
//
//   count   per-warp digit counters (shared atomics) over the warp's contiguous segment;
//   scan    first slot of (digit, warp) = keys of smaller digits + keys of this digit in the
//           warps before it (digit-major exclusive scan over 256 x 16 counters);
//   rank    each warp re-walks its segment in input order, 32 keys per round, and puts each key
//           at its (digit, warp) counter's next slot in the other buffer.  Stable: with the
//           shared-atomic lane order (selftest.cu) a single atomicAdd per key returns the slot;
//           otherwise eight ballots find the lanes with equal digits and the lowest one
//           advances the counter for the group.
//
// A pass whose digit is constant over all keys is skipped (the counts show it).  Keys are
// transformed (a1) only to extract digits; the buffers hold the raw keys.
//
// Above its capacity (20480 32-bit / 10240 64-bit keys) the one-CTA-per-SM variant
// (small_grid.cuh) takes over.
#pragma once

#include "common.cuh"

namespace bsort {
namespace small_detail {

constexpr int THREADS = 512;
constexpr int WARPS = THREADS / 32;

// keys that fit: the input and its per-pass copy, 2 x 80 KB of shared memory
template <typename U>
__host__ __device__ constexpr uint32_t max_n() {
  return sizeof(U) == 4 ? 20480u : 10240u;
}

template <typename U>
__host__ __device__ constexpr size_t smem_bytes() {
  return 2 * (size_t)max_n<U>() * sizeof(U) + (size_t)WARPS * 256 * 4;
}

}  // namespace small_detail

template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(small_detail::THREADS, 1)
    k_small_sort(U* __restrict__ keys, uint32_t n, int lane_atomics) {
  using namespace small_detail;
  extern __shared__ __align__(128) unsigned char smem[];
  U* sa = reinterpret_cast<U*>(smem);
  U* sb = sa + max_n<U>();
  uint32_t* wc = reinterpret_cast<uint32_t*>(sb + max_n<U>());  // [WARPS][256]
  __shared__ uint32_t wsum[8];
  __shared__ int trivial;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t seg = (n + WARPS - 1) / WARPS;  // warp w's keys: [w seg, min(n, (w+1) seg))
  const uint32_t w_lo = min((uint32_t)w * seg, n), w_hi = min(w_lo + seg, n);

  if ((uintptr_t)keys % 16 == 0) {
    constexpr uint32_t V = 16 / sizeof(U);
    const uint32_t nv = n / V;
#pragma unroll 4
    for (uint32_t j = tid; j < nv; j += THREADS) reinterpret_cast<uint4*>(sa)[j] = reinterpret_cast<const uint4*>(keys)[j];
    for (uint32_t i = nv * V + tid; i < n; i += THREADS) sa[i] = keys[i];
  } else {
#pragma unroll 4
    for (uint32_t i = tid; i < n; i += THREADS) sa[i] = keys[i];
  }

  U* cur = sa;
  U* oth = sb;
  for (int p = 0; p < (int)sizeof(U); ++p) {
    const int sh = 8 * p;
    auto digit = [&](U x) { return uint32_t(key_encode<KIND, DESC>(x) >> sh) & 0xFFu; };
    __syncthreads();  // the previous pass's ranking is done with wc and the buffers
    for (int i = tid; i < WARPS * 256; i += THREADS) wc[i] = 0;
    if (tid == 0) trivial = 0;
    __syncthreads();
    for (uint32_t i = w_lo + lane; i < w_hi; i += 32) atomicAdd(&wc[w * 256 + digit(cur[i])], 1u);
    __syncthreads();
    // digit-major exclusive scan over (digit, warp): thread d < 256 owns digit d's 16 counters
    uint32_t tot = 0;
    if (tid < 256) {
#pragma unroll
      for (int k = 0; k < WARPS; ++k) tot += wc[k * 256 + tid];
      if (tot == n) trivial = 1;
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[w] = x;
      tot = x - tot;  // exclusive within the warp's 32 digits
    }
    __syncthreads();
    if (trivial) continue;  // one digit value: the pass would not move a key
    if (tid < 256) {
      uint32_t f = tot;
      for (int k = 0; k < w; ++k) f += wsum[k];
#pragma unroll
      for (int k = 0; k < WARPS; ++k) {
        const uint32_t e = wc[k * 256 + tid];
        wc[k * 256 + tid] = f;
        f += e;
      }
    }
    __syncthreads();
    uint32_t* slot = wc + w * 256;
    if (lane_atomics) {
      // every lane runs the same number of rounds, so the atomics of one round are ONE warp
      // instruction (if some lanes had one round fewer, the compiler's remainder handling could
      // let the two lane groups run a round in different instructions, in either order)
      for (uint32_t r = w_lo; r < w_hi; r += 32) {
        const uint32_t i = r + lane;
        __syncwarp();
        if (i < w_hi) {
          const U x = cur[i];
          oth[atomicAdd(&slot[digit(x)], 1u)] = x;
        }
      }
    } else {
      for (uint32_t r = w_lo; r < w_hi; r += 32) {
        const uint32_t i = r + lane;
        const bool ok = i < w_hi;
        const U x = ok ? cur[i] : U(0);
        const uint32_t d = ok ? digit(x) : 256u;
        uint32_t peers = __ballot_sync(0xFFFFFFFFu, ok);
        if (!ok) peers = ~peers;  // invalid lanes group among themselves and store nothing
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (d >> b) & 1u);
          peers &= ((d >> b) & 1u) ? bal : ~bal;
        }
        const int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (ok && lane == leader) {  // distinct digits have distinct leaders: no conflicts
          b = slot[d];
          slot[d] = b + __popc(peers);
        }
        b = __shfl_sync(0xFFFFFFFFu, b, leader);
        if (ok) oth[b + __popc(peers & lanemask_lt())] = x;
      }
    }
    U* t = cur;
    cur = oth;
    oth = t;
  }
  __syncthreads();
  if ((uintptr_t)keys % 16 == 0) {
    constexpr uint32_t V = 16 / sizeof(U);
    const uint32_t nv = n / V;
#pragma unroll 4
    for (uint32_t j = tid; j < nv; j += THREADS) reinterpret_cast<uint4*>(keys)[j] = reinterpret_cast<const uint4*>(cur)[j];
    for (uint32_t i = nv * V + tid; i < n; i += THREADS) keys[i] = cur[i];
  } else {
    for (uint32_t i = tid; i < n; i += THREADS) keys[i] = cur[i];
  }
}

// Keys-only sorts of at most small_max_n<U>() keys take this path (BSORT_SMALL=0 disables it;
// BSORT_SMALL_MAX lowers the bound from what fits: 20480 / 10240 keys).
template <typename U>
inline uint64_t small_max_n() {
  static const uint64_t v = [] {
    const char* e = getenv("BSORT_SMALL");
    if (e && e[0] == '0') return (uint64_t)0;
    const char* mx = getenv("BSORT_SMALL_MAX");
    const uint64_t cap = small_detail::max_n<U>();
    return mx ? min64(strtoull(mx, nullptr, 10), cap) : cap;
  }();
  return v;
}

template <int KIND, bool DESC, typename U>
bsort_status_t launch_small(U* keys, uint64_t n, cudaStream_t s) {
  using namespace small_detail;
  auto kern = k_small_sort<KIND, DESC, U>;
  constexpr size_t SMEM = smem_bytes<U>();
  static DeviceOnce attr;
  if (attr.pending()) {
    BSORT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr.mark();
  }
  if (n > max_n<U>()) return BSORT_ERROR_INVALID_ARGUMENT;  // caller checks small_max_n
  const int lane_atomics = atomics_lane_ordered(s) ? 1 : 0;
  BSORT_LAUNCH(PROF_PASS, s, kern<<<1, THREADS, SMEM, s>>>(keys, (uint32_t)n, lane_atomics));
  return BSORT_SUCCESS;
}

}  // namespace bsort
