// onesweep.cuh — a3/a4: one-sweep multi-digit histogram and the per-digit stable scatter
// pass with decoupled look-back (templates shared by the LSD sort and the MSD partition).
//
// Paper mapping.  Algorithm 1 splits a range on ONE bit per scan and Algorithm 2
// recurses MSB-first, so a w-bit key costs w full scans (Theorem 4; "64 complete
// array scans").  Here each scan is a stable 256-way split on an 8-bit digit of the
// transformed key, least-significant digit first: ceil(w/8) scans instead of w, branch-free
// ranking instead of the mispredicted bit test, no recursion.  LSD order is
// correct because every pass is stable (a stable sort on digit p preserves the order of
// digits < p), which is why the ranking below follows global index order exactly.
#pragma once
#include "common.cuh"
#include "scan.cuh"

namespace bsort {

// Look-back descriptor: [flag:2 | value:(W-2)], flag 0 = not ready, 1 = aggregate (this tile's
// count only), 2 = inclusive prefix (count of all tiles <= this one).  One word => no fence.
template <typename D> struct LookbackBits;
template <> struct LookbackBits<uint32_t> {
  static constexpr int SH = 30;
  static constexpr uint32_t AGG = 1u << 30, INC = 2u << 30, VAL = (1u << 30) - 1;
};
template <> struct LookbackBits<unsigned long long> {
  static constexpr int SH = 62;
  static constexpr unsigned long long AGG = 1ull << 62, INC = 2ull << 62, VAL = (1ull << 62) - 1;
};

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename U> __device__ __forceinline__ U ldg_nc(const U* p);
template <> __device__ __forceinline__ uint32_t ldg_nc(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ unsigned long long ldg_nc(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Device-resident pass plan written by k_plan (device-side trivial-digit skipping, so the
// whole sort is enqueued without a host sync).
struct PassPlan {
  uint32_t skip[8];     // digit p is trivial (one bin holds all n keys): pass p not executed
  uint32_t src_alt[8];  // executed pass p reads the scratch buffer (and writes the user buffer)
  uint32_t final_copy;  // odd number of executed passes: result is in scratch, copy back
  uint32_t executed;    // number of executed passes
  uint32_t pad[14];
};

// Digit of LSD pass p: byte p of the transformed key.
template <int KIND, bool DESC, typename U>
struct RadixDigit {
  int shift;
  __device__ __forceinline__ uint32_t operator()(U x) const {
    return uint32_t(key_encode<KIND, DESC>(x) >> shift) & 0xFFu;
  }
};

// Digit of the MSD partition: destination rank of the key's top-16-bit bin.
template <int KIND, bool DESC, typename U>
struct RankDigit {
  uint32_t cuts[BSORT_DIST_MAX_RANKS + 1];
  int nranks;
  __device__ __forceinline__ uint32_t operator()(U x) const {
    const uint32_t b = uint32_t(key_encode<KIND, DESC>(x) >> (sizeof(U) * 8 - 16));
    uint32_t lo = 0, hi = (uint32_t)nranks;  // largest q in [0,nranks) with cuts[q] <= b
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (cuts[mid] <= b) lo = mid; else hi = mid;
    }
    return lo;
  }
};

// ---------------------------------------------------------------------------------------
// a3: one read of all keys, P = sizeof(U) digit histograms of 256 bins.  Counters are
// lane-banked (address = bin*LANES + lane%LANES, bank = lane) so the shared-memory atomics of a
// warp never conflict; one CTA of 1024 threads per SM, grid-stride, 128-bit loads.
constexpr int HIST_THREADS = 1024;

template <int KIND, bool DESC, typename U, int LANES>
__global__ void __launch_bounds__(HIST_THREADS, 1)
    k_onesweep_hist(const U* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ ghist) {
  constexpr int P = sizeof(U);
  extern __shared__ uint32_t hs[];  // [P][256][LANES]
  for (int i = threadIdx.x; i < P * 256 * LANES; i += HIST_THREADS) hs[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & (LANES - 1);
  auto add = [&](U x) {
    const U k = key_encode<KIND, DESC>(x);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint32_t d = uint32_t(k >> (8 * p)) & 0xFFu;
      atomicAdd(&hs[(p * 256 + d) * LANES + lane], 1u);
    }
  };
  constexpr int PER_VEC = 16 / sizeof(U);
  const uint64_t T = (uint64_t)gridDim.x * HIST_THREADS;
  const uint64_t gt = (uint64_t)blockIdx.x * HIST_THREADS + threadIdx.x;
  const uint64_t head = min64(n, ((16 - ((uintptr_t)keys & 15)) & 15) / sizeof(U));
  for (uint64_t i = gt; i < head; i += T) add(keys[i]);
  const uint4* v = reinterpret_cast<const uint4*>(keys + head);
  const uint64_t nv = (n - head) / PER_VEC;
  auto vec = [&](uint4 q) {
    if constexpr (sizeof(U) == 4) {
      add(U(q.x)); add(U(q.y)); add(U(q.z)); add(U(q.w));
    } else {
      add(U(q.x) | (U(q.y) << 32));
      add(U(q.z) | (U(q.w) << 32));
    }
  };
  uint64_t i = gt;
  for (; i + 3 * T < nv; i += 4 * T) {
    uint4 q0 = __ldcs(v + i), q1 = __ldcs(v + i + T), q2 = __ldcs(v + i + 2 * T), q3 = __ldcs(v + i + 3 * T);
    vec(q0); vec(q1); vec(q2); vec(q3);
  }
  for (; i < nv; i += T) vec(__ldcs(v + i));
  for (uint64_t j = head + nv * PER_VEC + gt; j < n; j += T) add(keys[j]);
  __syncthreads();
  for (int b = threadIdx.x; b < P * 256; b += HIST_THREADS) {
    uint32_t s = 0;
#pragma unroll 8
    for (int l = 0; l < LANES; ++l) s += hs[b * LANES + ((l + b) & (LANES - 1))];
    if (s) atomicAdd(&ghist[b], (unsigned long long)s);
  }
}

// Plan: exclusive scan of every digit histogram into global digit bases, trivial-digit
// detection, ping-pong buffer assignment, tile-counter reset.  One CTA of 256 threads.
__global__ void __launch_bounds__(256)
    k_plan(const unsigned long long* __restrict__ ghist, uint64_t n, int P, unsigned long long* __restrict__ bases,
           PassPlan* __restrict__ plan, uint32_t* __restrict__ tile_counters) {
  __shared__ unsigned long long wt[256 / 32 + 1];
  __shared__ uint32_t skip_s[8];
  for (int p = 0; p < P; ++p) {
    const unsigned long long c = ghist[p * 256 + threadIdx.x];
    const unsigned long long ex = block_exclusive_scan<256>(c, wt, (unsigned long long*)nullptr);
    bases[p * 256 + threadIdx.x] = ex;
    const int trivial = __syncthreads_or(c == n);
    if (threadIdx.x == 0) skip_s[p] = trivial;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t alt = 0, executed = 0;
    for (int p = 0; p < 8; ++p) {
      const uint32_t sk = (p < P) ? skip_s[p] : 1u;
      plan->skip[p] = sk;
      plan->src_alt[p] = alt;
      if (!sk) {
        alt ^= 1u;
        ++executed;
      }
    }
    plan->final_copy = alt;
    plan->executed = executed;
  }
  if (threadIdx.x < 8) tile_counters[threadIdx.x] = 0;
}

// ---------------------------------------------------------------------------------------
// a4: one stable scatter pass.  Persistent CTAs take tiles of THREADS*ITEMS keys in order from
// an atomic counter (forward progress for the look-back: a tile only waits on smaller tiles,
// which were taken earlier by CTAs that are running).  Per tile:
//   1. warp-striped coalesced loads (warp w owns a contiguous 32*ITEMS segment, item k of lane
//      l is element 32k+l of it, so (warp, item, lane) order IS global index order);
//   2. stable warp ranking: __match_any_sync groups equal digits, the group's highest lane
//      bumps the warp's per-digit counter, rank = counter + lanes below in the group;
//   3. per-digit tile counts published early to the look-back array (flag AGG), block scan of
//      the counts => per-(warp, digit) offsets, keys staged in smem in digit order;
//   4. decoupled look-back per digit (one thread per digit) => global digit offset, INC publish;
//   5. coalesced scatter of the smem-sorted tile: runs of equal digits are contiguous.
template <int THREADS, int ITEMS, typename U>
struct PassSmem {
  static constexpr int WARPS = THREADS / 32;
  static constexpr int TILE = THREADS * ITEMS;
  static constexpr size_t keys_off = 0;
  static constexpr size_t wcnt_off = align_up(keys_off + sizeof(U) * TILE, 16);
  static constexpr size_t gofs_off = align_up(wcnt_off + sizeof(uint32_t) * WARPS * 256, 16);
  static constexpr size_t wt_off = align_up(gofs_off + sizeof(unsigned long long) * 256, 16);
  static constexpr size_t misc_off = align_up(wt_off + sizeof(uint32_t) * (WARPS + 1), 16);
  static constexpr size_t bytes = align_up(misc_off + 16, 128);
};

template <typename U, int THREADS, int ITEMS, int MINB, typename DescT, typename DigitF>
__global__ void __launch_bounds__(THREADS, MINB)
    k_onesweep_pass(const U* a_ptr, U* b_ptr, uint64_t n, DigitF digit,
                    const unsigned long long* __restrict__ bases, DescT* __restrict__ lookback,
                    uint32_t* __restrict__ tile_counter, uint32_t num_tiles,
                    const PassPlan* __restrict__ plan, int pass) {
  using L = PassSmem<THREADS, ITEMS, U>;
  using LB = LookbackBits<DescT>;
  constexpr int TILE = L::TILE;
  constexpr int WARPS = L::WARPS;
  static_assert(THREADS >= 256, "one thread per digit");
  static_assert(32 * ITEMS <= 0xFFFF, "rank fits 16 bits");
  extern __shared__ __align__(128) unsigned char smem[];
  U* keys_s = reinterpret_cast<U*>(smem + L::keys_off);
  uint32_t(*wcnt)[256] = reinterpret_cast<uint32_t(*)[256]>(smem + L::wcnt_off);
  unsigned long long* gofs = reinterpret_cast<unsigned long long*>(smem + L::gofs_off);
  uint32_t* wt = reinterpret_cast<uint32_t*>(smem + L::wt_off);
  uint32_t* tile_s = reinterpret_cast<uint32_t*>(smem + L::misc_off);

  const U* src = a_ptr;
  U* dst = b_ptr;
  if (plan != nullptr) {
    if (plan->skip[pass]) return;
    if (plan->src_alt[pass]) {
      src = b_ptr;
      dst = const_cast<U*>(a_ptr);
    }
  }
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t t = threadIdx.x;

  for (;;) {
    if (t == 0) *tile_s = atomicAdd(tile_counter, 1u);
    __syncthreads();  // publishes tile id; previous tile's smem is dead
    const uint32_t tile = *tile_s;
    if (tile >= num_tiles) break;
    const uint64_t tile_base = (uint64_t)tile * TILE;
    const bool full = tile_base + TILE <= n;

    for (int j = lane; j < 256; j += 32) wcnt[warp][j] = 0;

    // 1. load
    const uint64_t seg = tile_base + (uint64_t)warp * (32 * ITEMS) + lane;
    U keys[ITEMS];
    if (full) {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) keys[k] = ldg_nc(src + seg + 32 * k);
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) keys[k] = (seg + 32 * k < n) ? ldg_nc(src + seg + 32 * k) : U(0);
    }
    __syncwarp();

    // 2. rank
    uint32_t rk[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t d = (full || seg + 32 * k < n) ? digit(keys[k]) : 255u;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t leader = 31 - __clz(peers);
      const uint32_t below = __popc(peers & lanemask_lt());
      uint32_t old = 0;
      if (lane == leader) {
        old = wcnt[warp][d];
        wcnt[warp][d] = old + __popc(peers);
      }
      __syncwarp();
      old = __shfl_sync(0xffffffffu, old, leader);
      rk[k] = (d << 16) | (old + below);
    }
    __syncthreads();

    // 3. per-digit totals, early publish, tile-local offsets
    uint32_t total = 0;
    if (t < 256) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const uint32_t c = wcnt[w][t];
        wcnt[w][t] = total;
        total += c;
      }
      if (!full && t == 255) total -= (uint32_t)(tile_base + TILE - n);  // invalid tail keys
      st_relaxed(&lookback[(uint64_t)tile * 256 + t], (tile == 0 ? LB::INC : LB::AGG) | DescT(total));
    }
    const uint32_t tile_excl = block_exclusive_scan<THREADS>(t < 256 ? total : 0u, wt, (uint32_t*)nullptr);
    if (t < 256) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) wcnt[w][t] += tile_excl;
    }
    __syncthreads();

#pragma unroll
    for (int k = 0; k < ITEMS; ++k) keys_s[wcnt[warp][rk[k] >> 16] + (rk[k] & 0xFFFFu)] = keys[k];

    // 4. decoupled look-back
    if (t < 256) {
      DescT excl = 0;
      if (tile > 0) {
        uint32_t j = tile - 1;
        for (;;) {
          const DescT v = ld_relaxed(&lookback[(uint64_t)j * 256 + t]);
          const DescT flag = v >> LB::SH;
          if (flag == 0) continue;
          excl += v & LB::VAL;
          if (flag == 2 || j == 0) break;
          --j;
        }
        st_relaxed(&lookback[(uint64_t)tile * 256 + t], LB::INC | (excl + DescT(total)));
      }
      gofs[t] = bases[t] + (unsigned long long)excl - tile_excl;
    }
    __syncthreads();

    // 5. scatter
    const uint32_t valid = full ? (uint32_t)TILE : (uint32_t)(n - tile_base);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t i = t + k * THREADS;
      if (i < valid) {
        const U x = keys_s[i];
        dst[gofs[digit(x)] + i] = x;
      }
    }
  }
}

// Final placement when an odd number of passes executed (result sits in the scratch buffer).
template <typename U>
__global__ void __launch_bounds__(256) k_copy_back(U* __restrict__ a, const U* __restrict__ b, uint64_t n,
                                                   const PassPlan* __restrict__ plan) {
  if (!plan->final_copy) return;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) a[i] = b[i];
}

}  // namespace bsort
