// Mid-size LSD sort in ONE cooperative launch (DESIGN.md §6 "Small n"): one CTA per SM for
// n between the single-CTA kernel's bound (small.cuh) and SMALL_GRID_MAX keys.
//
// Every LSD pass is three phases of one persistent kernel with grid-wide barriers between them
// instead of kernel boundaries:
//
//   A  each CTA stages its contiguous chunk of the current buffer in shared memory and counts the
//      pass's digits per warp (shared atomics), then publishes the CTA's 256 counts (u16) into
//      column c of a digit-major matrix cnt[d][c] in global memory;                  grid barrier
//   B  each CTA reads, for every digit d, row d of the matrix (two threads per row, 128-bit
//      loads of the first G columns, all in flight): the total T[d] and the count of the CTAs before it, P[d].  The CTA's
//      first slot for digit d is  sum_{d' < d} T[d'] + P[d]  (Algorithm 2's prefix over bins,
//      P:174-184, split by source chunk); per warp, plus the counts of the warps before it;
//   C  each warp re-walks its segment in input order, 32 keys per round, and puts every key at its
//      (digit, warp) counter's next slot of a second shared buffer (stable: lane-ordered shared
//      atomics, checked by selftest.cu, or eight ballots); the CTA then writes that buffer out in
//      slot order (a digit's keys are one contiguous run in the destination);        grid barrier
//
// A pass whose digit is constant over all keys (T[d] == n) is skipped by every CTA alike.  The
// count matrix is double-buffered by pass parity.  The grid barrier is cooperative groups'
// grid.sync() on the barrier word the runtime keeps for a cooperative launch, so the launch
// needs no memset of a counter of ours (one launch per sort instead of memset + launch:
// ~2 us at cfg1); with BSORT_GRID_CG=0 it is a counter in the workspace zeroed by a 4-byte
// memset before the launch (one release-add per CTA, relaxed polls, one acquire fence).  Both
// cost 1.2 us per barrier on B200 (tools/exp/gridbar.cu).  The launch is cooperative for its
// co-residency guarantee.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace bsort {
namespace grid_detail {

constexpr int THREADS = 512;
constexpr int WARPS = THREADS / 32;
constexpr int MAX_CTAS = 160;  // >= the SM count of a B200 (148); matrix rows padded to 8
constexpr int ROW = (MAX_CTAS + 7) / 8 * 8;

// keys per CTA at most: the chunk and its digit-sorted copy, 2 x 80 KB of shared memory
template <typename U>
__host__ __device__ constexpr uint32_t max_chunk() {
  return sizeof(U) == 4 ? 20480u : 10240u;
}

template <typename U>
__host__ __device__ constexpr size_t smem_bytes() {
  return 2 * (size_t)max_chunk<U>() * sizeof(U) + (size_t)WARPS * 256 * 4 + 3 * 256 * 4;
}

// workspace: the count matrix (two parities x 256 digits x ROW CTAs, u16), then the barrier word
__host__ __device__ constexpr size_t barrier_offset() { return 2ull * 256 * ROW * 2; }
__host__ __device__ constexpr size_t workspace_bytes() { return barrier_offset() + 256; }

__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  if (ctr == nullptr) {  // cooperative groups' barrier (no workspace word, no memset)
    cooperative_groups::this_grid().sync();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // bar.sync above + a cumulative release: the CTA's writes are published
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

}  // namespace grid_detail

// LSD sort of m <= max_chunk keys held in shared memory by one CTA of grid_detail::THREADS
// threads, on digits 0 .. NP-1 (small.cuh's passes: per-warp counters, digit-major scan, stable
// ranking by lane-ordered atomics or eight ballots; trivial digits skipped).  a holds the keys,
// b is the other buffer; returns the buffer with the result.  Every thread of the CTA calls it.
// Group form: NT threads (NT / 32 warps, NT >= 256) starting at warp `w0` of the CTA, synced by
// named barrier `bar` (the whole CTA: NT = THREADS, bar 0); wc, wsum, trivial are the group's.
__device__ __forceinline__ void group_sync(int bar, int nt) {
  if (bar == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nt) : "memory");
}
// ENC: the buffers hold encoded keys (a1 applied once at load), digits are plain shifts
template <int KIND, bool DESC, typename U, int NP, int NT = grid_detail::THREADS, bool ENC = false>
__device__ __forceinline__ U* small_lsd(U* a, U* b, uint32_t m, uint32_t* wc, uint32_t* wsum, int* trivial,
                                        int lane_atomics, int bar = 0) {
  constexpr int GW = NT / 32;  // warps of the group
  static_assert(NT >= 256 && NT % 32 == 0, "one thread per digit in the scan");
  const int tid = (int)threadIdx.x % NT, lane = tid & 31, w = tid >> 5;
  const uint32_t seg = (m + GW - 1) / GW;
  const uint32_t w_lo = min((uint32_t)w * seg, m), w_hi = min(w_lo + seg, m);
  U* cur = a;
  U* oth = b;
  for (int p = 0; p < NP; ++p) {
    const int sh = 8 * p;
    auto digit = [&](U x) {
      if constexpr (ENC) return uint32_t(x >> sh) & 0xFFu;
      else return uint32_t(key_encode<KIND, DESC>(x) >> sh) & 0xFFu;
    };
    group_sync(bar, NT);  // keys staged / the previous pass is done with wc and the buffers
    for (int i = tid; i < GW * 256; i += NT) wc[i] = 0;
    if (tid == 0) *trivial = 0;
    group_sync(bar, NT);
    for (uint32_t i = w_lo + lane; i < w_hi; i += 32) atomicAdd(&wc[w * 256 + digit(cur[i])], 1u);
    group_sync(bar, NT);
    uint32_t tot = 0;
    if (tid < 256) {
#pragma unroll
      for (int k = 0; k < GW; ++k) tot += wc[k * 256 + tid];
      if (tot == m) *trivial = 1;
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[w] = x;
      tot = x - tot;
    }
    group_sync(bar, NT);
    if (*trivial) continue;
    if (tid < 256) {
      uint32_t f = tot;
      for (int k = 0; k < w; ++k) f += wsum[k];
#pragma unroll
      for (int k = 0; k < GW; ++k) {
        const uint32_t e = wc[k * 256 + tid];
        wc[k * 256 + tid] = f;
        f += e;
      }
    }
    group_sync(bar, NT);
    uint32_t* slot = wc + w * 256;
    if (lane_atomics) {
      // four rounds per iteration: the keys are loaded first, then ranked in index order (one
      // converged atomic instruction per round; equal trip counts across lanes)
      for (uint32_t r = w_lo; r < w_hi; r += 128) {
        U x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t i = r + 32 * j + lane;
          x[j] = i < w_hi ? cur[i] : U(0);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __syncwarp();
          if (r + 32 * j + lane < w_hi) oth[atomicAdd(&slot[digit(x[j])], 1u)] = x[j];
        }
      }
    } else {
      for (uint32_t r = w_lo; r < w_hi; r += 32) {
        const uint32_t i = r + lane;
        const bool ok = i < w_hi;
        const U x = ok ? cur[i] : U(0);
        const uint32_t d = ok ? digit(x) : 256u;
        uint32_t peers = __ballot_sync(0xFFFFFFFFu, ok);
        if (!ok) peers = ~peers;
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) {
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (d >> bb) & 1u);
          peers &= ((d >> bb) & 1u) ? bal : ~bal;
        }
        const int leader = __ffs(peers) - 1;
        uint32_t q = 0;
        if (ok && lane == leader) {
          q = slot[d];
          slot[d] = q + __popc(peers);
        }
        q = __shfl_sync(0xFFFFFFFFu, q, leader);
        if (ok) oth[q + __popc(peers & lanemask_lt())] = x;
      }
    }
    U* t = cur;
    cur = oth;
    oth = t;
  }
  group_sync(bar, NT);
  return cur;
}

template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(grid_detail::THREADS, 1)
    k_grid_sort(U* __restrict__ keys, U* __restrict__ scratch, uint64_t n, uint32_t chunk,
                uint16_t* __restrict__ cnt, int keys_vec, int lane_atomics, int msd, int cgsync) {
  using namespace grid_detail;
  extern __shared__ __align__(128) unsigned char smem[];
  U* sk = reinterpret_cast<U*>(smem);                                  // the chunk, input order
  U* so = sk + max_chunk<U>();                                         // the chunk, digit order
  uint32_t* wc = reinterpret_cast<uint32_t*>(so + max_chunk<U>());    // [WARPS][256]
  uint32_t* tot = wc + WARPS * 256;                                    // totals -> global first slot
  uint32_t* first = tot + 256;                                         // counts of earlier CTAs
  uint32_t* lstart = first + 256;                                      // first local slot
  __shared__ uint32_t wsum[16], lsum[8];
  __shared__ int gtriv[2];  // MSD bucket groups' trivial flags
  __shared__ int trivial;
  __shared__ uint32_t bT[256], bS[256], bmax;  // MSD: bucket sizes and starts, largest bucket
  unsigned* bar = cgsync ? nullptr : reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(cnt) + barrier_offset());

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint64_t lo = (uint64_t)c * chunk;
  const uint32_t m = lo < n ? (uint32_t)min64(chunk, n - lo) : 0u;
  const uint32_t seg = (m + WARPS - 1) / WARPS;  // warp w's keys: [w seg, min(m, (w+1) seg))
  const uint32_t w_lo = min((uint32_t)w * seg, m), w_hi = min(w_lo + seg, m);
  unsigned nbar = 0;

  constexpr uint32_t V = 16 / sizeof(U);
  U* cur = keys;
  U* oth = scratch;
  // one grid-wide pass on digit p (count -> barrier -> scan -> rank -> write-out -> barrier);
  // record: keep the digit totals and global starts (bT, bS) and the largest total (bmax)
  auto pass = [&](int p, bool record) {
    const int sh = 8 * p;
    auto digit = [&](U x) { return uint32_t(key_encode<KIND, DESC>(x) >> sh) & 0xFFu; };
    uint16_t* cm = cnt + (size_t)(p & 1) * 256 * ROW;
    const bool vec = cur == scratch || keys_vec;  // chunk starts are 16-byte aligned (chunk % V == 0)

    // ---- A: stage the chunk (other CTAs' stores: through L2), count per warp, publish
    if (vec) {
      const uint4* src = reinterpret_cast<const uint4*>(cur + lo);
      uint4* dst = reinterpret_cast<uint4*>(sk);
      const uint32_t nv = m / V;
#pragma unroll 4
      for (uint32_t j = tid; j < nv; j += THREADS) dst[j] = __ldcg(src + j);
      for (uint32_t i = nv * V + tid; i < m; i += THREADS) sk[i] = __ldcg(cur + lo + i);
    } else {
#pragma unroll 4
      for (uint32_t i = tid; i < m; i += THREADS) sk[i] = __ldcg(cur + lo + i);
    }
    for (int i = tid; i < WARPS * 256; i += THREADS) wc[i] = 0;
    __syncthreads();
    for (uint32_t i = w_lo + lane; i < w_hi; i += 32) atomicAdd(&wc[w * 256 + digit(sk[i])], 1u);
    __syncthreads();
    if (tid < 256) {
      // per-warp first local slots within the digit; the CTA's count per digit
      uint32_t s = 0;
#pragma unroll
      for (int k = 0; k < WARPS; ++k) {
        const uint32_t e = wc[k * 256 + tid];
        wc[k * 256 + tid] = s;
        s += e;
      }
      cm[(size_t)tid * ROW + c] = (uint16_t)s;
      lstart[tid] = s;
    }
    if (tid == 0) trivial = 0;
    grid_barrier(bar, ++nbar * G);

    // ---- B: totals and the counts of the CTAs before this one, digit by digit.  Thread
    // (h, d) = (tid / 256, tid % 256) reads half h of row d: h is warp-uniform, so vectors past
    // G are skipped without divergence; the row's loads are all in flight at once.
    {
      const uint32_t d = tid & 255u, h = tid >> 8;
      const uint32_t half = (uint32_t)ROW / 2;  // a multiple of 8 halves: 16-byte aligned
      const uint4* row = reinterpret_cast<const uint4*>(cm + (size_t)d * ROW + h * half);
      uint32_t all = 0, before = 0;
      uint4 q[ROW / 16];
#pragma unroll
      for (uint32_t v = 0; v < half / 8; ++v)
        if (h * half + v * 8 < G) q[v] = __ldcg(row + v);
#pragma unroll
      for (uint32_t v = 0; v < half / 8; ++v) {
        const uint32_t base = h * half + v * 8;
        if (base < G) {
          const uint32_t x[4] = {q[v].x, q[v].y, q[v].z, q[v].w};
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t val = (x[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
            all += base + j < G ? val : 0u;  // entries past G were never written
            before += base + j < c ? val : 0u;
          }
        }
      }
      if (h == 1) {  // staged for the h = 0 thread of the same digit
        tot[d] = all;
        first[d] = before;
      }
      __syncthreads();
      if (h == 0) {
        all += tot[d];
        before += first[d];
        tot[d] = all;
        first[d] = before;
        if ((uint64_t)all == n) trivial = 1;
        if (record) {
          bT[d] = all;
          atomicMax(&bmax, all);
        }
      }
    }
    __syncthreads();
    if (trivial) return;  // every CTA saw the same totals: all skip this pass's scatter
    // exclusive scans over digits of the totals (global first slot) and of this CTA's counts
    if (tid < 256) {
      const uint32_t t = tot[tid], l = lstart[tid];
      uint32_t x = t, y = l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t xu = __shfl_up_sync(0xFFFFFFFFu, x, o);
        const uint32_t yu = __shfl_up_sync(0xFFFFFFFFu, y, o);
        if (lane >= o) {
          x += xu;
          y += yu;
        }
      }
      if (lane == 31) {
        wsum[w] = x;
        lsum[w] = y;
      }
      tot[tid] = x - t;
      lstart[tid] = y - l;
    }
    __syncthreads();
    if (tid < 256) {
      uint32_t add = 0, ladd = 0;
      for (int k = 0; k < w; ++k) {
        add += wsum[k];
        ladd += lsum[k];
      }
      tot[tid] += add + first[tid];
      if (record) bS[tid] = tot[tid] - first[tid];
      const uint32_t ls = lstart[tid] + ladd;
      lstart[tid] = ls;
#pragma unroll
      for (int k = 0; k < WARPS; ++k) wc[k * 256 + tid] += ls;
    }
    __syncthreads();

    // ---- C: stable local ranking into digit order ...
    uint32_t* slot = wc + w * 256;
    if (lane_atomics) {
      for (uint32_t r = w_lo; r < w_hi; r += 32) {  // equal trip counts: one instruction per round
        const uint32_t i = r + lane;
        __syncwarp();
        if (i < w_hi) {
          const U x = sk[i];
          so[atomicAdd(&slot[digit(x)], 1u)] = x;
        }
      }
    } else {
      for (uint32_t r = w_lo; r < w_hi; r += 32) {
        const uint32_t i = r + lane;
        const bool ok = i < w_hi;
        const U x = ok ? sk[i] : U(0);
        const uint32_t d = ok ? digit(x) : 256u;
        uint32_t peers = __ballot_sync(0xFFFFFFFFu, ok);
        if (!ok) peers = ~peers;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (d >> b) & 1u);
          peers &= ((d >> b) & 1u) ? bal : ~bal;
        }
        const int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (ok && lane == leader) {
          b = slot[d];
          slot[d] = b + __popc(peers);
        }
        b = __shfl_sync(0xFFFFFFFFu, b, leader);
        if (ok) so[b + __popc(peers & lanemask_lt())] = x;
      }
    }
    __syncthreads();
    // ... and the coalesced write-out: local slot i of digit d goes to tot[d] + i - lstart[d]
#pragma unroll 4
    for (uint32_t i = tid; i < m; i += THREADS) {
      const U x = so[i];
      const uint32_t d = digit(x);
      oth[tot[d] + (i - lstart[d])] = x;
    }
    U* t = cur;
    cur = oth;
    oth = t;
    grid_barrier(bar, ++nbar * G);
  };

  if (msd) {
    // MSD first (32-bit keys): one grid pass on the top digit partitions the keys into 256
    // contiguous buckets (in scratch); when every bucket fits one CTA's shared memory, CTA c
    // sorts buckets c, c + G, ... by the low three digits in shared memory (small.cuh's passes)
    // and writes them to their final place -- 2 grid barriers instead of 8.  Otherwise the LSD
    // passes below run on the partitioned keys (LSD does not depend on the input order).
    if (tid == 0) bmax = 0;
    if (tid < 256) {
      bT[tid] = 0;
      bS[tid] = 0;
    }
    __syncthreads();
    pass((int)sizeof(U) - 1, true);
    __syncthreads();
    if (trivial) {  // one top digit for all keys: the pass moved nothing; sizes are the totals
      if (tid < 256) {
        bS[tid] = 0;
      }
    }
    __syncthreads();
    // two groups of 8 warps sort two buckets at a time, each in half of the buffers
    constexpr uint32_t HALF = max_chunk<U>() / 2;
    if (bmax <= HALF) {
      const U* src = trivial ? keys : scratch;  // where the partitioned keys are
      const int g = w >> 3, gt = tid & 255;
      U* ga = sk + g * HALF;
      U* gb = so + g * HALF;
      __syncthreads();  // bT / bS / trivial read by everyone before the groups reuse `trivial`
      for (uint32_t d = c + (uint32_t)g * G; d < 256; d += 2 * G) {
        const uint32_t mb = bT[d], sb = bS[d];
        if (mb == 0) continue;
        group_sync(1 + g, 256);  // the group's previous bucket is written out
        for (uint32_t i = gt; i < mb; i += 256) ga[i] = key_encode<KIND, DESC>(__ldcg(src + sb + i));
        const U* r = small_lsd<KIND, DESC, U, (int)sizeof(U) - 1, 256, true>(ga, gb, mb, wc + g * 8 * 256,
                                                                           wsum + 8 * g, &gtriv[g], lane_atomics, 1 + g);
        for (uint32_t i = gt; i < mb; i += 256) keys[sb + i] = key_decode<KIND, DESC>(r[i]);
      }
      return;
    }
  }
  for (int p = 0; p < (int)sizeof(U); ++p) pass(p, false);
  if (cur != keys)
    for (uint32_t i = tid; i < m; i += THREADS) keys[lo + i] = __ldcg(cur + lo + i);
}

// Keys-only sorts with grid_min_n<U>() <= n <= grid_max_n<U>() (and above the single-CTA bound)
// take this path (BSORT_GRID=0 disables it; BSORT_GRID_MAX lowers the bound from SMs x
// max_chunk).  64-bit keys (8 passes, ~12 us of fixed cost each) only from 2^18 keys: below
// that the multi-launch path is as fast (tools/time_small.py).
template <typename U>
inline uint64_t grid_min_n() {
  return sizeof(U) == 4 ? 0 : (1ull << 18);
}
template <typename U>
inline uint64_t grid_max_n() {
  static const uint64_t v = [] {
    const char* e = getenv("BSORT_GRID");
    if (e && e[0] == '0') return (uint64_t)0;
    const uint64_t cap = min64((uint64_t)num_sms(), (uint64_t)grid_detail::MAX_CTAS) * grid_detail::max_chunk<U>();
    const char* mx = getenv("BSORT_GRID_MAX");
    return min64(mx ? strtoull(mx, nullptr, 10) : cap, cap);
  }();
  return v;
}

template <int KIND, bool DESC, typename U>
bsort_status_t launch_grid(U* keys, U* scratch, uint64_t n, uint16_t* cnt, cudaStream_t s) {
  using namespace grid_detail;
  auto kern = k_grid_sort<KIND, DESC, U>;
  constexpr size_t SMEM = smem_bytes<U>();
  static DeviceOnce attr;
  if (attr.pending()) {
    BSORT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr.mark();
  }
  static const uint64_t min_chunk = [] {
    const char* e = getenv("BSORT_GRID_CHUNK");
    return min64(e ? max64(256, strtoull(e, nullptr, 10)) : (uint64_t)4096, (uint64_t)max_chunk<U>());
  }();
  // CTAs: one per min_chunk keys, at most max_ctas (fewer, fuller CTAs win once every SM has
  // work: the count scan and the barriers grow with the grid), more only when chunks overflow
  static const uint64_t max_ctas = [] {
    const char* e = getenv("BSORT_GRID_CTAS");
    return e ? max64(1, strtoull(e, nullptr, 10)) : (uint64_t)128;
  }();
  constexpr uint64_t V = 16 / sizeof(U);
  const uint64_t sms = min64((uint64_t)num_sms(), (uint64_t)MAX_CTAS);
  uint64_t g = max64(1, min64((n + min_chunk - 1) / min_chunk, min64(max_ctas, sms)));
  if ((n + g - 1) / g > max_chunk<U>()) g = min64((n + max_chunk<U>() - 1) / max_chunk<U>(), sms);
  uint32_t chunk = (uint32_t)align_up((n + g - 1) / g, V);  // 16-byte aligned chunk starts
  if (chunk > max_chunk<U>()) return BSORT_ERROR_INVALID_ARGUMENT;  // caller checks grid_max_n
  g = (n + chunk - 1) / chunk;
  int keys_vec = (uintptr_t)keys % 16 == 0;
  int lane_atomics = atomics_lane_ordered(s) ? 1 : 0;
  // MSD-first fast path for 32-bit keys (BSORT_GRID_MSD=0: the plain LSD passes)
  static const bool msd_on = [] {
    const char* e = getenv("BSORT_GRID_MSD");
    return !(e && e[0] == '0');
  }();
  // (small grids would sort 256 / G buckets per CTA one after the other: 2^16 keys on 16 CTAs
  // took 72 us against 35 us for the LSD passes)
  int msd = (sizeof(U) == 4 && msd_on && g >= 64) ? 1 : 0;
  static const int cgsync = [] {
    const char* e = getenv("BSORT_GRID_CG");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  int cg = cgsync;
  void* args[] = {&keys, &scratch, &n, &chunk, &cnt, &keys_vec, &lane_atomics, &msd, &cg};
  if (!cg) {
    BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(reinterpret_cast<unsigned char*>(cnt) + barrier_offset(), 0, 4, s));
  }
  BSORT_LAUNCH(PROF_PASS, s, cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)g), dim3(THREADS), args,
                                                         SMEM, s));
  return BSORT_SUCCESS;
}

}  // namespace bsort
