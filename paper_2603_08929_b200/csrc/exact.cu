// exact.cu — exact splitting for the multi-GPU path.
//
// The bin-granular MSD split (a7/a8) cuts between top-16-bit bins, so a heavy bin (many equal or
// nearly equal keys) lands on one rank.  Exact splitting finds, for every rank boundary r, the
// transformed key K_r of global rank floor(r*N/P) by refining the boundary bins 16 bits at a time
// (k_dist_refine_hist + all-reduce, host search), and then partitions by CLASS: with the distinct
// split keys V_0 < ... < V_{m-1}, class(x) = 2j for V_{j-1} < enc(x) < V_j and 2j+1 for
// enc(x) == V_j.  Classes are contiguous in the partitioned buffer and increase with the key, so
// every destination's share is one contiguous slice of it: equal keys are split by COUNT at the
// class boundaries (equal keys are interchangeable, reading Q12), giving every rank exactly
// floor((r+1)N/P) - floor(rN/P) keys whatever the skew.
#include "lsd_impl.cuh"

namespace bsort {
using namespace lsd_detail;

namespace {

// Destination class of a key against the distinct split keys v[0..m) (encoded, increasing).
template <int KIND, bool DESC, typename U>
struct ClassDigit {
  static constexpr bool REMOTE = false;
  unsigned long long v[BSORT_DIST_MAX_RANKS];
  int m;
  __device__ __forceinline__ uint32_t operator()(U x) const {
    const U e = key_encode<KIND, DESC>(x);
    int lo = 0, hi = m;  // lower bound: first j with v[j] >= e
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (U(v[mid]) < e) lo = mid + 1; else hi = mid;
    }
    return 2u * (uint32_t)lo + ((lo < m && U(v[lo]) == e) ? 1u : 0u);
  }
  __device__ __forceinline__ uint32_t digit_low(U x, U* low) const {
    *low = U(0);
    return (*this)(x);
  }
};

struct RefineParams {
  unsigned long long prefix[BSORT_DIST_MAX_RANKS];  // unresolved boundary prefixes, increasing
  int m;
  int shift_prefix;  // e >> shift_prefix is a key's prefix
  int shift_bin;     // (e >> shift_bin) & 0xFFFF is its next 16 bits
};

constexpr int EX_THREADS = 512;

// hist[j * 65536 + b] += #{keys whose prefix == prefix[j] and next 16 bits == b}.  Whole warps
// step through the keys together; a warp whose 32 keys hit one bin adds once (runs of equal
// keys are exactly the case exact splitting exists for).
template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(EX_THREADS)
    k_dist_refine_hist(const U* __restrict__ keys, uint64_t n, RefineParams p,
                       unsigned long long* __restrict__ hist) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (EX_THREADS / 32);
  const uint64_t w = (uint64_t)blockIdx.x * (EX_THREADS / 32) + (threadIdx.x >> 5);
  for (uint64_t base = w * 32; base < n; base += warps * 32) {
    const uint64_t i = base + lane;
    uint32_t slot = 0xFFFFFFFFu;
    if (i < n) {
      const U e = key_encode<KIND, DESC>(keys[i]);
      const unsigned long long pre = (unsigned long long)(e >> p.shift_prefix);
      int lo = 0, hi = p.m;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (p.prefix[mid] < pre) lo = mid + 1; else hi = mid;
      }
      if (lo < p.m && p.prefix[lo] == pre) slot = (uint32_t)lo * 65536u + (uint32_t((e >> p.shift_bin) & 0xFFFFu));
    }
    const uint32_t s0 = __shfl_sync(0xffffffffu, slot, 0);
    if (__all_sync(0xffffffffu, slot == s0)) {
      if (lane == 0 && s0 != 0xFFFFFFFFu) atomicAdd(&hist[s0], 32ull);
    } else if (slot != 0xFFFFFFFFu) {
      atomicAdd(&hist[slot], 1ull);
    }
  }
}

// counts[c] = #{keys of class c}, c < 2m+1.  Lane-banked smem counters (bank = lane): no
// conflicts and no same-address serialization even when every key is equal.
template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(EX_THREADS)
    k_dist_class_hist(const U* __restrict__ keys, uint64_t n, ClassDigit<KIND, DESC, U> cd,
                      unsigned long long* __restrict__ counts) {
  __shared__ uint32_t h[(2 * BSORT_DIST_MAX_RANKS + 1) * 32];
  const int classes = 2 * cd.m + 1;
  for (int i = threadIdx.x; i < classes * 32; i += EX_THREADS) h[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t T = (uint64_t)gridDim.x * EX_THREADS;
  for (uint64_t i = (uint64_t)blockIdx.x * EX_THREADS + threadIdx.x; i < n; i += T)
    atomicAdd(&h[cd(keys[i]) * 32 + lane], 1u);
  __syncthreads();
  for (int c = threadIdx.x; c < classes; c += EX_THREADS) {
    uint32_t s = 0;
    for (int l = 0; l < 32; ++l) s += h[c * 32 + l];
    if (s) atomicAdd(&counts[c], (unsigned long long)s);
  }
}

template <int KIND, bool DESC, typename U>
ClassDigit<KIND, DESC, U> make_class_digit(const uint64_t* values, int m) {
  ClassDigit<KIND, DESC, U> cd;
  for (int j = 0; j < BSORT_DIST_MAX_RANKS; ++j) cd.v[j] = j < m ? values[j] : ~0ull;
  cd.m = m;
  return cd;
}

template <int KIND, bool DESC, typename U>
bsort_status_t refine_run(const U* keys, uint64_t n, const uint64_t* prefixes, int m, int prefix_bits,
                          uint64_t* hist, cudaStream_t s) {
  RefineParams p;
  for (int j = 0; j < BSORT_DIST_MAX_RANKS; ++j) p.prefix[j] = j < m ? prefixes[j] : ~0ull;
  p.m = m;
  p.shift_prefix = (int)sizeof(U) * 8 - prefix_bits;
  p.shift_bin = p.shift_prefix - 16;
  auto* h = reinterpret_cast<unsigned long long*>(hist);
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(h, 0, (size_t)m * 65536 * 8, s));
  if (n == 0) return BSORT_SUCCESS;
  const uint64_t grid = max64(1, min64((n + EX_THREADS - 1) / EX_THREADS, (uint64_t)num_sms() * 4));
  BSORT_LAUNCH(PROF_DIST_HIST, s, k_dist_refine_hist<KIND, DESC, U><<<(unsigned)grid, EX_THREADS, 0, s>>>(keys, n, p, h));
  return BSORT_SUCCESS;
}

template <int KIND, bool DESC, typename U>
bsort_status_t class_hist_run(const U* keys, uint64_t n, const uint64_t* values, int m, uint64_t* counts,
                              cudaStream_t s) {
  auto* c = reinterpret_cast<unsigned long long*>(counts);
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(c, 0, (size_t)(2 * m + 1) * 8, s));
  if (n == 0) return BSORT_SUCCESS;
  const uint64_t grid = max64(1, min64((n + EX_THREADS - 1) / EX_THREADS, (uint64_t)num_sms() * 4));
  BSORT_LAUNCH(PROF_DIST_HIST, s,
               k_dist_class_hist<KIND, DESC, U><<<(unsigned)grid, EX_THREADS, 0, s>>>(
                   keys, n, make_class_digit<KIND, DESC, U>(values, m), c));
  return BSORT_SUCCESS;
}

size_t class_layout(size_t* counter_off, size_t* bases_off, size_t* gcount_off) {
  size_t off = 0;
  *counter_off = off; off = align_up(off + 64, 256);
  *bases_off = off;   off = align_up(off + 256 * 8, 256);
  *gcount_off = off;  off = align_up(off + 256 * 8, 256);
  return off;
}

template <int KIND, bool DESC, typename U>
bsort_status_t class_part_run(const U* in, uint64_t n, const uint64_t* values, int m, const uint64_t* counts,
                              U* out, unsigned char* ws, cudaStream_t s) {
  size_t co, bo, go;
  const size_t total = class_layout(&co, &bo, &go);
  unsigned long long hb[256];
  unsigned long long acc = 0;
  for (int c = 0; c < 256; ++c) {
    hb[c] = acc;
    if (c < 2 * m + 1) acc += counts[c];
  }
  if (acc != n) return BSORT_ERROR_INVALID_ARGUMENT;
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(ws, 0, total, s));
  BSORT_CUDA(cudaMemcpyAsync(ws + bo, hb, sizeof(hb), cudaMemcpyHostToDevice, s));
  return launch_pass<U, RANK_UNSTABLE, uint32_t>(in, out, n, make_class_digit<KIND, DESC, U>(values, m),
                                                 reinterpret_cast<unsigned long long*>(ws + bo), (uint32_t*)nullptr,
                                                 reinterpret_cast<unsigned long long*>(ws + go),
                                                 reinterpret_cast<uint32_t*>(ws + co), nullptr, 0, s);
}

// dispatch over (key width, kind, direction)
#define BSORT_EXACT_DISPATCH(...)                                                        \
  switch ((di.bytes == 4 ? 0 : 6) + di.kind * 2 + (desc ? 1 : 0)) {                       \
    case 0: { using U = uint32_t; constexpr int K = KIND_U; constexpr bool D = false; __VA_ARGS__ } \
    case 1: { using U = uint32_t; constexpr int K = KIND_U; constexpr bool D = true; __VA_ARGS__ }  \
    case 2: { using U = uint32_t; constexpr int K = KIND_I; constexpr bool D = false; __VA_ARGS__ } \
    case 3: { using U = uint32_t; constexpr int K = KIND_I; constexpr bool D = true; __VA_ARGS__ }  \
    case 4: { using U = uint32_t; constexpr int K = KIND_F; constexpr bool D = false; __VA_ARGS__ } \
    case 5: { using U = uint32_t; constexpr int K = KIND_F; constexpr bool D = true; __VA_ARGS__ }  \
    case 6: { using U = unsigned long long; constexpr int K = KIND_U; constexpr bool D = false; __VA_ARGS__ } \
    case 7: { using U = unsigned long long; constexpr int K = KIND_U; constexpr bool D = true; __VA_ARGS__ }  \
    case 8: { using U = unsigned long long; constexpr int K = KIND_I; constexpr bool D = false; __VA_ARGS__ } \
    case 9: { using U = unsigned long long; constexpr int K = KIND_I; constexpr bool D = true; __VA_ARGS__ }  \
    case 10: { using U = unsigned long long; constexpr int K = KIND_F; constexpr bool D = false; __VA_ARGS__ } \
    default: { using U = unsigned long long; constexpr int K = KIND_F; constexpr bool D = true; __VA_ARGS__ } \
  }

}  // namespace

bsort_status_t dist_refine_hist(const DtypeInfo& di, const void* keys, uint64_t n, bool desc,
                                const uint64_t* prefixes, int m, int prefix_bits, uint64_t* hist, cudaStream_t s) {
  BSORT_EXACT_DISPATCH(return refine_run<K, D, U>(static_cast<const U*>(keys), n, prefixes, m, prefix_bits, hist, s);)
}

bsort_status_t dist_class_hist(const DtypeInfo& di, const void* keys, uint64_t n, bool desc, const uint64_t* values,
                               int m, uint64_t* counts, cudaStream_t s) {
  BSORT_EXACT_DISPATCH(return class_hist_run<K, D, U>(static_cast<const U*>(keys), n, values, m, counts, s);)
}

size_t dist_class_partition_workspace_bytes() {
  size_t a, b, c;
  return class_layout(&a, &b, &c);
}

bsort_status_t dist_partition_classes(const DtypeInfo& di, const void* in, uint64_t n, bool desc,
                                      const uint64_t* values, int m, const uint64_t* class_counts, void* out,
                                      void* ws, cudaStream_t s) {
  auto* w = static_cast<unsigned char*>(ws);
  BSORT_EXACT_DISPATCH(return class_part_run<K, D, U>(static_cast<const U*>(in), n, values, m, class_counts,
                                                      static_cast<U*>(out), w, s);)
}

}  // namespace bsort
