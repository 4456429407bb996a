// dist.cu — the MSD building blocks of the multi-GPU path (§8 rows a7, a9, N1): top-16-bit
// histogram and the (local or fused-remote) partition by destination rank.
#include "lsd_impl.cuh"

namespace bsort {
using namespace lsd_detail;

// ---------------------------------------------------------------- MSD partition (a7, a9)

namespace {
constexpr int TOP_BINS = BSORT_DIST_BINS;

// Top-16-bit histogram of the transformed keys: 65536 u32 bins do not fit next to a useful
// occupancy, so each CTA counts into a 16-bit-index smem table of 32768 u32 for its half of
// the bins (CTA pairs, as in the 16-bit counting path) and flushes with global atomics.
template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(1024, 1)
    k_dist_tophist(const U* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t th[];
  const uint32_t half = blockIdx.x & 1;
  const uint32_t chunk = blockIdx.x >> 1;
  const uint32_t pairs = gridDim.x >> 1;
  for (int i = threadIdx.x; i < TOP_BINS / 2; i += 1024) th[i] = 0;
  __syncthreads();
  const uint64_t per = (n + pairs - 1) / pairs;
  const uint64_t s0 = min64(n, (uint64_t)chunk * per), s1 = min64(n, s0 + per);
  for (uint64_t i = s0 + threadIdx.x; i < s1; i += 1024) {
    const uint32_t b = uint32_t(key_encode<KIND, DESC>(keys[i]) >> (sizeof(U) * 8 - 16));
    if ((b >> 15) == half) atomicAdd(&th[b & 0x7FFF], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < TOP_BINS / 2; b += 1024)
    if (th[b]) atomicAdd(&hist[half * (TOP_BINS / 2) + b], (unsigned long long)th[b]);
}

template <int KIND, bool DESC, typename U>
bsort_status_t tophist_run(const U* keys, uint64_t n, uint64_t* hist, cudaStream_t s) {
  auto* h = reinterpret_cast<unsigned long long*>(hist);
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(h, 0, TOP_BINS * 8, s));
  if (n == 0) return BSORT_SUCCESS;
  auto k = k_dist_tophist<KIND, DESC, U>;
  constexpr int smem = TOP_BINS / 2 * 4;
  static DeviceOnce attr;
  if (attr.pending()) {
    BSORT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr.mark();
  }
  const int pairs = max(1, num_sms() / 2);
  BSORT_LAUNCH(PROF_DIST_HIST, s, k<<<2 * pairs, 1024, smem, s>>>(keys, n, h));
  return BSORT_SUCCESS;
}

// Workspace of the MSD partition: tile counter, bucket bases, per-bucket running counts.  The
// partition is an unstable pass (order inside a destination bucket is irrelevant: every rank
// sorts what it receives), so it needs no look-back array.
size_t part_layout(size_t* counters_off, size_t* bases_off, size_t* gcount_off) {
  size_t off = 0;
  *counters_off = off; off = align_up(off + 64, 256);
  *bases_off = off;    off = align_up(off + 256 * 8, 256);
  *gcount_off = off;   off = align_up(off + 256 * 8, 256);
  return off;
}

template <int KIND, bool DESC, typename U>
bsort_status_t part_run(const U* in, uint64_t n, const uint32_t* cuts, int nranks, U* out, unsigned char* ws,
                        const unsigned long long* host_bases, const unsigned long long* host_dst, cudaStream_t s) {
  size_t co, bo, go;
  const size_t total = part_layout(&co, &bo, &go);
  auto* counter = reinterpret_cast<uint32_t*>(ws + co);
  auto* bases = reinterpret_cast<unsigned long long*>(ws + bo);
  auto* gcount = reinterpret_cast<unsigned long long*>(ws + go);
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(ws, 0, total, s));
  // bases: exclusive offsets of each destination bucket (from the caller's send counts; the
  // pageable copy is staged before cudaMemcpyAsync returns).
  BSORT_CUDA(cudaMemcpyAsync(bases, host_bases, 256 * 8, cudaMemcpyHostToDevice, s));
  auto fill = [&](auto& dg) {
    for (int q = 0; q <= nranks; ++q) dg.cuts[q] = cuts[q];
    for (int q = nranks + 1; q <= BSORT_DIST_MAX_RANKS; ++q) dg.cuts[q] = TOP_BINS;
    dg.nranks = nranks;
  };
  if (host_dst != nullptr) {  // fused partition + exchange: write into the owners' buffers
    RankDigit<KIND, DESC, U, true> dg;
    fill(dg);
    for (int q = 0; q < BSORT_DIST_MAX_RANKS; ++q) dg.dst_base[q] = q < nranks ? host_dst[q] : 0ull;
    return launch_pass<U, RANK_UNSTABLE, uint32_t>(in, const_cast<U*>(in), n, dg, bases, (uint32_t*)nullptr, gcount,
                                                   counter, nullptr, 0, s);
  }
  RankDigit<KIND, DESC, U> dg;
  fill(dg);
  return launch_pass<U, RANK_UNSTABLE, uint32_t>(in, out, n, dg, bases, (uint32_t*)nullptr, gcount, counter, nullptr,
                                                 0, s);
}

}  // namespace

bsort_status_t dist_top_hist(const DtypeInfo& di, const void* keys, uint64_t n, bool desc, uint64_t* hist,
                             cudaStream_t s) {
#define TOPH(U_)                                                                                                  \
  switch (di.kind) {                                                                                              \
    case KIND_U: return desc ? tophist_run<KIND_U, true>((const U_*)keys, n, hist, s)                             \
                             : tophist_run<KIND_U, false>((const U_*)keys, n, hist, s);                           \
    case KIND_I: return desc ? tophist_run<KIND_I, true>((const U_*)keys, n, hist, s)                             \
                             : tophist_run<KIND_I, false>((const U_*)keys, n, hist, s);                           \
    default: return desc ? tophist_run<KIND_F, true>((const U_*)keys, n, hist, s)                                 \
                         : tophist_run<KIND_F, false>((const U_*)keys, n, hist, s);                               \
  }
  if (di.bytes == 4) { TOPH(uint32_t) }
  TOPH(unsigned long long)
#undef TOPH
}

size_t dist_partition_workspace_bytes(int bytes, uint64_t n, int nranks) {
  (void)bytes;
  (void)n;
  (void)nranks;
  size_t a, b, c;
  return part_layout(&a, &b, &c);
}

bsort_status_t dist_partition(const DtypeInfo& di, const void* in, uint64_t n, bool desc, const uint32_t* cuts,
                              const uint64_t* send_counts, int nranks, void* out, const uint64_t* dst_addrs,
                              void* ws, size_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < dist_partition_workspace_bytes(di.bytes, n, nranks)) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  if (n == 0) return BSORT_SUCCESS;
  unsigned long long hb[256];
  unsigned long long acc = 0;
  for (int q = 0; q < 256; ++q) {
    hb[q] = acc;
    if (q < nranks) acc += send_counts[q];
  }
  if (acc != n) return BSORT_ERROR_INVALID_ARGUMENT;
  auto* w = static_cast<unsigned char*>(ws);
  const auto* hd = reinterpret_cast<const unsigned long long*>(dst_addrs);
#define PART(U_)                                                                                                  \
  {                                                                                                               \
    const U_* i_ = static_cast<const U_*>(in);                                                                    \
    U_* o_ = static_cast<U_*>(out);                                                                               \
    switch (di.kind * 2 + (desc ? 1 : 0)) {                                                                       \
      case 0: return part_run<KIND_U, false, U_>(i_, n, cuts, nranks, o_, w, hb, hd, s);                              \
      case 1: return part_run<KIND_U, true, U_>(i_, n, cuts, nranks, o_, w, hb, hd, s);                               \
      case 2: return part_run<KIND_I, false, U_>(i_, n, cuts, nranks, o_, w, hb, hd, s);                              \
      case 3: return part_run<KIND_I, true, U_>(i_, n, cuts, nranks, o_, w, hb, hd, s);                               \
      case 4: return part_run<KIND_F, false, U_>(i_, n, cuts, nranks, o_, w, hb, hd, s);                              \
      default: return part_run<KIND_F, true, U_>(i_, n, cuts, nranks, o_, w, hb, hd, s);                              \
    }                                                                                                             \
  }
  if (di.bytes == 4) PART(uint32_t)
  PART(unsigned long long)
#undef PART
}

}  // namespace bsort
