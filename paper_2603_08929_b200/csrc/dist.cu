// dist.cu — the MSD building blocks of the multi-GPU path (§8 rows a7, a9, N1): top-16-bit
// histogram and the (local or fused-remote) partition by destination rank.
#include "lsd_impl.cuh"

namespace bsort {
using namespace lsd_detail;

// ---------------------------------------------------------------- MSD partition (a7, a9)

namespace {
constexpr int TOP_BINS = BSORT_DIST_BINS;

// Top-16-bit histogram of the transformed keys (a7), one read of the keys: one CTA of 1024
// threads per SM holds all 65536 bins as u16 halves of 32768 smem words (128 KB); a half that
// reaches 0x8000 is drained into the global count (as the 16-bit counting path does), so the
// table never overflows.  Keys are read with 128-bit streaming loads, grid-stride; each CTA adds
// its nonzero bins to the global histogram at the end.  (Round 1: CTA pairs each read ALL keys
// and kept half of the bins -- 2x the algorithmic bytes.)
__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(1024, 1)
    k_dist_tophist(const U* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t th[];  // bin 2w in the low half of word w, 2w + 1 in the high half
  for (int i = threadIdx.x; i < TOP_BINS / 2; i += 1024) th[i] = 0;
  __syncthreads();
  constexpr int SH = (int)sizeof(U) * 8 - 16;
  auto add = [&](U x) {
    const uint32_t b = uint32_t(key_encode<KIND, DESC>(x) >> SH);
    const uint32_t sh = (b & 1u) << 4;
    const uint32_t old = atomicAdd(&th[b >> 1], 1u << sh);
    if (((old >> sh) & 0xFFFFu) == 0x7FFFu) {  // this add made the half 0x8000: drain it
      atomicAdd(&th[b >> 1], 0u - (0x8000u << sh));
      atomicAdd(&hist[b], 0x8000ull);
    }
  };
  constexpr int PER_VEC = 16 / (int)sizeof(U);
  const uint64_t T = (uint64_t)gridDim.x * 1024;
  const uint64_t gt = (uint64_t)blockIdx.x * 1024 + threadIdx.x;
  const uint64_t head = min64(n, ((16 - ((uintptr_t)keys & 15)) & 15) / sizeof(U));
  for (uint64_t i = gt; i < head; i += T) add(keys[i]);
  const U* vbase = keys + head;
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
    const uint4 q0 = ldg_stream16(vbase + i * PER_VEC), q1 = ldg_stream16(vbase + (i + T) * PER_VEC);
    const uint4 q2 = ldg_stream16(vbase + (i + 2 * T) * PER_VEC), q3 = ldg_stream16(vbase + (i + 3 * T) * PER_VEC);
    vec(q0); vec(q1); vec(q2); vec(q3);
  }
  for (; i < nv; i += T) vec(ldg_stream16(vbase + i * PER_VEC));
  for (uint64_t j = head + nv * PER_VEC + gt; j < n; j += T) add(keys[j]);
  __syncthreads();
  for (int w = threadIdx.x; w < TOP_BINS / 2; w += 1024) {
    const uint32_t c = th[w];
    if (c & 0xFFFFu) atomicAdd(&hist[2 * w], (unsigned long long)(c & 0xFFFFu));
    if (c >> 16) atomicAdd(&hist[2 * w + 1], (unsigned long long)(c >> 16));
  }
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
  BSORT_LAUNCH(PROF_DIST_HIST, s, k<<<num_sms(), 1024, smem, s>>>(keys, n, h));
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
