// lsd.cu — entry points of the 32/64-bit LSD path (§8 rows a2-a5): workspace size and the
// dispatch to the per-(key width, payload) translation units.
#include <algorithm>

#include "lsd_impl.cuh"

namespace bsort {

bsort_status_t lsd_sort_w4_asc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);
bsort_status_t lsd_sort_w4_desc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);
bsort_status_t lsd_sort_w4_kv_asc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);
bsort_status_t lsd_sort_w4_kv_desc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);
bsort_status_t lsd_sort_w8_asc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);
bsort_status_t lsd_sort_w8_desc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);
bsort_status_t lsd_sort_w8_kv_asc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);
bsort_status_t lsd_sort_w8_kv_desc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s);

size_t lsd_workspace_bytes(int bytes, uint64_t n, bool kv) {
  if (n <= 1) return 0;
  auto total = [&](uint64_t m) {
    return bytes == 4 ? lsd_detail::lsd_layout<uint32_t>(m, kv).total
                      : lsd_detail::lsd_layout<unsigned long long>(m, kv).total;
  };
  // Monotone in n (a workspace sized for n serves every m <= n: Sorter, in-place groups): below
  // WS_MIN_N the layout holds two look-back regions, so at and above it take at least the
  // largest layout below it.
  const uint64_t below = lsd_detail::WS_MIN_N - 1;
  return n >= lsd_detail::WS_MIN_N ? std::max(total(n), total(below)) : total(n);
}

bsort_status_t lsd_sort(const DtypeInfo& di, void* keys, uint32_t* vals, uint64_t n, bool desc, void* ws,
                        size_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < lsd_workspace_bytes(di.bytes, n, vals != nullptr)) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  auto* w = static_cast<unsigned char*>(ws);
  const int k = di.kind;
  if (di.bytes == 4) {
    if (vals) return desc ? lsd_sort_w4_kv_desc(k, keys, vals, n, w, s) : lsd_sort_w4_kv_asc(k, keys, vals, n, w, s);
    return desc ? lsd_sort_w4_desc(k, keys, nullptr, n, w, s) : lsd_sort_w4_asc(k, keys, nullptr, n, w, s);
  }
  if (vals) return desc ? lsd_sort_w8_kv_desc(k, keys, vals, n, w, s) : lsd_sort_w8_kv_asc(k, keys, vals, n, w, s);
  return desc ? lsd_sort_w8_desc(k, keys, nullptr, n, w, s) : lsd_sort_w8_asc(k, keys, nullptr, n, w, s);
}

}  // namespace bsort
