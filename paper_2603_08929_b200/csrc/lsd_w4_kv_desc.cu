// lsd_w4_kv_desc.cu — instantiates the LSD path for 32-bit keys with a u32 payload, descending (see lsd_impl.cuh).
#include "lsd_impl.cuh"

namespace bsort {
bsort_status_t lsd_sort_w4_kv_desc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s) {
  return lsd_detail::lsd_dispatch<uint32_t, true, true>(kind, static_cast<uint32_t*>(keys), vals, n, ws, s);
}
}  // namespace bsort
