// lsd_w8_desc.cu — instantiates the LSD path for 64-bit keys, descending (see lsd_impl.cuh).
#include "lsd_impl.cuh"

namespace bsort {
bsort_status_t lsd_sort_w8_desc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s) {
  return lsd_detail::lsd_dispatch<unsigned long long, false, true>(kind, static_cast<unsigned long long*>(keys), vals, n, ws, s);
}
}  // namespace bsort
