// lsd_w8_asc.cu — instantiates the LSD path for 64-bit keys, ascending (see lsd_impl.cuh).
#include "lsd_impl.cuh"

namespace bsort {
bsort_status_t lsd_sort_w8_asc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s) {
  return lsd_detail::lsd_dispatch<unsigned long long, false, false>(kind, static_cast<unsigned long long*>(keys), vals, n, ws, s);
}
}  // namespace bsort
