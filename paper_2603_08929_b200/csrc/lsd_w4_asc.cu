// lsd_w4_asc.cu — instantiates the LSD path for 32-bit keys, ascending (see lsd_impl.cuh).
#include "lsd_impl.cuh"

namespace bsort {
bsort_status_t lsd_sort_w4_asc(int kind, void* keys, uint32_t* vals, uint64_t n, unsigned char* ws,
                              cudaStream_t s) {
  return lsd_detail::lsd_dispatch<uint32_t, false, false>(kind, static_cast<uint32_t*>(keys), vals, n, ws, s);
}
}  // namespace bsort
