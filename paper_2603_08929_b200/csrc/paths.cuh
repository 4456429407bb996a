// paths.cuh — host entry points of the two sort paths (internal, not ABI).
#pragma once
#include "common.cuh"

namespace bsort {

struct DtypeInfo {
  int bytes;  // key width in bytes
  int kind;   // KIND_U / KIND_I / KIND_F
};
bool dtype_info(bsort_dtype_t dt, DtypeInfo* out);

// a6: 8/16-bit counting path (in place).
size_t counting_workspace_bytes(int bytes, uint64_t n);
bsort_status_t counting_sort(const DtypeInfo& di, void* keys, uint64_t n, bool desc, void* ws,
                             size_t ws_bytes, cudaStream_t s);

// a3-a5: 32/64-bit one-sweep LSD path.
// vals (nullable): 32-bit payload sorted along with the keys (key-value sort, §8 N3).
size_t lsd_workspace_bytes(int bytes, uint64_t n, bool kv = false);
bsort_status_t lsd_sort(const DtypeInfo& di, void* keys, uint32_t* vals, uint64_t n, bool desc, void* ws,
                        size_t ws_bytes, cudaStream_t s);

// §8 N4: in-place MSD partition(s) + LSD of bucket groups of at most `chunk` keys (inplace.cu).
uint64_t inplace_default_chunk(uint64_t n);
size_t inplace_workspace_bytes(int bytes, uint64_t n, uint64_t chunk);
bsort_status_t inplace_sort(const DtypeInfo& di, void* keys, uint64_t n, bool desc, uint64_t chunk, void* ws,
                            size_t ws_bytes, cudaStream_t s);

// a7/a9: distributed building blocks.
bsort_status_t dist_top_hist(const DtypeInfo& di, const void* keys, uint64_t n, bool desc,
                             uint64_t* dev_hist, cudaStream_t s);
size_t dist_partition_workspace_bytes(int bytes, uint64_t n, int nranks);
// dst_addrs == nullptr: bucketed copy into `out`; else (fused exchange) key of destination q
// goes to the device byte address range starting at dst_addrs[q].
bsort_status_t dist_partition(const DtypeInfo& di, const void* in, uint64_t n, bool desc,
                              const uint32_t* cuts, const uint64_t* send_counts, int nranks,
                              void* out, const uint64_t* dst_addrs, void* ws,
                              size_t ws_bytes, cudaStream_t s);

// §8 N2: exact splitting (csrc/exact.cu).
bsort_status_t dist_refine_hist(const DtypeInfo& di, const void* keys, uint64_t n, bool desc,
                                const uint64_t* prefixes, int m, int prefix_bits, uint64_t* hist,
                                cudaStream_t s);
bsort_status_t dist_class_hist(const DtypeInfo& di, const void* keys, uint64_t n, bool desc,
                               const uint64_t* values, int m, uint64_t* counts, cudaStream_t s);
size_t dist_class_partition_workspace_bytes();
bsort_status_t dist_partition_classes(const DtypeInfo& di, const void* in, uint64_t n, bool desc,
                                      const uint64_t* values, int m, const uint64_t* class_counts,
                                      void* out, void* ws, cudaStream_t s);

}  // namespace bsort
