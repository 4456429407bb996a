// Microbenchmark: throughput of 1-D bulk copies shared -> global (cp.async.bulk.global.shared::cta)
// of S bytes to scattered 16-byte-aligned destinations, vs the same data written by STG from
// threads.  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each CTA: ITER rounds; per round 256 copies of S bytes (one per thread of the first 256 threads...
// issued by `issuers` threads) from a 64 KB smem buffer to dst + pseudo-random 16B-aligned offsets
template <int S, bool STREAM>
__global__ void k_bulk(unsigned char* dst, size_t dst_bytes, int iters, int copies_per_round) {
  const size_t stream_bytes = dst_bytes / 256;
  extern __shared__ __align__(128) unsigned char sm[];
  const int t = threadIdx.x;
  for (int i = t; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  uint32_t r = (blockIdx.x * 1024 + t) * 2654435761u;
  const size_t nslots = dst_bytes / 4096;
  for (int it = 0; it < iters; ++it) {
    for (int c = t; c < copies_per_round; c += blockDim.x) {
      r = r * 1664525u + 1013904223u;
      // stream c % 256: consecutive chunks of a stream come from consecutive CTAs / rounds
      const size_t off = STREAM ? ((size_t)(c & 255) * stream_bytes + ((size_t)it * gridDim.x + blockIdx.x) * (S * (copies_per_round / 256)) + (c >> 8) * S)
                                : (size_t)(r % nslots) * 4096 + ((r >> 7) & 15) * 16;
      const uint32_t src = smem_u32(sm + (((c * 160) % (65536 - 1024)) & ~15));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(src), "n"(S)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// same bytes with STG from warps: each warp writes its runs of S bytes (32 lanes x 4B per row)
template <int S, bool STREAM>
__global__ void k_stg(unsigned char* dst, size_t dst_bytes, int iters, int copies_per_round) {
  const size_t stream_bytes = dst_bytes / 256;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  uint32_t r = (blockIdx.x * 1024 + warp) * 2654435761u;
  const size_t nslots = dst_bytes / 4096;
  for (int it = 0; it < iters; ++it) {
    for (int c = warp; c < copies_per_round; c += nw) {
      r = r * 1664525u + 1013904223u;
      const size_t off = STREAM ? ((size_t)(c & 255) * stream_bytes + ((size_t)it * gridDim.x + blockIdx.x) * (S * (copies_per_round / 256)) + (c >> 8) * S)
                                : (size_t)(r % nslots) * 4096 + ((r >> 7) & 15) * 16;
      uint32_t* d = reinterpret_cast<uint32_t*>(dst + off);
      for (int i = lane; i < S / 4; i += 32) d[i] = i + c;
    }
    __syncthreads();
  }
}

int main() {
  const size_t bytes = 1ull << 32;
  unsigned char* d;
  cudaMalloc(&d, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, void (*k)(unsigned char*, size_t, int, int), int S, int threads, int cpr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int iters = 400;
    k<<<148, threads, 65536>>>(d, bytes, 4, cpr);
    cudaEventRecord(a);
    k<<<148, threads, 65536>>>(d, bytes, iters, cpr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double tot = 148.0 * iters * cpr * S;
    printf("%-10s S=%4d copies/round=%4d threads=%4d: %.3f ms  %.0f GB/s  %.1f ns/copy/SM  err=%s\n", name, S, cpr,
           threads, ms, tot / (ms * 1e-3) / 1e9, ms * 1e6 / (iters * (double)cpr), cudaGetErrorString(cudaGetLastError()));
  };
  for (int cpr : {256}) {
    time("bulk-rand", k_bulk<128, false>, 128, 256, cpr);
    time("bulk-strm", k_bulk<128, true>, 128, 256, cpr);
    time("bulk-strm", k_bulk<160, true>, 160, 256, cpr);
    time("bulk-strm", k_bulk<256, true>, 256, 256, cpr);
    time("stg-rand", k_stg<128, false>, 128, 512, cpr);
    time("stg-strm", k_stg<128, true>, 128, 512, cpr);
    time("stg-strm", k_stg<160, true>, 160, 512, cpr);
    time("stg-strm", k_stg<256, true>, 256, 512, cpr);
  }
  return 0;
}
