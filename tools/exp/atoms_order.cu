// Microbenchmark / probe: (1) the order in which ATOMS.ADD (shared atomicAdd with return) hands
// out old values to lanes of one warp instruction that hit the same address; (2) throughput of
// shared-atomic ranking variants.  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// every warp: ITER rounds; per round each lane draws a bin (mod NB, skew by mask), does
// atomicAdd on its warp-private table, records whether old values are ascending in lane order
// among same-bin lanes.  bad[0] counts violations (ascending), bad[1] violations (descending).
template <int NB>
__global__ void k_order(uint32_t seed, int iters, unsigned long long* bad, uint32_t skewmask) {
  __shared__ uint32_t tab[32][NB];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = l; i < NB; i += 32) tab[w][i] = 0;
  __syncwarp();
  unsigned long long asc_bad = 0, desc_bad = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t r = mix(seed ^ mix(blockIdx.x * 977 + threadIdx.x * 131 + it * 7919));
    uint32_t d = (r & skewmask) % NB;
    uint32_t old = atomicAdd(&tab[w][d], 1u);
    // compare with every lower lane with the same bin
    for (int j = 0; j < 32; ++j) {
      uint32_t dj = __shfl_sync(0xffffffffu, d, j);
      uint32_t oj = __shfl_sync(0xffffffffu, old, j);
      if (j < l && dj == d) {
        if (!(oj < old)) asc_bad++;
        if (!(oj > old)) desc_bad++;
      }
    }
  }
  atomicAdd(&bad[0], asc_bad);
  atomicAdd(&bad[1], desc_bad);
}

// partial-warp (divergent) variant: only lanes with bit set in a random mask participate
template <int NB>
__global__ void k_order_div(uint32_t seed, int iters, unsigned long long* bad) {
  __shared__ uint32_t tab[32][NB];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = l; i < NB; i += 32) tab[w][i] = 0;
  __syncwarp();
  unsigned long long asc_bad = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t r = mix(seed ^ mix(blockIdx.x * 977 + threadIdx.x * 131 + it * 7919));
    uint32_t act = mix(seed + it * 31 + w);
    uint32_t d = r % NB;
    uint32_t old = 0xffffffffu;
    if ((act >> l) & 1) old = atomicAdd(&tab[w][d], 1u);
    for (int j = 0; j < 32; ++j) {
      uint32_t dj = __shfl_sync(0xffffffffu, d, j);
      uint32_t oj = __shfl_sync(0xffffffffu, old, j);
      bool aj = (act >> j) & 1, al = (act >> l) & 1;
      if (j < l && dj == d && aj && al && !(oj < old)) asc_bad++;
    }
  }
  atomicAdd(&bad[0], asc_bad);
}

// throughput: per warp-private tables (NB bins x REP replicas), ITEMS atomics per lane per round
template <int NB, int REP, bool RET>
__global__ void k_tput(uint32_t seed, int iters, uint32_t* sink, uint32_t skewmask) {
  extern __shared__ uint32_t tab[];  // [warps][NB*REP]
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  uint32_t* t = tab + w * NB * REP;
  for (int i = l; i < NB * REP; i += 32) t[i] = 0;
  __syncwarp();
  uint32_t acc = 0;
  uint32_t r = mix(seed ^ (blockIdx.x * 1024 + threadIdx.x));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      r = r * 1664525u + 1013904223u;
      uint32_t d = ((r >> 8) & skewmask) % NB;
      uint32_t a = d * REP + (REP > 1 ? (l % REP) : 0);
      if (RET) acc += atomicAdd(&t[a], 1u);
      else atomicAdd(&t[a], 1u);
    }
  }
  if (acc == 0x12345678) sink[0] = acc;
  if (!RET && l == 0) sink[1 + (blockIdx.x & 7)] = t[0];
}

int main() {
  unsigned long long* bad;
  cudaMalloc(&bad, 16);
  uint32_t* sink;
  cudaMalloc(&sink, 64);
  const uint32_t masks[] = {0xffffffffu, 0x7u, 0x3u, 0x1u, 0x0u, 0x1fu};
  for (uint32_t m : masks) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bad, 0, 16);
      k_order<256><<<296, 1024>>>(1234u + rep * 77 + m, 200, bad, m);
      unsigned long long h[2];
      cudaMemcpy(h, bad, 16, cudaMemcpyDeviceToHost);
      printf("order NB=256 skewmask=%08x rep %d: asc_violations=%llu desc_violations=%llu\n", m, rep, h[0], h[1]);
    }
  }
  cudaMemset(bad, 0, 16);
  k_order<16><<<296, 1024>>>(99u, 500, bad, 0xffffffffu);
  { unsigned long long h[2]; cudaMemcpy(h, bad, 16, cudaMemcpyDeviceToHost);
    printf("order NB=16: asc_violations=%llu desc_violations=%llu\n", h[0], h[1]); }
  cudaMemset(bad, 0, 16);
  k_order_div<64><<<296, 1024>>>(5u, 500, bad);
  { unsigned long long h[2]; cudaMemcpy(h, bad, 16, cudaMemcpyDeviceToHost);
    printf("order divergent NB=64: asc_violations=%llu\n", h[0]); }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*kern)(uint32_t, int, uint32_t*, uint32_t), int nb, int rep, uint32_t m) {
    int smem = 32 * nb * rep * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 200;
    kern<<<148, 1024, smem>>>(1, iters, sink, m);
    cudaEventRecord(e0);
    kern<<<148, 1024, smem>>>(2, iters, sink, m);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * 1024 * iters * 16;
    printf("%-28s skew=%08x: %.3f ms  %.3f SM-cycles per lane-op (at 1.965 GHz)\n", name, m, ms,
           ms * 1e-3 * 1.965e9 * 148 / ops);
  };
  for (uint32_t m : {0xffffffffu, 0x7u, 0x0u}) {
    run("ret NB=256 REP=1", k_tput<256, 1, true>, 256, 1, m);
    run("ret NB=256 REP=4", k_tput<256, 4, true>, 256, 4, m);
    run("noret NB=256 REP=1", k_tput<256, 1, false>, 256, 1, m);
    run("noret NB=256 REP=4", k_tput<256, 4, false>, 256, 4, m);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
