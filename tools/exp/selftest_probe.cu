// Lane-order self-test kernel (csrc/selftest.cu's pattern) run N times; prints the violation
// count of each run.  Used to check whether the check is stable, e.g. under an ncu session that
// does not profile it.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t st_mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void k_probe_lane_order(unsigned long long* bad) {
  __shared__ uint32_t tab[32][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = l; i < 256; i += 32) tab[w][i] = 0;
  __syncwarp();
  unsigned long long v = 0;
  for (int it = 0; it < 64; ++it) {
    const uint32_t r = st_mix(blockIdx.x * 7919u + threadIdx.x * 131u + it * 104729u);
    const int pattern = it % 3;
    uint32_t d = r & 255u;
    if (pattern == 1) d = (r >> 8) & 3u;
    const uint32_t act = pattern == 2 ? st_mix(it * 31u + w + blockIdx.x) | 1u : 0xFFFFFFFFu;
    const bool on = (act >> l) & 1u;
    uint32_t old = 0xFFFFFFFFu;
    if (on) old = atomicAdd(&tab[w][d], 1u);
    __syncwarp();
    for (int j = 0; j < 32; ++j) {
      const uint32_t dj = __shfl_sync(0xFFFFFFFFu, d, j);
      const uint32_t oj = __shfl_sync(0xFFFFFFFFu, old, j);
      if (j < l && on && ((act >> j) & 1u) && dj == d && !(oj < old)) ++v;
    }
  }
  if (v) atomicAdd(bad, v);
}
int main(int argc, char** argv) {
  int reps = argc > 1 ? atoi(argv[1]) : 10;
  unsigned long long* d; cudaMalloc(&d, 8);
  for (int r = 0; r < reps; ++r) {
    cudaMemset(d, 0, 8);
    k_probe_lane_order<<<148, 1024>>>(d);
    unsigned long long h = ~0ull;
    cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("run %d: violations %llu (%s)\n", r, h, cudaGetErrorString(e));
  }
  return 0;
}
