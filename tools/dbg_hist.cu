// Standalone check of k_onesweep_hist_joint (debug harness).
#include <cstdio>
#include <cstdlib>
#include "onesweep.cuh"
namespace bsort {
void prof_begin(int, cudaStream_t) {}
void prof_end(int, cudaStream_t) {}
void count_launch() {}
int num_sms() { return 148; }
void set_last_cuda_error(cudaError_t) {}
}  // namespace bsort
using namespace bsort;
__global__ void fill(unsigned long long* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = z ^ (z >> 31);
  }
}
template <typename U, int JL>
void run(uint64_t n) {
  U* k; unsigned long long *gh, *gj;
  cudaMalloc(&k, n * sizeof(U)); cudaMalloc(&gh, 8 * 256 * 8); cudaMalloc(&gj, 65536 * 8);
  fill<<<1024, 256>>>((unsigned long long*)k, n * sizeof(U) / 8);
  cudaMemset(gh, 0, 8 * 256 * 8); cudaMemset(gj, 0, 65536 * 8);
  constexpr int P = sizeof(U);
  auto hk = k_onesweep_hist_joint<0, false, U, JL>;
  const int hsmem = (32768 + (P - 2) * 256 * JL) * 4;
  printf("setattr %d\n", (int)cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem));
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, hk);
  printf("regs %d local %zu smem %d\n", fa.numRegs, fa.localSizeBytes, hsmem); fflush(stdout);
  hk<<<148, HIST_THREADS, hsmem>>>(k, n, gh, gj);
  printf("launch %d\n", (int)cudaGetLastError()); fflush(stdout);
  printf("sync %d\n", (int)cudaDeviceSynchronize()); fflush(stdout);
  static unsigned long long h[65536], g[2048];
  cudaMemcpy(h, gj, sizeof(h), cudaMemcpyDeviceToHost); cudaMemcpy(g, gh, sizeof(g), cudaMemcpyDeviceToHost);
  unsigned long long sj = 0, s2 = 0; for (int i = 0; i < 65536; ++i) sj += h[i]; for (int i = 512; i < 768; ++i) s2 += g[i];
  printf("P=%d n=%llu joint sum %llu digit2 sum %llu\n", P, (unsigned long long)n, sj, s2);
}
int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 0) : 16789561;
  run<uint32_t, 32>(n);
  run<unsigned long long, 8>(n);
}
