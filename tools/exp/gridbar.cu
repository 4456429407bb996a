// Grid-barrier cost on B200 (one CTA per SM, 512 threads, cooperative launch): flat counter,
// counters spread over 8 / 16 L2 lines, and cooperative groups' grid.sync.  Not part of the
// library; informs csrc/small.cuh.
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

template <int SPREAD>
__device__ __forceinline__ void bar(unsigned* ctr, unsigned k) {
  __syncthreads();
  const unsigned G = gridDim.x;
  if (threadIdx.x < SPREAD) {
    const unsigned i = threadIdx.x;
    // CTAs c with c % SPREAD == i arrive on counter i (32 u32 = 128 B apart)
    const unsigned members = G / SPREAD + (i < G % SPREAD ? 1u : 0u);
    if (blockIdx.x % SPREAD == i) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + 32 * i) : "memory");
    unsigned v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr + 32 * i) : "memory");
    } while (v < k * members);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

template <int SPREAD>
__global__ void k_bar(unsigned* ctr, int iters) {
  for (int k = 1; k <= iters; ++k) bar<SPREAD>(ctr, k);
}

__global__ void k_cg(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int k = 0; k < iters; ++k) g.sync();
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* ctr;
  cudaMalloc(&ctr, 4096 * 4);
  int iters = 1000;
  for (int G : {32, 64, 148}) {
    if (G > sms) continue;
    auto run = [&](auto kern) {
      return timeit([&] {
        cudaMemset(ctr, 0, 4096 * 4);
        void* args[] = {&ctr, &iters};
        cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(512), args, 0, 0);
      });
    };
    float f1 = run(k_bar<1>), f8 = run(k_bar<8>), f16 = run(k_bar<16>), f32 = run(k_bar<32>);
    float fc = timeit([&] {
      void* args[] = {&iters};
      cudaLaunchCooperativeKernel((const void*)k_cg, dim3(G), dim3(512), args, 0, 0);
    });
    printf("G=%d us/barrier: flat %.2f  spread8 %.2f  spread16 %.2f  spread32 %.2f  cg %.2f  (%s)\n", G,
           f1 * 1e3 / iters, f8 * 1e3 / iters, f16 * 1e3 / iters, f32 * 1e3 / iters, fc * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
