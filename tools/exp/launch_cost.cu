// Host cost of enqueueing work on B200: an empty kernel (small / large dynamic smem), a 16-byte
// memset, and one bsort_sort_ws of n keys (i32) through libbsort.  Not part of the library.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -Iinclude tools/exp/launch_cost.cu
//      -Lpaper_2603_08929_b200 -lbsort -Xlinker -rpath=$PWD/paper_2603_08929_b200 -o tools/exp/launch_cost
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bsort.h"

__global__ void k_empty(int* p) {
  if (p && threadIdx.x == 9999) *p = 1;
}

template <typename F>
double host_us(F f, int reps) {
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : (1u << 20);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int* d;
  cudaMalloc(&d, 1 << 20);
  const int reps = 2000;
  printf("empty <<<148,1024,0>>>       %.2f us\n", host_us([&] { k_empty<<<148, 1024, 0, s>>>(d); }, reps));
  printf("empty <<<148,1024,200KB>>>   %.2f us\n", host_us([&] { k_empty<<<148, 1024, 200 * 1024, s>>>(d); }, reps));
  printf("memset 16 B                  %.2f us\n", host_us([&] { cudaMemsetAsync(d, 0, 16, s); }, reps));
  printf("cudaGetLastError             %.3f us\n", host_us([&] { cudaGetLastError(); }, reps * 10));
  int dev;
  printf("cudaGetDevice                %.3f us\n", host_us([&] { cudaGetDevice(&dev); }, reps * 10));
  std::vector<int> h(n);
  for (uint64_t i = 0; i < n; ++i) h[i] = (int)(i * 2654435761u);
  int* keys;
  cudaMalloc(&keys, n * 4);
  cudaMemcpy(keys, h.data(), n * 4, cudaMemcpyHostToDevice);
  size_t wsb = bsort_workspace_bytes(BSORT_I32, n);
  void* ws;
  cudaMalloc(&ws, wsb);
  bsort_sort_ws(BSORT_I32, keys, n, BSORT_ASCENDING, ws, wsb, s);
  printf("bsort_sort_ws n=%llu          %.2f us host (launches per call: ", (unsigned long long)n,
         host_us([&] { bsort_sort_ws(BSORT_I32, keys, n, BSORT_ASCENDING, ws, wsb, s); }, 200));
  uint64_t c0 = bsort_launch_count();
  bsort_sort_ws(BSORT_I32, keys, n, BSORT_ASCENDING, ws, wsb, s);
  printf("%llu)\n", (unsigned long long)(bsort_launch_count() - c0));
  cudaStreamSynchronize(s);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
