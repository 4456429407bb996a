// Run-time checks of hardware behaviour the fast paths rely on (bsort_selftest, include/bsort.h).
//
// Check 1 -- shared-atomic lane order: when lanes of ONE warp instruction `atomicAdd` the same
// shared word, the hardware hands out the old values in ascending lane order.  The stable
// rankings of k_pass2 (pass2.cuh) and of the small-n kernel (small.cuh) take a key's position
// from that return value, which is stable exactly when this holds.  The CUDA programming guide
// leaves the order unspecified; sm_100 measured it lane-ordered in every pattern tried
// (tools/exp/atoms_order.cu).  The check below re-measures it once per device on first use:
// 148 CTAs x 32 warps x 64 rounds of uniform, skewed (few bins) and partial-warp patterns.  If
// any violation shows up, those kernels are not used on that device (the look-back passes fall
// back to k_onesweep_pass_ws, the small kernel to ballot-based peer ranking).
#include <cuda_runtime.h>

#include <mutex>

#include "bsort.h"
#include "common.cuh"

namespace bsort {
namespace {

__device__ __forceinline__ uint32_t st_mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void k_selftest_lane_order(unsigned long long* bad) {
  __shared__ uint32_t tab[32][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = l; i < 256; i += 32) tab[w][i] = 0;
  __syncwarp();
  unsigned long long v = 0;
  for (int it = 0; it < 64; ++it) {
    const uint32_t r = st_mix(blockIdx.x * 7919u + threadIdx.x * 131u + it * 104729u);
    const int pattern = it % 3;
    uint32_t d = r & 255u;                      // uniform over 256 counters
    if (pattern == 1) d = (r >> 8) & 3u;        // skewed: 4 counters
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

std::mutex g_mu;
int g_state[64] = {};  // 0 = not run, 1 = holds, 2 = violated / could not run

int run_lane_order_check() {
  unsigned long long* d = nullptr;
  cudaStream_t st = nullptr;
  int state = 2;
  if (cudaMalloc(&d, 8) == cudaSuccess && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
      cudaMemsetAsync(d, 0, 8, st) == cudaSuccess) {
    k_selftest_lane_order<<<num_sms(), 1024, 0, st>>>(d);
    unsigned long long h = ~0ull;
    if (cudaGetLastError() == cudaSuccess && cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
        cudaStreamSynchronize(st) == cudaSuccess)
      state = h == 0 ? 1 : 2;
  }
  cudaGetLastError();
  if (st) cudaStreamDestroy(st);
  if (d) cudaFree(d);
  return state;
}

}  // namespace

bool atomics_lane_ordered(cudaStream_t s) {
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_mu);
  if (g_state[dev] == 0) {
    // never allocate or synchronise while the caller's stream is being captured into a graph:
    // use the order-free paths for this call and check on the next uncaptured one
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (s && cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return false;
    cudaGetLastError();
    g_state[dev] = run_lane_order_check();
  }
  return g_state[dev] == 1;
}

}  // namespace bsort

extern "C" int bsort_selftest(void) {
  if (!bsort::atomics_lane_ordered(nullptr)) {
    int dev = 0;
    return cudaGetDevice(&dev) == cudaSuccess ? 1 : -1;
  }
  return 0;
}
