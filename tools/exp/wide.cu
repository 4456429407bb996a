// wide.cu — standalone harness for the 3-pass LSD (csrc/wide.cuh): histogram + three passes
// (11 / 11 / 10-bit digits) of 2^k cfg3-like f32 keys (or uniform u32), full check (sorted +
// multiset checksum), per-pass CUDA-event timing.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_2603_08929_b200/csrc -Itools/exp \
//        --expt-relaxed-constexpr -lineinfo -o tools/exp/wide tools/exp/wide.cu
//   tools/exp/wide [log2n=30] [reps=10] [dist=cfg3|u32]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#include "wide.cuh"

namespace bsort {
void prof_begin(int, cudaStream_t) {}
void prof_end(int, cudaStream_t) {}
void count_launch() {}
int num_sms() { return 148; }
void set_last_cuda_error(cudaError_t) {}
}  // namespace bsort
using namespace bsort;

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) {                                                                  \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));      \
      exit(1);                                                                                \
    }                                                                                         \
  } while (0)

__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_fill(uint32_t* p, uint64_t n, unsigned long long seed, int dist) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
    if (dist == 1) { p[i] = (uint32_t)b; continue; }
    if (dist == 2) { p[i] = (uint32_t)(mix64(b % 16)); continue; }  // 16 distinct
    const uint32_t cls = (uint32_t)((b >> 24) % 10000);
    float f;
    if (cls < 50) f = 0.0f;
    else if (cls < 100) f = -0.0f;
    else if (cls < 105) f = __int_as_float(0x7f800000);
    else if (cls < 110) f = __int_as_float(0xff800000);
    else if (b & 1) f = (float)((b >> 40) & 0xFFFFFF) * (1.0f / 16777216.0f) * 2e6f - 1e6f;
    else {
      const unsigned long long c = mix64(b);
      const float u1 = ((c >> 40) + 1) * (1.0f / 16777217.0f), u2 = ((c >> 16) & 0xFFFFFF) * (1.0f / 16777216.0f);
      f = sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
    }
    p[i] = __float_as_uint(f);
  }
}
// checksum of encoded keys + count of adjacent pairs out of order (encoded)
template <int KIND>
__global__ void k_check(const uint32_t* out, uint64_t n, bool raw, unsigned long long* res) {
  unsigned long long s = 0, b = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k0 = raw ? key_encode<KIND, false>(out[i]) : out[i];
    s += mix64(k0);
    if (i + 1 < n) {
      const uint32_t k1 = raw ? key_encode<KIND, false>(out[i + 1]) : out[i + 1];
      if (k0 > k1) ++b;
    }
  }
  atomicAdd(&res[0], b);
  atomicAdd(&res[1], s);
}
// digit-order check of an intermediate (encoded) array: pairs out of order by (digit at SHIFT, BITS)
__global__ void k_check_digit(const uint32_t* a, uint64_t n, int lo_bits, unsigned long long* res) {
  unsigned long long b = 0;
  const uint32_t m = lo_bits >= 32 ? 0xFFFFFFFFu : (1u << lo_bits) - 1u;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x)
    if ((a[i] & m) > (a[i + 1] & m)) ++b;
  atomicAdd(&res[0], b);
}

struct Ctx {
  uint64_t n;
  uint32_t *in, *m1, *m2, *out, *tmp, *ring, *gcount, *counter, *hist, *bases;
  cudaEvent_t e0, e1;
};

template <int SHIFT, int BITS, int MODE, int NT, int ITEMS, int MINB, int G = 4>
float pass(Ctx& C, const uint32_t* src, uint32_t* dst, const uint32_t* bases, uint32_t flags, int reps,
           const char* tag) {
  using L = WideSmem<NT, ITEMS, BITS, MODE>;
  auto kern = k_wide<KIND_F, false, SHIFT, BITS, MODE, NT, ITEMS, MINB, G>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, L::bytes));
  const uint32_t tiles = (uint32_t)((C.n + L::TILE - 1) / L::TILE);
  const uint32_t grid = std::min<uint32_t>(tiles, 148u * occ);
  float best = 1e30f, sum = 0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaMemsetAsync(C.ring, 0, (size_t)(WIDE_RING / 2) * (1 << BITS) * 4));
    CK(cudaMemsetAsync(C.gcount, 0, 4 * 2048));
    CK(cudaMemsetAsync(C.counter, 0, 4));
    CK(cudaEventRecord(C.e0));
    kern<<<grid, NT, L::bytes>>>(src, dst, (uint32_t)C.n, bases, C.ring, C.gcount, C.counter, tiles, flags);
    CK(cudaEventRecord(C.e1));
    CK(cudaEventSynchronize(C.e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, C.e0, C.e1));
    best = std::min(best, ms);
    sum += ms;
  }
  printf("%-34s smem %6zu occ %d tiles %7u  best %.3f ms  avg %.3f ms  (%.1f GB/s)\n", tag, L::bytes, occ, tiles,
         best, sum / reps, 8.0 * C.n / best / 1e6);
  return best;
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 30;
  const int reps = argc > 2 ? atoi(argv[2]) : 10;
  const char* dname = argc > 3 ? argv[3] : "cfg3";
  const int dist = !strcmp(dname, "u32") ? 1 : (!strcmp(dname, "d16") ? 2 : 0);
  const uint64_t n = (argc > 4) ? strtoull(argv[4], nullptr, 10) : (1ull << lg);
  Ctx C;
  C.n = n;
  CK(cudaMalloc(&C.in, n * 4));
  CK(cudaMalloc(&C.m1, n * 4));
  CK(cudaMalloc(&C.m2, n * 4));
  CK(cudaMalloc(&C.out, n * 4));
  CK(cudaMalloc(&C.tmp, n * 4));
  CK(cudaMalloc(&C.ring, (size_t)WIDE_RING * 2048 * 4));
  CK(cudaMemset(C.ring, 0, (size_t)WIDE_RING * 2048 * 4));
  CK(cudaMalloc(&C.gcount, 4 * 2048));
  CK(cudaMalloc(&C.counter, 64));
  CK(cudaMalloc(&C.hist, 4 * 5120));
  CK(cudaMalloc(&C.bases, 4 * 5120));
  CK(cudaEventCreate(&C.e0));
  CK(cudaEventCreate(&C.e1));
  unsigned long long* res;
  CK(cudaMalloc(&res, 16));
  k_fill<<<148 * 8, 256>>>(C.in, n, 12345, dist);
  CK(cudaDeviceSynchronize());

  // histogram
  {
    auto hk = k_wide_hist<KIND_F, false, 1024>;
    const int hb = 4 * 5120 * 4;
    CK(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, hb));
    float best = 1e30f;
    for (int r = 0; r < std::max(1, reps / 2); ++r) {
      CK(cudaMemset(C.hist, 0, 4 * 5120));
      CK(cudaEventRecord(C.e0));
      hk<<<148, 1024, hb>>>(C.in, (uint32_t)n, C.hist);
      CK(cudaEventRecord(C.e1));
      CK(cudaEventSynchronize(C.e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, C.e0, C.e1));
      best = std::min(best, ms);
    }
    printf("%-34s best %.3f ms (%.1f GB/s)\n", "hist 11/11/10 (simple)", best, 4.0 * n / best / 1e6);
  }
  std::vector<uint32_t> h(5120), b(5120);
  CK(cudaMemcpy(h.data(), C.hist, 4 * 5120, cudaMemcpyDeviceToHost));
  const int off[3] = {0, 2048, 4096}, nb[3] = {2048, 2048, 1024};
  uint32_t min_nz0 = 0xFFFFFFFFu;
  for (int p = 0; p < 3; ++p) {
    uint64_t r = 0;
    for (int d = 0; d < nb[p]; ++d) {
      b[off[p] + d] = (uint32_t)r;
      r += h[off[p] + d];
      if (p == 0 && h[d]) min_nz0 = std::min(min_nz0, h[d]);
    }
    if (r != n) { printf("hist total %d = %llu != n\n", p, (unsigned long long)r); return 1; }
  }
  printf("min nonzero digit-0 bucket %u (RUN2 needs >= tile 8192)\n", min_nz0);
  CK(cudaMemcpy(C.bases, b.data(), 4 * 5120, cudaMemcpyHostToDevice));

  // reference checksum
  CK(cudaMemset(res, 0, 16));
  k_check<KIND_F><<<148 * 8, 256>>>(C.in, n, true, res);
  unsigned long long r0[2];
  CK(cudaMemcpy(r0, res, 16, cudaMemcpyDeviceToHost));

  const bool run2 = min_nz0 >= 8192;
  float t0 = pass<0, 11, WM_UNSTABLE, 512, 16, 2>(C, C.in, C.m1, C.bases, WF_ENC, 1, "P0 unstable 11b 512x16");
  float t1 = run2 ? pass<11, 11, WM_RUN2, 512, 16, 2>(C, C.m1, C.m2, C.bases + 2048, 0, 1, "P1 run2 11b 512x16")
                  : pass<11, 11, WM_STABLE, 512, 16, 1>(C, C.m1, C.m2, C.bases + 2048, 0, 1, "P1 stable 11b 512x16");
  float t2 = pass<22, 10, WM_STABLE, 256, 32, 2>(C, C.m2, C.out, C.bases + 4096, WF_DEC, 1, "P2 stable 10b 256x32");
  (void)t0; (void)t1; (void)t2;
  CK(cudaMemset(res, 0, 16));
  k_check_digit<<<148 * 8, 256>>>(C.m1, n, 11, res);
  unsigned long long c1;
  CK(cudaMemcpy(&c1, res, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemset(res, 0, 16));
  k_check_digit<<<148 * 8, 256>>>(C.m2, n, 22, res);
  unsigned long long c2;
  CK(cudaMemcpy(&c2, res, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemset(res, 0, 16));
  k_check<KIND_F><<<148 * 8, 256>>>(C.out, n, true, res);
  unsigned long long r3[2];
  CK(cudaMemcpy(r3, res, 16, cudaMemcpyDeviceToHost));
  const bool ok = c1 == 0 && c2 == 0 && r3[0] == 0 && r3[1] == r0[1];
  printf("check: P0 out-of-order(11b) %llu  P1 out-of-order(22b) %llu  final out-of-order %llu  checksum %s  => %s\n",
         c1, c2, r3[0], r3[1] == r0[1] ? "ok" : "MISMATCH", ok ? "PASS" : "FAIL");
  if (!ok) return 2;

  // timing (each pass from its own input)
  float a = pass<0, 11, WM_UNSTABLE, 512, 16, 2>(C, C.in, C.tmp, C.bases, WF_ENC, reps, "P0 unstable 11b 512x16");
  float bb = run2 ? pass<11, 11, WM_RUN2, 512, 16, 2>(C, C.m1, C.tmp, C.bases + 2048, 0, reps, "P1 run2 11b 512x16")
                  : pass<11, 11, WM_STABLE, 512, 16, 1>(C, C.m1, C.tmp, C.bases + 2048, 0, reps, "P1 stable 11b 512x16");
  float c = pass<22, 10, WM_STABLE, 256, 32, 2>(C, C.m2, C.tmp, C.bases + 4096, WF_DEC, reps, "P2 stable 10b 256x32");
  pass<22, 10, WM_STABLE, 512, 16, 1>(C, C.m2, C.tmp, C.bases + 4096, WF_DEC, reps, "P2 stable 10b 512x16 (1 CTA)");
  pass<11, 11, WM_STABLE, 512, 16, 1>(C, C.m1, C.tmp, C.bases + 2048, 0, reps, "P1 stable 11b 512x16 (fallback)");
  printf("passes total %.3f ms (+ hist)\n", a + bb + c);
  return 0;
}
