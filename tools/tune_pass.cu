// tune_pass.cu — standalone tuning harness for the LSD scatter pass (k_onesweep_pass).
// Times one pass (digit 0 of f32-encoded keys / u64 keys) over 2^30 keys for several
// (THREADS, ITEMS, MINB, BULK) configurations, checks the output is digit-sorted and a
// permutation of the input (sum/xor of keys), and prints one line per configuration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2603_08929_b200/csrc --expt-relaxed-constexpr -o build/tune_pass tools/tune_pass.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "onesweep_ws.cuh"

namespace bsort {
// The kernels only reference these through BSORT_LAUNCH, unused here.
void prof_begin(int, cudaStream_t) {}
void prof_end(int, cudaStream_t) {}
void count_launch() {}
int num_sms() { return 148; }
void set_last_cuda_error(cudaError_t) {}
}  // namespace bsort

using namespace bsort;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
template <typename U>
__global__ void k_fill(U* p, uint64_t n, unsigned long long seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = U(mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull) >> (64 - 8 * sizeof(U)));
}
template <typename U, typename DigitF>
__global__ void k_check(const U* out, uint64_t n, DigitF digit, unsigned long long* bad,
                        unsigned long long* sum) {
  unsigned long long s = 0, b = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    s += (unsigned long long)out[i] * 0x9E3779B97F4A7C15ull + (out[i] >> 7);
    if (i + 1 < n && digit(out[i]) > digit(out[i + 1])) ++b;
  }
  atomicAdd(bad, b);
  atomicAdd(sum, s);
}
template <typename U>
__global__ void k_sum(const U* in, uint64_t n, unsigned long long* sum) {
  unsigned long long s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    s += (unsigned long long)in[i] * 0x9E3779B97F4A7C15ull + (in[i] >> 7);
  atomicAdd(sum, s);
}

template <typename U, int THREADS, int ITEMS, int MINB, bool BULK, int RANK = RANK_STABLE, int LBG = 8>
void run(const U* in, U* out, uint64_t n, const unsigned long long* bases, uint32_t* lookback, uint32_t* counter, unsigned long long* gcount,
         unsigned long long ref_sum, unsigned long long* dbg) {
  using DigitF = RadixDigit<sizeof(U) == 4 ? KIND_F : KIND_I, false, U, 0>;
  using L = PassSmem<THREADS, ITEMS, U, RANK>;
  auto kern = k_onesweep_pass<U, THREADS, ITEMS, MINB, BULK, uint32_t, DigitF, RANK, LBG>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, L::bytes));
  const uint64_t tiles = (n + L::TILE - 1) / L::TILE;
  const unsigned grid = (unsigned)min64(tiles, (uint64_t)148 * occ);
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f, tot = 0.f;
  const int reps = 6;
  for (int r = 0; r < reps; ++r) {
    CK(cudaMemset(lookback, 0, tiles * 256 * 4));
    CK(cudaMemset(counter, 0, 4));
    CK(cudaMemset(gcount, 0, 256 * 8));
    CK(cudaEventRecord(a));
    kern<<<grid, THREADS, L::bytes>>>(in, out, n, DigitF{}, bases, lookback, gcount, counter, (uint32_t)tiles, nullptr, 0, KvPtrs{});
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (r > 0) {
      tot += ms;
      best = ms < best ? ms : best;
    }
  }
  CK(cudaMemset(dbg, 0, 16));
  k_check<<<1184, 256>>>(out, n, DigitF{}, dbg, dbg + 1);
  unsigned long long h[2];
  CK(cudaMemcpy(h, dbg, 16, cudaMemcpyDeviceToHost));
  const double avg = tot / (reps - 1);
  const double gbs = 2.0 * n * sizeof(U) / (avg * 1e-3) / 1e9;
  printf("{\"lbg\": %d, \"rank\": %d, \"key_bytes\": %d, \"threads\": %d, \"items\": %d, \"minb\": %d, \"bulk\": %d, \"occ\": %d, \"regs\": %d, "
         "\"local\": %zu, \"smem\": %zu, \"avg_ms\": %.4f, \"best_ms\": %.4f, \"GBps\": %.1f, \"digit_sorted\": %d, "
         "\"perm\": %d}\n",
         LBG, RANK, (int)sizeof(U), THREADS, ITEMS, MINB, (int)BULK, occ, fa.numRegs, fa.localSizeBytes, L::bytes, avg, best, gbs,
         h[0] == 0, h[1] == ref_sum);
  fflush(stdout);
}

template <typename U, int RT, int ITEMS, int RANK, int MINB = 1>
void run_ws(const U* in, U* out, uint64_t n, const unsigned long long* bases, uint32_t* lookback, uint32_t* counter,
            unsigned long long ref_sum, unsigned long long* dbg, unsigned long long* gcount = nullptr) {
  using DigitF = RadixDigit<sizeof(U) == 4 ? KIND_F : KIND_I, false, U, 0>;
  using L = PassSmemWS<RT, ITEMS, U>;
  auto kern = k_onesweep_pass_ws<U, RT, ITEMS, uint32_t, DigitF, RANK, 8, MINB>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, RT + 256, L::bytes));
  const uint64_t tiles = (n + L::TILE - 1) / L::TILE;
  const unsigned grid = (unsigned)min64(tiles, (uint64_t)148 * occ);
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float tot = 0.f;
  const int reps = 6;
  for (int r = 0; r < reps; ++r) {
    CK(cudaMemset(lookback, 0, tiles * 256 * 4));
    CK(cudaMemset(counter, 0, 4));
    if (gcount) CK(cudaMemset(gcount, 0, 256 * 8));
    CK(cudaEventRecord(a));
    kern<<<grid, RT + 256, L::bytes>>>(in, out, n, DigitF{}, bases, lookback, counter, (uint32_t)tiles, nullptr, 0,
                                        KvPtrs{}, gcount);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (r > 0) tot += ms;
  }
  CK(cudaMemset(dbg, 0, 16));
  k_check<<<1184, 256>>>(out, n, DigitF{}, dbg, dbg + 1);
  unsigned long long h[2];
  CK(cudaMemcpy(h, dbg, 16, cudaMemcpyDeviceToHost));
  const double avg = tot / (reps - 1);
  printf("{\"ws\": 1, \"minb\": %d, \"rank\": %d, \"key_bytes\": %d, \"threads\": %d, \"items\": %d, \"occ\": %d, \"regs\": %d, "
         "\"local\": %zu, \"smem\": %zu, \"avg_ms\": %.4f, \"digit_sorted\": %d, \"perm\": %d}\n",
         MINB, RANK, (int)sizeof(U), RT, ITEMS, occ, fa.numRegs, fa.localSizeBytes, L::bytes, avg, h[0] == 0, h[1] == ref_sum);
  fflush(stdout);
}

template <typename U>
void suite(uint64_t n) {
  U *in, *out;
  unsigned long long *ghist, *bases, *dbg, *gcount;
  uint32_t *lookback, *counter, *tc;
  PassPlan* plan;
  CK(cudaMalloc(&in, n * sizeof(U)));
  CK(cudaMalloc(&out, n * sizeof(U)));
  CK(cudaMalloc(&ghist, 8 * 256 * 8));
  CK(cudaMalloc(&bases, 8 * 256 * 8));
  CK(cudaMalloc(&dbg, 16));
  CK(cudaMalloc(&gcount, 256 * 8));
  CK(cudaMalloc(&plan, sizeof(PassPlan)));
  CK(cudaMalloc(&tc, 64));
  CK(cudaMalloc(&lookback, (n / 2048 + 1) * 256 * 4));
  CK(cudaMalloc(&counter, 4));
  k_fill<<<4096, 256>>>(in, n, 12345);
  CK(cudaMemset(ghist, 0, 8 * 256 * 8));
  constexpr int P = sizeof(U);
  constexpr int LANES = sizeof(U) == 4 ? 32 : 16;
  auto hk = k_onesweep_hist<sizeof(U) == 4 ? KIND_F : KIND_I, false, U, LANES>;
  CK(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, P * 256 * LANES * 4));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  hk<<<148, HIST_THREADS, P * 256 * LANES * 4>>>(in, n, ghist, nullptr);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float hms;
  CK(cudaEventElapsedTime(&hms, a, b));
  printf("{\"hist_ms\": %.4f, \"hist_GBps\": %.1f}\n", hms, n * sizeof(U) / (hms * 1e-3) / 1e9);
  k_plan<<<1, 256>>>(ghist, n, P, bases, plan, tc, nullptr, nullptr);
  CK(cudaMemset(dbg, 0, 16));
  k_sum<<<1184, 256>>>(in, n, dbg + 1);
  unsigned long long h[2];
  CK(cudaMemcpy(h, dbg, 16, cudaMemcpyDeviceToHost));
  const unsigned long long ref = h[1];
  // One pass on uniform keys with digit shift 0: RUN2 sees a single run (the fast path).
  if constexpr (sizeof(U) == 4) {
#ifdef TUNE_WS
    run_ws<U, 512, 16, RANK_STABLE>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 16, RANK_RUN2>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 20, RANK_STABLE>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 20, RANK_RUN2>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 640, 16, RANK_STABLE>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 640, 16, RANK_RUN2>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 24, RANK_STABLE>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 24, RANK_RUN2>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 20, RANK_UNSTABLE>(in, out, n, bases, lookback, counter, ref, dbg, gcount);
    run_ws<U, 512, 16, RANK_UNSTABLE>(in, out, n, bases, lookback, counter, ref, dbg, gcount);
#endif
    run<U, 512, 16, 2, true, RANK_STABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 512, 16, 2, true, RANK_RUN2, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 512, 16, 2, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
#ifdef TUNE_UNSTABLE
    run<U, 1024, 16, 1, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 512, 24, 2, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 512, 20, 2, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 768, 16, 1, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
#endif
  } else {
    run<U, 384, 12, 2, true, RANK_STABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 384, 12, 2, true, RANK_RUN2, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 384, 12, 2, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
#ifdef TUNE_WS
    run_ws<U, 512, 12, RANK_STABLE>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 12, RANK_RUN2>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 14, RANK_STABLE>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 14, RANK_RUN2>(in, out, n, bases, lookback, counter, ref, dbg);
    run_ws<U, 512, 14, RANK_UNSTABLE>(in, out, n, bases, lookback, counter, ref, dbg, gcount);
#endif
#ifdef TUNE_U64_SWEEP
    run<U, 256, 16, 2, true, RANK_STABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 256, 16, 2, true, RANK_RUN2, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 256, 16, 2, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 512, 8, 2, true, RANK_STABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 512, 8, 2, true, RANK_RUN2, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 512, 8, 2, true, RANK_UNSTABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 256, 12, 3, true, RANK_STABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 256, 12, 3, true, RANK_RUN2, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 384, 16, 1, true, RANK_STABLE, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
    run<U, 384, 16, 1, true, RANK_RUN2, 8>(in, out, n, bases, lookback, counter, gcount, ref, dbg);
#endif
  }
  cudaFree(in);
  cudaFree(out);
  cudaFree(lookback);
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], nullptr, 0) : (1ull << 30);
  const int which = argc > 2 ? atoi(argv[2]) : 0;
  if (which == 0 || which == 4) suite<uint32_t>(n);
  if (which == 0 || which == 8) suite<unsigned long long>(n / 2);
  return 0;
}
