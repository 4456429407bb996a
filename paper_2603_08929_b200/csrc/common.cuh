// common.cuh — shared device/host helpers of the bsort CUDA path (sm_100a).
//
// Nothing here is shared with oracle/ (the CPU checker); this is the product side only.
#pragma once
#include <functional>

#include <cuda_runtime.h>
#include <stdint.h>

#include "bsort.h"

namespace bsort {

enum Kind : int { KIND_U = 0, KIND_I = 1, KIND_F = 2 };

template <int BYTES> struct Bits;
template <> struct Bits<1> { using U = uint8_t;  using S = int8_t; };
template <> struct Bits<2> { using U = uint16_t; using S = int16_t; };
template <> struct Bits<4> { using U = uint32_t; using S = int32_t; };
template <> struct Bits<8> { using U = unsigned long long; using S = long long; };

// ---------------------------------------------------------------------------------------
// a1: order-preserving key transform.  Encoded keys compare as unsigned integers in the
// paper's order (DESIGN.md §"Key transform"):
//   unsigned: identity                        (Algorithm 2 sorts raw bits)
//   signed:   flip the sign bit               (Algorithm 3's sign pass with not-asc)
//   float:    negative ? ~x : x | SIGN        (sign pass with not-asc + negatives in the inverse
//                                              direction for exponent and mantissa)
//   descending: complement of the ascending key (Algorithm 1's `asc` flag)
// The transform is a bijection on w-bit patterns, so the sorted bit sequence is unique.
template <int KIND, bool DESC, typename U>
__host__ __device__ __forceinline__ U key_encode(U x) {
  constexpr int W = int(sizeof(U) * 8);
  constexpr U SIGN = U(U(1) << (W - 1));
  U k;
  if constexpr (KIND == KIND_U) {
    k = x;
  } else if constexpr (KIND == KIND_I) {
    k = U(x ^ SIGN);
  } else {
    using S = typename Bits<sizeof(U)>::S;
    U m = U(U(S(x) >> (W - 1)) | SIGN);  // all-ones for negatives, SIGN otherwise
    k = U(x ^ m);
  }
  if constexpr (DESC) k = U(~k);
  return k;
}

template <int KIND, bool DESC, typename U>
__host__ __device__ __forceinline__ U key_decode(U k) {
  constexpr int W = int(sizeof(U) * 8);
  constexpr U SIGN = U(U(1) << (W - 1));
  if constexpr (DESC) k = U(~k);
  if constexpr (KIND == KIND_U) {
    return k;
  } else if constexpr (KIND == KIND_I) {
    return U(k ^ SIGN);
  } else {
    // (k & SIGN) ? k ^ SIGN : ~k, branch-free: t is all-ones when the sign bit is set
    using S = typename Bits<sizeof(U)>::S;
    const U t = U(S(k) >> (W - 1));
    return U(k ^ (U(~t) | SIGN));
  }
}

// Byte-parallel form for 8/16-bit keys packed in a 32-bit word: the transform of u8/i8/u16/i16
// is an XOR with a constant (no float kinds at these widths), so 4 (or 2) keys are encoded by
// one LOP.  Returns the XOR constant replicated over the word.
template <int KIND, bool DESC, int BYTES>
__host__ __device__ constexpr uint32_t packed_xor() {
  static_assert(KIND != KIND_F, "half floats use Float16 in counting.cu, not an XOR constant");
  uint32_t lane = (KIND == KIND_I) ? (1u << (BYTES * 8 - 1)) : 0u;
  if (DESC) lane ^= (BYTES == 1) ? 0xFFu : 0xFFFFu;
  return BYTES == 1 ? lane * 0x01010101u : lane * 0x00010001u;
}

// ---------------------------------------------------------------------------------------
// Host-side bookkeeping shared by the translation units (defined in api.cu).
enum ProfKind : int {
  PROF_MEMSET = 0,
  PROF_HIST = 1,
  PROF_SCAN = 2,
  PROF_PASS = 3,
  PROF_COPY = 4,
  PROF_COUNT_HIST = 5,
  PROF_COUNT_SCAN = 6,
  PROF_COUNT_FILL = 7,
  PROF_DIST_HIST = 8,
  PROF_DIST_PART = 9,
  PROF_H2D = 10,
  PROF_D2H = 11,
  PROF_DIST_A2A = 12,  // bsort_sort_dist's grouped NCCL send/recv (not a libbsort kernel)
};
static_assert(BSORT_PROF_KINDS == 13, "keep ProfKind in sync with the header");

void prof_begin(int kind, cudaStream_t s);
int current_device();  // cudaGetDevice, clamped to [0, 64)

// Per-device state of the one-time launch set-up (cudaFuncSetAttribute and the occupancy query
// act on the CURRENT device only, so a cache keyed by nothing would skip a second GPU).
struct DeviceOnce {
  bool done[64] = {};
  bool pending() const { return !done[current_device()]; }
  void mark() { done[current_device()] = true; }
};
struct DeviceInt {
  int v[64] = {};
  int& get() { return v[current_device()]; }
};
void prof_end(int kind, cudaStream_t s);
void count_launch();
int num_sms();
// graphs.cu: replay of a sort's launch sequence as a cached CUDA graph.  The key holds every
// argument the launch sequence depends on (all 64-bit: no padding, compared with memcmp).
struct GraphKey {
  uint64_t dtype, desc, device, n;
  uint64_t keys, vals, ws, wsb;
};
bsort_status_t run_graphed(const GraphKey& key, cudaStream_t s,
                           const std::function<bsort_status_t(cudaStream_t)>& run);
bool profiling_on();
uint64_t launch_count_now();
void add_launches(int64_t k);
// selftest.cu: shared atomicAdd hands out old values in lane order on this device (checked
// once per device on first use; false while `s` is being captured before the check has run)
bool atomics_lane_ordered(cudaStream_t s);
void set_last_cuda_error(cudaError_t e);

// Launch helper: profile-bracket, launch, count (kernels only, not memsets), check.
#define BSORT_LAUNCH(kind, stream, ...)                                   \
  do {                                                                    \
    ::bsort::prof_begin((kind), (stream));                                \
    __VA_ARGS__;                                                          \
    if ((kind) != ::bsort::PROF_MEMSET) ::bsort::count_launch();          \
    cudaError_t _e = cudaGetLastError();                                  \
    ::bsort::prof_end((kind), (stream));                                  \
    if (_e != cudaSuccess) {                                              \
      ::bsort::set_last_cuda_error(_e);                                   \
      return BSORT_ERROR_CUDA;                                            \
    }                                                                     \
  } while (0)

#define BSORT_CUDA(call)                                                  \
  do {                                                                    \
    cudaError_t _e = (call);                                              \
    if (_e != cudaSuccess) {                                              \
      ::bsort::set_last_cuda_error(_e);                                   \
      return BSORT_ERROR_CUDA;                                            \
    }                                                                     \
  } while (0)

__host__ __device__ constexpr uint64_t min64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ constexpr uint64_t max64(uint64_t a, uint64_t b) { return a > b ? a : b; }
__host__ __device__ constexpr uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Device-side helpers ------------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

}  // namespace bsort
