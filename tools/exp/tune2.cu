// tune2.cu — standalone harness for k_pass2 (csrc/pass2.cuh): one LSD pass over 2^k keys per
// configuration, exact check against a host stable counting pass at small n, digit-order +
// checksum check at full n, CUDA-event timing.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_2603_08929_b200/csrc \
//        --expt-relaxed-constexpr -lineinfo -o tools/exp/tune2 tools/exp/tune2.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#include "pass3.cuh"

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
// cfg3-like f32 mix (bits): 1% +-0, 0.1% +-inf, else half U[-1e6,1e6], half N(0,1)
__global__ void k_fill_cfg3(uint32_t* p, uint64_t n, unsigned long long seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
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
// joint histogram of (digit at SP >> 3, digit at SQ) of keys (encoded if ENC)
template <bool ENC>
__global__ void k_joint(const uint32_t* p, uint64_t n, int sp, int sq, unsigned long long* h) {
  __shared__ uint32_t s[32 * 256];
  for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) s[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t k = p[i];
    if (ENC) k = key_encode<KIND_F, false>(k);
    const uint32_t g = ((k >> sp) & 0xFF) >> 3, d = (k >> sq) & 0xFF;
    atomicAdd(&s[g * 256 + d], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x)
    if (s[i]) atomicAdd(&h[i], (unsigned long long)s[i]);
}
// enc: the array holds raw keys (encode to get digits); checksum over ENCODED keys
// full joint histogram of (digit 1, digit 0) of (encoded) keys: h[d1 * 256 + d0]
__global__ void k_joint16(const uint32_t* p, uint64_t n, unsigned long long* h) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[p[i] & 0xFFFFu], 1ull);
}
__global__ void k_check(const uint32_t* out, uint64_t n, int sq, bool enc, unsigned long long* res) {
  unsigned long long s = 0, b = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k0 = enc ? key_encode<KIND_F, false>(out[i]) : out[i];
    s += mix64(k0);
    if (i + 1 < n) {
      const uint32_t k1 = enc ? key_encode<KIND_F, false>(out[i + 1]) : out[i + 1];
      if (((k0 >> sq) & 0xFF) > ((k1 >> sq) & 0xFF)) ++b;
    }
  }
  atomicAdd(&res[0], b);
  atomicAdd(&res[1], s);
}

struct Bufs {
  uint32_t *in, *mid, *out, *lb, *counter;
  unsigned long long *bases, *gcount, *res, *jc;
  uint32_t* disp;
  unsigned long long* cstart;
  uint32_t *ctile, *jp;
  uint64_t n;
};

// host plan of a chunked pass from the joint histogram
struct HostPlan {
  std::vector<unsigned long long> bases, cstart;
  std::vector<uint32_t> ctile, jp, disp;
  uint32_t tiles;
};
int g_merge = 1;  // chunks = 32 / g_merge (coarser chains)
bool g_rr = false;  // dispatch by chunk_rr (no table)
HostPlan make_plan(const std::vector<unsigned long long>& jc_in, uint64_t tile) {
  std::vector<unsigned long long> jc(32 * 256, 0);
  for (int g = 0; g < 32; ++g)
    for (int d = 0; d < 256; ++d) jc[(g / g_merge) * 256 + d] += jc_in[g * 256 + d];
  HostPlan P;
  P.bases.assign(256, 0);
  std::vector<unsigned long long> marg(256, 0), grp(32, 0);
  for (int g = 0; g < 32; ++g)
    for (int d = 0; d < 256; ++d) { marg[d] += jc[g * 256 + d]; grp[g] += jc[g * 256 + d]; }
  unsigned long long r = 0;
  for (int d = 0; d < 256; ++d) { P.bases[d] = r; r += marg[d]; }
  P.cstart.assign(33, 0);
  for (int g = 0; g < 32; ++g) P.cstart[g + 1] = P.cstart[g] + grp[g];
  P.jp.assign(32 * 256, 0);
  std::vector<unsigned long long> acc(P.bases);
  for (int g = 0; g < 32; ++g)
    for (int d = 0; d < 256; ++d) { P.jp[g * 256 + d] = (uint32_t)acc[d]; acc[d] += jc[g * 256 + d]; }
  std::vector<uint32_t> nt(32);
  P.ctile.assign(33, 0);
  uint32_t maxk = 0;
  for (int g = 0; g < 32; ++g) {
    nt[g] = (uint32_t)((grp[g] + tile - 1) / tile);
    P.ctile[g + 1] = P.ctile[g] + nt[g];
    maxk = std::max(maxk, nt[g]);
  }
  P.tiles = P.ctile[32];
  for (uint32_t k = 0; k < maxk; ++k)
    for (int g = 0; g < 32; ++g)
      if (k < nt[g]) P.disp.push_back(((uint32_t)g << 24) | k);
  return P;
}

template <int SHIFT, int RT, int WT, int ITEMS, int MODE, bool CHUNKED, int LBV, int V3 = 0, int HALVES = 1, int P2MB = 1>
void run(const char* tag, Bufs& B, bool exact_check, const uint32_t* in, uint32_t flags) {
  // V3 > 0: k_pass3 with RT threads, V3 CTAs per SM (WT unused)
  using L2 = Pass2Smem<RT, (WT > 0 ? WT : 256), ITEMS, uint32_t, MODE, HALVES>;
  using L3 = Pass3Smem<RT, ITEMS, uint32_t, MODE>;
  constexpr int LTILE = V3 ? L3::TILE : L2::TILE;
  constexpr size_t LBYTES = V3 ? L3::bytes : L2::bytes;
  using KT = void (*)(const uint32_t*, uint32_t*, uint64_t, const unsigned long long*, uint32_t*, unsigned long long*,
                     uint32_t*, uint32_t, const PassPlan*, int, uint32_t, ChunkMap);
  KT kern;
  if constexpr (V3 > 0)
    kern = k_pass3<uint32_t, KIND_F, false, SHIFT, RT, ITEMS, MODE, CHUNKED, LBV, (V3 > 0 ? V3 : 1)>;
  else
    kern = k_pass2<uint32_t, KIND_F, false, SHIFT, RT, WT, ITEMS, MODE, CHUNKED, LBV, HALVES, P2MB>;
  const int nthreads = V3 ? RT : RT + WT;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LBYTES));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  const uint64_t n = B.n;
  const bool enc_in = flags & P2_ENC;
  // joint histogram (g of digit SHIFT-8, digit SHIFT), bases, chunk plan
  CK(cudaMemset(B.jc, 0, 32 * 256 * 8));
  if (enc_in) k_joint<true><<<296, 512>>>(in, n, SHIFT >= 8 ? SHIFT - 8 : 0, SHIFT, B.jc);
  else k_joint<false><<<296, 512>>>(in, n, SHIFT >= 8 ? SHIFT - 8 : 0, SHIFT, B.jc);
  std::vector<unsigned long long> jc(32 * 256);
  CK(cudaMemcpy(jc.data(), B.jc, jc.size() * 8, cudaMemcpyDeviceToHost));
  HostPlan P = make_plan(jc, LTILE);
  CK(cudaMemcpy(B.bases, P.bases.data(), 256 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B.cstart, P.cstart.data(), 33 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B.ctile, P.ctile.data(), 33 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B.jp, P.jp.data(), 32 * 256 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B.disp, P.disp.data(), P.disp.size() * 4, cudaMemcpyHostToDevice));
  ChunkMap cm{g_rr ? nullptr : B.disp, B.cstart, B.ctile, B.jp, (uint32_t)(32 / g_merge)};
  const uint32_t tiles = CHUNKED ? P.tiles : (uint32_t)((n + LTILE - 1) / LTILE);
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, 148 * (V3 ? V3 : P2MB));
  CK(cudaMemset(B.res, 0, 16));
  k_check<<<296, 512>>>(in, n, SHIFT, enc_in, B.res);
  unsigned long long ref[2];
  CK(cudaMemcpy(ref, B.res, 16, cudaMemcpyDeviceToHost));
  const size_t lb_bytes = ((tiles + 3) / 4) * 4 * 256 * 4;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f, tot = 0.f;
  const int reps = 5;
  std::vector<unsigned long long> seg;
  if (MODE == R2_J01) {  // segment starts of (d1, d0): bases[d1] + sum_{d0' < d0} J[d1][d0']
    CK(cudaMemset(B.gcount, 0, 65536 * 8));
    k_joint16<<<1184, 256>>>(in, n, B.gcount);
    std::vector<unsigned long long> J(65536);
    CK(cudaMemcpy(J.data(), B.gcount, 65536 * 8, cudaMemcpyDeviceToHost));
    seg.assign(65536, 0);
    for (int a = 0; a < 256; ++a) {
      unsigned long long r = P.bases[a];
      for (int b = 0; b < 256; ++b) { seg[b * 256 + a] = r; r += J[a * 256 + b]; }
    }
  }
  for (int r = 0; r < reps; ++r) {
    CK(cudaMemset(B.lb, 0, lb_bytes));
    CK(cudaMemset(B.counter, 0, 4));
    CK(cudaMemset(B.gcount, 0, 256 * 8));
    if (MODE == R2_J01) CK(cudaMemcpy(B.gcount, seg.data(), 65536 * 8, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(e0));
    kern<<<grid, nthreads, LBYTES>>>(in, B.out, n, B.bases, B.lb, B.gcount, B.counter, tiles, nullptr, 0, flags, cm);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
    if (r > 0) tot += ms;
  }
  // output: decoded if P2_DEC, else encoded; check digit order + multiset (of the same
  // representation as the input)
  const bool out_enc = !(flags & P2_DEC) && (enc_in || true);
  (void)out_enc;
  bool ok = true;
  {
    unsigned long long res[2];
    CK(cudaMemset(B.res, 0, 16));
    k_check<<<296, 512>>>(B.out, n, SHIFT, (flags & P2_DEC) != 0, B.res);
    CK(cudaMemcpy(res, B.res, 16, cudaMemcpyDeviceToHost));
    ok = res[0] == 0 && res[1] == ref[1];
  }
  long long mism = -1;
  {
    std::vector<uint32_t> hin, hout;
    if (exact_check) {
      hin.resize(n);
      hout.resize(n);
      CK(cudaMemcpy(hin.data(), in, n * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(hout.data(), B.out, n * 4, cudaMemcpyDeviceToHost));
      std::vector<uint32_t> exp(n);
      std::vector<unsigned long long> pos(P.bases);
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t k = enc_in ? key_encode<KIND_F, false>(hin[i]) : hin[i];
        const uint32_t d = (k >> SHIFT) & 0xFF;
        exp[pos[d]++] = (flags & P2_DEC) ? key_decode<KIND_F, false>(k) : k;
      }
      mism = 0;
      for (uint64_t i = 0; i < n; ++i) mism += exp[i] != hout[i];
      if (MODE == R2_STABLE) ok = ok && mism == 0;
      else {  // unstable: same digit order, same multiset
        std::vector<uint32_t> a(exp), b2(hout);
        bool dig = true;
        for (uint64_t i = 0; i < n; ++i) {
          const uint32_t ka = (flags & P2_DEC) ? key_encode<KIND_F, false>(a[i]) : a[i];
          const uint32_t kb = (flags & P2_DEC) ? key_encode<KIND_F, false>(b2[i]) : b2[i];
          dig &= ((ka >> SHIFT) & 0xFF) == ((kb >> SHIFT) & 0xFF);
        }
        std::sort(a.begin(), a.end());
        std::sort(b2.begin(), b2.end());
        ok = ok && dig && a == b2;
      }
    }
  }
  const double avg = tot / (reps - 1);
  printf("{\"tag\":\"%s\",\"n\":%llu,\"shift\":%d,\"mode\":%d,\"chunked\":%d,\"RT\":%d,\"WT\":%d,\"items\":%d,\"lbv\":%d,"
         "\"regs\":%d,\"smem\":%zu,\"v3\":%d,\"tiles\":%u,\"best_ms\":%.4f,\"avg_ms\":%.4f,\"GBps\":%.0f,\"ok\":%d,\"mismatch\":%lld}\n",
         tag, (unsigned long long)n, SHIFT, MODE, CHUNKED ? 1 : 0, RT, WT, ITEMS, LBV, fa.numRegs, LBYTES, V3, tiles, best,
         avg, 2.0 * 4 * n / (avg * 1e-3) / 1e9, ok ? 1 : 0, mism);
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int logn = argc > 1 ? atoi(argv[1]) : 30;
  Bufs B;
  B.n = 1ull << logn;
  CK(cudaMalloc(&B.in, B.n * 4));
  CK(cudaMalloc(&B.mid, B.n * 4));
  CK(cudaMalloc(&B.out, B.n * 4));
  CK(cudaMalloc(&B.lb, ((B.n / 4096) + 64) * 4 * 256 * 4));
  CK(cudaMalloc(&B.counter, 64));
  CK(cudaMalloc(&B.bases, 256 * 8));
  CK(cudaMalloc(&B.gcount, 65536 * 8));
  CK(cudaMalloc(&B.res, 16));
  CK(cudaMalloc(&B.jc, 32 * 256 * 8));
  CK(cudaMalloc(&B.disp, ((B.n / 4096) + 64) * 4));
  CK(cudaMalloc(&B.cstart, 33 * 8));
  CK(cudaMalloc(&B.ctile, 33 * 4));
  CK(cudaMalloc(&B.jp, 32 * 256 * 4));
  k_fill_cfg3<<<1184, 256>>>(B.in, B.n, 42);
  CK(cudaDeviceSynchronize());
  const bool exact = logn <= 24;
  // realistic inputs of passes 2 and 3: encoded keys sorted by the low 16 / 24 bits
  uint32_t* m2;
  uint32_t* m3;
  CK(cudaMalloc(&m2, B.n * 4));
  CK(cudaMalloc(&m3, B.n * 4));
  run<0, 512, 256, 20, R2_UNSTABLE, false, 2>("unstable_d0_enc", B, exact, B.in, P2_ENC);
  CK(cudaMemcpy(B.mid, B.out, B.n * 4, cudaMemcpyDeviceToDevice));
  run<8, 512, 256, 18, R2_J01, false, 2>("j01_512_18", B, exact, B.mid, 0);
  CK(cudaMemcpy(m2, B.out, B.n * 4, cudaMemcpyDeviceToDevice));
  run<16, 640, 256, 16, R2_STABLE, false, 2>("p2_stable_640_16", B, exact, m2, 0);
  CK(cudaMemcpy(m3, B.out, B.n * 4, cudaMemcpyDeviceToDevice));
  g_merge = 8;
  g_rr = true;
  run<16, 512, 256, 20, R2_STABLE, true, 2>("p2_chunked4_512x20", B, exact, m2, 0);
  run<16, 256, 256, 20, R2_STABLE, true, 2, 0, 1, 2>("p2_ch4_256x20_2cta", B, exact, m2, 0);
  run<16, 256, 256, 16, R2_STABLE, true, 2, 0, 1, 2>("p2_ch4_256x16_2cta", B, exact, m2, 0);
  run<16, 384, 256, 12, R2_STABLE, true, 2, 0, 1, 2>("p2_ch4_384x12_2cta", B, exact, m2, 0);
  run<24, 640, 256, 15, R2_STABLE, true, 2, 0, 2>("p3_chunked4_halves", B, exact, m3, P2_DEC);
  run<24, 256, 256, 21, R2_STABLE, true, 2, 0, 2, 2>("p3_ch4_256x21_h2_2cta", B, exact, m3, P2_DEC);
  g_merge = 1;
  g_rr = false;
  return 0;
}
