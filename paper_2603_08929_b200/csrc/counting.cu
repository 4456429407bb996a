// counting.cu — a6: the small-word counting path for 8/16-bit keys (BASELINE.json cfg2).
//
// Keys of w <= 16 bits are sorted by one histogram over all 2^w transformed values followed by
// a regeneration of the array from the bin prefix (Theorem 5's in-place property, P:761-775,
// is kept: O(2^w) auxiliary counters, no second key buffer).  Exact because equal transformed
// keys are equal bit patterns (the transform is a bijection), so the multiset of bins IS the
// multiset of keys.
//
//   k_count_hist8   256 lane-banked counters per CTA (bank = lane => conflict-free smem
//                   atomics), one read of the keys with 128-bit loads, flush to 256 global u64.
//   k_count_fill8   every CTA scans the 256 counts in smem; each thread regenerates 16-byte
//                   output vectors (binary search of the first key's bin, 128-bit stores).
//   k_count_hist16  one CTA per SM, all 65536 bins as u16 halves in 128 KB of smem (drained
//                   to a global overflow counter at 0x8000), one read of the keys; per-CTA
//                   rows of residual counts.
//   k_count_scan16  64 CTAs: bin totals over the rows + overflow, block-local exclusive scan.
//   k_count_fill16  warp-contiguous output ranges; one two-level binary search per lane, then a
//                   forward walk over the bin starts (L2-resident); 128-bit stores.
#include "paths.cuh"
#include "scan.cuh"

namespace bsort {
namespace {

constexpr int CNT_THREADS = 1024;
constexpr int FILL_THREADS = 256;
constexpr int BINS16 = 65536;

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------------------------------ 8-bit

template <uint32_t X>
__global__ void __launch_bounds__(CNT_THREADS, 2)
    k_count_hist8(const uint8_t* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ hist) {
  __shared__ uint32_t h[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += CNT_THREADS) h[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t T = (uint64_t)gridDim.x * CNT_THREADS;
  const uint64_t gt = (uint64_t)blockIdx.x * CNT_THREADS + threadIdx.x;
  const uint64_t head = min64(n, (16 - ((uintptr_t)keys & 15)) & 15);
  auto add = [&](uint32_t bin) { atomicAdd(&h[(bin << 5) | lane], 1u); };
  auto word = [&](uint32_t w) {
    w ^= X;
    add(w & 0xFF);
    add((w >> 8) & 0xFF);
    add((w >> 16) & 0xFF);
    add(w >> 24);
  };
  auto vec = [&](uint4 q) {
    word(q.x);
    word(q.y);
    word(q.z);
    word(q.w);
  };
  for (uint64_t i = gt; i < head; i += T) add((keys[i] ^ X) & 0xFF);
  const uint4* v = reinterpret_cast<const uint4*>(keys + head);
  const uint64_t nv = (n - head) >> 4;
  uint64_t i = gt;
  for (; i + 3 * T < nv; i += 4 * T) {
    uint4 q0 = ldg_stream(v + i), q1 = ldg_stream(v + i + T);
    uint4 q2 = ldg_stream(v + i + 2 * T), q3 = ldg_stream(v + i + 3 * T);
    vec(q0);
    vec(q1);
    vec(q2);
    vec(q3);
  }
  for (; i < nv; i += T) vec(ldg_stream(v + i));
  for (uint64_t j = head + (nv << 4) + gt; j < n; j += T) add((keys[j] ^ X) & 0xFF);
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += CNT_THREADS) {
    uint32_t s = 0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) s += h[(b << 5) | ((l + b) & 31)];
    if (s) atomicAdd(&hist[b], (unsigned long long)s);
  }
}

template <uint32_t X>
__global__ void __launch_bounds__(FILL_THREADS)
    k_count_fill8(uint8_t* __restrict__ keys, uint64_t n, const unsigned long long* __restrict__ hist) {
  __shared__ unsigned long long pre[257];
  __shared__ unsigned long long wt[FILL_THREADS / 32 + 1];
  unsigned long long ex = block_exclusive_scan<FILL_THREADS>(hist[threadIdx.x], wt,
                                                             (unsigned long long*)nullptr);
  pre[threadIdx.x] = ex;
  if (threadIdx.x == 0) pre[256] = n;
  __syncthreads();
  // largest b in [0, 256) with pre[b] <= p  (pre[0] = 0 <= p < n = pre[256])
  auto bin_of = [&](uint64_t p) -> uint32_t {
    uint32_t lo = 0, hi = 256;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (pre[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
  };
  const uint64_t T = (uint64_t)gridDim.x * FILL_THREADS;
  const uint64_t gt = (uint64_t)blockIdx.x * FILL_THREADS + threadIdx.x;
  const uint64_t head = min64(n, (16 - ((uintptr_t)keys & 15)) & 15);
  for (uint64_t i = gt; i < head; i += T) keys[i] = uint8_t(bin_of(i) ^ X);
  uint4* v = reinterpret_cast<uint4*>(keys + head);
  const uint64_t nv = (n - head) >> 4;
  // warp-contiguous vector ranges (coalesced stores); each lane's position only moves forward,
  // so one binary search per lane, then a forward walk over the bin starts
  const uint64_t warps = T / 32;
  const uint64_t wid = gt / 32;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t per = ((nv + warps - 1) / warps + 31) & ~uint64_t(31);
  const uint64_t v0 = min64(nv, wid * per), v1 = min64(nv, v0 + per);
  uint32_t b = 0;
  bool init = false;
  for (uint64_t i = v0 + lane; i < v1; i += 32) {
    const uint64_t p0 = head + (i << 4);
    if (!init) {
      b = bin_of(p0);
      init = true;
    }
    while (pre[b + 1] <= p0) ++b;
    uint4 q;
    if (pre[b + 1] >= p0 + 16) {
      const uint32_t w = (b * 0x01010101u) ^ X;
      q = make_uint4(w, w, w, w);
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
      uint32_t bb = b;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        while (pre[bb + 1] <= p0 + j) ++bb;
        w[j >> 2] |= bb << ((j & 3) * 8);
      }
      q = make_uint4(w[0] ^ X, w[1] ^ X, w[2] ^ X, w[3] ^ X);
    }
    v[i] = q;
  }
  for (uint64_t j = head + (nv << 4) + gt; j < n; j += T) keys[j] = uint8_t(bin_of(j) ^ X);
}

// ----------------------------------------------------------------------------- 16-bit

// Transforms of two 16-bit keys packed in a u32 (enc2: key -> order key; dec2: inverse).
// Integers: an XOR with a constant (sign flip and/or complement).  Half floats (f16, bf16):
// per half, negative ? ~h : h | 0x8000 (the paper's sign -> exponent -> mantissa order with
// negatives inverted), complemented for descending.
template <uint32_t X>
struct Xor16 {
  __device__ __forceinline__ static uint32_t enc2(uint32_t w) { return w ^ X; }
  __device__ __forceinline__ static uint32_t dec2(uint32_t e) { return e ^ X; }
};
template <bool DESC>
struct Float16 {
  static constexpr uint32_t D = DESC ? 0xFFFFFFFFu : 0u;
  __device__ __forceinline__ static uint32_t enc2(uint32_t w) {
    const uint32_t neg = ((w >> 15) & 0x00010001u) * 0xFFFFu;  // 0xFFFF in negative halves
    return (w ^ (neg | 0x80008000u)) ^ D;
  }
  __device__ __forceinline__ static uint32_t dec2(uint32_t e) {
    e ^= D;
    const uint32_t pos = (e >> 15) & 0x00010001u;  // encoded top bit set <=> non-negative key
    return e ^ (((pos ^ 0x00010001u) * 0xFFFFu) | (pos * 0x8000u));
  }
};

constexpr int SCAN16_BLOCK = 1024;
constexpr int SCAN16_BLOCKS = BINS16 / SCAN16_BLOCK;  // 64

// One CTA per SM counts its contiguous chunk into all 65536 bins held as u16 halves of 32768 u32
// words (128 KB of smem; each key is read once, every lane of a warp is busy).  A half that
// reaches 0x8000 is drained: the one thread whose atomicAdd returned 0x7FFF subtracts 0x8000
// from the half and adds 0x8000 to the bin's global overflow counter.  At most CNT_THREADS
// increments are in flight, so a half never wraps.  The CTA's residual u16 counts are written
// as a row of `partial` (no atomics).
template <typename TR>
__global__ void __launch_bounds__(CNT_THREADS, 1)
    k_count_hist16(const uint16_t* __restrict__ keys, uint64_t n, uint16_t* __restrict__ partial,
                   unsigned long long* __restrict__ ovf) {
  extern __shared__ uint32_t h16[];  // 32768 words: bin 2w in the low half, 2w+1 in the high half
  for (int i = threadIdx.x; i < BINS16 / 2; i += CNT_THREADS) h16[i] = 0;
  __syncthreads();
  auto add = [&](uint32_t k) {
    const uint32_t sh = (k & 1u) << 4;
    const uint32_t old = atomicAdd(&h16[k >> 1], 1u << sh);
    if (((old >> sh) & 0xFFFFu) == 0x7FFFu) {
      atomicAdd(&h16[k >> 1], 0u - (0x8000u << sh));
      atomicAdd(&ovf[k], 0x8000ull);
    }
  };
  auto vec = [&](uint4 q) {
    uint32_t w[4] = {TR::enc2(q.x), TR::enc2(q.y), TR::enc2(q.z), TR::enc2(q.w)};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      add(w[j] & 0xFFFF);
      add(w[j] >> 16);
    }
  };
  const uint64_t head = min64(n, ((16 - ((uintptr_t)keys & 15)) & 15) >> 1);
  const uint4* v = reinterpret_cast<const uint4*>(keys + head);
  const uint64_t nv = (n - head) >> 3;
  const uint64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const uint64_t vs = min64(nv, (uint64_t)blockIdx.x * per);
  const uint64_t ve = min64(nv, vs + per);
  if (blockIdx.x == 0)
    for (uint64_t i = threadIdx.x; i < head; i += CNT_THREADS) add(TR::enc2(keys[i]) & 0xFFFF);
  if (blockIdx.x == gridDim.x - 1)
    for (uint64_t i = head + (nv << 3) + threadIdx.x; i < n; i += CNT_THREADS) add(TR::enc2(keys[i]) & 0xFFFF);
  uint64_t i = vs + threadIdx.x;
  for (; i + 3 * CNT_THREADS < ve; i += 4 * CNT_THREADS) {
    uint4 q0 = ldg_stream(v + i), q1 = ldg_stream(v + i + CNT_THREADS);
    uint4 q2 = ldg_stream(v + i + 2 * CNT_THREADS), q3 = ldg_stream(v + i + 3 * CNT_THREADS);
    vec(q0);
    vec(q1);
    vec(q2);
    vec(q3);
  }
  for (; i < ve; i += CNT_THREADS) vec(ldg_stream(v + i));
  __syncthreads();
  uint32_t* row = reinterpret_cast<uint32_t*>(partial + (uint64_t)blockIdx.x * BINS16);  // same packing
  for (int w = threadIdx.x; w < BINS16 / 2; w += CNT_THREADS) row[w] = h16[w];
}

// Bin totals (sum of the per-CTA rows + overflow) and exclusive scan, 64 CTAs x 1024 bins:
// local[b] = prefix of b inside its 1024-bin block; tot[blk] = the block's total.
__global__ void __launch_bounds__(SCAN16_BLOCK)
    k_count_scan16(const uint16_t* __restrict__ partial, int rows, const unsigned long long* __restrict__ ovf,
                   unsigned long long* __restrict__ local, unsigned long long* __restrict__ tot) {
  __shared__ unsigned long long wt[SCAN16_BLOCK / 32 + 1];
  const uint32_t b = blockIdx.x * SCAN16_BLOCK + threadIdx.x;
  unsigned long long c = ovf[b];
#pragma unroll 8
  for (int r = 0; r < rows; ++r) c += partial[(uint64_t)r * BINS16 + b];
  unsigned long long t;
  local[b] = block_exclusive_scan<SCAN16_BLOCK>(c, wt, &t);
  if (threadIdx.x == 0) tot[blockIdx.x] = t;
}

// Regenerate the sorted keys in place.  Bin starts: pre(b) = ctot[b >> 10] + local[b] (ctot in
// smem, local L2-resident).  Warp w owns a contiguous range of 16-byte output vectors, lane l
// takes vectors l, l+32, ...: stores are coalesced and each lane's position only moves forward,
// so after one two-level binary search the lane finds its bin by walking forward.
template <typename TR>
__global__ void __launch_bounds__(FILL_THREADS)
    k_count_fill16(uint16_t* __restrict__ keys, uint64_t n, const unsigned long long* __restrict__ local,
                   const unsigned long long* __restrict__ tot) {
  __shared__ unsigned long long ctot[SCAN16_BLOCKS + 1];
  if (threadIdx.x < 32) {  // exclusive scan of the 64 block totals
    unsigned long long a = tot[threadIdx.x], b2 = tot[threadIdx.x + 32];
    const unsigned long long ia = warp_inclusive_scan(a);
    const unsigned long long sa = __shfl_sync(0xffffffffu, ia, 31);
    const unsigned long long ib = warp_inclusive_scan(b2) + sa;
    ctot[threadIdx.x] = ia - a;
    ctot[threadIdx.x + 32] = ib - b2;
    if (threadIdx.x == 31) ctot[SCAN16_BLOCKS] = ib;
  }
  __syncthreads();
  auto pre = [&](uint32_t b) -> uint64_t { return b < (uint32_t)BINS16 ? ctot[b >> 10] + local[b] : n; };
  auto bin_of = [&](uint64_t p) -> uint32_t {  // largest b with pre(b) <= p  (pre(0) = 0 <= p < n)
    uint32_t lo = 0, hi = SCAN16_BLOCKS;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (ctot[mid] <= p) lo = mid; else hi = mid;
    }
    const uint64_t base = ctot[lo];
    uint32_t blo = lo * SCAN16_BLOCK, bhi = blo + SCAN16_BLOCK;
    while (bhi - blo > 1) {
      const uint32_t mid = (blo + bhi) >> 1;
      if (base + local[mid] <= p) blo = mid; else bhi = mid;
    }
    return blo;
  };
  const uint64_t head = min64(n, ((16 - ((uintptr_t)keys & 15)) & 15) >> 1);
  const uint64_t gt = (uint64_t)blockIdx.x * FILL_THREADS + threadIdx.x;
  const uint64_t T = (uint64_t)gridDim.x * FILL_THREADS;
  for (uint64_t i = gt; i < head; i += T) keys[i] = uint16_t(TR::dec2(bin_of(i)));
  uint4* v = reinterpret_cast<uint4*>(keys + head);
  const uint64_t nv = (n - head) >> 3;
  const uint64_t warps = T / 32;
  const uint64_t wid = gt / 32;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t per = ((nv + warps - 1) / warps + 31) & ~uint64_t(31);
  const uint64_t v0 = min64(nv, wid * per), v1 = min64(nv, v0 + per);
  uint32_t b = 0;
  uint64_t nxt = 0;
  bool init = false;
  for (uint64_t i = v0 + lane; i < v1; i += 32) {
    const uint64_t p0 = head + (i << 3);
    if (!init) {
      b = bin_of(p0);
      nxt = pre(b + 1);
      init = true;
    }
    while (nxt <= p0) nxt = pre(++b + 1);
    uint4 q;
    if (nxt >= p0 + 8) {
      const uint32_t w = TR::dec2(b * 0x00010001u);
      q = make_uint4(w, w, w, w);
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
      uint32_t bb = b;
      uint64_t nn = nxt;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        while (nn <= p0 + j) nn = pre(++bb + 1);
        w[j >> 1] |= bb << ((j & 1) * 16);
      }
      q = make_uint4(TR::dec2(w[0]), TR::dec2(w[1]), TR::dec2(w[2]), TR::dec2(w[3]));
    }
    v[i] = q;
  }
  for (uint64_t j = head + (nv << 3) + gt; j < n; j += T) keys[j] = uint16_t(TR::dec2(bin_of(j)));
}

// ------------------------------------------------------------------------ host launch

int fill_grid(uint64_t vectors) {
  uint64_t want = (vectors + FILL_THREADS - 1) / FILL_THREADS;
  uint64_t cap = (uint64_t)num_sms() * 8;
  return (int)max64(1, min64(want, cap));
}

template <uint32_t X>
bsort_status_t run8(uint8_t* keys, uint64_t n, void* ws, cudaStream_t s) {
  auto* hist = reinterpret_cast<unsigned long long*>(ws);
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), s));
  const int grid = num_sms() * 2;
  BSORT_LAUNCH(PROF_COUNT_HIST, s, k_count_hist8<X><<<grid, CNT_THREADS, 0, s>>>(keys, n, hist));
  BSORT_LAUNCH(PROF_COUNT_FILL, s,
               k_count_fill8<X><<<fill_grid(n / 16 + 1), FILL_THREADS, 0, s>>>(keys, n, hist));
  return BSORT_SUCCESS;
}

struct Count16Layout {
  size_t ovf, local, tot, partial, total;
};
Count16Layout count16_layout() {
  Count16Layout l;
  size_t off = 0;
  l.ovf = off;     off = align_up(off + BINS16 * 8, 256);
  l.local = off;   off = align_up(off + BINS16 * 8, 256);
  l.tot = off;     off = align_up(off + SCAN16_BLOCKS * 8, 256);
  l.partial = off; off = align_up(off + (size_t)num_sms() * BINS16 * sizeof(uint16_t), 256);
  l.total = off;
  return l;
}

template <typename TR>
bsort_status_t run16(uint16_t* keys, uint64_t n, void* ws, cudaStream_t s) {
  const Count16Layout l = count16_layout();
  auto* w = static_cast<unsigned char*>(ws);
  auto* ovf = reinterpret_cast<unsigned long long*>(w + l.ovf);
  auto* local = reinterpret_cast<unsigned long long*>(w + l.local);
  auto* tot = reinterpret_cast<unsigned long long*>(w + l.tot);
  auto* partial = reinterpret_cast<uint16_t*>(w + l.partial);
  const int smem = (BINS16 / 2) * sizeof(uint32_t);
  static DeviceOnce attr;  // per device; idempotent, benign race
  if (attr.pending()) {
    BSORT_CUDA(cudaFuncSetAttribute(k_count_hist16<TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr.mark();
  }
  const int rows = num_sms();
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(ovf, 0, BINS16 * sizeof(unsigned long long), s));
  BSORT_LAUNCH(PROF_COUNT_HIST, s, k_count_hist16<TR><<<rows, CNT_THREADS, smem, s>>>(keys, n, partial, ovf));
  BSORT_LAUNCH(PROF_COUNT_SCAN, s,
               k_count_scan16<<<SCAN16_BLOCKS, SCAN16_BLOCK, 0, s>>>(partial, rows, ovf, local, tot));
  BSORT_LAUNCH(PROF_COUNT_FILL, s,
               k_count_fill16<TR><<<fill_grid(n / 8 + 1), FILL_THREADS, 0, s>>>(keys, n, local, tot));
  return BSORT_SUCCESS;
}

}  // namespace

size_t counting_workspace_bytes(int bytes, uint64_t n) {
  if (n <= 1) return 0;
  if (bytes == 1) return 256 * sizeof(unsigned long long);
  return count16_layout().total;
}

bsort_status_t counting_sort(const DtypeInfo& di, void* keys, uint64_t n, bool desc, void* ws,
                             size_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < counting_workspace_bytes(di.bytes, n)) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  auto* k8 = static_cast<uint8_t*>(keys);
  auto* k16 = static_cast<uint16_t*>(keys);
  if (di.bytes == 1) {
    if (di.kind == KIND_U)
      return desc ? run8<packed_xor<KIND_U, true, 1>()>(k8, n, ws, s)
                  : run8<packed_xor<KIND_U, false, 1>()>(k8, n, ws, s);
    return desc ? run8<packed_xor<KIND_I, true, 1>()>(k8, n, ws, s)
                : run8<packed_xor<KIND_I, false, 1>()>(k8, n, ws, s);
  }
  if (di.kind == KIND_U)
    return desc ? run16<Xor16<packed_xor<KIND_U, true, 2>()>>(k16, n, ws, s)
                : run16<Xor16<packed_xor<KIND_U, false, 2>()>>(k16, n, ws, s);
  if (di.kind == KIND_I)
    return desc ? run16<Xor16<packed_xor<KIND_I, true, 2>()>>(k16, n, ws, s)
                : run16<Xor16<packed_xor<KIND_I, false, 2>()>>(k16, n, ws, s);
  return desc ? run16<Float16<true>>(k16, n, ws, s) : run16<Float16<false>>(k16, n, ws, s);
}

}  // namespace bsort
