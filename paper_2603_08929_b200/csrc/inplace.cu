// inplace.cu — SURVEY §8 N4: the paper-faithful in-place mode and hybrid (DESIGN.md §"In-place").
//
// The paper's Algorithm 1 partitions a range in place by one bit and Algorithm 2
// recurses on the two halves from the most significant bit down; Theorem 5 bounds
// the extra space by the recursion depth.  Here the same MSD recursion is taken 8
// bits at a time (a 256-way in-place partition generalising Alg. 1's 2-way one), and the
// recursion stops as soon as a group of consecutive buckets fits a caller-chosen chunk of
// `chunk` keys, which the one-sweep LSD path then sorts with `chunk` keys of scratch (the
// paper's §V hybrid).  Extra memory: O(n/B) slot flags + O(SMs * 256 * B) overflow + the LSD
// scratch of one chunk, instead of the n-key ping-pong buffer of bsort_sort.
//
// 256-way in-place partition of a[0, n) by the digit (enc(x) >> shift) & 255, in slots of
// B = 512 bytes (B keys) counted from a[0]:
//   P1 k_ip_classify  stripe per CTA: keys are read tile by tile and appended to 256 per-bucket
//                     shared-memory buffers of B keys; every full buffer is written back as a
//                     whole slot ("block") at the stripe's write pointer, which never passes
//                     the read pointer.  Per stripe: blocks at its front, < B leftover keys per
//                     bucket saved to an overflow area, per-bucket key/block counts.
//   host              bucket starts S_b (exclusive prefix of the counts); bucket b's f_b blocks
//                     go to the aligned slots D_b = ceil(S_b/B) .. D_b+f_b-1 (disjoint over b).
//   P2 k_ip_permute   warp workers move every block once: claim an unprocessed slot (CAS on its
//                     flag), read it, claim the next destination slot of its bucket (atomicAdd),
//                     and if that slot still holds an unread block, read it before writing and
//                     carry it on (cycle following); a destination being read by another warp
//                     is written after its reader marks it free.
//   P3 k_ip_collect / k_ip_fill   the keys of bucket b's last block that lie past S_{b+1} are set
//                     aside, then b's gaps ([S_b, D_b*B) and after its last block) are filled
//                     with its overflow keys and those set-aside keys.
// Order inside a bucket is unspecified (every bucket is sorted afterwards).
#include <algorithm>
#include <vector>

#include "onesweep.cuh"
#include "paths.cuh"
#include "scan.cuh"

namespace bsort {
namespace {

constexpr int IP_THREADS = 1024;
constexpr int IP_ITEMS = 8;
constexpr int IP_TILE = IP_THREADS * IP_ITEMS;
constexpr int IP_BLOCK_BYTES = 512;
constexpr uint32_t F_EMPTY = 0, F_UNPROC = 1, F_READING = 2, F_FREE = 3;

template <typename U> constexpr int ip_block() { return IP_BLOCK_BYTES / (int)sizeof(U); }

template <int KIND, bool DESC, typename U>
struct ShiftDigit {
  int shift;
  __device__ __forceinline__ uint32_t operator()(U x) const {
    return uint32_t(key_encode<KIND, DESC>(x) >> shift) & 0xFFu;
  }
};

// P1.  grid = number of stripes; dynamic smem = 256 * B keys of bucket buffers + one tile.
// Per tile: rank by shared atomics, restage the tile bucket-sorted, then every block that a
// bucket completes (its buffered keys + the first of its new keys) is copied out by one warp as
// 512 contiguous bytes; the rest of the bucket's new keys refill its buffer.
template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(IP_THREADS, 1)
    k_ip_classify(U* __restrict__ a, uint64_t n, int shift, uint64_t stripe_len, U* __restrict__ ovf,
                  uint32_t* __restrict__ ovc, uint32_t* __restrict__ flags, unsigned long long* __restrict__ count,
                  unsigned long long* __restrict__ fblocks) {
  constexpr int B = ip_block<U>();
  constexpr int NW = IP_THREADS / 32;
  extern __shared__ __align__(16) unsigned char ip_smem[];
  U* sbuf = reinterpret_cast<U*>(ip_smem);  // [256][B]
  U* ts = sbuf + 256 * B;                    // [IP_TILE] the tile, bucket-sorted
  __shared__ uint32_t cbuf[256], cnt[256], nbk[256], boff[256], toff[256], nbsum[256], tcount[256];
  constexpr int MAXBLK = (IP_TILE + 256 * (B - 1)) / B;  // blocks one tile can complete
  __shared__ uint8_t blkmap[MAXBLK];                      // completed block -> its bucket
  __shared__ uint32_t wt[NW + 1];
  __shared__ uint32_t tot_blocks;
  const ShiftDigit<KIND, DESC, U> dg{shift};
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint64_t s = blockIdx.x;
  const uint64_t lo = s * stripe_len;
  const uint64_t hi = min64(n, lo + stripe_len);
  if (t < 256) {
    cbuf[t] = 0;
    nbsum[t] = 0;
    tcount[t] = 0;
  }
  uint64_t wp = lo;
  // register double buffer: tile tb+IP_TILE is loaded while tile tb is processed (this
  // iteration's writes end at or before tb+IP_TILE, the next one's are ordered after these
  // loads by the barriers that follow their use in ranking)
  U nxt[IP_ITEMS];
  auto load = [&](uint64_t tb) {
#pragma unroll
    for (int k = 0; k < IP_ITEMS; ++k) {
      const uint64_t i = tb + warp * (32 * IP_ITEMS) + k * 32 + lane;
      nxt[k] = i < hi ? a[i] : U(0);
    }
  };
  if (lo < hi) load(lo);
  for (uint64_t tb = lo; tb < hi; tb += IP_TILE) {
    U keys[IP_ITEMS];
    uint32_t info[IP_ITEMS];
#pragma unroll
    for (int k = 0; k < IP_ITEMS; ++k) keys[k] = nxt[k];
    if (tb + IP_TILE < hi) load(tb + IP_TILE);
    if (t < 256) cnt[t] = 0;
    __syncthreads();  // tile loaded by everyone (this iteration's writes may land on it); cnt zeroed
#pragma unroll
    for (int k = 0; k < IP_ITEMS; ++k) {
      const uint64_t i = tb + warp * (32 * IP_ITEMS) + k * 32 + lane;
      if (i < hi) {
        const uint32_t d = dg(keys[k]);
        info[k] = d | (atomicAdd(&cnt[d], 1u) << 8);
      } else {
        info[k] = 0xFFFFFFFFu;
      }
    }
    __syncthreads();
    // one scan of {blocks completed : 16 | tile count : 16} per bucket
    uint32_t packed = 0;
    if (t < 256) {
      const uint32_t nb = (cbuf[t] + cnt[t]) / (uint32_t)B;
      nbk[t] = nb;
      nbsum[t] += nb;
      tcount[t] += cnt[t];
      packed = (nb << 16) | cnt[t];
    }
    uint32_t total = 0;
    const uint32_t ex = block_exclusive_scan<IP_THREADS>(packed, wt, &total);
    if (t < 256) {
      boff[t] = ex >> 16;
      toff[t] = ex & 0xFFFFu;
    }
    if (t == 0) tot_blocks = total >> 16;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < IP_ITEMS; ++k)
      if (info[k] != 0xFFFFFFFFu) ts[toff[info[k] & 0xFFu] + (info[k] >> 8)] = keys[k];
    if (t < 256)
      for (uint32_t j = 0; j < nbk[t]; ++j) blkmap[boff[t] + j] = (uint8_t)t;
    __syncthreads();
    // completed blocks, one warp per block: 512 contiguous bytes at wp + g*B
    const uint32_t nblk = tot_blocks;
    for (uint32_t g = warp; g < nblk; g += NW) {
      const uint32_t d = blkmap[g], j = g - boff[d], c = cbuf[d];
#pragma unroll
      for (int e = 0; e < B / 32; ++e) {
        const uint32_t v = j * B + e * 32 + lane;
        a[wp + (uint64_t)g * B + e * 32 + lane] = v < c ? sbuf[d * B + v] : ts[toff[d] + (v - c)];
      }
    }
    __syncthreads();
    // the rest of each bucket's new keys go to its buffer
#pragma unroll
    for (int k = 0; k < IP_ITEMS; ++k) {
      if (info[k] != 0xFFFFFFFFu) {
        const uint32_t d = info[k] & 0xFFu;
        const uint32_t v = cbuf[d] + (info[k] >> 8);
        const uint32_t full = nbk[d] * (uint32_t)B;
        if (v >= full) sbuf[d * B + (v - full)] = keys[k];
      }
    }
    __syncthreads();
    if (t < 256) cbuf[t] = cbuf[t] + cnt[t] - nbk[t] * (uint32_t)B;
    wp += (uint64_t)nblk * B;
  }
  __syncthreads();
  if (t < 256) {
    ovc[s * 256 + t] = cbuf[t];
    if (tcount[t]) atomicAdd(&count[t], (unsigned long long)tcount[t]);
    if (nbsum[t]) atomicAdd(&fblocks[t], (unsigned long long)nbsum[t]);
  }
  for (uint32_t b = warp; b < 256; b += NW)
    for (uint32_t v = lane; v < cbuf[b]; v += 32) ovf[(s * 256 + b) * B + v] = sbuf[b * B + v];
  if (lo < n) {
    const uint64_t j0 = lo / B, jw = wp / B, j1 = (hi + B - 1) / B;
    for (uint64_t j = j0 + t; j < j1; j += IP_THREADS) flags[j] = j < jw ? F_UNPROC : F_EMPTY;
  }
}

// Slot j covers a[j*B, j*B+B); positions >= n (only in the last, partial slot) live in tail[].
template <typename U, int B>
__device__ __forceinline__ void slot_read(const U* a, const U* tail, uint64_t n, uint64_t j, U (&v)[B / 32]) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < B / 32; ++k) {
    const uint64_t p = j * B + k * 32 + lane;
    v[k] = p < n ? __ldcg(a + p) : __ldcg(tail + (p - n));
  }
}
template <typename U, int B>
__device__ __forceinline__ void slot_write(U* a, U* tail, uint64_t n, uint64_t j, const U (&v)[B / 32]) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < B / 32; ++k) {
    const uint64_t p = j * B + k * 32 + lane;
    if (p < n)
      __stcg(a + p, v[k]);
    else
      __stcg(tail + (p - n), v[k]);
  }
}

// P2.  One warp = one worker; slots are handed out 32 at a time.  Flag protocol: UNPROC (a
// block not read yet) -> READING (claimed by the warp that will read it); a warp that read a
// SOURCE slot marks it FREE, because the warp that later claims that slot as a destination must
// not overwrite it before the read completed.  A destination slot that its claimer read itself
// needs no mark (nobody else targets it).  The read of a destination is issued together with the
// CAS that claims it: an UNPROC slot is never written, so the data is valid whenever the CAS wins.
template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(256)
    k_ip_permute(U* __restrict__ a, uint64_t n, int shift, uint32_t* flags, uint64_t nslots,
                 const unsigned long long* __restrict__ dstart, unsigned long long* wcnt, unsigned long long* next_slot,
                 U* tail) {
  constexpr int B = ip_block<U>();
  const ShiftDigit<KIND, DESC, U> dg{shift};
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next_slot, 32ull);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (base >= nslots) break;
    const uint64_t mine = base + lane;
    uint32_t cand = __ballot_sync(0xFFFFFFFFu, mine < nslots && __ldcg(&flags[mine]) == F_UNPROC);
    while (cand) {
      const uint32_t l = __ffs(cand) - 1;
      cand &= cand - 1;
      const uint64_t j = base + l;
      U v[B / 32];
      slot_read<U, B>(a, tail, n, j, v);  // speculative: used only if the claim succeeds
      uint32_t got = 0;
      if (lane == 0) got = atomicCAS(&flags[j], F_UNPROC, F_READING) == F_UNPROC;
      if (!__shfl_sync(0xFFFFFFFFu, got, 0)) continue;
      uint32_t bkt = dg(__shfl_sync(0xFFFFFFFFu, v[0], 0));
      __threadfence();  // our reads of slot j are complete (their values are in use above)
      __syncwarp();
      if (lane == 0) atomicExch(&flags[j], F_FREE);
      for (;;) {  // carry block v (bucket bkt) to its next destination slot
        unsigned long long d = 0;
        if (lane == 0) d = dstart[bkt] + atomicAdd(&wcnt[bkt], 1ull);
        d = __shfl_sync(0xFFFFFFFFu, d, 0);
        U w[B / 32];
        slot_read<U, B>(a, tail, n, d, w);  // speculative, as above
        uint32_t prev = 0;
        if (lane == 0) prev = atomicCAS(&flags[d], F_UNPROC, F_READING);
        prev = __shfl_sync(0xFFFFFFFFu, prev, 0);
        if (prev == F_UNPROC) {  // an unread block: take it along, put ours in its place
          const uint32_t nb = dg(__shfl_sync(0xFFFFFFFFu, w[0], 0));
          slot_write<U, B>(a, tail, n, d, v);
#pragma unroll
          for (int k = 0; k < B / 32; ++k) v[k] = w[k];
          bkt = nb;
          continue;
        }
        if (prev == F_READING) {  // a source being read by another warp: wait until free
          if (lane == 0)
            while (atomicAdd(&flags[d], 0u) != F_FREE) __nanosleep(32);
          __syncwarp();
        }
        slot_write<U, B>(a, tail, n, d, v);
        break;
      }
    }
  }
}

struct IpBucket {
  unsigned long long S, S1, D, f;  // [S, S1) final range; blocks at slots D .. D+f-1
};

// P3a.  One CTA per bucket: keys of its blocks past S1 -> extra[b].
template <typename U>
__global__ void __launch_bounds__(256) k_ip_collect(const U* __restrict__ a, uint64_t n, const U* __restrict__ tail,
                                                    const IpBucket* __restrict__ bk, U* __restrict__ extra,
                                                    uint32_t* __restrict__ extra_n) {
  constexpr int B = ip_block<U>();
  const IpBucket q = bk[blockIdx.x];
  const uint64_t end = (q.D + q.f) * B;
  const uint64_t from = max64(q.S1, q.D * B);
  const uint64_t m = end > from ? end - from : 0;  // < B
  for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint64_t p = from + i;
    extra[(uint64_t)blockIdx.x * B + i] = p < n ? a[p] : tail[p - n];
  }
  if (threadIdx.x == 0) extra_n[blockIdx.x] = (uint32_t)m;
}

// P3b.  One CTA per bucket: fill [S, min(D*B, S1)) then [(D+f)*B, S1) from the overflow of every
// stripe and the set-aside keys.
template <typename U>
__global__ void __launch_bounds__(256) k_ip_fill(U* __restrict__ a, const IpBucket* __restrict__ bk,
                                                 const U* __restrict__ ovf, const uint32_t* __restrict__ ovc,
                                                 int stripes, const U* __restrict__ extra,
                                                 const uint32_t* __restrict__ extra_n) {
  constexpr int B = ip_block<U>();
  const uint32_t b = blockIdx.x;
  const IpBucket q = bk[b];
  const uint64_t g1_end = min64(q.D * B, q.S1);
  const uint64_t g1 = g1_end > q.S ? g1_end - q.S : 0;
  const uint64_t g2_start = (q.D + q.f) * B;
  auto pos = [&](uint64_t g) -> uint64_t { return g < g1 ? q.S + g : g2_start + (g - g1); };
  uint64_t base = 0;
  for (int s = 0; s < stripes; ++s) {
    const uint32_t c = ovc[(uint64_t)s * 256 + b];
    for (uint32_t v = threadIdx.x; v < c; v += blockDim.x) a[pos(base + v)] = ovf[((uint64_t)s * 256 + b) * B + v];
    base += c;
  }
  const uint32_t e = extra_n[b];
  for (uint32_t v = threadIdx.x; v < e; v += blockDim.x) a[pos(base + v)] = extra[(uint64_t)b * B + v];
}

// ---------------------------------------------------------------------------------- host

struct IpLayout {
  size_t ovf, ovc, flags, count, fblocks, dstart, wcnt, next, bk, extra, extra_n, tail, lsd, total;
  int stripes;
  uint64_t chunk;
};

IpLayout ip_layout(int bytes, uint64_t n, uint64_t chunk) {
  IpLayout l{};
  const uint64_t B = IP_BLOCK_BYTES / bytes;
  l.stripes = num_sms();
  l.chunk = chunk;
  size_t off = 0;
  auto take = [&](size_t sz) {
    const size_t o = off;
    off = align_up(off + sz, 256);
    return o;
  };
  l.ovf = take((size_t)l.stripes * 256 * IP_BLOCK_BYTES);
  l.ovc = take((size_t)l.stripes * 256 * 4);
  l.flags = take((size_t)((n + B - 1) / B + 1) * 4);
  l.count = take(256 * 8);
  l.fblocks = take(256 * 8);
  l.dstart = take(256 * 8);
  l.wcnt = take(256 * 8);
  l.next = take(8);
  l.bk = take(256 * sizeof(IpBucket));
  l.extra = take(256 * IP_BLOCK_BYTES);
  l.extra_n = take(256 * 4);
  l.tail = take(IP_BLOCK_BYTES);
  l.lsd = off;
  off = align_up(off + lsd_workspace_bytes(bytes, chunk), 256);
  l.total = off;
  return l;
}

template <int KIND, bool DESC, typename U>
bsort_status_t ip_partition(U* a, uint64_t n, int shift, char* ws, const IpLayout& l, uint64_t* counts_out,
                            cudaStream_t s) {
  constexpr int B = ip_block<U>();
  auto* count = reinterpret_cast<unsigned long long*>(ws + l.count);
  auto* fblocks = reinterpret_cast<unsigned long long*>(ws + l.fblocks);
  auto* flags = reinterpret_cast<uint32_t*>(ws + l.flags);
  // count, fblocks, dstart, wcnt, next are consecutive: one memset
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(ws + l.count, 0, l.bk - l.count, s));
  const uint64_t stripe_len = align_up((n + l.stripes - 1) / l.stripes, IP_TILE);
  const uint64_t grid = (n + stripe_len - 1) / stripe_len;
  static DeviceOnce attr;
  auto k1 = k_ip_classify<KIND, DESC, U>;
  const int smem = 256 * IP_BLOCK_BYTES + IP_TILE * (int)sizeof(U);
  if (attr.pending()) {
    BSORT_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr.mark();
  }
  BSORT_LAUNCH(PROF_PASS, s,
               k1<<<(unsigned)grid, IP_THREADS, smem, s>>>(a, n, shift, stripe_len, reinterpret_cast<U*>(ws + l.ovf),
                                                           reinterpret_cast<uint32_t*>(ws + l.ovc), flags, count,
                                                           fblocks));
  // unused stripes (grid < l.stripes) contribute no overflow
  if ((int)grid < l.stripes)
    BSORT_LAUNCH(PROF_MEMSET, s,
                 cudaMemsetAsync(ws + l.ovc + grid * 256 * 4, 0, (size_t)(l.stripes - grid) * 256 * 4, s));
  unsigned long long h[512];
  BSORT_CUDA(cudaMemcpyAsync(h, ws + l.count, sizeof(h), cudaMemcpyDeviceToHost, s));
  BSORT_CUDA(cudaStreamSynchronize(s));
  IpBucket bk[256];
  unsigned long long dst[256];
  uint64_t S = 0;
  for (int b = 0; b < 256; ++b) {
    bk[b].S = S;
    S += h[b];
    bk[b].S1 = S;
    bk[b].D = (bk[b].S + B - 1) / B;
    bk[b].f = h[256 + b];
    dst[b] = bk[b].D;
    counts_out[b] = h[b];
  }
  if (S != n) return BSORT_ERROR_CUDA;  // cannot happen unless a kernel failed silently
  BSORT_CUDA(cudaMemcpyAsync(ws + l.dstart, dst, sizeof(dst), cudaMemcpyHostToDevice, s));
  BSORT_CUDA(cudaMemcpyAsync(ws + l.bk, bk, sizeof(bk), cudaMemcpyHostToDevice, s));
  const uint64_t nslots = (n + B - 1) / B;
  U* tail = reinterpret_cast<U*>(ws + l.tail);
  const unsigned pgrid = (unsigned)max64(1, min64((nslots + 7) / 8, (uint64_t)num_sms() * 8));
  BSORT_LAUNCH(PROF_PASS, s,
               k_ip_permute<KIND, DESC, U><<<pgrid, 256, 0, s>>>(
                   a, n, shift, flags, nslots, reinterpret_cast<const unsigned long long*>(ws + l.dstart),
                   reinterpret_cast<unsigned long long*>(ws + l.wcnt),
                   reinterpret_cast<unsigned long long*>(ws + l.next), tail));
  BSORT_LAUNCH(PROF_PASS, s,
               k_ip_collect<U><<<256, 256, 0, s>>>(a, n, tail, reinterpret_cast<const IpBucket*>(ws + l.bk),
                                                   reinterpret_cast<U*>(ws + l.extra),
                                                   reinterpret_cast<uint32_t*>(ws + l.extra_n)));
  BSORT_LAUNCH(PROF_PASS, s,
               k_ip_fill<U><<<256, 256, 0, s>>>(a, reinterpret_cast<const IpBucket*>(ws + l.bk),
                                                reinterpret_cast<const U*>(ws + l.ovf),
                                                reinterpret_cast<const uint32_t*>(ws + l.ovc), l.stripes,
                                                reinterpret_cast<const U*>(ws + l.extra),
                                                reinterpret_cast<const uint32_t*>(ws + l.extra_n)));
  return BSORT_SUCCESS;
}

template <int KIND, bool DESC, typename U>
bsort_status_t ip_sort(const DtypeInfo& di, U* a, uint64_t n, int shift, char* ws, const IpLayout& l,
                       cudaStream_t s) {
  if (n <= 1) return BSORT_SUCCESS;
  if (n <= l.chunk) return lsd_sort(di, a, nullptr, n, DESC, ws + l.lsd, l.total - l.lsd, s);
  if (shift < 0) return BSORT_SUCCESS;  // every digit consumed: all keys of this range are equal
  uint64_t c[256];
  bsort_status_t st = ip_partition<KIND, DESC, U>(a, n, shift, ws, l, c, s);
  if (st != BSORT_SUCCESS) return st;
  uint64_t start = 0, gstart = 0, glen = 0;
  auto flush = [&]() -> bsort_status_t {
    bsort_status_t r = BSORT_SUCCESS;
    if (glen > 1) r = lsd_sort(di, a + gstart, nullptr, glen, DESC, ws + l.lsd, l.total - l.lsd, s);
    glen = 0;
    return r;
  };
  for (int b = 0; b < 256; ++b) {
    if (c[b] > l.chunk) {
      if ((st = flush()) != BSORT_SUCCESS) return st;
      if ((st = ip_sort<KIND, DESC, U>(di, a + start, c[b], shift - 8, ws, l, s)) != BSORT_SUCCESS) return st;
    } else {
      if (glen + c[b] > l.chunk && (st = flush()) != BSORT_SUCCESS) return st;
      if (glen == 0) gstart = start;
      glen += c[b];
    }
    start += c[b];
  }
  return flush();
}

}  // namespace

uint64_t inplace_default_chunk(uint64_t n) {
  return min64(n, max64(1ull << 22, n / 32));
}

size_t inplace_workspace_bytes(int bytes, uint64_t n, uint64_t chunk) {
  if (n <= 1) return 0;
  if (bytes <= 2) return counting_workspace_bytes(bytes, n);
  if (chunk == 0) chunk = inplace_default_chunk(n);
  chunk = min64(chunk, n);
  if (chunk >= n) return lsd_workspace_bytes(bytes, n);
  return ip_layout(bytes, n, chunk).total;
}

bsort_status_t inplace_sort(const DtypeInfo& di, void* keys, uint64_t n, bool desc, uint64_t chunk, void* ws,
                            size_t ws_bytes, cudaStream_t s) {
  if (n <= 1) return BSORT_SUCCESS;
  if (di.bytes <= 2) return counting_sort(di, keys, n, desc, ws, ws_bytes, s);
  if (chunk == 0) chunk = inplace_default_chunk(n);
  chunk = min64(chunk, n);
  if (chunk >= n) return lsd_sort(di, keys, nullptr, n, desc, ws, ws_bytes, s);
  const IpLayout l = ip_layout(di.bytes, n, chunk);
  if (ws_bytes < l.total) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  char* w = static_cast<char*>(ws);
  const int top = di.bytes * 8 - 8;
#define BSORT_IP(KIND, U)                                                                               \
  return desc ? ip_sort<KIND, true, U>(di, static_cast<U*>(keys), n, top, w, l, s)                      \
              : ip_sort<KIND, false, U>(di, static_cast<U*>(keys), n, top, w, l, s)
  if (di.bytes == 4) {
    if (di.kind == KIND_U) BSORT_IP(KIND_U, uint32_t);
    if (di.kind == KIND_I) BSORT_IP(KIND_I, uint32_t);
    BSORT_IP(KIND_F, uint32_t);
  }
  if (di.kind == KIND_U) BSORT_IP(KIND_U, unsigned long long);
  if (di.kind == KIND_I) BSORT_IP(KIND_I, unsigned long long);
  BSORT_IP(KIND_F, unsigned long long);
#undef BSORT_IP
}

}  // namespace bsort
