// onesweep.cuh — a3/a4: one-sweep multi-digit histogram and the per-digit stable scatter
// pass with decoupled look-back (templates shared by the LSD sort and the MSD partition).
//
// Paper mapping.  Algorithm 1 splits a range on ONE bit per scan and Algorithm 2
// recurses MSB-first, so a w-bit key costs w full scans (Theorem 4; "64 complete
// array scans").  Here each scan is a stable 256-way split on an 8-bit digit of the
// transformed key, least-significant digit first: ceil(w/8) scans instead of w, branch-free
// ranking instead of the mispredicted bit test, no recursion.  LSD order is
// correct because every pass is stable (a stable sort on digit p preserves the order of
// digits < p), which is why the ranking below follows global index order exactly.
#pragma once
#include "common.cuh"
#include "scan.cuh"

namespace bsort {

// Look-back descriptor: [flag:2 | value:(W-2)], flag 0 = not ready, 1 = aggregate (this tile's
// count only), 2 = inclusive prefix (count of all tiles <= this one).  One word => no fence.
template <typename D> struct LookbackBits;
template <> struct LookbackBits<uint32_t> {
  static constexpr int SH = 30;
  static constexpr uint32_t AGG = 1u << 30, INC = 2u << 30, VAL = (1u << 30) - 1;
};
template <> struct LookbackBits<unsigned long long> {
  static constexpr int SH = 62;
  static constexpr unsigned long long AGG = 1ull << 62, INC = 2ull << 62, VAL = (1ull << 62) - 1;
};

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back, one thread per digit t (descriptors tile-major: [tile][256 digits], so
// the 256 walking threads of a CTA read 128-byte coalesced rows).  Each step issues G
// independent loads for the G nearest unfolded predecessors, so one L2 round trip folds in up
// to G tiles: at B200 tile rates (hundreds of CTAs on consecutive tiles) a one-load-per-step
// walk is a serial chain of L2 latencies.
template <int G, typename DescT>
__device__ __forceinline__ void lookback_issue(const DescT* lookback, uint32_t t, int64_t j, DescT (&v)[G]) {
#pragma unroll
  for (int q = 0; q < G; ++q) v[q] = (j - q >= 0) ? ld_relaxed(&lookback[(uint64_t)(j - q) * 256 + t]) : DescT(0);
}
// Folds the window v (predecessors j, j-1, ..., j-G+1, loaded by lookback_issue) and walks on
// until an inclusive prefix is found.  Returns the exclusive prefix of the tile.
template <int G, typename DescT>
__device__ __forceinline__ DescT lookback_finish(const DescT* lookback, uint32_t t, int64_t j, DescT (&v)[G]) {
  using LB = LookbackBits<DescT>;
  DescT excl = 0;
  for (;;) {
    bool stop = false, fin = false;
    int adv = G;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      if (!stop) {
        const DescT f = v[q] >> LB::SH;
        if (f == 0) {
          stop = true;  // not published yet: poll again from here
          adv = q;
        } else {
          excl += v[q] & LB::VAL;
          if (f == 2) stop = fin = true;
        }
      }
    }
    if (fin) return excl;  // tile 0 holds an inclusive prefix, so the walk ends there at the latest
    j -= adv;
    lookback_issue<G>(lookback, t, j, v);
  }
}
template <int G, typename DescT>
__device__ __forceinline__ DescT lookback_walk(const DescT* lookback, uint32_t t, uint32_t tile) {
  DescT v[G];
  lookback_issue<G>(lookback, t, (int64_t)tile - 1, v);
  return lookback_finish<G>(lookback, t, (int64_t)tile - 1, v);
}

template <typename U> __device__ __forceinline__ U ldg_nc(const U* p);
template <> __device__ __forceinline__ uint32_t ldg_nc(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ unsigned long long ldg_nc(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Device-resident pass plan written by k_plan (device-side trivial-digit skipping, so the
// whole sort is enqueued without a host sync).
struct PassPlan {
  uint32_t skip[8];     // digit p is trivial (one bin holds all n keys): pass p not executed
  uint32_t src_alt[8];  // executed pass p reads the scratch buffer (and writes the user buffer)
  uint32_t final_copy;  // odd number of executed passes: result is in scratch, copy back
  uint32_t executed;    // number of executed passes
  uint32_t j01;         // pass 1 runs as RANK_J01 (every nonzero digit-0 bucket >= one tile)
  uint32_t reverse;     // input already in the opposite order: no pass, k_copy_back reverses
  uint32_t first;       // first executed pass (8: none) -- k_pass2 encodes keys as it loads them
  uint32_t last;        // last executed pass (8: none) -- k_pass2 decodes keys as it writes them
  uint32_t run2;        // pass 2 runs as R2_RUN2 (every nonzero (digit 1, digit 0) bin >= one tile)
  uint32_t skew;        // bit p: one bin of digit p holds > n/8 keys (pass2.cuh half-warp counters)
  uint32_t fewruns;     // bit p: pass p's input has few distinct lower-bit values (long runs): the
                        // run-ranking look-back kernel replaces k_pass2 (k_plan_joint)
  uint32_t pad[7];
};

// Presorted-input check (§8 a3 "sortedness test"), folded into the histogram sweep: for every
// adjacent pair (j, j+1) of the input, order[0] |= enc(x_j) > enc(x_j+1) (not already in the
// requested order) and order[1] |= enc(x_j) < enc(x_j+1) (not in the opposite order).  The key
// order is a total order on bit patterns, so an input with order[0] == 0 IS the sorted output,
// and one with order[1] == 0 reversed is (equal keys have equal bits).
struct OrderFlags {
  uint32_t up = 0, down = 0;
  template <typename U>
  __device__ __forceinline__ void pair(U a, U b) {  // encoded keys, a before b
    up |= a > b;
    down |= a < b;
  }
  __device__ __forceinline__ bool done() const { return up & down; }  // both set: nothing to learn
  // keys kv[0..V) at positions j0.., plus the pair (kv[V-1], x[j0+V]); once this thread has seen
  // both violations (any unsorted input, within a vector or two) the check is skipped.  The
  // next vector's first key comes from the next lane when it is active (consecutive lanes hold
  // consecutive vectors), else from memory.
  template <int KIND, bool DESC, typename U, int V>
  __device__ __forceinline__ void vector(const U (&kv)[V], uint64_t j0, const U* keys, uint64_t n) {
    const uint32_t m = __activemask();
    if (__all_sync(m, done())) return;  // the common case for unsorted input: one vote
    const uint32_t lane = threadIdx.x & 31;
    const U nb = shfl_down_u(m, kv[0]);
    if (done()) return;
    U e[V];
#pragma unroll
    for (int j = 0; j < V; ++j) e[j] = key_encode<KIND, DESC>(kv[j]);
#pragma unroll
    for (int j = 0; j + 1 < V; ++j) pair(e[j], e[j + 1]);
    const uint64_t nx = j0 + V;
    if (nx < n) {
      const bool have = lane < 31 && ((m >> (lane + 1)) & 1u);
      pair(e[V - 1], key_encode<KIND, DESC>(have ? nb : keys[nx]));
    }
  }
  template <typename U>
  static __device__ __forceinline__ U shfl_down_u(uint32_t m, U v) {
    if constexpr (sizeof(U) == 4) {
      return U(__shfl_down_sync(m, (uint32_t)v, 1));
    } else {
      const uint32_t lo = __shfl_down_sync(m, (uint32_t)v, 1), hi = __shfl_down_sync(m, (uint32_t)(v >> 32), 1);
      return U(lo) | (U(hi) << 32);
    }
  }
  // block-wide reduce + one atomic per block (every thread of the block must call it)
  __device__ __forceinline__ void flush(uint32_t* order) {
    const int u = __syncthreads_or(up), d = __syncthreads_or(down);
    if (threadIdx.x == 0 && order != nullptr) {
      if (u) atomicOr(&order[0], 1u);
      if (d) atomicOr(&order[1], 1u);
    }
  }
};

// Digit of LSD pass p: byte p of the transformed key (SHIFT = 8p is a compile-time constant so
// the digit is one funnel-shift + mask after the transform).
template <int KIND, bool DESC, typename U, int SHIFT>
struct RadixDigit {
  static constexpr bool REMOTE = false;
  __device__ __forceinline__ uint32_t operator()(U x) const {
    return uint32_t(key_encode<KIND, DESC>(x) >> SHIFT) & 0xFFu;
  }
  // digit and the bits below it (the digits the earlier LSD passes sorted by), one encode
  __device__ __forceinline__ uint32_t digit_low(U x, U* low) const {
    const U e = key_encode<KIND, DESC>(x);
    if constexpr (SHIFT == 0)
      *low = U(0);
    else
      *low = U(e & U((U(1) << SHIFT) - 1));
    return uint32_t(e >> SHIFT) & 0xFFu;
  }
};

// Digit of the MSD partition: destination rank of the key's top-16-bit bin.
// REMOTE (fused partition + exchange, §8 N1): dst_base[q] is the byte address (peer-mapped
// over NVLink when q is another GPU) of the first slot this rank owns in rank q's receive
// buffer; the pass writes each key there directly instead of into a local bucketed copy.
template <int KIND, bool DESC, typename U, bool REMOTE_ = false>
struct RankDigit {
  static constexpr bool REMOTE = REMOTE_;
  uint32_t cuts[BSORT_DIST_MAX_RANKS + 1];
  int nranks;
  unsigned long long dst_base[REMOTE_ ? BSORT_DIST_MAX_RANKS : 1];
  __device__ __forceinline__ uint32_t operator()(U x) const {
    const uint32_t b = uint32_t(key_encode<KIND, DESC>(x) >> (sizeof(U) * 8 - 16));
    uint32_t lo = 0, hi = (uint32_t)nranks;  // largest q in [0,nranks) with cuts[q] <= b
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (cuts[mid] <= b) lo = mid; else hi = mid;
    }
    return lo;
  }
  __device__ __forceinline__ uint32_t digit_low(U x, U* low) const {
    *low = U(0);
    return (*this)(x);
  }
};

// A region a kernel zeroes (grid-stride, 16-byte stores): look-back descriptors of later passes,
// so no memset launch per pass (lsd_impl.cuh: the pass kernels below 2^22 keys, the joint
// histogram sweep above 2^24).
struct ZeroSpan {
  uint4* p;
  uint32_t n16;
};

// ---------------------------------------------------------------------------------------
// a3: one read of all keys, P = sizeof(U) digit histograms of 256 bins.  Counters are
// lane-banked (address = bin*LANES + lane%LANES, bank = lane) so the shared-memory atomics of a
// warp never conflict; one CTA of 1024 threads per SM, grid-stride, 128-bit loads.
constexpr int HIST_THREADS = 1024;

// Forward declaration: the fused-plan epilogue below.
template <int NT>
__device__ __forceinline__ void plan_body(const unsigned long long* ghist, uint64_t n, int P,
                                          unsigned long long* __restrict__ bases, PassPlan* __restrict__ plan,
                                          uint32_t* __restrict__ tile_counters,
                                          unsigned long long* __restrict__ gcount, const uint32_t* order);

// What the fused-plan histogram kernel needs for k_plan's work (FUSE_PLAN; order[2] is the
// arrival ticket, zeroed with the histograms).
struct PlanArgs {
  unsigned long long* bases;
  PassPlan* plan;
  uint32_t* tile_counters;
  unsigned long long* gcount;
};

template <int KIND, bool DESC, typename U, int LANES, bool FUSE_PLAN = false>
__global__ void __launch_bounds__(HIST_THREADS, 1)
    k_onesweep_hist(const U* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ ghist,
                    uint32_t* __restrict__ order = nullptr, PlanArgs pa = {}) {
  constexpr int P = sizeof(U);
  OrderFlags of;
  // pair (j, j+1) for a scalar key j
  auto check1 = [&](uint64_t j, U kj) {
    if (j + 1 < n) of.pair(kj, key_encode<KIND, DESC>(ldg_nc(keys + j + 1)));
  };
  extern __shared__ uint32_t hs[];  // [P][256][LANES]
  for (int i = threadIdx.x; i < P * 256 * LANES; i += HIST_THREADS) hs[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & (LANES - 1);
  auto add = [&](U x) {
    const U k = key_encode<KIND, DESC>(x);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint32_t d = uint32_t(k >> (8 * p)) & 0xFFu;
      atomicAdd(&hs[(p * 256 + d) * LANES + lane], 1u);
    }
  };
  constexpr int PER_VEC = 16 / sizeof(U);
  const uint64_t T = (uint64_t)gridDim.x * HIST_THREADS;
  const uint64_t gt = (uint64_t)blockIdx.x * HIST_THREADS + threadIdx.x;
  const uint64_t head = min64(n, ((16 - ((uintptr_t)keys & 15)) & 15) / sizeof(U));
  for (uint64_t i = gt; i < head; i += T) add(keys[i]);
  const uint4* v = reinterpret_cast<const uint4*>(keys + head);
  const uint64_t nv = (n - head) / PER_VEC;
  // vector i: its keys, the pairs inside it and the pair (its last key, the next key)
  auto vec = [&](uint4 q, uint64_t i) {
    U kv[PER_VEC];
    if constexpr (sizeof(U) == 4) {
      kv[0] = U(q.x); kv[1] = U(q.y); kv[2] = U(q.z); kv[3] = U(q.w);
    } else {
      kv[0] = U(q.x) | (U(q.y) << 32);
      kv[1] = U(q.z) | (U(q.w) << 32);
    }
#pragma unroll
    for (int j = 0; j < PER_VEC; ++j) add(kv[j]);
    of.vector<KIND, DESC>(kv, head + i * PER_VEC, keys, n);
  };
  for (uint64_t i = gt; i < head; i += T) check1(i, key_encode<KIND, DESC>(keys[i]));
  uint64_t i = gt;
  for (; i + 3 * T < nv; i += 4 * T) {
    uint4 q0 = __ldcs(v + i), q1 = __ldcs(v + i + T), q2 = __ldcs(v + i + 2 * T), q3 = __ldcs(v + i + 3 * T);
    vec(q0, i); vec(q1, i + T); vec(q2, i + 2 * T); vec(q3, i + 3 * T);
  }
  for (; i < nv; i += T) vec(__ldcs(v + i), i);
  for (uint64_t j = head + nv * PER_VEC + gt; j < n; j += T) {
    add(keys[j]);
    check1(j, key_encode<KIND, DESC>(keys[j]));
  }
  of.flush(order);
  __syncthreads();
  for (int b = threadIdx.x; b < P * 256; b += HIST_THREADS) {
    uint32_t s = 0;
#pragma unroll 8
    for (int l = 0; l < LANES; ++l) s += hs[b * LANES + ((l + b) & (LANES - 1))];
    if (s) atomicAdd(&ghist[b], (unsigned long long)s);
  }
  if constexpr (FUSE_PLAN) {
    // the last CTA to finish plans (k_plan's work without its launch): small sorts are bound by
    // launch count (DESIGN.md §6 small n)
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&order[2], 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      plan_body<HIST_THREADS>(ghist, n, P, pa.bases, pa.plan, pa.tile_counters, pa.gcount, order);
    }
  }
}

// a3 with the joint histogram of the two lowest digits (pass 1 without look-back, RANK_J01):
// J[d1 * 256 + d0] counted in 65536 u16 halves of 32768 smem words (a half that reaches 0x8000
// is drained to the global count), the digits >= 2 lane-banked as above.  d0 is the fast index
// so that nearly sorted keys spread over banks; a warp whose 32 keys share one joint bin (runs
// of equal keys) adds once.  The marginals of digits 0 and 1 are derived from J by k_plan.  One
// read of the keys.
// Presorted check as a sweep of its own (joint-histogram sizes): order[0] |= some adjacent pair
// out of the requested order, order[1] |= some pair out of the opposite order (OrderFlags).  Warps
// publish a flag as soon as they see it and stop once both flags are set anywhere, so an unsorted
// input costs each warp about one vector (microseconds), while a presorted, reversed or
// all-equal input -- the cases where the result is decided here -- is read once, and the
// histogram sweep then returns at once (k_onesweep_hist_joint, prechecked).
template <int KIND, bool DESC, typename U>
__global__ void __launch_bounds__(HIST_THREADS) k_order_check(const U* __restrict__ keys, uint64_t n,
                                                              uint32_t* __restrict__ order) {
  constexpr int PER_VEC = 16 / sizeof(U);
  OrderFlags of;
  const uint64_t T = (uint64_t)gridDim.x * HIST_THREADS;
  const uint64_t gt = (uint64_t)blockIdx.x * HIST_THREADS + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t head = min64(n, ((16 - ((uintptr_t)keys & 15)) & 15) / sizeof(U));
  for (uint64_t j = gt; j < head; j += T)
    if (j + 1 < n) of.pair(key_encode<KIND, DESC>(keys[j]), key_encode<KIND, DESC>(keys[j + 1]));
  const uint4* v = reinterpret_cast<const uint4*>(keys + head);
  const uint64_t nv = (n - head) / PER_VEC;
  auto check_vec = [&](uint4 q, uint64_t i) {
    if constexpr (sizeof(U) == 4) {
      const U kv[4] = {U(q.x), U(q.y), U(q.z), U(q.w)};
      of.vector<KIND, DESC>(kv, head + i * PER_VEC, keys, n);
    } else {
      const U kv[2] = {U(q.x) | (U(q.y) << 32), U(q.z) | (U(q.w) << 32)};
      of.vector<KIND, DESC>(kv, head + i * PER_VEC, keys, n);
    }
  };
  // round 0, the whole CTA: one vector per thread, one flag publication per CTA.  An unsorted
  // input ends here (every CTA meets both violations in its first vectors).
  if (gt < nv) check_vec(__ldcs(v + gt), gt);
  {
    const int u = __syncthreads_or(of.up), d = __syncthreads_or(of.down);
    if (threadIdx.x == 0) {
      if (u) atomicOr(&order[0], 1u);
      if (d) atomicOr(&order[1], 1u);
    }
    if (u && d) return;
    of.up = u;  // a flag the CTA has published needs no further checking
    of.down = d;
  }
  const volatile uint32_t* vo = order;
  uint32_t told = (of.up ? 1u : 0u) | (of.down ? 2u : 0u);  // flags already published
  uint32_t polled = 0;  // lane 0: global flags read at the previous poll (not waited on)
  auto publish = [&]() -> bool {  // whole warp; true once both flags are set globally
    const uint32_t f = __reduce_or_sync(0xffffffffu, (of.up ? 1u : 0u) | (of.down ? 2u : 0u));
    uint32_t both = 0;
    if (lane == 0) {
      if ((f & 1u) && !(told & 1u)) atomicOr(&order[0], 1u);
      if ((f & 2u) && !(told & 2u)) atomicOr(&order[1], 1u);
      both = polled;
      polled = vo[0] & vo[1];
    }
    told |= f;
    return __shfl_sync(0xffffffffu, both, 0) != 0u;
  };
  // later rounds: four vectors per thread in flight; warp-uniform bounds (collectives inside).
  // Whole warps hold 32 consecutive vectors: the key after a lane's vector is the next lane's
  // first key (shuffle), and lane 31's is loaded with the vectors (no dependent load later).
  const uint64_t wbase = gt - lane;
  auto check_full = [&](uint4 q, U nxt) {
    U e[PER_VEC];
    if constexpr (sizeof(U) == 4) {
      e[0] = U(q.x); e[1] = U(q.y); e[2] = U(q.z); e[3] = U(q.w);
    } else {
      e[0] = U(q.x) | (U(q.y) << 32); e[1] = U(q.z) | (U(q.w) << 32);
    }
    const U nb = OrderFlags::shfl_down_u(0xffffffffu, e[0]);
#pragma unroll
    for (int j = 0; j < PER_VEC; ++j) e[j] = key_encode<KIND, DESC>(e[j]);
#pragma unroll
    for (int j = 0; j + 1 < PER_VEC; ++j) of.pair(e[j], e[j + 1]);
    of.pair(e[PER_VEC - 1], key_encode<KIND, DESC>(lane < 31 ? nb : nxt));
  };
  uint64_t r = T;
  for (uint32_t round = 0; wbase + r + 3 * T + 32 < nv; r += 4 * T, ++round) {
    const uint64_t i = gt + r;
    const uint4 q0 = __ldcs(v + i), q1 = __ldcs(v + i + T), q2 = __ldcs(v + i + 2 * T), q3 = __ldcs(v + i + 3 * T);
    U x0 = 0, x1 = 0, x2 = 0, x3 = 0;  // lane 31: the key after its vector (inside the array)
    if (lane == 31) {
      const U* kb = keys + head + (i + 1) * PER_VEC;
      x0 = kb[0];
      x1 = kb[T * PER_VEC];
      x2 = kb[2 * T * PER_VEC];
      x3 = kb[3 * T * PER_VEC];
    }
    check_full(q0, x0);
    check_full(q1, x1);
    check_full(q2, x2);
    check_full(q3, x3);
    if ((round & 3u) == 3u && publish()) return;
  }
  for (; wbase + r < nv; r += T) {
    const uint64_t i = gt + r;
    if (i < nv) check_vec(__ldcs(v + i), i);
  }
  for (uint64_t j = head + nv * PER_VEC + gt; j < n; j += T)
    if (j + 1 < n) of.pair(key_encode<KIND, DESC>(keys[j]), key_encode<KIND, DESC>(keys[j + 1]));
  publish();
}

// Chunked look-back of LSD pass 2 of 32-bit keys (pass2.cuh CHUNKED): its input is sorted by the
// low 16 bits, so it splits into LB_NC contiguous chunks by the top two bits of digit 1, and every
// chunk is its own look-back chain.  The start of (chunk c, digit d) in the output is
// base_2[d] + sum_{c' < c} C[c'][d], C = the coarse joint histogram of (digit 1 >> 6, digit 2),
// which the histogram sweep counts instead of a plain digit-2 histogram (its marginal).  (Pass 3
// chunked the same way measured slower in the sort: 3.94 -> 4.12 ms.)
constexpr int LB_NC = 4;
#ifndef HIST_PLAIN_VEC
#define HIST_PLAIN_VEC 1
#endif
// coarse-joint shared counters [256 digits][LB_NC chunks][CJ_LANES lane banks]: lanes l and l + 16
// share a bank only when their chunks have equal parity
constexpr int CJ_LANES = 16;
// pass 3's coarse joint (digit 3, digit 2 >> 6): 8 lane banks (the 16-bank pass-2 table and the
// 65,536-bin joint fill the rest of the 227 KB)
constexpr int CJ3_LANES = 8;

// shared words of k_onesweep_hist_joint: 65,536 u16 joint bins + digit counters (32-bit keys:
// digit 3 lane-banked + the pass-2 coarse joint; 64-bit keys: digits 2-7 with LANES banks)
template <int P, int LANES>
__host__ __device__ constexpr int hist_joint_words() {
  return 32768 + (P == 4 ? 256 * LB_NC * (CJ3_LANES + CJ_LANES) : (P - 2) * 256 * LANES);
}

template <int KIND, bool DESC, typename U, int LANES>
__global__ void __launch_bounds__(HIST_THREADS, 1)
    k_onesweep_hist_joint(const U* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ ghist,
                          unsigned long long* __restrict__ gjoint, uint32_t* __restrict__ order = nullptr,
                          bool prechecked = false, unsigned long long* __restrict__ gcoarse = nullptr,
                          ZeroSpan zs = {}) {
  constexpr int P = sizeof(U);
  // 32-bit keys: digits 2 and 3 counted as the coarse joints of passes 2 and 3 (LB_NC; the launch
  // sizes shared memory by hist_joint_words)
  constexpr bool COARSE = P == 4;
  static_assert(!COARSE || LANES == 32, "digit-3 counters lane-banked");
  OrderFlags of;
  if (prechecked) {
    // k_order_check ran first: a presorted (or reversed) input needs no histogram -- no pass
    // runs -- and otherwise both violations are known, so this sweep checks no pairs
    if (__ldcg(&order[0]) == 0 || __ldcg(&order[1]) == 0) return;
    of.up = of.down = 1;
  }
  auto check1 = [&](uint64_t j, U kj) {
    if (j + 1 < n) of.pair(kj, key_encode<KIND, DESC>(ldg_nc(keys + j + 1)));
  };
  extern __shared__ uint32_t hs[];  // [32768 joint words][P-2][256][LANES]
  uint32_t* hj = hs;
  uint32_t* hd = hs + 32768;
  for (int i = threadIdx.x; i < hist_joint_words<P, LANES>(); i += HIST_THREADS) hs[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & (LANES - 1);
  auto add_joint = [&](uint32_t jb, uint32_t inc) {  // jb = d1 * 256 + d0
    const uint32_t sh = (jb & 1u) << 4;
    const uint32_t old = atomicAdd(&hj[jb >> 1], inc << sh);
    const uint32_t h = (old >> sh) & 0xFFFFu;
    if (h < 0x8000u && h + inc >= 0x8000u) {  // this add took the half to >= 0x8000: drain
      atomicAdd(&hj[jb >> 1], 0u - (0x8000u << sh));
      atomicAdd(&gjoint[jb], 0x8000ull);
    }
  };
  auto add_high = [&](U k) {
    if constexpr (COARSE) {
      const uint32_t x = uint32_t(k);
      // (digit 3, digit 2 >> 6) = bits 22-31 and (digit 2, digit 1 >> 6) = bits 14-23 of the key,
      // as index digit * LB_NC + chunk
      atomicAdd(&hd[(x >> 22) * CJ3_LANES + (lane & (CJ3_LANES - 1))], 1u);
      atomicAdd(&hd[256 * LB_NC * CJ3_LANES + ((x >> 14) & 0x3FFu) * CJ_LANES + (lane & (CJ_LANES - 1))], 1u);
    } else {
#pragma unroll
      for (int p = 2; p < P; ++p) {
        const uint32_t d = uint32_t(k >> (8 * p)) & 0xFFu;
        atomicAdd(&hd[((p - 2) * 256 + d) * LANES + lane], 1u);
      }
    }
  };
  // scalar keys (ragged head/tail, divergent): no warp collectives
  auto add = [&](U x) {
    const U k = key_encode<KIND, DESC>(x);
    add_joint(uint32_t(k) & 0xFFFFu, 1u);
    add_high(k);
  };
  constexpr int PER_VEC = 16 / sizeof(U);
  // a full vector of PER_VEC consecutive keys, called by whole warps: equal joint bins within
  // the thread, and within the warp, are added once (runs of equal keys do not serialize)
  auto add_vec = [&](const U (&kv)[PER_VEC]) {
    if constexpr (COARSE && HIST_PLAIN_VEC) {
      // 32-bit keys: single increments (the drain test is one compare), except that a warp whose
      // 128 keys share one joint bin (long runs of equal keys that are not presorted: those
      // never reach this sweep, k_order_check) adds once
      U k[PER_VEC];
      uint32_t jb[PER_VEC];
#pragma unroll
      for (int j = 0; j < PER_VEC; ++j) {
        k[j] = key_encode<KIND, DESC>(kv[j]);
        jb[j] = uint32_t(k[j]) & 0xFFFFu;
      }
      const uint32_t j0 = __shfl_sync(0xffffffffu, jb[0], 0);
      const bool uniform = __all_sync(0xffffffffu, ((jb[0] ^ j0) | (jb[1] ^ j0) | (jb[2] ^ j0) | (jb[3] ^ j0)) == 0u);
      if (uniform) {
        if ((threadIdx.x & 31) == 0) add_joint(jb[0], 32u * PER_VEC);
      } else {
#pragma unroll
        for (int j = 0; j < PER_VEC; ++j) {
          const uint32_t sh = (jb[j] & 1u) << 4;
          const uint32_t old = atomicAdd(&hj[jb[j] >> 1], 1u << sh);
          if (((old >> sh) & 0xFFFFu) == 0x7FFFu) {  // this add took the half to 0x8000: drain
            atomicAdd(&hj[jb[j] >> 1], 0u - (0x8000u << sh));
            atomicAdd(&gjoint[jb[j]], 0x8000ull);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < PER_VEC; ++j) add_high(k[j]);
      return;
    }
    U k[PER_VEC];
    uint32_t jb[PER_VEC];
    bool same = true;
#pragma unroll
    for (int j = 0; j < PER_VEC; ++j) {
      k[j] = key_encode<KIND, DESC>(kv[j]);
      jb[j] = uint32_t(k[j]) & 0xFFFFu;
      same &= jb[j] == jb[0];
    }
    const uint32_t j0 = __shfl_sync(0xffffffffu, jb[0], 0);  // every lane (no short-circuit)
    const bool uniform = __all_sync(0xffffffffu, same & (jb[0] == j0));
    if (uniform) {
      if ((threadIdx.x & 31) == 0) add_joint(jb[0], 32u * PER_VEC);
    } else if (same) {
      add_joint(jb[0], PER_VEC);
    } else {
#pragma unroll
      for (int j = 0; j < PER_VEC; ++j) add_joint(jb[j], 1u);
    }
#pragma unroll
    for (int j = 0; j < PER_VEC; ++j) add_high(k[j]);
  };
  const uint64_t T = (uint64_t)gridDim.x * HIST_THREADS;
  const uint64_t gt = (uint64_t)blockIdx.x * HIST_THREADS + threadIdx.x;
  const uint64_t head = min64(n, ((16 - ((uintptr_t)keys & 15)) & 15) / sizeof(U));
  for (uint64_t i = gt; i < head; i += T) add(keys[i]);
  const uint4* v = reinterpret_cast<const uint4*>(keys + head);
  const uint64_t nv = (n - head) / PER_VEC;
  auto order_vec = [&](const U (&kv)[PER_VEC], uint64_t i) { of.vector<KIND, DESC>(kv, head + i * PER_VEC, keys, n); };
  auto vec = [&](uint4 q, uint64_t i, bool check) {
    if constexpr (sizeof(U) == 4) {
      const U kv[4] = {U(q.x), U(q.y), U(q.z), U(q.w)};
      add_vec(kv);
      if (check) order_vec(kv, i);
    } else {
      const U kv[2] = {U(q.x) | (U(q.y) << 32), U(q.z) | (U(q.w) << 32)};
      add_vec(kv);
      if (check) order_vec(kv, i);
    }
  };
  for (uint64_t i = gt; i < head; i += T) check1(i, key_encode<KIND, DESC>(keys[i]));
  // whole warps iterate together (collectives inside): the loop bound is warp-uniform
  const uint64_t wbase = gt & ~uint64_t(31);
  uint64_t i = gt;
  // order check only until every lane of the warp has seen both violations (an unsorted input:
  // the first iteration or two), then the plain loop
  for (; wbase + (i - gt) + 3 * T + 31 < nv && !__all_sync(0xffffffffu, of.done()); i += 4 * T) {
    uint4 q0 = __ldcs(v + i), q1 = __ldcs(v + i + T), q2 = __ldcs(v + i + 2 * T), q3 = __ldcs(v + i + 3 * T);
    vec(q0, i, true); vec(q1, i + T, true); vec(q2, i + 2 * T, true); vec(q3, i + 3 * T, true);
  }
  for (; wbase + (i - gt) + 3 * T + 31 < nv; i += 4 * T) {
    uint4 q0 = __ldcs(v + i), q1 = __ldcs(v + i + T), q2 = __ldcs(v + i + 2 * T), q3 = __ldcs(v + i + 3 * T);
    vec(q0, i, false); vec(q1, i + T, false); vec(q2, i + 2 * T, false); vec(q3, i + 3 * T, false);
  }
  for (; i < nv; i += T) {  // remaining vectors: per key (a warp may be partial here)
    const uint4 q = __ldcs(v + i);
    if constexpr (sizeof(U) == 4) {
      const U kv[4] = {U(q.x), U(q.y), U(q.z), U(q.w)};
      add(kv[0]); add(kv[1]); add(kv[2]); add(kv[3]);
      order_vec(kv, i);
    } else {
      const U kv[2] = {U(q.x) | (U(q.y) << 32), U(q.z) | (U(q.w) << 32)};
      add(kv[0]); add(kv[1]);
      order_vec(kv, i);
    }
  }
  for (uint64_t j = head + nv * PER_VEC + gt; j < n; j += T) {
    add(keys[j]);
    check1(j, key_encode<KIND, DESC>(keys[j]));
  }
  // the look-back regions of the LSD passes (lsd_run): zeroed here, where HBM has room (this
  // sweep is bound by shared atomics), instead of one memset launch per look-back pass
  for (uint64_t i = gt; i < zs.n16; i += T) __stcs(&zs.p[i], make_uint4(0u, 0u, 0u, 0u));
  of.flush(order);
  __syncthreads();
  for (int w = threadIdx.x; w < 32768; w += HIST_THREADS) {
    const uint32_t c = hj[w];
    if (c & 0xFFFFu) atomicAdd(&gjoint[2 * w], (unsigned long long)(c & 0xFFFFu));
    if (c >> 16) atomicAdd(&gjoint[2 * w + 1], (unsigned long long)(c >> 16));
  }
  if constexpr (COARSE) {
    static_assert(LB_NC == 4, "shared index digit * 4 + chunk");
    // coarse joints to gcoarse[pass - 2][chunk][digit]; their marginals are digits 2 and 3
    for (int b = threadIdx.x; b < LB_NC * 256; b += HIST_THREADS) {  // pass 3
      uint32_t s = 0;
#pragma unroll
      for (int l = 0; l < CJ3_LANES; ++l) s += hd[b * CJ3_LANES + ((l + b) & (CJ3_LANES - 1))];
      if (s) {
        const int d = b >> 2, c = b & 3;
        atomicAdd(&gcoarse[(LB_NC + c) * 256 + d], (unsigned long long)s);
        atomicAdd(&ghist[768 + d], (unsigned long long)s);
      }
    }
    const uint32_t* hc = hd + 256 * LB_NC * CJ3_LANES;  // pass 2
    for (int b = threadIdx.x; b < LB_NC * 256; b += HIST_THREADS) {
      uint32_t s = 0;
#pragma unroll
      for (int l = 0; l < CJ_LANES; ++l) s += hc[b * CJ_LANES + ((l + b) & (CJ_LANES - 1))];
      if (s) {
        const int d = b >> 2, c = b & 3;  // shared index: digit * LB_NC + chunk
        atomicAdd(&gcoarse[c * 256 + d], (unsigned long long)s);
        atomicAdd(&ghist[512 + d], (unsigned long long)s);
      }
    }
  } else {
    for (int b = threadIdx.x; b < (P - 2) * 256; b += HIST_THREADS) {
      uint32_t s = 0;
#pragma unroll 8
      for (int l = 0; l < LANES; ++l) s += hd[b * LANES + ((l + b) & (LANES - 1))];
      if (s) atomicAdd(&ghist[512 + b], (unsigned long long)s);
    }
  }
}

// Marginals and row prefixes of the joint (digit 1, digit 0) histogram, one CTA per digit-1 value
// a (256 CTAs x 256 threads; thread b = digit-0 value), instead of one CTA reading all 65,536
// bins twice: the digit-1 marginal ghist[256 + a], the digit-0 marginal ghist[b] (atomics; the
// histogram region is zeroed before the sweep), the number of nonzero bins (*nz, zeroed with it)
// and J01's segment starts relative to digit a's base, seg[b * 256 + a] = sum_{b' < b} J[a][b']
// (the J01 pass adds the base).
static __global__ void __launch_bounds__(256)
    k_joint_marg(const unsigned long long* __restrict__ gjoint, unsigned long long* __restrict__ ghist,
                 unsigned long long* __restrict__ seg, uint32_t* __restrict__ nz) {
  __shared__ unsigned long long wt[256 / 32 + 1];
  const uint32_t a = blockIdx.x, b = threadIdx.x;
  const unsigned long long v = gjoint[a * 256 + b];
  unsigned long long total = 0;
  const unsigned long long ex = block_exclusive_scan<256>(v, wt, &total);
  seg[b * 256 + a] = ex;
  if (v) atomicAdd(&ghist[b], v);
  const int c = __syncthreads_count(v != 0);
  if (b == 0) {
    ghist[256 + a] = total;
    if (c) atomicAdd(nz, (uint32_t)c);
  }
}

// Joint plan for RANK_J01 (one CTA of 256 threads, after k_plan): pass 1 may skip the look-back
// when every nonzero digit-0 bucket holds at least `tile` keys -- then any tile-sized window of
// the pass-0 output meets at most two digit-0 runs.  Segment (d1 = a, d0 = b) of the pass-1
// output starts at bases1[a] + sum_{b' < b} J[a][b']; those starts seed the allocation counters
// (seg[b * 256 + a], the layout RANK_J01 indexes by (run's d0, digit)).
// Chunk map of LSD pass 2 of 32-bit keys (pass2.cuh CHUNKED; LB_NC above), written by
// k_plan_joint (arrays sized for passes 2 and 3): cstart[LB_NC + 1] (chunk c starts where digit 1 reaches 64c),
// ctile[LB_NC + 1] (first linear tile of each chunk, tiles of `tile` keys) and
// jp[LB_NC][256] = base_p[d] + sum_{c' < c} C_p[c'][d].
struct ChunkPlanArgs {
  const unsigned long long* bases;    // [P][256] digit bases (k_plan)
  const unsigned long long* gcoarse;  // [2][LB_NC][256] coarse joints (histogram sweep)
  unsigned long long* cstart;         // [2][LB_NC + 1]
  uint32_t* ctile;                    // [2][LB_NC + 1]
  uint32_t* jp;                       // [2][LB_NC][256]
  uint64_t tile, n;                   // nullptr jp: no chunked passes
  uint64_t tile_skew;                 // tile of the half-warp-row kernel (passes whose digit is skewed)
};

static __global__ void __launch_bounds__(256)
    k_plan_joint(const unsigned long long* __restrict__ gjoint, const unsigned long long* __restrict__ ghist,
                 const unsigned long long* __restrict__ bases1, uint64_t tile, PassPlan* __restrict__ plan,
                 unsigned long long* __restrict__ seg, uint64_t run2_tile = 0, uint64_t fewruns_tile = 0,
                 uint64_t fewruns_n = 0, ChunkPlanArgs cp = {}) {
  const uint32_t t = threadIdx.x;
  // RUN2 for pass 2 (pass2.cuh): its input is sorted by the low 16 bits, whose runs are the joint
  // bins; a tile meets at most two of them when every nonzero bin is at least a tile long
  bool ok2 = run2_tile > 0;
  for (int b = 0; b < 256 && ok2; ++b) {
    const unsigned long long c = gjoint[t * 256 + b];
    ok2 = c == 0 || c >= run2_tile;
  }
  const int run2 = __syncthreads_and(ok2);
  // Few distinct lower-bit values (fewruns_tile > 0, 32-bit keys): pass 2's input is sorted by
  // the low 16 bits, whose distinct values are the nonzero joint bins (nz16); pass 3's by the
  // low 24 bits, at most nz16 x (nonzero digit-2 bins) distinct values.  When the average run is
  // at least 4 tiles, almost every tile meets at most two runs, and the run-ranking kernel (one
  // unstable atomic per key, per-tile fallback to the stable ranking) beats the lane-ordered
  // stable pass, whose same-word atomics serialize on few distinct digits (cfg4 16-distinct).
  __shared__ uint32_t few_s;
  if (fewruns_tile > 0) {  // nz16 was counted by k_plan (plan->pad[0])
    const uint32_t nz2 = (uint32_t)__syncthreads_count(ghist[512 + t] != 0);
    if (t == 0) {
      const unsigned long long r2 = plan->pad[0], r3 = r2 * nz2, lim = fewruns_n / (4 * fewruns_tile);
      few_s = (r2 <= lim ? 4u : 0u) | (r3 <= lim ? 8u : 0u);
      plan->fewruns = few_s;
    }
  } else if (t == 0) {
    few_s = 0;
  }
  __syncthreads();
  // pass 2 by runs unless the few-runs kernel takes it
  const bool run2_on = run2 && !plan->skip[2] && !(few_s & 4u);
  if (t == 0) plan->run2 = run2_on ? 1u : 0u;
  if (cp.jp != nullptr) {
    for (int q = 0; q < 2; ++q) {  // passes 2 and 3 (index q = pass - 2)
      unsigned long long run = cp.bases[(2 + q) * 256 + t];
      for (int c = 0; c < LB_NC; ++c) {
        cp.jp[(q * LB_NC + c) * 256 + t] = (uint32_t)run;
        run += cp.gcoarse[(q * LB_NC + c) * 256 + t];
      }
      if (t == 0) {
        unsigned long long* cs = cp.cstart + q * (LB_NC + 1);
        uint32_t* ct = cp.ctile + q * (LB_NC + 1);
        for (int c = 0; c < LB_NC; ++c) cs[c] = cp.bases[(1 + q) * 256 + 64 * c];
        cs[LB_NC] = cp.n;
        ct[0] = 0;
        // the pass runs k_pass2's half-warp-row variant when its digit is skewed (k_plan's skew
        // bit), pass 2 the chunked RUN2 launch when run2 is set
        const uint64_t tl = (q == 0 && run2_on) ? run2_tile
                            : ((plan->skew >> (2 + q)) & 1u) ? cp.tile_skew : cp.tile;
        for (int c = 0; c < LB_NC; ++c) ct[c + 1] = ct[c] + (uint32_t)((cs[c + 1] - cs[c] + tl - 1) / tl);
      }
    }
  }
  const unsigned long long c0 = ghist[t];  // digit-0 marginal
  const int eligible = __syncthreads_and(c0 == 0 || c0 >= tile);
  if (t == 0) plan->j01 = (uint32_t)eligible && !plan->skip[1];
  (void)eligible;  // the segment starts (relative to digit 1's bases) are k_joint_marg's
  (void)seg;
  (void)bases1;
}

// Plan: exclusive scan of every digit histogram into global digit bases, trivial-digit
// detection, ping-pong buffer assignment, tile-counter reset.  Run by a block of NT >= 256
// threads (thread d < 256 owns digit d; every thread takes part in the block barriers): k_plan
// below, or the last CTA of the fused histogram kernel (k_onesweep_hist<..., FUSE_PLAN>).
template <int NT>
__device__ __forceinline__ void plan_body(const unsigned long long* ghist, uint64_t n, int P,
                                          unsigned long long* __restrict__ bases, PassPlan* __restrict__ plan,
                                          uint32_t* __restrict__ tile_counters,
                                          unsigned long long* __restrict__ gcount, const uint32_t* order) {
  __shared__ unsigned long long wt[NT / 32 + 1];
  __shared__ uint32_t skip_s[8], skew_s[8];
  const uint32_t t = threadIdx.x;
  for (int p = 0; p < P; ++p) {
    const unsigned long long c = t < 256 ? __ldcg(&ghist[p * 256 + t]) : 0ull;
    const unsigned long long ex = block_exclusive_scan<NT>(c, wt, (unsigned long long*)nullptr);
    if (t < 256) bases[p * 256 + t] = ex;
    const int trivial = __syncthreads_or(t < 256 && c == n);
    const int skewed = __syncthreads_or(t < 256 && c * 8 > n);
    if (t == 0) {
      skip_s[p] = trivial;
      skew_s[p] = skewed;
    }
  }
  __syncthreads();
  if (t == 0) {
    uint32_t alt = 0, executed = 0, first = 8, last = 8;
    for (int p = 0; p < 8; ++p) {
      const uint32_t sk = (p < P) ? skip_s[p] : 1u;
      plan->skip[p] = sk;
      plan->src_alt[p] = alt;
      if (!sk) {
        alt ^= 1u;
        ++executed;
        if (first == 8) first = p;
        last = p;
      }
    }
    plan->first = first;
    plan->last = last;
    uint32_t skew = 0;
    for (int p = 0; p < P; ++p) skew |= skew_s[p] << p;
    plan->skew = skew;
    plan->final_copy = alt;
    plan->executed = executed;
    plan->j01 = 0;  // k_plan_joint (if launched) may enable the look-back-free pass 1
    plan->run2 = 0;  // ... and pass 2 ranked by runs (pass2.cuh R2_RUN2)
    plan->fewruns = 0;  // ... and passes 2-3 of 32-bit keys ranked by runs (k_onesweep_pass_ws)
    plan->reverse = 0;
    const bool in_order = order != nullptr && __ldcg(&order[0]) == 0;
    const bool reversed = order != nullptr && !in_order && __ldcg(&order[1]) == 0;
    if (in_order || reversed) {  // presorted input: no pass; reversed input is reversed in place
      for (int p = 0; p < 8; ++p) {
        plan->skip[p] = 1;
        plan->src_alt[p] = 0;
      }
      plan->final_copy = 0;
      plan->executed = 0;
      plan->first = plan->last = 8;
      plan->reverse = reversed;
    }
  }
  if (t < 16) tile_counters[t] = 0;  // 8 passes + the J01 pass
  if (gcount != nullptr && t < 256)
    for (int p = 0; p < P; ++p) gcount[p * 256 + t] = 0;  // unstable-pass digit counters
}

static __global__ void __launch_bounds__(256)
    k_plan(unsigned long long* __restrict__ ghist, uint64_t n, int P, unsigned long long* __restrict__ bases,
           PassPlan* __restrict__ plan, uint32_t* __restrict__ tile_counters,
           unsigned long long* __restrict__ gcount, const unsigned long long* __restrict__ gjoint,
           const uint32_t* __restrict__ order = nullptr) {
  if (gjoint != nullptr) {  // marginals of digits 1 (row sums) and 0 (column sums) of J[d1][d0]
    unsigned long long r = 0, c = 0;
    const ulonglong2* row = reinterpret_cast<const ulonglong2*>(gjoint + threadIdx.x * 256);
#pragma unroll 8
    for (int a = 0; a < 128; ++a) {
      const ulonglong2 q = row[a];
      r += q.x + q.y;
    }
    uint32_t nz = 0;  // nonzero joint bins = distinct low-16-bit values (k_plan_joint's fewruns)
#pragma unroll 8
    for (int b = 0; b < 256; ++b) {
      const unsigned long long v = gjoint[b * 256 + threadIdx.x];
      c += v;
      nz += v != 0;
    }
    ghist[threadIdx.x] = c;
    ghist[256 + threadIdx.x] = r;
    __shared__ uint32_t nz_s;
    if (threadIdx.x == 0) nz_s = 0;
    __syncthreads();
    atomicAdd(&nz_s, nz);
    __syncthreads();
    if (threadIdx.x == 0) plan->pad[0] = nz_s;
  }
  plan_body<256>(ghist, n, P, bases, plan, tile_counters, gcount, order);
  // k_joint_marg counted the nonzero joint bins into order[2] (k_plan_joint's fewruns)
  if (gjoint == nullptr && order != nullptr && threadIdx.x == 0) plan->pad[0] = __ldcg(&order[2]);
}

// ---------------------------------------------------------------------------------------
// a4: one scatter pass.  Persistent CTAs (grid = resident CTAs) take tiles of THREADS*ITEMS keys
// in increasing order from an atomic counter, which gives the decoupled look-back its forward
// progress (a tile only waits on smaller tiles, all held by running CTAs).  Per tile:
//   0. BULK: the tile was prefetched into smem buffer `cur` by a 1-D TMA bulk copy
//      (cp.async.bulk, mbarrier completion) issued while the previous tile was processed.
//      !BULK (source not 16-byte aligned): coalesced per-warp loads.
//   1. keys -> registers: half-warp h of warp w owns the contiguous keys
//      [w*32*ITEMS + h*16*ITEMS, +16*ITEMS), item k of its lane l is element 16k+l of them, so
//      (warp, half, item, lane) order IS index order (order-free modes read warp-striped).
//   2. ranking (MODE):
//      RANK_STABLE: half-warp multisplit in index order.  Each half-warp keeps one smem word per
//        digit, {count so far : 16 | match mask : 16}.  Per item every lane ORs its bit into
//        its digit's word and reads the word back (its group of equal digits and the count
//        before this item, in one load); the group's highest lane stores the new count with
//        a cleared mask; rank = old count + lanes below in the group.  (MATCH.ANY, 8-ballot and
//        leader-election grouping, and separate mask/count words per warp, were measured
//        slower on sm_100: DESIGN.md §6.)
//      RANK_UNSTABLE (first LSD pass, MSD partition: the input order carries no information):
//        one shared atomicAdd per key on block counters; the tile's per-digit global offsets
//        come from one global atomicAdd per digit -- no look-back.
//      RANK_RUN2 (LSD passes p >= 1): the array is sorted by the low 8p bits L (the digits of
//        the earlier passes), so a tile holds runs of equal L in increasing order.  If the tile
//        has at most two distinct L (those of its first and last key), keys are ranked unstably
//        by (run, digit) over 512 block counters -- keys with equal (run, digit) have equal low
//        8(p+1) bits, so their order is irrelevant, and run 0 precedes run 1 within a digit:
//        exactly the stable order.  Otherwise the tile falls back to RANK_STABLE.
//      RANK_J01 (LSD pass 1 when k_plan_joint found every nonzero digit-0 bucket at least one
//        tile long): as RUN2's unstable path, but the (digit-1, digit-0) segment of every key is
//        known from the joint histogram, so each (run, digit) bin of the tile takes its global
//        offset with one atomicAdd on its segment counter -- no look-back (order inside a
//        segment is irrelevant: equal low 16 bits).
//   3. per-digit totals; look-back modes publish the tile's counts early (flag AGG; tile 0
//      publishes INC); block scan => tile offsets; keys restaged in smem in digit order (in
//      buffer `cur`; its keys now live in registers).
//   4. look-back modes: decoupled look-back => global digit offsets.
//   5. coalesced write-out of the digit-sorted tile: runs of equal digits are contiguous.
enum RankMode : int { RANK_STABLE = 0, RANK_UNSTABLE = 1, RANK_RUN2 = 2, RANK_J01 = 3 };

// Block counters of the unstable ranking are replicated BREP ways (replica = lane % BREP): lanes
// of one warp instruction that share a digit hit BREP different words, so same-address atomic
// serialization is at most 32/BREP-way (skewed digits, runs of equal keys).
constexpr int BREP = 4;  // the offset code below reads one uint4 per bin

template <int THREADS, int ITEMS, typename U, int MODE, bool KV = false>
struct PassSmem {
  static constexpr int WARPS = THREADS / 32;
  static constexpr int TILE = THREADS * ITEMS;
  // multisplit tables: per half-warp 256 words {count:16 | mask:16} (+16 words of padding so the
  // two halves of a warp start 16 banks apart); 512 x BREP block counters
  static constexpr int HALF_WORDS = 272;
  // multisplit tables only where a tile may rank stably (J01 and unstable never do)
  static constexpr int rows = (MODE == RANK_STABLE || MODE == RANK_RUN2) ? WARPS : 0;
  static constexpr size_t buf_off = 0;  // U[2][TILE]
  static constexpr size_t rows_off = align_up(buf_off + 2 * sizeof(U) * TILE, 16);
  static constexpr size_t bcnt_off = align_up(rows_off + 2 * HALF_WORDS * 4 * rows, 16);
  static constexpr size_t gofs_off = align_up(bcnt_off + sizeof(uint32_t) * 512 * BREP, 16);
  static constexpr size_t wt_off = align_up(gofs_off + sizeof(unsigned long long) * 512, 16);
  static constexpr size_t mbar_off = align_up(wt_off + sizeof(uint32_t) * (WARPS + 1), 16);
  static constexpr size_t tile_off = mbar_off + 16;  // uint32 tile id held by each buffer
  static constexpr size_t vbuf_off = align_up(tile_off + 16, 128);  // KV: uint32 values [2][TILE]
  static constexpr size_t bytes = align_up(vbuf_off + (KV ? 2 * sizeof(uint32_t) * TILE : 0), 128);
};

// Payload of a key-value sort (§8 N3): 32-bit values ping-ponged like the keys.
struct KvPtrs {
  const uint32_t* va;
  uint32_t* vb;
};


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  } while (!done);
}
// One thread: arm `bar` for `bytes` (+ `bytes2`) and start 1-D bulk copies global -> shared
// (sizes % 16 == 0, addresses 16-byte aligned).  Zero bytes just arrive.
__device__ __forceinline__ void bulk_copy(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  if (bytes)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar,
                                          void* dst2 = nullptr, const void* src2 = nullptr, uint32_t bytes2 = 0) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes + bytes2)
               : "memory");
  bulk_copy(dst_smem, src, bytes, bar);
  bulk_copy(dst2, src2, bytes2, bar);
}

template <typename U, int THREADS, int ITEMS, int MINB, bool BULK, typename DescT, typename DigitF, int MODE,
          int LBG = 8, bool KV = false>
__global__ void __launch_bounds__(THREADS, MINB)
    k_onesweep_pass(const U* a_ptr, U* b_ptr, uint64_t n, DigitF digit,
                    const unsigned long long* __restrict__ bases, DescT* __restrict__ lookback,
                    unsigned long long* __restrict__ gcount, uint32_t* __restrict__ tile_counter,
                    uint32_t num_tiles, const PassPlan* __restrict__ plan, int pass, KvPtrs kvp = {},
                    ZeroSpan zs = {}) {
  using L = PassSmem<THREADS, ITEMS, U, MODE, KV>;
  using LB = LookbackBits<DescT>;
  constexpr int TILE = L::TILE;
  constexpr int WARPS = L::WARPS;
  constexpr int SEG = 32 * ITEMS;  // keys per warp segment
  constexpr bool LOOKBACK = MODE == RANK_STABLE || MODE == RANK_RUN2;
  constexpr bool RUNS = MODE == RANK_RUN2 || MODE == RANK_J01;  // bins carry the digit-0 run
  static_assert(THREADS >= 256 && THREADS % 32 == 0, "one thread per digit");
  static_assert(TILE < (1 << 22), "rank fits 22 bits");
  static_assert((TILE * sizeof(U)) % 16 == 0, "bulk copies need 16-byte tiles");
  extern __shared__ __align__(128) unsigned char smem[];
  U* bufs = reinterpret_cast<U*>(smem + L::buf_off);
  uint32_t* rows = reinterpret_cast<uint32_t*>(smem + L::rows_off);  // [warp][half][HALF_WORDS]
  uint32_t* bcnt = reinterpret_cast<uint32_t*>(smem + L::bcnt_off);  // [512 bins][BREP]
  unsigned long long* gofs = reinterpret_cast<unsigned long long*>(smem + L::gofs_off);
  uint32_t* wt = reinterpret_cast<uint32_t*>(smem + L::wt_off);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L::mbar_off);
  uint32_t* tile_s = reinterpret_cast<uint32_t*>(smem + L::tile_off);

  const U* src = a_ptr;
  U* dst = b_ptr;
  uint32_t* vbufs = reinterpret_cast<uint32_t*>(smem + L::vbuf_off);
  const uint32_t* vsrc = kvp.va;
  uint32_t* vdst = kvp.vb;
  (void)vbufs;
  for (uint32_t i = blockIdx.x * THREADS + threadIdx.x; i < zs.n16; i += gridDim.x * THREADS)
    zs.p[i] = make_uint4(0u, 0u, 0u, 0u);
  if (plan != nullptr) {
    if (plan->skip[pass]) return;
    if constexpr (MODE == RANK_J01) {
      if (!plan->j01) return;  // the RUN2 launch of this pass runs instead
    } else if constexpr (MODE == RANK_RUN2) {
      if (pass == 1 && plan->j01) return;  // the J01 launch of this pass runs instead
    }
    if (plan->src_alt[pass]) {
      src = b_ptr;
      dst = const_cast<U*>(a_ptr);
      vsrc = kvp.vb;
      vdst = const_cast<uint32_t*>(kvp.va);
    }
  }
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t t = threadIdx.x;
  const uint32_t lt = (1u << lane) - 1u;
  constexpr int HW = L::HALF_WORDS;
  const uint32_t half = lane >> 4;
  const uint32_t l16 = lane & 15;
  const uint32_t lt16 = (1u << l16) - 1u;
  // this half-warp's table: word d = {count of digit d so far : 16 | match mask : 16}
  uint32_t* wc = rows + (2 * warp + half) * HW;
  (void)lt;

  auto tile_valid = [&](uint32_t tile) -> uint32_t {
    const uint64_t b = (uint64_t)tile * TILE;
    return (uint32_t)min64((uint64_t)TILE, n - b);
  };
  // bulk-copied prefix of a tile (keys); the rest of a ragged last tile is loaded directly
  auto bulk_keys = [&](uint32_t valid) -> uint32_t {
    return (uint32_t)((valid * sizeof(U)) & ~(size_t)15) / (uint32_t)sizeof(U);
  };
  auto bulk_vals = [&](uint32_t valid) -> uint32_t { return valid & ~3u; };
  // arm buffer b's barrier and copy tile `id` (keys, and values for KV) into it
  auto issue = [&](int b, uint32_t id) {
    const uint32_t v = tile_valid(id);
    if constexpr (KV)
      bulk_load(bufs + b * TILE, src + (uint64_t)id * TILE, bulk_keys(v) * (uint32_t)sizeof(U), &mbar[b],
                vbufs + b * TILE, vsrc + (uint64_t)id * TILE, bulk_vals(v) * 4u);
    else
      bulk_load(bufs + b * TILE, src + (uint64_t)id * TILE, bulk_keys(v) * (uint32_t)sizeof(U), &mbar[b]);
  };

  uint32_t phase0 = 0, phase1 = 0;
  if constexpr (BULK) {
    if (t == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int b = 0; b < 2; ++b) {
        const uint32_t id = atomicAdd(tile_counter, 1u);
        tile_s[b] = id;
        if (id < num_tiles) issue(b, id);
      }
    }
    __syncthreads();
  }

  for (uint32_t it = 0;; ++it) {
    const uint32_t cur = it & 1u;
    U* buf = bufs + cur * TILE;
    uint32_t tile;
    uint32_t next_id = 0;
    if constexpr (BULK) {
      tile = tile_s[cur];
      if (tile >= num_tiles) break;
      if (t == 0) next_id = atomicAdd(tile_counter, 1u);  // refill of this buffer, used at the end
    } else {
      if (t == 0) tile_s[0] = atomicAdd(tile_counter, 1u);
      __syncthreads();  // publishes the tile id; previous tile's smem is dead
      tile = tile_s[0];
      if (tile >= num_tiles) break;
    }
    const uint64_t tile_base = (uint64_t)tile * TILE;
    const uint32_t valid = tile_valid(tile);
    const bool full = valid == (uint32_t)TILE;

    // zero the counters (every read of them happened before the previous tile's last barrier)
    if constexpr (MODE == RANK_STABLE || MODE == RANK_RUN2) {  // both half tables of this warp
#pragma unroll
      for (int j = 0; j < 16; ++j) wc[l16 + 16 * j] = 0;
    }
    if constexpr (MODE != RANK_STABLE) {
      for (int j = t; j < 512 * BREP / 4; j += THREADS) reinterpret_cast<uint4*>(bcnt)[j] = make_uint4(0, 0, 0, 0);
    }

    // 1. keys -> registers
    // tile-local index of item 0.  Stable-capable modes: half-warp h of warp w owns the
    // contiguous keys [w*SEG + h*16*ITEMS, +16*ITEMS), item k of its lane l16 is element
    // 16k + l16 of them.  Order-free modes: warp-striped (conflict-free loads from the buffer).
    // full tiles of 32-bit keys-only sorts take loops without the per-item bounds test (the 64-bit
    // and key-value instantiations measured 0.4-1% slower with the duplicated loops)
    constexpr bool SPLIT_FULL = sizeof(U) == 4 && !KV;
    constexpr bool HALF_MAP = MODE == RANK_STABLE || MODE == RANK_RUN2;
    constexpr uint32_t IS = HALF_MAP ? 16u : 32u;  // index stride between items
    const uint32_t seg = HALF_MAP ? warp * SEG + half * (16 * ITEMS) + l16 : warp * SEG + lane;
    U keys[ITEMS];
    uint32_t vals[KV ? ITEMS : 1];
    uint32_t* vbuf = vbufs + cur * TILE;
    (void)vals;
    (void)vbuf;
    U first_key = U(0), last_key = U(0);
    if constexpr (BULK) {
      mbar_wait(&mbar[cur], cur ? phase1 : phase0);
      if (cur) phase1 ^= 1u; else phase0 ^= 1u;
      if (full) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) keys[k] = buf[seg + IS * k];
        if constexpr (KV) {
#pragma unroll
          for (int k = 0; k < ITEMS; ++k) vals[k] = vbuf[seg + IS * k];
        }
        if constexpr (RUNS) {
          first_key = buf[0];
          last_key = buf[TILE - 1];
        }
      } else {
        const uint32_t bk = bulk_keys(valid);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t i = seg + IS * k;
          keys[k] = i < bk ? buf[i] : (i < valid ? ldg_nc(src + tile_base + i) : U(0));
        }
        if constexpr (KV) {
          const uint32_t bv = bulk_vals(valid);
#pragma unroll
          for (int k = 0; k < ITEMS; ++k) {
            const uint32_t i = seg + IS * k;
            vals[k] = i < bv ? vbuf[i] : (i < valid ? ldg_nc(vsrc + tile_base + i) : 0u);
          }
        }
        if constexpr (RUNS) {
          first_key = bk > 0 ? buf[0] : ldg_nc(src + tile_base);
          last_key = valid - 1 < bk ? buf[valid - 1] : ldg_nc(src + tile_base + valid - 1);
        }
      }
    } else {
      if (full) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) keys[k] = ldg_nc(src + tile_base + seg + IS * k);
      } else {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          keys[k] = (seg + IS * k < valid) ? ldg_nc(src + tile_base + seg + IS * k) : U(0);
      }
      if constexpr (KV) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          vals[k] = (full || seg + IS * k < valid) ? ldg_nc(vsrc + tile_base + seg + IS * k) : 0u;
      }
      if constexpr (RUNS) {
        first_key = ldg_nc(src + tile_base);
        last_key = ldg_nc(src + tile_base + valid - 1);
      }
    }

    // Ranking strategy of this tile (block-uniform); the barrier also orders the zeroing of
    // the block counters before their first atomic.
    bool unstable_rank = MODE == RANK_UNSTABLE || MODE == RANK_J01;
    U low_first = U(0), low_last = U(0);
    if constexpr (MODE == RANK_J01) {
      digit.digit_low(first_key, &low_first);
      digit.digit_low(last_key, &low_last);
      __syncthreads();  // counters zeroed before the atomics
    } else if constexpr (MODE == RANK_RUN2) {
      U lo;
      digit.digit_low(first_key, &low_first);
      digit.digit_low(last_key, &low_last);
      bool bad = false;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        digit.digit_low(keys[k], &lo);
        bad |= (full || seg + IS * k < valid) && lo != low_first && lo != low_last;
      }
      unstable_rank = !__syncthreads_or(bad);
    } else if constexpr (MODE == RANK_UNSTABLE) {
      __syncthreads();
    }

    // 2. ranking.  info = bin | rank << 9 (bin = digit, + 256 for run 1 in RUN2).
    uint32_t info[ITEMS];
    if (unstable_rank) {
      auto rank_item = [&](int k) {
        U lo;
        uint32_t bin = digit.digit_low(keys[k], &lo);
        if constexpr (RUNS) bin |= (lo != low_first) ? 256u : 0u;
        info[k] = bin | (atomicAdd(&bcnt[bin * BREP + (lane & (BREP - 1))], 1u) << 9);
      };
      if (SPLIT_FULL && full) {  // no per-item bounds branch (a BSSY / BSYNC pair per key otherwise)
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) rank_item(k);
      } else {  // invalid tail slots are not counted at all
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          if (full || seg + IS * k < valid) rank_item(k);
          else info[k] = 0xFFFFFFFFu;
        }
      }
    } else if constexpr (MODE == RANK_STABLE || MODE == RANK_RUN2) {
      // Invalid tail slots take digit 255: they sit at the end of the tile in index order, so
      // they rank after every valid key of digit 255 and are dropped at write-out.
      __syncwarp();  // tables zeroed by this warp
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const uint32_t d = (full || seg + IS * k < valid) ? digit(keys[k]) : 255u;
        atomicOr(&wc[d], 1u << l16);
        __syncwarp();
        const uint32_t w = wc[d];  // {count before this item | this item's group}
        const uint32_t peers = w & 0xFFFFu;
        const uint32_t below = __popc(peers & lt16);
        const uint32_t old = w >> 16;
        __syncwarp();
        if ((peers >> l16) == 1u) wc[d] = (old + below + 1u) << 16;  // highest lane: count, clear mask
        info[k] = d | ((old + below) << 9);
      }
    }
    __syncthreads();  // (A) counters complete; all warps done reading buf

    // 3. per-digit totals, early publish, tile offsets
    uint32_t total = 0, c0 = 0;
    unsigned long long jg0 = 0, jg1 = 0;
    (void)c0;
    (void)jg0;
    (void)jg1;
    if (t < 256) {
      if (unstable_rank) {
        const uint4 r0 = reinterpret_cast<const uint4*>(bcnt)[t];
        c0 = r0.x + r0.y + r0.z + r0.w;
        total = c0;
        if constexpr (RUNS) {
          const uint4 r1 = reinterpret_cast<const uint4*>(bcnt)[256 + t];
          total += r1.x + r1.y + r1.z + r1.w;
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2 * WARPS; ++h) total += rows[h * HW + t] >> 16;
        if (!full && t == 255) total -= (uint32_t)TILE - valid;  // invalid tail slots
      }
      if constexpr (LOOKBACK) {
        st_relaxed(&lookback[(uint64_t)tile * 256 + t], (tile == 0 ? LB::INC : LB::AGG) | DescT(total));
      }
      if constexpr (MODE == RANK_J01) {  // allocate in the (digit, run) segments, tile order free
        const uint32_t c1 = total - c0;
        if (c0) jg0 = atomicAdd(&gcount[(uint32_t)low_first * 256 + t], (unsigned long long)c0);
        if (c1) jg1 = atomicAdd(&gcount[(uint32_t)low_last * 256 + t], (unsigned long long)c1);
      }
    }
    const uint32_t tile_excl = block_exclusive_scan<THREADS>(t < 256 ? total : 0u, wt, (uint32_t*)nullptr);
    unsigned long long gbase = 0;
    if (t < 256) {
      if (unstable_rank) {
        // replica start offsets: run 0 replicas 0..3, then run 1 replicas 0..3
        uint4 r0 = reinterpret_cast<const uint4*>(bcnt)[t];
        uint32_t run = tile_excl;
        uint4 o0;
        o0.x = run; run += r0.x;
        o0.y = run; run += r0.y;
        o0.z = run; run += r0.z;
        o0.w = run; run += r0.w;
        reinterpret_cast<uint4*>(bcnt)[t] = o0;
        if constexpr (RUNS) {
          uint4 r1 = reinterpret_cast<const uint4*>(bcnt)[256 + t];
          uint4 o1;
          o1.x = run; run += r1.x;
          o1.y = run; run += r1.y;
          o1.z = run; run += r1.z;
          o1.w = run;
          reinterpret_cast<uint4*>(bcnt)[256 + t] = o1;
        }
        if constexpr (MODE == RANK_UNSTABLE)
          if (total) gbase = atomicAdd(&gcount[t], (unsigned long long)total);  // tile order is free
      } else {
        uint32_t run = tile_excl;
#pragma unroll
        for (int h = 0; h < 2 * WARPS; ++h) {
          const uint32_t c = rows[h * HW + t] >> 16;
          rows[h * HW + t] = run;
          run += c;
        }
      }
    }
    __syncthreads();  // (B)

    if (unstable_rank) {
      auto place_item = [&](int k) {
        const uint32_t pos = bcnt[(info[k] & 0x1FFu) * BREP + (lane & (BREP - 1))] + (info[k] >> 9);
        buf[pos] = keys[k];
        if constexpr (KV) vbuf[pos] = vals[k];
      };
      if (SPLIT_FULL && full) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) place_item(k);
      } else {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          if (info[k] != 0xFFFFFFFFu) place_item(k);
      }
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const uint32_t pos = wc[info[k] & 0xFFu] + (info[k] >> 9);
        buf[pos] = keys[k];
        if constexpr (KV) vbuf[pos] = vals[k];
      }
    }

    // 4. global digit offsets
    if (t < 256) {
      if constexpr (LOOKBACK) {
        DescT excl = 0;
        if (tile > 0) {
          excl = lookback_walk<LBG>(lookback, t, tile);
          st_relaxed(&lookback[(uint64_t)tile * 256 + t], LB::INC | (excl + DescT(total)));
        }
        gofs[t] = bases[t] + (unsigned long long)excl - tile_excl;
      } else if constexpr (MODE == RANK_J01) {
        gofs[t] = bases[t] + jg0 - tile_excl;  // seg holds starts relative to digit t's base
        gofs[256 + t] = bases[t] + jg1 - (tile_excl + c0);
      } else {
        if constexpr (DigitF::REMOTE)  // byte address of element 0 of this tile's run for t
          gofs[t] = t < 256u && total ? digit.dst_base[t < (uint32_t)BSORT_DIST_MAX_RANKS ? t : 0] +
                                            (gbase - tile_excl) * sizeof(U)
                                      : 0ull;
        else
          gofs[t] = bases[t] + gbase - tile_excl;
      }
    }
    __syncthreads();  // (C)

    // 5. write-out (full tiles without the per-item bounds branch)
    auto write_item = [&](int k) {
      const uint32_t i = t + k * THREADS;
      const U x = buf[i];
      if constexpr (DigitF::REMOTE) {
        reinterpret_cast<U*>(gofs[digit(x)])[i] = x;  // st.global to the owner's buffer
      } else {
        unsigned long long o;
        if constexpr (MODE == RANK_J01) {
          U lo;
          const uint32_t d = digit.digit_low(x, &lo);
          o = gofs[d + (lo != low_first ? 256u : 0u)] + i;
        } else {
          o = gofs[digit(x)] + i;
        }
        dst[o] = x;
        if constexpr (KV) vdst[o] = vbuf[i];
      }
    };
    if (SPLIT_FULL && full) {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) write_item(k);
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k)
        if (full || t + k * THREADS < valid) write_item(k);
    }
    if constexpr (BULK) {
      __syncthreads();  // (D) buffer `cur` fully read: refill it with the tile after next
      if (t == 0) {
        tile_s[cur] = next_id;
        if (next_id < num_tiles) issue((int)cur, next_id);
      }
    }
  }
}

// Final placement when an odd number of passes executed (result sits in the scratch buffer).
template <typename U>
__global__ void __launch_bounds__(256) k_copy_back(U* __restrict__ a, const U* __restrict__ b, uint64_t n,
                                                   const PassPlan* __restrict__ plan) {
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  if (plan->reverse) {  // input was in the opposite order (no pass ran): reverse in place
    constexpr uint32_t V = 16 / sizeof(U);
    if ((uintptr_t)a % 16 == 0 && n % V == 0) {
      // 16-byte vectors: vector k and its mirror nv-1-k swap with their elements reversed
      const uint64_t nv = n / V;
      uint4* av = reinterpret_cast<uint4*>(a);
      auto rev = [](uint4 q) {
        if constexpr (sizeof(U) == 4) return make_uint4(q.w, q.z, q.y, q.x);
        else return make_uint4(q.z, q.w, q.x, q.y);
      };
      uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
      const uint64_t hv = nv / 2;
      for (; k + T < hv; k += 2 * T) {  // two swaps in flight per thread
        const uint4 x0 = av[k], y0 = av[nv - 1 - k], x1 = av[k + T], y1 = av[nv - 1 - k - T];
        av[k] = rev(y0);
        av[nv - 1 - k] = rev(x0);
        av[k + T] = rev(y1);
        av[nv - 1 - k - T] = rev(x1);
      }
      for (; k < hv; k += T) {
        const uint4 x = av[k], y = av[nv - 1 - k];
        av[k] = rev(y);
        av[nv - 1 - k] = rev(x);
      }
      if ((nv & 1) && blockIdx.x == 0 && threadIdx.x == 0) av[hv] = rev(av[hv]);  // the middle vector
      return;
    }
    const uint64_t h = n / 2;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * T < h; i += 4 * T) {  // four independent swaps in flight per thread
      U x[4], y[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x[k] = a[i + k * T];
        y[k] = a[n - 1 - (i + k * T)];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a[i + k * T] = y[k];
        a[n - 1 - (i + k * T)] = x[k];
      }
    }
    for (; i < h; i += T) {
      const U x = a[i], y = a[n - 1 - i];
      a[i] = y;
      a[n - 1 - i] = x;
    }
    return;
  }
  if (!plan->final_copy) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) a[i] = b[i];
}

}  // namespace bsort
