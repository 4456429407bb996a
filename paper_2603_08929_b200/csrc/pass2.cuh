// pass2.cuh — a4 (round 2): the LSD scatter pass ranked by lane-ordered shared atomics.
//
// Paper mapping as in onesweep.cuh: one pass = a stable 256-way split of the transformed key on
// one 8-bit digit (Algorithm 1's one-bit split of P:141-160, widened to a digit; LSD order needs
// every pass after the first to be stable).
//
// What is new against k_onesweep_pass / k_onesweep_pass_ws (round 1):
//  * Stable ranking costs one shared atomic per key.  A warp keeps one counter per digit; its
//    keys are read item-major (index = warp segment + 32 * item + lane) and ranked with
//    atomicAdd(&cnt[warp][digit], 4).  Items of one warp are ordered by program order, and lanes
//    of ONE atomic instruction that hit the same word receive their old values in ascending
//    lane order on sm_100 (measured: tools/exp/atoms_order.cu, 0 violations in >10^9 same-word
//    lane pairs, random / skewed / divergent patterns; selftest.cu re-checks it once per device
//    on first use, and where it fails the library launches the round-1 kernels instead).  So the returned value
//    IS the stable rank inside the warp; a per-digit scan over warps gives the tile rank.  The
//    round-1 half-warp multisplit needed three shared accesses per key.
//  * Chunked look-back.  Pass p+1's input is sorted by digit p, so it splits into NC = 32
//    contiguous chunks by the top 5 bits of digit p, and the global start of (chunk c, digit d)
//    is base[d] + sum_{c' < c} J[c'][d], where J = the coarse joint histogram of (digit p >> 3,
//    digit p+1) counted by the histogram kernel.  Tiles are laid inside chunks and dispatched
//    round-robin over chunks, so every decoupled look-back chain (one per chunk) only has to
//    advance at 1/32 of the tile rate: round 1's single chain (one L2 round trip per 8 tiles)
//    bounded a look-back pass at ~3.6 ms per 2^30 keys whatever the ranking cost.
//  * Unstable passes (LSD pass 0) count with lane-banked counters (bank = lane: conflict-free);
//    the atomic's return value is the key's rank within (digit, lane), and a scan over lanes and
//    digits turns the table into staging offsets, so placing a key costs one conflict-free load
//    instead of a second, conflicting atomic.  Consecutive tiles use the two u16 halves of the
//    table's words (the scan of one tile zeroes the other half for the next).
//  * Keys stay ENCODED (a1's order-preserving transform) between passes: the first executed
//    pass encodes as it loads, the last one decodes as it writes (PassPlan::first / last), so
//    the passes in between extract digits with one shift.
//  * Separate TMA input buffers (2) and staging buffers (2): an input buffer is re-armed as soon
//    as its keys are in registers, so the TMA prefetch never waits for a write-out or a walk.
//  * Counters count in units of 4 (bytes of a 4-byte key): placing a key is load + add + store.
//    Offsets are 32-bit (n < 2^32).  Full tiles take a path without bounds checks; staging
//    addresses are computed for all of a thread's keys before the first store.
//
// Structure (one persistent CTA per SM): RT ranker threads + WT writer threads.  Rankers: wait
// for the tile, rank, publish the tile's per-digit counts (-> writers start the look-back),
// scan, stage the keys in digit order, hand the tile over and go on.  Writers: take the tile's
// global digit offsets (look-back walk / global atomics), write the staged tile out coalesced.
#pragma once
#include <type_traits>

#include "onesweep_ws.cuh"

namespace bsort {

enum Rank2 : int { R2_STABLE = 0, R2_UNSTABLE = 1, R2_J01 = 2, R2_RUN2 = 3 };
// ranking by (digit, run of the lower bits) in lane-banked tables: J01 and RUN2
constexpr bool p2_runs(int mode) { return mode == R2_J01 || mode == R2_RUN2; }
constexpr int P2_NC = 32;  // look-back chains (chunks) of a chunked stable pass
#ifndef P2_SCAN1
#define P2_SCAN1 1  // stable passes: one-barrier digit scan (scan256_1bar)
#endif

// Chunk map of a stable pass (device arrays written by the plan kernel).
struct ChunkMap {
  const uint32_t* disp;              // dispatch order: disp[t] = chunk << 24 | tile within chunk
                                     // (nullptr: round-robin over the nc chunks, computed on the fly)
  const unsigned long long* cstart;  // [nc + 1] chunk starts (keys)
  const uint32_t* ctile;             // [nc + 1] linear id of each chunk's first tile
  const uint32_t* jp;                // [nc][256] global start of (chunk, digit)
  uint32_t nc;                       // chunks (<= P2_NC; disp == nullptr needs nc <= 8)
};

// Round-robin dispatch without a table: tiles are handed out k-major (tile k of every chunk that
// has one, in chunk order, then tile k + 1 ...).  Between consecutive distinct chunk tile counts
// the set of chunks still dispatching is fixed, so dispatch ids split into at most nc segments of
// slope m (the number of such chunks): ChunkRR holds them, built once per CTA by one thread.
struct ChunkRR {
  unsigned long long cstart[9];  // the map's chunk starts and first tiles (shared-memory copies)
  uint32_t ctile[9];
  uint32_t kstart[8], idstart[9], m[8], nseg;
  uint8_t act[8][8];             // chunks still dispatching in segment j, in chunk order
};
__device__ __forceinline__ void chunk_rr_build(const ChunkMap& cm, ChunkRR* r) {
  uint32_t nt[8];
  for (uint32_t c = 0; c <= cm.nc && c < 9; ++c) {
    r->cstart[c] = cm.cstart[c];
    r->ctile[c] = cm.ctile[c];
  }
  for (uint32_t c = 0; c < 8; ++c) nt[c] = c < cm.nc ? r->ctile[c + 1] - r->ctile[c] : 0u;
  uint32_t k0 = 0, id0 = 0, j = 0;
  for (; j < 8; ++j) {
    uint32_t m = 0, next = 0xFFFFFFFFu;
    for (uint32_t c = 0; c < 8; ++c)
      if (nt[c] > k0) {
        r->act[j][m++] = (uint8_t)c;
        next = min(next, nt[c]);
      }
    if (m == 0) break;
    r->kstart[j] = k0;
    r->idstart[j] = id0;
    r->m[j] = m;
    id0 += (next - k0) * m;
    k0 = next;
  }
  r->idstart[j] = id0;
  r->nseg = j;
}
// false past the last tile
__device__ __forceinline__ bool chunk_rr(const ChunkRR* r, uint32_t id, uint32_t& chunk, uint32_t& k) {
  const uint32_t ns = r->nseg;
  uint32_t j = 0;
  while (j < ns && id >= r->idstart[j + 1]) ++j;
  if (j >= ns) return false;
  const uint32_t off = id - r->idstart[j], m = r->m[j];
  k = r->kstart[j] + off / m;
  chunk = r->act[j][off % m];
  return true;
}

// Vectorised look-back descriptors (u32 = {2-bit flag | 30-bit count}, LookbackBits<uint32_t>):
// (linear tile q, digit d) lives at lb[((q >> 2) * 256 + d) * 4 + (q & 3)].
__host__ __device__ __forceinline__ uint64_t lb2_index(uint64_t q, uint32_t d) {
  return ((q >> 2) * 256 + d) * 4 + (q & 3);
}
__device__ __forceinline__ uint4 ld_relaxed_v4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
// shared-window accesses by 32-bit address (volatile: kept in program order)
__device__ __forceinline__ uint32_t s_atom_add(uint32_t a, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t s_ld(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
  return r;
}
template <typename U>
__device__ __forceinline__ U s_ldk(uint32_t a) {
  if constexpr (sizeof(U) == 4) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return U(r);
  } else {
    unsigned long long r;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(r) : "r"(a));
    return U(r);
  }
}
template <typename U>
__device__ __forceinline__ void s_st(uint32_t a, U v) {
  if constexpr (sizeof(U) == 4)
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"((uint32_t)v) : "memory");
  else
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"((unsigned long long)v) : "memory");
}
// st.global of v at base + o * sizeof(U) + IMM bytes (one mad.wide for the address)
template <int IMM, typename U>
__device__ __forceinline__ void st_global_at(const U* base, uint32_t o, U v) {
  unsigned long long a;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(o), "n"((int)sizeof(U)), "l"(base));
  if constexpr (sizeof(U) == 4)
    asm volatile("st.global.b32 [%0+%1], %2;" ::"l"(a), "n"(IMM), "r"((uint32_t)v) : "memory");
  else
    asm volatile("st.global.b64 [%0+%1], %2;" ::"l"(a), "n"(IMM), "l"((unsigned long long)v) : "memory");
}
// f(integral_constant<int, I>) for I = 0 .. N-1 (compile-time indices for immediates)
template <int N, int I = 0, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, I + 1>(f);
  }
}
// Staging-buffer swizzle of the unstable passes: key p lives at p ^ (row(p) mod keys-per-row),
// a permutation inside every 128-byte row.  The unstable ranking gives each (digit, lane) pair a
// sub-run; when a tile holds few digits those sub-runs have equal lengths and the 32 lanes of a
// store would hit one bank.  Rows read back whole stay conflict-free.
template <typename U>
__device__ __forceinline__ uint32_t p2_swz(uint32_t p) {
  constexpr uint32_t KPR = 128 / sizeof(U);
  return p ^ ((p / KPR) & (KPR - 1));
}
template <int SHIFT, typename U>
__device__ __forceinline__ uint32_t p2_digit(U k) {
  if constexpr (SHIFT >= 32)
    return uint32_t(uint64_t(k) >> SHIFT) & 0xFFu;
  else
    return (uint32_t(k) >> SHIFT) & 0xFFu;
}

// Exclusive scan over the first 256 threads of a named-barrier group of NT threads (the others
// pass 0): ONE barrier -- every warp adds the totals of the warps before it itself (at most 7
// broadcast loads) instead of waiting for warp 0 to scan them behind a second barrier.  The
// totals array is rewritten only after the group's next barriers.
template <int NT, uint32_t BAR>
__device__ __forceinline__ uint32_t scan256_1bar(uint32_t v, uint32_t* warp_tot) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t inc = warp_inclusive_scan(v);
  if (lane == 31 && warp < 8) warp_tot[warp] = inc;
  named_bar_sync(BAR, NT);
  uint32_t base = 0;
  if (warp < 8)
    for (uint32_t w = 0; w < warp; ++w) base += warp_tot[w];
  return base + inc - v;
}

// Exclusive prefix of linear tile T for digit d: fold predecessors T-1, T-2, ... (aggregates)
// until an inclusive prefix; LBV vector loads (4 tiles each) per L2 round trip.  The first tile
// of every chain publishes an inclusive prefix, so the walk ends there at the latest.
template <int LBV>
__device__ __forceinline__ uint32_t lookback_walk_v4(const uint32_t* lb, uint32_t d, uint32_t T) {
  using LB = LookbackBits<uint32_t>;
  uint32_t excl = 0;
  int64_t j = (int64_t)T - 1;  // highest tile not folded yet
  for (;;) {
    const int64_t g0 = j >> 2;
    uint4 v[LBV];
#pragma unroll
    for (int i = 0; i < LBV; ++i)
      v[i] = (g0 - i >= 0) ? ld_relaxed_v4(lb + ((uint64_t)(g0 - i) * 256 + d) * 4) : make_uint4(0, 0, 0, 0);
    bool stop = false, fin = false;
    int64_t next = (g0 - LBV + 1) * 4 - 1;
#pragma unroll
    for (int i = 0; i < LBV; ++i) {
      const uint32_t e[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
      for (int k = 3; k >= 0; --k) {
        const int64_t q = (g0 - i) * 4 + k;
        if (!stop && q <= j) {
          const uint32_t f = e[k] >> LB::SH;
          if (f == 0) {
            stop = true;  // not published yet: poll again from q
            next = q;
          } else {
            excl += e[k] & LB::VAL;
            if (f == 2) stop = fin = true;
          }
        }
      }
    }
    if (fin) return excl;
    if (stop) __nanosleep(128);  // a predecessor has not published yet: do not hammer L2
    j = next;
  }
}

// What a tile is (written by the refill thread before its TMA copy is armed; copied to the
// staging slot for the writers).
struct SlotInfo {
  uint32_t lin;    // linear tile id (P2_END: no more tiles)
  uint32_t len;    // keys in the tile
  uint32_t off;    // input-buffer key of the tile's first key (< 16 bytes in)
  uint32_t bk;     // tile keys covered by the bulk copy (the rest: ld.global)
  uint32_t chunk;  // chunked pass: chunk of the tile
  uint32_t first;  // first tile of its look-back chain
  unsigned long long start;  // first key (index into the source array)
};
static_assert(sizeof(SlotInfo) == 32, "slot layout");
constexpr uint32_t P2_END = 0xFFFFFFFFu;

template <int RT, int WT, int ITEMS, typename U, int MODE, int HALVES = 1>
struct Pass2Smem {
  static constexpr int RW = RT / 32;
  static constexpr int TILE = RT * ITEMS;
  static constexpr int KPV = 16 / (int)sizeof(U);  // keys per 16-byte vector
  static constexpr int IBUFK = TILE + KPV;         // a tile starts at input-buffer key < KPV
  // STABLE: per-warp counters [RW][256]; UNSTABLE: lane-banked table [256 digits][32 lanes];
  // J01: lane-banked counts [256][32] of (run 0 | run 1 << 16) and the staging offsets, same shape
  static constexpr int NG = MODE == R2_J01 ? 512 : 256;  // write-out bins (J01: 2 * digit + run)
  // STABLE with HALVES = 2: one row per half-warp, rows 272 words apart (the halves' counters of
  // one digit sit 16 banks apart), for skewed digits
  static constexpr int HW = HALVES == 2 ? 272 : 256;
  static constexpr int CNT_WORDS = MODE == R2_STABLE ? RW * HALVES * HW : (p2_runs(MODE) ? 2 : 1) * 256 * 32;
  static constexpr size_t ibuf_off = 0;  // U[2][IBUFK] TMA input
  static constexpr size_t sbuf_off = align_up(ibuf_off + 2 * sizeof(U) * IBUFK, 16);  // U[2][TILE] staging
  static constexpr size_t cnt_off = align_up(sbuf_off + 2 * sizeof(U) * TILE, 16);
  static constexpr size_t meta_off = align_up(cnt_off + 4 * (size_t)CNT_WORDS, 16);  // uint4[2][256]
  static constexpr size_t gofs_off = align_up(meta_off + 16 * 2 * 256, 16);   // u32[2][NG]
  static constexpr size_t wt_off = align_up(gofs_off + 4 * 2 * NG, 16);       // u32[RW + 1]
  static constexpr size_t mbar_off = align_up(wt_off + 4 * (RW + 1), 16);     // u64[2]
  static constexpr size_t islot_off = mbar_off + 16;                          // SlotInfo[2] input
  static constexpr size_t sslot_off = islot_off + 64;                         // SlotInfo[2] staged
  static constexpr size_t rr_off = sslot_off + 64;  // ChunkRR (round-robin chunk dispatch)
  static constexpr size_t bytes = align_up(rr_off + sizeof(ChunkRR), 128);
};

// named barriers: 0 = __syncthreads; R = rankers; W = writers; per staging slot s:
// COUNTED + s (tile counts published), STAGED + s (tile staged), SFREE + s (slot written out)
constexpr uint32_t P2_BAR_R = 1, P2_BAR_W = 2, P2_BAR_COUNTED = 3, P2_BAR_STAGED = 5, P2_BAR_SFREE = 7;
// flags (used when plan == nullptr): encode keys on load / decode on write-out
constexpr uint32_t P2_ENC = 1, P2_DEC = 2;
// P2_RAW: keys are raw (not encoded) in both buffers whatever the plan says -- the pass encodes as
// it loads and decodes as it writes (passes of round-1 kernels run before / after it)
constexpr uint32_t P2_RAW = 4;
// P2_SKEWVAR: one of a pair of STABLE launches for the same pass; the HALVES = 2 kernel works when
// the plan marks the pass's digit skewed, the HALVES = 1 kernel otherwise
constexpr uint32_t P2_SKEWVAR = 8;
// P2_FEWALT: a run-ranking launch (k_onesweep_pass_ws, only_fewruns) follows for the same pass; this
// launch does no work when the plan marks the pass's input as having few distinct lower bits
constexpr uint32_t P2_FEWALT = 16;

// MODE R2_STABLE: look-back pass; with CHUNKED the chains of `cm`, else one chain over tiles of
//   TILE keys (gcount unused).
// MODE R2_UNSTABLE: tile offsets from one global atomicAdd per digit on gcount[256].
// MODE R2_J01 (LSD pass 1 when every nonzero digit-0 bucket is at least a tile long, so a tile
//   meets at most two digit-0 runs): keys ranked unstably by (digit, run) -- equal (digit, run)
//   means equal low 16 bits, whose order is irrelevant -- and each bin's global offset is one
//   atomicAdd on its (digit 1, digit 0) segment counter gcount[d0 * 256 + d1] seeded by
//   k_plan_joint: no look-back.  The plan's j01 flag picks this launch or the R2_STABLE one.
// MODE R2_RUN2 (LSD pass p >= 2 when every nonzero joint bin of the digits below is at least a
//   tile long: a tile meets at most two runs of equal lower bits L): ranked unstably by (digit,
//   run) as J01 -- keys with equal digit and equal L are interchangeable, run 0 precedes run 1 --
//   with R2_STABLE's look-back for the order between tiles.  The plan's run2 flag picks this
//   launch or the R2_STABLE one.
// Keys: digit SHIFT/8 of the encoded key; n < 2^32 (32-bit offsets), n <= 2^30 for R2_STABLE
// (30-bit look-back counts).
template <typename U, int KIND, bool DESC, int SHIFT, int RT, int WT, int ITEMS, int MODE, bool CHUNKED = false,
          int LBV = 2, int HALVES = 1, int MINB = 1>
__global__ void __launch_bounds__(RT + WT, MINB)
    k_pass2(const U* a_ptr, U* b_ptr, uint64_t n, const unsigned long long* __restrict__ bases,
            uint32_t* __restrict__ lookback, unsigned long long* __restrict__ gcount,
            uint32_t* __restrict__ tile_counter, uint32_t num_tiles, const PassPlan* __restrict__ plan, int pass,
            uint32_t flags, ChunkMap cm) {
  using L = Pass2Smem<RT, WT, ITEMS, U, MODE, HALVES>;
  using LB = LookbackBits<uint32_t>;
  constexpr int TILE = L::TILE;
  constexpr int RW = L::RW;
  constexpr int NROW = RW * HALVES;  // STABLE counter rows, in index order
  constexpr int HW = L::HW;
  static_assert(HALVES == 1 || (MODE == R2_STABLE && ITEMS % 2 == 1), "half-warp rows: stable, odd ITEMS");
  constexpr int SEG = 32 * ITEMS;
  constexpr uint32_t KS = sizeof(U) == 4 ? 2 : 3;  // log2 key bytes
  static_assert(RT >= 256 && RT % 32 == 0 && WT >= 256 && WT % 32 == 0, "one ranker / writer per digit");
  static_assert(MODE == R2_STABLE || TILE * sizeof(U) < (1 << 16), "staging offsets fit u16");
  static_assert((TILE * sizeof(U)) % 16 == 0 && L::bytes < (1 << 18) && L::bytes <= 227 * 1024,
                "16-byte tiles; addresses fit 18 bits; fits shared memory");
  static_assert(!CHUNKED || MODE == R2_STABLE || MODE == R2_RUN2, "chunks are look-back chains");
  extern __shared__ __align__(128) unsigned char smem[];
  U* ibufs = reinterpret_cast<U*>(smem + L::ibuf_off);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L::cnt_off);
  uint4* meta = reinterpret_cast<uint4*>(smem + L::meta_off);
  uint32_t* gofs = reinterpret_cast<uint32_t*>(smem + L::gofs_off);
  uint32_t* wt = reinterpret_cast<uint32_t*>(smem + L::wt_off);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L::mbar_off);
  volatile SlotInfo* islot = reinterpret_cast<volatile SlotInfo*>(smem + L::islot_off);
  volatile SlotInfo* sslot = reinterpret_cast<volatile SlotInfo*>(smem + L::sslot_off);
  ChunkRR* rr = reinterpret_cast<ChunkRR*>(smem + L::rr_off);  // thread 0 only
  const uint32_t smem_base = smem_u32(smem);

  const U* src = a_ptr;
  U* dst = b_ptr;
  bool enc_in = (flags & P2_ENC) != 0, dec_out = (flags & P2_DEC) != 0;
  if (plan != nullptr) {
    if (plan->skip[pass]) return;
    if constexpr (MODE == R2_J01) {
      if (!plan->j01) return;
    } else if constexpr (MODE == R2_RUN2) {
      if (!plan->run2) return;
    } else if constexpr (MODE == R2_STABLE) {
      if (pass == 1 && plan->j01) return;
      if (pass == 2 && plan->run2) return;
      if (flags & P2_SKEWVAR)
        if ((((plan->skew >> pass) & 1u) != 0) != (HALVES == 2)) return;
      if ((flags & P2_FEWALT) && ((plan->fewruns >> pass) & 1u)) return;
    }
    if (plan->src_alt[pass]) {
      src = b_ptr;
      dst = const_cast<U*>(a_ptr);
    }
    if (!(flags & P2_RAW)) {
      enc_in = plan->first == (uint32_t)pass;
      dec_out = plan->last == (uint32_t)pass;
    }
  }
  const uint32_t t = threadIdx.x;
  // one thread: give input buffer b the next tile (geometry in islot[b]), or mark the end
  auto refill = [&](int b) {
    const uint32_t id = atomicAdd(tile_counter, 1u);
    if (id >= num_tiles) {
      islot[b].lin = P2_END;
      mbar_arrive(&mbar[b]);
      return;
    }
    uint32_t lin, len, chunk = 0, first;
    unsigned long long start;
    if constexpr (CHUNKED) {
      uint32_t k = 0;
      unsigned long long cs, ce;
      if (cm.disp != nullptr) {
        const uint32_t v = cm.disp[id];
        chunk = v >> 24;
        k = v & 0xFFFFFFu;
        cs = cm.cstart[chunk];
        ce = cm.cstart[chunk + 1];
        lin = cm.ctile[chunk] + k;
      } else {
        if (!chunk_rr(rr, id, chunk, k)) {
          islot[b].lin = P2_END;
          mbar_arrive(&mbar[b]);
          return;
        }
        cs = rr->cstart[chunk];
        ce = rr->cstart[chunk + 1];
        lin = rr->ctile[chunk] + k;
      }
      start = cs + (unsigned long long)k * TILE;
      len = (uint32_t)min64((uint64_t)TILE, ce - start);
      first = k == 0;
    } else {
      lin = id;
      start = (unsigned long long)id * TILE;
      len = (uint32_t)min64((uint64_t)TILE, n - start);
      first = id == 0;
    }
    // bulk-copy the 16-byte-aligned span around [start, start + len) (at the end of the array:
    // inside it); the tile begins `off` keys into the buffer, keys the span misses are read
    // with ld.global
    const uintptr_t s0 = (uintptr_t)(src + start), s1 = (uintptr_t)(src + start + len);
    const uintptr_t a0 = s0 & ~(uintptr_t)15;
    const uintptr_t a1 = start + len == n ? s1 & ~(uintptr_t)15 : (s1 + 15) & ~(uintptr_t)15;
    islot[b].lin = lin;
    islot[b].len = len;
    islot[b].off = (uint32_t)((s0 - a0) / sizeof(U));
    islot[b].bk = a1 > s0 ? (uint32_t)min64(len, (a1 - s0) / sizeof(U)) : 0u;
    islot[b].chunk = chunk;
    islot[b].first = first;
    islot[b].start = start;
    bulk_load(ibufs + b * L::IBUFK, reinterpret_cast<const void*>(a0), a1 > a0 ? (uint32_t)(a1 - a0) : 0u,
              &mbar[b]);
  };
  if (t == 0) {
    if constexpr (CHUNKED) {
      if (cm.disp == nullptr) chunk_rr_build(cm, rr);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&mbar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < 2; ++b) refill(b);
  }
  if constexpr (MODE != R2_STABLE) {
    for (int i = t; i < L::CNT_WORDS / 4; i += RT + WT) reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  constexpr uint32_t OFS = p2_runs(MODE) ? 256 * 32 : 0;  // J01 / RUN2: offsets table after the counts
  constexpr uint32_t LOWMASK = SHIFT >= 32 ? 0xFFFFFFFFu : (1u << SHIFT) - 1u;  // bits below the digit

  if (t < (uint32_t)RT) {
    // ---------------------------------------------------------------- rankers
    const uint32_t lane = t & 31, warp = t >> 5;
    // STABLE: this thread's counter row (warp, or half-warp when HALVES == 2); item k of the thread
    // is tile key seg + IS * k, so (row, item, lane in row) is index order
    const uint32_t half = HALVES == 2 ? lane >> 4 : 0u;
    constexpr uint32_t IS = HALVES == 2 ? 16u : 32u;
    const uint32_t wcnt_a = smem_base + (uint32_t)L::cnt_off + (warp * HALVES + half) * (uint32_t)(HW * 4);
    const uint32_t lane_a = smem_base + (uint32_t)L::cnt_off + lane * 4u;     // UNSTABLE: lane column
    const uint32_t seg = HALVES == 2 ? warp * SEG + half * (16 * ITEMS) + (lane & 15) : warp * SEG + lane;
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it & 1u;  // input buffer and staging slot
      if (it >= 2) named_bar_sync(P2_BAR_SFREE + s, RT + WT);  // writers done with tile it - 2
      if constexpr (MODE == R2_STABLE) {
        // this warp's previous staging (the only reader of its row after the scan) is done
        uint4* w4 = reinterpret_cast<uint4*>(cnt + warp * HALVES * HW);
#pragma unroll
        for (int j = 0; j < (HALVES * HW / 4 + 31) / 32; ++j)
          if (lane + 32 * j < (uint32_t)(HALVES * HW / 4)) w4[lane + 32 * j] = make_uint4(0, 0, 0, 0);
      }
      mbar_wait(&mbar[s], (it >> 1) & 1u);
      const uint32_t lin = islot[s].lin;
      if (lin == P2_END) {
        if (t == 0) sslot[s].lin = P2_END;
        named_bar_arrive(P2_BAR_COUNTED + s, RT + WT);
        break;
      }
      const uint32_t valid = islot[s].len;
      const bool first_tile = islot[s].first != 0;
      const uint32_t ibuf_a = smem_base + (uint32_t)L::ibuf_off + s * (uint32_t)(L::IBUFK * sizeof(U)) +
                              islot[s].off * (uint32_t)sizeof(U);
      const uint32_t sbuf_a = smem_base + (uint32_t)L::sbuf_off + s * (uint32_t)(TILE * sizeof(U));
      const uint32_t hsh = (it & 1u) << 4;  // UNSTABLE: this tile's half of the table words
      if (t == 0) {
        sslot[s].lin = lin;
        sslot[s].len = valid;
        sslot[s].chunk = islot[s].chunk;
        sslot[s].first = islot[s].first;
      }

      auto tile_body = [&](auto full_c) {
        constexpr bool FULL = decltype(full_c)::value;
        // keys -> registers (encoded); rk = ranks (x4) of items 2j, 2j + 1 as u16 halves (the
        // counter address is recomputed from the key when staging: fewer live registers)
        U keys[ITEMS];
        uint32_t rk[(ITEMS + 1) / 2];
#pragma unroll
        for (int j = 0; j < (ITEMS + 1) / 2; ++j) rk[j] = 0;
        if constexpr (FULL) {
#pragma unroll
          for (int k = 0; k < ITEMS; ++k) keys[k] = s_ldk<U>(ibuf_a + (seg + IS * k) * (uint32_t)sizeof(U));
        } else {
          const uint32_t bk = islot[s].bk;
          const U* gsrc = src + islot[s].start;
#pragma unroll
          for (int k = 0; k < ITEMS; ++k) {
            const uint32_t i = seg + IS * k;
            keys[k] = i < bk ? s_ldk<U>(ibuf_a + i * (uint32_t)sizeof(U)) : (i < valid ? ldg_nc(gsrc + i) : U(0));
          }
        }
        if (enc_in) {
#pragma unroll
          for (int k = 0; k < ITEMS; ++k) keys[k] = key_encode<KIND, DESC>(keys[k]);
        }
        uint32_t lf = 0;  // J01 / RUN2: lower bits of the tile's first key (run 0)
        if constexpr (p2_runs(MODE)) {
          const uint32_t bk = islot[s].bk;
          const U* gsrc = src + islot[s].start;
          U fk = bk > 0 ? s_ldk<U>(ibuf_a) : ldg_nc(gsrc);
          U lk = valid - 1 < bk ? s_ldk<U>(ibuf_a + (valid - 1) * (uint32_t)sizeof(U)) : ldg_nc(gsrc + valid - 1);
          if (enc_in) {
            fk = key_encode<KIND, DESC>(fk);
            lk = key_encode<KIND, DESC>(lk);
          }
          lf = uint32_t(fk) & LOWMASK;
          if (t == 0) {
            meta[s * 256 + 254].w = lf;
            meta[s * 256 + 255].w = uint32_t(lk) & LOWMASK;
          }
        }
        auto run_of = [&](U key) -> uint32_t { return (uint32_t(key) & LOWMASK) != lf ? 1u : 0u; };
        (void)run_of;
        if constexpr (MODE == R2_STABLE) __syncwarp();  // row zeroed
        // counter of key k: STABLE this warp's digit counter; UNSTABLE (digit, lane), bank = lane
        auto counter = [&](U key) -> uint32_t {
          const uint32_t d = p2_digit<SHIFT>(key);
          if constexpr (MODE == R2_STABLE)
            return wcnt_a + d * 4u;
          else
            return lane_a + d * 128u;
        };
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          if (FULL || seg + IS * k < valid) {
            uint32_t r;
            if constexpr (MODE == R2_STABLE) {
              r = s_atom_add(counter(keys[k]), 4u);
            } else if constexpr (MODE == R2_UNSTABLE) {
              r = (s_atom_add(counter(keys[k]), 4u << hsh) >> hsh) & 0xFFFFu;
            } else {  // J01 / RUN2
              const uint32_t sh = run_of(keys[k]) << 4;
              r = (s_atom_add(counter(keys[k]), 4u << sh) >> sh) & 0xFFFFu;
            }
            rk[k >> 1] |= r << ((k & 1) * 16);
          }
        }
        named_bar_sync(P2_BAR_R, RT);  // (A) counts complete; the input buffer is read
        if (t == 0) refill((int)s);    // tile it + 2

        if constexpr (MODE == R2_STABLE) {
          uint32_t tot = 0;
          if (t < 256) {
#pragma unroll
            for (int w = 0; w < NROW; ++w) tot += cnt[w * HW + t];
            tot >>= 2;
            st_relaxed(&lookback[lb2_index(lin, t)], (first_tile ? LB::INC : LB::AGG) | tot);
            meta[s * 256 + t].y = tot;
          }
          named_bar_arrive(P2_BAR_COUNTED + s, RT + WT);  // writers may start the look-back
          const uint32_t excl = P2_SCAN1 ? scan256_1bar<RT, P2_BAR_R>(t < 256 ? tot : 0u, wt)
                                         : group_exclusive_scan<RT, P2_BAR_R>(t < 256 ? tot : 0u, wt);
          if (t < 256) {
            uint32_t run = sbuf_a + (excl << KS);
#pragma unroll
            for (int w = 0; w < NROW; ++w) {
              const uint32_t c = cnt[w * HW + t];
              cnt[w * HW + t] = run;
              run += c << (KS - 2);
            }
            meta[s * 256 + t].x = excl;
          }
        } else if constexpr (p2_runs(MODE)) {
          // as UNSTABLE below, with both u16 halves (runs 0 / 1) of every word counted, the
          // offsets written to the second table and the counts zeroed
          const uint32_t qr = t & 7u;
          uint4* row = reinterpret_cast<uint4*>(cnt + (t & 255u) * 32);
          uint4* orow = reinterpret_cast<uint4*>(cnt + OFS + (t & 255u) * 32);
          uint32_t tot = 0, upper = 0;  // packed run 0 | run 1 << 16, units of 4
          if (t < 256) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t q = (uint32_t)(i + qr) & 7u;
              if (q == 0) upper = tot;
              const uint4 v = row[q];
              tot += v.x + v.y + v.z + v.w;
            }
            if (qr == 0) upper = tot;
          }
          const uint32_t t0 = (tot & 0xFFFFu) >> 2, t1 = tot >> 18;
          if (t < 256) {
            if constexpr (MODE == R2_RUN2)
              st_relaxed(&lookback[lb2_index(lin, t)], (first_tile ? LB::INC : LB::AGG) | (t0 + t1));
            meta[s * 256 + t].y = t0 + t1;
            meta[s * 256 + t].z = t0;
          }
          named_bar_arrive(P2_BAR_COUNTED + s, RT + WT);  // writers may take the global offsets
          const uint32_t excl = group_exclusive_scan<RT, P2_BAR_R>(t < 256 ? t0 + t1 : 0u, wt);
          if (t < 256) {
            meta[s * 256 + t].x = excl;
            const uint32_t e0 = excl << KS, e1 = (excl + t0) << KS;
            uint32_t r0 = e0 + (((tot & 0xFFFFu) - (upper & 0xFFFFu)) << (KS - 2));
            uint32_t r1 = e1 + (((tot >> 16) - (upper >> 16)) << (KS - 2));
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t q = (uint32_t)(i + qr) & 7u;
              if (q == 0) {
                r0 = e0;
                r1 = e1;
              }
              const uint4 v = row[q];
              uint4 o;
              o.x = r0 | (r1 << 16); r0 += (v.x & 0xFFFFu) << (KS - 2); r1 += (v.x >> 16) << (KS - 2);
              o.y = r0 | (r1 << 16); r0 += (v.y & 0xFFFFu) << (KS - 2); r1 += (v.y >> 16) << (KS - 2);
              o.z = r0 | (r1 << 16); r0 += (v.z & 0xFFFFu) << (KS - 2); r1 += (v.z >> 16) << (KS - 2);
              o.w = r0 | (r1 << 16); r0 += (v.w & 0xFFFFu) << (KS - 2); r1 += (v.w >> 16) << (KS - 2);
              orow[q] = o;
              row[q] = make_uint4(0, 0, 0, 0);
            }
          }
        } else {
          // pass 1 over digit t's row (this tile's u16 halves), one 16-byte quad of lanes at a
          // time, quads visited from qr = t & 7 on (conflict-free): totals and the sum over
          // quads >= qr (units of 4)
          const uint32_t qr = t & 7u;
          uint4* row = reinterpret_cast<uint4*>(cnt + (t & 255u) * 32);
          uint32_t tot = 0, upper = 0;
          if (t < 256) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t q = (uint32_t)(i + qr) & 7u;
              if (q == 0) upper = tot;  // quads qr..7 summed
              const uint4 v = row[q];
              tot += ((v.x >> hsh) & 0xFFFFu) + ((v.y >> hsh) & 0xFFFFu) + ((v.z >> hsh) & 0xFFFFu) +
                     ((v.w >> hsh) & 0xFFFFu);
            }
            if (qr == 0) upper = tot;
            meta[s * 256 + t].y = tot >> 2;
          }
          named_bar_arrive(P2_BAR_COUNTED + s, RT + WT);  // writers may take the global offsets
          const uint32_t excl = group_exclusive_scan<RT, P2_BAR_R>(t < 256 ? tot >> 2 : 0u, wt);
          if (t < 256) {
            meta[s * 256 + t].x = excl;
            // pass 2: staging offset (bytes from the staging buffer) of (digit, lane) = digit's
            // tile offset + its keys in lanes below; quads < qr come after the wrap.  The other
            // half of every word is zeroed for the next tile.
            const uint32_t e = excl << KS;
            uint32_t run = e + ((tot - upper) << (KS - 2));
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t q = (uint32_t)(i + qr) & 7u;
              if (q == 0) run = e;
              const uint4 v = row[q];
              uint4 o;
              o.x = run << hsh; run += ((v.x >> hsh) & 0xFFFFu) << (KS - 2);
              o.y = run << hsh; run += ((v.y >> hsh) & 0xFFFFu) << (KS - 2);
              o.z = run << hsh; run += ((v.z >> hsh) & 0xFFFFu) << (KS - 2);
              o.w = run << hsh; run += ((v.w >> hsh) & 0xFFFFu) << (KS - 2);
              row[q] = o;
            }
          }
        }
        named_bar_sync(P2_BAR_R, RT);  // (B) staging addresses ready

        // stage: address = counter's staging address + rank; loads of a group before its stores
        constexpr int SG = 10;  // keys per staging group
#pragma unroll
        for (int k0 = 0; k0 < ITEMS; k0 += SG) {
          uint32_t pos[SG];
#pragma unroll
          for (int j = 0; j < SG; ++j) {
            const int k = k0 + j;
            if (k < ITEMS && (FULL || seg + IS * k < valid)) {
              const uint32_t w = s_ld(counter(keys[k]) + OFS * 4u);
              const uint32_t r = (rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
              if constexpr (MODE == R2_STABLE)
                pos[j] = w + (r << (KS - 2));
              else if constexpr (p2_runs(MODE))
                pos[j] = sbuf_a + ((w >> (run_of(keys[k]) << 4)) & 0xFFFFu) + (r << (KS - 2));
              else
                pos[j] = sbuf_a + (p2_swz<U>((((w >> hsh) & 0xFFFFu) >> KS) + (r >> 2)) << KS);  // swizzled
            }
          }
#pragma unroll
          for (int j = 0; j < SG; ++j) {
            const int k = k0 + j;
            if (k < ITEMS && (FULL || seg + IS * k < valid)) s_st(pos[j], keys[k]);
          }
        }
      };
      if (valid == (uint32_t)TILE && islot[s].bk == (uint32_t)TILE)
        tile_body(std::true_type{});
      else
        tile_body(std::false_type{});
      named_bar_arrive(P2_BAR_STAGED + s, RT + WT);  // hand the staged tile to the writers
    }
  } else {
    // ---------------------------------------------------------------- writers
    const uint32_t w = t - RT;
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it & 1u;
      named_bar_sync(P2_BAR_COUNTED + s, RT + WT);  // tile counts published (or the end)
      const uint32_t lin = sslot[s].lin;
      if (lin == P2_END) break;
      const uint32_t valid = sslot[s].len;
      const uint32_t chunk = sslot[s].chunk;
      const bool first_tile = sslot[s].first != 0;
      const uint32_t sbuf_a = smem_base + (uint32_t)L::sbuf_off + s * (uint32_t)(TILE * sizeof(U));
      uint32_t* gof = gofs + s * L::NG;
      uint32_t lf = 0, ll = 0;  // J01: the tile's digit-0 runs
      if constexpr (MODE == R2_J01) {
        lf = meta[s * 256 + 254].w;
        ll = meta[s * 256 + 255].w;
      }
      unsigned long long g0 = 0, g1 = 0;  // global start of this tile's run of digit w (J01: runs 0 / 1)
      uint32_t c0 = 0;
      if (w < 256) {
        const uint32_t c = meta[s * 256 + w].y;
        if constexpr (MODE == R2_STABLE || MODE == R2_RUN2) {
          uint32_t excl = 0;
          if (!first_tile) {
            excl = lookback_walk_v4<LBV>(lookback, w, lin);
            st_relaxed(&lookback[lb2_index(lin, w)], LB::INC | (excl + c));
          }
          if constexpr (CHUNKED)
            g0 = (unsigned long long)cm.jp[chunk * 256 + w] + excl;
          else
            g0 = bases[w] + excl;
        } else if constexpr (MODE == R2_UNSTABLE) {
          if (c) g0 = bases[w] + atomicAdd(&gcount[w], (unsigned long long)c);  // tile order is free
        } else {
          c0 = meta[s * 256 + w].z;
          if (c0) g0 = atomicAdd(&gcount[lf * 256 + w], (unsigned long long)c0);
          if (c - c0) g1 = atomicAdd(&gcount[ll * 256 + w], (unsigned long long)(c - c0));
        }
      }
      (void)chunk;
      named_bar_sync(P2_BAR_STAGED + s, RT + WT);  // rankers staged this tile
      if (w < 256) {
        const uint32_t x0 = meta[s * 256 + w].x;  // tile-exclusive offset of digit w
        if constexpr (MODE == R2_J01) {
          gof[2 * w] = (uint32_t)(g0 - x0);
          gof[2 * w + 1] = (uint32_t)(g1 - (x0 + c0));
        } else {
          gof[w] = (uint32_t)(g0 - x0);  // >= 0: the digits below w hold >= x0 keys globally
        }
      }
      named_bar_sync(P2_BAR_W, WT);
      constexpr int WB = 8;  // keys per writer per batch
      auto write_out = [&](auto full_c, auto dec_c) {
        constexpr bool FULL = decltype(full_c)::value;
        constexpr bool DEC = decltype(dec_c)::value;
        for (uint32_t base = w; base < valid; base += WB * WT) {
          U x[WB];
          uint32_t o[WB];
#pragma unroll
          for (int j = 0; j < WB; ++j) {
            const uint32_t i = base + j * WT;
            const uint32_t si = MODE == R2_UNSTABLE ? p2_swz<U>(i) : i;
            x[j] = (FULL || i < valid) ? s_ldk<U>(sbuf_a + si * (uint32_t)sizeof(U)) : U(0);
          }
#pragma unroll
          for (int j = 0; j < WB; ++j) {
            if constexpr (MODE == R2_J01)
              o[j] = gof[2 * p2_digit<SHIFT>(x[j]) + ((uint32_t(x[j]) & 0xFFu) != lf ? 1u : 0u)];
            else
              o[j] = gof[p2_digit<SHIFT>(x[j])];
          }
          const U* db = dst + base;
          static_for<WB>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            if (FULL || base + j * WT < valid) {
              U v = x[j];
              if constexpr (DEC) v = key_decode<KIND, DESC>(v);
              st_global_at<j * WT * (int)sizeof(U)>(db, o[j], v);
            }
          });
        }
      };
      constexpr bool WHOLE = TILE % (WB * WT) == 0;  // full tiles are whole batches
      if (WHOLE && valid == (uint32_t)TILE) {
        if (dec_out) write_out(std::bool_constant<WHOLE>{}, std::true_type{});
        else write_out(std::bool_constant<WHOLE>{}, std::false_type{});
      } else {
        if (dec_out) write_out(std::false_type{}, std::true_type{});
        else write_out(std::false_type{}, std::false_type{});
      }
      named_bar_arrive(P2_BAR_SFREE + s, RT + WT);  // staging slot s may be reused
    }
  }
}

}  // namespace bsort
