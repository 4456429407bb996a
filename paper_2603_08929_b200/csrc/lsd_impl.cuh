// lsd_impl.cuh — host orchestration of the 32/64-bit one-sweep LSD path (§8 rows a2-a5) and the
// launch helpers shared with the MSD partition.  Included by the per-(key width, payload,
// direction) translation units lsd_w{4,8}[_kv]_{asc,desc}.cu and by dist.cu / exact.cu, so the
// kernel instantiations compile in parallel.
//
//   memset(hist) -> k_onesweep_hist[_joint] -> k_plan [-> k_plan_joint]
//   -> P x { memset(look-back) ; k_onesweep_pass } -> k_copy_back (no-op unless an odd number of
//   passes executed).  Everything is stream-ordered on the caller's stream; no host sync.
#pragma once
#include <cstdlib>
#include <type_traits>

#include "onesweep.cuh"
#include "onesweep_ws.cuh"
#include "pass2.cuh"
#include "small.cuh"
#include "small_grid.cuh"
#include "paths.cuh"

namespace bsort {
namespace lsd_detail {


// Tile configuration per key width and ranking mode (tuned on B200 with tools/tune_pass.cu;
// profiles/r1/tune_*.jsonl).  Two CTAs per SM of 512 (384) threads, 8192 (4608) keys per tile.
// One 1024-thread CTA per SM shortens the look-back chains of a pure RUN2 pass (3.64 -> 3.38 ms)
// but its 16384-key tiles break RUN2's two-run condition in pass 2 (runs of ~16K keys at
// n = 2^30) and 8 keys per thread lose too much ILP (profiles/r1: cfg3 16.1 vs 16.6 / 19.7 ms).
// Key-value sorts (KV) carry ITEMS more registers and a second tile buffer pair: one CTA per SM.
template <typename U, int MODE, bool KV = false> struct PassCfg;
template <int MODE, bool KV> struct PassCfg<uint32_t, MODE, KV> {
  static constexpr int THREADS = 512, ITEMS = 16, MINB = KV ? 1 : 2, LBG = 8;
};
// The first LSD pass and the MSD partitions (unstable, no look-back): 10240-key tiles rank a
// little faster (tools/tune_pass -DTUNE_UNSTABLE: 2.45 -> 2.37 ms per 2^30 keys; x24 spills).
// The two-CTA look-back kernel keeps 8192 (the look-back array is sized for it).
template <> struct PassCfg<uint32_t, RANK_UNSTABLE, false> {
  static constexpr int THREADS = 512, ITEMS = 20, MINB = 2, LBG = 8;
};
// J01 (pass 1 without look-back) likewise; its eligibility is planned for this tile (J01_TILE).
template <> struct PassCfg<uint32_t, RANK_J01, false> {
  static constexpr int THREADS = 512, ITEMS = 20, MINB = 2, LBG = 8;
};
template <> struct PassCfg<unsigned long long, RANK_J01, false> {
  static constexpr int THREADS = 512, ITEMS = 12, MINB = 2, LBG = 8;
};
template <int MODE, bool KV> struct PassCfg<unsigned long long, MODE, KV> {
  static constexpr int THREADS = 384, ITEMS = 12, MINB = KV ? 1 : 2, LBG = 8;
};

template <typename U, bool KV = false> struct WsCfg;
template <> struct WsCfg<uint32_t, false> { static constexpr int RT = 512, ITEMS = 20; };
template <> struct WsCfg<unsigned long long, false> { static constexpr int RT = 512, ITEMS = 14; };
// key-value: three value buffers too; 512 x 16 (u32 keys, 192 KB + tables) / 512 x 10 (u64 keys)
template <> struct WsCfg<uint32_t, true> { static constexpr int RT = 512, ITEMS = 12; };
template <> struct WsCfg<unsigned long long, true> { static constexpr int RT = 512, ITEMS = 9; };

template <typename U> constexpr int hist_lanes() { return sizeof(U) == 4 ? 32 : 16; }

struct LsdLayout {
  size_t scratch, vscratch, ghist, bases, gcount, joint, seg, plan, counters, lookback, total;
  size_t lb_bytes;    // one look-back region
  int lb_regions;     // 2 below WS_MIN_N (alternating), 3 for 32-bit keys-only joint sorts (passes
                      // 1-3 each their own, zeroed by the histogram sweep), else 1 (memset per pass)
  size_t grid;        // k_grid_sort (small_grid.cuh): per-pass count matrix + barrier word
  uint64_t lb_tiles;  // look-back descriptor rows: tiles of the smallest look-back tile in use
};

// Smallest tile among the kernels that use the look-back array for (U, payload).
template <typename U, bool KV>
constexpr uint64_t lookback_tile() {
  constexpr uint64_t a = (uint64_t)PassCfg<U, RANK_RUN2, KV>::THREADS * PassCfg<U, RANK_RUN2, KV>::ITEMS;
  constexpr uint64_t b = (uint64_t)WsCfg<U, KV>::RT * WsCfg<U, KV>::ITEMS;
  return a < b ? a : b;
}

// Pass 1 may run look-back-free (RANK_J01) from the joint histogram of digits 0 and 1; below
// this size the digit-0 buckets are shorter than a tile anyway and the joint histogram's fixed
// cost (65536 bins) is not worth it.
constexpr uint64_t JOINT_MIN_N = 1ull << 24;

// Smallest n for the warp-specialised / round-2 look-back passes (lsd_run).
constexpr uint64_t WS_MIN_N = 1ull << 22;
// Smallest look-back tile of the kernels that use the three look-back regions of 32-bit
// keys-only joint sorts (k_pass2's half-warp-row variant: 640 x 15; checked below)
constexpr uint64_t TRI_MIN_TILE = 9600;

template <typename U>
LsdLayout lsd_layout(uint64_t n, bool kv = false) {
  const uint64_t TILE = kv ? lookback_tile<U, true>() : lookback_tile<U, false>();
  constexpr int P = sizeof(U);
  const uint64_t tiles = (n + TILE - 1) / TILE;
  const size_t desc = (n <= (1ull << 30)) ? 4 : 8;
  LsdLayout l;
  size_t off = 0;
  l.scratch = off;  off = align_up(off + n * sizeof(U), 256);
  l.vscratch = off; off = align_up(off + (kv ? n * sizeof(uint32_t) : 0), 256);
  l.ghist = off;    off = align_up(off + P * 256 * 8 + 16, 256);  // + the two order flags
  l.bases = off;    off = align_up(off + P * 256 * 8, 256);
  l.gcount = off;   off = align_up(off + P * 256 * 8, 256);
  const size_t jbytes = n >= JOINT_MIN_N ? 65536 * 8 : 0;  // joint histogram + segment starts
  // + the coarse joints of passes 2-3 and their chunk maps (32-bit keys; LB_NC)
  const size_t cbytes = n >= JOINT_MIN_N ? 2 * LB_NC * 256 * 8 + 2 * (LB_NC + 1) * 8 + 2 * (LB_NC + 1) * 4 +
                                               2 * LB_NC * 256 * 4 + 64
                                         : 0;
  l.joint = off;    off = align_up(off + jbytes + cbytes, 256);
  l.seg = off;      off = align_up(off + jbytes, 256);
  l.plan = off;     off = align_up(off + sizeof(PassPlan), 256);
  l.counters = off; off = align_up(off + 16 * 4, 256);
  // below WS_MIN_N two look-back regions alternate by pass parity (each pass kernel zeroes the
  // next pass's region: no memset launches, lsd_run)
  l.lb_regions = n < WS_MIN_N ? 2 : ((sizeof(U) == 4 && !kv && n >= JOINT_MIN_N && n <= (1ull << 30)) ? 3 : 1);
  // three regions: only k_pass2 (tiles >= TRI_MIN_TILE keys, + one partial tile per chunk) and the
  // few-runs kernel (10,240-key tiles) use them, so they are sized for those tiles
  const uint64_t lbt = l.lb_regions == 3 ? n / TRI_MIN_TILE + 16 : tiles;
  l.lb_bytes = align_up(lbt * 256 * desc, 256);
  l.lookback = off; off += l.lb_regions * l.lb_bytes;
  // just above 2^30 keys one (64-bit) region is smaller than the three regions at 2^30: pad, so
  // the workspace stays monotone in n (a workspace sized for n serves every smaller n)
  if (sizeof(U) == 4 && !kv && n > (1ull << 30)) {
    const uint64_t tri = 3 * align_up(((1ull << 30) / TRI_MIN_TILE + 16) * 256 * 4, 256);
    if (tri > l.lb_regions * l.lb_bytes) off += tri - l.lb_regions * l.lb_bytes;
  }
  l.grid = off;     off = align_up(off + grid_detail::workspace_bytes(), 256);  // k_grid_sort counts
  l.lb_tiles = tiles;
  l.total = off;
  return l;
}

template <typename U, bool BULK, int RANK, bool KV, typename DescT, typename DigitF>
bsort_status_t launch_pass_t(const U* a, U* b, uint64_t n, DigitF digit, const unsigned long long* bases,
                             DescT* lookback, unsigned long long* gcount, uint32_t* counter, const PassPlan* plan,
                             int pass, KvPtrs kvp, cudaStream_t s, ZeroSpan zs = {}) {
  using C = PassCfg<U, RANK, KV>;
  using L = PassSmem<C::THREADS, C::ITEMS, U, RANK, KV>;
  auto kern = k_onesweep_pass<U, C::THREADS, C::ITEMS, C::MINB, BULK, DescT, DigitF, RANK, C::LBG, KV>;
  static DeviceInt occ_d;  // per instantiation and device; benign race (idempotent)
  int& occ = occ_d.get();
  if (occ == 0) {
    BSORT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes));
    int o = 0;
    BSORT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, C::THREADS, L::bytes));
    occ = o > 0 ? o : 1;
  }
  const uint64_t tiles = (n + L::TILE - 1) / L::TILE;
  // persistent grid: every CTA resident at once (look-back forward progress)
  const uint64_t grid = min64(tiles, (uint64_t)num_sms() * occ);
  BSORT_LAUNCH(PROF_PASS, s,
               kern<<<(unsigned)grid, C::THREADS, L::bytes, s>>>(a, b, n, digit, bases, lookback, gcount, counter,
                                                                 (uint32_t)tiles, plan, pass, kvp, zs));
  return BSORT_SUCCESS;
}

// TMA bulk prefetch needs 16-byte aligned sources: both ping-pong buffers (the scratch buffer
// always is; the caller's array may be only element-aligned).
template <typename U, int RANK, typename DescT, bool KV = false, typename DigitF>
bsort_status_t launch_pass(const U* a, U* b, uint64_t n, DigitF digit, const unsigned long long* bases,
                           DescT* lookback, unsigned long long* gcount, uint32_t* counter, const PassPlan* plan,
                           int pass, cudaStream_t s, KvPtrs kvp = {}, ZeroSpan zs = {}) {
  bool aligned = ((uintptr_t)a % 16 == 0) && (plan == nullptr || (uintptr_t)b % 16 == 0);
  if (KV) aligned = aligned && (uintptr_t)kvp.va % 16 == 0 && (uintptr_t)kvp.vb % 16 == 0;
  if (aligned)
    return launch_pass_t<U, true, RANK, KV, DescT>(a, b, n, digit, bases, lookback, gcount, counter, plan, pass, kvp,
                                                   s, zs);
  return launch_pass_t<U, false, RANK, KV, DescT>(a, b, n, digit, bases, lookback, gcount, counter, plan, pass, kvp,
                                                  s, zs);
}

// Warp-specialised look-back pass (onesweep_ws.cuh) for keys without payload: rankers never wait
// for the look-back walk.  One CTA of 512 rankers + 256 writers per SM, larger tiles than
// PassCfg's (the look-back array, sized by PassCfg, is then large enough): 32-bit keys 512 x 20 =
// 10240 (three 40 KB buffers; tools/tune_pass -DTUNE_WS: stable 4.24 -> 3.79 ms, RUN2 3.65 -> 3.22
// ms per 2^30 keys; x16 and x24 were slower), 64-bit keys 512 x 14 = 7168 (three 56 KB buffers,
// 223 KB of shared memory: stable 3.18 -> 2.51 ms, RUN2 2.73 -> 2.27 ms per 2^29 keys; x12: 2.77 /
// 2.57).  RUN2's two-run condition holds for pass 2 of 2^30 keys (runs of ~16K keys).
// BSORT_WS=0 selects k_onesweep_pass instead (A/B).

// Below this size a pass has too few tiles to keep the walk off the critical path anyway, and
// the two-CTA kernel's smaller tiles spread a small input over more SMs (cfg1: 2^20 keys).
inline bool ws_enabled() {
  static const bool on = [] {
    const char* e = getenv("BSORT_WS");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename U, typename DescT, bool KV = false, int MODE = RANK_RUN2, typename DigitF>
bsort_status_t launch_pass_ws(const U* a, U* b, uint64_t n, DigitF digit, const unsigned long long* bases,
                              DescT* lookback, uint32_t* counter, const PassPlan* plan, int pass, cudaStream_t s,
                              KvPtrs kvp = {}, unsigned long long* gcount = nullptr, uint32_t only_fewruns = 0) {
  constexpr int WS_RT = WsCfg<U, KV>::RT;
  using L = PassSmemWS<WS_RT, WsCfg<U, KV>::ITEMS, U, KV>;
  static_assert(L::bytes <= 227 * 1024, "fits one CTA per SM");
  auto kern = k_onesweep_pass_ws<U, WS_RT, WsCfg<U, KV>::ITEMS, DescT, DigitF, MODE, 8, 1, KV>;
  static DeviceInt occ_d;
  int& occ = occ_d.get();
  if (occ == 0) {
    BSORT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes));
    int o = 0;
    BSORT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, WS_RT + 256, L::bytes));
    occ = o > 0 ? o : 1;
  }
  const uint64_t tiles = (n + L::TILE - 1) / L::TILE;
  const uint64_t grid = min64(tiles, (uint64_t)num_sms() * occ);  // all resident (look-back progress)
  BSORT_LAUNCH(PROF_PASS, s,
               kern<<<(unsigned)grid, WS_RT + 256, L::bytes, s>>>(a, b, n, digit, bases, lookback, counter,
                                                                  (uint32_t)tiles, plan, pass, kvp, gcount,
                                                                  only_fewruns));
  return BSORT_SUCCESS;
}

// Round-2 look-back pass (pass2.cuh) for 32-bit keys: ranking by lane-ordered warp atomics,
// separate input / staging buffers, vectorised look-back.  Keys stay raw in the buffers (P2_RAW):
// the passes before it are round-1 kernels.  640 rankers x 16 keys + 256 writers
// (tools/exp/tune2.cu: 3.45 ms per 2^30-key pass on cfg3 vs 3.65 / 4.16 ms for round 1's RUN2 /
// stable passes).  Needs n <= 2^30 (30-bit look-back counts).
template <int MODE> struct P2Cfg {
  static constexpr int RT = 512, WT = 256, ITEMS = 20;  // chunked passes 2 / 3: 2.97 -> 2.91 / 3.44 -> 3.37 ms vs 640 x 16
};
// RUN2 holds two lane-banked tables (counts, offsets): 640 x 15 = 9600-key tiles (TRI_MIN_TILE:
// the chunked RUN2 pass 2 uses the three look-back regions; 225 KB of shared memory)
template <> struct P2Cfg<R2_RUN2> {
  static constexpr int RT = 640, WT = 256, ITEMS = 15;
};
template <int MODE> constexpr uint64_t p2_tile() { return (uint64_t)P2Cfg<MODE>::RT * P2Cfg<MODE>::ITEMS; }
// skewed digits (plan->skew): half-warp counter rows, odd ITEMS (conflict-free key loads)
#ifndef P2SKEW_RT
#define P2SKEW_RT 640
#endif
#ifndef P2SKEW_ITEMS
#define P2SKEW_ITEMS 15
#endif
struct P2SkewCfg {
  static constexpr int RT = P2SKEW_RT, WT = 256, ITEMS = P2SKEW_ITEMS;
};
constexpr uint64_t P2_MAX_N = 1ull << 30;
static_assert((uint64_t)P2SkewCfg::RT * P2SkewCfg::ITEMS >= TRI_MIN_TILE &&
                  (uint64_t)P2Cfg<R2_STABLE>::RT * P2Cfg<R2_STABLE>::ITEMS >= TRI_MIN_TILE &&
                  p2_tile<R2_RUN2>() >= TRI_MIN_TILE &&
                  (uint64_t)WsCfg<uint32_t, false>::RT * WsCfg<uint32_t, false>::ITEMS >= TRI_MIN_TILE,
              "the three look-back regions are sized for TRI_MIN_TILE-key tiles");
// RUN2 for pass 2 measured slower than the stable pass on cfg3 (4.25 vs 3.6 ms, ALU-bound):
// off unless BSORT_P2_RUN2=1
inline bool p2_run2_enabled() {
  static const bool on = [] {
    const char* e = getenv("BSORT_P2_RUN2");
    return e && e[0] == '1';
  }();
  return on;
}
inline bool p2_enabled() {
  static const bool on = [] {
    const char* e = getenv("BSORT_P2");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <int KIND, bool DESC, int SHIFT, int MODE = R2_STABLE, int HALVES = 1, bool CHUNKED = false, typename U>
bsort_status_t launch_pass2(const U* a, U* b, uint64_t n, const unsigned long long* bases, uint32_t* lookback,
                            uint32_t* counter, const PassPlan* plan, int pass, cudaStream_t s, uint32_t xflags = 0,
                            ChunkMap cm = {}) {
  using C = std::conditional_t<HALVES == 2, P2SkewCfg, P2Cfg<MODE>>;
  using L = Pass2Smem<C::RT, C::WT, C::ITEMS, U, MODE, HALVES>;
  auto kern = k_pass2<U, KIND, DESC, SHIFT, C::RT, C::WT, C::ITEMS, MODE, CHUNKED, 2, HALVES>;
  static DeviceOnce attr;  // per instantiation and device
  if (attr.pending()) {
    BSORT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes));
    attr.mark();
  }
  // chunked: at most one partial tile per chunk more (the kernel stops at the map's tile count)
  const uint64_t tiles = (n + L::TILE - 1) / L::TILE + (CHUNKED ? cm.nc : 0);
  const uint64_t grid = min64(tiles, (uint64_t)num_sms());  // one CTA per SM, all resident
  BSORT_LAUNCH(PROF_PASS, s,
               kern<<<(unsigned)grid, C::RT + C::WT, L::bytes, s>>>(
                   a, b, n, bases, lookback, nullptr, counter, (uint32_t)tiles, plan, pass,
                   P2_RAW | P2_ENC | P2_DEC | xflags, cm));
  return BSORT_SUCCESS;
}

inline bsort_status_t memset_async(void* p, size_t bytes, cudaStream_t s) {
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(p, 0, bytes, s));
  return BSORT_SUCCESS;
}

template <int KIND, bool DESC, typename U, typename DescT, bool KV>
bsort_status_t lsd_run(U* keys, uint32_t* vals, uint64_t n, unsigned char* ws, cudaStream_t s) {
  // J01's eligibility (every nonzero digit-0 bucket at least one J01 tile) is planned for J01's tile
  constexpr uint64_t J01_TILE = (uint64_t)PassCfg<U, RANK_J01, KV>::THREADS * PassCfg<U, RANK_J01, KV>::ITEMS;
  constexpr int P = sizeof(U);
  constexpr int LANES = hist_lanes<U>();
  const LsdLayout l = lsd_layout<U>(n, KV);
  U* scratch = reinterpret_cast<U*>(ws + l.scratch);
  const KvPtrs kvp{vals, reinterpret_cast<uint32_t*>(ws + l.vscratch)};
  auto* ghist = reinterpret_cast<unsigned long long*>(ws + l.ghist);
  auto* bases = reinterpret_cast<unsigned long long*>(ws + l.bases);
  auto* gcount = reinterpret_cast<unsigned long long*>(ws + l.gcount);
  auto* joint = reinterpret_cast<unsigned long long*>(ws + l.joint);
  // coarse joints of passes 2-3 and their chunk maps, after the joint histogram (lsd_layout)
  auto* gcoarse = joint + 65536;
  auto* cstart = gcoarse + 2 * LB_NC * 256;
  auto* ctile = reinterpret_cast<uint32_t*>(cstart + 2 * (LB_NC + 1));
  auto* cjp = ctile + 2 * (LB_NC + 1);
  auto* seg = reinterpret_cast<unsigned long long*>(ws + l.seg);
  auto* plan = reinterpret_cast<PassPlan*>(ws + l.plan);
  auto* counters = reinterpret_cast<uint32_t*>(ws + l.counters);
  auto* lookback = reinterpret_cast<DescT*>(ws + l.lookback);

  // small n: the whole sort in one single-CTA launch (small.cuh)
  if constexpr (!KV) {
    if (n <= small_max_n<U>()) return launch_small<KIND, DESC, U>(keys, n, s);
    // mid-size: one cooperative launch, one CTA per SM (small_grid.cuh)
    if (n <= grid_max_n<U>() && n >= grid_min_n<U>())
      return launch_grid<KIND, DESC, U>(keys, scratch, n, reinterpret_cast<uint16_t*>(ws + l.grid), s);
  }

  static const bool joint_off = getenv("BSORT_NO_JOINT") != nullptr;  // A/B and debugging
  const bool use_joint = n >= JOINT_MIN_N && !joint_off;
  // passes 1-3 of 32-bit keys-only joint sorts use three look-back regions that the histogram
  // sweep zeroes (no memset launch per pass)
  // They are sized for TRI_MIN_TILE-key tiles (lsd_layout).  Where neither k_pass2 (BSORT_P2=0, or
  // a device that fails the lane-order self-test) nor the warp-specialised kernel (BSORT_WS=0, or
  // a caller pointer that is not 16-byte aligned) can run, the look-back passes fall back to
  // k_onesweep_pass, whose smaller tiles need more descriptor rows than one region holds: then
  // the three regions serve as one (3 x lb_bytes >= l.lb_tiles rows), zeroed by a memset per pass.
  bool tri = use_joint && l.lb_regions == 3;
  if constexpr (sizeof(U) == 4 && !KV) {
    if (tri) {
      const bool p2_ok = p2_enabled() && atomics_lane_ordered(s);
      const bool ws_ok = ws_enabled() && (uintptr_t)keys % 16 == 0;
      if (!p2_ok && !ws_ok) tri = false;
    }
  }
  // passes 2-3 of 32-bit keys: k_pass2, or the run-ranking warp-specialised kernel when the plan
  // finds few distinct lower-bit values (k_plan_joint's fewruns; both launched, one works)
  const bool few_alt = sizeof(U) == 4 && !KV && use_joint && n >= WS_MIN_N && n <= P2_MAX_N && p2_enabled() &&
                       ws_enabled() && (uintptr_t)keys % 16 == 0;
  // passes 2-3 of 32-bit keys with LB_NC look-back chains (the histogram sweep counted the coarse
  // joints); BSORT_P2_CHUNKED=0 turns it off (A/B)
  static const bool chunk_on = [] {
    const char* e = getenv("BSORT_P2_CHUNKED");
    return !(e && e[0] == '0');
  }();
  const bool chunked = sizeof(U) == 4 && !KV && use_joint && n <= P2_MAX_N && chunk_on;
  // digit histograms and, right after them, the presorted-input flags (k_onesweep_hist*)
  auto* order = reinterpret_cast<uint32_t*>(ghist + P * 256);
  BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(ghist, 0, P * 256 * 8 + 16, s));
  if (use_joint) {
    constexpr int JL = sizeof(U) == 4 ? 32 : 16;  // lanes of the digit >= 2 counters (224 KB for u64)
    auto hk = k_onesweep_hist_joint<KIND, DESC, U, JL>;
    constexpr int hsmem = hist_joint_words<P, JL>() * 4;
    static DeviceOnce hattr;
    if (hattr.pending()) {
      BSORT_CUDA(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem));
      hattr.mark();
    }
    BSORT_LAUNCH(PROF_MEMSET, s, cudaMemsetAsync(joint, 0, (65536 + 2 * LB_NC * 256) * 8, s));
    // presorted check first (stops early on unsorted input); the histogram sweep then checks no
    // pairs, and does nothing for a presorted / reversed input
    BSORT_LAUNCH(PROF_HIST, s, k_order_check<KIND, DESC, U><<<num_sms(), HIST_THREADS, 0, s>>>(keys, n, order));
    BSORT_LAUNCH(PROF_HIST, s,
                 hk<<<num_sms(), HIST_THREADS, hsmem, s>>>(
                     keys, n, ghist, joint, order, true, gcoarse,
                     tri ? ZeroSpan{reinterpret_cast<uint4*>(lookback), (uint32_t)(3 * l.lb_bytes / 16)} : ZeroSpan{}));
  } else {
    // the histogram kernel's last CTA also plans (no k_plan launch)
    auto hk = k_onesweep_hist<KIND, DESC, U, LANES, true>;
    constexpr int hsmem = P * 256 * LANES * 4;
    static DeviceOnce hattr;
    if (hattr.pending()) {
      BSORT_CUDA(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem));
      hattr.mark();
    }
    BSORT_LAUNCH(PROF_HIST, s,
                 hk<<<num_sms(), HIST_THREADS, hsmem, s>>>(keys, n, ghist, order,
                                                           PlanArgs{bases, plan, counters, gcount}));
  }
  if (use_joint) {
    // marginals, nonzero-bin count (order[2]) and J01's relative segment starts: 256 CTAs
    BSORT_LAUNCH(PROF_SCAN, s, k_joint_marg<<<256, 256, 0, s>>>(joint, ghist, seg, order + 2));
    BSORT_LAUNCH(PROF_SCAN, s, k_plan<<<1, 256, 0, s>>>(ghist, n, P, bases, plan, counters, gcount, nullptr, order));
  }
  if (use_joint)
    BSORT_LAUNCH(PROF_SCAN, s,
                 k_plan_joint<<<1, 256, 0, s>>>(joint, ghist, bases + 256, J01_TILE, plan, seg,
                                                (sizeof(U) == 4 && !KV && n <= P2_MAX_N && p2_enabled() && p2_run2_enabled())
                                                    ? p2_tile<R2_RUN2>()
                                                    : 0,
                                                few_alt ? (uint64_t)WsCfg<U, false>::RT * WsCfg<U, false>::ITEMS : 0,
                                                n,
                                                chunked ? ChunkPlanArgs{bases, gcoarse, cstart, ctile, cjp,
                                                                        p2_tile<R2_STABLE>(), n,
                                                                        (uint64_t)P2SkewCfg::RT * P2SkewCfg::ITEMS}
                                                        : ChunkPlanArgs{}));
  bsort_status_t st = BSORT_SUCCESS;
  const bool fold = n < WS_MIN_N;  // look-back zeroing folded into the pass kernels
  auto one_pass = [&](auto shift_c) {
    constexpr int SH = decltype(shift_c)::value;
    constexpr int p = SH / 8;
    if (p >= P || st != BSORT_SUCCESS) return;
    // below WS_MIN_N only k_onesweep_pass runs: it zeroes the other look-back region for the
    // next pass (fold), else one memset per look-back pass
    DescT* lb = lookback;
    ZeroSpan zs{};
    if (fold) {
      lb = reinterpret_cast<DescT*>(reinterpret_cast<unsigned char*>(lookback) + (p & 1) * l.lb_bytes);
      if (p + 1 < P)
        zs = ZeroSpan{reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(lookback) + ((p + 1) & 1) * l.lb_bytes),
                      (uint32_t)(l.lb_bytes / 16)};
    } else if constexpr (p > 0) {
      if (tri && p <= 3) {
        lb = reinterpret_cast<DescT*>(reinterpret_cast<unsigned char*>(lookback) + (p - 1) * l.lb_bytes);
      } else {
        st = memset_async(lookback, l.lb_tiles * 256 * sizeof(DescT), s);
        if (st != BSORT_SUCCESS) return;
      }
    }
    // The first LSD pass may order equal digits arbitrarily (the input order carries no
    // information); every later pass must be stable.
    if constexpr (p == 0) {
      // 64-bit keys: the warp-specialised kernel is faster for the unstable pass too (tune_pass
      // -DTUNE_WS: 1.90 -> 1.78 ms per 2^29 keys); 32-bit keys keep two CTAs per SM (2.37 vs 2.81)
      bool done = false;
      if constexpr (sizeof(U) == 8 && !KV) {
        if (n >= WS_MIN_N && ws_enabled() && (uintptr_t)keys % 16 == 0) {
          st = launch_pass_ws<U, DescT, false, RANK_UNSTABLE>(keys, scratch, n, RadixDigit<KIND, DESC, U, SH>{},
                                                              bases, lb, counters, plan, p, s, KvPtrs{},
                                                              gcount);
          done = true;
        }
      }
      if (!done)
        st = launch_pass<U, RANK_UNSTABLE, DescT, KV>(keys, scratch, n, RadixDigit<KIND, DESC, U, SH>{}, bases,
                                                      lookback, gcount, counters, plan, p, s, kvp, zs);
    } else {
      bool done = false;
      if constexpr (sizeof(U) == 4 && !KV) {
        if (n >= WS_MIN_N && n <= P2_MAX_N && p2_enabled() && (uintptr_t)keys % sizeof(U) == 0 &&
            atomics_lane_ordered(s)) {
          // (below 2^24 keys, unchunked: half-warp counter rows for skewed digits measured no
          // faster, 3.98 vs 3.92 ms; with chunked chains they are, below)
          const bool alt = few_alt && p >= 2;
          if (chunked && p >= 2) {
            const int q = p - 2;
            const ChunkMap cm{nullptr, cstart + q * (LB_NC + 1), ctile + q * (LB_NC + 1), cjp + q * LB_NC * 256,
                              (uint32_t)LB_NC};
            // skewed digit (plan->skew: one bin > n/8, e.g. cfg3's sign + exponent byte): half-warp
            // counter rows halve same-word atomic serialization (chunked pass 3: 3.44 -> 3.30 ms);
            // both launched, the plan's skew bit lets one work (its tile size is in the chunk map)
            const uint32_t xf = (alt ? P2_FEWALT : 0u) | P2_SKEWVAR;
            st = launch_pass2<KIND, DESC, SH, R2_STABLE, 1, true>(keys, scratch, n, bases + p * 256,
                                                                  reinterpret_cast<uint32_t*>(lb), counters + p,
                                                                  plan, p, s, xf, cm);
            if (st == BSORT_SUCCESS)
              st = launch_pass2<KIND, DESC, SH, R2_STABLE, 2, true>(keys, scratch, n, bases + p * 256,
                                                                    reinterpret_cast<uint32_t*>(lb),
                                                                    counters + p, plan, p, s, xf, cm);
            // pass 2 ranked by runs (chunked, same chains) when the plan sets run2; the stable
            // launches above then return at once
            if constexpr (p == 2)
              if (st == BSORT_SUCCESS && p2_run2_enabled())
                st = launch_pass2<KIND, DESC, SH, R2_RUN2, 1, true>(keys, scratch, n, bases + p * 256,
                                                                    reinterpret_cast<uint32_t*>(lb),
                                                                    counters + 12, plan, p, s, 0u, cm);
          } else {
            st = launch_pass2<KIND, DESC, SH>(keys, scratch, n, bases + p * 256,
                                              reinterpret_cast<uint32_t*>(lb), counters + p, plan, p, s,
                                              alt ? P2_FEWALT : 0u);
          }
          if (st == BSORT_SUCCESS && alt)
            st = launch_pass_ws<U, DescT, false, RANK_RUN2>(keys, scratch, n, RadixDigit<KIND, DESC, U, SH>{},
                                                            bases + p * 256, lb, counters + p, plan, p, s,
                                                            KvPtrs{}, nullptr, 1u);
          // pass 2 ranked by runs when the plan allows it (each launch checks plan->run2)
          if constexpr (p == 2)
            if (st == BSORT_SUCCESS && use_joint && !chunked && p2_run2_enabled())
              st = launch_pass2<KIND, DESC, SH, R2_RUN2>(keys, scratch, n, bases + p * 256,
                                                         reinterpret_cast<uint32_t*>(lb), counters + 12, plan, p,
                                                         s);
          done = true;
        }
      }
      // TMA on both buffers (the scratch buffers are aligned)
      if (!done && n >= WS_MIN_N && ws_enabled() && (uintptr_t)keys % 16 == 0 && (!KV || (uintptr_t)vals % 16 == 0)) {
        st = launch_pass_ws<U, DescT, KV>(keys, scratch, n, RadixDigit<KIND, DESC, U, SH>{}, bases + p * 256,
                                          lb, counters + p, plan, p, s, kvp);
        done = true;
      }
      if (!done)
        st = launch_pass<U, RANK_RUN2, DescT, KV>(keys, scratch, n, RadixDigit<KIND, DESC, U, SH>{},
                                                  bases + p * 256, lb, gcount + p * 256, counters + p,
                                                  plan, p, s, kvp, zs);
    }
    // pass 1 without look-back when the joint plan allows it (each launch checks plan->j01
    // and exactly one of the two does the work)
    if constexpr (p == 1)
      if (st == BSORT_SUCCESS && use_joint)
        st = launch_pass<U, RANK_J01, DescT, KV>(keys, scratch, n, RadixDigit<KIND, DESC, U, SH>{}, bases + 256,
                                                 lb, seg, counters + 8, plan, p, s, kvp);
  };
  one_pass(std::integral_constant<int, 0>{});
  one_pass(std::integral_constant<int, 8>{});
  one_pass(std::integral_constant<int, 16>{});
  one_pass(std::integral_constant<int, 24>{});
  if constexpr (P == 8) {
    one_pass(std::integral_constant<int, 32>{});
    one_pass(std::integral_constant<int, 40>{});
    one_pass(std::integral_constant<int, 48>{});
    one_pass(std::integral_constant<int, 56>{});
  }
  if (st != BSORT_SUCCESS) return st;
  const int cgrid = (int)min64((n + 255) / 256, (uint64_t)num_sms() * 16);
  BSORT_LAUNCH(PROF_COPY, s, k_copy_back<U><<<cgrid, 256, 0, s>>>(keys, scratch, n, plan));
  if constexpr (KV)
    BSORT_LAUNCH(PROF_COPY, s, k_copy_back<uint32_t><<<cgrid, 256, 0, s>>>(vals, kvp.vb, n, plan));
  return BSORT_SUCCESS;
}


template <int KIND, bool DESC, typename U, bool KV>
bsort_status_t lsd_dispatch_desc(U* keys, uint32_t* vals, uint64_t n, unsigned char* ws, cudaStream_t s) {
  if (n <= (1ull << 30)) return lsd_run<KIND, DESC, U, uint32_t, KV>(keys, vals, n, ws, s);
  return lsd_run<KIND, DESC, U, unsigned long long, KV>(keys, vals, n, ws, s);
}

// Instantiates the LSD path for one key width, payload mode and direction (one translation unit
// each, so the 64-bit instantiations -- the longest -- compile in parallel halves).
template <typename U, bool KV, bool DESC>
bsort_status_t lsd_dispatch(int kind, U* keys, uint32_t* vals, uint64_t n, unsigned char* ws, cudaStream_t s) {
  switch (kind) {
    case KIND_U:
      return lsd_dispatch_desc<KIND_U, DESC, U, KV>(keys, vals, n, ws, s);
    case KIND_I:
      return lsd_dispatch_desc<KIND_I, DESC, U, KV>(keys, vals, n, ws, s);
    default:
      return lsd_dispatch_desc<KIND_F, DESC, U, KV>(keys, vals, n, ws, s);
  }
}

}  // namespace lsd_detail
}  // namespace bsort
