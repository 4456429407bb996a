// wide.cuh (tools/exp; NOT part of the library -- a measured negative result): LSD passes with 11- and 10-bit digits, so 32-bit keys sort in THREE
// scatter passes (digits 11 / 11 / 10) instead of four 8-bit ones.
//
// Paper mapping as in onesweep.cuh: one pass = a stable 2^b-way split of the transformed key on
// one digit (Algorithm 1's one-bit split of P:141-160, widened to b bits; LSD order needs every
// pass after the first to be stable).  Why wider digits: on B200 an 8-bit pass is bound by the
// shared-memory pipe (16-25 wavefronts per 32 keys, ~0.6-1.0 SM-cycles per key),
// not by HBM, so the cost of a sort is roughly (passes x per-key ranking work); per-key work
// hardly depends on the digit width (one shared atomic, one restaging store), per-TILE work does
// (2^b counters to scan, 2^b look-back descriptors), and tiles of 8192 keys amortise 2048 bins.
//
// One kernel, three ranking modes (all: persistent CTAs, tiles from an atomic counter, TMA bulk
// prefetch of the next tile, in-place restaging, coalesced write-out):
//   WM_UNSTABLE  (pass 0): CTA-wide counters, rank = the atomic's return value; each tile takes
//                its per-digit global offsets with one global atomicAdd per nonzero digit.
//   WM_RUN2      (pass 1, when every nonzero digit-0 bucket is at least a tile long, so a tile
//                meets at most two runs of equal lower bits): ranked unstably by (digit, run) in
//                u16 halves of one word per digit -- keys of equal digit and equal lower bits are
//                interchangeable, run 0 precedes run 1 -- plus a decoupled look-back for the order
//                between tiles.
//   WM_STABLE    (last pass, or pass 1 when RUN2 does not hold): lane-ordered per-warp atomics
//                (pass2.cuh: a warp's same-word atomics return old values in lane order on sm_100,
//                checked at run time by bsort_selftest), per-digit scan over the warps, look-back.
// Look-back descriptors live in a ring of WIDE_RING tiles (u32: 0 = not published, bit 31 =
// inclusive prefix, else aggregate + 1); a tile that has published its inclusive prefix clears the
// slot WIDE_RING / 2 tiles ahead of it, which last held a tile WIDE_RING / 2 behind it.
#pragma once
#include "pass2.cuh"

namespace bsort {

enum WideMode : int { WM_UNSTABLE = 0, WM_RUN2 = 1, WM_STABLE = 2 };
constexpr uint32_t WIDE_RING = 4096;          // look-back ring (tiles); a power of two
constexpr uint32_t WIDE_INC = 0x80000000u;    // descriptor: inclusive prefix

// flags
constexpr uint32_t WF_ENC = 1, WF_DEC = 2;

template <int NT, int ITEMS, int BITS, int MODE>
struct WideSmem {
  static constexpr int NW = NT / 32;
  static constexpr int TILE = NT * ITEMS;
  static constexpr int BINS = 1 << BITS;
  static constexpr int CNT_WORDS = MODE == WM_STABLE ? NW * BINS : BINS;
  static constexpr size_t buf_off = 0;                                                  // u32[2][TILE]
  static constexpr size_t cnt_off = align_up(buf_off + 2 * 4 * (size_t)TILE, 16);
  static constexpr size_t excl_off = align_up(cnt_off + 4 * (size_t)CNT_WORDS, 16);   // u32[BINS]
  static constexpr size_t gofs_off = align_up(excl_off + 4 * (size_t)BINS, 16);       // u32[BINS]
  static constexpr size_t wt_off = align_up(gofs_off + 4 * (size_t)BINS, 16);         // u32[NW + 1]
  static constexpr size_t mbar_off = align_up(wt_off + 4 * (NW + 1), 16);             // u64[2]
  static constexpr size_t tile_off = mbar_off + 16;                                   // u32[2]
  static constexpr size_t bytes = align_up(tile_off + 16, 128);
};

template <int N>
__device__ __forceinline__ void ld_relaxed_vec(const uint32_t* p, uint32_t (&v)[N]) {
  if constexpr (N == 4) {
    asm volatile("ld.relaxed.gpu.global.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "l"(p)
                 : "memory");
  } else if constexpr (N == 2) {
    asm volatile("ld.relaxed.gpu.global.v2.b32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "l"(p) : "memory");
  } else {
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v[0]) : "l"(p) : "memory");
  }
}
template <int N>
__device__ __forceinline__ void st_relaxed_vec(uint32_t* p, const uint32_t (&v)[N]) {
  if constexpr (N == 4) {
    asm volatile("st.relaxed.gpu.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3])
                 : "memory");
  } else if constexpr (N == 2) {
    asm volatile("st.relaxed.gpu.global.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(v[0]), "r"(v[1]) : "memory");
  } else {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v[0]) : "memory");
  }
}

// Exclusive prefix over tiles < T of the BPT digits at ring + b0 (G predecessors per L2 round
// trip).  The first tile publishes inclusive prefixes, so every walk ends.
template <int BINS, int BPT, int G>
__device__ __forceinline__ void wide_walk(const uint32_t* ring, uint32_t b0, uint32_t T, uint32_t (&ex)[BPT]) {
  uint32_t done = 0;
#pragma unroll
  for (int i = 0; i < BPT; ++i) ex[i] = 0;
  int64_t j = (int64_t)T - 1;
  for (;;) {
    uint32_t v[G][BPT];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t q = j - g;
      if (q >= 0)
        ld_relaxed_vec<BPT>(ring + (size_t)((uint32_t)q & (WIDE_RING - 1)) * BINS + b0, v[g]);
      else
#pragma unroll
        for (int i = 0; i < BPT; ++i) v[g][i] = WIDE_INC;  // never reached: tile 0 is inclusive
    }
    bool stall = false;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!stall && done != (1u << BPT) - 1u) {
        bool ready = true;
#pragma unroll
        for (int i = 0; i < BPT; ++i)
          if (!((done >> i) & 1u) && v[g][i] == 0u) ready = false;
        if (!ready) {
          stall = true;
          j -= g;  // retry from this predecessor
        } else {
#pragma unroll
          for (int i = 0; i < BPT; ++i) {
            if (!((done >> i) & 1u)) {
              const uint32_t e = v[g][i];
              if (e & WIDE_INC) {
                ex[i] += e & ~WIDE_INC;
                done |= 1u << i;
              } else {
                ex[i] += e - 1u;
              }
            }
          }
        }
      }
    }
    if (done == (1u << BPT) - 1u) return;
    if (stall)
      __nanosleep(64);
    else
      j -= G;
  }
}

// One LSD pass over 32-bit (encoded) keys: digit = (key >> SHIFT) & (2^BITS - 1).
//   src -> dst, n < 2^31 keys; bases[d] = global start of digit d (exclusive histogram prefix);
//   ring: WIDE_RING x 2^BITS descriptors, all zero before the first launch that uses it (every
//   launch leaves it zero); gcount[2^BITS] zeroed (UNSTABLE); tile_counter zeroed.
template <int KIND, bool DESC, int SHIFT, int BITS, int MODE, int NT, int ITEMS, int MINB, int G = 4>
__global__ void __launch_bounds__(NT, MINB)
    k_wide(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, uint32_t n,
           const uint32_t* __restrict__ bases, uint32_t* __restrict__ ring, uint32_t* __restrict__ gcount,
           uint32_t* __restrict__ tile_counter, uint32_t num_tiles, uint32_t flags) {
  using L = WideSmem<NT, ITEMS, BITS, MODE>;
  constexpr int TILE = L::TILE, BINS = L::BINS, NW = L::NW;
  constexpr int BPT = BINS / NT;  // digits per thread in the scan / walk
  static_assert(BINS % NT == 0 && (BPT == 1 || BPT == 2 || BPT == 4), "digits per thread");
  static_assert(ITEMS % 4 == 0 && TILE < 65536, "vector loads; u16 ranks");
  static_assert(MODE != WM_RUN2 || SHIFT > 0, "RUN2 needs lower bits");
  constexpr uint32_t DM = BINS - 1;
  constexpr uint32_t LOWMASK = SHIFT > 0 ? (1u << SHIFT) - 1u : 0u;
  constexpr bool LOOKBACK = MODE != WM_UNSTABLE;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* bufs = reinterpret_cast<uint32_t*>(smem + L::buf_off);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L::cnt_off);
  uint32_t* excl = reinterpret_cast<uint32_t*>(smem + L::excl_off);
  uint32_t* gofs = reinterpret_cast<uint32_t*>(smem + L::gofs_off);
  uint32_t* wt = reinterpret_cast<uint32_t*>(smem + L::wt_off);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L::mbar_off);
  volatile uint32_t* tile_s = reinterpret_cast<volatile uint32_t*>(smem + L::tile_off);
  const uint32_t cnt_a = smem_u32(cnt), excl_a = smem_u32(excl), gofs_a = smem_u32(gofs);
  const bool enc = (flags & WF_ENC) != 0, dec = (flags & WF_DEC) != 0;
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t b0 = t * BPT;  // this thread's digits in the scan / walk

  auto valid_of = [&](uint32_t id) -> uint32_t { return min((uint32_t)TILE, n - id * (uint32_t)TILE); };
  auto issue = [&](int b, uint32_t id) {
    const uint32_t v = valid_of(id);
    bulk_load(bufs + b * TILE, src + (size_t)id * TILE, (v * 4u) & ~15u, &mbar[b]);
  };
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
  for (int i = t; i < L::CNT_WORDS; i += NT) cnt[i] = 0;
  __syncthreads();

  for (uint32_t it = 0;; ++it) {
    const uint32_t cur = it & 1u;
    const uint32_t tile = tile_s[cur];
    if (tile >= num_tiles) break;
    const uint32_t valid = valid_of(tile);
    const uint32_t bk = ((valid * 4u) & ~15u) >> 2;  // keys the bulk copy brought
    const uint32_t* gsrc = src + (size_t)tile * TILE;
    uint32_t* buf = bufs + cur * TILE;
    const uint32_t buf_a = smem_u32(buf);
    if constexpr (MODE == WM_STABLE) {
      // zero this warp's counter row (last read by this warp's staging of the previous tile)
      uint4* r4 = reinterpret_cast<uint4*>(cnt + warp * BINS);
#pragma unroll
      for (int j = 0; j < BINS / 128; ++j) r4[lane + 32 * j] = make_uint4(0, 0, 0, 0);
      __syncwarp();
    }
    mbar_wait(&mbar[cur], (it >> 1) & 1u);

    auto body = [&](auto full_c) {
      constexpr bool FULL = decltype(full_c)::value;
      uint32_t keys[ITEMS];
      uint32_t rk[ITEMS / 2];
      // item k of this thread: STABLE index order (warp, item, lane); else 16-byte vectors
      auto idx = [&](int k) -> uint32_t {
        if constexpr (MODE == WM_STABLE)
          return warp * (32 * ITEMS) + k * 32 + lane;
        else
          return (uint32_t)(k >> 2) * (NT * 4) + t * 4 + (k & 3);
      };
      if constexpr (MODE == WM_STABLE) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t i = idx(k);
          keys[k] = (FULL || i < bk) ? s_ld(buf_a + i * 4) : (i < valid ? ldg_nc(gsrc + i) : 0u);
        }
      } else {
#pragma unroll
        for (int j = 0; j < ITEMS / 4; ++j) {
          const uint32_t i0 = (uint32_t)j * (NT * 4) + t * 4;
          if (FULL || i0 + 4 <= bk) {
            const uint4 v = *reinterpret_cast<const uint4*>(buf + i0);
            keys[4 * j] = v.x;
            keys[4 * j + 1] = v.y;
            keys[4 * j + 2] = v.z;
            keys[4 * j + 3] = v.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t i = i0 + e;
              keys[4 * j + e] = i < bk ? buf[i] : (i < valid ? ldg_nc(gsrc + i) : 0u);
            }
          }
        }
      }
      if (enc) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) keys[k] = key_encode<KIND, DESC>(keys[k]);
      }
      uint32_t lf = 0;
      if constexpr (MODE == WM_RUN2) {
        uint32_t fk = bk > 0 ? buf[0] : ldg_nc(gsrc);
        if (enc) fk = key_encode<KIND, DESC>(fk);
        lf = fk & LOWMASK;
      }
      auto digit = [&](uint32_t x) -> uint32_t { return (x >> SHIFT) & DM; };
      // ---- rank
#pragma unroll
      for (int k = 0; k < ITEMS / 2; ++k) rk[k] = 0;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        if (FULL || idx(k) < valid) {
          const uint32_t d = digit(keys[k]);
          uint32_t r;
          if constexpr (MODE == WM_STABLE) {
            r = s_atom_add(cnt_a + (warp * BINS + d) * 4u, 1u);
          } else if constexpr (MODE == WM_UNSTABLE) {
            r = atomicAdd(cnt + d, 1u);
          } else {
            const uint32_t sh = ((keys[k] & LOWMASK) != lf) ? 16u : 0u;
            r = (atomicAdd(cnt + d, 1u << sh) >> sh) & 0xFFFFu;
          }
          rk[k >> 1] |= r << ((k & 1) * 16);
        }
      }
      __syncthreads();  // (A) counts complete; every key of the buffer is in registers

      // ---- scan: digits b0 .. b0 + BPT - 1
      uint32_t c[BPT], c0[BPT], eo[BPT];
      if constexpr (MODE == WM_STABLE) {
#pragma unroll
        for (int i = 0; i < BPT; ++i) c[i] = 0;
#pragma unroll 4
        for (int w = 0; w < NW; ++w) {
          if constexpr (BPT == 2) {
            const uint2 v = *reinterpret_cast<const uint2*>(cnt + w * BINS + b0);
            c[0] += v.x;
            c[1] += v.y;
          } else if constexpr (BPT == 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(cnt + w * BINS + b0);
            c[0] += v.x;
            c[1] += v.y;
            c[2] += v.z;
            c[3] += v.w;
          } else {
            c[0] += cnt[w * BINS + b0];
          }
        }
      } else {
        uint32_t v[BPT];
#pragma unroll
        for (int i = 0; i < BPT; ++i) v[i] = cnt[b0 + i];
#pragma unroll
        for (int i = 0; i < BPT; ++i) cnt[b0 + i] = 0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
          if constexpr (MODE == WM_RUN2) {
            c0[i] = v[i] & 0xFFFFu;
            c[i] = c0[i] + (v[i] >> 16);
          } else {
            c[i] = v[i];
          }
        }
      }
      uint32_t tot = 0;
#pragma unroll
      for (int i = 0; i < BPT; ++i) tot += c[i];
      // publish this tile's aggregates early (look-back), before the scan's barriers
      uint32_t* slot = ring + (size_t)(tile & (WIDE_RING - 1)) * BINS + b0;
      if constexpr (LOOKBACK) {
        uint32_t pv[BPT];
#pragma unroll
        for (int i = 0; i < BPT; ++i) pv[i] = tile == 0 ? (WIDE_INC | c[i]) : c[i] + 1u;
        st_relaxed_vec<BPT>(slot, pv);
      }
      const uint32_t e = block_exclusive_scan<NT>(tot, wt, (uint32_t*)nullptr);
      {
        uint32_t run = e;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
          eo[i] = run;
          run += c[i];
        }
      }
      if constexpr (MODE == WM_STABLE) {
        // rows -> staging offsets: row w of digit d = tile offset of d + keys of d in warps < w
        uint32_t run[BPT];
#pragma unroll
        for (int i = 0; i < BPT; ++i) run[i] = eo[i];
#pragma unroll 4
        for (int w = 0; w < NW; ++w) {
#pragma unroll
          for (int i = 0; i < BPT; ++i) {
            const uint32_t v = cnt[w * BINS + b0 + i];
            cnt[w * BINS + b0 + i] = run[i];
            run[i] += v;
          }
        }
      } else if constexpr (MODE == WM_RUN2) {
#pragma unroll
        for (int i = 0; i < BPT; ++i) excl[b0 + i] = eo[i] | ((eo[i] + c0[i]) << 16);
      } else {
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
          excl[b0 + i] = eo[i];
          if (c[i]) gofs[b0 + i] = bases[b0 + i] + atomicAdd(&gcount[b0 + i], c[i]) - eo[i];
        }
      }
      __syncthreads();  // (B) staging offsets ready

      // ---- stage the tile in digit order (in place)
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        if (FULL || idx(k) < valid) {
          const uint32_t d = digit(keys[k]);
          const uint32_t r = (rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
          uint32_t p;
          if constexpr (MODE == WM_STABLE) {
            p = s_ld(cnt_a + (warp * BINS + d) * 4u) + r;
          } else if constexpr (MODE == WM_RUN2) {
            const uint32_t sh = ((keys[k] & LOWMASK) != lf) ? 16u : 0u;
            p = ((s_ld(excl_a + d * 4u) >> sh) & 0xFFFFu) + r;
          } else {
            p = s_ld(excl_a + d * 4u) + r;
          }
          s_st<uint32_t>(buf_a + p * 4u, keys[k]);
        }
      }
      // ---- look-back: global start of this tile's digits
      if constexpr (LOOKBACK) {
        uint32_t ex[BPT];
        if (tile > 0) {
          wide_walk<BINS, BPT, G>(ring, b0, tile, ex);
          uint32_t pv[BPT];
#pragma unroll
          for (int i = 0; i < BPT; ++i) pv[i] = WIDE_INC | (ex[i] + c[i]);
          st_relaxed_vec<BPT>(slot, pv);
        } else {
#pragma unroll
          for (int i = 0; i < BPT; ++i) ex[i] = 0;
        }
        // clear the slot WIDE_RING / 2 tiles ahead (held a tile WIDE_RING / 2 behind this one)
        {
          uint32_t z[BPT];
#pragma unroll
          for (int i = 0; i < BPT; ++i) z[i] = 0;
          st_relaxed_vec<BPT>(ring + (size_t)((tile + WIDE_RING / 2) & (WIDE_RING - 1)) * BINS + b0, z);
        }
#pragma unroll
        for (int i = 0; i < BPT; ++i) gofs[b0 + i] = bases[b0 + i] + ex[i] - eo[i];
      }
      __syncthreads();  // (C) tile staged; offsets ready

      // ---- write-out: runs of equal digits are contiguous
      constexpr int WB = 8;
#pragma unroll
      for (int j0 = 0; j0 < ITEMS; j0 += WB) {
        uint32_t x[WB], o[WB];
#pragma unroll
        for (int j = 0; j < WB; ++j) {
          const uint32_t i = (uint32_t)(j0 + j) * NT + t;
          x[j] = (FULL || i < valid) ? s_ld(buf_a + i * 4u) : 0u;
        }
#pragma unroll
        for (int j = 0; j < WB; ++j) {
          const uint32_t i = (uint32_t)(j0 + j) * NT + t;
          o[j] = s_ld(gofs_a + digit(x[j]) * 4u) + i;
        }
#pragma unroll
        for (int j = 0; j < WB; ++j) {
          const uint32_t i = (uint32_t)(j0 + j) * NT + t;
          if (FULL || i < valid) dst[o[j]] = dec ? key_decode<KIND, DESC>(x[j]) : x[j];
        }
      }
    };
    if (valid == (uint32_t)TILE)
      body(std::true_type{});
    else
      body(std::false_type{});
    __syncthreads();  // (D) the buffer is free
    if (t == 0) {
      const uint32_t id = atomicAdd(tile_counter, 1u);
      tile_s[cur] = id;
      if (id < num_tiles) issue((int)cur, id);
    }
  }
}

// Histograms of the three digits (11 / 11 / 10 bits) of the encoded keys, one read: per-CTA
// shared counters, flushed with global atomics.  hist: u32[2048 + 2048 + 1024] (zeroed).
template <int KIND, bool DESC, int NT>
__global__ void __launch_bounds__(NT, 1) k_wide_hist(const uint32_t* __restrict__ src, uint32_t n,
                                                     uint32_t* __restrict__ hist) {
  constexpr int NB = 2048 + 2048 + 1024;
  constexpr int R = 4;  // replicas (by warp)
  extern __shared__ __align__(16) uint32_t sh[];  // [R][NB]
  for (int i = threadIdx.x; i < R * NB; i += NT) sh[i] = 0;
  __syncthreads();
  uint32_t* h = sh + ((threadIdx.x >> 5) % R) * NB;
  const uint32_t nv = n / 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < nv; i += gridDim.x * NT) {
    const uint4 v = __ldcs(s4 + i);
    const uint32_t k[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t x = key_encode<KIND, DESC>(k[e]);
      atomicAdd(&h[x & 2047u], 1u);
      atomicAdd(&h[2048 + ((x >> 11) & 2047u)], 1u);
      atomicAdd(&h[4096 + (x >> 22)], 1u);
    }
  }
  for (uint32_t i = nv * 4 + blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
    const uint32_t x = key_encode<KIND, DESC>(src[i]);
    atomicAdd(&h[x & 2047u], 1u);
    atomicAdd(&h[2048 + ((x >> 11) & 2047u)], 1u);
    atomicAdd(&h[4096 + (x >> 22)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += NT) {
    uint32_t s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += sh[r * NB + i];
    if (s) atomicAdd(&hist[i], s);
  }
}

}  // namespace bsort
