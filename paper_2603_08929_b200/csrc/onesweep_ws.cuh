// onesweep_ws.cuh — warp-specialised LSD pass for the look-back ranking modes (RANK_RUN2,
// RANK_STABLE).  Same algorithm and output as k_onesweep_pass; what changes is who waits for
// the decoupled look-back.  In k_onesweep_pass every thread of the CTA idles at a barrier while
// 256 threads walk (≈ 1.1 ms of a 4.2 ms RUN2 pass on 2^30 keys).  Here a CTA has
//   * RT "ranker" threads: wait for the tile's TMA bulk copy, rank it, publish its aggregate,
//     restage it in digit order, hand it over and move on to the next tile at once;
//   * 256 "writer" threads (one per digit): walk the look-back for the handed-over tile, publish
//     its inclusive prefix, write the tile out, and re-arm the freed buffer with the next tile.
// Three tile buffers rotate (ranked / being written / in flight), so rankers never wait for a walk.
// Hand-over and buffer reuse are ordered by named barriers (bar.arrive by rankers, bar.sync by
// writers, one id per buffer) and by the buffers' mbarriers (TMA completion).
#pragma once
#include "onesweep.cuh"

namespace bsort {

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ bool named_bar_or(uint32_t id, uint32_t n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, %2, %3, p;\n selp.u32 %0, 1, 0, q;\n}\n"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// block_exclusive_scan over the NT threads that share named barrier BAR.
template <int NT, uint32_t BAR, typename T>
__device__ __forceinline__ T group_exclusive_scan(T v, T* warp_tot) {
  constexpr int NW = NT / 32;
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) warp_tot[warp] = inc;
  named_bar_sync(BAR, NT);
  if (warp == 0) {
    T w = (lane < (uint32_t)NW) ? warp_tot[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane < (uint32_t)NW) warp_tot[lane] = wi - w;
  }
  named_bar_sync(BAR, NT);
  return warp_tot[warp] + inc - v;
}

template <int RT, int ITEMS, typename U, bool KV = false>
struct PassSmemWS {
  static constexpr int RW = RT / 32;
  static constexpr int TILE = RT * ITEMS;
  static constexpr int HALF_WORDS = 272;
  static constexpr size_t buf_off = 0;  // U[3][TILE]
  static constexpr size_t rows_off = align_up(buf_off + 3 * sizeof(U) * TILE, 16);
  static constexpr size_t bcnt_off = align_up(rows_off + 2 * HALF_WORDS * 4 * RW, 16);
  static constexpr size_t meta_off = align_up(bcnt_off + sizeof(uint32_t) * 512 * BREP, 16);  // uint2[3][256]
  static constexpr size_t gofs_off = align_up(meta_off + 8 * 3 * 256, 16);  // u64[256], writers
  static constexpr size_t wt_off = align_up(gofs_off + 8 * 256, 16);        // u32[RW + 1], rankers
  static constexpr size_t mbar_off = align_up(wt_off + 4 * (RW + 1), 16);   // u64[3]
  static constexpr size_t tile_off = mbar_off + 32;                         // u32[3] tile id per buffer
  static constexpr size_t vbuf_off = align_up(tile_off + 16, 128);          // KV: u32 values [3][TILE]
  static constexpr size_t bytes = align_up(vbuf_off + (KV ? 3 * sizeof(uint32_t) * TILE : 0), 128);
};

constexpr uint32_t WS_BAR_R = 1, WS_BAR_W = 2, WS_BAR_STAGED = 3;  // + buffer index (3 ids)

// Grid: one CTA of RT + 256 threads per SM (persistent).  BULK only (both ping-pong buffers, and
// for KV both value buffers, 16-byte aligned), no remote write-out.  KV: a u32 payload per key
// (§8 N3) is bulk-copied with its tile, restaged beside the keys and written out with them.
template <typename U, int RT, int ITEMS, typename DescT, typename DigitF, int MODE, int LBG = 8, int MINB = 1,
          bool KV = false>
__global__ void __launch_bounds__(RT + 256, MINB)
    k_onesweep_pass_ws(const U* a_ptr, U* b_ptr, uint64_t n, DigitF digit,
                       const unsigned long long* __restrict__ bases, DescT* __restrict__ lookback,
                       uint32_t* __restrict__ tile_counter, uint32_t num_tiles, const PassPlan* __restrict__ plan,
                       int pass, KvPtrs kvp = {}, unsigned long long* __restrict__ gcount = nullptr,
                       uint32_t only_fewruns = 0) {
  static_assert(MODE == RANK_RUN2 || MODE == RANK_STABLE || MODE == RANK_UNSTABLE, "no J01");
  constexpr bool LOOKBACK = MODE != RANK_UNSTABLE;
  static_assert(RT >= 256 && RT % 32 == 0, "at least one ranker per digit");
  using L = PassSmemWS<RT, ITEMS, U, KV>;
  using LB = LookbackBits<DescT>;
  constexpr int TILE = L::TILE;
  constexpr int SEG = 32 * ITEMS;
  constexpr int HW = L::HALF_WORDS;
  constexpr bool RUNS = MODE == RANK_RUN2;
  static_assert(TILE < (1 << 22), "rank fits 22 bits");
  static_assert((TILE * sizeof(U)) % 16 == 0, "bulk copies need 16-byte tiles");
  static_assert(TILE % 256 == 0, "writers stride the tile by 256");
  extern __shared__ __align__(128) unsigned char smem[];
  U* bufs = reinterpret_cast<U*>(smem + L::buf_off);
  uint32_t* rows = reinterpret_cast<uint32_t*>(smem + L::rows_off);
  uint32_t* bcnt = reinterpret_cast<uint32_t*>(smem + L::bcnt_off);
  uint2* meta = reinterpret_cast<uint2*>(smem + L::meta_off);
  unsigned long long* gofs = reinterpret_cast<unsigned long long*>(smem + L::gofs_off);
  uint32_t* wt = reinterpret_cast<uint32_t*>(smem + L::wt_off);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L::mbar_off);
  volatile uint32_t* tile_s = reinterpret_cast<volatile uint32_t*>(smem + L::tile_off);
  uint32_t* vbufs = reinterpret_cast<uint32_t*>(smem + L::vbuf_off);
  (void)vbufs;

  const U* src = a_ptr;
  U* dst = b_ptr;
  const uint32_t* vsrc = kvp.va;
  uint32_t* vdst = kvp.vb;
  if (plan != nullptr) {
    if (plan->skip[pass]) return;
    if constexpr (MODE == RANK_RUN2) {
      if (pass == 1 && plan->j01) return;  // the J01 launch of this pass runs instead
    }
    // launched as the few-runs alternative of a k_pass2 launch: works only when the plan says so
    if (only_fewruns && !((plan->fewruns >> pass) & 1u)) return;
    if (plan->src_alt[pass]) {
      src = b_ptr;
      dst = const_cast<U*>(a_ptr);
      vsrc = kvp.vb;
      vdst = const_cast<uint32_t*>(kvp.va);
    }
  }
  const uint32_t t = threadIdx.x;
  auto tile_valid = [&](uint32_t tile) -> uint32_t {
    const uint64_t b = (uint64_t)tile * TILE;
    return (uint32_t)min64((uint64_t)TILE, n - b);
  };
  auto bulk_keys = [&](uint32_t valid) -> uint32_t {
    return (uint32_t)((valid * sizeof(U)) & ~(size_t)15) / (uint32_t)sizeof(U);
  };
  // one thread: give buffer b the next tile (or, past the end, complete its phase empty)
  auto bulk_vals = [&](uint32_t valid) -> uint32_t { return valid & ~3u; };
  auto refill = [&](int b) {
    const uint32_t id = atomicAdd(tile_counter, 1u);
    tile_s[b] = id;
    if (id < num_tiles) {
      const uint32_t v = tile_valid(id);
      if constexpr (KV)
        bulk_load(bufs + b * TILE, src + (uint64_t)id * TILE, bulk_keys(v) * (uint32_t)sizeof(U), &mbar[b],
                  vbufs + b * TILE, vsrc + (uint64_t)id * TILE, bulk_vals(v) * 4u);
      else
        bulk_load(bufs + b * TILE, src + (uint64_t)id * TILE, bulk_keys(v) * (uint32_t)sizeof(U), &mbar[b]);
    } else {
      mbar_arrive(&mbar[b]);
    }
  };
  if (t == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&mbar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < 3; ++b) refill(b);
  }
  __syncthreads();

  if (t < (uint32_t)RT) {
    // ------------------------------------------------------------------ rankers
    const uint32_t lane = t & 31, warp = t >> 5;
    const uint32_t half = lane >> 4, l16 = lane & 15, lt16 = (1u << l16) - 1u;
    uint32_t* wc = rows + (2 * warp + half) * HW;
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % 3;
      U* buf = bufs + slot * TILE;
      mbar_wait(&mbar[slot], (it / 3) & 1u);
      const uint32_t tile = tile_s[slot];
      if (tile >= num_tiles) break;
      const uint64_t tile_base = (uint64_t)tile * TILE;
      const uint32_t valid = tile_valid(tile);
      const bool full = valid == (uint32_t)TILE;
      named_bar_sync(WS_BAR_R, RT);  // the previous tile's reads of the tables are done

      if constexpr (MODE == RANK_STABLE) {
#pragma unroll
        for (int j = 0; j < 16; ++j) wc[l16 + 16 * j] = 0;
      }
      if constexpr (MODE != RANK_STABLE)
        for (int j = t; j < 512 * BREP / 4; j += RT) reinterpret_cast<uint4*>(bcnt)[j] = make_uint4(0, 0, 0, 0);

      // keys -> registers, half-warp index order (as k_onesweep_pass)
      const uint32_t seg = warp * SEG + half * (16 * ITEMS) + l16;
      U keys[ITEMS];
      uint32_t vals[KV ? ITEMS : 1];
      uint32_t* vbuf = vbufs + slot * TILE;
      (void)vals;
      (void)vbuf;
      U first_key = U(0), last_key = U(0);
      const uint32_t bk = bulk_keys(valid);
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const uint32_t i = seg + 16u * k;
        keys[k] = full ? buf[i] : (i < bk ? buf[i] : (i < valid ? ldg_nc(src + tile_base + i) : U(0)));
      }
      if constexpr (KV) {
        const uint32_t bv = bulk_vals(valid);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t i = seg + 16u * k;
          vals[k] = full ? vbuf[i] : (i < bv ? vbuf[i] : (i < valid ? ldg_nc(vsrc + tile_base + i) : 0u));
        }
      }
      if constexpr (RUNS) {
        first_key = bk > 0 ? buf[0] : ldg_nc(src + tile_base);
        last_key = valid - 1 < bk ? buf[valid - 1] : ldg_nc(src + tile_base + valid - 1);
      }

      bool unstable_rank = MODE == RANK_UNSTABLE;
      U low_first = U(0), low_last = U(0);
      if constexpr (MODE == RANK_UNSTABLE) {
        named_bar_sync(WS_BAR_R, RT);  // counters zeroed before the atomics
      } else if constexpr (MODE == RANK_RUN2) {
        U lo;
        digit.digit_low(first_key, &low_first);
        digit.digit_low(last_key, &low_last);
        bool bad = false;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          digit.digit_low(keys[k], &lo);
          bad |= (full || seg + 16u * k < valid) && lo != low_first && lo != low_last;
        }
        unstable_rank = !named_bar_or(WS_BAR_R, RT, bad);  // also orders the zeroing before the atomics
      }

      uint32_t info[ITEMS];
      if (unstable_rank) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          if (full || seg + 16u * k < valid) {
            U lo;
            uint32_t bin = digit.digit_low(keys[k], &lo);
            if constexpr (RUNS) bin |= (lo != low_first) ? 256u : 0u;
            info[k] = bin | (atomicAdd(&bcnt[bin * BREP + (lane & (BREP - 1))], 1u) << 9);
          } else {
            info[k] = 0xFFFFFFFFu;
          }
        }
      } else {
        if constexpr (MODE == RANK_RUN2) {  // a RUN2 tile that falls back: zero this warp's tables
          // now (the previous tile's reads of them ended before its barrier B / our restage)
#pragma unroll
          for (int j = 0; j < 16; ++j) wc[l16 + 16 * j] = 0;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t d = (full || seg + 16u * k < valid) ? digit(keys[k]) : 255u;
          atomicOr(&wc[d], 1u << l16);
          __syncwarp();
          const uint32_t w = wc[d];
          const uint32_t peers = w & 0xFFFFu;
          const uint32_t below = __popc(peers & lt16);
          const uint32_t old = w >> 16;
          __syncwarp();
          if ((peers >> l16) == 1u) wc[d] = (old + below + 1u) << 16;
          info[k] = d | ((old + below) << 9);
        }
      }
      named_bar_sync(WS_BAR_R, RT);  // (A) counters complete

      uint32_t total = 0;
      if (t < 256) {
        if (unstable_rank) {
          const uint4 r0 = reinterpret_cast<const uint4*>(bcnt)[t];
          total = r0.x + r0.y + r0.z + r0.w;
          if constexpr (RUNS) {
            const uint4 r1 = reinterpret_cast<const uint4*>(bcnt)[256 + t];
            total += r1.x + r1.y + r1.z + r1.w;
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2 * L::RW; ++h) total += rows[h * HW + t] >> 16;
          if (!full && t == 255) total -= (uint32_t)TILE - valid;
        }
        if constexpr (LOOKBACK)
          st_relaxed(&lookback[(uint64_t)tile * 256 + t], (tile == 0 ? LB::INC : LB::AGG) | DescT(total));
      }
      const uint32_t tile_excl = group_exclusive_scan<RT, WS_BAR_R>(t < 256 ? total : 0u, wt);
      if (t < 256) {
        if (unstable_rank) {
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
        } else {
          uint32_t run = tile_excl;
#pragma unroll
          for (int h = 0; h < 2 * L::RW; ++h) {
            const uint32_t c = rows[h * HW + t] >> 16;
            rows[h * HW + t] = run;
            run += c;
          }
        }
        meta[slot * 256 + t] = make_uint2(tile_excl, total);
      }
      named_bar_sync(WS_BAR_R, RT);  // (B) offsets ready; every ranker has read buf

      if (unstable_rank) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
          if (info[k] != 0xFFFFFFFFu) {
            const uint32_t pos = bcnt[(info[k] & 0x1FFu) * BREP + (lane & (BREP - 1))] + (info[k] >> 9);
            buf[pos] = keys[k];
            if constexpr (KV) vbuf[pos] = vals[k];
          }
      } else {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t pos = wc[info[k] & 0xFFu] + (info[k] >> 9);
          buf[pos] = keys[k];
          if constexpr (KV) vbuf[pos] = vals[k];
        }
      }
      named_bar_arrive(WS_BAR_STAGED + slot, RT + 256);  // hand the staged tile to the writers
    }
  } else {
    // ------------------------------------------------------------------ writers
    const uint32_t w = t - RT;  // digit of this writer
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % 3;
      const uint32_t tile = tile_s[slot];
      if (tile >= num_tiles) break;
      const U* buf = bufs + slot * TILE;
      const uint32_t* vbuf = vbufs + slot * TILE;
      (void)vbuf;
      named_bar_sync(WS_BAR_STAGED + slot, RT + 256);  // rankers staged this tile
      const uint2 m = meta[slot * 256 + w];
      unsigned long long excl = 0;
      if constexpr (LOOKBACK) {
        if (tile > 0) {
          const DescT e = lookback_walk<LBG>(lookback, w, tile);
          st_relaxed(&lookback[(uint64_t)tile * 256 + w], LB::INC | (e + DescT(m.y)));
          excl = (unsigned long long)e;
        }
      } else {
        if (m.y) excl = atomicAdd(&gcount[w], (unsigned long long)m.y);  // tile order is free
      }
      gofs[w] = bases[w] + excl - m.x;
      named_bar_sync(WS_BAR_W, 256);
      const uint32_t valid = tile_valid(tile);
#pragma unroll 4
      for (uint32_t i = w; i < valid; i += 256) {
        const U x = buf[i];
        const unsigned long long o = gofs[digit(x)] + i;
        dst[o] = x;
        if constexpr (KV) vdst[o] = vbuf[i];
      }
      named_bar_sync(WS_BAR_W, 256);  // buffer and gofs fully read
      if (w == 0) refill((int)slot);
    }
  }
}

}  // namespace bsort
