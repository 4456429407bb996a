// pass3.cuh — a4 (round 2): non-warp-specialised LSD scatter pass, several CTAs per SM.
//
// Same ranking as k_pass2 (pass2.cuh: lane-ordered per-warp atomics for stable passes, lane-banked
// tables for unstable ones, chunked look-back, encoded intermediates), but every thread of a CTA
// ranks, scans, stages and writes its tile, and MINB CTAs share an SM: while one CTA waits at a
// barrier, a global atomic or a look-back walk, the others issue.  Two TMA tile buffers per CTA;
// a tile is staged in place in its own buffer (its keys are in registers by then) and the other
// buffer is being filled meanwhile.
#pragma once
#include "pass2.cuh"

namespace bsort {

template <int NT, int ITEMS, typename U, int MODE>
struct Pass3Smem {
  static constexpr int NW = NT / 32;
  static constexpr int TILE = NT * ITEMS;
  static constexpr int KPV = 16 / (int)sizeof(U);
  static constexpr int BUFK = TILE + KPV;
  // STABLE: per-warp counters [NW][256]; UNSTABLE: lane-banked table [256][32] (u16 halves
  // alternate between consecutive tiles)
  static constexpr int CNT_WORDS = MODE == R2_STABLE ? NW * 256 : 256 * 32;
  static constexpr size_t buf_off = 0;  // U[2][BUFK]
  static constexpr size_t cnt_off = align_up(buf_off + 2 * sizeof(U) * BUFK, 16);
  static constexpr size_t gofs_off = align_up(cnt_off + 4 * (size_t)CNT_WORDS, 16);  // u32[256]
  static constexpr size_t wt_off = align_up(gofs_off + 4 * 256, 16);                  // u32[NW + 1]
  static constexpr size_t mbar_off = align_up(wt_off + 4 * (NW + 1), 16);             // u64[2]
  static constexpr size_t slot_off = mbar_off + 16;                                   // SlotInfo[2]
  static constexpr size_t bytes = align_up(slot_off + 64, 128);
};

template <typename U, int KIND, bool DESC, int SHIFT, int NT, int ITEMS, int MODE, bool CHUNKED = false, int LBV = 2,
          int MINB = 2>
__global__ void __launch_bounds__(NT, MINB)
    k_pass3(const U* a_ptr, U* b_ptr, uint64_t n, const unsigned long long* __restrict__ bases,
            uint32_t* __restrict__ lookback, unsigned long long* __restrict__ gcount,
            uint32_t* __restrict__ tile_counter, uint32_t num_tiles, const PassPlan* __restrict__ plan, int pass,
            uint32_t flags, ChunkMap cm) {
  using L = Pass3Smem<NT, ITEMS, U, MODE>;
  using LB = LookbackBits<uint32_t>;
  constexpr int TILE = L::TILE;
  constexpr int NW = L::NW;
  constexpr int SEG = 32 * ITEMS;
  constexpr uint32_t KS = sizeof(U) == 4 ? 2 : 3;
  static_assert(NT >= 256 && NT % 32 == 0, "one thread per digit in the scan");
  static_assert(MODE != R2_UNSTABLE || TILE * sizeof(U) < (1 << 16), "staging offsets fit u16");
  static_assert((TILE * sizeof(U)) % 16 == 0 && L::bytes < (1 << 18), "16-byte tiles; 18-bit addresses");
  static_assert(!CHUNKED || MODE == R2_STABLE, "chunks are look-back chains");
  extern __shared__ __align__(128) unsigned char smem[];
  U* bufs = reinterpret_cast<U*>(smem + L::buf_off);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L::cnt_off);
  uint32_t* gofs = reinterpret_cast<uint32_t*>(smem + L::gofs_off);
  uint32_t* wt = reinterpret_cast<uint32_t*>(smem + L::wt_off);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L::mbar_off);
  volatile SlotInfo* slots = reinterpret_cast<volatile SlotInfo*>(smem + L::slot_off);
  const uint32_t smem_base = smem_u32(smem);

  const U* src = a_ptr;
  U* dst = b_ptr;
  bool enc_in = (flags & P2_ENC) != 0, dec_out = (flags & P2_DEC) != 0;
  if (plan != nullptr) {
    if (plan->skip[pass]) return;
    if (plan->src_alt[pass]) {
      src = b_ptr;
      dst = const_cast<U*>(a_ptr);
    }
    enc_in = plan->first == (uint32_t)pass;
    dec_out = plan->last == (uint32_t)pass;
  }
  const uint32_t t = threadIdx.x;
  auto refill = [&](int b) {
    const uint32_t id = atomicAdd(tile_counter, 1u);
    if (id >= num_tiles) {
      slots[b].lin = P2_END;
      mbar_arrive(&mbar[b]);
      return;
    }
    uint32_t lin, len, chunk = 0, first;
    unsigned long long start;
    if constexpr (CHUNKED) {
      const uint32_t v = cm.disp[id];
      chunk = v >> 24;
      const uint32_t k = v & 0xFFFFFFu;
      const unsigned long long cs = cm.cstart[chunk], ce = cm.cstart[chunk + 1];
      start = cs + (unsigned long long)k * TILE;
      len = (uint32_t)min64((uint64_t)TILE, ce - start);
      lin = cm.ctile[chunk] + k;
      first = k == 0;
    } else {
      lin = id;
      start = (unsigned long long)id * TILE;
      len = (uint32_t)min64((uint64_t)TILE, n - start);
      first = id == 0;
    }
    const uintptr_t s0 = (uintptr_t)(src + start), s1 = (uintptr_t)(src + start + len);
    const uintptr_t a0 = s0 & ~(uintptr_t)15;
    const uintptr_t a1 = start + len == n ? s1 & ~(uintptr_t)15 : (s1 + 15) & ~(uintptr_t)15;
    slots[b].lin = lin;
    slots[b].len = len;
    slots[b].off = (uint32_t)((s0 - a0) / sizeof(U));
    slots[b].bk = a1 > s0 ? (uint32_t)min64(len, (a1 - s0) / sizeof(U)) : 0u;
    slots[b].chunk = chunk;
    slots[b].first = first;
    slots[b].start = start;
    bulk_load(bufs + b * L::BUFK, reinterpret_cast<const void*>(a0), a1 > a0 ? (uint32_t)(a1 - a0) : 0u, &mbar[b]);
  };
  if (t == 0) {
    for (int b = 0; b < 2; ++b) mbar_init(&mbar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < 2; ++b) refill(b);
  }
  if constexpr (MODE == R2_UNSTABLE) {
    for (int i = t; i < L::CNT_WORDS / 4; i += NT) reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();

  const uint32_t lane = t & 31, warp = t >> 5;
  const uint32_t wcnt_a = smem_base + (uint32_t)L::cnt_off + warp * 1024u;
  const uint32_t lane_a = smem_base + (uint32_t)L::cnt_off + lane * 4u;
  const uint32_t seg = warp * SEG + lane;
  for (uint32_t it = 0;; ++it) {
    const uint32_t b = it & 1u;
    if constexpr (MODE == R2_STABLE) {
      uint4* w4 = reinterpret_cast<uint4*>(cnt + warp * 256);
      w4[lane] = make_uint4(0, 0, 0, 0);
      w4[lane + 32] = make_uint4(0, 0, 0, 0);
    }
    mbar_wait(&mbar[b], (it >> 1) & 1u);
    const uint32_t lin = slots[b].lin;
    if (lin == P2_END) break;
    const uint32_t valid = slots[b].len;
    const bool first_tile = slots[b].first != 0;
    const uint32_t chunk = slots[b].chunk;
    (void)chunk;
    const uint32_t buf_a = smem_base + (uint32_t)L::buf_off + b * (uint32_t)(L::BUFK * sizeof(U));
    const uint32_t ibuf_a = buf_a + slots[b].off * (uint32_t)sizeof(U);
    const uint32_t hsh = (it & 1u) << 4;

    auto tile_body = [&](auto full_c) {
      constexpr bool FULL = decltype(full_c)::value;
      U keys[ITEMS];
      uint32_t rk[(ITEMS + 1) / 2];
#pragma unroll
      for (int j = 0; j < (ITEMS + 1) / 2; ++j) rk[j] = 0;
      if constexpr (FULL) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) keys[k] = s_ldk<U>(ibuf_a + (seg + 32u * k) * (uint32_t)sizeof(U));
      } else {
        const uint32_t bk = slots[b].bk;
        const U* gsrc = src + slots[b].start;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
          const uint32_t i = seg + 32u * k;
          keys[k] = i < bk ? s_ldk<U>(ibuf_a + i * (uint32_t)sizeof(U)) : (i < valid ? ldg_nc(gsrc + i) : U(0));
        }
      }
      if (enc_in) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) keys[k] = key_encode<KIND, DESC>(keys[k]);
      }
      auto counter = [&](U key) -> uint32_t {
        const uint32_t d = p2_digit<SHIFT>(key);
        if constexpr (MODE == R2_STABLE)
          return wcnt_a + d * 4u;
        else
          return lane_a + d * 128u;
      };
      if constexpr (MODE == R2_STABLE) __syncwarp();
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        if (FULL || seg + 32u * k < valid) {
          uint32_t r;
          if constexpr (MODE == R2_STABLE)
            r = s_atom_add(counter(keys[k]), 4u);
          else
            r = (s_atom_add(counter(keys[k]), 4u << hsh) >> hsh) & 0xFFFFu;
          rk[k >> 1] |= r << ((k & 1) * 16);
        }
      }
      __syncthreads();  // (A) counts complete, every key of the buffer is in registers

      // per-digit totals and tile offsets; global offsets of this tile's digit runs
      uint32_t tot = 0, upper = 0;
      if (t < 256) {
        if constexpr (MODE == R2_STABLE) {
#pragma unroll
          for (int w = 0; w < NW; ++w) tot += cnt[w * 256 + t];
          tot >>= 2;
          st_relaxed(&lookback[lb2_index(lin, t)], (first_tile ? LB::INC : LB::AGG) | tot);
        } else {
          const uint32_t qr = t & 7u;
          const uint4* row = reinterpret_cast<const uint4*>(cnt + t * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t q = (uint32_t)(i + qr) & 7u;
            if (q == 0) upper = tot;
            const uint4 v = row[q];
            tot += ((v.x >> hsh) & 0xFFFFu) + ((v.y >> hsh) & 0xFFFFu) + ((v.z >> hsh) & 0xFFFFu) +
                   ((v.w >> hsh) & 0xFFFFu);
          }
          if (qr == 0) upper = tot;
          tot >>= 2;
          upper >>= 2;
        }
      }
      unsigned long long g0 = 0;
      if (t < 256) {  // issue the global step before the block scan (its latency overlaps)
        if constexpr (MODE == R2_STABLE) {
          uint32_t excl = 0;
          if (!first_tile) {
            excl = lookback_walk_v4<LBV>(lookback, t, lin);
            st_relaxed(&lookback[lb2_index(lin, t)], LB::INC | (excl + tot));
          }
          if constexpr (CHUNKED)
            g0 = (unsigned long long)cm.jp[chunk * 256 + t] + excl;
          else
            g0 = bases[t] + excl;
        } else {
          if (tot) g0 = bases[t] + atomicAdd(&gcount[t], (unsigned long long)tot);
        }
      }
      const uint32_t excl = block_exclusive_scan<NT>(t < 256 ? tot : 0u, wt, (uint32_t*)nullptr);
      if (t < 256) {
        gofs[t] = (uint32_t)(g0 - excl);
        if constexpr (MODE == R2_STABLE) {
          uint32_t run = buf_a + (excl << KS);
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const uint32_t c = cnt[w * 256 + t];
            cnt[w * 256 + t] = run;
            run += c << (KS - 2);
          }
        } else {
          const uint32_t qr = t & 7u;
          uint4* row = reinterpret_cast<uint4*>(cnt + t * 32);
          const uint32_t e = excl << KS;
          uint32_t run = e + ((tot - upper) << KS);
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
      __syncthreads();  // (B) staging addresses and global offsets ready

      constexpr int SG = 10;
#pragma unroll
      for (int k0 = 0; k0 < ITEMS; k0 += SG) {
        uint32_t pos[SG];
#pragma unroll
        for (int j = 0; j < SG; ++j) {
          const int k = k0 + j;
          if (k < ITEMS && (FULL || seg + 32u * k < valid)) {
            const uint32_t w = s_ld(counter(keys[k]));
            const uint32_t r = (rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
            if constexpr (MODE == R2_STABLE)
              pos[j] = w + (r << (KS - 2));
            else
              pos[j] = buf_a + ((w >> hsh) & 0xFFFFu) + (r << (KS - 2));
          }
        }
#pragma unroll
        for (int j = 0; j < SG; ++j) {
          const int k = k0 + j;
          if (k < ITEMS && (FULL || seg + 32u * k < valid)) s_st(pos[j], keys[k]);
        }
      }
    };
    if (valid == (uint32_t)TILE && slots[b].bk == (uint32_t)TILE)
      tile_body(std::true_type{});
    else
      tile_body(std::false_type{});
    __syncthreads();  // (C) staged

    constexpr int WB = 8;
    auto write_out = [&](auto full_c, auto dec_c) {
      constexpr bool FULL = decltype(full_c)::value;
      constexpr bool DEC = decltype(dec_c)::value;
      for (uint32_t base = t; base < valid; base += WB * NT) {
        U x[WB];
        uint32_t o[WB];
#pragma unroll
        for (int j = 0; j < WB; ++j) {
          const uint32_t i = base + j * NT;
          x[j] = (FULL || i < valid) ? s_ldk<U>(buf_a + i * (uint32_t)sizeof(U)) : U(0);
        }
#pragma unroll
        for (int j = 0; j < WB; ++j) o[j] = gofs[p2_digit<SHIFT>(x[j])];
        const U* db = dst + base;
        static_for<WB>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          if (FULL || base + j * NT < valid) {
            U v = x[j];
            if constexpr (DEC) v = key_decode<KIND, DESC>(v);
            st_global_at<j * NT * (int)sizeof(U)>(db, o[j], v);
          }
        });
      }
    };
    constexpr bool WHOLE = TILE % (WB * NT) == 0;
    if (WHOLE && valid == (uint32_t)TILE) {
      if (dec_out) write_out(std::bool_constant<WHOLE>{}, std::true_type{});
      else write_out(std::bool_constant<WHOLE>{}, std::false_type{});
    } else {
      if (dec_out) write_out(std::false_type{}, std::true_type{});
      else write_out(std::false_type{}, std::false_type{});
    }
    __syncthreads();  // (D) buffer b and gofs read
    if (t == 0) refill((int)b);
  }
}

}  // namespace bsort
