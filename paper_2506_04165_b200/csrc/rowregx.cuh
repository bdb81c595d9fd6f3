// rowregx.cuh -- the register row stream of rowreg.cuh for the other bucket
// shapes of the C3 K' sweep (BASELINE configs[2]): K' in {2, 4, 8} with
// B = 128 CPL buckets, CPL in {1, 2, 4}, B K' = 1024 candidates per row
// (K' = 2 / B = 512, K' = 4 / B = 256, K' = 8 / B = 128), and K' = 2 / B = 1024
// (2048 candidates: 64 slots per lane, packed to <= 32 before the sort).
//
// Same design, generalised (rowreg.cuh has the argument and the references):
//   * one warp per row; lane l owns the 4 CPL buckets 4 (l + 32 k) + j of the
//     CPL chunk columns k (8 bytes of every stride-row each) and streams the
//     chunk columns one after the other: every load is a 256-byte warp access;
//   * per chunk column the hit pass of rowreg.cuh (packed compare + packed
//     a * 2 + hit per word, tiles of 7 stride-rows through a staging tile),
//     the hits inserted into the bucket's K'-slot state in Alg. 1 order
//     (topk.cpp:80-102);
//   * M = the filled slots >= K proves the predicted level; otherwise the
//     maxima pass (K' disjoint groups of stride-rows per bucket), the bisection
//     of the K-th largest group maximum and a second hit pass; L = -inf takes
//     the exact path (Alg. 1 of every bucket, a sort of the B K' rank keys);
//   * stage 2: a bitonic sort of the 1024 slots in registers (32 per lane).
#pragma once

#include "rowreg.cuh"

namespace atkg {

template <int S, int KP>
__host__ __device__ constexpr int rx_group(int s) {
  int g = 0;
  while (g < KP - 1 && (g + 1) * S / KP <= s) ++g;
  return g;
}

// per warp: staging tile 2 KB | state [32 lanes][4 CPL buckets][K'] u32 (the sorted keys after the
// pass); a lane's slots are padded by 16 bytes so that the lanes' 16-byte accesses spread over the banks
template <int KP, int CPL>
__host__ __device__ constexpr uint32_t rx_lane_words() { return 4u * CPL * KP + 4; }
template <int KP, int CPL>
__host__ __device__ constexpr uint32_t rx_warp_smem() { return 8 * 256 + rx_lane_words<KP, CPL>() * 4 * 32; }

// insert e (code << 16 | position) into the K' slots sv[] kept in Alg. 1 order
template <int KP>
__device__ __forceinline__ bool rx_insert(uint32_t (&sv)[KP], uint32_t e) {
  if (sv[KP - 1] > (e | 0xffffu)) return false;  // value < v[K' - 1]
  const uint32_t eb = e & 0xffff0000u;
  bool above[KP];  // slot i stays above e (a later equal element never passes an earlier one)
#pragma unroll
  for (int i = 0; i < KP - 1; ++i) above[i] = sv[i] >= eb;
  above[KP - 1] = false;
#pragma unroll
  for (int i = KP - 1; i >= 1; --i) sv[i] = above[i] ? sv[i] : (above[i - 1] ? e : sv[i - 1]);
  sv[0] = above[0] ? sv[0] : e;
  return true;
}

template <int KP>
__device__ __forceinline__ void rx_load_state(const uint32_t* st, uint32_t (&sv)[KP]) {
  if constexpr (KP == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(st);
    sv[0] = v.x; sv[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < KP / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4*>(st)[q];
      sv[4 * q] = v.x; sv[4 * q + 1] = v.y; sv[4 * q + 2] = v.z; sv[4 * q + 3] = v.w;
    }
  }
}
template <int KP>
__device__ __forceinline__ void rx_store_state(uint32_t* st, const uint32_t (&sv)[KP]) {
  if constexpr (KP == 2) {
    *reinterpret_cast<uint2*>(st) = make_uint2(sv[0], sv[1]);
  } else {
#pragma unroll
    for (int q = 0; q < KP / 4; ++q)
      reinterpret_cast<uint4*>(st)[q] = make_uint4(sv[4 * q], sv[4 * q + 1], sv[4 * q + 2], sv[4 * q + 3]);
  }
}

// the hit pass over chunk column k (see rg_hits): bit 8 u + 6 - i of a tile's
// mask = element slot u of stride-row i (u = 0, 1, 2, 3 <-> element 0, 2, 1, 3)
template <int S, int KP, int CPL, bool POS>
__device__ __forceinline__ void rx_hits(const uint2* p, int k, uint32_t L2, uint32_t lane, uint2* stage, uint32_t* lst,
                                        uint32_t& nan) {
  constexpr int NB = (S + kRgTile - 1) / kRgTile;
  constexpr uint32_t B = 128u * CPL;
  const uint2* pk = p + k * 32;  // stride-row s of this chunk column: pk[s * 32 * CPL]
  uint2 buf[2][kRgTile];
#pragma unroll
  for (int i = 0; i < kRgTile; ++i)
    if (i < S) buf[0][i] = rg_ldg(pk + i * 32 * CPL);
  const uint8_t* col = reinterpret_cast<const uint8_t*>(stage + lane);
  uint32_t* stk = lst + (uint32_t)k * 4 * KP;  // the lane's buckets of this chunk column
  const uint32_t bk0 = 4 * (lane + 32 * (uint32_t)k);
#pragma unroll
  for (int bt = 0; bt < NB; ++bt) {
    if (bt + 1 < NB) {
#pragma unroll
      for (int i = 0; i < kRgTile; ++i) {
        const int s = (bt + 1) * kRgTile + i;
        if (s < S) buf[(bt + 1) & 1][i] = rg_ldg(pk + s * 32 * CPL);
      }
    }
    uint32_t ax = 0x3f803f80u, ay = 0x3f803f80u;
#pragma unroll
    for (int i = 0; i < kRgTile; ++i) {
      const int s = bt * kRgTile + i;
      if (s < S) {
        const uint2 v = buf[bt & 1][i];
        ax = rg_shl_add(ax, rg_geu1(v.x, L2));
        ay = rg_shl_add(ay, rg_geu1(v.y, L2));
        stage[(6 - i) * 32 + lane] = v;
      } else {
        ax = rg_shl_add(ax, 0u);
        ay = rg_shl_add(ay, 0u);
      }
    }
    uint32_t m = (ax & 0x007f007fu) | ((ay & 0x007f007fu) << 8);
    while (m) {
      uint32_t b;
      asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(m));
      m ^= 1u << b;
      const uint32_t r = b & 7u;
      const uint32_t j = ((b >> 2) & 2u) | (b >> 4);
      uint32_t val = *reinterpret_cast<const uint16_t*>(col + r * 256 + j * 2);
      if (!POS) {
        if ((val & 0x7fffu) > 0x7f80u) nan = 1u;
        val = asc_code16(val);
      }
      const uint32_t e = (val << 16) | ((uint32_t)(bt * kRgTile + 6) * B - r * B + bk0 + j);
      uint32_t sv[KP];
      rx_load_state<KP>(stk + j * KP, sv);
      if (rx_insert<KP>(sv, e)) rx_store_state<KP>(stk + j * KP, sv);
    }
  }
}

// the maxima pass: gm[(2 k + w) * KP + g] = maximum of group g of word w of chunk column k
template <int S, int KP, int CPL>
__device__ __forceinline__ void rx_max(const uint2* p, uint32_t (&gm)[2 * CPL * KP]) {
  constexpr int U = 14;
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
#pragma unroll
    for (int s0 = 0; s0 < S; s0 += U) {
      uint2 v[U];
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (s0 + i < S) v[i] = rg_ldg(p + k * 32 + (s0 + i) * 32 * CPL);
#pragma unroll
      for (int i = 0; i < U; ++i) {
        if (s0 + i < S) {
          const int g = rx_group<S, KP>(s0 + i);
          gm[(2 * k) * KP + g] = bmax_nan(gm[(2 * k) * KP + g], v[i].x);
          gm[(2 * k + 1) * KP + g] = bmax_nan(gm[(2 * k + 1) * KP + g], v[i].y);
        }
      }
    }
  }
}

template <int NG>
__device__ __forceinline__ uint32_t rx_count_ge(const uint32_t (&gm)[NG], uint32_t L2) {
  static_assert(NG <= 32, "one bit pair per register, two accumulators");
  uint32_t t0 = 0, t1 = 0;
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    if (i < 16) t0 |= rg_ge(gm[i], L2) & (0x00010001u << i);
    else t1 |= rg_ge(gm[i], L2) & (0x00010001u << (i - 16));
  }
  return __popc(t0) + __popc(t1);
}

// warp: the largest code t with at least K of the group maxima >= t (0: none)
template <int NG>
__device__ __forceinline__ uint32_t rx_bisect(const uint32_t (&gm)[NG], uint32_t K) {
  uint32_t cur = 0;
#pragma unroll 1
  for (int bit = 15; bit >= 0; --bit) {
    const uint32_t t = cur | (1u << bit);
    if (__reduce_add_sync(0xffffffffu, rx_count_ge<NG>(gm, rg_bits2(t))) >= K) cur = t;
  }
  return cur;
}

// The exact path: Alg. 1 of every bucket as the reference runs it (topk.cpp:
// 80-102, sentinels {-inf, 0} of topk.cpp:118-121), the B K' rank keys sorted
// as 32-bit keys (~code << 16 | position: bf16 values, n <= 65536), the first K written.
template <int S, int KP, int CPL>
__device__ __noinline__ void rx_exact(const uint16_t* xr, uint32_t lane, uint32_t K, uint32_t* srt, float* ov,
                                      uint32_t* oi) {
  constexpr uint32_t B = 128u * CPL;
#pragma unroll 1
  for (int q = 0; q < 4 * CPL; ++q) {
    const uint32_t bk = 4 * (lane + 32 * (uint32_t)(q >> 2)) + (q & 3);
    float v[KP];
    uint32_t ix[KP];
#pragma unroll
    for (int t = 0; t < KP; ++t) { v[t] = neg_inf(); ix[t] = 0; }
#pragma unroll 2
    for (int r = 0; r < S; ++r) {
      const uint32_t pos = r * B + bk;
      const float x = __uint_as_float((uint32_t)__ldg(xr + pos) << 16);
      const bool take = x >= v[KP - 1];
      v[KP - 1] = take ? x : v[KP - 1];
      ix[KP - 1] = take ? pos : ix[KP - 1];
#pragma unroll
      for (int t = KP - 1; t >= 1; --t) {
        const bool up = x > v[t - 1];
        const float va = v[t], vb = v[t - 1];
        v[t] = up ? vb : va;
        v[t - 1] = up ? va : vb;
        const uint32_t ia = ix[t], ib = ix[t - 1];
        ix[t] = up ? ib : ia;
        ix[t - 1] = up ? ia : ib;
      }
    }
#pragma unroll
    for (int t = 0; t < KP; ++t)
      srt[(lane * 4 * CPL + q) * KP + t] = ((~asc_code16(__float_as_uint(v[t]) >> 16) & 0xffffu) << 16) | ix[t];
  }
  __syncwarp();
  warp_bitonic_sort<uint32_t>(srt, 128u * CPL * KP, lane);
  for (uint32_t q = lane; q < K; q += 32) {
    ov[q] = __uint_as_float(code16_bits(~(srt[q] >> 16) & 0xffffu) << 16);
    oi[q] = srt[q] & 0xffffu;
  }
  __syncwarp();
}

// bitonic sort of NS keys per lane (element g = NS lane + i), every merge
// ascending (first step g <-> g ^ (size - 1)); the keys arrive as ascending
// runs of RUN
template <int NS, int RUN>
__device__ __forceinline__ void rx_sort(uint32_t (&k)[NS], uint32_t lane) {
#pragma unroll
  for (int size = 2 * RUN; size <= 32 * NS; size <<= 1) {
    if (size <= NS) {
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const int q = i ^ (size - 1);
        if (i < q) { const uint32_t x = k[i], y = k[q]; k[i] = min(x, y); k[q] = max(x, y); }
      }
    } else {
      const uint32_t lm = (uint32_t)(size / NS) - 1u;
      const bool lower = (lane & (uint32_t)(size / NS / 2)) == 0;
#pragma unroll
      for (int i = 0; i < NS / 2; ++i) {
        const uint32_t ya = __shfl_xor_sync(0xffffffffu, k[NS - 1 - i], lm);
        const uint32_t yb = __shfl_xor_sync(0xffffffffu, k[i], lm);
        k[i] = lower ? min(k[i], ya) : max(k[i], ya);
        k[NS - 1 - i] = lower ? min(k[NS - 1 - i], yb) : max(k[NS - 1 - i], yb);
      }
    }
#pragma unroll
    for (int dist = size >> 2; dist > 0; dist >>= 1) {
      if (dist >= NS) {
        const uint32_t ld = (uint32_t)(dist / NS);
        const bool lower = (lane & ld) == 0;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const uint32_t y = __shfl_xor_sync(0xffffffffu, k[i], ld);
          k[i] = lower ? min(k[i], y) : max(k[i], y);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NS; ++i)
          if ((i & dist) == 0) { const uint32_t x = k[i], y = k[i | dist]; k[i] = min(x, y); k[i | dist] = max(x, y); }
      }
    }
  }
}

// S stride-rows, K' = KP slots per bucket, B = 128 CPL buckets.  One CTA of
// NW warps per SM; rows, prediction and prologue as in row_reg_kernel.
template <int S, int KP, int CPL, int NW>
__global__ void __launch_bounds__(32 * NW, 1) row_regx_kernel(RgArgs a) {
  constexpr uint32_t B = 128u * CPL, n = B * S;
  constexpr int NBK = 4 * CPL, NS = NBK * KP, NG = 2 * CPL * KP;  // buckets, slots, packed group maxima per lane
  constexpr uint32_t WS = rx_warp_smem<KP, CPL>();
  static_assert(NG <= 32 && NS <= 64, "group maxima registers, slots per lane");
  extern __shared__ __align__(128) uint8_t rg_smem[];
  __shared__ uint32_t queue;
  __shared__ volatile uint32_t pred;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.k;
  uint8_t* wsm = rg_smem + (size_t)wid * WS;
  uint2* stage = reinterpret_cast<uint2*>(wsm);
  uint32_t* state = reinterpret_cast<uint32_t*>(wsm + 8 * 256);  // [32 lanes][NBK][KP] (+ pad), 0 = empty
  constexpr uint32_t LS = rx_lane_words<KP, CPL>();
  uint32_t* lst = state + lane * LS;
  const uint64_t r0 = a.rows * blockIdx.x / gridDim.x, r1 = a.rows * (blockIdx.x + 1) / gridDim.x;
  const uint32_t nrows = (uint32_t)(r1 - r0);
  if (threadIdx.x == 0) {
    queue = 0;
    pred = 0xffffffffu;
  }
  // ---- prologue: the first prediction from the CTA's first row ------------
  if (a.force == 0) {
    const uint2* p0 = reinterpret_cast<const uint2*>(a.in + r0 * n) + lane;
    uint32_t pm[NG];
#pragma unroll
    for (int i = 0; i < NG; ++i) pm[i] = 0xff80ff80u;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
#pragma unroll
      for (int g = 0; g < KP; ++g) {
        const int s1 = g == KP - 1 ? S : (g + 1) * S / KP;
        for (int s = g * S / KP + (int)wid; s < s1; s += NW) {
          const uint2 v = rg_ldg(p0 + k * 32 + s * 32 * CPL);
          pm[(2 * k) * KP + g] = bmax_nan(pm[(2 * k) * KP + g], v.x);
          pm[(2 * k + 1) * KP + g] = bmax_nan(pm[(2 * k + 1) * KP + g], v.y);
        }
      }
    }
    uint32_t* part = reinterpret_cast<uint32_t*>(wsm);  // [NG][32] per warp, from the start of its region
#pragma unroll
    for (int i = 0; i < NG; ++i) part[i * 32 + lane] = pm[i];
    __syncthreads();
    static_assert(2 * NG * 128 <= WS, "partial maxima and the folded result share warp 0's region");
    uint32_t* res = reinterpret_cast<uint32_t*>(rg_smem + NG * 128);  // behind warp 0's partials: [NG][32]
    for (uint32_t q = wid; q < (uint32_t)NG; q += NW) {  // a warp folds register q of every warp's share
      uint32_t m = 0xff80ff80u;
      for (uint32_t w2 = 0; w2 < (uint32_t)NW; ++w2)
        m = bmax_nan(m, reinterpret_cast<const uint32_t*>(rg_smem + (size_t)w2 * WS)[q * 32 + lane]);
      res[q * 32 + lane] = m;
    }
    __syncthreads();
    if (wid == 0) {
      uint32_t gm0[NG];
#pragma unroll
      for (int i = 0; i < NG; ++i) gm0[i] = res[i * 32 + lane];
      const uint32_t cur = rx_bisect<NG>(gm0, K);
      if (cur > kRgKeyNegInf && lane == 0) pred = cur << 4;
    }
  }
  __syncthreads();

  auto pop = [&]() {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(&queue, 1u);
    return __shfl_sync(0xffffffffu, r, 0);
  };
#pragma unroll 1
  for (;;) {
    const uint32_t rr = pop();
    if (rr >= nrows) break;
    const uint64_t row = r0 + rr;
    const uint16_t* xr = a.in + row * n;
    const uint2* p = reinterpret_cast<const uint2*>(xr) + lane;
    float* ov = a.out_v + row * K;
    uint32_t* oi = a.out_i + row * K;

    auto clear_state = [&]() {
#pragma unroll
      for (int q = 0; q < NS / 4; ++q) reinterpret_cast<uint4*>(lst)[q] = make_uint4(0, 0, 0, 0);
    };
    auto filled = [&]() {  // M = sum_b min(K', c_b)
      uint32_t f = 0;
#pragma unroll
      for (int q = 0; q < NS / 4; ++q) {
        const uint4 sv = reinterpret_cast<const uint4*>(lst)[q];
        f += (sv.x ? 1u : 0u) + (sv.y ? 1u : 0u) + (sv.z ? 1u : 0u) + (sv.w ? 1u : 0u);
      }
      return __reduce_add_sync(0xffffffffu, f);
    };
    uint32_t nan = 0;
    auto hit_pass = [&](uint32_t Lk) {
      clear_state();
      const uint32_t L2 = rg_bits2(Lk);
      if (Lk > 0x8000u) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) rx_hits<S, KP, CPL, true>(p, k, L2, lane, stage, lst, nan);
      } else {
#pragma unroll
        for (int k = 0; k < CPL; ++k) rx_hits<S, KP, CPL, false>(p, k, L2, lane, stage, lst, nan);
      }
      return filled();
    };
    const uint32_t pr = pred;  // running mean of the rows' K-th candidate levels, x 16
    const bool have = pr != 0xffffffffu && a.force == 0;
    uint32_t Lkey = max(pr >> 4, kRgKeyNegInf + 1 + a.margin) - a.margin;
    uint32_t M = have ? hit_pass(Lkey) : 0u;
    bool exact = a.force == 2;
    if (M < K) {  // no usable prediction: maxima, the guaranteed level, a second hit pass
      uint32_t gm[NG];
#pragma unroll
      for (int i = 0; i < NG; ++i) gm[i] = 0xff80ff80u;
      rx_max<S, KP, CPL>(p, gm);
      uint32_t mm = gm[0];
#pragma unroll
      for (int i = 1; i < NG; ++i) mm = bmax_nan(mm, gm[i]);
      nan = ((mm & 0x7fffu) > 0x7f80u || ((mm >> 16) & 0x7fffu) > 0x7f80u) ? 1u : 0u;
      if (__reduce_or_sync(0xffffffffu, nan)) {  // the reference rejects the input
        if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
        continue;
      }
      Lkey = rx_bisect<NG>(gm, K);
      if (Lkey <= kRgKeyNegInf) exact = true;
      else M = hit_pass(Lkey);
    }
    if (exact) {
      __syncwarp();
      rx_exact<S, KP, CPL>(xr, lane, K, state, ov, oi);
      continue;
    }
    const bool posmode = Lkey > 0x8000u;
    // ---- stage 2: sort the lane's slots with the warp's -----------------------
    constexpr int NK = NS > 32 ? 32 : NS;  // keys per lane in the sort
    uint32_t ks[NK];
    if constexpr (NS <= 32) {  // each bucket's K' slots are already ascending
#pragma unroll
      for (int q = 0; q < NS / 4; ++q) {
        const uint4 sv = reinterpret_cast<const uint4*>(lst)[q];
        ks[4 * q] = sv.x ^ 0xffff0000u;
        ks[4 * q + 1] = sv.y ^ 0xffff0000u;
        ks[4 * q + 2] = sv.z ^ 0xffff0000u;
        ks[4 * q + 3] = sv.w ^ 0xffff0000u;
      }
      rx_sort<NK, KP>(ks, lane);
    } else {
      // 64 slots per lane, ~12 filled: the lane packs its filled slots to the front of its region
      // (the write index never passes the read index) and sorts 32; a lane with more goes exact
      uint32_t c = 0;
#pragma unroll 4
      for (int q = 0; q < NS; ++q) {
        const uint32_t e = lst[q];
        if (e) {
          lst[c] = e;
          ++c;
        }
      }
      if (__reduce_max_sync(0xffffffffu, c) > 32u) {
        __syncwarp();
        rx_exact<S, KP, CPL>(xr, lane, K, state, ov, oi);
        continue;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 sv = reinterpret_cast<const uint4*>(lst)[q];
        ks[4 * q] = (uint32_t)(4 * q) < c ? sv.x ^ 0xffff0000u : 0xffff0000u;
        ks[4 * q + 1] = (uint32_t)(4 * q + 1) < c ? sv.y ^ 0xffff0000u : 0xffff0000u;
        ks[4 * q + 2] = (uint32_t)(4 * q + 2) < c ? sv.z ^ 0xffff0000u : 0xffff0000u;
        ks[4 * q + 3] = (uint32_t)(4 * q + 3) < c ? sv.w ^ 0xffff0000u : 0xffff0000u;
      }
      rx_sort<NK, 1>(ks, lane);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NK / 4; ++q)  // the lane's own region again: element NK lane + i
      reinterpret_cast<uint4*>(lst)[q] = make_uint4(ks[4 * q], ks[4 * q + 1], ks[4 * q + 2], ks[4 * q + 3]);
    __syncwarp();
    if (posmode && ((~(state[0] >> 16)) & 0x7fffu) > 0x7f80u) nan = 1u;  // a NaN hit sorts first
    if (__reduce_or_sync(0xffffffffu, nan)) {
      if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
      __syncwarp();
      continue;
    }
    for (uint32_t x = lane; x < K; x += 32) {  // sorted element x lives in lane x / NK
      const uint32_t key = state[(x / NK) * LS + x % NK], code = ~(key >> 16) & 0xffffu;
      ov[x] = __uint_as_float((posmode ? code : code16_bits(code)) << 16);
      oi[x] = key & 0xffffu;
    }
    const uint32_t ck = ~(state[((K - 1) / NK) * LS + (K - 1) % NK] >> 16) & 0xffffu;
    const uint32_t Lstar = posmode ? (ck | 0x8000u) : ck;
    if (lane == 0) {
      const uint32_t pv = pred;
      pred = pv == 0xffffffffu ? Lstar << 4 : (uint32_t)((int)pv + (((int)(Lstar << 4) - (int)pv) >> 2));
    }
    __syncwarp();
  }
}

}  // namespace atkg
