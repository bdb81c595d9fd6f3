// rowreg.cuh -- approx_top_k for short bf16 rows streamed ONCE from HBM, one
// warp per row, many rows in flight per SM: the FFN-activation config C3
// (rows of 14336 = 128 buckets x 112 stride-rows, K' = 4, K = 287).
//
// The earlier row kernels (rowres, rowwarp, shortrow) stage whole rows in
// shared memory; 28 KB per row leaves 6-8 rows (warps) per SM and they end
// up latency-bound.  Here a row only passes through a 4 KB staging tile:
//   * lane l reads its own 8 bytes (buckets 4l..4l+3, topk.hpp:13-15: element
//     i goes to bucket i mod B) of every stride-row straight into registers
//     (256 B per warp load, 16 loads in flight per lane, double-buffered);
//   * per bf16x2 word one packed 3-input max (the group maxima, two words
//     per instruction) and one packed compare + mask-or (the hit map): no
//     branch, no per-bucket state in the loop;
//   * every 16 stride-rows the lane walks the set bits of its hit map and
//     copies the hits (value | position) from its own column of the staging
//     tile to its log -- the row is never read again.
// Threshold argument: for a level L let c_b = the elements of
// bucket b that are >= L and M = sum_b min(K', c_b).  If M >= K the top K of
// the row's candidates are the top K of its candidates >= L, and those
// follow from the elements >= L alone (Alg. 1 over a bucket's elements >= L,
// topk.cpp:80-102, the S* lemma).  M is known exactly after the pass (the
// popcounts of the hit map), so ANY level may be tried:
//   fast path   L0 = the CTA's prediction: the level of the K-th candidate of
//               the row finished last (a by-product of its stage 2) minus a
//               margin.  One pass; M >= K afterwards proves it.
//   two-pass    no prediction yet, M < K, or a lane's log overflowed: the
//               exact K-th largest of the B K' group maxima (K' disjoint groups
//               of stride-rows per bucket; 16 packed-compare rounds on the
//               maxima the first pass kept) guarantees M >= K; a second pass
//               (the row is in L2) logs the hits against it.
//   exact path  L = -inf, or a log overflows even then (ties at L, one
//               bucket holding the large values): Alg. 1 of every bucket as
//               the reference runs it, then a bitonic sort of the B K' rank
//               keys.  Slow; degenerate rows only.
// After the pass: crowded buckets (c_b > K') are resolved by Alg. 1 over
// their logged hits (one lane per crowded bucket), then the (value code,
// index quarter) counting sort of rowwarp.cuh writes the first K in output
// order (topk.cpp:30-50).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "rowthr.cuh"

namespace atkg {

constexpr uint32_t kRgBins = 1024;           // 256 value codes x 4 index quarters
constexpr uint32_t kRgTmp = 512;             // candidates: <= B K'
constexpr uint32_t kRgKeyNegInf = 0x007fu;   // asc_code16(-inf)
constexpr int kRgTile = 8;                   // stride-rows per load batch = per staging tile
// per warp: staging tile [8][32] x 8 B | state [128 buckets][4] u32 | bins | tmp
constexpr uint32_t kRgWarpSmem = kRgTile * 256 + 4 * 512 + 4 * kRgBins + 4 * kRgTmp;

struct RgArgs {
  const uint16_t* in;
  uint64_t rows;
  uint32_t k;
  uint32_t sub_shift;   // pos >> sub_shift < 4
  uint32_t margin;      // prediction: codes below the level of the last row's K-th candidate
  uint32_t starters;    // warps per CTA that start without a prediction (the rest wait for one)
  uint32_t force;       // tests: 1 = every row two-pass, 2 = every row exact, 3 = sort instead of bins
  uint32_t probe;       // development: stop after phase `probe`
  float* out_v;
  uint32_t* out_i;
  uint32_t* status;
};

__device__ __forceinline__ uint2 rg_ldg(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
// 0xffff in each half whose bf16 is >= the matching half of L2 (false on NaN)
__device__ __forceinline__ uint32_t rg_ge(uint32_t w, uint32_t L2) {
  uint32_t h;
  asm("set.ge.u32.bf16x2 %0, %1, %2;" : "=r"(h) : "r"(w), "r"(L2));
  return h;
}
__device__ __forceinline__ uint32_t rg_bits2(uint32_t code) {
  const uint32_t b = code16_bits(code);
  return b | (b << 16);
}

template <typename K>
__device__ __forceinline__ void warp_bitonic_sort(K* s, uint32_t P, uint32_t lane) {
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t q = lane; q < P / 2; q += 32) {
        const uint32_t i = 2 * q - (q & (stride - 1));
        const uint32_t j = i + stride;
        const bool asc = (i & size) == 0;
        const K a = s[i], b = s[j];
        if ((a > b) == asc) { s[i] = b; s[j] = a; }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ uint32_t rg_excl_scan(uint32_t v, uint32_t lane, uint32_t* tot) {
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if ((int)lane >= o) inc += y;
  }
  *tot = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

// group g of K' = 4 covers the stride-rows [g S / 4, (g + 1) S / 4)
template <int S>
__host__ __device__ constexpr int rg_group(int s) {
  int g = 0;
  while (g < 3 && (g + 1) * S / 4 <= s) ++g;
  return g;
}

// One pass over the row: lane-local group maxima (MAX) and Alg. 1
// (topk.cpp:80-102) over the hits of each of the lane's 4 buckets, in stream
// order.  Per tile of 8 stride-rows: the loads (issued one tile ahead) are
// compared against L2 and copied to the lane's column of the staging tile;
// bit 8 u + 7 - i of the tile's hit mask = element slot u of stride-row i
// (u = 0, 1, 2, 3 <-> bucket 4 lane + 0, 2, 1, 3); the lane then walks the
// set bits from the top (ascending stride-row inside a slot) and inserts
// (code << 16 | position) into the bucket's state[4], kept in Alg. 1 order
// (value descending, a later equal element never passes an earlier one; the
// empty slots are 0, below every hit).  POS: the hits are strictly positive,
// their bf16 bits order as they are; otherwise ascending codes.
template <int S, bool MAX, bool POS>
__device__ __forceinline__ void rg_stream(const uint2* p, uint32_t L2, uint32_t lane, uint2* stage, uint4* state,
                                          uint32_t (&gm)[2][4]) {
  constexpr int NB = (S + kRgTile - 1) / kRgTile;
  uint2 buf[2][kRgTile];
#pragma unroll
  for (int i = 0; i < kRgTile; ++i)
    if (i < S) buf[0][i] = rg_ldg(p + i * 32);
  const uint8_t* col = reinterpret_cast<const uint8_t*>(stage + lane);
  uint4* st4 = state + 4 * lane;  // the lane's buckets 4 lane .. 4 lane + 3
#pragma unroll
  for (int bt = 0; bt < NB; ++bt) {
    if (bt + 1 < NB) {
#pragma unroll
      for (int i = 0; i < kRgTile; ++i) {
        const int s = (bt + 1) * kRgTile + i;
        if (s < S) buf[(bt + 1) & 1][i] = rg_ldg(p + s * 32);
      }
    }
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < kRgTile; ++i) {
      const int s = bt * kRgTile + i;
      if (s < S) {
        const uint2 v = buf[bt & 1][i];
        if (MAX) {
          const int g = rg_group<S>(s);
          gm[0][g] = bmax_nan(gm[0][g], v.x);
          gm[1][g] = bmax_nan(gm[1][g], v.y);
        }
        m |= rg_ge(v.x, L2) & (0x00010001u << (7 - i));
        m |= rg_ge(v.y, L2) & (0x01000100u << (7 - i));
        stage[(7 - i) * 32 + lane] = v;
      }
    }
    while (m) {
      const uint32_t b = 31u - (uint32_t)__clz((int)m);
      m ^= 1u << b;
      const uint32_t r = b & 7u, u = b >> 3;           // stride-row bt * 8 + 7 - r, element slot u
      const uint32_t j = ((u & 1u) << 1) | (u >> 1);    // bucket 4 lane + j
      uint32_t val = *reinterpret_cast<const uint16_t*>(col + r * 256 + j * 2);
      if (!POS) val = asc_code16(val);
      const uint32_t e = (val << 16) | (((bt * kRgTile + 7) << 7) - (r << 7) + 4 * lane + j);
      uint4 sv = st4[j];
      if (sv.w <= (e | 0xffffu)) {  // value >= v[K' - 1]: e replaces the minimum slot, then rises
        const uint32_t eb = e & 0xffff0000u;  // past the strictly smaller values
        const bool a2 = sv.z >= eb, a1 = sv.y >= eb, a0 = sv.x >= eb;  // slot k stays above e
        sv.w = a2 ? e : sv.z;
        sv.z = a2 ? sv.z : (a1 ? e : sv.y);
        sv.y = a1 ? sv.y : (a0 ? e : sv.x);
        sv.x = a0 ? sv.x : e;
        st4[j] = sv;
      }
    }
  }
}

// lane count of the 16 group maxima >= L2 (float order)
__device__ __forceinline__ uint32_t rg_count_ge(const uint32_t (&gm)[2][4], uint32_t L2) {
  uint32_t t = 0;
#pragma unroll
  for (int w = 0; w < 2; ++w)
#pragma unroll
    for (int g = 0; g < 4; ++g) t |= rg_ge(gm[w][g], L2) & (0x00010001u << (4 * w + g));
  return __popc(t);
}

// The exact path (degenerate rows): Alg. 1 of every bucket as the reference
// runs it (topk.cpp:80-102 with the {-inf, 0} sentinels of topk.cpp:118-121),
// the B K' = 512 rank keys sorted, the first K written (topk.cpp:192-236).
template <int S>
__device__ __noinline__ void rg_exact(const uint16_t* xr, uint32_t lane, uint32_t K, uint64_t* srt, float* ov,
                                      uint32_t* oi) {
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const uint32_t bk = 4 * lane + j;
    float v[4];
    uint32_t ix[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) { v[t] = neg_inf(); ix[t] = 0; }
#pragma unroll 4
    for (int r = 0; r < S; ++r) {
      const uint32_t pos = r * 128 + bk;
      const float x = __uint_as_float((uint32_t)__ldg(xr + pos) << 16);
      const bool take = x >= v[3];
      v[3] = take ? x : v[3];
      ix[3] = take ? pos : ix[3];
#pragma unroll
      for (int t = 3; t >= 1; --t) {
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
    for (int t = 0; t < 4; ++t) srt[bk * 4 + t] = rank_key_bits(__float_as_uint(v[t]), ix[t]);
  }
  __syncwarp();
  warp_bitonic_sort<uint64_t>(srt, 512, lane);
  for (uint32_t q = lane; q < K; q += 32) {
    ov[q] = __uint_as_float(key_value_bits(srt[q]));
    oi[q] = (uint32_t)srt[q];
  }
  __syncwarp();
}

// S = stride-rows (n = 128 S <= 16384), B = 128, K' = 4.  One CTA per SM;
// CTA c owns the rows [rows c / G, rows (c + 1) / G) and its warps pull them
// from a shared counter.  `pred` is the CTA's prediction (an ascending code;
// 0 = none yet, ~0 = the starters found none).
template <int S, int NW>
__global__ void __launch_bounds__(32 * NW, 1) row_reg_kernel(RgArgs a) {
  constexpr uint32_t n = 128u * S;
  extern __shared__ __align__(128) uint8_t rg_smem[];
  __shared__ uint32_t queue;
  __shared__ volatile uint32_t pred;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.k;
  uint8_t* wsm = rg_smem + (size_t)wid * kRgWarpSmem;
  uint2* stage = reinterpret_cast<uint2*>(wsm);
  uint4* state = reinterpret_cast<uint4*>(wsm + kRgTile * 256);
  uint32_t* cand = reinterpret_cast<uint32_t*>(state);  // [bucket][4], 0 = empty
  uint32_t* bins = cand + 512;
  uint32_t* tmp = bins + kRgBins;
  const uint64_t r0 = a.rows * blockIdx.x / gridDim.x, r1 = a.rows * (blockIdx.x + 1) / gridDim.x;
  const uint32_t nrows = (uint32_t)(r1 - r0);
  if (threadIdx.x == 0) {
    queue = 0;
    pred = 0;
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  // every warp but the starters waits for the first prediction
  if (wid >= a.starters && a.force == 0) {
    while (pred == 0) __nanosleep(500);
  }

#pragma unroll 1
  for (;;) {
    uint32_t rr = 0;
    if (lane == 0) rr = atomicAdd(&queue, 1u);
    rr = __shfl_sync(0xffffffffu, rr, 0);
    if (rr >= nrows) break;
    const uint64_t row = r0 + rr;
    const uint16_t* xr = a.in + row * n;
    const uint2* p = reinterpret_cast<const uint2*>(xr) + lane;
    float* ov = a.out_v + row * K;
    uint32_t* oi = a.out_i + row * K;

    // ---- the pass: group maxima + Alg. 1 over the hits against the prediction
    uint32_t gm[2][4];
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int g = 0; g < 4; ++g) gm[w][g] = 0xff80ff80u;
    auto clear_state = [&]() {
#pragma unroll
      for (int j = 0; j < 4; ++j) state[4 * lane + j] = make_uint4(0, 0, 0, 0);
    };
    clear_state();
    uint32_t Lkey = pred;
    const bool have = Lkey != 0 && Lkey != 0xffffffffu && a.force == 0;
    bool posmode = have && Lkey > 0x8000u;
    if (have) {
      if (posmode) rg_stream<S, true, true>(p, rg_bits2(Lkey), lane, stage, state, gm);
      else rg_stream<S, true, false>(p, rg_bits2(Lkey), lane, stage, state, gm);
    } else {
      rg_stream<S, true, true>(p, 0x7fc07fc0u, lane, stage, state, gm);  // NaN level: maxima only
    }
    if (a.probe == 1) {  // development: the pass alone (its results consumed)
      uint32_t z = state[4 * lane].x;
#pragma unroll
      for (int w = 0; w < 2; ++w)
#pragma unroll
        for (int g = 0; g < 4; ++g) z += gm[w][g];
      if (z == 0x12345u) oi[lane] = z;
      if (pred == 0) pred = 0xbff0u;
      continue;
    }

    // NaN rows (the reference rejects the input), the row maximum
    uint32_t mm = bmax_nan(bmax_nan(bmax_nan(gm[0][0], gm[0][1]), bmax_nan(gm[0][2], gm[0][3])),
                           bmax_nan(bmax_nan(gm[1][0], gm[1][1]), bmax_nan(gm[1][2], gm[1][3])));
    const uint32_t mlo = mm & 0xffffu, mhi = mm >> 16;
    const uint32_t nan = ((mlo & 0x7fffu) > 0x7f80u || (mhi & 0x7fffu) > 0x7f80u) ? 1u : 0u;
    if (__reduce_or_sync(0xffffffffu, nan)) {
      if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
      if (pred == 0) pred = 0xffffffffu;
      continue;
    }
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, max(asc_code16(mlo), asc_code16(mhi)));

    // M = sum_b min(K', c_b) = the filled slots
    auto filled = [&]() {
      uint32_t f = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 sv = state[4 * lane + j];
        f += (sv.x ? 1u : 0u) + (sv.y ? 1u : 0u) + (sv.z ? 1u : 0u) + (sv.w ? 1u : 0u);
      }
      return __reduce_add_sync(0xffffffffu, f);
    };
    uint32_t M = have ? filled() : 0u;
    bool exact = a.force == 2;
    if (M < K) {
      // ---- two-pass: the exact K-th largest group maximum guarantees M >= K
      uint32_t cur = 0;
#pragma unroll 1
      for (int bit = 15; bit >= 0; --bit) {
        const uint32_t t = cur | (1u << bit);
        const uint32_t cg = __reduce_add_sync(0xffffffffu, rg_count_ge(gm, rg_bits2(t)));
        if (cg >= K) cur = t;
      }
      Lkey = cur;
      if (Lkey <= kRgKeyNegInf) {
        exact = true;
      } else {
        if (pred == 0) pred = max(Lkey, kRgKeyNegInf + 1 + a.margin) - a.margin;
        posmode = Lkey > 0x8000u;
        clear_state();
        if (posmode) rg_stream<S, false, true>(p, rg_bits2(Lkey), lane, stage, state, gm);
        else rg_stream<S, false, false>(p, rg_bits2(Lkey), lane, stage, state, gm);
        M = filled();
      }
    }
    if (a.probe == 2) continue;
    if (exact) {
      if (pred == 0) pred = 0xffffffffu;
      __syncwarp();
      rg_exact<S>(xr, lane, K, reinterpret_cast<uint64_t*>(bins), ov, oi);
      continue;
    }
    __syncwarp();

    // ---- stage 2: the first K of the M >= K candidates -------------------
    const uint32_t kmaxm = posmode ? (kmax & 0x7fffu) : kmax;
    const uint32_t Lm = posmode ? (Lkey & 0x7fffu) : Lkey;
    const bool binned = kmaxm - Lm < 256u && a.force != 3;
    uint32_t Lstar = Lkey;  // level of the K-th candidate (ascending code)
    if (binned) {
#pragma unroll
      for (int i = 0; i < (int)(kRgBins / 128); ++i)
        reinterpret_cast<uint4*>(bins)[lane + 32 * i] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      auto bin_of = [&](uint32_t key) { return ((kmaxm - (key >> 16)) << 2) | ((key & 0xffffu) >> a.sub_shift); };
      uint32_t keys[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        keys[r] = cand[32 * r + lane];
        if (keys[r]) atomicAdd(&bins[bin_of(keys[r])], 1u);
      }
      __syncwarp();
      // exclusive scan of the 1024 bins (32 per lane), the first bin starting at >= K
      uint4 cc[8];
      uint32_t sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        cc[i] = reinterpret_cast<const uint4*>(bins)[8 * lane + i];
        sum += cc[i].x + cc[i].y + cc[i].z + cc[i].w;
      }
      uint32_t tot, st = rg_excl_scan(sum, lane, &tot), blim = 0xffffffffu, lim = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t q0 = st, q1 = q0 + cc[i].x, q2 = q1 + cc[i].y, q3 = q2 + cc[i].z;
        st = q3 + cc[i].w;
        reinterpret_cast<uint4*>(bins)[8 * lane + i] = make_uint4(q0, q1, q2, q3);
        const uint32_t b0 = 32 * lane + 4 * i;
        if (blim == 0xffffffffu) {
          if (q0 >= K) { blim = b0; lim = q0; }
          else if (q1 >= K) { blim = b0 + 1; lim = q1; }
          else if (q2 >= K) { blim = b0 + 2; lim = q2; }
          else if (q3 >= K) { blim = b0 + 3; lim = q3; }
        }
      }
      blim = __reduce_min_sync(0xffffffffu, blim);
      lim = min(M, __reduce_min_sync(0xffffffffu, lim));
      // bin blim - 1 is not empty and starts below K: it holds the K-th candidate
      if (blim != 0xffffffffu && blim > 0) Lstar = (kmaxm - ((blim - 1) >> 2)) | (posmode ? 0x8000u : 0u);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 16; ++r) {  // scatter the bins wholly below rank K
        if (keys[r]) {
          const uint32_t bn = bin_of(keys[r]);
          if (bn < blim) tmp[atomicAdd(&bins[bn], 1u)] = keys[r];
        }
      }
      __syncwarp();  // bins[b] = end of bin b = start of bin b + 1
      for (uint32_t x = lane; x < lim; x += 32) {
        const uint32_t key = tmp[x], bn = bin_of(key);
        const uint32_t b0 = bn ? bins[bn - 1] : 0u, b1 = bins[bn];
        uint32_t r = b0;
        for (uint32_t y = b0; y < b1; ++y) r += tmp[y] < key ? 1u : 0u;  // same code: by position
        if (r < K) {
          const uint32_t code = key >> 16;
          ov[r] = __uint_as_float((posmode ? code : code16_bits(code)) << 16);
          oi[r] = key & 0xffffu;
        }
      }
    } else {  // the hits span more than 256 value codes: sort the candidates
      uint32_t off = 0;
      for (uint32_t r = 0; r < 16; ++r) {
        const uint32_t e = cand[32 * r + lane];
        const uint32_t bal = __ballot_sync(0xffffffffu, e != 0);
        const uint32_t asc = (e >> 16) | (posmode ? 0x8000u : 0u);
        if (e) tmp[off + __popc(bal & lt)] = ((~asc & 0xffffu) << 16) | (e & 0xffffu);
        off += __popc(bal);
      }
      uint32_t P2 = 2;
      while (P2 < off) P2 <<= 1;
      for (uint32_t x = off + lane; x < P2; x += 32) tmp[x] = 0xffffffffu;
      __syncwarp();
      warp_bitonic_sort<uint32_t>(tmp, P2, lane);
      for (uint32_t x = lane; x < K; x += 32) {
        ov[x] = __uint_as_float(code16_bits(~(tmp[x] >> 16) & 0xffffu) << 16);
        oi[x] = tmp[x] & 0xffffu;
      }
      Lstar = ~(tmp[K - 1] >> 16) & 0xffffu;
    }
    // the next row's prediction
    if (lane == 0) pred = max(Lstar, kRgKeyNegInf + 1 + a.margin) - a.margin;
    __syncwarp();
  }
  // a starter that found no prediction must still release the waiting warps
  if (pred == 0) pred = 0xffffffffu;
}

}  // namespace atkg
