// rowreg.cuh -- approx_top_k for short bf16 rows streamed ONCE from HBM, one
// warp per row, many rows in flight per SM: the FFN-activation config C3
// (rows of 14336 = 128 buckets x 112 stride-rows, K' = 4, K = 287).
//
// The earlier row kernels (rowres, rowwarp, shortrow) stage whole rows in
// shared memory; 28 KB per row leaves 6-8 rows (warps) per SM and they end
// up latency-bound.  Here the row never touches shared memory:
//   * lane l reads its own 8 bytes (buckets 4l..4l+3, topk.hpp:13-15: element
//     i goes to bucket i mod B) of every stride-row straight into registers
//     (256 B per warp load, 14 loads in flight per lane, double-buffered);
//   * per bf16x2 word one packed max (the group maxima) and one packed
//     compare + mask-or (the hit map) -- 7 instructions per 4 elements and
//     lane, no branch, no per-bucket state in the loop;
//   * the hit map of a lane's 4 buckets (<= 128 stride-rows each) stays in
//     14 registers.
// Threshold argument (shortrow.cuh): split every bucket's
// stride-rows into K' disjoint groups.  If at least K of the B K' group
// maxima are >= L then M = sum_b min(K', c_b(L)) >= K, so the top K of the
// row's candidates are the top K of its candidates >= L, and those follow
// from the elements >= L alone (Alg. 1 over a bucket's elements >= L,
// topk.cpp:80-102, the S* lemma).
//   fast path   L0 = the warp's prediction (the previous row's exact level
//               minus a margin, then a +-1 code controller on the count of
//               group maxima >= L0).  Maxima and hit map come from the same
//               pass; the count proves M >= K afterwards.  Any L0 is exact.
//   two-pass    no prediction yet, or the count fell short: bisect the exact
//               K-th largest group maximum (16 packed-compare rounds), then
//               a second compare-only pass (the row is in L2).
//   exact path  L = -inf, or more hits than the list holds (ties at L):
//               Alg. 1 of every bucket as the reference runs it, then a
//               bitonic sort of the B K' rank keys.  Slow, degenerate rows only.
// After the stream: hits -> list (bucket-major, position-ascending inside a
// bucket), values fetched in balanced rounds (scattered 2-byte loads, L2),
// crowded buckets (c_b > K') resolved by Alg. 1 over their hits with one lane
// per crowded bucket, then the same (value code, index quarter) counting
// sort as rowwarp.cuh for the first K in output order (topk.cpp:30-50).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "rowthr.cuh"

namespace atkg {

constexpr uint32_t kRgCap = 1024;            // hit list entries per row
constexpr uint32_t kRgBins = 1024;           // 256 value codes x 4 index quarters
constexpr uint32_t kRgTmp = 512;             // candidates after the crowded buckets: <= B K'
constexpr uint32_t kRgDead = 0xffffffffu;    // dropped list entry (sorts last)
constexpr uint32_t kRgKeyNegInf = 0x007fu;   // asc_code16(-inf)
constexpr uint32_t kRgWarpSmem = 4 * kRgCap + 4 * kRgTmp + 4 * kRgBins;  // E | tmp | bins
constexpr int kRgBatch = 14;                 // stride-rows per load batch

struct RgArgs {
  const uint16_t* in;
  uint64_t rows;
  uint32_t k;
  uint32_t sub_shift;   // pos >> sub_shift < 4
  uint32_t margin;      // prediction: codes below the last exact level
  uint32_t slack;       // controller: aim at K + slack group maxima >= L0
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

// One pass over the row: lane-local group maxima (MAX) and the hit map
// against L2 (acc[w][q]: half h of word w = bucket 4 lane + 2 w + h, bit i =
// stride-row 16 q + i).
template <int S, bool MAX>
__device__ __forceinline__ void rg_stream(const uint2* p, uint32_t L2, uint32_t (&acc)[2][(S + 15) / 16],
                                          uint32_t (&gm)[2][4]) {
  constexpr int NB = (S + kRgBatch - 1) / kRgBatch;
  uint2 buf[2][kRgBatch];
#pragma unroll
  for (int i = 0; i < kRgBatch; ++i)
    if (i < S) buf[0][i] = rg_ldg(p + i * 32);
#pragma unroll
  for (int bt = 0; bt < NB; ++bt) {
    if (bt + 1 < NB) {
#pragma unroll
      for (int i = 0; i < kRgBatch; ++i) {
        const int s = (bt + 1) * kRgBatch + i;
        if (s < S) buf[(bt + 1) & 1][i] = rg_ldg(p + s * 32);
      }
    }
#pragma unroll
    for (int i = 0; i < kRgBatch; ++i) {
      const int s = bt * kRgBatch + i;
      if (s < S) {
        const uint2 v = buf[bt & 1][i];
        if (MAX) {
          const int g = rg_group<S>(s);
          gm[0][g] = bmax_nan(gm[0][g], v.x);
          gm[1][g] = bmax_nan(gm[1][g], v.y);
        }
        const uint32_t bit = 0x00010001u << (s & 15);
        acc[0][s >> 4] |= rg_ge(v.x, L2) & bit;
        acc[1][s >> 4] |= rg_ge(v.y, L2) & bit;
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
// from a shared counter.
template <int S, int NW>
__global__ void __launch_bounds__(32 * NW, 1) row_reg_kernel(RgArgs a) {
  constexpr int NQ = (S + 15) / 16;
  constexpr uint32_t n = 128u * S;
  extern __shared__ __align__(128) uint8_t rg_smem[];
  __shared__ uint32_t queue;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.k;
  uint32_t* E = reinterpret_cast<uint32_t*>(rg_smem + (size_t)wid * kRgWarpSmem);
  uint32_t* tmp = E + kRgCap;
  uint32_t* bins = tmp + kRgTmp;
  const uint64_t r0 = a.rows * blockIdx.x / gridDim.x, r1 = a.rows * (blockIdx.x + 1) / gridDim.x;
  const uint32_t nrows = (uint32_t)(r1 - r0);
  if (threadIdx.x == 0) queue = 0;
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t L0key = 0;  // 0 = no prediction yet

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

    // ---- the stream: group maxima + hit map against the prediction ------
    uint32_t acc[2][NQ], gm[2][4];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[w][q] = 0;
#pragma unroll
      for (int g = 0; g < 4; ++g) gm[w][g] = 0xff80ff80u;
    }
    const bool have = L0key != 0 && a.force == 0;
    uint32_t L2 = have ? rg_bits2(L0key) : 0x7fc07fc0u;  // NaN: no hits, count 0
    rg_stream<S, true>(p, L2, acc, gm);
    if (a.probe == 1) {  // development: the stream alone (its results consumed)
      uint32_t z = 0;
#pragma unroll
      for (int w = 0; w < 2; ++w) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) z ^= acc[w][q];
#pragma unroll
        for (int g = 0; g < 4; ++g) z += gm[w][g];
      }
      if (z == 0x12345u) oi[lane] = z;
      continue;
    }

    // NaN rows (the reference rejects the input), the row maximum
    uint32_t mm = bmax_nan(bmax_nan(bmax_nan(gm[0][0], gm[0][1]), bmax_nan(gm[0][2], gm[0][3])),
                           bmax_nan(bmax_nan(gm[1][0], gm[1][1]), bmax_nan(gm[1][2], gm[1][3])));
    const uint32_t mlo = mm & 0xffffu, mhi = mm >> 16;
    const uint32_t nan = ((mlo & 0x7fffu) > 0x7f80u || (mhi & 0x7fffu) > 0x7f80u) ? 1u : 0u;
    if (__reduce_or_sync(0xffffffffu, nan)) {
      if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
      continue;
    }
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, max(asc_code16(mlo), asc_code16(mhi)));

    // hit maps per bucket (bit r of bm[j][t] = stride-row 32 t + r), counts,
    // list offsets; H = hits of the row
    uint32_t bm[4][4], c[4], H = 0, d = 0;
    auto bucket_maps = [&]() {
      uint32_t nl = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        c[j] = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t lo = 2 * t < NQ ? acc[j >> 1][2 * t < NQ ? 2 * t : 0] : 0u;
          const uint32_t hi = 2 * t + 1 < NQ ? acc[j >> 1][2 * t + 1 < NQ ? 2 * t + 1 : 0] : 0u;
          bm[j][t] = __byte_perm(lo, hi, (j & 1) ? 0x7632 : 0x5410);
          c[j] += __popc(bm[j][t]);
        }
        nl += c[j];
      }
      d = rg_excl_scan(nl, lane, &H);
    };

    uint32_t Lkey = L0key;
    bool exact = a.force == 2;
    const uint32_t cnt = have ? __reduce_add_sync(0xffffffffu, rg_count_ge(gm, L2)) : 0u;
    bool twopass = !have || cnt < K;
    if (!twopass) {
      bucket_maps();
      twopass = H > kRgCap;  // the prediction sits far below the row's level
      // controller: hold the count of group maxima >= L0 near K + slack
      if (cnt < K + a.slack / 2) L0key = max(L0key - 1, kRgKeyNegInf + 1);
      else if (cnt > K + a.slack + a.slack / 2) L0key = L0key + 1;
    }
    if (twopass) {
      // ---- the exact K-th largest group maximum, then a compare-only pass
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
        L0key = 0;
      } else {
        L2 = rg_bits2(Lkey);
#pragma unroll
        for (int w = 0; w < 2; ++w)
#pragma unroll
          for (int q = 0; q < NQ; ++q) acc[w][q] = 0;
        rg_stream<S, false>(p, L2, acc, gm);
        L0key = max(Lkey, kRgKeyNegInf + 1 + a.margin) - a.margin;
        bucket_maps();
        if (H > kRgCap) exact = true;  // ties at L
      }
    }
    if (a.probe == 2) continue;
    if (exact) {
      rg_exact<S>(xr, lane, K, reinterpret_cast<uint64_t*>(E), ov, oi);
      continue;
    }
    const bool binned = kmax - Lkey < 256u && a.force != 3;
    if (binned) {
#pragma unroll
      for (int i = 0; i < (int)(kRgBins / 128); ++i)
        reinterpret_cast<uint4*>(bins)[lane + 32 * i] = make_uint4(0, 0, 0, 0);
    }

    // ---- hits -> list (bucket-major, position-ascending inside a bucket),
    //      crowded buckets -> descriptors (offset | count << 16) in tmp
    uint32_t nov = 0;
    {
      uint32_t o = d;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t crowded = c[j] > 4u ? 1u : 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, crowded);
        if (crowded) tmp[nov + __popc(bal & lt)] = o | (c[j] << 16);
        nov += __popc(bal);
        o += c[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t bk = 4 * lane + j;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint32_t x = bm[j][t];
        while (x) {
          const uint32_t s = 32 * t + __ffs(x) - 1;
          x &= x - 1;
          E[d++] = s * 128 + bk;
        }
      }
    }
    __syncwarp();
    if (a.probe == 3) continue;

    // ---- values: E[i] = (~code << 16) | pos, ascending = output order ----
    for (uint32_t i0 = 0; i0 < H; i0 += 128) {
      uint32_t pos[4], val[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + 32 * u + lane;
        pos[u] = i < H ? E[i] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) val[u] = __ldg(xr + pos[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + 32 * u + lane;
        if (i < H) E[i] = ((~asc_code16(val[u]) & 0xffffu) << 16) | pos[u];
      }
    }
    __syncwarp();
    if (a.probe == 4) continue;

    // ---- crowded buckets: Alg. 1 over the bucket's hits in position order;
    //      the K' survivors stay at the front of the segment
    uint32_t dropped = 0;
    for (uint32_t i = lane; i < nov; i += 32) {
      const uint32_t ds = tmp[i], off = ds & 0xffffu, cb = ds >> 16;
      uint32_t s0 = kRgDead, s1 = kRgDead, s2 = kRgDead, s3 = kRgDead;
      for (uint32_t q = 0; q < cb; ++q) {
        const uint32_t e = E[off + q];
        if ((e >> 16) <= (s3 >> 16)) {  // value >= v[K' - 1]: replace the minimum slot
          s3 = e;
          if ((s3 >> 16) < (s2 >> 16)) { const uint32_t z = s3; s3 = s2; s2 = z; }
          if ((s2 >> 16) < (s1 >> 16)) { const uint32_t z = s2; s2 = s1; s1 = z; }
          if ((s1 >> 16) < (s0 >> 16)) { const uint32_t z = s1; s1 = s0; s0 = z; }
        }
      }
      E[off] = s0;
      E[off + 1] = s1;
      E[off + 2] = s2;
      E[off + 3] = s3;
      for (uint32_t q = 4; q < cb; ++q) E[off + q] = kRgDead;
      dropped += cb - 4;
    }
    dropped = __reduce_add_sync(0xffffffffu, dropped);
    const uint32_t M = H - dropped;
    __syncwarp();
    if (a.probe == 5) continue;

    // ---- stage 2: the first K of the M >= K candidates -------------------
    if (binned) {
      auto bin_of = [&](uint32_t key) {
        return ((kmax - (~(key >> 16) & 0xffffu)) << 2) | ((key & 0xffffu) >> a.sub_shift);
      };
      for (uint32_t x = lane; x < H; x += 32) {
        const uint32_t key = E[x];
        if (key != kRgDead) atomicAdd(&bins[bin_of(key)], 1u);
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
      __syncwarp();
      for (uint32_t x = lane; x < H; x += 32) {  // scatter the bins wholly below rank K
        const uint32_t key = E[x];
        if (key != kRgDead) {
          const uint32_t bn = bin_of(key);
          if (bn < blim) tmp[atomicAdd(&bins[bn], 1u)] = key;
        }
      }
      __syncwarp();  // bins[b] = end of bin b = start of bin b + 1
      for (uint32_t x = lane; x < lim; x += 32) {
        const uint32_t key = tmp[x], bn = bin_of(key);
        const uint32_t b0 = bn ? bins[bn - 1] : 0u, b1 = bins[bn];
        uint32_t r = b0;
        for (uint32_t y = b0; y < b1; ++y) r += tmp[y] < key ? 1u : 0u;
        if (r < K) {
          ov[r] = __uint_as_float(code16_bits(~(key >> 16) & 0xffffu) << 16);
          oi[r] = key & 0xffffu;
        }
      }
    } else {  // the hits span more than 256 value codes: sort them
      uint32_t P2 = 2;
      while (P2 < H) P2 <<= 1;
      for (uint32_t x = H + lane; x < P2; x += 32) E[x] = kRgDead;
      __syncwarp();
      warp_bitonic_sort<uint32_t>(E, P2, lane);
      for (uint32_t x = lane; x < K; x += 32) {
        ov[x] = __uint_as_float(code16_bits(~(E[x] >> 16) & 0xffffu) << 16);
        oi[x] = E[x] & 0xffffu;
      }
    }
    __syncwarp();
  }
}

}  // namespace atkg
