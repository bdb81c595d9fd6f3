// rowwarp.cuh -- approx_top_k for bf16 rows held in shared memory, one warp
// per row: the FFN-activation config C3 (rows of 14336, K = 287, B = 128)
// and the K' sweep points with B in {128, 256, 512} (<= 128 stride-rows).
//
// Same threshold argument as shortrow.cuh: L = the K-th largest of the B*K'
// group maxima (K' disjoint groups of consecutive stride-rows per bucket)
// guarantees M = sum_b min(K', c_b) >= K, so the top K of the row's
// candidates are the top K of its candidates >= L, and those follow from the
// elements >= L (Alg. 1 over a bucket's elements >= L, topk.cpp:80-102, the
// S* lemma of DESIGN.md 4).  Here every lane owns whole buckets -- chunk
// column c = lane + 32 k holds the 4 buckets 4c..4c+3 (B = 128 CPL) -- so
// the group maxima, the per-bucket hit masks (registers: bit r of word w =
// stride-row 32 w + r), the counts and Alg. 1 over a crowded bucket are all
// lane-local; the warp only cooperates in the threshold select and stage 2.
// One warp per CTA and ~6 CTAs per SM keep as many rows in flight; the row
// arrives by one 1-D TMA bulk copy, and the next row's copy is issued as soon
// as this row's values are no longer read (before stage 2).
//   pass 1   max over each group's stride-rows (packed bf16x2, NaN-propagating);
//   select   256-bin histogram of the group maxima's ascending 16-bit keys,
//            binned down from the row maximum (finer second level when the
//            bins are wider than 4 codes) -> L, a lower bound of the K-th;
//   pass 2   one packed compare per word sets the hit-mask bits;
//   collect  an uncrowded bucket (c_b <= K') keeps its hits, a crowded one
//            runs Alg. 1 over them in position order; candidates (32-bit
//            rank keys ~key16 << 16 | pos, ascending = output order,
//            topk.cpp:30-50) go to a warp list at scanned offsets;
//   stage 2  counting sort on (value code, index quarter) bins, ranks inside
//            a bin by comparison, the first K written out.
// Rows with L = -inf or more candidates than the list holds take the exact
// path (Alg. 1 summaries of every bucket, summ.cuh, then a bitonic sort of
// the B*K' candidates); NaN rows raise ATKG_FLAG_NAN.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "ptx.cuh"
#include "rowthr.cuh"
#include "summ.cuh"

namespace atkg {

constexpr uint32_t kRwBins = 1024;          // stage 2: 256 value codes x 4 index quarters
constexpr uint32_t kRwKeyNegInf = 0x007fu;  // asc_code16(-inf)

struct RwArgs {
  const void* in;
  uint64_t rows;
  uint32_t n, S, k;
  uint32_t cap;         // candidate list (pow2)
  uint32_t row_bytes;   // n * 2
  uint32_t slot_bytes;  // row region (>= row_bytes, >= the exact path's sort)
  uint32_t P;           // exact path: pow2 >= B * K'
  uint32_t sub_shift;   // stage 2: pos >> sub_shift < 4
  uint32_t force_slow;  // tests: every row takes the exact path
  uint32_t probe;       // development: stop after phase `probe` (0 = off)
  uint64_t* gws;        // exact path scratch, [grid][P]
  float* out_v;
  uint32_t* out_i;
  uint32_t* status;
};

// smem (dynamic): row[slot_bytes] | cand[cap] u32 | tmp[cap] u32 | bins[1024] u32
__host__ __device__ constexpr size_t rw_smem_bytes(uint32_t slot_bytes, uint32_t cap) {
  return (size_t)slot_bytes + 8ull * cap + 4ull * kRwBins;
}

__device__ __forceinline__ uint2 rw_vmax(uint2 a, uint2 b) { return make_uint2(bmax_nan(a.x, b.x), bmax_nan(a.y, b.y)); }

// halves of a bf16x2 word >= L: mlo |= bit, mhi |= bit
__device__ __forceinline__ void rw_mark(uint32_t w, uint32_t L2, uint32_t bit, uint32_t& mlo, uint32_t& mhi) {
  asm("{\n\t.reg .pred p, q;\n\t"
      "setp.ge.bf16x2 p|q, %2, %3;\n\t"
      "@p or.b32 %0, %0, %4;\n\t"
      "@q or.b32 %1, %1, %4;\n\t}"
      : "+r"(mlo), "+r"(mhi)
      : "r"(w), "r"(L2), "r"(bit));
}

// warp-wide exclusive scan (returns the exclusive prefix; *tot = the sum)
__device__ __forceinline__ uint32_t rw_excl_scan(uint32_t v, uint32_t lane, uint32_t* tot) {
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if ((int)lane >= o) inc += y;
  }
  *tot = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

// KP = K'; CPL = 8-byte chunk columns per lane (B = 128 CPL); W = mask words
// per bucket (stride-rows <= 32 W)
template <int KP, int CPL, int W>
__global__ void __launch_bounds__(32) row_warp_kernel(RwArgs a) {
  constexpr uint32_t B = 128 * CPL, CPS = 32 * CPL;  // buckets, 8-byte chunks per stride-row
  constexpr int NB = 4 * CPL;                        // buckets per lane
  extern __shared__ __align__(128) uint8_t rw_smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t lane = threadIdx.x;
  const uint32_t S = a.S, K = a.k;
  uint8_t* rowp = rw_smem;
  const uint2* ch = reinterpret_cast<const uint2*>(rowp);
  const uint16_t* xh = reinterpret_cast<const uint16_t*>(rowp);
  uint32_t* cand = reinterpret_cast<uint32_t*>(rw_smem + a.slot_bytes);
  uint32_t* tmp = cand + a.cap;
  uint32_t* bins = tmp + a.cap;  // also the select histogram (256)
  const uint64_t pol = ptx::policy_evict_first();
  const uint8_t* in = static_cast<const uint8_t*>(a.in);
  const uint32_t lt = (1u << lane) - 1u;
  if (lane == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](uint64_t r) {  // lane 0: row r into the slot
    if (lane == 0 && r < a.rows) {
      ptx::mbar_arrive_expect_tx(&bar, a.row_bytes);
      ptx::bulk_g2s(rowp, in + r * a.row_bytes, a.row_bytes, &bar, pol);
    }
  };
  uint64_t row = blockIdx.x;
  issue(row);
#pragma unroll 1
  for (uint32_t it = 0; row < a.rows; ++it, row += gridDim.x) {
    const uint64_t nrow = row + gridDim.x;
    ptx::mbar_wait(&bar, it & 1);
    float* ov = a.out_v + row * K;
    uint32_t* oi = a.out_i + row * K;

    // ---- pass 1: group maxima -> ascending keys gk[k][j][g] --------------
    uint32_t gk[NB][KP];
    uint32_t kmax = 0, kmin = 0xffffffffu, nan = 0;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const uint2* p = ch + lane + 32 * k;
#pragma unroll
      for (int g = 0; g < KP; ++g) {
        const uint32_t r0 = g * S / KP, r1 = (g + 1) * S / KP;
        uint2 acc = make_uint2(0xff80ff80u, 0xff80ff80u);
        uint32_t r = r0;
        for (; r + 4 <= r1; r += 4)
          acc = rw_vmax(rw_vmax(acc, rw_vmax(p[r * CPS], p[(r + 1) * CPS])),
                        rw_vmax(p[(r + 2) * CPS], p[(r + 3) * CPS]));
        for (; r < r1; ++r) acc = rw_vmax(acc, p[r * CPS]);
        const uint32_t h[4] = {acc.x & 0xffffu, acc.x >> 16, acc.y & 0xffffu, acc.y >> 16};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          nan |= (h[j] & 0x7fffu) > 0x7f80u ? 1u : 0u;
          const uint32_t kk = asc_code16(h[j]);
          gk[4 * k + j][g] = kk;
          kmax = max(kmax, kk);
          kmin = min(kmin, kk);
        }
      }
    }
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    if (__reduce_or_sync(0xffffffffu, nan)) {  // the reference rejects the input
      if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
      ptx::fence_proxy_async();
      __syncwarp();
      issue(nrow);
      continue;
    }

    // ---- select: L = a lower bound of the K-th largest group maximum -----
    const uint32_t span = kmax - kmin;
    const uint32_t shf = span < 256u ? 0u : (uint32_t)(32 - __clz(span >> 8));
    auto zero_hist = [&]() {
      reinterpret_cast<uint4*>(bins)[lane] = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint4*>(bins)[lane + 32] = make_uint4(0, 0, 0, 0);
    };
    // the first bin whose cumulative count reaches `need`, and the count before it
    auto scan_bins = [&](uint32_t need, uint32_t& bin, uint32_t& before) {
      const uint4 c0 = reinterpret_cast<const uint4*>(bins)[2 * lane];
      const uint4 c1 = reinterpret_cast<const uint4*>(bins)[2 * lane + 1];
      const uint32_t c8[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      uint32_t sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += c8[i];
      uint32_t tot;
      uint32_t cum = rw_excl_scan(sum, lane, &tot), jb = 0xffffffffu, bef = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (jb == 0xffffffffu && cum + c8[i] >= need) { jb = lane * 8 + i; bef = cum; }
        cum += c8[i];
      }
      bin = __reduce_min_sync(0xffffffffu, jb);
      before = __shfl_sync(0xffffffffu, bef, (bin >> 3) & 31);
    };
    zero_hist();
    __syncwarp();
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int g = 0; g < KP; ++g) atomicAdd(&bins[min(255u, (kmax - gk[b][g]) >> shf)], 1u);
    __syncwarp();
    uint32_t j1, before;
    scan_bins(K, j1, before);
    uint64_t w1 = ((uint64_t)(j1 + 1) << shf) - 1;  // bin j1 = keys kmax - [j1 << shf, w1]
    uint32_t Lkey = (j1 >= 255u || w1 >= (uint64_t)span) ? kmin : kmax - (uint32_t)w1;
    if (shf > 2 && j1 < 255u) {  // refine inside bin j1
      const uint32_t shf2 = shf > 8 ? shf - 8 : 0, need = K - before;
      __syncwarp();
      zero_hist();
      __syncwarp();
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int g = 0; g < KP; ++g) {
          const uint32_t d = kmax - gk[b][g];
          if ((d >> shf) == j1) atomicAdd(&bins[min(255u, (d - (j1 << shf)) >> shf2)], 1u);
        }
      __syncwarp();
      uint32_t j2, b2;
      scan_bins(need, j2, b2);
      const uint64_t w2 = ((uint64_t)j1 << shf) + ((uint64_t)(j2 + 1) << shf2) - 1;
      Lkey = w2 >= (uint64_t)span ? kmin : kmax - (uint32_t)w2;
    }
    __syncwarp();
    bool slow = Lkey <= kRwKeyNegInf || a.force_slow;
    if (a.probe == 2) { ptx::fence_proxy_async(); __syncwarp(); issue(nrow); continue; }

    // ---- pass 2: hit masks m[b][w] (bit r = stride-row 32 w + r) ---------
    uint32_t m[NB][W];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int w = 0; w < W; ++w) m[b][w] = 0;
    uint32_t cnt[NB], M = 0, d = 0;
    if (!slow) {
      const uint32_t Lb = code16_bits(Lkey), L2 = Lb | (Lb << 16);
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const uint2* p = ch + lane + 32 * k;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          if (32 * w < (int)S) {
            const uint32_t nr = min(32u, S - 32 * w);
            const uint2* pw = p + 32 * w * CPS;
            uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0, bit = 1, i = 0;
            for (; i + 4 <= nr; i += 4) {
              const uint2 v0 = pw[i * CPS], v1 = pw[(i + 1) * CPS], v2 = pw[(i + 2) * CPS], v3 = pw[(i + 3) * CPS];
              rw_mark(v0.x, L2, bit, m0, m1);
              rw_mark(v0.y, L2, bit, m2, m3);
              rw_mark(v1.x, L2, bit << 1, m0, m1);
              rw_mark(v1.y, L2, bit << 1, m2, m3);
              rw_mark(v2.x, L2, bit << 2, m0, m1);
              rw_mark(v2.y, L2, bit << 2, m2, m3);
              rw_mark(v3.x, L2, bit << 3, m0, m1);
              rw_mark(v3.y, L2, bit << 3, m2, m3);
              bit <<= 4;
            }
            for (; i < nr; ++i, bit <<= 1) {
              const uint2 v = pw[i * CPS];
              rw_mark(v.x, L2, bit, m0, m1);
              rw_mark(v.y, L2, bit, m2, m3);
            }
            m[4 * k + 0][w] = m0;
            m[4 * k + 1][w] = m1;
            m[4 * k + 2][w] = m2;
            m[4 * k + 3][w] = m3;
          }
        }
      }
      // counts, candidate slots (warp scan)
      uint32_t mine = 0;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        cnt[b] = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) cnt[b] += __popc(m[b][w]);
        mine += min(cnt[b], (uint32_t)KP);
      }
      d = rw_excl_scan(mine, lane, &M);
      slow = M > a.cap;  // uniform: heavy ties at L
      if (a.probe == 3) { ptx::fence_proxy_async(); __syncwarp(); issue(nrow); continue; }
    }
    const bool binned = !slow && kmax - Lkey < 256u;
    if (!slow) {
      if (binned) {
#pragma unroll
        for (int i = 0; i < (int)(kRwBins / 128); ++i)
          reinterpret_cast<uint4*>(bins)[lane + 32 * i] = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      // ---- collect: candidates of every bucket this lane owns ------------
      auto put = [&](uint32_t key, uint32_t pos) {
        cand[d++] = ((~key & 0xffffu) << 16) | pos;
        if (binned) atomicAdd(&bins[((kmax - key) << 2) | (pos >> a.sub_shift)], 1u);
      };
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const uint32_t bk = 4 * (lane + 32 * (b >> 2)) + (b & 3);  // bucket index
        if (cnt[b] <= (uint32_t)KP) {  // every hit survives
#pragma unroll
          for (int w = 0; w < W; ++w) {
            uint32_t x = m[b][w];
            while (x) {
              const uint32_t pos = (32 * w + __ffs(x) - 1) * B + bk;
              x &= x - 1;
              put(asc_code16(xh[pos]), pos);
            }
          }
        } else {  // Alg. 1 (topk.cpp:80-102) on ascending keys; sentinels below every hit (L > -inf)
          uint32_t kv[KP], kq[KP];
#pragma unroll
          for (int j = 0; j < KP; ++j) { kv[j] = 0; kq[j] = 0; }
#pragma unroll
          for (int w = 0; w < W; ++w) {
            uint32_t x = m[b][w];
            while (x) {
              const uint32_t pos = (32 * w + __ffs(x) - 1) * B + bk;
              x &= x - 1;
              const uint32_t key = asc_code16(xh[pos]);
              if (key >= kv[KP - 1]) {
                kv[KP - 1] = key;
                kq[KP - 1] = pos;
#pragma unroll
                for (int j = KP - 1; j >= 1; --j) {
                  if (kv[j] > kv[j - 1]) {
                    const uint32_t tv = kv[j]; kv[j] = kv[j - 1]; kv[j - 1] = tv;
                    const uint32_t tq = kq[j]; kq[j] = kq[j - 1]; kq[j - 1] = tq;
                  }
                }
              }
            }
          }
#pragma unroll
          for (int j = 0; j < KP; ++j) put(kv[j], kq[j]);
        }
      }
      // the row is no longer read: the next row's copy overlaps stage 2
      ptx::fence_proxy_async();
      __syncwarp();
      issue(nrow);
      if (a.probe == 4) continue;

      // ---- stage 2: the first K of the M >= K candidates ---------------
      if (binned) {
        // exclusive scan of the 1024 bins (32 per lane), the first bin starting at >= K
        uint4 c[8];
        uint32_t sum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          c[i] = reinterpret_cast<const uint4*>(bins)[8 * lane + i];
          sum += c[i].x + c[i].y + c[i].z + c[i].w;
        }
        uint32_t tot, st = rw_excl_scan(sum, lane, &tot), blim = 0xffffffffu, lim = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t s0 = st, s1 = s0 + c[i].x, s2 = s1 + c[i].y, s3 = s2 + c[i].z;
          st = s3 + c[i].w;
          reinterpret_cast<uint4*>(bins)[8 * lane + i] = make_uint4(s0, s1, s2, s3);
          const uint32_t b0 = 32 * lane + 4 * i;
          if (blim == 0xffffffffu) {
            if (s0 >= K) { blim = b0; lim = s0; }
            else if (s1 >= K) { blim = b0 + 1; lim = s1; }
            else if (s2 >= K) { blim = b0 + 2; lim = s2; }
            else if (s3 >= K) { blim = b0 + 3; lim = s3; }
          }
        }
        blim = __reduce_min_sync(0xffffffffu, blim);
        lim = min(M, __reduce_min_sync(0xffffffffu, lim));
        __syncwarp();
        auto bin_of = [&](uint32_t key) {
          return ((kmax - (~(key >> 16) & 0xffffu)) << 2) | ((key & 0xffffu) >> a.sub_shift);
        };
        for (uint32_t x = lane; x < M; x += 32) {  // scatter the bins wholly below rank K
          const uint32_t key = cand[x], bn = bin_of(key);
          if (bn < blim) tmp[atomicAdd(&bins[bn], 1u)] = key;
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
      } else {  // candidate values span more than 256 codes: sort them
        uint32_t P2 = 2;
        while (P2 < M) P2 <<= 1;
        for (uint32_t x = M + lane; x < P2; x += 32) cand[x] = ~0u;  // cand | tmp hold 2 cap >= P2
        __syncwarp();
        group_bitonic_sort<uint32_t>(cand, P2, lane, 32);
        for (uint32_t x = lane; x < K; x += 32) {
          ov[x] = __uint_as_float(code16_bits(~(cand[x] >> 16) & 0xffffu) << 16);
          oi[x] = cand[x] & 0xffffu;
        }
      }
      __syncwarp();
      continue;
    }

    // ---- exact path: Alg. 1 summaries of every bucket this lane owns ------
    uint64_t* gx = a.gws + (uint64_t)blockIdx.x * a.P;
    uint32_t nn = 0;
#pragma unroll 1
    for (int b = 0; b < NB; ++b) {
      const uint32_t bk = 4 * (lane + 32 * (b >> 2)) + (b & 3);
      Summ<KP> sm;
      sm.clear();
      for (uint32_t r = 0; r < S; ++r) sm.push(__uint_as_float((uint32_t)xh[r * B + bk] << 16), r * B + bk, nn);
      float fv[KP];
      uint32_t fi[KP];
      sm.finalize(fv, fi);
#pragma unroll
      for (int j = 0; j < KP; ++j) gx[bk * KP + j] = rank_key_bits(__float_as_uint(fv[j]), fi[j]);
    }
    for (uint32_t q = B * KP + lane; q < a.P; q += 32) gx[q] = ~0ull;
    __syncwarp();
    uint64_t* srt = reinterpret_cast<uint64_t*>(rowp);  // the row is dead; P * 8 <= slot_bytes
    for (uint32_t q = lane; q < a.P; q += 32) srt[q] = gx[q];
    __syncwarp();
    group_bitonic_sort<uint64_t>(srt, a.P, lane, 32);
    for (uint32_t q = lane; q < K; q += 32) {
      ov[q] = __uint_as_float(key_value_bits(srt[q]));
      oi[q] = (uint32_t)srt[q];
    }
    ptx::fence_proxy_async();
    __syncwarp();
    issue(nrow);
  }
}

}  // namespace atkg
