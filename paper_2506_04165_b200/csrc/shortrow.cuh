// shortrow.cuh -- approx_top_k for bf16 rows that fit in shared memory: the
// FFN-activation config (rows of 14336, K = 287) and its K' sweep.
//
// approx_top_k (/root/reference/proj/core/src/topk.cpp:238-258) returns the
// top K of the B*K' stage-1 candidates.  For a row threshold L let c_b =
// #elements of bucket b (= i mod B, topk.hpp:13-15) that are >= L and
// M = sum_b min(K', c_b).  If M >= K, the top K of the candidates are the
// top K of the candidates >= L, and those follow from the elements >= L
// alone: Alg. 1 (topk.cpp:80-102) over the subsequence of a bucket's
// elements >= L ends, restricted to entries >= L, in the reference state
// (c_b <= K': every such element survives; c_b > K': v*_b >= L, the
// subsequence holds every element >= v*_b -- the S* lemma).
//
// Guaranteed threshold.  Cut every bucket into K' disjoint groups of
// consecutive stride-rows and let L = the K-th largest of the B*K' group
// maxima.  At least K groups have a maximum >= L, each holds an element
// >= L, and a bucket owns at most K' groups, so M >= K.  No sampled guess,
// no retry.
//
// One CTA (8 warps) per row at a time, persistent over rows, two row slots
// filled by 1-D TMA bulk copies (the next row loads while this one runs).
// A group's stride-rows are cut into parts of <= 32; a unit = (8-byte chunk
// column c = 4 buckets, mask word q = (group, part)).
//   pass 1   per unit: NaN-propagating packed max over the part's rows;
//   select   the K-th largest group maximum (max over the parts) by a
//            256-bin histogram of the ascending 16-bit keys binned down
//            from the row maximum (a second, finer histogram inside the
//            chosen bin when those bins are wide) -> L, a lower bound of it;
//   pass 2   per unit: one packed compare per word sets the bits of the
//            per-(bucket, word) hit masks -- no lists, no atomics;
//   count    thread = bucket: c_b = sum of its words' popcounts; crowded
//            buckets (c_b > K') are queued;
//   collect  per unit: the hits of uncrowded buckets become candidates
//            (warp scan + one atomic per warp for their slots); per queued
//            bucket: Alg. 1 over its hits in position order (values read
//            back from the resident row);
//   stage 2  counting sort of the M >= K candidates' 32-bit rank keys
//            (~key16 << 16 | pos: value desc, index asc; topk.cpp:30-50)
//            on (value code, index quarter) bins, ranks inside a bin by
//            comparison, the first K written out.
// Rows with L = -inf (sentinel semantics) or more candidates than the
// candidate buffer takes run the exact path in the kernel: Alg. 1
// summaries of every bucket from the resident row (summ.cuh), a bitonic sort
// of the B*K' candidates, the first K emitted.  NaN rows raise
// ATKG_FLAG_NAN (the reference throws "input contains NaN").
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "ptx.cuh"
#include "rowthr.cuh"
#include "summ.cuh"

namespace atkg {

constexpr int kSrThreads = 256;
constexpr int kSrWarps = kSrThreads / 32;
constexpr uint32_t kSrKeyNegInf = 0x007fu;  // asc_code16(-inf)
constexpr uint32_t kSrMaxWords = 64;        // mask words per bucket (K' * parts)
constexpr uint32_t kSrBins = 1024;          // stage 2: 256 value codes x 4 index quarters

struct SrArgs {
  const void* in;
  uint64_t rows;
  uint32_t n, B, S, k;
  uint32_t cps;         // 8-byte chunks per stride-row (B / 4)
  uint32_t npart;       // parts per group
  uint32_t pl;          // stride-rows per part (<= 32)
  uint32_t cap;         // candidate buffer
  uint32_t slot_bytes;  // one row slot: the row, later the stage-2 scratch
  uint32_t row_bytes;
  uint32_t P;           // exact path: pow2 >= B * K'
  uint32_t sub_shift;   // stage 2: pos >> sub_shift < 4
  uint32_t force_slow;  // tests: every row takes the exact path
  uint32_t probe;       // development: stream the rows only
  uint64_t* gws;        // exact path scratch, [grid][P]
  const uint32_t* row_list;   // optional: only these rows (rowmax1.cuh leaves it the rows it could not settle)
  const uint32_t* row_count;  //           how many (device)
  float* out_v;
  uint32_t* out_i;
  uint32_t* status;
};

// smem (dynamic): slot[2] | cand[cap] u32 | rm[nw * B] u32 | cnt[B] u32 |
// gmp[nw * B] u16 | crowd[cap / K'] u32 | seg[cap] u32,  nw = K' * npart
__host__ __device__ constexpr size_t sr_smem_bytes(uint32_t slot_bytes, uint32_t cap, uint32_t kp, uint32_t npart,
                                                   uint32_t B) {
  return 2ull * slot_bytes + 4ull * cap + 4ull * kp * npart * B + 4ull * B +
         ((2ull * kp * npart * B + 15) / 16 * 16) + 4ull * cap / kp + 4ull * cap;
}

__device__ __forceinline__ uint2 sr_vmax(uint2 a, uint2 b) {
  return make_uint2(bmax_nan(a.x, b.x), bmax_nan(a.y, b.y));
}

// marks the halves of a bf16x2 word that are >= L: mlo |= bit, mhi |= bit
__device__ __forceinline__ void sr_mark(uint32_t w, uint32_t L2, uint32_t bit, uint32_t& mlo, uint32_t& mhi) {
  asm("{\n\t.reg .pred p, q;\n\t"
      "setp.ge.bf16x2 p|q, %2, %3;\n\t"
      "@p or.b32 %0, %0, %4;\n\t"
      "@q or.b32 %1, %1, %4;\n\t}"
      : "+r"(mlo), "+r"(mhi)
      : "r"(w), "r"(L2), "r"(bit));
}

// Alg. 1 keeps a hit of a crowded bucket?  (closed form of summ.cuh
// finalize over the bucket's hits, as in st_finish_kernel): g = #greater,
// eq = #equal (itself included), e = #equal and earlier, maxg / lasteq =
// last position among the greater / the equal ones.
template <int KP>
__device__ __forceinline__ bool sr_kept(uint32_t g, uint32_t eq, uint32_t e, uint32_t maxg, uint32_t lasteq) {
  if (g + eq <= (uint32_t)KP - 1) return true;  // above v*
  if (g > (uint32_t)KP - 1) return false;       // below v*
  const uint32_t ct = KP - g;                   // slots left for the ties at v*
  if (e + 2 <= ct) return true;                 // one of the first ct - 1 ties
  return (g == 0 || lasteq > maxg) ? (e + 1 == eq) : (e + 1 == ct);
}

template <int KP>
__global__ void __launch_bounds__(kSrThreads) short_row_kernel(SrArgs a) {
  extern __shared__ __align__(128) uint8_t sr_smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t red_max[kSrWarps], red_min[kSrWarps], red_nan[kSrWarps], red_s[kSrWarps];
  __shared__ uint32_t hist[256];
  __shared__ __align__(16) uint32_t ebin[kSrBins];
  __shared__ uint32_t rbase[kSrMaxWords], rlen[kSrMaxWords];
  __shared__ uint32_t sh_L, sh_j1, sh_need, sh_ncl, sh_m, sh_cs, sh_lim, sh_blim;
  __shared__ uint32_t red[32];
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t B = a.B, S = a.S, cps = a.cps, npart = a.npart;
  constexpr uint32_t kNone = 0xffffffffu;
  const uint32_t nw = KP * npart;
  uint8_t* slots = sr_smem;
  uint32_t* cand = reinterpret_cast<uint32_t*>(sr_smem + 2ull * a.slot_bytes);
  uint32_t* rm = cand + a.cap;                                        // [q * B + b] hit masks
  uint32_t* cnt = rm + (size_t)nw * B;                                // [b] hits per bucket
  uint16_t* gmp = reinterpret_cast<uint16_t*>(cnt + B);               // [q * B + b] part-maximum keys
  uint32_t* crowd = reinterpret_cast<uint32_t*>(gmp + (((size_t)nw * B + 7) & ~7ull));  // [cap / K']
  uint32_t* seg = crowd + a.cap / KP;                                 // [cap] crowded buckets' hits
  const uint32_t U = cps * nw;                                        // units (word q, chunk column c)
  const uint32_t upt = (U + kSrThreads - 1) / kSrThreads;
  const uint32_t bpt = (B + kSrThreads - 1) / kSrThreads;
  const uint64_t pol = ptx::policy_evict_first();
  const uint8_t* in = static_cast<const uint8_t*>(a.in);
  for (uint32_t q = t; q < nw; q += kSrThreads) {
    const uint32_t g = q / npart, p = q - g * npart;
    const uint32_t r0 = g * S / KP + p * a.pl, r1 = min((g + 1) * S / KP, r0 + a.pl);
    rbase[q] = r0;
    rlen[q] = r1 > r0 ? r1 - r0 : 0u;
  }
  if (t == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint64_t nwork = a.row_list ? (uint64_t)*a.row_count : a.rows;
  auto row_of = [&](uint64_t i) { return a.row_list ? (uint64_t)a.row_list[i] : i; };
  uint64_t widx = blockIdx.x;
  if (t == 0 && widx < nwork) {
    ptx::mbar_arrive_expect_tx(&bar[0], a.row_bytes);
    ptx::bulk_g2s(slots, in + row_of(widx) * a.row_bytes, a.row_bytes, &bar[0], pol);
  }
#pragma unroll 1
  for (uint32_t it = 0; widx < nwork; ++it, widx += gridDim.x) {
    const uint64_t row = row_of(widx);
    const uint32_t s = it & 1;
    uint8_t* rowp = slots + (size_t)s * a.slot_bytes;
    const uint2* ch = reinterpret_cast<const uint2*>(rowp);
    const uint16_t* xh = reinterpret_cast<const uint16_t*>(rowp);
    {  // the next row into the other slot (its last use ended at the previous barrier)
      const uint64_t nidx = widx + gridDim.x;
      if (t == 0 && nidx < nwork) {
        ptx::mbar_arrive_expect_tx(&bar[s ^ 1], a.row_bytes);
        ptx::bulk_g2s(slots + (size_t)(s ^ 1) * a.slot_bytes, in + row_of(nidx) * a.row_bytes, a.row_bytes,
                      &bar[s ^ 1], pol);
      }
    }
    hist[t & 255] = 0;
    for (uint32_t i = t; i < kSrBins; i += kSrThreads) ebin[i] = 0;
    if (t == 0) { sh_ncl = 0; sh_m = 0; sh_cs = 0; }
    ptx::mbar_wait(&bar[s], (it >> 1) & 1);
    if (a.probe == 1) {  // development: the row pipeline alone (no compute, no output)
      __syncthreads();
      continue;
    }

    // ---- pass 1: part maxima (keys) ------------------------------------
    uint32_t kmax = 0, kmin = 0xffffffffu, nan = 0;
#pragma unroll 1
    for (uint32_t uu = 0; uu < upt; ++uu) {
      const uint32_t u = t + uu * kSrThreads;
      if (u >= U) break;
      const uint32_t q = u / cps, c = u - q * cps;
      const uint32_t len = rlen[q];
      const uint2* p = ch + (size_t)rbase[q] * cps + c;
      uint2 acc = make_uint2(0xff80ff80u, 0xff80ff80u);
#pragma unroll 4
      for (uint32_t i = 0; i < len; ++i) acc = sr_vmax(acc, p[i * cps]);
      uint32_t k4[4] = {acc.x & 0xffffu, acc.x >> 16, acc.y & 0xffffu, acc.y >> 16};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        nan |= (k4[j] & 0x7fffu) > 0x7f80u ? 1u : 0u;
        k4[j] = asc_code16(k4[j]);
        kmax = max(kmax, k4[j]);
        kmin = min(kmin, k4[j]);
      }
      *reinterpret_cast<uint2*>(gmp + (size_t)q * B + c * 4) = make_uint2(k4[0] | (k4[1] << 16), k4[2] | (k4[3] << 16));
    }
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    nan = __reduce_or_sync(0xffffffffu, nan);
    if (lane == 0) { red_max[warp] = kmax; red_min[warp] = kmin; red_nan[warp] = nan; }
    __syncthreads();
    kmax = 0; kmin = 0xffffffffu; nan = 0;
#pragma unroll
    for (int w = 0; w < kSrWarps; ++w) { kmax = max(kmax, red_max[w]); kmin = min(kmin, red_min[w]); nan |= red_nan[w]; }
    if (nan) {  // uniform: the reference rejects the input
      if (t == 0) atomicOr(a.status, ATKG_FLAG_NAN);
      ptx::fence_proxy_async();
      __syncthreads();
      continue;
    }

    // ---- select: L = a lower bound of the K-th largest group maximum -----
    // level 1: 256 bins of width 2^shf below kmax; level 2 (only when those
    // bins are wider than 4 codes): 256 bins of width 2^(shf-8) inside the
    // bin that reaches rank K.  L = the lowest key of the final bin.
    const uint32_t span = kmax - kmin;
    const uint32_t shf = span < 256u ? 0u : (uint32_t)(32 - __clz(span >> 8));
    const uint32_t nkeys = KP * B;
    auto gkey = [&](uint32_t i) {  // group maximum i = g * B + b: max over the group's parts
      const uint32_t g = i / B, b = i - g * B;
      uint32_t m = 0;
      for (uint32_t p = 0; p < npart; ++p) m = max(m, (uint32_t)gmp[(size_t)(g * npart + p) * B + b]);
      return m;
    };
    for (uint32_t i = t; i < nkeys; i += kSrThreads) atomicAdd(&hist[min(255u, (kmax - gkey(i)) >> shf)], 1u);
    __syncthreads();
    // warp 0: the first bin whose cumulative count reaches `need`, and the
    // count before it
    auto scan_bins = [&](uint32_t need, uint32_t& bin, uint32_t& before) {
      uint32_t c8[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { c8[i] = hist[lane * 8 + i]; sum += c8[i]; }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      uint32_t cum = incl - sum, jb = kNone, bef = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (jb == kNone && cum + c8[i] >= need) { jb = lane * 8 + i; bef = cum; }
        cum += c8[i];
      }
      const uint32_t j = __reduce_min_sync(0xffffffffu, jb);
      before = __shfl_sync(0xffffffffu, bef, (j >> 3) & 31);
      bin = j;
    };
    if (warp == 0) {
      uint32_t j1, before;
      scan_bins(a.k, j1, before);
      if (lane == 0) {
        sh_j1 = j1;
        sh_need = a.k - before;
        const uint64_t w = ((uint64_t)(j1 + 1) << shf) - 1;  // bin j1 = keys kmax - [j1 << shf, w]
        sh_L = (j1 >= 255u || w >= (uint64_t)span) ? kmin : kmax - (uint32_t)w;
      }
    }
    __syncthreads();
    if (shf > 2) {  // uniform: refine inside bin j1 (bins of <= 4 codes are fine as they are)
      const uint32_t j1 = sh_j1, shf2 = shf > 8 ? shf - 8 : 0;
      const uint32_t need = sh_need;
      __syncthreads();  // every thread has read sh_j1 / sh_need
      hist[t & 255] = 0;
      __syncthreads();
      if (j1 < 255u) {  // the clamped last bin needs no refinement (L = kmin)
        for (uint32_t i = t; i < nkeys; i += kSrThreads) {
          const uint32_t d = kmax - gkey(i);
          if ((d >> shf) == j1) atomicAdd(&hist[min(255u, (d - (j1 << shf)) >> shf2)], 1u);
        }
      }
      __syncthreads();
      if (warp == 0 && j1 < 255u) {
        uint32_t j2, before;
        scan_bins(need, j2, before);
        if (lane == 0) {
          const uint64_t w = ((uint64_t)j1 << shf) + ((uint64_t)(j2 + 1) << shf2) - 1;
          sh_L = w >= (uint64_t)span ? kmin : kmax - (uint32_t)w;
        }
      }
      __syncthreads();
    }
    const uint32_t Lkey = sh_L;
    const uint32_t Lb = code16_bits(Lkey);
    const uint32_t L2 = Lb | (Lb << 16);
    bool slow = Lkey <= kSrKeyNegInf || a.force_slow;  // uniform
    if (a.probe == 2) {  // development: pass 1 + select only
      ptx::fence_proxy_async();
      __syncthreads();
      continue;
    }

    if (!slow) {
      // ---- pass 2: hit masks, one bit per (bucket, stride-row) ----------
#pragma unroll 1
      for (uint32_t uu = 0; uu < upt; ++uu) {
        const uint32_t u = t + uu * kSrThreads;
        if (u >= U) break;
        const uint32_t q = u / cps, c = u - q * cps;
        const uint32_t len = rlen[q];
        const uint2* p = ch + (size_t)rbase[q] * cps + c;
        uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0, bit = 1;
#pragma unroll 4
        for (uint32_t i = 0; i < len; ++i, bit <<= 1) {
          const uint2 v = p[i * cps];
          sr_mark(v.x, L2, bit, m0, m1);
          sr_mark(v.y, L2, bit, m2, m3);
        }
        *reinterpret_cast<uint4*>(rm + (size_t)q * B + c * 4) = make_uint4(m0, m1, m2, m3);
      }
      __syncthreads();
      if (a.probe == 3) {  // development: through pass 2
        ptx::fence_proxy_async();
        __syncthreads();
        continue;
      }
      // ---- count: c_b per bucket.  A crowded bucket (c_b > K') gets a
      // segment of its hits (seg[base, base + c_b), in position order: word
      // q's hits start at base + pfx[q][b]); cnt[b] = c_b | base << 16.
      for (uint32_t i = 0; i < bpt; ++i) {
        const uint32_t b = t + i * kSrThreads;
        if (b >= B) break;
        uint32_t cb = 0;
        for (uint32_t q = 0; q < nw; ++q) cb += __popc(rm[(size_t)q * B + b]);
        uint32_t base = 0;
        if (cb > (uint32_t)KP) {
          base = atomicAdd(&sh_cs, cb);
          crowd[min(atomicAdd(&sh_ncl, 1u), a.cap / KP - 1)] = b;
          uint32_t pf = 0;
          for (uint32_t q = 0; q < nw; ++q) {  // gmp (dead since select) holds the word prefixes
            gmp[(size_t)q * B + b] = (uint16_t)pf;
            pf += __popc(rm[(size_t)q * B + b]);
          }
        }
        cnt[b] = cb | (min(base, 0xffffu) << 16);
      }
      __syncthreads();
      if (a.probe == 5) {  // development: through count
        ptx::fence_proxy_async();
        __syncthreads();
        continue;
      }
      const uint32_t ncl = sh_ncl, cs = sh_cs;
      slow = ncl > a.cap / KP || cs > a.cap;  // uniform: heavy ties at L -> exact path
      uint32_t MU = 0;
      if (!slow) {
        // ---- collect: every hit's position -> cand[0, MU) (uncrowded) or
        // its crowded bucket's segment (one flat loop per unit)
#pragma unroll 1
        for (uint32_t uu = 0; uu < upt; ++uu) {  // warp-uniform trip count
          const uint32_t u = t + uu * kSrThreads;
          uint32_t m[4] = {0, 0, 0, 0}, sb[4] = {0, 0, 0, 0}, q = 0, c = 0, n = 0, cm = 0;
          if (u < U) {
            q = u / cps;
            c = u - q * cps;
            const uint4 mm = *reinterpret_cast<const uint4*>(rm + (size_t)q * B + c * 4);
            const uint4 cc = *reinterpret_cast<const uint4*>(cnt + c * 4);
            m[0] = mm.x; m[1] = mm.y; m[2] = mm.z; m[3] = mm.w;
            const uint32_t ce[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if ((ce[j] & 0xffffu) > (uint32_t)KP) {
                cm |= 1u << j;
                sb[j] = (ce[j] >> 16) + gmp[(size_t)q * B + c * 4 + j];
              } else {
                n += __popc(m[j]);
              }
            }
          }
          uint32_t incl = n;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += y;
          }
          uint32_t wbase = 0;
          if (lane == 31 && incl) wbase = atomicAdd(&sh_m, incl);
          uint32_t d = __shfl_sync(0xffffffffu, wbase, 31) + incl - n;
          const uint32_t pb = (u < U ? rbase[q] : 0u) * B + c * 4;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w = m[j];
            const bool crowded = (cm >> j) & 1u;
            uint32_t e = crowded ? sb[j] : d;
            while (w) {
              const uint32_t pos = pb + (uint32_t)(__ffs(w) - 1) * B + j;
              w &= w - 1;
              if (crowded) seg[e] = pos;
              else if (e < a.cap) cand[e] = pos;
              ++e;
            }
            if (!crowded) d = e;
          }
        }
        __syncthreads();
        MU = sh_m;
        slow = MU + (uint32_t)KP * ncl > a.cap;  // uniform
      }
      if (a.probe == 6) {  // development: through collect
        ptx::fence_proxy_async();
        __syncthreads();
        continue;
      }
      const bool binned = kmax - Lkey < 256u;  // uniform: candidate keys lie in [L, kmax]
      auto note = [&](uint32_t key, uint32_t pos) {  // stage-2 bin: (value code, index quarter)
        if (binned) atomicAdd(&ebin[((kmax - key) << 2) | (pos >> a.sub_shift)], 1u);
      };
      if (!slow) {
        // ---- candidates: the uncrowded hits' rank keys (~key16 << 16 | pos,
        // ascending = output order), in place; then per crowded bucket (one
        // thread each) Alg. 1 (topk.cpp:80-102) over its segment, which holds
        // its hits in position order, on ascending keys (the K' sentinels
        // rank below every hit: L > -inf)
        for (uint32_t x = t; x < MU; x += kSrThreads) {
          const uint32_t pos = cand[x], key = asc_code16(xh[pos]);
          cand[x] = ((~key & 0xffffu) << 16) | pos;
          note(key, pos);
        }
        for (uint32_t qc = t; qc < ncl; qc += kSrThreads) {  // thread = crowded bucket: Alg. 1 over its segment
          const uint32_t b = crowd[qc], ce = cnt[b], c = ce & 0xffffu;
          const uint32_t* sg = seg + (ce >> 16);
          uint32_t kv[KP], kq[KP];
#pragma unroll
          for (int j = 0; j < KP; ++j) { kv[j] = 0; kq[j] = 0; }
          for (uint32_t j = 0; j < c; ++j) {
            const uint32_t pos = sg[j], key = asc_code16(xh[pos]);
            if (key >= kv[KP - 1]) {
              kv[KP - 1] = key;
              kq[KP - 1] = pos;
#pragma unroll
              for (int i = KP - 1; i >= 1; --i) {
                if (kv[i] > kv[i - 1]) {
                  const uint32_t tv = kv[i]; kv[i] = kv[i - 1]; kv[i - 1] = tv;
                  const uint32_t tq = kq[i]; kq[i] = kq[i - 1]; kq[i - 1] = tq;
                }
              }
            }
          }
          const uint32_t wb = atomicAdd(&sh_m, (uint32_t)KP);
#pragma unroll
          for (int j = 0; j < KP; ++j) {
            cand[wb + j] = ((~kv[j] & 0xffffu) << 16) | kq[j];
            note(kv[j], kq[j]);
          }
        }
        __syncthreads();  // candidates complete; the row is dead (its slot: stage-2 scratch)
      }
      if (a.probe == 4) {  // development: through the candidates
        ptx::fence_proxy_async();
        __syncthreads();
        continue;
      }
      const uint32_t M = sh_m;
      if (!slow) {
        // ---- stage 2: the first K of the M >= K candidates -----------------
        float* ov = a.out_v + row * a.k;
        uint32_t* oi = a.out_i + row * a.k;
        auto cand_at = [&](uint32_t x) { return cand[x]; };
        if (!binned) {
          uint32_t* keys = reinterpret_cast<uint32_t*>(rowp);  // contiguous copy (the emit sorts in place)
          for (uint32_t x = t; x < M; x += kSrThreads) keys[x] = cand_at(x);
          __syncthreads();
          uint32_t P2 = 2;
          while (P2 < M) P2 <<= 1;
          thr_sort_emit(keys, keys + P2, red, M, a.k, true, a.sub_shift, ov, oi);
        } else {
          uint32_t* tmp = reinterpret_cast<uint32_t*>(rowp);
          // exclusive scan of the bins (4 per thread), the first bin starting at >= k
          const uint4 c4 = *reinterpret_cast<const uint4*>(ebin + 4 * t);
          const uint32_t sum = c4.x + c4.y + c4.z + c4.w;
          uint32_t inc = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if ((int)lane >= o) inc += y;
          }
          if (lane == 31) red_s[warp] = inc;
          if (t == 0) { sh_blim = kNone; sh_lim = M; }
          __syncthreads();
          uint32_t st = inc - sum;
#pragma unroll
          for (int w = 0; w < kSrWarps; ++w) st += w < (int)warp ? red_s[w] : 0u;
          const uint32_t s0 = st, s1 = s0 + c4.x, s2 = s1 + c4.y, s3 = s2 + c4.z;
          *reinterpret_cast<uint4*>(ebin + 4 * t) = make_uint4(s0, s1, s2, s3);
          uint32_t bl = kNone, lm = kNone;
          if (s3 >= a.k) {
            bl = s0 >= a.k ? 4 * t : s1 >= a.k ? 4 * t + 1 : s2 >= a.k ? 4 * t + 2 : 4 * t + 3;
            lm = s0 >= a.k ? s0 : s1 >= a.k ? s1 : s2 >= a.k ? s2 : s3;
          }
          bl = __reduce_min_sync(0xffffffffu, bl);
          lm = __reduce_min_sync(0xffffffffu, lm);
          if (lane == 0 && bl != kNone) { atomicMin(&sh_blim, bl); atomicMin(&sh_lim, lm); }
          __syncthreads();
          const uint32_t blim = sh_blim, lim = sh_lim;
          auto bin_of = [&](uint32_t key) {
            return ((kmax - (~(key >> 16) & 0xffffu)) << 2) | ((key & 0xffffu) >> a.sub_shift);
          };
          for (uint32_t x = t; x < M; x += kSrThreads) {  // scatter (bins wholly below rank k)
            const uint32_t key = cand_at(x), bn = bin_of(key);
            if (bn < blim) tmp[atomicAdd(&ebin[bn], 1u)] = key;
          }
          __syncthreads();  // ebin[b] = end of bin b = start of bin b + 1
          for (uint32_t x = t; x < lim; x += kSrThreads) {
            const uint32_t key = tmp[x], bn = bin_of(key);
            const uint32_t b0 = bn ? ebin[bn - 1] : 0u, b1 = ebin[bn];
            uint32_t r = b0;
            for (uint32_t y = b0; y < b1; ++y) r += tmp[y] < key ? 1u : 0u;
            if (r < a.k) {
              ov[r] = __uint_as_float(code16_bits(~(key >> 16) & 0xffffu) << 16);
              oi[r] = key & 0xffffu;
            }
          }
        }
      }
    }
    if (slow) {  // uniform
      // ---- exact path: Alg. 1 per bucket from the resident row ------------
      uint64_t* gx = a.gws + (uint64_t)blockIdx.x * a.P;
      uint32_t nn = 0;
      for (uint32_t b = t; b < B; b += kSrThreads) {
        Summ<KP> sm;
        sm.clear();
        for (uint32_t r = 0; r < S; ++r) sm.push(__uint_as_float((uint32_t)xh[r * B + b] << 16), r * B + b, nn);
        float fv[KP];
        uint32_t fi[KP];
        sm.finalize(fv, fi);
#pragma unroll
        for (int j = 0; j < KP; ++j) gx[b * KP + j] = rank_key_bits(__float_as_uint(fv[j]), fi[j]);
      }
      for (uint32_t q = B * KP + t; q < a.P; q += kSrThreads) gx[q] = ~0ull;
      __syncthreads();  // the row is dead: its slot becomes the sort buffer when it fits
      uint64_t* srt = gx;
      if ((size_t)a.P * 8 <= a.slot_bytes) {
        srt = reinterpret_cast<uint64_t*>(rowp);
        for (uint32_t q = t; q < a.P; q += kSrThreads) srt[q] = gx[q];
        __syncthreads();
      }
      group_bitonic_sort<uint64_t>(srt, a.P, t, kSrThreads);
      float* ov = a.out_v + row * a.k;
      uint32_t* oi = a.out_i + row * a.k;
      for (uint32_t q = t; q < a.k; q += kSrThreads) {
        ov[q] = __uint_as_float(key_value_bits(srt[q]));
        oi[q] = (uint32_t)srt[q];
      }
    }
    // generic-proxy use of this slot ends before the TMA refill
    ptx::fence_proxy_async();
    __syncthreads();
  }
}

}  // namespace atkg
