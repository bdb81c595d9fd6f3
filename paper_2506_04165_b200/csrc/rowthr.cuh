// rowthr.cuh -- row-threshold approximate top-k for bf16 rows that fit in
// shared memory (the FFN-activation config: rows of 14336, 128 buckets of
// 112 elements).
//
// approx_top_k only needs the top K of the B*K' stage-1 candidates, not the
// grid.  One CTA owns one row (staged in shared memory by one 1-D TMA bulk
// copy); thread t = (word column p = t/2, row half h = t%2), a word holding
// the E = 2 adjacent buckets 2p, 2p+1.  Instead of exact per-bucket K'-th
// values the CTA works against one row threshold L:
//   sample   per-bucket maxima over every 4th stride-row (packed bf16x2
//            max), L = the r-th largest of those B maxima (bisection over
//            the 16-bit value code); r is set by the host so that about
//            1.7 K elements of a row are >= L;
//   collect  one packed compare per word marks the elements >= L in 16-row
//            mask words (each thread: its column, its half of the rows);
//   verify   c_b = #marks of bucket b, M = sum_b min(K', c_b).  If M >= K,
//            every candidate below L ranks after >= K candidates >= L, so
//            the top K of the row's candidates are the top K of its
//            candidates >= L -- and those are known exactly:
//              c_b <= K': the candidates of bucket b that are >= L are its
//                         marked elements themselves (all exceed v*_b, or
//                         are its only ties);
//              c_b >  K': v*_b >= L, so the marked elements contain every
//                         element >= v*_b, and the closed form of Alg. 1
//                         over them (the S* lemma and finalize in
//                         stage1.cuh / summ.cuh) is the reference state
//                         (/root/reference/proj/core/src/topk.cpp:80-102);
//            otherwise (M < K, L = -inf/NaN, too many marks) the CTA runs the
//            exact slow path: Alg. 1 summaries over every element;
//   extract  marks of small buckets are written straight out as rank keys
//            (value desc, index asc; topk.cpp:30-50); marks of large buckets
//            are listed bucket-major and every thread decides an equal share
//            of them from counts over their bucket's marks (greater /
//            equal-and-earlier / equal), which give v*, the bigs and the kept
//            ties directly -- no per-bucket serial loops;
//   select   the M keys are counting-sorted on (value code, index quarter),
//            ties ranked by index inside their bin (bitonic when the values
//            spread too far), and the first K emitted.
// Results are bit-identical to approx_top_k (topk.cpp:238-258).
#pragma once

#include "rowres.cuh"

namespace atkg {

constexpr int kThrNV = 256;      // counting sort: value codes the candidates may span
constexpr int kThrSub = 4;       // counting sort: index sub-bins per value code
constexpr int kThrNB = kThrNV * kThrSub;
constexpr int kThrRun = 64;      // counting sort: longest bin ranked by scanning
constexpr int kThrRPW = 16;      // stride-rows per mask word (bits [16e, 16e+16) = element e)
constexpr int kThrHalf = 4;      // mask words per row half (rows <= 2 * 4 * 16 = 128)
constexpr uint32_t kThrGCap = 512;   // marks of large buckets listed per row

// ascending order code of bf16 bits (-0 == +0) and back
__device__ __forceinline__ uint32_t asc_code16(uint32_t h) {
  if (h == 0x8000u) h = 0;
  return (h & 0x8000u) ? (~h & 0xffffu) : (h | 0x8000u);
}
__device__ __forceinline__ uint32_t code16_bits(uint32_t c) { return (c & 0x8000u) ? (c & 0x7fffu) : (~c & 0xffffu); }

__device__ __forceinline__ uint32_t bf2_max(uint32_t a, uint32_t b) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a), y = *reinterpret_cast<__nv_bfloat162*>(&b);
  const __nv_bfloat162 m = __hmax2(x, y);
  return *reinterpret_cast<const uint32_t*>(&m);
}
__device__ __forceinline__ float bf_at(const uint8_t* row, uint32_t pos) {
  return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(row)[pos] << 16);
}
__device__ __forceinline__ void emit_key32(uint32_t key, float* ov, uint32_t* oi) {
  *ov = key32_value_bf16(key);
  *oi = key & 0xffffu;
}

// exclusive block scan of a 64-bit value (all threads); *total = the sum
__device__ __forceinline__ uint64_t block_excl_scan64(uint64_t v, uint64_t* wsum, uint64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  uint64_t pre = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    const uint64_t s = wsum[w];
    pre += w < warp ? s : 0ull;
    tot += s;
  }
  *total = tot;
  __syncthreads();  // wsum reusable
  return pre + incl - v;
}

// The CTA emits the first k (ascending) of the M keys in keys[0..M).  Unique
// keys are counting-sorted: bin = (value code - lowest) * kThrSub + index >>
// sub_shift, so a bin holds equal values from one quarter of the row and is
// ranked by a short scan; when the values span more than kThrNV codes or a
// bin outgrows kThrRun -- or keys may repeat (the slow path's sentinels) -- a
// bitonic sort runs instead (P = pow2 >= M must fit in keys[]).  scr (tmp[M]
// | start[NB+4] | cur[NB], 16-byte aligned) may alias the dead row; red is
// 32 words of reduction scratch.
__device__ __forceinline__ void thr_sort_emit(uint32_t* keys, uint32_t* scr, uint32_t* red, uint32_t M, uint32_t k,
                                              bool unique, uint32_t sub_shift, float* ov, uint32_t* oi) {
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  const int lane = t & 31, warp = t >> 5, nw = nt >> 5;
  if (unique) {
    uint32_t lo = 0xffffffffu, hi = 0;
    for (uint32_t q = t; q < M; q += nt) {
      const uint32_t d = keys[q] >> 16;
      lo = min(lo, d);
      hi = max(hi, d);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) { red[warp] = lo; red[16 + warp] = hi; }
    __syncthreads();
    lo = 0xffffffffu;
    hi = 0;
    for (int w = 0; w < nw; ++w) { lo = min(lo, red[w]); hi = max(hi, red[16 + w]); }
    if (hi - lo < (uint32_t)kThrNV) {  // uniform
      uint32_t* tmp = scr;
      uint32_t* start = scr + ((M + 3) & ~3u);
      uint32_t* cur = start + kThrNB + 4;
      auto bin = [&](uint32_t key) { return ((key >> 16) - lo) * kThrSub + ((key & 0xffffu) >> sub_shift); };
      const uint32_t per = kThrNB / nt;  // bins scanned per thread (>= 2)
      for (uint32_t i = 0; i < per; i += 2) *reinterpret_cast<uint2*>(start + t * per + i) = make_uint2(0, 0);
      __syncthreads();  // also: every thread has read red[]
      for (uint32_t q = t; q < M; q += nt) atomicAdd(&start[bin(keys[q])], 1u);
      __syncthreads();
      uint32_t s = 0, mx = 0;
      for (uint32_t i = 0; i < per; ++i) {
        const uint32_t c = start[t * per + i];
        s += c;
        mx = max(mx, c);
      }
      mx = __reduce_max_sync(0xffffffffu, mx);
      // block scan of s (warp totals in red[16..]), block max of mx (red[0..])
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) { red[16 + warp] = incl; red[warp] = mx; }
      __syncthreads();
      uint32_t ex = incl - s;
      mx = 0;
      for (int w = 0; w < nw; ++w) {
        ex += w < warp ? red[16 + w] : 0u;
        mx = max(mx, red[w]);
      }
      if (mx <= (uint32_t)kThrRun) {  // uniform
        for (uint32_t i = 0; i < per; ++i) {
          const uint32_t c = start[t * per + i];
          start[t * per + i] = ex;
          cur[t * per + i] = ex;
          ex += c;
        }
        if (t == nt - 1) start[kThrNB] = M;
        __syncthreads();
        for (uint32_t q = t; q < M; q += nt) {
          const uint32_t key = keys[q];
          tmp[atomicAdd(&cur[bin(key)], 1u)] = key;
        }
        __syncthreads();
        for (uint32_t q = t; q < M; q += nt) {
          const uint32_t key = tmp[q];
          const uint32_t d = bin(key);
          const uint32_t a = start[d], e = start[d + 1];
          uint32_t r = a;
          for (uint32_t x = a; x < e; ++x) r += tmp[x] < key ? 1u : 0u;
          if (r < k) emit_key32(key, ov + r, oi + r);
        }
        return;
      }
    }
    __syncthreads();
  }
  uint32_t P = 2;
  while (P < M) P <<= 1;
  for (uint32_t q = M + t; q < P; q += nt) keys[q] = ~0u;
  __syncthreads();
  group_bitonic_sort<uint32_t>(keys, P, t, nt);
  for (uint32_t q = t; q < k; q += nt) emit_key32(keys[q], ov + q, oi + q);
}

// CTA = B threads = one row (W = B/2 word columns, 2 threads per column).
// smem: row (region: rows rounded to 16 rows, >= the sort scratch) | keys[cap]
// | glist[kThrGCap] (value bits << 16 | position) | gord[kThrGCap] (u16) |
// goff[B], gcnt[B] (u16)
template <int KP, int B>
__global__ void __launch_bounds__(B) row_threshold_kernel(const __nv_bfloat16* __restrict__ in, uint32_t n,
                                                          uint32_t k, uint32_t cap, uint32_t rsel,
                                                          uint32_t row_region, float* out_v, uint32_t* out_i,
                                                          uint32_t* status) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t red64[16];
  __shared__ uint32_t red[32];
  const uint32_t t = threadIdx.x;
  const int lane = t & 31;
  const uint32_t p = t >> 1, h = t & 1;  // word column, row half (= element for extraction)
  constexpr uint32_t W = B / 2;
  const uint64_t row = blockIdx.x;
  const uint32_t row_bytes = n * 2u;
  if (t == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&bar, row_bytes);
    ptx::bulk_g2s(smem_raw, in + row * n, row_bytes, &bar, ptx::policy_evict_first());
  }
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw + row_region);
  uint32_t* glist = keys + cap;
  uint16_t* gord = reinterpret_cast<uint16_t*>(glist + kThrGCap);
  uint16_t* goff = gord + kThrGCap;
  uint16_t* gcnt = goff + B;
  uint32_t* codes_sm = keys;  // the B sampled maxima, dead before the first key is written
  const uint32_t nstr = n / B;
  const uint32_t filled = min((uint32_t)KP, nstr);
  const uint32_t b = 2 * p + h;  // this thread's bucket (extraction, slow path)
  __syncthreads();
  ptx::mbar_wait(&bar, 0);
  const uint32_t* words = reinterpret_cast<const uint32_t*>(smem_raw) + p;
  const uint32_t j0 = h * kThrHalf * kThrRPW;  // first stride-row of this half
  const uint32_t j1 = min(nstr, j0 + kThrHalf * kThrRPW);

  // ---- sample: per-bucket maxima over every 4th stride-row (all when < 16) --
  uint32_t mx = 0xff80ff80u;
  if (nstr >= 16) {
#pragma unroll 4
    for (uint32_t j = j0; j < j1; j += 4) mx = bf2_max(mx, words[j * W]);
  } else {
    for (uint32_t j = j0; j < j1; ++j) mx = bf2_max(mx, words[j * W]);
  }
  mx = bf2_max(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  codes_sm[b] = asc_code16(h ? (mx >> 16) : (mx & 0xffffu));
  __syncthreads();
  // ---- L = rsel-th largest maximum: warp 0 bisects the B codes -------------
  if (t < 32) {
    uint32_t cr[B / 32];
#pragma unroll
    for (int i = 0; i < B / 32; ++i) cr[i] = codes_sm[i * 32 + lane];
    uint32_t pre = 0;
#pragma unroll 1
    for (int bit = 15; bit >= 0; --bit) {
      const uint32_t tt = pre | (1u << bit);
      uint32_t c = 0;
#pragma unroll
      for (int i = 0; i < B / 32; ++i) c += cr[i] >= tt ? 1u : 0u;
      c = __reduce_add_sync(0xffffffffu, c);
      if (c >= rsel) pre = tt;
    }
    if (t == 0) red[31] = pre;
  }
  __syncthreads();  // codes_sm (= keys) is overwritten below
  const uint32_t pre = red[31];
  bool fast = pre > 0x007fu && pre <= 0xff80u;  // L strictly above -inf, at most +inf
  const uint32_t L = code16_bits(pre), L2 = L | (L << 16);

  uint32_t nan = 0;
  uint32_t bm[kThrHalf];  // this bucket's marks, 32 stride-rows per word
  uint32_t cb = 0;
  if (fast) {  // uniform
    // ---- collect (own half of the column) ------------------------------------
    uint32_t m[kThrHalf];
#pragma unroll
    for (int i = 0; i < kThrHalf; ++i) {
      m[i] = 0;
      const uint32_t jc = j0 + i * kThrRPW;
      if (jc < j1) {
        const uint32_t* wp = words + jc * W;
        uint32_t a0 = 0, a1 = 0;
#pragma unroll
        for (int q = 0; q < kThrRPW; q += 2) {
          a0 |= WordNet<__nv_bfloat16>::hitmask(wp[q * W], L2) & (0x00010001u << q);
          a1 |= WordNet<__nv_bfloat16>::hitmask(wp[(q + 1) * W], L2) & (0x00010001u << (q + 1));
        }
        const uint32_t rem = j1 - jc;
        m[i] = (a0 | a1) & (rem >= (uint32_t)kThrRPW ? 0xffffffffu : ((1u << rem) - 1u) * 0x00010001u);
      }
    }
    // ---- both halves of the column; this thread's bucket is element e = h ----
    uint32_t fm[2 * kThrHalf];
#pragma unroll
    for (int i = 0; i < kThrHalf; ++i) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, m[i], 1);
      fm[i] = h ? o : m[i];
      fm[kThrHalf + i] = h ? m[i] : o;
    }
#pragma unroll
    for (int c = 0; c < kThrHalf; ++c) {
      const uint32_t lo16 = h ? (fm[2 * c] >> 16) : (fm[2 * c] & 0xffffu);
      const uint32_t hi16 = h ? (fm[2 * c + 1] >> 16) : (fm[2 * c + 1] & 0xffffu);
      bm[c] = lo16 | (hi16 << 16);
      cb += __popc(bm[c]);
    }
  }
  // ---- verify (block-uniform) ------------------------------------------------
  // scan fields: [0,16) small-bucket marks, [16,32) large buckets, [32,64)
  // large-bucket marks; M = small marks + K' * large buckets
  const bool large = cb > (uint32_t)KP;
  uint64_t tot;
  const uint64_t off = block_excl_scan64(
      fast ? (large ? (1ull << 16) | ((uint64_t)cb << 32) : (uint64_t)cb) : 0ull, red64, &tot);
  const uint32_t S = (uint32_t)(tot & 0xffffu), NL = (uint32_t)((tot >> 16) & 0xffffu), G = (uint32_t)(tot >> 32);
  uint32_t M = S + KP * NL;
  fast = fast && M >= k && G <= kThrGCap;
#ifdef ATKG_THR_STATS
  if (t == 0) {
    atomicAdd(status + 1, fast ? 0u : 1u);
    atomicAdd(status + 2, S + G);
    atomicAdd(status + 3, M);
    atomicAdd(status + 4, G);
    atomicAdd(status + 5, G > kThrGCap ? 1u : 0u);
  }
#endif
  if (fast) {
    // ---- small buckets: keys out; large buckets: marks listed ----------------
    const uint16_t* row16 = reinterpret_cast<const uint16_t*>(smem_raw);
    if (!large) {
      uint32_t o = (uint32_t)(off & 0xffffu);
#pragma unroll
      for (int c = 0; c < kThrHalf; ++c) {
        uint32_t w = bm[c];
        while (w) {
          const uint32_t pos = (32 * c + __ffs(w) - 1) * B + b;
          w &= w - 1;
          const uint32_t hv = (uint32_t)row16[pos] << 16;
          if (__uint_as_float(hv) != __uint_as_float(hv)) nan = 1u;
          keys[o++] = rank_key32_bf16(hv, pos);
        }
      }
    } else {
      const uint32_t ord = (uint32_t)((off >> 16) & 0xffffu);
      uint32_t o = (uint32_t)(off >> 32);
      goff[ord] = (uint16_t)o;
      gcnt[ord] = (uint16_t)cb;
#pragma unroll
      for (int c = 0; c < kThrHalf; ++c) {
        uint32_t w = bm[c];
        while (w) {
          const uint32_t pos = (32 * c + __ffs(w) - 1) * B + b;
          w &= w - 1;
          gord[o] = (uint16_t)ord;
          glist[o++] = ((uint32_t)row16[pos] << 16) | pos;
        }
      }
    }
    __syncthreads();
    // ---- large buckets: every thread decides an equal share of the marks ------
    // With g = #greater, e = #equal and earlier, eq = #equal (self included)
    // among the bucket's marks:
    //   big (x > v*)   iff g + eq <= K'-1      -> slot g + e
    //   tie (x == v*)  iff g <= K'-1 < g + eq  (nb = g, c = K' - g, t = e+1):
    //                  kept if t <= c-1 (slot g + e) or if it is X = the last
    //                  tie when that follows the last big (or there is no
    //                  big), else the c-th tie (slot K'-1)  (summ.cuh finalize)
    for (uint32_t q = t; q < G; q += B) {
      const uint32_t hv = glist[q];
      const uint32_t pos = hv & 0xffffu, ord = gord[q];
      const float x = __uint_as_float(hv & 0xffff0000u);
      if (x != x) {
        nan = 1u;
        continue;
      }
      const uint32_t ho = goff[ord], c = gcnt[ord];
      uint32_t g = 0, e = 0, eq = 0, maxg = 0, lasteq = pos;
      for (uint32_t r = ho; r < ho + c; ++r) {
        const uint32_t hr = glist[r];
        const float xr = __uint_as_float(hr & 0xffff0000u);
        const uint32_t pr = hr & 0xffffu;
        g += xr > x ? 1u : 0u;
        maxg = xr > x ? max(maxg, pr) : maxg;
        const bool same = xr == x;
        eq += same ? 1u : 0u;
        e += (same && pr < pos) ? 1u : 0u;
        lasteq = same ? max(lasteq, pr) : lasteq;
      }
      uint32_t slot = 0xffffffffu;
      if (g + eq <= (uint32_t)KP - 1) {
        slot = g + e;
      } else if (g <= (uint32_t)KP - 1) {
        const uint32_t ct = KP - g;
        if (e + 2 <= ct) slot = g + e;
        else if ((g == 0 || lasteq > maxg) ? (e + 1 == eq) : (e + 1 == ct)) slot = KP - 1;
      }
      if (slot != 0xffffffffu) keys[S + KP * ord + slot] = rank_key32_bf16(hv & 0xffff0000u, pos);
    }
  } else {
    // ---- exact slow path: Alg. 1 summary of bucket b over every element -------
    M = filled * B;
    Summ<KP> s;
    s.clear();
    for (uint32_t j = 0; j < nstr; ++j) s.push(bf_at(smem_raw, j * B + b), j * B + b, nan);
    float fv[KP];
    uint32_t fi[KP];
    s.finalize(fv, fi);
#pragma unroll
    for (int kk = 0; kk < KP; ++kk)
      if ((uint32_t)kk < filled) keys[b * filled + kk] = rank_key32_bf16(__float_as_uint(fv[kk]), fi[kk]);
  }
  if (__syncthreads_or(nan)) {  // the reference rejects NaN before ranking
    if (t == 0) atomicOr(status, ATKG_FLAG_NAN);
    return;
  }
  const uint32_t sub_shift = n > 4 ? (uint32_t)max(0, 32 - __clz((int)(n - 1)) - 2) : 0u;
  thr_sort_emit(keys, reinterpret_cast<uint32_t*>(smem_raw), red, M, k, fast, sub_shift, out_v + row * k,
                out_i + row * k);
}

}  // namespace atkg
