// rowpipe.cuh -- persistent row pipeline for bf16 rows that fit in shared
// memory (the FFN-activation config: rows of 14336, B = 128 buckets of 112).
//
// approx_top_k (/root/reference/proj/core/src/topk.cpp:238-258) needs the top
// K of the B*K' stage-1 candidates.  With a row threshold L and c_b = #marks
// (elements >= L) of bucket b, M = sum_b min(K', c_b): if M >= K the answer
// is the top K of the candidates >= L, and those follow from the marks alone
// (rowthr.cuh, streamthr.cuh).  Here every bucket runs Alg. 1
// (topk.cpp:80-102) over its marks in position order, from the reference's
// sentinel state {-inf, 0}: for c_b >= K' the marks hold every element >=
// v*_b (v*_b >= L) and Alg. 1 over that subsequence ends in the reference
// state (the S* lemma); for c_b < K' its entries >= L are the marks
// themselves.  Otherwise (M < K, L = -inf, NaN) the row takes the exact slow
// path: Alg. 1 summaries over every element.
//
// Layout: one CTA per SM, NG groups of B threads; group g owns two row
// buffers and processes every NG-th row of the CTA while the other buffer
// loads (1-D TMA bulk copy, mbarrier completion).  Thread t of a group owns
// bucket t (word column t/2, element t%2 of the packed bf16x2 words):
//   sample  per-bucket maxima over every 4th stride-row; L = the rsel-th
//           largest of the B maxima (warp bisection over the 16-bit code);
//   mark    one packed compare per word -> 4 x 32-row hit masks per bucket;
//   Alg. 1  over the set bits in ascending position, K' (value, index) in
//           registers; candidates >= L -> 32-bit rank keys (value desc,
//           index asc; topk.cpp:30-50);
//   emit    counting sort on the value code, ranks inside a bin by
//           comparison, the first K written.
#pragma once

#include "rowthr.cuh"

namespace atkg {

constexpr int kPipeNB = 512;   // emit: bins = value code x kPipeSub index sub-bins
constexpr int kPipeSub = 2;
constexpr int kPipeRun = 64;   // emit: longest bin ranked by comparison
constexpr int kPipeRed = 64;   // reduction words per group

struct PipeArgs {
  const __nv_bfloat16* in;
  uint64_t rows;
  uint32_t n, k, rsel, cap;
  uint32_t slot_bytes;   // one row buffer (rows padded to 16 stride-rows)
  uint32_t scr_words;    // per-group scratch words
  uint32_t force_slow;
  float* out_v;
  uint32_t* out_i;
  uint32_t* status;
};

// group-wide exclusive scan of v (B threads, named barrier id); *total = sum
template <int B>
__device__ __forceinline__ uint32_t pipe_scan(uint32_t v, uint32_t* wsum, int bar, uint32_t* total) {
  const int t = threadIdx.x % B, lane = t & 31, warp = t >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(B) : "memory");
  uint32_t pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < B / 32; ++w) {
    const uint32_t s = wsum[w];
    pre += w < warp ? s : 0u;
    tot += s;
  }
  *total = tot;
  return pre + incl - v;
}

template <int KP, int B, int NG>
__global__ void __launch_bounds__(B * NG, 1) row_pipe_kernel(PipeArgs a) {
  extern __shared__ __align__(128) uint8_t pipe_smem[];
  __shared__ __align__(8) uint64_t full_bar[NG][2];
  constexpr uint32_t W = B / 2;  // words per stride-row
  const int g = threadIdx.x / B, t = threadIdx.x % B, lane = t & 31, warp = t >> 5;
  const int bar = 1 + g;
  auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(B) : "memory"); };
  const uint32_t p = t >> 1, h = t & 1;
  const uint32_t nstr = a.n / B;
  const uint32_t filled = min((uint32_t)KP, nstr);
  uint8_t* bufs = pipe_smem + (size_t)g * 2 * a.slot_bytes;
  uint32_t* scr = reinterpret_cast<uint32_t*>(pipe_smem + (size_t)NG * 2 * a.slot_bytes) + (size_t)g * a.scr_words;
  uint32_t* keys = scr;                  // cap
  uint32_t* mem = keys + a.cap;          // cap
  uint32_t* hist = mem + a.cap;          // kPipeNB + 1
  uint32_t* curs = hist + kPipeNB + 1;   // kPipeNB
  uint32_t* red = curs + kPipeNB;        // kPipeRed
  const uint32_t row_bytes = a.n * 2u;
  // this CTA's rows: blockIdx.x + G * i; group g takes i = g, g + NG, ...
  const uint64_t G = gridDim.x;
  auto row_of = [&](uint32_t q) { return (uint64_t)blockIdx.x + G * ((uint64_t)g + (uint64_t)NG * q); };
  if (t == 0) {
    ptx::mbar_init(&full_bar[g][0], 1);
    ptx::mbar_init(&full_bar[g][1], 1);
    ptx::fence_mbar_init();
  }
  gsync();
  const uint64_t pol = ptx::policy_evict_first();
  auto issue = [&](uint32_t q) {  // thread 0 of the group
    const uint64_t row = row_of(q);
    if (row >= a.rows) return;
    uint64_t* fb = &full_bar[g][q & 1];
    ptx::mbar_arrive_expect_tx(fb, row_bytes);
    ptx::bulk_g2s(bufs + (q & 1) * a.slot_bytes, a.in + row * a.n, row_bytes, fb, pol);
  };
  if (t == 0) { issue(0); issue(1); }
  const uint32_t j0 = h * kThrHalf * kThrRPW;  // first stride-row of this half
  const uint32_t j1 = min(nstr, j0 + kThrHalf * kThrRPW);
  uint32_t nan = 0;
#pragma unroll 1
  for (uint32_t q = 0; row_of(q) < a.rows; ++q) {
    const uint64_t row = row_of(q);
    ptx::mbar_wait(&full_bar[g][q & 1], (q >> 1) & 1);
    const uint8_t* rb = bufs + (q & 1) * a.slot_bytes;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(rb) + p;
    const uint16_t* row16 = reinterpret_cast<const uint16_t*>(rb);
    // ---- sample: per-bucket maxima over every 4th stride-row ---------------
    uint32_t mx = 0xff80ff80u;
    if (nstr >= 16) {
#pragma unroll 4
      for (uint32_t j = j0; j < j1; j += 4) mx = bf2_max(mx, words[j * W]);
    } else {
      for (uint32_t j = j0; j < j1; ++j) mx = bf2_max(mx, words[j * W]);
    }
    mx = bf2_max(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    keys[t] = asc_code16(h ? (mx >> 16) : (mx & 0xffffu));
    gsync();
    if (warp == 0) {  // L = rsel-th largest maximum (bisection over the code)
      uint32_t cr[B / 32];
#pragma unroll
      for (int i = 0; i < B / 32; ++i) cr[i] = keys[i * 32 + lane];
      uint32_t pre = 0;
#pragma unroll 1
      for (int bit = 15; bit >= 0; --bit) {
        const uint32_t tt = pre | (1u << bit);
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < B / 32; ++i) c += cr[i] >= tt ? 1u : 0u;
        if (__reduce_add_sync(0xffffffffu, c) >= a.rsel) pre = tt;
      }
      if (lane == 0) red[32] = pre;
    }
    gsync();
    const uint32_t pre = red[32];
    bool fast = pre > 0x007fu && pre <= 0xff80u && !a.force_slow;  // -inf < L <= +inf
    const uint32_t L = code16_bits(pre), L2 = L | (L << 16);
    const float Lf = __uint_as_float(L << 16);
    uint32_t nc = 0;
    float v[KP];
    uint32_t ip[KP];
    if (fast) {
      // ---- mark (own column half) -> this bucket's 4 x 32-row masks --------
      uint32_t m[kThrHalf];
#pragma unroll
      for (int i = 0; i < kThrHalf; ++i) {
        m[i] = 0;
        const uint32_t jc = j0 + i * kThrRPW;
        if (jc < j1) {
          const uint32_t* wp = words + jc * W;
          uint32_t a0 = 0, a1 = 0;
#pragma unroll
          for (int qq = 0; qq < kThrRPW; qq += 2) {
            a0 |= WordNet<__nv_bfloat16>::hitmask(wp[qq * W], L2) & (0x00010001u << qq);
            a1 |= WordNet<__nv_bfloat16>::hitmask(wp[(qq + 1) * W], L2) & (0x00010001u << (qq + 1));
          }
          const uint32_t rem = j1 - jc;
          m[i] = (a0 | a1) & (rem >= (uint32_t)kThrRPW ? 0xffffffffu : ((1u << rem) - 1u) * 0x00010001u);
        }
      }
      uint32_t fm[2 * kThrHalf];
#pragma unroll
      for (int i = 0; i < kThrHalf; ++i) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, m[i], 1);
        fm[i] = h ? o : m[i];
        fm[kThrHalf + i] = h ? m[i] : o;
      }
      // ---- Alg. 1 over the marks in ascending position --------------------
#pragma unroll
      for (int k2 = 0; k2 < KP; ++k2) { v[k2] = -INFINITY; ip[k2] = 0; }
#pragma unroll
      for (int c = 0; c < kThrHalf; ++c) {
        const uint32_t lo16 = h ? (fm[2 * c] >> 16) : (fm[2 * c] & 0xffffu);
        const uint32_t hi16 = h ? (fm[2 * c + 1] >> 16) : (fm[2 * c + 1] & 0xffffu);
        uint32_t bm = lo16 | (hi16 << 16);
#pragma unroll 1
        while (bm) {
          const uint32_t pos = (32 * c + __ffs(bm) - 1) * B + t;
          bm &= bm - 1;
          const float x = __uint_as_float((uint32_t)row16[pos] << 16);
          if (x != x) { nan = 1u; continue; }
          if (x >= v[KP - 1]) {
            v[KP - 1] = x;
            ip[KP - 1] = pos;
#pragma unroll
            for (int k2 = KP - 1; k2 >= 1; --k2) {
              const bool up = v[k2] > v[k2 - 1];
              const float tv = v[k2];
              const uint32_t ti = ip[k2];
              v[k2] = up ? v[k2 - 1] : tv;
              ip[k2] = up ? ip[k2 - 1] : ti;
              v[k2 - 1] = up ? tv : v[k2 - 1];
              ip[k2 - 1] = up ? ti : ip[k2 - 1];
            }
          }
        }
      }
#pragma unroll
      for (int k2 = 0; k2 < KP; ++k2) nc += v[k2] >= Lf ? 1u : 0u;
    }
    // ---- candidates -> keys (group scan for offsets); verify M >= K ------
    uint32_t M;
    const uint32_t off = pipe_scan<B>(nc, red, bar, &M);
    fast = fast && M >= a.k && M <= a.cap;  // group-uniform
    float* ov = a.out_v + row * a.k;
    uint32_t* oi = a.out_i + row * a.k;
    bool sorted = false;
    if (fast) {
#pragma unroll
      for (int k2 = 0; k2 < KP; ++k2)
        if ((uint32_t)k2 < nc) keys[off + k2] = rank_key32_bf16(__float_as_uint(v[k2]), ip[k2]);
      // ---- emit: counting sort on the value code ---------------------------
      uint32_t lo = 0xffffu, hi = 0;
      for (uint32_t qq = t; qq < M; qq += B) {
        const uint32_t c = keys[qq] >> 16;
        lo = min(lo, c);
        hi = max(hi, c);
      }
      lo = __reduce_min_sync(0xffffffffu, lo);
      hi = __reduce_max_sync(0xffffffffu, hi);
      if (lane == 0) { red[33 + warp] = lo; red[33 + B / 32 + warp] = hi; }
      for (uint32_t i = t; i <= (uint32_t)kPipeNB; i += B) hist[i] = 0;
      gsync();
      lo = 0xffffu;
      hi = 0;
#pragma unroll
      for (int w2 = 0; w2 < B / 32; ++w2) { lo = min(lo, red[33 + w2]); hi = max(hi, red[33 + B / 32 + w2]); }
      // bin = (value code - lo) * kPipeSub + index quarter: ascending bins =
      // ascending keys, a bin holds equal values from one quarter of the row
      static_assert(kPipeSub == 1 || kPipeSub == 2 || kPipeSub == 4, "index sub-bins");
      const uint32_t sub_shift = (uint32_t)max(0, 32 - __clz((int)(a.n - 1)) - (kPipeSub == 4 ? 2 : kPipeSub == 2 ? 1 : 0));
      auto bin = [&](uint32_t key) { return ((key >> 16) - lo) * kPipeSub + ((key & 0xffffu) >> sub_shift); };
      if ((hi - lo) * kPipeSub < (uint32_t)kPipeNB) {  // group-uniform
        for (uint32_t qq = t; qq < M; qq += B) atomicAdd(&hist[bin(keys[qq])], 1u);
        gsync();
        if (warp == 0) {
          constexpr int PER = kPipeNB / 32;
          uint32_t c[PER], tot = 0, mxc = 0;
#pragma unroll
          for (int i = 0; i < PER; ++i) { c[i] = hist[lane * PER + i]; tot += c[i]; mxc = max(mxc, c[i]); }
          uint32_t incl = tot;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          uint32_t ex = incl - tot;
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            hist[lane * PER + i] = ex;
            curs[lane * PER + i] = ex;
            ex += c[i];
          }
          mxc = __reduce_max_sync(0xffffffffu, mxc);
          if (lane == 0) { hist[kPipeNB] = M; red[kPipeRed - 1] = mxc; }
        }
        gsync();
        if (red[kPipeRed - 1] <= (uint32_t)kPipeRun) {  // group-uniform
          for (uint32_t qq = t; qq < M; qq += B) {
            const uint32_t key = keys[qq];
            mem[atomicAdd(&curs[bin(key)], 1u)] = key;
          }
          gsync();
          for (uint32_t qq = t; qq < M; qq += B) {
            const uint32_t key = mem[qq];
            const uint32_t bn = bin(key);
            const uint32_t b0 = hist[bn], b1 = hist[bn + 1];
            uint32_t r = b0;
            for (uint32_t o = b0; o < b1; ++o) r += mem[o] < key ? 1u : 0u;
            if (r < a.k) emit_key32(key, ov + r, oi + r);
          }
          sorted = true;
        }
      }
    } else {
      // ---- exact slow path: Alg. 1 summary of bucket t over every element ---
      M = B * filled;
      Summ<KP> sm;
      sm.clear();
      for (uint32_t j = 0; j < nstr; ++j) sm.push(bf_at(rb, j * B + t), j * B + t, nan);
      float fv[KP];
      uint32_t fi[KP];
      sm.finalize(fv, fi);
#pragma unroll
      for (int k2 = 0; k2 < KP; ++k2)
        if ((uint32_t)k2 < filled) keys[t * filled + k2] = rank_key32_bf16(__float_as_uint(fv[k2]), fi[k2]);
    }
    if (!sorted) {  // group-uniform: bitonic sort of the M keys (repeats allowed)
      uint32_t P = 2;
      while (P < M) P <<= 1;
      gsync();
      for (uint32_t qq = M + t; qq < P; qq += B) keys[qq] = ~0u;
      gsync();
      for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
          for (uint32_t qq = t; qq < P / 2; qq += B) {
            const uint32_t i = 2 * qq - (qq & (stride - 1));
            const uint32_t j = i + stride;
            const bool asc = (i & size) == 0;
            const uint32_t x = keys[i], y = keys[j];
            if ((x > y) == asc) { keys[i] = y; keys[j] = x; }
          }
          gsync();
        }
      }
      for (uint32_t qq = t; qq < a.k; qq += B) emit_key32(keys[qq], ov + qq, oi + qq);
    }
    gsync();  // row buffer and scratch free
    if (t == 0) issue(q + 2);
  }
  if (nan) atomicOr(a.status, ATKG_FLAG_NAN);
}

}  // namespace atkg
