// rowres.cuh -- row-resident approximate top-k for short rows (the FFN
// activation config: bf16 rows of 14336, buckets of 112 elements).
//
// Buckets this short make any streaming insertion scheme branch-heavy (about
// 15 % of elements change a bucket's top-K').  Instead a CTA stages whole
// rows in shared memory with one 1-D TMA bulk copy per row and makes two
// passes over them:
//   pass 1  every thread owns one 32-bit word column (E = 4/sizeof(T)
//           adjacent buckets) and runs a branch-free min/max sorting network
//           over its stride-rows (packed bf16x2 ops for bf16) -> each
//           bucket's exact K'-th largest value v*;
//   pass 2  the same thread marks the elements >= v* in per-bucket bit
//           masks (one packed compare per word, a predicated OR per
//           element), then pushes only the marked elements, in position
//           order, through the exact summary update (summ.cuh
//           Summ::push).  By the S* lemma, Alg. 1
//           over the subsequence {x >= v*} ends in the same state as over
//           the whole bucket (/root/reference/proj/core/src/topk.cpp:80-102),
//           so finalize() yields the reference grid bit-for-bit;
//   stage 2 the row's candidate rank keys (value desc, index asc) are
//           sorted (warp register bitonic sorts; two warps each sort half
//           and a merge-path pass emits the first K) and the top K emitted.
#pragma once

#include <cuda_bf16.h>

#include <type_traits>

#include "common.cuh"
#include "emit.cuh"
#include "ptx.cuh"
#include "stage1.cuh"
#include "stage2.cuh"

namespace atkg {

// bitonic sort of P keys by the `nt` threads of one row group (t = rank in
// group); every group runs the same schedule, so __syncthreads is uniform
template <typename K>
__device__ __forceinline__ void group_bitonic_sort(K* s, uint32_t P, uint32_t t, uint32_t nt) {
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t q = t; q < P / 2; q += nt) {
        const uint32_t i = 2 * q - (q & (stride - 1));
        const uint32_t j = i + stride;
        const bool asc = (i & size) == 0;
        const K a = s[i], b = s[j];
        if ((a > b) == asc) { s[i] = b; s[j] = a; }
      }
      __syncthreads();
    }
  }
}


// bf16 candidate -> 32-bit rank key (value desc, index asc; -0.0 == +0.0)
__device__ __forceinline__ uint32_t rank_key32_bf16(uint32_t f32bits, uint32_t index) {
  uint32_t h = f32bits >> 16;
  if (h == 0x8000u) h = 0;
  const uint32_t asc = (h & 0x8000u) ? (~h & 0xffffu) : (h | 0x8000u);
  return ((~asc & 0xffffu) << 16) | index;
}
__device__ __forceinline__ float key32_value_bf16(uint32_t key) {
  const uint32_t asc = ~(key >> 16) & 0xffffu;
  const uint32_t h = (asc & 0x8000u) ? (asc & 0x7fffu) : (~asc & 0xffffu);
  return __uint_as_float(h << 16);
}


// Moves the k smallest of P unique keys to s[0..k) (unordered) and pads
// s[k..next_pow2(k)) with ~0.  MSB-first 8-bit radix select with a shared
// histogram (`scr` = 264 words per row group); every group runs the same
// schedule, so the __syncthreads are uniform.
template <typename K>
__device__ __forceinline__ void group_select_front(K* s, uint32_t P, uint32_t k, uint32_t t, uint32_t nt,
                                                   uint32_t* scr) {
  constexpr int BITS = sizeof(K) * 8;
  uint32_t* hist = scr;        // 256 bins
  uint32_t* ctl = scr + 256;   // [0] digit, [1] remaining k, [2] counter
  K prefix = 0, mask = 0;
  uint32_t krem = k;
  for (int shift = BITS - 8; shift >= 0; shift -= 8) {
    for (uint32_t q = t; q < 256; q += nt) hist[q] = 0;
    __syncthreads();
    for (uint32_t q = t; q < P; q += nt) {
      const K key = s[q];
      if ((key & mask) == prefix) atomicAdd(&hist[(uint32_t)(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (t < 32) {  // warp scan: lane owns bins [8 t, 8 t + 8)
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { c[q] = hist[t * 8 + q]; tot += c[q]; }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)t >= o) incl += y;
      }
      const uint32_t excl = incl - tot;
      if (excl < krem && krem <= incl) {
        uint32_t acc = excl;
        int d = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (d == 0 && acc + c[q] >= krem) { d = q + 1; break; }
          acc += c[q];
        }
        ctl[0] = t * 8 + (d - 1);
        ctl[1] = krem - acc;
      }
    }
    __syncthreads();
    prefix |= (K)ctl[0] << shift;
    mask |= (K)0xff << shift;
    krem = ctl[1];
    __syncthreads();
  }
  // prefix is now the k-th smallest key; gather keys <= it (exactly k)
  if (t == 0) ctl[2] = 0;
  __syncthreads();
  for (uint32_t q = t; q < P; q += nt) {
    const K key = s[q];
    if (key <= prefix) {
      const uint32_t slot = atomicAdd(&ctl[2], 1u);
      s[P + slot] = key;
    }
  }
  __syncthreads();
  uint32_t kp2 = 2;
  while (kp2 < k) kp2 <<= 1;
  for (uint32_t q = t; q < kp2; q += nt) s[q] = q < k ? s[P + q] : (K)~(K)0;
  __syncthreads();
}

template <typename T>
struct WordNet;  // packed top-KP values of the E buckets of one 32-bit word

template <>
struct WordNet<__nv_bfloat16> {
  static constexpr int E = 2;
  template <int KP>
  __device__ __forceinline__ static void init(uint32_t (&net)[KP]) {
#pragma unroll
    for (int k = 0; k < KP; ++k) net[k] = 0xff80ff80u;  // -inf, -inf
  }
  template <int KP>
  __device__ __forceinline__ static void add(uint32_t (&net)[KP], uint32_t w) {
    __nv_bfloat162 c = *reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      __nv_bfloat162 cur = *reinterpret_cast<__nv_bfloat162*>(&net[k]);
      const __nv_bfloat162 hi = __hmax2(cur, c);
      c = __hmin2(cur, c);
      net[k] = *reinterpret_cast<const uint32_t*>(&hi);
    }
  }
  __device__ __forceinline__ static float lane(uint32_t w, int e) {
    return __uint_as_float(e ? (w & 0xffff0000u) : (w << 16));
  }
  // per-half !(x < v*) (NaN included) as 0xffff / 0 halves (one HSET2)
  __device__ __forceinline__ static uint32_t hitmask(uint32_t w, uint32_t vs) {
    uint32_t r;
    asm("set.geu.u32.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(vs));
    return r;
  }
  // per-half !(x < v*) (NaN included) as two predicates from one HSETP2
  __device__ __forceinline__ static void hit(uint32_t w, uint32_t vs, bool (&h)[2]) {
    uint32_t lo, hi;
    asm("{\n\t.reg .pred p, q;\n\t"
        "setp.geu.bf16x2 p|q, %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "selp.u32 %1, 1, 0, q;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "r"(w), "r"(vs));
    h[0] = lo != 0;
    h[1] = hi != 0;
  }
};

template <>
struct WordNet<float> {
  static constexpr int E = 1;
  template <int KP>
  __device__ __forceinline__ static void init(uint32_t (&net)[KP]) {
#pragma unroll
    for (int k = 0; k < KP; ++k) net[k] = 0xff800000u;
  }
  template <int KP>
  __device__ __forceinline__ static void add(uint32_t (&net)[KP], uint32_t w) {
    float c = __uint_as_float(w);
    if (c != c) c = neg_inf();  // NaN is caught in pass 2
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const float cur = __uint_as_float(net[k]);
      net[k] = __float_as_uint(fmaxf(cur, c));
      c = fminf(cur, c);
    }
  }
  __device__ __forceinline__ static float lane(uint32_t w, int) { return __uint_as_float(w); }
  __device__ __forceinline__ static uint32_t hitmask(uint32_t w, uint32_t vs) {
    uint32_t r;
    asm("set.geu.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(w)), "f"(__uint_as_float(vs)));
    return r;
  }
  __device__ __forceinline__ static void hit(uint32_t w, uint32_t vs, bool (&h)[1]) {
    h[0] = !(__uint_as_float(w) < __uint_as_float(vs));
  }
};

// CTA = R row groups of TPR threads (TPR a multiple of 32).
// smem: R rows of n elements | R x key_stride candidate keys | R x 264 words
// of select scratch (P > 512 only)
#ifndef ATKG_RR_RANK_MIN
#define ATKG_RR_RANK_MIN 512  // rank emit for P in (ATKG_RR_RANK_MIN, 1024]
#endif
constexpr int kRowFastChunks = 4;       // closed-form pass 2 for buckets of <= 128

// first k of the merge of two ascending runs a[0..na), b[0..nb) of unique keys
// (merge path: thread t emits outputs [d0, d1))
template <typename K, typename Emit>
__device__ __forceinline__ void merge_path_emit(const K* a, uint32_t na, const K* b, uint32_t nb, uint32_t k,
                                                uint32_t t, uint32_t nt, Emit&& emit) {
  const uint32_t per = (k + nt - 1) / nt;
  const uint32_t d0 = t * per, d1 = min(k, d0 + per);
  if (d0 >= d1) return;
  // i + j = d0 with a[i-1] < b[j] and b[j-1] < a[i]
  uint32_t lo = d0 > nb ? d0 - nb : 0, hi = min(d0, na);
  while (lo < hi) {
    const uint32_t i = (lo + hi) / 2, j = d0 - i;
    if (a[i] < b[j - 1]) lo = i + 1;
    else hi = i;
  }
  uint32_t i = lo, j = d0 - lo;
  for (uint32_t d = d0; d < d1; ++d) {
    const bool take_a = j >= nb || (i < na && a[i] < b[j]);
    emit(d, take_a ? a[i++] : b[j++]);
  }
}

template <typename T, int KP>
__global__ void __launch_bounds__(256)
row_resident_kernel(const T* __restrict__ in, uint64_t rows, uint32_t n, uint32_t B, uint32_t R, uint32_t k,
                    uint32_t filled, uint32_t P, uint32_t fast, float* out_v, uint32_t* out_i, float* grid_v,
                    uint32_t* grid_i,
                    uint32_t* status) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using Net = WordNet<T>;
  constexpr int E = Net::E;
  // 32-bit keys when the value has 16 bits (bf16) and indices fit 16 bits
  constexpr bool K32 = sizeof(T) == 2;
  using Key = typename std::conditional<K32, uint32_t, uint64_t>::type;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t TPR = blockDim.x / R;
  const uint32_t g = threadIdx.x / TPR, t = threadIdx.x % TPR;
  const uint64_t row0 = (uint64_t)blockIdx.x * R;
  const uint32_t nrows = (uint32_t)umin64(R, rows - row0);
  const uint32_t row_bytes = n * sizeof(T);
  const uint32_t row_stride_b = (row_bytes + 127) & ~127u;
  const uint32_t key_stride = P > 512u ? 2 * P : P;  // + select scratch
  Key* keys = reinterpret_cast<Key*>(smem_raw + (size_t)R * row_stride_b);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(keys) + (size_t)R * key_stride * sizeof(Key));
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&bar, nrows * row_bytes);
    const uint64_t pol = ptx::policy_evict_first();
    for (uint32_t r = 0; r < nrows; ++r)
      ptx::bulk_g2s(smem_raw + r * row_stride_b, in + (row0 + r) * n, row_bytes, &bar, pol);
  }
  for (uint32_t q = threadIdx.x; q < R * key_stride; q += blockDim.x) keys[q] = (Key)~(Key)0;
  __syncthreads();
  ptx::mbar_wait(&bar, 0);

  const bool row_ok = g < nrows;
  const uint64_t row = row0 + g;
  const uint32_t* words = reinterpret_cast<const uint32_t*>(smem_raw + g * row_stride_b);
  const uint32_t W = B / E;      // words per stride-row
  const uint32_t nstr = n / B;   // stride-rows
  Key* rkeys = keys + (uint64_t)g * key_stride;
  uint32_t nan = 0;
  for (uint32_t p = t; row_ok && p < W; p += TPR) {
    // pass 1: exact K'-th largest values of the E buckets of word column p
    uint32_t net[KP];
    Net::template init<KP>(net);
#ifdef ATKG_RR_ILP2
    {  // two independent chains (even / odd stride-rows), merged at the end
      uint32_t net2[KP];
      Net::template init<KP>(net2);
      uint32_t j = 0;
      for (; j + 1 < nstr; j += 2) {
        Net::template add<KP>(net, words[j * W + p]);
        Net::template add<KP>(net2, words[(j + 1) * W + p]);
      }
      if (j < nstr) Net::template add<KP>(net, words[j * W + p]);
#pragma unroll
      for (int k = 0; k < KP; ++k) Net::template add<KP>(net, net2[k]);
    }
#else
    for (uint32_t j = 0; j < nstr; ++j) Net::template add<KP>(net, words[j * W + p]);
#endif
    const uint32_t vs = net[KP - 1];  // packed v* of the word's buckets
#ifdef ATKG_RR_NOPASS2
    {
      float ov[KP];
      uint32_t oi[KP];
#pragma unroll
      for (int e = 0; e < E; ++e) {
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) { ov[kk] = Net::lane(net[kk], e); oi[kk] = kk * B + p * E + e; }
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) {
          if (grid_v) {
            grid_v[row * KP * B + (uint64_t)kk * B + p * E + e] = ov[kk];
            grid_i[row * KP * B + (uint64_t)kk * B + p * E + e] = oi[kk];
          }
          if ((uint32_t)kk < filled) {
            if constexpr (K32) rkeys[(uint64_t)kk * B + p * E + e] = rank_key32_bf16(__float_as_uint(ov[kk]), oi[kk]);
            else rkeys[(uint64_t)kk * B + p * E + e] = rank_key_bits(__float_as_uint(ov[kk]), oi[kk]);
          }
        }
      }
      continue;
    }
#endif
    auto store = [&](uint32_t b, const float (&ov)[KP], const uint32_t (&oi)[KP]) {
#pragma unroll
      for (int kk = 0; kk < KP; ++kk) {
        if (grid_v) {
          grid_v[row * KP * B + (uint64_t)kk * B + b] = ov[kk];
          grid_i[row * KP * B + (uint64_t)kk * B + b] = oi[kk];
        }
        if ((uint32_t)kk < filled) {
          if constexpr (K32) rkeys[(uint64_t)kk * B + b] = rank_key32_bf16(__float_as_uint(ov[kk]), oi[kk]);
          else rkeys[(uint64_t)kk * B + b] = rank_key_bits(__float_as_uint(ov[kk]), oi[kk]);
        }
      }
    };
    uint32_t done = 0;  // buckets of this word finished by the closed form
    if (fast) {  // nstr <= 32 * kRowFastChunks and padded shared memory (host)
      // pass 2: mark the elements >= v* (NaN included).  Chunk c holds
      // CH = 32/E consecutive stride-rows 16c.. with bit q + e*CH for
      // bucket e (one SET + one LOP3 per word).  Rows past nstr read the
      // shared-memory padding that follows the row and are masked off.
      constexpr int CH = 32 / E;
      constexpr int NCH = 32 * kRowFastChunks / CH;
      uint32_t mk[NCH];
      auto qbits = [](int q) {
        uint32_t m = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) m |= 1u << (q + e * CH);
        return m;
      };
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint32_t jc = CH * c;
        mk[c] = 0;
        if (jc < nstr) {
          const uint32_t* wp = words + jc * W + p;
          uint32_t a0 = 0, a1 = 0;  // two chains for ILP
#pragma unroll
          for (int q = 0; q < CH; q += 2) {
            a0 |= Net::hitmask(wp[q * W], vs) & qbits(q);
            a1 |= Net::hitmask(wp[(q + 1) * W], vs) & qbits(q + 1);
          }
          const uint32_t rem = nstr - jc;
          const uint32_t valid = rem >= (uint32_t)CH ? 0xffffffffu : ((1u << rem) - 1u) * qbits(0);
          mk[c] = (a0 | a1) & valid;
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t b = p * E + e;
        const float vst = Net::lane(vs, e);
        if (!(vst > neg_inf())) continue;  // v* = -inf: sentinel rules, general path
        // this bucket's marks as 32-row masks m[k] (rows 32k..32k+31)
        uint32_t m[kRowFastChunks];
#pragma unroll
        for (int k = 0; k < kRowFastChunks; ++k) {
          if constexpr (E == 2) m[k] = __byte_perm(mk[2 * k], mk[2 * k + 1], e ? 0x7632 : 0x5410);
          else m[k] = mk[k];
        }
#ifdef ATKG_RR_NOEXTRACT
        {
          float ov[KP];
          uint32_t oi[KP];
#pragma unroll
          for (int kk = 0; kk < KP; ++kk) { ov[kk] = vst; oi[kk] = __popc(m[kk % kRowFastChunks]) + b; }
          store(b, ov, oi);
          done |= 1u << e;
          continue;
        }
#endif
        // closed form of Alg. 1 over S* = {x >= v*} (summ.cuh finalize):
        // keep every big (x > v*), the first c-1 ties (x == v*, c = K' -
        // #bigs) and X = the last tie if it comes after the last big, else
        // the c-th tie.  One pass over the marked elements, no list updates.
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < kRowFastChunks; ++k) cnt += __popc(m[k]);
        float bv[KP];
        uint32_t bp[KP], tp[KP];
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) { bv[kk] = neg_inf(); bp[kk] = kEmptyPos; tp[kk] = 0; }
        uint32_t nb = 0, nt = 0, last_big = 0, last_tie = 0;
        for (uint32_t h = 0; h < cnt; ++h) {
          // lowest marked row: first nonzero mask word
          const uint32_t w0 = m[0] ? m[0] : (m[1] ? m[1] : (m[2] ? m[2] : m[3]));
          const uint32_t k0 = m[0] ? 0u : (m[1] ? 1u : (m[2] ? 2u : 3u));
          const uint32_t j = 32 * k0 + (__ffs(w0) - 1);
          const uint32_t wc = w0 & (w0 - 1);
#pragma unroll
          for (int k = 0; k < kRowFastChunks; ++k)
            if ((uint32_t)k == k0) m[k] = wc;
          const float x = Net::lane(words[j * W + p], e);
          const uint32_t pos = j * B + b;
          if (x != x) {
            nan = 1u;
          } else if (x > vst) {
#pragma unroll
            for (int kk = 0; kk < KP - 1; ++kk)
              if ((uint32_t)kk == nb) { bv[kk] = x; bp[kk] = pos; }
            ++nb;
            last_big = pos;
          } else {
#pragma unroll
            for (int kk = 0; kk < KP; ++kk)
              if ((uint32_t)kk == nt) tp[kk] = pos;
            ++nt;
            last_tie = pos;
          }
        }
        // bigs: stable sort by value desc (empty slots are -inf and sink)
#pragma unroll
        for (int i = 1; i < KP - 1; ++i) {
#pragma unroll
          for (int kk = i; kk >= 1; --kk) {
            const bool sw = bv[kk] > bv[kk - 1];
            const float tv = bv[kk];
            const uint32_t ti = bp[kk];
            bv[kk] = sw ? bv[kk - 1] : tv;
            bp[kk] = sw ? bp[kk - 1] : ti;
            bv[kk - 1] = sw ? tv : bv[kk - 1];
            bp[kk - 1] = sw ? ti : bp[kk - 1];
          }
        }
        const uint32_t c = KP - nb;  // ties kept (>= 1)
        uint32_t tc = 0;             // the c-th tie
#pragma unroll
        for (int kk = 0; kk < KP; ++kk)
          if ((uint32_t)kk + 1 == c) tc = tp[kk];
        const uint32_t X = (nb == 0 || last_tie > last_big) ? last_tie : tc;
        float ov[KP];
        uint32_t oi[KP];
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) {
          if ((uint32_t)kk < nb) {
            ov[kk] = bv[kk];
            oi[kk] = bp[kk];
          } else {
            const uint32_t ti = kk - nb;  // tie rank
            uint32_t tpos = X;
#pragma unroll
            for (int q = 0; q < KP; ++q)
              if ((uint32_t)q == ti && ti + 1 < c) tpos = tp[q];
            ov[kk] = vst;
            oi[kk] = tpos;
          }
        }
        store(b, ov, oi);
        done |= 1u << e;
      }
    }
    // general path (long buckets, v* = -inf): exact summary update over the
    // elements >= v* in position order
#pragma unroll 1
    for (int e = 0; e < E; ++e) {
      if (done >> e & 1u) continue;
      const uint32_t b = p * E + e;
      const float vst = Net::lane(vs, e);
      Summ<KP> sm;
      sm.clear();
      for (uint32_t j = 0; j < nstr; ++j) {
        const float x = Net::lane(words[j * W + p], e);
        if (!(x < vst)) sm.push(x, j * B + b, nan);
      }
      float ov[KP];
      uint32_t oi[KP];
      sm.finalize(ov, oi);
      store(b, ov, oi);
    }
  }
  if (nan) atomicOr(status, ATKG_FLAG_NAN);
  if (!out_v) return;  // stage-1 only (uniform across the CTA)
  __syncthreads();
  uint32_t nsort = P;
  if constexpr (K32) {
    // large candidate sets, one row per CTA: counting-sort rank emit over the
    // value code, only the bins before rank k ranked (the dead row buffer
    // holds the scratch); rows with -inf candidates (repeatable sentinel
    // keys) or crowded bins take the radix-select path below
    if (P > (uint32_t)ATKG_RR_RANK_MIN && P <= 1024u && R == 1 && filled * B * 4 <= row_bytes) {  // measured: slower at 4096
      __shared__ uint32_t rr_sent;
      if (threadIdx.x == 0) rr_sent = 0;
      __syncthreads();
      const uint32_t M = filled * B;
      uint32_t sflag = 0;
      for (uint32_t q = threadIdx.x; q < M; q += blockDim.x)
        sflag |= key32_value_bf16(rkeys[q]) == neg_inf() ? 1u : 0u;
      if (sflag) atomicOr(&rr_sent, 1u);
      __syncthreads();
      if (!rr_sent && emit_ranked<uint32_t>(rkeys, reinterpret_cast<uint32_t*>(smem_raw), M, k,
                                            [&](uint32_t r, uint32_t key) {
                                              out_v[row * k + r] = key32_value_bf16(key);
                                              out_i[row * k + r] = key & 0xffffu;
                                            }))
        return;
      __syncthreads();
    }
  }
  if (P > 512u) {
    // large candidate sets: radix-select the k smallest (unique) keys into
    // the front, then sort only those
    group_select_front<Key>(rkeys, P, k, t, TPR, scratch + (uint64_t)g * 264);
    nsort = 2;
    while (nsort < k) nsort <<= 1;
  }
  auto emit = [&](uint32_t q, Key key) {
    if constexpr (K32) {
      out_v[row * k + q] = key32_value_bf16(key);
      out_i[row * k + q] = key & 0xffffu;
    } else {
      out_v[row * k + q] = __uint_as_float(key_value_bits(key));
      out_i[row * k + q] = (uint32_t)key;
    }
  };
  if (nsort == 512u && TPR >= 64) {
    // two warps each sort 256 keys in registers; merge path emits the first k
    if (row_ok && t < 64) {
      Key kk[8];
      Key* half = rkeys + (t / 32) * 256;
      const uint32_t l = t % 32;
#pragma unroll
      for (int r = 0; r < 8; ++r) kk[r] = half[l * 8 + r];
      warp_bitonic_sort<Key, 8>(kk, (int)l);
#pragma unroll
      for (int r = 0; r < 8; ++r) half[l * 8 + r] = kk[r];
    }
    __syncthreads();
    if (!row_ok || (*status & ATKG_FLAG_NAN)) return;
    merge_path_emit<Key>(rkeys, 256, rkeys + 256, 256, k, t, TPR, emit);
    return;
  }
  if (nsort == 512u || nsort == 256u) {
    // one warp of the row group sorts in registers
    if (row_ok && t < 32) {
      if (nsort == 512u) {
        Key kk[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) kk[r] = rkeys[t * 16 + r];
        warp_bitonic_sort<Key, 16>(kk, (int)t);
#pragma unroll
        for (int r = 0; r < 16; ++r) rkeys[t * 16 + r] = kk[r];
      } else {
        Key kk[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) kk[r] = rkeys[t * 8 + r];
        warp_bitonic_sort<Key, 8>(kk, (int)t);
#pragma unroll
        for (int r = 0; r < 8; ++r) rkeys[t * 8 + r] = kk[r];
      }
    }
    __syncthreads();
  } else {
    group_bitonic_sort<Key>(rkeys, nsort, t, TPR);
  }
  if (!row_ok || (*status & ATKG_FLAG_NAN)) return;
  for (uint32_t q = t; q < k; q += TPR) emit(q, rkeys[q]);
}

}  // namespace atkg
