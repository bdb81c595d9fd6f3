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
//   pass 2  the same thread pushes only elements >= v* through the exact
//           summary update (stage1.cuh Summ::push).  By the S* lemma, Alg. 1
//           over the subsequence {x >= v*} ends in the same state as over
//           the whole bucket (/root/reference/proj/core/src/topk.cpp:80-102),
//           so finalize() yields the reference grid bit-for-bit;
//   stage 2 the row's candidate rank keys (value desc, index asc) are
//           bitonic-sorted in shared memory and the top K emitted.
#pragma once

#include <cuda_bf16.h>

#include <type_traits>

#include "common.cuh"
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


// ---------------------------------------------------------------------------
// single-warp register bitonic sort, ascending, N keys per lane in
// lane-major order (element i = lane * N + r); strides < N stay in
// registers, larger strides exchange whole registers across lanes.
// ---------------------------------------------------------------------------
template <typename K>
__device__ __forceinline__ K shfl_key(K v, int m) {
  if constexpr (sizeof(K) == 8) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
    return ((uint64_t)hi << 32) | lo;
  } else {
    return __shfl_xor_sync(0xffffffffu, v, m);
  }
}

template <typename K, int N>
__device__ __forceinline__ void warp_bitonic_sort(K (&k)[N], int lane) {
  constexpr int TOT = 32 * N;
#pragma unroll
  for (int size = 2; size <= TOT; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= N) {
        const int m = stride / N;  // partner lane distance
        const bool low = (lane & m) == 0;
#pragma unroll
        for (int r = 0; r < N; ++r) {
          const int i = lane * N + r;
          const bool asc = (i & size) == 0;
          const K o = shfl_key(k[r], m);
          const K mn = k[r] < o ? k[r] : o, mx = k[r] < o ? o : k[r];
          k[r] = (low == asc) ? mn : mx;
        }
      } else {
#pragma unroll
        for (int r = 0; r < N; ++r) {
          if ((r & stride) == 0) {
            const int i = lane * N + r;
            const bool asc = (i & size) == 0;
            const K a = k[r], b = k[r + stride];
            const bool sw = (a > b) == asc;
            k[r] = sw ? b : a;
            k[r + stride] = sw ? a : b;
          }
        }
      }
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
};

// CTA = R row groups of TPR threads (TPR a multiple of 32).
// smem: R rows of n elements | R x P candidate keys | R x E x LOGC x TPR
// pass-2 position logs.
constexpr int kRowLog = 8;  // positions logged per (thread, bucket) in pass 2

template <typename T, int KP, int WN>
__global__ void __launch_bounds__(256)
row_resident_kernel(const T* __restrict__ in, uint64_t rows, uint32_t n, uint32_t B, uint32_t R, uint32_t k,
                    uint32_t filled, uint32_t P, float* out_v, uint32_t* out_i, float* grid_v, uint32_t* grid_i,
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
  Key* keys = reinterpret_cast<Key*>(smem_raw + (size_t)R * row_stride_b);
  uint32_t* logs = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(keys) + (size_t)R * P * sizeof(Key));
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&bar, nrows * row_bytes);
    const uint64_t pol = ptx::policy_evict_first();
    for (uint32_t r = 0; r < nrows; ++r)
      ptx::bulk_g2s(smem_raw + r * row_stride_b, in + (row0 + r) * n, row_bytes, &bar, pol);
  }
  for (uint32_t q = threadIdx.x; q < R * P; q += blockDim.x) keys[q] = (Key)~(Key)0;
  __syncthreads();
  ptx::mbar_wait(&bar, 0);

  const bool row_ok = g < nrows;
  const uint64_t row = row0 + g;
  const uint32_t* words = reinterpret_cast<const uint32_t*>(smem_raw + g * row_stride_b);
  const uint32_t W = B / E;      // words per stride-row
  const uint32_t nstr = n / B;   // stride-rows
  Key* rkeys = keys + (uint64_t)g * P;
  uint32_t* mylog = logs + (uint64_t)g * E * kRowLog * TPR + t;  // [e][q][TPR]
  uint32_t nan = 0;
  for (uint32_t p = t; row_ok && p < W; p += TPR) {
    // pass 1: exact K'-th largest values of the E buckets of word column p
    uint32_t net[KP];
    Net::template init<KP>(net);
    for (uint32_t j = 0; j < nstr; ++j) Net::template add<KP>(net, words[j * W + p]);
    float vstar[E];
#pragma unroll
    for (int e = 0; e < E; ++e) vstar[e] = Net::lane(net[KP - 1], e);
    // pass 2a: log the stride-rows of the elements >= v* (branch-free)
    uint32_t cnt[E];
#pragma unroll
    for (int e = 0; e < E; ++e) cnt[e] = 0;
    for (uint32_t j = 0; j < nstr; ++j) {
      const uint32_t w = words[j * W + p];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float x = Net::lane(w, e);
        const bool h = !(x < vstar[e]);
        if (h && cnt[e] < (uint32_t)kRowLog) mylog[(e * kRowLog + cnt[e]) * TPR] = j;
        cnt[e] += h ? 1u : 0u;
      }
    }
    // pass 2b: exact summaries of the logged elements (S* = {x >= v*});
    // a bucket with more than kRowLog such elements (heavy ties) replays
    // its whole stride-row sequence instead
#pragma unroll
    for (int e = 0; e < E; ++e) {
      Summ<KP> s;
      s.clear();
      const uint32_t b = p * E + e;
      if (cnt[e] <= (uint32_t)kRowLog) {
        for (uint32_t q = 0; q < cnt[e]; ++q) {
          const uint32_t j = mylog[(e * kRowLog + q) * TPR];
          s.push(Net::lane(words[j * W + p], e), j * B + b, nan);
        }
      } else {
        for (uint32_t j = 0; j < nstr; ++j) {
          const float x = Net::lane(words[j * W + p], e);
          if (!(x < vstar[e])) s.push(x, j * B + b, nan);
        }
      }
      float ov[KP];
      uint32_t oi[KP];
      s.finalize(ov, oi);
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
    }
  }
  if (nan) atomicOr(status, ATKG_FLAG_NAN);
  if (!out_v) return;  // stage-1 only (uniform across the CTA)
  __syncthreads();
  if (WN > 0 && P == 32u * WN) {
    // one warp of the row group sorts the row's P keys in registers
    if (row_ok && t < 32) {
      Key kk[WN > 0 ? WN : 1];
#pragma unroll
      for (int r = 0; r < WN; ++r) kk[r] = rkeys[t * WN + r];
      warp_bitonic_sort<Key, (WN > 0 ? WN : 1)>(kk, (int)t);
#pragma unroll
      for (int r = 0; r < WN; ++r) rkeys[t * WN + r] = kk[r];
    }
    __syncthreads();
  } else {
    group_bitonic_sort<Key>(rkeys, P, t, TPR);
  }
  if (!row_ok || (*status & ATKG_FLAG_NAN)) return;
  for (uint32_t q = t; q < k; q += TPR) {
    if constexpr (K32) {
      out_v[row * k + q] = key32_value_bf16(rkeys[q]);
      out_i[row * k + q] = rkeys[q] & 0xffffu;
    } else {
      out_v[row * k + q] = __uint_as_float(key_value_bits(rkeys[q]));
      out_i[row * k + q] = (uint32_t)rkeys[q];
    }
  }
}

}  // namespace atkg
