// stage2.cuh -- exact top-K of the stage-1 candidates (stage 2).
//
// Reference: select_top_k_candidates + top_k_from_keys,
// /root/reference/proj/core/src/topk.cpp:192-202, 219-236: drop candidates
// with index >= index_limit, reject NaN, sort 64-bit rank keys
// (value desc, index asc; -0.0 == +0.0) and keep the first K, rebuilding the
// value from the key (so -0.0 is emitted as +0.0).
//
// Device form: one CTA per row sorts the row's keys in shared memory with a
// bitonic network (keys are unique up to duplicate sentinels, whose order is
// irrelevant because equal keys produce identical outputs).
#pragma once

#include "common.cuh"

namespace atkg {

constexpr uint32_t kFlagFew = 2u;  // "fewer candidates than k"

// in-place ascending bitonic sort of P (power of two) keys in shared memory
__device__ __forceinline__ void block_bitonic_sort(uint64_t* s, uint32_t P) {
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const uint32_t i = 2 * t - (t & (stride - 1));
        const uint32_t j = i + stride;
        const bool asc = (i & size) == 0;
        const uint64_t a = s[i], b = s[j];
        if ((a > b) == asc) { s[i] = b; s[j] = a; }
      }
      __syncthreads();
    }
  }
}

// row r candidates: vals/idx[r*stride + c], c < count
static __global__ void stage2_bitonic_kernel(const float* __restrict__ vals, const uint32_t* __restrict__ idx,
                                      uint64_t count, uint64_t stride, uint32_t k, uint64_t index_limit,
                                      uint32_t P, float* out_v, uint32_t* out_i, uint32_t* status) {
  extern __shared__ uint64_t keys[];
  __shared__ uint32_t survivors;
  __shared__ uint32_t nan;
  const uint64_t row = blockIdx.x;
  if (threadIdx.x == 0) { survivors = 0; nan = 0; }
  __syncthreads();
  uint32_t mine = 0, bad = 0;
  for (uint32_t c = threadIdx.x; c < P; c += blockDim.x) {
    uint64_t key = ~0ull;
    if (c < count) {
      const float v = vals[row * stride + c];
      const uint32_t ix = idx[row * stride + c];
      bad |= (v != v);
      if ((uint64_t)ix < index_limit) { key = rank_key_bits(__float_as_uint(v), ix); ++mine; }
    }
    keys[c] = key;
  }
  if (mine) atomicAdd(&survivors, mine);
  if (bad) atomicOr(&nan, 1u);
  __syncthreads();
  if (nan) {
    if (threadIdx.x == 0) atomicOr(status, ATKG_FLAG_NAN);
    return;
  }
  if (survivors < k) {
    if (threadIdx.x == 0) atomicOr(status, kFlagFew);
    return;
  }
  block_bitonic_sort(keys, P);
  for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) {
    const uint64_t key = keys[t];
    out_v[row * k + t] = __uint_as_float(key_value_bits(key));
    out_i[row * k + t] = (uint32_t)key;
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


// one warp per row for count <= 32*N candidates: keys in registers (lane-major,
// element i = lane*N + r), warp bitonic sort, first k emitted
template <int N>
__global__ void __launch_bounds__(256) stage2_warp_kernel(const float* __restrict__ vals,
                                                          const uint32_t* __restrict__ idx, uint64_t rows,
                                                          uint32_t count, uint64_t stride, uint32_t k,
                                                          uint64_t index_limit, float* out_v, uint32_t* out_i,
                                                          uint32_t* status) {
  // no early exits: every lane of the warp reaches the shuffles, so they
  // compile to plain SHFL (no collective fix-up code)
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t row0 = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const bool live = row0 < rows;
  const uint64_t row = live ? row0 : rows - 1;
  const float* vr = vals + row * stride;
  const uint32_t* ir = idx + row * stride;
  uint64_t key[N];
  uint32_t mine = 0, bad = 0;
#pragma unroll
  for (int r = 0; r < N; ++r) {
    const uint32_t c = lane * N + r;
    key[r] = ~0ull;
    if (c < count) {
      const float v = vr[c];
      const uint32_t ix = ir[c];
      bad |= (v != v);
      if ((uint64_t)ix < index_limit) { key[r] = rank_key_bits(__float_as_uint(v), ix); ++mine; }
    }
  }
  const bool any_bad = __any_sync(0xffffffffu, bad);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  warp_bitonic_sort<uint64_t, N>(key, (int)lane);
  if (!live) return;
  if (any_bad || mine < k) {
    if (lane == 0) atomicOr(status, any_bad ? ATKG_FLAG_NAN : kFlagFew);
    return;
  }
#pragma unroll
  for (int r = 0; r < N; ++r) {
    const uint32_t c = lane * N + r;
    if (c < k) {
      out_v[row * k + c] = __uint_as_float(key_value_bits(key[r]));
      out_i[row * k + c] = (uint32_t)key[r];
    }
  }
}
}  // namespace atkg
