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
__global__ void stage2_bitonic_kernel(const float* __restrict__ vals, const uint32_t* __restrict__ idx,
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

}  // namespace atkg
