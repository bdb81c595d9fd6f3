// common.cuh -- shared device helpers for the atkg kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "../../include/atkg.h"

namespace atkg {

constexpr uint32_t kEmptyPos = 0xffffffffu;  // unfilled summary slot / "none"

#define ATKG_HD __host__ __device__ __forceinline__

ATKG_HD float neg_inf() { return -INFINITY; }
ATKG_HD uint32_t umax32(uint32_t a, uint32_t b) { return a > b ? a : b; }
ATKG_HD uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Sortable 64-bit rank key (src/topk.cpp:30-39): high 32 bits order by value
// descending over the IEEE total order with -0.0 canonicalised to +0.0, low
// 32 bits by index ascending; ascending key order = output order.
__host__ __device__ __forceinline__ uint64_t rank_key_bits(uint32_t bits, uint32_t index) {
  if (bits == 0x80000000u) bits = 0;
  const uint32_t asc = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
  return ((uint64_t)(~asc) << 32) | index;
}
// key_value (src/topk.cpp:41-46): -0.0 comes back as +0.0
__host__ __device__ __forceinline__ uint32_t key_value_bits(uint64_t key) {
  const uint32_t asc = (uint32_t)~(key >> 32);
  return (asc & 0x80000000u) ? (asc & 0x7fffffffu) : ~asc;
}

// element loads, upcast to fp32 exactly
template <typename T>
struct Elem;
template <>
struct Elem<float> {
  __device__ __forceinline__ static float to_f32(float x) { return x; }
};
template <>
struct Elem<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
};

// V consecutive elements as one vector load (16/8/4/2 bytes)
template <typename T, int V>
struct VecLoad {
  static constexpr int kBytes = sizeof(T) * V;
  __device__ __forceinline__ static void load(const T* p, float (&out)[V]) {
    if constexpr (kBytes == 16) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
      unpack(&u.x, out);
    } else if constexpr (kBytes == 8) {
      uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
      unpack(&u.x, out);
    } else if constexpr (kBytes == 4) {
      uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(p));
      unpack(&u, out);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) out[v] = Elem<T>::to_f32(p[v]);
    }
  }
  __device__ __forceinline__ static void unpack(const uint32_t* w, float (&out)[V]) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int v = 0; v < V; ++v) out[v] = __uint_as_float(w[v]);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint32_t word = w[v / 2];
        out[v] = __uint_as_float((v & 1) ? (word & 0xffff0000u) : (word << 16));
      }
    }
  }
};

#ifdef __CUDACC__
// ascending order key of a non-NaN float, -0 == +0
__device__ __forceinline__ uint32_t st_okey(float x) {
  uint32_t u = __float_as_uint(x);
  if (u == 0x80000000u) u = 0;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float st_oval(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
constexpr uint32_t kStKeyNegInf = 0x007fffffu;  // st_okey(-inf)

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint32_t bmax_nan(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

#endif

__host__ __device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

}  // namespace atkg
