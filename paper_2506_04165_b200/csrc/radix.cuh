// radix.cuh -- exact radix-select top-k (recall measurement, and stage 2
// for candidate sets too large for one CTA's shared memory).
//
// Reference: exact_top_k (/root/reference/proj/core/src/topk.cpp:206-217)
// fully sorts 64-bit rank keys (value desc, index asc, -0.0 == +0.0) and keeps
// the first k.  Device form per row, no host round trips:
//   passes 0-3  8-bit MSB-first histograms of the 32-bit value order key u
//               (smaller u = larger value) among elements matching the
//               prefix so far -> threshold value u* and how many of the
//               elements equal to u* are still needed;
//   passes 4-7  only when more elements equal u* than needed: the same on
//               the index bits among elements with u == u* -> index
//               threshold (indices are unique in a dense row);
//   gather      keys strictly below the (u*, i*) threshold, then the
//               threshold key itself up to k (duplicate candidate keys are
//               interchangeable);
//   sort        bitonic sort of the k selected keys in shared memory.
#pragma once

#include "common.cuh"
#include "stage2.cuh"

namespace atkg {

struct RowSel {
  uint32_t prefix, mask;    // value-key bits decided so far
  uint32_t krem;            // still needed among elements matching the prefix
  uint32_t iprefix, imask;  // index bits decided so far (tie passes)
  uint32_t need_index;      // ties at u* exceed krem
  uint32_t thr_u, thr_i;    // final threshold key
  uint32_t taken;           // gather counter
  uint32_t pad[3];
};

__device__ __forceinline__ uint32_t order_key_u(uint32_t bits) {
  // high 32 bits of rank_key: ~asc(bits), -0.0 canonicalised
  if (bits == 0x80000000u) bits = 0;
  const uint32_t asc = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
  return ~asc;
}

template <typename T>
struct DenseSrc {
  const T* base;
  uint64_t n;        // row length
  __device__ __forceinline__ uint64_t count() const { return n; }
  // returns false when the element is filtered out
  __device__ __forceinline__ bool get(uint64_t row, uint64_t c, uint32_t& u, uint32_t& ix, uint32_t& nan) const {
    const float x = Elem<T>::to_f32(base[row * n + c]);
    nan |= (x != x) ? 1u : 0u;
    u = order_key_u(__float_as_uint(x));
    ix = (uint32_t)c;
    return true;
  }
};

struct CandSrc {
  const float* vals;
  const uint32_t* idx;
  uint64_t cnt, stride, limit;
  __device__ __forceinline__ uint64_t count() const { return cnt; }
  __device__ __forceinline__ bool get(uint64_t row, uint64_t c, uint32_t& u, uint32_t& ix, uint32_t& nan) const {
    const float x = vals[row * stride + c];
    nan |= (x != x) ? 1u : 0u;
    ix = idx[row * stride + c];
    u = order_key_u(__float_as_uint(x));
    return (uint64_t)ix < limit;
  }
};

__global__ void radix_init_kernel(RowSel* sel, uint32_t* hist, uint64_t rows, uint32_t k) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < rows) {
    RowSel s = {};
    s.krem = k;
    sel[t] = s;
  }
  for (uint64_t i = t; i < rows * 256; i += (uint64_t)gridDim.x * blockDim.x) hist[i] = 0;
}

template <class Src>
__global__ void radix_hist_kernel(Src src, int pass, RowSel* sel, uint32_t* hist, uint32_t* status) {
  __shared__ uint32_t h[256];
  const uint64_t row = blockIdx.y;
  const RowSel s = sel[row];
  if (pass >= 4 && !s.need_index) return;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t n = src.count();
  const uint64_t per = ceil_div(n, gridDim.x);
  const uint64_t c0 = blockIdx.x * per, c1 = min(n, c0 + per);
  uint32_t nan = 0;
  const int shift = 24 - 8 * (pass & 3);
  for (uint64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    uint32_t u, ix;
    if (!src.get(row, c, u, ix, nan)) continue;
    if (pass < 4) {
      if ((u & s.mask) == s.prefix) atomicAdd(&h[(u >> shift) & 255u], 1u);
    } else {
      if (u == s.thr_u && (ix & s.imask) == s.iprefix) atomicAdd(&h[(ix >> shift) & 255u], 1u);
    }
  }
  if (nan && pass == 0) atomicOr(status, ATKG_FLAG_NAN);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[row * 256 + i], h[i]);
}

// one warp per row: scan the 256-bin histogram, pick the digit, reset bins
__global__ void radix_select_kernel(int pass, RowSel* sel, uint32_t* hist, uint64_t rows, uint32_t* status) {
  const uint64_t row = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  RowSel s = sel[row];
  if (pass >= 4 && !s.need_index) return;
  uint32_t* h = hist + row * 256;
  // lane owns bins [8 lane, 8 lane + 8)
  uint32_t c[8], tot = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) { c[q] = h[lane * 8 + q]; tot += c[q]; h[lane * 8 + q] = 0; }
  uint32_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t excl = incl - tot;
  const uint32_t grand = __shfl_sync(0xffffffffu, incl, 31);
  const int shift = 24 - 8 * (pass & 3);
  if (pass == 0 && grand < s.krem) {  // fewer elements than k
    if (lane == 0) atomicOr(status, kFlagFew);
    return;
  }
  // the lane whose range contains the krem-th element
  const bool mine = excl < s.krem && s.krem <= incl;
  const unsigned who = __ballot_sync(0xffffffffu, mine);
  if (!mine) return;
  (void)who;
  uint32_t before = excl;
  int d = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (before + c[q] >= s.krem) { d = lane * 8 + q; break; }
    before += c[q];
  }
  uint32_t bin = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) if (lane * 8 + q == d) bin = c[q];
  s.krem -= before;
  if (pass < 4) {
    s.prefix |= (uint32_t)d << shift;
    s.mask |= 0xffu << shift;
    if (pass == 3) {
      s.thr_u = s.prefix;
      s.need_index = bin > s.krem ? 1u : 0u;
      s.thr_i = 0xffffffffu;
    }
  } else {
    s.iprefix |= (uint32_t)d << shift;
    s.imask |= 0xffu << shift;
    if (pass == 7) s.thr_i = s.iprefix;
  }
  sel[row] = s;
}

template <class Src>
__global__ void radix_gather_kernel(Src src, RowSel* sel, uint64_t* keys, uint32_t k, uint64_t kstride) {
  const uint64_t row = blockIdx.y;
  const uint32_t tu = sel[row].thr_u, ti = sel[row].thr_i;
  const uint64_t n = src.count();
  const uint64_t per = ceil_div(n, gridDim.x);
  const uint64_t c0 = blockIdx.x * per, c1 = min(n, c0 + per);
  uint32_t nan = 0;
  for (uint64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    uint32_t u, ix;
    if (!src.get(row, c, u, ix, nan)) continue;
    if (u < tu || (u == tu && ix <= ti)) {
      const uint32_t slot = atomicAdd(&sel[row].taken, 1u);
      if (slot < k) keys[row * kstride + slot] = ((uint64_t)u << 32) | ix;
    }
  }
}

__global__ void sort_emit_kernel(const uint64_t* keys, uint32_t k, uint32_t P, float* out_v, uint32_t* out_i,
                                 const uint32_t* status) {
  extern __shared__ uint64_t s[];
  const uint64_t row = blockIdx.x;
  if (*status) return;
  for (uint32_t c = threadIdx.x; c < P; c += blockDim.x) s[c] = c < k ? keys[row * k + c] : ~0ull;
  __syncthreads();
  block_bitonic_sort(s, P);
  for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) {
    out_v[row * k + t] = __uint_as_float(key_value_bits(s[t]));
    out_i[row * k + t] = (uint32_t)s[t];
  }
}

// ---- k above one CTA's shared memory (k > 16384): a bitonic network over
// the row's P = pow2 >= k keys in global memory, [rows][P] padded with ~0.
// Blocks of kSortBlock keys are sorted in shared memory (alternating
// direction, as the network has it after every size <= kSortBlock); each
// larger size then takes global compare-exchange steps down to stride
// kSortBlock and one shared-memory pass for the smaller strides.
constexpr uint32_t kSortBlock = 16384;

__global__ void big_sort_block_kernel(uint64_t* keys, uint64_t P, uint32_t k) {
  extern __shared__ uint64_t sb[];
  const uint64_t row = blockIdx.y, base = (uint64_t)blockIdx.x * kSortBlock;
  uint64_t* g = keys + row * P + base;
  for (uint32_t c = threadIdx.x; c < kSortBlock; c += blockDim.x) sb[c] = base + c < k ? g[c] : ~0ull;
  __syncthreads();
  const bool desc = (blockIdx.x & 1u) != 0;
  for (uint32_t size = 2; size <= kSortBlock; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < kSortBlock / 2; t += blockDim.x) {
        const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
        const bool asc = ((i & size) == 0) != (desc && size == kSortBlock);
        const uint64_t a = sb[i], b = sb[j];
        if ((a > b) == asc) { sb[i] = b; sb[j] = a; }
      }
      __syncthreads();
    }
  }
  for (uint32_t c = threadIdx.x; c < kSortBlock; c += blockDim.x) g[c] = sb[c];
}

__global__ void big_sort_global_step(uint64_t* keys, uint64_t P, uint64_t size, uint64_t stride) {
  const uint64_t row = blockIdx.y;
  uint64_t* g = keys + row * P;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < P / 2; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = 2 * t - (t & (stride - 1)), j = i + stride;
    const bool asc = (i & size) == 0;
    const uint64_t a = g[i], b = g[j];
    if ((a > b) == asc) { g[i] = b; g[j] = a; }
  }
}

__global__ void big_sort_block_merge(uint64_t* keys, uint64_t P, uint64_t size) {
  extern __shared__ uint64_t sb[];
  const uint64_t row = blockIdx.y, base = (uint64_t)blockIdx.x * kSortBlock;
  uint64_t* g = keys + row * P + base;
  for (uint32_t c = threadIdx.x; c < kSortBlock; c += blockDim.x) sb[c] = g[c];
  __syncthreads();
  const bool asc = (base & size) == 0;
  for (uint32_t stride = kSortBlock >> 1; stride > 0; stride >>= 1) {
    for (uint32_t t = threadIdx.x; t < kSortBlock / 2; t += blockDim.x) {
      const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
      const uint64_t a = sb[i], b = sb[j];
      if ((a > b) == asc) { sb[i] = b; sb[j] = a; }
    }
    __syncthreads();
  }
  for (uint32_t c = threadIdx.x; c < kSortBlock; c += blockDim.x) g[c] = sb[c];
}

__global__ void big_sort_emit(const uint64_t* keys, uint64_t P, uint32_t k, uint64_t rows, float* out_v,
                              uint32_t* out_i, const uint32_t* status) {
  if (*status) return;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * k;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = t / k, c = t - row * k;
    const uint64_t key = keys[row * P + c];
    out_v[t] = __uint_as_float(key_value_bits(key));
    out_i[t] = (uint32_t)key;
  }
}

}  // namespace atkg
