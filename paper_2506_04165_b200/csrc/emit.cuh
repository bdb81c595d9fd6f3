// emit.cuh -- the first k (ascending) of M unique sort keys without a full
// sort: bins on the key's high half (ascending with the key), a counting sort
// into `mem`, ranks inside a bin by comparison (rank keys: value desc, index
// asc, /root/reference/proj/core/src/topk.cpp:30-50).  Block-wide (every
// thread of the CTA calls it); returns false (nothing written) when a bin is
// too crowded -- the caller sorts instead.
#pragma once

#include <stdint.h>

namespace atkg {

template <typename K, typename Emit>
__device__ __forceinline__ bool emit_ranked(const K* keys, K* mem, uint32_t M, uint32_t k, Emit&& emit) {
  constexpr uint32_t NB = 256, RUN = 48;
  constexpr int HB = sizeof(K) * 4;  // bits in the high half
  __shared__ uint32_t er_lo, er_hi, er_hist[NB + 1], er_curs[NB], er_max, er_lim;
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  if (t == 0) { er_lo = 0xffffffffu; er_hi = 0; er_max = 0; }
  for (uint32_t b = t; b <= NB; b += nt) er_hist[b] = 0;
  __syncthreads();
  auto high = [](K key) { return (uint32_t)(key >> HB); };
  uint32_t lo = 0xffffffffu, hi = 0;
  for (uint32_t q = t; q < M; q += nt) {
    const uint32_t h = high(keys[q]);
    lo = min(lo, h);
    hi = max(hi, h);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((t & 31) == 0) { atomicMin(&er_lo, lo); atomicMax(&er_hi, hi); }
  __syncthreads();
  lo = er_lo;
  const uint32_t span = er_hi - lo;
  const uint32_t shift = span < NB ? 0u : (uint32_t)(32 - __clz((int)(span >> 8)));  // span >> shift < NB
  auto bin = [&](K key) { return (high(key) - lo) >> shift; };
  for (uint32_t q = t; q < M; q += nt) atomicAdd(&er_hist[bin(keys[q])], 1u);
  __syncthreads();
  if (t < 32) {  // exclusive scan of NB bins, NB/32 per lane
    uint32_t c[NB / 32], tot = 0, mx = 0;
#pragma unroll
    for (int i = 0; i < (int)(NB / 32); ++i) { c[i] = er_hist[t * (NB / 32) + i]; tot += c[i]; }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)t >= o) incl += y;
    }
    uint32_t ex = incl - tot;
#pragma unroll
    for (int i = 0; i < (int)(NB / 32); ++i) {
      er_hist[t * (NB / 32) + i] = ex;
      er_curs[t * (NB / 32) + i] = ex;
      if (ex < k) mx = max(mx, c[i]);  // crowded bins past rank k do not matter
      ex += c[i];
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    // er_lim = the first bin start >= k (the bins before it hold ranks < k)
    uint32_t lim = M, st = incl - tot;
#pragma unroll
    for (int i = 0; i < (int)(NB / 32); ++i) {
      if (st >= k) lim = min(lim, st);
      st += c[i];
    }
    lim = __reduce_min_sync(0xffffffffu, lim);
    if (t == 0) { er_hist[NB] = M; er_max = mx; er_lim = lim; }
  }
  __syncthreads();
  if (er_max > RUN) return false;  // uniform
  // only bins that start before rank k can hold output keys; they fill
  // mem[0, er_lim)
  for (uint32_t q = t; q < M; q += nt) {
    const K key = keys[q];
    const uint32_t b = bin(key);
    if (er_hist[b] < k) mem[atomicAdd(&er_curs[b], 1u)] = key;
  }
  __syncthreads();
  const uint32_t lim = er_lim;
  for (uint32_t q = t; q < lim; q += nt) {
    const K key = mem[q];
    const uint32_t b = bin(key);
    const uint32_t b0 = er_hist[b], b1 = er_hist[b + 1];
    uint32_t r = b0;
    for (uint32_t o = b0; o < b1; ++o) r += mem[o] < key ? 1u : 0u;
    if (r < k) emit(r, key);
  }
  return true;
}

}  // namespace atkg
