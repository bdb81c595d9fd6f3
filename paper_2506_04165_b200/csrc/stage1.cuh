// stage1.cuh -- exact stage 1 of the two-stage approximate top-k on sm_100a.
//
// Reference semantics (Alg. 1, /root/reference/proj/core/src/topk.cpp:80-102,
// PAPER.md:307-323): bucket b = i mod B keeps K' slots; an incoming x
// replaces the minimum slot if x >= min (a LATER equal element wins), then
// bubbles forward while x > slot[k-1] (never past an equal one).
//
// The reference runs each bucket strictly sequentially.  On a B200 a row is
// instead split into segments processed in parallel, and the per-segment
// results are merged EXACTLY.  The device state of a bucket over a stretch of
// its stream is a *summary*:
//   list[0..K')  the segment's top-K' elements in rank order
//                (value desc, position asc), empty slots {-inf, kEmptyPos};
//   lt, ltv      when the list is full: the LAST position (and raw bits) of
//                any element equal to list[K'-1].value (the K'-th value).
// Summaries merge associatively (merge_into below), and the final Alg. 1
// state follows in closed form from the whole-bucket summary (finalize):
//   v* = K'-th value, big = entries > v* (all kept, rank order), ties
//   e_1..e_c = entries == v* (first c by position); Alg. 1 keeps
//   big ++ e_1..e_{c-1} ++ X with X = (last element == v*) if it comes after
//   the last big element, else e_c.  With v* == -inf the K' initial
//   sentinels {-inf, 0} of the reference are the first tie elements.
// This reproduces the reference grid bit-for-bit (tests/test_gpu_parity.py
// checks duplicate-heavy, +-0, +-inf and tiny-bucket streams against the
// reference library).
#pragma once

#include "common.cuh"
#include "ptx.cuh"

namespace atkg {

// ---------------------------------------------------------------------------
// per-bucket summary, fully register resident (all indices compile-time)
// ---------------------------------------------------------------------------
template <int KP>
struct Summ {
  float v[KP];
  uint32_t p[KP];
  uint32_t lt;   // valid when full
  float ltv;

  ATKG_HD void clear() {
#pragma unroll
    for (int k = 0; k < KP; ++k) { v[k] = neg_inf(); p[k] = kEmptyPos; }
    lt = kEmptyPos;
    ltv = neg_inf();
  }
  ATKG_HD bool full() const { return p[KP - 1] != kEmptyPos; }

  // prologue insert of the t-th element of a segment (t < KP; the caller's
  // loop over t is unrolled so every index below is compile-time)
  ATKG_HD void fill(int t, float x, uint32_t i) {
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (k == t) { v[k] = x; p[k] = i; }
#pragma unroll
    for (int k = KP - 1; k >= 1; --k) {
      if (k <= t && x > v[k - 1]) {
        const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
        const uint32_t tp = p[k]; p[k] = p[k - 1]; p[k - 1] = tp;
      }
    }
    if (t == KP - 1) { lt = p[KP - 1]; ltv = v[KP - 1]; }
  }

  // main-loop update of a FULL list with x at position i (> every position
  // seen).  Caller has established !(x < v[KP-1]) (NaN included).
  ATKG_HD void slow(float x, uint32_t i, uint32_t& nan) {
    if (x != x) { nan = 1u; return; }
    const float old = v[KP - 1];
    if (x == old) { lt = i; ltv = x; return; }
    v[KP - 1] = x;
    p[KP - 1] = i;
#pragma unroll
    for (int k = KP - 1; k >= 1; --k) {
      if (x > v[k - 1]) {
        const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
        const uint32_t tp = p[k]; p[k] = p[k - 1]; p[k - 1] = tp;
      }
    }
    if (v[KP - 1] != old) { lt = p[KP - 1]; ltv = v[KP - 1]; }
  }

  // streaming update with one element at position i (> every position seen);
  // works on partially filled lists (the accumulator's ragged edges)
  ATKG_HD void push(float x, uint32_t i, uint32_t& nan) {
    if (x != x) { nan = 1u; return; }
    if (full()) {
      if (!(x < v[KP - 1])) slow(x, i, nan);
      return;
    }
    int c = 0;
#pragma unroll
    for (int k = 0; k < KP; ++k) c += (p[k] != kEmptyPos) ? 1 : 0;
    fill(c, x, i);
  }

  // max position among entries equal to `val` (entries sorted so the last
  // equal one has the max position); kEmptyPos if none
  ATKG_HD void last_eq(float val, uint32_t& pos, float& bits) const {
    pos = kEmptyPos;
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (p[k] != kEmptyPos && v[k] == val) { pos = p[k]; bits = v[k]; }
  }

  // this = merge(this [earlier positions], o [later positions])
  ATKG_HD void merge_later(const Summ& o) {
    const bool a_full = full();
    const float a_min = v[KP - 1];
    const uint32_t a_lt = lt;
    const float a_ltv = ltv;
    Summ a = *this;  // pre-merge copy for the tie bookkeeping
    // insert o's entries (rank-sorted) one by one; rank: value desc, pos asc,
    // empty last.  o's positions all exceed ours.
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const float x = o.v[j];
      const uint32_t xp = o.p[j];
      if (xp == kEmptyPos) continue;
      // x enters iff it ranks before the current last slot
      const bool enter = (p[KP - 1] == kEmptyPos) || (x > v[KP - 1]);
      if (!enter) continue;
      v[KP - 1] = x;
      p[KP - 1] = xp;
#pragma unroll
      for (int k = KP - 1; k >= 1; --k) {
        const bool up = (p[k - 1] == kEmptyPos) || (x > v[k - 1]);
        if (up) {
          const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
          const uint32_t tp = p[k]; p[k] = p[k - 1]; p[k - 1] = tp;
        }
      }
    }
    if (!full()) { lt = kEmptyPos; ltv = neg_inf(); return; }
    const float c_min = v[KP - 1];
    uint32_t pos; float bits;
    // later segment first: any equal element there is after all of ours
    if (o.full() && o.v[KP - 1] == c_min) { pos = o.lt; bits = o.ltv; }
    else o.last_eq(c_min, pos, bits);
    if (pos == kEmptyPos) {
      if (a_full && a_min == c_min) { pos = a_lt; bits = a_ltv; }
      else a.last_eq(c_min, pos, bits);
    }
    lt = pos;
    ltv = bits;
  }

  // whole-bucket summary -> reference Alg. 1 state (value bits, index)
  ATKG_HD void finalize(float (&ov)[KP], uint32_t (&oi)[KP]) const {
    const bool f = full();
    const float vmin = v[KP - 1];
    if (f && vmin != neg_inf()) {
      uint32_t L = kEmptyPos;  // max position of entries > v*
      bool anybig = false;
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        ov[k] = v[k];
        oi[k] = p[k];
        if (v[k] > vmin) { L = anybig ? umax32(L, p[k]) : p[k]; anybig = true; }
      }
      if (!anybig || lt > L) { ov[KP - 1] = ltv; oi[KP - 1] = lt; }
      return;
    }
    // v* == -inf: the reference's K' sentinels {-inf, 0} are tie elements
    // that precede the stream
    uint32_t L = 0;
    bool anybig = false;
    uint32_t T = kEmptyPos;  // last real element equal to -inf
    if (f) T = lt;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (p[k] != kEmptyPos && v[k] > neg_inf()) {
        L = anybig ? umax32(L, p[k]) : p[k];
        anybig = true;
      } else if (!f && p[k] != kEmptyPos) {
        T = p[k];
      }
    }
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const bool big = p[k] != kEmptyPos && v[k] > neg_inf();
      ov[k] = big ? v[k] : neg_inf();
      oi[k] = big ? p[k] : 0u;
    }
    if (T != kEmptyPos && (!anybig || T > L)) { ov[KP - 1] = neg_inf(); oi[KP - 1] = T; }
  }
};

// summary <-> memory, layout per summary block: v[KP][B], p[KP][B], lt[B], ltv[B]
template <int KP>
__device__ __forceinline__ void store_summ(uint32_t* blk, uint64_t B, uint64_t b, const Summ<KP>& s) {
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    blk[(uint64_t)k * B + b] = __float_as_uint(s.v[k]);
    blk[(uint64_t)(KP + k) * B + b] = s.p[k];
  }
  blk[(uint64_t)(2 * KP) * B + b] = s.lt;
  blk[(uint64_t)(2 * KP + 1) * B + b] = __float_as_uint(s.ltv);
}
template <int KP>
__device__ __forceinline__ void load_summ(const uint32_t* blk, uint64_t B, uint64_t b, Summ<KP>& s) {
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    s.v[k] = __uint_as_float(blk[(uint64_t)k * B + b]);
    s.p[k] = blk[(uint64_t)(KP + k) * B + b];
  }
  s.lt = blk[(uint64_t)(2 * KP) * B + b];
  s.ltv = __uint_as_float(blk[(uint64_t)(2 * KP + 1) * B + b]);
}

// ---------------------------------------------------------------------------
// segment kernel: CTA = W warps over one 32*V-bucket tile of one row; warp w
// streams segment (cta_seg0 + w); the CTA tree-merges its W segment
// summaries in shared memory and writes one summary block.
// ---------------------------------------------------------------------------
struct SegArgs {
  const void* in;        // row-major [rows][row_stride] elements
  uint64_t row_stride;   // elements between rows
  uint64_t rows;
  uint64_t B;            // buckets
  uint64_t nstr;         // stride-rows in the processed range (len / B)
  uint64_t index_offset; // position of the first element (slice sharding)
  uint64_t seg_len;      // stride-rows per segment (>= KP unless nstr < KP)
  uint32_t segs;         // segments per row
  uint32_t cta_per_row_tile;  // summary blocks per (row, tile) = ceil(segs / G)
  uint32_t group;        // G: warps that cooperate on one (row, tile), power of 2 <= W
  uint64_t groups;       // rows * tiles * cta_per_row_tile
  uint32_t tiles;        // ceil(B / (32 V))
  uint32_t* out;         // summary blocks [rows][cta_per_row_tile][words]
                         // (W/G groups per CTA; group = G consecutive segments)
  uint32_t* status;
};

template <int KP, int V>
__device__ __forceinline__ void smem_put(uint32_t* sm, int lane, const Summ<KP> (&s)[V]) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      sm[((k)*V + v) * 32 + lane] = __float_as_uint(s[v].v[k]);
      sm[((KP + k) * V + v) * 32 + lane] = s[v].p[k];
    }
    sm[((2 * KP) * V + v) * 32 + lane] = s[v].lt;
    sm[((2 * KP + 1) * V + v) * 32 + lane] = __float_as_uint(s[v].ltv);
  }
}
template <int KP, int V>
__device__ __forceinline__ void smem_get(const uint32_t* sm, int lane, Summ<KP> (&s)[V]) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      s[v].v[k] = __uint_as_float(sm[((k)*V + v) * 32 + lane]);
      s[v].p[k] = sm[((KP + k) * V + v) * 32 + lane];
    }
    s[v].lt = sm[((2 * KP) * V + v) * 32 + lane];
    s[v].ltv = __uint_as_float(sm[((2 * KP + 1) * V + v) * 32 + lane]);
  }
}

// group tree merge: after the step, warp gw (gw % 2step == 0) holds the
// merge of its group's warps [gw, gw + 2 step); warp 0 of the group writes
// the group's summary block.
template <int KP, int V, int W>
__device__ __forceinline__ void group_merge_store(uint32_t* smem, int warp, int lane, int gw, uint32_t G,
                                                  bool lane_ok, uint64_t row, uint32_t cseg, uint64_t b0,
                                                  const SegArgs& a, Summ<KP> (&s)[V]) {
  constexpr int kWords = (2 * KP + 2) * V * 32;
#pragma unroll
  for (int step = 1; step < W; step *= 2) {
    if (step >= (int)G) break;  // uniform across the CTA
    if ((gw % (2 * step)) == step) smem_put<KP, V>(smem + (warp / (2 * step)) * kWords, lane, s);
    __syncthreads();
    if ((gw % (2 * step)) == 0 && gw + step < (int)G) {
      Summ<KP> o[V];
      smem_get<KP, V>(smem + (warp / (2 * step)) * kWords, lane, o);
#pragma unroll
      for (int v = 0; v < V; ++v) s[v].merge_later(o[v]);
    }
    __syncthreads();
  }
  if (gw == 0 && lane_ok) {
    const uint64_t words = (uint64_t)(2 * KP + 2) * a.B;
    uint32_t* dst = a.out + (row * a.cta_per_row_tile + cseg) * words;
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (b0 + v < a.B) store_summ<KP>(dst, a.B, b0 + v, s[v]);
  }
}

template <typename T, int KP, int V, int W, int D>
__global__ void __launch_bounds__(W * 32)
stage1_segments_kernel(SegArgs a) {
  extern __shared__ uint32_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t G = a.group;
  const int gw = warp & (G - 1);  // warp within its group
  uint64_t grp = (uint64_t)blockIdx.x * (W / G) + warp / G;
  const bool grp_ok = grp < a.groups;
  const uint32_t cseg = (uint32_t)(grp % a.cta_per_row_tile);
  grp /= a.cta_per_row_tile;
  const uint32_t tile = (uint32_t)(grp % a.tiles);
  const uint64_t row = grp / a.tiles;
  const uint64_t b0 = ((uint64_t)tile * 32 + lane) * V;  // first bucket of this lane
  const bool lane_ok = grp_ok && b0 < a.B;
  const uint32_t seg = cseg * G + gw;

  Summ<KP> s[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s[v].clear();
  uint32_t nan = 0;

  if (lane_ok && seg < a.segs) {
    const uint64_t j0 = (uint64_t)seg * a.seg_len;
    const uint64_t j1 = min(j0 + a.seg_len, a.nstr);
    const T* base = reinterpret_cast<const T*>(a.in) + row * a.row_stride + b0;
    const uint64_t B = a.B;
    const uint32_t ioff = (uint32_t)(a.index_offset + b0);
    // prologue: first KP stride-rows fill the lists in rank order
    uint64_t j = j0;
#pragma unroll
    for (int t = 0; t < KP; ++t) {
      if (j < j1) {
        float x[V];
        VecLoad<T, V>::load(base + j * B, x);
        const uint32_t i = ioff + (uint32_t)(j * B);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          nan |= (x[v] != x[v]) ? 1u : 0u;
          s[v].fill(t, x[v], i + v);
        }
        ++j;
      }
    }
    // main loop, D stride-rows per batch, next batch prefetched
    float buf[D][V];
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (j + d < j1) VecLoad<T, V>::load(base + (j + d) * B, buf[d]);
    while (j < j1) {
      float nxt[D][V];
#pragma unroll
      for (int d = 0; d < D; ++d)
        if (j + D + d < j1) VecLoad<T, V>::load(base + (j + D + d) * B, nxt[d]);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        if (j + d < j1) {
          const uint32_t i = ioff + (uint32_t)((j + d) * B);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const float x = buf[d][v];
            if (!(x < s[v].v[KP - 1])) s[v].slow(x, i + v, nan);
          }
        }
      }
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int v = 0; v < V; ++v) buf[d][v] = nxt[d][v];
      j += D;
    }
  }
  if (nan) atomicOr(a.status, ATKG_FLAG_NAN);

  group_merge_store<KP, V, W>(smem, warp, lane, gw, G, lane_ok, row, cseg, b0, a, s);
}

// ---------------------------------------------------------------------------
// merge kernel: one thread per (row, bucket) folds the row's `parts` summary
// blocks in index order, then writes the Alg. 1 grid and/or the summary.
// ---------------------------------------------------------------------------
template <int KP>
__global__ void merge_finalize_kernel(const uint32_t* __restrict__ in, uint32_t parts, uint64_t rows,
                                      uint64_t B, float* grid_v, uint32_t* grid_i, uint64_t grid_stride,
                                      uint32_t* summ_out, const uint32_t* prefix) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * B) return;
  const uint64_t row = t / B, b = t % B;
  const uint64_t words = (uint64_t)(2 * KP + 2) * B;
  const uint32_t* base = in + row * parts * words;
  Summ<KP> acc;
  uint32_t q0 = 0;
  if (prefix) {
    load_summ<KP>(prefix + row * words, B, b, acc);
  } else {
    load_summ<KP>(base, B, b, acc);
    q0 = 1;
  }
  for (uint32_t q = q0; q < parts; ++q) {
    Summ<KP> o;
    load_summ<KP>(base + q * words, B, b, o);
    acc.merge_later(o);
  }
  if (summ_out) store_summ<KP>(summ_out + row * words, B, b, acc);
  if (grid_v) {
    float ov[KP];
    uint32_t oi[KP];
    acc.finalize(ov, oi);
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      grid_v[row * grid_stride + (uint64_t)k * B + b] = ov[k];
      grid_i[row * grid_stride + (uint64_t)k * B + b] = oi[k];
    }
  }
}

// ---------------------------------------------------------------------------
// generic reference-semantics kernel for local_k beyond the register-resident
// specialisations: one thread per (row, bucket) runs Alg. 1 directly on the
// output grid (global memory), exact by construction.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void stage1_generic_kernel(const T* __restrict__ in, uint64_t rows, uint64_t n, uint64_t B,
                                      uint32_t kp, float* grid_v, uint32_t* grid_i, uint32_t* status) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * B) return;
  const uint64_t row = t / B, b = t % B;
  float* v = grid_v + row * kp * B + b;
  uint32_t* ix = grid_i + row * kp * B + b;
  for (uint32_t k = 0; k < kp; ++k) { v[(uint64_t)k * B] = neg_inf(); ix[(uint64_t)k * B] = 0; }
  uint32_t nan = 0;
  const T* r = in + row * n;
  for (uint64_t i = b; i < n; i += B) {
    const float x = Elem<T>::to_f32(r[i]);
    if (x != x) { nan = 1; continue; }
    float* vm = v + (uint64_t)(kp - 1) * B;
    if (x >= *vm) { *vm = x; ix[(uint64_t)(kp - 1) * B] = (uint32_t)i; }
    else continue;
    for (uint32_t k = kp - 1; k >= 1; --k) {
      float* va = v + (uint64_t)k * B;
      float* vb = va - B;
      if (x > *vb) {
        const float tv = *va; *va = *vb; *vb = tv;
        uint32_t* ia = ix + (uint64_t)k * B;
        uint32_t* ib = ia - B;
        const uint32_t tp = *ia; *ia = *ib; *ib = tp;
      } else {
        break;
      }
    }
  }
  if (nan) atomicOr(status, ATKG_FLAG_NAN);
}

// ---------------------------------------------------------------------------
// streaming accumulator kernels (Stage1Accumulator::consume, topk.hpp:59-94):
// fold the elements of positions [start, start+count) into per-bucket state,
// one thread per bucket, in index order.
// ---------------------------------------------------------------------------
template <typename T, int KP>
__global__ void fold_summary_kernel(uint32_t* summ, uint64_t B, const T* __restrict__ blk, uint64_t start,
                                    uint64_t count, uint32_t* status) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Summ<KP> s;
  load_summ<KP>(summ, B, b, s);
  uint32_t nan = 0;
  uint64_t q = start + ((b + B - start % B) % B);  // first position >= start in bucket b
  for (; q < start + count; q += B) s.push(Elem<T>::to_f32(blk[q - start]), (uint32_t)q, nan);
  store_summ<KP>(summ, B, b, s);
  if (nan) atomicOr(status, ATKG_FLAG_NAN);
}

template <int KP>
__global__ void summary_clear_kernel(uint32_t* summ, uint64_t B) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Summ<KP> s;
  s.clear();
  store_summ<KP>(summ, B, b, s);
}

// generic local_k: Alg. 1 directly on the [kp][B] grid
template <typename T>
__global__ void fold_grid_kernel(float* gv, uint32_t* gi, uint64_t B, uint32_t kp, const T* __restrict__ blk,
                                 uint64_t start, uint64_t count, uint32_t* status) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  uint32_t nan = 0;
  uint64_t q = start + ((b + B - start % B) % B);
  for (; q < start + count; q += B) {
    const float x = Elem<T>::to_f32(blk[q - start]);
    if (x != x) { nan = 1; continue; }
    float* vm = gv + (uint64_t)(kp - 1) * B + b;
    if (!(x >= *vm)) continue;
    *vm = x;
    gi[(uint64_t)(kp - 1) * B + b] = (uint32_t)q;
    for (uint32_t k = kp - 1; k >= 1; --k) {
      float* va = gv + (uint64_t)k * B + b;
      float* vb = va - B;
      if (!(x > *vb)) break;
      const float tv = *va; *va = *vb; *vb = tv;
      uint32_t* ia = gi + (uint64_t)k * B + b;
      uint32_t* ib = ia - B;
      const uint32_t tp = *ia; *ia = *ib; *ib = tp;
    }
  }
  if (nan) atomicOr(status, ATKG_FLAG_NAN);
}

__global__ void grid_init_kernel(float* gv, uint32_t* gi, uint64_t count) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) { gv[t] = neg_inf(); gi[t] = 0; }
}

}  // namespace atkg

// ---------------------------------------------------------------------------
// TMA-fed streaming kernel (the hot path).  Every warp streams one long
// segment of one (row, 32*V-bucket tile) through its own ring of NS shared-
// memory slots filled by 1-D bulk copies (cp.async.bulk -> UBLKCP), so
// memory-level parallelism comes from the ring depth, not from thread count,
// and segments can be long -- long segments keep the Alg. 1 insert rate (and
// with it the divergent slow path) low.  Lane l owns buckets tile*32V + l*V
// .. +V-1 and reads its V elements of every stride-row from shared memory.
// ---------------------------------------------------------------------------

namespace atkg {

template <typename T, int V>
__device__ __forceinline__ void lds_vec(const uint8_t* p, float (&out)[V]) {
  constexpr int kBytes = sizeof(T) * V;
  uint32_t w[(kBytes + 3) / 4];
  if constexpr (kBytes == 16) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    w[0] = u.x; w[1] = u.y; w[2] = u.z; w[3] = u.w;
  } else if constexpr (kBytes == 8) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    w[0] = u.x; w[1] = u.y;
  } else {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
  VecLoad<T, V>::unpack(w, out);
}

// Hot loop = filter -> log -> flush.  Per element the common path is one
// compare against a per-bucket threshold f plus a predicated append to a
// per-lane log in shared memory -- 4 instructions, no branch, full SIMT
// width.  f never exceeds the exact current K'-th value of the bucket (it is
// refreshed at every flush), so the log holds every element the sequential
// algorithm would send down its slow path (plus some it rejects on replay).
// A flush replays each lane's logs in index order through the exact summary
// update (Summ::push), warp-synchronously, then raises f.
// Loads are 128-bit (V elements per lane), D stride-rows per block with the
// next block prefetched into registers while the current one is filtered.
// Log layout per warp (structure of arrays, lane-minor, conflict-free):
//   float    val[V][LOGC][32]   element value
//   uint16_t row[V][LOGC][32]   stride-row offset j - j0 of the element
__device__ __forceinline__ void log_append(uint32_t& pv, uint32_t& pj, float x, float f, uint16_t jrel) {
  // appends (x, jrel) when !(x < f) -- NaN included -- and bumps both cursors
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.geu.f32 p, %2, %3;\n\t"
      "@p st.shared.f32 [%0], %2;\n\t"
      "@p st.shared.u16 [%1], %4;\n\t"
      "@p add.u32 %0, %0, 128;\n\t"
      "@p add.u32 %1, %1, 64;\n\t}"
      : "+r"(pv), "+r"(pj)
      : "f"(x), "f"(f), "h"(jrel)
      : "memory");
}

template <typename T, int KP, int V, int W, int NS, int CR, int LOGC, int Q0>
__global__ void __launch_bounds__(W * 32)
stage1_stream_kernel(SegArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  static_assert(LOGC >= 2 * CR, "log must absorb a chunk between flush checks");
  constexpr int LB = V * sizeof(T);              // bytes per lane per stride-row
  constexpr int SB = CR * 32 * LB;               // bytes per ring slot
  constexpr int RING = NS * SB;
  constexpr int LOGV = V * LOGC * 32;            // log entries per warp
  constexpr int WARP_BYTES = RING + LOGV * 6;    // ring + val[] + row[]
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint8_t* ring = smem_raw + warp * WARP_BYTES;
  uint8_t* lbase = ring + RING;
  const float* logv = reinterpret_cast<const float*>(lbase);
  const uint16_t* logj = reinterpret_cast<const uint16_t*>(lbase + LOGV * 4);
  const uint32_t sv0 = (uint32_t)__cvta_generic_to_shared(lbase) + lane * 4;
  const uint32_t sj0 = (uint32_t)__cvta_generic_to_shared(lbase + LOGV * 4) + lane * 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + W * WARP_BYTES) + warp * NS;

  const uint32_t G = a.group;
  const int gw = warp & (G - 1);
  uint64_t grp = (uint64_t)blockIdx.x * (W / G) + warp / G;
  const bool grp_ok = grp < a.groups;
  const uint32_t cseg = (uint32_t)(grp % a.cta_per_row_tile);
  grp /= a.cta_per_row_tile;
  const uint32_t tile = (uint32_t)(grp % a.tiles);
  const uint64_t row = grp / a.tiles;
  const uint64_t tb0 = (uint64_t)tile * 32 * V;
  const uint64_t b0 = tb0 + (uint64_t)lane * V;
  const bool lane_ok = grp_ok && b0 < a.B;
  const uint32_t seg = cseg * G + gw;
  const uint64_t B = a.B;
  const uint64_t j0 = (uint64_t)seg * a.seg_len;
  // trip counts are warp-uniform (warp-synchronous flushes); lanes past the
  // last bucket read lane 0's data (real input, so a NaN there is a real
  // NaN) and filter with f = +inf
  const uint64_t j1 = (grp_ok && seg < a.segs) ? umin64(j0 + a.seg_len, a.nstr) : j0;
  const uint32_t ioff = (uint32_t)(a.index_offset + b0);
  const uint32_t Bu = (uint32_t)B;
  const uint32_t tw = grp_ok ? (uint32_t)(umin64(32 * V, B - tb0) * sizeof(T)) : 0u;  // bytes per row
  const bool contiguous = (a.tiles == 1) && ((uint64_t)tw == B * sizeof(T));
  const uint32_t nch = (uint32_t)((j1 - j0 + CR - 1) / CR);
  const char* gbase = reinterpret_cast<const char*>(a.in) + (row * a.row_stride + tb0) * sizeof(T);
  const uint64_t gstride = B * sizeof(T);
  const uint32_t lane_off = lane_ok ? lane * LB : 0u;

  // ---- TMA ring: lane 0 keeps NS chunks of CR stride-rows in flight --------
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) ptx::mbar_init(&bars[q], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = ptx::policy_evict_first();
  auto issue = [&](uint32_t c) {
    const uint32_t slot = c % NS;
    const uint64_t jr = j0 + (uint64_t)c * CR;
    const uint32_t rows = (uint32_t)umin64(CR, j1 - jr);
    ptx::mbar_arrive_expect_tx(&bars[slot], rows * tw);
    if (contiguous) {
      ptx::bulk_g2s(ring + slot * SB, gbase + jr * gstride, rows * tw, &bars[slot], pol);
    } else {
      for (uint32_t r = 0; r < rows; ++r)
        ptx::bulk_g2s(ring + slot * SB + r * tw, gbase + (jr + r) * gstride, tw, &bars[slot], pol);
    }
  };
  if (lane == 0)
    for (uint32_t c = 0; c < (nch < (uint32_t)NS ? nch : (uint32_t)NS); ++c) issue(c);

  Summ<KP> s[V];
  float f[V];
#pragma unroll
  for (int v = 0; v < V; ++v) { s[v].clear(); f[v] = neg_inf(); }
  uint32_t nan = 0;

  // ---- phase 0: threshold from a sample ------------------------------------
  // Each warp takes the top-KP values (a sorting network on values only) of
  // the first Q0 stride-rows of its segment; the warps of a group (same row
  // and tile) pool them in shared memory and every bucket gets
  // tau = KP-th largest of the pooled sample.  Any subset's KP-th value is a
  // lower bound of the bucket's final KP-th value v*, and Alg. 1 over any
  // subsequence that contains every element >= v* ends in the same state, so
  // filtering with f >= tau from the first element on is exact -- and skips
  // the cold start of every segment.  (The sample reads go through L2, where
  // the ring's bulk copies of the same rows then hit.)
  {
    float net[V][KP];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int k = 0; k < KP; ++k) net[v][k] = neg_inf();
    const T* sbase = reinterpret_cast<const T*>(gbase + lane_off);
    const uint64_t qend = umin64(j0 + Q0, j1);
    for (uint64_t q = j0; q < qend; ++q) {
      float x[V];
      VecLoad<T, V>::load(sbase + q * B, x);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float c = x[v];
        if (c != c) c = neg_inf();  // NaN is caught by the filter below
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const float hi = fmaxf(net[v][k], c);
          c = fminf(net[v][k], c);
          net[v][k] = hi;
        }
      }
    }
    // exchange area: the (still unused) log of every warp
    float* mine = reinterpret_cast<float*>(lbase);
#pragma unroll
    for (int k = 0; k < KP; ++k)
#pragma unroll
      for (int v = 0; v < V; ++v) mine[(k * V + v) * 32 + lane] = net[v][k];
    __syncthreads();
    const int g0 = warp - gw;
    for (int w2 = g0; w2 < g0 + (int)G; ++w2) {
      if (w2 == warp) continue;
      const float* other = reinterpret_cast<const float*>(smem_raw + w2 * WARP_BYTES + RING);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          float c = other[(k * V + v) * 32 + lane];
#pragma unroll
          for (int kk = 0; kk < KP; ++kk) {
            const float hi = fmaxf(net[v][kk], c);
            c = fminf(net[v][kk], c);
            net[v][kk] = hi;
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) f[v] = lane_ok ? net[v][KP - 1] : __int_as_float(0x7f800000);
    __syncthreads();  // exchange area becomes the logs
  }
  float tau[V];
#pragma unroll
  for (int v = 0; v < V; ++v) tau[v] = f[v];

  uint32_t ptr[V], pj[V];
#pragma unroll
  for (int v = 0; v < V; ++v) { ptr[v] = sv0 + v * LOGC * 128; pj[v] = sj0 + v * LOGC * 64; }

  auto flush = [&]() {
    uint32_t cnt[V], m = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      cnt[v] = (ptr[v] - (sv0 + v * LOGC * 128)) >> 7;
      m = cnt[v] > m ? cnt[v] : m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, m, o);
      m = y > m ? y : m;
    }
    for (uint32_t e = 0; e < m; ++e) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (e < cnt[v]) {
          const float x = logv[(v * LOGC + e) * 32 + lane];
          const uint32_t jj = (uint32_t)j0 + logj[(v * LOGC + e) * 32 + lane];
          s[v].push(x, ioff + v + jj * Bu, nan);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      ptr[v] = sv0 + v * LOGC * 128;
      pj[v] = sj0 + v * LOGC * 64;
      f[v] = s[v].full() ? fmaxf(s[v].v[KP - 1], tau[v]) : tau[v];
    }
  };

  for (uint32_t c = 0; c < nch; ++c) {
    const uint32_t slot = c % NS;
    ptx::mbar_wait(&bars[slot], (c / NS) & 1u);
    const uint32_t jrel0 = c * CR;
    const uint32_t rows = (uint32_t)umin64(CR, j1 - (j0 + jrel0));
    const uint8_t* sl = ring + slot * SB + lane_off;
    if (rows == CR) {
#pragma unroll
      for (int r = 0; r < CR; ++r) {
        float x[V];
        lds_vec<T, V>(sl + r * tw, x);
#pragma unroll
        for (int v = 0; v < V; ++v) log_append(ptr[v], pj[v], x[v], f[v], (uint16_t)(jrel0 + r));
      }
    } else {
      for (uint32_t r = 0; r < rows; ++r) {
        float x[V];
        lds_vec<T, V>(sl + r * tw, x);
#pragma unroll
        for (int v = 0; v < V; ++v) log_append(ptr[v], pj[v], x[v], f[v], (uint16_t)(jrel0 + r));
      }
    }
    __syncwarp();
    if (lane == 0 && c + NS < nch) issue(c + NS);
    bool need = false;
#pragma unroll
    for (int v = 0; v < V; ++v) need |= ptr[v] > sv0 + (uint32_t)(v * LOGC + (LOGC - CR - 1)) * 128;
    if (__any_sync(0xffffffffu, need)) flush();
  }
  flush();
  if (nan) atomicOr(a.status, ATKG_FLAG_NAN);
  __syncthreads();  // rings drained and logs done before the merge reuses smem
  group_merge_store<KP, V, W>(reinterpret_cast<uint32_t*>(smem_raw), warp, lane, gw, G, lane_ok, row, cseg, b0,
                              a, s);
}

template <typename T, int KP, int V, int W, int NS, int CR, int LOGC>
constexpr size_t stream_smem_bytes() {
  static_assert((size_t)KP * V * 32 * 4 <= (size_t)V * LOGC * 32 * 6, "sample must fit a warp's log area");
  constexpr size_t work = (size_t)W * (NS * CR * 32 * V * sizeof(T) + V * LOGC * 32 * 6) + (size_t)W * NS * 8;
  constexpr size_t merge = (size_t)(W / 2) * (2 * KP + 2) * V * 32 * 4;
  return work > merge ? work : merge;
}

}  // namespace atkg
