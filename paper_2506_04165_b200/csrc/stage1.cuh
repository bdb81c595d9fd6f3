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
#include "stage2.cuh"
#include "summ.cuh"

namespace atkg {

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

static __global__ void grid_init_kernel(float* gv, uint32_t* gi, uint64_t count) {
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

// ---------------------------------------------------------------------------
// Hot loop = filter -> log -> flush.  Per element the common path is one
// compare against a per-bucket threshold f plus a predicated append to a
// per-lane log in shared memory -- 4 instructions, no branch, full SIMT
// width.  f never exceeds the exact current K'-th value of the bucket (it is
// refreshed at every flush), so the log holds every element the sequential
// algorithm would send down its slow path (plus some it rejects on replay).
// A flush replays each lane's logs in index order through the exact summary
// update (Summ::push), warp-synchronously, then raises f.
// Log layout per warp (structure of arrays, lane-minor, conflict-free):
//   float    val[V][LOGC][32]   element value
//   uint32_t row[V][LOGC][32]   stride-row index j of the element
// ---------------------------------------------------------------------------
template <int ROWOFF>
__device__ __forceinline__ void log_append(uint32_t& pv, float x, float f, uint32_t j) {
  // appends (x, j) when !(x < f) -- NaN included -- and bumps the cursor;
  // the row array sits ROWOFF bytes after the value array
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.geu.f32 p, %1, %2;\n\t"
      "@p st.shared.f32 [%0], %1;\n\t"
      "@p st.shared.u32 [%0+%4], %3;\n\t"
      "@p add.u32 %0, %0, 128;\n\t}"
      : "+r"(pv)
      : "f"(x), "f"(f), "r"(j), "n"(ROWOFF)
      : "memory");
}

// Balanced flat partition.  The work is the flattened space of
// (unit = (row, 32V-bucket tile), stride-row j) pairs, cut into equal
// contiguous ranges, one per warp, so every SM streams the same number of
// bytes whatever the row count.  A warp walks its range in chunks of CR
// stride-rows (never crossing a unit), fed by its own ring of NS shared-memory
// slots that 1-D TMA bulk copies (cp.async.bulk -> UBLKCP) keep full.  Each
// unit piece of the range yields one exact summary, stored as part
// (w - first warp of the unit) of that unit; merge_parts_kernel folds a unit's
// parts in index order.
//
// Before filtering a piece, the warp takes tau = K'-th largest value of the
// piece's first Q0 stride-rows (a value-only sorting network).  Any subset's
// K'-th value is a lower bound of the bucket's final K'-th value v*, and
// Alg. 1 over any subsequence that contains every element >= v* ends in the
// same state, so filtering with f >= tau from the first element on is exact
// -- and skips the cold start of every piece.
struct FlatArgs {
  const void* in;
  uint64_t row_stride;    // elements between rows
  uint64_t B;             // buckets
  uint64_t nstr;          // stride-rows per unit
  uint64_t index_offset;  // position of the first element (slice sharding)
  uint64_t total;         // units * nstr
  uint64_t len;           // stride-rows per warp
  uint32_t tiles;         // ceil(B / 32V)
  uint32_t parts;         // part slots per unit
  uint64_t warps;         // warps in the grid with work
  uint32_t* out;          // summary blocks [rows][parts][words(B)]
  uint32_t* status;
};

template <typename T, int KP, int V, int W, int NS, int CR, int LOGC, int Q0>
__global__ void __launch_bounds__(W * 32)
stage1_flat_kernel(FlatArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  static_assert(LOGC > CR, "log must absorb a chunk between flush checks");
  constexpr int LB = V * sizeof(T);              // bytes per lane per stride-row
  constexpr int SB = CR * 32 * LB;               // bytes per ring slot
  constexpr int RING = NS * SB;
  constexpr int LOGV = V * LOGC * 32;            // log entries per warp
  constexpr int WARP_BYTES = RING + LOGV * 8;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint8_t* ring = smem_raw + warp * WARP_BYTES;
  uint8_t* lbase = ring + RING;
  const float* logv = reinterpret_cast<const float*>(lbase);
  const uint32_t* logj = reinterpret_cast<const uint32_t*>(lbase + LOGV * 4);
  const uint32_t sv0 = (uint32_t)__cvta_generic_to_shared(lbase) + lane * 4;
  const uint64_t w = (uint64_t)blockIdx.x * W + warp;
  if (w >= a.warps) return;  // warp-uniform; no CTA-wide barriers below
  const uint64_t F0 = w * a.len;
  const uint64_t F1 = umin64(F0 + a.len, a.total);
  const uint64_t B = a.B;
  const uint64_t gstride = B * sizeof(T);
  const uint32_t Bu = (uint32_t)B;

  // chunk sequence of this warp: [F, F + rows) with rows <= CR, cut at unit
  // ends; producer and consumer walk it incrementally (no divisions per chunk)
  auto unit_src = [&](uint64_t u, uint32_t& tw, bool& contiguous) -> const char* {
    const uint64_t row = u / a.tiles, tile = u - row * a.tiles;
    const uint64_t tb0 = tile * 32 * V;
    tw = (uint32_t)(umin64(32 * V, B - tb0) * sizeof(T));
    contiguous = (a.tiles == 1) && ((uint64_t)tw == gstride);
    return reinterpret_cast<const char*>(a.in) + (row * a.row_stride + tb0) * sizeof(T);
  };

  // ---- ring fill: every lane copies its own LB bytes of each stride-row ----
  // (cp.async -> LDGSTS; a lane only ever reads back what it copied, so the
  // per-thread wait_group is the only synchronisation the ring needs)
  uint64_t Fi = F0;
  uint64_t ui = F0 / a.nstr;
  uint64_t ji = F0 - ui * a.nstr;
  uint32_t ci = 0, twi = 0;
  bool conti = false;
  const char* srci = unit_src(ui, twi, conti);
  uint32_t lofi = ((uint64_t)lane * LB < twi) ? lane * LB : 0u;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  auto issue_next = [&]() {  // all lanes; always commits one group
    if (Fi < F1) {
      if (ji == a.nstr) {
        ++ui;
        ji = 0;
        srci = unit_src(ui, twi, conti);
        lofi = ((uint64_t)lane * LB < twi) ? lane * LB : 0u;
      }
      const uint32_t slot = ci % NS;
      const uint64_t left = umin64(F1 - Fi, a.nstr - ji);
      const uint32_t dst = ring_s + slot * SB;
      if (conti && twi == 32 * LB && left >= CR) {
        // full tile, full chunk: one contiguous CR x 32LB block, lanes stride
        // through it with compile-time offsets
        const char* src = srci + ji * gstride + lane * LB;
#pragma unroll
        for (int r = 0; r < CR; ++r) ptx::cp_async<LB>(dst + r * 32 * LB + lane * LB, src + r * 32 * LB);
        Fi += CR;
        ji += CR;
      } else {
        const uint32_t rows = (uint32_t)umin64(CR, left);
        const char* src = srci + ji * gstride + lofi;
        for (uint32_t r = 0; r < rows; ++r) {
          ptx::cp_async<LB>(dst + r * twi + lofi, src);
          src += gstride;
        }
        Fi += rows;
        ji += rows;
      }
      ++ci;
    }
    ptx::cp_async_commit();
  };
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) issue_next();

  uint32_t nan = 0;
#ifdef ATKG_COUNT_LOG
  uint32_t dbg_logged = 0, dbg_taken = 0, dbg_flushes = 0;
#endif
  uint64_t F = F0;  // consumer position
  uint32_t c = 0;   // chunks consumed
  while (F < F1) {
    // ---- a unit piece: [F, piece_end) of unit u ----------------------------
    const uint64_t u = F / a.nstr;  // once per piece
    const uint64_t piece_end = umin64((u + 1) * a.nstr, F1);
    const uint64_t row = u / a.tiles, tile = u - row * a.tiles;
    const uint64_t b0 = (tile * 32 + lane) * V;
    const bool lane_ok = b0 < B;
    const uint32_t ioff = (uint32_t)(a.index_offset + b0);
    const uint64_t jp0 = F - u * a.nstr;
    const uint64_t plen = piece_end - F;
    const uint32_t lane_off = lane_ok ? lane * LB : 0u;

    Summ<KP> s[V];
    float f[V], tau[V];
    {
      // threshold tau from the piece's first Q0 stride-rows (through L2)
      float net[V][KP];
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int k = 0; k < KP; ++k) net[v][k] = neg_inf();
      const T* sbase = reinterpret_cast<const T*>(reinterpret_cast<const char*>(a.in) +
                                                  (row * a.row_stride + tile * 32 * V) * sizeof(T) + lane_off) +
                       jp0 * B;
      const uint64_t qn = umin64(Q0, plen);
      constexpr int QB = 8;
      for (uint64_t q0 = 0; q0 < qn; q0 += QB) {
        float x[QB][V];
#pragma unroll
        for (int r = 0; r < QB; ++r) {
          if (q0 + r < qn) VecLoad<T, V>::load(sbase + (q0 + r) * B, x[r]);
          else {
#pragma unroll
            for (int v = 0; v < V; ++v) x[r][v] = neg_inf();
          }
        }
#pragma unroll
        for (int r = 0; r < QB; ++r) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            float cc = x[r][v];
            if (cc != cc) cc = neg_inf();  // NaN is caught by the filter below
#pragma unroll
            for (int k = 0; k < KP; ++k) {
              const float hi = fmaxf(net[v][k], cc);
              cc = fminf(net[v][k], cc);
              net[v][k] = hi;
            }
          }
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        s[v].clear();
        tau[v] = lane_ok ? net[v][KP - 1] : __int_as_float(0x7f800000);
        f[v] = tau[v];
      }
    }
    uint32_t ptr[V];
#pragma unroll
    for (int v = 0; v < V; ++v) ptr[v] = sv0 + v * LOGC * 128;
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
            const uint32_t jj = logj[(v * LOGC + e) * 32 + lane];
#ifdef ATKG_COUNT_LOG
            dbg_logged++;
            if (!(s[v].full() && x < s[v].v[KP - 1])) dbg_taken++;
#endif
            s[v].push(x, ioff + v + jj * Bu, nan);
          }
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        ptr[v] = sv0 + v * LOGC * 128;
        f[v] = s[v].full() ? fmaxf(s[v].v[KP - 1], tau[v]) : tau[v];
      }
    };

    uint32_t tw;
    bool contiguous;
    (void)unit_src(u, tw, contiguous);
    uint32_t jabs0 = (uint32_t)jp0;
    while (F < piece_end) {
      const uint32_t slot = c % NS;
      issue_next();                       // chunk c + NS - 1 into the free slot
      ptx::cp_async_wait<NS - 1>();       // chunk c has landed (this lane's bytes)
      const uint32_t rows = (uint32_t)umin64(CR, piece_end - F);
      const uint8_t* sl = ring + slot * SB + lane_off;
      if (rows == CR) {
        // all shared-memory loads first: the appends are asm volatile with a
        // memory clobber, so loads placed after one cannot be hoisted
        float x[CR][V];
#pragma unroll
        for (int r = 0; r < CR; ++r) lds_vec<T, V>(sl + r * tw, x[r]);
#pragma unroll
        for (int r = 0; r < CR; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v) log_append<LOGV * 4>(ptr[v], x[r][v], f[v], jabs0 + r);
      } else {
        for (uint32_t r = 0; r < rows; ++r) {
          float x[V];
          lds_vec<T, V>(sl + r * tw, x);
#pragma unroll
          for (int v = 0; v < V; ++v) log_append<LOGV * 4>(ptr[v], x[v], f[v], jabs0 + r);
        }
      }
      F += rows;
      jabs0 += rows;
      ++c;
      bool need = false;
#pragma unroll
      for (int v = 0; v < V; ++v) need |= ptr[v] > sv0 + (uint32_t)(v * LOGC + (LOGC - CR - 1)) * 128;
      if (__any_sync(0xffffffffu, need)) {
#ifdef ATKG_COUNT_LOG
        dbg_flushes++;
#endif
        flush();
      }
    }
    flush();
    // part index of this piece within its unit
    const uint64_t wfirst = (u * a.nstr) / a.len;
    const uint64_t part = w - wfirst;
    const uint64_t words = (uint64_t)(2 * KP + 2) * B;
    uint32_t* dst = a.out + (row * a.parts + part) * words;
    if (lane_ok) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (b0 + v < B) store_summ<KP>(dst, B, b0 + v, s[v]);
    }
  }
  if (nan) atomicOr(a.status, ATKG_FLAG_NAN);
#ifdef ATKG_COUNT_LOG
  atomicAdd(a.status + 1, dbg_logged);
  atomicAdd(a.status + 2, dbg_taken);
  if (lane == 0) atomicAdd(a.status + 3, dbg_flushes);
#endif
}

template <typename T, int KP, int V, int W, int NS, int CR, int LOGC>
constexpr size_t flat_smem_bytes() {
  return (size_t)W * (NS * CR * 32 * V * sizeof(T) + V * LOGC * 32 * 8);
}

// ---------------------------------------------------------------------------
// hierarchical merge of a unit's parts: CTA = 32 buckets x Y part-ranges;
// thread (y, b) folds parts [y*n/Y, (y+1)*n/Y) of bucket b in order, then a
// shared-memory tree folds the Y partial summaries; writes the Alg. 1 grid
// and/or the merged summary.
// ---------------------------------------------------------------------------
template <int KP, int Y>
__global__ void __launch_bounds__(32 * Y)
merge_parts_kernel(const uint32_t* __restrict__ in, uint32_t parts, uint64_t nstr, uint64_t len, uint32_t tiles,
                   uint32_t vec, uint64_t rows, uint64_t B, float* grid_v, uint32_t* grid_i, uint64_t grid_stride,
                   uint32_t* summ_out) {
  __shared__ uint32_t sm[(Y / 2 > 0 ? Y / 2 : 1) * (2 * KP + 2) * 32];
  const int lane = threadIdx.x & 31, y = threadIdx.x >> 5;
  const uint64_t bgroups = (B + 31) / 32;
  const uint64_t row = blockIdx.x / bgroups;
  const uint64_t b = (blockIdx.x % bgroups) * 32 + lane;
  const bool ok = row < rows && b < B;
  const uint64_t bb = ok ? b : 0;
  // parts of this bucket's unit (row, tile)
  const uint64_t u = row * tiles + bb / (32ull * vec);
  const uint64_t w0 = (u * nstr) / len, w1 = ((u + 1) * nstr - 1) / len;
  const uint32_t n = (uint32_t)(w1 - w0 + 1);
  const uint64_t words = (uint64_t)(2 * KP + 2) * B;
  const uint32_t* base = in + row * parts * words;
  const uint32_t q0 = (uint32_t)((uint64_t)n * y / Y), q1 = (uint32_t)((uint64_t)n * (y + 1) / Y);
  Summ<KP> acc;
  acc.clear();
  if (ok)
    for (uint32_t q = q0; q < q1; ++q) {
      Summ<KP> o;
      load_summ<KP>(base + q * words, B, bb, o);
      acc.merge_later(o);
    }
  // tree over y: after the step, y (y % 2step == 0) holds [y, y + 2 step)
#pragma unroll
  for (int step = 1; step < Y; step *= 2) {
    uint32_t* slot = sm + (y / (2 * step)) * (2 * KP + 2) * 32;
    if ((y % (2 * step)) == step) {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        slot[k * 32 + lane] = __float_as_uint(acc.v[k]);
        slot[(KP + k) * 32 + lane] = acc.p[k];
      }
      slot[(2 * KP) * 32 + lane] = acc.lt;
      slot[(2 * KP + 1) * 32 + lane] = __float_as_uint(acc.ltv);
    }
    __syncthreads();
    if ((y % (2 * step)) == 0 && y + step < Y) {
      Summ<KP> o;
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        o.v[k] = __uint_as_float(slot[k * 32 + lane]);
        o.p[k] = slot[(KP + k) * 32 + lane];
      }
      o.lt = slot[(2 * KP) * 32 + lane];
      o.ltv = __uint_as_float(slot[(2 * KP + 1) * 32 + lane]);
      acc.merge_later(o);
    }
    __syncthreads();
  }
  if (y != 0 || !ok) return;
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
// fused tail for the flat path: one CTA per row stages the row's part
// summaries in shared memory (coalesced 16-byte loads, all in flight), every
// thread folds its buckets' parts in index order and finalizes the Alg. 1
// state, then the CTA sorts the row's candidate rank keys (bitonic, shared
// memory) and emits the top K -- stage 2 without a grid round trip.
// Optionally also writes the grid (stage1_partial_reduce).
// ---------------------------------------------------------------------------
template <int KP>
__global__ void __launch_bounds__(512)
merge_select_kernel(const uint32_t* __restrict__ in, uint32_t parts, uint64_t nstr, uint64_t len, uint32_t tiles,
                    uint32_t vec, uint64_t B, uint32_t filled, uint32_t P, uint32_t k, float* out_v,
                    uint32_t* out_i, float* grid_v, uint32_t* grid_i, uint32_t* status) {
  extern __shared__ __align__(16) uint32_t sm[];
  const uint64_t row = blockIdx.x;
  const uint64_t words = (uint64_t)(2 * KP + 2) * B;
  uint32_t* stage = sm;                                                      // [parts][words]
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm + ((parts * words + 3) & ~3ull));  // [P]
  {
    const uint4* src = reinterpret_cast<const uint4*>(in + row * parts * words);
    uint4* dst = reinterpret_cast<uint4*>(stage);
    const uint64_t n4 = parts * words / 4;
    for (uint64_t t = threadIdx.x; t < n4; t += blockDim.x) dst[t] = src[t];
  }
  for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) keys[t] = ~0ull;
  __syncthreads();
  for (uint64_t b = threadIdx.x; b < B; b += blockDim.x) {
    const uint64_t u = row * tiles + b / (32ull * vec);
    const uint64_t w0 = (u * nstr) / len, w1 = ((u + 1) * nstr - 1) / len;
    const uint32_t n = (uint32_t)(w1 - w0 + 1);
    Summ<KP> acc;
    load_summ<KP>(stage, B, b, acc);
    for (uint32_t q = 1; q < n; ++q) {
      Summ<KP> o;
      load_summ<KP>(stage + q * words, B, b, o);
      acc.merge_later(o);
    }
    float ov[KP];
    uint32_t oi[KP];
    acc.finalize(ov, oi);
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
      if (grid_v) {
        grid_v[row * KP * B + (uint64_t)kk * B + b] = ov[kk];
        grid_i[row * KP * B + (uint64_t)kk * B + b] = oi[kk];
      }
      if ((uint32_t)kk < filled) keys[(uint64_t)kk * B + b] = rank_key_bits(__float_as_uint(ov[kk]), oi[kk]);
    }
  }
  __syncthreads();
  if (*status & ATKG_FLAG_NAN) return;  // the reference rejects NaN before ranking
  block_bitonic_sort(keys, P);
  for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) {
    out_v[row * k + t] = __uint_as_float(key_value_bits(keys[t]));
    out_i[row * k + t] = (uint32_t)keys[t];
  }
}

}  // namespace atkg
