// streamthr.cuh -- approx_top_k for long rows (the LM-logit config: fp32
// rows of 262144; the giant row) by a bucket-agnostic threshold stream.
//
// approx_top_k (/root/reference/proj/core/src/topk.cpp:238-258) returns the
// top K of the B*K' stage-1 candidates.  For a row threshold L, let c_b =
// #elements of bucket b (= i mod B, topk.hpp:13-15) that are >= L and
// M = sum_b min(K', c_b).  The candidates >= L are known exactly from the
// elements >= L alone:
//   c_b <= K'  every marked element is a candidate (it beats v*_b, or it is
//              one of the bucket's only ties);
//   c_b >  K'  v*_b >= L, so the marked elements hold every element >= v*_b
//              and Alg. 1 over them (topk.cpp:80-102) ends in the reference
//              state (the S* lemma; closed form as in summ.cuh finalize).
// If M >= K, every candidate below L ranks after K candidates >= L, so the
// top K of the row are the top K of those M -- bit-identical to the
// reference.  Otherwise the row takes the exact fallback (Alg. 1 summaries
// over every element of the row).
//
// stream kernel (persistent, one CTA per SM slot): the flattened input is
//   cut into G equal pieces of 16-byte vectors; a producer warp streams each
//   piece through an NS-slot shared-memory ring with 1-D TMA bulk copies
//   (chunks never cross a row), and 8 consumer warps each own 1/8 of every
//   chunk.  A warp keeps a threshold L_w and a shared-memory log of the
//   elements >= L_w of its sub-stream of the current row segment; per lane
//   and batch of 8 vectors it needs one NaN-propagating max tree and one
//   compare (the log path runs only when some lane's max reaches L_w).  When
//   the log fills, L_w is raised to the R-th largest logged key and the log
//   compacted; at a row boundary the warp flushes {entries >= L_w, L_w} to a
//   fixed slot (piece, segment, warp) -- no atomics, no zeroed workspace.
//   Invariant: the slot holds every element of the sub-stream >= its L_w.
// finish kernel (one CTA per row): L = max of the row's slot thresholds
//   (every element >= L is in some slot), gather the entries >= L, count
//   per bucket, decide each entry of a bucket with c_b > K' by counting
//   (greater / equal-and-earlier / equal, as rowthr.cuh), bitonic-sort the
//   M candidate rank keys (topk.cpp:30-50) and emit the first K.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "emit.cuh"
#include "ptx.cuh"
#include "rowthr.cuh"
#include "summ.cuh"
#include "stconst.hpp"

namespace atkg {

#ifndef ATKG_ST_NW
#define ATKG_ST_NW 8
#endif
constexpr int kStNW = ATKG_ST_NW;           // consumer warps per CTA
#ifndef ATKG_ST_LOG
#define ATKG_ST_LOG 256
#endif
#ifndef ATKG_ST_SLOTS
#define ATKG_ST_SLOTS 2
#endif
constexpr uint32_t kStLog = ATKG_ST_LOG;   // log entries per warp
constexpr uint32_t kStWarpCap = 128;  // entries a warp keeps at a flush
constexpr uint32_t kStFewSlots = 3;         // finish: one-round-trip gather up to this many slots

struct StArgs {
  const void* in;
  uint64_t n;          // row length
  uint64_t vtot;       // 16-byte vectors in the whole input
  uint64_t psz;        // vectors per piece
  uint32_t G;          // pieces (= grid)
  uint32_t smax;       // slot segments per piece
  uint32_t slot_bytes; // ring slot size
  uint32_t ns;         // ring slots
  float rfac;          // per-warp rank target: R = 8 + rfac * (warp share of the segment)
  float lfac;          // sampled start: expected sample count above the row's safe level, per element
  float cfac;          // entries kept per row segment: Rc = 8 + cfac * (segment elements)
  uint32_t warp_sample;  // sampled start per warp (no CTA barrier) instead of per CTA
  uint32_t* slots;     // [G][smax][kStSlotWords]
  uint32_t* gate;      // giant rows: set by the finish kernel when a row needs the exact path
  uint32_t* status;
};

// piece c = vectors [c * psz, min(vtot, (c + 1) * psz))
__host__ __device__ __forceinline__ uint64_t st_piece_start(uint64_t vtot, uint64_t psz, uint32_t c) {
  const uint64_t v = psz * c;
  return v < vtot ? v : vtot;
}

// warp: the r-th largest of the n logged keys (n >= r >= 1), by MSB-first
// bisection over the 32-bit key
__device__ __forceinline__ uint32_t st_warp_rth(const uint32_t* keys, uint32_t n, uint32_t r, int lane) {
  uint32_t k[kStLog / 32];
#pragma unroll
  for (int i = 0; i < (int)(kStLog / 32); ++i) {
    const uint32_t q = i * 32 + lane;
    k[i] = q < n ? keys[q] : 0u;
  }
  uint32_t ans = 0;
#pragma unroll 1
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t cand = ans | (1u << bit);
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < (int)(kStLog / 32); ++i) c += k[i] >= cand ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= r) ans = cand;
  }
  return ans;
}

// warp: keep the logged entries with key >= t (in place); returns the count
__device__ __forceinline__ uint32_t st_warp_keep(uint32_t* keys, uint32_t* pos, uint32_t n, uint32_t t, int lane) {
  uint32_t k[kStLog / 32], p[kStLog / 32];
#pragma unroll
  for (int i = 0; i < (int)(kStLog / 32); ++i) {
    const uint32_t q = i * 32 + lane;
    k[i] = q < n ? keys[q] : 0u;
    p[i] = q < n ? pos[q] : 0u;
  }
  __syncwarp();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < (int)(kStLog / 32); ++i) {
    const bool keep = (uint32_t)(i * 32 + lane) < n && k[i] >= t;
    const uint32_t b = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const uint32_t d = m + __popc(b & lt);
      keys[d] = k[i];
      pos[d] = p[i];
    }
    m += __popc(b);
  }
  __syncwarp();
  return m;
}

// warp: raise the threshold so that at most `cap` entries stay, keeping
// about r (the r-th largest key; one above it when ties overflow `cap`)
__device__ __forceinline__ uint32_t st_warp_compact(uint32_t* keys, uint32_t* pos, uint32_t n, uint32_t r,
                                                    uint32_t cap, uint32_t& tkey, int lane) {
  if (n < r) return n;
  uint32_t t = st_warp_rth(keys, n, r, lane);
  if (t < tkey) t = tkey;
  uint32_t m = st_warp_keep(keys, pos, n, t, lane);
  while (m > cap && t < 0xff800000u) {  // ties: drop the tied key as well (never past +inf)
    t = t + 1;
    m = st_warp_keep(keys, pos, m, t, lane);
  }
  tkey = t;
  return m;
}

template <typename T>
struct StVec;  // 16-byte vector of T: max tree, per-element access
template <>
struct StVec<float> {
  static constexpr int VE = 4;
  __device__ __forceinline__ static float vmax(const uint4& v) {
    return fmax_nan(fmax_nan(__uint_as_float(v.x), __uint_as_float(v.y)),
                    fmax_nan(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
  __device__ __forceinline__ static float elem(const uint4& v, int j) {
    const uint32_t w = j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
    return __uint_as_float(w);
  }
  // packed max of a batch -> scalar
  using Acc = float;
  __device__ __forceinline__ static Acc acc_init() { return -INFINITY; }
  __device__ __forceinline__ static Acc acc_add(Acc a, const uint4& v) { return fmax_nan(a, vmax(v)); }
  __device__ __forceinline__ static float acc_val(Acc a) { return a; }
};
template <>
struct StVec<__nv_bfloat16> {
  static constexpr int VE = 8;
  __device__ __forceinline__ static float elem(const uint4& v, int j) {
    const uint32_t w = (j >> 1) == 0 ? v.x : (j >> 1) == 1 ? v.y : (j >> 1) == 2 ? v.z : v.w;
    return __uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16));
  }
  using Acc = uint32_t;
  __device__ __forceinline__ static Acc acc_init() { return 0xff80ff80u; }
  __device__ __forceinline__ static Acc acc_add(Acc a, const uint4& v) {
    return bmax_nan(a, bmax_nan(bmax_nan(v.x, v.y), bmax_nan(v.z, v.w)));
  }
  __device__ __forceinline__ static float acc_val(Acc a) {
    const uint32_t m = bmax_nan(a, __byte_perm(a, 0, 0x1032));
    return __uint_as_float(m << 16);
  }
  __device__ __forceinline__ static float vmax(const uint4& v) { return acc_val(acc_add(acc_init(), v)); }
};

// per-warp log state of the current row segment
struct StWarp {
  uint32_t* keys;
  uint32_t* poss;
  uint32_t n, r, tkey, nan, bad;
  float L;
};

// raise L and compact a full log (warp-collective; rare, out of line)
__device__ __noinline__ void st_make_room(StWarp& w, int lane) {
  w.n = st_warp_compact(w.keys, w.poss, w.n, w.r, kStLog - 64, w.tkey, lane);
  w.L = st_oval(w.tkey);
  if (w.n + 32 > kStLog) w.bad = 1u;  // ties fill the log: the row takes the exact path
}

// log the elements >= L of one 16-byte vector per lane (warp-collective);
// runs only for vectors where some lane reaches L
template <typename T>
__device__ __forceinline__ void st_log_vec(StWarp& w, uint4 x, uint32_t pbase, int lane) {
  using V = StVec<T>;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < V::VE; ++j) {
    if (w.n + 32 > kStLog) st_make_room(w, lane);
    const float xv = V::elem(x, j);
    const bool isnan = xv != xv;
    w.nan |= isnan ? 1u : 0u;
    const bool p = !(xv < w.L) && !isnan && !w.bad;
    const uint32_t m = __ballot_sync(0xffffffffu, p);
    if (p) {
      const uint32_t d = w.n + __popc(m & lt);
      w.keys[d] = st_okey(xv);
      w.poss[d] = pbase + j;
    }
    w.n += __popc(m);
  }
  __syncwarp();
}

// flush a segment's log to its slot {count | kStBadCount, Lkey, keys, positions}
__device__ __noinline__ void st_warp_trim(StWarp& w, int lane) {
  if (w.n > kStWarpCap) w.n = st_warp_compact(w.keys, w.poss, w.n, w.r, kStWarpCap, w.tkey, lane);
  if (w.n > kStWarpCap) w.bad = 1u;
}

// warp: the s-th largest of the CTA's 32 * kStNW sampled keys (bisection)
__device__ __forceinline__ uint32_t st_sample_rth(const uint32_t* samp, uint32_t s, int lane) {
  uint32_t k[kStNW];
#pragma unroll
  for (int i = 0; i < kStNW; ++i) k[i] = samp[i * 32 + lane];
  uint32_t ans = 0;
#pragma unroll 1
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t cand = ans | (1u << bit);
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < kStNW; ++i) c += k[i] >= cand ? 1u : 0u;
    if (__reduce_add_sync(0xffffffffu, c) >= s) ans = cand;
  }
  return ans;
}

__device__ __forceinline__ uint4 st_ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// 16-bit-prefix bisection: the largest t = p << 16 with #(keys >= t) >= s,
// a lower bound of the s-th largest key (keys[i * 32 + lane], i < N)
template <int N>
__device__ __forceinline__ uint32_t st_warp_rth16(const uint32_t (&k)[N], uint32_t s) {
  uint32_t ans = 0;
#pragma unroll 1
  for (int bit = 31; bit >= 16; --bit) {
    const uint32_t cand = ans | (1u << bit);
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) c += k[i] >= cand ? 1u : 0u;
    if (__reduce_add_sync(0xffffffffu, c) >= s) ans = cand;
  }
  return ans;
}

// One CTA = kStNW warps walks its piece in steps of kStNW * 32 * UNR
// vectors (a step never crosses a row).  Warp w owns the contiguous w-th
// eighth of every step and streams it through its own kStSlots-deep ring of
// shared-memory slots with 1-D TMA bulk copies (no cross-warp hand-off: the
// warp refills a slot as soon as it has read it).
constexpr int kStSlots = ATKG_ST_SLOTS;

template <typename T, int UNR>
__global__ void __launch_bounds__(kStNW * 32, 16 / kStNW) st_stream_kernel(StArgs a) {
  extern __shared__ __align__(128) uint8_t st_smem[];
  using V = StVec<T>;
  constexpr int VE = V::VE;
  constexpr uint32_t WV = 32 * UNR;             // vectors per warp per step
  constexpr uint32_t STEP = kStNW * WV;         // vectors per step
  __shared__ uint32_t samp[kStNW * 32];
  __shared__ uint32_t wcnt[kStNW];
  __shared__ __align__(8) uint64_t full_bar[kStNW][kStSlots];
  __shared__ uint32_t fl_l[kStNW], fl_n[kStNW], fl_ctr, fl_bad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    fl_ctr = 0;
    fl_bad = 0;
  }
  const uint32_t c = blockIdx.x;
  const uint64_t v0 = st_piece_start(a.vtot, a.psz, c), v1 = st_piece_start(a.vtot, a.psz, c + 1);
  const uint64_t nvrow = a.n / VE;  // vectors per row
  const uint4* in = static_cast<const uint4*>(a.in);
  uint4* ring = reinterpret_cast<uint4*>(st_smem + (size_t)kStNW * 2 * kStLog * 4) + warp * kStSlots * WV;
  StWarp w;
  w.keys = reinterpret_cast<uint32_t*>(st_smem) + warp * 2 * kStLog;
  w.poss = w.keys + kStLog;
  w.n = 0; w.r = 16; w.tkey = 0; w.nan = 0; w.bad = 0;
  w.L = -INFINITY;
  const uint64_t row0 = v0 / nvrow;
  const uint4 pad = sizeof(T) == 2 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                                   : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
  // PDL: the launch overlaps the previous kernel's tail; wait for its
  // completion (and memory) before reading the input or writing slots
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.gate) *a.gate = 0u;
  if (lane == 0) {
    for (int s = 0; s < kStSlots; ++s) ptx::mbar_init(&full_bar[warp][s], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  // step cursor, 32-bit offsets relative to v0: [cur, cur + len) within
  // row row0 + row, which ends at row_end
  const uint32_t plen = (uint32_t)(v1 - v0);
  struct Step {
    uint32_t cur, row, row_end, len;
  };
  auto make_step = [&](uint32_t cur, uint32_t row, uint32_t row_end) {
    if (cur >= row_end) { ++row; row_end += (uint32_t)nvrow; }
    Step st;
    st.cur = cur;
    st.row = row;
    st.row_end = row_end;
    st.len = cur < plen ? min(min(STEP, plen - cur), row_end - cur) : 0u;
    return st;
  };
  auto wlen_of = [&](const Step& st) {  // this warp's vectors of a step
    const uint32_t b = warp * WV;
    return st.len > b ? min(WV, st.len - b) : 0u;
  };
  const uint64_t pol = ptx::policy_evict_first();
  auto issue = [&](const Step& st, uint32_t k) {  // lane 0
    const uint32_t s = k % kStSlots;
    const uint32_t wl = wlen_of(st);
    ptx::mbar_arrive_expect_tx(&full_bar[warp][s], wl * 16);
    if (wl) ptx::bulk_g2s(ring + s * WV, in + v0 + st.cur + warp * WV, wl * 16, &full_bar[warp][s], pol);
  };
  uint32_t seg_len_e = 0;  // elements of the current row segment in this piece
  // CTA-level flush of a row segment (uniform over the CTA): Lc = max of the
  // warps' thresholds; every warp appends its entries >= Lc to the slot
  auto flush = [&](uint32_t seg) {  // seg = row - row0
    st_warp_trim(w, lane);
    if (lane == 0) {
      fl_l[warp] = w.tkey;
      fl_n[warp] = w.n;
      if (w.bad) fl_bad = 1u;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kStNW * 32) : "memory");
    uint32_t Lc = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < kStNW; ++i) { Lc = max(Lc, fl_l[i]); tot += fl_n[i]; }
    // keep about Rc entries per segment: when the warps logged far more
    // (a row cut into many pieces), warp 0 raises Lc to the Rc-th largest
    // logged key (16-bit prefix bisection; any Lc above the warps' own
    // thresholds keeps the slot exact)
    const uint32_t Rc = (uint32_t)fminf(768.f, 8.f + ceilf(fminf(1e6f, a.cfac * (float)seg_len_e)));
    if (tot > 2 * Rc) {  // uniform
      if (warp == 0) {
        const uint32_t* lk = reinterpret_cast<const uint32_t*>(st_smem);
        uint32_t ans = 0;
#pragma unroll 1
        for (int bit = 31; bit >= 16; --bit) {
          const uint32_t cand = ans | (1u << bit);
          uint32_t cnt = 0;
          for (int i = 0; i < kStNW; ++i) {
            const uint32_t* kk = lk + i * 2 * kStLog;
            const uint32_t ni = fl_n[i];
            for (uint32_t e = lane; e < ni; e += 32) cnt += kk[e] >= cand ? 1u : 0u;
          }
          if (__reduce_add_sync(0xffffffffu, cnt) >= Rc) ans = cand;
        }
        if (lane == 0) fl_l[0] = max(Lc, ans);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kStNW * 32) : "memory");
      Lc = fl_l[0];
    }
    uint32_t* sl = a.slots + ((uint64_t)c * a.smax + seg) * kStSlotWords;
    for (uint32_t e0 = 0; e0 < w.n; e0 += 32) {
      const uint32_t e = e0 + lane;
      const bool keep = e < w.n && w.keys[e] >= Lc;
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      uint32_t base = 0;
      if (lane == 0 && bal) base = atomicAdd(&fl_ctr, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const uint32_t d = base + __popc(bal & ((1u << lane) - 1u));
        if (d < kStSlotCap) {
          sl[2 + d] = w.keys[e];
          sl[2 + kStSlotCap + d] = w.poss[e];
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kStNW * 32) : "memory");
    if (threadIdx.x == 0) {
      sl[0] = (fl_bad || fl_ctr > kStSlotCap) ? kStBadCount : fl_ctr;
      sl[1] = Lc;
      fl_ctr = 0;
      fl_bad = 0;
    }
  };
  uint32_t row = ~0u;
  auto process = [&](const Step& st, const uint4* sl) {
    const bool first = st.row != row;  // first step of a row segment (uniform over the CTA)
    if (first) {
      if (row != ~0u) flush(row);
      row = st.row;
      w.n = 0;
      w.bad = 0;
      w.tkey = 0;
      w.L = -INFINITY;
      const uint32_t seg = min(plen, st.row_end) - st.cur;  // vectors of this row in the piece
      seg_len_e = seg * VE;
      const float share = (float)seg * (float)VE / (float)kStNW;
      w.r = (uint32_t)fminf(96.f, fmaxf(16.f, 8.f + ceilf(a.rfac * share)));
    }
    const uint32_t wl = wlen_of(st);
    uint4 x[UNR];
    float m[UNR];  // per-vector maxima (NaN-propagating)
    if (wl == WV) {  // full slot: plain loads
#pragma unroll
      for (int i = 0; i < UNR; ++i) x[i] = sl[i * 32 + lane];
    } else {
#pragma unroll
      for (int i = 0; i < UNR; ++i) x[i] = (uint32_t)(i * 32 + lane) < wl ? sl[i * 32 + lane] : pad;
    }
#pragma unroll
    for (int i = 0; i < UNR; ++i) m[i] = V::vmax(x[i]);
    float mx = m[0];
#pragma unroll
    for (int i = 1; i < UNR; ++i) mx = fmax_nan(mx, m[i]);
    if (first) {
      // sampled start: the s-th largest lane maximum of the segment's first
      // step is below the row's safe level with high probability; any start
      // value is exact (the slot records the threshold actually used)
      uint32_t t0;
      if (a.warp_sample) {
        // per-warp sample: the warp's own 32 lane maxima, no CTA barrier
        const uint32_t k1[1] = {mx != mx ? 0u : st_okey(mx)};
        const uint32_t wl = wlen_of(st);
        const float mu = a.lfac * (float)(wl * VE);
        const uint32_t sr = (uint32_t)fminf(32.f, ceilf(mu + 4.5f * sqrtf(mu) + 3.f));
        t0 = st_warp_rth16<1>(k1, sr);
      } else {
      samp[warp * 32 + lane] = mx != mx ? 0u : st_okey(mx);
      asm volatile("bar.sync 1, %0;" ::"n"(kStNW * 32) : "memory");
      if (warp == 0) {
        uint32_t k8[kStNW];
#pragma unroll
        for (int i = 0; i < kStNW; ++i) k8[i] = samp[i * 32 + lane];
        const float mu = a.lfac * (float)(st.len * VE);
        const uint32_t sr = (uint32_t)fminf((float)(kStNW * 32), ceilf(mu + 4.5f * sqrtf(mu) + 3.f));
        const uint32_t t = st_warp_rth16<kStNW>(k8, sr);
        __syncwarp();
        if (lane == 0) samp[0] = t;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kStNW * 32) : "memory");
      t0 = samp[0];
      }
      if (t0 > w.tkey) {
        w.tkey = t0;
        w.L = st_oval(t0);
      }
    }
    if (!__any_sync(0xffffffffu, !(mx < w.L))) return;
    // element offset of this warp's first vector in its row
    const uint32_t off_e = (st.cur + (uint32_t)nvrow - st.row_end + warp * WV) * VE;
    if (w.n + 64 > kStLog) st_make_room(w, lane);
    // lanes append their hits with shared-memory atomics (divergent, rare):
    // per-lane hit bits (element k = i * VE + j), one rolled loop over them
    if (lane == 0) wcnt[warp] = w.n;
    __syncwarp();
    uint32_t ovf = 0;
    if (!(mx < w.L)) {
      constexpr int HW = (UNR * VE + 31) / 32;
      uint32_t hm[HW];
#pragma unroll
      for (int h = 0; h < HW; ++h) hm[h] = 0;
#pragma unroll
      for (int i = 0; i < UNR; ++i) {
        if (!(m[i] < w.L) && (uint32_t)(i * 32 + lane) < wl) {  // padding (-inf) hits only when L = -inf
#pragma unroll
          for (int j = 0; j < VE; ++j)
            hm[(i * VE + j) / 32] |= (!(V::elem(x[i], j) < w.L) ? 1u : 0u) << ((i * VE + j) % 32);
        }
      }
#pragma unroll
      for (int h = 0; h < HW; ++h) {
#pragma unroll 1
        while (hm[h]) {
          const int kk = h * 32 + __ffs(hm[h]) - 1;
          hm[h] &= hm[h] - 1;
          const int i = kk / VE, j = kk % VE;
          const float xv = sizeof(T) == 4
                               ? reinterpret_cast<const float*>(sl + i * 32 + lane)[j]
                               : __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(sl + i * 32 + lane)[j] << 16);
          if (xv != xv) {
            w.nan = 1u;
          } else {
            const uint32_t d = atomicAdd(&wcnt[warp], 1u);
            if (d < kStLog) {
              w.keys[d] = st_okey(xv);
              w.poss[d] = off_e + (i * 32 + lane) * VE + j;
            } else {
              ovf = 1u;
            }
          }
        }
      }
    }
    __syncwarp();
    if (!__any_sync(0xffffffffu, ovf)) {
      w.n = wcnt[warp];
      return;
    }
    // the batch overflowed the log: drop its entries and log it vector by
    // vector, making room (raising L) as needed
#pragma unroll 1
    for (int i = 0; i < UNR; ++i) {
      const uint4 xi = (uint32_t)(i * 32 + lane) < wl ? sl[i * 32 + lane] : pad;
      if (__any_sync(0xffffffffu, !(V::vmax(xi) < w.L))) st_log_vec<T>(w, xi, off_e + (i * 32 + lane) * VE, lane);
    }
    __syncwarp();
  };
  // prologue: fill the ring
  Step sp = make_step(0, 0, (uint32_t)((row0 + 1) * nvrow - v0));  // processing cursor
  Step si = sp;                                                     // issue cursor
  uint32_t ki = 0;
  for (; ki < kStSlots && si.len; ++ki) {
    if (lane == 0) issue(si, ki);
    si = make_step(si.cur + si.len, si.row, si.row_end);
  }
#pragma unroll 1
  for (uint32_t k = 0; sp.len; ++k) {
    const uint32_t s = k % kStSlots;
    ptx::mbar_wait(&full_bar[warp][s], (k / kStSlots) & 1);
    process(sp, ring + s * WV);
    __syncwarp();
    if (si.len) {  // refill the slot just read with step k + kStSlots
      if (lane == 0) issue(si, ki);
      ++ki;
      si = make_step(si.cur + si.len, si.row, si.row_end);
    }
    sp = make_step(sp.cur + sp.len, sp.row, sp.row_end);
  }
  if (row != ~0u) flush(row);
  if (__any_sync(0xffffffffu, w.nan) && lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// first k of M unique 64-bit rank keys (emit.cuh); false: bins too crowded
__device__ __forceinline__ bool st_emit_ranked(const uint64_t* keys, uint32_t* mem32, uint32_t M, uint32_t k,
                                               float* ov, uint32_t* oi) {
  return emit_ranked<uint64_t>(keys, reinterpret_cast<uint64_t*>(mem32), M, k, [&](uint32_t r, uint64_t key) {
    ov[r] = __uint_as_float(key_value_bits(key));
    oi[r] = (uint32_t)key;
  });
}

// Stage 2 (select_top_k_candidates, topk.cpp:192-236) for 128 < count <=
// 1024 candidates per row: one CTA of 128 threads per row, survivors
// (index < limit) compacted into shared memory, then the counting-sort rank
// emit; rows holding -inf (sentinel keys may repeat) or crowded bins sort
// with a bitonic network instead.  smem: keys[P] | mem[P] (u64).
__global__ void __launch_bounds__(512) stage2_rank_kernel(const float* __restrict__ vals,
                                                          const uint32_t* __restrict__ idx, uint32_t count,
                                                          uint64_t stride, uint32_t k, uint64_t index_limit,
                                                          uint32_t P, float* out_v, uint32_t* out_i,
                                                          uint32_t* status) {
  extern __shared__ __align__(16) uint64_t s2_keys[];
  __shared__ uint32_t nsurv, flags;
  uint64_t* keys = s2_keys;
  uint32_t* mem32 = reinterpret_cast<uint32_t*>(s2_keys + P);
  const uint64_t row = blockIdx.x;
  const uint32_t t = threadIdx.x;
  if (t == 0) { nsurv = 0; flags = 0; }
  __syncthreads();
  uint32_t f = 0;
  for (uint32_t c = t; c < count; c += blockDim.x) {
    const float v = vals[row * stride + c];
    const uint32_t ix = idx[row * stride + c];
    if (v != v) f |= 1u;
    if (v == -INFINITY) f |= 2u;
    if ((uint64_t)ix < index_limit) keys[atomicAdd(&nsurv, 1u)] = rank_key_bits(__float_as_uint(v), ix);
  }
  if (f) atomicOr(&flags, f);
  __syncthreads();
  const uint32_t M = nsurv;
  if (flags & 1u) {
    if (t == 0) atomicOr(status, ATKG_FLAG_NAN);
    return;
  }
  if (M < k) {
    if (t == 0) atomicOr(status, kFlagFew);
    return;
  }
  if (!(flags & 2u) && st_emit_ranked(keys, mem32, M, k, out_v + row * k, out_i + row * k)) return;
  for (uint32_t q = M + t; q < P; q += blockDim.x) keys[q] = ~0ull;
  __syncthreads();
  block_bitonic_sort(keys, P);
  for (uint32_t q = t; q < k; q += blockDim.x) {
    out_v[row * k + q] = __uint_as_float(key_value_bits(keys[q]));
    out_i[row * k + q] = (uint32_t)keys[q];
  }
}

struct StFinArgs {
  const void* in;
  uint64_t n, vtot, psz;
  uint32_t G, smax, B, k;
  uint32_t slot_cap;    // entries per slot (kStSlotCap for the stream's own slots)
  uint32_t ecap;   // gathered-entry capacity (shared memory)
  uint32_t force_slow;  // tests: every row takes the exact fallback
  uint32_t* gate;       // giant rows: no in-kernel fallback, flag the row for the host instead
  const uint32_t* slots;
  float* out_v;
  uint32_t* out_i;
  uint32_t* status;
};

// one CTA (256 threads; 1024 for a few long rows) per row.  smem: ent keys[ecap] | ent pos[ecap] |
// grouped keys[ecap] | grouped pos[ecap] | cnt[B] | off[B] | cur[B]; the
// candidate keys (u64, <= max(B*K', ecap)) alias the first two arrays.
template <typename T, int KP>
__global__ void __launch_bounds__(1024) st_finish_kernel(StFinArgs a) {
  extern __shared__ __align__(128) uint8_t st_smem[];
  uint8_t* smem = st_smem;
  __shared__ uint32_t sh_l, sh_ne, sh_nk, sh_bad, sh_nc, sh_m;
  __shared__ uint32_t pfx[kStMaxRowPieces + 1];
  __shared__ uint64_t red64[32];
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  const uint64_t row = blockIdx.x;
  constexpr int VE = 16 / sizeof(T);
  const uint64_t nvrow = a.n / VE;
  uint32_t* ek = reinterpret_cast<uint32_t*>(smem);
  uint32_t* ep = ek + a.ecap;
  uint32_t* gk = ep + a.ecap;
  uint32_t* gp = gk + a.ecap;
  uint32_t* cnt = gp + a.ecap;
  uint32_t* off = cnt + a.B;
  uint32_t* cur = off + a.B;
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem);
  const uint32_t B = a.B;
  const bool pow2 = (B & (B - 1)) == 0;
  auto bucket = [&](uint32_t p) { return pow2 ? (p & (B - 1)) : p % B; };  // partition_index, topk.hpp:13-15
  if (t == 0) { sh_l = 0; sh_ne = 0; sh_nk = 0; sh_bad = 0; sh_nc = 0; }
  for (uint32_t b = t; b < B; b += nt) cnt[b] = 0;
  // pieces overlapping this row; the row is segment 0 of every piece but
  // the first (those start inside the row)
  const uint64_t va = row * nvrow, vb = (row + 1) * nvrow - 1;
  const uint32_t ca = (uint32_t)(va / a.psz), cb = (uint32_t)(vb / a.psz);
  const uint32_t seg_a = (uint32_t)(row - (uint64_t)ca * a.psz / nvrow);
  const uint32_t nslots = cb - ca + 1;
  auto slot_ptr = [&](uint32_t q) {
    return a.slots + ((uint64_t)(ca + q) * a.smax + (q == 0 ? seg_a : 0u)) * (2ull + 2ull * a.slot_cap);
  };
  __syncthreads();  // counters initialised
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the stream kernel's slots are complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // slot headers -> L = max of the slot thresholds (every element >= L is in
  // some slot), entry counts -> prefix pfx[]
  const int lane = t & 31;
  uint32_t Lk;
  if (nslots <= kStFewSlots && a.ecap >= 1024 && nt >= 256 && kStSlotCap % nt == 0 && a.slot_cap == kStSlotCap) {
    // few slots (rows over a handful of pieces): every thread reads the
    // headers (broadcast) and, speculatively, its share of every slot's
    // entries in the same round trip; filter against L = max threshold
    constexpr uint32_t PER = kStSlotCap / 256;  // entries per thread at 256 threads
    const uint32_t per = kStSlotCap / nt;
    uint32_t kk[kStFewSlots][PER], pp[kStFewSlots][PER], mq[kStFewSlots];
    Lk = 0;
    bool bad = false;
#pragma unroll
    for (uint32_t q = 0; q < kStFewSlots; ++q) {
      if (q < nslots) {
        const uint32_t* sl = slot_ptr(q);
        mq[q] = sl[0];
        Lk = max(Lk, sl[1]);
        bad |= mq[q] > kStSlotCap;
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
          if (i < per) {
            kk[q][i] = sl[2 + i * nt + t];
            pp[q][i] = sl[2 + kStSlotCap + i * nt + t];
          }
        }
      } else {
        mq[q] = 0;
      }
    }
    if (t == 0) { sh_l = Lk; if (bad) sh_bad = 1u; }
    if (!bad) {
#pragma unroll
      for (uint32_t q = 0; q < kStFewSlots; ++q) {
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
          const uint32_t e = i * nt + t;
          if (i < per && e < mq[q] && kk[q][i] >= Lk) {
            const uint32_t d = atomicAdd(&sh_ne, 1u);
            if (d < a.ecap) {
              ek[d] = kk[q][i];
              ep[d] = pp[q][i];
              atomicAdd(&cnt[bucket(pp[q][i])], 1u);
            }
          }
        }
      }
    }
  } else {
  if (nslots <= 32) {  // one warp: headers, max, prefix by shuffles
    if (t < 32) {
      const uint32_t* sl = lane < (int)nslots ? slot_ptr(lane) : nullptr;
      const uint32_t m0 = sl ? sl[0] : 0u, l0 = sl ? sl[1] : 0u;
      const bool bad = m0 > a.slot_cap;
      const uint32_t m = bad ? 0u : m0;
      uint32_t incl = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane < (int)nslots) pfx[lane] = incl - m;
      if (lane == (int)nslots - 1) pfx[nslots] = incl;
      const uint32_t lmax = __reduce_max_sync(0xffffffffu, l0);
      if (__any_sync(0xffffffffu, bad) && lane == 0) sh_bad = 1u;
      if (lane == 0) sh_l = lmax;
    }
  } else {
    uint32_t lmax = 0;
    const uint32_t per = (nslots + nt - 1) / nt;
    const uint32_t q0 = min(nslots, t * per), q1 = min(nslots, q0 + per);
    uint32_t sum = 0;
    for (uint32_t q = q0; q < q1; ++q) {
      const uint32_t* sl = slot_ptr(q);
      const uint32_t m = sl[0];
      lmax = max(lmax, sl[1]);
      if (m > a.slot_cap) sh_bad = 1u;
      pfx[q] = m > a.slot_cap ? 0u : m;
      sum += m > a.slot_cap ? 0u : m;
    }
    lmax = __reduce_max_sync(0xffffffffu, lmax);
    if (lane == 0 && lmax) atomicMax(&sh_l, lmax);
    uint64_t tot;
    uint32_t ex = (uint32_t)block_excl_scan64(sum, red64, &tot);
    for (uint32_t q = q0; q < q1; ++q) {
      const uint32_t m = pfx[q];
      pfx[q] = ex;
      ex += m;
    }
    if (t == 0) pfx[nslots] = (uint32_t)tot;
  }
  __syncthreads();
  Lk = sh_l;
  const uint32_t E = pfx[nslots];
  // every entry >= L, flattened over the slots (binary search for the slot);
  // four entries per thread per trip so their loads overlap
  auto slot_of = [&](uint32_t e) {  // pfx[lo] <= e < pfx[lo + 1]
    uint32_t lo = 0, hi = nslots;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pfx[mid] <= e) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  for (uint32_t e0 = 0; e0 < E; e0 += 4 * nt) {
    uint32_t key[4], q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t e = e0 + u * nt + t;
      q[u] = e < E ? slot_of(e) : 0u;
      key[u] = e < E ? slot_ptr(q[u])[2 + (e - pfx[q[u]])] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t e = e0 + u * nt + t;
      if (e < E && key[u] >= Lk) {
        const uint32_t d = atomicAdd(&sh_ne, 1u);
        if (d < a.ecap) {
          const uint32_t pos = slot_ptr(q[u])[2 + a.slot_cap + (e - pfx[q[u]])];
          ek[d] = key[u];
          ep[d] = pos;
          atomicAdd(&cnt[bucket(pos)], 1u);
        }
      }
    }
  }
  }
  __syncthreads();
  const uint32_t ne_all = sh_ne;
  bool fast = sh_bad == 0 && Lk > kStKeyNegInf && !a.force_slow && ne_all <= a.ecap;
  if (fast) {
    const uint32_t ne = ne_all;
    {
      // M and bucket offsets (block scan over buckets; thread owns a run)
      const uint32_t per = (B + nt - 1) / nt;
      const uint32_t b0 = min(B, t * per), b1 = min(B, b0 + per);
      uint32_t s = 0, mm = 0;
      for (uint32_t b = b0; b < b1; ++b) { s += cnt[b]; mm += min((uint32_t)KP, cnt[b]); }
      uint64_t tot;
      const uint64_t ex = block_excl_scan64(((uint64_t)mm << 32) | s, red64, &tot);
      uint32_t o = (uint32_t)ex;
      for (uint32_t b = b0; b < b1; ++b) { off[b] = o; cur[b] = o; o += cnt[b]; }
      if (t == 0) sh_m = (uint32_t)(tot >> 32);
      __syncthreads();
      for (uint32_t q = t; q < ne_all; q += nt) {
        const uint32_t d = atomicAdd(&cur[bucket(ep[q])], 1u);
        gk[d] = ek[q];
        gp[d] = ep[q];
      }
      __syncthreads();
      fast = sh_m >= a.k;
      if (fast) {
        // every entry: kept in its bucket's final state?  (cand aliases ek/ep)
        for (uint32_t q = t; q < ne; q += nt) {
          const uint32_t key = gk[q], pos = gp[q], b = bucket(pos);
          const uint32_t cb_ = cnt[b];
          bool kept = true;
          if (cb_ > (uint32_t)KP) {
            const uint32_t o0 = off[b];
            uint32_t g = 0, e = 0, eq = 0, maxg = 0, lasteq = pos;
            for (uint32_t rr = o0; rr < o0 + cb_; ++rr) {
              const uint32_t kr = gk[rr], pr = gp[rr];
              g += kr > key ? 1u : 0u;
              maxg = kr > key ? max(maxg, pr) : maxg;
              const bool same = kr == key;
              eq += same ? 1u : 0u;
              e += (same && pr < pos) ? 1u : 0u;
              lasteq = same ? max(lasteq, pr) : lasteq;
            }
            kept = false;
            if (g + eq <= (uint32_t)KP - 1) {
              kept = true;
            } else if (g <= (uint32_t)KP - 1) {
              const uint32_t ct = KP - g;
              if (e + 2 <= ct) kept = true;
              else if ((g == 0 || lasteq > maxg) ? (e + 1 == eq) : (e + 1 == ct)) kept = true;
            }
          }
          if (kept) {
            const uint32_t d = atomicAdd(&sh_nc, 1u);
            cand[d] = rank_key_bits(__float_as_uint(st_oval(key)), pos);
          }
        }
      }
    }
  }
  __syncthreads();
  uint32_t M = sh_nc;
  if (!fast && a.gate) {  // giant row: the host reruns the exact path
    if (t == 0) atomicOr(a.gate, 1u);
    return;
  }
  if (!fast) {
    // exact fallback: Alg. 1 summaries of every bucket over the whole row
    const T* x = static_cast<const T*>(a.in) + row * a.n;
    const uint32_t nstr = (uint32_t)(a.n / B);
    const uint32_t filled = min((uint32_t)KP, nstr);
    uint32_t nan = 0;
    for (uint32_t b = t; b < B; b += nt) {
      Summ<KP> sm;
      sm.clear();
      for (uint32_t j = 0; j < nstr; ++j) sm.push(Elem<T>::to_f32(x[(uint64_t)j * B + b]), j * B + b, nan);
      float fv[KP];
      uint32_t fi[KP];
      sm.finalize(fv, fi);
#pragma unroll
      for (int kk = 0; kk < KP; ++kk)
        if ((uint32_t)kk < filled) cand[b * filled + kk] = rank_key_bits(__float_as_uint(fv[kk]), fi[kk]);
    }
    if (nan) atomicOr(a.status, ATKG_FLAG_NAN);
    M = B * filled;
  }
  if (fast) {
    // unique keys (real elements >= L > -inf): counting sort on the key's
    // value word (ascending = value descending), ranks inside a bin by
    // comparison; the first k ranks are the output
    if (st_emit_ranked(cand, gk, M, a.k, a.out_v + row * a.k, a.out_i + row * a.k)) return;
  }
  uint32_t P = 2;
  while (P < M) P <<= 1;
  for (uint32_t q = M + t; q < P; q += nt) cand[q] = ~0ull;
  __syncthreads();
  group_bitonic_sort<uint64_t>(cand, P, t, nt);
  for (uint32_t q = t; q < a.k; q += nt) {
    const uint64_t key = cand[q];
    a.out_v[row * a.k + q] = __uint_as_float(key_value_bits(key));
    a.out_i[row * a.k + q] = (uint32_t)key;
  }
}

// ---------------------------------------------------------------------------
// Slices of one row on different GPUs (the sharded giant row).
// A slice runs the threshold stream as a row of its own; this kernel then
// folds the slice's stream slots into ONE payload slot {count, Lkey,
// keys[cap], positions[cap]} holding every element of the slice >= Lkey (Lkey
// = the max of the slots' thresholds), positions made global by
// index_offset.  The payloads of all slices are exchanged (all-gather) and
// st_finish_kernel runs on them as the slots of one row: L = the max of the
// slice thresholds, exact for the same reason as within one GPU.  A payload
// with count kStBadCount (a slot overflowed, the slice held a NaN, or more
// than cap entries) sends every rank to the exact summary path.
// ---------------------------------------------------------------------------
struct StPayArgs {
  const uint32_t* slots;  // the slice's stream slots [G][smax][kStSlotWords]; the slice is segment 0
  uint32_t G, smax, cap;
  uint64_t index_offset;
  const uint32_t* status;  // the stream kernel's flags (NaN)
  uint32_t* payload;       // [2 + 2 cap]
};

__global__ void __launch_bounds__(1024) st_slice_payload_kernel(StPayArgs a) {
  __shared__ uint32_t sh_l, sh_bad, sh_n;
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  if (t == 0) { sh_l = 0; sh_bad = (*a.status & ATKG_FLAG_NAN) ? 1u : 0u; sh_n = 0; }
  __syncthreads();
  auto slot = [&](uint32_t q) { return a.slots + (uint64_t)q * a.smax * kStSlotWords; };
  uint32_t lmax = 0, bad = 0;
  for (uint32_t q = t; q < a.G; q += nt) {
    const uint32_t* sl = slot(q);
    bad |= sl[0] > kStSlotCap ? 1u : 0u;
    lmax = max(lmax, sl[1]);
  }
  lmax = __reduce_max_sync(0xffffffffu, lmax);
  if ((t & 31) == 0) atomicMax(&sh_l, lmax);
  if (bad) sh_bad = 1u;
  __syncthreads();
  const uint32_t L = sh_l;
  if (!sh_bad) {
    // every entry >= L, one warp per slot (entries strided over its lanes)
    const uint32_t warp = t >> 5, lane = t & 31, nw = nt >> 5;
    for (uint32_t q = warp; q < a.G; q += nw) {
      const uint32_t* sl = slot(q);
      const uint32_t m = sl[0];
      for (uint32_t e0 = 0; e0 < m; e0 += 32) {
        const uint32_t e = e0 + lane;
        const uint32_t key = e < m ? sl[2 + e] : 0u;
        const bool keep = e < m && key >= L;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(&sh_n, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
          const uint32_t d = base + __popc(bal & ((1u << lane) - 1u));
          if (d < a.cap) {
            a.payload[2 + d] = key;
            a.payload[2 + a.cap + d] = (uint32_t)(sl[2 + kStSlotCap + e] + a.index_offset);
          }
        }
      }
    }
  }
  __syncthreads();
  if (t == 0) {
    a.payload[0] = (sh_bad || sh_n > a.cap) ? kStBadCount : sh_n;
    a.payload[1] = L;
  }
}

}  // namespace atkg
