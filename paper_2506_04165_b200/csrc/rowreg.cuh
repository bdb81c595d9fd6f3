// rowreg.cuh -- approx_top_k for short bf16 rows streamed ONCE from HBM, one
// warp per row, many rows in flight per SM: the FFN-activation config C3
// (rows of 14336 = 128 buckets x 112 stride-rows, K' = 4, K = 287).
//
// The earlier row kernels (rowres, rowwarp, shortrow) stage whole rows in
// shared memory; 28 KB per row leaves 6-8 rows (warps) per SM and they end
// up latency-bound.  Here a row only passes through a 4 KB staging tile:
//   * lane l reads its own 8 bytes (buckets 4l..4l+3, topk.hpp:13-15: element
//     i goes to bucket i mod B) of every stride-row straight into registers
//     (256 B per warp load, 16 loads in flight per lane, double-buffered);
//   * per bf16x2 word one packed compare against the level (set.geu) and one
//     packed a*2 + hit (fma.rn.bf16x2): after a tile of 7 stride-rows each
//     half holds 128 + its 7 hit bits; no branch, no per-bucket state in the
//     loop;
//   * after every tile the lane walks the set bits and inserts the hits
//     (code << 16 | position, read back from its own column of the staging
//     tile) into the bucket's 4-slot state in Alg. 1 order (topk.cpp:80-102)
//     -- the row is never read again.
// Threshold argument: for a level L let c_b = the elements of
// bucket b that are >= L and M = sum_b min(K', c_b).  If M >= K the top K of
// the row's candidates are the top K of its candidates >= L, and those
// follow from the elements >= L alone (Alg. 1 over a bucket's elements >= L,
// the S* lemma).  M is known exactly after the pass (the filled slots), so
// ANY level may be tried:
//   fast path   the CTA's prediction of the level of the row's K-th
//               candidate minus a margin: the running mean of the previous
//               rows' levels, or -- when the rows' scales differ -- the
//               row's own scale statistic plus the mean offset (kRgSigmas
//               below).  One pass; M >= K afterwards proves it.
//   two-pass    no prediction yet or M < K: the exact K-th largest of the
//               B K' group maxima (K' disjoint groups of stride-rows per
//               bucket) guarantees M >= K; a second pass (the row is in L2)
//               inserts the hits against it.
//   exact path  L = -inf: Alg. 1 of every bucket as the reference runs it,
//               then a bitonic sort of the B K' rank keys.  Slow; degenerate
//               rows only.
// After the pass the states hold the row's candidates >= L; a bitonic sort
// of the 512 slots in registers writes the first K in output order
// (topk.cpp:30-50).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "rowthr.cuh"

namespace atkg {

constexpr uint32_t kRgTmp = 512;             // candidates: <= B K'
constexpr uint32_t kRgKeyNegInf = 0x007fu;   // asc_code16(-inf)
constexpr int kRgTile = 7;                   // stride-rows per load batch = per staging tile (7 hit bits per
                                             // bucket and tile fit a bf16 counter exactly: 128 + bits)
// per warp: staging tile [8][32] x 8 B (the sorted keys after the pass) | state [128 buckets][4] u32
constexpr uint32_t kRgLaneQ = 5;            // uint4 per lane in the state: 4 buckets + 16 bytes of padding (banks)
constexpr uint32_t kRgWarpSmem = 8 * 256 + 16 * kRgLaneQ * 32;
static_assert(8 * 256 == 4 * kRgTmp, "the sorted keys reuse the staging tile");

struct RgArgs {
  const uint16_t* in;
  uint64_t rows;
  uint32_t S;           // stride-rows per bucket (n = 128 S)
  uint32_t k;
  uint32_t robust;      // 0: per CTA, by the spread of its first rows' scale statistics; 1: always; 2: never
  uint32_t margin;      // prediction: codes below the level of the last row's K-th candidate
  uint32_t force;       // tests: 1 = every row two-pass, 2 = every row exact
  uint32_t probe;       // development: stop after phase `probe`
  float* out_v;
  uint32_t* out_i;
  uint32_t* status;
};

__device__ __forceinline__ uint2 rg_ldg(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
// 0xffff in each half whose bf16 is >= the matching half of L2 (false on NaN)
__device__ __forceinline__ uint32_t rg_ge(uint32_t w, uint32_t L2) {
  uint32_t h;
  asm("set.ge.u32.bf16x2 %0, %1, %2;" : "=r"(h) : "r"(w), "r"(L2));
  return h;
}
// 1.0 (bf16) in each half whose bf16 is >= the matching half of L2 or unordered (a NaN element
// counts as a hit: it reaches stage 2 and is reported there)
__device__ __forceinline__ uint32_t rg_geu1(uint32_t w, uint32_t L2) {
  uint32_t h;
  asm("set.geu.bf16x2.bf16x2 %0, %1, %2;" : "=r"(h) : "r"(w), "r"(L2));
  return h;
}
// packed bf16 a * 2 + b on the FMA pipe (the ALU pipe is this kernel's bottleneck)
__device__ __forceinline__ uint32_t rg_shl_add(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(0x40004000u), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t rg_bits2(uint32_t code) {
  const uint32_t b = code16_bits(code);
  return b | (b << 16);
}

template <typename K>
__device__ __forceinline__ void warp_bitonic_sort(K* s, uint32_t P, uint32_t lane) {
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t q = lane; q < P / 2; q += 32) {
        const uint32_t i = 2 * q - (q & (stride - 1));
        const uint32_t j = i + stride;
        const bool asc = (i & size) == 0;
        const K a = s[i], b = s[j];
        if ((a > b) == asc) { s[i] = b; s[j] = a; }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ uint32_t rg_excl_scan(uint32_t v, uint32_t lane, uint32_t* tot) {
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if ((int)lane >= o) inc += y;
  }
  *tot = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

// group g of K' = 4 covers the stride-rows [g S / 4, (g + 1) S / 4)
template <int S>
__host__ __device__ constexpr int rg_group(int s) {
  int g = 0;
  while (g < 3 && (g + 1) * S / 4 <= s) ++g;
  return g;
}

// The hit pass over the row: Alg. 1 (topk.cpp:80-102) over the hits (>= L2,
// or NaN) of each of the lane's 4 buckets, in stream order.  Per tile of 7
// stride-rows: the loads (issued PF tiles ahead) are compared against L2 --
// one packed compare (ALU pipe) and one packed a * 2 + hit (FMA pipe) per
// word, so after 7 stride-rows each bf16 half holds 128 + its 7 hit bits
// exactly -- and copied to the lane's column of the staging tile.  Bit
// 8 u + 6 - i of the tile's hit mask = element slot u of stride-row i
// (u = 0, 1, 2, 3 <-> bucket 4 lane + 0, 2, 1, 3); the lane then walks the
// set bits from the top (ascending stride-row inside a slot) and inserts
// (code << 16 | position) into the bucket's state[4], kept in Alg. 1 order
// (value descending, a later equal element never passes an earlier one; the
// empty slots are 0, below every hit).  POS: the hits are strictly positive,
// their bf16 bits order as they are (a NaN sorts first); otherwise ascending
// codes, and a NaN raises `nan`.
template <int S, bool POS, int PF>
__device__ __forceinline__ void rg_hits(const uint2* p, const uint8_t* nxt, uint32_t L2, uint32_t lane, uint2* stage,
                                        uint4* state, uint32_t& nan, uint2 (&buf)[2][kRgTile]) {
  static_assert(PF == 1, "the caller preloads tiles 0 and 1 (the row's scale is read from them)");
  constexpr int NB = (S + kRgTile - 1) / kRgTile;
  constexpr int AH = 3;                    // L2 prefetch distance in tiles (7 x 256 B = 14 lines each)
  constexpr uint32_t TB = kRgTile * 256;   // bytes per tile
  const uint8_t* rowb = reinterpret_cast<const uint8_t*>(p) - 8 * lane;
  const uint8_t* col = reinterpret_cast<const uint8_t*>(stage + lane);
  uint4* st4 = state + kRgLaneQ * lane;  // the lane's buckets 4 lane .. 4 lane + 3
#pragma unroll
  for (int bt = 0; bt < NB; ++bt) {
    if (bt >= 1 && bt + 1 < NB) {  // tile 1 came with the caller's preload
#pragma unroll
      for (int i = 0; i < kRgTile; ++i) {
        const int s = (bt + 1) * kRgTile + i;
        if (s < S) buf[(bt + 1) & 1][i] = rg_ldg(p + s * 32);
      }
    }
    // pull the tile AH ahead into L2 (of this row, then of the warp's next row): the register
    // loads one tile ahead then wait on L2, not on DRAM
    if (lane < TB / 128) {
      const uint8_t* q = bt + AH < NB ? rowb + (bt + AH) * TB : (nxt ? nxt + (bt + AH - NB) * TB : nullptr);
      if (q && (bt + AH < NB ? (bt + AH) * TB + lane * 128 < (uint32_t)S * 256 : true))
        asm volatile("prefetch.global.L2 [%0];" ::"l"(q + lane * 128));
    }
    uint32_t ax = 0x3f803f80u, ay = 0x3f803f80u;  // 1.0 | 1.0
#pragma unroll
    for (int i = 0; i < kRgTile; ++i) {
      const int s = bt * kRgTile + i;
      if (s < S) {
        const uint2 v = buf[bt & 1][i];
        ax = rg_shl_add(ax, rg_geu1(v.x, L2));
        ay = rg_shl_add(ay, rg_geu1(v.y, L2));
        stage[(6 - i) * 32 + lane] = v;
      } else {
        ax = rg_shl_add(ax, 0u);
        ay = rg_shl_add(ay, 0u);
      }
    }
    uint32_t m = (ax & 0x007f007fu) | ((ay & 0x007f007fu) << 8);
    while (m) {
      uint32_t b;
      asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(m));
      m ^= 1u << b;
      const uint32_t r = b & 7u;                         // stride-row bt * 7 + 6 - r
      const uint32_t j = ((b >> 2) & 2u) | (b >> 4);     // element slot b >> 3 -> bucket 4 lane + j
      uint32_t val = *reinterpret_cast<const uint16_t*>(col + r * 256 + j * 2);
      if (!POS) {
        if ((val & 0x7fffu) > 0x7f80u) nan = 1u;
        val = asc_code16(val);
      }
      const uint32_t e = (val << 16) | (((bt * kRgTile + 6) << 7) - (r << 7) + 4 * lane + j);
      uint4 sv = st4[j];
      if (sv.w <= (e | 0xffffu)) {  // value >= v[K' - 1]: e replaces the minimum slot, then rises
        const uint32_t eb = e & 0xffff0000u;  // past the strictly smaller values
        const bool a2 = sv.z >= eb, a1 = sv.y >= eb, a0 = sv.x >= eb;  // slot k stays above e
        sv.w = a2 ? e : sv.z;
        sv.z = a2 ? sv.z : (a1 ? e : sv.y);
        sv.y = a1 ? sv.y : (a0 ? e : sv.x);
        sv.x = a0 ? sv.x : e;
        st4[j] = sv;
      }
    }
  }
}

// The maxima pass (rows without a usable prediction): lane-local maxima of
// the K' = 4 groups of stride-rows of the lane's buckets, NaN-propagating.
template <int S>
__device__ __forceinline__ void rg_max(const uint2* p, uint32_t (&gm)[2][4]) {
  constexpr int U = 14;
#pragma unroll
  for (int s0 = 0; s0 < S; s0 += U) {
    uint2 v[U];
#pragma unroll
    for (int i = 0; i < U; ++i)
      if (s0 + i < S) v[i] = rg_ldg(p + (s0 + i) * 32);
#pragma unroll
    for (int i = 0; i < U; ++i) {
      if (s0 + i < S) {
        const int g = rg_group<S>(s0 + i);
        gm[0][g] = bmax_nan(gm[0][g], v[i].x);
        gm[1][g] = bmax_nan(gm[1][g], v[i].y);
      }
    }
  }
}

// The same two passes for a row length known only at run time (S = 0
// instantiation: any 8 <= S <= 512): tiles in pairs through two register
// buffers, the ragged last tile with per-stride-row checks.
template <bool POS>
__device__ __forceinline__ void rg_hits_rt(const uint2* p, const uint8_t* nxt, int S, uint32_t L2, uint32_t lane,
                                           uint2* stage, uint4* state, uint32_t& nan, uint2 (&pre)[2][kRgTile]) {
  constexpr int AH = 3;
  constexpr uint32_t TB = kRgTile * 256;
  const int NB = (S + kRgTile - 1) / kRgTile;
  const uint8_t* rowb = reinterpret_cast<const uint8_t*>(p) - 8 * lane;
  const uint8_t* col = reinterpret_cast<const uint8_t*>(stage + lane);
  uint4* st4 = state + kRgLaneQ * lane;
  // a stride-row past the end loads as -inf: never a hit (the level is above -inf)
  auto load = [&](uint2 (&b)[kRgTile], int t) {
    const int s0 = t * kRgTile;
    const uint2* pt = p + s0 * 32;  // immediate offsets from one pointer per tile
    if (s0 + kRgTile <= S) {
#pragma unroll
      for (int i = 0; i < kRgTile; ++i) b[i] = rg_ldg(pt + i * 32);
    } else {
#pragma unroll
      for (int i = 0; i < kRgTile; ++i) {
        b[i] = make_uint2(0xff80ff80u, 0xff80ff80u);
        if (s0 + i < S) b[i] = rg_ldg(pt + i * 32);
      }
    }
  };
  uint2* stl = stage + lane;
  auto process = [&](const uint2 (&b)[kRgTile], int t) {
    {
      const int ta = t + AH;
      const uint32_t off = (uint32_t)(ta < NB ? ta : ta - NB) * TB + lane * 128;
      const uint8_t* q = ta < NB ? rowb : nxt;
      if (lane < TB / 128 && q && off < (uint32_t)S * 256) asm volatile("prefetch.global.L2 [%0];" ::"l"(q + off));
    }
    const int s0 = t * kRgTile;
    uint32_t ax = 0x3f803f80u, ay = 0x3f803f80u;
#pragma unroll
    for (int i = 0; i < kRgTile; ++i) {
      ax = rg_shl_add(ax, rg_geu1(b[i].x, L2));
      ay = rg_shl_add(ay, rg_geu1(b[i].y, L2));
      stl[(6 - i) * 32] = b[i];
    }
    uint32_t m = (ax & 0x007f007fu) | ((ay & 0x007f007fu) << 8);
    const uint32_t pbase = ((uint32_t)(s0 + 6) << 7) + 4 * lane;
    while (m) {
      uint32_t bb;
      asm("bfind.u32 %0, %1;" : "=r"(bb) : "r"(m));
      m ^= 1u << bb;
      const uint32_t r = bb & 7u;
      const uint32_t j = ((bb >> 2) & 2u) | (bb >> 4);
      uint32_t val = *reinterpret_cast<const uint16_t*>(col + r * 256 + j * 2);
      if (!POS) {
        if ((val & 0x7fffu) > 0x7f80u) nan = 1u;
        val = asc_code16(val);
      }
      const uint32_t e = (val << 16) | (pbase - (r << 7) + j);
      uint4 sv = st4[j];
      if (sv.w <= (e | 0xffffu)) {
        const uint32_t eb = e & 0xffff0000u;
        const bool a2 = sv.z >= eb, a1 = sv.y >= eb, a0 = sv.x >= eb;
        sv.w = a2 ? e : sv.z;
        sv.z = a2 ? sv.z : (a1 ? e : sv.y);
        sv.y = a1 ? sv.y : (a0 ? e : sv.x);
        sv.x = a0 ? sv.x : e;
        st4[j] = sv;
      }
    }
  };
  uint2 (&b0)[kRgTile] = pre[0];  // tiles 0 and 1 came with the caller's preload
  uint2 (&b1)[kRgTile] = pre[1];
#pragma unroll 1
  for (int bt = 0; bt < NB; bt += 2) {
    if (bt >= 2 && bt + 1 < NB) load(b1, bt + 1);
    process(b0, bt);
    if (bt + 1 < NB) {
      if (bt + 2 < NB) load(b0, bt + 2);
      process(b1, bt + 1);
    }
  }
}

__device__ __forceinline__ void rg_max_rt(const uint2* p, int S, uint32_t (&gm)[2][4]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int s1 = g == 3 ? S : (g + 1) * S / 4;
#pragma unroll 1
    for (int s = g * S / 4; s < s1; s += 4) {
      uint2 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = s + i < s1 ? rg_ldg(p + (s + i) * 32) : make_uint2(0xff80ff80u, 0xff80ff80u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        gm[0][g] = bmax_nan(gm[0][g], v[i].x);
        gm[1][g] = bmax_nan(gm[1][g], v[i].y);
      }
    }
  }
}

// lane count of the 16 group maxima >= L2 (float order)
__device__ __forceinline__ uint32_t rg_count_ge(const uint32_t (&gm)[2][4], uint32_t L2) {
  uint32_t t = 0;
#pragma unroll
  for (int w = 0; w < 2; ++w)
#pragma unroll
    for (int g = 0; g < 4; ++g) t |= rg_ge(gm[w][g], L2) & (0x00010001u << (4 * w + g));
  return __popc(t);
}

// The exact path (degenerate rows): Alg. 1 of every bucket as the reference
// runs it (topk.cpp:80-102 with the {-inf, 0} sentinels of topk.cpp:118-121),
// the B K' = 512 rank keys sorted, the first K written (topk.cpp:192-236).
static __device__ __noinline__ void rg_exact(const uint16_t* xr, int S, uint32_t lane, uint32_t K, uint64_t* srt, float* ov,
                                      uint32_t* oi) {
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const uint32_t bk = 4 * lane + j;
    float v[4];
    uint32_t ix[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) { v[t] = neg_inf(); ix[t] = 0; }
#pragma unroll 4
    for (int r = 0; r < S; ++r) {
      const uint32_t pos = r * 128 + bk;
      const float x = __uint_as_float((uint32_t)__ldg(xr + pos) << 16);
      const bool take = x >= v[3];
      v[3] = take ? x : v[3];
      ix[3] = take ? pos : ix[3];
#pragma unroll
      for (int t = 3; t >= 1; --t) {
        const bool up = x > v[t - 1];
        const float va = v[t], vb = v[t - 1];
        v[t] = up ? vb : va;
        v[t - 1] = up ? va : vb;
        const uint32_t ia = ix[t], ib = ix[t - 1];
        ix[t] = up ? ib : ia;
        ix[t - 1] = up ? ia : ib;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) srt[bk * 4 + t] = rank_key_bits(__float_as_uint(v[t]), ix[t]);
  }
  __syncwarp();
  warp_bitonic_sort<uint64_t>(srt, 512, lane);
  for (uint32_t q = lane; q < K; q += 32) {
    ov[q] = __uint_as_float(key_value_bits(srt[q]));
    oi[q] = (uint32_t)srt[q];
  }
  __syncwarp();
}

template <int S, bool POS, int PF>
__device__ __forceinline__ void rg_hits_any(const uint2* p, const uint8_t* nxt, int Sx, uint32_t L2, uint32_t lane,
                                            uint2* stage, uint4* state, uint32_t& nan, uint2 (&pre)[2][kRgTile]) {
  if constexpr (S != 0) rg_hits<S, POS, PF>(p, nxt, L2, lane, stage, state, nan, pre);
  else rg_hits_rt<POS>(p, nxt, Sx, L2, lane, stage, state, nan, pre);
}

// S = stride-rows (n = 128 S <= 65536; 0 = a run-time argument), B = 128, K' = 4.  CPS CTAs of NW warps per SM;
// CTA c owns the rows [rows c / G, rows (c + 1) / G) and its warps pull them
// from a shared counter.  `pred` is the CTA's prediction (an ascending code;
// ~0 = none).
// The row's first two tiles (14 stride-rows), loaded ahead of the hit pass:
// the pass consumes them as its tiles 0 and 1, and rg_row_scale reads the
// row's scale from them.
template <int S>
__device__ __forceinline__ void rg_preload(const uint2* p, int Sx, uint2 (&pre)[2][kRgTile]) {
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int i = 0; i < kRgTile; ++i) {
      const int s = t * kRgTile + i;
      if (S != 0 ? s < S : s < Sx) pre[t][i] = rg_ldg(p + s * 32);
      else pre[t][i] = make_uint2(0xff80ff80u, 0xff80ff80u);
    }
}
// Scale statistic of a row: the mean of 128 log2 (= bf16 codes per octave) of
// the buckets' largest magnitudes over the first 14 stride-rows, x 16.  A row
// scaled by s moves it (and a positive K-th candidate level, in the same
// unit) by 128 log2 s; over i.i.d. normal rows it has sigma ~3.9 codes (the
// signed maximum has ~19: a bucket whose samples are all small or negative
// moves the mean by hundreds of codes).  Buckets holding an infinity (masked
// columns), a NaN or a subnormal do not count.  kRgNoScale = no bucket qualifies.
constexpr int kRgNoScale = 0x7fffffff;
// max(|a|, |b|) per half (the sign of the result is not used); NaN wins
__device__ __forceinline__ uint32_t rg_amax(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ int rg_row_scale(const uint2 (&pre)[2][kRgTile]) {
  uint32_t mx = pre[0][0].x, my = pre[0][0].y;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int i = 0; i < kRgTile; ++i) {
      if (t == 0 && i == 0) continue;
      mx = rg_amax(mx, pre[t][i].x);
      my = rg_amax(my, pre[t][i].y);
    }
  mx &= 0x7fff7fffu;
  my &= 0x7fff7fffu;
  const uint32_t c[4] = {mx & 0xffffu, mx >> 16, my & 0xffffu, my >> 16};
  float sum = 0.f;
  uint32_t cnt = 0;
#pragma unroll
  for (int h = 0; h < 4; ++h)
    if (c[h] < 0x7f80u && c[h] >= 0x0080u) {  // finite and normal
      sum += __log2f(__uint_as_float(c[h] << 16));
      cnt += 1u;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (cnt == 0u) return kRgNoScale;
  return __float2int_rn(__fdividef(sum * 2048.f, (float)cnt));
}
// a positive level's ascending code <-> 128 log2(value) x 16 (bf16 codes are piecewise linear in
// the logarithm: up to 11 codes off, which a row's scale would otherwise move in and out of)
__device__ __forceinline__ int rg_level_log(uint32_t code) {
  return __float2int_rn(__log2f(__uint_as_float((code & 0x7fffu) << 16)) * 2048.f);
}
__device__ __forceinline__ uint32_t rg_log_level(int l16) {  // rounds down
  const float v = exp2f((float)l16 * (1.f / 2048.f));
  return min(max(__float_as_uint(v) >> 16, 0x0080u), 0x7f7fu) | 0x8000u;
}

// Two predictions of a row's K-th candidate level, each with the spread it
// has shown over the CTA's rows so far: the running mean of the previous
// rows' levels (precise while the rows keep their scale: sigma ~2-3 codes on
// i.i.d. rows) and the row's own scale statistic plus the mean offset between
// level and statistic (sigma ~4.5 codes whatever the rows' scales do).  A row
// passes against the one with the smaller sigma, kRgSigmas of them below it
// (never less than the margin argument); an outlier row by the statistic
// takes the second.  The spreads are sums over the CTA's rows (the warps run
// in step, so a last-writer running value would see one update per 28 rows),
// started from the prologue's estimates as kRgPriorRows pseudo-rows and
// halved every kRgWindow rows.  Levels and offsets are summed relative to the
// first row's (float sums of small numbers), in codes.
constexpr float kRgSigmas = 5.2f;
constexpr float kRgLevelVar = 5.3f;   // codes^2: spread of the K-th level over i.i.d. rows (sigma 2.3)
constexpr float kRgStatVar = 15.f;    // codes^2: sampling noise of the scale statistic (sigma 3.9)
constexpr float kRgStableVar = 13.f;  // codes^2: 3 sigma of that variance's estimate over 28 rows
constexpr float kRgPriorRows = 8.f;
constexpr uint32_t kRgWindow = 512;
constexpr float kRgOutlier = 20.f;    // codes: statistic and running mean disagree
constexpr int kRgOffStep = 64 << 4;   // codes x 16: a row's offset counts within this of the first row's
constexpr int kRgLevStep = 127 << 4;  // and its level within this (the sums of squares stay below 2^32)

template <int S, int NW, int PF, int CPS>
__global__ void __launch_bounds__(32 * NW, CPS) row_reg_kernel(RgArgs a) {
  const int Sx = S ? S : (int)a.S;  // S = 0: the row length is a run-time argument
  const uint32_t n = 128u * (uint32_t)Sx;
  extern __shared__ __align__(128) uint8_t rg_smem[];
  __shared__ uint32_t queue;
  __shared__ volatile uint32_t pred;
  // the predictions' statistics (see kRgSigmas); tracked = the prologue produced the references
  __shared__ volatile uint32_t tracked;
  // rows of one scale (the statistic's spread over the warps' first rows is its sampling noise) pass
  // against the running mean alone and skip the statistic; the first failed prediction ends that
  __shared__ volatile uint32_t robust;
  __shared__ volatile int ref_l, ref_o;        // the first row's level (code x 16) and log level - statistic
  __shared__ volatile float var_l0, var_o0;    // prior variances, codes^2
  // rows, sum and sum of squares of (level - ref_l) and (log level - statistic - ref_o), x 16 and x 256:
  // integers, so that the updates are plain shared-memory adds (a float add is a compare-and-swap loop)
  __shared__ volatile uint32_t acc_n, acc_l2, acc_ns, acc_o2;
  __shared__ volatile int acc_l, acc_o;
  // what the rows read, refreshed from the sums every fourth row: the two margins, which prediction,
  // the statistic's offset (x 16), the outlier distance (x 16), the sigmas (statistics only)
  __shared__ volatile uint32_t d_mgp, d_mgo, d_by;
  __shared__ volatile int d_off;
  __shared__ volatile float d_out, d_sgp, d_sgo;
  auto derive = [&]() {
    const float n = (float)acc_n, sl = (float)acc_l * (1.f / 16.f), sl2 = (float)acc_l2 * (1.f / 256.f);
    const float ns = (float)acc_ns, so = (float)acc_o * (1.f / 16.f), so2 = (float)acc_o2 * (1.f / 256.f);
    const float var_l = (kRgPriorRows * var_l0 + fmaxf(sl2 - sl * sl * __frcp_rn(fmaxf(n, 1.f)), 0.f)) *
                        __frcp_rn(kRgPriorRows + n);
    const float var_o = (kRgPriorRows * var_o0 + fmaxf(so2 - so * so * __frcp_rn(fmaxf(ns, 1.f)), 0.f)) *
                        __frcp_rn(kRgPriorRows + ns);
    const float inv1 = __frcp_rn(1.f + ns);        // the first row's offset is one sample of the mean
    const float sg_p = sqrtf(var_l * 1.07f);       // the running mean itself carries ~a quarter sigma
    const float sg_o = sqrtf(var_o * (1.f + inv1));
    if ((threadIdx.x & 31) == 0) {
      d_mgp = max(a.margin, (uint32_t)fminf(ceilf(kRgSigmas * sg_p), 4096.f));
      d_mgo = max(a.margin, (uint32_t)fminf(ceilf(kRgSigmas * sg_o), 4096.f));
      d_by = sg_p <= sg_o ? 1u : 0u;
      d_off = ref_o + (int)(16.f * so * inv1);
      d_out = 16.f * fmaxf(kRgOutlier, 4.f * sg_o);
      d_sgp = sg_p;
      d_sgo = sg_o;
    }
  };
  __shared__ int scale0[32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.k;
  uint8_t* wsm = rg_smem + (size_t)wid * kRgWarpSmem;
  uint2* stage = reinterpret_cast<uint2*>(wsm);
  uint4* state = reinterpret_cast<uint4*>(wsm + kRgTile * 256);
  uint32_t* tmp = reinterpret_cast<uint32_t*>(wsm);     // the staging tile is dead after the pass
  const uint64_t r0 = a.rows * blockIdx.x / gridDim.x, r1 = a.rows * (blockIdx.x + 1) / gridDim.x;
  const uint32_t nrows = (uint32_t)(r1 - r0);
  if (threadIdx.x == 0) {
    queue = 0;
    pred = 0xffffffffu;
    tracked = 0;
    robust = 0;
    acc_n = acc_l2 = acc_ns = acc_o2 = 0;
    acc_l = acc_o = 0;
  }
  // ---- prologue: the first prediction from the CTA's first row.  Every warp
  // takes a share of its stride-rows (one DRAM round trip for the CTA instead
  // of a lone warp's latency-bound pass), the group maxima are combined in
  // shared memory and warp 0 bisects the guaranteed level (K-th largest group
  // maximum).  A NaN or -inf-heavy first row leaves no prediction.
  if (a.force == 0) {
    const uint2* p0 = reinterpret_cast<const uint2*>(a.in + r0 * n) + lane;
    // the scale statistic of the warps' first rows: row r0's pairs with the prediction, their spread
    // tells whether the rows keep their scale.  Loaded first, so that it shares the round trip of
    // the warp's share of row r0.
    uint2 pre0[2][kRgTile];
    rg_preload<S>(reinterpret_cast<const uint2*>(a.in + (r0 + min((uint32_t)wid, nrows ? nrows - 1 : 0u)) * n) + lane, Sx,
                  pre0);
    uint32_t pm[2][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      pm[0][g] = pm[1][g] = 0xff80ff80u;
      const int s1 = g == 3 ? Sx : (g + 1) * Sx / 4;
      for (int s = g * Sx / 4 + (int)wid; s < s1; s += NW) {
        const uint2 v = rg_ldg(p0 + s * 32);
        pm[0][g] = bmax_nan(pm[0][g], v.x);
        pm[1][g] = bmax_nan(pm[1][g], v.y);
      }
    }
    {
      const int c0 = rg_row_scale(pre0);
      if (lane == 0) scale0[wid] = c0;
    }
    uint32_t* part = reinterpret_cast<uint32_t*>(wsm);  // [8][32] per warp, in its staging tile
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int g = 0; g < 4; ++g) part[(4 * w + g) * 32 + lane] = pm[w][g];
    __syncthreads();
    if (wid < 8) {  // warp q folds word q of every warp's share
      uint32_t m = 0xff80ff80u;
      for (uint32_t w2 = 0; w2 < (uint32_t)NW; ++w2)
        m = bmax_nan(m, reinterpret_cast<const uint32_t*>(rg_smem + (size_t)w2 * kRgWarpSmem)[wid * 32 + lane]);
      part[256 + lane] = m;
    }
    __syncthreads();
    if (wid == 0) {
      uint32_t gm0[2][4];
#pragma unroll
      for (int w = 0; w < 2; ++w)
#pragma unroll
        for (int g = 0; g < 4; ++g)
          gm0[w][g] = reinterpret_cast<const uint32_t*>(rg_smem + (size_t)(4 * w + g) * kRgWarpSmem)[256 + lane];
      uint32_t cur = 0;
#pragma unroll 1
      for (int bit = 15; bit >= 0; --bit) {
        const uint32_t t = cur | (1u << bit);
        const uint32_t cg = __reduce_add_sync(0xffffffffu, rg_count_ge(gm0, rg_bits2(t)));
        if (cg >= K) cur = t;
      }
      const bool in = lane < (uint32_t)NW;
      const int c = in ? scale0[lane] : 0;
      // tracked only for positive levels (a negative level moves against the rows' scale)
      const bool stat = !__any_sync(0xffffffffu, in && c == kRgNoScale) && cur > 0x8080u;
      const int mean = (int)__reduce_add_sync(0xffffffffu, c) / NW;
      const int mad = (int)__reduce_add_sync(0xffffffffu, in ? abs(c - mean) : 0) / NW;
      if (cur > kRgKeyNegInf && lane == 0) {
        // the spread of the statistic over the warps' first rows, less its sampling noise, is the
        // rows' scale spread: it widens the running mean's expected error
        if (stat) {
          const float sc = (float)mad * (1.f / (0.8f * 16.f));
          ref_l = (int)(cur << 4);
          ref_o = rg_level_log(cur) - scale0[0];
          var_l0 = kRgLevelVar + fmaxf(sc * sc - kRgStatVar - 4.f, 0.f);  // less a sigma of the estimate
          var_o0 = kRgLevelVar + kRgStatVar;
          tracked = 1;
          robust = (a.robust == 1 || (a.robust == 0 && sc * sc - kRgStatVar > kRgStableVar)) ? 1u : 0u;
        }
        pred = cur << 4;
      }
      __syncwarp();
      if (tracked) derive();
    }
  }
  __syncthreads();

  auto pop = [&]() {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(&queue, 1u);
    return __shfl_sync(0xffffffffu, r, 0);
  };
  uint32_t rnext = pop();
#pragma unroll 1
  for (;;) {
    const uint32_t rr = rnext;
    if (rr >= nrows) break;
    rnext = pop();  // one row ahead: its first tiles are prefetched into L2 during this row
    const uint8_t* nxt = rnext < nrows ? reinterpret_cast<const uint8_t*>(a.in + (r0 + rnext) * n) : nullptr;
    const uint64_t row = r0 + rr;
    const uint16_t* xr = a.in + row * n;
    const uint2* p = reinterpret_cast<const uint2*>(xr) + lane;
    float* ov = a.out_v + row * K;
    uint32_t* oi = a.out_i + row * K;

    // ---- the hit pass against the prediction: Alg. 1 over the hits ---------
    auto clear_state = [&]() {
#pragma unroll
      for (int j = 0; j < 4; ++j) state[kRgLaneQ * lane + j] = make_uint4(0, 0, 0, 0);
    };
    // M = sum_b min(K', c_b) = the filled slots
    auto filled = [&]() {
      uint32_t f = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 sv = state[kRgLaneQ * lane + j];
        f += (sv.x ? 1u : 0u) + (sv.y ? 1u : 0u) + (sv.z ? 1u : 0u) + (sv.w ? 1u : 0u);
      }
      return __reduce_add_sync(0xffffffffu, f);
    };
    const uint32_t pr = pred;  // running mean of the rows' K-th candidate levels, x 16
    const bool have = pr != 0xffffffffu && a.force == 0;
    uint2 pre[2][kRgTile];
    rg_preload<S>(p, Sx, pre);
    // the level to pass against (see kRgSigmas)
    const bool trk = tracked != 0;
    const bool rb = trk && robust != 0;
    const int crow = rb ? rg_row_scale(pre) : kRgNoScale;
    bool by_pred = true, both = false;
    uint32_t mg = a.margin, mg_o = 0;
    int est = 0;  // the statistic's prediction, log level x 16
    if (trk) {
      mg = d_mgp;
      if (crow != kRgNoScale) {
        est = crow + d_off;
        mg_o = d_mgo;
        by_pred = d_by != 0;
        // rows that keep their scale, but this row's statistic says otherwise: the lower of the two
        both = by_pred && fabsf((float)((int)(rg_log_level(est) << 4) - (int)pr)) > d_out;
      }
    }
    uint32_t Lkey = max(pr >> 4, kRgKeyNegInf + 1 + mg) - mg;
    if (!by_pred || both) {
      const uint32_t Lo = rg_log_level(est - 16 * (int)mg_o);
      Lkey = by_pred ? min(Lkey, Lo) : Lo;
    }
    bool posmode = Lkey > 0x8000u;
    uint32_t M = 0, nan = 0;
    if (have) {
      clear_state();
      if (posmode) rg_hits_any<S, true, PF>(p, nxt, Sx, rg_bits2(Lkey), lane, stage, state, nan, pre);
      else rg_hits_any<S, false, PF>(p, nxt, Sx, rg_bits2(Lkey), lane, stage, state, nan, pre);
      M = filled();
    }
    if (a.probe == 1) {  // development: the pass alone (its results consumed)
      if (M == 0x12345u) oi[lane] = M;
      continue;
    }
    bool exact = a.force == 2;
    const bool twopass = M < K;
    if (twopass) {
      if (have && trk && a.robust != 2 && lane == 0) robust = 1;
      // ---- no usable prediction: the group maxima, the exact K-th largest of
      //      them (it guarantees M >= K), then the hit pass against it
      uint32_t gm[2][4];
#pragma unroll
      for (int w = 0; w < 2; ++w)
#pragma unroll
        for (int g = 0; g < 4; ++g) gm[w][g] = 0xff80ff80u;
      if constexpr (S != 0) rg_max<S>(p, gm);
      else rg_max_rt(p, Sx, gm);
      const uint32_t mm = bmax_nan(bmax_nan(bmax_nan(gm[0][0], gm[0][1]), bmax_nan(gm[0][2], gm[0][3])),
                                   bmax_nan(bmax_nan(gm[1][0], gm[1][1]), bmax_nan(gm[1][2], gm[1][3])));
      nan = ((mm & 0x7fffu) > 0x7f80u || ((mm >> 16) & 0x7fffu) > 0x7f80u) ? 1u : 0u;
      if (__reduce_or_sync(0xffffffffu, nan)) {  // the reference rejects the input
        if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
        continue;
      }
      uint32_t cur = 0;
#pragma unroll 1
      for (int bit = 15; bit >= 0; --bit) {
        const uint32_t t = cur | (1u << bit);
        const uint32_t cg = __reduce_add_sync(0xffffffffu, rg_count_ge(gm, rg_bits2(t)));
        if (cg >= K) cur = t;
      }
      Lkey = cur;
      if (Lkey <= kRgKeyNegInf) {
        exact = true;
      } else {
        posmode = Lkey > 0x8000u;
        clear_state();
        rg_preload<S>(p, Sx, pre);
        if (posmode) rg_hits_any<S, true, PF>(p, nxt, Sx, rg_bits2(Lkey), lane, stage, state, nan, pre);
        else rg_hits_any<S, false, PF>(p, nxt, Sx, rg_bits2(Lkey), lane, stage, state, nan, pre);
        M = filled();
      }
    }
    if (a.probe == 2) continue;
    if (exact) {
      __syncwarp();
      rg_exact(xr, Sx, lane, K, reinterpret_cast<uint64_t*>(wsm), ov, oi);  // tile | state: 4 KB
      continue;
    }
    __syncwarp();

    // ---- stage 2: the first K of the M >= K candidates -------------------
    // A bitonic sort of the 512 slots in registers (16 per lane: the lane's
    // own 4 buckets, each already in Alg. 1 order = ascending key).  Key =
    // (~code << 16) | position: ascending = output order (value descending,
    // index ascending, topk.cpp:30-39); an empty slot sorts last.
    uint32_t Lstar;
    {
      uint32_t k[16];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 sv = state[kRgLaneQ * lane + j];
        k[4 * j] = sv.x ^ 0xffff0000u;
        k[4 * j + 1] = sv.y ^ 0xffff0000u;
        k[4 * j + 2] = sv.z ^ 0xffff0000u;
        k[4 * j + 3] = sv.w ^ 0xffff0000u;
      }
      // every merge ascending: its first step pairs g with g ^ (size - 1) (two ascending runs
      // head to tail), the others g with g ^ dist; element g = 16 lane + i
#pragma unroll
      for (int size = 8; size <= 512; size <<= 1) {
        if (size <= 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int q = i ^ (size - 1);
            if (i < q) { const uint32_t x = k[i], y = k[q]; k[i] = min(x, y); k[q] = max(x, y); }
          }
        } else {
          const uint32_t lm = (uint32_t)(size >> 4) - 1u;
          const bool lower = (lane & (uint32_t)(size >> 5)) == 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t ya = __shfl_xor_sync(0xffffffffu, k[15 - i], lm);  // partner's 15 - i -> my i
            const uint32_t yb = __shfl_xor_sync(0xffffffffu, k[i], lm);       // partner's i -> my 15 - i
            k[i] = lower ? min(k[i], ya) : max(k[i], ya);
            k[15 - i] = lower ? min(k[15 - i], yb) : max(k[15 - i], yb);
          }
        }
#pragma unroll
        for (int dist = size >> 2; dist > 0; dist >>= 1) {
          if (dist >= 16) {
            const uint32_t ld = (uint32_t)dist >> 4;
            const bool lower = (lane & ld) == 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t y = __shfl_xor_sync(0xffffffffu, k[i], ld);
              k[i] = lower ? min(k[i], y) : max(k[i], y);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if ((i & dist) == 0) { const uint32_t x = k[i], y = k[i | dist]; k[i] = min(x, y); k[i | dist] = max(x, y); }
            }
          }
        }
      }
      // sorted element x = 16 lane + i goes to tq[(x / 16) * 20 + x % 16]: 80-byte lane stride
      // (16-byte stores without bank conflicts) over the dead staging tile and state
      __syncwarp();
      uint32_t* tq = tmp;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<uint4*>(tq)[kRgLaneQ * lane + q] = make_uint4(k[4 * q], k[4 * q + 1], k[4 * q + 2], k[4 * q + 3]);
      __syncwarp();
      auto sorted = [&](uint32_t x) { return tq[(x >> 4) * (4 * kRgLaneQ) + (x & 15u)]; };
      // a NaN element was a hit (unordered compare): as raw bits it sorts first
      if (posmode && ((~(sorted(0) >> 16)) & 0x7fffu) > 0x7f80u) nan = 1u;
      if (__reduce_or_sync(0xffffffffu, nan)) {  // the reference rejects the input
        if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
        continue;
      }
      if (a.probe == 9) {  // development: path statistics instead of results (out_i[0..1] zeroed by the caller)
        if (lane == 0) {
          atomicAdd(a.out_i, twopass ? 1u : 0u);
          atomicAdd(a.out_i + 1, M);
          atomicAdd(a.out_i + 2, by_pred ? 1u : 0u);
          atomicAdd(a.out_i + 3, by_pred ? mg : mg_o);
          atomicAdd(a.out_i + 4, (uint32_t)(16.f * d_sgp));
          atomicAdd(a.out_i + 5, (uint32_t)(16.f * d_sgo));
          atomicAdd(a.out_i + 6, rb ? 1u : 0u);
        }
      } else {
        for (uint32_t x = lane; x < K; x += 32) {
          const uint32_t key = sorted(x), code = ~(key >> 16) & 0xffffu;
          ov[x] = __uint_as_float((posmode ? code : code16_bits(code)) << 16);
          oi[x] = key & 0xffffu;
        }
      }
      const uint32_t ck = ~(sorted(K - 1) >> 16) & 0xffffu;  // the K-th candidate's level
      Lstar = posmode ? (ck | 0x8000u) : ck;
    }
    // the next rows' prediction (a racing update by another warp is as good)
    if (lane == 0) {
      const uint32_t pv = pred;
      const int ls = (int)(Lstar << 4);
      pred = pv == 0xffffffffu ? (uint32_t)ls : (uint32_t)((int)pv + ((ls - (int)pv) >> 2));
      if (rb) {
        const int dl = min(max(ls - ref_l, -kRgLevStep), kRgLevStep);
        atomicAdd(const_cast<int*>(&acc_l), dl);
        atomicAdd(const_cast<uint32_t*>(&acc_l2), (uint32_t)(dl * dl));
        atomicAdd(const_cast<uint32_t*>(&acc_n), 1u);
        if (crow != kRgNoScale && Lstar > 0x8080u) {
          const int dn = min(max(rg_level_log(Lstar) - crow - ref_o, -kRgOffStep), kRgOffStep);
          atomicAdd(const_cast<int*>(&acc_o), dn);
          atomicAdd(const_cast<uint32_t*>(&acc_o2), (uint32_t)(dn * dn));
          atomicAdd(const_cast<uint32_t*>(&acc_ns), 1u);
        }
        if (acc_n >= kRgWindow) {  // forget: racing updates lose a row or two
          acc_n = acc_n >> 1;
          acc_l = acc_l / 2;
          acc_l2 = acc_l2 >> 1;
          acc_ns = acc_ns >> 1;
          acc_o = acc_o / 2;
          acc_o2 = acc_o2 >> 1;
        }
      }
    }
    __syncwarp();
    if (rb && (acc_n & 3u) == 0u) derive();
  }
}

}  // namespace atkg
