// rowmax1.cuh -- approx_top_k with K' = 1 (the original two-stage algorithm,
// the baseline of the C3 K' sweep: B = 3584 and 7168 buckets of 4 and 2
// stride-rows) on the register row stream of rowreg.cuh.
//
// With K' = 1 a bucket's candidate is its maximum, at the LAST position that
// holds it (Alg. 1 with one slot, topk.cpp:80-102: `value >= v[0]` replaces).
// A bucket has only S = n / B <= 8 elements, so there is no state to keep:
// lane l owns the 4 buckets 4 (l + 32 k) + j of every chunk column k, loads
// the S stride-rows of a chunk column (8 bytes each, 256 B per warp load, the
// next chunk column in flight), takes the packed maximum and the last
// stride-row equal to it, compares the maximum with the level L and appends
// the hits (code << 16 | position) to its log.
//   * M = the number of hits = the candidates >= L.  M >= K: the top K of the
//     row's candidates are the top K of the hits (threshold argument of
//     rowreg.cuh with K' = 1: c_b is 0 or 1).
//   * The level is the CTA's running mean of the rows' K-th candidate minus a
//     margin; a warp without one bisects the maxima of a sample of the first
//     row's buckets.  M < K or a full log: the level moves and the pass
//     repeats (the row is in L2), at most 3 times.
//   * Rows that stay unsettled (ties across most buckets, -inf rows, NaN)
//     go to a list; short_row_kernel (shortrow.cuh) finishes them exactly.
//   * Stage 2: a bitonic sort of 32 log slots per lane in registers
//     (rowregx.cuh), the first K written in output order (topk.cpp:30-50).
#pragma once

#include "rowregx.cuh"

namespace atkg {

struct RmArgs {
  const uint16_t* in;
  uint64_t rows;
  uint32_t CPL;          // chunk columns per lane: B = 128 CPL
  uint32_t k;
  uint32_t margin;
  uint32_t force;        // tests: 1 = every row to the list (exact kernel)
  float* out_v;
  uint32_t* out_i;
  uint32_t* status;
  uint32_t* hard_count;  // rows left to the exact kernel (zeroed before the launch)
  uint32_t* hard_list;
};

constexpr uint32_t kRmLane = 36;                      // log words per lane: 32 + 16 bytes of padding (banks)
constexpr uint32_t kRmWarpSmem = kRmLane * 4 * 32;    // 4608 B per warp

// 0xffff in each half where the bf16 halves compare equal (false on NaN)
__device__ __forceinline__ uint32_t rm_eq(uint32_t a, uint32_t b) {
  uint32_t h;
  asm("set.eq.u32.bf16x2 %0, %1, %2;" : "=r"(h) : "r"(a), "r"(b));
  return h;
}

// One pass over the row against L2: the hits -> the lane's log; returns the
// lane's hit count (logged or not); nanacc collects the maxima (NaN-propagating).
template <int S, bool POS>
__device__ __forceinline__ uint32_t rm_pass(const uint2* p, uint32_t CPL, uint32_t L2, uint32_t lane, uint32_t* lg,
                                            uint32_t& nanacc) {
  const uint32_t B = 128u * CPL, rs = 32u * CPL;  // stride-row stride in 8-byte chunks
  uint32_t cnt = 0;
  auto load = [&](uint2 (&v)[S], uint32_t k) {
#pragma unroll
    for (int r = 0; r < S; ++r) v[r] = rg_ldg(p + k * 32 + r * rs);
  };
  auto process = [&](const uint2 (&v)[S], uint32_t k) {
    uint32_t mx = v[0].x, my = v[0].y;
#pragma unroll
    for (int r = 1; r < S; ++r) {
      mx = bmax_nan(mx, v[r].x);
      my = bmax_nan(my, v[r].y);
    }
    nanacc = bmax_nan(nanacc, bmax_nan(mx, my));
    const uint32_t hx = rg_geu1(mx, L2), hy = rg_geu1(my, L2);  // 0x3f80 per hit half
    if ((hx | hy) != 0) {
      // the last stride-row equal to the maximum, per half
      uint32_t rx = 0, ry = 0;
#pragma unroll
      for (int r = 1; r < S; ++r) {
        const uint32_t ex = rm_eq(v[r].x, mx), ey = rm_eq(v[r].y, my);
        rx = (ex & (uint32_t)(r * 0x00010001)) | (~ex & rx);
        ry = (ey & (uint32_t)(r * 0x00010001)) | (~ey & ry);
      }
      const uint32_t pb = 4 * (lane + 32 * k);
      auto put = [&](uint32_t hit, uint32_t val, uint32_t r, uint32_t j) {
        if (hit) {
          if (!POS) val = asc_code16(val);
          if (cnt < 32) lg[cnt] = (val << 16) | (r * B + pb + j);
          ++cnt;
        }
      };
      put(hx & 0xffffu, mx & 0xffffu, rx & 0xffffu, 0);
      put(hx >> 16, mx >> 16, rx >> 16, 1);
      put(hy & 0xffffu, my & 0xffffu, ry & 0xffffu, 2);
      put(hy >> 16, my >> 16, ry >> 16, 3);
    }
  };
  uint2 v0[S], v1[S];
  load(v0, 0);
#pragma unroll 1
  for (uint32_t k = 0; k < CPL; k += 2) {
    if (k + 1 < CPL) load(v1, k + 1);
    process(v0, k);
    if (k + 1 < CPL) {
      if (k + 2 < CPL) load(v0, k + 2);
      process(v1, k + 1);
    }
  }
  return cnt;
}

// S = stride-rows per bucket (2, 4 or 8); B = 128 CPL; n = B S <= 65536.
template <int S, int NW>
__global__ void __launch_bounds__(32 * NW, 1) row_max1_kernel(RmArgs a) {
  extern __shared__ __align__(128) uint8_t rm_smem[];
  __shared__ uint32_t queue;
  __shared__ volatile uint32_t pred;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.k, CPL = a.CPL, B = 128u * CPL, n = B * S;
  uint32_t* keys = reinterpret_cast<uint32_t*>(rm_smem + (size_t)wid * kRmWarpSmem);
  uint32_t* lg = keys + lane * kRmLane;
  const uint64_t r0 = a.rows * blockIdx.x / gridDim.x, r1 = a.rows * (blockIdx.x + 1) / gridDim.x;
  const uint32_t nrows = (uint32_t)(r1 - r0);
  if (threadIdx.x == 0) {
    queue = 0;
    pred = 0xffffffffu;
  }
  __syncthreads();
  auto pop = [&]() {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(&queue, 1u);
    return __shfl_sync(0xffffffffu, r, 0);
  };
#pragma unroll 1
  for (;;) {
    const uint32_t rr = pop();
    if (rr >= nrows) break;
    const uint64_t row = r0 + rr;
    const uint2* p = reinterpret_cast<const uint2*>(a.in + row * n) + lane;
    float* ov = a.out_v + row * K;
    uint32_t* oi = a.out_i + row * K;
    auto defer = [&]() {  // the exact kernel finishes this row
      if (lane == 0) a.hard_list[atomicAdd(a.hard_count, 1u)] = (uint32_t)row;
    };
    if (a.force == 1) { defer(); continue; }

    uint32_t pr = pred;  // running mean of the rows' K-th candidate levels, x 16
    uint32_t Lkey;
    if (pr == 0xffffffffu) {
      // no prediction yet: the maxima of the buckets of the lane's first chunk columns (up to 4:
      // 16 per lane, 512 per warp) and the level that leaves K x (their share of B) of them
      const uint32_t nk = min(CPL, 4u);
      uint32_t gm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) gm[i] = 0xff80ff80u;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if ((uint32_t)kk < nk) {
#pragma unroll
          for (int r = 0; r < S; ++r) {
            const uint2 v = rg_ldg(p + kk * 32 + r * 32 * CPL);
            gm[2 * kk] = bmax_nan(gm[2 * kk], v.x);
            gm[2 * kk + 1] = bmax_nan(gm[2 * kk + 1], v.y);
          }
        }
      }
      const uint32_t ks = max(1u, (K * nk + CPL - 1) / CPL);
      Lkey = rx_bisect<8>(gm, ks);
      Lkey = max(Lkey, kRgKeyNegInf + 1 + a.margin + 8) - a.margin - 8;
    } else {
      Lkey = max(pr >> 4, kRgKeyNegInf + 1 + a.margin) - a.margin;
    }
    // ---- the pass, repeated while the level does not settle the row --------
    uint32_t M = 0, cnt = 0, nan = 0;
    bool ok = false;
#pragma unroll 1
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      uint32_t nanacc = 0xff80ff80u;
      const uint32_t L2 = rg_bits2(Lkey);
      cnt = Lkey > 0x8000u ? rm_pass<S, true>(p, CPL, L2, lane, lg, nanacc)
                           : rm_pass<S, false>(p, CPL, L2, lane, lg, nanacc);
      nan = ((nanacc & 0x7fffu) > 0x7f80u || ((nanacc >> 16) & 0x7fffu) > 0x7f80u) ? 1u : 0u;
      if (__reduce_or_sync(0xffffffffu, nan)) break;
      M = __reduce_add_sync(0xffffffffu, cnt);
      const bool full = __reduce_max_sync(0xffffffffu, cnt) > 32u;
      if (M >= K && !full) {
        ok = true;
      } else if (full) {
        Lkey += 6u << attempt;  // too many hits for a lane's log: a higher level
      } else {
        const uint32_t down = 24u << (2 * attempt);  // too few: 24, 96, 384 codes lower
        if (Lkey <= kRgKeyNegInf + 1) break;
        Lkey = Lkey > kRgKeyNegInf + 1 + down ? Lkey - down : kRgKeyNegInf + 1;
      }
    }
    if (__reduce_or_sync(0xffffffffu, nan)) {  // the reference rejects the input
      if (lane == 0) atomicOr(a.status, ATKG_FLAG_NAN);
      continue;
    }
    if (!ok) { defer(); continue; }
    const bool posmode = Lkey > 0x8000u;
    // ---- stage 2: sort the 32 log slots per lane (unused slots sort last) ----
    uint32_t ks[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 e = reinterpret_cast<const uint4*>(lg)[q];
      ks[4 * q] = (uint32_t)(4 * q) < cnt ? e.x ^ 0xffff0000u : 0xffff0000u;
      ks[4 * q + 1] = (uint32_t)(4 * q + 1) < cnt ? e.y ^ 0xffff0000u : 0xffff0000u;
      ks[4 * q + 2] = (uint32_t)(4 * q + 2) < cnt ? e.z ^ 0xffff0000u : 0xffff0000u;
      ks[4 * q + 3] = (uint32_t)(4 * q + 3) < cnt ? e.w ^ 0xffff0000u : 0xffff0000u;
    }
    rx_sort<32, 1>(ks, lane);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q)
      reinterpret_cast<uint4*>(lg)[q] = make_uint4(ks[4 * q], ks[4 * q + 1], ks[4 * q + 2], ks[4 * q + 3]);
    __syncwarp();
    auto sorted = [&](uint32_t x) { return keys[(x >> 5) * kRmLane + (x & 31u)]; };
    for (uint32_t x = lane; x < K; x += 32) {
      const uint32_t key = sorted(x), code = ~(key >> 16) & 0xffffu;
      ov[x] = __uint_as_float((posmode ? code : code16_bits(code)) << 16);
      oi[x] = key & 0xffffu;
    }
    const uint32_t ck = ~(sorted(K - 1) >> 16) & 0xffffu;
    const uint32_t Lstar = posmode ? (ck | 0x8000u) : ck;
    if (lane == 0) {
      const uint32_t pv = pred;
      pred = pv == 0xffffffffu ? Lstar << 4 : (uint32_t)((int)pv + (((int)(Lstar << 4) - (int)pv) >> 2));
    }
    __syncwarp();
  }
}

}  // namespace atkg
