// mips.cu -- fp32 MIPS scoring for the mips_unfused / mips_fused mirror.
//
// score_block (mips.cpp:57-91): out[q, c] = sum_j queries[q, j] * database[c, j],
// one fp32 accumulator from 0, j ascending, multiply and add rounded
// separately (the reference builds with -ffp-contract=off).  Columns
// [n, n_padded) get -inf (mips.cpp:112).  The kernel keeps that exact order
// per output, so the scores -- and every top-k built on them -- are
// bit-identical to the reference.  128x128 output tiles staged through shared
// memory in 16-wide slices of the dimension; 8x8 outputs per thread.
//
// The bf16 tcgen05 path with stage 1 in the epilogue is atkg_fused_gemm_top_k
// (fused_gemm.cu); this one is the fp32 reference-exact scorer.
#include <cuda_runtime.h>

#include "internal.hpp"

namespace atkg {
namespace {

constexpr int kTile = 128, kSlice = 16, kPer = 8;  // 128x128 tile, 8x8 outputs per thread

__global__ void __launch_bounds__(256, 2) mips_score_kernel(const float* __restrict__ q, uint64_t b,
                                                            const float* __restrict__ db, uint64_t n,
                                                            uint64_t d, float* __restrict__ out,
                                                            uint64_t stride, uint64_t n_padded) {
  // two slice buffers: the global loads of slice s+1 are in flight (registers)
  // while slice s is multiplied out of shared memory
  __shared__ __align__(16) float qs[2][kSlice][kTile + 4];  // +4: the transposing stores hit 16 banks, not 2
  __shared__ __align__(16) float ws[2][kSlice][kTile + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const uint64_t q0 = uint64_t(blockIdx.y) * kTile, c0 = uint64_t(blockIdx.x) * kTile;
  constexpr int kLoads = kTile * kSlice / 256;
  float pq[kLoads], pw[kLoads];
  auto fetch = [&](uint64_t j0) {
#pragma unroll
    for (int l = 0; l < kLoads; ++l) {
      const int e = threadIdx.x + l * 256, r = e / kSlice, j = e % kSlice;
      const uint64_t qq = q0 + r, cc = c0 + r, jj = j0 + j;
      pq[l] = (qq < b && jj < d) ? __ldg(q + qq * d + jj) : 0.0f;
      pw[l] = (cc < n && jj < d) ? __ldg(db + cc * d + jj) : 0.0f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int l = 0; l < kLoads; ++l) {
      const int e = threadIdx.x + l * 256, r = e / kSlice, j = e % kSlice;
      qs[buf][j][r] = pq[l];
      ws[buf][j][r] = pw[l];
    }
  };
  float acc[kPer][kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i)
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[i][j] = 0.0f;
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (uint64_t j0 = 0; j0 < d; j0 += kSlice, buf ^= 1) {
    const bool more = j0 + kSlice < d;
    if (more) fetch(j0 + kSlice);
    const int jn = static_cast<int>(d - j0 < uint64_t(kSlice) ? d - j0 : kSlice);
    for (int j = 0; j < jn; ++j) {
      float a[kPer], w[kPer];
      const float4 a0 = *reinterpret_cast<const float4*>(&qs[buf][j][ty * kPer]);
      const float4 a1 = *reinterpret_cast<const float4*>(&qs[buf][j][ty * kPer + 4]);
      const float4 w0 = *reinterpret_cast<const float4*>(&ws[buf][j][tx * kPer]);
      const float4 w1 = *reinterpret_cast<const float4*>(&ws[buf][j][tx * kPer + 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w; w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
#pragma unroll
      for (int i = 0; i < kPer; ++i)
#pragma unroll
        for (int k = 0; k < kPer; ++k) acc[i][k] = __fadd_rn(acc[i][k], __fmul_rn(a[i], w[k]));
    }
    if (more) stash(buf ^ 1);  // the other buffer was last read before the previous barrier
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const uint64_t qq = q0 + ty * kPer + i;
    if (qq >= b) continue;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint64_t cc = c0 + tx * kPer + k;
      if (cc < n)
        out[qq * stride + cc] = acc[i][k];
      else if (cc < n_padded)
        out[qq * stride + cc] = -__int_as_float(0x7f800000);
    }
  }
}

}  // namespace
}  // namespace atkg

using namespace atkg;

extern "C" int atkg_mips_score(const float* d_queries, uint64_t b, const float* d_database, uint64_t n,
                               uint64_t d, float* d_out, uint64_t out_stride, uint64_t n_padded,
                               void* stream) {
  return guarded([&] {
    if (d == 0) throw Inval("mips: dims must be >= 1");
    if (n == 0) throw Inval("mips: database must not be empty");
    if (b == 0) throw Inval("mips: queries must not be empty");
    if (n_padded < n || out_stride < n_padded) throw Inval("mips: out_stride >= n_padded >= n required");
    if (!d_queries || !d_database || !d_out) throw Inval("mips: null buffer");
    const uint64_t gx = (n_padded + kTile - 1) / kTile, gy = (b + kTile - 1) / kTile;
    if (gx > 0x7fffffffull || gy > 65535) throw Unsupported("mips: shape exceeds the launch grid");
    mips_score_kernel<<<dim3(unsigned(gx), unsigned(gy)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_queries, b, d_database, n, d, d_out, out_stride, n_padded);
    check_launch();
  });
}
