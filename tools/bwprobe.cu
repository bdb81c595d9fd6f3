// bwprobe.cu -- read-bandwidth probe on B200 (development aid, not product).
// How many bytes in flight per SM does a pure streaming read need, and what
// read rate can LDG.128 / per-warp cp.async.bulk rings / a CTA-wide bulk ring
// reach?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwprobe bwprobe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2506_04165_b200/csrc/ptx.cuh"

using namespace atkg;

template <int U>
__global__ void __launch_bounds__(256) ldg_max(const float4* __restrict__ in, size_t n4, float* out) {
  float m = -1e30f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
  }
  for (; i < n4; i += stride) { float4 v = in[i]; m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w))); }
  if (m == 12345.f) out[0] = m;
}

// per-warp ring: lane 0 issues NS-1 slots ahead, all lanes read the slot
template <int NS, int SLOT>
__global__ void __launch_bounds__(256) warp_ring(const char* __restrict__ in, size_t bytes, int wpb, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[8][NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = sm + warp * NS * SLOT;
  uint64_t* bar = bars[warp];
  const size_t nw = (size_t)gridDim.x * wpb;
  const size_t w = (size_t)blockIdx.x * wpb + warp;
  const size_t chunks = bytes / SLOT;
  const size_t c0 = chunks * w / nw, c1 = chunks * (w + 1) / nw;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) ptx::mbar_init(&bar[s], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = ptx::policy_evict_first();
  if (lane == 0)
    for (int s = 0; s < NS - 1; ++s)
      if (c0 + s < c1) {
        ptx::mbar_arrive_expect_tx(&bar[s], SLOT);
        ptx::bulk_g2s(ring + s * SLOT, in + (c0 + s) * SLOT, SLOT, &bar[s], pol);
      }
  float m = -1e30f;
  for (size_t c = c0; c < c1; ++c) {
    const int s = (int)((c - c0) % NS);
    const uint32_t par = (uint32_t)(((c - c0) / NS) & 1);
    if (lane == 0) {
      const size_t cn = c + NS - 1;
      if (cn < c1) {
        const int sn = (int)((cn - c0) % NS);
        ptx::mbar_arrive_expect_tx(&bar[sn], SLOT);
        ptx::bulk_g2s(ring + sn * SLOT, in + cn * SLOT, SLOT, &bar[sn], pol);
      }
    }
    ptx::mbar_wait(&bar[s], par);
    const float4* p = reinterpret_cast<const float4*>(ring + s * SLOT);
#pragma unroll 4
    for (int q = lane; q < SLOT / 16; q += 32) {
      const float4 v = p[q];
      m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    __syncwarp();
  }
  if (m == 12345.f) out[0] = m;
}

// CTA ring: thread 0 produces, all warps consume every stage (full + empty barriers)
template <int NS, int SLOT>
__global__ void __launch_bounds__(256) cta_ring(const char* __restrict__ in, size_t bytes, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int nwarps = blockDim.x >> 5;
  const size_t chunks = bytes / SLOT;
  const size_t c0 = chunks * blockIdx.x / gridDim.x, c1 = chunks * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], nwarps); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = ptx::policy_evict_first();
  if (threadIdx.x == 0)
    for (int s = 0; s < NS; ++s)
      if (c0 + s < c1) {
        ptx::mbar_arrive_expect_tx(&full[s], SLOT);
        ptx::bulk_g2s(sm + s * SLOT, in + (c0 + s) * SLOT, SLOT, &full[s], pol);
      }
  float m = -1e30f;
  for (size_t c = c0; c < c1; ++c) {
    const int s = (int)((c - c0) % NS);
    const uint32_t par = (uint32_t)(((c - c0) / NS) & 1);
    ptx::mbar_wait(&full[s], par);
    const float4* p = reinterpret_cast<const float4*>(sm + s * SLOT);
#pragma unroll 4
    for (int q = threadIdx.x; q < SLOT / 16; q += blockDim.x) {
      const float4 v = p[q];
      m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && c + NS < c1) {
      ptx::mbar_wait(&empty[s], par);
      ptx::mbar_arrive_expect_tx(&full[s], SLOT);
      ptx::bulk_g2s(sm + s * SLOT, in + (c + NS) * SLOT, SLOT, &full[s], pol);
    }
  }
  if (m == 12345.f) out[0] = m;
}

template <typename F>
float timeit(F f, int iters = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / iters;
}

int main() {
  const size_t bytes = (size_t)1 << 30;
  char* d;
  float* out;
  cudaMalloc(&d, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(d, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms) { printf("%-40s %8.1f GB/s\n", name, bytes / ms / 1e6); };
  for (int k : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg U=4 ctas=%d x 256", sms * k);
    rep(nm, timeit([&] { ldg_max<4><<<sms * k, 256>>>((const float4*)d, bytes / 16, out); }));
    snprintf(nm, 64, "ldg U=8 ctas=%d x 256", sms * k);
    rep(nm, timeit([&] { ldg_max<8><<<sms * k, 256>>>((const float4*)d, bytes / 16, out); }));
  }
#define WR(NS, SLOT, WPB, CPS)                                                                           \
  {                                                                                                      \
    auto kern = warp_ring<NS, SLOT>;                                                                     \
    const int smem = WPB * NS * SLOT;                                                                    \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                      \
    char nm[96];                                                                                         \
    snprintf(nm, 96, "warp_ring NS=%d slot=%d wpb=%d cta/sm=%d (%dKB fly/SM)", NS, SLOT, WPB, CPS,       \
             (NS - 1) * SLOT * WPB * CPS / 1024);                                                        \
    rep(nm, timeit([&] { kern<<<sms * CPS, WPB * 32, smem>>>(d, bytes, WPB, out); }));                   \
    cudaError_t e = cudaGetLastError();                                                                  \
    if (e) printf("  err %s\n", cudaGetErrorString(e));                                                  \
  }
  WR(3, 4096, 8, 1) WR(3, 4096, 4, 2) WR(4, 4096, 8, 1) WR(4, 8192, 4, 1) WR(4, 8192, 8, 1) WR(3, 8192, 8, 1)
  WR(6, 4096, 8, 1) WR(5, 8192, 5, 1) WR(3, 16384, 4, 1) WR(4, 16384, 3, 1) WR(2, 16384, 6, 1)
  WR(8, 2048, 8, 1) WR(6, 2048, 8, 2)
#define CR_(NS, SLOT, TH, CPS)                                                                            \
  {                                                                                                      \
    auto kern = cta_ring<NS, SLOT>;                                                                      \
    const int smem = NS * SLOT;                                                                          \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                      \
    char nm[96];                                                                                         \
    snprintf(nm, 96, "cta_ring NS=%d slot=%d thr=%d cta/sm=%d (%dKB ring/SM)", NS, SLOT, TH, CPS,       \
             NS * SLOT * CPS / 1024);                                                                    \
    rep(nm, timeit([&] { kern<<<sms * CPS, TH, smem>>>(d, bytes, out); }));                              \
    cudaError_t e = cudaGetLastError();                                                                  \
    if (e) printf("  err %s\n", cudaGetErrorString(e));                                                  \
  }
  CR_(4, 16384, 256, 1) CR_(6, 16384, 256, 1) CR_(8, 16384, 256, 1) CR_(12, 16384, 256, 1)
  CR_(6, 32768, 256, 1) CR_(4, 32768, 256, 1) CR_(4, 16384, 128, 2) CR_(6, 16384, 128, 2) CR_(3, 32768, 128, 2)
  CR_(8, 8192, 256, 1) CR_(12, 8192, 128, 2)
  return 0;
}
