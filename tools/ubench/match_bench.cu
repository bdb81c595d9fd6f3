// match.any / vote / shfl / atoms cost on sm_100a (development microbenchmark)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t seed) {
  __shared__ uint32_t sm[1024];
  uint32_t lane = threadIdx.x & 31, x = (threadIdx.x * 2654435761u + seed) >> 27, acc = 0;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) { uint32_t m = __match_any_sync(0xffffffffu, x); acc += __popc(m & ((1u << lane) - 1)); x = (x + m) & 31; }
    if (MODE == 1) { uint32_t m = __ballot_sync(0xffffffffu, x & 1); acc += m; x = (x + m + i) & 31; }
    if (MODE == 2) { uint32_t m = __shfl_sync(0xffffffffu, x, (lane + 1) & 31); acc += m; x = (x + m + i) & 31; }
    if (MODE == 3) { uint32_t m = atomicAdd(&sm[(threadIdx.x >> 5) * 32 + x], 1u); acc += m; x = (x + m + i) & 31; }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)((t1 - t0) / iters);
}
int main() {
  uint32_t* d; cudaMalloc(&d, 148 * 1024 * 4);
  const char* names[] = {"match.any", "ballot", "shfl", "atoms(spread 32)"};
  for (int warps : {1, 8, 28}) for (int mode = 0; mode < 4; ++mode) {
    uint32_t h = 0;
    auto run = [&](auto kern) { kern<<<148, warps * 32>>>(d, 2000, 12345u); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost); };
    if (mode == 0) run(k<0>); if (mode == 1) run(k<1>); if (mode == 2) run(k<2>); if (mode == 3) run(k<3>);
    printf("%-18s warps/SM=%2d  %u cycles per dependent iteration (per warp)\n", names[mode], warps, h);
  }
  return 0;
}
