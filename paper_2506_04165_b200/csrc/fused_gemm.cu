// fused_gemm.cu -- placeholder until the tcgen05 GEMM + stage-1 epilogue lands.
#include "../../include/atkg.h"
#include "host_common.hpp"

using namespace atkg;

extern "C" {
int atkg_fused_workspace_size(uint64_t, uint64_t, const atkg_params*, size_t* bytes) {
  *bytes = 0;
  return ATKG_OK;
}
int atkg_fused_gemm_top_k(const void*, const void*, uint64_t, uint64_t, const atkg_params*, float*, uint32_t*,
                          float*, void*, size_t, uint32_t*, void*) {
  return guarded([] { throw Unsupported("fused GEMM path not built yet"); });
}
int atkg_gemm_bf16(const void*, const void*, uint64_t, uint64_t, uint64_t, float*, void*) {
  return guarded([] { throw Unsupported("GEMM path not built yet"); });
}
}
