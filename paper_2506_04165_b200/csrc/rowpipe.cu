// rowpipe.cu -- host planner + launcher of row_pipe_kernel (rowpipe.cuh), the
// approx_top_k path for bf16 rows that fit in shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "internal.hpp"
#include "rowpipe.cuh"

namespace atkg {

namespace {

uint64_t env_flag(const char* name) {
  const char* e = std::getenv(name);
  return e ? std::strtoull(e, nullptr, 10) : 0;
}

constexpr int kNG = 3;  // row groups per CTA (two row buffers each)

template <int KP, int B>
void launch(const PipePlan& pp, const PipeArgs& a, cudaStream_t st) {
  auto kern = row_pipe_kernel<KP, B, kNG>;
  static size_t attr = 0;
  if (attr < pp.smem) {
    CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.smem));
    attr = pp.smem;
  }
  kern<<<pp.grid, B * kNG, pp.smem, st>>>(a);
  check_launch();
}

}  // namespace

PipePlan plan_rowpipe(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k) {
  PipePlan pp;
  // measured on B200 (C3): 181 us vs 106 us for row_resident_kernel -- the
  // per-row phase chain is barrier/latency bound at 12 warps per SM; kept as
  // an opt-in path (ATKG_ROWPIPE=1) with its parity tests
  if (!env_flag("ATKG_ROWPIPE")) return pp;
  if (dtype != ATKG_BF16 || (kp != 1 && kp != 2 && kp != 4 && kp != 8)) return pp;
  if (B != 128 && B != 256) return pp;
  if (n % B != 0 || (n * 2) % 16 != 0 || reinterpret_cast<uintptr_t>(in) % 16 != 0) return pp;
  const uint64_t nstr = n / B;
  if (nstr < 16 || nstr > 2ull * kThrHalf * kThrRPW) return pp;
  const uint64_t filled = std::min<uint64_t>(kp, nstr);
  uint64_t cap = 512;
  while (cap < filled * B) cap <<= 1;
  pp.cap = (uint32_t)cap;
  pp.slot_bytes = (uint32_t)((nstr + kThrRPW - 1) / kThrRPW * kThrRPW * B * 2);
  pp.scr_words = (uint32_t)(2 * cap + 2 * kPipeNB + 1 + kPipeRed + 3) & ~3u;
  pp.smem = (size_t)kNG * 2 * pp.slot_bytes + (size_t)kNG * pp.scr_words * 4;
  if (pp.smem > 220 * 1024) return pp;
  // row threshold: about 1.7 K elements of a row above it (the sampled
  // maxima cover every 4th stride-row)
  const double ns = (double)((nstr + 3) / 4);
  const double q = std::min(1.0, 1.7 * (double)k / (double)n);
  const double frac = 1.0 - std::pow(1.0 - q, ns);
  pp.rsel = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(B, (uint64_t)std::ceil((double)B * frac)));
  pp.grid = (uint32_t)std::min<uint64_t>((uint64_t)sm_count(), (rows + kNG - 1) / kNG);
  pp.ok = true;
  return pp;
}

void run_rowpipe(const PipePlan& pp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                 float* ov, uint32_t* oi, uint32_t* status, cudaStream_t st) {
  PipeArgs a;
  a.in = static_cast<const __nv_bfloat16*>(in);
  a.rows = rows;
  a.n = (uint32_t)n;
  a.k = k;
  a.rsel = pp.rsel;
  a.cap = pp.cap;
  a.slot_bytes = pp.slot_bytes;
  a.scr_words = pp.scr_words;
  a.force_slow = (uint32_t)env_flag("ATKG_PIPE_FORCE_SLOW");
  a.out_v = ov;
  a.out_i = oi;
  a.status = status;
  g_prof.bracket_begin(st);
#define ATKG_PIPE_B(KP_)                                      \
  if (B == 128) launch<KP_, 128>(pp, a, st);                  \
  else launch<KP_, 256>(pp, a, st);
  switch (kp) {
    case 1: ATKG_PIPE_B(1) break;
    case 2: ATKG_PIPE_B(2) break;
    case 4: ATKG_PIPE_B(4) break;
    default: ATKG_PIPE_B(8) break;
  }
#undef ATKG_PIPE_B
  g_prof.bracket_end(st);
}

}  // namespace atkg
