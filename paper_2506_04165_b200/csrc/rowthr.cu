// rowthr.cu -- host planner + launcher of row_threshold_kernel (rowthr.cuh),
// the approx_top_k path for rows that fit in shared memory.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "internal.hpp"
#include "rowthr.cuh"

namespace atkg {

namespace {

template <int KP, int B>
void launch(const ThrPlan& tp, const __nv_bfloat16* in, uint64_t rows, uint32_t n, uint32_t k, float* ov,
            uint32_t* oi, uint32_t* status, cudaStream_t st) {
  auto kern = row_threshold_kernel<KP, B>;
  ensure_smem_fn(kern, tp.smem);
  kern<<<(unsigned)rows, B, tp.smem, st>>>(in, n, k, tp.cap, tp.rsel, tp.region, ov, oi, status);
  check_launch();
}

}  // namespace

ThrPlan plan_rowthr(int dtype, const void* in, uint64_t n, uint64_t B, uint32_t kp, uint32_t k) {
  ThrPlan tp;
  if (opt("no_rowthr", 0)) return tp;
  if (dtype != ATKG_BF16 || (kp != 1 && kp != 2 && kp != 4 && kp != 8)) return tp;
  // measured on B200 (C3 shapes): the row threshold wins where the exact
  // per-bucket network of row_resident_kernel is long (K' = 8: 2x); at K' <= 4
  // that kernel is faster.  Option rowthr=1 forces this path (tests).
  if (kp < 8 && !opt("rowthr", 0)) return tp;
  const uint64_t row_bytes = n * 2;
  if (row_bytes > 64 * 1024 || row_bytes % 16 != 0 || reinterpret_cast<uintptr_t>(in) % 16 != 0) return tp;
  // one thread per (word column, row half): B threads
  if ((B != 64 && B != 128 && B != 256 && B != 512) || n % B != 0) return tp;
  const uint64_t nstr = n / B;
  if (nstr == 0 || nstr > 2ull * kThrHalf * kThrRPW) return tp;
  const uint64_t filled = std::min<uint64_t>(kp, nstr);
  uint64_t cap = 512;
  while (cap < filled * B) cap <<= 1;
  // row (the mask pass reads whole 16-row chunks) | keys | large-bucket marks
  // | their bucket ordinals | per-bucket offsets and counts; the row region
  // doubles as the counting-sort scratch once the row is dead
  const uint64_t rows16 = (nstr + kThrRPW - 1) / kThrRPW * kThrRPW * B * 2;
  const uint64_t scratch = (cap + 2ull * kThrNB + 8) * 4;
  tp.region = (uint32_t)align_up(std::max<uint64_t>(rows16, scratch), 128);
  tp.smem = tp.region + cap * 4 + kThrGCap * 4 + kThrGCap * 2 + 2 * B * 2;
  if (tp.smem > 200 * 1024) return tp;
  tp.cap = (uint32_t)cap;
  // rank r of the row threshold among the B bucket maxima sampled on every
  // 4th stride-row (each half starts on a multiple of 4), so that about
  // 1.7 K elements lie above it
  const uint64_t stride = nstr >= 16 ? 4 : 1;
  const double ns = (double)((nstr + stride - 1) / stride);
  const double q = std::min(1.0, 1.7 * (double)k / (double)n);
  const double frac = 1.0 - std::pow(1.0 - q, ns);
  const uint64_t r = (uint64_t)std::ceil((double)B * frac);
  tp.rsel = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(B, r));
  const uint64_t rr = opt("rowthr_r", 0);
  if (rr) tp.rsel = (uint32_t)std::min<uint64_t>(B, rr);
  tp.ok = true;
  return tp;
}

uint64_t rowthr_ws_bytes(uint64_t rows, const ThrPlan& tp) {
  (void)rows;
  (void)tp;
  return 0;
}

void run_rowthr(int dtype, const ThrPlan& tp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp,
                uint32_t k, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st) {
  (void)dtype;
  (void)ws;
  const auto* x = static_cast<const __nv_bfloat16*>(in);
  g_prof.bracket_begin(st);
#define ATKG_THR_B(KP_)                                                               \
  switch (B) {                                                                        \
    case 64: launch<KP_, 64>(tp, x, rows, (uint32_t)n, k, ov, oi, status, st); break;   \
    case 128: launch<KP_, 128>(tp, x, rows, (uint32_t)n, k, ov, oi, status, st); break; \
    case 256: launch<KP_, 256>(tp, x, rows, (uint32_t)n, k, ov, oi, status, st); break; \
    default: launch<KP_, 512>(tp, x, rows, (uint32_t)n, k, ov, oi, status, st); break;  \
  }
  switch (kp) {
    case 1: ATKG_THR_B(1) break;
    case 2: ATKG_THR_B(2) break;
    case 4: ATKG_THR_B(4) break;
    default: ATKG_THR_B(8) break;
  }
#undef ATKG_THR_B
  g_prof.bracket_end(st);
}

}  // namespace atkg
