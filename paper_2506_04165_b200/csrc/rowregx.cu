// rowregx.cu -- host planner + launcher of row_regx_kernel (rowregx.cuh): the C3 K' sweep shapes
// with B K' = 1024 candidates (bf16 rows of 14336: K' = 2 / B = 512, K' = 4 / B = 256, K' = 8 / B = 128).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.hpp"
#include "rowregx.cuh"

namespace atkg {

namespace {

template <int S, int KP, int CPL, int NW>
void rx_launch(const RgPlan& rp, const RgArgs& a, cudaStream_t st) {
  auto kern = row_regx_kernel<S, KP, CPL, NW>;
  ensure_smem_fn(kern, rp.smem);
  kern<<<rp.grid, 32 * NW, rp.smem, st>>>(a);
  check_launch();
}

template <int S, int KP, int CPL>
void rx_dispatch(const RgPlan& rp, const RgArgs& a, cudaStream_t st) {
  switch (rp.warps) {
    case 16: rx_launch<S, KP, CPL, 16>(rp, a, st); break;
    case 20: rx_launch<S, KP, CPL, 20>(rp, a, st); break;
    case 24: rx_launch<S, KP, CPL, 24>(rp, a, st); break;
    default: rx_launch<S, KP, CPL, 28>(rp, a, st); break;
  }
}

}  // namespace

RgPlan plan_rowregx(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                    bool for_size) {
  RgPlan rp;
  if (!for_size && (!opt("rowregx", 1) || opt("short", 0) || opt("rowwarp", 0))) return rp;
  if (dtype != ATKG_BF16 || n != 14336) return rp;
  const bool big = kp == 2 && B == 1024;  // 2048 candidates: 64 slots per lane, 20 warps
  if (!((kp == 2 && B == 512) || (kp == 4 && B == 256) || (kp == 8 && B == 128) || big)) return rp;
  if (k > 1024 || reinterpret_cast<uintptr_t>(in) % 8 != 0) return rp;
  rp.S = (uint32_t)(n / B);
  const uint32_t w = (uint32_t)opt("rowregx_warps", big ? 20 : 28);
  rp.warps = w <= 16 ? 16 : w <= 20 || big ? 20 : w <= 24 ? 24 : 28;
  // the same for the three 1024-candidate shapes (K' CPL = 8)
  rp.smem = (size_t)rp.warps * (big ? rx_warp_smem<2, 8>() : rx_warp_smem<4, 2>());
  rp.grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(rows, (uint64_t)sm_count()));
  rp.ok = true;
  return rp;
}

void run_rowregx(const RgPlan& rp, const void* in, uint64_t rows, uint64_t B, uint32_t kp, uint32_t k, float* ov,
                 uint32_t* oi, uint32_t* status, cudaStream_t st) {
  RgArgs a{};
  a.in = static_cast<const uint16_t*>(in);
  a.rows = rows;
  a.S = rp.S;
  a.k = k;
  a.margin = (uint32_t)opt("rowreg_margin", 12);
  a.force = (uint32_t)opt("rowreg_force", 0);
  a.probe = 0;
  a.out_v = ov;
  a.out_i = oi;
  a.status = status;
  g_prof.bracket_begin(st);
  if (kp == 2 && B == 1024) {
    if (rp.warps == 16) rx_launch<14, 2, 8, 16>(rp, a, st);
    else rx_launch<14, 2, 8, 20>(rp, a, st);
  } else if (kp == 2) rx_dispatch<28, 2, 4>(rp, a, st);
  else if (kp == 4) rx_dispatch<56, 4, 2>(rp, a, st);
  else rx_dispatch<112, 8, 1>(rp, a, st);
  g_prof.bracket_end(st);
}

}  // namespace atkg
