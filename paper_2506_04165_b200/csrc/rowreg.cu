// rowreg.cu -- host planner + launcher of row_reg_kernel (rowreg.cuh), the
// approx_top_k path for short bf16 rows with B = 128, K' = 4 (config C3).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.hpp"
#include "rowreg.cuh"

namespace atkg {

namespace {

template <int S, int NW, int PF, int CPS>
void rg_launch(const RgPlan& rp, const RgArgs& a, cudaStream_t st) {
  auto kern = row_reg_kernel<S, NW, PF, CPS>;
  ensure_smem_fn(kern, rp.smem);
  kern<<<rp.grid, 32 * NW, rp.smem, st>>>(a);
  check_launch();
}

// rp.warps = warps per SM (one CTA): 29 / 33 = 28 / 32 warps with the loads issued one tile ahead
template <int S>
void rg_dispatch(const RgPlan& rp, const RgArgs& a, cudaStream_t st) {
  switch (rp.warps) {
    case 16: rg_launch<S, 16, 1, 1>(rp, a, st); break;
    case 20: rg_launch<S, 20, 1, 1>(rp, a, st); break;
    case 24: rg_launch<S, 24, 1, 1>(rp, a, st); break;
    case 29: rg_launch<S, 28, 1, 1>(rp, a, st); break;
    default: rg_launch<S, 32, 1, 1>(rp, a, st); break;
  }
}

}  // namespace

RgPlan plan_rowreg(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                   bool for_size) {
  RgPlan rp;
  // default for its shapes; the explicit opt-ins of the other row kernels win
  if (!for_size && (!opt("rowreg", 1) || opt("short", 0) || opt("rowwarp", 0))) return rp;
  if (dtype != ATKG_BF16 || B != 128 || kp != 4 || n % 128 != 0) return rp;
  const uint64_t S = n / 128;
  if (S < 8 || S > 512) return rp;  // positions are 16-bit; K' = 4 groups of >= 2 stride-rows
  if (k > kRgTmp || (uint64_t)k > B * kp) return rp;
  if (reinterpret_cast<uintptr_t>(in) % 8 != 0) return rp;
  rp.S = (uint32_t)S;
  // warps per CTA (= per SM); 29 / 33 = 28 / 32 warps with the loads issued one tile ahead
  // the unrolled instantiations run best at 28 warps with the loads one tile ahead (72 registers); the
  // run-time row length needs 96 registers to keep its addresses (20 warps: 71 us vs 84 us on the C3 shape)
  const bool unrolled = S == 112 || S == 128 || S == 56 || S == 28;
  const bool unrolled28 = S == 32 || S == 64 || S == 86 || S == 96 || S == 108;  // 28 warps only
  uint32_t w = (uint32_t)opt("rowreg_warps", 0);
  if (w == 0) {
    if (opt("rowreg_rt", 0) || (!unrolled && !unrolled28)) {
      w = 20;
    } else if (unrolled28) {
      w = 29;
    } else {
      // every warp runs whole rows one after the other and the kernel is issue-bound, so its time goes
      // with waves x warps: the warp count with the fewest idle warp-rows per SM (ties: more warps)
      const uint64_t rps = (rows + (uint64_t)sm_count() - 1) / (uint64_t)sm_count();
      uint64_t best = ~0ull;
      for (uint32_t c : {16u, 20u, 24u, 28u}) {
        const uint64_t cost = (rps + c - 1) / c * c;
        if (cost <= best) { best = cost; w = c; }
      }
      if (w == 28) w = 29;  // 28 warps: the loads one tile ahead fit in 72 registers
    }
  }
  rp.warps = w <= 16 ? 16 : w <= 20 ? 20 : w <= 24 ? 24 : w <= 29 ? 29 : 33;
  const uint32_t cps = 1;
  rp.smem = (size_t)(rp.warps == 29 ? 28 : rp.warps == 33 ? 32 : rp.warps) * kRgWarpSmem;
  rp.grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(rows, (uint64_t)sm_count() * cps));
  rp.ok = true;
  return rp;
}

void run_rowreg(const RgPlan& rp, const void* in, uint64_t rows, uint32_t k, float* ov, uint32_t* oi,
                uint32_t* status, cudaStream_t st) {
  RgArgs a{};
  a.in = static_cast<const uint16_t*>(in);
  a.rows = rows;
  a.S = rp.S;
  a.k = k;
  a.robust = (uint32_t)opt("rowreg_robust", 0);
  a.margin = (uint32_t)opt("rowreg_margin", 12);  // floor; the kernel widens it by the predictions' tracked spread
  a.force = (uint32_t)opt("rowreg_force", 0);
  a.probe = (uint32_t)opt("rowreg_probe", 0);
  a.out_v = ov;
  a.out_i = oi;
  a.status = status;
  g_prof.bracket_begin(st);
  // unrolled instantiations for the common row lengths, else the row length as a run-time argument
  const bool rt = opt("rowreg_rt", 0) != 0;
  if (rp.S == 112 && !rt) rg_dispatch<112>(rp, a, st);
  else if (rp.S == 128 && !rt) rg_dispatch<128>(rp, a, st);
  else if (rp.S == 56 && !rt) rg_dispatch<56>(rp, a, st);
  else if (rp.S == 28 && !rt) rg_dispatch<28>(rp, a, st);
  // other common FFN widths (4096, 8192, 11008, 12288, 13824): one unrolled instantiation each
  else if (rp.S == 32 && rp.warps == 29 && !rt) rg_launch<32, 28, 1, 1>(rp, a, st);
  else if (rp.S == 64 && rp.warps == 29 && !rt) rg_launch<64, 28, 1, 1>(rp, a, st);
  else if (rp.S == 86 && rp.warps == 29 && !rt) rg_launch<86, 28, 1, 1>(rp, a, st);
  else if (rp.S == 96 && rp.warps == 29 && !rt) rg_launch<96, 28, 1, 1>(rp, a, st);
  else if (rp.S == 108 && rp.warps == 29 && !rt) rg_launch<108, 28, 1, 1>(rp, a, st);
  else rg_dispatch<0>(rp, a, st);
  g_prof.bracket_end(st);
}

}  // namespace atkg
