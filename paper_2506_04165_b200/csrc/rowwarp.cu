// rowwarp.cu -- host planner + launcher of row_warp_kernel (rowwarp.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.hpp"
#include "rowwarp.cuh"

namespace atkg {

namespace {

// the instantiated (K', chunk columns per lane, mask words) combinations:
// registers hold K' group keys and W mask words for each of the 4 CPL
// buckets a lane owns
constexpr bool rw_combo(uint32_t kp, uint32_t cpl, uint32_t w) {
  return (kp == 1 || kp == 2 || kp == 4 || kp == 8) && kp * cpl <= 8 &&
         ((cpl == 1 && w == 4) || (cpl == 2 && w == 2) || (cpl == 4 && w == 1) || (cpl == 1 && w == 2) ||
          (cpl == 1 && w == 1) || (cpl == 2 && w == 1));
}

template <int KP, int CPL, int W>
void rw_launch(const RwPlan& rp, const RwArgs& a, cudaStream_t st) {
  auto kern = row_warp_kernel<KP, CPL, W>;
  ensure_smem_fn(kern, rp.smem);
  kern<<<rp.grid, 32, rp.smem, st>>>(a);
  check_launch();
}

template <int KP>
void rw_dispatch_kp(const RwPlan& rp, const RwArgs& a, cudaStream_t st) {
  const uint32_t c = rp.cpl, w = rp.w;
  if (c == 1 && w == 4) rw_launch<KP, 1, 4>(rp, a, st);
  else if (c == 1 && w == 2) rw_launch<KP, 1, 2>(rp, a, st);
  else if (c == 1 && w == 1) rw_launch<KP, 1, 1>(rp, a, st);
  else if constexpr (KP <= 4) {
    if (c == 2 && w == 2) rw_launch<KP, 2, 2>(rp, a, st);
    else if (c == 2 && w == 1) rw_launch<KP, 2, 1>(rp, a, st);
    else if constexpr (KP <= 2) {
      if (c == 4 && w == 1) rw_launch<KP, 4, 1>(rp, a, st);
    }
  }
}

}  // namespace

RwPlan plan_rowwarp(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                    bool for_size) {
  RwPlan rp;
  if (!for_size && (opt("no_rowwarp", 0) || !opt("rowwarp", 0))) return rp;  // opt-in
  if (dtype != ATKG_BF16) return rp;
  if (B != 128 && B != 256 && B != 512) return rp;
  const uint64_t row_bytes = n * 2;
  if (n % B != 0 || row_bytes % 16 != 0 || row_bytes > 40 * 1024) return rp;
  if (reinterpret_cast<uintptr_t>(in) % 16 != 0) return rp;
  const uint64_t S = n / B;
  if (S < kp || S > 128) return rp;
  rp.cpl = (uint32_t)(B / 128);
  rp.w = S <= 32 ? 1 : S <= 64 ? 2 : 4;
  if (!rw_combo(kp, rp.cpl, rp.w)) return rp;
  uint64_t cap = 512;  // candidates: M <= B K'; i.i.d. rows ~1.4 K
  while (cap < std::min<uint64_t>(B * kp, 2 * (uint64_t)k + 256)) cap <<= 1;
  rp.cap = (uint32_t)cap;
  uint64_t P = 2;
  while (P < B * kp) P <<= 1;
  rp.P = (uint32_t)P;
  rp.slot_bytes = (uint32_t)align_up(std::max<uint64_t>(row_bytes, P * 8), 128);
  rp.sub_shift = 0;
  while ((n - 1) >> rp.sub_shift >= 4) ++rp.sub_shift;
  rp.smem = rw_smem_bytes(rp.slot_bytes, rp.cap);
  if (rp.smem > 100 * 1024) return rp;
  // CTAs (one warp each) per SM: as many as shared memory allows (<= 227 KB
  // per SM, 1 KB reserved per CTA)
  const uint64_t per_sm = std::min<uint64_t>(16, (227 * 1024) / (rp.smem + 1024 + 256));
  if (per_sm < 1) return rp;
  rp.grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(rows, (uint64_t)sm_count() * per_sm));
  rp.ws_bytes = (uint64_t)rp.grid * P * 8 + 256;
  rp.ok = true;
  return rp;
}

void run_rowwarp(const RwPlan& rp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                 float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st) {
  RwArgs a{};
  a.in = in;
  a.rows = rows;
  a.n = (uint32_t)n;
  a.S = (uint32_t)(n / B);
  a.k = k;
  a.cap = rp.cap;
  a.row_bytes = (uint32_t)(n * 2);
  a.slot_bytes = rp.slot_bytes;
  a.P = rp.P;
  a.sub_shift = rp.sub_shift;
  a.force_slow = (uint32_t)opt("rowwarp_force_slow", 0);
  a.probe = (uint32_t)opt("short_probe", 0);
  a.gws = static_cast<uint64_t*>(ws);
  a.out_v = ov;
  a.out_i = oi;
  a.status = status;
  g_prof.bracket_begin(st);
  switch (kp) {
    case 1: rw_dispatch_kp<1>(rp, a, st); break;
    case 2: rw_dispatch_kp<2>(rp, a, st); break;
    case 4: rw_dispatch_kp<4>(rp, a, st); break;
    default: rw_dispatch_kp<8>(rp, a, st); break;
  }
  g_prof.bracket_end(st);
}

}  // namespace atkg
