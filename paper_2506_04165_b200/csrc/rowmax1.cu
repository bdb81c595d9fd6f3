// rowmax1.cu -- host planner + launcher of row_max1_kernel (rowmax1.cuh): approx_top_k with K' = 1 for
// bf16 rows whose buckets hold 2, 4 or 8 elements (the C3 sweep baseline: B = 3584 and 7168).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.hpp"
#include "rowmax1.cuh"

namespace atkg {

namespace {

template <int S>
void rm_launch(const RmPlan& rp, const RmArgs& a, cudaStream_t st) {
  auto kern = row_max1_kernel<S, 28>;
  ensure_smem_fn(kern, rp.smem);
  kern<<<rp.grid, 32 * 28, rp.smem, st>>>(a);
  check_launch();
}

}  // namespace

RmPlan plan_rowmax1(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                    bool for_size) {
  RmPlan rp;
  if (!for_size && (!opt("rowmax1", 1) || opt("short", 0) || opt("rowwarp", 0))) return rp;
  if (dtype != ATKG_BF16 || kp != 1 || B % 128 != 0 || n % B != 0 || n > 65536) return rp;
  const uint64_t S = n / B;
  if (S != 2 && S != 4 && S != 8) return rp;
  if (k > 512 || k > B || reinterpret_cast<uintptr_t>(in) % 8 != 0) return rp;  // the log holds 1024 hits
  if (rows >= (1ull << 32)) return rp;  // the row list holds 32-bit row indices
  // the exact kernel for the rows left over must take the shape too
  rp.fallback = plan_short(dtype, in, rows, n, B, kp, k, true);
  if (!rp.fallback.ok || reinterpret_cast<uintptr_t>(in) % 16 != 0) return rp;
  rp.S = (uint32_t)S;
  rp.cpl = (uint32_t)(B / 128);
  rp.warps = 28;
  rp.smem = (size_t)rp.warps * kRmWarpSmem;
  rp.grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(rows, (uint64_t)sm_count()));
  rp.ws_bytes = align_up(rp.fallback.ws_bytes) + 256 + rows * 4;
  rp.ok = true;
  return rp;
}

void run_rowmax1(const RmPlan& rp, int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t k,
                 float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st) {
  char* w = static_cast<char*>(ws);
  uint32_t* count = reinterpret_cast<uint32_t*>(w + align_up(rp.fallback.ws_bytes));
  uint32_t* list = count + 64;
  CUDA_OK(cudaMemsetAsync(count, 0, 4, st));
  RmArgs a{};
  a.in = static_cast<const uint16_t*>(in);
  a.rows = rows;
  a.CPL = rp.cpl;
  a.k = k;
  a.margin = (uint32_t)opt("rowreg_margin", 12);
  a.force = (uint32_t)opt("rowmax1_force", 0);
  a.out_v = ov;
  a.out_i = oi;
  a.status = status;
  a.hard_count = count;
  a.hard_list = list;
  g_prof.bracket_begin(st);
  if (rp.S == 2) rm_launch<2>(rp, a, st);
  else if (rp.S == 4) rm_launch<4>(rp, a, st);
  else rm_launch<8>(rp, a, st);
  g_prof.bracket_end(st);
  // the rows it could not settle: the exact short-row kernel over the list (no work: it exits at once)
  run_short(dtype, rp.fallback, in, rows, n, B, 1, k, ov, oi, ws, status, st, list, count);
}

}  // namespace atkg
