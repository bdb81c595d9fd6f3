// shortrow.cu -- host planner + launcher of short_row_kernel (shortrow.cuh),
// the approx_top_k path for bf16 rows that fit in shared memory.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.hpp"
#include "shortrow.cuh"

namespace atkg {

namespace {

// resident CTAs per SM (memoised per device, K' and shared-memory size: the
// planner runs on every call)
template <int KP>
bool sr_fit(SrPlan& sp) {
  if (sp.smem > 220 * 1024) return false;
  struct Ent {
    int dev;
    size_t smem;
    int occ;
  };
  thread_local Ent memo[8] = {};
  thread_local int next = 0;
  const int dev = current_device();
  int occ = -1;
  for (const Ent& e : memo)
    if (e.smem == sp.smem && e.dev == dev && e.occ >= 0 && e.smem) occ = e.occ;
  if (occ < 0) {
    auto kern = short_row_kernel<KP>;
    ensure_smem_fn(kern, sp.smem);
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kSrThreads, sp.smem));
    memo[next] = Ent{dev, sp.smem, occ};
    next = (next + 1) % 8;
  }
  sp.per_sm = (uint32_t)std::min(occ, 4);
  return occ > 0;
}

template <int KP>
void sr_launch(const SrPlan& sp, const SrArgs& a, cudaStream_t st) {
  auto kern = short_row_kernel<KP>;
  ensure_smem_fn(kern, sp.smem);
  kern<<<sp.grid, kSrThreads, sp.smem, st>>>(a);
  check_launch();
}

}  // namespace

SrPlan plan_short(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                  bool for_size) {
  SrPlan sp;
  if (!for_size && opt("no_short", 0)) return sp;
  if (dtype != ATKG_BF16 || (kp != 1 && kp != 2 && kp != 4 && kp != 8)) return sp;
  const uint64_t row_bytes = n * 2;
  // rows that fit a shared-memory slot twice over, 16-byte aligned for TMA
  if (row_bytes > 64 * 1024 || row_bytes % 16 != 0) return sp;
  if (reinterpret_cast<uintptr_t>(in) % 16 != 0) return sp;
  if (B % 4 != 0 || n % B != 0) return sp;
  const uint64_t S = n / B;
  if (S < kp) return sp;  // fewer stride-rows than K': every element is a candidate
  // parts of <= 32 stride-rows per group, more of them while the units do
  // not cover the CTA
  const uint64_t gl = (S + kp - 1) / kp;
  uint64_t npart = (gl + 31) / 32;
  while ((B / 4) * kp * npart < (uint64_t)kSrThreads && npart * 2 <= gl && kp * npart * 2 <= kSrMaxWords) npart *= 2;
  if (kp * npart > kSrMaxWords) return sp;
  sp.npart = (uint32_t)npart;
  sp.pl = (uint32_t)((gl + npart - 1) / npart);
  // candidates: M <= B * K'; i.i.d. rows give ~1.4 K, rows with more (heavy
  // ties at L) take the exact path
  uint64_t cap = 512;
  while (cap < std::min<uint64_t>(B * kp, 2 * (uint64_t)k + 256)) cap <<= 1;
  if (cap > 65536) return sp;
  sp.cap = (uint32_t)cap;
  uint64_t P = 2;
  while (P < B * kp) P <<= 1;
  sp.P = (uint32_t)P;
  // stage-2 scratch in the dead row slot: keys[2 cap] | emit scratch
  sp.slot_bytes = (uint32_t)align_up(std::max<uint64_t>(row_bytes, (2 * cap + 2 * kThrNB + 64) * 4), 128);
  sp.sub_shift = 0;
  while ((n - 1) >> sp.sub_shift >= 4) ++sp.sub_shift;
  sp.smem = sr_smem_bytes(sp.slot_bytes, sp.cap, kp, sp.npart, (uint32_t)B);
  bool fit = false;
  switch (kp) {
    case 1: fit = sr_fit<1>(sp); break;
    case 2: fit = sr_fit<2>(sp); break;
    case 4: fit = sr_fit<4>(sp); break;
    default: fit = sr_fit<8>(sp); break;
  }
  if (!fit) return sp;
  sp.grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(rows, (uint64_t)sm_count() * sp.per_sm));
  sp.ws_bytes = (uint64_t)sp.grid * P * 8 + 256;
  sp.ok = true;
  return sp;
}

void run_short(int dtype, const SrPlan& sp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp,
               uint32_t k, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st,
               const uint32_t* row_list, const uint32_t* row_count) {
  (void)dtype;
  SrArgs a{};
  a.in = in;
  a.rows = rows;
  a.n = (uint32_t)n;
  a.B = (uint32_t)B;
  a.S = (uint32_t)(n / B);
  a.k = k;
  a.cps = (uint32_t)(B / 4);
  a.npart = sp.npart;
  a.pl = sp.pl;
  a.cap = sp.cap;
  a.slot_bytes = sp.slot_bytes;
  a.row_bytes = (uint32_t)(n * 2);
  a.P = sp.P;
  a.sub_shift = sp.sub_shift;
  a.force_slow = (uint32_t)opt("short_force_slow", 0);
  a.probe = (uint32_t)opt("short_probe", 0);
  a.gws = static_cast<uint64_t*>(ws);
  a.row_list = row_list;
  a.row_count = row_count;
  a.out_v = ov;
  a.out_i = oi;
  a.status = status;
  g_prof.bracket_begin(st);
  switch (kp) {
    case 1: sr_launch<1>(sp, a, st); break;
    case 2: sr_launch<2>(sp, a, st); break;
    case 4: sr_launch<4>(sp, a, st); break;
    default: sr_launch<8>(sp, a, st); break;
  }
  g_prof.bracket_end(st);
}

}  // namespace atkg
