// streamthr.cu -- host planner + launchers of the threshold-stream
// approx_top_k (streamthr.cuh) for long rows.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "internal.hpp"
#include "streamthr.cuh"

namespace atkg {

namespace {

// E[min(K', X)], X ~ Poisson(lambda)
double mean_min_poisson(double lambda, uint32_t kp) {
  double p = std::exp(-lambda), cdf = 0.0, m = 0.0;
  for (uint32_t j = 0; j < kp; ++j) {
    m += j * p;
    cdf += p;
    p *= lambda / (j + 1);
  }
  return m + kp * (1.0 - cdf);
}

// programmatic dependent launch: the kernel may start while the previous one
// on the stream drains; it synchronises with griddepcontrol.wait before
// touching what the previous kernel reads or writes
template <typename K, typename A>
void launch_pdl(K kern, unsigned grid, unsigned block, size_t smem, cudaStream_t st, const A& args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = opt("no_pdl", 0) ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, kern, args));
  check_launch();
}

template <typename T, int UNR>
void launch_stream(const StPlan& sp, const StArgs& a, cudaStream_t st) {
  auto kern = st_stream_kernel<T, UNR>;
  ensure_smem_fn(kern, sp.smem_stream);
  launch_pdl(kern, sp.G, kStNW * 32, sp.smem_stream, st, a);
}

template <typename T, int KP>
void launch_finish(const StPlan& sp, uint64_t rows, const StFinArgs& a, cudaStream_t st) {
  auto kern = st_finish_kernel<T, KP>;
  ensure_smem_fn(kern, sp.smem_fin);
  // a few rows (the giant row): one CTA per row is latency-bound, so give it
  // 32 warps; many rows: 8 warps per row, several rows per SM
  const unsigned threads = rows < 64 ? 1024u : (unsigned)opt("st_fin_threads", 256);
  launch_pdl(kern, (unsigned)rows, threads, sp.smem_fin, st, a);
}

}  // namespace

// target count T of row elements >= L: B * E[min(K', Poisson(T/B))] must
// clear K with margin
double streamthr_target(uint64_t n, uint64_t B, uint32_t kp, uint32_t k) {
  const double need = 1.2 * k + 4.0 * std::sqrt((double)k) + 8.0;
  thread_local uint64_t t_n = 0, t_B = 0, t_kp = 0, t_k = 0;
  thread_local double t_T = 1.0;
  if (t_n != n || t_B != B || t_kp != kp || t_k != k) {
    double T0 = 1.0;
    while (T0 < (double)n && (double)B * mean_min_poisson(T0 / (double)B, kp) < need) T0 *= 1.05;
    t_n = n; t_B = B; t_kp = kp; t_k = k; t_T = T0;
  }
  return t_T;
}

StPlan plan_streamthr(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                      bool for_size, double t_scale) {
  StPlan sp;
  if (!for_size && opt("no_streamthr", 0)) return sp;
  if (kp != 1 && kp != 2 && kp != 4 && kp != 8) return sp;
  // Many rows with a large K: the per-row finish (rebuild + rank of >= K
  // survivors) outweighs the stream's saving over the exact grid stage 1 +
  // stage 2 (MIPS shape 1024 x 1,000,448, K = 1024, B = 1024, K' = 4:
  // 13.6 -> 6.2 ms per batch after the tcgen05 GEMM).  Sizing keeps the
  // stream's workspace either way.
  if (!for_size && k >= 1024 && rows >= opt("streamthr_bigk_rows", 64)) return sp;
  const uint64_t es = dtype == ATKG_BF16 ? 2 : 4;
  const uint64_t ve = 16 / es;
  if (n < opt("streamthr_min_n", 32768) || n % ve != 0) return sp;
  // rows beyond 2^24 elements (the giant row) do not take the in-kernel exact
  // fallback; a failed row is flagged and rerun on the exact path by the host
  sp.giant = n > opt("st_giant_n", 1ull << 24);
  if (n > 0xffffffffull) return sp;
  if (reinterpret_cast<uintptr_t>(in) % 16 != 0) return sp;
  const uint64_t filled = std::min<uint64_t>(kp, n / B);
  if (B > 4096 || B * filled > 8192 || k > B * filled) return sp;
  sp.vtot = rows * n / ve;
  if (sp.vtot >= (1ull << 50)) return sp;
  if (sp.vtot / std::max<uint64_t>(1, (uint64_t)sm_count()) >= (1ull << 31)) return sp;  // 32-bit piece offsets
  // bytes per CTA step = kStNW warps x 32 lanes x UNR 16-byte vectors, UNR in {4, 8}
  sp.slot_bytes = (uint32_t)opt("st_step", (uint64_t)kStNW * 4096);
  if (sp.slot_bytes != (uint32_t)kStNW * 2048 && sp.slot_bytes != (uint32_t)kStNW * 4096) return sp;
  sp.ns = 0;
  const uint64_t per_sm = opt("st_ctas", 16 / kStNW);
  uint64_t G = (uint64_t)sm_count() * per_sm;
  G = std::max<uint64_t>(1, std::min<uint64_t>(G, sp.vtot / 1024));
  sp.psz = (sp.vtot + G - 1) / G;
  sp.G = (uint32_t)((sp.vtot + sp.psz - 1) / sp.psz);
  // rows spanned by any piece
  const uint64_t nvrow = n / ve;
  // (memoised: the planner runs on every call)
  thread_local uint64_t m_vtot = 0, m_psz = 0, m_nvrow = 0, m_smax = 1;
  if (m_vtot != sp.vtot || m_psz != sp.psz || m_nvrow != nvrow) {
    uint64_t smax = 1;
    for (uint32_t c = 0; c < sp.G; ++c) {
      const uint64_t v0 = st_piece_start(sp.vtot, sp.psz, c), v1 = st_piece_start(sp.vtot, sp.psz, c + 1);
      if (v1 > v0) smax = std::max<uint64_t>(smax, (v1 - 1) / nvrow - v0 / nvrow + 1);
    }
    m_vtot = sp.vtot; m_psz = sp.psz; m_nvrow = nvrow; m_smax = smax;
  }
  sp.smax = (uint32_t)m_smax;
  // every warp sub-stream keeps ~2x its share of the target T (a slice of a
  // sharded row: t_scale = its share of the row's target)
  const double T = std::max(8.0, streamthr_target(n, B, kp, k) * t_scale);
  sp.rfac = (float)(2.0 * T / (double)n);
  sp.lfac = (float)(T / 1.5 / (double)n);
  // rows cut into many pieces (the giant row): cap each slot at ~3x its share
  // of T, else the row threshold (max over the slots) gathers too much;
  // rows over a few pieces never need it (a slot holds <= 8 * kStWarpCap)
  sp.cfac = (n / ve > 8 * sp.psz) ? (float)(3.0 * T / (double)n) : 1e30f;
  // gathered entries per row: ~T, but up to ~2.4 per warp sub-stream when a
  // few rows are cut into many pieces (the max of many sub-stream thresholds)
  uint64_t ecap = rows >= 64 ? 4096 : 8192;
  while (ecap < B * filled) ecap <<= 1;
  sp.ecap = (uint32_t)ecap;
  sp.smem_stream = (size_t)kStNW * 2 * kStLog * 4 + (size_t)kStSlots * sp.slot_bytes;  // logs | per-warp rings
  sp.smem_fin = (size_t)ecap * 16 + (size_t)B * 12;
  if (sp.smem_stream > 220 * 1024 || sp.smem_fin > 220 * 1024) return sp;
  if (sp.G > kStMaxRowPieces) return sp;
  sp.ws_bytes = (uint64_t)sp.G * sp.smax * kStSlotWords * 4 + 256;  // slots | gate
  sp.ok = true;
  return sp;
}

void run_streamthr(int dtype, const StPlan& sp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp,
                   uint32_t k, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st) {
  StArgs a;
  a.in = in;
  a.n = n;
  a.vtot = sp.vtot;
  a.psz = sp.psz;
  a.G = sp.G;
  a.smax = sp.smax;
  a.slot_bytes = sp.slot_bytes;
  a.ns = sp.ns;
  a.rfac = sp.rfac;
  a.lfac = sp.lfac;
  a.cfac = sp.cfac;
  a.warp_sample = (uint32_t)opt("st_warp_sample", 0);
  a.slots = static_cast<uint32_t*>(ws);
  uint32_t* gate = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + (sp.ws_bytes - 256));
  a.gate = sp.giant ? gate : nullptr;
  a.status = status;
  StFinArgs f;
  f.in = in;
  f.n = n;
  f.vtot = sp.vtot;
  f.psz = sp.psz;
  f.G = sp.G;
  f.smax = sp.smax;
  f.B = (uint32_t)B;
  f.k = k;
  f.slot_cap = kStSlotCap;
  f.ecap = sp.ecap;
  f.slots = static_cast<const uint32_t*>(ws);
  f.out_v = ov;
  f.out_i = oi;
  f.status = status;
  f.force_slow = (uint32_t)opt("st_force_slow", 0);
  f.gate = a.gate;
  g_prof.bracket_begin(st);
  if (dtype == ATKG_BF16) {
    if (sp.slot_bytes == (uint32_t)kStNW * 4096) launch_stream<__nv_bfloat16, 8>(sp, a, st);
    else launch_stream<__nv_bfloat16, 4>(sp, a, st);
  } else {
    if (sp.slot_bytes == (uint32_t)kStNW * 4096) launch_stream<float, 8>(sp, a, st);
    else launch_stream<float, 4>(sp, a, st);
  }
  g_prof.bracket_end(st);
#define ATKG_ST_FIN(T_)                                   \
  switch (kp) {                                           \
    case 1: launch_finish<T_, 1>(sp, rows, f, st); break; \
    case 2: launch_finish<T_, 2>(sp, rows, f, st); break; \
    case 4: launch_finish<T_, 4>(sp, rows, f, st); break; \
    default: launch_finish<T_, 8>(sp, rows, f, st); break; \
  }
  if (dtype == ATKG_BF16) {
    ATKG_ST_FIN(__nv_bfloat16)
  } else {
    ATKG_ST_FIN(float)
  }
#undef ATKG_ST_FIN
}

// the stream kernel alone (no finish): slots of rows x n into ws
void run_stream_only(int dtype, const StPlan& sp, const void* in, uint64_t n, void* ws, uint32_t* status,
                     cudaStream_t st) {
  StArgs a;
  a.in = in;
  a.n = n;
  a.vtot = sp.vtot;
  a.psz = sp.psz;
  a.G = sp.G;
  a.smax = sp.smax;
  a.slot_bytes = sp.slot_bytes;
  a.ns = sp.ns;
  a.rfac = sp.rfac;
  a.lfac = sp.lfac;
  a.cfac = sp.cfac;
  a.warp_sample = (uint32_t)opt("st_warp_sample", 0);
  a.slots = static_cast<uint32_t*>(ws);
  a.gate = nullptr;
  a.status = status;
  g_prof.bracket_begin(st);
  if (dtype == ATKG_BF16) {
    if (sp.slot_bytes == (uint32_t)kStNW * 4096) launch_stream<__nv_bfloat16, 8>(sp, a, st);
    else launch_stream<__nv_bfloat16, 4>(sp, a, st);
  } else {
    if (sp.slot_bytes == (uint32_t)kStNW * 4096) launch_stream<float, 8>(sp, a, st);
    else launch_stream<float, 4>(sp, a, st);
  }
  g_prof.bracket_end(st);
}

// st_finish_kernel over `parts` slice payloads (slots of slot_cap entries) as
// the slots of one row of n elements; gate mode (no input to fall back on)
void run_payload_finish(const uint32_t* payloads, uint32_t parts, uint32_t slot_cap, uint64_t n, uint64_t B,
                        uint32_t kp, uint32_t k, float* ov, uint32_t* oi, uint32_t* gate, uint32_t* status,
                        cudaStream_t st) {
  StPlan sp;
  sp.ecap = 8192;
  while (sp.ecap < B * std::min<uint64_t>(kp, n / B)) sp.ecap <<= 1;
  sp.smem_fin = (size_t)sp.ecap * 16 + (size_t)B * 12;
  StFinArgs f{};
  f.in = nullptr;
  f.n = n;
  const uint64_t nvrow = n / 4;  // the geometry only locates the slots: one row over `parts` pieces
  f.vtot = nvrow;
  f.psz = (nvrow + parts - 1) / parts;
  f.G = parts;
  f.smax = 1;
  f.B = (uint32_t)B;
  f.k = k;
  f.slot_cap = slot_cap;
  f.ecap = sp.ecap;
  f.force_slow = (uint32_t)opt("st_force_slow", 0);
  f.gate = gate;
  f.slots = payloads;
  f.out_v = ov;
  f.out_i = oi;
  f.status = status;
  switch (kp) {
    case 1: launch_finish<float, 1>(sp, 1, f, st); break;
    case 2: launch_finish<float, 2>(sp, 1, f, st); break;
    case 4: launch_finish<float, 4>(sp, 1, f, st); break;
    default: launch_finish<float, 8>(sp, 1, f, st); break;
  }
}

void run_slice_payload(const StPlan& sp, const uint32_t* slots, uint32_t cap, uint64_t index_offset,
                       const uint32_t* status, uint32_t* payload, cudaStream_t st) {
  StPayArgs a;
  a.slots = slots;
  a.G = sp.G;
  a.smax = sp.smax;
  a.cap = cap;
  a.index_offset = index_offset;
  a.status = status;
  a.payload = payload;
  st_slice_payload_kernel<<<1, 1024, 0, st>>>(a);
  check_launch();
}

bool run_select_ranked(const float* vals, const uint32_t* idx, uint64_t rows, uint64_t count, uint64_t stride,
                       uint32_t k, uint64_t limit, float* ov, uint32_t* oi, uint32_t* status, cudaStream_t st) {
  if (opt("no_rank_select", 0) || count <= 128 || count > 1024) return false;
  uint32_t P = 2;
  while (P < count) P <<= 1;
  const unsigned threads = (unsigned)opt("s2_threads", 128);
  stage2_rank_kernel<<<(unsigned)rows, threads, (size_t)P * 16, st>>>(vals, idx, (uint32_t)count, stride, k, limit,
                                                                       P, ov, oi, status);
  check_launch();
  return true;
}

}  // namespace atkg
