// atkg_api.cu -- the C ABI (include/atkg.h): validation, workspace planning,
// kernel dispatch, host-buffer drop-in entry points and the streaming
// accumulator.  Kernels live in stage1.cuh / stage2.cuh / radix.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/atkg.h"
#include "host_common.hpp"
#include "internal.hpp"
#include "radix.cuh"
#include "rowres.cuh"
#include "stage1.cuh"
#include "stage2.cuh"

namespace atkg {

thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

std::atomic<uint64_t> g_launches{0};
Profiler g_prof;

constexpr int kSegWarps = 8;   // warps (= segments) per stage-1 CTA
constexpr int kPrefetch = 4;   // stride-rows per batch in the stage-1 loop
constexpr uint32_t kMaxSortKeys = 16384;  // one CTA's shared-memory sort (128 KB)

constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

int sm_count() {
  static std::atomic<int> cache[kMaxDevices] = {};
  const int dev = current_device();
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    int c = 0;
    if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c <= 0) c = 148;
    cache[dev].store(c, std::memory_order_relaxed);
    n = c;
  }
  return n;
}

void ensure_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, size_t>> done;  // (device, kernel) -> bytes set
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first.first == dev && e.first.second == kern) {
      if (e.second >= bytes) return;
      CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      e.second = bytes;
      return;
    }
  CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done.push_back({{dev, kern}, bytes});
}

namespace {
struct OptSlot {
  char name[48];
  std::atomic<uint64_t> val;
};
constexpr int kMaxOpts = 64;
OptSlot g_opts[kMaxOpts];
std::atomic<int> g_nopts{0};
std::mutex g_opt_mu;
}  // namespace

uint64_t opt(const char* name, uint64_t dflt) {
  const int n = g_nopts.load(std::memory_order_acquire);
  for (int i = 0; i < n; ++i)
    if (std::strcmp(g_opts[i].name, name) == 0) {
      const uint64_t v = g_opts[i].val.load(std::memory_order_relaxed);
      return v == ~0ull ? dflt : v;
    }
  return dflt;
}

void set_opt(const char* name, uint64_t v) {
  if (!name || std::strlen(name) >= sizeof(OptSlot::name)) throw_inval("option name too long");
  std::lock_guard<std::mutex> lk(g_opt_mu);
  const int n = g_nopts.load(std::memory_order_relaxed);
  for (int i = 0; i < n; ++i)
    if (std::strcmp(g_opts[i].name, name) == 0) {
      g_opts[i].val.store(v, std::memory_order_relaxed);
      return;
    }
  if (n >= kMaxOpts) throw_inval("too many options");
  std::strcpy(g_opts[n].name, name);
  g_opts[n].val.store(v, std::memory_order_relaxed);
  g_nopts.store(n + 1, std::memory_order_release);
}

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

uint32_t next_pow2(uint64_t x) {
  uint32_t p = 2;
  while (p < x) p <<= 1;
  return p;
}

void validate(const atkg_params& p) {  // src/topk.cpp:54-67, same messages
  if (p.n == 0) throw_inval("n must be >= 1");
  if (p.n > 0xffffffffull) throw_inval("n exceeds the 32-bit index range");
  if (p.num_buckets == 0) throw_inval("num_buckets must be >= 1");
  if (p.n % p.num_buckets != 0) throw_inval("num_buckets must divide n");
  if (p.lane_multiple == 0) throw_inval("lane_multiple must be >= 1");
  if (p.num_buckets % p.lane_multiple != 0) throw_inval("num_buckets must be a multiple of lane_multiple");
  if (p.local_k == 0) throw_inval("local_k must be >= 1");
  if (p.global_k == 0) throw_inval("global_k must be >= 1");
  if (p.global_k > p.n) throw_inval("global_k must not exceed n");
  if (p.num_buckets * static_cast<uint64_t>(p.local_k) < p.global_k)
    throw_inval("num_buckets * local_k must be >= global_k");
}

bool kp_specialised(uint32_t kp) { return (kp >= 1 && kp <= 8) || kp == 16; }

// ---------------------------------------------------------------------------
// stage-1 launch plan
//   flat     the balanced TMA-fed streaming kernel (stage1_flat_kernel) --
//            the hot path; needs 16-byte aligned rows and copy sizes
//   segments LDG fallback for 4-element-aligned inputs
//   generic  one thread per bucket running Alg. 1 directly (any shape, any K')
// Both summary paths leave `parts` summary blocks per row in the workspace,
// folded by run_merge.
// ---------------------------------------------------------------------------
#ifndef ATKG_SLOTS
#define ATKG_SLOTS 3
#endif
#ifndef ATKG_LOGC
#define ATKG_LOGC 16
#endif
#ifndef ATKG_FLAT_W
#define ATKG_FLAT_W 4
#endif
constexpr int kFlatSlots = ATKG_SLOTS;  // TMA ring slots per warp
#ifndef ATKG_CR
#define ATKG_CR 8
#endif
constexpr int kFlatRows = ATKG_CR;       // stride-rows per ring slot
constexpr int kFlatWarps = ATKG_FLAT_W; // warps per CTA (independent)
constexpr int kLogCap = ATKG_LOGC;      // log entries per (lane, bucket)
// lanes own V adjacent buckets; fewer for long lists to bound registers
// (at least 4 bytes per lane per row: the cp.async granule)
#ifndef ATKG_FLAT_V4
#define ATKG_FLAT_V4 4
#endif
constexpr int flat_vec(int kp, int esz = 4) {
  const int v = kp <= 4 ? ATKG_FLAT_V4 : (kp <= 8 ? 2 : 1);
  return v * esz >= 4 ? v : 4 / esz;
}
// stride-rows sampled for the starting threshold of every piece
#ifndef ATKG_Q0
#define ATKG_Q0 48
#endif
constexpr int flat_q0(int kp) { return kp <= 2 ? ATKG_Q0 : ATKG_Q0 / 2 * kp; }

template <typename T, int KP>
auto flat_kernel_fn() {
  return stage1_flat_kernel<T, KP, flat_vec(KP, sizeof(T)), kFlatWarps, kFlatSlots, kFlatRows, kLogCap, flat_q0(KP)>;
}
template <typename T, int KP>
constexpr size_t flat_smem() {
  return flat_smem_bytes<T, KP, flat_vec(KP, sizeof(T)), kFlatWarps, kFlatSlots, kFlatRows, kLogCap>();
}

template <typename T>
int flat_occupancy(uint32_t kp) {
  const void* k = nullptr;
  size_t smem = 0;
  switch (kp) {
#define ATKG_OCC(K) case K: k = reinterpret_cast<const void*>(flat_kernel_fn<T, K>()); smem = flat_smem<T, K>(); break;
    ATKG_OCC(1) ATKG_OCC(2) ATKG_OCC(3) ATKG_OCC(4) ATKG_OCC(5) ATKG_OCC(6) ATKG_OCC(7) ATKG_OCC(8) ATKG_OCC(16)
#undef ATKG_OCC
    default: return 1;
  }
  ensure_smem(k, smem);
  int n = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kFlatWarps * 32, smem));
  return n > 0 ? n : 1;
}

int flat_ctas_per_sm(int dtype, uint32_t kp) {
  static std::atomic<int> cache[kMaxDevices][2][17] = {};
  const int dev = current_device();
  std::atomic<int>& c = cache[dev][dtype == ATKG_BF16 ? 1 : 0][kp <= 16 ? kp : 0];
  int v = c.load(std::memory_order_relaxed);
  if (v == 0) {
    int cc = 0;
    cudaDeviceGetAttribute(&cc, cudaDevAttrComputeCapabilityMajor, dev);
    if (cc < 10) return 2;  // planning without an sm_100 device (workspace sizing)
    v = dtype == ATKG_BF16 ? flat_occupancy<__nv_bfloat16>(kp) : flat_occupancy<float>(kp);
    c.store(v, std::memory_order_relaxed);
  }
  return v;
}

struct S1Plan {
  enum Kind { kGeneric, kFlat, kSegments } kind = kGeneric;
  int V = 4;
  uint64_t nstr = 0;
  uint32_t tiles = 0;
  // flat
  uint64_t units = 0, total = 0, len = 0, warps = 0;
  uint32_t parts = 1;
  // segments
  uint32_t segs = 0, cpr = 0, group = 1;
  uint64_t groups = 0, seg_len = 0;
  size_t smem = 0;
};

// rows x (nstr stride-rows of B buckets), row_stride elements apart
S1Plan plan_stage1(int dtype, const void* in, uint64_t rows, uint64_t len, uint64_t row_stride, uint64_t B,
                   uint32_t kp) {
  S1Plan pl;
  const int esz = dtype == ATKG_BF16 ? 2 : 4;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(in);
  pl.nstr = len / B;
  if (!kp_specialised(kp) || pl.nstr == 0) return pl;
  const int Vf = flat_vec(kp, esz);
  const bool tma_ok = (addr % 16 == 0) && ((row_stride * esz) % 16 == 0) && ((B * esz) % 16 == 0) && (B % Vf == 0);
  if (tma_ok && opt("no_flat", 0) == 0) {
    pl.kind = S1Plan::kFlat;
    pl.V = Vf;
    pl.tiles = static_cast<uint32_t>(ceil_div(B, 32ull * Vf));
    pl.units = rows * pl.tiles;
    pl.total = pl.units * pl.nstr;
    const uint64_t target = opt("flat_warps", static_cast<uint64_t>(sm_count()) * flat_ctas_per_sm(dtype, kp) * kFlatWarps);
    pl.len = std::max<uint64_t>(1, ceil_div(pl.total, std::max<uint64_t>(1, target)));
    pl.warps = ceil_div(pl.total, pl.len);
    pl.parts = static_cast<uint32_t>(ceil_div(pl.nstr, pl.len) + 1);
    return pl;
  }
  const bool aligned = (addr % (4 * esz) == 0) && (row_stride % 4 == 0) && (B % 4 == 0);
  if (!aligned) return pl;
  pl.kind = S1Plan::kSegments;
  pl.V = 4;
  pl.tiles = static_cast<uint32_t>(ceil_div(B, 128ull));
  const uint64_t units = rows * pl.tiles;
  const uint64_t target_warps = static_cast<uint64_t>(sm_count()) * 32;
  const uint64_t min_len = std::max<uint64_t>(kp, 32);
  const uint64_t max_segs = std::max<uint64_t>(1, pl.nstr / min_len);
  const uint64_t segs = std::min<uint64_t>(max_segs, std::max<uint64_t>(1, ceil_div(target_warps, units)));
  pl.seg_len = std::max<uint64_t>(1, ceil_div(pl.nstr, segs));
  if (pl.nstr >= kp) pl.seg_len = std::max<uint64_t>(pl.seg_len, kp);
  pl.segs = static_cast<uint32_t>(std::max<uint64_t>(1, ceil_div(pl.nstr, pl.seg_len)));
  pl.group = 1;
  while (pl.group < (uint32_t)kSegWarps && pl.group < pl.segs) pl.group <<= 1;
  pl.cpr = static_cast<uint32_t>(ceil_div(pl.segs, pl.group));
  pl.parts = pl.cpr;
  pl.groups = rows * pl.tiles * pl.cpr;
  pl.smem = pl.group > 1 ? static_cast<size_t>(kSegWarps / 2) * (2 * kp + 2) * 4 * 32 * 4 : 0;
  return pl;
}

uint64_t stage1_ws_bytes(const S1Plan& pl, uint64_t rows, uint64_t B, uint32_t kp) {
  if (pl.kind == S1Plan::kGeneric) return 0;
  return align_up(rows * pl.parts * (2ull * kp + 2) * B * 4);
}

template <typename T, int KP>
void launch_stage1(const S1Plan& pl, const void* in, uint64_t rows, uint64_t row_stride, uint64_t B,
                   uint64_t index_offset, uint32_t* out, uint32_t* status, cudaStream_t st) {
  if (pl.kind == S1Plan::kFlat) {
    FlatArgs a{};
    a.in = in;
    a.row_stride = row_stride;
    a.B = B;
    a.nstr = pl.nstr;
    a.index_offset = index_offset;
    a.total = pl.total;
    a.len = pl.len;
    a.tiles = pl.tiles;
    a.parts = pl.parts;
    a.warps = pl.warps;
    a.out = out;
    a.status = status;
    auto kern = flat_kernel_fn<T, KP>();
    constexpr size_t smem = flat_smem<T, KP>();
    ensure_smem_fn(kern, smem);
    g_prof.bracket_begin(st);
    kern<<<static_cast<unsigned>(ceil_div(pl.warps, kFlatWarps)), kFlatWarps * 32, smem, st>>>(a);
    check_launch();
    g_prof.bracket_end(st);
    return;
  }
  SegArgs a{};
  a.in = in;
  a.row_stride = row_stride;
  a.rows = rows;
  a.B = B;
  a.nstr = pl.nstr;
  a.index_offset = index_offset;
  a.seg_len = pl.seg_len;
  a.segs = pl.segs;
  a.cta_per_row_tile = pl.cpr;
  a.group = pl.group;
  a.groups = pl.groups;
  a.tiles = pl.tiles;
  a.out = out;
  a.status = status;
  auto kern = stage1_segments_kernel<T, KP, 4, kSegWarps, kPrefetch>;
  ensure_smem_fn(kern, 160 * 1024);
  g_prof.bracket_begin(st);
  kern<<<static_cast<unsigned>(ceil_div(pl.groups, kSegWarps / pl.group)), kSegWarps * 32, pl.smem, st>>>(a);
  check_launch();
  g_prof.bracket_end(st);
}

#define ATKG_KP_SWITCH(kp, CALL)                   \
  switch (kp) {                                    \
    case 1: { constexpr int K_ = 1; CALL; } break;  \
    case 2: { constexpr int K_ = 2; CALL; } break;  \
    case 3: { constexpr int K_ = 3; CALL; } break;  \
    case 4: { constexpr int K_ = 4; CALL; } break;  \
    case 5: { constexpr int K_ = 5; CALL; } break;  \
    case 6: { constexpr int K_ = 6; CALL; } break;  \
    case 7: { constexpr int K_ = 7; CALL; } break;  \
    case 8: { constexpr int K_ = 8; CALL; } break;  \
    case 16: { constexpr int K_ = 16; CALL; } break; \
    default: throw Unsupported("local_k has no specialised kernel"); \
  }

// stage-1 summaries of rows x (len elements) into ws (plan kinds flat/segments)
void run_stage1_summaries(int dtype, const S1Plan& pl, const void* in, uint64_t rows, uint64_t row_stride,
                          uint64_t B, uint32_t kp, uint64_t index_offset, void* ws, uint32_t* status,
                          cudaStream_t st) {
  uint32_t* out = static_cast<uint32_t*>(ws);
  if (dtype == ATKG_BF16) {
    ATKG_KP_SWITCH(kp, (launch_stage1<__nv_bfloat16, K_>(pl, in, rows, row_stride, B, index_offset, out, status, st)));
  } else {
    ATKG_KP_SWITCH(kp, (launch_stage1<float, K_>(pl, in, rows, row_stride, B, index_offset, out, status, st)));
  }
}

template <int KP>
void launch_merge(const uint32_t* in, uint32_t parts, uint64_t rows, uint64_t B, float* gv, uint32_t* gi,
                  uint64_t gstride, uint32_t* summ_out, const uint32_t* prefix, cudaStream_t st) {
  const uint64_t threads = rows * B;
  merge_finalize_kernel<KP><<<static_cast<unsigned>(ceil_div(threads, 128)), 128, 0, st>>>(
      in, parts, rows, B, gv, gi, gstride, summ_out, prefix);
  check_launch();
}

void dispatch_merge(uint32_t kp, const uint32_t* in, uint32_t parts, uint64_t rows, uint64_t B, float* gv,
                    uint32_t* gi, uint64_t gstride, uint32_t* summ_out, cudaStream_t st,
                    const uint32_t* prefix = nullptr) {
  ATKG_KP_SWITCH(kp, (launch_merge<K_>(in, parts, rows, B, gv, gi, gstride, summ_out, prefix, st)));
}

template <int KP>
void launch_merge_parts(const S1Plan& pl, const uint32_t* in, uint64_t rows, uint64_t B, float* gv, uint32_t* gi,
                        uint64_t gstride, uint32_t* summ_out, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(rows * ceil_div(B, 32));
  if (pl.parts >= 32)
    merge_parts_kernel<KP, 8><<<grid, 256, 0, st>>>(in, pl.parts, pl.nstr, pl.len, pl.tiles, pl.V, rows, B, gv, gi,
                                                     gstride, summ_out);
  else if (pl.parts >= 8)
    merge_parts_kernel<KP, 4><<<grid, 128, 0, st>>>(in, pl.parts, pl.nstr, pl.len, pl.tiles, pl.V, rows, B, gv, gi,
                                                     gstride, summ_out);
  else
    merge_parts_kernel<KP, 1><<<grid, 32, 0, st>>>(in, pl.parts, pl.nstr, pl.len, pl.tiles, pl.V, rows, B, gv, gi,
                                                    gstride, summ_out);
  check_launch();
}

// folds the summaries of run_stage1_summaries: grid (Alg. 1 state) and/or merged summary
void run_merge(const S1Plan& pl, uint32_t kp, const uint32_t* ws, uint64_t rows, uint64_t B, float* gv,
               uint32_t* gi, uint64_t gstride, uint32_t* summ_out, cudaStream_t st) {
  if (pl.kind == S1Plan::kFlat) {
    ATKG_KP_SWITCH(kp, (launch_merge_parts<K_>(pl, ws, rows, B, gv, gi, gstride, summ_out, st)));
  } else {
    dispatch_merge(kp, ws, pl.parts, rows, B, gv, gi, gstride, summ_out, st);
  }
}

// ---------------------------------------------------------------------------
// row-resident path (rowres.cuh) for rows that fit in shared memory
// ---------------------------------------------------------------------------
struct RowPlan {
  bool ok = false;
  uint32_t R = 1, TPR = 32, P = 2;
  uint32_t fast = 0;  // closed-form pass 2 (short buckets, window padding affordable)
  size_t smem = 0;
};
RowPlan plan_rowres(int dtype, const void* in, uint64_t n, uint64_t B, uint32_t kp) {
  RowPlan rp;
  const uint64_t esz = dtype == ATKG_BF16 ? 2 : 4, E = 4 / esz;
  const uint64_t row_bytes = n * esz;
  if (!kp_specialised(kp) || opt("no_rowres", 0)) return rp;
  if (row_bytes > 64 * 1024 || row_bytes % 16 != 0 || reinterpret_cast<uintptr_t>(in) % 16 != 0) return rp;
  if (B % E != 0 || n / B > 4096) return rp;
  const uint64_t filled = std::min<uint64_t>(kp, n / B) * B;
  rp.P = next_pow2(filled);
  if (rp.P > 4096) return rp;
  const uint64_t W = B / E;
  rp.TPR = static_cast<uint32_t>(std::min<uint64_t>(256, (W + 31) / 32 * 32));
  const size_t key_bytes = esz == 2 ? 4 : 8;  // bf16 rows use 32-bit rank keys
  // keys (+ P more as the select scratch for large P) | select histogram
  const size_t keys = (size_t)(rp.P + (rp.P > 512 ? rp.P : 0)) * key_bytes;
  const size_t scratch = 264 * 4;
  const size_t per_row = ((row_bytes + 127) & ~127ull) + keys + scratch;
  // small CTAs (one row when rows are large) keep many rows in flight per SM
  const uint64_t rmax = opt("rowres_rows", 0);
  rp.R = static_cast<uint32_t>(
      rmax ? rmax : std::max<uint64_t>(1, std::min<uint64_t>(128 / rp.TPR, (48 * 1024) / per_row)));
  // pass 2 reads whole 32/E-row windows: rows past the end land in the
  // bytes that follow the last row (keys, scratch, then padding)
  const uint64_t CH = 32 / E, nstr = n / B;
  const size_t over = (size_t)((CH - nstr % CH) % CH) * B * esz;  // window overrun past the row
  const size_t tail = rp.R * (keys + scratch);
  const size_t pad = over > tail ? over - tail : 0;
  rp.fast = (nstr <= 128 && pad <= 4096 && !opt("rowres_slow", 0)) ? 1u : 0u;
  rp.smem = rp.R * per_row + (rp.fast ? pad : 0);
  rp.ok = true;
  return rp;
}
template <typename T, int KP>
void launch_rowres(const RowPlan& rp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t k,
                   float* ov, uint32_t* oi, float* gv, uint32_t* gi, uint32_t* status, cudaStream_t st) {
  auto kern = row_resident_kernel<T, KP>;
  ensure_smem_fn(kern, rp.smem);
  const uint32_t filled = (uint32_t)std::min<uint64_t>(KP, n / B);
  g_prof.bracket_begin(st);
  kern<<<static_cast<unsigned>(ceil_div(rows, rp.R)), rp.R * rp.TPR, rp.smem, st>>>(
      static_cast<const T*>(in), rows, (uint32_t)n, (uint32_t)B, rp.R, k, filled, rp.P, rp.fast, ov, oi, gv, gi,
      status);
  check_launch();
  g_prof.bracket_end(st);
}
void run_rowres(int dtype, const RowPlan& rp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp,
                uint32_t k, float* ov, uint32_t* oi, float* gv, uint32_t* gi, uint32_t* status, cudaStream_t st) {
  if (dtype == ATKG_BF16) {
    ATKG_KP_SWITCH(kp, (launch_rowres<__nv_bfloat16, K_>(rp, in, rows, n, B, k, ov, oi, gv, gi, status, st)));
  } else {
    ATKG_KP_SWITCH(kp, (launch_rowres<float, K_>(rp, in, rows, n, B, k, ov, oi, gv, gi, status, st)));
  }
}

// stage 1 into a grid (grid_stride elements between rows)
void run_stage1_grid(int dtype, const void* in, uint64_t rows, const atkg_params& p, float* gv, uint32_t* gi,
                     uint64_t gstride, void* ws, uint32_t* status, cudaStream_t st) {
  const uint64_t B = p.num_buckets;
  const uint32_t kp = p.local_k;
  const RowPlan rp = plan_rowres(dtype, in, p.n, B, kp);
  if (rp.ok && gstride == kp * B) {
    run_rowres(dtype, rp, in, rows, p.n, B, kp, 0, nullptr, nullptr, gv, gi, status, st);
    return;
  }
  const S1Plan pl = plan_stage1(dtype, in, rows, p.n, p.n, B, kp);
  if (pl.kind == S1Plan::kGeneric) {
    if (gstride != kp * B) throw Unsupported("generic stage 1 needs a dense grid");
    const uint64_t threads = rows * B;
    if (dtype == ATKG_BF16)
      stage1_generic_kernel<__nv_bfloat16><<<static_cast<unsigned>(ceil_div(threads, 128)), 128, 0, st>>>(
          static_cast<const __nv_bfloat16*>(in), rows, p.n, B, kp, gv, gi, status);
    else
      stage1_generic_kernel<float><<<static_cast<unsigned>(ceil_div(threads, 128)), 128, 0, st>>>(
          static_cast<const float*>(in), rows, p.n, B, kp, gv, gi, status);
    check_launch();
    return;
  }
  run_stage1_summaries(dtype, pl, in, rows, p.n, B, kp, 0, ws, status, st);
  run_merge(pl, kp, static_cast<const uint32_t*>(ws), rows, B, gv, gi, gstride, nullptr, st);
}

// ---------------------------------------------------------------------------
// stage 2 / exact selection
// ---------------------------------------------------------------------------
// keys per row in the radix path's buffer: k, or the pow2 >= k of the
// global-memory sort when k exceeds one CTA's shared-memory sort
uint64_t radix_key_stride(uint32_t k) { return k <= kMaxSortKeys ? k : next_pow2(k); }

uint64_t radix_ws_bytes(uint64_t rows, uint32_t k) {
  return align_up(rows * sizeof(RowSel)) + align_up(rows * 256 * 4) + align_up(rows * radix_key_stride(k) * 8);
}

template <class Src>
void run_radix(const Src& src, uint64_t rows, uint64_t count, uint32_t k, float* ov, uint32_t* oi, void* ws,
               uint32_t* status, cudaStream_t st) {
  char* w = static_cast<char*>(ws);
  RowSel* sel = reinterpret_cast<RowSel*>(w);
  w += align_up(rows * sizeof(RowSel));
  uint32_t* hist = reinterpret_cast<uint32_t*>(w);
  w += align_up(rows * 256 * 4);
  uint64_t* keys = reinterpret_cast<uint64_t*>(w);
  radix_init_kernel<<<static_cast<unsigned>(std::max<uint64_t>(1, ceil_div(rows * 256, 256))), 256, 0, st>>>(
      sel, hist, rows, k);
  check_launch();
  const uint64_t ctas_total = static_cast<uint64_t>(sm_count()) * 8;
  uint64_t cpr = std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(count, 4096), ceil_div(ctas_total, rows)));
  const dim3 grid(static_cast<unsigned>(cpr), static_cast<unsigned>(rows));
  for (int pass = 0; pass < 8; ++pass) {
    radix_hist_kernel<Src><<<grid, 256, 0, st>>>(src, pass, sel, hist, status);
    check_launch();
    radix_select_kernel<<<static_cast<unsigned>(ceil_div(rows, 8)), 256, 0, st>>>(pass, sel, hist, rows, status);
    check_launch();
  }
  const uint64_t kstride = radix_key_stride(k);
  radix_gather_kernel<Src><<<grid, 256, 0, st>>>(src, sel, keys, k, kstride);
  check_launch();
  if (k > kMaxSortKeys) {  // global-memory bitonic network over P = kstride keys per row
    const uint64_t P = kstride;
    const unsigned blocks = static_cast<unsigned>(P / kSortBlock);
    const size_t smem = kSortBlock * 8;
    ensure_smem_fn(big_sort_block_kernel, smem);
    ensure_smem_fn(big_sort_block_merge, smem);
    big_sort_block_kernel<<<dim3(blocks, static_cast<unsigned>(rows)), 1024, smem, st>>>(keys, P, k);
    check_launch();
    for (uint64_t size = 2ull * kSortBlock; size <= P; size <<= 1) {
      for (uint64_t stride = size >> 1; stride >= kSortBlock; stride >>= 1) {
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(P / 2, 256), 4096));
        big_sort_global_step<<<dim3(g, static_cast<unsigned>(rows)), 256, 0, st>>>(keys, P, size, stride);
        check_launch();
      }
      big_sort_block_merge<<<dim3(blocks, static_cast<unsigned>(rows)), 1024, smem, st>>>(keys, P, size);
      check_launch();
    }
    const unsigned eg = static_cast<unsigned>(std::min<uint64_t>(ceil_div(rows * k, 256), 65535));
    big_sort_emit<<<eg, 256, 0, st>>>(keys, P, k, rows, ov, oi, status);
    check_launch();
    return;
  }
  const uint32_t P = next_pow2(k);
  ensure_smem_fn(sort_emit_kernel, kMaxSortKeys * 8);
  sort_emit_kernel<<<static_cast<unsigned>(rows), std::min<uint32_t>(1024, P / 2), P * 8, st>>>(keys, k, P, ov, oi,
                                                                                             status);
  check_launch();
}

uint64_t select_ws_bytes(uint64_t rows, uint64_t count, uint32_t k) {
  if (next_pow2(count) <= kMaxSortKeys) return 0;
  return radix_ws_bytes(rows, k);
}

void run_select(const float* vals, const uint32_t* idx, uint64_t rows, uint64_t count, uint64_t stride, uint32_t k,
                uint64_t limit, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st) {
  const uint32_t P = next_pow2(count);
  if (run_select_ranked(vals, idx, rows, count, stride, k, limit, ov, oi, status, st)) return;
  if (P <= 512) {  // one warp per row, keys in registers
    const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
    const uint32_t c32 = static_cast<uint32_t>(count);
    if (P <= 64)
      stage2_warp_kernel<2><<<grid, 256, 0, st>>>(vals, idx, rows, c32, stride, k, limit, ov, oi, status);
    else if (P <= 128)
      stage2_warp_kernel<4><<<grid, 256, 0, st>>>(vals, idx, rows, c32, stride, k, limit, ov, oi, status);
    else if (P <= 256)
      stage2_warp_kernel<8><<<grid, 256, 0, st>>>(vals, idx, rows, c32, stride, k, limit, ov, oi, status);
    else
      stage2_warp_kernel<16><<<grid, 256, 0, st>>>(vals, idx, rows, c32, stride, k, limit, ov, oi, status);
    check_launch();
    return;
  }
  if (P <= kMaxSortKeys) {
    ensure_smem_fn(stage2_bitonic_kernel, kMaxSortKeys * 8);
    stage2_bitonic_kernel<<<static_cast<unsigned>(rows), std::min<uint32_t>(1024, P / 2), P * 8, st>>>(
        vals, idx, count, stride, k, limit, P, ov, oi, status);
    check_launch();
    return;
  }
  CandSrc src{vals, idx, count, stride, limit};
  run_radix(src, rows, count, k, ov, oi, ws, status, st);
}

uint64_t grid_bytes(uint64_t rows, const atkg_params& p) { return align_up(rows * p.local_k * p.num_buckets * 8); }

uint64_t filled_count(const atkg_params& p) {  // topk.cpp:250-253
  return std::min<uint64_t>(p.local_k, p.n / p.num_buckets) * p.num_buckets;
}

// fused merge + stage 2 (merge_select_kernel) for the flat path
size_t merge_select_smem(const S1Plan& pl, const atkg_params& p) {
  const uint64_t words = (2ull * p.local_k + 2) * p.num_buckets;
  const uint64_t staged = (pl.parts * words + 3) & ~3ull;
  return staged * 4 + (size_t)next_pow2(filled_count(p)) * 8;
}
bool fused_tail_ok(const S1Plan& pl, const atkg_params& p) {
  return pl.kind == S1Plan::kFlat && merge_select_smem(pl, p) <= 200 * 1024 &&
         next_pow2(filled_count(p)) <= kMaxSortKeys && ((2ull * p.local_k + 2) * p.num_buckets) % 4 == 0;
}
template <int KP>
void launch_merge_select(const S1Plan& pl, const atkg_params& p, const uint32_t* ws, uint64_t rows, float* ov,
                         uint32_t* oi, float* gv, uint32_t* gi, uint32_t* status, cudaStream_t st) {
  const size_t smem = merge_select_smem(pl, p);
  ensure_smem_fn(merge_select_kernel<KP>, smem);
  const uint32_t P = next_pow2(filled_count(p));
  const uint32_t threads = std::min<uint32_t>(512, std::max<uint32_t>(64, (uint32_t)std::max<uint64_t>(p.num_buckets, P / 2)));
  const uint32_t filled = (uint32_t)std::min<uint64_t>(p.local_k, p.n / p.num_buckets);
  merge_select_kernel<KP><<<static_cast<unsigned>(rows), (threads + 31) / 32 * 32, smem, st>>>(
      ws, pl.parts, pl.nstr, pl.len, pl.tiles, pl.V, p.num_buckets, filled, P, p.global_k, ov, oi, gv, gi, status);
  check_launch();
}
void run_merge_select(const S1Plan& pl, const atkg_params& p, const uint32_t* ws, uint64_t rows, float* ov,
                      uint32_t* oi, float* gv, uint32_t* gi, uint32_t* status, cudaStream_t st) {
  ATKG_KP_SWITCH(p.local_k, (launch_merge_select<K_>(pl, p, ws, rows, ov, oi, gv, gi, status, st)));
}

// ---------------------------------------------------------------------------
// device scratch cache for the host-buffer entry points
// ---------------------------------------------------------------------------
struct HostCtx {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  void* buf[6] = {};
  size_t cap[6] = {};
  void* get(int slot, size_t bytes) {
    if (bytes == 0) bytes = 256;
    if (cap[slot] < bytes) {
      if (buf[slot]) CUDA_OK(cudaFree(buf[slot]));
      CUDA_OK(cudaMalloc(&buf[slot], bytes));
      cap[slot] = bytes;
    }
    return buf[slot];
  }
  cudaStream_t s() {
    if (!stream) CUDA_OK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    return stream;
  }
};
// one context per device: its stream and buffers live on that device
HostCtx& host_ctx() {
  static HostCtx* ctx[kMaxDevices] = {};
  static std::mutex mu;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  if (!ctx[dev]) ctx[dev] = new HostCtx();
  return *ctx[dev];
}

// caller-supplied workspace must cover what the dispatch will use
void check_ws(size_t have, size_t need) {
  if (have < need) throw_inval("workspace smaller than atkg_workspace_size");
}

void check_status_sync(const uint32_t* d_status, cudaStream_t st) {
  uint32_t flags = 0;
  CUDA_OK(cudaMemcpyAsync(&flags, d_status, 4, cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaStreamSynchronize(st));
  if (flags & ATKG_FLAG_NAN) throw NanInput();
  if (flags & kFlagFew) throw_inval("fewer candidates than k");
}

// workspace bytes for `op` (atkg_workspace_size): the maximum over every
// dispatch path the call may take, for 16-byte aligned and unaligned inputs
size_t ws_need_uncached(int op, int dtype, uint64_t rows, const atkg_params& pr) {
  const atkg_params* p = &pr;
  size_t bytes = 0;
  for (uintptr_t addr : {uintptr_t(256), uintptr_t(264), uintptr_t(258)}) {
    const void* in = reinterpret_cast<const void*>(addr);
    size_t b = 0;
    switch (op) {
      case ATKG_OP_STAGE1: {
        const S1Plan pl = plan_stage1(dtype, in, rows, p->n, p->n, p->num_buckets, p->local_k);
        b = stage1_ws_bytes(pl, rows, p->num_buckets, p->local_k);
        break;
      }
      case ATKG_OP_APPROX: {
        const S1Plan pl = plan_stage1(dtype, in, rows, p->n, p->n, p->num_buckets, p->local_k);
        b = stage1_ws_bytes(pl, rows, p->num_buckets, p->local_k) + grid_bytes(rows, *p) +
            select_ws_bytes(rows, filled_count(*p), p->global_k);
        const ThrPlan tp = plan_rowthr(dtype, in, p->n, p->num_buckets, p->local_k, p->global_k);
        if (tp.ok) b = std::max<size_t>(b, rowthr_ws_bytes(rows, tp));
        const StPlan sp = plan_streamthr(dtype, in, rows, p->n, p->num_buckets, p->local_k, p->global_k, true);
        if (sp.ok) b = std::max<size_t>(b, sp.ws_bytes);
        const RwPlan rwp = plan_rowwarp(dtype, in, rows, p->n, p->num_buckets, p->local_k, p->global_k, true);
        if (rwp.ok) b = std::max<size_t>(b, rwp.ws_bytes);
        const SrPlan srp = plan_short(dtype, in, rows, p->n, p->num_buckets, p->local_k, p->global_k, true);
        if (srp.ok) b = std::max<size_t>(b, srp.ws_bytes);
        const RmPlan rmp = plan_rowmax1(dtype, in, rows, p->n, p->num_buckets, p->local_k, p->global_k, true);
        if (rmp.ok) b = std::max<size_t>(b, rmp.ws_bytes + 256);
        break;
      }
      case ATKG_OP_SELECT:
        b = select_ws_bytes(rows, p->n, p->global_k);
        break;
      case ATKG_OP_EXACT:
        b = radix_ws_bytes(rows, p->global_k);
        break;
      case ATKG_OP_SUMMARY: {
        const S1Plan pl = plan_stage1(dtype, in, 1, p->n, p->n, p->num_buckets, p->local_k);
        b = stage1_ws_bytes(pl, 1, p->num_buckets, p->local_k);
        break;
      }
      case ATKG_OP_MERGE:
        b = grid_bytes(1, *p) + select_ws_bytes(1, filled_count(*p), p->global_k);
        break;
      default:
        throw_inval("unknown workspace op");
    }
    bytes = std::max(bytes, b);
  }
  // slack so every device path can align its pointers
  return bytes + 512;
}

// memoised per thread: the check runs on every call (host critical path)
size_t ws_need(int op, int dtype, uint64_t rows, const atkg_params& p) {
  struct Ent {
    int op, dtype, dev;
    uint64_t rows;
    atkg_params p;
    size_t bytes;
  };
  thread_local Ent memo[8];
  thread_local int next = 0;
  const int dev = current_device();
  for (const Ent& e : memo)
    if (e.bytes && e.op == op && e.dtype == dtype && e.dev == dev && e.rows == rows && e.p.n == p.n &&
        e.p.num_buckets == p.num_buckets && e.p.local_k == p.local_k && e.p.global_k == p.global_k &&
        e.p.lane_multiple == p.lane_multiple)
      return e.bytes;
  const size_t b = ws_need_uncached(op, dtype, rows, p);
  memo[next] = Ent{op, dtype, dev, rows, p, b};
  next = (next + 1) % 8;
  return b;
}

}  // namespace atkg

using namespace atkg;

// ===========================================================================
extern "C" {

const char* atkg_last_error(void) { return g_last_error.c_str(); }
const char* atkg_version(void) { return "atkg 0.1 (sm_100a)"; }

int atkg_set_device(int device) {
  return guarded([&] { CUDA_OK(cudaSetDevice(device)); });
}

int atkg_set_option(const char* name, uint64_t value) {
  return guarded([&] { set_opt(name, value); });
}

uint64_t atkg_get_option(const char* name, uint64_t dflt) { return opt(name, dflt); }

void atkg_profile_begin(void) { atkg_profile_begin_every(1); }

void atkg_profile_begin_every(uint32_t every) {
  g_prof.on = true;
  g_prof.used = 0;
  g_prof.every = every ? every : 1;
  g_prof.seen = 0;
  g_prof.open = false;
}

int atkg_profile_end(double* total_ms, uint64_t* launches) {
  return guarded([&] {
    g_prof.on = false;
    double sum = 0.0;
    for (size_t q = 0; q < g_prof.used; q += 2) {
      CUDA_OK(cudaEventSynchronize(g_prof.ev[q + 1]));
      float ms = 0.f;
      CUDA_OK(cudaEventElapsedTime(&ms, g_prof.ev[q], g_prof.ev[q + 1]));
      sum += ms;
    }
    *total_ms = sum;
    *launches = g_prof.used / 2;
  });
}

uint64_t atkg_launch_count(void) { return g_launches.load(); }

int atkg_validate(const atkg_params* p) {
  return guarded([&] { validate(*p); });
}

int atkg_workspace_size(int op, int dtype, uint64_t rows, const atkg_params* p, size_t* bytes) {
  return guarded([&] { *bytes = ws_need(op, dtype, rows, *p); });
}

int atkg_stage1(int dtype, const void* d_in, uint64_t rows, const atkg_params* p, float* d_grid_vals,
                uint32_t* d_grid_idx, void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    validate(*p);
    if (rows == 0) return;
    check_ws(ws_bytes, ws_need(ATKG_OP_STAGE1, dtype, rows, *p));
    run_stage1_grid(dtype, d_in, rows, *p, d_grid_vals, d_grid_idx, (uint64_t)p->local_k * p->num_buckets, d_ws,
                    d_status, static_cast<cudaStream_t>(stream));
  });
}

int atkg_select_candidates(const float* d_vals, const uint32_t* d_idx, uint64_t rows, uint64_t count,
                           uint64_t stride, uint32_t k, uint64_t index_limit, float* d_out_vals,
                           uint32_t* d_out_idx, void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    if (k == 0) throw_inval("k must be >= 1");
    if (rows == 0) return;
    if (count < k) throw_inval("fewer candidates than k");
    check_ws(ws_bytes, ws_need(ATKG_OP_SELECT, ATKG_F32, rows, atkg_params{count, 1, 1, k, 1}));
    run_select(d_vals, d_idx, rows, count, stride, k, index_limit, d_out_vals, d_out_idx, d_ws, d_status,
               static_cast<cudaStream_t>(stream));
  });
}

int atkg_approx_top_k(int dtype, const void* d_in, uint64_t rows, const atkg_params* p, float* d_out_vals,
                      uint32_t* d_out_idx, void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    validate(*p);
    if (rows == 0) return;
    check_ws(ws_bytes, ws_need(ATKG_OP_APPROX, dtype, rows, *p));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const RgPlan rgp = plan_rowreg(dtype, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k);
    if (rgp.ok) {  // bf16 rows up to 65536 with B = 128, K' = 4: one warp per row, streamed once into registers (rowreg.cuh)
      run_rowreg(rgp, d_in, rows, p->global_k, d_out_vals, d_out_idx, d_status, st);
      return;
    }
    const RmPlan rmp = plan_rowmax1(dtype, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k);
    if (rmp.ok) {  // K' = 1 with buckets of 2-8 elements: the register row stream, exact kernel for the rest
      run_rowmax1(rmp, dtype, d_in, rows, p->n, p->num_buckets, p->global_k, d_out_vals, d_out_idx,
                  reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(d_ws))), d_status, st);
      return;
    }
    const RgPlan rxp = plan_rowregx(dtype, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k);
    if (rxp.ok) {  // the C3 sweep shapes with 1024 candidates per row (rowregx.cuh)
      run_rowregx(rxp, d_in, rows, p->num_buckets, p->local_k, p->global_k, d_out_vals, d_out_idx, d_status, st);
      return;
    }
    const StPlan sp = plan_streamthr(dtype, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k);
    if (sp.ok) {  // long rows: threshold stream + per-row finish (exact fallback per row)
      void* sws = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(d_ws)));
      run_streamthr(dtype, sp, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k, d_out_vals, d_out_idx,
                    sws, d_status, st);
      if (!sp.giant) return;
      // giant rows: read the gate (4 bytes) and rerun the exact path if a
      // row's threshold failed (the device cannot afford that fallback)
      uint32_t gate = 0;
      CUDA_OK(cudaMemcpyAsync(&gate, static_cast<char*>(sws) + (sp.ws_bytes - 256), 4, cudaMemcpyDeviceToHost, st));
      CUDA_OK(cudaStreamSynchronize(st));
      if (!gate) return;
    }
    const S1Plan pl = plan_stage1(dtype, d_in, rows, p->n, p->n, p->num_buckets, p->local_k);
    char* w = static_cast<char*>(d_ws);
    w = reinterpret_cast<char*>(align_up(reinterpret_cast<uintptr_t>(w)));
    void* s1ws = w;
    w += stage1_ws_bytes(pl, rows, p->num_buckets, p->local_k);
    const uint64_t gstride = (uint64_t)p->local_k * p->num_buckets;
    float* gv = reinterpret_cast<float*>(w);
    uint32_t* gi = reinterpret_cast<uint32_t*>(w + rows * gstride * 4);
    w += grid_bytes(rows, *p);
    // the guaranteed-threshold row kernels (rowwarp.cuh, shortrow.cuh) are
    // bit-exact but not yet faster than row_resident_kernel where that one
    // applies; they run where it does not, or when selected
    const RowPlan rrp = plan_rowres(dtype, d_in, p->n, p->num_buckets, p->local_k);
    const bool row_new = !rrp.ok || opt("short", 0) || opt("rowwarp", 0);
    const RwPlan rwp = row_new ? plan_rowwarp(dtype, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k)
                               : RwPlan{};
    if (rwp.ok) {  // one warp per row in shared memory, guaranteed row threshold (rowwarp.cuh)
      run_rowwarp(rwp, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k, d_out_vals, d_out_idx,
                  reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(d_ws))), d_status, st);
      return;
    }
    const SrPlan srp = row_new ? plan_short(dtype, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k)
                               : SrPlan{};
    if (srp.ok) {  // rows in shared memory, guaranteed row threshold (shortrow.cuh)
      run_short(dtype, srp, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k, d_out_vals, d_out_idx,
                reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(d_ws))), d_status, st);
      return;
    }
    const ThrPlan tp = plan_rowthr(dtype, d_in, p->n, p->num_buckets, p->local_k, p->global_k);
    if (tp.ok) {  // row-resident, row threshold: stage 1 + stage 2 in one warp per row
      run_rowthr(dtype, tp, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k, d_out_vals, d_out_idx,
                 s1ws, d_status, st);
      return;
    }
    const RowPlan rp = plan_rowres(dtype, d_in, p->n, p->num_buckets, p->local_k);
    if (rp.ok) {  // row-resident: stage 1 + stage 2 in one kernel
      run_rowres(dtype, rp, d_in, rows, p->n, p->num_buckets, p->local_k, p->global_k, d_out_vals, d_out_idx,
                 nullptr, nullptr, d_status, st);
      return;
    }
    if (fused_tail_ok(pl, *p)) {
      // stage 1 summaries, then one fused merge + stage-2 kernel per row
      run_stage1_summaries(dtype, pl, d_in, rows, p->n, p->num_buckets, p->local_k, 0, s1ws, d_status, st);
      run_merge_select(pl, *p, static_cast<const uint32_t*>(s1ws), rows, d_out_vals, d_out_idx, nullptr, nullptr,
                       d_status, st);
      return;
    }
    run_stage1_grid(dtype, d_in, rows, *p, gv, gi, gstride, s1ws, d_status, st);
    run_select(gv, gi, rows, filled_count(*p), gstride, p->global_k, UINT64_MAX, d_out_vals, d_out_idx, w,
               d_status, st);
  });
}

}  // extern "C"

namespace atkg {

// select_parameters is deterministic in its request (seed included) and runs
// an adaptive Monte Carlo sweep: memoise the plans of recent requests
atkg_plan_result cached_plan(const atkg_plan_request& req) {
  struct Ent {
    uint64_t n, k, seed;
    double target;
    uint32_t lane;
    std::vector<uint32_t> kps;
    atkg_plan_result res;
  };
  static std::mutex mu;
  static std::vector<Ent> memo;
  std::vector<uint32_t> kps(req.allowed_local_k, req.allowed_local_k + req.num_allowed_local_k);
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const Ent& e : memo)
      if (e.n == req.n && e.k == req.k && e.seed == req.seed && e.target == req.recall_target &&
          e.lane == req.lane_multiple && e.kps == kps)
        return e.res;
  }
  atkg_plan_result r{};
  rethrow(atkg_select_parameters(&req, &r));
  std::lock_guard<std::mutex> lk(mu);
  if (memo.size() >= 32) memo.erase(memo.begin());
  memo.push_back(Ent{req.n, req.k, req.seed, req.recall_target, req.lane_multiple, kps, r});
  return r;
}

atkg_params plan_params(const atkg_plan_request& req, const atkg_plan_result& r) {  // PlanResult::params
  return atkg_params{req.n, r.num_buckets, r.local_k, static_cast<uint32_t>(req.k), req.lane_multiple};
}

}  // namespace atkg

extern "C" {

int atkg_approx_at_recall_workspace_size(int dtype, uint64_t rows, const atkg_plan_request* req, size_t* bytes) {
  return guarded([&] {
    const atkg_params p = plan_params(*req, cached_plan(*req));
    *bytes = ws_need(ATKG_OP_APPROX, dtype, rows, p);
  });
}

int atkg_approx_top_k_at_recall(int dtype, const void* d_in, uint64_t rows, const atkg_plan_request* req,
                                atkg_plan_result* plan_out, float* d_out_vals, uint32_t* d_out_idx, void* d_ws,
                                size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    const atkg_plan_result r = cached_plan(*req);
    if (plan_out) *plan_out = r;
    const atkg_params p = plan_params(*req, r);
    rethrow(atkg_approx_top_k(dtype, d_in, rows, &p, d_out_vals, d_out_idx, d_ws, ws_bytes, d_status, stream));
  });
}

int atkg_exact_top_k(int dtype, const void* d_in, uint64_t rows, uint64_t n, uint32_t k, float* d_out_vals,
                     uint32_t* d_out_idx, void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    if (k == 0) throw_inval("k must be >= 1");
    if (n > 0xffffffffull + 1) throw_inval("input exceeds the 32-bit index range");
    if (k > n) throw_inval("k must not exceed the input length");
    if (rows == 0) return;
    check_ws(ws_bytes, ws_need(ATKG_OP_EXACT, dtype, rows, atkg_params{n, 1, 1, k, 1}));
    char* w = reinterpret_cast<char*>(align_up(reinterpret_cast<uintptr_t>(d_ws)));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == ATKG_BF16) {
      DenseSrc<__nv_bfloat16> src{static_cast<const __nv_bfloat16*>(d_in), n};
      run_radix(src, rows, n, k, d_out_vals, d_out_idx, w, d_status, st);
    } else {
      DenseSrc<float> src{static_cast<const float*>(d_in), n};
      run_radix(src, rows, n, k, d_out_vals, d_out_idx, w, d_status, st);
    }
  });
}

int atkg_stage1_summary(int dtype, const void* d_slice, uint64_t len, uint64_t index_offset, const atkg_params* p,
                        uint32_t* d_summary, void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    validate(*p);
    const uint64_t B = p->num_buckets;
    if (len % B != 0 || index_offset % B != 0) throw_inval("slice length and offset must be multiples of num_buckets");
    if (index_offset + len > p->n) throw_inval("slice exceeds the row");
    check_ws(ws_bytes, ws_need(ATKG_OP_SUMMARY, dtype, 1, atkg_params{len, B, p->local_k, 1, 1}));
    if (!kp_specialised(p->local_k)) throw Unsupported("local_k has no specialised summary kernel");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const S1Plan pl = plan_stage1(dtype, d_slice, 1, len, len, B, p->local_k);
    if (pl.kind == S1Plan::kGeneric) throw Unsupported("summary path needs num_buckets % 4 == 0 and aligned input");
    char* w = reinterpret_cast<char*>(align_up(reinterpret_cast<uintptr_t>(d_ws)));
    run_stage1_summaries(dtype, pl, d_slice, 1, len, B, p->local_k, index_offset, w, d_status, st);
    run_merge(pl, p->local_k, reinterpret_cast<const uint32_t*>(w), 1, B, nullptr, nullptr, 0, d_summary, st);
  });
}

int atkg_summary_merge_top_k(const uint32_t* d_summaries, uint32_t parts, const atkg_params* p, float* d_grid_vals,
                             uint32_t* d_grid_idx, float* d_out_vals, uint32_t* d_out_idx, void* d_ws,
                             size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    validate(*p);
    if (parts == 0) throw_inval("need at least one summary");
    if (!kp_specialised(p->local_k)) throw Unsupported("local_k has no specialised merge kernel");
    check_ws(ws_bytes, ws_need(ATKG_OP_MERGE, ATKG_F32, 1, *p));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* w = reinterpret_cast<char*>(align_up(reinterpret_cast<uintptr_t>(d_ws)));
    const uint64_t gstride = (uint64_t)p->local_k * p->num_buckets;
    float* gv = d_grid_vals;
    uint32_t* gi = d_grid_idx;
    if (!gv) {
      gv = reinterpret_cast<float*>(w);
      gi = reinterpret_cast<uint32_t*>(w + gstride * 4);
    }
    w += grid_bytes(1, *p);
    dispatch_merge(p->local_k, d_summaries, parts, 1, p->num_buckets, gv, gi, gstride, nullptr, st);
    if (d_out_vals)
      run_select(gv, gi, 1, filled_count(*p), gstride, p->global_k, UINT64_MAX, d_out_vals, d_out_idx, w, d_status,
                 st);
  });
}

int atkg_check_status(const uint32_t* d_status, void* stream) {
  return guarded([&] { check_status_sync(d_status, static_cast<cudaStream_t>(stream)); });
}

// ---- host-buffer drop-in ----------------------------------------------------
int atkg_stage1_host(const float* in, uint64_t rows, const atkg_params* p, float* grid_vals, uint32_t* grid_idx) {
  return guarded([&] {
    validate(*p);
    HostCtx& c = host_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    cudaStream_t st = c.s();
    size_t ws = 0;
    if (int rc = atkg_workspace_size(ATKG_OP_STAGE1, ATKG_F32, rows, p, &ws)) throw Inval(g_last_error);
    const uint64_t nin = rows * p->n, ng = rows * p->local_k * p->num_buckets;
    float* din = static_cast<float*>(c.get(0, nin * 4));
    float* gv = static_cast<float*>(c.get(1, ng * 4));
    uint32_t* gi = static_cast<uint32_t*>(c.get(2, ng * 4));
    void* dws = c.get(3, ws);
    uint32_t* status = static_cast<uint32_t*>(c.get(4, 4));
    CUDA_OK(cudaMemsetAsync(status, 0, 4, st));
    CUDA_OK(cudaMemcpyAsync(din, in, nin * 4, cudaMemcpyHostToDevice, st));
    run_stage1_grid(ATKG_F32, din, rows, *p, gv, gi, p->local_k * p->num_buckets, dws, status, st);
    check_status_sync(status, st);
    CUDA_OK(cudaMemcpyAsync(grid_vals, gv, ng * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(grid_idx, gi, ng * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

int atkg_select_candidates_host(const float* vals, const uint32_t* idx, uint64_t count, uint32_t k,
                                uint64_t index_limit, float* out_vals, uint32_t* out_idx) {
  return guarded([&] {
    if (k == 0) throw_inval("k must be >= 1");
    if (count < k) {
      // NaN is rejected before the count check (topk.cpp:225-234)
      for (uint64_t i = 0; i < count; ++i)
        if (vals[i] != vals[i]) throw NanInput();
      throw_inval("fewer candidates than k");
    }
    HostCtx& c = host_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    cudaStream_t st = c.s();
    float* dv = static_cast<float*>(c.get(0, count * 4));
    uint32_t* di = static_cast<uint32_t*>(c.get(1, count * 4));
    float* ov = static_cast<float*>(c.get(2, (uint64_t)k * 4));
    uint32_t* oi = static_cast<uint32_t*>(c.get(3, (uint64_t)k * 4));
    void* dws = c.get(5, select_ws_bytes(1, count, k) + 512);
    uint32_t* status = static_cast<uint32_t*>(c.get(4, 4));
    CUDA_OK(cudaMemsetAsync(status, 0, 4, st));
    CUDA_OK(cudaMemcpyAsync(dv, vals, count * 4, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(di, idx, count * 4, cudaMemcpyHostToDevice, st));
    run_select(dv, di, 1, count, count, k, index_limit, ov, oi,
               reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(dws))), status, st);
    check_status_sync(status, st);
    CUDA_OK(cudaMemcpyAsync(out_vals, ov, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(out_idx, oi, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

int atkg_approx_top_k_host(const float* rows_in, uint64_t rows, const atkg_params* p, float* out_vals,
                           uint32_t* out_idx) {
  return guarded([&] {
    validate(*p);
    if (rows == 0) return;
    HostCtx& c = host_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    cudaStream_t st = c.s();
    size_t ws = 0;
    if (atkg_workspace_size(ATKG_OP_APPROX, ATKG_F32, rows, p, &ws)) throw Inval(g_last_error);
    const uint64_t nin = rows * p->n, no = rows * p->global_k;
    float* din = static_cast<float*>(c.get(0, nin * 4));
    float* ov = static_cast<float*>(c.get(1, no * 4));
    uint32_t* oi = static_cast<uint32_t*>(c.get(2, no * 4));
    void* dws = c.get(3, ws);
    uint32_t* status = static_cast<uint32_t*>(c.get(4, 4));
    CUDA_OK(cudaMemsetAsync(status, 0, 4, st));
    CUDA_OK(cudaMemcpyAsync(din, rows_in, nin * 4, cudaMemcpyHostToDevice, st));
    const int rc = atkg_approx_top_k(ATKG_F32, din, rows, p, ov, oi, dws, ws, status, st);
    if (rc) throw Inval(g_last_error);
    check_status_sync(status, st);
    CUDA_OK(cudaMemcpyAsync(out_vals, ov, no * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(out_idx, oi, no * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

int atkg_approx_top_k_at_recall_host(const float* rows_in, uint64_t rows, const atkg_plan_request* req,
                                     atkg_plan_result* plan_out, float* out_vals, uint32_t* out_idx) {
  return guarded([&] {
    const atkg_plan_result r = cached_plan(*req);
    if (plan_out) *plan_out = r;
    const atkg_params p = plan_params(*req, r);
    rethrow(atkg_approx_top_k_host(rows_in, rows, &p, out_vals, out_idx));
  });
}

int atkg_exact_top_k_host(const float* in, uint64_t n, uint32_t k, float* out_vals, uint32_t* out_idx) {
  return guarded([&] {
    if (k == 0) throw_inval("k must be >= 1");
    if (n > 0xffffffffull + 1) throw_inval("input exceeds the 32-bit index range");
    if (k > n) throw_inval("k must not exceed the input length");
    HostCtx& c = host_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    cudaStream_t st = c.s();
    float* din = static_cast<float*>(c.get(0, n * 4));
    float* ov = static_cast<float*>(c.get(1, (uint64_t)k * 4));
    uint32_t* oi = static_cast<uint32_t*>(c.get(2, (uint64_t)k * 4));
    void* dws = c.get(3, radix_ws_bytes(1, k) + 512);
    uint32_t* status = static_cast<uint32_t*>(c.get(4, 4));
    CUDA_OK(cudaMemsetAsync(status, 0, 4, st));
    CUDA_OK(cudaMemcpyAsync(din, in, n * 4, cudaMemcpyHostToDevice, st));
    DenseSrc<float> src{din, n};
    run_radix(src, 1, n, k, ov, oi, reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(dws))), status, st);
    check_status_sync(status, st);
    CUDA_OK(cudaMemcpyAsync(out_vals, ov, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(out_idx, oi, (uint64_t)k * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

// measure_recall (topk.cpp:275-297): |approx ∩ exact| / K by sorted merge
int atkg_measure_recall(const uint32_t* approx_idx, uint64_t approx_k, const uint32_t* exact_idx,
                        uint64_t exact_k, double* out) {
  return guarded([&] {
    if (approx_k != exact_k) throw_inval("recall needs results of equal size");
    if (approx_k == 0) throw_inval("recall of empty results is undefined");
    std::vector<uint32_t> a(approx_idx, approx_idx + approx_k), b(exact_idx, exact_idx + exact_k);
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    uint64_t hits = 0, i = 0, j = 0;
    while (i < a.size() && j < b.size()) {
      if (a[i] < b[j]) ++i;
      else if (b[j] < a[i]) ++j;
      else { ++hits; ++i; ++j; }
    }
    *out = static_cast<double>(hits) / static_cast<double>(exact_k);
  });
}

}  // extern "C"

// ===========================================================================
// streaming accumulator (Stage1Accumulator, include/atk/topk.hpp:68-94)
// ===========================================================================
struct atkg_accumulator {
  atkg_params p;
  uint64_t consumed = 0;
  bool summary_mode = false;
  uint32_t* summ = nullptr;   // summary mode: (2kp+2)*B words
  float* gv = nullptr;        // grid mode / candidates scratch
  uint32_t* gi = nullptr;
  uint32_t* status = nullptr;
  void* ws = nullptr;         // segment-kernel scratch for aligned bodies
  size_t ws_cap = 0;
};

namespace atkg {

template <int KP>
void launch_clear(uint32_t* summ, uint64_t B, cudaStream_t st) {
  summary_clear_kernel<KP><<<static_cast<unsigned>(ceil_div(B, 128)), 128, 0, st>>>(summ, B);
  check_launch();
}
template <typename T, int KP>
void launch_fold(uint32_t* summ, uint64_t B, const void* blk, uint64_t start, uint64_t count, uint32_t* status,
                 cudaStream_t st) {
  fold_summary_kernel<T, KP><<<static_cast<unsigned>(ceil_div(B, 128)), 128, 0, st>>>(
      summ, B, static_cast<const T*>(blk), start, count, status);
  check_launch();
}
void acc_fold(atkg_accumulator* a, int dtype, const void* blk, uint64_t start, uint64_t count, cudaStream_t st) {
  if (count == 0) return;
  const uint64_t B = a->p.num_buckets;
  if (a->summary_mode) {
    if (dtype == ATKG_BF16) { ATKG_KP_SWITCH(a->p.local_k, (launch_fold<__nv_bfloat16, K_>(a->summ, B, blk, start, count, a->status, st))); }
    else { ATKG_KP_SWITCH(a->p.local_k, (launch_fold<float, K_>(a->summ, B, blk, start, count, a->status, st))); }
  } else {
    if (dtype == ATKG_BF16)
      fold_grid_kernel<__nv_bfloat16><<<static_cast<unsigned>(ceil_div(B, 128)), 128, 0, st>>>(
          a->gv, a->gi, B, a->p.local_k, static_cast<const __nv_bfloat16*>(blk), start, count, a->status);
    else
      fold_grid_kernel<float><<<static_cast<unsigned>(ceil_div(B, 128)), 128, 0, st>>>(
          a->gv, a->gi, B, a->p.local_k, static_cast<const float*>(blk), start, count, a->status);
    check_launch();
  }
}

}  // namespace atkg

extern "C" {

int atkg_accumulator_create(const atkg_params* p, atkg_accumulator** out) {
  return guarded([&] {
    validate(*p);
    auto* a = new atkg_accumulator();
    a->p = *p;
    const uint64_t B = p->num_buckets, kp = p->local_k;
    a->summary_mode = kp_specialised(p->local_k);
    CUDA_OK(cudaMalloc(&a->status, 4));
    CUDA_OK(cudaMemset(a->status, 0, 4));
    CUDA_OK(cudaMalloc(&a->gv, kp * B * 4));
    CUDA_OK(cudaMalloc(&a->gi, kp * B * 4));
    if (a->summary_mode) {
      CUDA_OK(cudaMalloc(&a->summ, (2 * kp + 2) * B * 4));
      ATKG_KP_SWITCH(p->local_k, (launch_clear<K_>(a->summ, B, 0)));
    } else {
      grid_init_kernel<<<static_cast<unsigned>(ceil_div(kp * B, 256)), 256>>>(a->gv, a->gi, kp * B);
      check_launch();
    }
    CUDA_OK(cudaDeviceSynchronize());
    *out = a;
  });
}

// consume(): positions consumed()..+len-1, any length and alignment
// (topk.cpp:123-172).  The bucket-aligned body of a large block runs through
// the segment kernels; ragged edges and odd layouts fold element-wise.
int atkg_accumulator_consume(atkg_accumulator* a, int dtype, const void* d_block, uint64_t len, void* stream) {
  return guarded([&] {
    if (a->consumed + len > a->p.n) throw_inval("stage 1 fed more than n elements");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t B = a->p.num_buckets;
    const uint64_t esz = dtype == ATKG_BF16 ? 2 : 4;
    const char* blk = static_cast<const char*>(d_block);
    uint64_t start = a->consumed;
    const uint64_t end = start + len;
    if (a->summary_mode && len >= 4 * B) {
      const uint64_t h = std::min(end, ceil_div(start, B) * B);
      acc_fold(a, dtype, blk, start, h - start, st);
      const uint64_t body = (end - h) / B * B;
      const void* bptr = blk + (h - start) * esz;
      const S1Plan pl = plan_stage1(dtype, bptr, 1, body, body, B, a->p.local_k);
      if (body > 0 && pl.kind != S1Plan::kGeneric) {
        const size_t words = (2ull * a->p.local_k + 2) * B * 4;
        const size_t need = stage1_ws_bytes(pl, 1, B, a->p.local_k) + align_up(words);
        if (a->ws_cap < need) {
          if (a->ws) CUDA_OK(cudaFree(a->ws));
          CUDA_OK(cudaMalloc(&a->ws, need));
          a->ws_cap = need;
        }
        uint32_t* parts = static_cast<uint32_t*>(a->ws);
        uint32_t* body_summ = reinterpret_cast<uint32_t*>(static_cast<char*>(a->ws) + stage1_ws_bytes(pl, 1, B, a->p.local_k));
        run_stage1_summaries(dtype, pl, bptr, 1, body, B, a->p.local_k, h, parts, a->status, st);
        run_merge(pl, a->p.local_k, parts, 1, B, nullptr, nullptr, 0, body_summ, st);
        // acc = merge(acc, body) in index order
        dispatch_merge(a->p.local_k, body_summ, 1, 1, B, nullptr, nullptr, 0, a->summ, st, a->summ);
        acc_fold(a, dtype, blk + (h + body - start) * esz, h + body, end - h - body, st);
      } else {
        acc_fold(a, dtype, blk + (h - start) * esz, h, end - h, st);
      }
    } else {
      acc_fold(a, dtype, blk, start, len, st);
    }
    a->consumed = end;
  });
}

uint64_t atkg_accumulator_consumed(const atkg_accumulator* a) { return a->consumed; }

int atkg_accumulator_candidates(atkg_accumulator* a, float* d_vals, uint32_t* d_idx, void* stream) {
  return guarded([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t B = a->p.num_buckets, kp = a->p.local_k;
    if (a->summary_mode) {
      dispatch_merge(a->p.local_k, a->summ, 1, 1, B, d_vals, d_idx, kp * B, nullptr, st);
    } else {
      CUDA_OK(cudaMemcpyAsync(d_vals, a->gv, kp * B * 4, cudaMemcpyDeviceToDevice, st));
      CUDA_OK(cudaMemcpyAsync(d_idx, a->gi, kp * B * 4, cudaMemcpyDeviceToDevice, st));
    }
    check_status_sync(a->status, st);
  });
}

int atkg_accumulator_consume_host(atkg_accumulator* a, const float* block, uint64_t len) {
  return guarded([&] {
    if (a->consumed + len > a->p.n) throw_inval("stage 1 fed more than n elements");
    for (uint64_t i = 0; i < len; ++i)  // topk.cpp:126: NaN is rejected up front
      if (block[i] != block[i]) throw NanInput();
    if (len == 0) return;
    HostCtx& c = host_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    cudaStream_t st = c.s();
    float* d = static_cast<float*>(c.get(0, len * 4));
    CUDA_OK(cudaMemcpyAsync(d, block, len * 4, cudaMemcpyHostToDevice, st));
    rethrow(atkg_accumulator_consume(a, ATKG_F32, d, len, st));
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

int atkg_accumulator_candidates_host(atkg_accumulator* a, float* vals, uint32_t* idx) {
  return guarded([&] {
    HostCtx& c = host_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    cudaStream_t st = c.s();
    const uint64_t g = a->p.num_buckets * (uint64_t)a->p.local_k;
    float* dv = static_cast<float*>(c.get(1, g * 4));
    uint32_t* di = static_cast<uint32_t*>(c.get(2, g * 4));
    rethrow(atkg_accumulator_candidates(a, dv, di, st));
    CUDA_OK(cudaMemcpyAsync(vals, dv, g * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(idx, di, g * 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

void atkg_accumulator_destroy(atkg_accumulator* a) {
  if (!a) return;
  cudaFree(a->summ);
  cudaFree(a->gv);
  cudaFree(a->gi);
  cudaFree(a->status);
  cudaFree(a->ws);
  delete a;
}

}  // extern "C"
