// internal.hpp -- host-side helpers shared by the library's translation
// units (atkg_api.cu, fused_gemm.cu); not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "host_common.hpp"

namespace atkg {

#define CUDA_OK(x)                                                                           \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// launch counter (atkg_launch_count) and the stage-1 event brackets
// (atkg_profile_begin/end)
extern std::atomic<uint64_t> g_launches;
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // pairs
  size_t used = 0;
  uint32_t every = 1, seen = 0;  // bracket every `every`-th launch
  bool open = false;
  void bracket_begin(cudaStream_t st) {
    if (!on) return;
    open = (seen++ % every) == 0;
    if (!open) return;
    if (used + 2 > ev.size()) {
      for (int q = 0; q < 2; ++q) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreate(&e));
        ev.push_back(e);
      }
    }
    CUDA_OK(cudaEventRecord(ev[used], st));
  }
  void bracket_end(cudaStream_t st) {
    if (!on || !open) return;
    open = false;
    CUDA_OK(cudaEventRecord(ev[used + 1], st));
    used += 2;
  }
};
extern Profiler g_prof;

inline void check_launch() {
  CUDA_OK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// SM count of the calling thread's current device (cached per device)
int sm_count();
int current_device();
// raises a kernel's dynamic shared-memory limit to >= bytes on the current
// device (the attribute is per device; cached per (device, kernel))
void ensure_smem(const void* kern, size_t bytes);
template <typename K>
inline void ensure_smem_fn(K* kern, size_t bytes) { ensure_smem(reinterpret_cast<const void*>(kern), bytes); }

// Path-selection and tuning overrides (atkg_set_option): tests force the
// rare fallbacks and alternative dispatch paths through these; every
// default is the measured production choice.  Process-wide.
uint64_t opt(const char* name, uint64_t dflt);

uint64_t align_up(uint64_t x, uint64_t a = 256);
uint32_t next_pow2(uint64_t x);
void validate(const atkg_params& p);
uint64_t select_ws_bytes(uint64_t rows, uint64_t count, uint32_t k);
void run_select(const float* vals, const uint32_t* idx, uint64_t rows, uint64_t count, uint64_t stride, uint32_t k,
                uint64_t limit, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st);

// row-threshold approx_top_k for rows that fit in shared memory (rowthr.cu)
struct ThrPlan {
  bool ok = false;
  uint32_t cap = 512, rsel = 1, region = 0;
  size_t smem = 0;
};
ThrPlan plan_rowthr(int dtype, const void* in, uint64_t n, uint64_t B, uint32_t kp, uint32_t k);
uint64_t rowthr_ws_bytes(uint64_t rows, const ThrPlan& tp);
void run_rowthr(int dtype, const ThrPlan& tp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp,
                uint32_t k, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st);

// short rows held in shared memory, guaranteed row threshold (shortrow.cu)
struct SrPlan {
  bool ok = false;
  uint32_t npart = 1, pl = 1, cap = 0, slot_bytes = 0, P = 0, sub_shift = 0, grid = 0, per_sm = 0;
  size_t smem = 0;
  uint64_t ws_bytes = 0;
};
SrPlan plan_short(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                  bool for_size = false);
// row_list / row_count (device): only those rows (the rows rowmax1.cu could not settle)
void run_short(int dtype, const SrPlan& sp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp,
               uint32_t k, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st,
               const uint32_t* row_list = nullptr, const uint32_t* row_count = nullptr);

// K' = 1 on the register row stream; the rows it cannot settle go to run_short (rowmax1.cu)
struct RmPlan {
  bool ok = false;
  uint32_t S = 0, cpl = 0, warps = 0, grid = 0;
  size_t smem = 0;
  SrPlan fallback;
  uint64_t ws_bytes = 0;  // the fallback's scratch | counter | row list
};
RmPlan plan_rowmax1(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                    bool for_size = false);
void run_rowmax1(const RmPlan& rp, int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t k,
                 float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st);

// one warp per bf16 row held in shared memory (rowwarp.cu)
struct RwPlan {
  bool ok = false;
  uint32_t cpl = 1, w = 4, cap = 0, P = 0, slot_bytes = 0, sub_shift = 0, grid = 0;
  size_t smem = 0;
  uint64_t ws_bytes = 0;
};
RwPlan plan_rowwarp(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                    bool for_size = false);
void run_rowwarp(const RwPlan& rp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                 float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st);

// one warp per bf16 row streamed once into registers, B = 128, K' = 4 (rowreg.cu)
struct RgPlan {
  bool ok = false;
  uint32_t S = 0, warps = 0, grid = 0;
  size_t smem = 0;
};
RgPlan plan_rowreg(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                   bool for_size = false);
void run_rowreg(const RgPlan& rp, const void* in, uint64_t rows, uint32_t k, float* ov, uint32_t* oi,
                uint32_t* status, cudaStream_t st);
// the same stream for the C3 sweep shapes with 1024 candidates per row (rowregx.cu)
RgPlan plan_rowregx(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                    bool for_size = false);
void run_rowregx(const RgPlan& rp, const void* in, uint64_t rows, uint64_t B, uint32_t kp, uint32_t k, float* ov,
                 uint32_t* oi, uint32_t* status, cudaStream_t st);

// stage 2 by counting-sort ranks for 128 < count <= 1024 (streamthr.cu);
// false if not applicable
bool run_select_ranked(const float* vals, const uint32_t* idx, uint64_t rows, uint64_t count, uint64_t stride,
                       uint32_t k, uint64_t limit, float* ov, uint32_t* oi, uint32_t* status, cudaStream_t st);

// threshold-stream approx_top_k for long rows (streamthr.cu)
struct StPlan {
  bool ok = false, giant = false;
  uint64_t vtot = 0, psz = 0, ws_bytes = 0;
  uint32_t G = 0, smax = 1, slot_bytes = 32768, ns = 3, ecap = 4096;
  float rfac = 0.f, lfac = 0.f, cfac = 0.f;
  size_t smem_stream = 0, smem_fin = 0;
};
// for_size: ignore the ATKG_NO_STREAMTHR switch (workspace sizing covers every path)
StPlan plan_streamthr(int dtype, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp, uint32_t k,
                      bool for_size = false, double t_scale = 1.0);
double streamthr_target(uint64_t n, uint64_t B, uint32_t kp, uint32_t k);
void run_stream_only(int dtype, const StPlan& sp, const void* in, uint64_t n, void* ws, uint32_t* status,
                     cudaStream_t st);
void run_slice_payload(const StPlan& sp, const uint32_t* slots, uint32_t cap, uint64_t index_offset,
                       const uint32_t* status, uint32_t* payload, cudaStream_t st);
void run_payload_finish(const uint32_t* payloads, uint32_t parts, uint32_t slot_cap, uint64_t n, uint64_t B,
                        uint32_t kp, uint32_t k, float* ov, uint32_t* oi, uint32_t* gate, uint32_t* status,
                        cudaStream_t st);
void run_streamthr(int dtype, const StPlan& sp, const void* in, uint64_t rows, uint64_t n, uint64_t B, uint32_t kp,
                   uint32_t k, float* ov, uint32_t* oi, void* ws, uint32_t* status, cudaStream_t st);

}  // namespace atkg
