// shard.cu -- one row sliced across GPUs (the sharded giant row, C5; SURVEY
// 8(e)): per-slice threshold-stream payloads, their exchange, the merge, and
// the C-ABI entry that runs the whole exchange over an NCCL communicator.
//
// The reference consumes a row's blocks in index order through
// Stage1Accumulator::consume (include/atk/topk.hpp:68-94, topk.cpp:123-172)
// and returns approx_top_k (topk.cpp:238-258); the slices here are those
// blocks, one per GPU.
//   fast path   every rank runs the threshold stream over its slice
//               (streamthr.cuh) and folds the slots into one payload: every
//               element of the slice >= the slice threshold L_s, global
//               positions.  The payloads are all-gathered; every rank runs
//               the per-row finish on them with L = max_s L_s -- exact, as
//               within one GPU (the threshold-stream argument).
//   fallback    when a payload is bad (slot overflow, NaN, too many entries)
//               or the candidates >= L do not reach K, every rank sees the
//               same gathered data and takes the exact path together: the
//               associative per-bucket summaries (atkg_stage1_summary),
//               all-gathered and merged in index order (summary words + one
//               NaN word per rank).
// NCCL is loaded at run time (dlopen, the process's own libnccl.so.2 if one
// is loaded): the library keeps no link-time dependency on it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"
#include "stconst.hpp"

namespace atkg {

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);  // the one already in the process
      if (!n.h) n.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(n.h, "ncclAllGather"));
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(n.h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
  });
  if (!n.h || !n.all_gather || !n.get_unique_id || !n.comm_init_rank || !n.comm_destroy)
    throw Unsupported("NCCL (libnccl.so.2) is not available");
  return n;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* m = nccl().error_string ? nccl().error_string(r) : "error";
    throw CudaError(std::string(what) + ": " + m);
  }
}

// entries a slice payload holds: every element of the slice >= its
// threshold, ~2x its share of the row target T with margin
uint32_t payload_cap(const atkg_params& p, uint32_t parts) {
  const double T = streamthr_target(p.n, p.num_buckets, p.local_k, p.global_k);
  const double want = 4.0 * T / std::max<uint32_t>(parts, 1) + 512.0;
  uint32_t cap = 1024;
  while (cap < want && cap < (1u << 20)) cap <<= 1;
  return cap;
}

void check_slice(const atkg_params& p, uint64_t len, uint64_t index_offset) {
  const uint64_t B = p.num_buckets;
  if (len % B != 0 || index_offset % B != 0) throw_inval("slice length and offset must be multiples of num_buckets");
  if (index_offset + len > p.n) throw_inval("slice exceeds the row");
  if (len == 0) throw_inval("empty slice");
}

StPlan slice_plan(int dtype, const void* d_slice, uint64_t len, const atkg_params& p, uint32_t parts) {
  // each slice keeps ~1.5x its share of the row's target (the max of the
  // slice thresholds stays below the row's safe level)
  const StPlan sp = plan_streamthr(dtype, d_slice, 1, len, p.num_buckets, p.local_k, p.global_k, false,
                                   1.5 / std::max<uint32_t>(parts, 1));
  return sp;
}

}  // namespace

uint64_t slice_payload_words(const atkg_params& p, uint32_t parts) { return 2ull + 2ull * payload_cap(p, parts); }

}  // namespace atkg

using namespace atkg;

extern "C" {

int atkg_slice_payload_words(const atkg_params* p, uint32_t parts, size_t* words) {
  return guarded([&] {
    validate(*p);
    if (parts == 0) throw_inval("need at least one slice");
    *words = slice_payload_words(*p, parts);
  });
}

int atkg_slice_payload_workspace(int dtype, uint64_t len, const atkg_params* p, uint32_t parts, size_t* bytes) {
  return guarded([&] {
    validate(*p);
    const void* aligned = reinterpret_cast<const void*>(static_cast<uintptr_t>(256));
    const StPlan sp = plan_streamthr(dtype, aligned, 1, len, p->num_buckets, p->local_k, p->global_k, true,
                                     1.5 / std::max<uint32_t>(parts, 1));
    *bytes = (sp.ok ? sp.ws_bytes : 0) + 512;
  });
}

int atkg_slice_payload(int dtype, const void* d_slice, uint64_t len, uint64_t index_offset, const atkg_params* p,
                       uint32_t parts, uint32_t* d_payload, void* d_ws, size_t ws_bytes, uint32_t* d_status,
                       void* stream) {
  return guarded([&] {
    validate(*p);
    check_slice(*p, len, index_offset);
    if (parts == 0) throw_inval("need at least one slice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t cap = payload_cap(*p, parts);
    const StPlan sp = slice_plan(dtype, d_slice, len, *p, parts);
    if (!sp.ok) {  // a slice the stream does not take: a bad payload sends every rank to the exact path
      const uint32_t hdr[2] = {kStBadCount, 0u};
      CUDA_OK(cudaMemcpyAsync(d_payload, hdr, 8, cudaMemcpyHostToDevice, st));
      CUDA_OK(cudaStreamSynchronize(st));
      return;
    }
    if (ws_bytes < sp.ws_bytes + 256) throw_inval("workspace smaller than atkg_slice_payload_workspace");
    void* sws = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(d_ws)));
    run_stream_only(dtype, sp, d_slice, len, sws, d_status, st);
    run_slice_payload(sp, static_cast<const uint32_t*>(sws), cap, index_offset, d_status, d_payload, st);
  });
}

int atkg_payload_merge_top_k(const uint32_t* d_payloads, uint32_t parts, const atkg_params* p, float* d_out_vals,
                             uint32_t* d_out_idx, uint32_t* d_gate, uint32_t* d_status, void* stream) {
  return guarded([&] {
    validate(*p);
    if (parts == 0 || parts > kStMaxRowPieces) throw_inval("slice count out of range");
    if (p->local_k != 1 && p->local_k != 2 && p->local_k != 4 && p->local_k != 8)
      throw Unsupported("local_k has no specialised finish kernel");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_OK(cudaMemsetAsync(d_gate, 0, 4, st));
    run_payload_finish(d_payloads, parts, payload_cap(*p, parts), p->n, p->num_buckets, p->local_k, p->global_k,
                       d_out_vals, d_out_idx, d_gate, d_status, st);
  });
}

int atkg_nccl_unique_id(char out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_ok(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
  });
}

int atkg_nccl_comm_init(void** comm, int nranks, const char id[128], int rank) {
  return guarded([&] {
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    ncclComm_t c = nullptr;
    nccl_ok(nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    *comm = c;
  });
}

int atkg_nccl_comm_destroy(void* comm) {
  return guarded([&] { nccl_ok(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy"); });
}

int atkg_sharded_workspace_size(int dtype, uint64_t len, const atkg_params* p, uint32_t world, size_t* bytes) {
  return guarded([&] {
    validate(*p);
    if (world == 0) throw_inval("need at least one rank");
    const uint64_t words = slice_payload_words(*p, world);
    size_t pay_ws = 0, sum_ws = 0, merge_ws = 0;
    rethrow(atkg_slice_payload_workspace(dtype, len, p, world, &pay_ws));
    atkg_params sp = *p;
    sp.n = len;
    sp.global_k = 1;
    sp.lane_multiple = 1;
    rethrow(atkg_workspace_size(ATKG_OP_SUMMARY, dtype, 1, &sp, &sum_ws));
    rethrow(atkg_workspace_size(ATKG_OP_MERGE, dtype, 1, p, &merge_ws));
    const uint64_t sw = ATKG_SUMMARY_WORDS(p) + 1;
    *bytes = align_up((1 + world) * words * 4) + 256 + align_up((1 + 2 * world) * sw * 4) +
             std::max(pay_ws, std::max(sum_ws, merge_ws)) + 512;
  });
}

int atkg_sharded_approx_top_k(int dtype, const void* d_slice, uint64_t len, uint64_t index_offset,
                              const atkg_params* p, void* nccl_comm, uint32_t world, float* d_out_vals,
                              uint32_t* d_out_idx, void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
  return guarded([&] {
    validate(*p);
    check_slice(*p, len, index_offset);
    if (world == 0) throw_inval("need at least one rank");
    size_t need = 0;
    rethrow(atkg_sharded_workspace_size(dtype, len, p, world, &need));
    if (ws_bytes < need) throw_inval("workspace smaller than atkg_sharded_workspace_size");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    const uint64_t words = slice_payload_words(*p, world);
    char* w = reinterpret_cast<char*>(align_up(reinterpret_cast<uintptr_t>(d_ws)));
    uint32_t* mine = reinterpret_cast<uint32_t*>(w);
    uint32_t* all = mine + words;
    w += align_up((1 + world) * words * 4);
    uint32_t* gate = reinterpret_cast<uint32_t*>(w);
    w += 256;
    const uint64_t sw = ATKG_SUMMARY_WORDS(p) + 1;  // summary | NaN word
    uint32_t* smine = reinterpret_cast<uint32_t*>(w);
    uint32_t* sall = smine + sw;                  // [world][sw] gathered
    uint32_t* scomp = sall + (uint64_t)world * sw;  // [world][sw - 1] the summaries, consecutive
    w += align_up((1 + 2 * world) * sw * 4);
    void* scratch = w;
    const size_t scratch_bytes = ws_bytes - (static_cast<size_t>(w - static_cast<char*>(d_ws)));
    // fast path: threshold-stream payloads
    rethrow(atkg_slice_payload(dtype, d_slice, len, index_offset, p, world, mine, scratch, scratch_bytes, d_status,
                               stream));
    nccl_ok(nccl().all_gather(mine, all, words, ncclUint32, comm, st), "ncclAllGather");
    rethrow(atkg_payload_merge_top_k(all, world, p, d_out_vals, d_out_idx, gate, d_status, stream));
    uint32_t g = 0;
    CUDA_OK(cudaMemcpyAsync(&g, gate, 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (!g) return;
    // exact path, on every rank together: per-bucket summaries + NaN word
    CUDA_OK(cudaMemsetAsync(d_status, 0, 4, st));
    rethrow(atkg_stage1_summary(dtype, d_slice, len, index_offset, p, smine, scratch, scratch_bytes, d_status,
                                stream));
    CUDA_OK(cudaMemcpyAsync(smine + sw - 1, d_status, 4, cudaMemcpyDeviceToDevice, st));
    nccl_ok(nccl().all_gather(smine, sall, sw, ncclUint32, comm, st), "ncclAllGather");
    std::vector<uint32_t> flags(world);
    for (uint32_t r = 0; r < world; ++r)
      CUDA_OK(cudaMemcpyAsync(&flags[r], sall + r * sw + sw - 1, 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    for (uint32_t r = 0; r < world; ++r)
      if (flags[r] & ATKG_FLAG_NAN) throw NanInput();
    // merge expects consecutive summaries: drop the NaN words
    CUDA_OK(cudaMemcpy2DAsync(scomp, (sw - 1) * 4, sall, sw * 4, (sw - 1) * 4, world, cudaMemcpyDeviceToDevice, st));
    rethrow(atkg_summary_merge_top_k(scomp, world, p, nullptr, nullptr, d_out_vals, d_out_idx, scratch, scratch_bytes,
                                     d_status, stream));
  });
}

}  // extern "C"
