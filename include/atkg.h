/*
 * atkg.h -- C ABI of the B200-native two-stage approximate top-k
 * (arXiv 2506.04165), the drop-in boundary for the reference `atk` core.
 *
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference/proj/core):
 *
 *   atkg_validate                 AlgoParams::validate        include/atk/params.hpp:40, src/topk.cpp:54-67
 *   atkg_validate_analysis        AlgoParams::validate_analysis  params.hpp:47, topk.cpp:69-76
 *   atkg_stage1                   stage1_partial_reduce       include/atk/topk.hpp:98-99, src/topk.cpp:178-186
 *   atkg_select_candidates        select_top_k_candidates     topk.hpp:109-112, topk.cpp:219-236
 *   atkg_approx_top_k             approx_top_k / _batch       topk.hpp:117-124, topk.cpp:238-273
 *   atkg_exact_top_k              exact_top_k                 topk.hpp:104, topk.cpp:206-217
 *   atkg_measure_recall           measure_recall              topk.hpp:128, topk.cpp:275-297
 *   atkg_stage1_summary /
 *   atkg_summary_merge_top_k      Stage1Accumulator::consume over a slice of one
 *                                 row + the cross-slice merge  topk.hpp:68-94, topk.cpp:123-172
 *   atkg_accumulator_*            Stage1Accumulator           topk.hpp:68-94
 *   atkg_exact_expected_recall    exact_expected_recall       include/atk/recall.hpp:39, src/recall.cpp:76-100
 *   atkg_mc_expected_recall       mc_expected_recall          recall.hpp:45-46, recall.cpp:102-154
 *   atkg_mc_expected_recall_adaptive  mc_expected_recall_adaptive  recall.hpp:50-51, recall.cpp:156-165
 *   atkg_legal_bucket_counts      legal_bucket_counts         include/atk/planner.hpp:61-62, src/planner.cpp:59-77
 *   atkg_select_parameters        select_parameters           planner.hpp:66-67, planner.cpp:79-147
 *   atkg_fused_gemm_top_k         mips_fused semantics (stage 1 in the matmul epilogue)
 *                                 include/atk/mips.hpp:50-52, src/mips.cpp:138-193
 *   atkg_approx_top_k_at_recall   select_parameters + PlanResult::params + approx_top_k
 *                                 planner.hpp:38,66-67, topk.hpp:117-124
 *   atkg_slice_payload /
 *   atkg_payload_merge_top_k /
 *   atkg_sharded_approx_top_k     approx_top_k of one row whose blocks live on different
 *                                 GPUs (Stage1Accumulator::consume order, topk.hpp:68-94)
 *
 * Conventions
 *   - Device entry points take DEVICE pointers and a cudaStream_t passed as
 *     void*; they only enqueue work (no host synchronisation).  Outputs are
 *     caller-owned.  Temporary storage is caller-supplied through `ws`
 *     (size from atkg_workspace_size), so concurrent streams never share state.
 *   - NaN detection is a device flag: kernels OR ATKG_FLAG_NAN into *d_status
 *     (a caller-zeroed uint32 in device memory).  atkg_check_status()
 *     synchronises the stream and maps the flags to ATKG_ENAN
 *     ("input contains NaN", the reference's std::invalid_argument).
 *   - *_host entry points are the drop-in form of the reference's span API:
 *     host buffers in, host buffers out, synchronous, errors returned with
 *     the reference's exact messages (atkg_last_error()).
 *   - Indices are uint32 element positions in the source row, identical to
 *     the reference's std::uint32_t (bit-identical to int32 for n < 2^31).
 *   - Values are fp32.  bf16 inputs are upcast exactly.
 */
#ifndef ATKG_H_
#define ATKG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; messages via atkg_last_error() (thread-local) */
#define ATKG_OK 0
#define ATKG_EINVAL 1         /* std::invalid_argument */
#define ATKG_ENAN 2           /* std::invalid_argument("input contains NaN") */
#define ATKG_EINFEASIBLE 3    /* atk::NoFeasibleConfigError */
#define ATKG_ECUDA 4          /* CUDA runtime failure */
#define ATKG_EUNSUPPORTED 5   /* shape outside what the device path implements */
#define ATKG_EFORMAT 6        /* atk::DatasetFormatError (dataset.hpp:14-16) */

#define ATKG_FLAG_NAN 1u

/* element types of the input rows */
#define ATKG_F32 0
#define ATKG_BF16 1

/* operations for atkg_workspace_size */
#define ATKG_OP_STAGE1 0
#define ATKG_OP_APPROX 1
#define ATKG_OP_SELECT 2
#define ATKG_OP_EXACT 3
#define ATKG_OP_SUMMARY 4
#define ATKG_OP_MERGE 5

/* AlgoParams (include/atk/params.hpp:20-48); lane_multiple default 128 */
typedef struct atkg_params {
  uint64_t n;
  uint64_t num_buckets;
  uint32_t local_k;
  uint32_t global_k;
  uint32_t lane_multiple;
} atkg_params;

const char* atkg_last_error(void);
const char* atkg_version(void);
/* Selects the CUDA device for subsequent calls on this host thread
 * (cudaSetDevice of the library's runtime). */
int atkg_set_device(int device);

/* Process-wide path-selection overrides, for tests and tuning only (no
 * effect on results: every path is bit-identical).  Unset options keep the
 * measured production choice; value UINT64_MAX resets one.  Names:
 *   no_streamthr, st_force_slow, st_giant_n (threshold stream), no_rowres,
 *   rowthr / no_rowthr, short / no_short / short_force_slow,
 *   rowwarp / no_rowwarp / rowwarp_force_slow (short-row kernels),
 *   fused_path (0 auto, 1 unfused), gemm_cg, sim_host_gen, no_pdl. */
int atkg_set_option(const char* name, uint64_t value);
uint64_t atkg_get_option(const char* name, uint64_t dflt);

int atkg_validate(const atkg_params* p);
int atkg_validate_analysis(const atkg_params* p);

/* ---- device entry points ------------------------------------------------ */

/* Bytes of caller-supplied workspace needed by `op`.  For ATKG_OP_SELECT,
 * p->n is the candidate count per row and p->global_k the k. For
 * ATKG_OP_EXACT, p->n is the row length and p->global_k the k. */
int atkg_workspace_size(int op, int dtype, uint64_t rows, const atkg_params* p,
                        size_t* bytes);

/* stage1_partial_reduce over `rows` contiguous rows of p->n elements:
 * writes the bucket-minor grid [rows][local_k][num_buckets] (topk.hpp:59-67),
 * bit-identical to the reference (Alg. 1 tie semantics, unfilled slots
 * {-inf, 0}). */
int atkg_stage1(int dtype, const void* d_in, uint64_t rows, const atkg_params* p,
                float* d_grid_vals, uint32_t* d_grid_idx, void* d_ws, size_t ws_bytes,
                uint32_t* d_status, void* stream);

/* select_top_k_candidates per row: candidates row r live at
 * d_vals[r*stride .. r*stride+count); indices >= index_limit are dropped;
 * output [rows][k] sorted by (value desc, index asc), -0.0 emitted as +0.0.
 * Rows with fewer than k surviving candidates raise ATKG_EINVAL
 * ("fewer candidates than k") at atkg_check_status. */
int atkg_select_candidates(const float* d_vals, const uint32_t* d_idx, uint64_t rows,
                           uint64_t count, uint64_t stride, uint32_t k, uint64_t index_limit,
                           float* d_out_vals, uint32_t* d_out_idx, void* d_ws, size_t ws_bytes,
                           uint32_t* d_status, void* stream);

/* approx_top_k_batch: stage 1 + stage 2 per row -> [rows][global_k].
 * Asynchronous on `stream`, except for rows longer than 2^24 elements: the
 * threshold stream then reads a 4-byte device gate after its finish kernel
 * (one stream synchronisation) and reruns the exact path if a row's
 * threshold failed -- the results are bit-identical either way. */
int atkg_approx_top_k(int dtype, const void* d_in, uint64_t rows, const atkg_params* p,
                      float* d_out_vals, uint32_t* d_out_idx, void* d_ws, size_t ws_bytes,
                      uint32_t* d_status, void* stream);

/* exact_top_k per row (recall measurement only). */
int atkg_exact_top_k(int dtype, const void* d_in, uint64_t rows, uint64_t n, uint32_t k,
                     float* d_out_vals, uint32_t* d_out_idx, void* d_ws, size_t ws_bytes,
                     uint32_t* d_status, void* stream);

/* Slice summaries for sharding one row (or streaming it in blocks).
 * The slice holds elements [index_offset, index_offset + len) of a row of
 * p->n elements; index_offset and len are multiples of num_buckets.
 * The summary of every bucket (ATKG_SUMMARY_WORDS(p) uint32 words) is exact
 * and associative: atkg_summary_merge_top_k over the G slices' summaries,
 * in index order, reproduces the reference stage-1 grid and its top-k
 * bit-for-bit.  This is what crosses NVLink in the sharded giant-row path. */
#define ATKG_SUMMARY_WORDS(p) ((2ull * (p)->local_k + 2ull) * (p)->num_buckets)
int atkg_stage1_summary(int dtype, const void* d_slice, uint64_t len, uint64_t index_offset,
                        const atkg_params* p, uint32_t* d_summary, void* d_ws, size_t ws_bytes,
                        uint32_t* d_status, void* stream);
/* Merges `parts` consecutive summaries (each ATKG_SUMMARY_WORDS words, in
 * index order).  Writes the Alg. 1 grid if d_grid_vals != NULL, and the
 * top-global_k if d_out_vals != NULL. */
int atkg_summary_merge_top_k(const uint32_t* d_summaries, uint32_t parts, const atkg_params* p,
                             float* d_grid_vals, uint32_t* d_grid_idx, float* d_out_vals,
                             uint32_t* d_out_idx, void* d_ws, size_t ws_bytes,
                             uint32_t* d_status, void* stream);

/* ---- one row sliced across GPUs: threshold-stream payloads --------------
 * The fast form of the slice exchange (the same reference contract as the
 * summaries above).  Each rank reduces its slice to a payload of
 * atkg_slice_payload_words(p, parts) uint32 words -- every element of the
 * slice >= the slice's threshold, global positions -- a few KB instead of
 * the exact summaries, at the streaming speed of the threshold stream.
 * atkg_payload_merge_top_k over the `parts` payloads (index order) writes the
 * top global_k, or sets *d_gate (device word) when the payloads cannot
 * settle the row (overflow, NaN, too few candidates); every rank sees the
 * same payloads, so all of them then take the exact summary path together. */
int atkg_slice_payload_words(const atkg_params* p, uint32_t parts, size_t* words);
int atkg_slice_payload_workspace(int dtype, uint64_t len, const atkg_params* p, uint32_t parts,
                                 size_t* bytes);
int atkg_slice_payload(int dtype, const void* d_slice, uint64_t len, uint64_t index_offset,
                       const atkg_params* p, uint32_t parts, uint32_t* d_payload, void* d_ws,
                       size_t ws_bytes, uint32_t* d_status, void* stream);
int atkg_payload_merge_top_k(const uint32_t* d_payloads, uint32_t parts, const atkg_params* p,
                             float* d_out_vals, uint32_t* d_out_idx, uint32_t* d_gate,
                             uint32_t* d_status, void* stream);

/* The whole sharded approx_top_k of one row over an NCCL communicator
 * (ncclComm_t passed as void*; rank r of `world` holds elements
 * [index_offset, index_offset + len)): slice payload -> ncclAllGather ->
 * merge; when the gate is set, exact summaries -> ncclAllGather -> merge.
 * Every rank returns the same top global_k, bit-identical to approx_top_k on
 * the whole row (topk.cpp:238-258).  Synchronises `stream` once (the gate).
 * NCCL is loaded at run time (libnccl.so.2, the process's own if loaded);
 * the helpers below create communicators with that same library. */
int atkg_sharded_workspace_size(int dtype, uint64_t len, const atkg_params* p, uint32_t world,
                                size_t* bytes);
int atkg_sharded_approx_top_k(int dtype, const void* d_slice, uint64_t len, uint64_t index_offset,
                              const atkg_params* p, void* nccl_comm, uint32_t world,
                              float* d_out_vals, uint32_t* d_out_idx, void* d_ws, size_t ws_bytes,
                              uint32_t* d_status, void* stream);
int atkg_nccl_unique_id(char out[128]);
int atkg_nccl_comm_init(void** comm, int nranks, const char id[128], int rank);
int atkg_nccl_comm_destroy(void* comm);

/* Synchronises `stream`, reads *d_status and maps the flags to a status
 * code (ATKG_ENAN / ATKG_EINVAL with the reference message). */
int atkg_check_status(const uint32_t* d_status, void* stream);

/* ---- streaming accumulator (Stage1Accumulator, topk.hpp:68-94) ---------- */
typedef struct atkg_accumulator atkg_accumulator;
int atkg_accumulator_create(const atkg_params* p, atkg_accumulator** out);
/* consume the next `len` elements (positions consumed()..+len-1) of the row
 * from device memory; any length, any alignment; stream-ordered */
int atkg_accumulator_consume(atkg_accumulator* acc, int dtype, const void* d_block,
                             uint64_t len, void* stream);
uint64_t atkg_accumulator_consumed(const atkg_accumulator* acc);
/* grid [local_k][num_buckets] (device pointers), synchronises */
int atkg_accumulator_candidates(atkg_accumulator* acc, float* d_vals, uint32_t* d_idx,
                                void* stream);
/* host-buffer forms (synchronous): consume() a host block (NaN rejected as
 * in topk.cpp:126), candidates() into host arrays of num_buckets*local_k */
int atkg_accumulator_consume_host(atkg_accumulator* acc, const float* block, uint64_t len);
int atkg_accumulator_candidates_host(atkg_accumulator* acc, float* vals, uint32_t* idx);
void atkg_accumulator_destroy(atkg_accumulator* acc);

/* ---- fused GEMM + stage 1 (C4: x[M,Kd] . W[Kd,N] -> top-k per row) ------ */
/* x bf16 row-major [M][Kd]; w_t bf16 row-major [N][Kd] (W transposed, i.e.
 * the MIPS "database" layout, mips.hpp:37-62).  Scores are fp32 accumulated
 * on tcgen05 tensor cores; stage 1 runs in the epilogue.  Optionally writes
 * the fp32 score matrix (d_scores != NULL, [M][N]) for oracle replay. */
int atkg_fused_gemm_top_k(const void* d_x, const void* d_w_t, uint64_t m, uint64_t kdim,
                          const atkg_params* p, float* d_out_vals, uint32_t* d_out_idx,
                          float* d_scores, void* d_ws, size_t ws_bytes, uint32_t* d_status,
                          void* stream);
int atkg_fused_workspace_size(uint64_t m, uint64_t kdim, const atkg_params* p, size_t* bytes);
/* plain tcgen05 bf16 GEMM, fp32 out (the unfused reference path) */
int atkg_gemm_bf16(const void* d_x, const void* d_w_t, uint64_t m, uint64_t kdim, uint64_t n,
                   float* d_out, void* stream);

/* fp32 MIPS scores, bit-identical to atk::score_block (mips.hpp:57-63,
 * mips.cpp:57-91): out[q*out_stride + c] = <queries[q], database[c]> for
 * c < n, -inf for n <= c < n_padded (mips.cpp:112). Device pointers. */
int atkg_mips_score(const float* d_queries, uint64_t b, const float* d_database, uint64_t n,
                    uint64_t d, float* d_out, uint64_t out_stride, uint64_t n_padded, void* stream);

/* ---- host-buffer drop-in entry points (synchronous) --------------------- */
int atkg_stage1_host(const float* in, uint64_t rows, const atkg_params* p, float* grid_vals,
                     uint32_t* grid_idx);
int atkg_select_candidates_host(const float* vals, const uint32_t* idx, uint64_t count,
                                uint32_t k, uint64_t index_limit, float* out_vals,
                                uint32_t* out_idx);
int atkg_approx_top_k_host(const float* rows_in, uint64_t rows, const atkg_params* p,
                           float* out_vals, uint32_t* out_idx);
int atkg_exact_top_k_host(const float* in, uint64_t n, uint32_t k, float* out_vals,
                          uint32_t* out_idx);

/* ---- host analysis / planner -------------------------------------------- */
int atkg_measure_recall(const uint32_t* approx_idx, uint64_t approx_k, const uint32_t* exact_idx,
                        uint64_t exact_k, double* out);
int atkg_exact_expected_recall(const atkg_params* p, double* out);
int atkg_mc_expected_recall(const atkg_params* p, uint64_t trials, uint64_t seed, double* mean,
                            double* std_error);
int atkg_mc_expected_recall_adaptive(const atkg_params* p, uint64_t seed, double* mean,
                                     double* std_error, uint64_t* trials);
uint64_t atkg_legal_bucket_counts(uint64_t n, uint64_t lane_multiple, uint64_t* out,
                                  uint64_t cap);

/* PlanRequest / PlanResult (planner.hpp:18-39) */
typedef struct atkg_plan_request {
  uint64_t n;
  uint64_t k;
  double recall_target;
  const uint32_t* allowed_local_k;
  uint32_t num_allowed_local_k;
  uint32_t lane_multiple;
  uint64_t seed;
} atkg_plan_request;
#define ATKG_RECALL_EXACT 0
#define ATKG_RECALL_MONTE_CARLO 1
typedef struct atkg_plan_result {
  uint32_t local_k;
  uint64_t num_buckets;
  uint64_t num_elements;
  double recall;
  int recall_method;       /* ATKG_RECALL_* */
  double recall_std_error; /* monte_carlo only, else 0 */
  uint64_t recall_trials;  /* monte_carlo only, else 0 */
  int high_target_warning;
} atkg_plan_result;
int atkg_select_parameters(const atkg_plan_request* req, atkg_plan_result* out);

/* approx_top_k at a recall target: the planner (select_parameters,
 * planner.cpp:79-147) picks (K', B) from the request -- global_k = req->k,
 * the allowed K' list, lane multiple, seed -- and the row reduction runs with
 * them ("taking either (B, K') or (recall_target, allowed K'
 * list), with the planner running on the host first").  Plans are memoised
 * per request (the planner is deterministic in it).  *plan_out (optional)
 * receives the plan used. */
int atkg_approx_at_recall_workspace_size(int dtype, uint64_t rows, const atkg_plan_request* req,
                                         size_t* bytes);
int atkg_approx_top_k_at_recall(int dtype, const void* d_in, uint64_t rows,
                                const atkg_plan_request* req, atkg_plan_result* plan_out,
                                float* d_out_vals, uint32_t* d_out_idx, void* d_ws, size_t ws_bytes,
                                uint32_t* d_status, void* stream);
int atkg_approx_top_k_at_recall_host(const float* rows_in, uint64_t rows,
                                     const atkg_plan_request* req, atkg_plan_result* plan_out,
                                     float* out_vals, uint32_t* out_idx);

/* ---- ATKV dataset container ------------------------------ */
/* Replaces atk::read_dataset_file / write_dataset_file (dataset.hpp:45-49,
 * dataset.cpp:45-124): "ATKV", version 1, rows u64 LE, dims u64 LE, then
 * rows*dims fp32 LE.  Format failures return ATKG_EFORMAT with the reference's
 * messages ("bad dataset magic", "dataset truncated: payload incomplete",
 * "dataset payload contains NaN", ...).  Synchronous. */
int atkg_dataset_read_header(const char* path, uint64_t* rows, uint64_t* dims);
/* host buffer of `capacity` floats (ATKG_EINVAL if rows*dims exceeds it) */
int atkg_dataset_read_file(const char* path, float* out, uint64_t capacity, uint64_t* rows,
                           uint64_t* dims);
int atkg_dataset_write_file(const char* path, const float* data, uint64_t rows, uint64_t dims);
/* Device variants: the payload streams through pinned double-buffered chunks
 * straight to/from HBM; NaN rejection is a
 * device scan.  For dumping fused activations / replaying inputs. */
int atkg_dataset_read_file_device(const char* path, float* d_out, uint64_t capacity,
                                  uint64_t* rows, uint64_t* dims, void* stream);
int atkg_dataset_write_file_device(const char* path, const float* d_in, uint64_t rows,
                                   uint64_t dims, void* stream);

/* ---- recall simulation ----------------------------------- */
/* Rows [first_row, first_row + rows) of atk::synth_distinct (dataset.cpp:132-170):
 * row r is a Fisher-Yates permutation of 1..n on derive_seed(seed, r); n <= 2^24.
 * Host, `threads` workers. */
int atkg_synth_distinct(uint64_t first_row, uint64_t rows, uint64_t n, uint64_t seed, float* out,
                        uint32_t threads);
/* The same rows generated in HBM (one CTA per row, n <= 2^16, else
 * ATKG_EUNSUPPORTED); bit-identical to atkg_synth_distinct. */
int atkg_synth_distinct_device(uint64_t first_row, uint64_t rows, uint64_t n, uint64_t seed,
                               float* d_out, void* stream);
/* atk::simulate_recall_many (simulate.hpp:31-34, simulate.cpp:53-113): rows
 * generated on the device for n <= 2^16 (else on `threads` host workers),
 * approx_top_k + recall counting on the
 * device (stream), mean / sample stddev per config identical to the
 * reference.  Synchronous. */
int atkg_simulate_recall_many(const atkg_params* configs, uint32_t num_configs, uint64_t runs,
                              uint64_t seed, uint32_t threads, double* mean_recall, double* stddev,
                              void* stream);

/* ---- seeded synthetic inputs (documented convention) --------- */
/* out[i] = mean + stddev * z_i, z from Box-Muller over xoshiro256++ streams
 * derive_seed(seed, i / 65536) (rng.hpp:25-81), fp32. */
void atkg_fill_normal(uint64_t seed, uint64_t count, float mean, float stddev, float* out,
                      uint32_t threads);
/* elements [start, start + count) of the same stream (start % 65536 == 0):
 * one rank's slice of a sharded row */
void atkg_fill_normal_range(uint64_t seed, uint64_t start, uint64_t count, float mean, float stddev,
                            float* out, uint32_t threads);
/* round-to-nearest-even fp32 -> bf16 bits */
void atkg_f32_to_bf16(const float* in, uint64_t count, uint16_t* out, uint32_t threads);
void atkg_bf16_to_f32(const uint16_t* in, uint64_t count, float* out, uint32_t threads);

/* ---- instrumentation (bench.py, profiling) ------------------------------ */
/* Between atkg_profile_begin() and atkg_profile_end(), every stage-1
 * streaming kernel (the dominant kernel) launched by this library is
 * bracketed by CUDA events on its own stream; profile_end synchronises and
 * returns the summed device duration and the number of such launches.
 * Process-wide; not for concurrent use. */
void atkg_profile_begin(void);
/* Same, bracketing only every `every`-th dominant-kernel launch: the event
 * records sit between a kernel and its PDL-launched successor, so sampling
 * keeps the timed loop's step time unperturbed. */
void atkg_profile_begin_every(uint32_t every);
int atkg_profile_end(double* total_ms, uint64_t* launches);
/* Kernels launched by this library so far (process-wide counter). */
uint64_t atkg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* ATKG_H_ */
