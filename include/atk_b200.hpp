// atk_b200.hpp -- the reference's C++ interface over the B200 library.
//
// A header-only drop-in for callers of the reference `atk` core: the same
// signatures, argument meaning, results and exception types as
// include/atk/topk.hpp, planner.hpp and recall.hpp
// (/root/reference/proj/core/include/atk/), computed by libatkg.so through
// its C ABI (include/atkg.h).  The types are the reference's own
// (atk/params.hpp, atk/planner.hpp, atk/recall.hpp are header-only), so a
// caller switches by calling atk_b200::f instead of atk::f (or with
// `namespace atk_impl = atk_b200;`) and linking -latkg instead of the
// reference's topk.cpp / planner.cpp.  Host buffers in, host buffers out,
// synchronous -- the reference's contract; device-resident callers use the
// stream-ordered entry points of atkg.h directly.
//
//   reference (include/atk/)                         here
//   approx_top_k            topk.hpp:117              approx_top_k
//   approx_top_k_batch      topk.hpp:121-124          approx_top_k_batch
//   stage1_partial_reduce   topk.hpp:98-99            stage1_partial_reduce
//   select_top_k_candidates topk.hpp:109-112          select_top_k_candidates
//   exact_top_k             topk.hpp:104              exact_top_k
//   measure_recall          topk.hpp:128              measure_recall
//   Stage1Accumulator       topk.hpp:68-94            Stage1Accumulator
//   select_parameters       planner.hpp:66-67         select_parameters (trace == nullptr)
//   PlanResult::params      planner.hpp:38            plan_params
//   legal_bucket_counts     planner.hpp:61-62         legal_bucket_counts
//   exact_expected_recall   recall.hpp:39             exact_expected_recall
//   mc_expected_recall(_adaptive) recall.hpp:45-51    mc_expected_recall(_adaptive)
//   (planner + approx_top_k)             approx_top_k_at_recall
//
// Errors: std::invalid_argument with the reference's messages (including
// "input contains NaN"), atk::NoFeasibleConfigError from the planner,
// std::runtime_error for CUDA failures.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "atk/params.hpp"
#include "atk/planner.hpp"
#include "atk/recall.hpp"
#include "atkg.h"

namespace atk_b200 {

namespace detail {

inline void check(int rc) {
  if (rc == ATKG_OK) return;
  const std::string m = atkg_last_error();
  if (rc == ATKG_EINVAL || rc == ATKG_ENAN) throw std::invalid_argument(m);
  if (rc == ATKG_EINFEASIBLE) throw atk::NoFeasibleConfigError(m);
  throw std::runtime_error(m);
}

inline atkg_params to_c(const atk::AlgoParams& p) {
  return atkg_params{p.n, p.num_buckets, p.local_k, p.global_k, p.lane_multiple};
}

inline atk::TopKResult result(const float* v, const uint32_t* i, std::size_t k) {
  atk::TopKResult r;
  r.values.assign(v, v + k);
  r.indices.assign(i, i + k);
  return r;
}

inline atkg_plan_request to_c(const atk::PlanRequest& req) {
  return atkg_plan_request{req.n,
                           req.k,
                           req.recall_target,
                           req.allowed_local_k.data(),
                           static_cast<uint32_t>(req.allowed_local_k.size()),
                           req.lane_multiple,
                           req.seed};
}

inline atk::PlanResult from_c(const atkg_plan_result& r) {
  atk::PlanResult out;
  out.local_k = r.local_k;
  out.num_buckets = r.num_buckets;
  out.num_elements = r.num_elements;
  out.estimated_recall.value = r.recall;
  if (r.recall_method == ATKG_RECALL_MONTE_CARLO) {
    out.estimated_recall.method = atk::RecallMethod::monte_carlo;
    out.estimated_recall.std_error = r.recall_std_error;
    out.estimated_recall.trials = r.recall_trials;
  } else {
    out.estimated_recall.method = atk::RecallMethod::exact;
  }
  out.high_target_warning = r.high_target_warning != 0;
  return out;
}

}  // namespace detail

// ---- topk.hpp ---------------------------------------------------------------

inline std::vector<atk::TopKResult> approx_top_k_batch(std::span<const float> rows, std::uint64_t row_count,
                                                       const atk::AlgoParams& params, unsigned threads = 1) {
  (void)threads;  // the device path is thread-count invariant, like the reference (threads.hpp:13-17)
  const atkg_params c = detail::to_c(params);
  detail::check(atkg_validate(&c));
  if (rows.size() != row_count * params.n) throw std::invalid_argument("batch length does not match row_count * n");
  const std::size_t k = params.global_k;
  std::vector<float> v(row_count * k);
  std::vector<uint32_t> i(row_count * k);
  if (row_count) detail::check(atkg_approx_top_k_host(rows.data(), row_count, &c, v.data(), i.data()));
  std::vector<atk::TopKResult> out(row_count);
  for (std::uint64_t r = 0; r < row_count; ++r) out[r] = detail::result(v.data() + r * k, i.data() + r * k, k);
  return out;
}

inline atk::TopKResult approx_top_k(std::span<const float> input, const atk::AlgoParams& params) {
  const atkg_params c = detail::to_c(params);
  detail::check(atkg_validate(&c));
  if (input.size() != params.n) throw std::invalid_argument("input length does not match params.n");
  return atk_b200::approx_top_k_batch(input, 1, params).front();
}

inline atk::TopKResult stage1_partial_reduce(std::span<const float> input, const atk::AlgoParams& params) {
  const atkg_params c = detail::to_c(params);
  detail::check(atkg_validate(&c));
  if (input.size() != params.n) throw std::invalid_argument("input length does not match params.n");
  atk::TopKResult g;
  g.values.resize(params.num_candidates());
  g.indices.resize(params.num_candidates());
  detail::check(atkg_stage1_host(input.data(), 1, &c, g.values.data(), g.indices.data()));
  return g;
}

inline atk::TopKResult exact_top_k(std::span<const float> input, std::uint32_t k) {
  std::vector<float> v(k ? k : 1);
  std::vector<uint32_t> i(k ? k : 1);
  detail::check(atkg_exact_top_k_host(input.data(), input.size(), k, v.data(), i.data()));
  return detail::result(v.data(), i.data(), k);
}

inline atk::TopKResult select_top_k_candidates(std::span<const float> values, std::span<const std::uint32_t> indices,
                                               std::uint32_t k, std::uint64_t index_limit = UINT64_MAX) {
  if (values.size() != indices.size()) throw std::invalid_argument("candidate value/index lengths differ");
  std::vector<float> v(k ? k : 1);
  std::vector<uint32_t> i(k ? k : 1);
  const float zf = 0.f;
  const uint32_t zi = 0;
  detail::check(atkg_select_candidates_host(values.empty() ? &zf : values.data(),
                                            indices.empty() ? &zi : indices.data(), values.size(), k, index_limit,
                                            v.data(), i.data()));
  return detail::result(v.data(), i.data(), k);
}

inline double measure_recall(const atk::TopKResult& approx, const atk::TopKResult& exact) {
  double r = 0.0;
  detail::check(atkg_measure_recall(approx.indices.data(), approx.indices.size(), exact.indices.data(),
                                    exact.indices.size(), &r));
  return r;
}

// Streaming stage 1 (topk.hpp:68-94): blocks in index order, any length
// and alignment, bit-identical for every blocking; the state lives on the GPU.
class Stage1Accumulator {
 public:
  explicit Stage1Accumulator(const atk::AlgoParams& params) : params_(params) {
    const atkg_params c = detail::to_c(params);
    detail::check(atkg_accumulator_create(&c, &acc_));
  }
  ~Stage1Accumulator() { atkg_accumulator_destroy(acc_); }
  Stage1Accumulator(const Stage1Accumulator&) = delete;
  Stage1Accumulator& operator=(const Stage1Accumulator&) = delete;

  void consume(std::span<const float> block) {
    detail::check(atkg_accumulator_consume_host(acc_, block.data(), block.size()));
    dirty_ = true;
  }
  std::uint64_t consumed() const { return atkg_accumulator_consumed(acc_); }
  const atk::AlgoParams& params() const { return params_; }
  const std::vector<float>& values() const { refresh(); return values_; }
  const std::vector<std::uint32_t>& indices() const { refresh(); return indices_; }
  atk::TopKResult candidates() const {
    refresh();
    atk::TopKResult r;
    r.values = values_;
    r.indices = indices_;
    return r;
  }

 private:
  void refresh() const {
    if (!dirty_) return;
    values_.resize(params_.num_candidates());
    indices_.resize(params_.num_candidates());
    detail::check(atkg_accumulator_candidates_host(acc_, values_.data(), indices_.data()));
    dirty_ = false;
  }
  atk::AlgoParams params_;
  atkg_accumulator* acc_ = nullptr;
  mutable std::vector<float> values_;
  mutable std::vector<std::uint32_t> indices_;
  mutable bool dirty_ = true;
};

// ---- planner.hpp / recall.hpp ---------------------------------------------

inline atk::PlanResult select_parameters(const atk::PlanRequest& req,
                                         std::vector<atk::PlanCandidate>* trace = nullptr) {
  if (trace) throw std::invalid_argument("select_parameters: the sweep trace is not exported by atk_b200");
  const atkg_plan_request c = detail::to_c(req);
  atkg_plan_result r{};
  detail::check(atkg_select_parameters(&c, &r));
  return detail::from_c(r);
}

inline atk::AlgoParams plan_params(const atk::PlanResult& plan, const atk::PlanRequest& req) {  // PlanResult::params
  atk::AlgoParams p;
  p.n = req.n;
  p.num_buckets = plan.num_buckets;
  p.local_k = plan.local_k;
  p.global_k = static_cast<std::uint32_t>(req.k);
  p.lane_multiple = req.lane_multiple;
  return p;
}

inline std::vector<std::uint64_t> legal_bucket_counts(std::uint64_t n, std::uint64_t lane_multiple) {
  if (n == 0) throw std::invalid_argument("n must be >= 1");
  if (lane_multiple == 0) throw std::invalid_argument("lane_multiple must be >= 1");
  const uint64_t cnt = atkg_legal_bucket_counts(n, lane_multiple, nullptr, 0);
  std::vector<std::uint64_t> out(cnt);
  if (cnt) atkg_legal_bucket_counts(n, lane_multiple, out.data(), cnt);
  return out;
}

inline atk::RecallEstimate exact_expected_recall(const atk::AlgoParams& params) {
  const atkg_params c = detail::to_c(params);
  atk::RecallEstimate e;
  detail::check(atkg_exact_expected_recall(&c, &e.value));
  e.method = atk::RecallMethod::exact;
  return e;
}

inline atk::RecallEstimate mc_expected_recall(const atk::AlgoParams& params, std::uint64_t trials,
                                              std::uint64_t seed) {
  const atkg_params c = detail::to_c(params);
  atk::RecallEstimate e;
  double se = 0.0;
  detail::check(atkg_mc_expected_recall(&c, trials, seed, &e.value, &se));
  e.method = atk::RecallMethod::monte_carlo;
  e.std_error = se;
  e.trials = trials;
  return e;
}

inline atk::RecallEstimate mc_expected_recall_adaptive(const atk::AlgoParams& params, std::uint64_t seed) {
  const atkg_params c = detail::to_c(params);
  atk::RecallEstimate e;
  double se = 0.0;
  uint64_t trials = 0;
  detail::check(atkg_mc_expected_recall_adaptive(&c, seed, &e.value, &se, &trials));
  e.method = atk::RecallMethod::monte_carlo;
  e.std_error = se;
  e.trials = trials;
  return e;
}

// ---- at a recall target ---------------------------------------

// select_parameters(req), then approx_top_k_batch with the planned (K', B):
// returns the plan and the rows' top req.k.
inline std::pair<atk::PlanResult, std::vector<atk::TopKResult>> approx_top_k_at_recall(
    std::span<const float> rows, std::uint64_t row_count, const atk::PlanRequest& req) {
  if (rows.size() != row_count * req.n) throw std::invalid_argument("batch length does not match row_count * n");
  const atkg_plan_request c = detail::to_c(req);
  const std::size_t k = req.k;
  std::vector<float> v(row_count * k);
  std::vector<uint32_t> i(row_count * k);
  atkg_plan_result r{};
  detail::check(atkg_approx_top_k_at_recall_host(rows.data(), row_count, &c, &r, v.data(), i.data()));
  std::vector<atk::TopKResult> out(row_count);
  for (std::uint64_t q = 0; q < row_count; ++q) out[q] = detail::result(v.data() + q * k, i.data() + q * k, k);
  return {detail::from_c(r), std::move(out)};
}

}  // namespace atk_b200
