// atk_b200_check.cpp -- TEST INFRASTRUCTURE: the C++ drop-in header
// (include/atk_b200.hpp) against the reference core itself.
//
// Built in the build container (the reference headers live there), linked
// against libatkg.so and oracle/_ref/libatk_ref.so (the unmodified reference
// core); run on the GPU box by tests/test_gpu_cpp_dropin.py.  Every check
// calls atk::f (reference) and atk_b200::f (this repo) on the same inputs
// and compares results bit for bit, or the exception type and message.
// Prints one "PASS name" / "FAIL name: why" line per check; exit code =
// number of failures.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "atk/params.hpp"
#include "atk/planner.hpp"
#include "atk/recall.hpp"
#include "atk/topk.hpp"
#include "atk_b200.hpp"

namespace {

int g_fail = 0;

void report(const std::string& name, bool ok, const std::string& why = "") {
  if (ok) std::printf("PASS %s\n", name.c_str());
  else { std::printf("FAIL %s: %s\n", name.c_str(), why.c_str()); ++g_fail; }
}

std::vector<float> normal_rows(std::size_t count, uint64_t seed, int quantize = 0) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> d(0.0, 1.0);
  std::vector<float> x(count);
  for (auto& v : x) {
    v = static_cast<float>(d(g));
    if (quantize) v = std::round(v * quantize) / quantize;
  }
  return x;
}

bool same(const atk::TopKResult& a, const atk::TopKResult& b, std::string* why) {
  if (a.values.size() != b.values.size() || a.indices.size() != b.indices.size()) {
    *why = "sizes differ";
    return false;
  }
  for (std::size_t i = 0; i < a.values.size(); ++i) {
    uint32_t x, y;
    std::memcpy(&x, &a.values[i], 4);
    std::memcpy(&y, &b.values[i], 4);
    if (x != y || a.indices[i] != b.indices[i]) {
      *why = "entry " + std::to_string(i) + " differs";
      return false;
    }
  }
  return true;
}

template <class F, class G>
void same_error(const std::string& name, F&& ref, G&& ours) {
  std::string rm = "none", om = "none";
  int rk = 0, ok = 0;
  try { ref(); } catch (const atk::NoFeasibleConfigError& e) { rk = 3; rm = e.what(); }
  catch (const std::invalid_argument& e) { rk = 1; rm = e.what(); } catch (const std::exception& e) { rk = 2; rm = e.what(); }
  try { ours(); } catch (const atk::NoFeasibleConfigError& e) { ok = 3; om = e.what(); }
  catch (const std::invalid_argument& e) { ok = 1; om = e.what(); } catch (const std::exception& e) { ok = 2; om = e.what(); }
  report(name, rk == ok && rk != 0 && rm == om, "reference [" + std::to_string(rk) + "] " + rm + " / ours [" +
                                                   std::to_string(ok) + "] " + om);
}

atk::AlgoParams P(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, uint32_t lane = 128) {
  atk::AlgoParams p;
  p.n = n;
  p.num_buckets = b;
  p.local_k = kp;
  p.global_k = k;
  p.lane_multiple = lane;
  return p;
}

}  // namespace

int main() {
  std::string why;
  // approx_top_k_batch / approx_top_k (topk.hpp:117-124)
  for (auto [rows, n, b, kp, k, q] : std::vector<std::tuple<uint64_t, uint64_t, uint64_t, uint32_t, uint32_t, int>>{
           {64, 14336, 128, 4, 287, 0}, {8, 262144, 128, 2, 64, 0}, {16, 32768, 512, 4, 128, 4}, {4, 65536, 256, 8, 1024, 0}}) {
    const auto x = normal_rows(rows * n, n + k, q);
    const auto p = P(n, b, kp, k);
    const auto r = atk::approx_top_k_batch(x, rows, p, 4);
    const auto o = atk_b200::approx_top_k_batch(x, rows, p, 4);
    bool ok = r.size() == o.size();
    for (std::size_t i = 0; ok && i < r.size(); ++i) ok = same(r[i], o[i], &why);
    report("approx_top_k_batch n=" + std::to_string(n) + " q=" + std::to_string(q), ok, why);
    const auto r1 = atk::approx_top_k(std::span<const float>(x.data(), n), p);
    const auto o1 = atk_b200::approx_top_k(std::span<const float>(x.data(), n), p);
    report("approx_top_k n=" + std::to_string(n), same(r1, o1, &why), why);
  }
  // stage1_partial_reduce (topk.hpp:98-99)
  {
    const auto x = normal_rows(65536, 3, 8);
    const auto p = P(65536, 256, 4, 100);
    report("stage1_partial_reduce", same(atk::stage1_partial_reduce(x, p), atk_b200::stage1_partial_reduce(x, p), &why),
           why);
  }
  // exact_top_k (topk.hpp:104), incl. k above one CTA's sort
  for (auto [n, k] : std::vector<std::pair<uint64_t, uint32_t>>{{100000, 1000}, {200000, 20000}, {7, 7}}) {
    const auto x = normal_rows(n, k, 16);
    report("exact_top_k k=" + std::to_string(k), same(atk::exact_top_k(x, k), atk_b200::exact_top_k(x, k), &why), why);
  }
  // select_top_k_candidates (topk.hpp:109-112) with index_limit
  {
    const auto v = normal_rows(5000, 11, 4);
    std::vector<uint32_t> ix(5000);
    for (uint32_t i = 0; i < 5000; ++i) ix[i] = (i * 7919u) % 9000u;
    report("select_top_k_candidates",
           same(atk::select_top_k_candidates(v, ix, 300, 8000), atk_b200::select_top_k_candidates(v, ix, 300, 8000),
                &why), why);
  }
  // measure_recall (topk.hpp:128)
  {
    const auto x = normal_rows(262144, 5);
    const auto p = P(262144, 128, 1, 64);
    const auto a = atk::approx_top_k(x, p);
    const auto e = atk::exact_top_k(x, 64);
    report("measure_recall", atk::measure_recall(a, e) == atk_b200::measure_recall(a, e));
  }
  // Stage1Accumulator (topk.hpp:68-94), ragged blocks
  {
    const auto x = normal_rows(100000, 9, 8);
    const auto p = P(100000, 1000, 3, 500, 8);
    atk::Stage1Accumulator ra(p);
    atk_b200::Stage1Accumulator oa(p);
    std::mt19937 g(1);
    std::size_t pos = 0;
    while (pos < x.size()) {
      const std::size_t len = std::min<std::size_t>(x.size() - pos, 1 + g() % 20000);
      ra.consume(std::span<const float>(x.data() + pos, len));
      oa.consume(std::span<const float>(x.data() + pos, len));
      pos += len;
    }
    report("Stage1Accumulator", same(ra.candidates(), oa.candidates(), &why) && ra.consumed() == oa.consumed(), why);
  }
  // planner / recall (planner.hpp:38,61-67; recall.hpp:39-51)
  {
    atk::PlanRequest req;
    req.n = 14336;
    req.k = 287;
    req.recall_target = 0.95;
    req.allowed_local_k = {1, 2, 4, 8};
    const auto r = atk::select_parameters(req);
    const auto o = atk_b200::select_parameters(req);
    report("select_parameters", r.local_k == o.local_k && r.num_buckets == o.num_buckets &&
                                    r.num_elements == o.num_elements &&
                                    r.estimated_recall.value == o.estimated_recall.value &&
                                    r.estimated_recall.method == o.estimated_recall.method &&
                                    r.high_target_warning == o.high_target_warning);
    const auto rp = r.params(req);
    const auto op = atk_b200::plan_params(o, req);
    report("PlanResult::params", rp.n == op.n && rp.num_buckets == op.num_buckets && rp.local_k == op.local_k &&
                                     rp.global_k == op.global_k && rp.lane_multiple == op.lane_multiple);
    report("legal_bucket_counts", atk::legal_bucket_counts(430080, 128) == atk_b200::legal_bucket_counts(430080, 128));
    report("exact_expected_recall",
           atk::exact_expected_recall(P(262144, 512, 4, 1024)).value ==
               atk_b200::exact_expected_recall(P(262144, 512, 4, 1024)).value);
    const auto rm = atk::mc_expected_recall(P(14336, 128, 4, 287), 10000, 3);
    const auto om = atk_b200::mc_expected_recall(P(14336, 128, 4, 287), 10000, 3);
    report("mc_expected_recall", rm.value == om.value && rm.std_error == om.std_error);
    const auto ra = atk::mc_expected_recall_adaptive(P(262144, 512, 4, 1024), 7);
    const auto oa = atk_b200::mc_expected_recall_adaptive(P(262144, 512, 4, 1024), 7);
    report("mc_expected_recall_adaptive", ra.value == oa.value && ra.trials == oa.trials);
    // at a recall target: the plan, then the rows
    const auto x = normal_rows(32 * 14336, 21);
    const auto [plan, res] = atk_b200::approx_top_k_at_recall(x, 32, req);
    const auto rr = atk::approx_top_k_batch(x, 32, r.params(req));
    bool ok = plan.local_k == r.local_k && plan.num_buckets == r.num_buckets && res.size() == rr.size();
    for (std::size_t i = 0; ok && i < rr.size(); ++i) ok = same(rr[i], res[i], &why);
    report("approx_top_k_at_recall", ok, why);
  }
  // errors: same exception type and message
  {
    auto x = normal_rows(4096, 1);
    x[77] = NAN;
    const auto p = P(4096, 128, 2, 64);
    same_error("nan approx_top_k", [&] { atk::approx_top_k(x, p); }, [&] { atk_b200::approx_top_k(x, p); });
    same_error("nan exact_top_k", [&] { atk::exact_top_k(x, 10); }, [&] { atk_b200::exact_top_k(x, 10); });
    const auto y = normal_rows(4096, 2);
    same_error("bad buckets", [&] { atk::approx_top_k(y, P(4096, 100, 2, 64)); },
               [&] { atk_b200::approx_top_k(y, P(4096, 100, 2, 64)); });
    same_error("global_k > candidates", [&] { atk::approx_top_k(y, P(4096, 128, 1, 200)); },
               [&] { atk_b200::approx_top_k(y, P(4096, 128, 1, 200)); });
    same_error("exact k > n", [&] { atk::exact_top_k(y, 5000); }, [&] { atk_b200::exact_top_k(y, 5000); });
    std::vector<uint32_t> ix(10, 3);
    same_error("fewer candidates", [&] { atk::select_top_k_candidates(std::span<const float>(y.data(), 10), ix, 5, 2); },
               [&] { atk_b200::select_top_k_candidates(std::span<const float>(y.data(), 10), ix, 5, 2); });
    atk::PlanRequest bad;  // no bucket count of n = 1000 is a multiple of lane 128
    bad.n = 1000;
    bad.k = 10;
    bad.recall_target = 0.95;
    bad.allowed_local_k = {1, 2};
    same_error("planner infeasible", [&] { atk::select_parameters(bad); }, [&] { atk_b200::select_parameters(bad); });
    bad.recall_target = 1.5;
    same_error("planner bad target", [&] { atk::select_parameters(bad); }, [&] { atk_b200::select_parameters(bad); });
  }
  std::printf("%d failure(s)\n", g_fail);
  return g_fail;
}
