// planner.cpp -- host planner: expected recall (Theorem 1), Monte-Carlo
// estimate and (B, K') selection at a recall target.
//
// Restates, for the host side of the B200 path, /root/reference/proj/core:
//   log_choose / Hypergeometric / HypergeometricSampler   src/hypergeom.cpp:10-103
//   bucket_excess_mean, exact_expected_recall             src/recall.cpp:33-56, 76-100
//   mc_expected_recall(_adaptive)                         src/recall.cpp:102-165
//   legal_bucket_counts, select_parameters                src/planner.cpp:59-147
// The floating-point expression order follows the reference so the planner
// picks the same (K', B) and reports the same recall (planner KATs in
// tests/test_planner.py; glibc lgamma/exp on both sides).
// The planner runs in well under 50 ms per config; it stays on the host.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/atkg.h"
#include "host_common.hpp"

namespace atkg {
namespace {

// ---- xoshiro256++ / splitmix64 (include/atk/rng.hpp:15-81) ---------------
struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& st) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& w : s) w = splitmix(sm);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

double log_choose(uint64_t n, uint64_t k) {
  if (k > n) return -std::numeric_limits<double>::infinity();
  return std::lgamma(static_cast<double>(n) + 1.0) - std::lgamma(static_cast<double>(k) + 1.0) -
         std::lgamma(static_cast<double>(n - k) + 1.0);
}

struct Hyper {
  uint64_t pop, succ, draws;
  uint64_t lo() const { const uint64_t miss = pop - succ; return draws > miss ? draws - miss : 0; }
  uint64_t hi() const { return std::min(succ, draws); }
  double mean() const { return static_cast<double>(draws) * static_cast<double>(succ) / static_cast<double>(pop); }
  double sd() const {
    if (pop <= 1) return 0.0;
    const double n = static_cast<double>(pop), p = static_cast<double>(succ) / n, s = static_cast<double>(draws);
    const double var = s * p * (1.0 - p) * (n - s) / (n - 1.0);
    return var > 0.0 ? std::sqrt(var) : 0.0;
  }
  double log_pmf(uint64_t r) const {
    if (r < lo() || r > hi()) return -std::numeric_limits<double>::infinity();
    return log_choose(succ, r) + log_choose(pop - succ, draws - r) - log_choose(pop, draws);
  }
};

// inverse-CDF table over mean +- 60 sigma (hypergeom.cpp:61-96)
struct Sampler {
  uint64_t base = 0;
  std::vector<double> cdf;
  explicit Sampler(const Hyper& h) {
    const uint64_t smin = h.lo(), smax = h.hi();
    const double mu = h.mean(), span = 60.0 * h.sd() + 2.0;
    uint64_t a = smin, b = smax;
    if (mu - span > static_cast<double>(smin)) a = static_cast<uint64_t>(mu - span);
    if (mu + span < static_cast<double>(smax)) b = static_cast<uint64_t>(mu + span) + 1;
    if (b < a) b = a;
    base = a;
    cdf.resize(static_cast<size_t>(b - a + 1));
    const double n = static_cast<double>(h.pop), k = static_cast<double>(h.succ), s = static_cast<double>(h.draws);
    double p = std::exp(h.log_pmf(a)), cum = 0.0;
    for (uint64_t r = a; r <= b; ++r) {
      cum += p;
      cdf[static_cast<size_t>(r - a)] = cum;
      const double rr = static_cast<double>(r);
      const double num = (k - rr) * (s - rr);
      const double den = (rr + 1.0) * (n - k - s + rr + 1.0);
      p = den > 0.0 ? p * (num / den) : 0.0;
    }
  }
  uint64_t draw(Rng& rng) const {
    const double u = rng.uniform();
    const auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
    if (it == cdf.end()) return base + cdf.size() - 1;
    return base + static_cast<uint64_t>(it - cdf.begin());
  }
};

double excess_mean(uint64_t n, uint64_t k, uint64_t s, uint32_t kp) {
  const Hyper h{n, k, s};
  const uint64_t rmax = h.hi();
  if (kp >= rmax) return 0.0;
  const uint64_t rmin = std::max<uint64_t>(static_cast<uint64_t>(kp) + 1, h.lo());
  const double lden = log_choose(n, s);
  const double mode = (static_cast<double>(s) + 1.0) * (static_cast<double>(k) + 1.0) / (static_cast<double>(n) + 2.0);
  double sum = 0.0, comp = 0.0;  // Kahan
  for (uint64_t r = rmin; r <= rmax; ++r) {
    const double lterm = log_choose(k, r) + log_choose(n - k, s - r) - lden;
    const double term = static_cast<double>(r - kp) * std::exp(lterm);
    const double y = term - comp;
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
    if (static_cast<double>(r) > mode + 2.0 && term <= sum * 1e-18) break;
  }
  return sum;
}

double clamp01(double x) { return std::min(1.0, std::max(0.0, x)); }

}  // namespace

uint64_t derive_seed(uint64_t seed, uint64_t stream) {  // rng.hpp:25-32
  uint64_t s = seed;
  (void)Rng::splitmix(s);
  s ^= 0x9e3779b97f4a7c15ull * (stream + 1);
  const uint64_t a = Rng::splitmix(s);
  const uint64_t b = Rng::splitmix(s);
  return a ^ (b >> 1);
}

double exact_recall(const atkg_params& p) {
  const uint64_t s_lo = p.n / p.num_buckets, chi = p.n % p.num_buckets, clo = p.num_buckets - chi;
  double excess = 0.0;
  if (clo > 0) excess += static_cast<double>(clo) * excess_mean(p.n, p.global_k, s_lo, p.local_k);
  if (chi > 0) excess += static_cast<double>(chi) * excess_mean(p.n, p.global_k, s_lo + 1, p.local_k);
  return clamp01(1.0 - excess / static_cast<double>(p.global_k));
}

void mc_recall(const atkg_params& p, uint64_t trials, uint64_t seed, double* mean_out, double* se_out) {
  const uint64_t n = p.n, b = p.num_buckets, k = p.global_k;
  const uint64_t s_lo = n / b, chi = n % b, clo = b - chi;
  const double kd = static_cast<double>(k);
  const uint64_t kp = p.local_k;
  const Sampler lo(Hyper{n, k, s_lo});
  const Sampler hi(chi > 0 ? Hyper{n, k, s_lo + 1} : Hyper{n, k, s_lo});
  Rng rng(seed);
  double mean = 0.0, m2 = 0.0;
  for (uint64_t t = 0; t < trials; ++t) {
    double excess = 0.0;
    if (clo > 0) {
      const uint64_t x = lo.draw(rng);
      if (x > kp) excess += static_cast<double>(clo) * static_cast<double>(x - kp);
    }
    if (chi > 0) {
      const uint64_t x = hi.draw(rng);
      if (x > kp) excess += static_cast<double>(chi) * static_cast<double>(x - kp);
    }
    const double rec = 1.0 - excess / kd;
    const double d = rec - mean;
    mean += d / static_cast<double>(t + 1);
    m2 += d * (rec - mean);
  }
  const double var = m2 / static_cast<double>(trials - 1);
  *mean_out = mean;
  *se_out = std::sqrt(std::max(0.0, var) / static_cast<double>(trials));
}

void mc_recall_adaptive(const atkg_params& p, uint64_t seed, double* mean, double* se, uint64_t* trials_out) {
  uint64_t trials = 4096;
  for (uint64_t attempt = 0;; ++attempt) {
    mc_recall(p, trials, derive_seed(seed, attempt), mean, se);
    if (3.0 * *se <= 0.005) {
      *trials_out = trials;
      return;
    }
    trials *= 2;
  }
}

std::vector<uint64_t> legal_buckets(uint64_t n, uint64_t lane) {
  if (n % lane != 0) return {};
  const uint64_t m = n / lane;
  std::vector<uint64_t> d;
  for (uint64_t x = 1; x * x <= m; ++x) {
    if (m % x) continue;
    d.push_back(x * lane);
    if (x != m / x) d.push_back((m / x) * lane);
  }
  std::sort(d.rbegin(), d.rend());
  return d;
}

}  // namespace atkg

using namespace atkg;

extern "C" {

int atkg_validate_analysis(const atkg_params* p) {
  return guarded([&] {
    if (p->n == 0) throw_inval("n must be >= 1");
    if (p->num_buckets == 0) throw_inval("num_buckets must be >= 1");
    if (p->num_buckets > p->n) throw_inval("num_buckets must not exceed n");
    if (p->local_k == 0) throw_inval("local_k must be >= 1");
    if (p->global_k == 0) throw_inval("global_k must be >= 1");
    if (p->global_k > p->n) throw_inval("global_k must not exceed n");
  });
}

int atkg_exact_expected_recall(const atkg_params* p, double* out) {
  const int rc = atkg_validate_analysis(p);
  if (rc) return rc;
  return guarded([&] { *out = exact_recall(*p); });
}

int atkg_mc_expected_recall(const atkg_params* p, uint64_t trials, uint64_t seed, double* mean,
                            double* std_error) {
  const int rc = atkg_validate_analysis(p);
  if (rc) return rc;
  return guarded([&] {
    if (trials < 2) throw_inval("mc_expected_recall needs trials >= 2");
    mc_recall(*p, trials, seed, mean, std_error);
  });
}

int atkg_mc_expected_recall_adaptive(const atkg_params* p, uint64_t seed, double* mean,
                                     double* std_error, uint64_t* trials) {
  const int rc = atkg_validate_analysis(p);
  if (rc) return rc;
  return guarded([&] { mc_recall_adaptive(*p, seed, mean, std_error, trials); });
}

uint64_t atkg_legal_bucket_counts(uint64_t n, uint64_t lane, uint64_t* out, uint64_t cap) {
  if (n == 0 || lane == 0) return 0;
  const auto v = legal_buckets(n, lane);
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  return v.size();
}

int atkg_select_parameters(const atkg_plan_request* req, atkg_plan_result* out) {
  return guarded([&] {
    if (req->n == 0) throw_inval("plan: n must be >= 1");
    if (req->k == 0 || req->k > req->n) throw_inval("plan: k must satisfy 1 <= k <= n");
    if (req->k > 0xffffffffull) throw_inval("plan: k exceeds the 32-bit result size");
    if (!(req->recall_target > 0.0) || !(req->recall_target < 1.0))
      throw_inval("plan: recall_target must be in (0, 1)");
    if (req->num_allowed_local_k == 0) throw_inval("plan: allowed_local_k must not be empty");
    for (uint32_t i = 0; i < req->num_allowed_local_k; ++i)
      if (req->allowed_local_k[i] == 0) throw_inval("plan: allowed_local_k entries must be >= 1");
    if (req->lane_multiple == 0) throw_inval("plan: lane_multiple must be >= 1");

    const bool warn = req->recall_target >= 0.995;
    const auto buckets = legal_buckets(req->n, req->lane_multiple);
    std::vector<uint32_t> kps(req->allowed_local_k, req->allowed_local_k + req->num_allowed_local_k);
    std::sort(kps.begin(), kps.end());
    kps.erase(std::unique(kps.begin(), kps.end()), kps.end());

    struct Cand { uint32_t kp; uint64_t b; double mean, se; uint64_t trials; };
    std::vector<Cand> pass;
    for (const uint32_t kp : kps) {
      const uint64_t kseed = derive_seed(req->seed, kp);
      for (const uint64_t b : buckets) {
        if (b * kp < req->k) break;
        atkg_params p{req->n, b, kp, static_cast<uint32_t>(req->k), req->lane_multiple};
        double mean, se;
        uint64_t tr;
        mc_recall_adaptive(p, derive_seed(kseed, b), &mean, &se, &tr);
        if (!(mean >= req->recall_target)) break;
        pass.push_back({kp, b, mean, se, tr});
      }
    }
    if (pass.empty())
      throw Infeasible("no legal (local_k, num_buckets) configuration meets the recall target");
    std::stable_sort(pass.begin(), pass.end(), [](const Cand& a, const Cand& b) {
      const uint64_t ea = a.b * a.kp, eb = b.b * b.kp;
      if (ea != eb) return ea < eb;
      return a.kp < b.kp;
    });
    for (const auto& c : pass) {
      atkg_plan_result r{};
      r.recall = c.mean;
      r.recall_method = ATKG_RECALL_MONTE_CARLO;
      r.recall_std_error = c.se;
      r.recall_trials = c.trials;
      if (std::min<uint64_t>(req->k, req->n / c.b) <= 10000) {
        atkg_params p{req->n, c.b, c.kp, static_cast<uint32_t>(req->k), req->lane_multiple};
        r.recall = exact_recall(p);
        r.recall_method = ATKG_RECALL_EXACT;
        r.recall_std_error = 0.0;
        r.recall_trials = 0;
        if (r.recall < req->recall_target) continue;
      }
      r.local_k = c.kp;
      r.num_buckets = c.b;
      r.num_elements = c.b * c.kp;
      r.high_target_warning = warn ? 1 : 0;
      *out = r;
      return;
    }
    throw Infeasible("every MC-passing configuration failed exact re-validation");
  });
}

}  // extern "C"
