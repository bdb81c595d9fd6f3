// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference `atk` core, compiled straight
// from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libatk_ref.so.  Used (a) to pin oracle/atk_oracle.c against the
// reference itself, (b) to generate tests/golden fixtures, and (c) as the CPU
// baseline arm of bench.py (`--impl reference`, cpu_baseline.kind
// "reference").  The product never loads it.
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "atk/planner.hpp"
#include "atk/recall.hpp"
#include "atk/topk.hpp"
#include "atk/mips.hpp"
#include "atk/dataset.hpp"
#include "atk/simulate.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const atk::DatasetFormatError& e) {
    g_err = e.what();
    return 6;
  } catch (const atk::NoFeasibleConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

atk::AlgoParams mk(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, uint32_t lane) {
  atk::AlgoParams p;
  p.n = n;
  p.num_buckets = b;
  p.local_k = kp;
  p.global_k = k;
  p.lane_multiple = lane;
  return p;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_validate(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, uint32_t lane) {
  return guard([&] { mk(n, b, kp, k, lane).validate(); });
}

int ref_update_bucket(float* v, uint32_t* ix, uint32_t kp, float value, uint32_t index) {
  return guard([&] {
    atk::BucketState s(kp);
    std::memcpy(s.values.data(), v, 4 * kp);
    std::memcpy(s.indices.data(), ix, 4 * kp);
    atk::update_bucket(s, value, index);
    std::memcpy(v, s.values.data(), 4 * kp);
    std::memcpy(ix, s.indices.data(), 4 * kp);
  });
}

int ref_stage1(const float* in, uint64_t n, uint64_t b, uint32_t kp, uint32_t lane,
               float* vals, uint32_t* idx) {
  return guard([&] {
    auto p = mk(n, b, kp, 1, lane);
    auto g = atk::stage1_partial_reduce(std::span<const float>(in, n), p);
    std::memcpy(vals, g.values.data(), 4 * g.values.size());
    std::memcpy(idx, g.indices.data(), 4 * g.indices.size());
  });
}

int ref_select_candidates(const float* v, const uint32_t* ix, uint64_t count, uint32_t k,
                          uint64_t index_limit, float* ov, uint32_t* oi) {
  return guard([&] {
    auto r = atk::select_top_k_candidates(std::span<const float>(v, count),
                                          std::span<const uint32_t>(ix, count), k,
                                          index_limit);
    std::memcpy(ov, r.values.data(), 4 * r.values.size());
    std::memcpy(oi, r.indices.data(), 4 * r.indices.size());
  });
}

int ref_exact_top_k(const float* in, uint64_t n, uint32_t k, float* ov, uint32_t* oi) {
  return guard([&] {
    auto r = atk::exact_top_k(std::span<const float>(in, n), k);
    std::memcpy(ov, r.values.data(), 4 * r.values.size());
    std::memcpy(oi, r.indices.data(), 4 * r.indices.size());
  });
}

int ref_approx_top_k_batch(const float* rows, uint64_t row_count, uint64_t n, uint64_t b,
                           uint32_t kp, uint32_t k, uint32_t lane, uint32_t threads,
                           float* ov, uint32_t* oi) {
  return guard([&] {
    auto p = mk(n, b, kp, k, lane);
    auto res = atk::approx_top_k_batch(std::span<const float>(rows, row_count * n),
                                       row_count, p, threads);
    for (uint64_t r = 0; r < row_count; ++r) {
      std::memcpy(ov + r * k, res[r].values.data(), 4ull * k);
      std::memcpy(oi + r * k, res[r].indices.data(), 4ull * k);
    }
  });
}

int ref_measure_recall(const float* av, const uint32_t* ai, const float* ev,
                       const uint32_t* ei, uint64_t k, double* out) {
  return guard([&] {
    atk::TopKResult a{std::vector<float>(av, av + k), std::vector<uint32_t>(ai, ai + k)};
    atk::TopKResult e{std::vector<float>(ev, ev + k), std::vector<uint32_t>(ei, ei + k)};
    *out = atk::measure_recall(a, e);
  });
}

int ref_exact_expected_recall(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, double* out) {
  return guard([&] { *out = atk::exact_expected_recall(mk(n, b, kp, k, 1)).value; });
}

int ref_mc_expected_recall(uint64_t n, uint64_t b, uint32_t kp, uint32_t k, uint64_t trials,
                           uint64_t seed, double* mean, double* se) {
  return guard([&] {
    auto e = atk::mc_expected_recall(mk(n, b, kp, k, 1), trials, seed);
    *mean = e.value;
    *se = e.std_error.value();
  });
}

uint64_t ref_legal_bucket_counts(uint64_t n, uint64_t lane, uint64_t* out, uint64_t cap) {
  auto v = atk::legal_bucket_counts(n, lane);
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  return v.size();
}

int ref_select_parameters(uint64_t n, uint64_t k, double target, const uint32_t* kps,
                          uint32_t nkps, uint32_t lane, uint64_t seed, uint32_t* kp_out,
                          uint64_t* b_out, double* recall_out, int* exact_out, int* warn_out) {
  return guard([&] {
    atk::PlanRequest req;
    req.n = n;
    req.k = k;
    req.recall_target = target;
    req.allowed_local_k.assign(kps, kps + nkps);
    req.lane_multiple = lane;
    req.seed = seed;
    auto r = atk::select_parameters(req);
    *kp_out = r.local_k;
    *b_out = r.num_buckets;
    *recall_out = r.estimated_recall.value;
    *exact_out = r.estimated_recall.method == atk::RecallMethod::exact;
    *warn_out = r.high_target_warning;
  });
}

void ref_score_block(const float* queries, uint64_t b, const float* database, uint64_t rows,
                     uint64_t d, uint64_t c0, uint64_t c1, float* out, uint64_t out_stride) {
  atk::VectorDataset q, db;
  q.rows = b;
  q.dims = d;
  q.data.assign(queries, queries + b * d);
  db.rows = rows;
  db.dims = d;
  db.data.assign(database, database + rows * d);
  atk::score_block(q, db, c0, c1, out, out_stride);
}

// reference MIPS pipeline (mips.cpp:138-193): database [rows][d], queries
// [b][d] fp32; block_cols 0 = default_block_cols; results [b][k]
int ref_mips_fused(const float* database, uint64_t rows, uint64_t d, const float* queries, uint64_t b,
                   uint64_t nb, uint32_t kp, uint32_t k, uint32_t lane, uint64_t block_cols, uint32_t threads,
                   float* ov, uint32_t* oi) {
  return guard([&] {
    atk::VectorDataset q, db;
    q.rows = b;
    q.dims = d;
    q.data.assign(queries, queries + b * d);
    db.rows = rows;
    db.dims = d;
    db.data.assign(database, database + rows * d);
    auto p = mk(rows, nb, kp, k, lane);
    const uint64_t bc = block_cols ? block_cols : atk::default_block_cols(p);
    auto res = atk::mips_fused(db, q, p, bc, threads);
    for (uint64_t r = 0; r < b; ++r) {
      std::memcpy(ov + r * k, res.per_query[r].values.data(), 4ull * k);
      std::memcpy(oi + r * k, res.per_query[r].indices.data(), 4ull * k);
    }
  });
}

// dataset.cpp:45-130 (ATKV container), file-path entry points
int ref_dataset_write_file(const char* path, const float* data, uint64_t rows, uint64_t dims) {
  return guard([&] {
    atk::VectorDataset ds;
    ds.rows = rows;
    ds.dims = dims;
    ds.data.assign(data, data + rows * dims);
    atk::write_dataset_file(ds, path);
  });
}

int ref_dataset_read_file(const char* path, float* out, uint64_t cap, uint64_t* rows, uint64_t* dims) {
  return guard([&] {
    const atk::VectorDataset ds = atk::read_dataset_file(path);
    if (ds.data.size() > cap) throw std::invalid_argument("capacity");
    std::memcpy(out, ds.data.data(), ds.data.size() * 4);
    *rows = ds.rows;
    *dims = ds.dims;
  });
}

// dataset.cpp:132-150
int ref_synth_distinct_row(uint64_t n, uint64_t seed, uint64_t row_index, float* out) {
  return guard([&] {
    const auto row = atk::synth_distinct_row(n, seed, row_index);
    std::memcpy(out, row.data(), row.size() * 4);
  });
}

// simulate.cpp:53-113; configs as (n, b, kp, k, lane) records
int ref_simulate_recall_many(const uint64_t* cfg, uint32_t num, uint64_t runs, uint64_t seed,
                             uint32_t threads, double* mean, double* sd) {
  return guard([&] {
    std::vector<atk::AlgoParams> ps;
    for (uint32_t c = 0; c < num; ++c)
      ps.push_back(mk(cfg[5 * c], cfg[5 * c + 1], static_cast<uint32_t>(cfg[5 * c + 2]),
                      static_cast<uint32_t>(cfg[5 * c + 3]), static_cast<uint32_t>(cfg[5 * c + 4])));
    const auto st = atk::simulate_recall_many(ps, runs, seed, threads);
    for (uint32_t c = 0; c < num; ++c) {
      mean[c] = st[c].mean_recall;
      sd[c] = st[c].stddev;
    }
  });
}

}  // extern "C"
