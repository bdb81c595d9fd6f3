// TEST INFRASTRUCTURE: host-side emulation of the stage-1 device logic.
//
// Compiles paper_2506_04165_b200/csrc/stage1.cuh with nvcc and drives the
// SAME Summ<KP> code the kernels run (fill / slow / push / merge_later /
// finalize are __host__ __device__) on the CPU, so the exact split-merge
// algorithm is checked against the reference Alg. 1 without a GPU
// (tests/test_summary_emulation.py).  Nothing here is product code.
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2506_04165_b200/csrc/stage1.cuh"

using namespace atkg;

template <int KP>
static void run(const float* row, uint64_t n, uint64_t B, const uint32_t* bounds, uint32_t nsegs, int mode,
                uint64_t seed, float* gv, uint32_t* gi, uint32_t* nan_out) {
  const uint64_t nstr = n / B;
  std::mt19937_64 rng(seed);
  uint32_t nan = 0;
  for (uint64_t b = 0; b < B; ++b) {
    Summ<KP> acc;
    if (mode == 2) {  // accumulator: element-wise push
      acc.clear();
      for (uint64_t j = 0; j < nstr; ++j) acc.push(row[j * B + b], (uint32_t)(j * B + b), nan);
    } else {
      std::vector<Summ<KP>> parts;
      for (uint32_t s = 0; s < nsegs; ++s) {
        Summ<KP> sm;
        sm.clear();
        const uint64_t j0 = bounds[s], j1 = bounds[s + 1];
        uint64_t j = j0;
        for (int t = 0; t < KP && j < j1; ++t, ++j) {
          const float x = row[j * B + b];
          nan |= (x != x);
          sm.fill(t, x, (uint32_t)(j * B + b));
        }
        for (; j < j1; ++j) {
          const float x = row[j * B + b];
          if (!(x < sm.v[KP - 1])) sm.slow(x, (uint32_t)(j * B + b), nan);
        }
        parts.push_back(sm);
      }
      if (mode == 0) {
        acc = parts[0];
        for (size_t q = 1; q < parts.size(); ++q) acc.merge_later(parts[q]);
      } else {  // random association order (adjacent pairs only)
        while (parts.size() > 1) {
          const size_t q = rng() % (parts.size() - 1);
          parts[q].merge_later(parts[q + 1]);
          parts.erase(parts.begin() + q + 1);
        }
        acc = parts[0];
      }
    }
    float ov[KP];
    uint32_t oi[KP];
    acc.finalize(ov, oi);
    for (int k = 0; k < KP; ++k) {
      gv[(uint64_t)k * B + b] = ov[k];
      gi[(uint64_t)k * B + b] = oi[k];
    }
  }
  *nan_out = nan;
}

extern "C" int emu_stage1(const float* row, uint64_t n, uint64_t B, uint32_t kp, const uint32_t* bounds,
                          uint32_t nsegs, int mode, uint64_t seed, float* gv, uint32_t* gi, uint32_t* nan) {
  switch (kp) {
    case 1: run<1>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 2: run<2>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 3: run<3>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 4: run<4>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 5: run<5>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 6: run<6>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 7: run<7>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 8: run<8>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    case 16: run<16>(row, n, B, bounds, nsegs, mode, seed, gv, gi, nan); return 0;
    default: return 5;
  }
}

// ---- slice summaries in the library's memory layout (atkg_stage1_summary):
// words = v[KP][B], p[KP][B], lt[B], ltv[B] ----------------------------------
template <int KP>
static void slice_summary(const float* x, uint64_t len, uint64_t offset, uint64_t B, uint32_t* words,
                          uint32_t* nan) {
  for (uint64_t b = 0; b < B; ++b) {
    Summ<KP> s;
    s.clear();
    for (uint64_t j = 0; j * B + b < len; ++j) s.push(x[j * B + b], (uint32_t)(offset + j * B + b), *nan);
    for (int k = 0; k < KP; ++k) {
      std::memcpy(&words[(uint64_t)k * B + b], &s.v[k], 4);
      words[(uint64_t)(KP + k) * B + b] = s.p[k];
    }
    words[(uint64_t)(2 * KP) * B + b] = s.lt;
    std::memcpy(&words[(uint64_t)(2 * KP + 1) * B + b], &s.ltv, 4);
  }
}

template <int KP>
static void merge_summaries(const uint32_t* words, uint32_t parts, uint64_t B, float* gv, uint32_t* gi) {
  const uint64_t W = (2ull * KP + 2) * B;
  for (uint64_t b = 0; b < B; ++b) {
    Summ<KP> acc;
    for (uint32_t g = 0; g < parts; ++g) {
      const uint32_t* w = words + g * W;
      Summ<KP> s;
      for (int k = 0; k < KP; ++k) {
        std::memcpy(&s.v[k], &w[(uint64_t)k * B + b], 4);
        s.p[k] = w[(uint64_t)(KP + k) * B + b];
      }
      s.lt = w[(uint64_t)(2 * KP) * B + b];
      std::memcpy(&s.ltv, &w[(uint64_t)(2 * KP + 1) * B + b], 4);
      if (g == 0) acc = s;
      else acc.merge_later(s);
    }
    float ov[KP];
    uint32_t oi[KP];
    acc.finalize(ov, oi);
    for (int k = 0; k < KP; ++k) {
      gv[(uint64_t)k * B + b] = ov[k];
      gi[(uint64_t)k * B + b] = oi[k];
    }
  }
}

#define EMU_KP_SWITCH(kp, CALL)  \
  switch (kp) {                  \
    case 1: { constexpr int K_ = 1; CALL; return 0; } \
    case 2: { constexpr int K_ = 2; CALL; return 0; } \
    case 4: { constexpr int K_ = 4; CALL; return 0; } \
    case 8: { constexpr int K_ = 8; CALL; return 0; } \
    default: return 5;           \
  }

extern "C" int emu_slice_summary(const float* x, uint64_t len, uint64_t offset, uint64_t B, uint32_t kp,
                                 uint32_t* words, uint32_t* nan) {
  EMU_KP_SWITCH(kp, (slice_summary<K_>(x, len, offset, B, words, nan)))
}

extern "C" int emu_merge_summaries(const uint32_t* words, uint32_t parts, uint64_t B, uint32_t kp, float* gv,
                                   uint32_t* gi) {
  EMU_KP_SWITCH(kp, (merge_summaries<K_>(words, parts, B, gv, gi)))
}
