// TEST INFRASTRUCTURE: host-side emulation of the stage-1 device logic.
//
// Compiles paper_2506_04165_b200/csrc/stage1.cuh with nvcc and drives the
// SAME Summ<KP> code the kernels run (fill / slow / push / merge_later /
// finalize are __host__ __device__) on the CPU, so the exact split-merge
// algorithm is checked against the reference Alg. 1 without a GPU
// (tests/test_summary_emulation.py).  Nothing here is product code.
#include <cstdint>
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
