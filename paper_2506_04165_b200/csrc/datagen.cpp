// datagen.cpp -- seeded synthetic inputs shared by the GPU path, the oracle
// and the CPU baseline (identical bytes everywhere).
//
// The reference has no normal generator (its fixtures are uniform or
// permutation rows, proj/tools/atk.cpp:286-288, dataset.cpp:132-150), so this
// is a documented build convention:
//   element i of a flat [rows * n] buffer = mean + stddev * z_i, where the
//   buffer is cut into blocks of 65536 elements, block q draws from
//   xoshiro256++(derive_seed(seed, q)) (rng.hpp:25-81), and each pair of
//   uniforms (u1, u2) gives z = sqrt(-2 ln(1-u1)) * (cos, sin)(2 pi u2)
//   evaluated in double and rounded once to fp32.
// bf16 inputs are the round-to-nearest-even conversion of that fp32 stream.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/atkg.h"

namespace atkg {
uint64_t derive_seed(uint64_t seed, uint64_t stream);
}

namespace {

constexpr uint64_t kBlock = 65536;

struct Xo {
  uint64_t s[4];
  static uint64_t sm(uint64_t& st) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  explicit Xo(uint64_t seed) { uint64_t st = seed; for (auto& w : s) w = sm(st); }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  double u() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

template <class F>
void parallel_blocks(uint64_t blocks, uint32_t threads, F&& f) {
  if (threads <= 1 || blocks <= 1) {
    for (uint64_t q = 0; q < blocks; ++q) f(q);
    return;
  }
  const uint64_t w = std::min<uint64_t>(threads, blocks);
  std::vector<std::thread> pool;
  for (uint64_t t = 0; t < w; ++t)
    pool.emplace_back([&, t] { for (uint64_t q = t; q < blocks; q += w) f(q); });
  for (auto& th : pool) th.join();
}

inline uint16_t to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);  // quiet NaN
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return static_cast<uint16_t>(u >> 16);
}

}  // namespace

extern "C" {

void atkg_fill_normal_range(uint64_t seed, uint64_t start, uint64_t count, float mean, float stddev, float* out,
                            uint32_t threads) {
  // elements [start, start + count) of the flat stream; start % kBlock == 0
  // (the caller checks), so every generator block is produced whole
  const uint64_t q0 = start / kBlock;
  const uint64_t blocks = (count + kBlock - 1) / kBlock;
  const double two_pi = 6.283185307179586476925286766559;
  parallel_blocks(blocks, threads, [&](uint64_t qq) {
    Xo rng(atkg::derive_seed(seed, q0 + qq));
    const uint64_t i0 = qq * kBlock, i1 = std::min(count, i0 + kBlock);
    for (uint64_t i = i0; i < i1; i += 2) {
      const double u1 = rng.u(), u2 = rng.u();
      const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
      const double a = two_pi * u2;
      out[i] = static_cast<float>(static_cast<double>(mean) + static_cast<double>(stddev) * (r * std::cos(a)));
      if (i + 1 < i1)
        out[i + 1] = static_cast<float>(static_cast<double>(mean) + static_cast<double>(stddev) * (r * std::sin(a)));
    }
  });
}

void atkg_fill_normal(uint64_t seed, uint64_t count, float mean, float stddev, float* out,
                      uint32_t threads) {
  atkg_fill_normal_range(seed, 0, count, mean, stddev, out, threads);
}

void atkg_f32_to_bf16(const float* in, uint64_t count, uint16_t* out, uint32_t threads) {
  const uint64_t blocks = (count + kBlock - 1) / kBlock;
  parallel_blocks(blocks, threads, [&](uint64_t q) {
    const uint64_t i1 = std::min(count, (q + 1) * kBlock);
    for (uint64_t i = q * kBlock; i < i1; ++i) out[i] = to_bf16_rne(in[i]);
  });
}

void atkg_bf16_to_f32(const uint16_t* in, uint64_t count, float* out, uint32_t threads) {
  const uint64_t blocks = (count + kBlock - 1) / kBlock;
  parallel_blocks(blocks, threads, [&](uint64_t q) {
    const uint64_t i1 = std::min(count, (q + 1) * kBlock);
    for (uint64_t i = q * kBlock; i < i1; ++i) {
      const uint32_t u = static_cast<uint32_t>(in[i]) << 16;
      std::memcpy(&out[i], &u, 4);
    }
  });
}

}  // extern "C"
