// simulate.cu -- empirical recall simulation with the top-k on the GPU.
//
// Restates simulate.cpp:53-113 and synth_distinct_row (dataset.cpp:132-150):
// run r is a Fisher-Yates permutation of 1..n on xoshiro256++(derive_seed(seed,
// r)); every configuration's approx_top_k runs on it; recall is |approx ∩ true|
// / k, where the true top-k set is the positions holding values > n - k.
//
// B200 split:
// * Row generation is a serial swap chain per row (bit-exact to the reference
//   needs the same draw order), so host threads build a batch of rows, one row
//   per thread at a time, into pinned memory while the GPU works on the
//   previous batch.
// * The batch is copied to HBM once and shared by every configuration:
//   atkg_approx_top_k (the hot path) then recall_hits_kernel, which gathers
//   row[idx] for the K winners and counts values > n - k.  Because the winners
//   are distinct positions this equals the reference's sorted intersection.
// * Only the per-run hit counts come back; mean / stddev are the reference's
//   Welford recurrence in run order, so the statistics match bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace atkg {
uint64_t derive_seed(uint64_t seed, uint64_t stream);  // planner.cpp (rng.hpp:25-32)

namespace {

constexpr uint64_t kMaxSynthN = 1ull << 24;  // dataset.cpp:15

struct Xoshiro {  // rng.hpp:34-81
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& w : s) {
      uint64_t z = (sm += 0x9e3779b97f4a7c15ull);
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      w = z ^ (z >> 31);
    }
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
  uint64_t below(uint64_t bound) {  // rng.hpp:59-73 (Lemire, rejection on the low word)
    using u128 = unsigned __int128;
    u128 m = static_cast<u128>(next()) * bound;
    uint64_t lo = static_cast<uint64_t>(m);
    if (lo < bound) {
      const uint64_t threshold = (0 - bound) % bound;
      while (lo < threshold) {
        m = static_cast<u128>(next()) * bound;
        lo = static_cast<uint64_t>(m);
      }
    }
    return static_cast<uint64_t>(m >> 64);
  }
};

void check_synth_n(uint64_t n) {
  if (n == 0) throw Inval("synth_distinct: n must be >= 1");
  if (n > kMaxSynthN) throw Inval("synth_distinct: n must be <= 2^24 so values stay fp32-exact");
}

// dataset.cpp:132-150
void synth_row(uint64_t n, uint64_t seed, uint64_t row_index, float* row) {
  for (uint64_t i = 0; i < n; ++i) row[i] = static_cast<float>(i + 1);
  Xoshiro rng(derive_seed(seed, row_index));
  for (uint64_t i = n - 1; i >= 1; --i) std::swap(row[i], row[rng.below(i + 1)]);
}

void synth_rows(uint64_t first, uint64_t rows, uint64_t n, uint64_t seed, float* out, unsigned threads) {
  threads = std::max(1u, std::min<unsigned>(threads, static_cast<unsigned>(std::max<uint64_t>(rows, 1))));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([=] {
      for (uint64_t r = t; r < rows; r += threads) synth_row(n, seed, first + r, out + r * n);
    });
  for (auto& th : pool) th.join();
}

// One warp per run: hits[run] = #{j < k : row[idx[j]] > n - k}.
__global__ void __launch_bounds__(256) recall_hits_kernel(const float* __restrict__ rows, uint64_t n,
                                                          const uint32_t* __restrict__ idx, uint32_t k,
                                                          uint64_t nrows, uint32_t* __restrict__ hits) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x / 32) + threadIdx.x / 32;
  if (r >= nrows) return;
  const unsigned lane = threadIdx.x & 31;
  const float thr = static_cast<float>(n - k);  // simulate.cpp:22
  const float* row = rows + r * n;
  const uint32_t* ir = idx + r * k;
  uint32_t c = 0;
  for (uint32_t j = lane; j < k; j += 32) c += __ldg(row + __ldg(ir + j)) > thr;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) hits[r] = c;
}

// Device Fisher-Yates, one CTA per row with the row in shared memory as u16
// (value - 1; n <= 2^16 keeps 128 KB per row).  The swap chain is serial by
// definition, so one thread walks it; the CTA fills and writes the row out
// coalesced.  Draws are the host Xoshiro's, bit for bit (rng.hpp:34-81).
constexpr uint64_t kDeviceSynthMaxN = 1ull << 16;

__device__ __forceinline__ uint64_t d_splitmix(uint64_t& st) {
  uint64_t z = (st += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t d_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__global__ void __launch_bounds__(128) synth_distinct_kernel(uint64_t first_row, uint64_t n, uint64_t seed,
                                                             float* __restrict__ out) {
  extern __shared__ uint16_t perm[];
  const uint64_t row = first_row + blockIdx.x;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) perm[i] = static_cast<uint16_t>(i);
  __syncthreads();
  if (threadIdx.x == 0) {
    // derive_seed(seed, row) (rng.hpp:25-32), then the xoshiro256++ state
    uint64_t st = seed;
    (void)d_splitmix(st);
    st ^= 0x9e3779b97f4a7c15ull * (row + 1);
    const uint64_t a = d_splitmix(st), b = d_splitmix(st);
    uint64_t sm = a ^ (b >> 1), s0, s1, s2, s3;
    s0 = d_splitmix(sm);
    s1 = d_splitmix(sm);
    s2 = d_splitmix(sm);
    s3 = d_splitmix(sm);
    for (uint64_t i = n - 1; i >= 1; --i) {
      const uint64_t bound = i + 1;
      uint64_t x = d_rotl(s0 + s3, 23) + s0;
      uint64_t t = s1 << 17;
      s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = d_rotl(s3, 45);
      uint64_t lo = x * bound, hi = __umul64hi(x, bound);
      if (lo < bound) {
        const uint64_t threshold = (0 - bound) % bound;
        while (lo < threshold) {
          x = d_rotl(s0 + s3, 23) + s0;
          t = s1 << 17;
          s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = d_rotl(s3, 45);
          lo = x * bound;
          hi = __umul64hi(x, bound);
        }
      }
      const uint16_t vi = perm[i], vj = perm[hi];
      perm[i] = vj;
      perm[hi] = vi;
    }
  }
  __syncthreads();
  float* o = out + blockIdx.x * n;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) o[i] = static_cast<float>(perm[i]) + 1.0f;
}

void launch_synth_distinct(uint64_t first_row, uint64_t rows, uint64_t n, uint64_t seed, float* d_out,
                           cudaStream_t s) {
  if (rows == 0) return;
  const size_t smem = n * sizeof(uint16_t);
  // the opt-in shared-memory limit is per device: set it on every call (cheap)
  CUDA_OK(cudaFuncSetAttribute(synth_distinct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kDeviceSynthMaxN * sizeof(uint16_t))));
  for (uint64_t r0 = 0; r0 < rows; r0 += 65535) {
    const unsigned g = static_cast<unsigned>(std::min<uint64_t>(65535, rows - r0));
    synth_distinct_kernel<<<g, 128, smem, s>>>(first_row + r0, n, seed, d_out + r0 * n);
    check_launch();
  }
}

struct Pinned {
  void* p = nullptr;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};
struct Device {
  void* p = nullptr;
  ~Device() {
    if (p) cudaFree(p);
  }
};

}  // namespace
}  // namespace atkg

using namespace atkg;

extern "C" {

int atkg_synth_distinct(uint64_t first_row, uint64_t rows, uint64_t n, uint64_t seed, float* out,
                        uint32_t threads) {
  return guarded([&] {
    check_synth_n(n);
    if (rows && !out) throw Inval("output buffer must not be null");
    synth_rows(first_row, rows, n, seed, out, threads);
  });
}

int atkg_synth_distinct_device(uint64_t first_row, uint64_t rows, uint64_t n, uint64_t seed, float* d_out,
                               void* stream) {
  return guarded([&] {
    check_synth_n(n);
    if (n > kDeviceSynthMaxN) throw Unsupported("synth_distinct on the device: n must be <= 2^16");
    if (rows && !d_out) throw Inval("output buffer must not be null");
    launch_synth_distinct(first_row, rows, n, seed, d_out, static_cast<cudaStream_t>(stream));
  });
}

int atkg_simulate_recall_many(const atkg_params* configs, uint32_t num_configs, uint64_t runs,
                              uint64_t seed, uint32_t threads, double* mean_recall, double* stddev,
                              void* stream) {
  return guarded([&] {
    // simulate.cpp:53-66
    if (num_configs == 0 || !configs) throw Inval("simulate: no configurations");
    if (runs == 0) throw Inval("simulate: runs must be >= 1");
    const uint64_t n = configs[0].n;
    for (uint32_t c = 0; c < num_configs; ++c) {
      if (atkg_validate(&configs[c]) != ATKG_OK) throw Inval(atkg_last_error());
      if (configs[c].n != n) throw Inval("simulate: configurations must share n");
    }
    check_synth_n(n);
    if (!mean_recall || !stddev) throw Inval("output pointers must not be null");
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    // Batches of runs: about 32 MiB of rows (at least one row per worker) per
    // pinned buffer, so pinning stays cheap and generation overlaps the GPU.
    // Rows of n <= 2^16 are generated on the device (synth_distinct_kernel):
    // no host generation, no H2D; larger rows come from host workers.
    const bool dev_gen = n <= kDeviceSynthMaxN && !opt("sim_host_gen", 0);
    const uint64_t workers = std::max<uint32_t>(threads, 1);
    const uint64_t batch = dev_gen ? std::min<uint64_t>(runs, 2048)
                                   : std::min<uint64_t>(runs, std::max<uint64_t>(workers, (1ull << 23) / n));
    uint32_t kmax = 0;
    size_t ws = 0;
    for (uint32_t c = 0; c < num_configs; ++c) {
      kmax = std::max(kmax, configs[c].global_k);
      size_t b = 0;
      if (atkg_workspace_size(ATKG_OP_APPROX, ATKG_F32, batch, &configs[c], &b) != ATKG_OK)
        throw Inval(atkg_last_error());
      ws = std::max(ws, b);
    }
    Pinned host[2], hits_h;
    Device d_rows, d_vals, d_idx, d_ws, d_hits, d_status;
    if (!dev_gen)
      for (auto& h : host) CUDA_OK(cudaHostAlloc(&h.p, batch * n * 4, cudaHostAllocDefault));
    CUDA_OK(cudaHostAlloc(&hits_h.p, size_t(num_configs) * runs * 4, cudaHostAllocDefault));
    CUDA_OK(cudaMalloc(&d_rows.p, batch * n * 4));
    CUDA_OK(cudaMalloc(&d_vals.p, batch * kmax * 4));
    CUDA_OK(cudaMalloc(&d_idx.p, batch * kmax * 4));
    CUDA_OK(cudaMalloc(&d_ws.p, std::max<size_t>(ws, 256)));
    CUDA_OK(cudaMalloc(&d_hits.p, size_t(num_configs) * runs * 4));
    CUDA_OK(cudaMalloc(&d_status.p, 4));
    CUDA_OK(cudaMemsetAsync(d_status.p, 0, 4, s));
    cudaEvent_t copied[2];
    for (auto& e : copied) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EvGuard {
      cudaEvent_t* e;
      ~EvGuard() {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
      }
    } ev_guard{copied};

    const uint64_t nbatches = (runs + batch - 1) / batch;
    auto gen = [&](uint64_t bi) {
      const uint64_t r0 = bi * batch, nr = std::min(batch, runs - r0);
      synth_rows(r0, nr, n, seed, static_cast<float*>(host[bi & 1].p), threads);
    };
    if (!dev_gen) gen(0);
    uint32_t* hits = static_cast<uint32_t*>(d_hits.p);
    for (uint64_t bi = 0; bi < nbatches; ++bi) {
      const uint64_t r0 = bi * batch, nr = std::min(batch, runs - r0);
      if (dev_gen) {
        launch_synth_distinct(r0, nr, n, seed, static_cast<float*>(d_rows.p), s);
      } else {
        CUDA_OK(cudaMemcpyAsync(d_rows.p, host[bi & 1].p, nr * n * 4, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaEventRecord(copied[bi & 1], s));
      }
      for (uint32_t c = 0; c < num_configs; ++c) {
        const int rc = atkg_approx_top_k(ATKG_F32, d_rows.p, nr, &configs[c], static_cast<float*>(d_vals.p),
                                         static_cast<uint32_t*>(d_idx.p), d_ws.p, ws,
                                         static_cast<uint32_t*>(d_status.p), stream);
        if (rc != ATKG_OK) throw Inval(atkg_last_error());
        const unsigned warps = 8;
        recall_hits_kernel<<<static_cast<unsigned>((nr + warps - 1) / warps), warps * 32, 0, s>>>(
            static_cast<const float*>(d_rows.p), n, static_cast<const uint32_t*>(d_idx.p), configs[c].global_k,
            nr, hits + uint64_t(c) * runs + r0);
        check_launch();
      }
      // generate the next batch while the GPU works on this one; the buffer it
      // overwrites was last read by the copy of batch bi - 1
      if (!dev_gen && bi + 1 < nbatches) {
        CUDA_OK(cudaEventSynchronize(copied[(bi + 1) & 1]));
        gen(bi + 1);
      }
      // d_rows is reused next batch: the next copy is stream-ordered after this batch's kernels
    }
    CUDA_OK(cudaMemcpyAsync(hits_h.p, d_hits.p, size_t(num_configs) * runs * 4, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    if (atkg_check_status(static_cast<uint32_t*>(d_status.p), stream) != ATKG_OK) throw Inval(atkg_last_error());
    // simulate.cpp:95-109: Welford over runs in order, sample stddev (ddof 1)
    const uint32_t* hh = static_cast<const uint32_t*>(hits_h.p);
    for (uint32_t c = 0; c < num_configs; ++c) {
      double mean = 0.0, m2 = 0.0;
      for (uint64_t r = 0; r < runs; ++r) {
        const double rec = static_cast<double>(hh[uint64_t(c) * runs + r]) /
                           static_cast<double>(configs[c].global_k);
        const double delta = rec - mean;
        mean += delta / static_cast<double>(r + 1);
        m2 += delta * (rec - mean);
      }
      mean_recall[c] = mean;
      stddev[c] = runs > 1 ? std::sqrt(m2 / static_cast<double>(runs - 1)) : 0.0;
    }
  });
}

}  // extern "C"
