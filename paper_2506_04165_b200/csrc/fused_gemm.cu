// fused_gemm.cu -- C4: bf16 x[M,Kd] . W[Kd,N] on tcgen05 tensor cores with
// stage 1 of the approximate top-K in the GEMM epilogue.
//
// Reference semantics: mips_fused / mips_unfused
// (/root/reference/proj/core/src/mips.cpp:109-193): score every (query, db
// row) pair, feed the scores of one query to stage 1 in column order, then
// stage 2.  The reference scores in fp32 on the CPU (score_block,
// mips.cpp:57-95); here the scores are fp32 tensor-core accumulations of bf16
// products, and the parity oracle is the reference's approx_top_k run on the
// fp32 scores this kernel produced (dumped through d_scores).
//
// Tiling ("bucket-complete tiles").  Column c lives in bucket c mod B at
// stride-row s = c / B, S = N / B stride-rows per bucket.  Viewing W^T
// [N][Kd] as a 3-D tensor [S][B][Kd], one TMA box of [S][NB][64] loads NB
// *complete* buckets (TN = NB*S <= 256 columns) for a 64-deep K slice.  The
// shared-memory B tile is therefore ordered n = s*NB + j (bucket b0 + j), and
// after the K loop every TMEM lane (= one query row) holds all S elements of
// NB buckets.  Stage 1 for those buckets is then a purely thread-local,
// in-order Alg. 1 pass (Summ<KP>, stage1.cuh) with no cross-tile state, and
// the epilogue emits K' candidates per bucket.  The M x N score matrix never
// touches HBM.
//
// Kernel shape: persistent, one CTA per SM, 6 warps.
//   warp 0      TMA producer (one lane): A box [128 rows][64], B box above,
//               kStages-deep smem ring (full/empty mbarriers)
//   warp 1      TMEM allocator + MMA issuer (one lane): 4 x
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=TN, K=16) per
//               stage, tcgen05.commit -> empty[stage]; -> tmem_full[acc]
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 (lane = row), Alg. 1 per
//               bucket, candidates to HBM; two TMEM accumulators (2*TN <= 512
//               columns) so the epilogue of tile t overlaps the MMAs of t+1.
// The plain GEMM (atkg_gemm_bf16) is the same kernel with a 2-D B box of
// 256 rows and an epilogue that stores fp32 scores.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/atkg.h"
#include "host_common.hpp"
#include "internal.hpp"
#include "ptx.cuh"
#include "summ.cuh"

namespace atkg {

constexpr uint32_t kBM = 128;      // rows per CTA tile (TMEM lanes)
constexpr uint32_t kBK = 64;       // K per stage: one 128-byte swizzle row
constexpr uint32_t kPlainTN = 256;  // columns per tile of the plain GEMM
constexpr uint32_t kSmemBudget = 227 * 1024;

struct GemmArgs {
  uint32_t m, kdim, n;
  uint32_t m_blocks, n_tiles, k_blocks;  // m_blocks counts CG*128-row blocks
  uint32_t tn;          // columns per tile (MMA N)
  uint32_t S;           // stride-rows per bucket (fused)
  uint32_t B;           // buckets (fused)
  uint32_t cand_stride; // candidates per row = B * KP (fused)
  uint32_t stages;      // smem ring depth
  uint32_t n_panel;     // tile order: panels of n_panel column tiles (their W stays in L2), rows inside
  float* out;           // plain: scores [m][n]; fused: optional score dump
  float* cand_v;        // fused: [m][B*KP]
  uint32_t* cand_i;
  uint32_t* status;
};

// Tile t -> (row block mb, column tile g).  Column tiles are taken in panels
// of n_panel: inside a panel the column tile runs fastest, then the row
// block, so the tiles in flight share one W panel (L2-resident, 3.2 MB per
// C4 column tile) and each x row block is read once per panel.
__device__ __forceinline__ void gemm_tile_coords(const GemmArgs& a, uint32_t t, uint32_t& mb, uint32_t& g) {
  const uint32_t per_panel = a.n_panel * a.m_blocks;
  const uint32_t pn = t / per_panel, r = t - pn * per_panel;
  const uint32_t g0 = pn * a.n_panel, w = min(a.n_panel, a.n_tiles - g0);  // the last panel may be narrower
  mb = r / w;
  g = g0 + (r - mb * w);
}

// per-CTA bytes of one pipeline stage: A [128][64] + this CTA's share of B
__host__ __device__ constexpr uint32_t gemm_stage_bytes(uint32_t tn, uint32_t cg) {
  return kBM * 128 + (tn / cg) * 128;
}
inline uint32_t gemm_stages(uint32_t tn, uint32_t cg) {
  const uint32_t st = (kSmemBudget - 2048) / gemm_stage_bytes(tn, cg);
  return st > 8 ? 8 : st;
}
inline size_t gemm_smem_bytes(uint32_t tn, uint32_t cg) {
  return 1024 /*alignment slack*/ + (size_t)gemm_stages(tn, cg) * gemm_stage_bytes(tn, cg) + 256 /*barriers*/;
}

// epilogue warps: 4 (one per TMEM lane quarter), or 8 for fused tiles with
// several buckets (two warps per quarter, each owning every other bucket)
__host__ __device__ constexpr int gemm_epi_warps(int nb) { return nb >= 2 ? 8 : 4; }
__host__ __device__ constexpr int gemm_threads(int nb) { return 64 + 32 * gemm_epi_warps(nb); }

// Alg. 1 over `W` consecutive stride-rows of one bucket, list already full
template <int KP, int W>
__device__ __forceinline__ void bucket_chunk(Summ<KP>& s, const uint32_t (&r)[W], uint32_t pos0, uint32_t B,
                                             uint32_t& nan) {
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const float x = __uint_as_float(r[e]);
    if (!(x < s.v[KP - 1])) s.slow(x, pos0 + e * B, nan);
  }
}

// CG: CTAs per MMA (1, or 2 = a CTA pair with cta_group::2, M = 256);
// NB: buckets per tile (0 = plain GEMM); KP: local_k
template <int CG, int NB, int KP>
__global__ void __launch_bounds__(gemm_threads(NB), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const GemmArgs a) {
  constexpr int kEpiWarps = gemm_epi_warps(NB);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t stage_bytes = gemm_stage_bytes(a.tn, CG);
  const uint32_t nst = a.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
  uint64_t* empty = full + nst;
  uint64_t* tmem_full = empty + nst;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;
  const uint32_t unit = blockIdx.x / CG, nunits = gridDim.x / CG;
  const uint32_t ntiles = a.m_blocks * a.n_tiles;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&map_a);
    ptx::prefetch_tmap(&map_b);
    for (uint32_t s = 0; s < nst; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tmem_full[s], 1);
      ptx::mbar_init(&tmem_empty[s], kEpiWarps * CG);  // one arrival per epilogue warp of the group
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) ptx::tc::alloc_pair(tmem_base_slot, 512);
    else ptx::tc::alloc(tmem_base_slot, 512);
  }
  ptx::tc::fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc::fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs of a pair)
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = unit; t < ntiles; t += nunits) {
        uint32_t mb, g;
        gemm_tile_coords(a, t, mb, g);
        const int32_t row0 = (int32_t)(mb * kBM * CG + rank * kBM);
        for (uint32_t kb = 0; kb < a.k_blocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * stage_bytes;
          uint8_t* sb = sa + kBM * 128;
          const int32_t k0 = (int32_t)(kb * kBK);
          if constexpr (CG == 1) {
            ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
            ptx::tma_load_2d(sa, &map_a, k0, row0, &full[stage]);
            if constexpr (NB == 0) {
              ptx::tma_load_2d(sb, &map_b, k0, (int32_t)(g * a.tn), &full[stage]);
            } else {
#pragma unroll
              for (int j = 0; j < NB; ++j)  // bucket-major: bucket j = rows [j*S, (j+1)*S)
                ptx::tma_load_3d(sb + j * a.S * 128, &map_b, k0, (int32_t)(g * NB + j), 0, &full[stage]);
            }
          } else {
            // the leader's barrier counts both CTAs' bytes
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);
            const uint32_t bar = ptx::mapa(ptx::smem_addr(&full[stage]), 0);
            ptx::tma_load_2d_pair(sa, &map_a, k0, row0, bar);
            if constexpr (NB == 0) {
              ptx::tma_load_2d_pair(sb, &map_b, k0, (int32_t)(g * a.tn + rank * (a.tn / 2)), bar);
            } else if constexpr (NB == 1) {  // half of the bucket's stride-rows each
              ptx::tma_load_3d_pair(sb, &map_b, k0, (int32_t)g, (int32_t)(rank * (a.S / 2)), bar);
            } else {  // half of the buckets each
#pragma unroll
              for (int j = 0; j < NB / 2; ++j)
                ptx::tma_load_3d_pair(sb + j * a.S * 128, &map_b, k0, (int32_t)(g * NB + rank * (NB / 2) + j), 0,
                                      bar);
            }
          }
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (leader CTA)
      const uint32_t idesc = ptx::tc::idesc_bf16(kBM * CG, a.tn);
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (uint32_t t = unit; t < ntiles; t += nunits) {
        ptx::mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        ptx::tc::fence_after();
        const uint32_t d = tmem_base + acc * a.tn;
        for (uint32_t kb = 0; kb < a.k_blocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc::fence_after();
          const uint32_t sa = ptx::smem_addr(smem + stage * stage_bytes);
          const uint64_t da = ptx::tc::desc_sw128(sa), db = ptx::tc::desc_sw128(sa + kBM * 128);
#pragma unroll
          for (uint32_t k = 0; k < kBK / 16; ++k) {  // +32 bytes along K per UMMA_K = 16
            if constexpr (CG == 2) ptx::tc::mma_bf16_pair(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
            else ptx::tc::mma_bf16(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          }
          if constexpr (CG == 2) ptx::tc::commit_pair(&empty[stage], 0x3);
          else ptx::tc::commit(&empty[stage]);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        if constexpr (CG == 2) ptx::tc::commit_pair(&tmem_full[acc], 0x3);
        else ptx::tc::commit(&tmem_full[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {  // ---------------------------- epilogue warps (both CTAs)
    const uint32_t q = warp & 3;           // TMEM lane quarter this warp may access
    const uint32_t eg = (warp - 2) / 4;    // epilogue group: buckets j = eg, eg + 2, ...
    uint32_t acc = 0, acc_phase = 0, nan = 0;
    const uint32_t release = CG == 2 ? ptx::mapa(ptx::smem_addr(&tmem_empty[0]), 0) : 0;
    for (uint32_t t = unit; t < ntiles; t += nunits) {
      uint32_t mb, g;
      gemm_tile_coords(a, t, mb, g);
      const uint32_t row = mb * kBM * CG + rank * kBM + q * 32 + lane;
      const bool live = row < a.m;
      ptx::mbar_wait(&tmem_full[acc], acc_phase);
      ptx::tc::fence_after();
      const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * a.tn;
      auto release_tmem = [&] {
        ptx::tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) ptx::mbar_arrive_cluster(release + acc * 8);
          else ptx::mbar_arrive(&tmem_empty[acc]);
        }
      };
      if constexpr (NB == 0) {
        const uint32_t c0 = g * a.tn;
        for (uint32_t c = 0; c < a.tn; c += 32) {
          uint32_t r[32];
          __syncwarp();
          ptx::tc::ld32x32(taddr + c, r);
          ptx::tc::wait_ld();
          if (live) {
            float* o = a.out + (uint64_t)row * a.n + c0 + c;
            if (c0 + c + 32 <= a.n && (a.n & 3) == 0) {
#pragma unroll
              for (int e = 0; e < 32; e += 4)
                *reinterpret_cast<float4*>(o + e) = make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                                                                __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (c0 + c + e < a.n) o[e] = __uint_as_float(r[e]);
            }
          }
        }
        release_tmem();
      } else {
        // bucket-major tile: bucket b0 + j = TMEM columns [j*S, (j+1)*S),
        // column j*S + s = stride-row s, element position s*B + b
        constexpr int kGroups = kEpiWarps / 4;
        float ov[NB / kGroups > 0 ? NB / kGroups : 1][KP];
        uint32_t oi[NB / kGroups > 0 ? NB / kGroups : 1][KP];
        const uint32_t S = a.S, B = a.B;
#pragma unroll
        for (int jj = 0; jj < NB / kGroups; ++jj) {
          const uint32_t j = eg + jj * kGroups;
          const uint32_t b = g * NB + j;
          const uint32_t col = taddr + j * S;
          Summ<KP> s;
          s.clear();
          {  // first 8 stride-rows fill the list (KP <= 8)
            uint32_t r[8];
            __syncwarp();
            ptx::tc::ld32x8(col, r);
            ptx::tc::wait_ld();
#pragma unroll
            for (int e = 0; e < 8; ++e) s.push(__uint_as_float(r[e]), e * B + b, nan);
            if (a.out != nullptr && live)
#pragma unroll
              for (int e = 0; e < 8; ++e) a.out[(uint64_t)row * a.n + (uint64_t)e * B + b] = __uint_as_float(r[e]);
          }
          uint32_t sr = 8;
          for (; sr + 32 <= S; sr += 32) {
            uint32_t r[32];
            __syncwarp();
            ptx::tc::ld32x32(col + sr, r);
            ptx::tc::wait_ld();
            bucket_chunk<KP, 32>(s, r, sr * B + b, B, nan);
            if (a.out != nullptr && live)
#pragma unroll
              for (int e = 0; e < 32; ++e)
                a.out[(uint64_t)row * a.n + (uint64_t)(sr + e) * B + b] = __uint_as_float(r[e]);
          }
          if (sr + 16 <= S) {
            uint32_t r[16];
            __syncwarp();
            ptx::tc::ld32x16(col + sr, r);
            ptx::tc::wait_ld();
            bucket_chunk<KP, 16>(s, r, sr * B + b, B, nan);
            if (a.out != nullptr && live)
#pragma unroll
              for (int e = 0; e < 16; ++e)
                a.out[(uint64_t)row * a.n + (uint64_t)(sr + e) * B + b] = __uint_as_float(r[e]);
            sr += 16;
          }
          if (sr + 8 <= S) {
            uint32_t r[8];
            __syncwarp();
            ptx::tc::ld32x8(col + sr, r);
            ptx::tc::wait_ld();
            bucket_chunk<KP, 8>(s, r, sr * B + b, B, nan);
            if (a.out != nullptr && live)
#pragma unroll
              for (int e = 0; e < 8; ++e)
                a.out[(uint64_t)row * a.n + (uint64_t)(sr + e) * B + b] = __uint_as_float(r[e]);
          }
          s.finalize(ov[jj], oi[jj]);
        }
        release_tmem();  // TMEM free before the HBM writes
        if (live) {
          float* cv = a.cand_v + (uint64_t)row * a.cand_stride + (uint64_t)g * NB * KP;
          uint32_t* ci = a.cand_i + (uint64_t)row * a.cand_stride + (uint64_t)g * NB * KP;
#pragma unroll
          for (int jj = 0; jj < NB / kGroups; ++jj) {
            const uint32_t j = eg + jj * kGroups;
#pragma unroll
            for (int k = 0; k < KP; ++k) { cv[j * KP + k] = ov[jj][k]; ci[j * KP + k] = oi[jj][k]; }
          }
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (nan) atomicOr(a.status, ATKG_FLAG_NAN);
  }
  ptx::tc::fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    ptx::tc::fence_after();
    if constexpr (CG == 2) ptx::tc::dealloc_pair(tmem_base, 512);
    else ptx::tc::dealloc(tmem_base, 512);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

CUtensorMap make_map(const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                     const cuuint32_t* box) {
  CUtensorMap m;
  cuuint32_t elem[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                                 strides_bytes, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

void check_gemm_operands(const void* x, const void* w_t, uint64_t m, uint64_t kdim, uint64_t n) {
  if (x == nullptr || w_t == nullptr) throw_inval("null operand");
  if (m == 0 || n == 0 || kdim == 0) throw_inval("empty GEMM");
  if (kdim % 8 != 0) throw_inval("kdim must be a multiple of 8 (16-byte rows for TMA)");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w_t)) & 15)
    throw_inval("operands must be 16-byte aligned");
  if (m >= (1ull << 31) || n >= (1ull << 31) || kdim >= (1ull << 31)) throw_inval("GEMM dimension too large");
}

// buckets per fused tile: largest NB in {4,2,1} with NB complete buckets in
// one MMA (NB*S <= 256, NB*S % 16 == 0) and S % 8 == 0 (TMEM chunks of 8);
// 0 = not fusable
uint32_t fused_nb(const atkg_params& p) {
  if (p.n % p.num_buckets != 0 || p.n >= (1ull << 31)) return 0;
  const uint64_t S = p.n / p.num_buckets;
  if (S > 256 || S % 8 != 0) return 0;
  if (!(p.local_k == 1 || p.local_k == 2 || p.local_k == 4 || p.local_k == 8)) return 0;
  for (uint32_t nb : {4u, 2u, 1u}) {
    if (p.num_buckets % nb) continue;
    const uint64_t tn = nb * S;
    if (tn <= 256 && tn % 16 == 0) return nb;
  }
  return 0;
}

// CTAs per MMA: a CTA pair (cta_group::2) halves each SM's B traffic; it
// needs the B tile to split into two 8-row-aligned halves (and, for the
// bucket-complete 3-D box, an even number of stride-rows)
uint32_t gemm_cg(uint32_t tn, uint32_t S, uint32_t nb) {
  const uint32_t forced = (uint32_t)opt("gemm_cg", 0);
  const bool pair_ok = (tn / 2) % 8 == 0 && (nb != 1 || S % 16 == 0);
  if (forced == 1 || !pair_ok) return 1;
  return 2;
}

template <int CG, int NB, int KP>
void launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, GemmArgs ga, cudaStream_t st) {
  const size_t smem = gemm_smem_bytes(ga.tn, CG);
  ga.stages = gemm_stages(ga.tn, CG);
  // column tiles per panel: W split into the fewest equal panels of <= 52 MB, inside one L2
  // partition (C4: 2 panels of 16 tiles; measured 359 MB DRAM reads per launch against 426 MB with
  // the row block running fastest over every column tile = option gemm_n_panel 1)
  const uint64_t w_bytes = (uint64_t)ga.tn * ga.kdim * 2 * ga.n_tiles;
  const uint64_t panels = std::max<uint64_t>(1, (w_bytes + (52ull << 20) - 1) / (52ull << 20));
  const uint64_t np = opt("gemm_n_panel", (ga.n_tiles + panels - 1) / panels);
  ga.n_panel = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(1, np), ga.n_tiles);
  ensure_smem_fn(gemm_tc_kernel<CG, NB, KP>, smem);
  const uint32_t tiles = ga.m_blocks * ga.n_tiles;
  const uint32_t units = std::min<uint32_t>(tiles, (uint32_t)sm_count() / CG);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * CG);
  cfg.blockDim = dim3(gemm_threads(NB));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CG;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<CG, NB, KP>, ma, mb, ga));
  check_launch();
}

// A: x [m][kdim] as 2-D {kdim, m}, box {64, 128}
CUtensorMap map_rows(const void* x, uint64_t m, uint64_t kdim) {
  const cuuint64_t d[2] = {kdim, m}, s[1] = {kdim * 2};
  const cuuint32_t b[2] = {kBK, kBM};
  return make_map(x, 2, d, s, b);
}

void run_plain_gemm(const void* x, const void* w_t, uint64_t m, uint64_t kdim, uint64_t n, float* out,
                    cudaStream_t st) {
  const uint32_t cg = gemm_cg(kPlainTN, 0, 0);
  const cuuint64_t db[2] = {kdim, n}, sb[1] = {kdim * 2};
  const cuuint32_t bb[2] = {kBK, kPlainTN / cg};
  const CUtensorMap ma = map_rows(x, m, kdim), mb = make_map(w_t, 2, db, sb, bb);
  GemmArgs ga{};
  ga.m = (uint32_t)m;
  ga.kdim = (uint32_t)kdim;
  ga.n = (uint32_t)n;
  ga.m_blocks = (uint32_t)((m + kBM * cg - 1) / (kBM * cg));
  ga.n_tiles = (uint32_t)((n + kPlainTN - 1) / kPlainTN);
  ga.k_blocks = (uint32_t)((kdim + kBK - 1) / kBK);
  ga.tn = kPlainTN;
  ga.out = out;
  if (cg == 2) launch_gemm<2, 0, 1>(ma, mb, ga, st);
  else launch_gemm<1, 0, 1>(ma, mb, ga, st);
}

// Unfused alternative for shapes the fused epilogue supports (plain GEMM ->
// grid stage 1 -> stage 2, identical results).  Off by default: no shape has
// measured faster this way yet.  Option fused_path=1 selects it (tests).
bool unfused_requested(const atkg_params& p) {
  if (p.local_k > p.n / p.num_buckets) return false;  // grid slots all filled
  return opt("fused_path", 0) == 1;
}

uint64_t fused_cand_bytes(uint64_t m, const atkg_params& p) {
  return align_up(m * p.num_buckets * p.local_k * 4ull);
}

}  // namespace
}  // namespace atkg

using namespace atkg;

extern "C" {

int atkg_fused_workspace_size(uint64_t m, uint64_t kdim, const atkg_params* p, size_t* bytes) {
  return guarded([&] {
    if (p == nullptr || bytes == nullptr) throw_inval("null argument");
    validate(*p);
    if (fused_nb(*p) != 0 && unfused_requested(*p)) {
      const uint64_t count = (uint64_t)p->num_buckets * p->local_k;
      size_t s1 = 0;
      if (atkg_workspace_size(ATKG_OP_STAGE1, ATKG_F32, m, p, &s1) != ATKG_OK) throw Inval(atkg_last_error());
      *bytes = align_up(m * p->n * 4ull) + 2 * fused_cand_bytes(m, *p) + align_up(s1) +
               select_ws_bytes(m, count, p->global_k);
    } else if (fused_nb(*p) != 0) {
      const uint64_t count = (uint64_t)p->num_buckets * p->local_k;
      *bytes = 2 * fused_cand_bytes(m, *p) + select_ws_bytes(m, count, p->global_k);
    } else {  // unfused: scores + the approx_top_k workspace
      size_t inner = 0;
      const int rc = atkg_workspace_size(ATKG_OP_APPROX, ATKG_F32, m, p, &inner);
      if (rc != ATKG_OK) throw Inval(atkg_last_error());
      *bytes = align_up(m * p->n * 4ull) + inner;
    }
  });
}

int atkg_fused_gemm_top_k(const void* d_x, const void* d_w_t, uint64_t m, uint64_t kdim, const atkg_params* p,
                          float* d_out_vals, uint32_t* d_out_idx, float* d_scores, void* d_ws, size_t ws_bytes,
                          uint32_t* d_status, void* stream) {
  return guarded([&] {
    if (p == nullptr) throw_inval("null params");
    validate(*p);
    check_gemm_operands(d_x, d_w_t, m, kdim, p->n);
    size_t need = 0;
    if (atkg_fused_workspace_size(m, kdim, p, &need) != ATKG_OK) throw Inval(atkg_last_error());
    if (ws_bytes < need) throw_inval("workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t nb = fused_nb(*p);
    if (nb == 0) {
      // shapes whose buckets do not fit one MMA tile: plain GEMM, then the
      // streaming approx_top_k on the fp32 scores
      float* scores = d_scores ? d_scores : static_cast<float*>(d_ws);
      uint8_t* inner = static_cast<uint8_t*>(d_ws) + align_up(m * p->n * 4ull);
      run_plain_gemm(d_x, d_w_t, m, kdim, p->n, scores, st);
      const int rc = atkg_approx_top_k(ATKG_F32, scores, m, p, d_out_vals, d_out_idx, inner,
                                       need - align_up(m * p->n * 4ull), d_status, stream);
      if (rc != ATKG_OK) throw Inval(atkg_last_error());
      return;
    }
    if (unfused_requested(*p)) {
      // write the fp32 scores, then the grid stage 1 + stage 2 (identical results)
      uint8_t* w = static_cast<uint8_t*>(d_ws);
      float* scores = d_scores ? d_scores : reinterpret_cast<float*>(w);
      w += align_up(m * p->n * 4ull);
      float* gv = reinterpret_cast<float*>(w);
      uint32_t* gi = reinterpret_cast<uint32_t*>(w + fused_cand_bytes(m, *p));
      w += 2 * fused_cand_bytes(m, *p);
      size_t s1 = 0;
      if (atkg_workspace_size(ATKG_OP_STAGE1, ATKG_F32, m, p, &s1) != ATKG_OK) throw Inval(atkg_last_error());
      run_plain_gemm(d_x, d_w_t, m, kdim, p->n, scores, st);
      const int rc = atkg_stage1(ATKG_F32, scores, m, p, gv, gi, w, s1, d_status, stream);
      if (rc != ATKG_OK) throw Inval(atkg_last_error());
      w += align_up(s1);
      const uint64_t count = (uint64_t)p->num_buckets * p->local_k;
      run_select(gv, gi, m, count, count, p->global_k, UINT64_MAX, d_out_vals, d_out_idx, w, d_status, st);
      return;
    }
    const uint64_t B = p->num_buckets, S = p->n / B;
    const uint32_t tn = (uint32_t)(nb * S), cg = gemm_cg(tn, (uint32_t)S, nb);
    // W^T as [S][B][Kd]; one box = one bucket (or half of it when a CTA
    // pair splits a single-bucket tile)
    const cuuint64_t db[3] = {kdim, B, S}, sb[2] = {kdim * 2, B * kdim * 2};
    const cuuint32_t bb[3] = {kBK, 1, (cuuint32_t)(nb == 1 ? S / cg : S)};
    const CUtensorMap ma = map_rows(d_x, m, kdim), mb = make_map(d_w_t, 3, db, sb, bb);
    GemmArgs ga{};
    ga.m = (uint32_t)m;
    ga.kdim = (uint32_t)kdim;
    ga.n = (uint32_t)p->n;
    ga.m_blocks = (uint32_t)((m + kBM * cg - 1) / (kBM * cg));
    ga.n_tiles = (uint32_t)(B / nb);
    ga.k_blocks = (uint32_t)((kdim + kBK - 1) / kBK);
    ga.tn = tn;
    ga.S = (uint32_t)S;
    ga.B = (uint32_t)B;
    ga.cand_stride = (uint32_t)(B * p->local_k);
    ga.out = d_scores;
    uint8_t* w = static_cast<uint8_t*>(d_ws);
    ga.cand_v = reinterpret_cast<float*>(w);
    ga.cand_i = reinterpret_cast<uint32_t*>(w + fused_cand_bytes(m, *p));
    ga.status = d_status;
    void* sel_ws = w + 2 * fused_cand_bytes(m, *p);
    g_prof.bracket_begin(st);
#define ATKG_FUSED_CASE(NBV, KPV)                               \
  if (nb == NBV && p->local_k == KPV) {                         \
    if (cg == 2) launch_gemm<2, NBV, KPV>(ma, mb, ga, st);      \
    else launch_gemm<1, NBV, KPV>(ma, mb, ga, st);              \
  }
    ATKG_FUSED_CASE(1, 1) ATKG_FUSED_CASE(1, 2) ATKG_FUSED_CASE(1, 4) ATKG_FUSED_CASE(1, 8)
    ATKG_FUSED_CASE(2, 1) ATKG_FUSED_CASE(2, 2) ATKG_FUSED_CASE(2, 4) ATKG_FUSED_CASE(2, 8)
    ATKG_FUSED_CASE(4, 1) ATKG_FUSED_CASE(4, 2) ATKG_FUSED_CASE(4, 4) ATKG_FUSED_CASE(4, 8)
#undef ATKG_FUSED_CASE
    g_prof.bracket_end(st);
    run_select(ga.cand_v, ga.cand_i, m, B * p->local_k, B * p->local_k, p->global_k, UINT64_MAX, d_out_vals,
               d_out_idx, sel_ws, d_status, st);
  });
}

int atkg_gemm_bf16(const void* d_x, const void* d_w_t, uint64_t m, uint64_t kdim, uint64_t n, float* d_out,
                   void* stream) {
  return guarded([&] {
    check_gemm_operands(d_x, d_w_t, m, kdim, n);
    if (d_out == nullptr) throw_inval("null output");
    run_plain_gemm(d_x, d_w_t, m, kdim, n, d_out, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
