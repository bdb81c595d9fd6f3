// summ.cuh -- the per-bucket stage-1 summary (Summ<KP>), shared by the
// streaming kernels (stage1.cuh, rowres.cuh) and the GEMM epilogue
// (fused_gemm.cu).  Semantics: see the comment block at the top of
// stage1.cuh (reference Alg. 1, /root/reference/proj/core/src/topk.cpp:80-102).
#pragma once

#include "common.cuh"

namespace atkg {

// ---------------------------------------------------------------------------
// per-bucket summary, fully register resident (all indices compile-time)
// ---------------------------------------------------------------------------
template <int KP>
struct Summ {
  float v[KP];
  uint32_t p[KP];
  uint32_t lt;   // valid when full
  float ltv;

  ATKG_HD void clear() {
#pragma unroll
    for (int k = 0; k < KP; ++k) { v[k] = neg_inf(); p[k] = kEmptyPos; }
    lt = kEmptyPos;
    ltv = neg_inf();
  }
  ATKG_HD bool full() const { return p[KP - 1] != kEmptyPos; }

  // prologue insert of the t-th element of a segment (t < KP; the caller's
  // loop over t is unrolled so every index below is compile-time)
  ATKG_HD void fill(int t, float x, uint32_t i) {
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (k == t) { v[k] = x; p[k] = i; }
#pragma unroll
    for (int k = KP - 1; k >= 1; --k) {
      if (k <= t && x > v[k - 1]) {
        const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
        const uint32_t tp = p[k]; p[k] = p[k - 1]; p[k - 1] = tp;
      }
    }
    if (t == KP - 1) { lt = p[KP - 1]; ltv = v[KP - 1]; }
  }

  // main-loop update of a FULL list with x at position i (> every position
  // seen).  Caller has established !(x < v[KP-1]) (NaN included).
  ATKG_HD void slow(float x, uint32_t i, uint32_t& nan) {
    if (x != x) { nan = 1u; return; }
    const float old = v[KP - 1];
    if (x == old) { lt = i; ltv = x; return; }
    v[KP - 1] = x;
    p[KP - 1] = i;
#pragma unroll
    for (int k = KP - 1; k >= 1; --k) {
      if (x > v[k - 1]) {
        const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
        const uint32_t tp = p[k]; p[k] = p[k - 1]; p[k - 1] = tp;
      }
    }
    if (v[KP - 1] != old) { lt = p[KP - 1]; ltv = v[KP - 1]; }
  }

  // streaming update with one element at position i (> every position seen);
  // works on partially filled lists (the accumulator's ragged edges)
  ATKG_HD void push(float x, uint32_t i, uint32_t& nan) {
    if (x != x) { nan = 1u; return; }
    if (full()) {
      if (!(x < v[KP - 1])) slow(x, i, nan);
      return;
    }
    int c = 0;
#pragma unroll
    for (int k = 0; k < KP; ++k) c += (p[k] != kEmptyPos) ? 1 : 0;
    fill(c, x, i);
  }

  // max position among entries equal to `val` (entries sorted so the last
  // equal one has the max position); kEmptyPos if none
  ATKG_HD void last_eq(float val, uint32_t& pos, float& bits) const {
    pos = kEmptyPos;
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (p[k] != kEmptyPos && v[k] == val) { pos = p[k]; bits = v[k]; }
  }

  // this = merge(this [earlier positions], o [later positions])
  ATKG_HD void merge_later(const Summ& o) {
    const bool a_full = full();
    const float a_min = v[KP - 1];
    const uint32_t a_lt = lt;
    const float a_ltv = ltv;
    Summ a = *this;  // pre-merge copy for the tie bookkeeping
    // insert o's entries (rank-sorted) one by one; rank: value desc, pos asc,
    // empty last.  o's positions all exceed ours.
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const float x = o.v[j];
      const uint32_t xp = o.p[j];
      if (xp == kEmptyPos) continue;
      // x enters iff it ranks before the current last slot
      const bool enter = (p[KP - 1] == kEmptyPos) || (x > v[KP - 1]);
      if (!enter) continue;
      v[KP - 1] = x;
      p[KP - 1] = xp;
#pragma unroll
      for (int k = KP - 1; k >= 1; --k) {
        const bool up = (p[k - 1] == kEmptyPos) || (x > v[k - 1]);
        if (up) {
          const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
          const uint32_t tp = p[k]; p[k] = p[k - 1]; p[k - 1] = tp;
        }
      }
    }
    if (!full()) { lt = kEmptyPos; ltv = neg_inf(); return; }
    const float c_min = v[KP - 1];
    uint32_t pos; float bits;
    // later segment first: any equal element there is after all of ours
    if (o.full() && o.v[KP - 1] == c_min) { pos = o.lt; bits = o.ltv; }
    else o.last_eq(c_min, pos, bits);
    if (pos == kEmptyPos) {
      if (a_full && a_min == c_min) { pos = a_lt; bits = a_ltv; }
      else a.last_eq(c_min, pos, bits);
    }
    lt = pos;
    ltv = bits;
  }

  // whole-bucket summary -> reference Alg. 1 state (value bits, index)
  ATKG_HD void finalize(float (&ov)[KP], uint32_t (&oi)[KP]) const {
    const bool f = full();
    const float vmin = v[KP - 1];
    if (f && vmin != neg_inf()) {
      uint32_t L = kEmptyPos;  // max position of entries > v*
      bool anybig = false;
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        ov[k] = v[k];
        oi[k] = p[k];
        if (v[k] > vmin) { L = anybig ? umax32(L, p[k]) : p[k]; anybig = true; }
      }
      if (!anybig || lt > L) { ov[KP - 1] = ltv; oi[KP - 1] = lt; }
      return;
    }
    // v* == -inf: the reference's K' sentinels {-inf, 0} are tie elements
    // that precede the stream
    uint32_t L = 0;
    bool anybig = false;
    uint32_t T = kEmptyPos;  // last real element equal to -inf
    if (f) T = lt;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (p[k] != kEmptyPos && v[k] > neg_inf()) {
        L = anybig ? umax32(L, p[k]) : p[k];
        anybig = true;
      } else if (!f && p[k] != kEmptyPos) {
        T = p[k];
      }
    }
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const bool big = p[k] != kEmptyPos && v[k] > neg_inf();
      ov[k] = big ? v[k] : neg_inf();
      oi[k] = big ? p[k] : 0u;
    }
    if (T != kEmptyPos && (!anybig || T > L)) { ov[KP - 1] = neg_inf(); oi[KP - 1] = T; }
  }
};

}  // namespace atkg
