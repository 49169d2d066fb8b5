// row_gj.cuh -- the register-row Gauss-Jordan inversion of a w x w (w <= 36)
// complex block used by the strip factorisation (strip_setup.cu: k_factor_rows,
// k_reduced, the two-level separator setup) and by tools/bench_gj.cu.
#pragma once
#include "common.cuh"

// e / w for 0 <= e < w^2 <= 36^2 without an integer division: (e + 1/2) / w in
// single precision stays at least 1/(2w) away from the next integer
__device__ __forceinline__ int div_w(int e, float invw) { return (int)(((float)e + 0.5f) * invw); }

#ifndef HELM_ROW_LPR
#define HELM_ROW_LPR 2      // threads per block row in the register-row Gauss-Jordan (2 or 4)
#endif
static constexpr int kRowW = 36;
static constexpr int kLPR = HELM_ROW_LPR;                 // lanes per row: column j = kLPR jj + h
static constexpr int kRowHW = kRowW / kLPR;               // columns (registers) per thread
static constexpr int kRowThreads = kLPR == 2 ? 96 : 160;  // >= kRowW kLPR threads, whole warps
static constexpr int kRowWarps = kRowThreads / 32;
static_assert(kRowW % kLPR == 0 && kRowW * kLPR <= kRowThreads, "row layout");

struct RowSmem {
  cplx mat[kRowW * kRowW];    // natural-order inverse of the current block / Y
  cplx tmat[kRowW * kRowW];   // U_c Y (kind 0, X[lo,hi] chain)
  cplx prow[2 * kRowW];       // row_invert_r: index 2 (slot + rot) + h, rot < kRowHW
  cplx pcol[2][kRowW];        // row_invert_g: pivot-column entries (multipliers), by step parity
  cplx pdinv;                 // row_invert_g: 1 / pivot
  unsigned redk[12];
  int redi[12];
  int pivrow[kRowW];
  long long gjp[4];           // HELM_GJ_PROF: thread 0's per-phase pivot-loop cycles
};

// a[kj] for a runtime index kj < N by a select tree on the bits of kj
template <int N>
__device__ __forceinline__ cplx sel_idx(const cplx (&a)[N], int kj) {
  cplx t[N];
#pragma unroll
  for (int u = 0; u < N; ++u) t[u] = a[u];
#pragma unroll
  for (int st = 1; st < N; st <<= 1) {
    const bool bit = kj & st;
#pragma unroll
    for (int u = 0; u + st < N; u += 2 * st) t[u] = bit ? t[u + st] : t[u];
  }
  return t[0];
}

// Gauss-Jordan inversion of the w x w block held LPR threads per row (thread
// (i, h) holds columns LPR jj + h), the same pivot rule and elementary operations
// as row_invert; the pivot row is broadcast raw with 1/pivot (the scaling of the
// pivot row itself and of the multipliers happens after the broadcast barrier,
// off its critical path), the multipliers through shared memory (rows may straddle
// warps).  Used by k_reduced with more threads per row (shorter pivot steps).
template <int LPR>
__device__ __forceinline__ int row_invert_g(cplx (&a)[kRowW / LPR], int w, RowSmem& sm) {
  constexpr int HW = kRowW / LPR;
  constexpr int NWR = (kRowW * LPR + 31) / 32;   // warps holding rows
  static_assert(kRowW % LPR == 0 && NWR <= 12, "row_invert_g layout");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = tid / LPR, h = tid % LPR;
  const bool active = i < w;
  bool used = false;
  int kstep = 0;
#ifdef HELM_GJ_PROF
  long long gp_s = 0, gp_p = 0, gp_u = 0;
#endif
#pragma unroll 1
  for (int k = 0; k < w; ++k) {
    const int kh = k % LPR, kj = k / LPR, par = k & 1;
#ifdef HELM_GJ_PROF
    const long long q0 = clock64();
#endif
    const cplx mine = sel_idx(a, kj);
    const bool cand = active && !used && h == kh;
    const unsigned key = cand ? (unsigned)__double2hiint(cabs2(mine)) + 1u : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    const unsigned who = __ballot_sync(0xffffffffu, key == kmax);
    if (lane == 0 && warp < NWR) { sm.redk[warp] = kmax; sm.redi[warp] = (warp * 32 + __ffs(who) - 1) / LPR; }
    if (active && h == kh) sm.pcol[par][i] = mine;
    __syncthreads();
#ifdef HELM_GJ_PROF
    const long long q1 = clock64();
    gp_s += q1 - q0;
#endif
    unsigned k0 = sm.redk[0];
    int p = sm.redi[0];
#pragma unroll
    for (int q = 1; q < NWR; ++q)
      if (sm.redk[q] > k0) { k0 = sm.redk[q]; p = sm.redi[q]; }
    if (k0 <= 1u || k0 > 0x7FF00000u) return 1;   // all candidates zero (key 1 = +0.0), or a NaN / Inf entry (exponent all ones)
    if (i == p) {
#pragma unroll
      for (int jj = 0; jj < HW; ++jj) sm.prow[LPR * jj + h] = a[jj];
      if (h == kh) {
        // the pivot column is broadcast as pivot + 1: a_ik - (a_ik / piv)(piv + 1) = -a_ik / piv
        sm.prow[k] = cmk(mine.x + 1.0, mine.y);
#ifdef HELM_GJ_DRCP
        { const double dd = __drcp_rn(cabs2(mine)); sm.pdinv = cmk(mine.x * dd, -mine.y * dd); }
#else
        sm.pdinv = cinv(mine);
#endif
      }
    }
    __syncthreads();
#ifdef HELM_GJ_PROF
    const long long q2 = clock64();
    gp_p += q2 - q1;
#endif
    const cplx dinv = sm.pdinv;
    if (i == p) {
#pragma unroll
      for (int jj = 0; jj < HW; ++jj) a[jj] = (h == kh && jj == kj) ? dinv : cmul(a[jj], dinv);
      used = true;
      kstep = k;
      if (h == 0) sm.pivrow[k] = p;
    } else if (active) {
      const cplx f = cmul(sm.pcol[par][i], dinv);
#pragma unroll
      for (int jj = 0; jj < HW; ++jj) {
        const cplx r = sm.prow[LPR * jj + h];
        a[jj].x = fma(-f.x, r.x, a[jj].x);
        a[jj].x = fma(f.y, r.y, a[jj].x);
        a[jj].y = fma(-f.x, r.y, a[jj].y);
        a[jj].y = fma(-f.y, r.x, a[jj].y);
      }
    }
#ifdef HELM_GJ_PROF
    gp_u += clock64() - q2;
#endif
  }
#ifdef HELM_GJ_PROF
  if (tid == 0) { sm.gjp[0] += gp_s; sm.gjp[1] += gp_p; sm.gjp[2] += gp_u; }
#endif
  __syncthreads();   // pivrow complete; everyone is done reading mat from the previous block
  if (active) {
#pragma unroll
    for (int jj = 0; jj < HW; ++jj) {
      const int j = LPR * jj + h;
      if (j < w) sm.mat[kstep * kRowW + sm.pivrow[j]] = a[jj];
    }
  }
  __syncthreads();
  return 0;
}

// Invert the w x w block held as described above; leaves the inverse in
// sm.mat (natural order, row stride kRowW).  Returns 1 (uniformly) on a zero pivot.
__device__ __forceinline__ int row_invert(cplx (&a)[kRowHW], int w, RowSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = tid / kLPR, h = tid % kLPR;
  const bool active = i < w;
  bool used = false;
  int kstep = 0;
  // the pivot loop is NOT unrolled (a fully unrolled loop thrashed the instruction
  // cache, ncu no_inst ~27%); the pivot-column entry a[k >> 1] is extracted and
  // written back with unrolled selects
#pragma unroll 1
  for (int k = 0; k < w; ++k) {
    const int kh = k % kLPR, kj = k / kLPR;
    // a[kj] by a select tree on the bits of kj (depth log2, not a chain)
    cplx mine;
    {
      cplx t1[(kRowHW + 1) / 2];
#pragma unroll
      for (int u = 0; u < kRowHW / 2; ++u) t1[u] = (kj & 1) ? a[2 * u + 1] : a[2 * u];
      if (kRowHW & 1) t1[kRowHW / 2] = a[kRowHW - 1];
      constexpr int n1 = (kRowHW + 1) / 2;
      cplx t2[(n1 + 1) / 2];
#pragma unroll
      for (int u = 0; u < n1 / 2; ++u) t2[u] = (kj & 2) ? t1[2 * u + 1] : t1[2 * u];
      if (n1 & 1) t2[n1 / 2] = t1[n1 - 1];
      constexpr int n2 = (n1 + 1) / 2;
      cplx t3[(n2 + 1) / 2];
#pragma unroll
      for (int u = 0; u < n2 / 2; ++u) t3[u] = (kj & 4) ? t2[2 * u + 1] : t2[2 * u];
      if (n2 & 1) t3[n2 / 2] = t2[n2 - 1];
      constexpr int n3 = (n2 + 1) / 2;
      if constexpr (n3 == 1) {
        mine = t3[0];
      } else {
        cplx t4[(n3 + 1) / 2];
#pragma unroll
        for (int u = 0; u < n3 / 2; ++u) t4[u] = (kj & 8) ? t3[2 * u + 1] : t3[2 * u];
        if (n3 & 1) t4[n3 / 2] = t3[n3 - 1];
        constexpr int n4 = (n3 + 1) / 2;
        static_assert(n4 <= 2, "select tree depth");
        if constexpr (n4 == 2) mine = (kj & 16) ? t4[1] : t4[0];
        else mine = t4[0];
      }
    }
    // pivot search: the largest |a_ik|^2 among unused rows, compared on the high
    // 32 bits of the (non-negative) double -- monotonic; candidates equal to ~1e-6
    // relative go to the lowest row -- with one warp max-reduction and a ballot
#ifdef HELM_GJ_NOPIVOT
    // ablation (timing only): diagonal pivots, no search
    const int p = k;
    (void)lane; (void)warp;
#else
    const double mag = (active && !used && h == kh) ? cabs2(mine) : 0.0;
    const unsigned key = (active && !used && h == kh) ? (unsigned)__double2hiint(mag) + 1u : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    const unsigned who = __ballot_sync(0xffffffffu, key == kmax);
    if (lane == 0 && warp < kRowWarps) { sm.redk[warp] = kmax; sm.redi[warp] = warp * (32 / kLPR) + (__ffs(who) - 1) / kLPR; }
    __syncthreads();
    unsigned k0 = sm.redk[0];
    int p = sm.redi[0];
#pragma unroll
    for (int q = 1; q < kRowWarps; ++q)
      if (sm.redk[q] > k0) { k0 = sm.redk[q]; p = sm.redi[q]; }
    if (k0 <= 1u || k0 > 0x7FF00000u) return 1;   // all candidates zero (key 1 = +0.0), or a NaN / Inf entry (exponent all ones)
#endif
    // pivot element to every lane of the pivot row; multiplier to every lane of the others
    cplx akk;
    {
      const int src = (lane & ~(kLPR - 1)) | kh;
      akk.x = __shfl_sync(0xffffffffu, mine.x, src);
      akk.y = __shfl_sync(0xffffffffu, mine.y, src);
    }
    if (i == p) {
      const cplx dinv = cinv(akk);
#pragma unroll
      for (int jj = 0; jj < kRowHW; ++jj) {
        const cplx v = (h == kh && jj == kj) ? cmk(1.0, 0.0) : a[jj];
        a[jj] = cmul(v, dinv);
        sm.prow[kLPR * jj + h] = a[jj];
      }
      // the pivot column is broadcast as 1 + 1/piv, so the generic update of the
      // other rows, a_ik - f (1 + 1/piv) with f = a_ik, leaves -f/piv there
      if (h == kh) sm.prow[k] = cmk(1.0 + dinv.x, dinv.y);
      used = true;
      kstep = k;
      if (h == 0) sm.pivrow[k] = p;
    }
    __syncthreads();
    if (active && i != p) {
      const cplx f = akk;
#pragma unroll
      for (int jj = 0; jj < kRowHW; ++jj) {   // a -= f r, four fused multiply-adds
        const cplx r = sm.prow[kLPR * jj + h];
        a[jj].x = fma(-f.x, r.x, a[jj].x);
        a[jj].x = fma(f.y, r.y, a[jj].x);
        a[jj].y = fma(-f.x, r.y, a[jj].y);
        a[jj].y = fma(-f.y, r.x, a[jj].y);
      }
    }
  }
  __syncthreads();   // pivrow complete; everyone is done reading mat from the previous block
  if (active) {
#pragma unroll
    for (int jj = 0; jj < kRowHW; ++jj) {
      const int j = kLPR * jj + h;
      if (j < w) sm.mat[kstep * kRowW + sm.pivrow[j]] = a[jj];
    }
  }
  __syncthreads();
  return 0;
}

// row_invert with rotating register slots (no register selects): during the
// pass of pivot pairs m0 .. m0 + UP - 1, slot jj holds column LPR ((jj + m0) mod
// HW) + h, so the pivot column of pivot k = LPR (m0 + u) + kh is the
// compile-time slot u; after each pass the slots rotate by UP (HW / UP passes
// restore the natural order).  The pivot row is published at index
// LPR (jj + m0) + h of the doubled sm.prow (no wrap-around arithmetic).  Same
// pivot rule and elementary operations as row_invert: bitwise the same inverse.
#ifndef HELM_ROW_UP
#define HELM_ROW_UP 3
#endif
template <int UP>
__device__ __forceinline__ int row_invert_r(cplx (&a)[kRowHW], int w, RowSmem& sm) {
  static_assert(kRowHW % UP == 0, "the slots rotate by UP");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = tid / kLPR, h = tid % kLPR;
  const bool active = i < w;
  bool used = false;
  int kstep = 0;
#pragma unroll 1
  for (int m0 = 0; m0 < kRowHW; m0 += UP) {
#pragma unroll
    for (int u = 0; u < UP; ++u) {
#pragma unroll
      for (int kh = 0; kh < kLPR; ++kh) {
        const int k = kLPR * (m0 + u) + kh;
        if (k < w) {
          const cplx mine = a[u];
          const double mag = (active && !used && h == kh) ? cabs2(mine) : 0.0;
          const unsigned key = (active && !used && h == kh) ? (unsigned)__double2hiint(mag) + 1u : 0u;
          const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
          const unsigned who = __ballot_sync(0xffffffffu, key == kmax);
          if (lane == 0 && warp < kRowWarps) { sm.redk[warp] = kmax; sm.redi[warp] = warp * (32 / kLPR) + (__ffs(who) - 1) / kLPR; }
          __syncthreads();
          unsigned k0 = sm.redk[0];
          int p = sm.redi[0];
#pragma unroll
          for (int q = 1; q < kRowWarps; ++q)
            if (sm.redk[q] > k0) { k0 = sm.redk[q]; p = sm.redi[q]; }
          if (k0 <= 1u || k0 > 0x7FF00000u) return 1;   // all candidates zero (key 1 = +0.0), or a NaN / Inf entry (exponent all ones)
          cplx akk;
          {
            const int src = (lane & ~(kLPR - 1)) | kh;
            akk.x = __shfl_sync(0xffffffffu, mine.x, src);
            akk.y = __shfl_sync(0xffffffffu, mine.y, src);
          }
          cplx* prow = sm.prow + kLPR * m0 + h;
          if (i == p) {
            const cplx dinv = cinv(akk);
#pragma unroll
            for (int jj = 0; jj < kRowHW; ++jj) {
              const cplx v = (jj == u && h == kh) ? cmk(1.0, 0.0) : a[jj];
              a[jj] = cmul(v, dinv);
              prow[kLPR * jj] = a[jj];
            }
            if (h == kh) prow[kLPR * u] = cmk(1.0 + dinv.x, dinv.y);
            used = true;
            kstep = k;
            if (h == 0) sm.pivrow[k] = p;
          }
          __syncthreads();
          if (active && i != p) {
            const cplx f = akk;
#pragma unroll
            for (int jj = 0; jj < kRowHW; ++jj) {   // a -= f r, four fused multiply-adds
              const cplx r = prow[kLPR * jj];
              a[jj].x = fma(-f.x, r.x, a[jj].x);
              a[jj].x = fma(f.y, r.y, a[jj].x);
              a[jj].y = fma(-f.x, r.y, a[jj].y);
              a[jj].y = fma(-f.y, r.x, a[jj].y);
            }
          }
        }
      }
    }
    cplx t[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) t[u] = a[u];
#pragma unroll
    for (int jj = 0; jj + UP < kRowHW; ++jj) a[jj] = a[jj + UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) a[kRowHW - UP + u] = t[u];
  }
  __syncthreads();   // pivrow complete; everyone is done reading mat from the previous block
  if (active) {
#pragma unroll
    for (int jj = 0; jj < kRowHW; ++jj) {
      const int j = kLPR * jj + h;
      if (j < w) sm.mat[kstep * kRowW + sm.pivrow[j]] = a[jj];
    }
  }
  __syncthreads();
  return 0;
}
