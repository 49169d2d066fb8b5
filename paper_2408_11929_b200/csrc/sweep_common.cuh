// sweep_common.cuh -- arguments and device helpers shared by the two sweep
// kernels (sweep_apply.cu: general TMA-ring kernel; sweep_fast.cu: register-
// streaming kernel for block rows of <= 36 nodes).
#pragma once
#include "common.cuh"

#define HELM_MAXDIR 8

struct DirArgs {
  int axis, order, N, P, nc, nxp1, is_double, ntile_max;
  int disc;              // HELM_DISC_P1 / HELM_DISC_FD5 (RHS row scaling of the FD5 strip systems)
  const int *a, *w, *own_lo, *own_hi, *seg_lo, *seg_hi;
  const cplx *cr, *ne;   // bands: U_c couplings, stride wmax per row, nc*wmax per strip
  const cplx* tc;        // transmission stencils [s][side][c][5]
  const cplx* fac;
  const cplx* facp;      // two-chain kernel: packed top-down inverses, NULL if absent
  const cplx* fac2;      // two-chain kernel: packed bottom-up inverses, NULL if absent
  const long* pfac_off;  // per-strip offsets of the packed arrays
  const long* fac_off;
  const cplx* red;
  const long* red_off;
  const cplx* R;         // source column
  cplx* Z;               // output column
  cplx *yb, *xs, *xb, *corr_prev, *corr_next;
  unsigned* cnt;         // [0] segment arrivals, [1] reducer releases
  unsigned* flag;        // fast kernel: per-separator publication flags (solve index + 1)
  const cplx* xinv;      // explicit separator-inverse rows (fast kernel), NULL if absent
  const float2* xinv32;  // their complex64 copy (inexact separator solve, two-chain kernel), NULL if off
  const long* xinv_off;
  const cplx* sep2;      // two-chain kernel: two-level separator panels (strip_setup.cu), NULL = full R^{-1} rows
  const long* sep2_off;
  const int* sep2_plan;
  int sep2_M, sep2_ld1, sep2_ld2;
  cplx* gh;              // two-level: the coarse right-hand sides [2][M][wmax]
  int wmax;
  int cta_base;
  int vec_rows;
};

struct ApplyArgs {
  DirArgs d[HELM_MAXDIR];
  int t;
  int rows_per_tile;  // R_t = consumer threads / 8
  int nstage;
  int stage_elems;    // cplx per stage
  int vec_elems;      // cplx per vector area (bseg / yseg / staged couplings)
  int pmax;           // max segments over directions
  int nsolve_max;     // max local solves per apply over directions
  int vec_global;     // vector areas in global scratch (shared memory too small)
  cplx* vec_scratch;  // per-CTA 4 * vec_elems when vec_global
  long long* prof;    // optional per-CTA cycle counters (8 per CTA), NULL = off
};

// per-thread profiling accumulators (thread 0 reports)
struct Prof {
  long long peek = 0, comp = 0, bar = 0, steps = 0, xwait = 0, xmv = 0;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// relaxed poll (no L1 invalidation per iteration); callers fence once after success
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ cplx ldcg(const cplx* p) { return __ldcg(p); }
// TMA bulk copy global -> shared with an L2 cache-policy hint
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// 16-byte asynchronous global -> shared copies (LDGSTS); zfill: src-size 0 writes zeros
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool zfill = false) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
               "r"(zfill ? 0 : 16)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// 16-byte shared-memory load by byte address
__device__ __forceinline__ cplx lds128(uint32_t addr) {
  cplx v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}


// ------------------------------------------------------------------ geometry helpers
__device__ __forceinline__ int sigma(const DirArgs& D, int m) { return D.order == 0 ? m : D.N - 1 - m; }
__device__ __forceinline__ int n_solves(const DirArgs& D) { return D.is_double ? 2 * D.N - 1 : D.N; }
// sweep step m and pass of solve i
__device__ __forceinline__ int step_of(const DirArgs& D, int i) { return i < D.N ? i : 2 * D.N - 2 - i; }
__device__ __forceinline__ bool is_bwd(const DirArgs& D, int i) { return i >= D.N; }
__device__ __forceinline__ bool writes_Z(const DirArgs& D, int i) { return D.is_double ? (i >= D.N - 1) : true; }
__device__ __forceinline__ long node_of(const DirArgs& D, int a, int c, int q) {
  return D.axis == 0 ? (long)c * D.nxp1 + (a + q) : (long)(a + q) * D.nxp1 + c;
}
// interface positions inside strip s: prev side / next side (0 = low line a_s, w-1 = high line b_s)
__device__ __forceinline__ int prev_side(const DirArgs& D) { return D.order == 0 ? 0 : 1; }
__device__ __forceinline__ int next_side(const DirArgs& D) { return D.order == 0 ? 1 : 0; }

// Correction (D8) for destination strip t, side, row c, from a source solution
// x_s accessed by a functor X(c', q).  Positions of the interface line and the
// outer line in the source strip (a_src).
// Variant with the destination strip's first line `at` and width `wt` passed in
// (no dependent loads of the strip geometry in front of the stencil loads).
template <class XF>
__device__ __forceinline__ cplx correction_aw(const DirArgs& D, int t, int at, int wt, int side, int c, int a_src,
                                              XF X) {
  const cplx* k = D.tc + (((long)t * 2 + side) * D.nc + c) * kTcW;
  const int bt = at + wt - 1;
  int qi, qo, qn, dd;
  if (side == 0) { qi = at - a_src; qo = at - 1 - a_src; qn = at + 1 - a_src; dd = -1; }
  else { qi = bt - a_src; qo = bt + 1 - a_src; qn = bt - 1 - a_src; dd = 1; }
  const cplx k0 = c >= 1 ? __ldg(k + 0) : cmk(0, 0);
  const cplx k1 = __ldg(k + 1);
  const cplx k2 = c + 1 < D.nc ? __ldg(k + 2) : cmk(0, 0);
  const cplx k3 = __ldg(k + 3);
  const bool h4 = c + dd >= 0 && c + dd < D.nc;
  const cplx k4 = h4 ? __ldg(k + 4) : cmk(0, 0);
  const cplx x1 = X(c, qi), x3 = X(c, qo);
  const cplx x0 = c >= 1 ? X(c - 1, qi) : cmk(0, 0);
  const cplx x2 = c + 1 < D.nc ? X(c + 1, qi) : cmk(0, 0);
  const cplx x4 = h4 ? X(c + dd, qo) : cmk(0, 0);
  cplx acc = cmul(k1, x1);
  cfma(acc, k3, x3);
  cfma(acc, k0, x0);
  cfma(acc, k2, x2);
  cfma(acc, k4, x4);
  if (D.disc == HELM_DISC_FD5) cfma(acc, __ldg(k + 5), X(c, qn));   // inner line (centred normal derivative)
  return acc;
}

template <class XF>
__device__ __forceinline__ cplx correction(const DirArgs& D, int t, int side, int c, int a_src, XF X) {
  const cplx* k = D.tc + (((long)t * 2 + side) * D.nc + c) * kTcW;
  int at = D.a[t], bt = at + D.w[t] - 1;
  int qi, qo, qn, dd;
  if (side == 0) { qi = at - a_src; qo = at - 1 - a_src; qn = at + 1 - a_src; dd = -1; }
  else { qi = bt - a_src; qo = bt + 1 - a_src; qn = bt - 1 - a_src; dd = 1; }
  cplx acc = cmul(__ldg(k + 1), X(c, qi));
  cfma(acc, __ldg(k + 3), X(c, qo));
  if (c >= 1) cfma(acc, __ldg(k + 0), X(c - 1, qi));
  if (c + 1 < D.nc) cfma(acc, __ldg(k + 2), X(c + 1, qi));
  if (c + dd >= 0 && c + dd < D.nc) cfma(acc, __ldg(k + 4), X(c + dd, qo));
  if (D.disc == HELM_DISC_FD5) cfma(acc, __ldg(k + 5), X(c, qn));
  return acc;
}

// RHS row scaling of the strip system actually factored: 1 for P1; for FD5 the
// strip matrix is S_s = D_s A_s (complex symmetric), so A_s v = f is solved as
// S_s v = D_s f (common.cuh fd5_d; the source and the corrections both scale)
__device__ __forceinline__ double rhs_scale(const DirArgs& D, int c, int q, int w) {
  return D.disc == HELM_DISC_FD5 ? fd5_d(q, w, c, D.nc) : 1.0;
}

