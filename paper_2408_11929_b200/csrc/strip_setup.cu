// strip_setup.cu -- sweep_setup (hot-path row a2): strip geometry (D6), local
// block-tridiagonal matrices (D7), transmission-correction stencils (D8), and
// the factorisation of every strip, "factored once" (P:L152 uses `\`; the
// north star asks for a banded / block-tridiagonal LU).
//
// Strip s, generic coordinates: block row c = cross index (n_c rows), position
// q = 0..w_s-1 along the axis (line a_s + q).  A_s is block tridiagonal:
//   D_c = tridiag(al[c][q-1], dg[c][q], al[c][q]),  U_c = bidiag(cr[c][q], ne[c][q]),
//   L_{c+1} = U_c^T  (A_s complex symmetric).
// Partitioned factorisation: the n_c rows are split into P
// segments separated by P-1 single separator rows.  Each segment is factored
// by block-Thomas with explicit inverses  S_lo = D_lo,
//   S_c = D_c - U_{c-1}^T S_{c-1}^{-1} U_{c-1},  Sinv_c = S_c^{-1}
// (unpivoted between blocks, Gauss-Jordan with partial pivoting inside a
// block; stable here).  The separator Schur complement
// (block tridiagonal with dense couplings) is factored by block-Thomas too and
// stored as Rinv_k, G_k = Rinv_k R_{k,k-1}, F_k = Rinv_k R_{k,k+1}.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "dense.cuh"
#include "p1_entries.cuh"
#include "sweep_common.cuh"

#ifndef HELM_SETUP_DMMA
#define HELM_SETUP_DMMA 1   // block products of the setup kernels on the FP64 tensor cores (dense.cuh blk_mm_dmma)
#endif
#ifndef HELM_GJ_BLOCKED
#define HELM_GJ_BLOCKED 1   // shared-memory Gauss-Jordan (wide strips): panels of 8 pivots, the other columns updated on the tensor cores
#endif
#define WIDE_GJ(S, w, piv, colv, ybuf, redv, flag) \
  ((ybuf) ? gj_invert_blk(S, w, w, piv, colv, ybuf, redv, flag) : gj_invert(S, w, piv, colv, redv, nullptr, flag))
#if HELM_SETUP_DMMA
#define SETUP_MM blk_mm_dmma
#else
#define SETUP_MM blk_mm_tiled
#endif

static constexpr int kXinvMaxW = 36;   // explicit separator inverse for the register-streaming kernel

// Factor sets are shared between handles that describe the same strips (LRL and
// RLR, BTB and TBT, or different gathers): same problem, axis, N, overlap, P.
struct SharedFactors {
  int refs;
  long prob_uid;
  int axis, N, overlap, P;
  cplx *dg, *al, *cr, *ne, *tc, *fac, *red, *xinv, *fac2, *facp;
  long factor_bytes;
  float2* xinv32 = nullptr;   // complex64 separator-inverse rows, made on the first sweep_set_precision(32)
  long xinv_elems = 0;
  cplx* sep2 = nullptr;       // two-level separator panels
  int* sep2_plan = nullptr;
  int sep2_M = 0, sep2_ld1 = 0, sep2_ld2 = 0;
};
static std::vector<SharedFactors*> g_shared;
static std::mutex g_shared_mu;   // setups of different axes may run on concurrent host threads

// ------------------------------------------------------------------ bands + corrections
struct StripGeo {
  const int* a;   // first line of each strip
  const int* w;   // width
  int N, nc, wmax, axis;
};

// Five-point scheme (the paper's; reading DESIGN.md §3 FD5): the strip
// matrix A_s has the global rows (u_E + u_W + u_N + u_S - 4 u)/h^2 + k^2 u with
// ghost-point Robin elimination (Eq. 1b / Eq. 4: inward neighbour 2/h^2,
// + 2ik/h on the diagonal) on every boundary line of the strip, physical or
// interface.  Stored: S_s = D_s A_s (complex symmetric), D_s = fd5_d:
//   S(p,p) = d_p (-4/h^2 + k^2 + 2ik/h [q edge] + 2ik/h [c edge])
//   S(p, along) = dc(c)/h^2,  S(p, cross) = dq(q)/h^2,  no diagonal coupling.
// The correction (Atilde_s - A) v on an interface row is
//   (1/h^2) v(inner line) + (2ik/h) v(interface line) - (1/h^2) v(outer line),
// unscaled (the kernels scale source + corrections by D_s together).
__global__ void k_strip_bands_fd5(GridView g, StripGeo sg, cplx* dg, cplx* al, cplx* cr, cplx* ne, cplx* tc) {
  const int s = blockIdx.y;
  const int w = sg.w[s];
  const int nc = sg.nc;
  const double ih2 = 1.0 / (g.h * g.h), k = g.omega;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nc * sg.wmax; e += gridDim.x * blockDim.x) {
    int c = e / sg.wmax, q = e % sg.wmax;
    long idx = ((long)s * nc + c) * sg.wmax + q;
    if (q >= w) {
      dg[idx] = al[idx] = cr[idx] = ne[idx] = cmk(0, 0);
      continue;
    }
    const bool qe = q == 0 || q == w - 1, ce = c == 0 || c == nc - 1;
    const double dq = qe ? 0.5 : 1.0, dc = ce ? 0.5 : 1.0;
    dg[idx] = cmk(dq * dc * (-4.0 * ih2 + k * k), dq * dc * (2.0 * k / g.h) * ((qe ? 1 : 0) + (ce ? 1 : 0)));
    al[idx] = (q + 1 < w) ? cmk(dc * ih2, 0.0) : cmk(0, 0);
    cr[idx] = (c + 1 < nc) ? cmk(dq * ih2, 0.0) : cmk(0, 0);
    ne[idx] = cmk(0, 0);
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * nc; e += gridDim.x * blockDim.x) {
    int side = e / nc, c = e % nc;
    cplx* o = tc + (((long)s * 2 + side) * nc + c) * kTcW;
    bool has = side == 0 ? (s > 0) : (s < sg.N - 1);
    for (int kk = 0; kk < kTcW; ++kk) o[kk] = cmk(0, 0);
    if (!has) continue;
    o[1] = cmk(0.0, 2.0 * k / g.h);   // interface line
    o[3] = cmk(-ih2, 0.0);            // outer line
    o[5] = cmk(ih2, 0.0);             // inner line
  }
}

__global__ void k_strip_bands(GridView g, StripGeo sg, cplx* dg, cplx* al, cplx* cr, cplx* ne, cplx* tc) {
  const int s = blockIdx.y;
  const int a = sg.a[s], w = sg.w[s], b = a + w - 1;
  CellSel loc{sg.axis, a, b, s > 0 ? 1 : 0, s < sg.N - 1 ? 1 : 0};
  CellSel all = sel_all();
  const int nc = sg.nc;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nc * sg.wmax; e += gridDim.x * blockDim.x) {
    int c = e / sg.wmax, q = e % sg.wmax;
    long idx = ((long)s * nc + c) * sg.wmax + q;
    if (q >= w) {
      dg[idx] = al[idx] = cr[idx] = ne[idx] = cmk(0, 0);
      continue;
    }
    int pa = a + q;
    dg[idx] = gen_diag(g, loc, sg.axis, pa, c);
    al[idx] = (q + 1 < w) ? gen_along(g, loc, sg.axis, pa, c) : cmk(0, 0);
    cr[idx] = (c + 1 < nc) ? gen_cross(g, loc, sg.axis, pa, c) : cmk(0, 0);
    ne[idx] = (c + 1 < nc && q + 1 < w) ? gen_ne(g, loc, sg.axis, pa, c) : cmk(0, 0);
  }
  // transmission-correction stencil (D8): (Atilde_s - A) on the interface rows.
  // tc[((s*2 + side)*nc + c)*kTcW + k], k: 0 v(L,c-1), 1 v(L,c), 2 v(L,c+1), 3 v(O,c),
  // 4 v(O,c+dd), 5 v(I,c) (inner line: zero for P1)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * nc; e += gridDim.x * blockDim.x) {
    int side = e / nc, c = e % nc;
    cplx* o = tc + (((long)s * 2 + side) * nc + c) * kTcW;
    bool has = side == 0 ? (s > 0) : (s < sg.N - 1);
    o[5] = cmk(0, 0);
    if (!has) {
      for (int k = 0; k < 5; ++k) o[k] = cmk(0, 0);
      continue;
    }
    int L = side == 0 ? a : b;
    o[0] = (c >= 1) ? csub(gen_cross(g, loc, sg.axis, L, c - 1), gen_cross(g, all, sg.axis, L, c - 1)) : cmk(0, 0);
    o[1] = csub(gen_diag(g, loc, sg.axis, L, c), gen_diag(g, all, sg.axis, L, c));
    o[2] = (c + 1 < nc) ? csub(gen_cross(g, loc, sg.axis, L, c), gen_cross(g, all, sg.axis, L, c)) : cmk(0, 0);
    if (side == 0) {
      o[3] = cscale(gen_along(g, all, sg.axis, L - 1, c), -1.0);
      o[4] = (c >= 1) ? cscale(gen_ne(g, all, sg.axis, L - 1, c - 1), -1.0) : cmk(0, 0);
    } else {
      o[3] = cscale(gen_along(g, all, sg.axis, L, c), -1.0);
      o[4] = (c + 1 < nc) ? cscale(gen_ne(g, all, sg.axis, L, c), -1.0) : cmk(0, 0);
    }
  }
}

// ------------------------------------------------------------------ segment factorisation
struct FacArgs {
  const int* w;
  const long* fac_off;
  const int* seg_lo;
  const int* seg_hi;
  const cplx *dg, *al, *cr, *ne;
  int nc, wmax, P;
  cplx* fac;
  cplx* scratch;   // per (s,p): 4 w^2: ping, pong, XLL, XLH
  long scratch_stride;
  int* status;     // first failure: (s*nc + c) + 1
  cplx* fac2;      // packed bottom-up inverses S'^{-1}_c, NULL = not kept
  cplx* facp;      // packed top-down inverses Sinv_c, NULL = not kept
  const long* pfac_off;
  int s0;          // first strip of this launch (the setup runs in strip chunks)
};

__device__ inline void build_D(cplx* S, const cplx* dg, const cplx* al, int w) {
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    int p = e / w, q = e % w;
    cplx v = cmk(0, 0);
    if (p == q) v = dg[p];
    else if (q == p + 1) v = al[p];
    else if (p == q + 1) v = al[q];
    S[e] = v;
  }
  __syncthreads();
}

__global__ void k_factor_segments(FacArgs fa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.y + fa.s0, pseg = blockIdx.x;
  const int w = fa.w[s];
  cplx* S = reinterpret_cast<cplx*>(smem_raw);
  cplx* colv = S + w * w;
  // gj_invert_blk needs the panel's pivot rows (8 w entries): used when the launch's shared memory holds them
  unsigned dsm;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsm));
  const bool gjblk = HELM_GJ_BLOCKED && dsm >= sizeof(cplx) * ((size_t)w * w + 9 * (size_t)w) + sizeof(int) * (w + 4) + 64;
  cplx* ybuf = gjblk ? colv + w : nullptr;
  double* redv = reinterpret_cast<double*>(colv + w + (gjblk ? 8 * w : 0));
  int* flag = reinterpret_cast<int*>(redv + 4);
  int* piv = flag + 4;
  const int lo = fa.seg_lo[pseg], hi = fa.seg_hi[pseg];
  const long band = (long)s * fa.nc * fa.wmax;
  cplx* fac = fa.fac + fa.fac_off[s];
  const long w2 = (long)w * w;
  auto Ub = [&](int c, int mode) { return Bidi{mode, fa.cr + band + (long)c * fa.wmax, fa.ne + band + (long)c * fa.wmax}; };
  const Bidi NONE{BD_NONE, nullptr, nullptr};

  // top-down block-Thomas over the segment
  for (int c = lo; c <= hi; ++c) {
    build_D(S, fa.dg + band + (long)c * fa.wmax, fa.al + band + (long)c * fa.wmax, w);
    if (c > lo) blk_lxr(S, fac + (long)(c - 1) * w2, Ub(c - 1, BD_UT), Ub(c - 1, BD_U), w, -1.0, true);
    if (WIDE_GJ(S, w, piv, colv, ybuf, redv, flag)) {
      if (threadIdx.x == 0) atomicCAS(fa.status, 0, s * fa.nc + c + 1);
      return;
    }
    blk_copy(fac + (long)c * w2, S, w);
  }
  if (fa.P == 1) return;
  cplx* scr = fa.scratch + ((long)s * fa.P + pseg) * fa.scratch_stride;
  cplx* ping = scr;
  cplx* pong = scr + w2;
  cplx* XLL = scr + 2 * w2;
  cplx* XLH = scr + 3 * w2;
  // bottom-up block-Thomas: S'_hi = D_hi, S'_c = D_c - U_c S'^{-1}_{c+1} U_c^T;
  // X[lo,lo] = S'^{-1}_lo (corner block of the segment inverse)
  for (int c = hi; c >= lo; --c) {
    build_D(S, fa.dg + band + (long)c * fa.wmax, fa.al + band + (long)c * fa.wmax, w);
    if (c < hi) blk_lxr(S, ping, Ub(c, BD_U), Ub(c, BD_UT), w, -1.0, true);
    if (WIDE_GJ(S, w, piv, colv, ybuf, redv, flag)) {
      if (threadIdx.x == 0) atomicCAS(fa.status, 0, s * fa.nc + c + 1);
      return;
    }
    blk_copy(c == lo ? XLL : ping, S, w);
  }
  // X[lo,hi]: Y_hi = Sinv_hi; Y_c = -Sinv_c U_c Y_{c+1}
  blk_copy(ping, fac + (long)hi * w2, w);
  cplx* cur = ping;
  cplx* nxt = pong;
  for (int c = hi - 1; c >= lo; --c) {
    // tmp = U_c Y_{c+1}  (into XLH as scratch), then nxt = -Sinv_c tmp
    blk_lxr(XLH, cur, Ub(c, BD_U), NONE, w, 1.0, false);
    SETUP_MM(nxt, w, fac + (long)c * w2, w, false, XLH, w, w, -1.0, false);
    cplx* t = cur; cur = nxt; nxt = t;
  }
  blk_copy(XLH, cur, w);
}

// ------------------------------------------------------------------ register-row factorisation (w <= 36)
// Same recurrences as k_factor_segments, laid out for throughput: one CTA of
// 96 threads per (segment, strip, kind).  Row i of the current block lives in
// the registers of the thread pair (2i, 2i+1), thread half h holding columns
// j = 2 jj + h.  The in-place Gauss-Jordan inversion uses implicit partial
// pivoting (rows stay in their threads; the pivot row is broadcast through
// shared memory, two barriers per pivot step; the permutation is undone when
// the inverse is written back in natural order).
//   kind 0: top-down Thomas S_c = D_c - U_{c-1}^T Sinv_{c-1} U_{c-1} (writes fac),
//           then X[lo,hi] by Y_hi = Sinv_hi, Y_c = -Sinv_c U_c Y_{c+1}
//   kind 1: bottom-up S'_c = D_c - U_c S'^{-1}_{c+1} U_c^T, X[lo,lo] = S'^{-1}_lo
// Pivot choice (largest |a_ik| among the rows not yet used, ties to the lower
// row) and the elementary operations are those of gj_invert.
#include "row_gj.cuh"


__device__ long long g_red_prof[8];   // diagnostics (setup_timing knob): block 0 sub-phase cycles

// a = row i of D_c - (L X R) with X = sm.mat:
//   td (kind 0): L = U_{c-1}^T, R = U_{c-1};  bu (kind 1): L = U_c, R = U_c^T
__device__ __forceinline__ void row_schur(cplx (&a)[kRowHW], int w, const cplx* dg, const cplx* al, const cplx* cr,
                                          const cplx* ne, bool has, bool td, const RowSmem& sm) {
  const int i = threadIdx.x / kLPR, h = threadIdx.x % kLPR;
  const cplx zero = cmk(0, 0);
  const cplx dgi = i < w ? __ldg(dg + i) : zero;
  const cplx ali = i + 1 < w ? __ldg(al + i) : zero;
  const cplx alm = (i >= 1 && i < w) ? __ldg(al + i - 1) : zero;
#pragma unroll
  for (int jj = 0; jj < kRowHW; ++jj) {
    const int q = kLPR * jj + h;
    a[jj] = q == i ? dgi : (q == i + 1 ? ali : (q + 1 == i ? alm : zero));
  }
  if (!has || i >= w) return;
  const cplx ci = __ldg(cr + i);
  const cplx* x0 = sm.mat + i * kRowW;
  if (td) {
    // (L X)[i] = cr[i] X[i] + ne[i-1] X[i-1];  v_q = cr[q] y_q + ne[q-1] y_{q-1}
    const cplx nm = i >= 1 ? __ldg(ne + i - 1) : zero;
    const cplx* x1 = sm.mat + (i >= 1 ? i - 1 : 0) * kRowW;
#pragma unroll
    for (int jj = 0; jj < kRowHW; ++jj) {
      const int q = kLPR * jj + h;
      if (q >= w) break;
      cplx yq = cmul(ci, x0[q]);
      if (i >= 1) cfma(yq, nm, x1[q]);
      cplx v = cmul(__ldg(cr + q), yq);
      if (q >= 1) {
        cplx yp = cmul(ci, x0[q - 1]);
        if (i >= 1) cfma(yp, nm, x1[q - 1]);
        cfma(v, __ldg(ne + q - 1), yp);
      }
      a[jj] = csub(a[jj], v);
    }
  } else {
    // (L X)[i] = cr[i] X[i] + ne[i] X[i+1];  v_q = cr[q] y_q + ne[q] y_{q+1}
    const cplx ni = i + 1 < w ? __ldg(ne + i) : zero;
    const cplx* x1 = sm.mat + (i + 1 < w ? i + 1 : i) * kRowW;
#pragma unroll
    for (int jj = 0; jj < kRowHW; ++jj) {
      const int q = kLPR * jj + h;
      if (q >= w) break;
      cplx yq = cmul(ci, x0[q]);
      if (i + 1 < w) cfma(yq, ni, x1[q]);
      cplx v = cmul(__ldg(cr + q), yq);
      if (q + 1 < w) {
        cplx yn = cmul(ci, x0[q + 1]);
        if (i + 1 < w) cfma(yn, ni, x1[q + 1]);
        cfma(v, __ldg(ne + q), yn);
      }
      a[jj] = csub(a[jj], v);
    }
  }
}

__device__ __forceinline__ void row_store(cplx* dst, int w, const RowSmem& sm) {
  const float invw = 1.0f / (float)w;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int r = div_w(e, invw);
    dst[e] = sm.mat[r * kRowW + (e - r * w)];
  }
}

// padded packed upper triangle (common.cuh pk_start) of the symmetrised block in sm.mat
__device__ __forceinline__ void row_store_packed(cplx* dst, int w, const RowSmem& sm) {
  for (int r = threadIdx.x >> 3; r < w; r += blockDim.x >> 3) {
    const int st = pk_start(r, w);
    for (int q = r + (threadIdx.x & 7); q < w; q += 8) {
      const cplx a = sm.mat[r * kRowW + q], b = sm.mat[q * kRowW + r];
      dst[st + (q - r)] = cmk(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
    }
  }
}

#ifndef HELM_FAC_G
#define HELM_FAC_G 0        // 1: k_factor_rows uses row_invert_g (raw pivot-row broadcast)
#endif
#ifndef HELM_FAC_ROT
#define HELM_FAC_ROT 0      // 1: rotating register slots (row_invert_r: 1.6x per CTA alone, slower in the setup at the register cap)
#endif
__device__ __forceinline__ int fac_invert(cplx (&a)[kRowHW], int w, RowSmem& sm) {
  if (HELM_FAC_G) return row_invert_g<kLPR>(a, w, sm);
  if (HELM_FAC_ROT) return row_invert_r<HELM_ROW_UP>(a, w, sm);
  return row_invert(a, w, sm);
}
#ifndef HELM_FAC_MINB
#define HELM_FAC_MINB 5   // 5 CTAs per SM (a few spills) beat 4 without
#endif
__global__ void __launch_bounds__(kRowThreads, HELM_FAC_MINB) k_factor_rows(FacArgs fa) {
  __shared__ RowSmem sm;
  const int s = blockIdx.y + fa.s0, pseg = blockIdx.x, kind = blockIdx.z;
  if (kind == 1 && fa.P == 1) return;
  const int w = fa.w[s];
  const int lo = fa.seg_lo[pseg], hi = fa.seg_hi[pseg];
  const long band = (long)s * fa.nc * fa.wmax;
  cplx* fac = fa.fac + fa.fac_off[s];
  const long w2 = (long)w * w;
  cplx* scr = fa.scratch + ((long)s * fa.P + pseg) * fa.scratch_stride;
  const int i = threadIdx.x / kLPR, h = threadIdx.x % kLPR;
  cplx a[kRowHW];
  auto B = [&](const cplx* base, int c) { return base + band + (long)c * fa.wmax; };
  if (kind == 0) {
    for (int c = lo; c <= hi; ++c) {
      row_schur(a, w, B(fa.dg, c), B(fa.al, c), B(fa.cr, c - 1), B(fa.ne, c - 1), c > lo, true, sm);
      if (fac_invert(a, w, sm)) {
        if (threadIdx.x == 0) atomicCAS(fa.status, 0, s * fa.nc + c + 1);
        return;
      }
      row_store(fac + (long)c * w2, w, sm);
      if (fa.facp) row_store_packed(fa.facp + fa.pfac_off[s] + (long)c * pk_size(w), w, sm);
    }
    if (fa.P == 1) return;
    // X[lo,hi]: Y_hi = Sinv_hi (in sm.mat); Y_c = -Sinv_c (U_c Y_{c+1})
#ifdef HELM_FAC_NOXCHAIN
    for (int c = hi - 1; c >= hi; --c) {   // ablation (timing only): no X chain
#else
    for (int c = hi - 1; c >= lo; --c) {
#endif
      const cplx* cr = B(fa.cr, c);
      const cplx* ne = B(fa.ne, c);
      // Sinv_c (stored by this CTA in the top-down pass) is read into registers first: its
      // L2 latency passes behind the coupling product below
      constexpr int kPre = (kRowW * kRowW + kRowThreads - 1) / kRowThreads;
      cplx pre[kPre];
      {
        const cplx* src = fac + (long)c * w2;
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          const int e = threadIdx.x + u * kRowThreads;
          pre[u] = e < w2 ? __ldcg(src + e) : cmk(0, 0);
        }
      }
      if (i < w) {
        const cplx ci = __ldg(cr + i);
        const cplx ni = i + 1 < w ? __ldg(ne + i) : cmk(0, 0);
        for (int q = h; q < w; q += kLPR) {
          cplx v = cmul(ci, sm.mat[i * kRowW + q]);
          if (i + 1 < w) cfma(v, ni, sm.mat[(i + 1) * kRowW + q]);
          sm.tmat[i * kRowW + q] = v;
        }
      }
      __syncthreads();
      // mat is free now: Sinv_c into it, then Y_c = -Sinv_c tmat
      {
        const float invw = 1.0f / (float)w;
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          const int e = threadIdx.x + u * kRowThreads;
          if (e < w2) {
            const int r = div_w(e, invw);
            sm.mat[r * kRowW + (e - r * w)] = pre[u];
          }
        }
      }
      __syncthreads();
#if HELM_SETUP_DMMA
      // Y_c = -Sinv_c tmat on the FP64 tensor cores, the warp's output tiles in registers
      // until every warp has read Sinv_c (the result replaces it in sm.mat)
      blk_mm_dmma_reg<(((kRowW + 7) / 8) * ((kRowW + 7) / 8) + kRowWarps - 1) / kRowWarps>(sm.mat, kRowW, sm.mat, kRowW,
                                                                                           sm.tmat, kRowW, w, -1.0);
#else
      {
        const int nt = (w + 3) >> 2;
        const int t = threadIdx.x;
        cplx acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = cmk(0, 0);
        const int i0 = (t / nt) * 4, j0 = (t % nt) * 4;
        const bool on = t < nt * nt;
        if (on) {
          for (int k = 0; k < w; ++k) {
            cplx av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              av[u] = sm.mat[(i0 + u) * kRowW + k];     // rows >= w hold finite leftovers, never stored
              bv[u] = sm.tmat[k * kRowW + j0 + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int v = 0; v < 4; ++v) cfma(acc[u][v], av[u], bv[v]);
          }
        }
        __syncthreads();
        if (on) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v)
              if (i0 + u < w && j0 + v < w) sm.mat[(i0 + u) * kRowW + j0 + v] = cscale(acc[u][v], -1.0);
        }
      }
      __syncthreads();
#endif
    }
    row_store(scr + 3 * w2, w, sm);
  } else {
    for (int c = hi; c >= lo; --c) {
      row_schur(a, w, B(fa.dg, c), B(fa.al, c), B(fa.cr, c), B(fa.ne, c), c < hi, false, sm);
      if (fac_invert(a, w, sm)) {
        if (threadIdx.x == 0) atomicCAS(fa.status, 0, s * fa.nc + c + 1);
        return;
      }
      if (fa.fac2) row_store_packed(fa.fac2 + fa.pfac_off[s] + (long)c * pk_size(w), w, sm);
    }
    row_store(scr + 2 * w2, w, sm);
  }
}

// ------------------------------------------------------------------ separator system
struct RedArgs {
  const int* w;
  const long* fac_off;
  const long* red_off;
  const int* seg_lo;
  const int* seg_hi;
  const cplx *dg, *al, *cr, *ne;
  int nc, wmax, P;
  const cplx* fac;
  const cplx* scratch;
  long scratch_stride;
  cplx* red;
  cplx* rscratch;  // per strip: 2 w^2 (R_{k,k+1} of the previous separator, temp)
  int* status;
  int s0;          // first strip of this launch
  cplx* rraw = nullptr;   // two-level separator solve: the raw blocks R_kk, R_{k,k+1} per separator (stride 2 wmax^2)
};

// One CTA (96 threads) per strip walks the K = P-1 separators in order (the
// separator block-Thomas is a chain).  Block inverses use the register-row
// Gauss-Jordan of k_factor_rows; products use register-tiled smem matmuls.
// Shared memory: RowSmem (static) + S, T1 (R_{k,k+1}), T2 (F_k) (dynamic).

// 384 threads: the register-row Gauss-Jordan uses the first 96 (the others only
// join its barriers); the products, stencil applications and copies use all.
static constexpr int kRedThreads = 384;
#ifndef HELM_RED_LPR
#define HELM_RED_LPR 9      // threads per block row of k_reduced's Gauss-Jordan (kRowW * LPR <= 384)
#endif
static constexpr int kRedLPR = HELM_RED_LPR;
#ifndef HELM_RED_OLDGJ
#define HELM_RED_OLDGJ 0    // 1: k_reduced uses row_invert (2 threads per row, normalised pivot-row broadcast)
#endif
#if HELM_SETUP_DMMA
#define RED_MM blk_mm_dmma
#else
#define RED_MM blk_mm_tiled2
#endif
__global__ void __launch_bounds__(kRedThreads) k_reduced(RedArgs ra) {
  __shared__ RowSmem sm;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.x + ra.s0;
  const int w = ra.w[s];
  const long w2 = (long)w * w;
  cplx* S = reinterpret_cast<cplx*>(smem_raw);
  cplx* T1 = S + w2;   // R_{k-1,k} of the previous separator, then R_{k,k+1}
  cplx* T2 = T1 + w2;  // F_{k-1}, then F_k
  // staged operands of separator k, double-buffered: [buf][Bh | Bl | Bx | bands(6w)]
  cplx* stage0 = T2 + w2;
  const long stage_sz = 3 * w2 + 6L * w;
  const long band = (long)s * ra.nc * ra.wmax;
  const cplx* fac = ra.fac + ra.fac_off[s];
  cplx* red = ra.red + ra.red_off[s];
  auto scr = [&](int p) { return ra.scratch + ((long)s * ra.P + p) * ra.scratch_stride; };
  const int P = ra.P;
#if HELM_RED_OLDGJ
  const int i = threadIdx.x / kLPR, h = threadIdx.x % kLPR;
#endif
  // cp.async the operands of separator k into buffer k & 1: Sinv_{h_k}, X_{k+1}[lo,lo],
  // X_{k+1}[lo,hi] and the couplings of rows h_k, s_k, h_{k+1}
  auto stage = [&](int k) {
    cplx* d = stage0 + (k & 1) * stage_sz;
    const int hk = ra.seg_hi[k], sk = hk + 1, hk1 = ra.seg_hi[k + 1];
    const cplx* g0 = fac + (long)hk * w2;
    const cplx* g1 = scr(k + 1) + 2 * w2;
    const cplx* g2 = scr(k + 1) + 3 * w2;
    for (int e = threadIdx.x; e < w2; e += blockDim.x) {
      cp_async16(d + e, g0 + e);
      cp_async16(d + w2 + e, g1 + e);
      cp_async16(d + 2 * w2 + e, g2 + e);
    }
    const int rows[3] = {hk, sk, hk1};
    for (int e = threadIdx.x; e < 3 * w; e += blockDim.x) {
      const int rr = e / w, q2 = e - rr * w;
      cp_async16(d + 3 * w2 + (2 * rr) * w + q2, ra.cr + band + (long)rows[rr] * ra.wmax + q2);
      cp_async16(d + 3 * w2 + (2 * rr + 1) * w + q2, ra.ne + band + (long)rows[rr] * ra.wmax + q2);
    }
    cp_async_commit();
  };
  if (threadIdx.x == 0) sm.gjp[0] = sm.gjp[1] = sm.gjp[2] = 0;
  stage(0);
  for (int k = 0; k <= P - 2; ++k) {
    const int hk = ra.seg_hi[k];          // last row of segment k
    const int sk = hk + 1;                // separator row
    cplx* Rinv = red + (long)k * 3 * w2;
    cplx* G = Rinv + w2;
    cplx* F = Rinv + 2 * w2;
    cp_async_wait_all();
    __syncthreads();
    if (k + 1 <= P - 2) stage(k + 1);     // overlaps this separator's work
    cplx* Bh = stage0 + (k & 1) * stage_sz;
    cplx* Bl = Bh + w2;
    cplx* Bx = Bl + w2;
    cplx* bands = Bx + w2;
    auto Ub = [&](int rr, int mode) { return Bidi{mode, bands + (2 * rr) * w, bands + (2 * rr + 1) * w}; };
    const bool pr = blockIdx.x == 0 && threadIdx.x == 0;
    long long c0 = pr ? clock64() : 0;
    // R_kk = D_sk - U_hk^T X_k[hi,hi] U_hk - U_sk X_{k+1}[lo,lo] U_sk^T
    build_D(S, ra.dg + band + (long)sk * ra.wmax, ra.al + band + (long)sk * ra.wmax, w);
    blk_lxr(S, Bh, Ub(0, BD_UT), Ub(0, BD_U), w, -1.0, true);
    blk_lxr(S, Bl, Ub(1, BD_U), Ub(1, BD_UT), w, -1.0, true);
    if (ra.rraw) {
      cplx* d = ra.rraw + ((long)s * (P - 1) + k) * 2 * ra.wmax * ra.wmax;
      for (int e = threadIdx.x; e < w * w; e += blockDim.x) d[e] = S[e];   // R_kk
      __syncthreads();
    }
    // - R_{k,k-1} Rinv_{k-1} R_{k-1,k} = - R_{k-1,k}^T F_{k-1}
    if (k >= 1) RED_MM(S, w, T1, w, true, T2, w, w, -1.0, true);
    long long c1 = pr ? clock64() : 0;
    if (pr) g_red_prof[0] += c1 - c0;
    // Rinv_k (register-row Gauss-Jordan; result in sm.mat, row stride kRowW)
#if HELM_RED_OLDGJ
    cplx a[kRowHW];
#pragma unroll
    for (int jj = 0; jj < kRowHW; ++jj) {
      const int col = kLPR * jj + h;
      a[jj] = (i < w && col < w) ? S[i * w + col] : cmk(0, 0);
    }
    if (row_invert(a, w, sm)) {
#else
    cplx a[kRowW / kRedLPR];
    {
      const int ir = threadIdx.x / kRedLPR, hr = threadIdx.x % kRedLPR;
#pragma unroll
      for (int jj = 0; jj < kRowW / kRedLPR; ++jj) {
        const int col = kRedLPR * jj + hr;
        a[jj] = (ir < w && col < w) ? S[ir * w + col] : cmk(0, 0);
      }
    }
    if (row_invert_g<kRedLPR>(a, w, sm)) {
#endif
      if (threadIdx.x == 0) atomicCAS(ra.status, 0, s * ra.nc + sk + 1);
      return;
    }
    long long c2 = pr ? clock64() : 0;
    if (pr) g_red_prof[1] += c2 - c1;
    row_store(Rinv, w, sm);
    if (k >= 1) {
      // G_k = Rinv_k R_{k,k-1} = Rinv_k R_{k-1,k}^T   (S <- T1^T; S is free now)
      const float invw = 1.0f / (float)w;
      for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
        const int p2 = div_w(e, invw), q2 = e - p2 * w;
        S[e] = T1[q2 * w + p2];
      }
      __syncthreads();
      RED_MM(G, w, sm.mat, kRowW, false, S, w, w, 1.0, false);
    }
    if (k <= P - 3) {
      // R_{k,k+1} = - U_sk X_{k+1}[lo,hi] U_{hk1};  F_k = Rinv_k R_{k,k+1}
      blk_lxr(T1, Bx, Ub(1, BD_U), Ub(2, BD_U), w, -1.0, false);
      if (ra.rraw) {
        cplx* d = ra.rraw + (((long)s * (P - 1) + k) * 2 + 1) * ra.wmax * ra.wmax;
        for (int e = threadIdx.x; e < w * w; e += blockDim.x) d[e] = T1[e];   // R_{k,k+1}
      }
      RED_MM(T2, w, sm.mat, kRowW, false, T1, w, w, 1.0, false);
      for (int e = threadIdx.x; e < w * w; e += blockDim.x) F[e] = T2[e];
    }
    __syncthreads();
    if (pr) g_red_prof[2] += clock64() - c2;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_red_prof[3] += sm.gjp[0]; g_red_prof[4] += sm.gjp[1]; g_red_prof[5] += sm.gjp[2];
  }
}

#undef RED_MM
// ------------------------------------------------------------------ two-level separator solve (setup)
// DESIGN.md §5 "Two-level separator solve".  The K separators of a strip are
// split into M coarse separators and M + 1 groups of fine ones between them
// (sep2_plan).  With R block tridiagonal (diagonal R_kk, couplings E_k = R_{k,k+1},
// R_{k+1,k} = E_k^T), Y^g = (R restricted to group g)^{-1} and, for a fine
// separator p of group g with coarse neighbours c_l = first - 1, c_r = last + 1,
//   x_p = (Y^g g_g)_p - V_p x_{c_l} - W_p x_{c_r},   V_p = Y^g_{p,first} E_{c_l}^T,
//                                                    W_p = Y^g_{p,last} E_last;
// the coarse values solve the block-tridiagonal Schur system
//   Rh x_C = gh,  gh_c = g_c - sum_j H_{c,j} g_j,
//   H_{c,j} = E_{c-1}^T Y^{left}_{last,j} (j in the left group), E_c Y^{right}_{first,j} (right group),
//   Rh_cc = R_cc - E_{c-1}^T Y^{left}_{last,last} E_{c-1} - E_c Y^{right}_{first,first} E_c^T,
//   Rh_{c,c'} = -E_c Y^{g}_{first,last} E_last   (c' the next coarse, g the group between).
// Every separator gets two row panels: panel 1 (its group's Y row, or for a
// coarse one [H left | H right]) and panel 2 (Q_p = V_p Xc_{c_l,.} + W_p Xc_{c_r,.}
// for a fine p, the row of Xc = Rh^{-1} for a coarse one), so that the apply
// forms x_p from ~K / sqrt(K) blocks instead of the K blocks of a row of R^{-1}.
static constexpr int kSep2MaxB = 8;                        // blocks per group (panel 1 of a coarse: <= 2 groups)
static constexpr int kSep2PlanHdr = 64;                    // ints: [0] M, [1] groups, [2] nb1 max, [8..] gstart, [32..] glen
static constexpr int kSep2PlanStride = 4 + 2 * kSep2MaxB;  // ints per separator: kind, n1, group / coarse index, -, idx1[]

struct Sep2Args {
  const int* w;
  int wmax, P, s0;
  const cplx* rraw;      // [s][k][2][wmax^2]: R_kk, E_k
  const int* plan;       // sep2 plan (device)
  cplx* ytmp;            // per (s, group): Li[B], Ri[B], Y[B^2] blocks of wmax^2
  long ytmp_stride;      // cplx per (s, group)
  cplx* vw;              // per (s, k): V_k, W_k
  cplx* cd;              // per (s, coarse j): [0] left diagonal term, [1] right diagonal term, [2] Rh_{j,j+1}
  cplx* xc;              // per s: Xc (M^2 blocks) and its temporaries (2M)
  cplx* sep2;            // panels
  const long* sep2_off;
  int ld1, ld2;
  int* status;
};

// C (+)= alpha op(A) op(B) on w x w blocks in shared memory (row stride w), 2 x 2 tiles
__device__ inline void s2_mm(cplx* C, const cplx* A, bool ta, const cplx* B, bool tb, int w, double alpha, bool acc) {
  const int nt = (w + 1) / 2;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) {
    const int i0 = (t / nt) * 2, j0 = (t % nt) * 2;
    cplx c[2][2] = {{cmk(0, 0), cmk(0, 0)}, {cmk(0, 0), cmk(0, 0)}};
    for (int r = 0; r < w; ++r) {
      cplx av[2], bv[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = i0 + u, j = j0 + u;
        av[u] = i < w ? (ta ? A[r * w + i] : A[i * w + r]) : cmk(0, 0);
        bv[u] = j < w ? (tb ? B[j * w + r] : B[r * w + j]) : cmk(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) cfma(c[u][v], av[u], bv[v]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = i0 + u, j = j0 + v;
        if (i < w && j < w) C[i * w + j] = acc ? cadd(C[i * w + j], cscale(c[u][v], alpha)) : cscale(c[u][v], alpha);
      }
  }
  __syncthreads();
}
__device__ inline void s2_ld(cplx* d, const cplx* g, int w) {
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) d[e] = __ldcg(g + e);
  __syncthreads();
}
__device__ inline void s2_st(cplx* g, const cplx* d, int w, bool trans = false) {
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int r = e / w, c = e - r * w;
    g[e] = trans ? d[c * w + r] : d[e];
  }
  __syncthreads();
}
// dst (global, row stride w) = S^{-1}; S in shared memory (row stride w)
__device__ inline int s2_inv(cplx* dst, const cplx* S, int w, RowSmem& sm) {
  cplx a[kRowW / kRedLPR];
  {
    const int ir = threadIdx.x / kRedLPR, hr = threadIdx.x % kRedLPR;
#pragma unroll
    for (int jj = 0; jj < kRowW / kRedLPR; ++jj) {
      const int col = kRedLPR * jj + hr;
      a[jj] = (ir < w && col < w) ? S[ir * w + col] : cmk(0, 0);
    }
  }
  if (row_invert_g<kRedLPR>(a, w, sm)) return 1;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int r = e / w, c = e - r * w;
    dst[e] = sm.mat[r * kRowW + c];
  }
  __syncthreads();
  return 0;
}

// Explicit inverse Y (nb x nb blocks, Y + (i nb + j) ws) of the block-tridiagonal
// matrix with diagonal blocks D(j) and couplings E(j) = block (j, j+1), block
// (j+1, j) = E(j)^T:  forward Schur complements L_j = D_j - E_{j-1}^T L_{j-1}^{-1} E_{j-1},
// backward ones R_j = D_j - E_j R_{j+1}^{-1} E_j^T, diagonal blocks
// Y_jj = (D_j - E_{j-1}^T L_{j-1}^{-1} E_{j-1} - E_j R_{j+1}^{-1} E_j^T)^{-1},
// off-diagonal Y_ij = -L_i^{-1} E_i Y_{i+1,j} (i < j), Y_ji = Y_ij^T.
// Li, Ri: nb blocks each (global scratch).  sA..sD: four w x w shared blocks.
template <class DF, class EF>
__device__ int s2_bt_inverse(int nb, int w, long ws, DF D, EF E, cplx* Li, cplx* Ri, cplx* Y, cplx* sA, cplx* sB,
                             cplx* sC, cplx* sS, RowSmem& sm) {
  // forward
  s2_ld(sS, D(0), w);
  if (s2_inv(Li, sS, w, sm)) return 1;
  for (int j = 1; j < nb; ++j) {
    s2_ld(sA, E(j - 1), w);
    s2_ld(sB, Li + (j - 1) * ws, w);
    s2_mm(sC, sB, false, sA, false, w, 1.0, false);      // L^{-1} E
    s2_ld(sS, D(j), w);
    s2_mm(sS, sA, true, sC, false, w, -1.0, true);       // - E^T L^{-1} E
    if (s2_inv(Li + j * ws, sS, w, sm)) return 1;
  }
  // backward
  s2_ld(sS, D(nb - 1), w);
  if (s2_inv(Ri + (nb - 1) * ws, sS, w, sm)) return 1;
  for (int j = nb - 2; j >= 1; --j) {
    s2_ld(sA, E(j), w);
    s2_ld(sB, Ri + (j + 1) * ws, w);
    s2_mm(sC, sB, false, sA, true, w, 1.0, false);       // R^{-1} E^T
    s2_ld(sS, D(j), w);
    s2_mm(sS, sA, false, sC, false, w, -1.0, true);      // - E R^{-1} E^T
    if (s2_inv(Ri + j * ws, sS, w, sm)) return 1;
  }
  // diagonal blocks
  for (int j = 0; j < nb; ++j) {
    s2_ld(sS, D(j), w);
    if (j >= 1) {
      s2_ld(sA, E(j - 1), w);
      s2_ld(sB, Li + (j - 1) * ws, w);
      s2_mm(sC, sB, false, sA, false, w, 1.0, false);
      s2_mm(sS, sA, true, sC, false, w, -1.0, true);
    }
    if (j + 1 < nb) {
      s2_ld(sA, E(j), w);
      s2_ld(sB, Ri + (j + 1) * ws, w);
      s2_mm(sC, sB, false, sA, true, w, 1.0, false);
      s2_mm(sS, sA, false, sC, false, w, -1.0, true);
    }
    if (s2_inv(Y + (j * nb + j) * ws, sS, w, sm)) return 1;
  }
  // off-diagonal blocks, column by column upwards from the diagonal
  for (int j = 1; j < nb; ++j) {
    s2_ld(sS, Y + (j * nb + j) * ws, w);                   // Y_{i+1, j}
    for (int i = j - 1; i >= 0; --i) {
      s2_ld(sA, E(i), w);
      s2_mm(sC, sA, false, sS, false, w, 1.0, false);      // E_i Y_{i+1,j}
      s2_ld(sB, Li + i * ws, w);
      s2_mm(sS, sB, false, sC, false, w, -1.0, false);     // Y_ij = -L_i^{-1} E_i Y_{i+1,j}
      s2_st(Y + (i * nb + j) * ws, sS, w);
      s2_st(Y + (j * nb + i) * ws, sS, w, true);
    }
  }
  return 0;
}

__device__ __forceinline__ cplx* s2_panel1(const Sep2Args& a, int s, int k, int w) {
  return a.sep2 + a.sep2_off[s] + (long)k * w * (a.ld1 + a.ld2);
}
__device__ __forceinline__ cplx* s2_panel2(const Sep2Args& a, int s, int k, int w) {
  return s2_panel1(a, s, k, w) + (long)w * a.ld1;
}
// block (rows of) a w x w smem block into panel columns [col0, col0 + w)
__device__ inline void s2_put(cplx* panel, int ld, int col0, const cplx* blk, int w) {
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int r = e / w, c = e - r * w;
    panel[(long)r * ld + col0 + c] = blk[e];
  }
  __syncthreads();
}

// One CTA per (group, strip): Y^g, the fine separators' panel 1 and V / W, the
// adjacent coarse separators' H parts and their Schur-system terms.
static constexpr int kSep2Threads = 384;
__global__ void __launch_bounds__(kSep2Threads) k_sep2_group(Sep2Args a) {
  __shared__ RowSmem sm;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.y + a.s0, g = blockIdx.x;
  const int w = a.w[s], K = a.P - 1, M = a.plan[0];
  const long ws = (long)a.wmax * a.wmax;
  const int first = a.plan[8 + g], nb = a.plan[32 + g], last = first + nb - 1;
  cplx* sA = reinterpret_cast<cplx*>(smem_raw);
  cplx *sB = sA + ws, *sC = sB + ws, *sS = sC + ws, *sT = sS + ws;
  const cplx* rr = a.rraw + (long)s * K * 2 * ws;
  auto D = [&](int j) { return rr + (long)(first + j) * 2 * ws; };
  auto E = [&](int j) { return rr + ((long)(first + j) * 2 + 1) * ws; };
  cplx* Li = a.ytmp + ((long)s * (M + 1) + g) * a.ytmp_stride;
  cplx* Ri = Li + kSep2MaxB * ws;
  cplx* Y = Ri + kSep2MaxB * ws;
  if (s2_bt_inverse(nb, w, ws, D, E, Li, Ri, Y, sA, sB, sC, sS, sm)) {
    if (threadIdx.x == 0) atomicCAS(a.status, 0, -(s * 1024 + first + 1));
    return;
  }
  const bool hasl = g > 0, hasr = g < M;
  const int cl = first - 1, cr = last + 1;
  for (int l = 0; l < nb; ++l) {
    const int p = first + l;
    cplx* p1 = s2_panel1(a, s, p, w);
    for (int j = 0; j < nb; ++j) {
      s2_ld(sS, Y + (l * nb + j) * ws, w);
      s2_put(p1, a.ld1, j * w, sS, w);
    }
    cplx* v = a.vw + ((long)s * K + p) * 2 * ws;
    if (hasl) {   // V_p = Y_{l,0} E_{cl}^T
      s2_ld(sS, Y + (l * nb) * ws, w);
      s2_ld(sA, rr + ((long)cl * 2 + 1) * ws, w);
      s2_mm(sC, sS, false, sA, true, w, 1.0, false);
      s2_st(v, sC, w);
    }
    if (hasr) {   // W_p = Y_{l,nb-1} E_last
      s2_ld(sS, Y + (l * nb + nb - 1) * ws, w);
      s2_ld(sA, E(nb - 1), w);
      s2_mm(sC, sS, false, sA, false, w, 1.0, false);
      s2_st(v + ws, sC, w);
    }
  }
  if (hasr) {
    // coarse c_r (index g): H left part = E_last^T Y_{nb-1, j}; Rh term -E_last^T Y_{nb-1,nb-1} E_last
    cplx* p1 = s2_panel1(a, s, cr, w);
    s2_ld(sA, E(nb - 1), w);
    for (int j = 0; j < nb; ++j) {
      s2_ld(sS, Y + ((nb - 1) * nb + j) * ws, w);
      s2_mm(sC, sA, true, sS, false, w, 1.0, false);
      s2_put(p1, a.ld1, j * w, sC, w);
      if (j == nb - 1) {
        s2_mm(sT, sC, false, sA, false, w, -1.0, false);
        s2_st(a.cd + ((long)s * M + g) * 3 * ws, sT, w);
      }
    }
  }
  if (hasl) {
    // coarse c_l (index g - 1): H right part = E_cl Y_{0, j} (after the left group's nbl blocks);
    // Rh term -E_cl Y_00 E_cl^T; Rh_{g-1, g} = -E_cl Y_{0,nb-1} E_last
    const int nbl = a.plan[32 + g - 1];
    cplx* p1 = s2_panel1(a, s, cl, w);
    s2_ld(sA, rr + ((long)cl * 2 + 1) * ws, w);
    for (int j = 0; j < nb; ++j) {
      s2_ld(sS, Y + j * ws, w);
      s2_mm(sC, sA, false, sS, false, w, 1.0, false);
      s2_put(p1, a.ld1, (nbl + j) * w, sC, w);
      if (j == 0) {
        s2_mm(sT, sC, false, sA, true, w, -1.0, false);
        s2_st(a.cd + ((long)s * M + g - 1) * 3 * ws + ws, sT, w);
      }
      if (j == nb - 1 && hasr) {
        s2_ld(sS, E(nb - 1), w);
        s2_mm(sT, sC, false, sS, false, w, -1.0, false);
        s2_st(a.cd + ((long)s * M + g - 1) * 3 * ws + 2 * ws, sT, w);
      }
    }
  }
}

// One CTA per strip: the coarse Schur system Rh (M blocks) and Xc = Rh^{-1};
// the coarse separators' panel 2 (rows of Xc).
__global__ void __launch_bounds__(kSep2Threads) k_sep2_coarse(Sep2Args a) {
  __shared__ RowSmem sm;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.x + a.s0;
  const int w = a.w[s], K = a.P - 1, M = a.plan[0];
  const long ws = (long)a.wmax * a.wmax;
  cplx* sA = reinterpret_cast<cplx*>(smem_raw);
  cplx *sB = sA + ws, *sC = sB + ws, *sS = sC + ws;
  const cplx* rr = a.rraw + (long)s * K * 2 * ws;
  cplx* xcs = a.xc + (long)s * (M * M + 3 * M) * ws;   // Xc, then Li, Ri, Dh
  cplx* Li = xcs + (long)M * M * ws;
  cplx* Ri = Li + (long)M * ws;
  cplx* Dh = Ri + (long)M * ws;
  const cplx* cd = a.cd + (long)s * M * 3 * ws;
  for (int j = 0; j < M; ++j) {   // Rh_jj = R_cc + left term + right term
    const int c = a.plan[8 + j + 1] - 1;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x)
      Dh[j * ws + e] = cadd(__ldcg(rr + (long)c * 2 * ws + e), cadd(__ldcg(cd + (long)j * 3 * ws + e), __ldcg(cd + ((long)j * 3 + 1) * ws + e)));
  }
  __syncthreads();
  auto D = [&](int j) { return (const cplx*)(Dh + j * ws); };
  auto E = [&](int j) { return cd + ((long)j * 3 + 2) * ws; };
  if (s2_bt_inverse(M, w, ws, D, E, Li, Ri, xcs, sA, sB, sC, sS, sm)) {
    if (threadIdx.x == 0) atomicCAS(a.status, 0, -(s * 1024 + 1000));
    return;
  }
  for (int j = 0; j < M; ++j) {
    const int c = a.plan[8 + j + 1] - 1;
    cplx* p2 = s2_panel2(a, s, c, w);
    for (int i = 0; i < M; ++i) {
      s2_ld(sS, xcs + ((long)j * M + i) * ws, w);
      s2_put(p2, a.ld2, i * w, sS, w);
    }
  }
}

// One CTA per (separator, strip): panel 2 of a fine separator, Q_p = V_p Xc_{cl,.} + W_p Xc_{cr,.}
__global__ void __launch_bounds__(kSep2Threads) k_sep2_q(Sep2Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.y + a.s0, p = blockIdx.x;
  const int w = a.w[s], K = a.P - 1, M = a.plan[0];
  if (p >= K) return;
  const int* pk = a.plan + kSep2PlanHdr + p * kSep2PlanStride;
  if (pk[0] != 0) return;   // coarse
  const int g = pk[2];
  const long ws = (long)a.wmax * a.wmax;
  cplx* sV = reinterpret_cast<cplx*>(smem_raw);
  cplx *sW = sV + ws, *sX = sW + ws, *sC = sX + ws;
  const cplx* xcs = a.xc + (long)s * (M * M + 3 * M) * ws;
  const cplx* v = a.vw + ((long)s * K + p) * 2 * ws;
  const bool hasl = g > 0, hasr = g < M;
  if (hasl) s2_ld(sV, v, w);
  if (hasr) s2_ld(sW, v + ws, w);
  cplx* p2 = s2_panel2(a, s, p, w);
  for (int i = 0; i < M; ++i) {
    bool any = false;
    if (hasl) { s2_ld(sX, xcs + ((long)(g - 1) * M + i) * ws, w); s2_mm(sC, sV, false, sX, false, w, 1.0, false); any = true; }
    if (hasr) { s2_ld(sX, xcs + ((long)g * M + i) * ws, w); s2_mm(sC, sW, false, sX, false, w, 1.0, any); any = true; }
    s2_put(p2, a.ld2, i * w, sC, w);
  }
}

// general block width (w > 36): generic smem Gauss-Jordan and matmuls
__global__ void k_reduced_generic(RedArgs ra) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.x + ra.s0;
  const int w = ra.w[s];
  const long w2 = (long)w * w;
  cplx* S = reinterpret_cast<cplx*>(smem_raw);
  cplx* colv = S + w * w;
  // gj_invert_blk needs the panel's pivot rows (8 w entries): used when the launch's shared memory holds them
  unsigned dsm;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsm));
  const bool gjblk = HELM_GJ_BLOCKED && dsm >= sizeof(cplx) * ((size_t)w * w + 9 * (size_t)w) + sizeof(int) * (w + 4) + 64;
  cplx* ybuf = gjblk ? colv + w : nullptr;
  double* redv = reinterpret_cast<double*>(colv + w + (gjblk ? 8 * w : 0));
  int* flag = reinterpret_cast<int*>(redv + 4);
  int* piv = flag + 4;
  const long band = (long)s * ra.nc * ra.wmax;
  const cplx* fac = ra.fac + ra.fac_off[s];
  cplx* red = ra.red + ra.red_off[s];
  cplx* Rprev = ra.rscratch + (long)s * 2 * ra.wmax * ra.wmax;  // R_{k-1,k}
  cplx* Tmp = Rprev + (long)ra.wmax * ra.wmax;
  auto Ub = [&](int c, int mode) { return Bidi{mode, ra.cr + band + (long)c * ra.wmax, ra.ne + band + (long)c * ra.wmax}; };
  auto scr = [&](int p) { return ra.scratch + ((long)s * ra.P + p) * ra.scratch_stride; };
  const int P = ra.P;
  for (int k = 0; k <= P - 2; ++k) {
    const int hk = ra.seg_hi[k];          // last row of segment k
    const int sk = hk + 1;                // separator row
    const int hk1 = ra.seg_hi[k + 1];     // last row of segment k+1
    cplx* Rinv = red + (long)k * 3 * w2;
    cplx* G = Rinv + w2;
    cplx* F = Rinv + 2 * w2;
    // R_kk = D_sk - U_hk^T X_k[hi,hi] U_hk - U_sk X_{k+1}[lo,lo] U_sk^T
    build_D(S, ra.dg + band + (long)sk * ra.wmax, ra.al + band + (long)sk * ra.wmax, w);
    blk_lxr(S, fac + (long)hk * w2, Ub(hk, BD_UT), Ub(hk, BD_U), w, -1.0, true);
    blk_lxr(S, scr(k + 1) + 2 * w2, Ub(sk, BD_U), Ub(sk, BD_UT), w, -1.0, true);
    if (k >= 1) {
      // - R_{k,k-1} Rinv_{k-1} R_{k-1,k} = - R_{k-1,k}^T F_{k-1}
      SETUP_MM(S, w, Rprev, w, true, red + (long)(k - 1) * 3 * w2 + 2 * w2, w, w, -1.0, true);
    }
    if (WIDE_GJ(S, w, piv, colv, ybuf, redv, flag)) {
      if (threadIdx.x == 0) atomicCAS(ra.status, 0, s * ra.nc + sk + 1);
      return;
    }
    blk_copy(Rinv, S, w);
    if (k >= 1) {
      // G_k = Rinv_k R_{k,k-1} = Rinv_k R_{k-1,k}^T  (Tmp = R_{k-1,k}^T)
      for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
        int p = e / w, q = e % w;
        Tmp[e] = Rprev[q * w + p];
      }
      __syncthreads();
      SETUP_MM(G, w, Rinv, w, false, Tmp, w, w, 1.0, false);
    }
    if (k <= P - 3) {
      // R_{k,k+1} = - U_sk X_{k+1}[lo,hi] U_{hk1}
      blk_lxr(Rprev, scr(k + 1) + 3 * w2, Ub(sk, BD_U), Ub(hk1, BD_U), w, -1.0, false);
      SETUP_MM(F, w, Rinv, w, false, Rprev, w, w, 1.0, false);
    }
  }
}

// ------------------------------------------------------------------ explicit separator inverse
// Rows of R^{-1} (R = the separator Schur complement, block tridiagonal with
// K = P-1 dense w x w blocks) for the register-streaming sweep kernel: the
// segment CTAs then obtain x_sep = R^{-1} g by a parallel dense mat-vec
// instead of a K-step dependent chain.  Computed from the block-Thomas
// factors (Rinv_k, G_k, F_k) applied to the identity, one CTA per
// (strip, column block j):  Z_j = Rinv_j E_j, Z_k = -G_k Z_{k-1} (k > j),
// X_{K-1} = Z_{K-1}, X_k = Z_k - F_k X_{k+1}.  Storage per strip:
// X[k] is w x (K w) row-major (the rows of separator k), contiguous.

#ifndef HELM_RINV_THREADS
#define HELM_RINV_THREADS 256   // C5 separator inverse per axis: 128: 1.43, 192: 1.33, 256: 1.17, 512: 1.20, 800: 1.23 ms
#endif
constexpr int kRinvThreads = HELM_RINV_THREADS;
template <int NT>
__global__ void __launch_bounds__(NT) k_reduced_inverse(RedArgs ra, cplx* xinv, const long* xinv_off) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.y + ra.s0, j = blockIdx.x;
  const int K = ra.P - 1;
  if (j >= K) return;
  const int w = ra.w[s];
  const long w2 = (long)w * w;
  const cplx* red = ra.red + ra.red_off[s];
  cplx* X = xinv + xinv_off[s];
  // three rotating w x w column blocks (current X_k / Z_k, next, prefetch target; leading
  // dimension lb) and a double-buffered factor block (leading dimension la), all staged
  // one step ahead with cp.async
  const int la = dmma_lda(w), lb = dmma_ldb(w);
  const long sb = (long)w * lb, sa = (long)w * la;
  cplx* vb[3] = {reinterpret_cast<cplx*>(smem_raw), reinterpret_cast<cplx*>(smem_raw) + sb,
                 reinterpret_cast<cplx*>(smem_raw) + 2 * sb};
  cplx* Mb = vb[2] + sb;
  const long ld = x_ld(K, w);   // row stride (128-byte aligned rows)
  auto blkX = [&](int k, int r, int c) -> cplx& { return X[((long)k * w + r) * ld + (long)j * w + c]; };
  const float invw = 1.0f / (float)w;   // e -> e / w by div_w (no integer division)
  auto rowof = [&](int e) { return div_w(e, invw); };
  auto mm = [&](cplx* C, const cplx* A, const cplx* B, bool acc) {
#if defined(HELM_RINV_ABL) && HELM_RINV_ABL == 1
    __syncthreads();   // ablation (timing only): no product
#else
    blk_mm_dmma(C, lb, A, la, false, B, lb, w, -1.0, acc);
#endif
  };
  auto stage_M = [&](int k, int which) {   // which = 1: G_k (forward), 2: F_k (backward)
    const cplx* G = red + ((long)k * 3 + which) * w2;
    cplx* d = Mb + (k & 1) * sa;
    for (int e = threadIdx.x; e < w2; e += NT) {
      const int r = rowof(e);
      cp_async16(d + r * la + (e - r * w), G + e);
    }
  };
  auto stage_Z = [&](int k, cplx* d) {
    for (int e = threadIdx.x; e < w2; e += NT) {
      const int r = rowof(e), c = e - r * w;
      cp_async16(d + r * lb + c, &blkX(k, r, c));
    }
  };
  auto store = [&](int k, const cplx* blk) {
    for (int e = threadIdx.x; e < w2; e += NT) {
      const int r = rowof(e), c = e - r * w;
      blkX(k, r, c) = blk[r * lb + c];
    }
  };
  // X = R^{-1} is complex symmetric (R is): this CTA forms the blocks (k, j),
  // k >= j, of its column block and mirrors them into (j, k), so the backward
  // recurrence stops at k = j (a third less work than the full column block)
  auto mirror = [&](int k, const cplx* blk) {   // block (j, k) = block(k, j)^T
    // consecutive threads write consecutive entries of a row of block (j, k) (coalesced;
    // the transposed reads are from shared memory)
    for (int e = threadIdx.x; e < w2; e += NT) {
      const int c = rowof(e), r = e - c * w;
      X[((long)j * w + c) * ld + (long)k * w + r] = blk[r * lb + c];
    }
  };
  // forward: k = j: Rinv_j; k > j: Z_k = -G_k Z_{k-1}
  if (j + 1 < K) { stage_M(j + 1, 1); cp_async_commit(); }
  int ic = 0;
  for (int e = threadIdx.x; e < w2; e += NT) {
    const cplx v = red[(long)j * 3 * w2 + e];
    const int r = rowof(e);
    vb[0][r * lb + (e - r * w)] = v;
    blkX(j, r, e - r * w) = v;
  }
  for (int k = j + 1; k < K; ++k) {
    cp_async_wait_all();
    __syncthreads();
    if (k + 1 < K) { stage_M(k + 1, 1); cp_async_commit(); }
    cplx* nx = vb[(ic + 1) % 3];
    mm(nx, Mb + (k & 1) * sa, vb[ic], false);
#if !(defined(HELM_RINV_ABL) && HELM_RINV_ABL == 2)
    store(k, nx);
#endif
    ic = (ic + 1) % 3;
  }
  // backward: vb[ic] holds X_{K-1}[:, j] = Z_{K-1}[:, j];  X_k = Z_k - F_k X_{k+1}, k >= j
  if (K - 1 > j) mirror(K - 1, vb[ic]);
  __syncthreads();   // every thread's forward stores precede the read-back
  if (K - 2 >= j) { stage_M(K - 2, 2); stage_Z(K - 2, vb[(ic + 1) % 3]); cp_async_commit(); }
  for (int k = K - 2; k >= j; --k) {
    cp_async_wait_all();
    __syncthreads();
    cplx* z = vb[(ic + 1) % 3];
    if (k - 1 >= j) { stage_M(k - 1, 2); stage_Z(k - 1, vb[(ic + 2) % 3]); cp_async_commit(); }
    mm(z, Mb + (k & 1) * sa, vb[ic], true);
#if !(defined(HELM_RINV_ABL) && HELM_RINV_ABL == 2)
    store(k, z);
    if (k > j) mirror(k, z);
#endif
    ic = (ic + 1) % 3;
  }
}

// Wide strips (w > 36): the same recurrences with every block in global memory
// (a w = 99 block is 157 KB, beyond shared memory).  Column block j of X is
// formed in place in the X rows: Z_j = Rinv_j, Z_k = -G_k Z_{k-1} (k > j), then
// X_k = Z_k - F_k X_{k+1} (k < K-1); the products are 4x4 register-tiled with
// operands from L1/L2.  The CTA only reads blocks it wrote itself (same SM: the
// write-through L1 stays coherent after the barrier ending each product).
__global__ void __launch_bounds__(512, 1) k_reduced_inverse_glb(RedArgs ra, cplx* xinv, const long* xinv_off) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = blockIdx.y + ra.s0, j = blockIdx.x;
  const int K = ra.P - 1;
  if (j >= K) return;
  const int w = ra.w[s];
  const long w2 = (long)w * w;
  const cplx* red = ra.red + ra.red_off[s];
  cplx* X = xinv + xinv_off[s];
  const long ld = x_ld(K, w);
  auto blk = [&](int k) { return X + (long)k * w * ld + (long)j * w; };   // block (k, j), row stride ld
  // the products stage their operands in shared memory (the factor block whole, the column
  // block in panels of 32 columns) when the launch provides it; straight from L1 / L2 the
  // tensor pipe ran at 0.23 of its peak (every warp re-reads its operand rows and columns)
  unsigned dsm;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsm));
  const bool staged = dsm >= sizeof(cplx) * (size_t)w * (dmma_lda(w) + kDmmaPanelLd);
  cplx* sA = reinterpret_cast<cplx*>(smem_raw);
  cplx* sB = sA + (long)w * dmma_lda(w);
  auto mm = [&](cplx* C, const cplx* A, const cplx* B, bool acc) {
    if (staged) blk_mm_dmma_staged(C, (int)ld, A, w, B, (int)ld, w, -1.0, acc, sA, sB);
    else SETUP_MM(C, (int)ld, A, w, false, B, (int)ld, w, -1.0, acc);
  };
  // blocks (k, j), k >= j, mirrored into (j, k) (X is symmetric; see k_reduced_inverse)
  auto mirror = [&](int k) {
    __syncthreads();
    const cplx* b = blk(k);
    for (long e = threadIdx.x; e < w2; e += blockDim.x) {   // (coalesced writes, strided L1/L2 reads)
      const long c = e / w, r = e % w;
      X[((long)j * w + c) * ld + (long)k * w + r] = b[r * ld + c];
    }
  };
  for (long e = threadIdx.x; e < w2; e += blockDim.x) blk(j)[(e / w) * ld + e % w] = red[(long)j * 3 * w2 + e];
  __syncthreads();
  for (int k = j + 1; k < K; ++k) mm(blk(k), red + ((long)k * 3 + 1) * w2, blk(k - 1), false);
  if (K - 1 > j) mirror(K - 1);
  for (int k = K - 2; k >= j; --k) {
    mm(blk(k), red + ((long)k * 3 + 2) * w2, blk(k + 1), true);
    if (k > j) mirror(k);
  }
}

// ------------------------------------------------------------------ host
// Segments per strip: the largest P <= 33 whose segments have >= 8 cross rows
// (C5, t = 4, 128-byte aligned separator-inverse rows: P = 29..37 measured 4.35,
// 4.32, 4.11, 4.19, 4.05, 4.20, 4.13, 4.12, 4.11 ms per apply -- 33 is the best,
// and 4 directions x 33 segments = 132 CTAs fit the 148 SMs; C2: 16 / 24 / 32
// segments 0.56 / 0.50 / 0.53 ms -- more, shorter segments pay while the
// separator system stays small).
#ifndef HELM_SEG_EXTRA
#define HELM_SEG_EXTRA 0   // where the segments with one more row go (0 first, 1 last, 2 middle)
#endif
static int choose_segments(int nc, int requested, int wmax) {
  if (requested > 0) return requested;
  // two-chain kernel (w <= 36): t = 4 batches of 36 segment CTAs fill 144 of the 148 SMs
  // (C5 t = 4 apply: P = 33 3.83, 36 3.75, 37 3.81 ms); wider strips (general kernel,
  // explicit separator rows formed in global memory) keep 33
  int P = wmax <= 36 ? 36 : 33;
  while (P > 1 && (nc - (P - 1)) / P < 8) --P;
  return P;
}

extern "C" int sweep_setup(helm_problem_t prob, int axis, int order, int n_strips, int overlap,
                           int is_double, int gather, int n_segments, void* stream, helm_sweep_t* out) {
  if (!prob || !out) { helm_set_error("sweep_setup: null argument"); return HELM_EINVAL; }
  *out = nullptr;
  if ((axis != 0 && axis != 1) || (order != 0 && order != 1) || n_strips < 1 || overlap < 0 ||
      (gather != 0 && gather != 1) || n_segments < 0) {
    helm_set_error("sweep_setup: bad axis/order/n_strips/overlap/gather/n_segments");
    return HELM_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n_axis = axis == 0 ? prob->nx : prob->ny;
  const int nc = (axis == 0 ? prob->ny : prob->nx) + 1;
  // partition lines p_0 = 0 < ... < p_N = n_axis, larger runs first (D6, A12)
  std::vector<int> pl(n_strips + 1, 0);
  int base = n_axis / n_strips, extra = n_axis % n_strips;
  for (int s = 0; s < n_strips; ++s) pl[s + 1] = pl[s] + base + (s < extra ? 1 : 0);
  if (n_strips > 1 && base < std::max(2 * overlap + 1, 2)) {
    helm_set_error("sweep_setup: strips of %d cells are too thin for overlap %d (need >= %d)", base,
                   overlap, std::max(2 * overlap + 1, 2));
    return HELM_EINVAL;
  }
  if (n_strips > n_axis) { helm_set_error("sweep_setup: more strips than cells"); return HELM_EINVAL; }
  if (prob->disc == HELM_DISC_FD5 && n_strips > 1 && overlap < 1) {
    // the FD5 transmission data use the centred difference across the interface
    // line, i.e. the neighbour's values one line inside this strip
    helm_set_error("sweep_setup: the five-point scheme needs overlap >= 1");
    return HELM_EINVAL;
  }
  helm_sweep_s* h = new helm_sweep_s();
  h->prob = prob;
  h->axis = axis; h->order = order; h->N = n_strips; h->overlap = overlap;
  h->is_double = is_double ? 1 : 0; h->gather = gather; h->nc = nc;
  h->disc = prob->disc;
  h->a.resize(n_strips); h->b.resize(n_strips); h->w.resize(n_strips);
  h->own_lo.resize(n_strips); h->own_hi.resize(n_strips);
  int wmax = 0;
  for (int s = 0; s < n_strips; ++s) {
    h->a[s] = std::max(pl[s] - overlap, 0);
    h->b[s] = std::min(pl[s + 1] + overlap, n_axis);
    h->w[s] = h->b[s] - h->a[s] + 1;
    wmax = std::max(wmax, h->w[s]);
    if (gather == 0) {
      h->own_lo[s] = 0; h->own_hi[s] = h->w[s] - 1;
    } else {  // core: lines p_s .. p_{s+1}-1 (last strip also p_N)
      h->own_lo[s] = pl[s] - h->a[s];
      h->own_hi[s] = (s == n_strips - 1 ? pl[s + 1] : pl[s + 1] - 1) - h->a[s];
    }
  }
  h->wmax = wmax;
  {
    // the generic (w > 36) factorisation holds one w x w block in shared memory
    const size_t need = sizeof(cplx) * ((size_t)wmax * wmax + wmax) + sizeof(int) * (wmax + 4) + 64;
    if (wmax > kRowW && need > 227u * 1024u) {
      helm_set_error("sweep_setup: strips of %d nodes exceed the factorisation's shared-memory block (max 119); "
                     "use more strips", wmax);
      delete h;
      return HELM_EINVAL;
    }
  }
  int P = choose_segments(nc, n_segments, wmax);
  if (P < 1 || nc - (P - 1) < P) {
    helm_set_error("sweep_setup: %d segments do not fit %d cross rows", P, nc);
    delete h;
    return HELM_EINVAL;
  }
  h->P = P;
  {
    int rows = nc - (P - 1), sb = rows / P, se = rows % P, c = 0;
    for (int p = 0; p < P; ++p) {
#if HELM_SEG_EXTRA == 1
      int m = sb + (p >= P - se ? 1 : 0);                 // the longer segments last
#elif HELM_SEG_EXTRA == 2
      int m = sb + ((p >= (P - se) / 2 && p < (P - se) / 2 + se) ? 1 : 0);   // in the middle
#else
      int m = sb + (p < se ? 1 : 0);
#endif
      h->seg_lo.push_back(c);
      h->seg_hi.push_back(c + m - 1);
      c += m + 1;  // skip the separator row
    }
  }
  // factor storage
  h->fac_off.resize(n_strips);
  h->red_off.resize(n_strips);
  long fac_total = 0, red_total = 0;
  for (int s = 0; s < n_strips; ++s) {
    h->fac_off[s] = fac_total;
    fac_total += (long)nc * h->w[s] * h->w[s];
    h->red_off[s] = red_total;
    red_total += (long)std::max(P - 1, 0) * 3 * h->w[s] * h->w[s];
  }
  const long bandN = (long)n_strips * nc * wmax;
  h->factor_bytes = (fac_total + red_total) * (long)sizeof(cplx);
  cudaError_t e = cudaSuccess;
  auto alloc = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = helm_dev_alloc(p, bytes);
  };
  // explicit separator-inverse offsets (register-streaming kernel only)
  // wide strips (w > 36): explicit separator-inverse rows too (formed in global
  // memory), used by the general kernel's segments instead of its reducer CTA's
  // sequential separator solve (C4: 19.1 -> 12.5 ms per t = 4 apply for +24 ms of
  // setup per axis); the no_wide_xinv knob keeps the reducer path
  const bool wide_xinv = wmax > kXinvMaxW && !helm_knob(KNOB_NO_WIDE_XINV);
  const bool want_xinv = P > 1 && (wmax <= kXinvMaxW || wide_xinv);
  // bottom-up inverses for the two-chain kernel (sweep_dual.cu): row factorisation only
  const bool want_fac2 = want_xinv && wmax <= kRowW && !helm_knob(KNOB_FACTOR_GENERIC);
  (void)wide_xinv;
  long pfac_total = 0;
  h->pfac_off.resize(n_strips);
  for (int s2 = 0; s2 < n_strips; ++s2) {
    h->pfac_off[s2] = pfac_total;
    pfac_total += (long)nc * pk_size(h->w[s2]);
  }
  if (want_fac2) h->factor_bytes += 2 * pfac_total * (long)sizeof(cplx);
  long xinv_total = 0;
  if (want_xinv) {
    h->xinv_off.resize(n_strips);
    for (int s2 = 0; s2 < n_strips; ++s2) {
      h->xinv_off[s2] = xinv_total;
      xinv_total += (long)(P - 1) * h->w[s2] * x_ld(P - 1, h->w[s2]);
    }
  }
  // two-level separator solve (k_sweep_dual): group / coarse plan and panel sizes
  const int Ksep = P - 1;
  // (opt-in, sep_two_level knob: parity-tested, measured slower than the full rows on C5 --
  // two dependent latency-bound rounds and a coarse barrier instead of one HBM-bound
  // mat-vec)
  const bool want_sep2 = want_fac2 && Ksep >= 8 && Ksep <= 80 && helm_knob(KNOB_SEP_TWO_LEVEL);
  std::vector<int> plan;
  int M2 = 0, ngr2 = 0, nbmax2 = 0, nb1max2 = 0;
  long sep2_total = 0;
  if (want_sep2) {
    M2 = std::max(1, (int)std::lround(std::sqrt(Ksep + 1.0)) - 1);
    while ((Ksep - M2 + M2) / (M2 + 1) > kSep2MaxB && M2 < 8) ++M2;   // ceil((K - M) / (M + 1)) <= kSep2MaxB
    ngr2 = M2 + 1;
    const int fine = Ksep - M2, base = fine / ngr2, extra = fine % ngr2;
    plan.assign(kSep2PlanHdr + Ksep * kSep2PlanStride, 0);
    plan[0] = M2;
    plan[1] = ngr2;
    std::vector<int> gs(ngr2), gl(ngr2);
    for (int g2 = 0, k = 0; g2 < ngr2; ++g2) {
      gl[g2] = base + (g2 < extra ? 1 : 0);
      gs[g2] = k;
      plan[8 + g2] = gs[g2];
      plan[32 + g2] = gl[g2];
      nbmax2 = std::max(nbmax2, gl[g2]);
      for (int l = 0; l < gl[g2]; ++l) {   // fine separators of group g2
        int* pk = &plan[kSep2PlanHdr + (k + l) * kSep2PlanStride];
        pk[0] = 0; pk[1] = gl[g2]; pk[2] = g2;
        for (int j = 0; j < gl[g2]; ++j) pk[4 + j] = k + j;
      }
      k += gl[g2];
      if (g2 < M2) {   // coarse separator g2 at k: both adjacent groups
        int* pk = &plan[kSep2PlanHdr + k * kSep2PlanStride];
        pk[0] = 1; pk[2] = g2;
        k += 1;
      }
    }
    for (int j = 0; j < M2; ++j) {
      const int c = gs[j + 1] - 1;
      int* pk = &plan[kSep2PlanHdr + c * kSep2PlanStride];
      pk[1] = gl[j] + gl[j + 1];
      for (int l = 0; l < gl[j]; ++l) pk[4 + l] = gs[j] + l;
      for (int l = 0; l < gl[j + 1]; ++l) pk[4 + gl[j] + l] = gs[j + 1] + l;
      nb1max2 = std::max(nb1max2, pk[1]);
    }
    nb1max2 = std::max(nb1max2, nbmax2);
    plan[2] = nb1max2;
    h->sep2_M = M2;
    h->sep2_ld1 = (nb1max2 * wmax + 7) / 8 * 8;
    h->sep2_ld2 = (M2 * wmax + 7) / 8 * 8;
    h->sep2_off.resize(n_strips);
    for (int s2 = 0; s2 < n_strips; ++s2) {
      h->sep2_off[s2] = sep2_total;
      sep2_total += (long)Ksep * h->w[s2] * (h->sep2_ld1 + h->sep2_ld2);
    }
    h->factor_bytes += sep2_total * (long)sizeof(cplx);
  }
  SharedFactors* sf = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_shared_mu);
    for (SharedFactors* c : g_shared)
      if (c->prob_uid == prob->uid && c->axis == axis && c->N == n_strips && c->overlap == overlap && c->P == P) sf = c;
    if (sf) sf->refs++;   // taken under the lock; released by sweep_destroy
  }
  h->shared = sf;
  h->d_a = h->d_w = h->d_own_lo = h->d_own_hi = h->d_seg_lo = h->d_seg_hi = nullptr;
  h->d_dg = h->d_al = h->d_cr = h->d_ne = h->d_tc = h->d_fac = h->d_red = nullptr;
  h->d_fac_off = h->d_red_off = nullptr;
  h->d_xinv = nullptr;
  h->d_xinv_off = nullptr;
  h->d_fac2 = nullptr;
  h->d_facp = nullptr;
  h->d_pfac_off = nullptr;
  alloc((void**)&h->d_a, sizeof(int) * n_strips);
  alloc((void**)&h->d_w, sizeof(int) * n_strips);
  alloc((void**)&h->d_own_lo, sizeof(int) * n_strips);
  alloc((void**)&h->d_own_hi, sizeof(int) * n_strips);
  alloc((void**)&h->d_seg_lo, sizeof(int) * P);
  alloc((void**)&h->d_seg_hi, sizeof(int) * P);
  alloc((void**)&h->d_fac_off, sizeof(long) * n_strips);
  alloc((void**)&h->d_pfac_off, sizeof(long) * n_strips);
  alloc((void**)&h->d_red_off, sizeof(long) * n_strips);
  if (want_xinv) alloc((void**)&h->d_xinv_off, sizeof(long) * n_strips);
  if (want_sep2) alloc((void**)&h->d_sep2_off, sizeof(long) * n_strips);
  if (!sf) {
    if (want_sep2) alloc((void**)&h->d_sep2, sizeof(cplx) * sep2_total);
    if (want_sep2) alloc((void**)&h->d_sep2_plan, sizeof(int) * plan.size());
    alloc((void**)&h->d_dg, sizeof(cplx) * bandN);
    alloc((void**)&h->d_al, sizeof(cplx) * bandN);
    alloc((void**)&h->d_cr, sizeof(cplx) * bandN);
    alloc((void**)&h->d_ne, sizeof(cplx) * bandN);
    alloc((void**)&h->d_tc, sizeof(cplx) * n_strips * 2 * nc * kTcW);
    alloc((void**)&h->d_fac, sizeof(cplx) * fac_total);
    alloc((void**)&h->d_red, sizeof(cplx) * std::max(red_total, 1L));
    if (want_xinv) alloc((void**)&h->d_xinv, sizeof(cplx) * xinv_total);
    if (want_fac2) alloc((void**)&h->d_fac2, sizeof(cplx) * pfac_total);
    if (want_fac2) alloc((void**)&h->d_facp, sizeof(cplx) * pfac_total);
  }
  if (e != cudaSuccess) {
    helm_set_error("sweep_setup: cudaMalloc (%.2f GB factors): %s", h->factor_bytes / 1e9, cudaGetErrorString(e));
    sweep_destroy(h);
    return HELM_ENOMEM;
  }
  auto h2d = [&](void* d, const void* s, size_t bytes) {
    if (e == cudaSuccess) e = cudaMemcpyAsync(d, s, bytes, cudaMemcpyHostToDevice, st);
  };
  h2d(h->d_a, h->a.data(), sizeof(int) * n_strips);
  h2d(h->d_w, h->w.data(), sizeof(int) * n_strips);
  h2d(h->d_own_lo, h->own_lo.data(), sizeof(int) * n_strips);
  h2d(h->d_own_hi, h->own_hi.data(), sizeof(int) * n_strips);
  h2d(h->d_seg_lo, h->seg_lo.data(), sizeof(int) * P);
  h2d(h->d_seg_hi, h->seg_hi.data(), sizeof(int) * P);
  h2d(h->d_fac_off, h->fac_off.data(), sizeof(long) * n_strips);
  h2d(h->d_pfac_off, h->pfac_off.data(), sizeof(long) * n_strips);
  h2d(h->d_red_off, h->red_off.data(), sizeof(long) * n_strips);
  if (want_xinv) h2d(h->d_xinv_off, h->xinv_off.data(), sizeof(long) * n_strips);
  if (want_sep2) h2d(h->d_sep2_off, h->sep2_off.data(), sizeof(long) * n_strips);
  if (want_sep2 && !sf) h2d(h->d_sep2_plan, plan.data(), sizeof(int) * plan.size());
  if (e != cudaSuccess) {
    helm_set_error("sweep_setup: copy geometry: %s", cudaGetErrorString(e));
    sweep_destroy(h);
    return HELM_ECUDA;
  }
  if (sf) {
    // same strips already factored: share the device factor set
    h->d_dg = sf->dg; h->d_al = sf->al; h->d_cr = sf->cr; h->d_ne = sf->ne; h->d_tc = sf->tc;
    h->d_fac = sf->fac; h->d_red = sf->red; h->d_xinv = sf->xinv; h->d_fac2 = sf->fac2; h->d_facp = sf->facp;
    h->d_sep2 = sf->sep2; h->d_sep2_plan = sf->sep2_plan;
    if (!h->d_sep2) { helm_dev_free(h->d_sep2_off); h->d_sep2_off = nullptr; h->sep2_M = 0; }
    h->factor_bytes = sf->factor_bytes;
    h->xinv_elems = sf->xinv_elems;
    h->shared = sf;
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      helm_set_error("sweep_setup: %s", cudaGetErrorString(e));
      sweep_destroy(h);
      return HELM_ECUDA;
    }
    *out = h;
    return HELM_OK;
  }
  GridView g{prob->nx, prob->ny, prob->h, prob->omega, prob->c};
  StripGeo sg{h->d_a, h->d_w, n_strips, nc, wmax, axis};
  const bool timing = helm_knob(KNOB_SETUP_TIMING) != 0;
  cudaEvent_t tev[6];
  if (timing) {
    for (auto& x : tev) cudaEventCreate(&x);
    cudaEventRecord(tev[0], st);
  }
  {
    dim3 grid((nc * wmax + 255) / 256, n_strips);
    if (prob->disc == HELM_DISC_FD5)
      k_strip_bands_fd5<<<grid, 256, 0, st>>>(g, sg, h->d_dg, h->d_al, h->d_cr, h->d_ne, h->d_tc);
    else
      k_strip_bands<<<grid, 256, 0, st>>>(g, sg, h->d_dg, h->d_al, h->d_cr, h->d_ne, h->d_tc);
    HELM_LAUNCH_CHECK();
  }
  // factorisation
  int* d_status = nullptr;
  cplx* scratch = nullptr;
  cplx* rscratch = nullptr;
  const long sstride = 4L * wmax * wmax;
  if (e == cudaSuccess) e = helm_dev_alloc((void**)&d_status, sizeof(int));
  if (e == cudaSuccess) e = cudaMemsetAsync(d_status, 0, sizeof(int), st);
  if (P > 1) {
    alloc((void**)&scratch, sizeof(cplx) * sstride * n_strips * P);
    alloc((void**)&rscratch, sizeof(cplx) * 2L * wmax * wmax * n_strips);
  }
  const long ws2 = (long)wmax * wmax;
  const long ytmp_stride = (2L * kSep2MaxB + (long)nbmax2 * nbmax2) * ws2;
  cplx *rraw = nullptr, *ytmp = nullptr, *vw = nullptr, *cdm = nullptr, *xcm = nullptr;
  if (want_sep2) {
    alloc((void**)&rraw, sizeof(cplx) * (long)n_strips * Ksep * 2 * ws2);
    alloc((void**)&ytmp, sizeof(cplx) * (long)n_strips * ngr2 * ytmp_stride);
    alloc((void**)&vw, sizeof(cplx) * (long)n_strips * Ksep * 2 * ws2);
    alloc((void**)&cdm, sizeof(cplx) * (long)n_strips * M2 * 3 * ws2);
    alloc((void**)&xcm, sizeof(cplx) * (long)n_strips * (M2 * M2 + 3 * M2) * ws2);
  }
  if (e != cudaSuccess) {
    helm_set_error("sweep_setup: scratch: %s", cudaGetErrorString(e));
    helm_dev_free(d_status); helm_dev_free(scratch); helm_dev_free(rscratch);
    helm_dev_free(rraw); helm_dev_free(ytmp); helm_dev_free(vw); helm_dev_free(cdm); helm_dev_free(xcm);
    sweep_destroy(h);
    return HELM_ENOMEM;
  }
  size_t smem = sizeof(cplx) * ((size_t)wmax * wmax + 9 * (size_t)wmax) + sizeof(int) * (wmax + 4) + 64;   // blocked Gauss-Jordan
  if (smem > 227u * 1024u) smem = sizeof(cplx) * ((size_t)wmax * wmax + wmax) + sizeof(int) * (wmax + 4) + 64;   // w > 115: unblocked
  cudaFuncSetAttribute(k_factor_segments, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_reduced_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int threads = wmax * wmax >= 1024 ? 512 : 256;
  FacArgs fa{h->d_w, h->d_fac_off, h->d_seg_lo, h->d_seg_hi, h->d_dg, h->d_al, h->d_cr, h->d_ne,
             nc, wmax, P, h->d_fac, scratch, sstride, d_status, h->d_fac2, h->d_facp, h->d_pfac_off};
  RedArgs ra{h->d_w, h->d_fac_off, h->d_red_off, h->d_seg_lo, h->d_seg_hi, h->d_dg, h->d_al, h->d_cr,
             h->d_ne, nc, wmax, P, h->d_fac, scratch, sstride, h->d_red, rscratch, d_status};
  ra.rraw = rraw;
  Sep2Args sa{h->d_w, wmax, P, 0, rraw, h->d_sep2_plan, ytmp, ytmp_stride, vw, cdm, xcm,
              h->d_sep2, h->d_sep2_off, h->sep2_ld1, h->sep2_ld2, d_status};
  if (want_sep2) {
    cudaFuncSetAttribute(k_sep2_group, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(5 * ws2 * sizeof(cplx)));
    cudaFuncSetAttribute(k_sep2_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * ws2 * sizeof(cplx)));
    cudaFuncSetAttribute(k_sep2_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * ws2 * sizeof(cplx)));
  }
  const size_t smr = sizeof(cplx) * (9 * (size_t)wmax * wmax + 12 * (size_t)wmax);
  const size_t sm3 = sizeof(cplx) * (size_t)wmax * (3 * dmma_ldb(wmax) + 2 * dmma_lda(wmax));
  if (P > 1 && wmax <= kRowW) cudaFuncSetAttribute(k_reduced, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
  if (P > 1 && want_xinv && wmax <= kXinvMaxW)
    cudaFuncSetAttribute(k_reduced_inverse<kRinvThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
  const bool rows_kernel = wmax <= kRowW && !helm_knob(KNOB_FACTOR_GENERIC);
  // strips [s0, s0 + ns): segment factors, separator factors, separator-inverse rows
  auto run_chunk = [&](cudaStream_t cs, int s0, int ns, cudaEvent_t fac_done) {
    FacArgs fc = fa;
    fc.s0 = s0;
    if (timing) cudaEventRecord(tev[1], cs);
    if (rows_kernel)
      k_factor_rows<<<dim3(P, ns, 2), kRowThreads, 0, cs>>>(fc);
    else
      k_factor_segments<<<dim3(P, ns), threads, smem, cs>>>(fc);
    if (fac_done) cudaEventRecord(fac_done, cs);
    if (timing) cudaEventRecord(tev[2], cs);
    g_helm_launches++;
    cudaError_t e2 = cudaGetLastError();
    if (e2 == cudaSuccess && P > 1) {
      RedArgs rc = ra;
      rc.s0 = s0;
      if (wmax <= kRowW) k_reduced<<<ns, kRedThreads, smr, cs>>>(rc);
      else k_reduced_generic<<<ns, threads, smem, cs>>>(rc);
      if (timing) cudaEventRecord(tev[3], cs);
      g_helm_launches++;
      e2 = cudaGetLastError();
      if (e2 == cudaSuccess && want_sep2) {
        Sep2Args sc = sa;
        sc.s0 = s0;
        k_sep2_group<<<dim3(ngr2, ns), kSep2Threads, 5 * ws2 * sizeof(cplx), cs>>>(sc);
        k_sep2_coarse<<<ns, kSep2Threads, 4 * ws2 * sizeof(cplx), cs>>>(sc);
        k_sep2_q<<<dim3(Ksep, ns), kSep2Threads, 4 * ws2 * sizeof(cplx), cs>>>(sc);
        g_helm_launches += 3;
        e2 = cudaGetLastError();
      }
      if (e2 == cudaSuccess && want_xinv) {
        // explicit separator inverse rows for the register-streaming kernel
        // (128 threads: 256 measured slower, round 1)
        if (wmax > kXinvMaxW) {
          size_t smg = sizeof(cplx) * (size_t)wmax * (dmma_lda(wmax) + kDmmaPanelLd);   // staged operands
          if (smg > 227u * 1024u) smg = 0;
          else cudaFuncSetAttribute(k_reduced_inverse_glb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smg);
          k_reduced_inverse_glb<<<dim3(P - 1, ns), 512, smg, cs>>>(rc, h->d_xinv, h->d_xinv_off);
        }
        else k_reduced_inverse<kRinvThreads><<<dim3(P - 1, ns), kRinvThreads, sm3, cs>>>(rc, h->d_xinv, h->d_xinv_off);
        if (timing) cudaEventRecord(tev[4], cs);
        g_helm_launches++;
        e2 = cudaGetLastError();
      }
    }
    if (e == cudaSuccess) e = e2;
  };
  // Optional (setup_chunks knob): the strips pipelined in chunks on forked
  // streams, chunk c + 1's segment factors starting when chunk c's are done, so
  // that chunk c's separator chain (long latency, one CTA per strip) runs beside
  // them.  Measured slower on C5 (both axes: 1 chunk 15.8 ms, 2: 16.9, 4: 18.5,
  // 8: 23.9) -- a chunk's segment factors are one long partial wave -- so the
  // default is one pass.
  int nchunk = helm_knob(KNOB_SETUP_CHUNKS);
  if (nchunk <= 0) nchunk = 1;
  if (timing) nchunk = 1;
  nchunk = std::min(std::min(nchunk, n_strips), 8);
  if (nchunk == 1) {
    run_chunk(st, 0, n_strips, nullptr);
  } else {
    // per host thread (the two axes are set up from two threads concurrently)
    thread_local cudaStream_t cs[8] = {};
    thread_local cudaEvent_t ev_fac[8] = {}, ev_done[8] = {}, ev_fork = nullptr;
    if (!ev_fork) {
      for (int c = 0; c < 8; ++c) {
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs[c], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_fac[c], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_done[c], cudaEventDisableTiming);
      }
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev_fork, st);
    for (int c = 0; c < nchunk && e == cudaSuccess; ++c) {
      const int s0 = (int)((long)n_strips * c / nchunk), s1 = (int)((long)n_strips * (c + 1) / nchunk);
      cudaStreamWaitEvent(cs[c], ev_fork, 0);
      if (c > 0) cudaStreamWaitEvent(cs[c], ev_fac[c - 1], 0);
      run_chunk(cs[c], s0, s1 - s0, ev_fac[c]);
      cudaEventRecord(ev_done[c], cs[c]);
      cudaStreamWaitEvent(st, ev_done[c], 0);
    }
  }
  if (P > 1 && want_xinv) h->factor_bytes += xinv_total * (long)sizeof(cplx);
  // wait for this setup's kernels first, then read the status: a pageable copy
  // issued while the stream is busy blocks inside the driver and serialises
  // setups running concurrently on other streams / host threads
  int status = 0;
  {
    // always drain this setup's stream before the scratch buffers are freed below,
    // also after a launch error (kernels queued earlier may still use them)
    const cudaError_t es = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = es;
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (timing && e == cudaSuccess) {
    float t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    cudaEventElapsedTime(&t1, tev[0], tev[1]);
    cudaEventElapsedTime(&t2, tev[1], tev[2]);
    if (P > 1) cudaEventElapsedTime(&t3, tev[2], tev[3]);
    if (P > 1 && want_xinv) cudaEventElapsedTime(&t4, tev[3], tev[4]);
    fprintf(stderr, "[sweep_setup] bands %.2f ms, segment factors %.2f ms, separator factors %.2f ms, separator inverse %.2f ms\n",
            t1, t2, t3, t4);
    long long rp[8];
    if (cudaMemcpyFromSymbol(rp, g_red_prof, sizeof(rp)) == cudaSuccess && P > 1) {
      fprintf(stderr, "[k_reduced] per separator (block 0): build+RtF %lld, invert %lld, store+G+F %lld cycles"
              " | per pivot: search %lld, publish %lld, update %lld\n",
              rp[0] / (P - 1), rp[1] / (P - 1), rp[2] / (P - 1), rp[3] / ((P - 1) * (long long)wmax),
              rp[4] / ((P - 1) * (long long)wmax), rp[5] / ((P - 1) * (long long)wmax));
      long long z[8] = {0};
      cudaMemcpyToSymbol(g_red_prof, z, sizeof(z));
    }
  }
  helm_dev_free(d_status);
  helm_dev_free(scratch);
  helm_dev_free(rscratch);
  helm_dev_free(rraw); helm_dev_free(ytmp); helm_dev_free(vw); helm_dev_free(cdm); helm_dev_free(xcm);
  if (e != cudaSuccess) {
    helm_set_error("sweep_setup: factorisation kernel: %s", cudaGetErrorString(e));
    sweep_destroy(h);
    return HELM_ECUDA;
  }
  if (status < 0) {
    helm_set_error("sweep_setup: zero pivot in the two-level separator system of strip %d", (-status - 1) / 1024);
    sweep_destroy(h);
    return HELM_ESINGULAR;
  }
  if (status != 0) {
    int s = (status - 1) / nc, c = (status - 1) % nc;
    helm_set_error("sweep_setup: zero pivot in strip %d, cross row %d", s, c);
    sweep_destroy(h);
    return HELM_ESINGULAR;
  }
  sf = new SharedFactors{1, prob->uid, axis, n_strips, overlap, P, h->d_dg, h->d_al, h->d_cr, h->d_ne, h->d_tc,
                         h->d_fac, h->d_red, h->d_xinv, h->d_fac2, h->d_facp, h->factor_bytes};
  sf->xinv_elems = h->xinv_elems = want_xinv ? xinv_total : 0;
  sf->sep2 = h->d_sep2; sf->sep2_plan = h->d_sep2_plan;
  sf->sep2_M = h->sep2_M; sf->sep2_ld1 = h->sep2_ld1; sf->sep2_ld2 = h->sep2_ld2;
  {
    std::lock_guard<std::mutex> lk(g_shared_mu);
    g_shared.push_back(sf);
  }
  h->shared = sf;
  *out = h;
  return HELM_OK;
}

extern "C" int sweep_info(helm_sweep_t h, long* info) {
  if (!h || !info) return HELM_EINVAL;
  info[0] = h->N;
  info[1] = h->nc;
  info[2] = h->wmax;
  info[3] = h->P;
  long solves = h->is_double ? 2L * h->N - 1 : h->N;
  info[4] = solves;
  info[5] = h->factor_bytes;
  // model bytes: per local solve 16 (2 n_c w^2 + 3 n_c w), summed
  // over the solves of one apply (strip sigma_N is solved once).
  // the strip solved once is sigma_N (order 0: strip N-1; order 1: strip 0)
  double model = 0.0;
  for (int s = 0; s < h->N; ++s) {
    double w = h->w[s];
    double per = 16.0 * (2.0 * h->nc * w * w + 3.0 * h->nc * w);
    int last = h->order == 0 ? h->N - 1 : 0;
    model += per * ((h->is_double && s != last) ? 2.0 : 1.0);
  }
  info[6] = (long)model;
  info[7] = h->axis;
  info[8] = h->order;
  info[9] = h->is_double;
  return HELM_OK;
}

// ------------------------------------------------------------------ inexact separator solve
__global__ void k_to_c64(const cplx* __restrict__ x, float2* __restrict__ y, long n) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
    y[e] = make_float2((float)x[e].x, (float)x[e].y);
}

extern "C" int sweep_set_precision(helm_sweep_t h, int separator_bits) {
  if (!h || (separator_bits != 32 && separator_bits != 64)) {
    helm_set_error("sweep_set_precision: need a handle and 32 or 64 separator bits");
    return HELM_EINVAL;
  }
  if (separator_bits == 64) { h->sep_fp32 = 0; return HELM_OK; }
  if (!h->d_xinv || h->xinv_elems <= 0) {
    helm_set_error("sweep_set_precision: this sweep has no explicit separator-inverse rows (P = 1)");
    return HELM_EINVAL;
  }
  SharedFactors* sf = h->shared;
  std::lock_guard<std::mutex> lk(g_shared_mu);
  if (!sf->xinv32) {
    float2* y = nullptr;
    cudaError_t e = helm_dev_alloc((void**)&y, sizeof(float2) * h->xinv_elems);
    cudaStream_t st = nullptr;
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
      k_to_c64<<<148 * 8, 256, 0, st>>>(h->d_xinv, y, h->xinv_elems);
      g_helm_launches++;
      e = cudaGetLastError();
      const cudaError_t es = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = es;
      cudaStreamDestroy(st);
    }
    if (e != cudaSuccess) {
      helm_dev_free(y);
      helm_set_error("sweep_set_precision: %s", cudaGetErrorString(e));
      return e == cudaErrorMemoryAllocation ? HELM_ENOMEM : HELM_ECUDA;
    }
    sf->xinv32 = y;
  }
  h->d_xinv32 = sf->xinv32;
  h->sep_fp32 = 1;
  return HELM_OK;
}

extern "C" void sweep_destroy(helm_sweep_t h) {
  if (!h) return;
  helm_dev_free(h->d_a); helm_dev_free(h->d_w); helm_dev_free(h->d_own_lo); helm_dev_free(h->d_own_hi);
  helm_dev_free(h->d_seg_lo); helm_dev_free(h->d_seg_hi); helm_dev_free(h->d_fac_off);
  helm_dev_free(h->d_pfac_off);
  helm_dev_free(h->d_red_off); helm_dev_free(h->d_xinv_off); helm_dev_free(h->d_sep2_off);
  bool free_factors = true;
  if (h->shared) {
    std::lock_guard<std::mutex> lk(g_shared_mu);
    SharedFactors* sf = h->shared;
    if (--sf->refs > 0) {
      free_factors = false;
    } else {
      for (size_t k = 0; k < g_shared.size(); ++k)
        if (g_shared[k] == sf) { g_shared.erase(g_shared.begin() + k); break; }
      helm_dev_free(sf->xinv32);
      delete sf;
    }
  }
  if (free_factors) {
    helm_dev_free(h->d_dg); helm_dev_free(h->d_al); helm_dev_free(h->d_cr); helm_dev_free(h->d_ne);
    helm_dev_free(h->d_tc); helm_dev_free(h->d_fac); helm_dev_free(h->d_red); helm_dev_free(h->d_xinv);
    helm_dev_free(h->d_fac2); helm_dev_free(h->d_facp);
    helm_dev_free(h->d_sep2); helm_dev_free(h->d_sep2_plan);
  }
  delete h;
}
