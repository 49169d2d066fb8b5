// sweep_fast.cu -- hot-path row a4 for block rows of <= 36 nodes (C1, C2, C3,
// C5 and the y-sweeps of C4): the batched, partitioned double sweep of
// sweep_apply.cu (one persistent cooperative launch for all t directions),
// with a data path designed from B200 measurements (tools/bench_*.cu,
// DESIGN.md §5):
//
//  * No reducer CTA.  After phase 1 the P segment CTAs of a direction do one
//    all-gather of their boundary rows; every CTA then forms the separator
//    right-hand side g itself and obtains its two separator values as rows of
//    R^{-1} g, a parallel dense mat-vec with the explicit separator-inverse
//    rows precomputed at setup (strip_setup.cu, k_reduced_inverse).  This
//    replaces the (2P-3)-step dependent chain of the reduced block-Thomas
//    solve by ~1 MB of streamed reads per CTA.
//  * Factor blocks are streamed L2 -> registers with plain 128-bit loads,
//    D = 3 block steps ahead (each thread holds the 9 complex entries of its
//    row slice), so every factor byte crosses the L1/shared-memory data path
//    once.  A helper warp keeps the next ~12 blocks (and the separator-inverse
//    rows of the next solve) warm in L2 with cp.async.bulk.prefetch.L2.
//  * 4 lanes per block row, 8 row slots per warp: 7 owned rows + 1 halo row.
//    The halo gives the writer lanes the neighbour value they need to form
//    the COMPLETE next input (b - L y or U x) with one shuffle: one input
//    vector, one 2-level butterfly and one named barrier per block step.
//    Forward rows are kept read-only during the backward pass (xsg holds the
//    final rows) so a halo slot never observes an owner's update.
//  * Exchange arrays are double-buffered by solve parity, so a CTA one solve
//    ahead never overwrites data a slower CTA still reads.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "sweep_common.cuh"

namespace fastk {
constexpr int LPR = 4;    // lanes per block row
constexpr int OWN = 7;    // owned rows per warp (8 slots, 1 halo)
constexpr int KPL = 9;    // complex entries per lane per block row (w <= 36)
constexpr int D = 3;      // register prefetch depth (block steps)
constexpr int WM = 40;    // vector stride
constexpr int PF = 12;    // L2 prefetch distance (block steps)
}  // namespace fastk

struct FastArgs {
  DirArgs d[HELM_MAXDIR];
  int t;
  int nw;           // consumer warps per CTA
  int vec_elems;    // cplx per vector area
  int nsolve_max;   // even
  int pmax;
  int nsx;          // stages of the separator-inverse row ring (0 = plain loads)
  int xrow_elems;   // cplx per ring stage (>= K*w of every direction)
  int sps_max;
  long long* prof;  // optional per-CTA counters (8 per CTA)
};

struct FastTab {
  const cplx* fac;
  const cplx* xinv;
  int w, a, s, pad;
};

// one entry of the per-CTA schedule of a solve
struct StepEnt {
  int row;      // block row c
  int kind;     // 0 forward step, 1 backward step
  int flags;    // bit0 high-halo mapping, bit4 phase 3, bits 8.. step within the phase
  int pad;
};

__device__ __forceinline__ StepEnt seg_entry(int e, int lo, int hi, int P) {
  const int m = hi - lo + 1, spp = 2 * m - 1, nph = P > 1 ? 2 : 1;
  const int ph = e / spp, js = e - ph * spp;
  StepEnt en;
  const int phase3 = nph == 2 ? ph : 1;
  int high;
  if (js < m) {
    en.kind = 0;
    en.row = lo + js;
    high = (js == m - 1 && m > 1) ? 1 : 0;
  } else {
    en.kind = 1;
    en.row = hi - 1 - (js - m);
    high = 1;
  }
  en.flags = high | (phase3 << 4) | (js << 8);
  en.pad = 0;
  return en;
}

// thread's block row for a step mapping
__device__ __forceinline__ int slot_row(int wi, int slot, int high) {
  return high ? fastk::OWN * wi + slot : fastk::OWN * wi + slot - 1;
}
__device__ __forceinline__ bool slot_owned(int slot, int high) { return high ? slot < 7 : slot >= 1; }

__device__ __forceinline__ void load_block(cplx (&dst)[fastk::KPL], const cplx* B, int w, int row, int q) {
  const bool ok = row >= 0 && row < w;
  const cplx* rp = B + (ok ? row * w + q : 0);
  const int kmax = ok ? w - q : 0;   // valid c: LPR*c < kmax
#pragma unroll
  for (int c = 0; c < fastk::KPL; ++c)
    dst[c] = (fastk::LPR * c < kmax) ? __ldg(rp + fastk::LPR * c) : cmk(0, 0);
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(32 * 8, 1) k_sweep_fast(const __grid_constant__ FastArgs A) {
  using namespace fastk;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int ncons = A.nw * 32;
  int d = 0;
  while (d + 1 < A.t && (int)blockIdx.x >= A.d[d + 1].cta_base) ++d;
  const DirArgs& D_ = A.d[d];
  const int p = blockIdx.x - D_.cta_base;
  const int P = D_.P, K = P - 1;

  cplx* vbuf = reinterpret_cast<cplx*>(smem_raw);   // [2][WM]
  cplx* xlo = vbuf + 2 * WM;                        // x_sep[p-1]
  cplx* xhi = xlo + WM;                             // x_sep[p]
  cplx* cpv = xhi + WM;                             // [pmax] prev-side separator corrections
  cplx* cnv = cpv + A.pmax;                         // [pmax] next-side separator corrections
  FastTab* tab = reinterpret_cast<FastTab*>(cnv + A.pmax);
  volatile int* prog = reinterpret_cast<volatile int*>(tab + A.nsolve_max);
  cplx* vec0 = reinterpret_cast<cplx*>(smem_raw + ((((char*)(prog + 4) - (char*)smem_raw) + 127) / 128) * 128);
  cplx* bseg = vec0;                                // RHS rows lo..hi
  cplx* yseg = bseg + A.vec_elems;                  // forward rows y
  cplx* bcr = yseg + A.vec_elems;                   // staged U couplings, rows lo-1..hi
  cplx* bne = bcr + A.vec_elems;
  cplx* xsg = bne + A.vec_elems;                    // final rows x
  cplx* gsm = xsg + A.vec_elems;                    // separator RHS g (K x w)
  StepEnt* sched = reinterpret_cast<StepEnt*>(gsm + A.vec_elems);
  // TMA ring for the rows of x_sep[p] = X_p g: mbarriers + stages (128-byte aligned)
  unsigned char* rb = reinterpret_cast<unsigned char*>(sched + A.sps_max);
  rb = reinterpret_cast<unsigned char*>((((uintptr_t)rb) + 127) & ~(uintptr_t)127);
  uint64_t* xfull = reinterpret_cast<uint64_t*>(rb);
  uint64_t* xempty = xfull + 16;
  cplx* xring = reinterpret_cast<cplx*>(rb + 256);

  const int nsolve = n_solves(D_);
  for (int i = tid; i < nsolve; i += blockDim.x) {
    const int s = sigma(D_, step_of(D_, i));
    tab[i].fac = D_.fac + D_.fac_off[s];
    tab[i].xinv = D_.xinv ? D_.xinv + D_.xinv_off[s] : nullptr;
    tab[i].w = D_.w[s];
    tab[i].a = D_.a[s];
    tab[i].s = s;
  }
  if (tid == 0) *prog = 0;
  const int lo = D_.seg_lo[p], hi = D_.seg_hi[p];
  const int m = hi - lo + 1;
  const int sps = (P > 1 ? 2 : 1) * (2 * m - 1);
  const int total = nsolve * sps;
  for (int e = tid; e < sps; e += blockDim.x) sched[e] = seg_entry(e, lo, hi, P);
  if (tid == 0 && A.nsx > 0) {
    for (int s2 = 0; s2 < A.nsx; ++s2) {
      mbar_init(&xfull[s2], 1);
      mbar_init(&xempty[s2], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // rows of X_p streamed per solve (0 when this CTA owns no separator)
  const bool own_sep = P > 1 && p < P - 1;

  if (tid >= ncons) {
    // ================================================================ L2 prefetch helper warp
    if (tid == ncons) {
      // lane 0: keep the factor blocks of the next PF steps warm in L2
      int pi = 0, ppos = 0;
      for (int jp = 0; jp < total; ++jp) {
        while (*prog + PF < jp) __nanosleep(500);
        const int w = tab[pi].w;
        const StepEnt en = sched[ppos];
        prefetch_l2(tab[pi].fac + (long)en.row * w * w, (uint32_t)(w * w * sizeof(cplx)));
        if (++ppos == sps) { ppos = 0; ++pi; }
      }
    } else if (tid == ncons + 32 && A.nsx > 0 && own_sep) {
      // second helper warp: TMA producer of the rows of X_p (separator inverse), solve after
      // solve; rows of the next solve are staged while the current one runs
      uint32_t f = 0;
      for (int i = 0; i < nsolve; ++i) {
        const int w = tab[i].w;
        const long Kw = (long)K * w;
        const uint32_t bytes = (uint32_t)(Kw * sizeof(cplx));
        const cplx* X = tab[i].xinv + (long)p * w * x_ld(K, w);
        for (int r = 0; r < w; ++r, ++f) {
          const int sidx = f % A.nsx;
          if (f >= (uint32_t)A.nsx) mbar_wait(&xempty[sidx], ((f / A.nsx) - 1) & 1);
          mbar_expect_tx(&xfull[sidx], bytes);
          bulk_g2s(xring + (long)sidx * A.xrow_elems, X + (long)r * x_ld(K, w), bytes, &xfull[sidx]);
        }
      }
    }
    return;
  }

  const int wi = tid >> 5, lane = tid & 31;
  const int slot = lane >> 2, q = lane & 3;
  const long band_stride = (long)D_.nc * D_.wmax;
  long long xwait = 0, t_sep = 0, t_pre = 0;
  const long long t_start = clock64();
  auto cbar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory"); };
  const long exs = 2L * P * D_.wmax;   // parity stride of yb / xb
  const long xss = (long)P * D_.wmax;  // parity stride of xs

  // register prefetch cursor (runs D steps ahead of the consumer)
  cplx pre[D][KPL];
  int pi = 0, ppos = 0, jp_next = 0;
  int pw = tab[0].w;
  const cplx* pbase = tab[0].fac;
  auto issue = [&](cplx (&dst)[KPL]) {
    if (jp_next < total) {
      const StepEnt en = sched[ppos];
      load_block(dst, pbase + (long)en.row * pw * pw, pw, slot_row(wi, slot, en.flags & 1), q);
      ++jp_next;
      if (++ppos == sps) {
        ppos = 0;
        if (++pi < nsolve) { pw = tab[pi].w; pbase = tab[pi].fac; }
      }
    }
  };
#pragma unroll
  for (int dd = 0; dd < D; ++dd) issue(pre[dd]);
  int ci_solve = 0, cpos = 0;
  int cur = 0;
  uint32_t xrow_base = 0;   // X rows consumed before the current solve (ring position)

  // ------------------------------------------------------------ per-solve actions
  // epilogue of solve i: gather into Z, publish boundary rows / separator, next correction
  auto seg_epilogue = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    const int par = i & 1;
    if (writes_Z(D_, i)) {
      const int olo = D_.own_lo[s], ohi = D_.own_hi[s], ow = ohi - olo + 1;
      for (int e = tid; e < m * ow; e += ncons) {
        int cl = e / ow, qq = olo + e % ow;
        D_.Z[node_of(D_, a, lo + cl, qq)] = xsg[cl * w + qq];
      }
      if (p < P - 1)
        for (int e = tid; e < ow; e += ncons) D_.Z[node_of(D_, a, hi + 1, olo + e)] = xhi[olo + e];
    }
    if (P > 1) {
      cplx* xb = D_.xb + par * exs + (long)p * 2 * D_.wmax;
      for (int e = tid; e < w; e += ncons) {
        xb[e] = xsg[e];
        xb[D_.wmax + e] = xsg[(m - 1) * w + e];
      }
    }
    int tdst = -1, side = 0;
    cplx* target = nullptr;
    if (!bwd) {
      if (st < D_.N - 1) { tdst = sigma(D_, st + 1); side = prev_side(D_); target = D_.corr_prev + (long)(st + 1) * D_.nc; }
      else if (D_.is_double && D_.N > 1) { tdst = sigma(D_, D_.N - 2); side = next_side(D_); target = D_.corr_next; }
    } else if (st >= 1) {
      tdst = sigma(D_, st - 1); side = next_side(D_); target = D_.corr_next;
    }
    if (tdst >= 0) {
      auto X = [&](int cc, int qq) -> cplx {
        if (cc < lo) return xlo[qq];
        if (cc > hi) return xhi[qq];
        return xsg[(cc - lo) * w + qq];
      };
      for (int c = lo + tid; c <= hi; c += ncons) target[c] = correction(D_, tdst, side, c, a, X);
    }
  };
  // RHS of solve i (rows lo..hi) and the couplings of rows lo-1..hi
  auto seg_rhs = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    const int qp = prev_side(D_) == 0 ? 0 : w - 1;
    const int qn = next_side(D_) == 0 ? 0 : w - 1;
    const cplx* cband = D_.cr + s * band_stride;
    const cplx* nband = D_.ne + s * band_stride;
    for (int e = tid; e < m * w; e += ncons) {
      int cl = e / w, qq = e % w, c = lo + cl;
      cplx v = __ldg(D_.R + node_of(D_, a, c, qq));
      if (st > 0 && qq == qp) v = cadd(v, D_.corr_prev[(long)st * D_.nc + c]);
      if (bwd && qq == qn) v = cadd(v, D_.corr_next[c]);
      bseg[cl * w + qq] = cscale(v, rhs_scale(D_, c, qq, w));
    }
    for (int e = tid; e < (m + 1) * w; e += ncons) {
      int cl = e / w, qq = e % w, c = lo - 1 + cl;
      bcr[e] = c >= 0 ? __ldg(cband + (long)c * D_.wmax + qq) : cmk(0, 0);
      bne[e] = c >= 0 ? __ldg(nband + (long)c * D_.wmax + qq) : cmk(0, 0);
    }
  };
  // separator stage of solve i (after phase 1): all-gather, g, x_sep = R^{-1} g rows
  auto seg_separators = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    const int par = i & 1, ppar = par ^ 1;
    const int qp = prev_side(D_) == 0 ? 0 : w - 1;
    const int qn = next_side(D_) == 0 ? 0 : w - 1;
    const cplx* cband = D_.cr + s * band_stride;
    const cplx* nband = D_.ne + s * band_stride;
    cplx* yb = D_.yb + par * exs + (long)p * 2 * D_.wmax;
    for (int e = tid; e < w; e += ncons) {
      yb[e] = xsg[e];
      yb[D_.wmax + e] = xsg[(m - 1) * w + e];
    }
    cbar();
    const long long cw0 = clock64();
    if (tid == 0) {
      __threadfence();
      red_release_add(&D_.cnt[0], 1u);
      while (ld_relaxed(&D_.cnt[0]) < (unsigned)(P * (i + 1))) __nanosleep(20);
      (void)ld_acquire(&D_.cnt[0]);
    }
    cbar();
    xwait += clock64() - cw0;
    // separator-row transmission corrections (from solve i-1) for every separator
    if (st > 0 || bwd) {
      const int aprev = i > 0 ? tab[i - 1].a : 0;
      for (int k = tid; k < K; k += ncons) {
        const int sk = D_.seg_hi[k] + 1;
        auto X = [&](int cc, int qq) -> cplx {
          if (cc == sk) return ldcg(D_.xs + ppar * xss + (long)k * D_.wmax + qq);
          if (cc == sk - 1) return ldcg(D_.xb + ppar * exs + (long)k * 2 * D_.wmax + D_.wmax + qq);
          return ldcg(D_.xb + ppar * exs + (long)(k + 1) * 2 * D_.wmax + qq);
        };
        cplx cp = cmk(0, 0), cn = cmk(0, 0);
        if (st > 0) {
          if (!bwd) {
            cp = correction(D_, s, prev_side(D_), sk, aprev, X);
            if (k == p) D_.corr_prev[(long)st * D_.nc + sk] = cp;   // kept for the backward pass
          } else {
            cp = ldcg(D_.corr_prev + (long)st * D_.nc + sk);
          }
        }
        if (bwd) cn = correction(D_, s, next_side(D_), sk, aprev, X);
        cpv[k] = cp;
        cnv[k] = cn;
      }
      cbar();
    }
    // g_k = b_{s_k} - U_{h_k}^T y_k[hi] - U_{s_k} y_{k+1}[lo]  (all K separators)
    const cplx* ybp = D_.yb + par * exs;
    for (int e = tid; e < K * w; e += ncons) {
      const int k = e / w, qq = e % w;
      const int hk = D_.seg_hi[k], sk = hk + 1;
      cplx v = __ldg(D_.R + node_of(D_, a, sk, qq));
      if (st > 0 && qq == qp) v = cadd(v, cpv[k]);
      if (bwd && qq == qn) v = cadd(v, cnv[k]);
      v = cscale(v, rhs_scale(D_, sk, qq, w));
      const cplx* yh = ybp + (long)k * 2 * D_.wmax + D_.wmax;
      const cplx* yl = ybp + (long)(k + 1) * 2 * D_.wmax;
      cplx tt = cmul(__ldg(cband + (long)hk * D_.wmax + qq), ldcg(yh + qq));
      if (qq >= 1) cfma(tt, __ldg(nband + (long)hk * D_.wmax + qq - 1), ldcg(yh + qq - 1));
      cfma(tt, __ldg(cband + (long)sk * D_.wmax + qq), ldcg(yl + qq));
      if (qq + 1 < w) cfma(tt, __ldg(nband + (long)sk * D_.wmax + qq), ldcg(yl + qq + 1));
      gsm[k * w + qq] = csub(v, tt);
    }
    cbar();
    // x_sep[p] = X_p g: the rows of X_p arrive through the TMA ring (one row per
    // stage, issued by the helper warp); warp wi reduces rows wi, wi + nw, ...
    const long Kw = (long)K * w;
    if (own_sep && A.nsx == 0) {
      // plain-load path: 4 rows per warp, 8 independent loads in flight per lane
      for (int rb = 4 * wi; rb < w; rb += 4 * A.nw) {
        const cplx* Xr[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ok[u] = rb + u < w;
          Xr[u] = tab[i].xinv + ((long)p * w + (ok[u] ? rb + u : 0)) * x_ld(K, w);
        }
        cplx acc[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
        for (long jj = lane; jj < Kw; jj += 64) {
          const bool two = jj + 32 < Kw;
          cplx xv[4][2];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            xv[u][0] = ok[u] ? __ldcg(Xr[u] + jj) : cmk(0, 0);
            xv[u][1] = (ok[u] && two) ? __ldcg(Xr[u] + jj + 32) : cmk(0, 0);
          }
          const cplx g0 = gsm[jj], g1 = two ? gsm[jj + 32] : cmk(0, 0);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            cfma(acc[u], xv[u][0], g0);
            cfma(acc[u], xv[u][1], g1);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            acc[u].x += __shfl_xor_sync(0xffffffffu, acc[u].x, off);
            acc[u].y += __shfl_xor_sync(0xffffffffu, acc[u].y, off);
          }
          if (lane == 0 && ok[u]) xhi[rb + u] = acc[u];
        }
      }
    } else if (own_sep) {
      for (int r = wi; r < w; r += A.nw) {
        const uint32_t f = xrow_base + r;
        const int sidx = f % A.nsx;
        mbar_wait(&xfull[sidx], (f / A.nsx) & 1);
        const cplx* Xr = xring + (long)sidx * A.xrow_elems;
        cplx a0 = cmk(0, 0), a1 = cmk(0, 0);
        long jj = lane;
        for (; jj + 32 < Kw; jj += 64) {
          cfma(a0, Xr[jj], gsm[jj]);
          cfma(a1, Xr[jj + 32], gsm[jj + 32]);
        }
        if (jj < Kw) cfma(a0, Xr[jj], gsm[jj]);
        cplx acc = cadd(a0, a1);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
        }
        __syncwarp();
        if (lane == 0) {
          xhi[r] = acc;
          mbar_arrive(&xempty[sidx]);
        }
      }
      xrow_base += w;
    }
    for (int e = tid; e < WM; e += ncons) {
      if (p == 0) xlo[e] = cmk(0, 0);
      if (p == P - 1) xhi[e] = cmk(0, 0);
    }
    cbar();
    // publish x_sep[p] (parity buffer; also the next solve's correction source),
    // then take x_sep[p-1] from the left neighbour
    if (p < P - 1) {
      for (int e = tid; e < w; e += ncons) D_.xs[par * xss + (long)p * D_.wmax + e] = xhi[e];
      cbar();
      if (tid == 0) {
        __threadfence();
        st_release(&D_.flag[p], (unsigned)(i + 1));
      }
    }
    if (p > 0) {
      const long long cw1 = clock64();
      if (tid == 0) {
        while (ld_relaxed(&D_.flag[p - 1]) < (unsigned)(i + 1)) __nanosleep(20);
        (void)ld_acquire(&D_.flag[p - 1]);
      }
      cbar();
      xwait += clock64() - cw1;
      for (int e = tid; e < w; e += ncons) xlo[e] = ldcg(D_.xs + par * xss + (long)(p - 1) * D_.wmax + e);
      cbar();
    }
    // phase-3 RHS: b_lo -= U_{lo-1}^T x_sep[p-1]; b_hi -= U_hi x_sep[p]
    for (int qq = tid; qq < w; qq += ncons) {
      if (p > 0) {
        cplx tt = cmul(bcr[qq], xlo[qq]);
        if (qq >= 1) cfma(tt, bne[qq - 1], xlo[qq - 1]);
        bseg[qq] = csub(bseg[qq], tt);
      }
      if (p < P - 1) {
        const cplx* crr = bcr + (long)m * w;      // row hi
        const cplx* ner = bne + (long)m * w;
        cplx tt = cmul(crr[qq], xhi[qq]);
        if (qq + 1 < w) cfma(tt, ner[qq], xhi[qq + 1]);
        bseg[(m - 1) * w + qq] = csub(bseg[(m - 1) * w + qq], tt);
      }
    }
  };

  // ------------------------------------------------------------ one block step
  auto do_step = [&](int j, cplx (&S)[KPL]) {
    const StepEnt en = sched[cpos];
    const int i = ci_solve;
    const int kind = en.kind, row_c = en.row, high = en.flags & 1;
    const int js = en.flags >> 8, ph3 = (en.flags >> 4) & 1;
    const int w = tab[i].w;
    // ---- pre-actions (uniform over the CTA)
    if (js == 0) {
      const long long cp0 = clock64();
      if (!ph3 || P == 1) {
        if (i > 0) {
          seg_epilogue(i - 1);
          cbar();
        }
        seg_rhs(i);
      } else {
        seg_separators(i);
      }
      cbar();
      for (int e = tid; e < w; e += ncons) vbuf[cur * WM + e] = bseg[e];
      cbar();
      if (!ph3 || P == 1) t_pre += clock64() - cp0;
      else t_sep += clock64() - cp0;
    }
    if (tid == 0) *prog = j;
    // ---- mat-vec on the block held in registers
    const int row = slot_row(wi, slot, high);
    const bool act = row >= 0 && row < w;
    const cplx* vin = vbuf + cur * WM;
    const int ci = row_c - lo;   // local block row
    cplx base = cmk(0, 0);
    if (act && kind == 1) base = yseg[ci * w + row];
    // 4 independent accumulator chains (dependent DFMA depth 3 x 2 instead of 5 x 2)
    cplx a0 = cmk(0, 0), a1 = cmk(0, 0), a2 = cmk(0, 0), a3 = cmk(0, 0);
#ifndef HELM_ABL_NOFMA
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int k = q + LPR * c;
      if (k < w) {
        const cplx v = vin[k];
        if ((c & 3) == 0) cfma(a0, S[c], v);
        else if ((c & 3) == 1) cfma(a1, S[c], v);
        else if ((c & 3) == 2) cfma(a2, S[c], v);
        else cfma(a3, S[c], v);
      }
    }
#else
    a0 = cadd(vin[q], S[0]);
#endif
    cplx acc = cadd(cadd(a0, a1), cadd(a2, a3));
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
    cplx o = kind == 1 ? csub(base, acc) : acc;
    if (!act) o = cmk(0, 0);
    // neighbour row value (r-1 for the low-halo mapping, r+1 for the high-halo one)
    cplx nb;
    if (high) {
      nb.x = __shfl_down_sync(0xffffffffu, o.x, 4);
      nb.y = __shfl_down_sync(0xffffffffu, o.y, 4);
    } else {
      nb.x = __shfl_up_sync(0xffffffffu, o.x, 4);
      nb.y = __shfl_up_sync(0xffffffffu, o.y, 4);
    }
    // register loads for step j + D (independent of this step's data)
#ifndef HELM_ABL_NOLDG
    issue(S);
#endif
#ifdef HELM_ABL_NOWRITER
    if (false) {
#else
    if (q == 0 && act && slot_owned(slot, high)) {
#endif
      cplx* vn = vbuf + (cur ^ 1) * WM;
      if (kind == 0) {
        yseg[ci * w + row] = o;
        if (js == m - 1) xsg[ci * w + row] = o;    // x_hi = y_hi
      } else {
        xsg[ci * w + row] = o;
      }
      if (kind == 0 && js < m - 1) {
        // forward-style input of row c+1: b_{c+1} - cr_c o - ne_c[r-1] o[r-1]
        const cplx* cr = bcr + (long)(ci + 1) * w;
        const cplx* ne = bne + (long)(ci + 1) * w;
        cplx v = csub(bseg[(ci + 1) * w + row], cmul(cr[row], o));
        if (row >= 1) v = csub(v, cmul(ne[row - 1], nb));
        vn[row] = v;
      } else if (kind == 0 ? (m > 1) : (row_c > lo)) {
        // backward-style input of row c' (fwd: hi-1, bwd: c-1): cr_c' o + ne_c' o[r+1]
        const int cp = kind == 0 ? hi - 1 : row_c - 1;
        const cplx* cr = bcr + (long)(cp - lo + 1) * w;
        const cplx* ne = bne + (long)(cp - lo + 1) * w;
        cplx v = cmul(cr[row], o);
        if (row + 1 < w) cfma(v, ne[row], nb);
        vn[row] = v;
      }
    }
    cbar();
    cur ^= 1;
    if (++cpos == sps) { cpos = 0; ++ci_solve; }
  };

  for (int j0 = 0; j0 < total; j0 += D) {
#pragma unroll
    for (int dd = 0; dd < D; ++dd) {
      const int j = j0 + dd;
      if (j < total) do_step(j, pre[dd]);
    }
  }
  seg_epilogue(nsolve - 1);
  if (A.prof && tid == 0) {
    long long* o = A.prof + (long)blockIdx.x * 8;
    o[0] = t_pre; o[1] = t_sep; o[2] = 0; o[3] = total; o[4] = xwait;
    o[5] = clock64() - t_start; o[6] = 0; o[7] = d;
  }
}

// ------------------------------------------------------------------ host
static constexpr int kFastSmemMax = 227 * 1024;
extern long long* helm_sweep_prof_buffer();

// Launches the register-streaming kernel if every direction fits it (w <= 36
// and, for P > 1, the explicit separator inverse was built at setup); returns
// -1 (not applicable) otherwise.
int sweep_apply_fast(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                     cudaStream_t st) {
  using namespace fastk;
  int wmax = 0, pmax = 1, nsolve_max = 1;
  for (int d = 0; d < t; ++d) {
    wmax = std::max(wmax, dirs[d]->wmax);
    pmax = std::max(pmax, dirs[d]->P);
    nsolve_max = std::max(nsolve_max, dirs[d]->is_double ? 2 * dirs[d]->N - 1 : dirs[d]->N);
    if (dirs[d]->P > 1 && !dirs[d]->d_xinv) return -1;
  }
  if (wmax > LPR * KPL || wmax > WM) return -1;
  nsolve_max = (nsolve_max + 1) & ~1;
  const int nw = (wmax + OWN - 1) / OWN;
  const int threads = nw * 32 + 64;   // consumers + L2-prefetch warp + TMA producer warp
  long vec_elems = 0;
  int ctas = 0, sps_max = 1;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    int mmax = 0;
    for (int p = 0; p < h->P; ++p) mmax = std::max(mmax, h->seg_hi[p] - h->seg_lo[p] + 1);
    vec_elems = std::max(vec_elems, (long)(mmax + 1) * h->wmax);
    vec_elems = std::max(vec_elems, (long)std::max(h->P - 1, 1) * h->wmax);
    sps_max = std::max(sps_max, (h->P > 1 ? 2 : 1) * (2 * mmax - 1));
    ctas += h->P;
  }
  vec_elems = (vec_elems + 7) / 8 * 8;
  size_t head = sizeof(cplx) * (4 * WM + 2 * pmax) + sizeof(FastTab) * nsolve_max + 16;
  head = (head + 127) / 128 * 128;
  size_t smem = head + sizeof(cplx) * 6 * vec_elems + sizeof(StepEnt) * sps_max;
  // separator-inverse row ring
  long xrow = 1;
  for (int d = 0; d < t; ++d) xrow = std::max(xrow, (long)std::max(dirs[d]->P - 1, 1) * dirs[d]->wmax);
  xrow = (xrow + 7) / 8 * 8;
  const size_t ring_fixed = 128 + 256;
  long room = (long)kFastSmemMax - (long)smem - (long)ring_fixed;
  int nsx = room > 0 ? (int)std::min<long>(8, room / (long)(sizeof(cplx) * xrow)) : 0;
  if (pmax > 1 && nsx < 2) nsx = 0;
  if (pmax == 1) nsx = 0;
  // (A TMA ring for the separator-inverse rows was tried in round 1 and hung
  // with >= ~96 co-resident CTAs; it is disabled: the rows are read from L2.)
  nsx = 0;
  smem += ring_fixed + (size_t)nsx * xrow * sizeof(cplx);
  if (smem > (size_t)kFastSmemMax) return -1;
  // per-direction scratch: counters, parity-buffered yb / xb / xs, corrections
  std::vector<size_t> off(t);
  size_t total = 0;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    off[d] = total;
    total += al(sizeof(unsigned) * (2 + h->P));               // counters + separator flags
    total += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax) * 2;   // yb, xb
    total += al(sizeof(cplx) * 2L * h->P * h->wmax);           // xs
    total += al(sizeof(cplx) * (long)h->N * h->nc);
    total += al(sizeof(cplx) * (long)h->nc);
  }
  unsigned char* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, total, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply: scratch alloc: %s", cudaGetErrorString(e));
    return HELM_ENOMEM;
  }
  const helm_problem_s* prob = dirs[0]->prob;
  FastArgs A;
  memset(&A, 0, sizeof(A));
  A.t = t;
  A.nw = nw;
  A.vec_elems = (int)vec_elems;
  A.nsolve_max = nsolve_max;
  A.pmax = pmax;
  A.nsx = nsx;
  A.xrow_elems = (int)xrow;
  A.sps_max = sps_max;
  A.prof = helm_sweep_prof_buffer();
  int base = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    DirArgs& D = A.d[d];
    D.axis = h->axis; D.order = h->order; D.N = h->N; D.P = h->P; D.nc = h->nc; D.disc = h->disc;
    D.nxp1 = prob->nx + 1; D.is_double = h->is_double; D.ntile_max = 1;
    D.a = h->d_a; D.w = h->d_w; D.own_lo = h->d_own_lo; D.own_hi = h->d_own_hi;
    D.seg_lo = h->d_seg_lo; D.seg_hi = h->d_seg_hi;
    D.cr = h->d_cr; D.ne = h->d_ne; D.tc = h->d_tc;
    D.fac = h->d_fac; D.fac_off = h->d_fac_off; D.red = h->d_red; D.red_off = h->d_red_off;
    D.xinv = h->d_xinv; D.xinv_off = h->d_xinv_off;
    D.R = Rdev + (ldr == 0 ? 0 : (long)d * ldr);
    D.Z = Zdev + (long)d * ldz;
    unsigned char* q = scratch + off[d];
    D.cnt = (unsigned*)q; D.flag = D.cnt + 2; q += al(sizeof(unsigned) * (2 + h->P));
    D.yb = (cplx*)q; q += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax);
    D.xb = (cplx*)q; q += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax);
    D.xs = (cplx*)q; q += al(sizeof(cplx) * 2L * h->P * h->wmax);
    D.corr_prev = (cplx*)q; q += al(sizeof(cplx) * (long)h->N * h->nc);
    D.corr_next = (cplx*)q;
    D.wmax = h->wmax;
    D.cta_base = base;
    base += h->P;
    if (e == cudaSuccess) e = cudaMemsetAsync(D.cnt, 0, sizeof(unsigned) * (2 + h->P), st);
  }
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_sweep_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 0, occ = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep_fast, threads, smem);
  if (e == cudaSuccess && occ * nsm < ctas) {
    helm_set_error("sweep_apply: %d CTAs cannot be co-resident (%d SMs x %d); reduce n_segments", ctas, nsm, occ);
    cudaFreeAsync(scratch, st);
    return HELM_ECUDA;
  }
  if (e == cudaSuccess) {
    void* args[] = {(void*)&A};
    e = cudaLaunchCooperativeKernel((void*)k_sweep_fast, dim3(ctas), dim3(threads), args, smem, st);
    g_helm_launches++;
  }
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply (fast): %s", cudaGetErrorString(e));
    return HELM_ECUDA;
  }
  return HELM_OK;
}
