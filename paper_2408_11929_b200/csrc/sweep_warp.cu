// sweep_warp.cu -- hot-path row a4, the default sweep kernel for block rows of
// <= 36 nodes and P > 1 segments: the two-chain partitioned double sweep of
// sweep_dual.cu (phase 1: top-down elimination with Sinv_c || bottom-up
// elimination with S'^{-1}_c; separator stage; phase 3: back substitution ||
// first-block-column correction; x = xa + fb), with each chain run by ONE warp:
//
//  * A block step is a complex w x w mat-vec.  Lane (a, b) = (lane & 3,
//    lane >> 2) owns rows 5b..5b+4 and columns a, a+4, .., a+32: 45 products,
//    five independent accumulators, a 2-level butterfly over a.  No barrier
//    per step: the next input vector is exchanged through shared memory with
//    __syncwarp only.
//  * Factor blocks are complex symmetric and stored as packed upper triangles
//    (w(w+1)/2 entries, half the HBM bytes of a full block).  The chain warp's
//    lane 0 streams them HBM/L2 -> shared memory with one cp.async.bulk per
//    block into an NST-stage ring (mbarrier complete_tx), NST-1 blocks ahead,
//    across phase and solve boundaries.  Each lane holds its 45 packed-triangle
//    offsets in registers (recomputed when the strip width changes), so a
//    product costs one LDS.128 and four DFMA.
//  * The per-solve stages (RHS, separator stage, epilogue) use all 8 warps.
// Numerics are those of sweep_dual.cu up to the summation order inside a row
// (DESIGN.md §5).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "sweep_common.cuh"

namespace warpk {
constexpr int WM = 40;      // vector stride (>= 8 row groups x 5 rows)
constexpr int NST = 4;      // ring stages per chain
constexpr int NTH = 256;    // threads per CTA (warps 0, 1: chains A, B)
constexpr int RPG = 5;      // rows per lane group
constexpr int CPL = 9;      // columns per lane (a + 4c)
constexpr int PWMAX = 36 * 37 / 2;
}  // namespace warpk

struct WarpArgs {
  DirArgs d[HELM_MAXDIR];
  int t;
  int vec_elems;    // cplx per vector area
  int nsolve_max;
  int pmax;
  int stage_elems;  // cplx per ring stage (>= max packed block + 1 zero entry)
  long long* prof;  // optional per-CTA counters (8 per CTA)
};

struct WarpTab {
  const cplx* fac;
  const cplx* fac2;
  const cplx* xinv;
  int w, a, s, pks;   // pks: entries per padded packed block (pk_size(w))
};

__device__ __forceinline__ uint64_t wl2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t wl2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ cplx wld_cg_hint(const cplx* a, uint64_t pol) {
  cplx v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void wprefetch_l2(const void* p, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
               : "memory");
}
__global__ void __launch_bounds__(warpk::NTH, 1) k_sweep_warp(const __grid_constant__ WarpArgs A) {
  using namespace warpk;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  constexpr int ncons = NTH;
  int d = 0;
  while (d + 1 < A.t && (int)blockIdx.x >= A.d[d + 1].cta_base) ++d;
  const DirArgs& D_ = A.d[d];
  const int p = blockIdx.x - D_.cta_base;
  const int P = D_.P, K = P - 1;

  // ring stages first (TMA destinations, 128-byte aligned), then barriers and vectors
  cplx* ring = reinterpret_cast<cplx*>(smem_raw);                 // [2][NST][stage_elems]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + 2L * NST * A.stage_elems);   // [2][NST]
  cplx* vbuf = reinterpret_cast<cplx*>(full + 2 * NST);            // [chain][2][WM]
  cplx* xlo = vbuf + 4 * WM;                                        // x_{p-1}
  cplx* xhi = xlo + WM;                                             // x_p
  cplx* zlo = xhi + WM;                                             // x0_lo (chain B phase 1)
  cplx* cpv = zlo + WM;
  cplx* cnv = cpv + A.pmax;
  WarpTab* tab = reinterpret_cast<WarpTab*>(cnv + A.pmax);
  cplx* vec0 = reinterpret_cast<cplx*>(
      smem_raw + ((((char*)(tab + A.nsolve_max) - (char*)smem_raw) + 127) / 128) * 128);
  cplx* bseg = vec0;                 // RHS rows lo..hi
  cplx* yseg = bseg + A.vec_elems;   // chain A phase 1 (y)
  cplx* xa = yseg + A.vec_elems;     // chain A phase 3 (aliased by g during the separator stage)
  cplx* fb = xa + A.vec_elems;       // chain B phase 3
  cplx* bcr = fb + A.vec_elems;      // staged U couplings, rows lo-1..hi
  cplx* bne = bcr + A.vec_elems;
  cplx* gsm = xa;                    // separator RHS g (K x w), dead before phase 3 writes xa

  const int nsolve = n_solves(D_);
  for (int i = tid; i < nsolve; i += blockDim.x) {
    const int s = sigma(D_, step_of(D_, i));
    tab[i].fac = D_.facp + D_.pfac_off[s];
    tab[i].fac2 = D_.fac2 + D_.pfac_off[s];
    tab[i].xinv = D_.xinv + D_.xinv_off[s];
    tab[i].w = D_.w[s];
    tab[i].a = D_.a[s];
    tab[i].s = s;
    tab[i].pks = pk_size(D_.w[s]);
  }
  for (int e = tid; e < 4 * WM; e += blockDim.x) vbuf[e] = cmk(0, 0);   // padding stays finite
  // the zero entry after each ring stage (target of the out-of-range offsets)
  for (int e = tid; e < 2 * NST; e += blockDim.x) ring[(long)e * A.stage_elems + A.stage_elems - 1] = cmk(0, 0);
  if (tid == 0) {
    for (int e = 0; e < 2 * NST; ++e) mbar_init(&full[e], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int lo = D_.seg_lo[p], hi = D_.seg_hi[p];
  const int m = hi - lo + 1;
  __syncthreads();

  const int wid = tid >> 5, lane = tid & 31;
  const long band_stride = (long)D_.nc * D_.wmax;
  long long xwait = 0, t_sep = 0, t_pre = 0, t_mbar = 0;
  const long long t_start = clock64();
  auto cbar = [&]() { __syncthreads(); };
  const long exs = 2L * P * D_.wmax;   // parity stride of yb / xb
  const long xss = (long)P * D_.wmax;  // parity stride of xs
  const uint64_t pol_last = wl2_policy_last(), pol_first = wl2_policy_first();
  int cur = 0;

  // ------------------------------------------------------------ per-solve actions (all consumers)
  // epilogue of solve i: x = xa + fb gathered into Z, boundary rows published, next correction
  auto seg_epilogue = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    const int par = i & 1;
    if (writes_Z(D_, i)) {
      const int olo = D_.own_lo[s], ohi = D_.own_hi[s], ow = ohi - olo + 1;
      for (int e = tid; e < m * ow; e += ncons) {
        int cl = e / ow, qq = olo + e % ow;
        D_.Z[node_of(D_, a, lo + cl, qq)] = cadd(xa[cl * w + qq], fb[cl * w + qq]);
      }
      if (p < P - 1)
        for (int e = tid; e < ow; e += ncons) D_.Z[node_of(D_, a, hi + 1, olo + e)] = xhi[olo + e];
    }
    cplx* xb = D_.xb + par * exs + (long)p * 2 * D_.wmax;
    for (int e = tid; e < w; e += ncons) {
      xb[e] = cadd(xa[e], fb[e]);
      xb[D_.wmax + e] = cadd(xa[(m - 1) * w + e], fb[(m - 1) * w + e]);
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
        return cadd(xa[(cc - lo) * w + qq], fb[(cc - lo) * w + qq]);
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
      bseg[cl * w + qq] = v;
    }
    for (int e = tid; e < (m + 1) * w; e += ncons) {
      int cl = e / w, qq = e % w, c = lo - 1 + cl;
      bcr[e] = c >= 0 ? __ldg(cband + (long)c * D_.wmax + qq) : cmk(0, 0);
      bne[e] = c >= 0 ? __ldg(nband + (long)c * D_.wmax + qq) : cmk(0, 0);
    }
  };
  // separator stage of solve i (after phase 1): all-gather of x0_lo / x0_hi, g,
  // x_p = X_p g, neighbour exchange, phase-3 chain inputs
  auto seg_separators = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    const int par = i & 1, ppar = par ^ 1;
    const int qp = prev_side(D_) == 0 ? 0 : w - 1;
    const int qn = next_side(D_) == 0 ? 0 : w - 1;
    const cplx* cband = D_.cr + s * band_stride;
    const cplx* nband = D_.ne + s * band_stride;
    const long Kw = (long)K * w;
    if (p < P - 1 && tid < 32) {
      // stream this CTA's rows of the separator inverse (w x Kw, contiguous) into L2
      // while the all-gather completes; the mat-vec below then reads L2
      const char* xp = reinterpret_cast<const char*>(tab[i].xinv + (long)p * w * x_ld(K, w));
      const long bytes = (long)w * x_ld(K, w) * (long)sizeof(cplx);
      for (long o = (long)tid * 32768; o < bytes; o += 32L * 32768)
        wprefetch_l2(xp + o, (uint32_t)(bytes - o < 32768L ? bytes - o : 32768L), pol_first);
    }
    cplx* yb = D_.yb + par * exs + (long)p * 2 * D_.wmax;
    for (int e = tid; e < w; e += ncons) {
      yb[e] = zlo[e];
      yb[D_.wmax + e] = yseg[(m - 1) * w + e];
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
    // g_k = b_{s_k} - U_{h_k}^T x0_k[hi] - U_{s_k} x0_{k+1}[lo]  (all K separators)
    const cplx* ybp = D_.yb + par * exs;
    for (int e = tid; e < K * w; e += ncons) {
      const int k = e / w, qq = e % w;
      const int hk = D_.seg_hi[k], sk = hk + 1;
      cplx v = __ldg(D_.R + node_of(D_, a, sk, qq));
      if (st > 0 && qq == qp) v = cadd(v, cpv[k]);
      if (bwd && qq == qn) v = cadd(v, cnv[k]);
      const cplx* yh = ybp + (long)k * 2 * D_.wmax + D_.wmax;
      const cplx* yl = ybp + (long)(k + 1) * 2 * D_.wmax;
      cplx tt = cmul(__ldg(cband + (long)hk * D_.wmax + qq), ldcg(yh + qq));
      if (qq >= 1) cfma(tt, __ldg(nband + (long)hk * D_.wmax + qq - 1), ldcg(yh + qq - 1));
      cfma(tt, __ldg(cband + (long)sk * D_.wmax + qq), ldcg(yl + qq));
      if (qq + 1 < w) cfma(tt, __ldg(nband + (long)sk * D_.wmax + qq), ldcg(yl + qq + 1));
      gsm[k * w + qq] = csub(v, tt);
    }
    cbar();
    // x_p = X_p g: 4 rows per warp, 16 independent loads in flight per lane
    const int cw = tid >> 5, ncw = ncons >> 5;
    if (p < P - 1) {
      for (int rb = 4 * cw; rb < w; rb += 4 * ncw) {
        const cplx* Xr[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ok[u] = rb + u < w;
          Xr[u] = tab[i].xinv + ((long)p * w + (ok[u] ? rb + u : 0)) * x_ld(K, w);
        }
        cplx acc[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
        for (long jj = lane; jj < Kw; jj += 128) {
          cplx xv[4][4], gv[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const bool in = jj + 32 * v < Kw;
            gv[v] = in ? gsm[jj + 32 * v] : cmk(0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u][v] = (ok[u] && in) ? wld_cg_hint(Xr[u] + jj + 32 * v, pol_first) : cmk(0, 0);
          }
#pragma unroll
          for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int u = 0; u < 4; ++u) cfma(acc[u], xv[u][v], gv[v]);
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
    }
    for (int e = tid; e < WM; e += ncons) {
      if (p == 0) xlo[e] = cmk(0, 0);
      if (p == P - 1) xhi[e] = cmk(0, 0);
    }
    cbar();
    // publish x_p (parity buffer; also the next solve's correction source),
    // then take x_{p-1} from the left neighbour
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
    // phase-3 inputs: chain A  U_hi x_p;  chain B  -U_{lo-1}^T x_{p-1}
    cplx* vA = vbuf + 0 * 2 * WM + cur * WM;
    cplx* vB = vbuf + 1 * 2 * WM + cur * WM;
    for (int qq = tid; qq < w; qq += ncons) {
      const cplx* crr = bcr + (long)m * w;      // row hi
      const cplx* ner = bne + (long)m * w;
      cplx ta = cmul(crr[qq], xhi[qq]);
      if (qq + 1 < w) cfma(ta, ner[qq], xhi[qq + 1]);
      vA[qq] = ta;
      cplx tb = cmul(bcr[qq], xlo[qq]);          // row lo-1
      if (qq >= 1) cfma(tb, bne[qq - 1], xlo[qq - 1]);
      vB[qq] = cscale(tb, -1.0);
    }
  };


  // ------------------------------------------------------------ chain warps
  // Block sequence of chain G: per solve, phase 0 then phase 1, m blocks each.
  // Lane 0 of the chain warp is the TMA producer of its own ring.
  const int G = wid;                       // valid for wid < 2
  const int ga = lane & 3, gb = lane >> 2;
  uint32_t fseq = 0;                       // blocks issued (producer, lane 0)
  uint32_t cseq = 0;                       // blocks consumed
  int pr_i = 0, pr_e = 0;                  // producer cursor (solve, step within solve)
  auto produce_one = [&]() {
    if (pr_i >= nsolve) return;
    const int pw = tab[pr_i].pks;
    const int ph = pr_e >= m ? 1 : 0, js = pr_e - ph * m;
    const bool up = (G == 0) == (ph == 0);
    const cplx* src = (G == 0 ? tab[pr_i].fac : tab[pr_i].fac2) + (long)(up ? lo + js : hi - js) * pw;
    const int st = fseq % NST;
    uint64_t* bar = &full[G * NST + st];
    const uint32_t bytes = (uint32_t)(pw * sizeof(cplx));
    mbar_expect_tx(bar, bytes);
    bulk_g2s_hint(ring + ((long)G * NST + st) * A.stage_elems, src, bytes, bar, ph == 0 ? pol_last : pol_first);
    ++fseq;
    if (++pr_e == 2 * m) { pr_e = 0; ++pr_i; }
  };
  if (wid < 2 && lane == 0)
    for (int k = 0; k < NST - 1; ++k) produce_one();

  // per-lane packed-triangle byte offsets of the 45 products (row 5b+i, column a+4c);
  // out-of-range products point at the zero entry at the end of the stage
  uint32_t off[RPG][CPL];
  int off_w = -1;
  auto set_offsets = [&](int w) {
    const int pw = w * (w + 1) / 2;
#pragma unroll
    for (int i = 0; i < RPG; ++i) {
      const int r = RPG * gb + i;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int k = ga + 4 * c;
        int idx;
        if (r >= w || k >= w) idx = A.stage_elems - 1;
        else idx = pk_index(r, k, w);
        off[i][c] = (uint32_t)idx * (uint32_t)sizeof(cplx);
      }
    }
    off_w = w;
    (void)pw;
  };

  auto run_phase = [&](int i, auto G_, auto PH_) {
    constexpr int GG = decltype(G_)::value;
    constexpr int PH = decltype(PH_)::value;
    constexpr bool up = (GG == 0) == (PH == 0);   // A1, B3 walk lo -> hi
    constexpr bool sub = GG == 0 && PH == 1;      // chain A back substitution: o = y_c - Sinv v
    const int w = tab[i].w;
    if (w != off_w) set_offsets(w);
    const uint32_t ring_base = smem_u32(ring + (long)GG * NST * A.stage_elems);
    const uint32_t stage_bytes = (uint32_t)A.stage_elems * (uint32_t)sizeof(cplx);
    cplx* myv = vbuf + GG * 2 * WM;
    for (int js = 0; js < m; ++js) {
      // keep the ring NST-1 blocks ahead (the stage refilled here was consumed in step js-1)
      if (lane == 0) produce_one();
      const int st = cseq % NST;
      const long long tw0 = clock64();
      mbar_wait(&full[GG * NST + st], (cseq / NST) & 1);
      t_mbar += clock64() - tw0;
      ++cseq;
      const uint32_t sb = ring_base + st * stage_bytes;
      const cplx* vin = myv + cur * WM;
      cplx acc[RPG];
#pragma unroll
      for (int r = 0; r < RPG; ++r) acc[r] = cmk(0, 0);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const cplx v = vin[ga + 4 * c];
#pragma unroll
        for (int r = 0; r < RPG; ++r) cfma(acc[r], lds128(sb + off[r][c]), v);
      }
#pragma unroll
      for (int r = 0; r < RPG; ++r) {
        acc[r].x += __shfl_xor_sync(0xffffffffu, acc[r].x, 1);
        acc[r].y += __shfl_xor_sync(0xffffffffu, acc[r].y, 1);
        acc[r].x += __shfl_xor_sync(0xffffffffu, acc[r].x, 2);
        acc[r].y += __shfl_xor_sync(0xffffffffu, acc[r].y, 2);
      }
      const int ci = up ? js : m - 1 - js;   // local block row
      // outputs of rows 5gb..5gb+4 (every lane of the group holds all five)
      cplx o[RPG];
#pragma unroll
      for (int r = 0; r < RPG; ++r) {
        const int row = RPG * gb + r;
        o[r] = acc[r];
        if (sub) o[r] = row < w ? csub(yseg[ci * w + row], acc[r]) : cmk(0, 0);
      }
      // neighbours across lane groups: o[row-1] of row 5gb and o[row+1] of row 5gb+4
      cplx prv, nxt;
      prv.x = __shfl_up_sync(0xffffffffu, o[RPG - 1].x, 4);
      prv.y = __shfl_up_sync(0xffffffffu, o[RPG - 1].y, 4);
      nxt.x = __shfl_down_sync(0xffffffffu, o[0].x, 4);
      nxt.y = __shfl_down_sync(0xffffffffu, o[0].y, 4);
      if (gb == 7) nxt = cmk(0, 0);
      cplx* vn = myv + (cur ^ 1) * WM;
      const bool last = js == m - 1;
      // lane a writes rows i = a and (a == 0) i = 4 of its group
#pragma unroll
      for (int r = 0; r < RPG; ++r) {
        if (!(r == ga || (r == 4 && ga == 0))) continue;
        const int row = RPG * gb + r;
        if (row >= w) continue;
        const cplx om = r > 0 ? o[r - 1] : prv;          // o[row-1]
        const cplx op = r < RPG - 1 ? o[r + 1] : nxt;    // o[row+1]
        if (GG == 0 && PH == 0) {
          // A1: y_c; next input b_{c+1} - U_c^T y_c
          yseg[ci * w + row] = o[r];
          if (!last) {
            const cplx* cr = bcr + (long)(ci + 1) * w;
            const cplx* ne = bne + (long)(ci + 1) * w;
            cplx v = csub(bseg[(ci + 1) * w + row], cmul(cr[row], o[r]));
            if (row >= 1) v = csub(v, cmul(ne[row - 1], om));
            vn[row] = v;
          }
        } else if (GG == 0) {
          // A3: xa_c; next input U_{c-1} xa_c
          xa[ci * w + row] = o[r];
          if (!last) {
            const cplx* cr = bcr + (long)ci * w;
            const cplx* ne = bne + (long)ci * w;
            cplx v = cmul(cr[row], o[r]);
            if (row + 1 < w) cfma(v, ne[row], op);
            vn[row] = v;
          }
        } else if (PH == 0) {
          // B1: z_c; next input b_{c-1} - U_{c-1} z_c; z_lo = x0_lo
          if (last) {
            zlo[row] = o[r];
          } else {
            const cplx* cr = bcr + (long)ci * w;
            const cplx* ne = bne + (long)ci * w;
            cplx v = cmul(cr[row], o[r]);
            if (row + 1 < w) cfma(v, ne[row], op);
            vn[row] = csub(bseg[(ci - 1) * w + row], v);
          }
        } else {
          // B3: f_c; next input -U_c^T f_c
          fb[ci * w + row] = o[r];
          if (!last) {
            const cplx* cr = bcr + (long)(ci + 1) * w;
            const cplx* ne = bne + (long)(ci + 1) * w;
            cplx v = cmul(cr[row], o[r]);
            if (row >= 1) cfma(v, ne[row - 1], om);
            vn[row] = cscale(v, -1.0);
          }
        }
      }
      __syncwarp();
      cur ^= 1;
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;

  auto solve_loop = [&](auto G_) {
    constexpr int GG = decltype(G_)::value;   // 0, 1: chain warps; 2: the other warps
    for (int i = 0; i < nsolve; ++i) {
      const int w = tab[i].w;
      // ---- pre-actions: epilogue of the previous solve, RHS, phase-1 inputs
      long long c0 = clock64();
      cbar();
      if (i > 0) {
        seg_epilogue(i - 1);
        cbar();
      }
      seg_rhs(i);
      cbar();
      for (int e = tid; e < w; e += ncons) {
        vbuf[0 * 2 * WM + cur * WM + e] = bseg[e];                // chain A: b_lo
        vbuf[1 * 2 * WM + cur * WM + e] = bseg[(m - 1) * w + e];  // chain B: b_hi
      }
      cbar();
      t_pre += clock64() - c0;
      if (GG < 2) run_phase(i, std::integral_constant<int, (GG < 2 ? GG : 0)>{}, I0{});
      else cur ^= m & 1;
      // ---- separator stage, phase-3 inputs
      c0 = clock64();
      cbar();
      seg_separators(i);
      cbar();
      t_sep += clock64() - c0;
      if (GG < 2) run_phase(i, std::integral_constant<int, (GG < 2 ? GG : 0)>{}, I1{});
      else cur ^= m & 1;
    }
  };
  if (wid == 0) solve_loop(I0{});
  else if (wid == 1) solve_loop(I1{});
  else solve_loop(std::integral_constant<int, 2>{});
  cbar();
  seg_epilogue(nsolve - 1);
  if (A.prof && tid == 0) {
    long long* o = A.prof + (long)blockIdx.x * 8;
    o[0] = t_pre; o[1] = t_sep; o[2] = t_mbar; o[3] = 2L * m * nsolve; o[4] = xwait;
    o[5] = clock64() - t_start; o[6] = 1; o[7] = d;
  }
}

// ------------------------------------------------------------------ host
static constexpr int kWarpSmemMax = 227 * 1024;
extern long long* helm_sweep_prof_buffer();

// Launches the warp-chain kernel if every direction fits it (w <= 36, P > 1,
// separator inverse and packed factor sets built at setup, shared memory);
// returns -1 (not applicable) otherwise.
int sweep_apply_warp(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                     cudaStream_t st) {
  using namespace warpk;
  int wmax = 0, pmax = 1, nsolve_max = 1;
  for (int d = 0; d < t; ++d) {
    wmax = std::max(wmax, dirs[d]->wmax);
    pmax = std::max(pmax, dirs[d]->P);
    nsolve_max = std::max(nsolve_max, dirs[d]->is_double ? 2 * dirs[d]->N - 1 : dirs[d]->N);
    if (dirs[d]->P < 2 || !dirs[d]->d_xinv || !dirs[d]->d_fac2 || !dirs[d]->d_facp) return -1;
  }
  if (wmax > 36) return -1;
  long vec_elems = 0;
  int ctas = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    int mmax = 0;
    for (int p = 0; p < h->P; ++p) mmax = std::max(mmax, h->seg_hi[p] - h->seg_lo[p] + 1);
    vec_elems = std::max(vec_elems, (long)(mmax + 1) * h->wmax);
    vec_elems = std::max(vec_elems, (long)(h->P - 1) * h->wmax);
    ctas += h->P;
  }
  vec_elems = (vec_elems + 7) / 8 * 8;
  const long stage_elems = pk_size(wmax) + 8;   // padded packed block + a zero entry, 128-byte multiple
  size_t smem = sizeof(cplx) * 2 * NST * stage_elems + sizeof(uint64_t) * 2 * NST +
                sizeof(cplx) * (7 * WM + 2 * pmax) + sizeof(WarpTab) * nsolve_max + 256;
  smem = (smem + 127) / 128 * 128 + sizeof(cplx) * 6 * vec_elems;
  if (smem > (size_t)kWarpSmemMax) return -1;
  std::vector<size_t> off(t);
  size_t total = 0;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    off[d] = total;
    total += al(sizeof(unsigned) * (2 + h->P));
    total += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax) * 2;
    total += al(sizeof(cplx) * 2L * h->P * h->wmax);
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
  WarpArgs A;
  memset(&A, 0, sizeof(A));
  A.t = t;
  A.vec_elems = (int)vec_elems;
  A.nsolve_max = nsolve_max;
  A.pmax = pmax;
  A.stage_elems = (int)stage_elems;
  A.prof = helm_sweep_prof_buffer();
  int base = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    DirArgs& D = A.d[d];
    D.axis = h->axis; D.order = h->order; D.N = h->N; D.P = h->P; D.nc = h->nc;
    D.nxp1 = prob->nx + 1; D.is_double = h->is_double; D.ntile_max = 1;
    D.a = h->d_a; D.w = h->d_w; D.own_lo = h->d_own_lo; D.own_hi = h->d_own_hi;
    D.seg_lo = h->d_seg_lo; D.seg_hi = h->d_seg_hi;
    D.cr = h->d_cr; D.ne = h->d_ne; D.tc = h->d_tc;
    D.fac = h->d_fac; D.fac2 = h->d_fac2; D.facp = h->d_facp; D.pfac_off = h->d_pfac_off; D.fac_off = h->d_fac_off;
    D.red = h->d_red; D.red_off = h->d_red_off;
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
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_sweep_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 0, occ = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep_warp, NTH, smem);
  if (e == cudaSuccess && occ * nsm < ctas) {
    cudaFreeAsync(scratch, st);
    return -1;
  }
  if (e == cudaSuccess) {
    void* args[] = {(void*)&A};
    e = cudaLaunchCooperativeKernel((void*)k_sweep_warp, dim3(ctas), dim3(NTH), args, smem, st);
    g_helm_launches++;
  }
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply (warp): %s", cudaGetErrorString(e));
    return HELM_ECUDA;
  }
  return HELM_OK;
}
