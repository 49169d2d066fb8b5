// sweep_fast.cu -- hot-path row a4 for block rows of <= 36 nodes (C1, C2, C3,
// C5 and the y-sweeps of C4): the same batched, partitioned double sweep as
// sweep_apply.cu (segment CTAs + reducer CTA per direction, one persistent
// cooperative launch for all t directions), with a data path designed from
// B200 measurements (tools/bench_*.cu):
//
//  * Factor blocks are streamed L2 -> registers with plain 128-bit loads,
//    D = 3 block steps ahead (each thread holds only the 9 complex entries of
//    its row slice), so every factor byte crosses the L1/shared-memory data
//    path once (the TMA ring crosses it twice and saturated it).  A helper
//    warp keeps the blocks of the next ~12 steps warm in L2
//    (cp.async.bulk.prefetch.L2) so the first (HBM) touch is hidden too.
//  * 4 lanes per block row, 8 row slots per warp: 7 owned rows + 1 halo row.
//    The halo row gives the writer lanes the neighbour value they need to
//    form the COMPLETE next input (b - L y or U x) with one shuffle, so each
//    step reads a single input vector and needs one 2-level butterfly and
//    one named barrier.  The halo sits below (forward-style next input) or
//    above (backward-style) the owned rows, chosen per step.
//  * The reducer computes h_k = Rinv_k g_k for all separators off the
//    dependent chain (no barriers), then runs z_k = h_k - G_k z_{k-1} and
//    x_k = z_k - F_k x_{k+1}: one block per chain step.
#include <algorithm>
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
  long long* prof;  // optional per-CTA counters (8 per CTA)
};

struct FastTab {
  const cplx* fac;
  const cplx* red;
  int w, a, s, pad;
};

// decoded block step
struct Step {
  int i;        // solve
  int kind;     // 0 seg fwd, 1 seg bwd, 2 red h (Rinv), 3 red fwd chain (G), 4 red bwd chain (F)
  int row;      // seg: block row; red: separator k
  int high;     // halo mapping: 1 = neighbour row r+1 available, 0 = r-1
  int js;       // step within the solve (red) or phase (seg)
  int ph;       // seg: 0 phase 1, 1 phase 3
};

__device__ __forceinline__ Step seg_decode(int j, int lo, int hi, int P) {
  const int m = hi - lo + 1, spp = 2 * m - 1, nph = P > 1 ? 2 : 1;
  Step s;
  s.i = j / (nph * spp);
  const int r1 = j - s.i * nph * spp;
  const int ph = r1 / spp;
  s.ph = nph == 2 ? ph : 1;
  s.js = r1 - ph * spp;
  if (s.js < m) {
    s.kind = 0;
    s.row = lo + s.js;
    s.high = (s.js == m - 1 && m > 1) ? 1 : 0;
  } else {
    s.kind = 1;
    s.row = hi - 1 - (s.js - m);
    s.high = 1;
  }
  return s;
}

__device__ __forceinline__ Step red_decode(int j, int K) {
  const int sps = 3 * K - 2;
  Step s;
  s.i = j / sps;
  s.js = j - s.i * sps;
  s.high = 0;
  s.ph = 0;
  if (s.js < K) { s.kind = 2; s.row = s.js; }
  else if (s.js < 2 * K - 1) { s.kind = 3; s.row = s.js - K + 1; }
  else { s.kind = 4; s.row = K - 2 - (s.js - (2 * K - 1)); }
  return s;
}

// Per-CTA schedule of one solve (identical for every solve of the apply, only
// the strip changes): built once in shared memory; the per-step cursor is a
// table lookup plus a solve counter (no division, little uniform arithmetic).
struct StepEnt {
  int blk;      // block index inside the strip's factor array (seg: row; red: 3k + {0,1,2})
  int row;      // seg: block row c; red: separator k
  int kind;     // 0 seg fwd, 1 seg bwd, 2 red h, 3 red fwd chain, 4 red bwd chain
  int flags;    // bit0 high-halo mapping, bits 8.. js (in phase/solve), bit4 phase (seg: 0/1)
};

// Incremental step cursor (no integer division on the per-step path).
struct Cursor {
  Step s;
  int m, spp, nph, K, lo, hi, P;
  bool red;
  int w;
  const cplx* base;   // factor (or reduced-system) base of the current solve
  __device__ __forceinline__ void derive(const FastTab* tab) {
    if (!red) {
      if (s.js < m) { s.kind = 0; s.row = lo + s.js; s.high = (s.js == m - 1 && m > 1) ? 1 : 0; }
      else { s.kind = 1; s.row = hi - 1 - (s.js - m); s.high = 1; }
    } else {
      s.high = 0;
      if (s.js < K) { s.kind = 2; s.row = s.js; }
      else if (s.js < 2 * K - 1) { s.kind = 3; s.row = s.js - K + 1; }
      else { s.kind = 4; s.row = K - 2 - (s.js - (2 * K - 1)); }
    }
  }
  __device__ __forceinline__ void load_solve(const FastTab* tab, int nsolve) {
    if (s.i < nsolve) {
      w = tab[s.i].w;
      base = red ? tab[s.i].red : tab[s.i].fac;
    }
  }
  __device__ __forceinline__ void init(int j0, bool red_, int lo_, int hi_, int P_, const FastTab* tab, int nsolve) {
    red = red_; lo = lo_; hi = hi_; P = P_; K = P_ - 1;
    m = hi - lo + 1; spp = 2 * m - 1; nph = P > 1 ? 2 : 1;
    s = red ? red_decode(j0, K) : seg_decode(j0, lo, hi, P);
    load_solve(tab, nsolve);
  }
  __device__ __forceinline__ void advance(const FastTab* tab, int nsolve) {
    if (!red) {
      if (++s.js == spp) {
        s.js = 0;
        if (nph == 2 && s.ph == 0) s.ph = 1;
        else { s.ph = nph == 2 ? 0 : 1; ++s.i; load_solve(tab, nsolve); }
      }
    } else {
      if (++s.js == 3 * K - 2) { s.js = 0; ++s.i; load_solve(tab, nsolve); }
    }
    derive(tab);
  }
  __device__ __forceinline__ const cplx* block() const {
    const long w2 = (long)w * w;
    if (!red) return base + (long)s.row * w2;
    return base + ((long)s.row * 3 + (s.kind - 2)) * w2;
  }
};

__device__ __forceinline__ const cplx* step_block(const Step& s, const FastTab* tab) {
  const int w = tab[s.i].w;
  const long w2 = (long)w * w;
  if (s.kind <= 1) return tab[s.i].fac + (long)s.row * w2;
  return tab[s.i].red + ((long)s.row * 3 + (s.kind - 2)) * w2;
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

__global__ void __launch_bounds__(32 * 7, 1) k_sweep_fast(const __grid_constant__ FastArgs A) {
  using namespace fastk;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int ncons = A.nw * 32;
  int d = 0;
  while (d + 1 < A.t && (int)blockIdx.x >= A.d[d + 1].cta_base) ++d;
  const DirArgs& D_ = A.d[d];
  const int role = blockIdx.x - D_.cta_base;
  const bool reducer = (D_.P > 1 && role == D_.P);
  const int p = role;
  const int P = D_.P, K = P - 1;

  cplx* vbuf = reinterpret_cast<cplx*>(smem_raw);   // [2][WM]
  cplx* xlo = vbuf + 2 * WM;
  cplx* xhi = xlo + WM;
  cplx* cnx = xhi + WM;                                // pmax
  FastTab* tab = reinterpret_cast<FastTab*>(cnx + A.pmax);
  volatile int* prog = reinterpret_cast<volatile int*>(tab + A.nsolve_max);
  cplx* vec0 = reinterpret_cast<cplx*>(smem_raw + ((((char*)(prog + 4) - (char*)smem_raw) + 127) / 128) * 128);
  cplx* vec1 = vec0 + A.vec_elems;
  cplx* bcr = vec1 + A.vec_elems;
  cplx* bne = bcr + A.vec_elems;
  cplx* xsg = bne + A.vec_elems;    // segment: final solution x of the block sweep

  const int nsolve = n_solves(D_);
  for (int i = tid; i < nsolve; i += blockDim.x) {
    const int s = sigma(D_, step_of(D_, i));
    tab[i].fac = D_.fac + D_.fac_off[s];
    tab[i].red = D_.red + D_.red_off[s];
    tab[i].w = D_.w[s];
    tab[i].a = D_.a[s];
    tab[i].s = s;
  }
  if (tid == 0) *prog = 0;
  __syncthreads();

  const int lo = reducer ? 0 : D_.seg_lo[p];
  const int hi = reducer ? 0 : D_.seg_hi[p];
  const int m = hi - lo + 1;
  const int total = reducer ? nsolve * (3 * K - 2) : nsolve * (P > 1 ? 2 : 1) * (2 * m - 1);

  if (tid >= ncons) {
    // ================================================================ L2 prefetch helper warp
    if (tid == ncons) {
      for (int jp = 0; jp < total; ++jp) {
        while (*prog + PF < jp) __nanosleep(500);
        Step s = reducer ? red_decode(jp, K) : seg_decode(jp, lo, hi, P);
        const int w = tab[s.i].w;
        prefetch_l2(step_block(s, tab), (uint32_t)(w * w * sizeof(cplx)));
      }
    }
    return;
  }

  const int wi = tid >> 5, lane = tid & 31;
  const int slot = lane >> 2, q = lane & 3;
  const long band_stride = (long)D_.nc * D_.wmax;
  long long xwait = 0;
  const long long t_start = clock64();
  auto cbar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory"); };

  cplx pre[D][KPL];
  // schedule of one solve in shared memory
  StepEnt* sched = reinterpret_cast<StepEnt*>(xsg + A.vec_elems);
  const int sps = reducer ? 3 * K - 2 : (P > 1 ? 2 : 1) * (2 * m - 1);
  for (int e = tid; e < sps; e += ncons) {
    Step st = reducer ? red_decode(e, K) : seg_decode(e, lo, hi, P);
    StepEnt en;
    en.row = st.row;
    en.kind = st.kind;
    en.blk = st.kind <= 1 ? st.row : st.row * 3 + (st.kind - 2);
    en.flags = (st.high ? 1 : 0) | (st.ph ? 16 : 0) | (st.js << 8);
    sched[e] = en;
  }
  cbar();
  // cursor of the next block to load into registers (runs D steps ahead of the consumer)
  int pi = 0, ppos = 0, jp_next = 0;
  int pw = tab[0].w;
  const cplx* pbase = reducer ? tab[0].red : tab[0].fac;
  auto issue = [&](cplx (&dst)[KPL]) {
    if (jp_next < total) {
      const StepEnt en = sched[ppos];
      load_block(dst, pbase + (long)en.blk * pw * pw, pw, slot_row(wi, slot, en.flags & 1), q);
      ++jp_next;
      if (++ppos == sps) {
        ppos = 0;
        if (++pi < nsolve) { pw = tab[pi].w; pbase = reducer ? tab[pi].red : tab[pi].fac; }
      }
    }
  };
#pragma unroll
  for (int dd = 0; dd < D; ++dd) issue(pre[dd]);
  int ci_solve = 0, cpos = 0;
  int cur = 0;

  // ------------------------------------------------------------ segment helpers
  cplx* bseg = vec0;
  cplx* yseg = vec1;
  // epilogue of solve i: gather into Z, publish boundary rows, next correction
  auto seg_epilogue = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    if (writes_Z(D_, i)) {
      const int olo = D_.own_lo[s], ohi = D_.own_hi[s], ow = ohi - olo + 1;
      for (int e = tid; e < m * ow; e += ncons) {
        int cl = e / ow, qq = olo + e % ow;
        D_.Z[node_of(D_, a, lo + cl, qq)] = xsg[cl * w + qq];
      }
    }
    if (P > 1) {
      cplx* xb = D_.xb + (long)p * 2 * D_.wmax;
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

  // ------------------------------------------------------------ reducer helpers
  cplx* g = vec0;   // K x WM reduced RHS
  cplx* z = vec1;   // K x WM: h_k, then z_k, then x_k (in place)
  auto red_start = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    const int qp = prev_side(D_) == 0 ? 0 : w - 1;
    const int qn = next_side(D_) == 0 ? 0 : w - 1;
    const cplx* cband = D_.cr + s * band_stride;
    const cplx* nband = D_.ne + s * band_stride;
    const long long cw0 = clock64();
    if (tid == 0) {
      while (ld_relaxed(&D_.cnt[0]) < (unsigned)(P * (i + 1))) __nanosleep(20);
      (void)ld_acquire(&D_.cnt[0]);
    }
    cbar();
    xwait += clock64() - cw0;
    if (i >= 1) {
      const int aprev = tab[i - 1].a;
      const int side = bwd ? next_side(D_) : prev_side(D_);
      for (int k = tid; k < K; k += ncons) {
        const int sk = D_.seg_hi[k] + 1;
        auto X = [&](int cc, int qq) -> cplx {
          if (cc == sk) return z[k * WM + qq];
          if (cc == sk - 1) return ldcg(D_.xb + (long)k * 2 * D_.wmax + D_.wmax + qq);
          return ldcg(D_.xb + (long)(k + 1) * 2 * D_.wmax + qq);
        };
        cplx cv = correction(D_, s, side, sk, aprev, X);
        if (!bwd) D_.corr_prev[(long)st * D_.nc + sk] = cv;
        else cnx[k] = cv;
      }
      cbar();
    }
    for (int e = tid; e < K * w; e += ncons) {
      const int k = e / w, qq = e % w;
      const int hk = D_.seg_hi[k], sk = hk + 1;
      cplx v = __ldg(D_.R + node_of(D_, a, sk, qq));
      if (st > 0 && qq == qp) v = cadd(v, D_.corr_prev[(long)st * D_.nc + sk]);
      if (bwd && qq == qn) v = cadd(v, cnx[k]);
      const cplx* yh = D_.yb + (long)k * 2 * D_.wmax + D_.wmax;
      const cplx* yl = D_.yb + (long)(k + 1) * 2 * D_.wmax;
      cplx t = cmul(__ldg(cband + (long)hk * D_.wmax + qq), ldcg(yh + qq));
      if (qq >= 1) cfma(t, __ldg(nband + (long)hk * D_.wmax + qq - 1), ldcg(yh + qq - 1));
      cfma(t, __ldg(cband + (long)sk * D_.wmax + qq), ldcg(yl + qq));
      if (qq + 1 < w) cfma(t, __ldg(nband + (long)sk * D_.wmax + qq), ldcg(yl + qq + 1));
      g[k * WM + qq] = csub(v, t);
    }
    cbar();
  };
  auto red_finish = [&](int i) {
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    for (int e = tid; e < K * w; e += ncons) {
      const int k = e / w, qq = e % w;
      D_.xs[(long)k * D_.wmax + qq] = z[k * WM + qq];
    }
    cbar();
    if (tid == 0) {
      __threadfence();
      st_release(&D_.cnt[1], (unsigned)(i + 1));
    }
    if (writes_Z(D_, i)) {
      const int olo = D_.own_lo[s], ohi = D_.own_hi[s], ow = ohi - olo + 1;
      for (int e = tid; e < K * ow; e += ncons) {
        const int k = e / ow, qq = olo + e % ow;
        D_.Z[node_of(D_, a, D_.seg_hi[k] + 1, qq)] = z[k * WM + qq];
      }
    }
  };

  // ------------------------------------------------------------ one block step
  auto do_step = [&](int j, cplx (&S)[KPL]) {
    Step s;
    {
      const StepEnt en = sched[cpos];
      s.i = ci_solve; s.kind = en.kind; s.row = en.row; s.high = en.flags & 1;
      s.js = en.flags >> 8; s.ph = reducer ? 0 : ((P > 1) ? ((en.flags >> 4) & 1) : 1);
    }
    const int w = tab[s.i].w;
    // ---- pre-actions (uniform over the CTA)
    if (!reducer) {
      if (s.js == 0 && (s.ph == 0 || P == 1)) {
        if (s.i > 0) {
          seg_epilogue(s.i - 1);
          cbar();
        }
        seg_rhs(s.i);
        cbar();
        for (int e = tid; e < w; e += ncons) vbuf[cur * WM + e] = bseg[e];
        cbar();
      } else if (s.js == 0 && s.ph == 1) {
        // end of phase 1: publish y[lo], y[hi]; wait for the separators; phase-3 RHS
        cplx* yb = D_.yb + (long)p * 2 * D_.wmax;
        for (int e = tid; e < w; e += ncons) {
          yb[e] = xsg[e];
          yb[D_.wmax + e] = xsg[(m - 1) * w + e];
        }
        cbar();
        const long long cw0 = clock64();
        if (tid == 0) {
          __threadfence();
          red_release_add(&D_.cnt[0], 1u);
          while (ld_relaxed(&D_.cnt[1]) < (unsigned)(s.i + 1)) __nanosleep(20);
          (void)ld_acquire(&D_.cnt[1]);
        }
        cbar();
        xwait += clock64() - cw0;
        for (int e = tid; e < w; e += ncons) {
          xlo[e] = p > 0 ? ldcg(D_.xs + (long)(p - 1) * D_.wmax + e) : cmk(0, 0);
          xhi[e] = p < P - 1 ? ldcg(D_.xs + (long)p * D_.wmax + e) : cmk(0, 0);
        }
        cbar();
        for (int qq = tid; qq < w; qq += ncons) {
          if (p > 0) {
            const cplx* crr = bcr;                    // row lo-1
            const cplx* ner = bne;
            cplx t = cmul(crr[qq], xlo[qq]);
            if (qq >= 1) cfma(t, ner[qq - 1], xlo[qq - 1]);
            bseg[qq] = csub(bseg[qq], t);
          }
          if (p < P - 1) {
            const cplx* crr = bcr + (long)m * w;      // row hi
            const cplx* ner = bne + (long)m * w;
            cplx t = cmul(crr[qq], xhi[qq]);
            if (qq + 1 < w) cfma(t, ner[qq], xhi[qq + 1]);
            bseg[(m - 1) * w + qq] = csub(bseg[(m - 1) * w + qq], t);
          }
        }
        cbar();
        for (int e = tid; e < w; e += ncons) vbuf[cur * WM + e] = bseg[e];
        cbar();
      }
    } else {
      if (s.js == 0) red_start(s.i);
    }
    if (tid == 0) *prog = j;
    // ---- mat-vec on the block held in registers
    const int row = slot_row(wi, slot, s.high);
    const bool act = row >= 0 && row < w;
    const cplx* vin;
    if (s.kind <= 1) vin = vbuf + cur * WM;
    else if (s.kind == 2) vin = g + s.row * WM;
    else if (s.kind == 3) vin = z + (s.row - 1) * WM;
    else vin = z + (s.row + 1) * WM;
    // base for "x = base - acc" steps
    cplx base = cmk(0, 0);
    const int ci = s.row - lo;   // segment local row
    if (act) {
      if (s.kind == 1) base = yseg[ci * w + row];
      else if (s.kind >= 3) base = z[s.row * WM + row];
    }
    cplx a0 = cmk(0, 0), a1 = cmk(0, 0);
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int k = q + LPR * c;
      if (k < w) {
        if (c & 1) cfma(a1, S[c], vin[k]);
        else cfma(a0, S[c], vin[k]);
      }
    }
    cplx acc = cadd(a0, a1);
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
    cplx o = (s.kind == 1 || s.kind >= 3) ? csub(base, acc) : acc;
    if (!act) o = cmk(0, 0);
    // neighbour row value (r-1 for the low-halo mapping, r+1 for the high-halo one)
    cplx nb;
    if (s.high) {
      nb.x = __shfl_down_sync(0xffffffffu, o.x, 4);
      nb.y = __shfl_down_sync(0xffffffffu, o.y, 4);
    } else {
      nb.x = __shfl_up_sync(0xffffffffu, o.x, 4);
      nb.y = __shfl_up_sync(0xffffffffu, o.y, 4);
    }
    // issue the register loads for step j + D (independent of this step's data)
    issue(S);
    if (q == 0 && act && slot_owned(slot, s.high)) {
      if (s.kind <= 1) {
        // forward rows go to yseg (read-only during the backward pass, so a halo
        // slot can never observe an owner's update); final rows go to xsg
        if (s.kind == 0) {
          yseg[ci * w + row] = o;
          if (s.js == m - 1) xsg[ci * w + row] = o;    // x_hi = y_hi
        } else {
          xsg[ci * w + row] = o;
        }
        cplx* vn = vbuf + (cur ^ 1) * WM;
        if (s.kind == 0 && s.js < m - 1) {
          // forward-style input of row c+1: b_{c+1} - cr_c o - ne_c[r-1] o[r-1]
          const cplx* cr = bcr + (long)(ci + 1) * w;
          const cplx* ne = bne + (long)(ci + 1) * w;
          cplx v = csub(bseg[(ci + 1) * w + row], cmul(cr[row], o));
          if (row >= 1) v = csub(v, cmul(ne[row - 1], nb));
          vn[row] = v;
        } else if (s.kind == 0 ? (m > 1) : (s.row > lo)) {
          // backward-style input of row c' = (fwd: hi-1, bwd: c-1): cr_c' o + ne_c' o[r+1]
          const int cp = s.kind == 0 ? hi - 1 : s.row - 1;
          const cplx* cr = bcr + (long)(cp - lo + 1) * w;
          const cplx* ne = bne + (long)(cp - lo + 1) * w;
          cplx v = cmul(cr[row], o);
          if (row + 1 < w) cfma(v, ne[row], nb);
          vn[row] = v;
        }
      } else {
        z[s.row * WM + row] = o;
      }
    }
    const bool need_bar = !(s.kind == 2 && s.js < K - 1);
    if (need_bar) cbar();
    if (s.kind <= 1) cur ^= 1;
    if (reducer && s.js == 3 * K - 3) red_finish(s.i);
    if (++cpos == sps) { cpos = 0; ++ci_solve; }
  };

  for (int j0 = 0; j0 < total; j0 += D) {
#pragma unroll
    for (int dd = 0; dd < D; ++dd) {
      const int j = j0 + dd;
      if (j < total) do_step(j, pre[dd]);
    }
  }
  if (!reducer) {
    seg_epilogue(nsolve - 1);
    cbar();
  }
  if (A.prof && tid == 0) {
    long long* o = A.prof + (long)blockIdx.x * 8;
    o[0] = 0; o[1] = 0; o[2] = 0; o[3] = total; o[4] = xwait;
    o[5] = clock64() - t_start; o[6] = reducer ? 1 : 0; o[7] = d;
  }
}

// ------------------------------------------------------------------ host
static constexpr int kFastSmemMax = 227 * 1024;
extern long long* helm_sweep_prof_buffer();

// Returns HELM_OK and launches if every direction fits the fast kernel
// (w <= 36); returns -1 (not applicable) otherwise.
int sweep_apply_fast(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                     cudaStream_t st) {
  using namespace fastk;
  int wmax = 0, pmax = 1, nsolve_max = 1;
  for (int d = 0; d < t; ++d) {
    wmax = std::max(wmax, dirs[d]->wmax);
    pmax = std::max(pmax, dirs[d]->P);
    nsolve_max = std::max(nsolve_max, dirs[d]->is_double ? 2 * dirs[d]->N - 1 : dirs[d]->N);
  }
  if (wmax > LPR * KPL || wmax > WM) return -1;
  nsolve_max = (nsolve_max + 1) & ~1;
  const int nw = (wmax + OWN - 1) / OWN;
  const int threads = nw * 32 + 32;
  long vec_elems = 0;
  int ctas = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    int mmax = 0;
    for (int p = 0; p < h->P; ++p) mmax = std::max(mmax, h->seg_hi[p] - h->seg_lo[p] + 1);
    vec_elems = std::max(vec_elems, (long)(mmax + 1) * h->wmax);
    vec_elems = std::max(vec_elems, (long)std::max(h->P - 1, 1) * WM);
    ctas += h->P + (h->P > 1 ? 1 : 0);
  }
  vec_elems = (vec_elems + 7) / 8 * 8;
  size_t head = sizeof(cplx) * (4 * WM + pmax) + sizeof(FastTab) * nsolve_max + 16;
  head = (head + 127) / 128 * 128;
  int sps_max = 1;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    int mmax = 0;
    for (int p = 0; p < h->P; ++p) mmax = std::max(mmax, h->seg_hi[p] - h->seg_lo[p] + 1);
    sps_max = std::max(sps_max, (h->P > 1 ? 2 : 1) * (2 * mmax - 1));
    sps_max = std::max(sps_max, 3 * h->P);
  }
  size_t smem = head + sizeof(cplx) * 5 * vec_elems + sizeof(StepEnt) * sps_max;
  if (smem > (size_t)kFastSmemMax) return -1;
  // per-direction scratch (same layout as the general kernel)
  std::vector<size_t> off(t);
  size_t total = 0;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    off[d] = total;
    total += al(sizeof(unsigned) * 2);
    total += al(sizeof(cplx) * 2L * h->P * h->wmax) * 2;
    total += al(sizeof(cplx) * (long)std::max(h->P - 1, 1) * h->wmax);
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
    D.fac = h->d_fac; D.fac_off = h->d_fac_off; D.red = h->d_red; D.red_off = h->d_red_off;
    D.R = Rdev + (ldr == 0 ? 0 : (long)d * ldr);
    D.Z = Zdev + (long)d * ldz;
    unsigned char* q = scratch + off[d];
    D.cnt = (unsigned*)q; q += al(sizeof(unsigned) * 2);
    D.yb = (cplx*)q; q += al(sizeof(cplx) * 2L * h->P * h->wmax);
    D.xb = (cplx*)q; q += al(sizeof(cplx) * 2L * h->P * h->wmax);
    D.xs = (cplx*)q; q += al(sizeof(cplx) * (long)std::max(h->P - 1, 1) * h->wmax);
    D.corr_prev = (cplx*)q; q += al(sizeof(cplx) * (long)h->N * h->nc);
    D.corr_next = (cplx*)q;
    D.wmax = h->wmax;
    D.cta_base = base;
    base += h->P + (h->P > 1 ? 1 : 0);
    if (e == cudaSuccess) e = cudaMemsetAsync(D.cnt, 0, sizeof(unsigned) * 2, st);
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
