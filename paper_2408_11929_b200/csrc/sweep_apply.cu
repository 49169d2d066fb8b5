// sweep_apply.cu -- hot-path row a4: z = M^{-1} r for t directional double
// sweeps, all directions batched in ONE persistent cooperative launch
// ("we can perform this part fully in parallel").
//
// The sweep (Eq. 2a-3c), per direction:
//   forward  v_{s1} = A^{-1} R r,  v_{sm} = A^{-1}(R r + C^prev(v_{s(m-1)}))
//   backward u_{sN} = v_{sN},      u_{sm} = A^{-1}(R r + C^prev(v_{s(m-1)}) + C^next(u_{s(m+1)}))
//   gather: u_{sN}, ..., u_{s1} written in that order ("most recent"),
// with C the 5-point transmission stencils (D8) precomputed by sweep_setup.
//
// Each local solve A_s x = b is the partitioned block-Thomas solve of
// strip_setup.cu: per direction, P "segment" CTAs and one
// "reducer" CTA:
//   phase 1 (segments, parallel): y_p = A_p^{-1} b_p       (fwd + bwd block sweep)
//   phase 2 (reducer):  g_k = b_{s_k} - L y_k[hi] - U y_{k+1}[lo];
//                       x_sep = Rsep^{-1} g               (block-Thomas, dense couplings)
//   phase 3 (segments): x_p = A_p^{-1}(b_p - A_{p,sep} x_sep)
// CTAs synchronise through per-direction arrival counters in global memory
// (release/acquire); co-residency is guaranteed by the cooperative launch.
//
// Data movement: every dense w x w factor block (explicit Schur inverse) is
// streamed HBM/L2 -> shared memory by the TMA bulk-copy engine
// (cp.async.bulk + mbarrier complete_tx) through an NSTAGE ring that runs
// ahead of the dependent chain across phase boundaries; one elected thread
// issues the copies.  The dependent block step is a shared-memory mat-vec:
// 8 lanes per output row (interleaved columns, bank-conflict free) and a
// 3-level xor-shuffle reduction; the sparse coupling L y / U x of the next
// step is folded into the producer lanes (one __syncthreads per block step).
#include <algorithm>
#include <cstring>

#include "common.cuh"

#define HELM_MAXDIR 8

struct DirArgs {
  int axis, order, N, P, nc, nxp1, is_double, ntile_max;
  const int *a, *w, *own_lo, *own_hi, *seg_lo, *seg_hi;
  const cplx *cr, *ne;   // bands: U_c couplings, stride wmax per row, nc*wmax per strip
  const cplx* tc;        // transmission stencils [s][side][c][5]
  const cplx* fac;
  const long* fac_off;
  const cplx* red;
  const long* red_off;
  const cplx* R;         // source column
  cplx* Z;               // output column
  cplx *yb, *xs, *xb, *corr_prev, *corr_next;
  unsigned* cnt;         // [0] segment arrivals, [1] reducer releases
  int wmax;
  int cta_base;
  int vec_rows;
};

struct ApplyArgs {
  DirArgs d[HELM_MAXDIR];
  int t;
  int rows_per_tile;  // R_t = blockDim/8
  int nstage;
  int stage_elems;    // cplx per stage
  int vec_elems;      // cplx per vector area (bseg / yseg)
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
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ cplx ldcg(const cplx* p) { return __ldcg(p); }

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
template <class XF>
__device__ __forceinline__ cplx correction(const DirArgs& D, int t, int side, int c, int a_src, XF X) {
  const cplx* k = D.tc + (((long)t * 2 + side) * D.nc + c) * 5;
  int at = D.a[t], bt = at + D.w[t] - 1;
  int qi, qo, dd;
  if (side == 0) { qi = at - a_src; qo = at - 1 - a_src; dd = -1; }
  else { qi = bt - a_src; qo = bt + 1 - a_src; dd = 1; }
  cplx acc = cmul(__ldg(k + 1), X(c, qi));
  cfma(acc, __ldg(k + 3), X(c, qo));
  if (c >= 1) cfma(acc, __ldg(k + 0), X(c - 1, qi));
  if (c + 1 < D.nc) cfma(acc, __ldg(k + 2), X(c + 1, qi));
  if (c + dd >= 0 && c + dd < D.nc) cfma(acc, __ldg(k + 4), X(c + dd, qo));
  return acc;
}

// ------------------------------------------------------------------ tile pipeline
struct Ring {
  uint64_t* bar;     // nstage mbarriers
  cplx* stage;       // nstage * stage_elems
  int nstage, stage_elems, R_t;
  uint32_t kc;       // consumer tile counter
  uint32_t kp;       // producer tile counter (thread 0)
};

__device__ __forceinline__ void ring_issue(Ring& rg, const cplx* src, uint32_t bytes) {
  // thread 0 only
  int sidx = rg.kp % rg.nstage;
  mbar_expect_tx(&rg.bar[sidx], bytes);
  bulk_g2s(rg.stage + (long)sidx * rg.stage_elems, src, bytes, &rg.bar[sidx]);
  rg.kp++;
}
__device__ __forceinline__ const cplx* ring_wait(Ring& rg) {
  int sidx = rg.kc % rg.nstage;
  mbar_wait(&rg.bar[sidx], (rg.kc / rg.nstage) & 1);
  return rg.stage + (long)sidx * rg.stage_elems;
}

// Producer cursors: the exact tile sequence the consumer will ask for.
struct SegCursor {
  int i, ph, j, tt;   // solve, phase index, step, tile
  bool done;
};
struct RedCursor {
  int i, part, k, tt, sub;  // solve, part (0 fwd, 1 bwd), separator, tile, sub-block
  bool done;
};

__device__ __forceinline__ int ntile_of(int w, int R_t) { return (w + R_t - 1) / R_t; }

__device__ bool seg_next_tile(const DirArgs& D, int p, int R_t, SegCursor& c, const cplx** src, uint32_t* bytes) {
  if (c.done) return false;
  const int lo = D.seg_lo[p], hi = D.seg_hi[p], m = hi - lo + 1;
  const int nph = D.P > 1 ? 2 : 1;
  const int s = sigma(D, step_of(D, c.i));
  const int w = D.w[s];
  const int nt = ntile_of(w, R_t);
  int row = c.j < m ? lo + c.j : hi - 1 - (c.j - m);
  int r0 = c.tt * R_t;
  int rows = min(R_t, w - r0);
  *src = D.fac + D.fac_off[s] + (long)row * w * w + (long)r0 * w;
  *bytes = (uint32_t)(rows * w * sizeof(cplx));
  // advance
  if (++c.tt == nt) {
    c.tt = 0;
    if (++c.j == 2 * m - 1) {
      c.j = 0;
      if (++c.ph == nph) {
        c.ph = 0;
        if (++c.i == n_solves(D)) c.done = true;
      }
    }
  }
  return true;
}

__device__ bool red_next_tile(const DirArgs& D, int R_t, RedCursor& c, const cplx** src, uint32_t* bytes) {
  if (c.done) return false;
  const int P = D.P;
  const int s = sigma(D, step_of(D, c.i));
  const int w = D.w[s];
  const int nt = ntile_of(w, R_t);
  const long w2 = (long)w * w;
  const cplx* base = D.red + D.red_off[s];
  int blk;  // 0 Rinv, 1 G, 2 F
  if (c.part == 0) blk = c.sub;  // sub 0 = Rinv_k, sub 1 = G_k
  else blk = 2;
  int r0 = c.tt * R_t;
  int rows = min(R_t, w - r0);
  *src = base + ((long)c.k * 3 + blk) * w2 + (long)r0 * w;
  *bytes = (uint32_t)(rows * w * sizeof(cplx));
  // advance: part 0: for k in 0..P-2: for tt: [Rinv tt, (k>=1) G tt]; part 1: for k = P-3..0: F tt
  if (c.part == 0) {
    if (c.sub == 0 && c.k >= 1) { c.sub = 1; return true; }
    c.sub = 0;
    if (++c.tt < nt) return true;
    c.tt = 0;
    if (++c.k <= P - 2) return true;
    c.part = 1;
    c.k = P - 3;
    if (c.k >= 0) return true;
  } else {
    if (++c.tt < nt) return true;
    c.tt = 0;
    if (--c.k >= 0) return true;
  }
  // next solve
  c.part = 0; c.k = 0; c.tt = 0; c.sub = 0;
  if (++c.i == n_solves(D)) c.done = true;
  return true;
}

// ------------------------------------------------------------------ block step
// One dependent block step over the tiles of a w x w block:
//   acc[r] = sum_k B[r][k] * (tA[k] + tB[k])
//   out[r] = acc (mode 0: forward, y = S^{-1} t) or ybase[r] - acc (mode 1: x = y - S^{-1} t)
// and, in the producer lanes, the next step's input
//   next 0: none; next 1 (forward-style): tA'[r] = bn[r] - crn[r] out[r], tB'[r+1] = -nen[r] out[r]
//   next 2 (backward-style): tA'[r] = crn[r] out[r], tB'[r-1] = nen[r-1] out[r]
struct StepIO {
  const cplx* tA; const cplx* tB;    // inputs (smem)
  cplx* out;                          // output row vector (smem), length w
  const cplx* ybase;                  // mode 1 base (smem)
  int mode;
  int next;                           // 0 none, 1 fwd-style, 2 bwd-style
  const cplx* bn;                     // next fwd rhs (smem)
  const cplx* crn; const cplx* nen;   // next couplings (global)
  cplx* tAn; cplx* tBn;               // next inputs (smem)
};

template <class Refill>
__device__ __forceinline__ void block_step(Ring& rg, int w, const StepIO& io, Refill refill) {
  const int tid = threadIdx.x;
  const int ri = tid >> 3, q = tid & 7;
  const int nt = ntile_of(w, rg.R_t);
  // prefetch next-step coefficients (independent of this step's data)
  for (int tt = 0; tt < nt; ++tt) {
    const int r0 = tt * rg.R_t;
    const int rows = min(rg.R_t, w - r0);
    const int r = r0 + ri;
    cplx crv = cmk(0, 0), nev = cmk(0, 0), nem = cmk(0, 0), bnv = cmk(0, 0);
    if (q == 0 && ri < rows && io.next) {
      crv = __ldg(io.crn + r);
      if (io.next == 1) { nev = __ldg(io.nen + r); bnv = io.bn[r]; }
      else if (r >= 1) nem = __ldg(io.nen + r - 1);
    }
    const cplx* B = ring_wait(rg);
    cplx acc = cmk(0, 0);
    if (ri < rows) {
      const cplx* Br = B + ri * w;
#pragma unroll 4
      for (int k = q; k < w; k += 8) {
        cplx v = cadd(io.tA[k], io.tB[k]);
        cfma(acc, Br[k], v);
      }
    }
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (q == 0 && ri < rows) {
      cplx o = io.mode == 0 ? acc : csub(io.ybase[r], acc);
      io.out[r] = o;
      if (io.next == 1) {
        io.tAn[r] = csub(bnv, cmul(crv, o));
        if (r + 1 < w) io.tBn[r + 1] = cscale(cmul(nev, o), -1.0);
        if (r == 0) io.tBn[0] = cmk(0, 0);
      } else if (io.next == 2) {
        io.tAn[r] = cmul(crv, o);
        if (r >= 1) io.tBn[r - 1] = cmul(nem, o);
        if (r == w - 1) io.tBn[w - 1] = cmk(0, 0);
      }
    }
    __syncthreads();
    refill();
  }
}

// two-block step for the reducer forward chain: out = A*u - B*v  (tile-interleaved A, B)
template <class Refill>
__device__ __forceinline__ void block_step2(Ring& rg, int w, const cplx* u, const cplx* v, bool hasB,
                                            cplx* out, Refill refill) {
  const int tid = threadIdx.x;
  const int ri = tid >> 3, q = tid & 7;
  const int nt = ntile_of(w, rg.R_t);
  for (int tt = 0; tt < nt; ++tt) {
    const int r0 = tt * rg.R_t;
    const int rows = min(rg.R_t, w - r0);
    const cplx* A = ring_wait(rg);
    rg.kc++;
    const cplx* B = nullptr;
    if (hasB) B = ring_wait(rg);
    rg.kc--;  // restore: refill() advances kc per consumed tile
    cplx acc = cmk(0, 0);
    if (ri < rows) {
      const cplx* Ar = A + ri * w;
      for (int k = q; k < w; k += 8) cfma(acc, Ar[k], u[k]);
      if (hasB) {
        const cplx* Br = B + ri * w;
        for (int k = q; k < w; k += 8) cfma(acc, Br[k], cscale(v[k], -1.0));
      }
    }
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (q == 0 && ri < rows) out[r0 + ri] = acc;
    __syncthreads();
    refill();
    if (hasB) refill();
  }
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(288, 1) k_sweep_apply(const __grid_constant__ ApplyArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  // which direction / role
  int d = 0;
  while (d + 1 < A.t && (int)blockIdx.x >= A.d[d + 1].cta_base) ++d;
  const DirArgs& D = A.d[d];
  const int role = blockIdx.x - D.cta_base;  // 0..P-1 segments, P = reducer
  const bool reducer = (D.P > 1 && role == D.P);

  Ring rg;
  rg.bar = reinterpret_cast<uint64_t*>(smem_raw);
  rg.stage = reinterpret_cast<cplx*>(smem_raw + 128);
  rg.nstage = A.nstage;
  rg.stage_elems = A.stage_elems;
  rg.R_t = A.rows_per_tile;
  rg.kc = 0;
  rg.kp = 0;
  cplx* vec0 = rg.stage + (long)A.nstage * A.stage_elems;  // bseg / g
  cplx* vec1 = vec0 + A.vec_elems;                           // yseg / z
  cplx* tbuf = vec1 + A.vec_elems;                           // 4 * wmax: tA0 tB0 tA1 tB1
  cplx* xlo = tbuf + 4 * D.wmax;                             // separator x above (p-1)
  cplx* xhi = xlo + D.wmax;                                  // separator x below (p)
  cplx* cnx = xhi + D.wmax;                                  // reducer: next-side corrections (P-1)

  if (tid == 0) {
    for (int s = 0; s < A.nstage; ++s) mbar_init(&rg.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int nsolve = n_solves(D);
  SegCursor sc{0, 0, 0, 0, false};
  RedCursor rc{0, 0, 0, 0, 0, false};
  const int p = role;
  auto next_tile = [&](const cplx** src, uint32_t* bytes) -> bool {
    return reducer ? red_next_tile(D, rg.R_t, rc, src, bytes) : seg_next_tile(D, p, rg.R_t, sc, src, bytes);
  };
  if (tid == 0) {
    const cplx* src;
    uint32_t bytes;
    for (int s = 0; s < A.nstage; ++s) {
      if (!next_tile(&src, &bytes)) break;
      ring_issue(rg, src, bytes);
    }
  }
  auto refill = [&]() {
    // called by all threads after the __syncthreads that ends a tile's use
    if (tid == 0) {
      const cplx* src;
      uint32_t bytes;
      if (next_tile(&src, &bytes)) ring_issue(rg, src, bytes);
    }
    rg.kc++;
  };

  const long band_stride = (long)D.nc * D.wmax;

  if (!reducer) {
    // ================================================================ segment CTA
    const int lo = D.seg_lo[p], hi = D.seg_hi[p], m = hi - lo + 1;
    cplx* bseg = vec0;
    cplx* yseg = vec1;
    for (int i = 0; i < nsolve; ++i) {
      const int st = step_of(D, i);
      const bool bwd = is_bwd(D, i);
      const int s = sigma(D, st);
      const int a = D.a[s], w = D.w[s];
      const int qp = prev_side(D) == 0 ? 0 : w - 1;
      const int qn = next_side(D) == 0 ? 0 : w - 1;
      const bool has_prev = st > 0;
      const bool has_next = bwd;  // backward solves carry C^next(u_{s(m+1)})
      const cplx* rsrc = D.R;
      const cplx* cband = D.cr + s * band_stride;
      const cplx* nband = D.ne + s * band_stride;
      // ---- RHS: R_s r + corrections (rows lo..hi)
      for (int e = tid; e < m * w; e += blockDim.x) {
        int cl = e / w, q = e % w, c = lo + cl;
        cplx v = __ldg(rsrc + node_of(D, a, c, q));
        if (has_prev && q == qp) v = cadd(v, D.corr_prev[(long)st * D.nc + c]);
        if (has_next && q == qn) v = cadd(v, D.corr_next[c]);
        bseg[cl * w + q] = v;
      }
      __syncthreads();

      // block-Thomas over the segment: fwd y_c = Sinv_c (b_c - L_c y_{c-1}); bwd x_c = y_c - Sinv_c U_c x_{c+1}
      auto thomas = [&]() {
        cplx* tA[2] = {tbuf, tbuf + 2 * D.wmax};
        cplx* tB[2] = {tbuf + D.wmax, tbuf + 3 * D.wmax};
        for (int e = tid; e < w; e += blockDim.x) { tA[0][e] = bseg[e]; tB[0][e] = cmk(0, 0); }
        __syncthreads();
        int cur = 0;
        for (int j = 0; j < m; ++j) {  // forward
          const int c = lo + j;
          StepIO io;
          io.tA = tA[cur]; io.tB = tB[cur];
          io.out = yseg + j * w; io.ybase = nullptr; io.mode = 0;
          if (j + 1 < m) {
            io.next = 1; io.bn = bseg + (j + 1) * w; io.crn = cband + (long)c * D.wmax; io.nen = nband + (long)c * D.wmax;
          } else if (m > 1) {
            io.next = 2; io.bn = nullptr; io.crn = cband + (long)(hi - 1) * D.wmax; io.nen = nband + (long)(hi - 1) * D.wmax;
          } else {
            io.next = 0; io.bn = nullptr; io.crn = nullptr; io.nen = nullptr;
          }
          io.tAn = tA[cur ^ 1]; io.tBn = tB[cur ^ 1];
          block_step(rg, w, io, refill);
          cur ^= 1;
        }
        for (int c = hi - 1; c >= lo; --c) {  // backward
          const int j = c - lo;
          StepIO io;
          io.tA = tA[cur]; io.tB = tB[cur];
          io.out = yseg + j * w; io.ybase = yseg + j * w; io.mode = 1;
          if (c > lo) {
            io.next = 2; io.bn = nullptr; io.crn = cband + (long)(c - 1) * D.wmax; io.nen = nband + (long)(c - 1) * D.wmax;
          } else {
            io.next = 0; io.bn = nullptr; io.crn = nullptr; io.nen = nullptr;
          }
          io.tAn = tA[cur ^ 1]; io.tBn = tB[cur ^ 1];
          block_step(rg, w, io, refill);
          cur ^= 1;
        }
      };

      if (D.P > 1) {
        // ---- phase 1: y_p = A_p^{-1} b_p; publish y[lo], y[hi]
        thomas();
        cplx* yb = D.yb + (long)p * 2 * D.wmax;
        for (int e = tid; e < w; e += blockDim.x) {
          yb[e] = yseg[e];
          yb[D.wmax + e] = yseg[(m - 1) * w + e];
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          red_release_add(&D.cnt[0], 1u);
          while (ld_acquire(&D.cnt[1]) < (unsigned)(i + 1)) __nanosleep(64);
          __threadfence();
        }
        __syncthreads();
        // ---- phase 3 RHS: b_lo -= U_{lo-1}^T x_sep[p-1]; b_hi -= U_hi x_sep[p]
        for (int e = tid; e < w; e += blockDim.x) {
          xlo[e] = p > 0 ? ldcg(D.xs + (long)(p - 1) * D.wmax + e) : cmk(0, 0);
          xhi[e] = p < D.P - 1 ? ldcg(D.xs + (long)p * D.wmax + e) : cmk(0, 0);
        }
        __syncthreads();
        for (int q = tid; q < w; q += blockDim.x) {
          if (p > 0) {
            const cplx* crr = cband + (long)(lo - 1) * D.wmax;
            const cplx* ner = nband + (long)(lo - 1) * D.wmax;
            cplx t = cmul(__ldg(crr + q), xlo[q]);
            if (q >= 1) cfma(t, __ldg(ner + q - 1), xlo[q - 1]);
            bseg[q] = csub(bseg[q], t);
          }
          if (p < D.P - 1) {
            const cplx* crr = cband + (long)hi * D.wmax;
            const cplx* ner = nband + (long)hi * D.wmax;
            cplx t = cmul(__ldg(crr + q), xhi[q]);
            if (q + 1 < w) cfma(t, __ldg(ner + q), xhi[q + 1]);
            bseg[(m - 1) * w + q] = csub(bseg[(m - 1) * w + q], t);
          }
        }
        __syncthreads();
      }
      // ---- phase 3 (or the whole solve when P == 1)
      thomas();
      // ---- epilogue: gather, boundary rows, next correction
      if (writes_Z(D, i)) {
        const int olo = D.own_lo[s], ohi = D.own_hi[s], ow = ohi - olo + 1;
        for (int e = tid; e < m * ow; e += blockDim.x) {
          int cl = e / ow, q = olo + e % ow;
          D.Z[node_of(D, a, lo + cl, q)] = yseg[cl * w + q];
        }
      }
      if (D.P > 1) {
        cplx* xb = D.xb + (long)p * 2 * D.wmax;
        for (int e = tid; e < w; e += blockDim.x) {
          xb[e] = yseg[e];
          xb[D.wmax + e] = yseg[(m - 1) * w + e];
        }
      }
      // correction for the next solve (destination strip t, side, target array)
      int tdst = -1, side = 0;
      cplx* target = nullptr;
      if (!bwd) {
        if (st < D.N - 1) { tdst = sigma(D, st + 1); side = prev_side(D); target = D.corr_prev + (long)(st + 1) * D.nc; }
        else if (D.is_double && D.N > 1) { tdst = sigma(D, D.N - 2); side = next_side(D); target = D.corr_next; }
      } else if (st >= 1) {
        tdst = sigma(D, st - 1); side = next_side(D); target = D.corr_next;
      }
      if (tdst >= 0) {
        auto X = [&](int cc, int q) -> cplx {
          if (cc < lo) return xlo[q];
          if (cc > hi) return xhi[q];
          return yseg[(cc - lo) * w + q];
        };
        for (int c = lo + tid; c <= hi; c += blockDim.x) target[c] = correction(D, tdst, side, c, a, X);
      }
      __syncthreads();
    }
  } else {
    // ================================================================ reducer CTA
    const int P = D.P, K = P - 1;
    cplx* g = vec0;   // K x wmax: reduced RHS
    cplx* z = vec1;   // K x wmax: forward results, then x_sep (in place)
    for (int i = 0; i < nsolve; ++i) {
      const int st = step_of(D, i);
      const bool bwd = is_bwd(D, i);
      const int s = sigma(D, st);
      const int a = D.a[s], w = D.w[s];
      const int qp = prev_side(D) == 0 ? 0 : w - 1;
      const int qn = next_side(D) == 0 ? 0 : w - 1;
      const cplx* cband = D.cr + s * band_stride;
      const cplx* nband = D.ne + s * band_stride;
      if (tid == 0) {
        while (ld_acquire(&D.cnt[0]) < (unsigned)(P * (i + 1))) __nanosleep(32);
        __threadfence();
      }
      __syncthreads();
      // (a) separator-row corrections from the previous solve's solution
      if (i >= 1) {
        const int sprev = sigma(D, step_of(D, i - 1));
        const int aprev = D.a[sprev];
        const int wprev = D.w[sprev];
        const int side = bwd ? next_side(D) : prev_side(D);
        for (int k = tid; k < K; k += blockDim.x) {
          const int sk = D.seg_hi[k] + 1;
          auto X = [&](int cc, int q) -> cplx {
            if (cc == sk) return z[k * D.wmax + q];
            if (cc == sk - 1) return ldcg(D.xb + (long)k * 2 * D.wmax + D.wmax + q);
            return ldcg(D.xb + (long)(k + 1) * 2 * D.wmax + q);  // cc == sk + 1
          };
          (void)wprev;
          cplx cv = correction(D, s, side, sk, aprev, X);
          if (!bwd) D.corr_prev[(long)st * D.nc + sk] = cv;
          else cnx[k] = cv;
        }
        __syncthreads();
      }
      // (b) reduced RHS g_k = b_{s_k} - U_{h_k}^T y_k[hi] - U_{s_k} y_{k+1}[lo]
      for (int e = tid; e < K * w; e += blockDim.x) {
        const int k = e / w, q = e % w;
        const int hk = D.seg_hi[k], sk = hk + 1;
        cplx v = __ldg(D.R + node_of(D, a, sk, q));
        if (st > 0 && q == qp) v = cadd(v, D.corr_prev[(long)st * D.nc + sk]);
        if (bwd && q == qn) v = cadd(v, cnx[k]);
        const cplx* yh = D.yb + (long)k * 2 * D.wmax + D.wmax;     // y_k[hi]
        const cplx* yl = D.yb + (long)(k + 1) * 2 * D.wmax;        // y_{k+1}[lo]
        cplx t = cmul(__ldg(cband + (long)hk * D.wmax + q), ldcg(yh + q));
        if (q >= 1) cfma(t, __ldg(nband + (long)hk * D.wmax + q - 1), ldcg(yh + q - 1));
        cfma(t, __ldg(cband + (long)sk * D.wmax + q), ldcg(yl + q));
        if (q + 1 < w) cfma(t, __ldg(nband + (long)sk * D.wmax + q), ldcg(yl + q + 1));
        g[k * D.wmax + q] = csub(v, t);
      }
      __syncthreads();
      // (c) block-Thomas on the separator system
      for (int k = 0; k < K; ++k) {
        block_step2(rg, w, g + k * D.wmax, k >= 1 ? z + (k - 1) * D.wmax : nullptr, k >= 1,
                    z + k * D.wmax, refill);
      }
      for (int k = K - 2; k >= 0; --k) {
        StepIO io;
        io.tA = z + (k + 1) * D.wmax;
        io.tB = tbuf;  // zeros
        if (k == K - 2) {
          for (int e = tid; e < w; e += blockDim.x) tbuf[e] = cmk(0, 0);
          __syncthreads();
        }
        io.out = z + k * D.wmax; io.ybase = z + k * D.wmax; io.mode = 1;
        io.next = 0; io.bn = nullptr; io.crn = nullptr; io.nen = nullptr; io.tAn = nullptr; io.tBn = nullptr;
        block_step(rg, w, io, refill);
      }
      // (d) publish x_sep
      for (int e = tid; e < K * w; e += blockDim.x) {
        const int k = e / w, q = e % w;
        D.xs[(long)k * D.wmax + q] = z[k * D.wmax + q];
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release(&D.cnt[1], (unsigned)(i + 1));
      }
      // (e) gather separator rows
      if (writes_Z(D, i)) {
        const int olo = D.own_lo[s], ohi = D.own_hi[s], ow = ohi - olo + 1;
        for (int e = tid; e < K * ow; e += blockDim.x) {
          const int k = e / ow, q = olo + e % ow;
          D.Z[node_of(D, a, D.seg_hi[k] + 1, q)] = z[k * D.wmax + q];
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ host
static constexpr int kSmemMax = 227 * 1024;

int sweep_apply_dev(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                    cudaStream_t st);

extern "C" int sweep_apply(const helm_sweep_t* dirs, int t, const double* Rin, long ldr, double* Zout,
                           long ldz, void* stream) {
  if (!dirs || !Rin || !Zout || t < 1 || t > HELM_MAXDIR) {
    helm_set_error("sweep_apply: need 1 <= t <= %d and non-null R, Z", HELM_MAXDIR);
    return HELM_EINVAL;
  }
  const helm_problem_s* prob = dirs[0]->prob;
  for (int d = 0; d < t; ++d) {
    if (!dirs[d]) { helm_set_error("sweep_apply: null direction handle"); return HELM_EINVAL; }
    if (dirs[d]->prob->n != prob->n || dirs[d]->prob->nx != prob->nx) {
      helm_set_error("sweep_apply: direction %d belongs to a different problem size", d);
      return HELM_EDIM;
    }
  }
  const long n = prob->n;
  if (ldr != 0 && ldr < n) { helm_set_error("sweep_apply: ldr < n"); return HELM_EINVAL; }
  if (ldz < n) { helm_set_error("sweep_apply: ldz < n"); return HELM_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  Staged sR, sZ;
  size_t rbytes = sizeof(cplx) * (ldr == 0 ? n : ldr * (t - 1) + n);
  size_t zbytes = sizeof(cplx) * (ldz * (t - 1) + n);
  HELM_TRY(helm_stage_in(Rin, rbytes, true, st, sR));
  HELM_TRY(helm_stage_in(Zout, zbytes, false, st, sZ));
  int rc = sweep_apply_dev(dirs, t, (const cplx*)sR.dev, ldr, (cplx*)sZ.dev, ldz, st);
  helm_stage_free(sR, st);
  if (rc != HELM_OK) {
    helm_stage_free(sZ, st);
    return rc;
  }
  return helm_stage_out(sZ, st);
}

int sweep_apply_dev(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                    cudaStream_t st) {
  const helm_problem_s* prob = dirs[0]->prob;
  // launch geometry
  int wmax = 0;
  for (int d = 0; d < t; ++d) wmax = std::max(wmax, dirs[d]->wmax);
  int threads = std::min(1024, ((8 * std::min(wmax, 36) + 31) / 32) * 32);
  const int R_t = threads / 8;
  long vec_elems = 0, stage_elems = 0;
  int ctas = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    int mmax = 0;
    for (int p = 0; p < h->P; ++p) mmax = std::max(mmax, h->seg_hi[p] - h->seg_lo[p] + 1);
    int vr = std::max(mmax, std::max(h->P - 1, 1));
    vec_elems = std::max(vec_elems, (long)vr * h->wmax);
    stage_elems = std::max(stage_elems, (long)std::min(R_t, h->wmax) * h->wmax);
    ctas += h->P + (h->P > 1 ? 1 : 0);
  }
  vec_elems = (vec_elems + 7) / 8 * 8;
  stage_elems = (stage_elems + 7) / 8 * 8;
  int pmax = 1;
  for (int d = 0; d < t; ++d) pmax = std::max(pmax, dirs[d]->P);
  long fixed = 128 + sizeof(cplx) * (2 * vec_elems + 7L * wmax + pmax + 8);
  int nstage = (int)std::min<long>(8, (kSmemMax - fixed) / (long)(sizeof(cplx) * stage_elems));
  if (nstage < 2) {
    helm_set_error("sweep_apply: shared memory too small (w=%d)", wmax);
    return HELM_EINVAL;
  }
  size_t smem = fixed + sizeof(cplx) * (size_t)nstage * stage_elems;
  // per-direction scratch
  std::vector<size_t> off(t);
  size_t total = 0;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    off[d] = total;
    total += al(sizeof(unsigned) * 2);
    total += al(sizeof(cplx) * 2L * h->P * h->wmax) * 2;          // yb, xb
    total += al(sizeof(cplx) * (long)std::max(h->P - 1, 1) * h->wmax);  // xs
    total += al(sizeof(cplx) * (long)h->N * h->nc);                // corr_prev
    total += al(sizeof(cplx) * (long)h->nc);                       // corr_next
  }
  unsigned char* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, total, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply: scratch alloc: %s", cudaGetErrorString(e));
    return HELM_ENOMEM;
  }
  ApplyArgs A;
  memset(&A, 0, sizeof(A));
  A.t = t;
  A.rows_per_tile = R_t;
  A.nstage = nstage;
  A.stage_elems = (int)stage_elems;
  A.vec_elems = (int)vec_elems;
  int base = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    DirArgs& D = A.d[d];
    D.axis = h->axis; D.order = h->order; D.N = h->N; D.P = h->P; D.nc = h->nc;
    D.nxp1 = prob->nx + 1; D.is_double = h->is_double; D.ntile_max = (h->wmax + R_t - 1) / R_t;
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
    e = cudaMemsetAsync(D.cnt, 0, sizeof(unsigned) * 2, st);
    if (e != cudaSuccess) break;
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_sweep_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 0, occ = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep_apply, threads, smem);
  if (e == cudaSuccess && occ * nsm < ctas) {
    helm_set_error("sweep_apply: %d CTAs cannot be co-resident (%d SMs x %d); reduce n_segments", ctas, nsm, occ);
    cudaFreeAsync(scratch, st);
    return HELM_ECUDA;
  }
  if (e == cudaSuccess) {
    void* args[] = {(void*)&A};
    e = cudaLaunchCooperativeKernel((void*)k_sweep_apply, dim3(ctas), dim3(threads), args, smem, st);
    g_helm_launches++;
  }
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply: launch: %s", cudaGetErrorString(e));
    return HELM_ECUDA;
  }
  return HELM_OK;
}
