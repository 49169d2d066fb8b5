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
#include <cstdlib>
#include <cstring>

#include "common.cuh"

#include "sweep_common.cuh"

#ifndef HELM_GEN_XPF
#define HELM_GEN_XPF 0     // 1: bulk L2 prefetch of the separator-inverse rows before the gather (C4 t = 1 / 4: 11.09 / 11.84 ms with, 10.55 / 11.02 without: 5 MB of rows per CTA overflow L2 and the issuing warp stalls in front of a barrier)
#endif
#ifndef HELM_GEN_XUN
#define HELM_GEN_XUN 1     // iterations of the separator mat-vec's column loop unrolled (4 * XCH loads per lane each)
#endif
constexpr int kGenXun = HELM_GEN_XUN;
#ifndef HELM_GEN_XCH
#define HELM_GEN_XCH 6     // 32-column chunks per row and iteration (4 rows per warp: 24 loads per lane in flight;
                           // C4 t = 1: XCH/XUN 4/1 8.96, 4/2 8.13-8.77, 4/4 8.12, 8/1 8.31, 6/1 8.03 ms)
#endif
constexpr int kGenXch = HELM_GEN_XCH;
#ifndef HELM_GEN_XPIPE
#define HELM_GEN_XPIPE 0   // 1: pipelined L2 prefetch of the separator-inverse rows (wide strips)
#endif

// ------------------------------------------------------------------ tile pipeline
// Warp-specialised ring: the last warp of the CTA is the TMA producer (one
// elected lane walks the exact tile sequence the consumers will ask for and
// issues cp.async.bulk into stage f % NS after waiting for the consumers'
// release of fill f - NS); the consumer warps wait on full[stage], compute,
// sync among themselves with named barrier 1, and one thread releases the
// stage through empty[stage].  The producer therefore runs up to NS tiles
// ahead across step, phase and solve boundaries, off the dependent chain.
struct Ring {
  uint64_t* full;    // nstage mbarriers (tx-count)
  uint64_t* empty;   // nstage mbarriers (consumer release)
  cplx* stage;       // nstage * stage_elems
  int nstage, stage_elems, R_t;
  uint32_t kc;       // consumer tile counter
};

__device__ __forceinline__ void cbar(int ncons) {
  asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory");
}
__device__ __forceinline__ const cplx* ring_peek(const Ring& rg, uint32_t k) {
  int sidx = k % rg.nstage;
  mbar_wait(&rg.full[sidx], (k / rg.nstage) & 1);
  return rg.stage + (long)sidx * rg.stage_elems;
}
// consumers: release `count` consumed tiles.  Every consumer warp arrives once per
// stage (the empty barriers are initialised with the number of consumer warps), so a
// warp that is done with a tile frees its share without a CTA barrier.
__device__ __forceinline__ void ring_release(Ring& rg, int count) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0)
    for (int c = 0; c < count; ++c) mbar_arrive(&rg.empty[(rg.kc + c) % rg.nstage]);
  rg.kc += count;
}

// Producer cursors: the exact tile sequence the consumer will ask for.  All
// geometry comes from registers and a per-solve table in shared memory
// (strip width and factor base of solve i), so the producer warp issues a
// tile in a few tens of cycles.
struct SolveTab {
  const cplx* fac;   // factor base of the strip solved at solve i
  const cplx* red;   // separator-system base
  int w;
  int pad;
};
struct SegCursor {
  int i, ph, j, tt;   // solve, phase index, step, tile
  int lo, hi, m, nph, nsolve, R_t;
  int w, nt;
  const cplx* fac;
  bool done;
};
struct RedCursor {
  int i, part, k, tt, sub;  // solve, part (0 fwd, 1 bwd), separator, tile, sub-block
  int P, nsolve, R_t, w, nt;
  const cplx* red;
  bool done;
};

__device__ __forceinline__ int ntile_of(int w, int R_t) { return (w + R_t - 1) / R_t; }

__device__ __forceinline__ void seg_load_solve(SegCursor& c, const SolveTab* tab) {
  c.w = tab[c.i].w;
  c.fac = tab[c.i].fac;
  c.nt = ntile_of(c.w, c.R_t);
}

__device__ __forceinline__ bool seg_next_tile(SegCursor& c, const SolveTab* tab, const cplx** src, uint32_t* bytes) {
  if (c.done) return false;
  const int w = c.w;
  int row = c.j < c.m ? c.lo + c.j : c.hi - 1 - (c.j - c.m);
  int r0 = c.tt * c.R_t;
  int rows = min(c.R_t, w - r0);
  *src = c.fac + (long)row * w * w + (long)r0 * w;
  *bytes = (uint32_t)(rows * w * sizeof(cplx));
  if (++c.tt == c.nt) {
    c.tt = 0;
    if (++c.j == 2 * c.m - 1) {
      c.j = 0;
      if (++c.ph == c.nph) {
        c.ph = 0;
        if (++c.i == c.nsolve) c.done = true;
        else seg_load_solve(c, tab);
      }
    }
  }
  return true;
}

__device__ __forceinline__ void red_load_solve(RedCursor& c, const SolveTab* tab) {
  c.w = tab[c.i].w;
  c.red = tab[c.i].red;
  c.nt = ntile_of(c.w, c.R_t);
}

__device__ __forceinline__ bool red_next_tile(RedCursor& c, const SolveTab* tab, const cplx** src, uint32_t* bytes) {
  if (c.done) return false;
  const int w = c.w;
  const long w2 = (long)w * w;
  const int blk = c.part == 0 ? c.sub : 2;  // 0 Rinv, 1 G, 2 F
  int r0 = c.tt * c.R_t;
  int rows = min(c.R_t, w - r0);
  *src = c.red + ((long)c.k * 3 + blk) * w2 + (long)r0 * w;
  *bytes = (uint32_t)(rows * w * sizeof(cplx));
  // part 0: for k in 0..P-2: for tt: [Rinv tt, (k>=1) G tt]; part 1: for k = P-3..0: F tt
  if (c.part == 0) {
    if (c.sub == 0 && c.k >= 1) { c.sub = 1; return true; }
    c.sub = 0;
    if (++c.tt < c.nt) return true;
    c.tt = 0;
    if (++c.k <= c.P - 2) return true;
    c.part = 1;
    c.k = c.P - 3;
    if (c.k >= 0) return true;
  } else {
    if (++c.tt < c.nt) return true;
    c.tt = 0;
    if (--c.k >= 0) return true;
  }
  c.part = 0; c.k = 0; c.tt = 0; c.sub = 0;
  if (++c.i == c.nsolve) c.done = true;
  else red_load_solve(c, tab);
  return true;
}

// ------------------------------------------------------------------ block step
// One dependent block step over the tiles of a w x w block:
//   acc[r] = sum_k B[r][k] * (tA[k] + tB[k])
//   out[r] = acc (mode 0: forward, y = S^{-1} t) or ybase[r] - acc (mode 1: x = y - S^{-1} t)
// and, in the writer lanes, the next step's input
//   next 0: none; next 1 (forward-style): tA'[r] = bn[r] - crn[r] out[r], tB'[r+1] = -nen[r] out[r]
//   next 2 (backward-style): tA'[r] = crn[r] out[r], tB'[r-1] = nen[r-1] out[r]
struct StepIO {
  const cplx* tA; const cplx* tB;    // inputs
  cplx* out;                          // output row vector, length w
  const cplx* ybase;                  // mode 1 base
  int mode;
  int next;                           // 0 none, 1 fwd-style, 2 bwd-style
  const cplx* bn;                     // next fwd rhs
  const cplx* crn; const cplx* nen;   // next couplings (staged)
  cplx* tAn; cplx* tBn;               // next inputs
};

// KP: complex entries per lane and block row (8 lanes per row: KP >= ceil(w / 8)).
// The combined input t = tA + tB is read once per block step into registers and
// serves every 36-row tile of the block; the tiles need no CTA barrier between
// them (each warp releases its share of a ring stage when it is done with it), only
// the end of the step does (the writers' next input).
template <int KP>
__device__ __forceinline__ void block_step(Ring& rg, int w, int ncons, const StepIO& io, Prof& pf) {
  const int tid = threadIdx.x;
  const int ri = tid >> 3, q = tid & 7;
  const int nt = ntile_of(w, rg.R_t);
  cplx tv[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i) {
    const int k = q + 8 * i;
    tv[i] = k < w ? cadd(io.tA[k], io.tB[k]) : cmk(0, 0);
  }
  for (int tt = 0; tt < nt; ++tt) {
    const int r0 = tt * rg.R_t;
    const int rows = min(rg.R_t, w - r0);
    const int r = r0 + ri;
    const bool writer = (q == 0 && ri < rows);
    // operands of the writer lanes, independent of this step's data
    cplx crv = cmk(0, 0), nev = cmk(0, 0), nem = cmk(0, 0), bnv = cmk(0, 0), ybv = cmk(0, 0);
    if (writer) {
      if (io.mode == 1) ybv = io.ybase[r];
      if (io.next) {
        crv = io.crn[r];
        if (io.next == 1) { nev = io.nen[r]; bnv = io.bn[r]; }
        else if (r >= 1) nem = io.nen[r - 1];
      }
    }
    long long c0 = clock64();
    const cplx* B = ring_peek(rg, rg.kc);
    long long c1 = clock64();
    cplx a0 = cmk(0, 0), a1 = cmk(0, 0), a2 = cmk(0, 0), a3 = cmk(0, 0);
    if (ri < rows) {
      const cplx* Br = B + ri * w + q;
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        if (q + 8 * i < w) {
          const cplx b = Br[8 * i];
          if ((i & 3) == 0) cfma(a0, b, tv[i]);
          else if ((i & 3) == 1) cfma(a1, b, tv[i]);
          else if ((i & 3) == 2) cfma(a2, b, tv[i]);
          else cfma(a3, b, tv[i]);
        }
      }
    }
    cplx acc = cadd(cadd(a0, a1), cadd(a2, a3));
    ring_release(rg, 1);   // this warp is done with the tile (its entries are in registers)
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (writer) {
      cplx o = io.mode == 0 ? acc : csub(ybv, acc);
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
    long long c2 = clock64();
    pf.peek += c1 - c0; pf.comp += c2 - c1; pf.steps++;
  }
  long long c2 = clock64();
  cbar(ncons);
  pf.bar += clock64() - c2;
}

// two-block step for the reducer forward chain: out = A*u - B*v  (tile-interleaved A, B)
__device__ __forceinline__ void block_step2(Ring& rg, int w, int ncons, const cplx* u, const cplx* v, bool hasB,
                                            cplx* out, Prof& pf) {
  const int tid = threadIdx.x;
  const int ri = tid >> 3, q = tid & 7;
  const int nt = ntile_of(w, rg.R_t);
  for (int tt = 0; tt < nt; ++tt) {
    const int r0 = tt * rg.R_t;
    const int rows = min(rg.R_t, w - r0);
    long long c0 = clock64();
    const cplx* A = ring_peek(rg, rg.kc);
    const cplx* B = hasB ? ring_peek(rg, rg.kc + 1) : nullptr;
    long long c1 = clock64();
    cplx acc0 = cmk(0, 0), acc1 = cmk(0, 0);
    if (ri < rows) {
      const cplx* Ar = A + ri * w;
      for (int k = q; k < w; k += 8) cfma(acc0, Ar[k], u[k]);
      if (hasB) {
        const cplx* Br = B + ri * w;
        for (int k = q; k < w; k += 8) cfma(acc1, Br[k], v[k]);
      }
    }
    cplx acc = csub(acc0, acc1);
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (q == 0 && ri < rows) out[r0 + ri] = acc;
    long long c2 = clock64();
    cbar(ncons);
    ring_release(rg, hasB ? 2 : 1);
    long long c3 = clock64();
    pf.peek += c1 - c0; pf.comp += c2 - c1; pf.bar += c3 - c2; pf.steps++;
  }
}

// ------------------------------------------------------------------ kernel
// blockDim = ncons consumer threads (8 lanes per block row) + 1 producer warp.
template <int KP>
__global__ void __launch_bounds__(320, 1) k_sweep_apply(const __grid_constant__ ApplyArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int ncons = blockDim.x - 32;
  // which direction / role
  int d = 0;
  while (d + 1 < A.t && (int)blockIdx.x >= A.d[d + 1].cta_base) ++d;
  const DirArgs& D = A.d[d];
  const int role = blockIdx.x - D.cta_base;  // 0..P-1 segments, P = reducer
  const bool reducer = (D.P > 1 && role == D.P);
  const int p = role;
  // X path: the segments solve the separator system with the explicit rows of
  // its inverse (as sweep_dual.cu does); the reducer CTA has nothing to do
  const bool xpath = D.P > 1 && D.xinv != nullptr;
  if (reducer && xpath) return;

  Ring rg;
  rg.full = reinterpret_cast<uint64_t*>(smem_raw);
  rg.empty = rg.full + 16;
  rg.stage = reinterpret_cast<cplx*>(smem_raw + 256);
  rg.nstage = A.nstage;
  rg.stage_elems = A.stage_elems;
  rg.R_t = A.rows_per_tile;
  rg.kc = 0;
  cplx* sm_tail = rg.stage + (long)A.nstage * A.stage_elems;
  cplx* tbuf = sm_tail;                  // 4 * wmax: tA0 tB0 tA1 tB1
  cplx* xlo = tbuf + 4 * D.wmax;         // separator x above (p-1)
  cplx* xhi = xlo + D.wmax;              // separator x below (p)
  cplx* cnx = xhi + D.wmax;              // reducer / X path: next-side corrections (P-1)
  cplx* cpx = cnx + A.pmax;              // X path: prev-side corrections (P-1)
  SolveTab* tab = reinterpret_cast<SolveTab*>(cpx + A.pmax);   // per-solve table (nsolve_max)
  cplx* vbase = reinterpret_cast<cplx*>(tab + A.nsolve_max);      // vector areas (smem) ...
  if (A.vec_global) vbase = A.vec_scratch + (long)blockIdx.x * 4 * A.vec_elems;  // ... or global
  cplx* vec0 = vbase;                    // bseg / g
  cplx* vec1 = vec0 + A.vec_elems;       // yseg / z
  cplx* bcr = vec1 + A.vec_elems;        // staged U couplings, rows lo-1..hi
  cplx* bne = bcr + A.vec_elems;

  if (tid == 0) {
    for (int s = 0; s < A.nstage; ++s) {
      mbar_init(&rg.full[s], 1);
      mbar_init(&rg.empty[s], ncons >> 5);   // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < n_solves(D); i += blockDim.x) {
    const int s = sigma(D, step_of(D, i));
    tab[i].fac = D.fac + D.fac_off[s];
    tab[i].red = D.red + D.red_off[s];
    tab[i].w = D.w[s];
  }
  __syncthreads();

  if (tid >= ncons) {
    // ================================================================ TMA producer warp
    if (tid == ncons) {
      SegCursor sc;
      RedCursor rc;
      if (!reducer) {
        sc.i = sc.ph = sc.j = sc.tt = 0;
        sc.lo = D.seg_lo[p]; sc.hi = D.seg_hi[p]; sc.m = sc.hi - sc.lo + 1;
        sc.nph = D.P > 1 ? 2 : 1; sc.nsolve = n_solves(D); sc.R_t = rg.R_t; sc.done = false;
        seg_load_solve(sc, tab);
      } else {
        rc.i = rc.part = rc.k = rc.tt = rc.sub = 0;
        rc.P = D.P; rc.nsolve = n_solves(D); rc.R_t = rg.R_t; rc.done = false;
        red_load_solve(rc, tab);
      }
      const cplx* src;
      uint32_t bytes;
      for (uint32_t f = 0;; ++f) {
        bool more = reducer ? red_next_tile(rc, tab, &src, &bytes) : seg_next_tile(sc, tab, &src, &bytes);
        if (!more) break;
        const int sidx = f % rg.nstage;
        if (f >= (uint32_t)rg.nstage) mbar_wait(&rg.empty[sidx], ((f / rg.nstage) - 1) & 1);
        mbar_expect_tx(&rg.full[sidx], bytes);
        bulk_g2s(rg.stage + (long)sidx * rg.stage_elems, src, bytes, &rg.full[sidx]);
      }
    }
    return;
  }

  const int nsolve = n_solves(D);
  const long band_stride = (long)D.nc * D.wmax;
  Prof pf;
  const long long t_start = clock64();

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
      const cplx* cband = D.cr + s * band_stride;
      const cplx* nband = D.ne + s * band_stride;
      // ---- RHS: R_s r + corrections (rows lo..hi); couplings of rows lo-1..hi
      for (int e = tid; e < m * w; e += ncons) {
        int cl = e / w, q = e % w, c = lo + cl;
        cplx v = __ldg(D.R + node_of(D, a, c, q));
        if (has_prev && q == qp) v = cadd(v, D.corr_prev[(long)st * D.nc + c]);
        if (has_next && q == qn) v = cadd(v, D.corr_next[c]);
        bseg[cl * w + q] = cscale(v, rhs_scale(D, c, q, w));
      }
      for (int e = tid; e < (m + 1) * w; e += ncons) {
        int cl = e / w, q = e % w, c = lo - 1 + cl;
        bcr[e] = c >= 0 ? __ldg(cband + (long)c * D.wmax + q) : cmk(0, 0);
        bne[e] = c >= 0 ? __ldg(nband + (long)c * D.wmax + q) : cmk(0, 0);
      }
      cbar(ncons);
      // staged couplings of row c: bcr + (c - lo + 1) * w
      auto crow = [&](int c) { return bcr + (long)(c - lo + 1) * w; };
      auto nrow = [&](int c) { return bne + (long)(c - lo + 1) * w; };

      // block-Thomas over the segment: fwd y_c = Sinv_c (b_c - L_c y_{c-1}); bwd x_c = y_c - Sinv_c U_c x_{c+1}
      auto thomas = [&]() {
        cplx* tA0 = tbuf;
        cplx* tB0 = tbuf + D.wmax;
        cplx* tA1 = tbuf + 2 * D.wmax;
        cplx* tB1 = tbuf + 3 * D.wmax;
        for (int e = tid; e < w; e += ncons) { tA0[e] = bseg[e]; tB0[e] = cmk(0, 0); }
        cbar(ncons);
        int cur = 0;
        for (int j = 0; j < m; ++j) {  // forward
          const int c = lo + j;
          StepIO io;
          io.tA = cur ? tA1 : tA0; io.tB = cur ? tB1 : tB0;
          io.tAn = cur ? tA0 : tA1; io.tBn = cur ? tB0 : tB1;
          io.out = yseg + j * w; io.ybase = nullptr; io.mode = 0;
          if (j + 1 < m) {
            io.next = 1; io.bn = bseg + (j + 1) * w; io.crn = crow(c); io.nen = nrow(c);
          } else if (m > 1) {
            io.next = 2; io.bn = nullptr; io.crn = crow(hi - 1); io.nen = nrow(hi - 1);
          } else {
            io.next = 0; io.bn = nullptr; io.crn = nullptr; io.nen = nullptr;
          }
          block_step<KP>(rg, w, ncons, io, pf);
          cur ^= 1;
        }
        for (int c = hi - 1; c >= lo; --c) {  // backward
          const int j = c - lo;
          StepIO io;
          io.tA = cur ? tA1 : tA0; io.tB = cur ? tB1 : tB0;
          io.tAn = cur ? tA0 : tA1; io.tBn = cur ? tB0 : tB1;
          io.out = yseg + j * w; io.ybase = yseg + j * w; io.mode = 1;
          if (c > lo) {
            io.next = 2; io.bn = nullptr; io.crn = crow(c - 1); io.nen = nrow(c - 1);
          } else {
            io.next = 0; io.bn = nullptr; io.crn = nullptr; io.nen = nullptr;
          }
          block_step<KP>(rg, w, ncons, io, pf);
          cur ^= 1;
        }
      };

      const int par = xpath ? (i & 1) : 0, ppar = par ^ 1;
      const long exs = 2L * D.P * D.wmax;   // parity strides of yb / xb and xs
      const long xss = (long)D.P * D.wmax;
      if (D.P > 1 && !xpath) {
        // ---- phase 1: y_p = A_p^{-1} b_p; publish y[lo], y[hi]
        thomas();
        cplx* yb = D.yb + (long)p * 2 * D.wmax;
        for (int e = tid; e < w; e += ncons) {
          yb[e] = yseg[e];
          yb[D.wmax + e] = yseg[(m - 1) * w + e];
        }
        cbar(ncons);
        long long cw0 = clock64();
        if (tid == 0) {
          __threadfence();
          red_release_add(&D.cnt[0], 1u);
          while (ld_relaxed(&D.cnt[1]) < (unsigned)(i + 1)) __nanosleep(20);
          (void)ld_acquire(&D.cnt[1]);
        }
        cbar(ncons);
        pf.xwait += clock64() - cw0;
        // ---- phase 3 RHS: b_lo -= U_{lo-1}^T x_sep[p-1]; b_hi -= U_hi x_sep[p]
        for (int e = tid; e < w; e += ncons) {
          xlo[e] = p > 0 ? ldcg(D.xs + (long)(p - 1) * D.wmax + e) : cmk(0, 0);
          xhi[e] = p < D.P - 1 ? ldcg(D.xs + (long)p * D.wmax + e) : cmk(0, 0);
        }
        cbar(ncons);
      } else if (D.P > 1) {
        // ---- phase 1: y_p = A_p^{-1} b_p; publish y[lo], y[hi] (parity buffers)
        thomas();
        const int K = D.P - 1;
        const long Kw = (long)K * w, xld = x_ld(K, w);
        if (HELM_GEN_XPF && p < D.P - 1 && tid < 32) {
          // this CTA's rows of the separator inverse into L2 during the gather
          // (HELM_GEN_XPIPE: only the rows of the mat-vec's first pass; each warp then
          // prefetches its next pass's rows while it computes the current one, so wide
          // strips -- 5 MB of rows per CTA at C4 -- do not overflow L2)
          const char* xp = reinterpret_cast<const char*>(D.xinv + D.xinv_off[s] + (long)p * w * xld);
          const long rows_pf = HELM_GEN_XPIPE ? std::min<long>(w, 4L * (ncons >> 5)) : w;
          const long bytes = rows_pf * xld * (long)sizeof(cplx);
          for (long o = (long)tid * 32768; o < bytes; o += 32L * 32768)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(xp + o),
                         "r"((uint32_t)(bytes - o < 32768L ? bytes - o : 32768L)) : "memory");
        }
        cplx* yb = D.yb + par * exs + (long)p * 2 * D.wmax;
        for (int e = tid; e < w; e += ncons) {
          yb[e] = yseg[e];
          yb[D.wmax + e] = yseg[(m - 1) * w + e];
        }
        cbar(ncons);
        long long cw0 = clock64();
        if (tid == 0) {
          __threadfence();
          red_release_add(&D.cnt[0], 1u);
          while (ld_relaxed(&D.cnt[0]) < (unsigned)(D.P * (i + 1))) __nanosleep(20);
          (void)ld_acquire(&D.cnt[0]);
        }
        cbar(ncons);
        pf.xwait += clock64() - cw0;
        // separator-row corrections (from solve i-1), every separator (reducer step (a))
        if (i >= 1) {
          const int aprev = D.a[sigma(D, step_of(D, i - 1))];
          for (int k = tid; k < K; k += ncons) {
            const int sk = D.seg_hi[k] + 1;
            auto X = [&](int cc, int q) -> cplx {
              if (cc == sk) return ldcg(D.xs + ppar * xss + (long)k * D.wmax + q);
              if (cc == sk - 1) return ldcg(D.xb + ppar * exs + (long)k * 2 * D.wmax + D.wmax + q);
              return ldcg(D.xb + ppar * exs + (long)(k + 1) * 2 * D.wmax + q);
            };
            cplx cp = cmk(0, 0), cn = cmk(0, 0);
            if (st > 0) {
              if (!bwd) {
                cp = correction(D, s, prev_side(D), sk, aprev, X);
                if (k == p) D.corr_prev[(long)st * D.nc + sk] = cp;   // kept for the backward pass
              } else {
                cp = ldcg(D.corr_prev + (long)st * D.nc + sk);
              }
            }
            if (bwd) cn = correction(D, s, next_side(D), sk, aprev, X);
            cpx[k] = cp;
            cnx[k] = cn;
          }
          cbar(ncons);
        }
        // g_k = b_{s_k} (+ corrections) - U_{h_k}^T y_k[hi] - U_{s_k} y_{k+1}[lo] (reducer step (b)), into yseg
        cplx* g = yseg;
        const cplx* ybp = D.yb + par * exs;
        for (int e = tid; e < K * w; e += ncons) {
          const int k = e / w, q = e % w;
          const int hk = D.seg_hi[k], sk = hk + 1;
          cplx v = __ldg(D.R + node_of(D, a, sk, q));
          if (st > 0 && q == qp) v = cadd(v, cpx[k]);
          if (bwd && q == qn) v = cadd(v, cnx[k]);
          v = cscale(v, rhs_scale(D, sk, q, w));
          const cplx* yh = ybp + (long)k * 2 * D.wmax + D.wmax;     // y_k[hi]
          const cplx* yl = ybp + (long)(k + 1) * 2 * D.wmax;        // y_{k+1}[lo]
          cplx t = cmul(__ldg(cband + (long)hk * D.wmax + q), ldcg(yh + q));
          if (q >= 1) cfma(t, __ldg(nband + (long)hk * D.wmax + q - 1), ldcg(yh + q - 1));
          cfma(t, __ldg(cband + (long)sk * D.wmax + q), ldcg(yl + q));
          if (q + 1 < w) cfma(t, __ldg(nband + (long)sk * D.wmax + q), ldcg(yl + q + 1));
          g[e] = csub(v, t);
        }
        cbar(ncons);
        // x_p = X_p g: 4 rows per warp, 16 independent loads in flight per lane
        const int cw = tid >> 5, ncw = ncons >> 5, lane = tid & 31;
        const long long cx0 = clock64();
        if (p < D.P - 1) {
          for (int rb = 4 * cw; rb < w; rb += 4 * ncw) {
            const cplx* Xr[4];
            bool ok[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              ok[u] = rb + u < w;
              Xr[u] = D.xinv + D.xinv_off[s] + ((long)p * w + (ok[u] ? rb + u : 0)) * xld;
            }
            if (HELM_GEN_XPIPE && lane < 4 && rb + 4 * ncw + lane < w)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                               D.xinv + D.xinv_off[s] + ((long)p * w + rb + 4 * ncw + lane) * xld),
                           "r"((uint32_t)(Kw * (long)sizeof(cplx))) : "memory");
            cplx acc[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
#pragma unroll kGenXun
            for (long jj = lane; jj < Kw; jj += 32 * kGenXch) {   // kGenXun iterations' loads in flight
              cplx xv[4][kGenXch], gv[kGenXch];
#pragma unroll
              for (int v = 0; v < kGenXch; ++v) {
                const bool in = jj + 32 * v < Kw;
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u][v] = (ok[u] && in) ? ldcg(Xr[u] + jj + 32 * v) : cmk(0, 0);
              }
#pragma unroll
              for (int v = 0; v < kGenXch; ++v) gv[v] = jj + 32 * v < Kw ? g[jj + 32 * v] : cmk(0, 0);
#pragma unroll
              for (int v = 0; v < kGenXch; ++v)
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
        for (int e = tid; e < D.wmax; e += ncons) {
          if (p == 0) xlo[e] = cmk(0, 0);
          if (p == D.P - 1) xhi[e] = cmk(0, 0);
        }
        cbar(ncons);
        pf.xmv += clock64() - cx0;
        // publish x_p (gather row and the next solve's corrections), take x_{p-1}
        if (p < D.P - 1) {
          for (int e = tid; e < w; e += ncons) D.xs[par * xss + (long)p * D.wmax + e] = xhi[e];
          if (writes_Z(D, i)) {
            const int olo = D.own_lo[s], ohi = D.own_hi[s];
            for (int q = olo + tid; q <= ohi; q += ncons) D.Z[node_of(D, a, hi + 1, q)] = xhi[q];
          }
          cbar(ncons);
          if (tid == 0) {
            __threadfence();
            st_release(&D.flag[p], (unsigned)(i + 1));
          }
        }
        if (p > 0) {
          long long cw1 = clock64();
          if (tid == 0) {
            while (ld_relaxed(&D.flag[p - 1]) < (unsigned)(i + 1)) __nanosleep(20);
            (void)ld_acquire(&D.flag[p - 1]);
          }
          cbar(ncons);
          pf.xwait += clock64() - cw1;
          for (int e = tid; e < w; e += ncons) xlo[e] = ldcg(D.xs + par * xss + (long)(p - 1) * D.wmax + e);
        }
        cbar(ncons);
      }
      if (D.P > 1) {
        for (int q = tid; q < w; q += ncons) {
          if (p > 0) {
            const cplx* crr = crow(lo - 1);
            const cplx* ner = nrow(lo - 1);
            cplx t = cmul(crr[q], xlo[q]);
            if (q >= 1) cfma(t, ner[q - 1], xlo[q - 1]);
            bseg[q] = csub(bseg[q], t);
          }
          if (p < D.P - 1) {
            const cplx* crr = crow(hi);
            const cplx* ner = nrow(hi);
            cplx t = cmul(crr[q], xhi[q]);
            if (q + 1 < w) cfma(t, ner[q], xhi[q + 1]);
            bseg[(m - 1) * w + q] = csub(bseg[(m - 1) * w + q], t);
          }
        }
        cbar(ncons);
      }
      // ---- phase 3 (or the whole solve when P == 1)
      thomas();
      // ---- epilogue: gather, boundary rows, next correction
      if (writes_Z(D, i)) {
        const int olo = D.own_lo[s], ohi = D.own_hi[s], ow = ohi - olo + 1;
        for (int e = tid; e < m * ow; e += ncons) {
          int cl = e / ow, q = olo + e % ow;
          D.Z[node_of(D, a, lo + cl, q)] = yseg[cl * w + q];
        }
      }
      if (D.P > 1) {
        cplx* xb = D.xb + par * exs + (long)p * 2 * D.wmax;
        for (int e = tid; e < w; e += ncons) {
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
        for (int c = lo + tid; c <= hi; c += ncons) target[c] = correction(D, tdst, side, c, a, X);
      }
      cbar(ncons);
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
      long long cw0 = clock64();
      if (tid == 0) {
        while (ld_relaxed(&D.cnt[0]) < (unsigned)(P * (i + 1))) __nanosleep(20);
        (void)ld_acquire(&D.cnt[0]);
      }
      cbar(ncons);
      pf.xwait += clock64() - cw0;
      // (a) separator-row corrections from the previous solve's solution
      if (i >= 1) {
        const int sprev = sigma(D, step_of(D, i - 1));
        const int aprev = D.a[sprev];
        const int side = bwd ? next_side(D) : prev_side(D);
        for (int k = tid; k < K; k += ncons) {
          const int sk = D.seg_hi[k] + 1;
          auto X = [&](int cc, int q) -> cplx {
            if (cc == sk) return z[k * D.wmax + q];
            if (cc == sk - 1) return ldcg(D.xb + (long)k * 2 * D.wmax + D.wmax + q);
            return ldcg(D.xb + (long)(k + 1) * 2 * D.wmax + q);  // cc == sk + 1
          };
          cplx cv = correction(D, s, side, sk, aprev, X);
          if (!bwd) D.corr_prev[(long)st * D.nc + sk] = cv;
          else cnx[k] = cv;
        }
        cbar(ncons);
      }
      // (b) reduced RHS g_k = b_{s_k} - U_{h_k}^T y_k[hi] - U_{s_k} y_{k+1}[lo]
      for (int e = tid; e < K * w; e += ncons) {
        const int k = e / w, q = e % w;
        const int hk = D.seg_hi[k], sk = hk + 1;
        cplx v = __ldg(D.R + node_of(D, a, sk, q));
        if (st > 0 && q == qp) v = cadd(v, D.corr_prev[(long)st * D.nc + sk]);
        if (bwd && q == qn) v = cadd(v, cnx[k]);
        v = cscale(v, rhs_scale(D, sk, q, w));
        const cplx* yh = D.yb + (long)k * 2 * D.wmax + D.wmax;     // y_k[hi]
        const cplx* yl = D.yb + (long)(k + 1) * 2 * D.wmax;        // y_{k+1}[lo]
        cplx t = cmul(__ldg(cband + (long)hk * D.wmax + q), ldcg(yh + q));
        if (q >= 1) cfma(t, __ldg(nband + (long)hk * D.wmax + q - 1), ldcg(yh + q - 1));
        cfma(t, __ldg(cband + (long)sk * D.wmax + q), ldcg(yl + q));
        if (q + 1 < w) cfma(t, __ldg(nband + (long)sk * D.wmax + q), ldcg(yl + q + 1));
        g[k * D.wmax + q] = csub(v, t);
      }
      for (int e = tid; e < w; e += ncons) tbuf[e] = cmk(0, 0);
      cbar(ncons);
      // (c) block-Thomas on the separator system
      for (int k = 0; k < K; ++k)
        block_step2(rg, w, ncons, g + k * D.wmax, k >= 1 ? z + (k - 1) * D.wmax : nullptr, k >= 1, z + k * D.wmax, pf);
      for (int k = K - 2; k >= 0; --k) {
        StepIO io;
        io.tA = z + (k + 1) * D.wmax;
        io.tB = tbuf;  // zeros
        io.out = z + k * D.wmax; io.ybase = z + k * D.wmax; io.mode = 1;
        io.next = 0; io.bn = nullptr; io.crn = nullptr; io.nen = nullptr; io.tAn = nullptr; io.tBn = nullptr;
        block_step<KP>(rg, w, ncons, io, pf);
      }
      // (d) publish x_sep
      for (int e = tid; e < K * w; e += ncons) {
        const int k = e / w, q = e % w;
        D.xs[(long)k * D.wmax + q] = z[k * D.wmax + q];
      }
      cbar(ncons);
      if (tid == 0) {
        __threadfence();
        st_release(&D.cnt[1], (unsigned)(i + 1));
      }
      // (e) gather separator rows
      if (writes_Z(D, i)) {
        const int olo = D.own_lo[s], ohi = D.own_hi[s], ow = ohi - olo + 1;
        for (int e = tid; e < K * ow; e += ncons) {
          const int k = e / ow, q = olo + e % ow;
          D.Z[node_of(D, a, D.seg_hi[k] + 1, q)] = z[k * D.wmax + q];
        }
      }
      cbar(ncons);
    }
  }
  if (A.prof && tid == 0) {
    long long* o = A.prof + (long)blockIdx.x * 8;
    o[0] = pf.peek; o[1] = pf.comp; o[2] = pf.bar; o[3] = pf.steps; o[4] = pf.xwait;
    o[5] = clock64() - t_start; o[6] = reducer ? 1 : 0; o[7] = pf.xmv;   // X mat-vec cycles (segment CTAs)
  }
}

// ------------------------------------------------------------------ host
static constexpr int kSmemMax = 227 * 1024;
static long long* g_sweep_prof = nullptr;   // set by helm_sweep_profile (diagnostics)

// Diagnostics (not part of the ABI header): when `buf` (device, 8 long long per
// CTA) is non-null, every subsequent sweep_apply records per-CTA cycle counters.
extern "C" void helm_sweep_profile(long long* buf) { g_sweep_prof = buf; }
long long* helm_sweep_prof_buffer() { return g_sweep_prof; }

int sweep_apply_fast(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                     cudaStream_t st);
int sweep_apply_dual(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                     cudaStream_t st);

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
  StageGuard gR(sR, st), gZ(sZ, st);
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

static const char* g_sweep_kernel = "";
extern "C" const char* helm_sweep_kernel_name(void) { return g_sweep_kernel; }

int sweep_apply_dev(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                    cudaStream_t st) {
  const helm_problem_s* prob = dirs[0]->prob;
  // The batched kernels are persistent and cooperative: all CTAs of all t
  // directions (P segment CTAs each, plus a reducer in the general kernel) must
  // be co-resident, one per SM.  A batch that cannot be (e.g. t = 8 with 33
  // segments) runs as two half batches, in order on the same stream.
  // kernel choice: the two-chain block kernel (sweep_dual.cu) where it applies
  // (w <= 36, P > 1), else the single-chain register-streaming kernel
  // (sweep_fast.cu, w <= 36), else the general TMA-ring kernel.
  // The sweep_kernel knob (helm_set_knob: 2 = fast, 3 = general) starts lower
  // (parity tests of every kernel); read per call.
  const int kn = helm_knob(KNOB_SWEEP_KERNEL);
  const int level = kn == 2 || kn == 3 ? kn : 1;
  static int nsm_dev = 0;
  if (!nsm_dev) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm_dev, cudaDevAttrMultiProcessorCount, dev);
  }
  long need = 0, need_dual = 0;   // CTAs: P per direction (two-chain), P + 1 (the others: a reducer each)
  for (int d = 0; d < t; ++d) {
    need += dirs[d]->P + 1;
    need_dual += dirs[d]->P;
  }
  if (level <= 1 && need_dual <= nsm_dev) {
    g_sweep_kernel = "k_sweep_dual";
    int rc = sweep_apply_dual(dirs, t, Rdev, ldr, Zdev, ldz, st);
    if (rc != -1) return rc;
  }
  if (t > 1 && need > nsm_dev) {
    const int h = t / 2;
    int rc = sweep_apply_dev(dirs, h, Rdev, ldr, Zdev, ldz, st);
    if (rc != HELM_OK) return rc;
    return sweep_apply_dev(dirs + h, t - h, Rdev + (ldr == 0 ? 0 : (long)h * ldr), ldr, Zdev + (long)h * ldz, ldz, st);
  }
  if (level <= 2) {
    g_sweep_kernel = "k_sweep_fast";
    int rc = sweep_apply_fast(dirs, t, Rdev, ldr, Zdev, ldz, st);
    if (rc != -1) return rc;
  }
  g_sweep_kernel = "k_sweep_apply";
  // launch geometry: 8 consumer lanes per block row (<= 36 rows per tile) + 1 TMA producer warp
  int wmax = 0, pmax = 1;
  for (int d = 0; d < t; ++d) {
    wmax = std::max(wmax, dirs[d]->wmax);
    pmax = std::max(pmax, dirs[d]->P);
  }
  const int ncons = ((8 * std::min(wmax, 36) + 31) / 32) * 32;
  const int threads = ncons + 32;
  const int R_t = ncons / 8;
  long vec_elems = 0, stage_elems = 0;
  int ctas = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    int mmax = 0;
    for (int p = 0; p < h->P; ++p) mmax = std::max(mmax, h->seg_hi[p] - h->seg_lo[p] + 1);
    int vr = std::max(mmax + 1, std::max(h->P - 1, 1));
    vec_elems = std::max(vec_elems, (long)vr * h->wmax);
    stage_elems = std::max(stage_elems, (long)std::min(R_t, h->wmax) * h->wmax);
    ctas += h->P + (h->P > 1 ? 1 : 0);
  }
  vec_elems = (vec_elems + 7) / 8 * 8;
  stage_elems = (stage_elems + 7) / 8 * 8;
  int nsolve_max = 1;
  for (int d = 0; d < t; ++d) nsolve_max = std::max(nsolve_max, dirs[d]->is_double ? 2 * dirs[d]->N - 1 : dirs[d]->N);
  nsolve_max = (nsolve_max + 1) & ~1;  // keeps the vector areas after the table 16-byte aligned
  const long tail = sizeof(cplx) * (7L * wmax + 2L * pmax + 8) + (long)sizeof(SolveTab) * nsolve_max + 32;
  const long stage_bytes = sizeof(cplx) * stage_elems;
  int vec_global = 0;
  long fixed = 256 + tail + sizeof(cplx) * 4 * vec_elems;
  if (kSmemMax - fixed < 2 * stage_bytes) {
    vec_global = 1;
    fixed = 256 + tail;
  }
  int nstage = (int)std::min<long>(8, (kSmemMax - fixed) / stage_bytes);
  if (nstage < 2) {
    helm_set_error("sweep_apply: shared memory too small (w=%d)", wmax);
    return HELM_EINVAL;
  }
  size_t smem = fixed + (size_t)nstage * stage_bytes;
  // per-direction scratch
  std::vector<size_t> off(t);
  size_t total = 0;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    off[d] = total;
    total += al(sizeof(unsigned) * (2 + h->P));                     // counters, neighbour flags
    total += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax) * 2;      // yb, xb (parity buffers)
    total += al(sizeof(cplx) * 2L * h->P * h->wmax);              // xs (parity buffers)
    total += al(sizeof(cplx) * (long)h->N * h->nc);                // corr_prev
    total += al(sizeof(cplx) * (long)h->nc);                       // corr_next
  }
  size_t vec_off = total;
  if (vec_global) total += al(sizeof(cplx) * 4L * vec_elems * ctas);
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
  A.pmax = pmax;
  A.nsolve_max = nsolve_max;
  A.vec_global = vec_global;
  A.vec_scratch = vec_global ? (cplx*)(scratch + vec_off) : nullptr;
  A.prof = g_sweep_prof;
  int base = 0;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    DirArgs& D = A.d[d];
    D.axis = h->axis; D.order = h->order; D.N = h->N; D.P = h->P; D.nc = h->nc; D.disc = h->disc;
    D.nxp1 = prob->nx + 1; D.is_double = h->is_double; D.ntile_max = (h->wmax + R_t - 1) / R_t;
    D.a = h->d_a; D.w = h->d_w; D.own_lo = h->d_own_lo; D.own_hi = h->d_own_hi;
    D.seg_lo = h->d_seg_lo; D.seg_hi = h->d_seg_hi;
    D.cr = h->d_cr; D.ne = h->d_ne; D.tc = h->d_tc;
    D.fac = h->d_fac; D.fac_off = h->d_fac_off; D.red = h->d_red; D.red_off = h->d_red_off;
    D.R = Rdev + (ldr == 0 ? 0 : (long)d * ldr);
    D.Z = Zdev + (long)d * ldz;
    unsigned char* q = scratch + off[d];
    D.cnt = (unsigned*)q; D.flag = D.cnt + 2; q += al(sizeof(unsigned) * (2 + h->P));
    D.yb = (cplx*)q; q += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax);
    D.xb = (cplx*)q; q += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax);
    D.xs = (cplx*)q; q += al(sizeof(cplx) * 2L * h->P * h->wmax);
    // explicit separator-inverse rows: the segments solve the separator system
    // themselves (X path) unless the general_reducer knob is set
    const bool force_reducer = helm_knob(KNOB_GENERAL_REDUCER) != 0;
    D.xinv = force_reducer ? nullptr : h->d_xinv;
    D.xinv_off = h->d_xinv_off;
    D.corr_prev = (cplx*)q; q += al(sizeof(cplx) * (long)h->N * h->nc);
    D.corr_next = (cplx*)q;
    D.wmax = h->wmax;
    D.cta_base = base;
    base += h->P + (h->P > 1 ? 1 : 0);
    e = cudaMemsetAsync(D.cnt, 0, sizeof(unsigned) * (2 + h->P), st);
    if (e != cudaSuccess) break;
  }
  // entries per lane and block row (8 lanes per row): the instantiation for the widest strip of the batch
  const void* kfun = wmax <= 40 ? (const void*)k_sweep_apply<5>
                     : wmax <= 104 ? (const void*)k_sweep_apply<13> : (const void*)k_sweep_apply<15>;
  if (wmax > 120) {
    helm_set_error("sweep_apply: strips wider than 120 nodes are not supported (w=%d)", wmax);
    cudaFreeAsync(scratch, st);
    return HELM_EINVAL;
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kfun, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 0, occ = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfun, threads, smem);
  if (e == cudaSuccess && occ * nsm < ctas) {
    helm_set_error("sweep_apply: %d CTAs cannot be co-resident (%d SMs x %d); reduce n_segments", ctas, nsm, occ);
    cudaFreeAsync(scratch, st);
    return HELM_ECUDA;
  }
  if (e == cudaSuccess) {
    void* args[] = {(void*)&A};
    e = cudaLaunchCooperativeKernel(kfun, dim3(ctas), dim3(threads), args, smem, st);
    g_helm_launches++;
  }
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply: launch: %s", cudaGetErrorString(e));
    return HELM_ECUDA;
  }
  return HELM_OK;
}
