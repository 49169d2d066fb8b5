// sweep_dual.cu -- hot-path row a4 for block rows of <= 36 nodes and P > 1
// segments: the batched, partitioned double sweep with TWO independent
// recurrence chains per segment, so that the dependent path of one local solve
// is ~2m block steps instead of the 4m - 2 of sweep_fast.cu.
//
// Segment [lo, hi] (m rows) of strip s, separators x_{p-1} (row lo-1) and
// x_p (row hi+1).  With top-down inverses Sinv_c (fac) and bottom-up inverses
// S'^{-1}_c (fac2, strip_setup.cu k_factor_rows kind 1):
//   phase 1 (independent, concurrent):
//     chain A  y_c  = Sinv_c (b_c - U_{c-1}^T y_{c-1}),      c = lo..hi   (y_hi = x0_hi)
//     chain B  z_c  = S'^{-1}_c (b_c - U_c z_{c+1}),          c = hi..lo   (z_lo = x0_lo)
//   separator stage (as sweep_fast.cu): g from x0_lo / x0_hi of all segments,
//     x_p = X_p g (explicit separator-inverse rows), neighbour exchange for x_{p-1}
//   phase 3 (independent, concurrent):
//     chain A  xa_c = y_c - Sinv_c U_c xa_{c+1},  xa_{hi+1} = x_p   c = hi..lo
//     chain B  f_c  = -S'^{-1}_c U_{c-1}^T f_{c-1}, f_{lo-1} = x_{p-1}  c = lo..hi
//   x_c = xa_c + f_c.
// Chain A phase 3 is the back substitution of the top-down Thomas factorisation
// with b_hi replaced by b_hi - U_hi x_p; chain B phase 3 adds the response
// T^{-1}[:, lo] (-U_{lo-1}^T x_{p-1}) through the first block column of the
// segment inverse, X[c][lo] = -S'^{-1}_c U_{c-1}^T X[c-1][lo].
// Both phases read Sinv and S'^{-1} once per row: 4 w^2 per row per solve, the
// same factor bytes as sweep_fast.cu, with half the dependent steps.
//
// Warps [0, nw) run chain A, [nw, 2 nw) chain B (named barriers 1 and 2);
// whole-consumer stages use barrier 3.  A block step: 4 lanes per block row,
// 7 owned + 1 halo row per warp (the halo gives the writer lanes the
// neighbour value of the bidiagonal coupling with one shuffle).  The packed
// factor blocks are streamed HBM/L2 -> shared memory by one cp.async.bulk per
// block into a per-chain NST-stage ring (mbarrier complete_tx) issued NST-1
// blocks ahead across phase and solve boundaries by lane 0 of the group; each
// lane reads its nine entries with precomputed byte offsets (the 16-byte
// register loads of an earlier revision cost ~1200 cycles per step in L1
// wavefronts and exposed latency, tools/bench_dualstep.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <type_traits>

#include "sweep_common.cuh"

#ifndef HELM_DUAL_SNPOS
#define HELM_DUAL_SNPOS 1   // where the next block's entries are read (see step(); 1 = interleaved with the FMAs)
#endif
#ifndef HELM_DUAL_WOPS_LATE
#define HELM_DUAL_WOPS_LATE 1   // 1: writer operands read after the FMAs (not before the input-vector loads)
#endif
#ifndef HELM_DUAL_GSRC
#define HELM_DUAL_GSRC 1   // 1: the separator-row source is staged into the g area at the pre-actions
#endif
#ifndef HELM_DUAL_XCH
#define HELM_DUAL_XCH 4     // 32-column chunks per row in flight in the X mat-vec (4 rows per warp)
#endif
#ifndef HELM_DUAL_ONELOOP
#define HELM_DUAL_ONELOOP 1   // 1: one copy of the solve loop (the chain phases dispatch on the group): half the code
#endif
#ifndef HELM_DUAL_NOFENCE
#define HELM_DUAL_NOFENCE 1   // 1: the counter / flag releases rely on red/st.release after the CTA barrier (no extra fence)
#endif
#if HELM_DUAL_NOFENCE
#define HELM_DUAL_FENCE() ((void)0)
#else
#define HELM_DUAL_FENCE() __threadfence()
#endif
#ifndef HELM_DUAL_S2PF
#define HELM_DUAL_S2PF 2   // two-level panels' L2 prefetch: 0 none, 1 normal priority, 2 evict_first
#endif
#ifndef HELM_DUAL_XPF_PROD
#define HELM_DUAL_XPF_PROD 1    // 1: the X-row L2 prefetch is issued by the chain-A producer warp when phase 1 ends
#endif
#ifndef HELM_DUAL_FPF
#define HELM_DUAL_FPF 7     // n > 0: the producers prefetch the factor block n steps ahead into L2 (C5 t = 4: off 3.74,
                            // 4: 3.74, 5: 3.72, 6: 3.71, 7: 3.69, 8: 3.70, 9: 3.73, 10: 3.74, 16: 3.78 ms)
#endif
#ifndef HELM_DUAL_FPF_P1
#define HELM_DUAL_FPF_P1 1  // 1: only phase-1 blocks are prefetched (phase 3 too: the same 3.69 ms)
#endif
#ifndef HELM_DUAL_EPIREL
#define HELM_DUAL_EPIREL 1    // 1: the epilogue counter is released by chain B's producer lane (not thread 0 before a barrier)
#endif
#ifndef HELM_DUAL_RHS_TMA
#define HELM_DUAL_RHS_TMA 0   // stage the next RHS by bulk copies (1) or per-element cp.async (0)
#endif
namespace dualk {
constexpr int LPR = 4;    // lanes per block row
constexpr int OWN = 7;    // owned rows per warp (8 slots, 1 halo)
constexpr int KPL = 9;    // complex entries per lane per block row (w <= 36)
constexpr int WM = 40;    // vector stride
#ifndef HELM_DUAL_NST
#define HELM_DUAL_NST 4
#endif
constexpr int NST = HELM_DUAL_NST;    // TMA ring stages per chain (NST-1 blocks in flight)
constexpr int MAXT = 5 * 64 + 64;   // 2 groups of <= 5 warps (w <= 35) + 2 TMA producer warps
}  // namespace dualk

// per-CTA cycle counters (tools/prof_sweep.py) only in the -DHELM_DUAL_PROF build
// (python -m paper_2408_11929_b200.build --prof); the per-step sub-phase counters
// (-DHELM_DUAL_PROF_STEP) keep clock values live across the step and spill
#ifdef HELM_DUAL_PROF
constexpr bool kProf = true;
#else
constexpr bool kProf = false;
#endif
#ifdef HELM_DUAL_PROF_STEP
constexpr bool kProfStep = kProf;
#else
constexpr bool kProfStep = false;
#endif
__device__ __forceinline__ long long pclk() {
  if constexpr (kProf) return clock64();
  else return 0;
}

struct DualArgs {
  DirArgs d[HELM_MAXDIR];
  int t;
  int nw;           // consumer warps per chain group
  int vec_elems;    // cplx per vector area
  int nsolve_max;
  int pmax;
  int stage_elems;  // cplx per ring stage (>= largest packed block + 1 zero entry)
  int mmax;         // largest segment (rows)
  long long* prof;  // optional per-CTA counters (32 per CTA)
};

// two-level separator plan layout (strip_setup.cu kSep2*)
constexpr int kS2PlanHdr = 64, kS2PlanStride = 4 + 2 * 8;

struct DualTab {
  const cplx* fac;
  const cplx* fac2;
  const cplx* xinv;
  const cplx* sep2;       // this strip's two-level panels (NULL: full rows)
  const float2* xinv32;   // complex64 rows (XF32 instantiation only)
  int w, a, s, pks;   // pks: entries per padded packed block (pk_size(w))
};

__device__ __forceinline__ int dslot_row(int wi, int slot, int high) {
  return high ? dualk::OWN * wi + slot : dualk::OWN * wi + slot - 1;
}
__device__ __forceinline__ bool dslot_owned(int slot, int high) { return high ? slot < 7 : slot >= 1; }

// L2 residency: factor blocks read in phase 1 are re-read in phase 3 of the
// same solve after ~2m block steps and the separator stage (~300 MB of other
// traffic for C5 t = 4, more than L2), so phase-1 loads carry evict_last and
// phase-3 / separator-inverse loads evict_first.
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ cplx ld_cg_hint(const cplx* a, uint64_t pol) {
  cplx v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(a), "l"(pol));
  return v;
}

__device__ __forceinline__ float2 ld_cg_hint_f2(const float2* a, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(a), "l"(pol));
  return v;
}

__device__ __forceinline__ void dprefetch_l2(const void* p, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
               : "memory");
}

// block row and halo mapping of step e (0 <= e < 2m) of chain g
__device__ __forceinline__ void chain_row(int g, int e, int m, int lo, int hi, int& row, int& high, int& js,
                                          int& ph) {
  ph = e >= m ? 1 : 0;
  js = e - ph * m;
  const bool up = (g == 0) == (ph == 0);   // A1, B3 walk lo -> hi
  row = up ? lo + js : hi - js;
  high = up ? 0 : 1;                       // lo -> hi steps need o[r-1]: low mapping
}

// GSEP: the separator RHS g (K w entries) has its own shared-memory area when it
// is longer than two segment vector areas (e.g. C2 with 28 segments of 8 rows);
// else it spans xa and the adjacent fb, which are free from the epilogue of the
// previous solve to phase 3 of this one.  A template parameter, not a runtime
// choice: the kernel is at its register cap.
template <bool GSEP, bool XF32>
__global__ void __launch_bounds__(dualk::MAXT, 1) k_sweep_dual(const __grid_constant__ DualArgs A) {
  using namespace dualk;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int gsz = A.nw * 32;
  const int ncons = 2 * gsz;
  int d = 0;
  while (d + 1 < A.t && (int)blockIdx.x >= A.d[d + 1].cta_base) ++d;
  const DirArgs& D_ = A.d[d];
  const int p = blockIdx.x - D_.cta_base;
  const int P = D_.P, K = P - 1;

  // ring stages first (TMA destinations, 128-byte aligned), then barriers, vectors
  cplx* ring = reinterpret_cast<cplx*>(smem_raw);                          // [2][NST][stage_elems]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + 2L * NST * A.stage_elems);   // [2][NST] block landed
  uint64_t* empty = full + 2 * NST;                                        // [2][NST] stage released
  // staging barriers (bulk copies, complete_tx): [0] inputs of the next solve, staged
  // during phase 3; [1] the couplings of the current solve; [2] the first RHS
  uint64_t* sbar = empty + 2 * NST;
  cplx* vbuf = reinterpret_cast<cplx*>(sbar + 4);                         // [group][2][WM]
  cplx* xlo = vbuf + 4 * WM;                        // x_{p-1}
  cplx* xhi = xlo + WM;                             // x_p
  cplx* zlo = xhi + WM;                             // x0_lo (chain B phase 1)
  cplx* cpv = zlo + WM;                             // [pmax] prev-side separator corrections
  cplx* cnv = cpv + A.pmax;                         // [pmax] next-side separator corrections
  DualTab* tab = reinterpret_cast<DualTab*>(cnv + A.pmax);
  int* pkst = reinterpret_cast<int*>(tab + A.nsolve_max);   // [WM] padded row starts of the current w
  int* sepr = pkst + WM;                                     // [pmax] separator rows s_k
  cplx* vec0 = reinterpret_cast<cplx*>(
      smem_raw + ((((char*)(sepr + A.pmax) - (char*)smem_raw) + 127) / 128) * 128);
  cplx* bseg = vec0;                                // RHS rows lo..hi, entry (cl, q) at cl * bsc + q * bsq
  cplx* yseg = bseg + A.vec_elems;                  // chain A phase 1 (y)
  cplx* xa = yseg + A.vec_elems;                    // chain A phase 3 (aliased by g in the separator stage)
  cplx* fb = xa + A.vec_elems;                      // chain B phase 3
  cplx* bcr = fb + A.vec_elems;                     // staged U couplings, rows lo-1..hi (row stride wmax)
  cplx* bne = bcr + A.vec_elems;
  cplx* gsm_own = bne + A.vec_elems + (2 + kTcW) * A.mmax;   // GSEP: after cs / cps / tcs
  cplx* gsm = GSEP ? gsm_own : xa;                  // separator RHS g (K x w): xa (+ fb), dead before phase 3
  cplx* cs = bne + A.vec_elems;                     // [mmax] corrections formed by the last epilogue (next RHS)
  cplx* cps = cs + A.mmax;                          // [mmax] forward-pass corr_prev rows (backward RHS), staged
  cplx* tcs = cps + A.mmax;                         // [kTcW mmax] transmission coefficients of the next epilogue, staged

  const int nsolve = n_solves(D_);
  for (int i = tid; i < nsolve; i += blockDim.x) {
    const int s = sigma(D_, step_of(D_, i));
    tab[i].fac = D_.facp + D_.pfac_off[s];
    tab[i].fac2 = D_.fac2 + D_.pfac_off[s];
    tab[i].xinv = D_.xinv + D_.xinv_off[s];
    tab[i].xinv32 = D_.xinv32 ? D_.xinv32 + D_.xinv_off[s] : nullptr;
    tab[i].sep2 = D_.sep2 ? D_.sep2 + D_.sep2_off[s] : nullptr;
    tab[i].w = D_.w[s];
    tab[i].a = D_.a[s];
    tab[i].s = s;
    tab[i].pks = pk_size(D_.w[s]);
  }
  for (int e = tid; e < 4 * WM; e += blockDim.x) vbuf[e] = cmk(0, 0);   // padding entries stay finite
  // the zero entry after each ring stage (target of out-of-range lanes)
  for (int e = tid; e < 2 * NST; e += blockDim.x) ring[(long)e * A.stage_elems + A.stage_elems - 1] = cmk(0, 0);
  if (tid == 0) {
    for (int e = 0; e < 2 * NST; ++e) {
      mbar_init(&full[e], 1);
      mbar_init(&empty[e], 1);
    }
    for (int e = 0; e < 4; ++e) mbar_init(&sbar[e], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int lo = D_.seg_lo[p], hi = D_.seg_hi[p];
  const int m = hi - lo + 1;
  const int bw = D_.wmax;                         // band row stride in bcr / bne
  // RHS layout: rows (x axis: a row of the strip is contiguous in the grid) or
  // columns (y axis: a line of the strip is contiguous), odd column stride
  const int bsq = D_.axis == 0 ? 1 : (m | 1);
  for (int k = tid; k < K; k += blockDim.x) sepr[k] = D_.seg_hi[k] + 1;
  // this segment's entry of the two-level separator plan (the same for every strip)
  __shared__ int spk[kS2PlanStride];
  if (D_.sep2 && p < K)
    for (int e = tid; e < kS2PlanStride; e += blockDim.x) spk[e] = D_.sep2_plan[kS2PlanHdr + p * kS2PlanStride + e];
  if (lo == 0)
    for (int e = tid; e < bw; e += blockDim.x) bcr[e] = bne[e] = cmk(0, 0);   // row -1 (never staged)
  const int total = nsolve * 2 * m;      // block steps per chain
  __syncthreads();

  if (tid >= ncons) {
    // ============================================================ TMA producer warps
    // warp ncons/32 + pg feeds chain pg: per solve, phase 0 then phase 1, m packed
    // blocks each, NST stages ahead; a stage is refilled once the chain group has
    // released it (empty barrier, arrived by the group after its step barrier)
    const int pg = (tid - ncons) >> 5;
    if ((tid & 31) == 0) {
      const uint64_t polL = l2_policy_last(), polF = l2_policy_first();
      uint32_t f = 0;
      for (int i2 = 0; i2 < nsolve; ++i2) {
        const int pw = tab[i2].pks;
        const cplx* fbase = pg == 0 ? tab[i2].fac : tab[i2].fac2;
        for (int e = 0; e < 2 * m; ++e, ++f) {
          const int ph = e >= m ? 1 : 0, js = e - ph * m;
          const bool up = (pg == 0) == (ph == 0);
          const cplx* src = fbase + (long)(up ? lo + js : hi - js) * pw;
          const int st = f % NST;
          if (f >= (uint32_t)NST) mbar_wait(&empty[pg * NST + st], ((f / NST) - 1) & 1);
#if HELM_DUAL_EPIREL
          if (pg == 1 && i2 >= 1 && e == std::min(NST - 1, 2 * m - 1)) {
            // the epilogue of solve i2 - 1 is complete (CTA-scope arrival of thread 0 after
            // the consumers' barrier): publish it to the other segments
            mbar_wait(&sbar[3], (i2 - 1) & 1);
            red_release_add(&D_.cnt[1], 1u);
          }
#endif
#if HELM_DUAL_XPF_PROD
          if (!XF32 && pg == 0 && e == std::min(m + NST - 1, 2 * m - 1) && p < P - 1) {
            // chain A has released its last phase-1 block: this solve's separator stage
            // starts now -- stream this CTA's separator-inverse rows into L2 from here
            // (off the consumers' barriers)
            const int w2 = tab[i2].w;
            const long ld = x_ld(K, w2);
            for (int r = 0; r < w2; ++r)
              dprefetch_l2(tab[i2].xinv + ((long)p * w2 + r) * ld, (uint32_t)((long)K * w2 * sizeof(cplx)), polF);
          }
#endif
          uint64_t* bar = &full[pg * NST + st];
          const uint32_t bytes = (uint32_t)(pw * sizeof(cplx));
#if HELM_DUAL_FPF
          {
            // L2 prefetch of the factor block HELM_DUAL_FPF steps ahead (same solve): the ring
            // holds only NST - 1 blocks in flight, ~3.5 k cycles of lookahead against HBM
            // latency spikes under load
            const int ea = e + HELM_DUAL_FPF;
            if (ea < (HELM_DUAL_FPF_P1 ? m : 2 * m)) {
              const int pha = ea >= m ? 1 : 0, jsa = ea - pha * m;
              const bool upa = (pg == 0) == (pha == 0);
              dprefetch_l2(fbase + (long)(upa ? lo + jsa : hi - jsa) * pw, bytes, pha == 0 ? polL : polF);
            }
          }
#endif
          mbar_expect_tx(bar, bytes);
          bulk_g2s_hint(ring + ((long)pg * NST + st) * A.stage_elems, src, bytes, bar, ph == 0 ? polL : polF);
        }
      }
    }
    return;
  }

  const int g = tid >= gsz ? 1 : 0;       // chain group
  const int gtid = tid - g * gsz;
  const int wi = gtid >> 5, lane = tid & 31;
  // lane -> (slot = row within the warp's 8, q = column residue mod 4); slot is the
  // fast index so that a quarter-warp reads 8 rows of one column (conflict-free with
  // the padded packed layout, common.cuh) and one broadcast input entry
  const int slot = lane & 7, q = lane >> 3;
  const long band_stride = (long)D_.nc * D_.wmax;
  // cycle counters of thread 0 (prof build only), kept in shared memory so that
  // they cost no registers: [0] pre-actions [1] separator stage [2] X mat-vec
  // [4] waits [8..11] step sub-phases (mat-vec, loads+reduce, writer, barrier)
  // [12] gather wait [13] neighbour wait [14] corrections + g
  __shared__ long long profs[32];
  auto pacc = [&](int k, long long v) {
    if constexpr (kProf) {
      if (tid == 0) profs[k] += v;
    }
  };
  if (kProf && tid == 0)
    for (int k = 0; k < 32; ++k) profs[k] = 0;
  const long long t_start = pclk();
  auto cbar = [&]() { asm volatile("bar.sync 3, %0;" ::"r"(ncons) : "memory"); };
  auto gbar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(gsz) : "memory"); };
  const long exs = 2L * P * D_.wmax;   // parity stride of yb / xb
  const long xss = (long)P * D_.wmax;  // parity stride of xs
  cplx* myv = vbuf + g * 2 * WM;
  const uint64_t pol_last = l2_policy_last(), pol_first = l2_policy_first();

  int cur = 0;

  // ------------------------------------------------------------ per-solve actions (all consumers)
  // the transmission correction the epilogue of solve i forms for solve i + 1:
  // destination strip, its side and the global buffer (none after the last solve)
  auto epi_target = [&](int i, int& tdst, int& side, cplx*& target) {
    const int st = step_of(D_, i);
    tdst = -1;
    side = 0;
    target = nullptr;
    if (!is_bwd(D_, i)) {
      if (st < D_.N - 1) { tdst = sigma(D_, st + 1); side = prev_side(D_); target = D_.corr_prev + (long)(st + 1) * D_.nc; }
      else if (D_.is_double && D_.N > 1) { tdst = sigma(D_, D_.N - 2); side = next_side(D_); target = D_.corr_next; }
    } else if (st >= 1) {
      tdst = sigma(D_, st - 1); side = next_side(D_); target = D_.corr_next;
    }
  };
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
    epi_target(i, tdst, side, target);
    if (tdst >= 0) {
      auto X = [&](int cc, int qq) -> cplx {
        if (cc < lo) return xlo[qq];
        if (cc > hi) return xhi[qq];
        return cadd(xa[(cc - lo) * w + qq], fb[(cc - lo) * w + qq]);
      };
      // the destination strip is the one solve i + 1 works on
      const int at = i + 1 < nsolve ? tab[i + 1].a : D_.a[tdst];
      const int wt = i + 1 < nsolve ? tab[i + 1].w : D_.w[tdst];
      const int bt = at + wt - 1;
      const int qi = side == 0 ? at - a : bt - a, qo = side == 0 ? at - 1 - a : bt + 1 - a;
      const int qin = side == 0 ? at + 1 - a : bt - 1 - a;
      const int dd = side == 0 ? -1 : 1;
      for (int c = lo + tid; c <= hi; c += ncons) {
        // D8 stencil with the coefficients staged in tcs (sweep_common.cuh correction_aw)
        const cplx* kk = tcs + (c - lo) * kTcW;
        const bool h4 = c + dd >= 0 && c + dd < D_.nc;
        cplx v = cmul(kk[1], X(c, qi));
        cfma(v, kk[3], X(c, qo));
        if (c >= 1) cfma(v, kk[0], X(c - 1, qi));
        if (c + 1 < D_.nc) cfma(v, kk[2], X(c + 1, qi));
        if (h4) cfma(v, kk[4], X(c + dd, qo));
        if (D_.disc == HELM_DISC_FD5) cfma(v, kk[5], X(c, qin));
        target[c] = v;
        cs[c - lo] = v;
      }
    }
  };
  // Staging by bulk copies (TMA, mbarrier complete_tx), issued by the lanes of warp 0:
  //  * the source rows lo..hi of solve i+1 go to bseg at the start of phase 3 of
  //    solve i (bseg is only read in phase 1), with the coefficients of epilogue
  //    i's correction and, for a backward solve i+1, its forward-pass corr_prev rows
  //    (barrier sbar[0], waited at the pre-actions of solve i+1);
  //  * the couplings of rows lo-1..hi go to bcr/bne at the start of the
  //    pre-actions (free after phase 3), overlapping the epilogue (sbar[1]).
  // The copies replace per-element cp.async, whose LSU traffic competed with the
  // block steps running at the same time.
  auto issue_copies = [&](int ncp, auto desc, uint64_t* bar) {
    // desc(j, dst, src, bytes) describes copy j; lane 0 arms the barrier with the total
    if (tid < 32) {
      uint32_t tot = 0;
      for (int j = 0; j < ncp; ++j) {
        cplx* dd;
        const cplx* sr;
        uint32_t by;
        desc(j, dd, sr, by);
        tot += by;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic accesses of the targets
      if (tid == 0) mbar_expect_tx(bar, tot);
      __syncwarp();
      for (int j = tid; j < ncp; j += 32) {
        cplx* dd;
        const cplx* sr;
        uint32_t by;
        desc(j, dd, sr, by);
        if (by) bulk_g2s_hint(dd, sr, by, bar, pol_first);
      }
    }
  };
  auto rhs_copy = [&](int i, int j, cplx*& dd, const cplx*& sr, uint32_t& by) {
    const int a = tab[i].a, w = tab[i].w;
    if (D_.axis == 0) { dd = bseg + (long)j * w; sr = D_.R + node_of(D_, a, lo + j, 0); by = (uint32_t)(w * sizeof(cplx)); }
    else { dd = bseg + (long)j * bsq; sr = D_.R + node_of(D_, a, lo, j); by = (uint32_t)(m * sizeof(cplx)); }
  };
  auto stage_rhs0 = [&]() {
    const int nr = D_.axis == 0 ? m : tab[0].w;
    issue_copies(nr, [&](int j, cplx*& dd, const cplx*& sr, uint32_t& by) { rhs_copy(0, j, dd, sr, by); }, &sbar[2]);
  };
  auto stage_next = [&](int i) {
    int tdst, side;
    cplx* target;
    epi_target(i, tdst, side, target);
    const bool rhs = i + 1 < nsolve;
    const bool cpb = rhs && is_bwd(D_, i + 1) && step_of(D_, i + 1) > 0;
#if HELM_DUAL_RHS_TMA
    const int nr = !rhs ? 0 : (D_.axis == 0 ? m : tab[i + 1].w);
#else
    // the source rows: per-element cp.async by all consumers (bulk copies of the
    // m rows / w lines queue in front of the factor stream in the TMA unit)
    const int nr = 0;
    if (rhs) {
      const int a1 = tab[i + 1].a, w1 = tab[i + 1].w;
      for (int e = tid; e < m * w1; e += ncons) {
        const int cl = e / w1, qq = e - cl * w1;
        cp_async16(bseg + (D_.axis == 0 ? cl * w1 + qq : qq * bsq + cl), D_.R + node_of(D_, a1, lo + cl, qq));
      }
      cp_async_commit();
    }
#endif
    issue_copies(nr + 2, [&](int j, cplx*& dd, const cplx*& sr, uint32_t& by) {
      if (j < nr) { rhs_copy(i + 1, j, dd, sr, by); return; }
      dd = j == nr ? tcs : cps;
      sr = j == nr ? D_.tc + (((long)(tdst < 0 ? 0 : tdst) * 2 + side) * D_.nc + lo) * kTcW
                   : D_.corr_prev + (long)step_of(D_, i + 1 < nsolve ? i + 1 : i) * D_.nc + lo;
      by = j == nr ? (tdst >= 0 ? (uint32_t)(kTcW * m * sizeof(cplx)) : 0u) : (cpb ? (uint32_t)(m * sizeof(cplx)) : 0u);
    }, &sbar[0]);
  };
  auto stage_bands = [&](int i) {
    const int s = tab[i].s;
    const int c0 = lo > 0 ? lo - 1 : 0;
    const long off = (long)s * band_stride + (long)c0 * bw;
    const uint32_t by = (uint32_t)((hi - c0 + 1) * bw * sizeof(cplx));
    cplx* d0 = lo > 0 ? bcr : bcr + bw;
    cplx* d1 = lo > 0 ? bne : bne + bw;
    issue_copies(2, [&](int j, cplx*& dd, const cplx*& sr, uint32_t& b2) {
      dd = j == 0 ? d0 : d1;
      sr = (j == 0 ? D_.cr : D_.ne) + off;
      b2 = by;
    }, &sbar[1]);
  };
  // RHS of solve i (rows lo..hi): the staged source plus the transmission
  // corrections on the interface columns (after cp.async.wait_all + barrier)
  auto seg_rhs = [&](int i) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int w = tab[i].w;
    const int qp = prev_side(D_) == 0 ? 0 : w - 1;
    const int qn = next_side(D_) == 0 ? 0 : w - 1;
    for (int cl = tid; cl < m; cl += ncons) {
      // corrections of the previous epilogue (cs) and, backward, the forward pass's (cps)
      const int bsc = D_.axis == 0 ? w : 1;
      if (st > 0) bseg[cl * bsc + qp * bsq] = cadd(bseg[cl * bsc + qp * bsq], bwd ? cps[cl] : cs[cl]);
      if (bwd) bseg[cl * bsc + qn * bsq] = cadd(bseg[cl * bsc + qn * bsq], cs[cl]);
      if (D_.disc == HELM_DISC_FD5) {
        // FD5: the factored strip matrix is D_s A_s, so the RHS is D_s (source + corrections)
        const int c = lo + cl;
        if (c == 0 || c == D_.nc - 1) {
          for (int qq = 0; qq < w; ++qq) bseg[cl * bsc + qq * bsq] = cscale(bseg[cl * bsc + qq * bsq], rhs_scale(D_, c, qq, w));
        } else {
          bseg[cl * bsc] = cscale(bseg[cl * bsc], 0.5);
          bseg[cl * bsc + (w - 1) * bsq] = cscale(bseg[cl * bsc + (w - 1) * bsq], 0.5);
        }
      }
    }
  };
  // separator stage of solve i (after phase 1): all-gather of x0_lo / x0_hi, g,
  // x_p = X_p g, neighbour exchange, phase-3 chain inputs
  auto seg_separators = [&](int i) __attribute__((always_inline)) {
    const int st = step_of(D_, i);
    const bool bwd = is_bwd(D_, i);
    const int s = tab[i].s, a = tab[i].a, w = tab[i].w;
    const int par = i & 1, ppar = par ^ 1;
    const int qp = prev_side(D_) == 0 ? 0 : w - 1;
    const int qn = next_side(D_) == 0 ? 0 : w - 1;
    const long long csep0 = pclk();
    if (p < P - 1 && tid < 32 && (!HELM_DUAL_XPF_PROD || XF32)) {
      // (the XF32 variant, or the XPF_PROD = 0 ablation) stream this CTA's rows of the
      // separator inverse into L2 while the all-gather completes
      const long ld = x_ld(K, w);
      if constexpr (XF32) {
        const uint32_t bytes = (uint32_t)((long)K * w * (long)sizeof(float2));
        for (int r = tid; r < w; r += 32) dprefetch_l2(tab[i].xinv32 + ((long)p * w + r) * ld, bytes, pol_first);
      } else {
        const uint32_t bytes = (uint32_t)((long)K * w * (long)sizeof(cplx));
        for (int r = tid; r < w; r += 32) dprefetch_l2(tab[i].xinv + ((long)p * w + r) * ld, bytes, pol_first);
      }
    }
    // publish this segment's contributions to its two separator right-hand sides:
    //   yb[0..w)   = U_{lo-1} x0_lo   (enters g_{p-1}),  yb[wmax..) = U_hi^T x0_hi  (enters g_p)
    // with the staged couplings of rows lo-1 (bcr/bne row 0) and hi (row m)
    cplx* yb = D_.yb + par * exs + (long)p * 2 * D_.wmax;
    for (int e = tid; e < w; e += ncons) {
      const cplx* xl = zlo;                       // x0_lo
      const cplx* xh = yseg + (long)(m - 1) * w;  // x0_hi = y_hi
      cplx tl = cmul(bcr[e], xl[e]);
      if (e + 1 < w) cfma(tl, bne[e], xl[e + 1]);
      cplx th = cmul(bcr[(long)m * bw + e], xh[e]);
      if (e >= 1) cfma(th, bne[(long)m * bw + e - 1], xh[e - 1]);
      yb[e] = tl;
      yb[D_.wmax + e] = th;
    }
    cbar();
    const long long cw0 = pclk();
    pacc(16, cw0 - csep0);
    const bool need_corr = st > 0 || bwd;
    if (tid == 0) {
      HELM_DUAL_FENCE();
      red_release_add(&D_.cnt[0], 1u);   // arrive: this segment's yb is published
      if (need_corr) {
        // every segment has published solve i-1's boundary rows (epilogue counter),
        // so the corrections can be formed while the slower segments finish phase 1
        while (ld_relaxed(&D_.cnt[1]) < (unsigned)(P * i)) __nanosleep(20);
        (void)ld_acquire(&D_.cnt[1]);
      }
    }
    cbar();
    // separator-row transmission corrections (from solve i-1) for every separator
    if (need_corr) {
      const int aprev = i > 0 ? tab[i - 1].a : 0;
      for (int k = tid; k < K; k += ncons) {
        const int sk = sepr[k];
        auto X = [&](int cc, int qq) -> cplx {
          if (cc == sk) return ldcg(D_.xs + ppar * xss + (long)k * D_.wmax + qq);
          if (cc == sk - 1) return ldcg(D_.xb + ppar * exs + (long)k * 2 * D_.wmax + D_.wmax + qq);
          return ldcg(D_.xb + ppar * exs + (long)(k + 1) * 2 * D_.wmax + qq);
        };
        cplx cp = cmk(0, 0), cn = cmk(0, 0);
        if (st > 0) {
          if (!bwd) {
            cp = correction_aw(D_, s, a, w, prev_side(D_), sk, aprev, X);
            if (k == p) D_.corr_prev[(long)st * D_.nc + sk] = cp;   // kept for the backward pass
          } else {
            cp = ldcg(D_.corr_prev + (long)st * D_.nc + sk);
          }
        }
        if (bwd) cn = correction_aw(D_, s, a, w, next_side(D_), sk, aprev, X);
        cpv[k] = cp;
        cnv[k] = cn;
      }
    }
    if (tid == 0) {
#ifndef HELM_DUAL_ABL_NOGW
      while (ld_relaxed(&D_.cnt[0]) < (unsigned)(P * (i + 1))) __nanosleep(20);
#endif
      (void)ld_acquire(&D_.cnt[0]);
    }
#if HELM_DUAL_GSRC
    cp_async_wait_all();   // the separator-row source staged at the pre-actions
#endif
    cbar();
    pacc(4, pclk() - cw0);
    pacc(12, pclk() - cw0);
    const long long cg0 = pclk();
    // g_k = b_{s_k} - U_{h_k}^T x0_k[hi] - U_{s_k} x0_{k+1}[lo]  (all K separators)
    const cplx* ybp = D_.yb + par * exs;
    // g_k = b_{s_k} (+ corrections) - U_{h_k}^T x0_k[hi] - U_{s_k} x0_{k+1}[lo]: the two
    // products were formed by the owning segments; four elements per thread and pass
    for (int e0 = tid; e0 < K * w; e0 += 4 * ncons) {
      cplx th[4], tl[4], gs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * ncons;
        const bool ok = e < K * w;
        const int k = ok ? e / w : 0, qq = ok ? e - k * w : 0;
        th[u] = ok ? ldcg(ybp + (long)k * 2 * D_.wmax + D_.wmax + qq) : cmk(0, 0);
        tl[u] = ok ? ldcg(ybp + (long)(k + 1) * 2 * D_.wmax + qq) : cmk(0, 0);
#if HELM_DUAL_GSRC
        gs[u] = ok ? gsm[e] : cmk(0, 0);                                    // source at the separator rows (staged)
#else
        gs[u] = ok ? ldcg(D_.R + node_of(D_, a, sepr[k], qq)) : cmk(0, 0);   // source at the separator rows
#endif
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * ncons;
        if (e >= K * w) break;
        const int k = e / w, qq = e - k * w;
        cplx v = gs[u];
        if (st > 0 && qq == qp) v = cadd(v, cpv[k]);
        if (bwd && qq == qn) v = cadd(v, cnv[k]);
        if (D_.disc == HELM_DISC_FD5) v = cscale(v, rhs_scale(D_, sepr[k], qq, w));
        gsm[e] = csub(csub(v, th[u]), tl[u]);
      }
    }
    cbar();
    // x_p = X_p g with X = R^{-1} complex symmetric: only the upper block triangle
    // is read, each of its blocks by its two users in the same stage (the second
    // read hits L2), so the separator-inverse HBM stream is halved:
    //   normal part      sum_{k >= p} X[p][r][k w + j] g_k[j]   (row r of block row p)
    //   transposed part  sum_{k <  p} X[k][i][p w + r] g_k[i]   (= X[p][r][k w + i])
    const long long cx0 = pclk();
    pacc(14, cx0 - cg0);
    const long Kw = (long)K * w, xld = x_ld(K, w);
    const int cw = tid >> 5, ncw = ncons >> 5;
#ifdef HELM_DUAL_ABL_NOXMV
    if (false) {
#else
    if (p < P - 1) {
#endif
      constexpr int XCH = HELM_DUAL_XCH;
      if constexpr (XF32) {
        // inexact separator solve (sweep_set_precision(32)): complex64 rows of R^{-1}, FP32
        // products and accumulation -- half the separator-inverse bytes, twice the columns
        // in flight for the same registers
        for (int rb = 4 * cw; rb < w; rb += 4 * ncw) {
          const float2* Xr[4];
          bool ok[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ok[u] = rb + u < w;
            Xr[u] = tab[i].xinv32 + ((long)p * w + (ok[u] ? rb + u : 0)) * xld;
          }
          float2 acc[4] = {make_float2(0, 0), make_float2(0, 0), make_float2(0, 0), make_float2(0, 0)};
          for (long jj = lane; jj < Kw; jj += 32 * 8) {
            float2 xv[4][8], gv[8];
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const bool in = jj + 32 * v < Kw;
              const cplx gd = in ? gsm[jj + 32 * v] : cmk(0, 0);
              gv[v] = make_float2((float)gd.x, (float)gd.y);
#pragma unroll
              for (int u = 0; u < 4; ++u) xv[u][v] = (ok[u] && in) ? ld_cg_hint_f2(Xr[u] + jj + 32 * v, pol_first) : make_float2(0, 0);
            }
#pragma unroll
            for (int v = 0; v < 8; ++v)
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                acc[u].x = fmaf(xv[u][v].x, gv[v].x, acc[u].x);
                acc[u].x = fmaf(-xv[u][v].y, gv[v].y, acc[u].x);
                acc[u].y = fmaf(xv[u][v].x, gv[v].y, acc[u].y);
                acc[u].y = fmaf(xv[u][v].y, gv[v].x, acc[u].y);
              }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              acc[u].x += __shfl_xor_sync(0xffffffffu, acc[u].x, off);
              acc[u].y += __shfl_xor_sync(0xffffffffu, acc[u].y, off);
            }
            if (lane == 0 && ok[u]) xhi[rb + u] = cmk((double)acc[u].x, (double)acc[u].y);
          }
        }
      } else {
      // Rounds of row-panel mat-vecs: one with the full explicit inverse (row block p of
      // R^{-1} times g), or two with the two-level panels (strip_setup.cu): panel 1 times
      // the gathered group separators' g (a coarse CTA then publishes its coarse RHS
      // gh = g_p - result), panel 2 times all coarse RHSs once published.
      const cplx* sep2 = tab[i].sep2;
      const int* pk = spk;
      const bool coarse = sep2 && pk[0] == 1;
      const int M2 = D_.sep2_M;
      cplx* vx = bseg;                       // gathered panel vector (bseg is free in this stage)
      cplx* ytmp = bseg + (long)(2 * 8 + 8) * w;   // round-1 result of a fine separator
      cplx* gh = D_.gh + (long)par * M2 * D_.wmax;
      const int nround = sep2 ? 2 : 1;
      long long crd = pclk();
      for (int rd = 0; rd < nround; ++rd) {
        const cplx* pbase;
        long ld, ncol;
        const cplx* vec;
        cplx* out;
        if (!sep2) {
          pbase = tab[i].xinv + (long)p * w * xld; ld = xld; ncol = Kw; vec = gsm; out = xhi;
        } else if (rd == 0) {
          const int n1 = pk[1];
          for (int e = tid; e < n1 * w; e += ncons) {
            const int b2 = e / w, qq = e - b2 * w;
            vx[e] = gsm[(long)pk[4 + b2] * w + qq];
          }
          cbar();
          pbase = sep2 + (long)p * w * (D_.sep2_ld1 + D_.sep2_ld2); ld = D_.sep2_ld1; ncol = (long)n1 * w; vec = vx;
          out = coarse ? xhi : ytmp;
        } else {
          // every coarse RHS is published: gather them
          if (tid == 0) {
            while (ld_relaxed(&D_.cnt[2]) < (unsigned)(M2 * (i + 1))) __nanosleep(20);
            (void)ld_acquire(&D_.cnt[2]);
          }
          cbar();
          pacc(24, pclk() - crd);   // (two-level) wait for the coarse RHSs
          crd = pclk();
          for (int e = tid; e < M2 * w; e += ncons) {
            const int j = e / w, qq = e - j * w;
            vx[e] = ldcg(gh + (long)j * D_.wmax + qq);
          }
          cbar();
          pbase = sep2 + (long)p * w * (D_.sep2_ld1 + D_.sep2_ld2) + (long)w * D_.sep2_ld1; ld = D_.sep2_ld2;
          ncol = (long)M2 * w; vec = vx; out = xhi;
        }
        // 4 rows per warp, lanes over the columns, XCH loads in flight per lane
        for (int rb = 4 * cw; rb < w; rb += 4 * ncw) {
          const cplx* Xr[4];
          bool ok[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ok[u] = rb + u < w;
            Xr[u] = pbase + (long)(ok[u] ? rb + u : 0) * ld;
          }
          cplx acc[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
          for (long jj = lane; jj < ncol; jj += 32 * XCH) {
            cplx xv[4][XCH], gv[XCH];
#pragma unroll
            for (int v = 0; v < XCH; ++v) {
              const bool in = jj + 32 * v < ncol;
              gv[v] = in ? vec[jj + 32 * v] : cmk(0, 0);
#pragma unroll
              for (int u = 0; u < 4; ++u) xv[u][v] = (ok[u] && in) ? ld_cg_hint(Xr[u] + jj + 32 * v, pol_first) : cmk(0, 0);
            }
#pragma unroll
            for (int v = 0; v < XCH; ++v)
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
            if (lane == 0 && ok[u]) out[rb + u] = acc[u];
          }
        }
        cbar();
        pacc(rd == 0 ? 25 : 26, pclk() - crd);   // (two-level) round 1 / round 2 mat-vecs (incl. gathers)
        crd = pclk();
        if (sep2 && rd == 0 && coarse) {
          // gh_c = g_p - H g (this coarse separator's index pk[2])
          for (int e = tid; e < w; e += ncons) gh[(long)pk[2] * D_.wmax + e] = csub(gsm[(long)p * w + e], xhi[e]);
          cbar();
          if (tid == 0) red_release_add(&D_.cnt[2], 1u);
        }
        if (sep2 && rd == 1 && !coarse)
          for (int e = tid; e < w; e += ncons) xhi[e] = csub(ytmp[e], xhi[e]);   // x_p = y_p - Q_p gh
      }
      }
    }
    cbar();
    for (int e = tid; e < WM; e += ncons) {
      if (p == 0) xlo[e] = cmk(0, 0);
      if (p == P - 1) xhi[e] = cmk(0, 0);
    }
    cbar();
    pacc(2, pclk() - cx0);
    // publish x_p (parity buffer; also the next solve's correction source),
    // then take x_{p-1} from the left neighbour
    if (p < P - 1) {
      for (int e = tid; e < w; e += ncons) D_.xs[par * xss + (long)p * D_.wmax + e] = xhi[e];
      cbar();
      if (tid == 0) {
        HELM_DUAL_FENCE();
        st_release(&D_.flag[p], (unsigned)(i + 1));
      }
    }
    pacc(17, pclk() - cx0);   // X mat-vec + fixups + publication
    if (p > 0) {
      const long long cw1 = pclk();
      if (tid == 0) {
        while (ld_relaxed(&D_.flag[p - 1]) < (unsigned)(i + 1)) __nanosleep(20);
        (void)ld_acquire(&D_.flag[p - 1]);
      }
      cbar();
      pacc(4, pclk() - cw1);
      pacc(13, pclk() - cw1);
      for (int e = tid; e < w; e += ncons) xlo[e] = ldcg(D_.xs + par * xss + (long)(p - 1) * D_.wmax + e);
      cbar();
    }
    const long long cvi = pclk();
    // phase-3 inputs: chain A  U_hi x_p;  chain B  -U_{lo-1}^T x_{p-1}
    cplx* vA = vbuf + 0 * 2 * WM + cur * WM;
    cplx* vB = vbuf + 1 * 2 * WM + cur * WM;
    for (int qq = tid; qq < w; qq += ncons) {
      const cplx* crr = bcr + (long)m * bw;     // row hi
      const cplx* ner = bne + (long)m * bw;
      cplx ta = cmul(crr[qq], xhi[qq]);
      if (qq + 1 < w) cfma(ta, ner[qq], xhi[qq + 1]);
      vA[qq] = ta;
      cplx tb = cmul(bcr[qq], xlo[qq]);          // row lo-1
      if (qq >= 1) cfma(tb, bne[qq - 1], xlo[qq - 1]);
      vB[qq] = cscale(tb, -1.0);
    }
    pacc(18, pclk() - cvi);
  };

  // ------------------------------------------------------------ one phase of this group's chain
  // Chain G, phase PH (0: forward elimination / bottom-up elimination, 1: the
  // phase-3 chain), m block steps on solve i.  Factor blocks are loaded into
  // registers two steps ahead (per-lane packed offsets precomputed per phase),
  // the mode-specific writer is resolved at compile time.
  uint32_t cseq = 0;   // blocks consumed by this chain group
  const uint32_t ring_base = smem_u32(ring + (long)g * NST * A.stage_elems);
  const uint32_t stage_bytes = (uint32_t)A.stage_elems * (uint32_t)sizeof(cplx);

  // ------------------------------------------------------------ one phase of this group's chain
  // Chain G, phase PH (0: top-down / bottom-up elimination, 1: the phase-3
  // chain), m block steps on solve i.  Each step waits for its packed block in
  // the ring, reads this lane's nine entries with precomputed byte offsets, and
  // the group's producer refills the stage freed by the previous step.
  auto run_phase = [&](int i, auto G_, auto PH_) {
    constexpr int G = decltype(G_)::value;
    constexpr int PH = decltype(PH_)::value;
    constexpr bool up = (G == 0) == (PH == 0);   // A1, B3 walk lo -> hi
    constexpr int high = up ? 0 : 1;             // lo -> hi steps need o[r-1]: low-halo mapping
    constexpr bool sub = G == 0 && PH == 1;      // chain A back substitution: o = y_c - Sinv v
    const int w = tab[i].w;
    const int bsc = D_.axis == 0 ? w : 1;
    const int row = dslot_row(wi, slot, high);
    const bool act = row >= 0 && row < w;
    const bool owned = q == 0 && act && dslot_owned(slot, high);
    // packed-triangle byte offsets of this lane's entries k = q + 4c: k >= row from
    // row `row`, k < row from row k (column `row`); others -> the zero entry
    uint32_t off[KPL];
    {
      const int rs = act ? pkst[row] : 0;
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        const int k = q + LPR * c;
        int idx = A.stage_elems - 1;
        if (act && k < w) idx = k >= row ? rs + (k - row) : pkst[k] + (row - k);
        off[c] = (uint32_t)idx * (uint32_t)sizeof(cplx);
      }
    }
    // this lane's nine entries of the block consumed as sequence number `seq`
    auto load_S = [&](cplx (&S)[KPL], uint32_t seq) {
      const int st = seq % NST;
      mbar_wait(&full[G * NST + st], (seq / NST) & 1);
      const uint32_t sb = ring_base + st * stage_bytes;
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
#if defined(HELM_DUAL_ABL_CFREE)
        S[c] = lds128(sb + (uint32_t)((gtid * KPL + c) % 600) * 16u);   // ablation: conflict-free, wrong values
#elif defined(HELM_DUAL_ABL_NOS)
        S[c] = cmk(1e-3 * c + 1e-4 * (sb & 7), 1e-3);                    // ablation: no block loads
#else
        S[c] = lds128(sb + off[c]);
#endif
      }
    };
    // one block step with this block's entries in Sc; the next block's entries are
    // read into Sn while the reductions, the writer and the barrier of this step
    // run, so only the input-vector loads sit on the dependent path
    // writer operands (independent of this step's result): couplings of the
    // next input and, for the sweeps that subtract, the source row
    auto load_wops = [&](int ci, bool last, cplx& wc, cplx& wn, cplx& wb, cplx& ysub) {
      constexpr bool cplus = (G == 0 && PH == 0) || (G == 1 && PH == 1);
      if (owned && !last) {
        const int crow = cplus ? ci + 1 : ci;
        wc = bcr[crow * bw + row];
        if (cplus) { if (row >= 1) wn = bne[crow * bw + row - 1]; }
        else if (row + 1 < w) wn = bne[crow * bw + row];
        if (G == 0 && PH == 0) wb = bseg[(ci + 1) * bsc + row * bsq];
        if (G == 1 && PH == 0) wb = bseg[(ci - 1) * bsc + row * bsq];
      }
      if (sub && act) ysub = yseg[ci * w + row];
#ifdef HELM_DUAL_ABL_NOWOPS
      wc = cmk(1e-3, 0); wn = cmk(1e-4, 0); wb = cmk(1e-5, 0); ysub = cmk(0, 0);   // ablation: no writer operand loads
#endif
    };
    auto step = [&](int js, cplx (&Sc)[KPL], cplx (&Sn)[KPL]) {
      long long q0 = 0;
      if (kProfStep && A.prof && tid == 0) q0 = pclk();
      const int st = cseq % NST;
      const int ci = up ? js : m - 1 - js;   // local block row
      const bool last = js == m - 1;
      const cplx* vin = myv + cur * WM;
      cplx wc = cmk(0, 0), wn = cmk(0, 0), wb = cmk(0, 0), ysub = cmk(0, 0);
#if !HELM_DUAL_WOPS_LATE
      load_wops(ci, last, wc, wn, wb, ysub);
#endif
      cplx vv[KPL];
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
#ifdef HELM_DUAL_ABL_NOVIN
        vv[c] = cmk(1e-3 * c, 0.0);     // ablation: no input-vector loads
#else
        vv[c] = vin[q + LPR * c];       // entries k >= w of the input are zero-padded
#endif
      }
      long long q1 = 0;
      if (kProfStep && A.prof && tid == 0) { q1 = pclk(); pacc(8, q1 - q0); }
      cplx a0 = cmk(0, 0), a1 = cmk(0, 0), a2 = cmk(0, 0), a3 = cmk(0, 0);
#if HELM_DUAL_SNPOS == 1
      // next block: wait for it, then read each entry right after its register pair is consumed
      uint32_t sbn = 0;
      if (!last) {
        const int stn = (cseq + 1) % NST;
        mbar_wait(&full[G * NST + stn], ((cseq + 1) / NST) & 1);
        sbn = ring_base + stn * stage_bytes;
      }
#elif HELM_DUAL_SNPOS == 2
      if (!last) load_S(Sn, cseq + 1);
#endif
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        if ((c & 3) == 0) cfma(a0, Sc[c], vv[c]);
        else if ((c & 3) == 1) cfma(a1, Sc[c], vv[c]);
        else if ((c & 3) == 2) cfma(a2, Sc[c], vv[c]);
        else cfma(a3, Sc[c], vv[c]);
#if HELM_DUAL_SNPOS == 1
        if (!last) Sn[c] = lds128(sbn + off[c]);
#endif
      }
      cplx acc = cadd(cadd(a0, a1), cadd(a2, a3));
#if HELM_DUAL_WOPS_LATE
      load_wops(ci, last, wc, wn, wb, ysub);   // behind the input-vector loads in the LSU queue
#endif
#if HELM_DUAL_SNPOS == 0
      if (!last) load_S(Sn, cseq + 1);   // Sc is dead: Sn can take its registers
#endif
#ifndef HELM_DUAL_ABL_NOSHFL
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 8);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 8);
#endif
      cplx o = acc;
      if (sub) o = act ? csub(ysub, acc) : cmk(0, 0);
      cplx nb;
      if (high) {
        nb.x = __shfl_down_sync(0xffffffffu, o.x, 1, 8);
        nb.y = __shfl_down_sync(0xffffffffu, o.y, 1, 8);
      } else {
        nb.x = __shfl_up_sync(0xffffffffu, o.x, 1, 8);
        nb.y = __shfl_up_sync(0xffffffffu, o.y, 1, 8);
      }
      long long q2 = 0;
      if (kProfStep && A.prof && tid == 0) { q2 = pclk(); pacc(9, q2 - q1); }
      if (owned) {
        cplx* vn = myv + (cur ^ 1) * WM;
        if (G == 0 && PH == 0) yseg[ci * w + row] = o;          // A1: y_c; next b_{c+1} - U_c^T y_c
        else if (G == 0) xa[ci * w + row] = o;                  // A3: xa_c; next U_{c-1} xa_c
        else if (PH == 1) fb[ci * w + row] = o;                 // B3: f_c; next -U_c^T f_c
        else if (last) zlo[row] = o;                            // B1: z_lo = x0_lo
        if (!last) {                                            // B1: next b_{c-1} - U_{c-1} z_c
          cplx t = cmul(wc, o);
          cfma(t, wn, nb);
          if (PH == 0) vn[row] = csub(wb, t);
          else vn[row] = G == 0 ? t : cscale(t, -1.0);
        }
      }
#if HELM_DUAL_SNPOS == 3
      if (!last) load_S(Sn, cseq + 1);
#endif
      long long q3 = 0;
      if (kProfStep && A.prof && tid == 0) { q3 = pclk(); pacc(10, q3 - q2); }
      gbar();
      if (gtid == 0) mbar_arrive(&empty[G * NST + st]);   // every lane of the group is done with the stage
      if (kProfStep && A.prof && tid == 0) pacc(11, pclk() - q3);
      ++cseq;
      cur ^= 1;
    };
    cplx SA[KPL], SB[KPL];
    load_S(SA, cseq);
    int js = 0;
    for (; js + 1 < m; js += 2) {
      step(js, SA, SB);
      step(js + 1, SB, SA);
    }
    if (js < m) step(js, SA, SB);
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;

  // the solve loop, instantiated per chain group (each group only carries the
  // registers of its own two phases)
  auto solve_loop = [&](auto G_) {
    for (int i = 0; i < nsolve; ++i) {
      const int w = tab[i].w;
      // ---- pre-actions: epilogue of the previous solve, RHS, phase-1 inputs
      long long c0 = pclk();
      cbar();
      if (!kProfStep) pacc(9, pclk() - c0);   // the other chain group's phase 3 tail
      const long long csb = pclk();
      stage_bands(i);
      pacc(22, pclk() - csb);
      if (i == 0) {
        stage_rhs0();
        mbar_wait(&sbar[2], 0);
      } else {
        mbar_wait(&sbar[0], (i - 1) & 1);   // staged during phase 3 of solve i-1
        cp_async_wait_all();
        pacc(23, pclk() - csb);
        seg_epilogue(i - 1);
        cbar();
        // epilogue counter: solve i-1's boundary rows (xb) and separators (xs) are
        // published; the separator stage of solve i forms its corrections from them
#if HELM_DUAL_EPIREL
        // (the release itself -- a gpu-scope fence behind this CTA's Z stores -- is
        // done by chain B's producer lane after this CTA-scope arrival, off the barrier)
        if (tid == 0) mbar_arrive(&sbar[3]);
#else
        if (tid == 0) red_release_add(&D_.cnt[1], 1u);
#endif
      }
      const long long cpb = pclk();
      if (!kProfStep) pacc(10, cpb - c0);
      mbar_wait(&sbar[1], i & 1);
      cbar();
      pacc(15, pclk() - cpb);   // couplings landed
      seg_rhs(i);
#if HELM_DUAL_GSRC
      {
        // the source at the separator rows is constant during the solve: copy it into
        // the g area now (free until the separator stage), off the stage's critical path
        const int a = tab[i].a;
        for (int e = tid; e < K * w; e += ncons) {
          const int k = e / w, qq = e - k * w;
          cp_async16(gsm + e, D_.R + node_of(D_, a, sepr[k], qq));
        }
        cp_async_commit();
      }
#endif
      cbar();
      for (int e = tid; e < w; e += ncons) {
        const int bsc = D_.axis == 0 ? w : 1;
        vbuf[0 * 2 * WM + cur * WM + e] = bseg[e * bsq];                  // chain A: b_lo
        vbuf[1 * 2 * WM + cur * WM + e] = bseg[(m - 1) * bsc + e * bsq];  // chain B: b_hi
      }
      if (tid == 0 && (i == 0 || tab[i - 1].w != w)) {
        for (int r = 0, x = 0; r < w; ++r) {   // padded packed row starts (common.cuh pk_start)
          pkst[r] = x;
          x += w - r;
          const int want = (2 * (r + 1)) & 7;
          while ((x & 7) != want) ++x;
        }
      }
      cbar();
      pacc(0, pclk() - c0);
      const long long cph1 = pclk();
#if HELM_DUAL_ONELOOP
      if (g == 0) run_phase(i, I0{}, I0{});
      else run_phase(i, I1{}, I0{});
#else
      run_phase(i, G_, I0{});
#endif
      // ---- separator stage, phase-3 inputs
      c0 = pclk();
      pacc(19, c0 - cph1);
      if (kProf && A.prof && tid == 0 && i < 64) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        A.prof[(long)gridDim.x * 32 + (long)blockIdx.x * 64 + i] = (long long)gt;   // phase-1 end, ns
      }
      cbar();
      seg_separators(i);
      cbar();
      pacc(1, pclk() - c0);
      const long long csn = pclk();
#ifndef HELM_DUAL_ABL_NONEXT
      stage_next(i);
#else
      if (tid == 0) mbar_expect_tx(&sbar[0], 0);
#endif
      const long long cph3 = pclk();
      pacc(21, cph3 - csn);
#if HELM_DUAL_ONELOOP
      if (g == 0) run_phase(i, I0{}, I1{});
      else run_phase(i, I1{}, I1{});
#else
      run_phase(i, G_, I1{});
#endif
      pacc(20, pclk() - cph3);
    }
  };
#if HELM_DUAL_ONELOOP
  solve_loop(I0{});   // one copy of the per-solve code; the chain phases dispatch on the group
#else
  if (g == 0) solve_loop(I0{});
  else solve_loop(I1{});
#endif
  cbar();
  mbar_wait(&sbar[0], (nsolve - 1) & 1);
  seg_epilogue(nsolve - 1);
  if (kProf && A.prof && tid == 0) {
    long long* o = A.prof + (long)blockIdx.x * 32;
    for (int k = 0; k < 32; ++k) o[k] = profs[k];
    o[3] = total;
    o[5] = pclk() - t_start; o[6] = 1; o[7] = d;
  }
}

// ------------------------------------------------------------------ host
static constexpr int kDualSmemMax = 227 * 1024;
extern long long* helm_sweep_prof_buffer();

// Launches the two-chain kernel if every direction fits it (w <= 36, P > 1,
// explicit separator inverse and bottom-up inverses built at setup); returns
// -1 (not applicable) otherwise.
int sweep_apply_dual(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                     cudaStream_t st) {
  using namespace dualk;
  int wmax = 0, pmax = 1, nsolve_max = 1;
  for (int d = 0; d < t; ++d) {
    wmax = std::max(wmax, dirs[d]->wmax);
    pmax = std::max(pmax, dirs[d]->P);
    nsolve_max = std::max(nsolve_max, dirs[d]->is_double ? 2 * dirs[d]->N - 1 : dirs[d]->N);
    if (dirs[d]->P < 2 || !dirs[d]->d_xinv || !dirs[d]->d_fac2 || !dirs[d]->d_facp) return -1;
  }
  if (wmax > LPR * KPL || wmax > WM) return -1;
  const int nw = (wmax + OWN - 1) / OWN;
  const int threads = 2 * nw * 32 + 64;   // two chain groups + two TMA producer warps
  if (threads > MAXT) return -1;
  long vec_elems = 0, gsm_elems = 0;
  int ctas = 0, mmax_all = 1;
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    int mmax = 0;
    for (int p = 0; p < h->P; ++p) mmax = std::max(mmax, h->seg_hi[p] - h->seg_lo[p] + 1);
    vec_elems = std::max(vec_elems, (long)(mmax + 1) * h->wmax);
    mmax_all = std::max(mmax_all, mmax);
    gsm_elems = std::max(gsm_elems, (long)(h->P - 1) * h->wmax);
    ctas += h->P;
  }
  vec_elems = (vec_elems + 7) / 8 * 8;
  const long stage_elems = pk_size(wmax) + 8;   // padded packed block + a zero entry, 128-byte multiple
  size_t smem = sizeof(cplx) * 2 * NST * stage_elems + sizeof(uint64_t) * (4 * NST + 4) +
                sizeof(cplx) * (7 * WM + 2 * pmax) + sizeof(DualTab) * nsolve_max + sizeof(int) * (WM + pmax) + 256;
  // g aliases xa and, when it is longer, the adjacent fb (both are free from the
  // epilogue to the end of the separator stage); its own area only beyond that
  const bool gsep = gsm_elems > 2 * vec_elems;
  smem = (smem + 127) / 128 * 128 + sizeof(cplx) * (6 * vec_elems + (2L + kTcW) * mmax_all + (gsep ? gsm_elems : 0));
  // inexact separator solve only when every direction of the batch asked for it
  bool xf32 = true;
  for (int d = 0; d < t; ++d) xf32 = xf32 && dirs[d]->sep_fp32 && dirs[d]->d_xinv32;
  const void* kfun = gsep ? (xf32 ? (const void*)k_sweep_dual<true, true> : (const void*)k_sweep_dual<true, false>)
                          : (xf32 ? (const void*)k_sweep_dual<false, true> : (const void*)k_sweep_dual<false, false>);
  if (smem > (size_t)kDualSmemMax) return -1;
  // scratch: the counters of every direction first (one memset), then per
  // direction the parity-buffered yb / xb / xs and the corrections
  std::vector<size_t> off(t), coff(t);
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t ncnt = 0;
  for (int d = 0; d < t; ++d) {
    coff[d] = ncnt;
    ncnt += 3 + dirs[d]->P;
  }
  size_t total = al(sizeof(unsigned) * ncnt);
  for (int d = 0; d < t; ++d) {
    const helm_sweep_s* h = dirs[d];
    off[d] = total;
    total += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax) * 2;
    total += al(sizeof(cplx) * 2L * h->P * h->wmax);
    total += al(sizeof(cplx) * (long)h->N * h->nc);
    total += al(sizeof(cplx) * (long)h->nc);
    total += al(sizeof(cplx) * 2L * 8 * h->wmax);   // gh (two-level coarse RHS, M <= 8)
  }
  unsigned char* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, total, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply: scratch alloc: %s", cudaGetErrorString(e));
    return HELM_ENOMEM;
  }
  const helm_problem_s* prob = dirs[0]->prob;
  DualArgs A;
  memset(&A, 0, sizeof(A));
  A.t = t;
  A.nw = nw;
  A.vec_elems = (int)vec_elems;
  A.nsolve_max = nsolve_max;
  A.pmax = pmax;
  A.stage_elems = (int)stage_elems;
  A.mmax = mmax_all;
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
    D.fac = h->d_fac; D.fac2 = h->d_fac2; D.facp = h->d_facp; D.pfac_off = h->d_pfac_off; D.fac_off = h->d_fac_off; D.red = h->d_red; D.red_off = h->d_red_off;
    D.xinv = h->d_xinv; D.xinv_off = h->d_xinv_off;
    D.xinv32 = xf32 ? h->d_xinv32 : nullptr;
    D.R = Rdev + (ldr == 0 ? 0 : (long)d * ldr);
    D.Z = Zdev + (long)d * ldz;
    unsigned char* q = scratch + off[d];
    D.cnt = reinterpret_cast<unsigned*>(scratch) + coff[d]; D.flag = D.cnt + 3;
    D.yb = (cplx*)q; q += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax);
    D.xb = (cplx*)q; q += al(sizeof(cplx) * 2L * 2 * h->P * h->wmax);
    D.xs = (cplx*)q; q += al(sizeof(cplx) * 2L * h->P * h->wmax);
    D.corr_prev = (cplx*)q; q += al(sizeof(cplx) * (long)h->N * h->nc);
    D.corr_next = (cplx*)q; q += al(sizeof(cplx) * (long)h->nc);
    D.gh = (cplx*)q;
    // two-level separator panels when the gathered panel vectors fit the RHS area
    const bool s2 = h->d_sep2 && !xf32 && vec_elems >= (long)(2 * 8 + 8 + 1) * h->wmax;
    D.sep2 = s2 ? h->d_sep2 : nullptr; D.sep2_off = h->d_sep2_off; D.sep2_plan = h->d_sep2_plan;
    D.sep2_M = h->sep2_M; D.sep2_ld1 = h->sep2_ld1; D.sep2_ld2 = h->sep2_ld2;
    D.wmax = h->wmax;
    D.cta_base = base;
    base += h->P;
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(scratch, 0, sizeof(unsigned) * ncnt, st);
  // the attribute / occupancy queries cost host time on every iteration's critical
  // path (the solve is host-synchronous): cache them per (kernel, shared memory)
  int dev = 0, nsm = 0, occ = 0;
  {
    // (the dynamic shared-memory attribute is raised to the largest size ever
    // launched, never lowered: a cached smaller setting must not cap a later launch)
    struct OccKey { const void* f; size_t smem; int threads, dev; int nsm, occ; };
    struct AttrMax { const void* f; int dev; size_t smem; };
    static std::mutex mu;
    static std::vector<OccKey> cache;
    static std::vector<AttrMax> attr;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    bool raised = false;
    for (AttrMax& a : attr)
      if (a.f == kfun && a.dev == dev) {
        raised = true;
        if (smem > a.smem && e == cudaSuccess) {
          e = cudaFuncSetAttribute(kfun, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          if (e == cudaSuccess) a.smem = smem;
        }
      }
    if (!raised && e == cudaSuccess) {
      e = cudaFuncSetAttribute(kfun, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) attr.push_back(AttrMax{kfun, dev, smem});
    }
    bool hit = false;
    for (const OccKey& c : cache)
      if (c.f == kfun && c.smem == smem && c.threads == threads && c.dev == dev) { nsm = c.nsm; occ = c.occ; hit = true; }
    if (!hit) {
      if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfun, threads, smem);
      if (e == cudaSuccess) cache.push_back(OccKey{kfun, smem, threads, dev, nsm, occ});
    }
  }
  if (e == cudaSuccess && occ * nsm < ctas) {
    cudaFreeAsync(scratch, st);
    return -1;   // not co-resident: the caller falls back to the single-chain kernel
  }
  if (e == cudaSuccess) {
    void* args[] = {(void*)&A};
    e = cudaLaunchCooperativeKernel(kfun, dim3(ctas), dim3(threads), args, smem, st);
    g_helm_launches++;
  }
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) {
    helm_set_error("sweep_apply (dual): %s", cudaGetErrorString(e));
    return HELM_ECUDA;
  }
  return HELM_OK;
}
