// warp_gj.cuh -- Gauss-Jordan inversion of a w x w (w <= 36) complex block by ONE
// warp, no CTA barrier: the strip factorisation's block inverses
// (Sinv_c = S_c^{-1}, S'^{-1}_c; DESIGN.md §5 "Strip factors"), laid out for
// throughput (thousands of independent segment chains, one per warp).
//
// Layout: lane i holds row i (i < 32) in registers, a[s] = column (s + k0) mod 36
// during the pass of pivots k0 .. k0 + U - 1 (the slots rotate by U after each
// pass, so the pivot column is always a compile-time slot: no register selects).
// Rows 32..w-1 ("extra" rows, w > 32) live in shared memory (g.ext[e][col]); lane
// l updates columns l and l + 32 of them.
// Implicit partial pivoting with the pivot rule of row_invert (row_gj.cuh): the
// largest |a_ik|^2 among unused rows, compared on the high 32 bits of the double,
// ties to the lowest row.  Deferred normalisation: the pivot row is published raw
// (its pivot entry set to 1) and every other row subtracts (a_ik / piv) times it;
// each row stays its normalised counterpart times its own pivot (elimination is
// linear per row), so one scaling by 1/pivot per row at the end gives the inverse
// (no per-pivot work on the pivot lane alone).  The pivot column is published as
// piv + 1 so that a_ik - (a_ik / piv)(piv + 1) leaves -a_ik / piv there.  One
// __syncwarp per pivot (the pivot row double-buffered by pivot parity).
#pragma once
#include "../paper_2408_11929_b200/csrc/common.cuh"

static constexpr int kWW = 36;   // register slots per lane (columns), also the row stride of the output
static constexpr int kWX = 4;    // extra rows (w - 32) at most

struct WarpGJ {
  cplx prow[2][2 * kWW];   // pivot row, index col (col >= k0) or col + 36 (col < k0)
  cplx fext[2][kWX];       // the extra rows' column-k entries
  cplx dx[kWX];            // 1 / pivot of each extra row
  int pivrow[kWW];         // row chosen at step k (extra rows: 32 + e)
  cplx ext[kWX][kWW];      // rows 32 .. w-1 (natural column order)
};

__device__ __forceinline__ void warp_gj_init(WarpGJ& g) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < 2 * 2 * kWW; e += 32) (&g.prow[0][0])[e] = cmk(0, 0);
  __syncwarp();
}

// In-place inversion.  On return (0) lane i's row was the pivot of step ks (its
// kstep), extra row e that of kx[e]; the natural-order inverse is
//   Ainv[kstep(i)][pivrow[j]] = (row i, column j)   (warp_gj_store).
// Returns 1 (warp-uniformly) when every candidate of a pivot column is zero.
template <int U>
__device__ __forceinline__ int warp_invert(cplx (&a)[kWW], int w, WarpGJ& g, int& ks, int (&kx)[kWX]) {
  static_assert(kWW % U == 0, "the slots rotate by U");
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int nx = w > 32 ? w - 32 : 0;
  bool used = lane >= w;
  cplx dmine = cmk(1.0, 0.0);   // 1 / pivot of this lane's row
  unsigned usedx = 0;
#pragma unroll
  for (int e = 0; e < kWX; ++e)
    if (e >= nx) usedx |= 1u << e;
#pragma unroll 1
  for (int k0 = 0; k0 < kWW; k0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u;
      if (k < w) {
        const int kl = k & 31;   // the lane that searches / publishes column k of the extra rows
        const int buf = k & 1;
        // ---- pivot search
        const unsigned km = used ? 0u : (unsigned)__double2hiint(cabs2(a[u])) + 1u;
        unsigned kxm = 0u;
        int ex = 0;
        if (lane == kl) {
#pragma unroll
          for (int e = 0; e < kWX; ++e) {
            const cplx v = g.ext[e][k];
            g.fext[buf][e] = v;
            if (!((usedx >> e) & 1u)) {
              const unsigned kk = (unsigned)__double2hiint(cabs2(v)) + 1u;
              if (kk > kxm) { kxm = kk; ex = e; }
            }
          }
        }
        const unsigned kmax = __reduce_max_sync(FULL, km > kxm ? km : kxm);
        if (kmax <= 1u) return 1;   // all candidates zero (key 1 = +0.0)
        const unsigned who = __ballot_sync(FULL, km == kmax);
        const bool pm = who != 0u;   // the pivot is a main row (lower rows win ties)
        const int p = pm ? __ffs(who) - 1 : __shfl_sync(FULL, ex, kl);
        const cplx mine = pm ? a[u] : g.ext[p][k];
        cplx akk;
        {
          const int src = pm ? p : kl;
          akk.x = __shfl_sync(FULL, mine.x, src);
          akk.y = __shfl_sync(FULL, mine.y, src);
        }
        const cplx dinv = cinv(akk);
        const cplx pone = cmk(akk.x + 1.0, akk.y);
        // ---- publish the raw pivot row (pivot entry piv + 1), keep it with a 1 there
        if (pm) {
          if (lane == p) {
#pragma unroll
            for (int s = 0; s < kWW; ++s) g.prow[buf][k0 + s] = (s == u) ? pone : a[s];
            a[u] = cmk(1.0, 0.0);
            dmine = dinv;
            used = true;
            ks = k;
          }
        } else {
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            const int col = lane + 32 * sl;
            if (col < w) {
              const int ix = col >= k0 ? col : col + kWW;
              if (col == k) {
                g.prow[buf][ix] = pone;
                g.ext[p][col] = cmk(1.0, 0.0);
              } else {
                g.prow[buf][ix] = g.ext[p][col];
              }
            }
          }
          if (lane == 0) g.dx[p] = dinv;
          usedx |= 1u << p;
#pragma unroll
          for (int e = 0; e < kWX; ++e)
            if (e == p) kx[e] = k;
        }
        if (lane == 0) g.pivrow[k] = pm ? p : 32 + p;
        __syncwarp();
        // ---- eliminate column k from every other row: the extra rows, then the register rows
#pragma unroll
        for (int e = 0; e < kWX; ++e) {
          if (e < nx && (pm || e != p)) {
            const cplx f = cmul(g.fext[buf][e], dinv);
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              const int col = lane + 32 * sl;
              if (col < w) {
                const cplx r = g.prow[buf][col >= k0 ? col : col + kWW];
                cplx v = g.ext[e][col];
                v.x = fma(-f.x, r.x, v.x);
                v.x = fma(f.y, r.y, v.x);
                v.y = fma(-f.x, r.y, v.y);
                v.y = fma(-f.y, r.x, v.y);
                g.ext[e][col] = v;
              }
            }
          }
        }
        asm volatile("" ::: "memory");
        if (lane < w && !(pm && lane == p)) {
          const cplx f = cmul(a[u], dinv);
#pragma unroll
          for (int s = 0; s < kWW; ++s) {   // a -= f r, four fused multiply-adds
            const cplx r = g.prow[buf][k0 + s];
            a[s].x = fma(-f.x, r.x, a[s].x);
            a[s].x = fma(f.y, r.y, a[s].x);
            a[s].y = fma(-f.x, r.y, a[s].y);
            a[s].y = fma(-f.y, r.x, a[s].y);
          }
        }
      }
    }
    // rotate the slots by U: slot s holds column (s + k0 + U) mod 36 next pass
    cplx t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = a[u];
#pragma unroll
    for (int s = 0; s + U < kWW; ++s) a[s] = a[s + U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[kWW - U + u] = t[u];
  }
  // ---- the deferred normalisation: every row by 1 / its pivot
#pragma unroll
  for (int s = 0; s < kWW; ++s) a[s] = cmul(a[s], dmine);
  __syncwarp();   // pivrow, dx, ext complete
#pragma unroll
  for (int e = 0; e < kWX; ++e) {
    if (e < nx) {
      const cplx d = g.dx[e];
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const int col = lane + 32 * sl;
        if (col < w) g.ext[e][col] = cmul(g.ext[e][col], d);
      }
    }
  }
  __syncwarp();
  return 0;
}

// Natural-order inverse into mat (row stride kWW): Ainv[kstep][pivrow[j]].
__device__ __forceinline__ void warp_gj_store(const cplx (&a)[kWW], int w, const WarpGJ& g, int ks,
                                              const int (&kx)[kWX], cplx* mat) {
  const int lane = threadIdx.x & 31;
  if (lane < w) {
#pragma unroll
    for (int s = 0; s < kWW; ++s)
      if (s < w) mat[ks * kWW + g.pivrow[s]] = a[s];
  }
  const int nx = w > 32 ? w - 32 : 0;
#pragma unroll
  for (int e = 0; e < kWX; ++e) {
    if (e < nx) {
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const int col = lane + 32 * sl;
        if (col < w) mat[kx[e] * kWW + g.pivrow[col]] = g.ext[e][col];
      }
    }
  }
  __syncwarp();
}
