// krylov.cu -- hot-path rows a3 (source selection), a5 (SpMM), a6 (BCGS2 +
// intra-block CGS2 with deflation), a7 (host Householder least squares) and a8
// (x = Z y, true residual): mpgmres_solve, selective MPGMRES with
// the paper's selection rules, following SURVEY D10 step by step.
//
// Tall-skinny reductions are deterministic two-stage sums (per-block partials
// in a fixed row order, then a fixed-order sum over blocks): no fp64 atomics,
// so reruns are bitwise reproducible.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <complex>
#include <mutex>

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

int helm_spmm_dev(const helm_problem_s* p, const cplx* X, cplx* Y, int ncols, long ld, cudaStream_t st);
int sweep_apply_dev(const helm_sweep_t* dirs, int t, const cplx* Rdev, long ldr, cplx* Zdev, long ldz,
                    cudaStream_t st);

static constexpr int kDotChunk = 4096;   // rows*t per block in the dot kernel (64 KB of W in smem)
static constexpr int kDotThreads = 256;
static constexpr int kMaxT = 8;

// partial[b][j*t + i] = sum_{r in block b} conj(V[j][r]) * W[i][r]
// V: m columns (ld), W: t columns (ldw).  Warp per V column; W chunk in smem.
__global__ void __launch_bounds__(kDotThreads) k_dots(long n, int rows_blk, const cplx* __restrict__ V, long ldv,
                                                      int m, const cplx* __restrict__ W, long ldw, int t,
                                                      cplx* __restrict__ partial) {
  extern __shared__ cplx Wsm[];
  const long r0 = (long)blockIdx.x * rows_blk;
  const int rows = (int)min((long)rows_blk, n - r0);
  for (int i = 0; i < t; ++i)
    for (int r = threadIdx.x; r < rows; r += blockDim.x) Wsm[i * rows_blk + r] = W[i * ldw + r0 + r];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int j = warp; j < m; j += nw) {
    cplx acc[kMaxT];
#pragma unroll
    for (int i = 0; i < kMaxT; ++i) acc[i] = cmk(0, 0);
    const cplx* v = V + j * ldv + r0;
    for (int r = lane; r < rows; r += 32) {
      cplx vv = __ldg(v + r);
#pragma unroll
      for (int i = 0; i < kMaxT; ++i)
        if (i < t) cfmaconj(acc[i], vv, Wsm[i * rows_blk + r]);
    }
#pragma unroll
    for (int i = 0; i < kMaxT; ++i) {
      if (i >= t) break;
      for (int off = 16; off > 0; off >>= 1) {
        acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, off);
        acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, off);
      }
    }
    if (lane == 0)
      for (int i = 0; i < t; ++i) partial[(long)blockIdx.x * m * t + j * t + i] = acc[i];
  }
}

// out[j*t+i] (+)= sum_b partial[b][j*t+i], fixed order over b
__global__ void k_reduce_partials(const cplx* __restrict__ partial, int nblk, int mt, cplx* out, int accumulate) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < mt; e += gridDim.x * blockDim.x) {
    cplx acc = cmk(0, 0);
    for (int b = 0; b < nblk; ++b) acc = cadd(acc, partial[(long)b * mt + e]);
    out[e] = accumulate ? cadd(out[e], acc) : acc;
  }
}

// W[:, i] -= sum_j V[:, j] C[j*t + i]   (C: m x t, row-major by j)
__global__ void __launch_bounds__(256) k_update(long n, const cplx* __restrict__ V, long ldv, int m,
                                                const cplx* __restrict__ C, cplx* __restrict__ W, long ldw,
                                                int t) {
  extern __shared__ cplx Cs[];
  for (int e = threadIdx.x; e < m * t; e += blockDim.x) Cs[e] = C[e];
  __syncthreads();
  for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < n; r += (long)gridDim.x * blockDim.x) {
    cplx acc[kMaxT];
#pragma unroll
    for (int i = 0; i < kMaxT; ++i) acc[i] = cmk(0, 0);
    for (int j = 0; j < m; ++j) {
      cplx v = __ldg(V + j * ldv + r);
#pragma unroll
      for (int i = 0; i < kMaxT; ++i)
        if (i < t) cfma(acc[i], v, Cs[j * t + i]);
    }
    for (int i = 0; i < t; ++i) W[i * ldw + r] = csub(W[i * ldw + r], acc[i]);
  }
}

// y = alpha * x  (complex alpha)
__global__ void k_scale(long n, const cplx* __restrict__ x, cplx alpha, cplx* __restrict__ y) {
  for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < n; r += (long)gridDim.x * blockDim.x)
    y[r] = cmul(alpha, x[r]);
}

// y = sum_{j<m} V[:, j]  (t >= 3 sum rule)
__global__ void k_colsum(long n, const cplx* __restrict__ V, long ldv, int m, cplx* __restrict__ y) {
  for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < n; r += (long)gridDim.x * blockDim.x) {
    cplx acc = cmk(0, 0);
    for (int j = 0; j < m; ++j) acc = cadd(acc, V[j * ldv + r]);
    y[r] = acc;
  }
}

// x = Z y (Z: ncols columns), r = b - x handled by caller
__global__ void k_gemv(long n, const cplx* __restrict__ Z, long ldz, int ncols, const cplx* __restrict__ y,
                       cplx* __restrict__ x) {
  for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < n; r += (long)gridDim.x * blockDim.x) {
    cplx acc = cmk(0, 0);
    for (int j = 0; j < ncols; ++j) cfma(acc, __ldg(Z + j * ldz + r), y[j]);
    x[r] = acc;
  }
}

__global__ void k_axpy_sub(long n, const cplx* __restrict__ b, const cplx* __restrict__ ax, cplx* __restrict__ r) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    r[i] = csub(b[i], ax[i]);
}


// ------------------------------------------------------------------ fused orthogonalisation
// One cooperative launch per iteration runs row a6 (D10 steps 4-5):
//   gram_i = ||A z_i||^2                               (deflation reference)
//   C1 = V^H W; W -= V C1; C2 = V^H W; W -= V C2         (BCGS2 against V_1..k)
//   for i = 0..t-1: two CGS passes of w_i against the new slots V[:, m..m+i),
//     nrm_i = ||w_i||, keep iff nrm_i > 1e-10 ||A z_i||, V[:, m+i] = w_i/nrm_i (else 0)
// Block b owns a contiguous row range and walks it in tiles of kOrthTile rows:
// a tile of W is updated (thread per row) and staged in shared memory, then the
// warps form the projections (warp per V column, lanes over rows) into per-block
// partials.  Reductions are two-stage in a fixed order (partials, grid sync, a
// fixed-order sum over blocks), so results are bitwise reproducible; norms are
// summed redundantly by every block, which saves the grid sync that would
// broadcast the keep/drop decision.  ~5 grid syncs per column instead of ~10
// launches and a host round trip per column.
#ifndef HELM_ORTH_TILE
#define HELM_ORTH_TILE 1024
#endif
static constexpr int kOrthTile = HELM_ORTH_TILE;
static constexpr int kOrthThreads = 256;
static constexpr int kIntraNV = 2 * 8 + 1;     // intra-block partial values per block (t <= 8)
static constexpr long kIntraMaxBlk = 1024;     // blocks the intra-block partial region covers

struct OrthArgs {
  long n;
  cplx* V;          // n x (m + t), ld n; the new slots start at column m
  int m, t;
  cplx* W;          // n x t (A Z_k on entry, orthogonalised on exit)
  cplx* part;       // nblk x S partial sums, S = (m + 1) * t
  cplx* out;        // [C1 m*t][C2 m*t][gram t*t][cv 2*t*t][nn t]  (host copy, one D2H)
  long rows;        // rows per block
  long long* prof;  // optional phase clock stamps of block 0 (diagnostics, orth_prof knob)
  cplx* ipart;      // [2][nblk][kIntraNV] intra-block partials, alternating per pass
};

// One pass over this block's rows.  Optional update W[:, wc0+i] -= sum_j Vb[:, j] Cs[j*tc+i]
// (i < tc); then optional projections outsm[j*tc+i] = sum conj(Vb[:, j]) W[:, wc0+i] (j < mcols)
// and squared norms outsm[mcols*tc + q] = ||W[:, nc0+q]||^2 (q < nn).
template <int TM>
__device__ void orth_pass(const OrthArgs& a, cplx* Wt, const cplx* Cs, cplx* outsm, const cplx* Vb, int mcols,
                          int wc0, int tc, bool upd, bool dots, int nc0, int nn, long r0, long r1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nout = (dots ? mcols * tc : 0) + nn;
  for (int e = threadIdx.x; e < nout; e += blockDim.x) outsm[e] = cmk(0, 0);
  __syncthreads();
  for (long t0 = r0; t0 < r1; t0 += kOrthTile) {
    const int rows = (int)min((long)kOrthTile, r1 - t0);
    for (int rr = threadIdx.x; rr < rows; rr += blockDim.x) {
      const long r = t0 + rr;
      cplx w[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i)
        if (i < tc) w[i] = a.W[(long)(wc0 + i) * a.n + r];
      if (upd) {
        cplx acc[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) acc[i] = cmk(0, 0);
        int j = 0;
        for (; j + 8 <= mcols; j += 8) {   // eight independent loads in flight per thread
          cplx v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcg(Vb + (long)(j + u) * a.n + r);
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < TM; ++i)
              if (i < tc) cfma(acc[i], v[u], Cs[(j + u) * tc + i]);
        }
        for (; j < mcols; ++j) {
          const cplx v = __ldcg(Vb + (long)j * a.n + r);
#pragma unroll
          for (int i = 0; i < TM; ++i)
            if (i < tc) cfma(acc[i], v, Cs[j * tc + i]);
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
          if (i < tc) {
            w[i] = csub(w[i], acc[i]);
            a.W[(long)(wc0 + i) * a.n + r] = w[i];
          }
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
        if (i < tc) Wt[i * kOrthTile + rr] = w[i];
    }
    __syncthreads();
    const int jn = (dots ? mcols : 0) + nn;
    // two projection columns per warp at a time (16 loads in flight per lane)
    if (dots && tc == a.t) {
      const int jd = mcols & ~1;
      for (int j = 2 * warp; j < jd; j += 2 * nw) {
        cplx acc0[TM], acc1[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) { acc0[i] = cmk(0, 0); acc1[i] = cmk(0, 0); }
        const cplx* v0 = Vb + (long)j * a.n + t0;
        const cplx* v1 = v0 + a.n;
        int rr = lane;
        for (; rr + 224 < rows; rr += 256) {
          cplx x0[8], x1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) { x0[u] = __ldcg(v0 + rr + 32 * u); x1[u] = __ldcg(v1 + rr + 32 * u); }
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < TM; ++i)
              if (i < tc) {
                const cplx wv = Wt[i * kOrthTile + rr + 32 * u];
                cfmaconj(acc0[i], x0[u], wv);
                cfmaconj(acc1[i], x1[u], wv);
              }
        }
        for (; rr < rows; rr += 32) {
          const cplx y0 = __ldcg(v0 + rr), y1 = __ldcg(v1 + rr);
#pragma unroll
          for (int i = 0; i < TM; ++i)
            if (i < tc) {
              const cplx wv = Wt[i * kOrthTile + rr];
              cfmaconj(acc0[i], y0, wv);
              cfmaconj(acc1[i], y1, wv);
            }
        }
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          if (i >= tc) break;
          for (int off = 16; off > 0; off >>= 1) {
            acc0[i].x += __shfl_xor_sync(0xffffffffu, acc0[i].x, off);
            acc0[i].y += __shfl_xor_sync(0xffffffffu, acc0[i].y, off);
            acc1[i].x += __shfl_xor_sync(0xffffffffu, acc1[i].x, off);
            acc1[i].y += __shfl_xor_sync(0xffffffffu, acc1[i].y, off);
          }
        }
        if (lane == 0) {
#pragma unroll
          for (int i = 0; i < TM; ++i)
            if (i < tc) {
              outsm[j * tc + i] = cadd(outsm[j * tc + i], acc0[i]);
              outsm[(j + 1) * tc + i] = cadd(outsm[(j + 1) * tc + i], acc1[i]);
            }
        }
      }
    }
    const int jstart = (dots && tc == a.t) ? (mcols & ~1) : 0;
    for (int j = jstart + warp; j < jn; j += nw) {
      const bool isdot = dots && j < mcols;
      cplx acc[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) acc[i] = cmk(0, 0);
      if (isdot) {
        const cplx* v = Vb + (long)j * a.n + t0;
        int rr = lane;
        for (; rr + 224 < rows; rr += 256) {   // eight independent loads in flight per lane
          cplx vv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) vv[u] = __ldcg(v + rr + 32 * u);
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < TM; ++i)
              if (i < tc) cfmaconj(acc[i], vv[u], Wt[i * kOrthTile + rr + 32 * u]);
        }
        for (; rr < rows; rr += 32) {
          const cplx vv = __ldcg(v + rr);
#pragma unroll
          for (int i = 0; i < TM; ++i)
            if (i < tc) cfmaconj(acc[i], vv, Wt[i * kOrthTile + rr]);
        }
      } else {
        const int c = nc0 + (j - (dots ? mcols : 0)) - wc0;
        for (int rr = lane; rr < rows; rr += 32) {
          const cplx ww = Wt[c * kOrthTile + rr];
          cfmaconj(acc[0], ww, ww);
        }
      }
      const int na = isdot ? tc : 1;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        if (i >= na) break;
        for (int off = 16; off > 0; off >>= 1) {
          acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, off);
          acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, off);
        }
      }
      if (lane == 0) {
        if (isdot) {
#pragma unroll
          for (int i = 0; i < TM; ++i)
            if (i < tc) outsm[j * tc + i] = cadd(outsm[j * tc + i], acc[i]);
        }
        else
          outsm[(dots ? mcols * tc : 0) + (j - (dots ? mcols : 0))] =
              cadd(outsm[(dots ? mcols * tc : 0) + (j - (dots ? mcols : 0))], acc[0]);
      }
    }
    __syncthreads();
  }
  const int S = (a.m + 1) * a.t;
  for (int e = threadIdx.x; e < nout; e += blockDim.x) a.part[(long)blockIdx.x * S + e] = outsm[e];
}

// dst[e] = sum_b part[b][off + e] for e < count, fixed order over b (grid-strided)
// sum over the blocks' partials, one warp per element: lanes take blocks b = lane,
// lane + 32, ... in order, then a fixed butterfly -- a fixed order, so the result
// is bitwise reproducible (a serial sum over ~300 blocks per thread was ~40k cycles)
__device__ __forceinline__ cplx warp_sum_partials(const OrthArgs& a, long idx) {
  const int S = (a.m + 1) * a.t;
  const int lane = threadIdx.x & 31;
  cplx acc = cmk(0, 0);
  for (int b = lane; b < (int)gridDim.x; b += 32) acc = cadd(acc, __ldcg(a.part + (long)b * S + idx));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  return acc;
}

// dst[e] = sum_b part[b][off + e] for e < count (warp per element, grid-strided)
__device__ __forceinline__ void orth_reduce(const OrthArgs& a, int off, int count, cplx* dst) {
  const long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwt = ((long)gridDim.x * blockDim.x) >> 5;
  for (long e = gw; e < count; e += nwt) {
    const cplx v = warp_sum_partials(a, off + e);
    if ((threadIdx.x & 31) == 0) dst[e] = v;
  }
}

// every block: the same fixed-order sum of one norm partial (no broadcast sync needed)
__device__ __forceinline__ double orth_norm2(const OrthArgs& a, int off) {
  __shared__ double s;
  if (threadIdx.x < 32) {
    const cplx v = warp_sum_partials(a, off);
    if (threadIdx.x == 0) s = v.x;
  }
  __syncthreads();
  const double v = s;
  __syncthreads();
  return v;
}

// One pass of the intra-block CGS2 over this block's rows (thread per row; a
// block only ever touches its own rows, so no grid sync is needed between a
// store and a later read of the same rows).  Column i of W:
//   vprev >= 0: first store Vn[:, vprev] = W[:, vprev] * sc_prev
//   upd:  w_i -= sum_{j<i} Vn_j c[j]
//   dself: projections Vn_j^H w_i (j < i)                       -> outputs [0, i)
//   nrm:  ||w_i||^2                                             -> output  o_n
//   nxt:  Vn_j^H w_{i+1} (j < i) and w_i^H w_{i+1}              -> outputs o_x .. o_x + i
// Per-block partial sums in a fixed order go to a.part[blockIdx.x * S + e].
template <int TM>
__device__ void intra_pass(const OrthArgs& a, int i, const cplx* c, int vprev, double sc_prev, bool upd, bool dself,
                           bool nrm, bool nxt, long r0, long r1, cplx* red, int par) {
  constexpr int NV = 2 * TM + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  cplx* Vn = a.V + (long)a.m * a.n;
  const int o_n = dself ? i : 0, o_x = o_n + (nrm ? 1 : 0);
  const int nv = o_x + (nxt ? i + 1 : 0);
  cplx accd[TM], accx[TM + 1];
  double accn = 0.0;
#pragma unroll
  for (int e = 0; e < TM; ++e) accd[e] = cmk(0, 0);
#pragma unroll
  for (int e = 0; e <= TM; ++e) accx[e] = cmk(0, 0);
  // four rows per thread and iteration: all loads of the four rows are issued
  // before their arithmetic (the stores to W / Vn would otherwise serialise them)
  constexpr int RU = TM <= 2 ? 4 : (TM <= 4 ? 2 : 1);
  for (long rb = r0 + threadIdx.x; rb < r1; rb += (long)RU * blockDim.x) {
    cplx vj[RU][TM], w[RU], wn[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const long r = rb + (long)u * blockDim.x;
      const bool in = r < r1;
#pragma unroll
      for (int j = 0; j < TM; ++j)
        if (j < i) vj[u][j] = in ? __ldcg((j == vprev ? a.W : Vn) + (long)j * a.n + r) : cmk(0, 0);
      w[u] = in ? __ldcg(a.W + (long)i * a.n + r) : cmk(0, 0);
      wn[u] = (nxt && in) ? __ldcg(a.W + (long)(i + 1) * a.n + r) : cmk(0, 0);
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const long r = rb + (long)u * blockDim.x;
      const bool in = r < r1;
      if (vprev >= 0) {
#pragma unroll
        for (int j = 0; j < TM; ++j)
          if (j == vprev) {
            vj[u][j] = cscale(vj[u][j], sc_prev);
            if (in) Vn[(long)vprev * a.n + r] = vj[u][j];
          }
      }
      if (upd) {
#pragma unroll
        for (int j = 0; j < TM; ++j)
          if (j < i) w[u] = csub(w[u], cmul(vj[u][j], c[j]));
        if (in) a.W[(long)i * a.n + r] = w[u];
      }
      if (dself) {
#pragma unroll
        for (int j = 0; j < TM; ++j)
          if (j < i) cfmaconj(accd[j], vj[u][j], w[u]);
      }
      if (nrm) accn += w[u].x * w[u].x + w[u].y * w[u].y;
      if (nxt) {
#pragma unroll
        for (int j = 0; j < TM; ++j)
          if (j < i) cfmaconj(accx[j], vj[u][j], wn[u]);
#pragma unroll
        for (int j = 0; j < TM; ++j)
          if (j == i) cfmaconj(accx[j], w[u], wn[u]);
      }
    }
  }
  // block reduction in a fixed order: butterflies, then warps in order
  auto wred = [&](cplx v, int e) {
    for (int off = 16; off > 0; off >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
    }
    if (lane == 0) red[warp * NV + e] = v;
  };
  if (dself) {
#pragma unroll
    for (int j = 0; j < TM; ++j)
      if (j < i) wred(accd[j], j);
  }
  if (nrm) wred(cmk(accn, 0.0), o_n);
  if (nxt) {
#pragma unroll
    for (int j = 0; j <= TM; ++j)
      if (j <= i) wred(accx[j], o_x + j);
  }
  __syncthreads();
  // alternate partial regions per pass: a fast block's next pass must not
  // overwrite partials a slower block is still summing
  cplx* dst = a.ipart + ((long)par * gridDim.x + blockIdx.x) * kIntraNV;
  for (int e = threadIdx.x; e < nv; e += blockDim.x) {
    cplx v = red[e];
    for (int q = 1; q < nw; ++q) v = cadd(v, red[q * NV + e]);
    dst[e] = v;
  }
  __syncthreads();
}

// after a grid sync: every block sums the first nv partials in the same fixed
// order (warp per value) into dst (shared memory); no broadcast sync is needed
__device__ __forceinline__ void intra_reduce(const OrthArgs& a, int nv, cplx* dst, int par) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const cplx* src = a.ipart + (long)par * gridDim.x * kIntraNV;
  for (int e = warp; e < nv; e += nw) {
    cplx acc = cmk(0, 0);
    for (int b = lane; b < (int)gridDim.x; b += 32) acc = cadd(acc, __ldcg(src + (long)b * kIntraNV + e));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) dst[e] = acc;
  }
  __syncthreads();
}

template <int TM>
__global__ void __launch_bounds__(kOrthThreads, 2) k_orth(OrthArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ cplx osm[];
  const int m = a.m, t = a.t;
  cplx* Wt = osm;                                  // kOrthTile * t
  cplx* Cs = Wt + (long)kOrthTile * t;             // m * t
  cplx* outsm = Cs + (long)m * t;                  // (m + 1) * t
  const long r0 = min(a.n, (long)blockIdx.x * a.rows), r1 = min(a.n, r0 + a.rows);
  cplx* C1 = a.out;
  cplx* C2 = C1 + (long)m * t;
  cplx* gram = C2 + (long)m * t;
  cplx* cv = gram + t * t;
  cplx* nn = cv + 2 * t * t;
  cplx* Vn = a.V + (long)m * a.n;
  auto load_C = [&](const cplx* C, int cnt) {
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) Cs[e] = __ldcg(C + e);
    __syncthreads();
  };
  const bool pr = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
  if (pr) a.prof[0] = clock64();
  // C1 = V^H W and ||w_i||^2 (the Gram diagonal)
  orth_pass<TM>(a, Wt, Cs, outsm, a.V, m, 0, t, false, true, 0, t, r0, r1);
  if (pr) a.prof[1] = clock64();
  grid.sync();
  orth_reduce(a, 0, m * t, C1);
  {
    // Gram diagonal: the t norm partials follow the m*t projections; the last t warps
    const long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long nwt = ((long)gridDim.x * blockDim.x) >> 5;
    const long e = gw - (nwt - t);
    if (e >= 0 && e < t) {
      const cplx v = warp_sum_partials(a, (long)m * t + e);
      if ((threadIdx.x & 31) == 0) gram[e * t + e] = v;
    }
  }
  grid.sync();
  if (pr) a.prof[2] = clock64();
  // W -= V C1; C2 = V^H W
  load_C(C1, m * t);
  orth_pass<TM>(a, Wt, Cs, outsm, a.V, m, 0, t, true, true, 0, 0, r0, r1);
  if (pr) a.prof[3] = clock64();
  grid.sync();
  orth_reduce(a, 0, m * t, C2);
  grid.sync();
  // W -= V C2
  if (pr) a.prof[4] = clock64();
  load_C(C2, m * t);
  orth_pass<TM>(a, Wt, Cs, outsm, a.V, m, 0, t, true, false, 0, 0, r0, r1);
  if (pr) a.prof[5] = clock64();
  // intra-block CGS2 (D10 step 5), two passes and two grid syncs per column:
  //   round 1 of column i comes with the norm pass of column i-1:
  //     c_j = Vn_j^H w_i (j < i-1),  c_{i-1} = sc_{i-1} w_{i-1}^H w_i  (Vn_{i-1} = sc_{i-1} w_{i-1})
  //   pass B: w_i -= Vn c;  c' = Vn^H w_i
  //   pass C: w_i -= Vn c'; ||w_i||^2 (and round 1 of column i+1)
  //   keep iff ||w_i|| > 1e-10 ||A z_i||; Vn_i = w_i / ||w_i|| (else 0), stored by the next pass
  cplx* red = outsm + (long)(m + 1) * t;   // [nw][2 TM + 1] block partials (beyond the BCGS2 outputs)
  cplx* vals = red + 8 * (2 * TM + 1);      // reduced values
  cplx* cc = Cs;                           // current projection coefficients
  double sc = 0.0;
  int par = 0;
  for (int i = 0; i < t; ++i) {
    if (i > 0) {
      // pass B (stores Vn_{i-1} first)
      intra_pass<TM>(a, i, cc, i - 1, sc, true, true, false, false, r0, r1, red, par);
      grid.sync();
      intra_reduce(a, i, vals, par);
      par ^= 1;
      for (int j = threadIdx.x; j < i; j += blockDim.x) {
        cc[j] = vals[j];
        if (blockIdx.x == 0) cv[(long)t * t + (long)i * t + j] = vals[j];
      }
      __syncthreads();
    }
    // pass C: w_i -= Vn c' (i > 0); ||w_i||^2; round 1 of column i+1
    const bool nx = i + 1 < t;
    intra_pass<TM>(a, i, cc, -1, 0.0, i > 0, false, true, nx, r0, r1, red, par);
    grid.sync();
    intra_reduce(a, 1 + (nx ? i + 1 : 0), vals, par);
    par ^= 1;
    // keep iff ||w_i|| > 1e-10 ||A z_i||; gram[i] is visible after the syncs above
    const double nrm = sqrt(fmax(vals[0].x, 0.0));
    const double naz = sqrt(fmax(__ldcg(gram + i * t + i).x, 0.0));
    sc = nrm > 1e-10 * naz ? 1.0 / nrm : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) nn[i] = cmk(nrm, 0.0);
    if (nx) {
      for (int j = threadIdx.x; j <= i; j += blockDim.x) {
        const cplx v = j < i ? vals[1 + j] : cscale(vals[1 + i], sc);
        cc[j] = v;
        if (blockIdx.x == 0) cv[(long)(i + 1) * t + j] = v;
      }
    }
    __syncthreads();
  }
  // the last new basis vector (own rows; the kernel's end orders it for the host)
  for (long r = r0 + threadIdx.x; r < r1; r += blockDim.x) Vn[(long)(t - 1) * a.n + r] = cscale(a.W[(long)(t - 1) * a.n + r], sc);
  if (pr) a.prof[6] = clock64();
}

namespace {

struct Work {
  long n;
  cudaStream_t st;
  cplx* partial = nullptr;
  int nblk = 0;
  cplx* dsmall = nullptr;  // device small results
  cplx* hsmall = nullptr;  // pinned host mirror
  size_t small_cap = 0;
};

long grid_for(long n) {
  long b = (n + 255) / 256;
  return b > 148L * 8 ? 148L * 8 : b;
}

// C[j*t+i] = V^H W  over all rows (device result in `out`)
int dots(Work& wk, const cplx* V, long ldv, int m, const cplx* W, long ldw, int t, cplx* out, bool accumulate) {
  const int rows_blk = kDotChunk / t;
  const int nblk = (int)((wk.n + rows_blk - 1) / rows_blk);
  const size_t sm = sizeof(cplx) * kDotChunk;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dots, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k_dots<<<nblk, kDotThreads, sm, wk.st>>>(wk.n, rows_blk, V, ldv, m, W, ldw, t, wk.partial);
  HELM_LAUNCH_CHECK();
  int mt = m * t;
  k_reduce_partials<<<(mt + 127) / 128, 128, 0, wk.st>>>(wk.partial, nblk, mt, out, accumulate ? 1 : 0);
  HELM_LAUNCH_CHECK();
  return HELM_OK;
}

int update(Work& wk, const cplx* V, long ldv, int m, const cplx* C, cplx* W, long ldw, int t) {
  size_t sm = sizeof(cplx) * (size_t)m * t;
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_update<<<grid_for(wk.n), 256, sm, wk.st>>>(wk.n, V, ldv, m, C, W, ldw, t);
  HELM_LAUNCH_CHECK();
  return HELM_OK;
}

int to_host(Work& wk, const cplx* dsrc, size_t count, std::vector<std::complex<double>>& out) {
  out.resize(count);
  if (count == 0) return HELM_OK;
  HELM_CUDA_TRY(cudaMemcpyAsync(wk.hsmall, dsrc, sizeof(cplx) * count, cudaMemcpyDeviceToHost, wk.st));
  HELM_CUDA_TRY(cudaStreamSynchronize(wk.st));
  for (size_t i = 0; i < count; ++i) out[i] = {wk.hsmall[i].x, wk.hsmall[i].y};
  return HELM_OK;
}

// Incremental Householder QR of the block Hessenberg matrix H~ (host)
// "minimises the Euclidean norm of the residual": min_y || beta e1 - H~ y ||.
// H~ can be rank deficient: a deflated column (D10 step 6) keeps its H~ column
// but gets no new row, and duplicate preconditioners give (numerically) equal
// columns.  A column whose part below the current rank vanishes after the
// previous reflectors (|tail| <= 1e-12 |column|) lies in the span of the
// earlier independent columns: it gets no reflector and y = 0 there, which
// leaves the minimal residual unchanged (the oracle's lstsq reaches the same
// residual and, for equal columns, the same x = Z y).
struct HouseholderLSQ {
  typedef std::complex<double> C;
  std::vector<std::vector<C>> R;   // columns of the triangularised H~ (entries 0..rank at append time)
  std::vector<int> piv;            // row of each column's pivot, -1 for a dependent column
  std::vector<std::vector<C>> v;   // reflector vectors (reflector q acts on rows q..)
  std::vector<C> tau;
  std::vector<C> g;                // transformed rhs
  int nrows = 0;

  void init(double beta) {
    g.assign(1, C(beta, 0.0));
    nrows = 1;
  }
  // apply reflector q (rows q..) to vector x
  void apply(int q, std::vector<C>& x) const {
    const std::vector<C>& vq = v[q];
    C s = 0;
    for (size_t k = 0; k < vq.size(); ++k) s += std::conj(vq[k]) * x[q + k];
    s *= tau[q];
    for (size_t k = 0; k < vq.size(); ++k) x[q + k] -= vq[k] * s;
  }
  // append a column (length new_nrows >= nrows); rows grow to new_nrows
  void append(std::vector<C> col, int new_nrows) {
    if (new_nrows > nrows) {
      g.resize(new_nrows, C(0));
      nrows = new_nrows;
    }
    col.resize(nrows, C(0));
    double cn = 0;
    for (auto& e : col) cn += std::norm(e);
    cn = std::sqrt(cn);
    const int rank = (int)v.size();
    for (int q = 0; q < rank; ++q) apply(q, col);
    // the part below the rank: a reflector rows rank.. (complex Householder)
    double xn = 0;
    for (int i = rank; i < nrows; ++i) xn += std::norm(col[i]);
    xn = std::sqrt(xn);
    if (rank >= nrows || !(xn > 1e-12 * cn)) {
      piv.push_back(-1);            // dependent: in the span of the earlier columns
      col.resize(rank);
      R.push_back(col);
      return;
    }
    std::vector<C> x(col.begin() + rank, col.end());
    // x -> beta e1 with beta = -e^{i arg x0} ||x||, v = x - beta e1, tau = 2/||v||^2
    C alpha = x[0];
    double aa = std::abs(alpha);
    C phase = aa > 0 ? alpha / aa : C(1.0, 0.0);
    C beta = -phase * xn;
    std::vector<C> vq = x;
    vq[0] = alpha - beta;
    double vn = 0;
    for (auto& e : vq) vn += std::norm(e);
    v.push_back(vq);
    tau.push_back(vn > 0 ? C(2.0 / vn) : C(0));
    apply(rank, col);
    apply(rank, g);
    col.resize(rank + 1);
    piv.push_back(rank);
    R.push_back(col);
  }
  // y = argmin: back substitution over the independent columns (y = 0 on the
  // dependent ones); res = || g[rank..] ||
  void solve(std::vector<C>& y, double& res) const {
    const int nc = (int)R.size();
    const int rank = (int)v.size();
    y.assign(nc, C(0));
    std::vector<int> colof(rank, -1);   // independent column of each pivot row
    for (int j = 0; j < nc; ++j)
      if (piv[j] >= 0) colof[piv[j]] = j;
    for (int q = rank - 1; q >= 0; --q) {
      const int j = colof[q];
      C s = g[q];
      for (int q2 = q + 1; q2 < rank; ++q2) s -= R[colof[q2]][q] * y[colof[q2]];
      y[j] = s / R[j][q];
    }
    double r2 = 0;
    for (int i = rank; i < nrows; ++i) r2 += std::norm(g[i]);
    res = std::sqrt(r2);
  }
};

}  // namespace

// ------------------------------------------------------------------ device-side block QR helpers
// scale[i] = keep ? 1/||w_i|| : 0 with the deflation rule of D10 step 5
// (drop if ||w_i|| <= 1e-10 ||A z_i||, ||A z_i|| from the Gram diagonal).
__global__ void k_decide(const cplx* nn, const cplx* gram, int t, int i, double* scale, double* nrm_out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double nrm = sqrt(fmax(nn[0].x, 0.0));
    double naz = sqrt(fmax(gram[i * t + i].x, 0.0));
    bool keep = nrm > 1e-10 * naz;
    scale[i] = keep ? 1.0 / nrm : 0.0;
    nrm_out[i] = nrm;
  }
}

__global__ void k_scale_dev(long n, const cplx* __restrict__ x, const double* __restrict__ s, int i,
                            cplx* __restrict__ y) {
  const double a = s[i];
  for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < n; r += (long)gridDim.x * blockDim.x)
    y[r] = cscale(x[r], a);
}

// ------------------------------------------------------------------ workspace
// The solve workspace lives with the problem handle and is reused across
// solves (grown on demand): V (n x (1 + icap t)), Z (n x icap t), W, sources,
// dot partials and pinned host mirrors.  No per-solve allocation.
struct KrylovWS {
  long n = 0;
  int tcap = 0;              // largest t the t-sized buffers (W, Rsrc) hold
  long vcap = 0, zcap = 0;   // V / Z capacities in columns
  int small_t = 0;           // t the small per-iteration buffers (dC1, dC2, dsm, partial) are sized for
  cplx *V = nullptr, *Z = nullptr, *W = nullptr, *Rsrc = nullptr, *tmp = nullptr, *partial = nullptr;
  cplx *dC1 = nullptr, *dC2 = nullptr, *dsm = nullptr, *dy = nullptr;
  double* dscal = nullptr;
  cplx* hsmall = nullptr;
  size_t small_cap = 0;
  long partial_cap = 0;
};

// Pinned host staging for the per-iteration small D2H copy.  One buffer per
// host thread, grown on demand and never returned: cudaFreeHost synchronises
// the device and can take hundreds of ms, so it must not run per problem.
static cplx* pinned_small(size_t count) {
  static thread_local cplx* buf = nullptr;
  static thread_local size_t cap = 0;
  if (count > cap) {
    cplx* nb = nullptr;
    if (cudaMallocHost((void**)&nb, sizeof(cplx) * count) != cudaSuccess) return nullptr;
    if (buf) cudaFreeHost(buf);
    buf = nb;
    cap = count;
  }
  return buf;
}

static void ws_free(KrylovWS* w) {
  if (!w) return;
  helm_dev_free(w->V); helm_dev_free(w->Z); helm_dev_free(w->W); helm_dev_free(w->Rsrc); helm_dev_free(w->tmp);
  helm_dev_free(w->partial); helm_dev_free(w->dC1); helm_dev_free(w->dC2); helm_dev_free(w->dsm); helm_dev_free(w->dy);
  helm_dev_free(w->dscal);
  delete w;
}

void helm_problem_free_ws(helm_problem_s* p) {
  ws_free(reinterpret_cast<KrylovWS*>(p->ws));
  p->ws = nullptr;
}

// ensure capacity for `iters` iterations of t columns; preserves the first
// `keepV` V columns and `keepZ` Z columns.  Capacities are tracked in columns
// (vcap, zcap) and the small per-iteration buffers are sized for the largest t
// seen (tcap), so one problem handle can be reused with any t in [1, 8].
static int ws_reserve(helm_problem_s* p, int t, int iters, long keepV, long keepZ, cudaStream_t st) {
  KrylovWS* w = reinterpret_cast<KrylovWS*>(p->ws);
  if (!w) { w = new KrylovWS(); p->ws = w; w->n = p->n; }
  const long n = p->n;
  cudaError_t e = cudaSuccess;
  if (t > w->tcap) {
    helm_dev_free(w->W); helm_dev_free(w->Rsrc); helm_dev_free(w->tmp); helm_dev_free(w->dscal);
    w->W = w->Rsrc = w->tmp = nullptr; w->dscal = nullptr;
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->W, sizeof(cplx) * n * t);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->Rsrc, sizeof(cplx) * n * t);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->tmp, sizeof(cplx) * n);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->dscal, sizeof(double) * 16);
    if (e == cudaSuccess) w->tcap = t;
  }
  const long need_v = 1 + (long)iters * t, need_z = (long)iters * t;
  if (e == cudaSuccess && (need_v > w->vcap || need_z > w->zcap)) {
    const long vc = std::max(need_v, w->vcap), zc = std::max(need_z, w->zcap);
    cplx *V2 = nullptr, *Z2 = nullptr;
    e = helm_dev_alloc((void**)&V2, sizeof(cplx) * n * vc);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&Z2, sizeof(cplx) * n * zc);
    if (e == cudaSuccess && keepV > 0) e = cudaMemcpyAsync(V2, w->V, sizeof(cplx) * n * keepV, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && keepZ > 0) e = cudaMemcpyAsync(Z2, w->Z, sizeof(cplx) * n * keepZ, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      helm_dev_free(V2); helm_dev_free(Z2);
      helm_set_error("mpgmres_solve: basis of %ld columns: %s", vc, cudaGetErrorString(e));
      return HELM_ENOMEM;
    }
    helm_dev_free(w->V); helm_dev_free(w->Z);
    w->V = V2; w->Z = Z2;
    w->vcap = vc; w->zcap = zc;
    w->small_t = 0;   // the small buffers depend on vcap / zcap: resize below
  }
  if (e == cudaSuccess && w->small_t < w->tcap) {
    // sized for vcap V columns and tcap new columns (the largest t any solve of this handle uses)
    const long vc = w->vcap, zc = w->zcap, tc = w->tcap;
    helm_dev_free(w->dC1); helm_dev_free(w->dC2); helm_dev_free(w->dsm); helm_dev_free(w->dy); helm_dev_free(w->partial);
    w->dC1 = w->dC2 = w->dsm = w->dy = w->partial = nullptr;
    w->hsmall = nullptr;
    w->partial_cap = std::max(((n + kDotChunk - 1) / kDotChunk) * kMaxT * vc * tc, 148L * 4 * (vc + 1) * tc);
    w->small_cap = 4 * vc * tc + 64;
    e = helm_dev_alloc((void**)&w->dC1, sizeof(cplx) * vc * tc);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->dC2, sizeof(cplx) * vc * tc);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->dsm, sizeof(cplx) * w->small_cap);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->dy, sizeof(cplx) * zc);
    if (e == cudaSuccess) e = helm_dev_alloc((void**)&w->partial, sizeof(cplx) * (w->partial_cap + 2 * kIntraMaxBlk * kIntraNV));
    if (e == cudaSuccess) {
      w->hsmall = pinned_small(w->small_cap);
      if (!w->hsmall) e = cudaErrorMemoryAllocation;
    }
    if (e == cudaSuccess) w->small_t = w->tcap;
  }
  if (e != cudaSuccess) {
    helm_set_error("mpgmres_solve: workspace: %s", cudaGetErrorString(e));
    return HELM_ENOMEM;
  }
  return HELM_OK;
}

// Launch k_orth cooperatively (one launch per iteration).  Returns 1 when it
// ran, 0 when the shapes exceed its shared-memory plan (the caller then uses
// the multi-launch sequence), -1 on a CUDA error (message set).
static int orth_fused(KrylovWS* ws, long n, cplx* V, int m, int t, cplx* W, cudaStream_t st) {
  if (helm_knob(KNOB_ORTH_UNFUSED)) return 0;
  const size_t smem = sizeof(cplx) * ((size_t)kOrthTile * t + (size_t)m * t + (size_t)(m + 1) * t + 9 * kIntraNV);
  if (smem > 200 * 1024) return 0;
  static int nsm = 0;
  int dev = 0;
  if (!nsm) {
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_orth<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_orth<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_orth<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_orth<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  const void* kfun = t <= 1 ? (const void*)k_orth<1> : t <= 2 ? (const void*)k_orth<2>
                   : t <= 4 ? (const void*)k_orth<4> : (const void*)k_orth<8>;
  // occupancy per (kernel, shared memory), cached: the query sits on the host-synchronous
  // iteration's critical path
  int occ = 0;
  cudaError_t e = cudaSuccess;
  {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, size_t>, int>> cache;
    bool hit = false;
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto& c : cache)
        if (c.first.first == kfun && c.first.second == smem) { occ = c.second; hit = true; }
    }
    if (!hit) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfun, kOrthThreads, smem);
      if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        cache.push_back({{kfun, smem}, occ});
      }
    }
  }
  if (e != cudaSuccess || occ < 1) return 0;
  long nblk = std::min<long>((long)nsm * std::min(occ, 4), (n + kOrthThreads - 1) / kOrthThreads);
  if ((long)nblk * (m + 1) * t > ws->partial_cap) nblk = ws->partial_cap / ((long)(m + 1) * t);
  if (nblk < 1) return 0;
  OrthArgs a;
  a.n = n; a.V = V; a.m = m; a.t = t; a.W = W; a.part = ws->partial; a.out = ws->dsm;
  a.ipart = ws->partial + ws->partial_cap;   // the tail region of the partial buffer
  if (nblk > kIntraMaxBlk) return 0;
  static long long* prof = nullptr;
  if (helm_knob(KNOB_ORTH_PROF) && !prof) cudaMallocManaged((void**)&prof, 16 * sizeof(long long));
  a.prof = prof;
  if (prof) {
    static int calls = 0;
    if (calls++ > 0) {
      cudaDeviceSynchronize();
      fprintf(stderr, "[k_orth m=%d] C1 pass %lld, reduce %lld, update+C2 %lld, reduce %lld, update+norm %lld, intra %lld cycles\n", m,
              prof[1] - prof[0], prof[2] - prof[1], prof[3] - prof[2], prof[4] - prof[3], prof[5] - prof[4],
              prof[6] - prof[5]);
    }
  }
  a.rows = (n + nblk - 1) / nblk;
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel(kfun, dim3((unsigned)nblk), dim3(kOrthThreads), args, smem, st);
  if (e != cudaSuccess) {
    helm_set_error("mpgmres_solve: k_orth: %s", cudaGetErrorString(e));
    return -1;
  }
  g_helm_launches++;
  return 1;
}

// One MPGMRES solve.  Direction-parallel mode: this
// rank applies only its t_local directions dirs[0..t_local) -- global directions
// rank*t_local .. -- and the new Z and W = A Z columns of all ranks are
// all-gathered through `gather` after the SpMM; everything else (source
// selection, BCGS2 + block QR, the host least squares) runs replicated on every
// rank from identical data, so every rank takes the same decisions.  gather ==
// nullptr: single process (t_local == t).
static int mpgmres_core(helm_problem_t prob, const helm_sweep_t* dirs, int t_local, int t, int rank,
                        helm_allgather_fn gather, void* gctx, const double* b_in, double* x_out, double tol,
                        int maxit, mpgmres_stats* stats, void* stream) {
  typedef std::complex<double> C;
  auto t0 = std::chrono::steady_clock::now();
  if (!prob || !dirs || !b_in || !x_out) { helm_set_error("mpgmres_solve: null argument"); return HELM_EINVAL; }
  if (t < 1 || t > kMaxT || !(tol > 0.0 && tol < 1.0) || maxit < 1) {
    helm_set_error("mpgmres_solve: need 1 <= t <= 8, 0 < tol < 1, maxit >= 1");
    return HELM_EINVAL;
  }
  for (int d = 0; d < t_local; ++d)
    if (!dirs[d] || dirs[d]->prob->n != prob->n) { helm_set_error("mpgmres_solve: direction %d size mismatch", d); return HELM_EDIM; }
  cudaStream_t st = (cudaStream_t)stream;
  const long n = prob->n;
  Staged sb, sx;
  HELM_TRY(helm_stage_in(b_in, sizeof(cplx) * n, true, st, sb));
  {
    const int rs = helm_stage_in(x_out, sizeof(cplx) * n, false, st, sx);
    if (rs != HELM_OK) { helm_stage_free(sb, st); return rs; }
  }
  const cplx* b = (const cplx*)sb.dev;
  cplx* x = (cplx*)sx.dev;

  int rc = ws_reserve(prob, t, std::min(maxit, 24), 0, 0, st);
  if (rc != HELM_OK) { helm_stage_free(sb, st); helm_stage_free(sx, st); return rc; }
  KrylovWS* ws = reinterpret_cast<KrylovWS*>(prob->ws);
  Work wk;
  wk.n = n;
  wk.st = st;
  wk.partial = ws->partial;
  wk.hsmall = pinned_small(ws->small_cap);   // re-fetched: the buffer is shared per thread
  wk.small_cap = ws->small_cap;
  cudaEvent_t ev[4];
  for (auto& e : ev) cudaEventCreate(&e);
  double sweep_ms = 0, spmv_ms = 0, orth_ms = 0;
  long inner = 0;
  int deflations = 0;
  std::vector<double> hist;
  int k_done = 0;
  bool converged = false, exhausted = false;
  double rho = 1.0, true_res = NAN;
  cudaError_t e = cudaSuccess;

  std::vector<C> hv;
  HouseholderLSQ lsq;
  std::vector<int> tags;        // origin tag of each V column (-1 for v1)
  long blk_start = 0, mV = 0;   // first column of the newest block, #V columns
  long nz = 0;                  // #Z columns
  double beta = 0;
  std::vector<C> y;
  // small device results, packed in ws->dsm: [gram t*t][cv 2*t*t][nn t]
  cplx* d_gram = ws->dsm;
  cplx* d_cv = d_gram + t * t;
  cplx* d_nn = d_cv + 2 * t * t;
  double* d_nrm = ws->dscal + 8;
  // beta = ||b||, V1 = b / beta
  rc = dots(wk, b, n, 1, b, n, 1, d_nn, false);
  if (rc == HELM_OK) rc = to_host(wk, d_nn, 1, hv);
  if (rc == HELM_OK) {
    beta = std::sqrt(hv[0].real());
    if (beta == 0.0) {
      cudaMemsetAsync(x, 0, sizeof(cplx) * n, st);
      converged = true;
      rho = 0.0;
      true_res = 0.0;
    } else {
      k_scale<<<grid_for(n), 256, 0, st>>>(n, b, cmk(1.0 / beta, 0.0), ws->V);
      g_helm_launches++;
      tags.push_back(-1);
      mV = 1;
      blk_start = 0;
      lsq.init(beta);
    }
  }
  for (int k = 1; rc == HELM_OK && !converged && k <= maxit; ++k) {
    if (1 + (long)k * t > ws->vcap || (long)k * t > ws->zcap) {
      rc = ws_reserve(prob, t, std::min(maxit, 2 * k), mV, nz, st);
      if (rc != HELM_OK) break;
      wk.partial = ws->partial; wk.hsmall = pinned_small(ws->small_cap); wk.small_cap = ws->small_cap;
      d_gram = ws->dsm; d_cv = d_gram + t * t; d_nn = d_cv + 2 * t * t;
    }
    cplx* V = ws->V;
    cplx* Z = ws->Z;
    cplx* W = ws->W;
    cplx* Rsrc = ws->Rsrc;
    // ---- a3: source selection (A19)
    const cplx* src = nullptr;
    long ldr = 0;
    const long nblk = mV - blk_start;
    if (k == 1) {
      src = V;
    } else if (t == 1) {
      src = V + (mV - 1) * n;
    } else if (t == 2) {
      long c0 = -1, c1 = -1;
      for (long c = blk_start; c < mV; ++c) {
        if (tags[c] == 0) c0 = c;
        if (tags[c] == 1) c1 = c;
      }
      if (c0 >= 0 && c1 >= 0) {
        cudaMemcpyAsync(Rsrc, V + c1 * n, sizeof(cplx) * n, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(Rsrc + n, V + c0 * n, sizeof(cplx) * n, cudaMemcpyDeviceToDevice, st);
        src = Rsrc;
        ldr = n;
      } else {
        src = V + blk_start * n;  // the survivor feeds both
      }
    } else {
      k_colsum<<<grid_for(n), 256, 0, st>>>(n, V + blk_start * n, n, (int)nblk, Rsrc);
      g_helm_launches++;
      src = Rsrc;
    }
    // ---- a4: Z_k = [M_i^{-1} src_i], one batched launch (this rank's directions)
    cplx* Zk = Z + nz * n;
    const long off = (long)rank * t_local;   // first global direction of this rank
    cudaEventRecord(ev[0], st);
    rc = sweep_apply_dev(dirs, t_local, ldr == 0 ? src : src + off * ldr, ldr, Zk + off * n, n, st);
    if (rc != HELM_OK) break;
    cudaEventRecord(ev[1], st);
    // ---- a5: W = A Z_k (this rank's columns)
    rc = helm_spmm_dev(prob, Zk + off * n, W + off * n, t_local, n, st);
    if (rc != HELM_OK) break;
    if (gather) {
      // direction-parallel: every rank receives all t new Z and W columns (in place)
      const long bytes = (long)t_local * n * (long)sizeof(cplx);
      if (gather(gctx, Zk + off * n, Zk, bytes, st) != 0 || gather(gctx, W + off * n, W, bytes, st) != 0) {
        helm_set_error("mpgmres_solve_dist: all-gather callback failed at iteration %d", k);
        rc = HELM_ECUDA;
        break;
      }
    }
    cudaEventRecord(ev[2], st);
    // ---- a6: Gram diagonal of A Z_k (for ||A z_i||), BCGS2 against V_1..k, intra-block CGS2
    const int m = (int)mV;
    std::vector<C> h1, h2, small;
    std::vector<double> nrm(t);
    int fused = orth_fused(ws, n, V, m, t, W, st);
    if (fused < 0) { rc = HELM_ECUDA; break; }
    if (fused) {
      // one device->host copy: [C1][C2][gram][cv][nn]
      cudaEventRecord(ev[3], st);
      std::vector<C> all;
      if ((rc = to_host(wk, ws->dsm, (size_t)(2 * m * t + 3 * t * t + t), all)) != HELM_OK) break;
      h1.assign(all.begin(), all.begin() + (size_t)m * t);
      h2.assign(all.begin() + (size_t)m * t, all.begin() + 2 * (size_t)m * t);
      small.assign(all.begin() + 2 * (size_t)m * t, all.end());
      for (int i = 0; i < t; ++i) nrm[i] = small[3 * t * t + i].real();
    } else {
      rc = dots(wk, W, n, t, W, n, t, d_gram, false);
      if (rc == HELM_OK) rc = dots(wk, V, n, m, W, n, t, ws->dC1, false);
      if (rc == HELM_OK) rc = update(wk, V, n, m, ws->dC1, W, n, t);
      if (rc == HELM_OK) rc = dots(wk, V, n, m, W, n, t, ws->dC2, false);
      if (rc == HELM_OK) rc = update(wk, V, n, m, ws->dC2, W, n, t);
      if (rc != HELM_OK) break;
      // intra-block CGS2 on the device: new column i is projected (twice) against
      // slots V[:, m .. m+i); a dropped column leaves a zero slot, so later
      // projections onto it vanish exactly as if it were skipped.
      for (int i = 0; i < t && rc == HELM_OK; ++i) {
        cplx* wi = W + (long)i * n;
        for (int pass = 0; pass < 2 && i > 0; ++pass) {
          cplx* cvi = d_cv + (long)pass * t * t + (long)i * t;
          rc = dots(wk, V + mV * n, n, i, wi, n, 1, cvi, false);
          if (rc == HELM_OK) rc = update(wk, V + mV * n, n, i, cvi, wi, n, 1);
          if (rc != HELM_OK) break;
        }
        if (rc != HELM_OK) break;
        rc = dots(wk, wi, n, 1, wi, n, 1, d_nn + i, false);
        if (rc != HELM_OK) break;
        k_decide<<<1, 32, 0, st>>>(d_nn + i, d_gram, t, i, ws->dscal, d_nrm);
        k_scale_dev<<<grid_for(n), 256, 0, st>>>(n, wi, ws->dscal, i, V + (mV + i) * n);
        g_helm_launches += 2;
      }
      if (rc != HELM_OK) break;
      cudaEventRecord(ev[3], st);
      if ((rc = to_host(wk, ws->dC1, (size_t)m * t, h1)) != HELM_OK) break;
      if ((rc = to_host(wk, ws->dC2, (size_t)m * t, h2)) != HELM_OK) break;
      if ((rc = to_host(wk, d_gram, (size_t)(3 * t * t + t), small)) != HELM_OK) break;
      e = cudaMemcpyAsync(nrm.data(), d_nrm, sizeof(double) * t, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) { helm_set_error("mpgmres_solve: %s", cudaGetErrorString(e)); rc = HELM_ECUDA; break; }
    }
    inner += 2L * m * t;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { helm_set_error("mpgmres_solve: %s", cudaGetErrorString(e)); rc = HELM_ECUDA; break; }
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[0], ev[1]); sweep_ms += ms;
    cudaEventElapsedTime(&ms, ev[1], ev[2]); spmv_ms += ms;
    cudaEventElapsedTime(&ms, ev[2], ev[3]); orth_ms += ms;
    const C* gram = small.data();
    const C* cv = gram + t * t;
    // failure detection: a non-finite Gram diagonal, projection or norm (a NaN / Inf
    // reached the new columns, e.g. from a singular strip solve) would otherwise be
    // "deflated" silently by the 1e-10 rule; stop with its own status instead
    {
      bool finite = true;
      for (int i = 0; i < t; ++i) finite = finite && std::isfinite(nrm[i]) && std::isfinite(gram[i * t + i].real());
      for (size_t j = 0; j < h1.size() && finite; ++j)
        finite = std::isfinite(h1[j].real()) && std::isfinite(h1[j].imag()) && std::isfinite(h2[j].real()) &&
                 std::isfinite(h2[j].imag());
      if (!finite) {
        helm_set_error("mpgmres_solve: non-finite values in the new block at iteration %d", k);
        rc = HELM_ENONFINITE;
        break;
      }
    }
    std::vector<int> kept;
    std::vector<std::vector<C>> Rb(t, std::vector<C>(t, C(0)));
    for (int i = 0; i < t; ++i) {
      double naz = std::sqrt(std::max(gram[i * t + i].real(), 0.0));
      for (int j = 0; j < i; ++j) Rb[j][i] = cv[i * t + j] + cv[t * t + i * t + j];
      inner += 2L * i + 1;
      if (!(nrm[i] > 1e-10 * naz)) { deflations++; continue; }
      Rb[i][i] = nrm[i];
      kept.push_back(i);
    }
    const int nk = (int)kept.size();
    // compact the kept slots to V[:, m .. m+nk)
    for (int jj = 0; jj < nk; ++jj)
      if (kept[jj] != jj)
        cudaMemcpyAsync(V + (mV + jj) * n, V + (mV + kept[jj]) * n, sizeof(cplx) * n, cudaMemcpyDeviceToDevice, st);
    // H block column: rows 0..m-1 = C1 + C2, then one row per kept column
    const int new_rows = (int)mV + nk;
    for (int i = 0; i < t; ++i) {
      std::vector<C> col(new_rows, C(0));
      for (int j = 0; j < m; ++j) col[j] = h1[j * t + i] + h2[j * t + i];
      for (int jj = 0; jj < nk; ++jj) col[m + jj] = Rb[kept[jj]][i];
      lsq.append(col, new_rows);
    }
    nz += t;
    blk_start = mV;
    for (int jj = 0; jj < nk; ++jj) tags.push_back(kept[jj]);
    mV += nk;
    double res = 0;
    lsq.solve(y, res);
    rho = res / beta;
    hist.push_back(rho);
    k_done = k;
    if (rho <= tol) { converged = true; break; }
    if (nk == 0) { exhausted = true; break; }
  }
  // ---- a8: x = Z y; true residual
  if (rc == HELM_OK && beta > 0.0 && nz > 0) {
    std::vector<cplx> yh(nz);
    for (long j = 0; j < nz; ++j) yh[j] = cmk(y[j].real(), y[j].imag());
    e = cudaMemcpyAsync(ws->dy, yh.data(), sizeof(cplx) * nz, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      k_gemv<<<grid_for(n), 256, 0, st>>>(n, ws->Z, n, (int)nz, ws->dy, x);
      g_helm_launches++;
      rc = helm_spmm_dev(prob, x, ws->tmp, 1, n, st);
      if (rc == HELM_OK) {
        k_axpy_sub<<<grid_for(n), 256, 0, st>>>(n, b, ws->tmp, ws->tmp);
        g_helm_launches++;
        rc = dots(wk, ws->tmp, n, 1, ws->tmp, n, 1, d_nn, false);
        std::vector<C> rr;
        if (rc == HELM_OK) rc = to_host(wk, d_nn, 1, rr);
        if (rc == HELM_OK) true_res = std::sqrt(std::max(rr[0].real(), 0.0)) / beta;
      }
    } else {
      helm_set_error("mpgmres_solve: %s", cudaGetErrorString(e));
      rc = HELM_ECUDA;
    }
  }
  if (rc == HELM_OK) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { helm_set_error("mpgmres_solve: %s", cudaGetErrorString(e)); rc = HELM_ECUDA; }
  }
  for (auto& ev_ : ev) cudaEventDestroy(ev_);
  helm_stage_free(sb, st);
  if (rc == HELM_OK) rc = helm_stage_out(sx, st);
  else helm_stage_free(sx, st);
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (stats) {
    stats->iterations = k_done;
    stats->converged = converged ? 1 : 0;
    stats->flags = (!converged && !exhausted ? 1 : 0) | (exhausted ? 2 : 0);
    stats->deflations = deflations;
    stats->proj_rel_res = rho;
    stats->true_rel_res = true_res;
    stats->solve_s = secs;
    stats->sweep_ms = sweep_ms;
    stats->spmv_ms = spmv_ms;
    stats->orth_ms = orth_ms;
    stats->matvecs = (long)k_done * t;
    stats->prec_applies = (long)k_done * t;
    stats->inner_products = inner;
    if (stats->history && stats->history_cap > 0)
      for (int i = 0; i < (int)hist.size() && i < stats->history_cap; ++i) stats->history[i] = hist[i];
  }
  if (rc != HELM_OK) return rc;
  if (exhausted) return HELM_EEXHAUSTED;
  if (!converged) return HELM_ENOCONV;
  return HELM_OK;
}

extern "C" int mpgmres_solve(helm_problem_t prob, const helm_sweep_t* dirs, int t, const double* b_in,
                             double* x_out, double tol, int maxit, mpgmres_stats* stats, void* stream) {
  return mpgmres_core(prob, dirs, t, t, 0, nullptr, nullptr, b_in, x_out, tol, maxit, stats, stream);
}

extern "C" int mpgmres_solve_dist(helm_problem_t prob, const helm_sweep_t* local_dirs, int t_local, int nranks,
                                  int rank, helm_allgather_fn allgather, void* ctx, const double* b, double* x,
                                  double tol, int maxit, mpgmres_stats* stats, void* stream) {
  if (nranks < 1 || rank < 0 || rank >= nranks || t_local < 1 || (nranks > 1 && !allgather)) {
    helm_set_error("mpgmres_solve_dist: need 0 <= rank < nranks, t_local >= 1 and an all-gather callback");
    return HELM_EINVAL;
  }
  return mpgmres_core(prob, local_dirs, t_local, t_local * nranks, rank, nranks > 1 ? allgather : nullptr, ctx, b, x,
                      tol, maxit, stats, stream);
}
