// dense.cuh -- CTA-wide dense complex w x w block helpers for the strip
// factorisation (setup only; the hot path is sweep_apply.cu).
// All blocks are row-major w x w; every helper must be called by the whole CTA
// and ends with __syncthreads().
#pragma once
#include "common.cuh"

// Bidiagonal coupling U of a strip (D7 block structure): row c couples to row
// c+1 through U_c with U[p][p] = cr[p], U[p][p+1] = ne[p].  L_{c+1} = U_c^T.
enum BidiMode { BD_NONE = 0, BD_U = 1, BD_UT = 2 };

struct Bidi {
  int mode;
  const cplx* cr;
  const cplx* ne;
};

// (L X)[p][s] for a left bidiagonal factor
__device__ __forceinline__ cplx bidi_left(const Bidi& L, const cplx* X, int w, int p, int s) {
  if (L.mode == BD_NONE) return X[p * w + s];
  cplx acc = cmul(L.cr[p], X[p * w + s]);
  if (L.mode == BD_U) {
    if (p + 1 < w) cfma(acc, L.ne[p], X[(p + 1) * w + s]);
  } else {
    if (p >= 1) cfma(acc, L.ne[p - 1], X[(p - 1) * w + s]);
  }
  return acc;
}

// out[p][q] (+)= alpha * (L X R)[p][q]; R applied on the right:
//   R = U : (Y U)[p][q] = cr[q] Y[p][q] + ne[q-1] Y[p][q-1]
//   R = UT: (Y U^T)[p][q] = cr[q] Y[p][q] + ne[q] Y[p][q+1]
__device__ inline void blk_lxr(cplx* out, const cplx* X, Bidi L, Bidi R, int w, double alpha,
                               bool accumulate) {
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    int p = e / w, q = e % w;
    cplx v;
    if (R.mode == BD_NONE) {
      v = bidi_left(L, X, w, p, q);
    } else {
      v = cmul(R.cr[q], bidi_left(L, X, w, p, q));
      if (R.mode == BD_U) {
        if (q >= 1) cfma(v, R.ne[q - 1], bidi_left(L, X, w, p, q - 1));
      } else {
        if (q + 1 < w) cfma(v, R.ne[q], bidi_left(L, X, w, p, q + 1));
      }
    }
    v = cscale(v, alpha);
    out[e] = accumulate ? cadd(out[e], v) : v;
  }
  __syncthreads();
}

// C (+)= alpha * op(A) * B, op(A) = A or A^T; C must not alias A or B.
__device__ inline void blk_matmul(cplx* C, const cplx* A, bool transA, const cplx* B, int w,
                                  double alpha, bool accumulate) {
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    int p = e / w, q = e % w;
    cplx acc = cmk(0.0, 0.0);
    if (!transA) {
      for (int r = 0; r < w; ++r) cfma(acc, A[p * w + r], B[r * w + q]);
    } else {
      for (int r = 0; r < w; ++r) cfma(acc, A[r * w + p], B[r * w + q]);
    }
    acc = cscale(acc, alpha);
    C[e] = accumulate ? cadd(C[e], acc) : acc;
  }
  __syncthreads();
}

// Register-tiled C (+)= alpha * op(A) B for w x w blocks with explicit leading
// dimensions (4 x 4 output tile per thread: 8 operand loads per 16 products).
// C must not alias A or B.  Whole CTA; ends with __syncthreads().
__device__ inline void blk_mm_tiled(cplx* C, int ldc, const cplx* A, int lda, bool transA, const cplx* B, int ldb,
                                    int w, double alpha, bool accumulate) {
  const int nt = (w + 3) / 4;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) {
    const int i0 = (t / nt) * 4, j0 = (t % nt) * 4;
    cplx acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = cmk(0, 0);
    for (int r = 0; r < w; ++r) {
      cplx av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        av[u] = i < w ? (transA ? A[(long)r * lda + i] : A[(long)i * lda + r]) : cmk(0, 0);
        const int j = j0 + u;
        bv[u] = j < w ? B[(long)r * ldb + j] : cmk(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) cfma(acc[u][v], av[u], bv[v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = i0 + u, j = j0 + v;
        if (i < w && j < w) {
          const cplx val = cscale(acc[u][v], alpha);
          C[(long)i * ldc + j] = accumulate ? cadd(C[(long)i * ldc + j], val) : val;
        }
      }
  }
  __syncthreads();
}

// FP64 tensor-core variant: C (+)= alpha * op(A) B on 8 x 8 output tiles, one warp per
// tile, k in steps of 4 (mma.sync.m8n8k4.f64: lane l holds A[l/4][l%4], B[l%4][l/4] and
// C[l/4][2 (l%4) + {0, 1}]).  The complex product is four real ones on the interleaved
// operands: Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br; one 16-byte operand load per lane and
// matrix feeds all four (the 4 x 4 register-tiled DFMA product needs eight loads per 16
// complex products and ran at ~0.2 of the FP64 peak in the setup kernels; tools/bench_dmma.cu:
// a 35^3 complex product takes 3.5-4.0 k SM-cycles from shared memory, the tensor pipe's
// peak is 37.2 TFLOP/s).  Every warp of the CTA must call it (whole warps execute the mma).
// Rows / columns / k >= w read as zero.  C must not alias A or B.  Ends with __syncthreads().
// A variant with two tiles and two k-split accumulator sets per warp measured slower.
__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ inline void blk_mm_dmma(cplx* C, int ldc, const cplx* A, int lda, bool transA, const cplx* B, int ldb,
                                   int w, double alpha, bool accumulate) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int nt = (w + 7) >> 3;
  const int lr = lane >> 2, lk = lane & 3;
  for (int t = warp; t < nt * nt; t += nw) {
    const int i0 = (t / nt) * 8, j0 = (t % nt) * 8;
    const int ia = i0 + lr, jb = j0 + lr;
    const bool aok = ia < w, bok = jb < w;
    const cplx* Ap = transA ? A + ia : A + (long)ia * lda;
    const long as = transA ? lda : 1;
    const cplx* Bp = B + jb;
    double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
#pragma unroll 3
    for (int k0 = 0; k0 < w; k0 += 4) {
      const int k = k0 + lk;
      const bool kok = k < w;
      const cplx a = (aok && kok) ? Ap[(long)k * as] : cmk(0, 0);
      const cplx b = (bok && kok) ? Bp[(long)k * ldb] : cmk(0, 0);
      dmma_884(cr0, cr1, a.x, b.x);
      dmma_884(cr0, cr1, -a.y, b.y);
      dmma_884(ci0, ci1, a.x, b.y);
      dmma_884(ci0, ci1, a.y, b.x);
    }
    if (aok) {
      const int j = j0 + 2 * lk;
      cplx* Cp = C + (long)ia * ldc + j;
      if (j < w) {
        const cplx v = cmk(alpha * cr0, alpha * ci0);
        Cp[0] = accumulate ? cadd(Cp[0], v) : v;
      }
      if (j + 1 < w) {
        const cplx v = cmk(alpha * cr1, alpha * ci1);
        Cp[1] = accumulate ? cadd(Cp[1], v) : v;
      }
    }
  }
  __syncthreads();
}

// Shared-memory leading dimensions of the tensor-core product's operands: A fragments
// (2 rows x 4 k per quarter-warp) are conflict-free when lda = 4 mod 8, B fragments
// (4 k x 2 columns) when ldb = 2 or 6 mod 8.
__host__ __device__ inline int dmma_lda(int w) { return w + ((4 - w % 8) + 8) % 8; }
__host__ __device__ inline int dmma_ldb(int w) { int l = w; while (l % 8 != 2 && l % 8 != 6) ++l; return l; }
constexpr int kDmmaPanel = 32, kDmmaPanelLd = 34;   // column panel of the staged product and its leading dimension

// C (+)= alpha A B for operands in global memory (wide blocks: w x w does not fit shared
// memory three times): A is staged whole into sA (w x dmma_lda(w)), B in panels of 32
// columns into sB (w x 34), each output tile by one warp as in blk_mm_dmma.  C must not
// alias A or B.  Whole CTA; ends with __syncthreads().
__device__ inline void blk_mm_dmma_staged(cplx* C, int ldc, const cplx* A, int lda, const cplx* B, int ldb, int w,
                                          double alpha, bool accumulate, cplx* sA, cplx* sB) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, nw = nthr >> 5, lane = tid & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int la = dmma_lda(w);
  const int ntr = (w + 7) >> 3;
  for (int e = tid; e < w * w; e += nthr) {
    const int r = e / w, c = e - r * w;
    sA[r * la + c] = __ldcg(A + (long)r * lda + c);
  }
  for (int c0 = 0; c0 < w; c0 += kDmmaPanel) {
    const int nc = min(kDmmaPanel, w - c0);
    __syncthreads();   // the previous panel's readers are done (and, the first time, sA is complete below)
    for (int e = tid; e < w * kDmmaPanel; e += nthr) {
      const int r = e >> 5, cc = e & 31;
      sB[r * kDmmaPanelLd + cc] = cc < nc ? __ldcg(B + (long)r * ldb + c0 + cc) : cmk(0.0, 0.0);
    }
    __syncthreads();
    const int ntc = (nc + 7) >> 3;
    for (int t = warp; t < ntr * ntc; t += nw) {
      const int ti = t / ntc, tj = t - ti * ntc;
      const int ia = ti * 8 + lr, jb = tj * 8 + lr;
      const bool aok = ia < w;
      const cplx* Ap = sA + ia * la;
      const cplx* Bp = sB + jb;
      double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
#pragma unroll 4
      for (int k0 = 0; k0 < w; k0 += 4) {
        const int k = k0 + lk;
        const bool kok = k < w;
        const cplx a = (aok && kok) ? Ap[k] : cmk(0, 0);
        const cplx b = kok ? Bp[k * kDmmaPanelLd] : cmk(0, 0);
        dmma_884(cr0, cr1, a.x, b.x);
        dmma_884(cr0, cr1, -a.y, b.y);
        dmma_884(ci0, ci1, a.x, b.y);
        dmma_884(ci0, ci1, a.y, b.x);
      }
      if (aok) {
        const int j = c0 + tj * 8 + 2 * lk;
        cplx* Cp = C + (long)ia * ldc + j;
        if (j < w) {
          const cplx v = cmk(alpha * cr0, alpha * ci0);
          Cp[0] = accumulate ? cadd(Cp[0], v) : v;
        }
        if (j + 1 < w) {
          const cplx v = cmk(alpha * cr1, alpha * ci1);
          Cp[1] = accumulate ? cadd(Cp[1], v) : v;
        }
      }
    }
  }
  __syncthreads();
}

// The same product with every output tile of the warp held in registers until all
// warps are done with the operands (MAXT >= tiles per warp): C may alias A or B.
template <int MAXT>
__device__ __forceinline__ void blk_mm_dmma_reg(cplx* C, int ldc, const cplx* A, int lda, const cplx* B, int ldb, int w,
                                                double alpha) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int nt = (w + 7) >> 3;
  const int lr = lane >> 2, lk = lane & 3;
  double c[MAXT][4];
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    c[u][0] = c[u][1] = c[u][2] = c[u][3] = 0.0;
    const int t = warp + u * nw;
    if (t < nt * nt) {   // warp-uniform
      const int ia = (t / nt) * 8 + lr, jb = (t % nt) * 8 + lr;
      const bool aok = ia < w, bok = jb < w;
      const cplx* Ap = A + ia * lda;
      const cplx* Bp = B + jb;
#pragma unroll 3
      for (int k0 = 0; k0 < w; k0 += 4) {
        const int k = k0 + lk;
        const bool kok = k < w;
        const cplx a = (aok && kok) ? Ap[k] : cmk(0, 0);
        const cplx b = (bok && kok) ? Bp[k * ldb] : cmk(0, 0);
        dmma_884(c[u][0], c[u][1], a.x, b.x);
        dmma_884(c[u][0], c[u][1], -a.y, b.y);
        dmma_884(c[u][2], c[u][3], a.x, b.y);
        dmma_884(c[u][2], c[u][3], a.y, b.x);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    const int t = warp + u * nw;
    if (t < nt * nt) {
      const int ia = (t / nt) * 8 + lr, j = (t % nt) * 8 + 2 * lk;
      if (ia < w) {
        if (j < w) C[ia * ldc + j] = cmk(alpha * c[u][0], alpha * c[u][2]);
        if (j + 1 < w) C[ia * ldc + j + 1] = cmk(alpha * c[u][1], alpha * c[u][3]);
      }
    }
  }
  __syncthreads();
}

// 2 x 2-tiled variant for large CTAs (324 tiles at w = 35)
__device__ inline void blk_mm_tiled2(cplx* C, int ldc, const cplx* A, int lda, bool transA, const cplx* B, int ldb,
                                     int w, double alpha, bool accumulate) {
  const int nt = (w + 1) / 2;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) {
    const int i0 = (t / nt) * 2, j0 = (t % nt) * 2;
    cplx acc[2][2] = {{cmk(0, 0), cmk(0, 0)}, {cmk(0, 0), cmk(0, 0)}};
    for (int r = 0; r < w; ++r) {
      cplx av[2], bv[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = i0 + u, j = j0 + u;
        av[u] = i < w ? (transA ? A[(long)r * lda + i] : A[(long)i * lda + r]) : cmk(0, 0);
        bv[u] = j < w ? B[(long)r * ldb + j] : cmk(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) cfma(acc[u][v], av[u], bv[v]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = i0 + u, j = j0 + v;
        if (i < w && j < w) {
          const cplx val = cscale(acc[u][v], alpha);
          C[(long)i * ldc + j] = accumulate ? cadd(C[(long)i * ldc + j], val) : val;
        }
      }
  }
  __syncthreads();
}

__device__ inline void blk_copy(cplx* dst, const cplx* src, int w) {
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) dst[e] = src[e];
  __syncthreads();
}

// In-place Gauss-Jordan inversion with partial (row) pivoting of a w x w block
// in shared memory.  piv: smem int[w]; col: smem cplx[w]; red: smem scratch of
// >= 2*32 doubles/ints.  Returns (to all threads) 0 on success, 1 if a pivot is 0.
__device__ inline int gj_invert(cplx* A, int w, int* piv, cplx* col, double* redv, int* redi,
                                int* flag) {
  const int tid = threadIdx.x;
  if (tid == 0) *flag = 0;
  __syncthreads();
  for (int k = 0; k < w; ++k) {
    // pivot search in column k (warp 0)
    if (tid < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < w; i += 32) {
        double v = cabs2(A[i * w + k]);
        if (v > best) { best = v; bi = i; }
      }
      for (int off = 16; off > 0; off >>= 1) {
        double ob = __shfl_down_sync(0xffffffffu, best, off);
        int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        piv[k] = bi;
        redv[0] = best;
        if (!(best > 0.0)) *flag = 1;
      }
    }
    __syncthreads();
    if (*flag) return 1;
    const int p = piv[k];
    if (p != k) {
      for (int j = tid; j < w; j += blockDim.x) {
        cplx t = A[k * w + j];
        A[k * w + j] = A[p * w + j];
        A[p * w + j] = t;
      }
      __syncthreads();
    }
    // save column k (multipliers), then scale row k
    for (int i = tid; i < w; i += blockDim.x) col[i] = A[i * w + k];
    __syncthreads();
    const cplx dinv = cinv(col[k]);
    for (int j = tid; j < w; j += blockDim.x) {
      cplx v = (j == k) ? cmk(1.0, 0.0) : A[k * w + j];
      A[k * w + j] = cmul(v, dinv);
    }
    __syncthreads();
    // eliminate column k from all other rows: a warp per row, lanes along the
    // row (no index division, contiguous shared-memory access); the pivot row is
    // held in registers (w <= 128: four entries per lane), read once per pivot
    {
      const int lane = tid & 31, nwarp = (int)(blockDim.x >> 5);
      if (w <= 128) {
        cplx rr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) rr[u] = lane + 32 * u < w ? A[k * w + lane + 32 * u] : cmk(0.0, 0.0);
        for (int i = tid >> 5; i < w; i += nwarp) {
          if (i == k) continue;
          const cplx f = col[i];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = lane + 32 * u;
            if (j < w) {
              const long e = (long)i * w + j;
              cplx a = (j == k) ? cmk(0.0, 0.0) : A[e];
              a.x -= f.x * rr[u].x - f.y * rr[u].y;
              a.y -= f.x * rr[u].y + f.y * rr[u].x;
              A[e] = a;
            }
          }
        }
      } else {
        for (int i = tid >> 5; i < w; i += nwarp) {
          if (i == k) continue;
          const cplx f = col[i];
          for (int j = lane; j < w; j += 32) {
            const long e = (long)i * w + j;
            cplx a = (j == k) ? cmk(0.0, 0.0) : A[e];
            const cplx r = A[k * w + j];
            a.x -= f.x * r.x - f.y * r.y;
            a.y -= f.x * r.y + f.y * r.x;
            A[e] = a;
          }
        }
      }
    }
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, in reverse order
  for (int k = w - 1; k >= 0; --k) {
    int p = piv[k];
    if (p != k) {
      for (int i = tid; i < w; i += blockDim.x) {
        cplx t = A[i * w + k];
        A[i * w + k] = A[i * w + p];
        A[i * w + p] = t;
      }
      __syncthreads();
    }
  }
  (void)redi;
  return 0;
}

// Blocked in-place Gauss-Jordan inversion with partial (row) pivoting, panels of 8 pivots.
// The elementary operations and the pivot rule are gj_invert's; only their order differs:
// within a panel the eliminations touch the panel's columns only (they then hold N = T e_J,
// the accumulated transformation T of the panel's pivot steps applied to the unit vectors),
// and every other column c gets the panel's row interchanges and steps afterwards,
// A[:, c] <- A[:, c] + (N - I_J) A[J, c]: the rows J outside the panel are saved to ybuf
// and cleared, then A += N ybuf on the FP64 tensor cores (mma.sync.m8n8k4: M = w, K = 8,
// N = w - 8).  97% of the flops of a 99 x 99 inversion move from a shared-memory-bound
// rank-1 sweep per pivot (five CTA barriers each) to the tensor pipe.  The panel itself
// (w x 8) is factored by the first ceil(w / 32) warps, a thread per row, synchronised by a
// named barrier (four per pivot) instead of CTA barriers; a single warp with four rows per
// lane measured slower.
// A has leading dimension ld.  ybuf: 8 * w entries of shared memory; col, redv: unused (kept
// for the call signature).
// Whole CTA (whole warps).  Returns 1 (to all threads) if a pivot is zero.
// For the 35 x 35 blocks of the narrow strips it measured 2.3x SLOWER than the register-row
// Gauss-Jordan (row_gj.cuh: 100 k against 44 k cycles per inversion in k_reduced, segment
// factors 9.5 against 5.1 ms per axis): five group barriers per pivot against two, and a
// product of only 20 tiles per panel.  Used for strips wider than 36 nodes only.
__device__ inline int gj_invert_blk(cplx* A, int ld, int w, int* piv, cplx* col, cplx* ybuf, double* redv, int* flag) {
  constexpr int NB = 8;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, nw = nthr >> 5, lane = tid & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int nt = (w + 7) >> 3;
  const int npw = (w + 31) >> 5;   // warps of the panel group (w <= 32 * warps of the CTA)
  (void)col; (void)redv;
  if (tid == 0) *flag = 0;
  __syncthreads();
  for (int j0 = 0; j0 < w; j0 += NB) {
    const int nb = min(NB, w - j0);
    // ---- the panel's columns, all rows: the first ceil(w / 32) warps, a thread per row,
    // synchronised among themselves by a named barrier (the other warps wait below)
    if (warp < npw) {
      const int i = tid;                       // this thread's row
      const bool row = i < w;
      double* rv = reinterpret_cast<double*>(ybuf);        // [npw] warp maxima (ybuf is free here)
      int* ri = reinterpret_cast<int*>(ybuf + 4);          // [npw] their rows
      auto pbar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(npw * 32) : "memory"); };
      for (int k = j0; k < j0 + nb; ++k) {
        double best = (row && i >= k) ? cabs2(A[i * ld + k]) : -1.0;
        int bi = i;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) { rv[warp] = best; ri[warp] = bi; }
        pbar();
        best = rv[0]; bi = ri[0];
        for (int q = 1; q < npw; ++q)
          if (rv[q] > best) { best = rv[q]; bi = ri[q]; }   // ties: the lower row (warps in row order)
        if (!(best > 0.0)) {   // uniform over the group
          if (tid == 0) *flag = 1;
          break;
        }
        const int p = bi;
        if (tid == 0) piv[k] = p;
        if (p != k && tid < nb) {
          const cplx t = A[k * ld + j0 + tid];
          A[k * ld + j0 + tid] = A[p * ld + j0 + tid];
          A[p * ld + j0 + tid] = t;
        }
        pbar();
        const cplx dinv = cinv(A[k * ld + k]);
        const cplx f = row ? A[i * ld + k] : cmk(0.0, 0.0);   // this row's multiplier
        cplx av[NB];
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) av[jj] = (row && jj < nb) ? A[i * ld + j0 + jj] : cmk(0.0, 0.0);
        pbar();
        if (i == k) {
#pragma unroll
          for (int jj = 0; jj < NB; ++jj)
            if (jj < nb) A[k * ld + j0 + jj] = cmul(j0 + jj == k ? cmk(1.0, 0.0) : av[jj], dinv);
        }
        pbar();
        if (row && i != k) {
#pragma unroll
          for (int jj = 0; jj < NB; ++jj) {
            if (jj < nb) {
              const cplx r = A[k * ld + j0 + jj];
              cplx a = (j0 + jj == k) ? cmk(0.0, 0.0) : av[jj];
              a.x -= f.x * r.x - f.y * r.y;
              a.y -= f.x * r.y + f.y * r.x;
              A[i * ld + j0 + jj] = a;
            }
          }
        }
        pbar();
      }
    }
    __syncthreads();
    if (*flag) return 1;
    // ---- the panel's row interchanges on every other column (a thread per column, in order)
    for (int c = tid; c < w; c += nthr) {
      if (c >= j0 && c < j0 + nb) continue;
      for (int k = j0; k < j0 + nb; ++k) {
        const int p = piv[k];
        if (p != k) {
          const cplx t = A[k * ld + c];
          A[k * ld + c] = A[p * ld + c];
          A[p * ld + c] = t;
        }
      }
    }
    __syncthreads();
    // ---- ybuf = A[J, :] outside the panel (zero inside), rows J cleared there
    for (int e = tid; e < NB * w; e += nthr) {
      const int kk = e / w, c = e - kk * w;
      const bool inpanel = c >= j0 && c < j0 + nb;
      cplx y = cmk(0.0, 0.0);
      if (kk < nb && !inpanel) {
        y = A[(j0 + kk) * ld + c];
        A[(j0 + kk) * ld + c] = cmk(0.0, 0.0);
      }
      ybuf[e] = y;
    }
    __syncthreads();
    // A += N ybuf on 8 x 8 tiles (one warp per tile), all tile columns but the panel's own
    const int tjp = j0 >> 3;
    for (int t = warp; t < nt * nt; t += nw) {
      const int ti = t / nt, tj = t - ti * nt;
      if (tj == tjp) continue;   // warp-uniform
      const int ia = ti * 8 + lr, jb = tj * 8 + lr;
      double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const int k = k0 + lk;
        const cplx a = (ia < w && k < nb) ? A[ia * ld + j0 + k] : cmk(0, 0);
        const cplx b = jb < w ? ybuf[k * w + jb] : cmk(0, 0);
        dmma_884(cr0, cr1, a.x, b.x);
        dmma_884(cr0, cr1, -a.y, b.y);
        dmma_884(ci0, ci1, a.x, b.y);
        dmma_884(ci0, ci1, a.y, b.x);
      }
      if (ia < w) {
        const int j = tj * 8 + 2 * lk;
        cplx* Cp = A + ia * ld + j;
        if (j < w) Cp[0] = cadd(Cp[0], cmk(cr0, ci0));
        if (j + 1 < w) Cp[1] = cadd(Cp[1], cmk(cr1, ci1));
      }
    }
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, in reverse order (a thread per row)
  for (int i = tid; i < w; i += nthr) {
    for (int k = w - 1; k >= 0; --k) {
      const int p = piv[k];
      if (p != k) {
        const cplx t = A[i * ld + k];
        A[i * ld + k] = A[i * ld + p];
        A[i * ld + p] = t;
      }
    }
  }
  __syncthreads();
  return 0;
}
