// krylov.cu -- hot-path rows a3 (source selection), a5 (SpMM), a6 (BCGS2 +
// intra-block CGS2 with deflation), a7 (host Householder least squares) and a8
// (x = Z y, true residual): mpgmres_solve, selective MPGMRES with
// the paper's selection rules, following SURVEY D10 step by step.
//
// Tall-skinny reductions are deterministic two-stage sums (per-block partials
// in a fixed row order, then a fixed-order sum over blocks): no fp64 atomics,
// so reruns are bitwise reproducible.
#include <chrono>
#include <cmath>
#include <complex>

#include "common.cuh"

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
struct HouseholderLSQ {
  typedef std::complex<double> C;
  std::vector<std::vector<C>> R;   // columns of the triangularised H~ (length nrows at append time)
  std::vector<std::vector<C>> v;   // reflector vectors (start at their column index)
  std::vector<C> tau;
  std::vector<C> g;                // transformed rhs
  int nrows = 0;

  void init(double beta) {
    g.assign(1, C(beta, 0.0));
    nrows = 1;
  }
  // apply reflector j to vector x (length >= its extent)
  void apply(int j, std::vector<C>& x) const {
    const std::vector<C>& vj = v[j];
    C s = 0;
    for (size_t k = 0; k < vj.size(); ++k) s += std::conj(vj[k]) * x[j + k];
    s *= tau[j];
    for (size_t k = 0; k < vj.size(); ++k) x[j + k] -= vj[k] * s;
  }
  // append a column (length new_nrows >= nrows); rows grow to new_nrows
  void append(std::vector<C> col, int new_nrows) {
    if (new_nrows > nrows) {
      g.resize(new_nrows, C(0));
      nrows = new_nrows;
    }
    col.resize(nrows, C(0));
    const int j = (int)R.size();
    for (int i = 0; i < j; ++i) apply(i, col);
    // reflector for rows j..nrows-1 (complex Householder, zeroes col[j+1..])
    std::vector<C> x(col.begin() + std::min(j, nrows), col.end());
    C tj = 0;
    std::vector<C> vj;
    if (!x.empty()) {
      double xn = 0;
      for (auto& e : x) xn += std::norm(e);
      xn = std::sqrt(xn);
      // x -> beta e1 with beta = -e^{i arg x0} ||x||, v = x - beta e1, tau = 2/||v||^2
      C alpha = x[0];
      double aa = std::abs(alpha);
      C phase = aa > 0 ? alpha / aa : C(1.0, 0.0);
      C beta = -phase * xn;
      vj = x;
      vj[0] = alpha - beta;
      double vn = 0;
      for (auto& e : vj) vn += std::norm(e);
      tj = vn > 0 ? C(2.0 / vn) : C(0);
    }
    v.push_back(vj);
    tau.push_back(tj);
    if (!vj.empty()) {
      apply(j, col);
      apply(j, g);
    }
    R.push_back(col);
  }
  // solve R y = g[0..ncols); entries with negligible |R_jj| are set to zero
  void solve(std::vector<C>& y, double& res) const {
    const int nc = (int)R.size();
    y.assign(nc, C(0));
    double rmax = 0;
    for (int j = 0; j < nc; ++j) rmax = std::max(rmax, std::abs(R[j][j]));
    for (int j = nc - 1; j >= 0; --j) {
      C s = g[j];
      for (int k = j + 1; k < nc; ++k) s -= R[k][j] * y[k];
      double d = std::abs(R[j][j]);
      y[j] = d > 1e-14 * rmax ? s / R[j][j] : C(0);
    }
    double r2 = 0;
    for (int i = nc; i < nrows; ++i) r2 += std::norm(g[i]);
    // columns with dropped pivots leave their g entry unmatched
    for (int j = 0; j < nc; ++j)
      if (!(std::abs(R[j][j]) > 1e-14 * rmax)) r2 += std::norm(g[j]);
    res = std::sqrt(r2);
  }
};

}  // namespace

extern "C" int mpgmres_solve(helm_problem_t prob, const helm_sweep_t* dirs, int t, const double* b_in,
                             double* x_out, double tol, int maxit, mpgmres_stats* stats, void* stream) {
  typedef std::complex<double> C;
  auto t0 = std::chrono::steady_clock::now();
  if (!prob || !dirs || !b_in || !x_out) { helm_set_error("mpgmres_solve: null argument"); return HELM_EINVAL; }
  if (t < 1 || t > kMaxT || !(tol > 0.0 && tol < 1.0) || maxit < 1) {
    helm_set_error("mpgmres_solve: need 1 <= t <= 8, 0 < tol < 1, maxit >= 1");
    return HELM_EINVAL;
  }
  for (int d = 0; d < t; ++d)
    if (!dirs[d] || dirs[d]->prob->n != prob->n) { helm_set_error("mpgmres_solve: direction %d size mismatch", d); return HELM_EDIM; }
  cudaStream_t st = (cudaStream_t)stream;
  const long n = prob->n;
  Staged sb, sx;
  HELM_TRY(helm_stage_in(b_in, sizeof(cplx) * n, true, st, sb));
  HELM_TRY(helm_stage_in(x_out, sizeof(cplx) * n, false, st, sx));
  const cplx* b = (const cplx*)sb.dev;
  cplx* x = (cplx*)sx.dev;

  const long vcols = 1 + (long)maxit * t;
  const long zcols = (long)maxit * t;
  cplx *V = nullptr, *Z = nullptr, *W = nullptr, *Rsrc = nullptr, *tmp = nullptr;
  cplx *dC1 = nullptr, *dC2 = nullptr, *dc = nullptr, *dy = nullptr;
  Work wk;
  wk.n = n;
  wk.st = st;
  wk.nblk = (int)((n + kDotChunk - 1) / kDotChunk) * kMaxT;  // upper bound over t
  cudaEvent_t ev[8];
  for (auto& e : ev) cudaEventCreate(&e);
  int rc = HELM_OK;
  double sweep_ms = 0, spmv_ms = 0, orth_ms = 0;
  long inner = 0;
  int deflations = 0;
  std::vector<double> hist;
  int k_done = 0;
  bool converged = false, exhausted = false;
  double rho = 1.0, true_res = NAN;

  auto fail = [&](int code) { rc = code; };
  cudaError_t e = cudaSuccess;
  e = cudaMallocAsync((void**)&V, sizeof(cplx) * n * vcols, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&Z, sizeof(cplx) * n * zcols, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&W, sizeof(cplx) * n * t, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&Rsrc, sizeof(cplx) * n * t, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&tmp, sizeof(cplx) * n, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&wk.partial, sizeof(cplx) * (size_t)wk.nblk * vcols * t, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dC1, sizeof(cplx) * vcols * t, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dC2, sizeof(cplx) * vcols * t, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dc, sizeof(cplx) * 64, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dy, sizeof(cplx) * zcols, st);
  wk.small_cap = (size_t)vcols * t + zcols + 64;
  if (e == cudaSuccess) e = cudaMallocHost((void**)&wk.hsmall, sizeof(cplx) * wk.small_cap);
  if (e != cudaSuccess) {
    helm_set_error("mpgmres_solve: allocation (%ld x %ld complex basis): %s", n, vcols, cudaGetErrorString(e));
    rc = HELM_ENOMEM;
  }
  std::vector<C> hv;
  HouseholderLSQ lsq;
  std::vector<int> tags;        // origin tag of each V column (-1 for v1)
  long blk_start = 0, mV = 0;   // first column of the newest block, #V columns
  long nz = 0;                  // #Z columns
  double beta = 0;
  std::vector<C> y;
  if (rc == HELM_OK) {
    // beta = ||b||, V1 = b / beta
    rc = dots(wk, b, n, 1, b, n, 1, dc, false);
    if (rc == HELM_OK) rc = to_host(wk, dc, 1, hv);
    if (rc == HELM_OK) {
      beta = std::sqrt(hv[0].real());
      if (beta == 0.0) {
        cudaMemsetAsync(x, 0, sizeof(cplx) * n, st);
        converged = true;
        rho = 0.0;
        true_res = 0.0;
      } else {
        k_scale<<<grid_for(n), 256, 0, st>>>(n, b, cmk(1.0 / beta, 0.0), V);
        g_helm_launches++;
        tags.push_back(-1);
        mV = 1;
        blk_start = 0;
        lsq.init(beta);
      }
    }
  }
  for (int k = 1; rc == HELM_OK && !converged && k <= maxit; ++k) {
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
    // ---- a4: Z_k = [M_i^{-1} src_i]
    cplx* Zk = Z + nz * n;
    cudaEventRecord(ev[0], st);
    rc = sweep_apply_dev(dirs, t, src, ldr, Zk, n, st);
    if (rc != HELM_OK) break;
    cudaEventRecord(ev[1], st);
    // ---- a5: W = A Z_k
    rc = helm_spmm_dev(prob, Zk, W, t, n, st);
    if (rc != HELM_OK) break;
    cudaEventRecord(ev[2], st);
    // ---- a6: norms of A z_i, BCGS2 against V_1..k
    rc = dots(wk, W, n, t, W, n, t, dc, false);
    if (rc != HELM_OK) break;
    const int m = (int)mV;
    rc = dots(wk, V, n, m, W, n, t, dC1, false);
    if (rc == HELM_OK) rc = update(wk, V, n, m, dC1, W, n, t);
    if (rc == HELM_OK) rc = dots(wk, V, n, m, W, n, t, dC2, false);
    if (rc == HELM_OK) rc = update(wk, V, n, m, dC2, W, n, t);
    if (rc != HELM_OK) break;
    inner += 2L * m * t;
    std::vector<C> gram, h1, h2;
    if ((rc = to_host(wk, dc, (size_t)t * t, gram)) != HELM_OK) break;
    std::vector<double> nAz(t);
    for (int i = 0; i < t; ++i) nAz[i] = std::sqrt(std::max(gram[i * t + i].real(), 0.0));
    // intra-block CGS2 with the 1e-10 deflation rule (D10 step 5)
    std::vector<std::vector<C>> Rb(t, std::vector<C>(t, C(0)));
    std::vector<int> kept;
    for (int i = 0; i < t && rc == HELM_OK; ++i) {
      cplx* wi = W + (long)i * n;
      const int nk = (int)kept.size();
      for (int pass = 0; pass < 2 && nk > 0; ++pass) {
        rc = dots(wk, V + mV * n, n, nk, wi, n, 1, dc, false);
        if (rc == HELM_OK) rc = update(wk, V + mV * n, n, nk, dc, wi, n, 1);
        if (rc != HELM_OK) break;
        std::vector<C> cv;
        if ((rc = to_host(wk, dc, nk, cv)) != HELM_OK) break;
        for (int j = 0; j < nk; ++j) Rb[kept[j]][i] += cv[j];
        inner += nk;
      }
      if (rc != HELM_OK) break;
      rc = dots(wk, wi, n, 1, wi, n, 1, dc, false);
      std::vector<C> nn;
      if (rc == HELM_OK) rc = to_host(wk, dc, 1, nn);
      if (rc != HELM_OK) break;
      inner += 1;
      double nrm = std::sqrt(std::max(nn[0].real(), 0.0));
      if (!(nrm > 1e-10 * nAz[i])) {
        deflations++;
        continue;
      }
      Rb[i][i] = nrm;
      k_scale<<<grid_for(n), 256, 0, st>>>(n, wi, cmk(1.0 / nrm, 0.0), V + (mV + nk) * n);
      g_helm_launches++;
      kept.push_back(i);
    }
    if (rc != HELM_OK) break;
    cudaEventRecord(ev[3], st);
    // H block column: rows 0..m-1 = C1 + C2, then one row per kept column
    if ((rc = to_host(wk, dC1, (size_t)m * t, h1)) != HELM_OK) break;
    if ((rc = to_host(wk, dC2, (size_t)m * t, h2)) != HELM_OK) break;
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[0], ev[1]); sweep_ms += ms;
    cudaEventElapsedTime(&ms, ev[1], ev[2]); spmv_ms += ms;
    cudaEventElapsedTime(&ms, ev[2], ev[3]); orth_ms += ms;
    const int nk = (int)kept.size();
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
    e = cudaMemcpyAsync(dy, yh.data(), sizeof(cplx) * nz, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      k_gemv<<<grid_for(n), 256, 0, st>>>(n, Z, n, (int)nz, dy, x);
      g_helm_launches++;
      rc = helm_spmm_dev(prob, x, tmp, 1, n, st);
      if (rc == HELM_OK) {
        k_axpy_sub<<<grid_for(n), 256, 0, st>>>(n, b, tmp, tmp);
        g_helm_launches++;
        rc = dots(wk, tmp, n, 1, tmp, n, 1, dc, false);
        std::vector<C> rr;
        if (rc == HELM_OK) rc = to_host(wk, dc, 1, rr);
        if (rc == HELM_OK) true_res = std::sqrt(std::max(rr[0].real(), 0.0)) / beta;
      }
    } else {
      fail(HELM_ECUDA);
    }
  }
  if (rc == HELM_OK) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { helm_set_error("mpgmres_solve: %s", cudaGetErrorString(e)); rc = HELM_ECUDA; }
  }
  cudaFreeAsync(V, st); cudaFreeAsync(Z, st); cudaFreeAsync(W, st); cudaFreeAsync(Rsrc, st);
  cudaFreeAsync(tmp, st); cudaFreeAsync(wk.partial, st); cudaFreeAsync(dC1, st); cudaFreeAsync(dC2, st);
  cudaFreeAsync(dc, st); cudaFreeAsync(dy, st);
  if (wk.hsmall) cudaFreeHost(wk.hsmall);
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
