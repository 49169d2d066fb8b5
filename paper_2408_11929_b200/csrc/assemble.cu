// assemble.cu -- helm_assemble (a1), helm_load_vector (a1, b = M1 f), helm_spmv
// (a5 SpMV/SpMM), error/staging plumbing of the helmsweep C ABI.
#include <cstdarg>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "p1_entries.cuh"

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";
std::atomic<long> g_helm_launches{0};

void helm_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* helm_last_error(void) { return g_err; }
extern "C" long helm_kernel_launches(void) { return g_helm_launches.load(); }

static std::atomic<int> g_knobs[KNOB_COUNT];
int helm_knob(int id) { return (id >= 0 && id < KNOB_COUNT) ? g_knobs[id].load() : 0; }

extern "C" int helm_set_knob(const char* name, int value) {
  static const char* names[KNOB_COUNT] = {"sweep_kernel", "general_reducer", "no_wide_xinv", "factor_generic",
                                          "orth_unfused", "setup_timing", "orth_prof", "setup_chunks", "sep_two_level"};
  if (!name) return HELM_EINVAL;
  for (int k = 0; k < KNOB_COUNT; ++k)
    if (strcmp(name, names[k]) == 0) {
      if (k == KNOB_SWEEP_KERNEL && value != 0 && value != 2 && value != 3) break;
      g_knobs[k] = value;
      return HELM_OK;
    }
  helm_set_error("helm_set_knob: unknown knob or value (%s = %d)", name, value);
  return HELM_EINVAL;
}

extern "C" const char* helm_strerror(int code) {
  switch (code) {
    case HELM_OK: return "ok";
    case HELM_EINVAL: return "invalid argument";
    case HELM_EDIM: return "dimension mismatch";
    case HELM_ESINGULAR: return "singular pivot in strip factorisation";
    case HELM_ECUDA: return "CUDA error";
    case HELM_ENOMEM: return "out of device memory";
    case HELM_ENOCONV: return "maxit reached without convergence";
    case HELM_EEXHAUSTED: return "search space exhausted (block fully deflated)";
    case HELM_ENONFINITE: return "non-finite values in the Krylov block";
    default: return "unknown status";
  }
}

// ------------------------------------------------------------------ device memory
// allocations and frees are ordered on a private non-blocking stream that carries no
// other work: the synchronisation in helm_dev_alloc returns at once and never waits for
// (or serialises with) kernels the caller runs on other streams -- e.g. the two axes'
// sweep_setup calls running concurrently -- and memory freed by a destroyed handle is
// reused by the next allocation without cross-stream ordering questions.  Handles must
// be destroyed only after the work that uses them has completed (every ABI call that
// launches work synchronises its stream before returning).
static cudaStream_t g_alloc_stream = nullptr;
static std::once_flag g_alloc_stream_ready;
static cudaStream_t alloc_stream() {
  std::call_once(g_alloc_stream_ready, []() { cudaStreamCreateWithFlags(&g_alloc_stream, cudaStreamNonBlocking); });
  return g_alloc_stream;
}

cudaError_t helm_dev_alloc(void** p, size_t bytes) {
  static std::once_flag pool_ready;
  std::call_once(pool_ready, []() {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  });
  cudaStream_t as = alloc_stream();
  cudaError_t e = cudaMallocAsync(p, bytes > 0 ? bytes : 16, as);
  if (e == cudaSuccess) e = cudaStreamSynchronize(as);
  return e;
}

void helm_dev_free(void* p) {
  if (p) cudaFreeAsync(p, alloc_stream());
}

// ------------------------------------------------------------------ staging
bool helm_is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int helm_stage_in(const void* ptr, size_t bytes, bool copy_in, cudaStream_t st, Staged& out) {
  out = Staged();
  out.bytes = bytes;
  if (ptr == nullptr || helm_is_device_ptr(ptr)) {
    out.dev = const_cast<void*>(ptr);
    return HELM_OK;
  }
  out.host = ptr;
  out.owned = true;
  HELM_CUDA_TRY(cudaMallocAsync(&out.dev, bytes, st));
  if (copy_in) HELM_CUDA_TRY(cudaMemcpyAsync(out.dev, ptr, bytes, cudaMemcpyHostToDevice, st));
  return HELM_OK;
}

int helm_stage_out(Staged& s, cudaStream_t st) {
  if (s.owned) {
    HELM_CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(s.host), s.dev, s.bytes, cudaMemcpyDeviceToHost, st));
    HELM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  helm_stage_free(s, st);
  return HELM_OK;
}

void helm_stage_free(Staged& s, cudaStream_t st) {
  if (s.owned && s.dev) cudaFreeAsync(s.dev, st);
  s.dev = nullptr;
  s.owned = false;
}

// ------------------------------------------------------------------ kernels
__global__ void k_assemble(GridView g, cplx* dC, cplx* dE, cplx* dN, cplx* dNE) {
  long n = (long)(g.nx + 1) * (g.ny + 1);
  CellSel all = sel_all();
  for (long gi = blockIdx.x * (long)blockDim.x + threadIdx.x; gi < n; gi += (long)gridDim.x * blockDim.x) {
    int i = (int)(gi % (g.nx + 1)), j = (int)(gi / (g.nx + 1));
    dC[gi] = entry_C(g, all, i, j);
    dE[gi] = entry_E(g, all, i, j);
    dN[gi] = entry_N(g, all, i, j);
    dNE[gi] = entry_NE(g, all, i, j);
  }
}

// Five-point scheme (the paper's own; DESIGN.md §3 FD5), constant k =
// omega: A = Delta_h + k^2 with ghost-point impedance rows (Eq. 1b).  Stored as
// the complex-symmetric S = D A (common.cuh fd5_d on the global grid) in the
// same 4 diagonals (NE = 0); k_spmm applies A = D^{-1} S.
__global__ void k_assemble_fd5(int nx, int ny, double h, double k, cplx* dC, cplx* dE, cplx* dN, cplx* dNE) {
  const long n = (long)(nx + 1) * (ny + 1);
  const double ih2 = 1.0 / (h * h);
  for (long gi = blockIdx.x * (long)blockDim.x + threadIdx.x; gi < n; gi += (long)gridDim.x * blockDim.x) {
    const int i = (int)(gi % (nx + 1)), j = (int)(gi / (nx + 1));
    const bool ie = i == 0 || i == nx, je = j == 0 || j == ny;
    const double di = ie ? 0.5 : 1.0, dj = je ? 0.5 : 1.0;
    dC[gi] = cmk(di * dj * (-4.0 * ih2 + k * k), di * dj * (2.0 * k / h) * ((ie ? 1 : 0) + (je ? 1 : 0)));
    dE[gi] = i < nx ? cmk(dj * ih2, 0.0) : cmk(0, 0);
    dN[gi] = j < ny ? cmk(di * ih2, 0.0) : cmk(0, 0);
    dNE[gi] = cmk(0, 0);
  }
}

// b = M1 f (D5): sum over the 6 triangles around node g of
// (h^2/24) (2 f_g + f_o1 + f_o2)  (consistent P1 mass, unit coefficient).
__global__ void k_load_vector(int nx, int ny, double h, const cplx* __restrict__ f, cplx* __restrict__ b) {
  long n = (long)(nx + 1) * (ny + 1);
  const double w = h * h / 24.0;
  const long s = nx + 1;
  for (long gi = blockIdx.x * (long)blockDim.x + threadIdx.x; gi < n; gi += (long)gridDim.x * blockDim.x) {
    int i = (int)(gi % s), j = (int)(gi / s);
    cplx fg = f[gi];
    cplx acc = cmk(0.0, 0.0);
    auto tri = [&](bool ok, long o1, long o2) {
      if (!ok) return;
      cplx t = cadd(cscale(fg, 2.0), cadd(f[o1], f[o2]));
      acc = cadd(acc, cscale(t, w));
    };
    bool ci = i < nx, cj = j < ny, pi = i > 0, pj = j > 0;
    tri(ci && cj, gi + 1, gi + s + 1);          // T_L(i,j): (i+1,j), (i+1,j+1)
    tri(ci && cj, gi + s + 1, gi + s);          // T_U(i,j): (i+1,j+1), (i,j+1)
    tri(pi && cj, gi - 1, gi + s);              // T_L(i-1,j): (i-1,j), (i,j+1)
    tri(pi && pj, gi - s - 1, gi - s);          // T_L(i-1,j-1): (i-1,j-1), (i,j-1)
    tri(pi && pj, gi - s - 1, gi - 1);          // T_U(i-1,j-1): (i-1,j-1), (i-1,j)
    tri(ci && pj, gi - s, gi + 1);              // T_U(i,j-1): (i,j-1), (i+1,j)
    b[gi] = acc;
  }
}

// Y = A X for ncols columns; A complex symmetric stored as 4 upper diagonals.
// One thread per row; the row's 4 stored coefficients (+3 mirrored) are read
// once and applied to every column (SpMM: one matrix read serves t columns).
// FD5 problems store S = D A: the row result is scaled by D^{-1} (fd5 = 1).
template <int NC>
__global__ void __launch_bounds__(256) k_spmm(long n, int nxp1, const cplx* __restrict__ dC,
                                              const cplx* __restrict__ dE, const cplx* __restrict__ dN,
                                              const cplx* __restrict__ dNE, const cplx* __restrict__ X,
                                              cplx* __restrict__ Y, int ncols, long ld, int fd5) {
  const long s = nxp1;
  const long nyl = n / nxp1 - 1;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < n; g += (long)gridDim.x * blockDim.x) {
    cplx c0 = __ldg(dC + g);
    cplx e = __ldg(dE + g);
    cplx nn = __ldg(dN + g);
    cplx ne = __ldg(dNE + g);
    cplx w = g >= 1 ? __ldg(dE + g - 1) : cmk(0, 0);
    cplx so = g >= s ? __ldg(dN + g - s) : cmk(0, 0);
    cplx sw = g >= s + 1 ? __ldg(dNE + g - s - 1) : cmk(0, 0);
    const int nc = NC > 0 ? NC : ncols;
    double dinv = 1.0;
    if (fd5) {
      const long i = g % s, j = g / s;
      dinv = ((i == 0 || i == s - 1) ? 2.0 : 1.0) * ((j == 0 || j == nyl) ? 2.0 : 1.0);
    }
#pragma unroll
    for (int col = 0; col < (NC > 0 ? NC : 8); ++col) {
      if (col >= nc) break;
      const cplx* x = X + col * ld;
      cplx acc = cmul(c0, __ldg(x + g));
      if (g + 1 < n) cfma(acc, e, __ldg(x + g + 1));
      if (g + s < n) cfma(acc, nn, __ldg(x + g + s));
      if (g + s + 1 < n) cfma(acc, ne, __ldg(x + g + s + 1));
      if (g >= 1) cfma(acc, w, __ldg(x + g - 1));
      if (g >= s) cfma(acc, so, __ldg(x + g - s));
      if (g >= s + 1) cfma(acc, sw, __ldg(x + g - s - 1));
      Y[col * ld + g] = fd5 ? cscale(acc, dinv) : acc;
    }
  }
}

int helm_spmm_dev(const helm_problem_s* p, const cplx* X, cplx* Y, int ncols, long ld, cudaStream_t st) {
  const int fd5 = p->disc == HELM_DISC_FD5 ? 1 : 0;
  int threads = 256;
  long blocks = (p->n + threads - 1) / threads;
  if (blocks > 148L * 16) blocks = 148L * 16;
  for (int c0 = 0; c0 < ncols; c0 += 8) {
    int nc = ncols - c0 < 8 ? ncols - c0 : 8;
    const cplx* x = X + (long)c0 * ld;
    cplx* y = Y + (long)c0 * ld;
    switch (nc) {
      case 1: k_spmm<1><<<blocks, threads, 0, st>>>(p->n, p->nx + 1, p->dC, p->dE, p->dN, p->dNE, x, y, nc, ld, fd5); break;
      case 2: k_spmm<2><<<blocks, threads, 0, st>>>(p->n, p->nx + 1, p->dC, p->dE, p->dN, p->dNE, x, y, nc, ld, fd5); break;
      case 4: k_spmm<4><<<blocks, threads, 0, st>>>(p->n, p->nx + 1, p->dC, p->dE, p->dN, p->dNE, x, y, nc, ld, fd5); break;
      default: k_spmm<0><<<blocks, threads, 0, st>>>(p->n, p->nx + 1, p->dC, p->dE, p->dN, p->dNE, x, y, nc, ld, fd5); break;
    }
    HELM_LAUNCH_CHECK();
  }
  return HELM_OK;
}

// ------------------------------------------------------------------ C ABI
static int assemble_impl(const helm_grid_desc* gd, int disc, void* stream, helm_problem_t* out);

extern "C" int helm_assemble(const helm_grid_desc* gd, void* stream, helm_problem_t* out) {
  return assemble_impl(gd, HELM_DISC_P1, stream, out);
}

extern "C" int helm_assemble_fd5(const helm_grid_desc* gd, void* stream, helm_problem_t* out) {
  if (gd && gd->c_nodes) {
    helm_set_error("helm_assemble_fd5: the five-point mode has constant k = omega (c_nodes must be NULL)");
    if (out) *out = nullptr;
    return HELM_EINVAL;
  }
  return assemble_impl(gd, HELM_DISC_FD5, stream, out);
}

static int assemble_impl(const helm_grid_desc* gd, int disc, void* stream, helm_problem_t* out) {
  if (!gd || !out) { helm_set_error("null argument"); return HELM_EINVAL; }
  *out = nullptr;
  if (gd->nx < 2 || gd->ny < 2 || !(gd->h > 0.0) || !(gd->omega > 0.0)) {
    helm_set_error("helm_assemble: need nx, ny >= 2, h > 0, omega > 0");
    return HELM_EINVAL;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    helm_set_error("no CUDA device (the library has no CPU fallback)");
    return HELM_ECUDA;
  }
  cudaStream_t st = (cudaStream_t)stream;
  static std::atomic<long> next_uid{1};
  helm_problem_s* p = new helm_problem_s();
  p->uid = next_uid++;
  p->disc = disc;
  p->nx = gd->nx; p->ny = gd->ny; p->h = gd->h; p->omega = gd->omega;
  p->n = (long)(gd->nx + 1) * (gd->ny + 1);
  size_t vb = sizeof(cplx) * p->n;
  cudaError_t e = cudaSuccess;
  p->c = nullptr; p->dC = p->dE = p->dN = p->dNE = nullptr;
  e = helm_dev_alloc((void**)&p->c, sizeof(double) * p->n);
  if (e == cudaSuccess) e = helm_dev_alloc((void**)&p->dC, vb);
  if (e == cudaSuccess) e = helm_dev_alloc((void**)&p->dE, vb);
  if (e == cudaSuccess) e = helm_dev_alloc((void**)&p->dN, vb);
  if (e == cudaSuccess) e = helm_dev_alloc((void**)&p->dNE, vb);
  if (e != cudaSuccess) {
    helm_set_error("helm_assemble: cudaMalloc: %s", cudaGetErrorString(e));
    helm_problem_destroy(p);
    return HELM_ENOMEM;
  }
  if (gd->c_nodes) {
    e = cudaMemcpyAsync(p->c, gd->c_nodes, sizeof(double) * p->n, cudaMemcpyDefault, st);
  } else {
    // c = 1 everywhere
    std::vector<double> ones(p->n, 1.0);
    e = cudaMemcpyAsync(p->c, ones.data(), sizeof(double) * p->n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (e != cudaSuccess) {
    helm_set_error("helm_assemble: copy c: %s", cudaGetErrorString(e));
    helm_problem_destroy(p);
    return HELM_ECUDA;
  }
  GridView g{p->nx, p->ny, p->h, p->omega, p->c};
  long blocks = (p->n + 255) / 256;
  if (blocks > 148L * 8) blocks = 148L * 8;
  if (disc == HELM_DISC_FD5)
    k_assemble_fd5<<<blocks, 256, 0, st>>>(p->nx, p->ny, p->h, p->omega, p->dC, p->dE, p->dN, p->dNE);
  else
    k_assemble<<<blocks, 256, 0, st>>>(g, p->dC, p->dE, p->dN, p->dNE);
  g_helm_launches++;
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    helm_set_error("helm_assemble: kernel: %s", cudaGetErrorString(e));
    helm_problem_destroy(p);
    return HELM_ECUDA;
  }
  *out = p;
  return HELM_OK;
}

extern "C" int helm_problem_info(helm_problem_t p, long* n, int* nx, int* ny) {
  if (!p) return HELM_EINVAL;
  if (n) *n = p->n;
  if (nx) *nx = p->nx;
  if (ny) *ny = p->ny;
  return HELM_OK;
}

extern "C" int helm_get_diagonals(helm_problem_t p, double* out, void* stream) {
  if (!p || !out) return HELM_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  size_t vb = sizeof(cplx) * p->n;
  char* o = reinterpret_cast<char*>(out);
  HELM_CUDA_TRY(cudaMemcpyAsync(o, p->dC, vb, cudaMemcpyDefault, st));
  HELM_CUDA_TRY(cudaMemcpyAsync(o + vb, p->dE, vb, cudaMemcpyDefault, st));
  HELM_CUDA_TRY(cudaMemcpyAsync(o + 2 * vb, p->dN, vb, cudaMemcpyDefault, st));
  HELM_CUDA_TRY(cudaMemcpyAsync(o + 3 * vb, p->dNE, vb, cudaMemcpyDefault, st));
  HELM_CUDA_TRY(cudaStreamSynchronize(st));
  return HELM_OK;
}

extern "C" int helm_load_vector(helm_problem_t p, const double* f, double* b, void* stream) {
  if (!p || !f || !b) { helm_set_error("helm_load_vector: null argument"); return HELM_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  size_t vb = sizeof(cplx) * p->n;
  Staged sf, sb;
  StageGuard gf(sf, st), gb(sb, st);
  HELM_TRY(helm_stage_in(f, vb, true, st, sf));
  HELM_TRY(helm_stage_in(b, vb, false, st, sb));
  long blocks = (p->n + 255) / 256;
  if (blocks > 148L * 8) blocks = 148L * 8;
  if (p->disc == HELM_DISC_FD5) {
    // five-point scheme: b = f at every node (the ghost-eliminated rows keep their source)
    HELM_CUDA_TRY(cudaMemcpyAsync(sb.dev, sf.dev, vb, cudaMemcpyDeviceToDevice, st));
  } else {
    k_load_vector<<<blocks, 256, 0, st>>>(p->nx, p->ny, p->h, (const cplx*)sf.dev, (cplx*)sb.dev);
    HELM_LAUNCH_CHECK();
  }
  helm_stage_free(sf, st);
  HELM_TRY(helm_stage_out(sb, st));
  return HELM_OK;
}

extern "C" int helm_spmv(helm_problem_t p, const double* X, double* Y, int ncols, void* stream) {
  if (!p || !X || !Y || ncols < 1) { helm_set_error("helm_spmv: bad argument"); return HELM_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  size_t vb = sizeof(cplx) * p->n * ncols;
  Staged sx, sy;
  StageGuard gx(sx, st), gy(sy, st);
  HELM_TRY(helm_stage_in(X, vb, true, st, sx));
  HELM_TRY(helm_stage_in(Y, vb, false, st, sy));
  HELM_TRY(helm_spmm_dev(p, (const cplx*)sx.dev, (cplx*)sy.dev, ncols, p->n, st));
  helm_stage_free(sx, st);
  HELM_TRY(helm_stage_out(sy, st));
  return HELM_OK;
}

extern "C" void helm_problem_destroy(helm_problem_t p) {
  if (!p) return;
  helm_problem_free_ws(p);
  helm_dev_free(p->c);
  helm_dev_free(p->dC);
  helm_dev_free(p->dE);
  helm_dev_free(p->dN);
  helm_dev_free(p->dNE);
  delete p;
}
