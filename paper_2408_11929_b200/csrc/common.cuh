// common.cuh -- shared device/host helpers of the helmsweep library (sm_100a).
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/helmsweep.h"

typedef double2 cplx;

// ------------------------------------------------------------------ complex
__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
// Products with an explicit FMA contraction (the compiler otherwise picks which of
// the two products it fuses per call site, and that choice -- a last-bit
// difference -- moved with unrelated code changes; C4's wide strips amplify it to
// ~1e-10 against the oracle).  h_mul: an uncontracted product.
__host__ __device__ __forceinline__ double h_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cmk(fma(a.x, b.x, -h_mul(a.y, b.y)), fma(a.x, b.y, h_mul(a.y, b.x)));
}
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return cmk(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return cmk(a.x, -a.y); }
// acc += a * b
__host__ __device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__host__ __device__ __forceinline__ void cfmaconj(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__host__ __device__ __forceinline__ double cabs2(cplx a) { return fma(a.x, a.x, h_mul(a.y, a.y)); }
__host__ __device__ __forceinline__ cplx cinv(cplx a) {
  double d = 1.0 / cabs2(a);
  return cmk(a.x * d, -a.y * d);
}

// ------------------------------------------------------------------ knobs
// Diagnostics / testing controls set through helm_set_knob (helmsweep.h); all 0
// by default (= the product choice).  The library reads no environment variable.
enum HelmKnob {
  KNOB_SWEEP_KERNEL = 0,    // 0 auto, 2 single-chain k_sweep_fast first, 3 general k_sweep_apply
  KNOB_GENERAL_REDUCER,     // 1: the general kernel solves the separators with its reducer CTA
  KNOB_NO_WIDE_XINV,        // 1: no explicit separator-inverse rows for w > 36
  KNOB_FACTOR_GENERIC,      // 1: generic shared-memory factorisation (no packed / bottom-up factors)
  KNOB_ORTH_UNFUSED,        // 1: multi-launch BCGS2 instead of the fused cooperative k_orth
  KNOB_SETUP_TIMING,        // 1: sweep_setup prints its phase times to stderr
  KNOB_ORTH_PROF,           // 1: k_orth phase clock stamps to stderr
  KNOB_SETUP_CHUNKS,        // 0 auto, n: sweep_setup pipelines its strips in n chunks (1 = one pass)
  KNOB_SEP_TWO_LEVEL,       // 1: sweep_setup builds the two-level separator panels and k_sweep_dual uses them
  KNOB_COUNT
};
int helm_knob(int id);

// ------------------------------------------------------------------ errors
void helm_set_error(const char* fmt, ...);
extern std::atomic<long> g_helm_launches;   // host counter of this library's launches (thread-safe)

#define HELM_CUDA_TRY(expr)                                                       \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      helm_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return (_e == cudaErrorMemoryAllocation) ? HELM_ENOMEM : HELM_ECUDA;        \
    }                                                                             \
  } while (0)

#define HELM_LAUNCH_CHECK()                                                       \
  do {                                                                            \
    g_helm_launches++;                                                            \
    cudaError_t _e = cudaGetLastError();                                          \
    if (_e != cudaSuccess) {                                                      \
      helm_set_error("%s:%d kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return HELM_ECUDA;                                                          \
    }                                                                             \
  } while (0)

#define HELM_TRY(expr)            \
  do {                            \
    int _rc = (expr);             \
    if (_rc != HELM_OK) return _rc; \
  } while (0)

// ------------------------------------------------------------------ device memory
// Handle and workspace memory comes from the device's default stream-ordered
// pool with an unlimited release threshold: freed blocks stay in the pool, so
// the per-problem / per-sweep buffers of repeated solves are reused instead of
// being mapped and unmapped by cudaMalloc / cudaFree every time.
cudaError_t helm_dev_alloc(void** p, size_t bytes);
void helm_dev_free(void* p);

// ------------------------------------------------------------------ padded packed triangles
// A complex-symmetric w x w block is stored as its upper triangle, row r holding
// columns r..w-1 from entry pk_start(r, w).  Row starts are padded so that
// pk_start(r) = 2r (mod 8), i.e. (pk_start(r) - r) = r (mod 8): in the sweep
// kernels a quarter-warp reads one column k of 8 consecutive rows; for k >= r the
// eight 16-byte entries pk_start(r) + k - r then fall into 8 different bank groups,
// for k < r they are 8 consecutive entries of row k -- both conflict-free.
// Average padding 3.5 entries per row.
__host__ __device__ inline int pk_start(int r, int w) {
  // x_{i+1} = x_i + (w - i) + pad_i with x_i = 2i (mod 8), so pad_i = (i + 2 - w) mod 8;
  // the pads repeat with period 8 (sum 28 per period): O(1) instead of a loop over
  // the rows (the loop was 11% of the factorisation kernel's stall samples)
  const int c = ((2 - w) % 8 + 8) % 8;
  int pad = 28 * (r >> 3);
  for (int i = r & ~7; i < r; ++i) pad += (i + c) & 7;
  return r * w - r * (r - 1) / 2 + pad;
}
// entries per padded block (a multiple of 8, so blocks stay 128-byte aligned)
__host__ __device__ inline int pk_size(int w) { return ((pk_start(w - 1, w) + 1) + 7) / 8 * 8; }
// Row stride of the explicit separator-inverse rows (k_reduced_inverse, sweep
// kernels): K w entries padded to a multiple of 8 (128-byte aligned rows, so the
// separator mat-vec's warp loads are whole cache lines for every P).
__host__ __device__ inline long x_ld(int K, int w) { return ((long)K * w + 7) / 8 * 8; }
// index of entry (r, k) of the symmetric block
__host__ __device__ inline int pk_index(int r, int k, int w) {
  return k >= r ? pk_start(r, w) + (k - r) : pk_start(k, w) + (r - k);
}

// ------------------------------------------------------------------ discretisations
enum { HELM_DISC_P1 = 0, HELM_DISC_FD5 = 1 };
// Transmission-correction stencil (D8) per interface node: kTcW coefficients on
// the source solution at (c-1, qi), (c, qi), (c+1, qi), (c, qo), (c+dd, qo),
// (c, qin): interface line qi, outer line qo, inner line qin of the destination
// strip (the last one is zero for P1; FD5's centred normal derivative uses it).
constexpr int kTcW = 6;
// FD5 row scaling of a strip (or of the global) matrix: S = D A is complex
// symmetric with d = 1/2 on each boundary line (physical or interface) the node
// lies on (ghost rows couple inward with 2/h^2, the inward rows back with 1/h^2).
__host__ __device__ __forceinline__ double fd5_d(int q, int w, int c, int nc) {
  return ((q == 0 || q == w - 1) ? 0.5 : 1.0) * ((c == 0 || c == nc - 1) ? 0.5 : 1.0);
}

// ------------------------------------------------------------------ handles
struct helm_problem_s {
  int nx, ny;
  long n;
  double h, omega;
  double* c;      // [dev] nodal wave speed (n)
  cplx* dC;       // [dev] diagonals: centre, east (g,g+1), north (g,g+nx+1), north-east (g,g+nx+2)
  cplx* dE;
  cplx* dN;
  cplx* dNE;
  int disc = 0;        // HELM_DISC_P1 (D4) or HELM_DISC_FD5 (five-point, the paper's own scheme)
  void* ws = nullptr;  // cached MPGMRES workspace (krylov.cu), grown on demand
  long uid = 0;        // unique id (factor-set sharing key; addresses can be reused)
};
void helm_problem_free_ws(helm_problem_s* p);

// One sweep preconditioner (one direction): strips + factors, all on device.
struct helm_sweep_s {
  helm_problem_s* prob;
  int axis, order, N, overlap, is_double, gather;
  int disc;        // discretisation of the problem (HELM_DISC_P1 / HELM_DISC_FD5)
  int nc;          // cross rows per strip (ny+1 for axis 0, nx+1 for axis 1)
  int wmax;        // max nodes per block row over strips
  int P;           // segments per strip
  // host copies of geometry
  std::vector<int> a, b, w;        // per strip: first/last along line, width
  std::vector<int> own_lo, own_hi; // per strip: gathered position range (core/recent)
  std::vector<int> seg_lo, seg_hi; // per segment: cross-row range (same for all strips)
  // device geometry (int arrays, N each)
  int* d_a; int* d_w; int* d_own_lo; int* d_own_hi;
  int* d_seg_lo; int* d_seg_hi;    // P each
  // strip bands (local matrix A_s, D7): per strip s, per row c, per position q:
  //   dg[s][c][q] = diagonal, al[s][c][q] = along coupling (q,q+1),
  //   cr[s][c][q] = cross coupling (c,q)-(c+1,q), ne[s][c][q] = (c,q)-(c+1,q+1)
  //   stored with stride wmax per row and nc*wmax per strip.
  cplx* d_dg; cplx* d_al; cplx* d_cr; cplx* d_ne;
  // transmission-correction coefficients (D8): [s][side][c][5]
  cplx* d_tc;
  // factors: per strip s, row c: Sinv (w_s x w_s row-major) at fac_off[s] + c*w_s^2
  cplx* d_fac; std::vector<long> fac_off; long* d_fac_off;
  // reduced (separator) system: per strip s, separator k (0..P-2): Rinv, G, F
  cplx* d_red; std::vector<long> red_off; long* d_red_off;
  // explicit rows of the separator inverse (w <= 36 only): per strip, separator k:
  // w x (K w) row-major at xinv_off[s] + k * w * K * w
  cplx* d_xinv = nullptr; std::vector<long> xinv_off; long* d_xinv_off = nullptr;
  long xinv_elems = 0;
  // opt-in inexact separator solve (sweep_set_precision): complex64 copy of the
  // explicit separator-inverse rows, shared by the handles of one factor set
  float2* d_xinv32 = nullptr;
  int sep_fp32 = 0;
  // two-chain kernel (sweep_dual.cu): the top-down inverses Sinv_c (d_facp) and the
  // bottom-up inverses S'^{-1}_c (d_fac2) of every segment row, complex symmetric,
  // stored as packed upper triangles (row r holds columns r..w-1), w(w+1)/2 per
  // row, at pfac_off[s] + c * w(w+1)/2
  cplx* d_facp = nullptr;
  cplx* d_fac2 = nullptr;
  std::vector<long> pfac_off; long* d_pfac_off = nullptr;
  // two-level separator solve (k_sweep_dual): per strip s, separator
  // k, two row panels (w rows of ld1, then w rows of ld2 complex) at
  // sep2_off[s] + k * w_s * (ld1 + ld2); the plan (group / coarse structure) is
  // the same for every strip.  NULL unless the sep_two_level knob is set (and K >= 8, w <= 36).
  cplx* d_sep2 = nullptr;
  std::vector<long> sep2_off; long* d_sep2_off = nullptr;
  int* d_sep2_plan = nullptr;
  int sep2_M = 0, sep2_ld1 = 0, sep2_ld2 = 0;
  // the band/factor arrays above are shared by every handle with the same
  // (problem, axis, N, overlap, P) -- e.g. LRL and RLR -- through this record
  struct SharedFactors* shared = nullptr;
  long factor_bytes;
};

// ------------------------------------------------------------------ staging
// Ensure `ptr` is device-accessible; for host pointers allocate a device
// buffer (and copy in when `copy_in`).  `dev` receives the device pointer.
struct Staged {
  void* dev = nullptr;
  const void* host = nullptr;
  size_t bytes = 0;
  bool owned = false;
};
int helm_stage_in(const void* ptr, size_t bytes, bool copy_in, cudaStream_t st, Staged& out);
int helm_stage_out(Staged& s, cudaStream_t st);  // copy back to host if staged, then free
void helm_stage_free(Staged& s, cudaStream_t st);
bool helm_is_device_ptr(const void* p);
// frees a staging buffer on every return path (helm_stage_free is idempotent)
struct StageGuard {
  Staged& s;
  cudaStream_t st;
  StageGuard(Staged& s_, cudaStream_t st_) : s(s_), st(st_) {}
  ~StageGuard() { helm_stage_free(s, st); }
};
