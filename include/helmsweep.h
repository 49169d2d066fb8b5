/*
 * helmsweep.h -- C ABI of the B200 (sm_100a) hot path of multipreconditioned
 * GMRES with directional double-sweep preconditioners for the 2D impedance
 * Helmholtz problem (Bootland & Rees, arXiv 2408.11929).
 *
 * Citations: P:Lnn = PAPER.md line nn (section / equation named), D1..D12 and
 * A1..A27 = SURVEY.md §8(c) definitions / readings (restated in DESIGN.md §3).
 *
 * Conventions (all entry points)
 *   - complex128 values are interleaved {re, im} doubles (cuDoubleComplex /
 *     double2 layout); passed here as `double*` pointing at 2*len doubles.
 *   - Node index g = j*(nx+1) + i, x fastest (D1).  Multi-column vectors are
 *     column-major with leading dimension `ld` (>= n) in complex elements.
 *   - Pointers marked [dev|host] may be device or host memory: the library
 *     detects host pointers (cudaPointerGetAttributes) and stages them
 *     through device buffers itself (this is the end-to-end path).  Pointers
 *     marked [dev] must be device memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Every call is asynchronous on `stream` unless stated otherwise.
 *   - The caller owns every vector buffer; the library owns the matrix and
 *     factor storage behind the handles (released by *_destroy).  Handles are
 *     immutable after setup, so concurrent applies on distinct outputs are safe.
 *   - Every call returns a status code (HELM_OK = 0) and never aborts; the
 *     message of the last failure is in helm_last_error().
 *   - There is no CPU fallback: without a CUDA device every compute call
 *     returns HELM_ECUDA.
 */
#ifndef HELMSWEEP_H
#define HELMSWEEP_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HELM_OK = 0,
  HELM_EINVAL = 1,      /* invalid argument (sizes, strips too thin, t out of range, tol) */
  HELM_EDIM = 2,        /* mismatched dimensions between handles */
  HELM_ESINGULAR = 3,   /* zero or non-finite (NaN / Inf) pivot while factoring a strip block */
  HELM_ECUDA = 4,       /* CUDA runtime error or no device */
  HELM_ENOMEM = 5,      /* device allocation failed */
  HELM_ENOCONV = 6,     /* maxit reached; x holds the last iterate */
  HELM_EEXHAUSTED = 7,  /* every new column of a block deflated (search space exhausted) */
  HELM_ENONFINITE = 8   /* a NaN / Inf reached the Krylov block (failure detection) */
};

typedef struct helm_problem_s* helm_problem_t;  /* device matrix (4 symmetric diagonals) + geometry + c */
typedef struct helm_sweep_s* helm_sweep_t;      /* device strip factors for one (axis, order, N, overlap) */

/* Grid and medium (D1, D3).  Omega = [0, nx h] x [0, ny h]. */
typedef struct {
  int nx, ny;            /* cells per axis (>= 2) */
  double h;              /* cell size */
  double omega;          /* angular frequency; k = omega / c */
  const double* c_nodes; /* [dev|host] (nx+1)(ny+1) nodal wave speed, NULL => c = 1 */
} helm_grid_desc;

/* helm_assemble -- the P1 matrix of Eq. 1a-1b on the "/" mesh (D2):
 *   A = -K + sum_T k_T^2 M_T + i sum_{e in dOmega} k_e B_e         (D4, A3)
 * k_T = omega / mean(c at the triangle's vertices), k_e = omega / mean(c at
 * the edge's ends) (D3, A5).  A is complex symmetric; it is stored as the 4
 * upper diagonals (centre, east, north, north-east), n complex each.
 * Errors: HELM_EINVAL (nx, ny < 2, h <= 0), HELM_ENOMEM, HELM_ECUDA. */
int helm_assemble(const helm_grid_desc* grid, void* stream, helm_problem_t* out);

/* helm_assemble_fd5 -- the paper's own discretisation (paper-calibration
 * mode): "the standard five-point finite difference
 * approximation on a regular Cartesian grid" (§4) of Eq. 1a-1b,
 *   A = Delta_h + k^2  (interior row (u_E + u_W + u_N + u_S - 4u)/h^2 + k^2 u),
 * impedance rows by ghost-point elimination of the centred normal derivative
 * through Eq. 1b (inward neighbour 2/h^2, + 2ik/h on the diagonal per boundary
 * line; reading DESIGN.md §3 FD5).  Constant k = omega: c_nodes must be NULL.
 * Stored as the complex-symmetric S = D A (D = 1/2 per boundary line the node
 * lies on), whose diagonals helm_get_diagonals returns (NE = 0); helm_spmv
 * applies A = D^{-1} S; helm_load_vector returns b = f; sweep_setup factors the
 * strip matrices D_s A_s (interface lines eliminated like boundary lines,
 * Eq. 4) and needs overlap >= 1.
 * Errors: HELM_EINVAL (c_nodes given, nx, ny < 2, h <= 0), HELM_ENOMEM, HELM_ECUDA. */
int helm_assemble_fd5(const helm_grid_desc* grid, void* stream, helm_problem_t* out);

/* n = (nx+1)(ny+1), nx, ny of a problem.  Host-only query. */
int helm_problem_info(helm_problem_t p, long* n, int* nx, int* ny);

/* Copy the 4 stored diagonals to out[4*n] (C, E, N, NE; entry g couples node g
 * to g, g+1, g+nx+1, g+nx+2).  [dev|host] out.  For parity tests. */
int helm_get_diagonals(helm_problem_t p, double* out, void* stream);

/* helm_load_vector -- b = M1 f (D5, A4): consistent unit-coefficient P1 mass
 * times the nodal complex source f.  [dev|host] f (n complex), b (n complex). */
int helm_load_vector(helm_problem_t p, const double* f, double* b, void* stream);

/* helm_spmv -- Y = A X for ncols columns (col-major, ld = n), with A the
 * matrix of helm_assemble: the "t matrix-vector products" of each MPGMRES
 * iteration (step 3 of D10).  [dev|host] X, Y (n x ncols complex).
 * 1 <= ncols <= 8.  Errors: HELM_EINVAL, HELM_ECUDA. */
int helm_spmv(helm_problem_t p, const double* X, double* Y, int ncols, void* stream);

/* sweep_setup -- build and factor one directional sweep preconditioner
 * (Eq. 2-4; strips D6, local matrices D7, transmission D8):
 *   axis       0 = x (strips are vertical slabs: LRL / RLR), 1 = y (BTB / TBT)
 *   order      0 = increasing (LRL, BTB), 1 = decreasing (RLR, TBT)
 *   n_strips   N >= 1; every strip needs >= max(2*overlap+1, 2) cells
 *   overlap    l >= 0 extra mesh lines per internal boundary (A11)
 *   is_double  1 = double sweep (2N-1 local solves), 0 = forward sweep only
 *   gather     0 = "recent" (P:L93 literal rule), 1 = "core" ownership (A16)
 *   n_segments P >= 1 cross-row segments per strip for the partitioned
 *              (separator) strip solve; 0 = choose automatically (the
 *              largest P <= 36 (<= 33 for strips wider than 36 nodes) whose
 *              segments have >= 8 cross rows: four
 *              directions of 36 segment CTAs fill a B200)
 * Each strip's local block-tridiagonal matrix is factored once on the device
 * (block-Thomas per segment plus the separator Schur complement).
 * Errors: HELM_EINVAL, HELM_ESINGULAR, HELM_ENOMEM, HELM_ECUDA.  Synchronous. */
int sweep_setup(helm_problem_t p, int axis, int order, int n_strips, int overlap,
                int is_double, int gather, int n_segments, void* stream,
                helm_sweep_t* out);

/* sweep_set_precision -- opt-in INEXACT separator solve (
 * "the subproblems can be solved to low accuracy without much deterioration",
 * P:L278): separator_bits = 32 makes the two-chain sweep kernel multiply the
 * separator right-hand side by a complex64 copy of the explicit
 * separator-inverse rows with FP32 products and accumulation (half the bytes
 * of that HBM-bound stage); 64 (default) restores the complex128 path.  The
 * preconditioner then differs from the exact strip solves by ~1e-6 relative
 * (the MPGMRES residual and x stay complex128); every other step is
 * unchanged.  Applies when every direction of a batch asked for it and the
 * two-chain kernel runs (strips <= 36 nodes, P > 1).  The complex64 copy is
 * made once per factor set (device memory: half of the rows').
 * Errors: HELM_EINVAL (bits not 32 / 64, or no separator rows), HELM_ENOMEM, HELM_ECUDA. */
int sweep_set_precision(helm_sweep_t s, int separator_bits);

/* Geometry / size report of a sweep handle (host-only query):
 *   info[0] n_strips, [1] n_c (cross rows), [2] w_max (nodes per block row),
 *   [3] n_segments, [4] local solves per apply, [5] factor bytes on device,
 *   [6] model bytes per apply (sum over solves of
 *       16*(2 n_c w^2 + 3 n_c w)), [7] axis, [8] order, [9] is_double. */
int sweep_info(helm_sweep_t s, long* info /* >= 10 */);

/* sweep_apply -- Z[:, d] = M_d^{-1} R[:, d] for the t directions dirs[0..t-1]
 * ("apply ... in parallel"), all batched in ONE persistent kernel launch.
 *   R   [dev|host] n x t col-major with leading dim ldr; ldr = 0 broadcasts one
 *       vector to all t directions (k = 1 and the t >= 3 sum rule).
 *   Z   [dev|host] n x t col-major, leading dim ldz (>= n).
 * All handles must belong to the same problem size.  1 <= t <= 8.  The t
 * directions run in one persistent launch when all their CTAs (n_segments
 * each, plus one) fit the SMs, else as consecutive half batches.
 * Errors: HELM_EINVAL, HELM_EDIM, HELM_ECUDA. */
int sweep_apply(const helm_sweep_t* dirs, int t, const double* R, long ldr,
                double* Z, long ldz, void* stream);

/* Solve statistics of mpgmres_solve. */
typedef struct {
  int iterations;        /* outer iterations k (each applies all t preconditioners, D11) */
  int converged;         /* projected rho_k <= tol */
  int flags;             /* bit0 maxit reached, bit1 search space exhausted */
  int deflations;        /* columns dropped by the 1e-10 rule (D10 step 5) */
  double proj_rel_res;   /* rho_k = ||beta e1 - H y|| / beta at exit */
  double true_rel_res;   /* ||b - A x|| / ||b|| recomputed */
  double solve_s;        /* wall seconds of the solve (host clock) */
  double sweep_ms;       /* device ms spent in sweep_apply launches (CUDA events) */
  double spmv_ms;        /* device ms in the SpMM launches */
  double orth_ms;        /* device ms in BCGS2 + block QR launches */
  long matvecs, prec_applies, inner_products;
  double* history;       /* optional host array of rho_k, capacity history_cap */
  int history_cap;
} mpgmres_stats;

/* mpgmres_solve -- selective MPGMRES with the paper's selection
 * rules (t = 2 cross rule, t >= 3 sum rule, k = 1 all on r0/||r0||),
 * block classical Gram-Schmidt with reorthogonalisation (BCGS2) and intra-
 * block CGS2 with the 1e-10 deflation rule (D10), projected least squares by
 * Householder QR on the host.  x0 = 0; stops when rho_k <= tol.
 *   b [dev|host] n complex; x [dev|host] n complex (output).
 * Host-synchronous (one small device->host copy per iteration).
 * One problem handle may be reused for solves with different t: its cached
 * workspace is sized in columns and for the largest t seen.
 * Errors: HELM_EINVAL (tol not in (0,1), t not in [1,8], maxit < 1),
 *         HELM_ENOCONV, HELM_EEXHAUSTED, HELM_ENONFINITE (NaN / Inf in the
 *         Gram diagonal, the BCGS2 coefficients or the new norms),
 *         HELM_ENOMEM, HELM_ECUDA. */
int mpgmres_solve(helm_problem_t p, const helm_sweep_t* dirs, int t,
                  const double* b, double* x, double tol, int maxit,
                  mpgmres_stats* stats, void* stream);

/* All-gather callback of the direction-parallel solve: every rank contributes
 * `bytes` from `send` (device memory, on `stream`) and receives all ranks'
 * contributions concatenated in rank order in `recv` (nranks * bytes; send ==
 * recv + rank * bytes, i.e. in place).  Returns 0 on success.  The caller
 * provides it (e.g. an NCCL all-gather over NVLink through torch.distributed);
 * the library itself holds no communicator. */
typedef int (*helm_allgather_fn)(void* ctx, const void* send, void* recv, long bytes, void* stream);

/* mpgmres_solve_dist -- the direction-parallel MPGMRES of SURVEY §8(e): the
 * t = nranks * t_local preconditioners are split over the ranks (one process
 * per GPU), rank r applying global directions r*t_local .. r*t_local+t_local-1
 * ("we can perform this part fully in parallel").  Per iteration each
 * rank sweeps its directions and forms its columns of W = A Z, then the new Z
 * and W columns are all-gathered (two callbacks); source selection, BCGS2 +
 * block QR and the host least squares run replicated and deterministic, so all
 * ranks hold the same x.  Every rank passes the same problem data, b, tol and
 * maxit; local_dirs are this rank's sweep handles.  nranks == 1 is
 * mpgmres_solve.  Errors: as mpgmres_solve, HELM_EINVAL for a bad rank /
 * missing callback, HELM_ECUDA if the callback fails. */
int mpgmres_solve_dist(helm_problem_t p, const helm_sweep_t* local_dirs, int t_local, int nranks, int rank,
                       helm_allgather_fn allgather, void* ctx, const double* b, double* x,
                       double tol, int maxit, mpgmres_stats* stats, void* stream);

void helm_problem_destroy(helm_problem_t p);
void sweep_destroy(helm_sweep_t s);
const char* helm_strerror(int code);
const char* helm_last_error(void);

/* Number of this library's kernel launches since load (host counter). */
long helm_kernel_launches(void);

/* Name of the sweep kernel the last sweep_apply / mpgmres_solve iteration of
 * this process launched ("k_sweep_dual", "k_sweep_fast", "k_sweep_apply"; ""
 * before the first apply).  Diagnostics: the choice depends on the strip
 * width, the segment count and the sweep_kernel knob. */
const char* helm_sweep_kernel_name(void);

/* helm_set_knob -- diagnostics / testing controls, process-wide, all 0 (the
 * product choice) by default; the library reads no environment variable.
 *   "sweep_kernel"     0 auto (two-chain k_sweep_dual where it applies),
 *                      2 start at the single-chain k_sweep_fast,
 *                      3 the general TMA-ring k_sweep_apply
 *   "general_reducer"  1: k_sweep_apply solves the separator system with its
 *                      reducer CTA instead of the explicit inverse rows
 *   "no_wide_xinv"     1: sweep_setup forms no explicit separator-inverse rows
 *                      for strips wider than 36 nodes
 *   "factor_generic"   1: sweep_setup uses the generic factorisation kernel
 *   "orth_unfused"     1: multi-launch BCGS2 instead of the fused k_orth
 *   "setup_timing"     1: sweep_setup prints its phase times to stderr
 *   "orth_prof"        1: k_orth prints phase clock stamps to stderr
 *   "setup_chunks"     n > 1: sweep_setup pipelines its strips in n chunks on forked streams (0 / 1: one pass)
 *   "sep_two_level"    1: sweep_setup also builds two-level separator panels (fine groups +
 *                      coarse Schur system, >= 8 separators) and k_sweep_dual uses them
 * Every knob selects a different, parity-tested kernel or schedule for the same
 * arithmetic.  Not synchronised with calls running on other host threads.
 * Errors: HELM_EINVAL (unknown name or value). */
int helm_set_knob(const char* name, int value);

#ifdef __cplusplus
}
#endif
#endif /* HELMSWEEP_H */
