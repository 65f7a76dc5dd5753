/*
 * jfftb200.h -- C ABI of libjfftb200.so, the B200-native (sm_100a) J-FFT PCG
 * hot path (arXiv 2508.02613).
 *
 * The reference (/root/reference/pkg/src/jfft) is pure Python on NumPy and has
 * no FFI of its own; its "operator API" is the set of module-level functions
 * re-exported by jfft/__init__.py:5-21.  Each entry point below replaces one
 * of those functions (cited per declaration).  The Python host layer
 * paper_2508_02613_b200/ binds this ABI with ctypes and keeps the reference's
 * call signatures; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Plain C types only: pointers + sizes, no torch/CUDA types in signatures
 *    (streams are passed as void*).
 *  - Every function returns an int status (JFFTB_OK = 0).  On failure a
 *    thread-local message is available from jfftb_last_error().  No C++
 *    exception crosses the boundary.
 *  - Array arguments are float64, C order, last index contiguous:
 *      scalar (pixel) field  n0 x ... x n_{d-1}
 *      vector field          d x n0 x ... x n_{d-1}
 *      quadrature field      M x d! x n0 x ...   (M = 3 in 2-D, 6 in 3-D)
 *      half spectrum         d x n0 x ... x (n_{d-1}/2+1) complex (re,im interleaved)
 *  - `where` selects the memory space of every array argument of that call:
 *    JFFTB_HOST (pageable or pinned host memory; the call copies and
 *    synchronises) or JFFTB_DEVICE (device pointers on the grid's device;
 *    the call is asynchronous on the grid's stream unless stated).
 *  - Handles are not thread-safe; use one grid handle per calling thread.
 */
#ifndef JFFTB200_H
#define JFFTB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mapped by the host layer to the reference's exceptions) */
#define JFFTB_OK          0  /* success */
#define JFFTB_EINVAL      1  /* invalid argument         -> ValueError       */
#define JFFTB_ENONFINITE  2  /* NaN/Inf in the recurrence -> SolverAbortError */
#define JFFTB_ECURVATURE  3  /* curvature <= 0            -> SolverAbortError */
#define JFFTB_ECUDA       4  /* CUDA / cuFFT failure      -> RuntimeError     */

#define JFFTB_HOST   0
#define JFFTB_DEVICE 1

/* preconditioner kinds, preconditioners.py:22 PRECONDITIONER_KINDS order */
#define JFFTB_PC_NONE          0
#define JFFTB_PC_GREEN         1
#define JFFTB_PC_JACOBI        2
#define JFFTB_PC_GREEN_JACOBI  3

/* SolveReport.terminated, solver.py:32-33 */
#define JFFTB_CONVERGED      0
#define JFFTB_ITERATION_CAP  1

typedef struct jfftb_grid   jfftb_grid;    /* grid.py:34 Grid (+ device, stream, FFT plans) */
typedef struct jfftb_op     jfftb_op;      /* operators.py:15 SystemOperator               */
typedef struct jfftb_green  jfftb_green;   /* preconditioners.py:29 GreenOperator          */
typedef struct jfftb_jacobi jfftb_jacobi;  /* preconditioners.py:38 JacobiDiagonal         */

/* ---- library ---------------------------------------------------------- */
const char* jfftb_last_error(void);
int jfftb_version(void);                   /* 100 * major + minor */
/* number of kernel launches issued by this thread since the last reset */
int64_t jfftb_launch_count(int reset);

/* ---- grid / context (grid.py:34-96 make_grid) -------------------------- */
/* d in {2,3}; n[d] nodes per axis (>= 2); lengths[d] > 0; CUDA device id. */
int jfftb_grid_create(int d, const int64_t* n, const double* lengths, int device,
                      jfftb_grid** out);
int jfftb_grid_destroy(jfftb_grid* g);
/* run all subsequent work of this grid (and its ops/greens/jacobis) on
 * `stream` (a cudaStream_t; cudaStreamLegacy = (void*)1 for the legacy
 * default stream); NULL selects the grid's own (non-blocking) stream. */
int jfftb_grid_set_stream(jfftb_grid* g, void* stream);
int jfftb_grid_synchronize(jfftb_grid* g);

/* ---- load cases (topopt.py:98-196 consumers of pcg) -----
 * `nload` (1..6) solutions u (nload vector fields back to back, `where`)
 * with macroscopic strains ebar (nload Mandel vectors, host).  Total strains
 * eps_g = ebar_g + B u_g are paired per voxel,
 *   P_gc(x) = sum_t eps_c^T C0 eps_g                (_strain_pairings)
 * and sigma_out (nload x nload, host) = (w/|Y|) sum_x rho P_gc  (_stress_matrix).
 * If field_out (N, `where`) is given, it receives sum_gc weights_gc P_gc(x)
 * (weights: nload x nload host; _stress_gradient before its scale). */
int jfftb_load_pairings(jfftb_op* op, int nload, const double* u, const double* ebar,
                        const double* weights, double* sigma_out, double* field_out,
                        int where);

/* ---- input generators (microstructures.py:73-115) ------
 * Scalar (pixel) fields of the grid, in place; `where` as above.  Host
 * arrays are copied to the device, processed and copied back. */
/* `passes` periodic passes of the separable binomial filter, one [1 2 1]/4
 * sweep per axis (axis 0 first): gaussian_filter, microstructures.py:73-82,
 * bit-identical to its NumPy rounding order (d-generic) */
int jfftb_binomial_filter(jfftb_grid* g, double* field, int passes, int where);
/* minimum and maximum of a field -> minmax2[0..1] (host) */
int jfftb_field_minmax(jfftb_grid* g, const double* field, double* minmax2, int where);
/* affine map onto [1/chi, 1], chi = inf -> [0, 1] (rescale_contrast,
 * microstructures.py:104-115; same operation order); EINVAL for chi < 1 or a
 * constant field */
int jfftb_rescale_contrast(jfftb_grid* g, double* field, double chi, int where);
/* 1 where v >= 0.5, else 1/chi (threshold, microstructures.py:94-101) */
int jfftb_threshold(jfftb_grid* g, double* field, double chi, int where);
/* BASELINE config-5 projection: v <- tanh(beta (v - 1/2)), min-max to
 * [0, 1], E = emin + v^3 */
int jfftb_simp_projection(jfftb_grid* g, double* field, double beta, double emin, int where);
/* field file layout (grid.py:225-295 save_field / load_field): convert
 * `planes` consecutive planes between the file's "x1-fastest" order (Fortran
 * order of the n0 x ... x n_{d-1} array) and C order: to_c = 1 file -> C,
 * 0 C -> file.  Not in place. */
int jfftb_field_layout(jfftb_grid* g, const double* src, double* dst, int planes, int to_c,
                       int where);

/* ---- FFT contract (grid.py:200-215 fft_forward / fft_inverse) ---------- */
int jfftb_fft_forward(jfftb_grid* g, const double* u, double* spec, int where);
int jfftb_fft_inverse(jfftb_grid* g, const double* spec, double* u, int where);

/* ---- system operator (operators.py:38-101) ----------------------------- */
/* make_operator (operators.py:38): density rho >= 0 (EINVAL otherwise),
 * isotropic material (material.py:25) lambda0, mu0. */
int jfftb_op_create(jfftb_grid* g, const double* rho, int where, double lambda0,
                    double mu0, jfftb_op** out);
int jfftb_op_destroy(jfftb_op* op);
/* apply_system (operators.py:51): out = K(rho) u */
int jfftb_apply_system(jfftb_op* op, const double* u, double* out, int where);
/* assemble_rhs (operators.py:61): out = -B^T W rho C0 E; eps_bar is a host
 * Mandel vector (3 or 6 entries, finite). */
int jfftb_assemble_rhs(jfftb_op* op, const double* eps_bar, double* out, int where);
/* total_strain (operators.py:79): quadrature field E + B u */
int jfftb_total_strain(jfftb_op* op, const double* u, const double* eps_bar,
                       double* out, int where);
/* residual_force (operators.py:86): -B^T W sigma(rho, E + B u) */
int jfftb_residual_force(jfftb_op* op, const double* u, const double* eps_bar,
                         double* out, int where);
/* homogenized_stress (operators.py:98): sigma_out (host, 3 or 6 entries) */
int jfftb_homogenized_stress(jfftb_op* op, const double* u, const double* eps_bar,
                             double* sigma_out, int where);

/* ---- Green operator (preconditioners.py:50-94) ------------------------- */
/* assemble_green (preconditioners.py:50): impulse responses of K_ref ->
 * spectrum -> Hermitised per-frequency pseudo-inverse (cutoff 1e-12 lambda_max),
 * zero-frequency block = 0.  EINVAL if C_ref is not positive definite. */
int jfftb_green_create(jfftb_grid* g, double lambda_ref, double mu_ref,
                       jfftb_green** out);
int jfftb_green_destroy(jfftb_green* green);
/* GreenOperator.blocks: host array (n0, ..., n_{d-1}/2+1, d, d) complex */
int jfftb_green_export_blocks(jfftb_green* green, double* out);
/* apply_green (preconditioners.py:83) */
int jfftb_apply_green(jfftb_green* green, const double* r, double* out, int where);

/* ---- Jacobi diagonal (preconditioners.py:97-136) ----------------------- */
/* assemble_jacobi (preconditioners.py:97): d * 2^d comb probes of K;
 * EINVAL for odd n or a negative / non-finite probed diagonal. */
int jfftb_jacobi_create(jfftb_op* op, jfftb_jacobi** out);
int jfftb_jacobi_destroy(jfftb_jacobi* jac);
/* JacobiDiagonal(grid, inv_sqrt) built by the caller (preconditioners.py:38-47
 * is a plain container; the reference's tests construct it directly) */
int jfftb_jacobi_from_array(jfftb_grid* g, const double* inv_sqrt, int where, jfftb_jacobi** out);
/* JacobiDiagonal.inv_sqrt (vector field layout) */
int jfftb_jacobi_export(jfftb_jacobi* jac, double* out, int where);

/* Preconditioner.apply (preconditioners.py:156-163) for every kind;
 * kind = JFFTB_PC_*; green / jac may be NULL when the kind does not use them
 * (apply_jacobi_half is exposed as kind = -1). */
int jfftb_apply_precond(int kind, jfftb_green* green, jfftb_jacobi* jac,
                        const double* r, double* out, int where);

/* ---- PCG (solver.py:64-140) -------------------------------------------- */
/* pcg(op, rhs, preconditioner, green, eta, max_iter).  `green_pc` is the
 * preconditioner's Green operator (kinds green / green-jacobi), `jac` its
 * Jacobi diagonal (jacobi / green-jacobi), `green_term` the Green operator of
 * the termination functional <r, G r>.  Outputs: x_out (solution, mean
 * subtracted, in `where` space), history_out (HOST, max_iter + 1 doubles;
 * entries 0..iterations valid), iterations, terminated (JFFTB_CONVERGED /
 * JFFTB_ITERATION_CAP), wall_s (host wall time of the call).  Returns
 * JFFTB_ENONFINITE / JFFTB_ECURVATURE like SolverAbortError. */
int jfftb_pcg(jfftb_op* op, int kind, jfftb_green* green_pc, jfftb_jacobi* jac,
              jfftb_green* green_term, const double* rhs, int where, double eta,
              int max_iter, double* x_out, double* history_out, int* iterations,
              int* terminated, double* wall_s);

/* pcg over nrhs right-hand sides at once (the load cases of
 * topopt.py:98-127 share one operator and preconditioner): rhs / x_out hold
 * nrhs vector fields back to back, history_out nrhs x (max_iter + 1),
 * iterations / terminated nrhs entries.  Every stage is one launch for all
 * solves (a grid dimension per right-hand side, a device PCG state each), so
 * rho, D^-1/2 and the Green planes are read once per stage for all of them;
 * each solve stops on its own test (solver.py semantics per solve).  Fused
 * 3-D grids, kinds green / green-jacobi. */
int jfftb_pcg_batch(jfftb_op* op, int kind, jfftb_green* green_pc, jfftb_jacobi* jac,
                    jfftb_green* green_term, int nrhs, const double* rhs, int where, double eta,
                    int max_iter, double* x_out, double* history_out, int* iterations,
                    int* terminated, double* wall_s);

/* ---- device-side stage profile (no reference counterpart; SolveReport's
 * wall_time, solver.py:88,139, is the reference's only timing) ----------- */
#define JFFTB_N_STAGES 8  /* stencil, alpha, update, fft_fwd, spectral,
                             finalize, fft_inv, pupdate */
/* reset and enable: CUDA events are recorded between the stages of every
 * PCG iteration of this grid, on the grid's stream */
int jfftb_profile_start(jfftb_grid* g);
/* stage_ms[JFFTB_N_STAGES] summed over the iterations completed since start
 * (iterations that ran past convergence are not counted); stop != 0 disables */
int jfftb_profile_read(jfftb_grid* g, double* stage_ms, int64_t* iterations, int stop);

/* ---- distributed 3-D solves (replaces the loop of
 * solver.py:113-136 and the FFT solve of preconditioners.py:83-94 on
 * slab-decomposed grids) --------------------------------------------------
 * Real space is split into P slabs of L1 = n1 / P rows along axis 1 (rank r
 * owns rows [r L1, (r+1) L1)); spectra into P slabs of axis-0 frequency rows.
 * A communicator is either NCCL (one process per GPU; rank 0 makes the
 * 128-byte unique id with jfftb_comm_unique_id and the caller broadcasts it)
 * or a loopback that emulates all P ranks in this process on one device
 * (ranks run one after the other; transfers are device copies).  Every
 * per-rank array argument below holds the LOCAL ranks' slabs back to back:
 * one slab (n0 x L1 x n2 scalars, 3 x n0 x L1 x n2 vectors) for NCCL, P for
 * the loopback. */
typedef struct jfftb_comm jfftb_comm;
typedef struct jfftb_dist jfftb_dist;
int jfftb_comm_unique_id(char* id128);
int jfftb_comm_create_nccl(const char* id128, int rank, int world, int device, jfftb_comm** out);
int jfftb_comm_create_local(int world, int device, jfftb_comm** out);
int jfftb_comm_destroy(jfftb_comm* comm);
/* make_operator + assemble_green + build_preconditioner on the slabs:
 * power-of-two n (16..2048), n1 / P >= 16, (n0 / 2) % P == 0; kind is
 * JFFTB_PC_GREEN or JFFTB_PC_GREEN_JACOBI; the Green operator (reference
 * material lambda_ref, mu_ref) serves the preconditioner and the
 * termination functional.  rho: the local density slabs (`where`). */
int jfftb_dist_create(jfftb_comm* comm, const int64_t* n, const double* lengths, const double* rho,
                      int where, double lambda0, double mu0, double lambda_ref, double mu_ref,
                      int kind, jfftb_dist** out);
int jfftb_dist_destroy(jfftb_dist* dist);
/* assemble_rhs (operators.py:61) into the local vector slabs */
int jfftb_dist_assemble_rhs(jfftb_dist* dist, const double* eps_bar, double* out, int where);
/* JacobiDiagonal.inv_sqrt of the local slabs (green-jacobi) */
int jfftb_dist_jacobi_export(jfftb_dist* dist, double* out, int where);
/* pcg (solver.py:64-140): rhs / x_out local vector slabs; history_out (host,
 * max_iter + 1) identical on every rank; same status codes as jfftb_pcg */
int jfftb_dist_pcg(jfftb_dist* dist, const double* rhs, int where, double eta, int max_iter,
                   double* x_out, double* history_out, int* iterations, int* terminated,
                   double* wall_s);
/* info8: world, L1, local ranks, first local rank, its k0lo, its k0 count,
 * nodes per slab, loopback flag */
int jfftb_dist_info(jfftb_dist* dist, int64_t* info8);

/* ---- diagnostics (tests only) ------------------------------------------ */
/* Run the fused Green(-Jacobi) application up to pass `upto` (1 axis-0 R2C,
 * 2 axis-1 FFT, 3 last-axis FFT + block solve + iFFT, 4 axis-1 iFFT,
 * 5 axis-0 C2R) on host input r; out receives the intermediate spectrum
 * (d x (n0/2+1) x n1 [x n2] complex) or, for upto = 5, the result.
 * EINVAL on grids without the fused path (non power-of-two, n < 16). */
int jfftb_debug_fused_apply(jfftb_green* green, jfftb_jacobi* jac, int upto, const double* r,
                            double* out);

#ifdef __cplusplus
}
#endif
#endif /* JFFTB200_H */
