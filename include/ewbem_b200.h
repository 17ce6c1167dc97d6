/*
 * ewbem_b200 — C ABI of the B200-native (sm_100a, FP64) per-frequency
 * elastodynamic BEM solve.  Drop-in boundary for the hot path of the CPU
 * reference `ewbem` 0.1.0 (arXiv 1212.3032), whose Python seams are listed
 * next to each entry point (file:line under /root/reference/pkg/src/ewbem).
 *
 * Conventions
 *   - Plain pointers and sizes only.  `void* stream` is a cudaStream_t.
 *   - Complex data is complex128 interleaved (re, im) — the memory layout of
 *     numpy.complex128 / torch.complex128.  Matrices are row-major (C order),
 *     DOF index = 3 * element + component (assembly.py:78-80).
 *   - Pointers named *_dev are device memory owned by the caller; the context
 *     owns only the per-mesh tables it uploads.  Host pointers are *_host.
 *   - Every call returns EWB_OK (0) or an error code; ewb_last_error() gives
 *     a thread-local message.  Calls are asynchronous on `stream` unless the
 *     comment says "synchronises".
 *   - A context is not thread-safe; use one per host thread.
 */
#ifndef EWBEM_B200_H
#define EWBEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EWB_ABI_VERSION 6

enum ewb_status {
  EWB_OK = 0,
  EWB_ERR_INVALID = 1,   /* bad argument: Python side raises ValueError   */
  EWB_ERR_CUDA = 2,      /* CUDA runtime error                             */
  EWB_ERR_NONFINITE = 3  /* non-finite entry assembled (FloatingPointError) */
};

enum ewb_window { EWB_WIN_RECTANGULAR = 0, EWB_WIN_HANNING = 1, EWB_WIN_BLACKMAN = 2 };

typedef struct ewb_ctx ewb_ctx;

/* result record of ewb_gmres (device memory, 32 bytes) — SolveStats, linsolve.py:28-48 */
typedef struct ewb_gmres_result {
  int32_t iterations;
  int32_t n_hist;      /* entries written to the residual history */
  int32_t converged;
  int32_t matvecs;    /* passes over A: iterations + true residuals + r0 */
  double init_residual;
  double final_residual;
} ewb_gmres_result;

/* head of the operator-GMRES state (ewb_opgmres_*), at the start of its
 * workspace; fields as SolveStats (linsolve.py:28-48) plus the gates */
typedef struct ewb_op_head {
  int32_t in_cycle;     /* gate: the next operator application is A P^{-1} v_j */
  int32_t lit_pending;  /* gate: the next operator application is A x          */
  int32_t done, converged;
  int32_t iterations, j, m, used;
  int32_t cycle_open, n_hist, applications, pad;
  double norm_b, rnorm, residual, init_residual, final_residual;
} ewb_op_head;

typedef struct ewb_sem_result {
  int32_t kept;        /* history columns used after the rank filter */
  int32_t fallback;    /* 1: newest column returned unchanged        */
} ewb_sem_result;

int ewb_abi_version(void);
const char* ewb_last_error(void);

/* Number of kernels this library has launched since load (all entry points);
 * the benchmark reports the delta across its timed region. */
int64_t ewb_launch_count(void);

/* Per-mesh context: replaces Assembler.__init__ + _prepare_geometry +
 * static_offdiag_rowsums (assembly.py:112-216).  Uploads the element
 * geometry (derived exactly as mesh.py:88-106), classifies every element
 * pair into far / mid / near tiers on the GPU with the reference's exact
 * rounding (assembly.py:132-136, quadrature.py:223-228), grades near pairs
 * (quadrature.py:230-235), builds the 384-point self rules
 * (quadrature.py:135-185) and runs the static pass (assembly.py:193-216).
 * Synchronises.
 *   centroids/normals_host: (n_e,3); areas/diameters_host: (n_e,);
 *   corners_host: (n_e,3,3) vertex coordinates of each element;
 *   gl8_host: 8 Gauss-Legendre nodes then 8 weights; gl16_host likewise (32);
 *   rules_host: concatenated [bary (Q,3), weights (Q,)] tables of 6 rules in
 *   the order gauss3, gauss7, gauss7-sub1..sub4 (quadrature.py:63-132);
 *   rule_off_host[7]: offsets (in doubles) of each table, rule_q_host[7]: Q. */
int ewb_ctx_create(const double* centroids_host, const double* normals_host,
                   const double* areas_host, const double* diameters_host,
                   const double* corners_host, int64_t n_elements, double lam, double mu,
                   double rho, const double* gl8_host, const double* gl16_host,
                   const double* rules_host, const int32_t* rule_off_host,
                   const int32_t* rule_q_host, void* stream, ewb_ctx** out);
int ewb_ctx_destroy(ewb_ctx* ctx);

/* Exterior-problem diagonal (NOT a reference mode, parity
 * unpinned): on != 0 adds +I to every T diagonal block (c + PV int T = I, an
 * unbounded medium) instead of the reference's interior identity
 * (assembly.py:243-246).  Default off. */
int ewb_ctx_set_exterior(ewb_ctx* ctx, int32_t on, void* stream);

/* counts_host[8] = n_e, far pairs, mid pairs, near pairs, near L1..L4. */
int ewb_ctx_counts(const ewb_ctx* ctx, int64_t* counts_host);

/* The context's pair tables (Assembler._prepare_geometry's buckets,
 * assembly.py:132-161) copied to host buffers (each nullable), rows sorted:
 * near_ptr/mid_ptr (n_e+1) CSR row pointers, near_j/near_lvl (n_near) column
 * and subdivision level 1..4 of each near pair, mid_j (n_mid) column of each
 * mid (gauss7) pair.  Every other off-diagonal pair is far (gauss3).
 * Synchronises. */
int ewb_ctx_pair_lists(const ewb_ctx* ctx, int32_t* near_ptr_host, int32_t* near_j_host,
                       int32_t* near_lvl_host, int32_t* mid_ptr_host, int32_t* mid_j_host,
                       void* stream);

/* Static off-diagonal traction row sums, (n_e,3,3) float64
 * (Assembler.static_offdiag_rowsums, assembly.py:174-182). */
int ewb_static_rowsums(ewb_ctx* ctx, double* out_dev, void* stream);

/* Static T, U with the rigid-body diagonal, real (N,N) float64
 * (Assembler.assemble_static_tu, assembly.py:184-216). */
int ewb_static_tu(ewb_ctx* ctx, double* t_dev, double* u_dev, void* stream);

/* Dense T, U at complex omega (Im <= 0), complex128 (N,N)
 * (Assembler.assemble_tu, assembly.py:219-254; omega == 0 is the caller's
 * static path). */
int ewb_assemble_tu(ewb_ctx* ctx, double omega_re, double omega_im, void* t_dev, void* u_dev,
                    void* stream);

/* Fused per-frequency system: assemble_tu + apply_bcs + block_diag_precond
 * (assembly.py:219-297, linsolve.py:80-104) without materialising T or U.
 *   kinds_dev: (N,) uint8 NEUMANN=0 / DIRICHLET=1; prescribed_dev: (N,) complex;
 *   a_dev (N,N), b_dev (N,), pinv_dev (n_e,3,3) inverse diagonal blocks of A. */
int ewb_assemble_system(ewb_ctx* ctx, double omega_re, double omega_im,
                        const uint8_t* kinds_dev, const void* prescribed_dev, void* a_dev,
                        void* b_dev, void* pinv_dev, void* stream);

/* Multi-frequency fused system: nf <= EWB_MAX_BATCH members
 * of one sweep in one pass over the element pairs; member f equals
 * ewb_assemble_system at omega[f] to <= 1e-13 of max|A| (the phase factors
 * e^{-i Re(k) r} are stepped across an equispaced batch instead of being
 * re-evaluated).  Replaces nf iterations of the per-frequency assembly in
 * run_sweep (driver.py:128-134).  Host arrays omega_re/omega_im (nf,);
 * device arrays: prescribed (nf,N), a (nf,N,N), b (nf,N), pinv (nf,n_e,3,3),
 * flags (nf,4) int32, zeroed by the caller: [f][0] != 0 non-finite entries,
 * [f][1] singular diagonal blocks (identity fallback). */
#define EWB_MAX_BATCH 32
int ewb_assemble_system_multi(ewb_ctx* ctx, int32_t nf, const double* omega_re_host,
                              const double* omega_im_host, const uint8_t* kinds_dev,
                              const void* prescribed_dev, void* a_dev, void* b_dev,
                              void* pinv_dev, int32_t* flags_dev, void* stream);

/* Read and clear the context's fault flags (non-finite entries, singular
 * diagonal blocks) raised by the calls above.  Synchronises. */
int ewb_ctx_flags(ewb_ctx* ctx, int32_t* nonfinite_host, int32_t* singular_host, void* stream);
/* Stream-ordered variant for pipelined sweeps: moves the four flag words
 * (non-finite, singular, reserved x2) into flags_dev (device int32[4]) and
 * clears them, without synchronising. */
int ewb_ctx_flags_async(ewb_ctx* ctx, int32_t* flags_dev, void* stream);

/* apply_bcs for caller-supplied T, U (assembly.py:263-297). */
int ewb_apply_bcs(const void* t_dev, const void* u_dev, const uint8_t* kinds_dev,
                  const void* prescribed_dev, int64_t n, void* a_dev, void* b_dev, void* stream);

/* block_diag_precond (linsolve.py:80-104): pinv (n/3,3,3); singular blocks
 * become the identity and are counted in *singular_dev (int32, accumulated). */
int ewb_blockdiag_inverse(const void* a_dev, int64_t n, void* pinv_dev, int32_t* singular_dev,
                          void* stream);

/* y_b = A_b x_b for `batch` dense (n,n) systems (the `mat @ v` of
 * _as_operator, linsolve.py:73-77). */
int ewb_gemv_batched(const void* a_dev, const void* x_dev, void* y_dev, int64_t n, int32_t batch,
                     void* stream);

/* CTA budget of the solver launches (ewb_gmres, ewb_sem_guess): 0 = one CTA
 * per SM (default).  A smaller budget leaves SMs to concurrent work on other
 * streams; the matvec's bandwidth scales with the SMs it streams through
 * (measured ~46 GB/s per SM), so the default is the fastest solve.
 * Process-wide; not thread-safe. */
int ewb_set_solver_ctas(int32_t ctas);
int32_t ewb_solver_ctas(void);
/* Whole restarted right-preconditioned GMRES solve in one cooperative launch
 * (linsolve.py:107-210).  pinv_dev may be NULL (no preconditioner); x_dev
 * holds x0 when has_x0 != 0 and receives the solution; hist_dev receives the
 * residual history (init, then one estimate per iteration).  ax0_dev
 * (optional, used only with has_x0) holds A x0 when the caller already has
 * it (ewb_sem_guess returns it): the initial residual b - A x0
 * (linsolve.py:144) then costs no pass over A unless it already meets tol.
 * Restart residuals are formed from the cycle's stored products; every exit
 * (converged or maxiter) is decided on, and reports, the literal
 * ||b - A x|| / ||b|| (linsolve.py:200-205), one pass over A.
 * workspace: ewb_gmres_workspace_bytes(n, restart) bytes of device memory. */
int64_t ewb_gmres_workspace_bytes(int64_t n, int32_t restart);
int ewb_gmres(const void* a_dev, const void* b_dev, const void* pinv_dev, void* x_dev,
              int32_t has_x0, const void* ax0_dev, int64_t n, double tol, int32_t restart,
              int32_t maxiter,
              void* workspace_dev, int64_t workspace_bytes, double* hist_dev, int32_t hist_cap,
              ewb_gmres_result* result_dev, void* stream);

/* Least-squares extrapolated initial guess (sem_initial_guess,
 * linsolve.py:213-242), K in [1, 8].  x_hist_dev: K history columns, newest first,
 * column c at x_hist_dev + c*n; writes x0_dev (n) and, if ax0_dev is not
 * NULL, A x0 = (A X) s from the same products (for ewb_gmres). */
int64_t ewb_sem_workspace_bytes(int64_t n, int32_t K);
int ewb_sem_guess(const void* a_dev, const void* b_dev, const void* x_hist_dev, int32_t K,
                  int64_t n, double rank_tol, void* x0_dev, void* ax0_dev, void* workspace_dev,
                  int64_t workspace_bytes, ewb_sem_result* result_dev, void* stream);

/* The same guess from caller-supplied products y_hist_dev = A X (K columns,
 * column c at +c*n) — the matrix-free seam, where Y comes from one
 * ewb_matfree_apply pass (linsolve.py:226-242 without the matvecs). */
int ewb_sem_from_products(const void* b_dev, const void* x_hist_dev, const void* y_hist_dev,
                          int32_t K, int64_t n, double rank_tol, void* x0_dev, void* ax0_dev,
                          void* workspace_dev, int64_t workspace_bytes,
                          ewb_sem_result* result_dev, void* stream);

/* Restarted right-preconditioned GMRES around an operator applied by the
 * caller (the matrix-free seam gmres(apply_a=callable), linsolve.py:73-77,
 * 107-210).  All solver state stays on the device (ewb_op_head at the start
 * of the workspace).  Phases (cooperative launches): 0 begin, 1 Arnoldi step
 * on w = A z, 2 cycle end (back substitution, x update), 3 settle (literal
 * residual b - A x).  The host enqueues
 *   begin; apply(lit); settle;  { apply(cycle); step } x chunk; cycle_end; apply(lit); settle
 * and reads `done` once per chunk; apply(cycle) / apply(lit) are operator
 * applications z -> w (or vt/vu -> w for ewb_matfree_apply) gated on the
 * gate words (ewb_opgmres_buffers): with the gate at 0 they must do no work,
 * which ewb_matfree_apply's gate_dev does.  Every exit is decided on, and
 * reports, the literal ||b - A x|| / ||b||.  pinv_dev (n/3,3,3) or NULL;
 * kinds_dev (n) NEUMANN/DIRICHLET or NULL (vt = z), split_u: also write
 * vu = -mask_D z. */
int64_t ewb_opgmres_workspace_bytes(int64_t n, int32_t restart);
int ewb_opgmres_buffers(void* workspace_dev, int64_t n, int32_t restart, void** z_dev,
                        void** vt_dev, void** vu_dev, void** w_dev, int32_t** gate_cycle_dev,
                        int32_t** gate_literal_dev);
int ewb_opgmres_phase(int32_t phase, void* workspace_dev, int64_t workspace_bytes,
                      const void* b_dev, void* x_dev, int32_t has_x0, const void* ax0_dev,
                      const void* pinv_dev, const uint8_t* kinds_dev, int32_t split_u, int64_t n,
                      double tol, int32_t restart, int32_t maxiter, double* hist_dev,
                      int32_t hist_cap, void* stream);

/* conjugate_fill + window_weights + inverse_mft (transform.py:137-203) for D
 * columns at once.  half_dev: (n_half, D) complex (row k = frequency k);
 * out_dev: (N, D) float64 with N = 2 (n_half - 1); residue_dev: (D,) the
 * imaginary-residue ratio the reference checks (raise > 1e-8). */
int ewb_window_idft(const void* half_dev, int64_t n_half, int64_t D, int32_t window,
                    double eta, double period, double* out_dev, double* residue_dev,
                    void* stream);

/* Matrix-free operator (north-star item 2; seam gmres(apply_a=callable),
 * linsolve.py:73-77): y_k = T vt_k + U vu_k for K <= 5 vectors (each (N,)
 * complex, vector k at +k*N), recomputing every element pair with the
 * dense assembler's ladder (assembly.py:122-254).  A v uses vt = mask_N v,
 * vu = -mask_D v; b uses vt = -mask_D p, vu = mask_N p (assembly.py:293-296).
 * vu_dev may be NULL (all-Neumann: U not applied).  If pinv_dev is non-NULL
 * the inverse 3x3 diagonal blocks of A (kinds_dev mixes the columns) are
 * written too (block_diag_precond, linsolve.py:80-104).  gate_dev (device
 * int32, nullable): when *gate_dev == 0 at execution time the application
 * does no work (ewb_opgmres_*). */
int64_t ewb_matfree_workspace_bytes(const ewb_ctx* ctx, int32_t K);
int ewb_matfree_apply(ewb_ctx* ctx, double omega_re, double omega_im, const void* vt_dev,
                      const void* vu_dev, int32_t K, void* y_dev, const uint8_t* kinds_dev,
                      void* pinv_dev, void* workspace_dev, int64_t workspace_bytes,
                      const int32_t* gate_dev, void* stream);
/* The same with per-vector masks: bit k of t_mask / u_mask clear = vt_k /
 * vu_k is known to be zero and its block product is skipped (the K + 1
 * vector pass of an all-Neumann frequency: b has vt = 0, SEM's columns vu = 0).
 * Bits at or beyond K are rejected. */
int ewb_matfree_apply_masked(ewb_ctx* ctx, double omega_re, double omega_im, const void* vt_dev,
                             const void* vu_dev, int32_t K, uint32_t t_mask, uint32_t u_mask,
                             void* y_dev, const uint8_t* kinds_dev, void* pinv_dev,
                             void* workspace_dev, int64_t workspace_bytes,
                             const int32_t* gate_dev, void* stream);

/* Pair-kernel microbenchmark (BASELINE cfg3): P points x M triangles x F
 * frequencies with gauss7 on every pair (pair_geometry + integrated_blocks,
 * kernels.py:292-317).  x_dev (P,3), tri_dev (M,3,3) corners, omega_host
 * (F,2) = (re, im).  _blocks writes full U, T (F,P,M,3,3) complex;
 * _reduce writes yu = sum_m U x_m, yt = sum_m T x_m, (F,P,3) complex. */
int ewb_pair_kernels_blocks(const double* x_dev, int64_t P, const double* tri_dev, int64_t M,
                            const double* omega_host, int32_t F, double lam, double mu,
                            double rho, void* u_dev, void* t_dev, void* stream);
int64_t ewb_pair_kernels_workspace_bytes(int64_t P, int64_t M, int32_t F);
int ewb_pair_kernels_reduce(const double* x_dev, int64_t P, const double* tri_dev, int64_t M,
                            const void* xvec_dev, const double* omega_host, int32_t F, double lam,
                            double mu, double rho, void* yu_dev, void* yt_dev,
                            void* workspace_dev, int64_t workspace_bytes, void* stream);

/* DFMA throughput probe (TFLOP/s) — the FP64 roofline denominator, which
 * MEASURED_PEAKS.json does not carry.  Synchronises. */
int ewb_fp64_peak_probe(int64_t iters, int32_t blocks_per_sm, double* tflops_host,
                        double* ms_host, void* stream);

/* The device sin/cos/exp the kernel phases use (ewb_common.cuh fast_sincos /
 * fast_exp), evaluated on n HOST arguments into host arrays: the accuracy
 * check against libm (tests).  Synchronises. */
int ewb_math_selftest(const double* x_host, int64_t n, double* sin_host, double* cos_host,
                      double* exp_host, void* stream);

/* The small-argument exponential (ewb_common.cuh exp_small) that steps the
 * damping factor e^{Im(k) r} from the first quadrature point of a far pair
 * to the other two in the matrix-free kernels, on n HOST arguments
 * |t| <= 2^-4 (EWB_ERR_INVALID beyond).  Synchronises. */
int ewb_math_selftest_delta(const double* t_host, int64_t n, double* exp_host, void* stream);

/* Debug-build self checks (library built with -DEWB_DEBUG_CHECKS; the
 * stand-in for compute-sanitizer): *failures = device-side
 * invariant violations recorded since the last reset (index bounds,
 * ring-slot bookkeeping, scratch capacity), *first_site = the first
 * violated check's id (0 if none).  A release build reports *failures = -1.
 * reset != 0 clears the counters after reading.  Synchronises the device. */
int ewb_debug_checks(int64_t* failures, int64_t* first_site, int32_t reset);

#ifdef __cplusplus
}
#endif

#endif /* EWBEM_B200_H */
