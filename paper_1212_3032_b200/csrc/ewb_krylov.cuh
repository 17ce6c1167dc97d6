// Internal interfaces of the Krylov kernels (ewb_krylov.cu).
#pragma once

#include <cuda_runtime.h>

#include "ewb_common.cuh"

namespace ewb {

constexpr int kMaxRestart = 128;   // Arnoldi cycle length cap (reference default 60)
constexpr int kMaxSem = 8;         // SEM history depth cap (reference default 4)

struct GmresOut {
  int iterations;
  int n_hist;
  int converged;
  int matvecs;   // dense passes over A (iterations + exit residuals + r0)
  double init_res;
  double final_res;
};

struct GmresArgs {
  const cplx* A;        // (n, n) row-major
  const cplx* b;        // (n,)
  const cplx* pinv;     // (n/3, 3, 3) or nullptr (no preconditioner)
  cplx* x;              // in: x0 if has_x0; out: solution
  const cplx* ax0;      // optional A x0 (initial residual without a pass over A)
  cplx* r;              // scratch (n)
  cplx* w;              // scratch (n)
  cplx* z;              // scratch (n)
  cplx* V;              // scratch ((restart+1) n)
  cplx* W;              // scratch (restart n): A P^{-1} v_j of the cycle (restart
                        // residuals without a pass over A), or nullptr
  cplx* rs;             // scratch (n): the cycle's starting residual (with W)
  cplx* H;              // scratch ((kMaxRestart+1) kMaxRestart)
  cplx* Gram;           // scratch ((kMaxRestart+1) kMaxRestart): <v_i, v_l>, l < i
  cplx* dpart;          // scratch (2 * grid * (2 kMaxRestart + 2)) batched-dot partials
  double* partial;      // scratch (2 * grid * 16)
  double* hist;         // residual history (hist_cap)
  GmresOut* out;
  long long n;
  int restart, maxiter, has_x0, hist_cap;
  double tol;
};

struct SemOut {
  int kept;
  int fallback;
};

struct SemArgs {
  const cplx* A;        // (n, n)
  const cplx* b;        // (n,)
  const cplx* X;        // K columns, column c at X + c n (newest first)
  cplx* Y;              // scratch K n
  cplx* Q;              // scratch K n
  cplx* x0;             // out (n)
  cplx* ax0;            // optional out (n): A x0 = Y s
  double* partial;
  SemOut* out;
  long long n;
  int K;
  double rank_tol;
};


// ---------------------------------------------------------------------
// GMRES around an operator that is applied by its own launches (the
// matrix-free seam gmres(apply_a=callable), linsolve.py:73-77).  The whole
// solver state lives on the device; the host enqueues
//   begin, [apply(x) if lit_pending], settle,
//   { [apply(z) if in_cycle], step } x chunk, cycle_end, [apply(x) if lit_pending], settle
// and reads `done` once per chunk.  Applications whose gate word is 0 exit
// at once, so a chunk may be enqueued past convergence without work.
struct OpHead {
  int in_cycle;         // gate of the Arnoldi applications: next apply is A z_j
  int lit_pending;      // gate of the literal applications: next apply is A x
  int done, converged;
  int its, j, m, used;
  int cycle_open, n_hist, applies, pad;
  double nb, rnorm, res, init_res, final_res;
};
struct OpState {
  OpHead h;
  cplx g[kMaxRestart + 1], cs[kMaxRestart], sn[kMaxRestart];
  cplx H[(kMaxRestart + 1) * kMaxRestart];   // H[i * kMaxRestart + j]
};

struct OpArgs {
  OpState* st;
  const cplx* b;        // (n,)
  cplx* x;              // in: x0 (has_x0); out: solution
  const cplx* ax0;      // optional A x0 (SEM's (A X) s)
  const cplx* pinv;     // (n/3,3,3) or nullptr
  const uint8_t* kinds; // per-DOF NEUMANN/DIRICHLET (nullable: vt only)
  cplx* z;              // (n) operator input: P^{-1} v_j, or x for a literal residual
  cplx* vt;             // (n) mask_N z  (A z = T vt + U vu, assembly.py:293-294)
  cplx* vu;             // (n) -mask_D z, or nullptr (all Neumann)
  const cplx* w;        // (n) operator output
  cplx* r;              // (n) residual
  cplx* rs;             // (n) the cycle's starting residual
  cplx* V;              // ((restart+1) n) Arnoldi basis
  cplx* W;              // (restart n) A P^{-1} v_j of the cycle
  double* hist;
  double* partial;      // (2 * grid * 16)
  long long n;
  int restart, maxiter, has_x0, hist_cap;
  double tol;
};

cudaError_t launch_op_gmres(int phase, OpArgs& args, cudaStream_t s);  // 0 begin 1 step 2 cycle_end 3 settle

int solver_grid_max();      // co-resident CTAs of the solver kernels (workspace sizing)
int solver_grid_blocks();   // CTAs the solver launches use (<= max, see set_solver_ctas)
void set_solver_ctas(int ctas);
long long ring_cplx_capacity();  // complex values the solver shared-memory ring holds
// debug build (-DEWB_DEBUG_CHECKS): per translation unit violation count + first site
void dbg_fetch_assembly(unsigned long long* o);
void dbg_fetch_krylov(unsigned long long* o);
void dbg_fetch_matfree(unsigned long long* o);
void dbg_fetch_spectral(unsigned long long* o);
void dbg_reset_assembly();
void dbg_reset_krylov();
void dbg_reset_matfree();
void dbg_reset_spectral();
cudaError_t launch_gmres(GmresArgs& args, cudaStream_t s);
cudaError_t launch_sem(SemArgs& args, cudaStream_t s);
// QR + solve of SEM from caller-supplied products Y = A X (args.A unused)
cudaError_t launch_sem_products(SemArgs& args, cudaStream_t s);
cudaError_t launch_gemv_batched(const cplx* A, const cplx* x, cplx* y, long long n, int batch,
                                cudaStream_t s);

}  // namespace ewb
