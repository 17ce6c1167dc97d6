// Internal interfaces of the Krylov kernels (ewb_krylov.cu).
#pragma once

#include <cuda_runtime.h>

#include "ewb_common.cuh"

namespace ewb {

constexpr int kMaxRestart = 128;   // Arnoldi cycle length cap (reference default 60)
constexpr int kMaxSem = 4;         // SEM history depth cap (reference default 4)

struct GmresOut {
  int iterations;
  int n_hist;
  int converged;
  int matvecs;   // dense passes over A (iterations + restarts + r0)
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
  cplx* W;              // scratch (restart n): A P^{-1} v_j of the cycle, or nullptr
                        // (then the cycle's true residual takes a pass over A)
  cplx* rs;             // scratch (n): the cycle's starting residual (with W)
  cplx* H;              // scratch ((kMaxRestart+1) kMaxRestart)
  cplx* Gram;           // scratch ((kMaxRestart+1) kMaxRestart): <v_i, v_l>, l < i
  cplx* dpart;          // scratch (2 * grid * (2 kMaxRestart + 2)) batched-dot partials
  double* partial;      // scratch (2 * grid * 16)
  double* hist;         // residual history (hist_cap)
  GmresOut* out;
  long long n;
  int restart, maxiter, has_x0, hist_cap;
  int ortho;            // 0: fused one-reduction MGS (default), 1: sequential MGS,
                        // 2: one-reduction MGS with separate vector phases
  unsigned long long* probe;  // optional phase trace (CTA 0): (phase << 56) | globaltimer
  int probe_cap;
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

int solver_grid_max();      // co-resident CTAs of the solver kernels (workspace sizing)
int solver_grid_blocks();   // CTAs the solver launches use (<= max, see set_solver_ctas)
void set_solver_ctas(int ctas);
cudaError_t launch_gmres(GmresArgs& args, cudaStream_t s);
cudaError_t launch_sem(SemArgs& args, cudaStream_t s);
// Row balance (see cta_rows): measure per-CTA matvec speed on A (n x n) and
// split rows accordingly for every later solver launch; stats (us): spread
// and mean of the per-CTA matvec time, equal split then calibrated split.
cudaError_t calibrate_rows(const cplx* A, long long n, int iters, double* stats, cudaStream_t s);
cudaError_t reset_row_balance(cudaStream_t s);
cudaError_t launch_gemv_batched(const cplx* A, const cplx* x, cplx* y, long long n, int batch,
                                cudaStream_t s);

}  // namespace ewb
