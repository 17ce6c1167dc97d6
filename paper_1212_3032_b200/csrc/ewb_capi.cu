// extern "C" boundary (include/ewbem_b200.h).  Validation, error codes and
// the thread-local error string live here; kernels live in the other files.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ewbem_b200.h"
#include "ewb_ctx.cuh"
#include "ewb_krylov.cuh"

namespace ewb {
cudaError_t launch_window_idft(const cplx* half, long long n_half, long long D, const double* win,
                               const cplx* tw, double eta_dt, double* out, double* residue,
                               cudaStream_t s);
}

struct ewb_ctx {
  ewb::Context c;
};

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void ewb::note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
  return fail(EWB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define EWB_CUDA(call, where)                 \
  do {                                        \
    cudaError_t e_ = (call);                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// The stream-ordered allocator's default pool returns freed memory to the
// driver at every synchronisation (release threshold 0), so the next small
// cudaMallocAsync can stall the host for tens of ms; keep it pooled.
static void keep_pool_memory() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

extern "C" {

int ewb_abi_version(void) { return EWB_ABI_VERSION; }

const char* ewb_last_error(void) { return g_err.c_str(); }

int64_t ewb_launch_count(void) { return g_launches.load(); }

int ewb_ctx_create(const double* centroids, const double* normals, const double* areas,
                   const double* diameters, const double* corners, int64_t n_elements,
                   double lam, double mu, double rho, const double* gl8, const double* gl16,
                   const double* rules, const int32_t* rule_off, const int32_t* rule_q,
                   void* stream, ewb_ctx** out) {
  if (!out || !centroids || !normals || !areas || !diameters || !corners || !gl8 || !gl16 ||
      !rules || !rule_off || !rule_q)
    return fail(EWB_ERR_INVALID, "ewb_ctx_create: null argument");
  if (n_elements < 1 || n_elements > (1LL << 22))
    return fail(EWB_ERR_INVALID, "ewb_ctx_create: n_elements out of range");
  if (!(mu > 0) || !(rho > 0) || !(lam + 2 * mu > 0))
    return fail(EWB_ERR_INVALID, "ewb_ctx_create: invalid material");
  for (int k = 0; k < 6; ++k)
    if (rule_q[k] < 1) return fail(EWB_ERR_INVALID, "ewb_ctx_create: empty rule table");
  auto* h = new ewb_ctx();
  h->c.n_e = (int)n_elements;
  h->c.lam = lam;
  h->c.mu = mu;
  h->c.rho = rho;
  cudaError_t e = ewb::setup_context(h->c, centroids, normals, areas, diameters, corners, gl8,
                                     gl16, rules, rule_off, rule_q, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  if (e != cudaSuccess) {
    for (void* p : h->c.owned) cudaFree(p);
    delete h;
    return cuda_fail(e, "ewb_ctx_create");
  }
  *out = h;
  return EWB_OK;
}

int ewb_ctx_destroy(ewb_ctx* ctx) {
  if (!ctx) return EWB_OK;
  cudaDeviceSynchronize();
  for (void* p : ctx->c.owned) cudaFree(p);
  delete ctx;
  return EWB_OK;
}

int ewb_ctx_set_exterior(ewb_ctx* ctx, int32_t on, void* stream) {
  if (!ctx) return fail(EWB_ERR_INVALID, "ewb_ctx_set_exterior: null argument");
  EWB_CUDA(ewb::set_exterior(ctx->c, on, S(stream)), "ewb_ctx_set_exterior");
  return EWB_OK;
}

int ewb_ctx_counts(const ewb_ctx* ctx, int64_t* counts) {
  if (!ctx || !counts) return fail(EWB_ERR_INVALID, "ewb_ctx_counts: null argument");
  counts[0] = ctx->c.n_e;
  counts[1] = ctx->c.n_far;
  counts[2] = ctx->c.n_mid;
  counts[3] = ctx->c.n_near;
  for (int L = 1; L <= 4; ++L) counts[3 + L] = ctx->c.n_near_lvl[L];
  return EWB_OK;
}

int ewb_ctx_pair_lists(const ewb_ctx* ctx, int32_t* near_ptr, int32_t* near_j, int32_t* near_lvl,
                       int32_t* mid_ptr, int32_t* mid_j, void* stream) {
  if (!ctx) return fail(EWB_ERR_INVALID, "ewb_ctx_pair_lists: null context");
  const ewb::Geo& g = ctx->c.g;
  const size_t n1 = sizeof(int32_t) * (ctx->c.n_e + 1);
  const size_t nn = sizeof(int32_t) * ctx->c.n_near, nm = sizeof(int32_t) * ctx->c.n_mid;
  struct { void* dst; const void* src; size_t bytes; } cp[] = {
      {near_ptr, g.near_ptr, n1}, {near_j, g.near_j, nn}, {near_lvl, g.near_lvl, nn},
      {mid_ptr, g.mid_ptr, n1}, {mid_j, g.mid_j, nm}};
  for (auto& c : cp)
    if (c.dst && c.bytes)
      EWB_CUDA(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToHost, S(stream)),
               "ewb_ctx_pair_lists");
  EWB_CUDA(cudaStreamSynchronize(S(stream)), "ewb_ctx_pair_lists");
  return EWB_OK;
}

int ewb_static_rowsums(ewb_ctx* ctx, double* out, void* stream) {
  if (!ctx || !out) return fail(EWB_ERR_INVALID, "ewb_static_rowsums: null argument");
  EWB_CUDA(cudaMemcpyAsync(out, ctx->c.rowsums, sizeof(double) * 9 * ctx->c.n_e,
                           cudaMemcpyDeviceToDevice, S(stream)),
           "ewb_static_rowsums");
  return EWB_OK;
}

int ewb_static_tu(ewb_ctx* ctx, double* t, double* u, void* stream) {
  if (!ctx || !t || !u) return fail(EWB_ERR_INVALID, "ewb_static_tu: null argument");
  EWB_CUDA(ewb::launch_static_pass(ctx->c, t, u, S(stream)), "ewb_static_tu");
  return EWB_OK;
}

static int check_omega(double ore, double oim, const char* who) {
  // material.py:92-93
  double mag = std::hypot(ore, oim);
  if (!std::isfinite(ore) || !std::isfinite(oim))
    return fail(EWB_ERR_INVALID, std::string(who) + ": non-finite frequency");
  if (oim > 1e-12 * (mag > 1.0 ? mag : 1.0))
    return fail(EWB_ERR_INVALID, std::string(who) + ": frequency has positive imaginary part");
  if (ore == 0.0 && oim == 0.0)
    return fail(EWB_ERR_INVALID, std::string(who) + ": omega == 0 takes the static path");
  return EWB_OK;
}

int ewb_assemble_tu(ewb_ctx* ctx, double ore, double oim, void* t, void* u, void* stream) {
  if (!ctx || !t || !u) return fail(EWB_ERR_INVALID, "ewb_assemble_tu: null argument");
  if (int rc = check_omega(ore, oim, "ewb_assemble_tu")) return rc;
  {
    const size_t nn = 9 * (size_t)ctx->c.n_e * ctx->c.n_e * 16;
    EWB_CUDA(ewb::dbg_poison(t, nn, S(stream)), "ewb_assemble_tu");
    EWB_CUDA(ewb::dbg_poison(u, nn, S(stream)), "ewb_assemble_tu");
  }
  EWB_CUDA(ewb::launch_assemble_tu(ctx->c, ore, oim, (ewb::cplx*)t, (ewb::cplx*)u, S(stream)),
           "ewb_assemble_tu");
  return EWB_OK;
}

int ewb_assemble_system(ewb_ctx* ctx, double ore, double oim, const uint8_t* kinds,
                        const void* p, void* a, void* b, void* pinv, void* stream) {
  if (!ctx || !kinds || !p || !a || !b || !pinv)
    return fail(EWB_ERR_INVALID, "ewb_assemble_system: null argument");
  if (int rc = check_omega(ore, oim, "ewb_assemble_system")) return rc;
  {
    const size_t N = 3 * (size_t)ctx->c.n_e;
    EWB_CUDA(ewb::dbg_poison(a, N * N * 16, S(stream)), "ewb_assemble_system");
    EWB_CUDA(ewb::dbg_poison(b, N * 16, S(stream)), "ewb_assemble_system");
    EWB_CUDA(ewb::dbg_poison(pinv, 3 * N * 16, S(stream)), "ewb_assemble_system");
  }
  EWB_CUDA(ewb::launch_assemble_system(ctx->c, ore, oim, kinds, (const ewb::cplx*)p,
                                       (ewb::cplx*)a, (ewb::cplx*)b, (ewb::cplx*)pinv, S(stream)),
           "ewb_assemble_system");
  return EWB_OK;
}

int ewb_assemble_system_multi(ewb_ctx* ctx, int32_t nf, const double* ore, const double* oim,
                              const uint8_t* kinds, const void* p, void* a, void* b, void* pinv,
                              int32_t* flags, void* stream) {
  if (!ctx || !ore || !oim || !kinds || !p || !a || !b || !pinv || !flags)
    return fail(EWB_ERR_INVALID, "ewb_assemble_system_multi: null argument");
  if (nf < 1 || nf > EWB_MAX_BATCH)
    return fail(EWB_ERR_INVALID, "ewb_assemble_system_multi: nf must be in [1, EWB_MAX_BATCH]");
  for (int f = 0; f < nf; ++f)
    if (int rc = check_omega(ore[f], oim[f], "ewb_assemble_system_multi")) return rc;
  {  // every entry of A, b, P^{-1} must have a writer
    const size_t N = 3 * (size_t)ctx->c.n_e;
    EWB_CUDA(ewb::dbg_poison(a, nf * N * N * 16, S(stream)), "ewb_assemble_system_multi");
    EWB_CUDA(ewb::dbg_poison(b, nf * N * 16, S(stream)), "ewb_assemble_system_multi");
    EWB_CUDA(ewb::dbg_poison(pinv, nf * 3 * N * 16, S(stream)), "ewb_assemble_system_multi");
  }
  EWB_CUDA(ewb::launch_assemble_system_multi(ctx->c, nf, ore, oim, kinds, (const ewb::cplx*)p,
                                             (ewb::cplx*)a, (ewb::cplx*)b, (ewb::cplx*)pinv,
                                             flags, S(stream)),
           "ewb_assemble_system_multi");
  return EWB_OK;
}

int ewb_ctx_flags(ewb_ctx* ctx, int32_t* nonfinite, int32_t* singular, void* stream) {
  if (!ctx) return fail(EWB_ERR_INVALID, "ewb_ctx_flags: null argument");
  int h[4] = {0, 0, 0, 0};
  EWB_CUDA(cudaMemcpyAsync(h, ctx->c.flags, 16, cudaMemcpyDeviceToHost, S(stream)), "ewb_ctx_flags");
  EWB_CUDA(cudaMemsetAsync(ctx->c.flags, 0, 16, S(stream)), "ewb_ctx_flags");
  EWB_CUDA(cudaStreamSynchronize(S(stream)), "ewb_ctx_flags");
  if (nonfinite) *nonfinite = h[0];
  if (singular) *singular = h[1];
  return EWB_OK;
}

int ewb_ctx_flags_async(ewb_ctx* ctx, int32_t* flags_dev, void* stream) {
  if (!ctx || !flags_dev) return fail(EWB_ERR_INVALID, "ewb_ctx_flags_async: null argument");
  EWB_CUDA(cudaMemcpyAsync(flags_dev, ctx->c.flags, 16, cudaMemcpyDeviceToDevice, S(stream)),
           "ewb_ctx_flags_async");
  EWB_CUDA(cudaMemsetAsync(ctx->c.flags, 0, 16, S(stream)), "ewb_ctx_flags_async");
  return EWB_OK;
}

int ewb_apply_bcs(const void* t, const void* u, const uint8_t* kinds, const void* p, int64_t n,
                  void* a, void* b, void* stream) {
  if (!t || !u || !kinds || !p || !a || !b || n < 1)
    return fail(EWB_ERR_INVALID, "ewb_apply_bcs: bad argument");
  EWB_CUDA(ewb::launch_apply_bcs((const ewb::cplx*)t, (const ewb::cplx*)u, kinds,
                                 (const ewb::cplx*)p, n, (ewb::cplx*)a, (ewb::cplx*)b, S(stream)),
           "ewb_apply_bcs");
  return EWB_OK;
}

int ewb_blockdiag_inverse(const void* a, int64_t n, void* pinv, int32_t* singular, void* stream) {
  if (!a || !pinv || !singular) return fail(EWB_ERR_INVALID, "ewb_blockdiag_inverse: null argument");
  if (n < 3 || n % 3)
    return fail(EWB_ERR_INVALID, "matrix must be square with size divisible by 3");
  EWB_CUDA(ewb::launch_blockdiag_inverse((const ewb::cplx*)a, n, (ewb::cplx*)pinv, singular,
                                         S(stream)),
           "ewb_blockdiag_inverse");
  return EWB_OK;
}

int ewb_gemv_batched(const void* a, const void* x, void* y, int64_t n, int32_t batch,
                     void* stream) {
  if (!a || !x || !y || n < 1 || batch < 1)
    return fail(EWB_ERR_INVALID, "ewb_gemv_batched: bad argument");
  EWB_CUDA(ewb::launch_gemv_batched((const ewb::cplx*)a, (const ewb::cplx*)x, (ewb::cplx*)y, n,
                                    batch, S(stream)),
           "ewb_gemv_batched");
  return EWB_OK;
}

int ewb_set_solver_ctas(int32_t ctas) {
  if (ctas < 0) return fail(EWB_ERR_INVALID, "ewb_set_solver_ctas: ctas must be >= 0");
  ewb::set_solver_ctas(ctas);
  return EWB_OK;
}

int32_t ewb_solver_ctas(void) { return ewb::solver_grid_blocks(); }

// workspace layout: r, w, z (3n), V ((restart+1) n), H, partial
int64_t ewb_gmres_workspace_bytes(int64_t n, int32_t restart) {
  int64_t cpl = 16;
  int64_t G = ewb::solver_grid_max();
  return cpl * (3 * n + (int64_t)(restart + 1) * n + (int64_t)(restart + 1) * n +
                2 * (int64_t)(ewb::kMaxRestart + 1) * ewb::kMaxRestart +
                2 * G * (2 * ewb::kMaxRestart + 2)) +
         8 * 2 * G * 16 + 256 * 8;
}

int ewb_gmres(const void* a, const void* b, const void* pinv, void* x, int32_t has_x0,
              const void* ax0, int64_t n, double tol, int32_t restart, int32_t maxiter, void* ws,
              int64_t ws_bytes,
              double* hist, int32_t hist_cap, ewb_gmres_result* result, void* stream) {
  if (!a || !b || !x || !ws || !hist || !result || n < 1)
    return fail(EWB_ERR_INVALID, "ewb_gmres: bad argument");
  if (!(tol > 0.0 && tol < 1.0)) return fail(EWB_ERR_INVALID, "tol must be in (0, 1)");
  if (restart < 1 || restart > ewb::kMaxRestart)
    return fail(EWB_ERR_INVALID, "ewb_gmres: restart must be in [1, 128]");
  if (maxiter < 0) return fail(EWB_ERR_INVALID, "ewb_gmres: maxiter must be >= 0");
  if (pinv && n % 3) return fail(EWB_ERR_INVALID, "ewb_gmres: preconditioner needs n % 3 == 0");
  if (ws_bytes < ewb_gmres_workspace_bytes(n, restart))
    return fail(EWB_ERR_INVALID, "ewb_gmres: workspace too small");
  // the update phase keeps max(RU, 512) + RU complex values of the idle
  // ring, RU = rows per CTA + the <= 2 rows completing its last element
  {
    const int64_t G = ewb::solver_grid_blocks();
    const int64_t ru = (n + G - 1) / G + 2;
    if ((ru > 512 ? ru : 512) + ru > ewb::ring_cplx_capacity())
      return fail(EWB_ERR_INVALID, "ewb_gmres: too many rows per solver CTA for the shared-memory "
                                   "ring (raise the solver CTA count, ewb_set_solver_ctas)");
  }
  ewb::GmresArgs g{};
  auto* base = (ewb::cplx*)ws;
  g.A = (const ewb::cplx*)a;
  g.b = (const ewb::cplx*)b;
  g.pinv = (const ewb::cplx*)pinv;
  g.x = (ewb::cplx*)x;
  g.ax0 = has_x0 ? (const ewb::cplx*)ax0 : nullptr;
  g.r = base;
  g.w = base + n;
  g.z = base + 2 * n;
  g.V = base + 3 * n;
  g.W = g.V + (int64_t)(restart + 1) * n;
  g.rs = g.W + (int64_t)restart * n;
  g.H = g.rs + n;
  g.Gram = g.H + (int64_t)(ewb::kMaxRestart + 1) * ewb::kMaxRestart;
  g.dpart = g.Gram + (int64_t)(ewb::kMaxRestart + 1) * ewb::kMaxRestart;
  g.partial = (double*)(g.dpart + 2 * (int64_t)ewb::solver_grid_max() *
                                      (2 * ewb::kMaxRestart + 2));
  g.hist = hist;
  g.out = (ewb::GmresOut*)result;
  g.n = n;
  g.restart = restart;
  g.maxiter = maxiter;
  g.has_x0 = has_x0;
  g.hist_cap = hist_cap;
  g.tol = tol;
  EWB_CUDA(ewb::dbg_poison(ws, (size_t)ws_bytes, S(stream)), "ewb_gmres");
  EWB_CUDA(ewb::launch_gmres(g, S(stream)), "ewb_gmres");
  return EWB_OK;
}

int64_t ewb_sem_workspace_bytes(int64_t n, int32_t K) {
  int64_t G = ewb::solver_grid_max();
  return 16 * (2 * (int64_t)K * n) + 8 * 2 * G * 16 + 256 * 8;
}

int ewb_sem_guess(const void* a, const void* b, const void* xh, int32_t K, int64_t n,
                  double rank_tol, void* x0, void* ax0, void* ws, int64_t ws_bytes,
                  ewb_sem_result* result, void* stream) {
  if (!a || !b || !xh || !x0 || !ws || !result || n < 1)
    return fail(EWB_ERR_INVALID, "ewb_sem_guess: bad argument");
  if (K < 1 || K > ewb::kMaxSem) return fail(EWB_ERR_INVALID, "ewb_sem_guess: K must be in [1, 8]");
  if (ws_bytes < ewb_sem_workspace_bytes(n, K))
    return fail(EWB_ERR_INVALID, "ewb_sem_guess: workspace too small");
  ewb::SemArgs s{};
  auto* base = (ewb::cplx*)ws;
  s.A = (const ewb::cplx*)a;
  s.b = (const ewb::cplx*)b;
  s.X = (const ewb::cplx*)xh;
  s.Y = base;
  s.Q = base + (int64_t)K * n;
  s.partial = (double*)(base + 2 * (int64_t)K * n);
  s.x0 = (ewb::cplx*)x0;
  s.ax0 = (ewb::cplx*)ax0;
  s.out = (ewb::SemOut*)result;
  s.n = n;
  s.K = K;
  s.rank_tol = rank_tol;
  EWB_CUDA(ewb::dbg_poison(ws, (size_t)ws_bytes, S(stream)), "ewb_sem_guess");
  EWB_CUDA(ewb::launch_sem(s, S(stream)), "ewb_sem_guess");
  return EWB_OK;
}

int ewb_sem_from_products(const void* b, const void* xh, const void* yh, int32_t K, int64_t n,
                          double rank_tol, void* x0, void* ax0, void* ws, int64_t ws_bytes,
                          ewb_sem_result* result, void* stream) {
  if (!b || !xh || !yh || !x0 || !ws || !result || n < 1)
    return fail(EWB_ERR_INVALID, "ewb_sem_from_products: bad argument");
  if (K < 1 || K > ewb::kMaxSem)
    return fail(EWB_ERR_INVALID, "ewb_sem_from_products: K must be in [1, 8]");
  if (ws_bytes < ewb_sem_workspace_bytes(n, K))
    return fail(EWB_ERR_INVALID, "ewb_sem_from_products: workspace too small");
  ewb::SemArgs s{};
  auto* base = (ewb::cplx*)ws;
  s.b = (const ewb::cplx*)b;
  s.X = (const ewb::cplx*)xh;
  s.Y = (ewb::cplx*)yh;
  s.Q = base;
  s.partial = (double*)(base + (int64_t)K * n);
  s.x0 = (ewb::cplx*)x0;
  s.ax0 = (ewb::cplx*)ax0;
  s.out = (ewb::SemOut*)result;
  s.n = n;
  s.K = K;
  s.rank_tol = rank_tol;
  EWB_CUDA(ewb::launch_sem_products(s, S(stream)), "ewb_sem_from_products");
  return EWB_OK;
}

// operator-GMRES workspace: state | z vt vu w r rs (6n) | V ((restart+1) n) |
// W (restart n) | partials
static_assert(sizeof(ewb_op_head) == sizeof(ewb::OpHead), "ewb_op_head mirrors OpHead");
static_assert(offsetof(ewb_op_head, final_residual) == offsetof(ewb::OpHead, final_res),
              "ewb_op_head mirrors OpHead");
static int64_t op_state_bytes() { return ((int64_t)sizeof(ewb::OpState) + 255) / 256 * 256; }

int64_t ewb_opgmres_workspace_bytes(int64_t n, int32_t restart) {
  if (n < 1 || restart < 1 || restart > ewb::kMaxRestart) return -1;
  const int64_t G = ewb::solver_grid_max();
  return op_state_bytes() + 16 * (6 * n + (int64_t)(2 * restart + 1) * n) + 8 * 2 * G * 16;
}

int ewb_opgmres_buffers(void* ws, int64_t n, int32_t restart, void** z, void** vt, void** vu,
                        void** w, int32_t** gate_cycle, int32_t** gate_literal) {
  if (!ws || n < 1 || restart < 1 || restart > ewb::kMaxRestart)
    return fail(EWB_ERR_INVALID, "ewb_opgmres_buffers: bad argument");
  auto* st = (ewb::OpState*)ws;
  auto* v = (ewb::cplx*)((unsigned char*)ws + op_state_bytes());
  if (z) *z = v;
  if (vt) *vt = v + n;
  if (vu) *vu = v + 2 * n;
  if (w) *w = v + 3 * n;
  if (gate_cycle) *gate_cycle = &st->h.in_cycle;
  if (gate_literal) *gate_literal = &st->h.lit_pending;
  return EWB_OK;
}

int ewb_opgmres_phase(int32_t phase, void* ws, int64_t ws_bytes, const void* b, void* x,
                      int32_t has_x0, const void* ax0, const void* pinv, const uint8_t* kinds,
                      int32_t split_u, int64_t n, double tol, int32_t restart, int32_t maxiter,
                      double* hist, int32_t hist_cap, void* stream) {
  if (phase < 0 || phase > 3 || !ws || !b || !x || !hist || n < 1)
    return fail(EWB_ERR_INVALID, "ewb_opgmres_phase: bad argument");
  if (!(tol > 0.0 && tol < 1.0)) return fail(EWB_ERR_INVALID, "tol must be in (0, 1)");
  if (restart < 1 || restart > ewb::kMaxRestart)
    return fail(EWB_ERR_INVALID, "ewb_opgmres_phase: restart must be in [1, 128]");
  if (maxiter < 0) return fail(EWB_ERR_INVALID, "ewb_opgmres_phase: maxiter must be >= 0");
  if ((pinv || kinds) && n % 3)
    return fail(EWB_ERR_INVALID, "ewb_opgmres_phase: preconditioner/kinds need n % 3 == 0");
  if (ws_bytes < ewb_opgmres_workspace_bytes(n, restart))
    return fail(EWB_ERR_INVALID, "ewb_opgmres_phase: workspace too small");
  ewb::OpArgs a{};
  a.st = (ewb::OpState*)ws;
  auto* v = (ewb::cplx*)((unsigned char*)ws + op_state_bytes());
  a.z = v;
  a.vt = v + n;
  a.vu = split_u ? v + 2 * n : nullptr;
  a.w = v + 3 * n;
  a.r = v + 4 * n;
  a.rs = v + 5 * n;
  a.V = v + 6 * n;
  a.W = a.V + (int64_t)(restart + 1) * n;
  a.partial = (double*)(a.W + (int64_t)restart * n);
  a.b = (const ewb::cplx*)b;
  a.x = (ewb::cplx*)x;
  a.ax0 = has_x0 ? (const ewb::cplx*)ax0 : nullptr;
  a.pinv = (const ewb::cplx*)pinv;
  a.kinds = kinds;
  a.hist = hist;
  a.hist_cap = hist_cap;
  a.n = n;
  a.restart = restart;
  a.maxiter = maxiter;
  a.has_x0 = has_x0;
  a.tol = tol;
  EWB_CUDA(ewb::launch_op_gmres(phase, a, S(stream)), "ewb_opgmres_phase");
  return EWB_OK;
}

int ewb_window_idft(const void* half, int64_t n_half, int64_t D, int32_t window, double eta,
                    double period, double* out, double* residue, void* stream) {
  if (!half || !out || !residue || n_half < 2 || D < 1)
    return fail(EWB_ERR_INVALID, "ewb_window_idft: bad argument");
  if (window < 0 || window > 2) return fail(EWB_ERR_INVALID, "ewb_window_idft: unknown window");
  const int64_t N = 2 * (n_half - 1);
  if (N > 4096) return fail(EWB_ERR_INVALID, "ewb_window_idft: N > 4096 unsupported");
  // host-exact tables: window_weights (transform.py:157-176) and e^{2 pi i m / N},
  // built and uploaded once per (N, window) and kept on the device: a
  // per-call stream-ordered malloc + free + synchronize showed 30-150 ms host
  // stalls in the benchmark's timed steps
  static std::mutex mu;
  static std::map<std::tuple<int, int64_t, int32_t>, void*> cache;
  void* dtab = nullptr;
  int dev = 0;
  EWB_CUDA(cudaGetDevice(&dev), "ewb_window_idft");
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, N, window});
    if (it != cache.end()) {
      dtab = it->second;
    } else {
      std::vector<double> tab(3 * N);
      for (int64_t k = 0; k < N; ++k) {
        double ph = 2.0 * M_PI * (double)k / (double)N;
        double w = 1.0;
        if (window == EWB_WIN_HANNING) w = 0.5 * (1.0 + std::cos(ph));
        else if (window == EWB_WIN_BLACKMAN) w = 0.42 + 0.5 * std::cos(ph) + 0.08 * std::cos(2.0 * ph);
        tab[k] = w;
        tab[N + 2 * k] = std::cos(ph);
        tab[N + 2 * k + 1] = std::sin(ph);
      }
      EWB_CUDA(cudaMalloc(&dtab, sizeof(double) * 3 * N), "ewb_window_idft");
      // ordered on the caller's stream (a non-blocking stream would not wait
      // for a legacy-stream copy); the host table must outlive the copy
      EWB_CUDA(cudaMemcpyAsync(dtab, tab.data(), sizeof(double) * 3 * N, cudaMemcpyHostToDevice,
                               S(stream)),
               "ewb_window_idft");
      EWB_CUDA(cudaStreamSynchronize(S(stream)), "ewb_window_idft");
      cache[{dev, N, window}] = dtab;
    }
  }
  double dt = period / (double)N;
  EWB_CUDA(ewb::launch_window_idft((const ewb::cplx*)half, n_half, D, (const double*)dtab,
                                   (const ewb::cplx*)((double*)dtab + N), eta * dt, out, residue,
                                   S(stream)),
           "ewb_window_idft");
  return EWB_OK;
}

}  // extern "C"

namespace ewb {
cudaError_t launch_math_selftest(const double* x, long long n, double* s, double* c, double* e,
                                 cudaStream_t st);
cudaError_t launch_math_selftest_delta(const double* t, long long n, double* e, cudaStream_t st);
}

// ---------------------------------------------------------------------
// matrix-free, pair-kernel microbenchmark, FP64 probe
// ---------------------------------------------------------------------
namespace ewb {
size_t mf_workspace_bytes(const Context& c, int K);
cudaError_t launch_matfree(Context& c, double ore, double oim, const cplx* vt, const cplx* vu,
                           int K, cplx* y, const uint8_t* kinds, cplx* pinv, void* ws,
                           const int* gate, cudaStream_t s, unsigned t_mask, unsigned u_mask);
cudaError_t launch_pair_blocks(const double* x, long long P, const double* tri, long long M,
                               const FreqConst* fcs_dev, int F, const double* b7, const double* w7,
                               cplx* u, cplx* t, cudaStream_t s);
cudaError_t launch_pair_reduce(const double* x, long long P, const double* tri, long long M,
                               const cplx* xv, const FreqConst* fcs_dev, int F, const double* b7,
                               const double* w7, cplx* yu, cplx* yt, cplx* part, int nchunk,
                               cudaStream_t s);
cudaError_t fp64_peak_probe(long long iters, int blocks_per_sm, double* tflops, double* ms,
                            cudaStream_t s);
}  // namespace ewb

// triangle chunks of the fused pair reduction: 148 x 16 CTAs per frequency
// (148 x 4 measured 1.4 % slower on cfg3: 7.60e9 vs 7.70e9 pair-evals/s)
#ifndef EWB_PK_CTAS_PER_SM
#define EWB_PK_CTAS_PER_SM 16
#endif
static int pair_chunks(int64_t P, int64_t M) {
  (void)M;
  int64_t pblocks = (P + 127) / 128;
  int64_t want = (148 * EWB_PK_CTAS_PER_SM + pblocks - 1) / pblocks;
  if (want < 1) want = 1;
  if (want > 16) want = 16;
  return (int)want;
}

// gauss7 tables exactly as quadrature.py:75-88 builds them.
static void gauss7_tables(double b7[21], double w7[7]) {
  double s15 = std::sqrt(15.0);
  double a = (6.0 + s15) / 21.0, b = (6.0 - s15) / 21.0;
  double wa = (155.0 + s15) / 1200.0, wb = (155.0 - s15) / 1200.0;
  b7[0] = b7[1] = b7[2] = 1.0 / 3;
  w7[0] = 9.0 / 40.0;
  int q = 1;
  for (int g = 0; g < 2; ++g) {
    double v = g == 0 ? a : b, w = g == 0 ? wa : wb, o = 1 - 2 * v;
    double pts[3][3] = {{v, v, o}, {v, o, v}, {o, v, v}};
    for (int k = 0; k < 3; ++k, ++q) {
      for (int c = 0; c < 3; ++c) b7[3 * q + c] = pts[k][c];
      w7[q] = w;
    }
  }
}

extern "C" {

int64_t ewb_matfree_workspace_bytes(const ewb_ctx* ctx, int32_t K) {
  if (!ctx || K < 1 || K > 5) return -1;
  return (int64_t)ewb::mf_workspace_bytes(ctx->c, K);
}

int ewb_matfree_apply_masked(ewb_ctx* ctx, double ore, double oim, const void* vt,
                             const void* vu, int32_t K, uint32_t t_mask, uint32_t u_mask, void* y,
                             const uint8_t* kinds, void* pinv, void* ws, int64_t ws_bytes,
                             const int32_t* gate, void* stream) {
  if (!ctx || !vt || !y || !ws) return fail(EWB_ERR_INVALID, "ewb_matfree_apply: null argument");
  if (K < 1 || K > 5) return fail(EWB_ERR_INVALID, "ewb_matfree_apply: K must be in [1, 5]");
  if (int rc = check_omega(ore, oim, "ewb_matfree_apply")) return rc;
  if (ws_bytes < (int64_t)ewb::mf_workspace_bytes(ctx->c, K))
    return fail(EWB_ERR_INVALID, "ewb_matfree_apply: workspace too small");
  const uint32_t all = (1u << K) - 1u;
  if ((t_mask & ~all) || (u_mask & ~all))
    return fail(EWB_ERR_INVALID, "ewb_matfree_apply: mask bits beyond K");
  if (!gate) {  // a gated call may skip its work and must leave y alone
    EWB_CUDA(ewb::dbg_poison(ws, (size_t)ws_bytes, S(stream)), "ewb_matfree_apply");
    EWB_CUDA(ewb::dbg_poison(y, (size_t)K * 3 * ctx->c.n_e * 16, S(stream)), "ewb_matfree_apply");
  }
  EWB_CUDA(ewb::launch_matfree(ctx->c, ore, oim, (const ewb::cplx*)vt, (const ewb::cplx*)vu, K,
                               (ewb::cplx*)y, kinds, (ewb::cplx*)pinv, ws, gate, S(stream),
                               t_mask, u_mask),
           "ewb_matfree_apply");
  return EWB_OK;
}

int ewb_matfree_apply(ewb_ctx* ctx, double ore, double oim, const void* vt, const void* vu,
                      int32_t K, void* y, const uint8_t* kinds, void* pinv, void* ws,
                      int64_t ws_bytes, const int32_t* gate, void* stream) {
  const uint32_t all = K >= 1 && K <= 5 ? (1u << K) - 1u : 0u;
  return ewb_matfree_apply_masked(ctx, ore, oim, vt, vu, K, all, all, y, kinds, pinv, ws,
                                  ws_bytes, gate, stream);
}

static int pair_prep(const double* omega_host, int32_t F, double lam, double mu, double rho,
                     cudaStream_t s, void** dev_tables) {
  // tables: FreqConst[F] | b7[21] | w7[7]
  ewb::Context tmp;
  tmp.lam = lam; tmp.mu = mu; tmp.rho = rho;
  std::vector<ewb::FreqConst> fcs(F);
  for (int f = 0; f < F; ++f) fcs[f] = ewb::freq_const(tmp, omega_host[2 * f], omega_host[2 * f + 1]);
  double b7[21], w7[7];
  gauss7_tables(b7, w7);
  size_t bytes = sizeof(ewb::FreqConst) * F + 28 * 8;
  std::vector<unsigned char> h(bytes);
  memcpy(h.data(), fcs.data(), sizeof(ewb::FreqConst) * F);
  memcpy(h.data() + sizeof(ewb::FreqConst) * F, b7, 21 * 8);
  memcpy(h.data() + sizeof(ewb::FreqConst) * F + 21 * 8, w7, 7 * 8);
  keep_pool_memory();
  EWB_CUDA(cudaMallocAsync(dev_tables, bytes, s), "pair kernels");
  EWB_CUDA(cudaMemcpyAsync(*dev_tables, h.data(), bytes, cudaMemcpyHostToDevice, s), "pair kernels");
  EWB_CUDA(cudaStreamSynchronize(s), "pair kernels");
  return EWB_OK;
}

int ewb_pair_kernels_blocks(const double* x, int64_t P, const double* tri, int64_t M,
                            const double* omega_host, int32_t F, double lam, double mu, double rho,
                            void* u, void* t, void* stream) {
  if (!x || !tri || !omega_host || !u || !t || P < 1 || M < 1 || F < 1)
    return fail(EWB_ERR_INVALID, "ewb_pair_kernels_blocks: bad argument");
  for (int f = 0; f < F; ++f)
    if (int rc = check_omega(omega_host[2 * f], omega_host[2 * f + 1], "ewb_pair_kernels_blocks"))
      return rc;
  void* tab = nullptr;
  if (int rc = pair_prep(omega_host, F, lam, mu, rho, S(stream), &tab)) return rc;
  auto* fcs = (const ewb::FreqConst*)tab;
  const double* b7 = (const double*)((unsigned char*)tab + sizeof(ewb::FreqConst) * F);
  EWB_CUDA(ewb::launch_pair_blocks(x, P, tri, M, fcs, F, b7, b7 + 21, (ewb::cplx*)u,
                                   (ewb::cplx*)t, S(stream)),
           "ewb_pair_kernels_blocks");
  EWB_CUDA(cudaFreeAsync(tab, S(stream)), "ewb_pair_kernels_blocks");
  return EWB_OK;
}

int64_t ewb_pair_kernels_workspace_bytes(int64_t P, int64_t M, int32_t F) {
  return (int64_t)pair_chunks(P, M) * F * P * 6 * 16;
}

int ewb_pair_kernels_reduce(const double* x, int64_t P, const double* tri, int64_t M,
                            const void* xv, const double* omega_host, int32_t F, double lam,
                            double mu, double rho, void* yu, void* yt, void* ws, int64_t ws_bytes,
                            void* stream) {
  if (!x || !tri || !xv || !omega_host || !yu || !yt || !ws || P < 1 || M < 1 || F < 1)
    return fail(EWB_ERR_INVALID, "ewb_pair_kernels_reduce: bad argument");
  if (ws_bytes < ewb_pair_kernels_workspace_bytes(P, M, F))
    return fail(EWB_ERR_INVALID, "ewb_pair_kernels_reduce: workspace too small");
  for (int f = 0; f < F; ++f)
    if (int rc = check_omega(omega_host[2 * f], omega_host[2 * f + 1], "ewb_pair_kernels_reduce"))
      return rc;
  void* tab = nullptr;
  if (int rc = pair_prep(omega_host, F, lam, mu, rho, S(stream), &tab)) return rc;
  auto* fcs = (const ewb::FreqConst*)tab;
  const double* b7 = (const double*)((unsigned char*)tab + sizeof(ewb::FreqConst) * F);
  EWB_CUDA(ewb::launch_pair_reduce(x, P, tri, M, (const ewb::cplx*)xv, fcs, F, b7, b7 + 21,
                                   (ewb::cplx*)yu, (ewb::cplx*)yt, (ewb::cplx*)ws,
                                   pair_chunks(P, M), S(stream)),
           "ewb_pair_kernels_reduce");
  EWB_CUDA(cudaFreeAsync(tab, S(stream)), "ewb_pair_kernels_reduce");
  return EWB_OK;
}

int ewb_fp64_peak_probe(int64_t iters, int32_t blocks_per_sm, double* tflops, double* ms,
                        void* stream) {
  if (!tflops || !ms || iters < 1 || blocks_per_sm < 1)
    return fail(EWB_ERR_INVALID, "ewb_fp64_peak_probe: bad argument");
  EWB_CUDA(ewb::fp64_peak_probe(iters, blocks_per_sm, tflops, ms, S(stream)), "ewb_fp64_peak_probe");
  return EWB_OK;
}

int ewb_math_selftest(const double* x, int64_t n, double* sin_out, double* cos_out,
                      double* exp_out, void* stream) {
  if (!x || !sin_out || !cos_out || !exp_out || n < 0)
    return fail(EWB_ERR_INVALID, "ewb_math_selftest: bad argument");
  if (n == 0) return EWB_OK;
  double* d = nullptr;
  EWB_CUDA(cudaMalloc(&d, sizeof(double) * 4 * n), "ewb_math_selftest");
  cudaStream_t s = S(stream);
  cudaError_t e = cudaMemcpyAsync(d, x, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (!e) e = ewb::launch_math_selftest(d, n, d + n, d + 2 * n, d + 3 * n, s);
  if (!e) e = cudaMemcpyAsync(sin_out, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaMemcpyAsync(cos_out, d + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaMemcpyAsync(exp_out, d + 3 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  cudaFree(d);
  EWB_CUDA(e, "ewb_math_selftest");
  return EWB_OK;
}

int ewb_math_selftest_delta(const double* t, int64_t n, double* exp_out, void* stream) {
  if (!t || !exp_out || n < 0) return fail(EWB_ERR_INVALID, "ewb_math_selftest_delta: bad argument");
  for (int64_t i = 0; i < n; ++i)
    if (!(t[i] >= -0.0625 && t[i] <= 0.0625))
      return fail(EWB_ERR_INVALID, "ewb_math_selftest_delta: |t| > 2^-4");
  if (n == 0) return EWB_OK;
  double* d = nullptr;
  EWB_CUDA(cudaMalloc(&d, sizeof(double) * 2 * n), "ewb_math_selftest_delta");
  cudaStream_t s = S(stream);
  cudaError_t e = cudaMemcpyAsync(d, t, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (!e) e = ewb::launch_math_selftest_delta(d, n, d + n, s);
  if (!e) e = cudaMemcpyAsync(exp_out, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  cudaFree(d);
  EWB_CUDA(e, "ewb_math_selftest_delta");
  return EWB_OK;
}

int ewb_debug_checks(int64_t* failures, int64_t* first_site, int32_t reset) {
  if (!failures || !first_site) return fail(EWB_ERR_INVALID, "ewb_debug_checks: null argument");
  EWB_CUDA(cudaDeviceSynchronize(), "ewb_debug_checks");
  if (!ewb::kDebugChecks) {
    *failures = -1;
    *first_site = 0;
    return EWB_OK;
  }
  unsigned long long v[4][2];
  ewb::dbg_fetch_assembly(v[0]);
  ewb::dbg_fetch_krylov(v[1]);
  ewb::dbg_fetch_matfree(v[2]);
  ewb::dbg_fetch_spectral(v[3]);
  int64_t total = 0, site = 0;
  for (auto& t : v) {
    total += (int64_t)t[0];
    if (!site && t[0]) site = (int64_t)t[1];
  }
  *failures = total;
  *first_site = site;
  if (reset) {
    ewb::dbg_reset_assembly();
    ewb::dbg_reset_krylov();
    ewb::dbg_reset_matfree();
    ewb::dbg_reset_spectral();
  }
  EWB_CUDA(cudaGetLastError(), "ewb_debug_checks");
  return EWB_OK;
}

}  // extern "C"
