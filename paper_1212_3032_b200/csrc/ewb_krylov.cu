// sm_100a Krylov solver: the reference's right-preconditioned restarted
// GMRES (linsolve.py:107-210), its least-squares solution-extrapolation
// initial guess (linsolve.py:213-242) and the dense complex matvec
// (linsolve.py:73-77), as persistent cooperative kernels.
//
// One launch runs a whole solve: the grid stays resident, phases are
// separated by grid-wide barriers, and every global reduction is summed in
// a fixed order (block partials -> every block re-reduces the same
// partials the same way), so all blocks agree bit-for-bit on every scalar
// (Arnoldi coefficients, Givens rotations, residual estimates) and make
// the same convergence decisions without a host round trip.  The host
// sees one launch and one small read-back per frequency.
//
// The matvec streams A once per application with 16-byte loads; a warp
// owns R rows at a time so each x-element load feeds R FMAs.  MGS is kept
// (not CGS) for iteration-count parity: step i of the orthogonalisation
// fuses "w -= h_i v_i" with the partial dot of step i+1, one barrier each.
#include <cooperative_groups.h>
#include <vector>
#include <cuda_runtime.h>

#include "ewb_common.cuh"
#include "ewb_krylov.cuh"

namespace cg = cooperative_groups;

namespace ewb {

#ifndef EWB_SOLVE_THREADS
#define EWB_SOLVE_THREADS 512
#endif
constexpr int kSolveThreads = EWB_SOLVE_THREADS;
// register cap 65536 / (kSolveThreads * kSolveMinBlocks) = 128: with 256 threads a
// solver CTA leaves half of the register file to co-resident assembly CTAs
constexpr int kSolveMinBlocks = 512 / kSolveThreads;
constexpr int kSolveWarps = kSolveThreads / 32;
constexpr int kMaxRed = 16;  // doubles per grid reduction

__device__ __forceinline__ cplx ldc(const cplx* p) {
  double2 v = __ldcs(reinterpret_cast<const double2*>(p));  // streaming (evict-first)
  return {v.x, v.y};
}
__device__ __forceinline__ cplx ldg(const cplx* p) {
  double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}

// Deterministic grid-wide sum of C doubles per thread.  `red` alternates
// between two partial buffers so a fast block never overwrites partials a
// slow block is still reading.
struct GridRed {
  double* partial;  // [2][G][kMaxRed]
  int parity;
};

template <int C>
__device__ void grid_sum(cg::grid_group& grid, GridRed& R, double (&v)[C]) {
  __shared__ double s_w[kSolveWarps][kMaxRed];
  __shared__ double s_out[kMaxRed];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    warp_sum(v[c]);
    if (lane == 0) s_w[wid][c] = v[c];
  }
  __syncthreads();
  double* part = R.partial + (size_t)R.parity * gridDim.x * kMaxRed;
  if (threadIdx.x < C) {
    double s = 0.0;
    for (int w = 0; w < kSolveWarps; ++w) s += s_w[w][threadIdx.x];
    part[(size_t)blockIdx.x * kMaxRed + threadIdx.x] = s;
  }
  grid.sync();
  if (wid == 0) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double s = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) s += part[(size_t)b * kMaxRed + c];
      warp_sum(s);
      if (lane == 0) s_out[c] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < C; ++c) v[c] = s_out[c];
  __syncthreads();
  R.parity ^= 1;
}

// y[:, k] = A x[:, k] for K right-hand sides (x, y stored column after
// column, leading dimension n).  Rows are dealt to warps R at a time.
template <int RR, int K>
__device__ void matvec_grid(const cplx* __restrict__ A, long long n, const cplx* x, cplx* y) {
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r0 = gw * RR; r0 < n; r0 += nw * RR) {
    cplx acc[RR][K];
#pragma unroll
    for (int a = 0; a < RR; ++a)
#pragma unroll
      for (int k = 0; k < K; ++k) acc[a][k] = {0.0, 0.0};
    const int nr = (int)min((long long)RR, n - r0);
    if (nr == RR) {
      const cplx* rowp = A + r0 * n;
#pragma unroll 2
      for (long long c = lane; c < n; c += 32) {
        cplx xv[K];
#pragma unroll
        for (int k = 0; k < K; ++k) xv[k] = ldg(x + k * n + c);
#pragma unroll
        for (int a = 0; a < RR; ++a) {
          cplx av = ldc(rowp + a * n + c);
#pragma unroll
          for (int k = 0; k < K; ++k) cfma(acc[a][k], av, xv[k]);
        }
      }
    } else {
      for (long long c = lane; c < n; c += 32) {
        cplx xv[K];
#pragma unroll
        for (int k = 0; k < K; ++k) xv[k] = ldg(x + k * n + c);
        for (int a = 0; a < nr; ++a) {
          cplx av = ldc(A + (r0 + a) * n + c);
#pragma unroll
          for (int k = 0; k < K; ++k) cfma(acc[a][k], av, xv[k]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < RR; ++a)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        warp_sum(acc[a][k]);
        if (lane == 0 && a < nr) y[k * n + r0 + a] = acc[a][k];
      }
  }
}

// ---------------------------------------------------------------------
// TMA (cp.async.bulk) matvec.  Row groups of kRR rows are dealt to CTAs
// round-robin; each CTA streams its groups through a kNS-stage ring of
// shared-memory tiles (kRR rows x kTC columns = 32 KB), one bulk copy per
// row segment, completion tracked by a transaction-count mbarrier per
// stage.  Thread t owns column t % kTC of every tile for kRR/2 rows; the
// per-row sums are reduced across the CTA at the end of each row group.
// Up to kNS x 32 KB = 192 KB per SM are in flight with no register cost.
// ---------------------------------------------------------------------
#ifndef EWB_RING_RR
#define EWB_RING_RR 16
#endif
#ifndef EWB_RING_TC
#define EWB_RING_TC 256
#endif
#ifndef EWB_RING_NS
#define EWB_RING_NS 3
#endif
constexpr int kRR = EWB_RING_RR;
constexpr int kTC = EWB_RING_TC;
constexpr int kNS = EWB_RING_NS;
constexpr int kStageElems = kRR * kTC;
constexpr int kRingBytes = kNS * kStageElems * 16;
constexpr int kSlices = kSolveThreads / kTC;     // row slices per tile
constexpr int kRpt = kRR / kSlices;              // rows per thread
static_assert(kSolveThreads % kTC == 0 && kRR % kSlices == 0, "tile geometry");

struct Ring {
  cplx* buf;            // dynamic shared memory, kNS stages
  uint64_t* bar;        // kNS mbarriers (static shared)
  unsigned pos;         // stages consumed so far by this CTA (uniform)
  unsigned evict_first; // L2 policy for A: evict_first (A larger than L2) or evict_last
};

// Optional L2 residency of part of A: the first kPinRows rows of every CTA's
// slice are loaded evict_last, the rest evict_first, so ~kPinRows x 148 rows
// stay in L2 across passes.  Measured (n = 15360): 2 rows lift a standalone
// GEMV from 6.76 to 6.88 TB/s but slow the cfg2 sweep from 4.02 to 4.09 s
// (the pinned rows crowd the Krylov basis out of L2), so it is off.
#ifndef EWB_X_PREFETCH
#define EWB_X_PREFETCH 0
#endif
#ifndef EWB_L2_PREFETCH_TILES
#define EWB_L2_PREFETCH_TILES 0
#endif
#ifndef EWB_PIN_ROWS
#define EWB_PIN_ROWS 0
#endif
constexpr int kPinRows = EWB_PIN_ROWS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void ring_init(Ring& R, bool evict_first) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&R.bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  R.evict_first = evict_first ? 1u : 0u;
  R.pos = 0;
  __syncthreads();
}

__device__ __forceinline__ void ring_issue(const Ring& R, unsigned pos, const cplx* A, long long n,
                                           long long row0, int nrows, long long c0, int tc,
                                           int npin = 0) {
  const int b = pos % kNS;
  const uint32_t bar = smem_u32(&R.bar[b]);
  const uint32_t bytes = (uint32_t)(nrows * tc * 16);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  // policies are made here (issuing thread only) instead of living in
  // registers of every thread across the whole solve
  uint64_t stream_pol, pin_pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pin_pol));
  if (R.evict_first)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream_pol));
  else
    stream_pol = pin_pol;
  if (kPinRows == 0) npin = 0;
  for (int r = 0; r < nrows; ++r) {
    const uint32_t dst = smem_u32(R.buf + (size_t)b * kStageElems + r * kTC);
    const cplx* src = A + (row0 + r) * n + c0;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(tc * 16), "r"(bar), "l"(r < npin ? pin_pol : stream_pol)
        : "memory");
  }
}

__device__ __forceinline__ void ring_wait(const Ring& R, unsigned pos) {
  const uint32_t bar = smem_u32(&R.bar[pos % kNS]);
  const uint32_t parity = (pos / kNS) & 1u;
#ifdef EWB_WAIT_HINT   // experiment: suspend-time hint (ns) for the waiting warps
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity), "n"(EWB_WAIT_HINT)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
#endif
}

// y[k] = A x[k] for K vectors (x, y: vector k at +k n), all CTAs cooperate;
// the caller separates phases with grid.sync().
template <int K>
__device__ void matvec_tma(Ring& R, const cplx* __restrict__ A, long long n, const cplx* x,
                           cplx* y) {
  __shared__ cplx s_red[kSolveWarps][kRpt][K];
  const long long ngroups = (n + kRR - 1) / kRR;
  const int ntile = (int)((n + kTC - 1) / kTC);
  const long long mine = ngroups > blockIdx.x ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long S = mine * ntile;
  auto coords = [&](long long s, long long& row0, int& nrows, long long& c0, int& tc) {
    const long long gi = s / ntile;
    const int t = (int)(s % ntile);
    row0 = (blockIdx.x + gi * gridDim.x) * kRR;
    nrows = (int)min((long long)kRR, n - row0);
    c0 = (long long)t * kTC;
    tc = (int)min((long long)kTC, n - c0);
  };
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (long long s = 0; s < S && s < kNS; ++s) {
      long long row0, c0;
      int nrows, tc;
      coords(s, row0, nrows, c0, tc);
      ring_issue(R, R.pos + (unsigned)s, A, n, row0, nrows, c0, tc);
    }
  }
  const int col = threadIdx.x % kTC, slice = threadIdx.x / kTC;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  cplx acc[kRpt][K];
#pragma unroll
  for (int r = 0; r < kRpt; ++r)
#pragma unroll
    for (int k = 0; k < K; ++k) acc[r][k] = {0.0, 0.0};
  for (long long s = 0; s < S; ++s) {
    long long row0, c0;
    int nrows, tc;
    coords(s, row0, nrows, c0, tc);
    const unsigned pos = R.pos + (unsigned)s;
    ring_wait(R, pos);
    if (col < tc) {
      cplx xv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) xv[k] = ldg(x + k * n + c0 + col);
      const cplx* tile = R.buf + (size_t)(pos % kNS) * kStageElems;
#pragma unroll
      for (int r = 0; r < kRpt; ++r) {
        const int row = slice * kRpt + r;
        if (row < nrows) {
          double2 a2 = *reinterpret_cast<const double2*>(tile + row * kTC + col);
          cplx av = {a2.x, a2.y};
#pragma unroll
          for (int k = 0; k < K; ++k) cfma(acc[r][k], av, xv[k]);
        }
      }
    }
    __syncthreads();  // every consumer is done with this stage's buffer
    if (threadIdx.x == 0 && s + kNS < S) {
      long long r2, c2;
      int n2, t2;
      coords(s + kNS, r2, n2, c2, t2);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      ring_issue(R, pos + kNS, A, n, r2, n2, c2, t2);
    }
    if (c0 + tc >= n) {  // last tile of the row group: reduce and store
#pragma unroll
      for (int r = 0; r < kRpt; ++r)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          warp_sum(acc[r][k]);
          if (lane == 0) s_red[wid][r][k] = acc[r][k];
          acc[r][k] = {0.0, 0.0};
        }
      __syncthreads();
      if (threadIdx.x < kRR * K) {
        const int row = threadIdx.x / K, k = threadIdx.x % K;
        const int h = row / kRpt, r = row % kRpt;
        constexpr int wps = kSolveWarps / kSlices;  // warps per row slice
        cplx sum = {0.0, 0.0};
        for (int w = 0; w < wps; ++w) sum = sum + s_red[h * wps + w][r][k];
        if (row < nrows) y[k * n + row0 + row] = sum;
      }
      __syncthreads();
    }
  }
  R.pos += (unsigned)S;
}

// One out-of-line copy of the single-vector matvec for the GMRES kernel:
// every call site shares the same (register-allocated once) code.  The ring
// travels by value and the new position is returned, so nothing is spilled.
__device__ __noinline__ unsigned matvec1_nl(Ring R, const cplx* __restrict__ A, long long n,
                                            const cplx* x, cplx* y) {
  matvec_tma<1>(R, A, n, x, y);
  return R.pos;
}
// (measured: the out-of-line copy is ~15 % slower than inlining; kept for
// A/B tests with -DEWB_MATVEC_NOINLINE)
#ifndef EWB_MATVEC_NOINLINE
#define EWB_MATVEC1(ring, A, n, x, y) matvec_tma<1>(ring, A, n, x, y)
#else
#define EWB_MATVEC1(ring, A, n, x, y) (ring).pos = matvec1_nl(ring, A, n, x, y)
#endif

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// optional phase trace (CTA 0): (phase << 56) | %globaltimer
#define EWB_PROBE(id)                                                                  \
  do {                                                                                 \
    if (a.probe && blockIdx.x == 0 && threadIdx.x == 0 && n_probe < a.probe_cap)       \
      a.probe[n_probe++] = ((unsigned long long)(id) << 56) |                          \
                           (gtimer() & ((1ull << 56) - 1));                            \
  } while (0)

// z = P^{-1} v  (3x3 blocks; identity when pinv == nullptr).  Grid-stride
// over elements: thread e owns DOFs 3e..3e+2.
__device__ __forceinline__ void precond_apply_elem(const cplx* pinv, long long e, const cplx* v,
                                                   cplx* z) {
  cplx v0 = v[3 * e], v1 = v[3 * e + 1], v2 = v[3 * e + 2];
  const cplx* P = pinv + 9 * e;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    // numpy einsum('bij,bj->bi') order: ((P0 v0 + P1 v1) + P2 v2)
    cplx s = P[3 * a] * v0;
    s = s + P[3 * a + 1] * v1;
    s = s + P[3 * a + 2] * v2;
    z[3 * e + a] = s;
  }
}

__device__ __forceinline__ long long gtid() {
  return (long long)blockIdx.x * blockDim.x + threadIdx.x;
}
__device__ __forceinline__ long long gthreads() { return (long long)gridDim.x * blockDim.x; }

// Givens state kept redundantly (and identically) in every block.
struct GivensShared {
  cplx cs[kMaxRestart], sn[kMaxRestart], g[kMaxRestart + 1];
  cplx h[kMaxRestart + 1];
};

// Classic sequential MGS (one grid barrier per projection) — kept as the
// GmresArgs::ortho == 1 variant for A/B parity checks.
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_gmres_mgs(GmresArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char ring_smem[];
  __shared__ uint64_t ring_bar[kNS];
  Ring ring{reinterpret_cast<cplx*>(ring_smem), ring_bar, 0u, 0u};
  ring_init(ring, 16.0 * (double)a.n * (double)a.n > 96e6);
  __shared__ GivensShared gs;
  __shared__ cplx s_y[kMaxRestart];
  const long long n = a.n;
  const long long tid = gtid(), nth = gthreads();
  const bool have_pc = a.pinv != nullptr;
  GridRed R{a.partial, 0};
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  // ||b||
  double v1[1] = {0.0};
  for (long long k = tid; k < n; k += nth) v1[0] += abs2(a.b[k]);
  grid_sum(grid, R, v1);
  const double nb = sqrt(v1[0]);
  if (nb == 0.0) {  // linsolve.py:136-140
    for (long long k = tid; k < n; k += nth) a.x[k] = {0.0, 0.0};
    if (tid == 0) { a.out->iterations = 0; a.out->init_res = 0; a.out->final_res = 0;
                    a.out->n_hist = 0; a.out->converged = 1; a.out->matvecs = 0; }
    return;
  }
  int n_mv = 0;
  // r = b - A x0  (skipped when x0 is all zero: linsolve.py:144)
  double anyv[1] = {0.0};
  if (a.has_x0)
    for (long long k = tid; k < n; k += nth) anyv[0] += (a.x[k].re != 0.0 || a.x[k].im != 0.0);
  else
    for (long long k = tid; k < n; k += nth) a.x[k] = {0.0, 0.0};
  grid_sum(grid, R, anyv);
  if (anyv[0] > 0.0) {
    matvec_tma<1>(ring, a.A, n, a.x, a.w);
    ++n_mv;
    grid.sync();
    for (long long k = tid; k < n; k += nth) a.r[k] = a.b[k] - a.w[k];
  } else {
    for (long long k = tid; k < n; k += nth) a.r[k] = a.b[k];
  }
  double rr[1] = {0.0};
  for (long long k = tid; k < n; k += nth) rr[0] += abs2(a.r[k]);
  grid_sum(grid, R, rr);
  double rnorm = sqrt(rr[0]);
  double res = rnorm / nb;
  int n_hist = 0;
  if (tid == 0) { a.out->init_res = res; a.hist[n_hist] = res; }
  n_hist++;
  int its = 0;
  while (res > a.tol && its < a.maxiter) {
    const int m = min(a.restart, a.maxiter - its);
    const double beta = rnorm;
    // V0 = r / beta ; z = P^{-1} V0
    for (long long k = tid; k < n; k += nth) {
      cplx v = a.r[k];
      a.V[k] = {v.re / beta, v.im / beta};
    }
    if (threadIdx.x == 0) {
      gs.g[0] = {beta, 0.0};
      for (int k = 1; k <= m; ++k) gs.g[k] = {0.0, 0.0};
    }
    grid.sync();
    int used = 0;
    for (int j = 0; j < m; ++j) {
      const cplx* vj = a.V + (size_t)j * n;
      // z = P^{-1} v_j
      if (have_pc) {
        for (long long e = tid; e < n / 3; e += nth) precond_apply_elem(a.pinv, e, vj, a.z);
      } else {
        for (long long k = tid; k < n; k += nth) a.z[k] = vj[k];
      }
      grid.sync();
      matvec_tma<1>(ring, a.A, n, a.z, a.w);
      ++n_mv;
      grid.sync();
      // MGS, fused: partial <v_0, w>
      double dv[2] = {0.0, 0.0};
      for (long long k = tid; k < n; k += nth) {
        cplx p = conj(a.V[k]) * a.w[k];
        dv[0] += p.re; dv[1] += p.im;
      }
      for (int i = 0; i <= j; ++i) {
        grid_sum(grid, R, dv);
        const cplx h = {dv[0], dv[1]};
        if (threadIdx.x == 0) gs.h[i] = h;
        const cplx* vi = a.V + (size_t)i * n;
        const cplx* vn = a.V + (size_t)(i + 1) * n;
        dv[0] = dv[1] = 0.0;
        if (i < j) {
          for (long long k = tid; k < n; k += nth) {
            cplx w = a.w[k] - h * vi[k];
            a.w[k] = w;
            cplx p = conj(vn[k]) * w;
            dv[0] += p.re; dv[1] += p.im;
          }
        } else {
          for (long long k = tid; k < n; k += nth) {
            cplx w = a.w[k] - h * vi[k];
            a.w[k] = w;
            dv[0] += abs2(w);
          }
        }
      }
      double nw[1] = {dv[0]};
      grid_sum(grid, R, nw);
      const double hn = sqrt(nw[0]);
      if (hn > 0.0) {
        cplx* vn = a.V + (size_t)(j + 1) * n;
        for (long long k = tid; k < n; k += nth) {
          cplx w = a.w[k];
          vn[k] = {w.re / hn, w.im / hn};
        }
      }
      // Givens (linsolve.py:171-194), identical in every block
      if (threadIdx.x == 0) {
        gs.h[j + 1] = {hn, 0.0};
        for (int i = 0; i < j; ++i) {
          cplx top = gs.cs[i] * gs.h[i] + gs.sn[i] * gs.h[i + 1];
          gs.h[i + 1] = (-conj(gs.sn[i])) * gs.h[i] + conj(gs.cs[i]) * gs.h[i + 1];
          gs.h[i] = top;
        }
        double ahj = hypot(gs.h[j].re, gs.h[j].im), ahn = hypot(gs.h[j + 1].re, gs.h[j + 1].im);
        double den = sqrt(ahj * ahj + ahn * ahn);
        if (den == 0.0) {
          gs.cs[j] = {1.0, 0.0}; gs.sn[j] = {0.0, 0.0};
        } else if (gs.h[j].re == 0.0 && gs.h[j].im == 0.0) {
          gs.cs[j] = {0.0, 0.0}; gs.sn[j] = {1.0, 0.0};
        } else {
          gs.cs[j] = {ahj / den, 0.0};
          cplx ph = {gs.h[j].re / ahj, gs.h[j].im / ahj};
          cplx t = ph * conj(gs.h[j + 1]);
          gs.sn[j] = {t.re / den, t.im / den};
        }
        gs.h[j] = gs.cs[j] * gs.h[j] + gs.sn[j] * gs.h[j + 1];
        gs.h[j + 1] = {0.0, 0.0};
        gs.g[j + 1] = (-conj(gs.sn[j])) * gs.g[j];
        gs.g[j] = gs.cs[j] * gs.g[j];
        if (blockIdx.x == 0) {
          for (int i = 0; i <= j; ++i) a.H[(size_t)i * kMaxRestart + j] = gs.h[i];
        }
      }
      __syncthreads();
      ++its;
      used = j + 1;
      const double est = hypot(gs.g[j + 1].re, gs.g[j + 1].im) / nb;
      if (tid == 0 && n_hist < a.hist_cap) a.hist[n_hist] = est;
      n_hist++;
      grid.sync();  // V_{j+1} complete, H visible
      if (est <= a.tol) break;
    }
    // back substitution (linsolve.py:196-198): warp 0 of every block
    if (wid == 0) {
      for (int i = used - 1; i >= 0; --i) {
        cplx s = {0.0, 0.0};
        for (int k = i + 1 + lane; k < used; k += 32) s = s + a.H[(size_t)i * kMaxRestart + k] * s_y[k];
        warp_sum(s);
        if (lane == 0) s_y[i] = cdiv(gs.g[i] - s, a.H[(size_t)i * kMaxRestart + i]);
        __syncwarp();
      }
    }
    __syncthreads();
    // x += P^{-1} (V^T y)   (u in w as scratch)
    for (long long k = tid; k < n; k += nth) {
      cplx u = {0.0, 0.0};
      for (int i = 0; i < used; ++i) cfma(u, a.V[(size_t)i * n + k], s_y[i]);
      a.w[k] = u;
    }
    if (have_pc) {
      grid.sync();
      for (long long e = tid; e < n / 3; e += nth) {
        precond_apply_elem(a.pinv, e, a.w, a.z);
        for (int c = 0; c < 3; ++c) a.x[3 * e + c] = a.x[3 * e + c] + a.z[3 * e + c];
      }
    } else {
      for (long long k = tid; k < n; k += nth) a.x[k] = a.x[k] + a.w[k];
    }
    grid.sync();
    // true residual (linsolve.py:200-201)
    matvec_tma<1>(ring, a.A, n, a.x, a.w);
    ++n_mv;
    grid.sync();
    double q[1] = {0.0};
    for (long long k = tid; k < n; k += nth) {
      cplx r = a.b[k] - a.w[k];
      a.r[k] = r;
      q[0] += abs2(r);
    }
    grid_sum(grid, R, q);
    rnorm = sqrt(q[0]);
    res = rnorm / nb;
  }
  if (tid == 0) {
    a.out->iterations = its;
    a.out->final_res = res;
    a.out->converged = res <= a.tol;
    a.out->n_hist = n_hist;
    a.out->matvecs = n_mv;
  }
}

// ---------------------------------------------------------------------
// One-reduction MGS-GMRES (default).  The reference's MGS computes
//   h_i = <v_i, w - sum_{l<i} h_l v_l> = d_i - sum_{l<i} <v_i, v_l> h_l,
// d_i = <v_i, w>, i.e. h = (I + L)^{-1} d with L the strictly lower part of
// the Gram matrix V^H V.  Row j of L (<v_j, v_l>, l < j) is reduced together
// with d in ONE grid reduction, the unit-triangular solve runs redundantly
// (and identically) in every CTA, and w -= h_0 v_0 -= h_1 v_1 ... (the MGS
// update order) plus |w|^2 take the second reduction.  Same algorithm and
// coefficients as MGS up to floating-point association — no approximation —
// with 4 grid barriers per Arnoldi step instead of j + 5.
// ---------------------------------------------------------------------
constexpr int kMaxDots = 2 * kMaxRestart + 2;

// CTA-partial dots over this CTA's DOF slice [k0, k1):
//   t < nd        : <V_t, w>
//   nd <= t < nd+ng: <v_j, V_{t-nd}>
__device__ void slice_dots(const cplx* V, long long n, const cplx* w, int nd, int ng, int j,
                           long long k0, long long k1, cplx* part) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int t = wid; t < nd + ng; t += kSolveWarps) {
    const cplx* p = t < nd ? V + (size_t)t * n : V + (size_t)j * n;
    const cplx* q = t < nd ? w : V + (size_t)(t - nd) * n;
    cplx s = {0.0, 0.0};
    for (long long k = k0 + lane; k < k1; k += 32) cfma(s, conj(p[k]), q[k]);
    warp_sum(s);
    if (lane == 0) part[(size_t)blockIdx.x * kMaxDots + t] = s;
  }
}

// Every CTA reduces the CTA partials in the same fixed order -> s_out.
__device__ void reduce_slices(const cplx* part, int cnt, cplx* s_out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int t = wid; t < cnt; t += kSolveWarps) {
    cplx s = {0.0, 0.0};
    for (int b = lane; b < (int)gridDim.x; b += 32) s = s + part[(size_t)b * kMaxDots + t];
    warp_sum(s);
    if (lane == 0) s_out[t] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void precond_regs(const cplx* pinv, long long e, const cplx v[3],
                                             cplx* z) {
  const cplx* P = pinv + 9 * e;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    cplx s = P[3 * r] * v[0];
    s = s + P[3 * r + 1] * v[1];
    s = s + P[3 * r + 2] * v[2];
    z[3 * e + r] = s;
  }
}

__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_gmres(GmresArgs a) {
  int n_probe = 0;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char ring_smem[];
  __shared__ uint64_t ring_bar[kNS];
  __shared__ GivensShared gs;
  __shared__ cplx s_y[kMaxRestart];
  __shared__ cplx s_dots[kMaxDots];
  __shared__ cplx s_h[kMaxRestart + 1];
  __shared__ double s_est;
  Ring ring{reinterpret_cast<cplx*>(ring_smem), ring_bar, 0u, 0u};
  ring_init(ring, 16.0 * (double)a.n * (double)a.n > 96e6);
  const long long n = a.n;
  const long long tid = gtid(), nth = gthreads();
  const bool pc = a.pinv != nullptr;
  const int ucnt = pc ? 3 : 1;
  const long long nunits = pc ? n / 3 : n;
  const long long k0 = (long long)blockIdx.x * n / gridDim.x;
  const long long k1 = (long long)(blockIdx.x + 1) * n / gridDim.x;
  GridRed R{a.partial, 0};
  int dpar = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  // ||b|| and "x0 has a nonzero entry", one reduction
  double v2[2] = {0.0, 0.0};
  for (long long k = tid; k < n; k += nth) {
    v2[0] += abs2(a.b[k]);
    if (a.has_x0) v2[1] += (a.x[k].re != 0.0 || a.x[k].im != 0.0);
    else a.x[k] = {0.0, 0.0};
  }
  grid_sum(grid, R, v2);
  const double nb = sqrt(v2[0]);
  if (nb == 0.0) {  // linsolve.py:136-140
    for (long long k = tid; k < n; k += nth) a.x[k] = {0.0, 0.0};
    if (tid == 0) { a.out->iterations = 0; a.out->init_res = 0; a.out->final_res = 0;
                    a.out->n_hist = 0; a.out->converged = 1; a.out->matvecs = 0; }
    return;
  }
  int n_mv = 0;
  if (v2[1] > 0.0) {  // r = b - A x0 (linsolve.py:144)
    EWB_MATVEC1(ring, a.A, n, a.x, a.w);
    ++n_mv;
    grid.sync();
    for (long long k = tid; k < n; k += nth) a.r[k] = a.b[k] - a.w[k];
  } else {
    for (long long k = tid; k < n; k += nth) a.r[k] = a.b[k];
  }
  double rr[1] = {0.0};
  for (long long k = tid; k < n; k += nth) rr[0] += abs2(a.r[k]);
  grid_sum(grid, R, rr);
  double rnorm = sqrt(rr[0]);
  double res = rnorm / nb;
  int n_hist = 0;
  if (tid == 0) { a.out->init_res = res; a.hist[0] = res; }
  n_hist++;
  int its = 0;
  while (res > a.tol && its < a.maxiter) {
    const int m = min(a.restart, a.maxiter - its);
    const double beta = rnorm;
    // V0 = r / beta and z = P^{-1} V0, per unit (element or DOF)
    for (long long u = tid; u < nunits; u += nth) {
      cplx v[3];
      for (int c = 0; c < ucnt; ++c) {
        const long long k = u * ucnt + c;
        v[c] = {a.r[k].re / beta, a.r[k].im / beta};
        a.V[k] = v[c];
      }
      if (pc) precond_regs(a.pinv, u, v, a.z);
      else a.z[u] = v[0];
    }
    if (threadIdx.x == 0) {
      gs.g[0] = {beta, 0.0};
      for (int k = 1; k <= m; ++k) gs.g[k] = {0.0, 0.0};
    }
    grid.sync();
    int used = 0;
    for (int j = 0; j < m; ++j) {
#ifdef EWB_DBG_LOOP_X
      EWB_MATVEC1(ring, a.A, n, a.x, a.w);   // timing experiment only
#else
      EWB_MATVEC1(ring, a.A, n, a.z, a.w);   // w = A P^{-1} v_j
#endif
      ++n_mv;
      grid.sync();
      // reduction 1: d_i = <v_i, w> (i <= j) and Gram row j: <v_j, v_l> (l < j)
      cplx* part = a.dpart + (size_t)dpar * gridDim.x * kMaxDots;
      dpar ^= 1;
      EWB_PROBE(20);
#ifdef EWB_DBG_WARM
      for (int rep = 0; rep < 2; ++rep) {  // second pass: same code and data, warm
        slice_dots(a.V, n, a.w, j + 1, j, j, k0, k1, part);
        EWB_PROBE(21 + rep);
      }
#else
      slice_dots(a.V, n, a.w, j + 1, j, j, k0, k1, part);
      EWB_PROBE(21);
#endif
      grid.sync();
      reduce_slices(part, 2 * j + 1, s_dots);
      // h = (I + L)^{-1} d  (warp 0, identical in every CTA).  The Gram rows
      // i < j are first staged (packed, one parallel round trip) into the
      // idle TMA ring — the matvec is complete, nothing is in flight.
      cplx* gsm = ring.buf;
      for (int i = 1; i < j; ++i)
        for (int l = threadIdx.x; l < i; l += blockDim.x)
          gsm[i * (i - 1) / 2 + l] = a.Gram[(size_t)i * kMaxRestart + l];
      __syncthreads();
      if (wid == 0) {
        for (int i = 0; i <= j; ++i) {
          cplx s = {0.0, 0.0};
          for (int l = lane; l < i; l += 32) {
            const cplx g = i == j ? s_dots[j + 1 + l] : gsm[i * (i - 1) / 2 + l];
            s = s + g * s_h[l];
          }
          warp_sum(s);
          if (lane == 0) s_h[i] = s_dots[i] - s;
          __syncwarp();
        }
        if (blockIdx.x == 0)
          for (int l = lane; l < j; l += 32) a.Gram[(size_t)j * kMaxRestart + l] = s_dots[j + 1 + l];
      }
      __syncthreads();
      // w <- (((w - h0 v0) - h1 v1) ... - hj vj)  and |w|^2 (reduction 2)
      double q[1] = {0.0};
      for (long long k = tid; k < n; k += nth) {
        cplx wk = a.w[k];
        for (int i = 0; i <= j; ++i) wk = wk - s_h[i] * a.V[(size_t)i * n + k];
        a.w[k] = wk;
        q[0] += abs2(wk);
      }
      grid_sum(grid, R, q);
      const double hn = sqrt(q[0]);
      // Givens (linsolve.py:171-194), identical in every CTA
      if (threadIdx.x == 0) {
        // apply the previous rotations; only `carry` (the running h_i) is
        // on the dependency chain
        cplx carry = s_h[0];
#pragma unroll 4
        for (int i = 0; i < j; ++i) {
          const cplx c = gs.cs[i], sn = gs.sn[i], hn1 = s_h[i + 1];
          gs.h[i] = c * carry + sn * hn1;
          carry = (-conj(sn)) * carry + conj(c) * hn1;
        }
        gs.h[j] = carry;
        gs.h[j + 1] = {hn, 0.0};
        double ahj = hypot(gs.h[j].re, gs.h[j].im), ahn = hypot(gs.h[j + 1].re, gs.h[j + 1].im);
        double den = sqrt(ahj * ahj + ahn * ahn);
        if (den == 0.0) {
          gs.cs[j] = {1.0, 0.0}; gs.sn[j] = {0.0, 0.0};
        } else if (gs.h[j].re == 0.0 && gs.h[j].im == 0.0) {
          gs.cs[j] = {0.0, 0.0}; gs.sn[j] = {1.0, 0.0};
        } else {
          gs.cs[j] = {ahj / den, 0.0};
          cplx ph = {gs.h[j].re / ahj, gs.h[j].im / ahj};
          cplx t = ph * conj(gs.h[j + 1]);
          gs.sn[j] = {t.re / den, t.im / den};
        }
        gs.h[j] = gs.cs[j] * gs.h[j] + gs.sn[j] * gs.h[j + 1];
        gs.h[j + 1] = {0.0, 0.0};
        gs.g[j + 1] = (-conj(gs.sn[j])) * gs.g[j];
        gs.g[j] = gs.cs[j] * gs.g[j];
        s_est = hypot(gs.g[j + 1].re, gs.g[j + 1].im) / nb;
        if (blockIdx.x == 0)
          for (int i = 0; i <= j; ++i) a.H[(size_t)i * kMaxRestart + j] = gs.h[i];
      }
      __syncthreads();
      ++its;
      used = j + 1;
      const double est = s_est;
      if (tid == 0 && n_hist < a.hist_cap) a.hist[n_hist] = est;
      n_hist++;
      if (est <= a.tol) {
        grid.sync();  // H visible to every CTA before the back substitution
        break;
      }
      // v_{j+1} = w / h_{j+1,j} and z = P^{-1} v_{j+1}
      if (hn > 0.0) {
        cplx* vn = a.V + (size_t)(j + 1) * n;
        for (long long u = tid; u < nunits; u += nth) {
          cplx v[3];
          for (int c = 0; c < ucnt; ++c) {
            const long long k = u * ucnt + c;
            v[c] = {a.w[k].re / hn, a.w[k].im / hn};
            vn[k] = v[c];
          }
          if (pc) precond_regs(a.pinv, u, v, a.z);
          else a.z[u] = v[0];
        }
      }
      grid.sync();
    }
    // back substitution (linsolve.py:196-198): warp 0 of every CTA, with
    // the upper triangle of H staged (packed) into the idle ring first.
    {
      cplx* hsm = ring.buf;
      for (int i = 0; i < used; ++i)
        for (int k = i + threadIdx.x; k < used; k += blockDim.x)
          hsm[i * used - i * (i - 1) / 2 + (k - i)] = a.H[(size_t)i * kMaxRestart + k];
      __syncthreads();
      if (wid == 0) {
        for (int i = used - 1; i >= 0; --i) {
          const cplx* row = hsm + i * used - i * (i - 1) / 2 - i;
          cplx s = {0.0, 0.0};
          for (int k = i + 1 + lane; k < used; k += 32) s = s + row[k] * s_y[k];
          warp_sum(s);
          if (lane == 0) s_y[i] = cdiv(gs.g[i] - s, row[i]);
          __syncwarp();
        }
      }
      __syncthreads();
    }
    // x += P^{-1} (V^T y), per unit
    for (long long u = tid; u < nunits; u += nth) {
      cplx uv[3];
      for (int c = 0; c < ucnt; ++c) {
        const long long k = u * ucnt + c;
        cplx s = {0.0, 0.0};
        for (int i = 0; i < used; ++i) cfma(s, a.V[(size_t)i * n + k], s_y[i]);
        uv[c] = s;
      }
      if (pc) {
        precond_regs(a.pinv, u, uv, a.z);
        for (int c = 0; c < 3; ++c) a.x[3 * u + c] = a.x[3 * u + c] + a.z[3 * u + c];
      } else {
        a.x[u] = a.x[u] + uv[0];
      }
    }
    grid.sync();
    EWB_MATVEC1(ring, a.A, n, a.x, a.w);  // true residual (linsolve.py:200-201)
    ++n_mv;
    grid.sync();
    double q2[1] = {0.0};
    for (long long k = tid; k < n; k += nth) {
      cplx r = a.b[k] - a.w[k];
      a.r[k] = r;
      q2[0] += abs2(r);
    }
    grid_sum(grid, R, q2);
    rnorm = sqrt(q2[0]);
    res = rnorm / nb;
  }
  if (tid == 0) {
    a.out->iterations = its;
    a.out->final_res = res;
    a.out->converged = res <= a.tol;
    a.out->n_hist = n_hist;
    a.out->matvecs = n_mv;
  }
}

// ---------------------------------------------------------------------
// Balanced row-block matvec with a per-block epilogue.
//
// CTA b owns the contiguous rows [b n / G, (b+1) n / G) (at most one row of
// imbalance, where the round-robin 16-row groups above leave up to 8 %),
// cut into ceil(R / kRR) near-equal blocks.  Each block streams through the
// same TMA ring; x is read one stage ahead so its L2 latency overlaps the
// current stage.  When a block's last column tile is consumed its per-row
// sums land in s_sum[row][k] and epi(row0, nrows, s_sum) runs on all
// threads (CTA-uniform), so vector work on the block's rows (scaling,
// residuals, partial dot products) happens while the next stages are
// already in flight.
// ---------------------------------------------------------------------
//
// Row balance.  The matvec bandwidth of an SM under full-GPU contention is
// not uniform: with equal row counts some SMs finish ~25 us (5 %) after the
// others, every pass, and the grid barrier waits for them.  The slowness
// follows the SM, not the rows (swapping the row chunks keeps the slow set:
// tools/gmres_trace.py), and the CTA -> SM map of the solver launches is
// fixed, so ewb_calibrate_rows measures each CTA's rows per second once and
// the row split follows those speeds: CTA b owns [cumw[b] n, cumw[b+1] n).
// Results stay bit-identical for a given split; splits from different
// calibrations change only the grouping of the dot-product partials
// (rounding level).  c_bal_g == 0 (default) or a different grid: equal split.
constexpr int kMaxBalGrid = 512;
__constant__ double c_cumw[kMaxBalGrid + 1];
__constant__ int c_bal_g;

__device__ __forceinline__ void cta_rows(long long n, long long& r0, long long& r1) {
#ifdef EWB_ROWS_REVERSED   // experiment: is a slow CTA slow because of its SM or its rows?
  const long long b = gridDim.x - 1 - blockIdx.x;
#else
  const long long b = blockIdx.x;
#endif
  if (c_bal_g == (int)gridDim.x) {
    r0 = llrint(c_cumw[b] * (double)n);
    r1 = llrint(c_cumw[b + 1] * (double)n);
  } else {
    r0 = b * n / gridDim.x;
    r1 = (b + 1) * n / gridDim.x;
  }
}
// host mirror of cta_rows' balanced split
static inline long long host_split(const double* cumw, int b, long long n) {
  return llrint(cumw[b] * (double)n);
}

struct NoPre {
  __device__ __forceinline__ void operator()(long long, int) const {}
};
#ifndef EWB_EPI_PREFETCH
#define EWB_EPI_PREFETCH 12
#endif
// pre(row0, nrows) runs EWB_EPI_PREFETCH tiles before a block's epilogue:
// the GMRES kernel prefetches the basis rows its dot products will read
// into L1 there, so the epilogue (during which this CTA consumes no ring
// stage) does not wait on L2.
template <int K, typename Epi, typename Pre = NoPre>
__device__ void matvec_rows(Ring& R, const cplx* __restrict__ A, long long n, const cplx* x,
                            long long r0, long long r1, Epi&& epi, Pre&& pre = Pre{}) {
  __shared__ cplx s_red[kSolveWarps][kRpt][K];
  __shared__ cplx s_sum[kRR][K];
  __shared__ int s_rel[kNS];  // warps done with each ring slot
  const int rows = (int)(r1 - r0);
  if (rows <= 0) return;
  const int nblk = (rows + kRR - 1) / kRR;
  const int ntile = (int)((n + kTC - 1) / kTC);
  const int S = nblk * ntile;
  const int last_tc = (int)(n - (long long)(ntile - 1) * kTC);
  // block q covers rows r0 + [q rows / nblk, (q+1) rows / nblk); stage
  // u = q ntile + t.  (32-bit arithmetic: rows per CTA << 2^31 / nblk.)
  // Stage u goes to ring slot (R.pos + u) % kNS; the LAST warp to finish
  // reading a slot refills it with stage u + kNS, so no warp ever waits for
  // another except on data arrival (no CTA barrier per stage).
  auto issue = [&](int u) {
    const int q = u / ntile, t = u - q * ntile;
    const int rel0 = q * rows / nblk, nr = (q + 1) * rows / nblk - rel0;
    const int tc = t == ntile - 1 ? last_tc : kTC;
    ring_issue(R, R.pos + (unsigned)u, A, n, r0 + rel0, nr, (long long)t * kTC, tc,
               max(0, min(nr, kPinRows - rel0)));
  };
  if (threadIdx.x < kNS) s_rel[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int u = 0; u < S && u < kNS; ++u) issue(u);
  }
  const int col = threadIdx.x % kTC, slice = threadIdx.x / kTC;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  cplx acc[kRpt][K];
#pragma unroll
  for (int r = 0; r < kRpt; ++r)
#pragma unroll
    for (int k = 0; k < K; ++k) acc[r][k] = {0.0, 0.0};
  cplx xn[K];  // x for the stage being consumed (prefetched one stage ahead)
#pragma unroll
  for (int k = 0; k < K; ++k) xn[k] = col < n ? ldg(x + k * n + col) : cplx{0.0, 0.0};
  int q = 0, t = 0;
  long long row0 = r0;
  int nrows = rows / nblk;
  for (int s = 0; s < S; ++s) {
    const long long c0 = (long long)t * kTC;
    const int tc = t == ntile - 1 ? last_tc : kTC;
    cplx xv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) xv[k] = xn[k];
    {  // prefetch the next stage's x
      const long long cn = (t == ntile - 1 ? 0 : c0 + kTC) + col;
#pragma unroll
      for (int k = 0; k < K; ++k) xn[k] = cn < n ? ldg(x + k * n + cn) : cplx{0.0, 0.0};
    }
    if (t == max(0, ntile - 1 - EWB_EPI_PREFETCH)) pre(row0, nrows);
    const unsigned pos = R.pos + (unsigned)s;
    ring_wait(R, pos);
    if (col < tc) {
      const cplx* tile = R.buf + (size_t)(pos % kNS) * kStageElems;
#pragma unroll
      for (int r = 0; r < kRpt; ++r) {
        const int row = slice * kRpt + r;
        if (row < nrows) {
          double2 a2 = *reinterpret_cast<const double2*>(tile + row * kTC + col);
          cplx av = {a2.x, a2.y};
#pragma unroll
          for (int k = 0; k < K; ++k) cfma(acc[r][k], av, xv[k]);
        }
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0 &&
        atomicAdd(&s_rel[pos % kNS], 1) == kSolveWarps - 1) {  // last reader of the slot
      s_rel[pos % kNS] = 0;
      if (s + kNS < S) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(s + kNS);
      }
    }
    if (t == ntile - 1) {  // last tile of the block: reduce, then the epilogue
#pragma unroll
      for (int r = 0; r < kRpt; ++r)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          warp_sum(acc[r][k]);
          if (lane == 0) s_red[wid][r][k] = acc[r][k];
          acc[r][k] = {0.0, 0.0};
        }
      __syncthreads();
      if (threadIdx.x < kRR * K) {
        const int row = threadIdx.x / K, k = threadIdx.x % K;
        const int h = row / kRpt, r = row % kRpt;
        constexpr int wps = kSolveWarps / kSlices;  // warps per row slice
        cplx sum = {0.0, 0.0};
        for (int w = 0; w < wps; ++w) sum = sum + s_red[h * wps + w][r][k];
        s_sum[row][k] = sum;
      }
      __syncthreads();
      epi(row0, nrows, s_sum);
      __syncthreads();
      t = 0;
      if (++q < nblk) {
        const int rel0 = q * rows / nblk;
        row0 = r0 + rel0;
        nrows = (q + 1) * rows / nblk - rel0;
      }
    } else {
      ++t;
    }
  }
  R.pos += (unsigned)S;
}

template <int K, typename Epi>
__device__ void matvec_rows_wide(Ring& R, const cplx* __restrict__ A, long long n, const cplx* x,
                            long long r0, long long r1, Epi&& epi) {
  // 4 row slices x 4 rows; a slice's 128 threads take columns col and
  // col + 128 of every tile: 4 x K accumulators and 2 x K prefetched x per
  // thread (K = 3, 4 fit the 128-register budget without spilling).
  constexpr int kSl = 4, kRw = kRR / kSl, kCols = kSolveThreads / kSl, kCp = kTC / kCols;
  static_assert(kRR % kSl == 0 && kTC % kCols == 0, "matvec_rows_wide layout");
  __shared__ cplx s_red[kSolveWarps][kRw][K];
  __shared__ cplx s_sum[kRR][K];
  __shared__ int s_rel[kNS];  // warps done with each ring slot
  const int rows = (int)(r1 - r0);
  if (rows <= 0) return;
  const int nblk = (rows + kRR - 1) / kRR;
  const int ntile = (int)((n + kTC - 1) / kTC);
  const int S = nblk * ntile;
  const int last_tc = (int)(n - (long long)(ntile - 1) * kTC);
  // block q covers rows r0 + [q rows / nblk, (q+1) rows / nblk); stage
  // u = q ntile + t.  (32-bit arithmetic: rows per CTA << 2^31 / nblk.)
  // Stage u goes to ring slot (R.pos + u) % kNS; the LAST warp to finish
  // reading a slot refills it with stage u + kNS, so no warp ever waits for
  // another except on data arrival (no CTA barrier per stage).
  auto issue = [&](int u) {
    const int q = u / ntile, t = u - q * ntile;
    const int rel0 = q * rows / nblk, nr = (q + 1) * rows / nblk - rel0;
    const int tc = t == ntile - 1 ? last_tc : kTC;
    ring_issue(R, R.pos + (unsigned)u, A, n, r0 + rel0, nr, (long long)t * kTC, tc,
               max(0, min(nr, kPinRows - rel0)));
  };
  if (threadIdx.x < kNS) s_rel[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int u = 0; u < S && u < kNS; ++u) issue(u);
  }
  const int col = threadIdx.x % kCols, slice = threadIdx.x / kCols;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  cplx acc[kRw][K];
#pragma unroll
  for (int r = 0; r < kRw; ++r)
#pragma unroll
    for (int k = 0; k < K; ++k) acc[r][k] = {0.0, 0.0};
  cplx xn[kCp][K];  // x of the stage being consumed (loaded after the previous stage's FMAs)
#pragma unroll
  for (int m = 0; m < kCp; ++m)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = col + m * kCols;
      xn[m][k] = c < n ? ldg(x + k * n + c) : cplx{0.0, 0.0};
    }
  int q = 0, t = 0;
  long long row0 = r0;
  int nrows = rows / nblk;
  for (int s = 0; s < S; ++s) {
    const long long c0 = (long long)t * kTC;
    const int tc = t == ntile - 1 ? last_tc : kTC;
    const unsigned pos = R.pos + (unsigned)s;
    ring_wait(R, pos);
    {
      const cplx* tile = R.buf + (size_t)(pos % kNS) * kStageElems;
#pragma unroll
      for (int m = 0; m < kCp; ++m) {
        const int c = col + m * kCols;
        if (c < tc) {
#pragma unroll
          for (int r = 0; r < kRw; ++r) {
            const int row = slice * kRw + r;
            if (row < nrows) {
              double2 a2 = *reinterpret_cast<const double2*>(tile + row * kTC + c);
              cplx av = {a2.x, a2.y};
#pragma unroll
              for (int k = 0; k < K; ++k) cfma(acc[r][k], av, xn[m][k]);
            }
          }
        }
      }
    }
    {  // x for the next stage
      const long long cb = (t == ntile - 1 ? 0 : c0 + kTC) + col;
#pragma unroll
      for (int m = 0; m < kCp; ++m)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const long long cn = cb + m * kCols;
          xn[m][k] = cn < n ? ldg(x + k * n + cn) : cplx{0.0, 0.0};
        }
    }
#if EWB_X_PREFETCH
    {  // the x columns of the stage after next into L1 (no registers held)
      const int t2 = (t + 2) % ntile;
      const long long c2 = (long long)t2 * kTC;
      constexpr int kLines = kTC * 16 / 128;   // 128-byte lines per vector segment
      if (threadIdx.x < K * kLines) {
        const int k = threadIdx.x / kLines, ln = threadIdx.x % kLines;
        const long long cc = c2 + ln * 8;
        if (cc < n) asm volatile("prefetch.global.L1 [%0];" ::"l"(x + k * n + cc));
      }
    }
#endif
    __syncwarp();
    if ((threadIdx.x & 31) == 0 &&
        atomicAdd(&s_rel[pos % kNS], 1) == kSolveWarps - 1) {  // last reader of the slot
      s_rel[pos % kNS] = 0;
      if (s + kNS < S) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(s + kNS);
      }
    }
    if (t == ntile - 1) {  // last tile of the block: reduce, then the epilogue
#pragma unroll
      for (int r = 0; r < kRw; ++r)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          warp_sum(acc[r][k]);
          if (lane == 0) s_red[wid][r][k] = acc[r][k];
          acc[r][k] = {0.0, 0.0};
        }
      __syncthreads();
      if (threadIdx.x < kRR * K) {
        const int row = threadIdx.x / K, k = threadIdx.x % K;
        const int h = row / kRw, r = row % kRw;
        constexpr int wps = kSolveWarps / kSl;  // warps per row slice
        cplx sum = {0.0, 0.0};
        for (int w = 0; w < wps; ++w) sum = sum + s_red[h * wps + w][r][k];
        s_sum[row][k] = sum;
      }
      __syncthreads();
      epi(row0, nrows, s_sum);
      __syncthreads();
      t = 0;
      if (++q < nblk) {
        const int rel0 = q * rows / nblk;
        row0 = r0 + rel0;
        nrows = (q + 1) * rows / nblk - rel0;
      }
    } else {
      ++t;
    }
  }
  R.pos += (unsigned)S;
}

// sum over aligned groups of G lanes (result in every lane of the group)
template <int G>
__device__ __forceinline__ void group_sum(cplx& v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    v.re += __shfl_xor_sync(0xffffffffu, v.re, o);
    v.im += __shfl_xor_sync(0xffffffffu, v.im, o);
  }
}

// Fixed-order reduction of `cnt` CTA partials (layout part[b * stride + t]):
// 8 threads per value, thread `sub` summing CTAs sub, sub + 8, ... with all
// of its loads issued before the first add (one L2 round trip per round
// instead of one per CTA), then a 3-step shuffle.  Identical in every CTA.
constexpr int kRedPer = 20;  // partial loads per thread: grids up to 160 CTAs

__device__ void reduce_parts(const cplx* part, int stride, int cnt, cplx* out) {
  const int sub = threadIdx.x & 7;
  const int G = gridDim.x;
  for (int base = 0; base < cnt; base += kSolveThreads / 8) {
    const int t = base + (threadIdx.x >> 3);
    cplx s = {0.0, 0.0};
    if (t < cnt) {
      if (G <= 8 * kRedPer) {
        cplx v[kRedPer];
#pragma unroll
        for (int i = 0; i < kRedPer; ++i) {
          const int b = sub + 8 * i;
          v[i] = b < G ? part[(size_t)b * stride + t] : cplx{0.0, 0.0};
        }
#pragma unroll
        for (int i = 0; i < kRedPer; ++i) s = s + v[i];
      } else {
        for (int b = sub; b < G; b += 8) s = s + part[(size_t)b * stride + t];
      }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      s.re += __shfl_xor_sync(0xffffffffu, s.re, o);
      s.im += __shfl_xor_sync(0xffffffffu, s.im, o);
    }
    if (sub == 0 && t < cnt) out[t] = s;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------
// GMRES with the Arnoldi vector work fused around the matvec (default,
// GmresArgs::ortho == 0).  Same algorithm as k_gmres (one-reduction MGS,
// linsolve.py:150-170 up to association), restructured so that an Arnoldi
// step costs one pass over A plus two grid barriers:
//
//   matvec   w = (A z') / h_{j,j-1} over the CTA's own rows; each finished
//            row block immediately adds <V_t, w>, t <= j, to CTA partials
//   S1       grid barrier
//   reduce   d_t and Gram row j (fixed order, every CTA); h = (I + L)^{-1} d
//            as d - L (d - L d), exact to O(|L|^3) with |L| the basis's loss
//            of orthogonality (~1e-15)
//   update   u = w - sum_i h_i V_i over own rows (+ the <= 2 rows completing
//            the last owned element), |u|^2 and <u, V_l> partials (the next
//            Gram row), z' = P^{-1} u for owned elements
//   S2       grid barrier
//   Givens   h_{j+1,j} = |u| (fixed-order reduce), rotations, residual
//            estimate; V_{j+1} = u / h_{j+1,j} written by the owning CTA
//
// The basis vector is normalised lazily: the next matvec runs on the
// unnormalised z' and scales its rows, so the norm reduction shares the
// barrier with the update instead of costing one of its own.
// ---------------------------------------------------------------------
constexpr int kNormSlot = kMaxDots - 1;
constexpr int kGrp = kRR <= 16 ? 16 : 32;  // lanes per epilogue dot


#ifdef EWB_GMRES_MAXNREG
__global__ void __maxnreg__(EWB_GMRES_MAXNREG)
#else
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks)
#endif
k_gmres_f(GmresArgs a) {
  int n_probe = 0;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char ring_smem[];
  __shared__ uint64_t ring_bar[kNS];
  __shared__ GivensShared gs;
  __shared__ cplx s_y[kMaxRestart];
  __shared__ cplx s_dots[kMaxDots];
  __shared__ cplx s_h[kMaxRestart + 1];
  __shared__ cplx s_h1[kMaxRestart + 1];
  __shared__ cplx s_dacc[kMaxRestart + 1];
  __shared__ cplx s_wblk[kRR];
  __shared__ double s_nrm[kSolveWarps];
  __shared__ double s_est;
  Ring ring{reinterpret_cast<cplx*>(ring_smem), ring_bar, 0u, 0u};
  ring_init(ring, 16.0 * (double)a.n * (double)a.n > 96e6);
  const long long n = a.n;
  const long long tid = gtid(), nth = gthreads();
  const bool pc = a.pinv != nullptr;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long k0, k1;
  cta_rows(n, k0, k1);
  // rows whose u this CTA computes: own rows plus the tail of the last
  // element it owns (element e is owned by the CTA owning row 3e)
  const long long e0 = pc ? (k0 + 2) / 3 : k0, e1 = pc ? (k1 + 2) / 3 : k1;
  const long long ka = k0, kb = pc ? max(k1, 3 * e1) : k1;
  const int RU = (int)(kb - ka);
  GridRed R{a.partial, 0};
  int dpar = 0;
  auto part_buf = [&](int p) { return a.dpart + (size_t)p * gridDim.x * kMaxDots; };

  // CTA-sum of one double per thread -> part[kNormSlot].re of buffer p
  auto cta_norm_partial = [&](double q, int p) {
    warp_sum(q);
    if (lane == 0) s_nrm[wid] = q;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kSolveWarps; ++w) s += s_nrm[w];
      part_buf(p)[(size_t)blockIdx.x * kMaxDots + kNormSlot] = {s, 0.0};
    }
  };
  // every CTA: sum of the kNormSlot partials of buffer p (fixed order)
  auto grid_norm = [&](int p) -> double {
    const cplx* part = part_buf(p);
    if (wid == 0) {
      double v[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int b = lane + 32 * i;
        v[i] = b < (int)gridDim.x ? part[(size_t)b * kMaxDots + kNormSlot].re : 0.0;
      }
      double s = (((v[0] + v[1]) + v[2]) + v[3]) + v[4];
      for (int b = lane + 160; b < (int)gridDim.x; b += 32) s += part[(size_t)b * kMaxDots + kNormSlot].re;
      warp_sum(s);
      if (lane == 0) s_est = s;
    }
    __syncthreads();
    const double v = s_est;
    __syncthreads();
    return v;
  };
  // r = b - A x over own rows (a.r), |r|^2 partial into buffer p; ends with
  // a grid barrier, returns |r|
  auto residual = [&](int p) -> double {
    double q = 0.0;
    matvec_rows<1>(ring, a.A, n, a.x, k0, k1, [&](long long row0, int nr, cplx (*sum)[1]) {
      if (threadIdx.x < nr) {
        const cplx r = a.b[row0 + threadIdx.x] - sum[threadIdx.x][0];
        a.r[row0 + threadIdx.x] = r;
        q += abs2(r);
      }
    });
    cta_norm_partial(q, p);
    grid.sync();
    return sqrt(grid_norm(p));
  };

  // ||b|| and "x0 has a nonzero entry", one reduction
  double v2[2] = {0.0, 0.0};
  for (long long k = tid; k < n; k += nth) {
    v2[0] += abs2(a.b[k]);
    if (a.has_x0) v2[1] += (a.x[k].re != 0.0 || a.x[k].im != 0.0);
    else a.x[k] = {0.0, 0.0};
  }
  grid_sum(grid, R, v2);
  const double nb = sqrt(v2[0]);
  if (nb == 0.0) {  // linsolve.py:136-140
    for (long long k = tid; k < n; k += nth) a.x[k] = {0.0, 0.0};
    if (tid == 0) { a.out->iterations = 0; a.out->init_res = 0; a.out->final_res = 0;
                    a.out->n_hist = 0; a.out->converged = 1; a.out->matvecs = 0; }
    return;
  }
  int n_mv = 0;
  double rnorm;
#ifndef EWB_NO_AX0
  if (v2[1] > 0.0 && a.ax0) {  // r = b - A x0 with A x0 supplied (SEM's Y s)
    double q = 0.0;
    for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      const cplx r = a.b[k] - a.ax0[k];
      a.r[k] = r;
      q += abs2(r);
    }
    cta_norm_partial(q, dpar);
    grid.sync();
    rnorm = sqrt(grid_norm(dpar));
    dpar ^= 1;
  } else
#endif
  if (v2[1] > 0.0) {  // r = b - A x0 (linsolve.py:144)
    rnorm = residual(dpar);
    dpar ^= 1;
    ++n_mv;
  } else {
    for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) a.r[k] = a.b[k];
    rnorm = nb;
    grid.sync();
  }
  double res = rnorm / nb;
  int n_hist = 0;
  if (tid == 0) { a.out->init_res = res; a.hist[0] = res; }
  n_hist++;
  int its = 0;
  cplx* const scr = ring.buf;  // idle ring = scratch between matvecs
  while (res > a.tol && its < a.maxiter) {
    const int m = min(a.restart, a.maxiter - its);
    // cycle start: u = r, h = beta; z' = P^{-1} r for owned elements
    const double beta = rnorm;
    if (pc) {
      for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        cplx v[3] = {a.r[3 * e], a.r[3 * e + 1], a.r[3 * e + 2]};
        precond_regs(a.pinv, e, v, a.z);
      }
    } else {
      for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) a.z[k] = a.r[k];
    }
    if (threadIdx.x == 0) {
      gs.g[0] = {beta, 0.0};
      for (int k = 1; k <= m; ++k) gs.g[k] = {0.0, 0.0};
    }
    for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      a.V[k] = {a.r[k].re / beta, a.r[k].im / beta};
      if (a.W) a.rs[k] = a.r[k];   // the cycle's starting (true) residual
    }
    grid.sync();
    double hprev = beta;
    int used = 0;
    for (int j = 0;; ++j) {
      // ---- matvec + <V_t, w> partials ------------------------------------
      const double sc = 1.0 / hprev;
      for (int t = threadIdx.x; t <= j; t += blockDim.x) s_dacc[t] = {0.0, 0.0};
      __syncthreads();
      EWB_PROBE(2);
      matvec_rows<1>(ring, a.A, n, a.z, k0, k1, [&](long long row0, int nr, cplx (*sum)[1]) {
        if (threadIdx.x < nr) {
          const cplx w = sum[threadIdx.x][0] * sc;
          a.w[row0 + threadIdx.x] = w;
          if (a.W) a.W[(size_t)j * n + row0 + threadIdx.x] = w;   // = A P^{-1} v_j
          s_wblk[threadIdx.x] = w;
        }
        __syncthreads();
        // kGrp lanes per dot (one row each), kSolveThreads / kGrp dots per round
        const int sub = threadIdx.x % kGrp;
        for (int t0 = 0; t0 <= j; t0 += 2 * (kSolveThreads / kGrp)) {
          const int ta = t0 + threadIdx.x / kGrp, tb = ta + kSolveThreads / kGrp;
          const bool ok = sub < nr;
          cplx va = ok && ta <= j ? a.V[(size_t)ta * n + row0 + sub] : cplx{0.0, 0.0};
          cplx vb = ok && tb <= j ? a.V[(size_t)tb * n + row0 + sub] : cplx{0.0, 0.0};
          const cplx wv = ok ? s_wblk[sub] : cplx{0.0, 0.0};
          cplx sa = conj(va) * wv, sb = conj(vb) * wv;
          group_sum<kGrp>(sa);
          group_sum<kGrp>(sb);
          if (sub == 0) {
            if (ta <= j) s_dacc[ta] = s_dacc[ta] + sa;
            if (tb <= j) s_dacc[tb] = s_dacc[tb] + sb;
          }
        }
      }, [&](long long row0, int nr) {
        // the same V entries the dot loop above reads, into L1 ahead of time
        const int sub = threadIdx.x % kGrp;
        if (sub < nr)
          for (int ta = threadIdx.x / kGrp; ta <= j; ta += kSolveThreads / kGrp)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.V + (size_t)ta * n + row0 + sub));
      });
      ++n_mv;
#if EWB_L2_PREFETCH_TILES > 0
      {  // the next pass's first tiles of this CTA's rows into L2 while the
         // grid waits at S1 and reduces (HBM otherwise idle)
        const int rows = (int)(k1 - k0), nblk = (rows + kRR - 1) / kRR;
        const int nr = rows / nblk;
        const int ntile = (int)((n + kTC - 1) / kTC);
        const int nt = min(EWB_L2_PREFETCH_TILES, ntile);
        for (int idx = threadIdx.x; idx < nr * nt; idx += blockDim.x) {
          const int r = idx % nr, t = idx / nr;
          const long long c0 = (long long)t * kTC;
          const uint32_t bytes = (uint32_t)(min((long long)kTC, n - c0) * 16);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.A + (k0 + r) * n + c0),
                       "r"(bytes)
                       : "memory");
        }
      }
#endif
      cplx* part = part_buf(dpar);
      for (int t = threadIdx.x; t <= j; t += blockDim.x)
        part[(size_t)blockIdx.x * kMaxDots + t] = s_dacc[t];
      EWB_PROBE(3);
      if (a.probe && threadIdx.x == 0 && j < 100 && its == j) {  // per-CTA matvec finish (cycle 0)
        a.probe[32768 + j * gridDim.x + blockIdx.x] = gtimer();
        if (j == 0) {
          unsigned sm;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
          a.probe[32768 + 100 * gridDim.x + blockIdx.x] = sm;   // which SM ran this CTA
        }
      }
      // Gram rows 1..j-1 (written in earlier steps) staged into the idle
      // ring while other CTAs finish their matvec
      cplx* gsm = scr;
      {
        const int tri = j * (j - 1) / 2;
        for (int q = threadIdx.x; q < tri; q += blockDim.x) {
          // packed index q -> (i, l), i >= 1, l < i
          int i = (int)((1.0 + sqrt(1.0 + 8.0 * q)) * 0.5);
          while (i * (i - 1) / 2 > q) --i;
          while ((i + 1) * i / 2 <= q) ++i;
          const int l = q - i * (i - 1) / 2;
          gsm[q] = a.Gram[(size_t)i * kMaxRestart + l];
        }
      }
      grid.sync();  // S1
      EWB_PROBE(4);
      // ---- d_t and Gram row j; h = (I + L)^{-1} d --------------------------
      {
        // reduce-scatter (CTA b sums value t = b mod G over the CTA partials
        // in a fixed order) + barrier + all-gather: every partial is read
        // once instead of once per CTA
        cplx* fin = reinterpret_cast<cplx*>(a.partial);
        const int cnt = 2 * j + 1;
#ifdef EWB_DBG_WARM
        for (int rep = 0; rep < 2; ++rep) {
        if (rep) EWB_PROBE(15);
#endif
        for (int t = blockIdx.x + wid * gridDim.x; t < cnt; t += kSolveWarps * gridDim.x) {
          cplx v[5];
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            const int b = lane + 32 * i;
            v[i] = b < (int)gridDim.x ? part[(size_t)b * kMaxDots + t] : cplx{0.0, 0.0};
          }
          cplx sum = (((v[0] + v[1]) + v[2]) + v[3]) + v[4];
          for (int b = lane + 160; b < (int)gridDim.x; b += 32) sum = sum + part[(size_t)b * kMaxDots + t];
          warp_sum(sum);
          if (lane == 0) fin[t] = t > j ? sum * sc : sum;  // <u, V_l> / h = <v_j, V_l>
        }
#ifdef EWB_DBG_WARM
        __syncthreads();
        }
#endif
        EWB_PROBE(11);
        grid.sync();  // S1b
        EWB_PROBE(12);
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) s_dots[t] = fin[t];
        __syncthreads();
        EWB_PROBE(8);
        if (blockIdx.x == 0)
          for (int l = threadIdx.x; l < j; l += blockDim.x)
            a.Gram[(size_t)j * kMaxRestart + l] = s_dots[j + 1 + l];
        // h = d - L (d - L d): two Jacobi sweeps, warp per row
        for (int sweep = 0; sweep < 2; ++sweep) {
          const cplx* hin = sweep == 0 ? s_dots : s_h1;
          cplx* hout = sweep == 0 ? s_h1 : s_h;
          for (int i = wid; i <= j; i += kSolveWarps) {
            cplx s = {0.0, 0.0};
            for (int l = lane; l < i; l += 32) {
              const cplx g = i == j ? s_dots[j + 1 + l] : gsm[i * (i - 1) / 2 + l];
              s = s + g * hin[l];
            }
            warp_sum(s);
            if (lane == 0) hout[i] = s_dots[i] - s;
          }
          __syncthreads();
          EWB_PROBE(9 + sweep);
        }
      }
      EWB_PROBE(5);
      // ---- update: u = w - sum_i h_i V_i over [ka, kb) --------------------
      {
        const int nv = j + 1;
        const int nc = max(1, min(nv, kSolveThreads / max(RU, 1)));
        cplx* pu = scr;            // [nc][RU] chunk partials
        cplx* su = scr + nc * RU;  // [RU] u
        for (int p = threadIdx.x; p < nc * RU; p += blockDim.x) {
          const int r = p % RU, c = p / RU;
          const int i0 = c * nv / nc, i1 = (c + 1) * nv / nc;
          cplx s = {0.0, 0.0};
#pragma unroll 8
          for (int i = i0; i < i1; ++i) cfma(s, s_h[i], a.V[(size_t)i * n + ka + r]);
          pu[p] = s;
        }
        __syncthreads();
        double q = 0.0;
        for (int r = threadIdx.x; r < RU; r += blockDim.x) {
          cplx u = a.w[ka + r];
          for (int c = 0; c < nc; ++c) u = u - pu[c * RU + r];
          su[r] = u;
          if (ka + r < k1) {
            a.r[ka + r] = u;
            q += abs2(u);
          }
        }
        __syncthreads();
        if (pc) {
          for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const cplx* u = su + (3 * e - ka);
            cplx v[3] = {u[0], u[1], u[2]};
            precond_regs(a.pinv, e, v, a.z);
          }
        } else {
          for (int r = threadIdx.x; r < RU; r += blockDim.x) a.z[ka + r] = su[r];
        }
        // next Gram row: <u, V_l>, l <= j, over own rows
        cplx* pn = part_buf(dpar ^ 1);
        const int own = (int)(k1 - k0);
        {
          const int sub = threadIdx.x & 15;
          for (int l0 = 0; l0 <= j; l0 += kSolveThreads / 16) {  // warp-uniform trip count
            const int l = l0 + (threadIdx.x >> 4);
            cplx s = {0.0, 0.0};
            if (l <= j) {
#pragma unroll 8
              for (int r = sub; r < own; r += 16) cfma(s, conj(su[r]), a.V[(size_t)l * n + k0 + r]);
            }
            group_sum<16>(s);
            if (sub == 0 && l <= j) pn[(size_t)blockIdx.x * kMaxDots + (j + 2) + l] = s;
          }
        }
        cta_norm_partial(q, dpar ^ 1);
      }
      dpar ^= 1;
      EWB_PROBE(6);
      grid.sync();  // S2
      EWB_PROBE(13);
      const double hn = sqrt(grid_norm(dpar));
      EWB_PROBE(14);
      // Givens (linsolve.py:171-194), identical in every CTA
      if (threadIdx.x == 0) {
        // apply the previous rotations; only `carry` (the running h_i) is
        // on the dependency chain
        cplx carry = s_h[0];
#pragma unroll 4
        for (int i = 0; i < j; ++i) {
          const cplx c = gs.cs[i], sn = gs.sn[i], hn1 = s_h[i + 1];
          gs.h[i] = c * carry + sn * hn1;
          carry = (-conj(sn)) * carry + conj(c) * hn1;
        }
        gs.h[j] = carry;
        gs.h[j + 1] = {hn, 0.0};
        double ahj = hypot(gs.h[j].re, gs.h[j].im), ahn = hypot(gs.h[j + 1].re, gs.h[j + 1].im);
        double den = sqrt(ahj * ahj + ahn * ahn);
        if (den == 0.0) {
          gs.cs[j] = {1.0, 0.0}; gs.sn[j] = {0.0, 0.0};
        } else if (gs.h[j].re == 0.0 && gs.h[j].im == 0.0) {
          gs.cs[j] = {0.0, 0.0}; gs.sn[j] = {1.0, 0.0};
        } else {
          gs.cs[j] = {ahj / den, 0.0};
          cplx ph = {gs.h[j].re / ahj, gs.h[j].im / ahj};
          cplx t = ph * conj(gs.h[j + 1]);
          gs.sn[j] = {t.re / den, t.im / den};
        }
        gs.h[j] = gs.cs[j] * gs.h[j] + gs.sn[j] * gs.h[j + 1];
        gs.h[j + 1] = {0.0, 0.0};
        gs.g[j + 1] = (-conj(gs.sn[j])) * gs.g[j];
        gs.g[j] = gs.cs[j] * gs.g[j];
        s_est = hypot(gs.g[j + 1].re, gs.g[j + 1].im) / nb;
        if (blockIdx.x == 0)
          for (int i = 0; i <= j; ++i) a.H[(size_t)i * kMaxRestart + j] = gs.h[i];
      }
      __syncthreads();
      EWB_PROBE(7);
      ++its;
      used = j + 1;
      const double est = s_est;
      if (tid == 0 && n_hist < a.hist_cap) a.hist[n_hist] = est;
      n_hist++;
      if (est <= a.tol || j + 1 == m) break;
      // V_{j+1} = u / h_{j+1,j} on own rows (u kept in a.r)
      if (hn > 0.0) {
        cplx* vn = a.V + (size_t)(j + 1) * n;
        for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x)
          vn[k] = {a.r[k].re / hn, a.r[k].im / hn};
      }
      hprev = hn > 0.0 ? hn : 1.0;
      __syncthreads();
    }
    grid.sync();  // H visible to every CTA before the back substitution
    // back substitution (linsolve.py:196-198): warp 0 of every CTA, with
    // the upper triangle of H staged (packed) into the idle ring first.
    {
      cplx* hsm = ring.buf;
      for (int i = 0; i < used; ++i)
        for (int k = i + threadIdx.x; k < used; k += blockDim.x)
          hsm[i * used - i * (i - 1) / 2 + (k - i)] = a.H[(size_t)i * kMaxRestart + k];
      __syncthreads();
      if (wid == 0) {
        for (int i = used - 1; i >= 0; --i) {
          const cplx* row = hsm + i * used - i * (i - 1) / 2 - i;
          cplx s = {0.0, 0.0};
          for (int k = i + 1 + lane; k < used; k += 32) s = s + row[k] * s_y[k];
          warp_sum(s);
          if (lane == 0) s_y[i] = cdiv(gs.g[i] - s, row[i]);
          __syncwarp();
        }
      }
      __syncthreads();
    }
    // x += P^{-1} (V y), per owned element (or own row)
    {
      const long long ua = pc ? e0 : k0, ub = pc ? e1 : k1;
      const int ucnt = pc ? 3 : 1;
      for (long long u = ua + threadIdx.x; u < ub; u += blockDim.x) {
        cplx uv[3];
        for (int c = 0; c < ucnt; ++c) {
          const long long k = u * ucnt + c;
          cplx s = {0.0, 0.0};
#pragma unroll 8
          for (int i = 0; i < used; ++i) cfma(s, a.V[(size_t)i * n + k], s_y[i]);
          uv[c] = s;
        }
        if (pc) {
          const cplx* P = a.pinv + 9 * u;
          for (int r = 0; r < 3; ++r) {
            cplx s = P[3 * r] * uv[0];
            s = s + P[3 * r + 1] * uv[1];
            s = s + P[3 * r + 2] * uv[2];
            a.x[3 * u + r] = a.x[3 * u + r] + s;
          }
        } else {
          a.x[u] = a.x[u] + uv[0];
        }
      }
    }
    grid.sync();
    if (a.W) {
      // true residual (linsolve.py:200-201) without another pass over A:
      // b - A x_new = r_start - sum_i y_i (A P^{-1} v_i), from the products
      // this cycle already computed (equal to b - A x_new up
      // to rounding of |A x|, ~1e-16 |b| against a tolerance of 1e-8 |b|)
      double q = 0.0;
      for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        cplx s = a.rs[k];
        for (int i = 0; i < used; ++i) s = s - s_y[i] * a.W[(size_t)i * n + k];
        a.r[k] = s;
        q += abs2(s);
      }
      cta_norm_partial(q, dpar);
      grid.sync();
      rnorm = sqrt(grid_norm(dpar));
    } else {
      rnorm = residual(dpar);  // true residual (linsolve.py:200-201)
      ++n_mv;
    }
    dpar ^= 1;
    res = rnorm / nb;
  }
  if (tid == 0) {
    a.out->iterations = its;
    a.out->final_res = res;
    a.out->converged = res <= a.tol;
    a.out->n_hist = n_hist;
    a.out->matvecs = n_mv;
  }
}

// ---------------------------------------------------------------------
// SEM (linsolve.py:213-242): Y = A X (one pass over A for all K columns),
// QR of Y[:, keep] by classical Gram-Schmidt with one re-orthogonalisation
// (|R_ii| agrees with Householder's to rounding), rank filter
// |R_ii| >= rank_tol * max|R_ii| (<= 2 passes), x0 = X s with R s = Q^H b;
// falls back to the newest column.
// ---------------------------------------------------------------------
template <int K>
__device__ void sem_body(cg::grid_group& grid, GridRed& R, const SemArgs& a) {
  const long long n = a.n, tid = gtid(), nth = gthreads();
  // Y = A X was produced by k_multi_gemv (its own launch: the K-vector
  // matvec needs more registers than this cooperative kernel can give it)
  __shared__ int keep[kMaxSem];
  __shared__ cplx Rm[kMaxSem][kMaxSem];
  __shared__ int nkeep;
  if (threadIdx.x == 0) {
    nkeep = a.K;
    for (int c = 0; c < a.K; ++c) keep[c] = c;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    const int kk = nkeep;
    // QR of Y[:, keep] -> Q (columns in a.Q), R (shared)
    for (int c = 0; c < kk; ++c) {
      const cplx* yc = a.Y + (size_t)keep[c] * n;
      cplx* qc = a.Q + (size_t)c * n;
      for (long long k = tid; k < n; k += nth) qc[k] = yc[k];
      if (threadIdx.x == 0)
        for (int i = 0; i < kMaxSem; ++i) Rm[i][c] = {0.0, 0.0};
      for (int rep = 0; rep < 2 && c > 0; ++rep) {
        double d[2 * kMaxSem];
#pragma unroll
        for (int i = 0; i < 2 * kMaxSem; ++i) d[i] = 0.0;
        for (long long k = tid; k < n; k += nth) {
          cplx qk = qc[k];
          for (int i = 0; i < c; ++i) {
            cplx p = conj(a.Q[(size_t)i * n + k]) * qk;
            d[2 * i] += p.re; d[2 * i + 1] += p.im;
          }
        }
        grid_sum(grid, R, d);
        for (long long k = tid; k < n; k += nth) {
          cplx qk = qc[k];
          for (int i = 0; i < c; ++i) qk = qk - cplx{d[2 * i], d[2 * i + 1]} * a.Q[(size_t)i * n + k];
          qc[k] = qk;
        }
        if (threadIdx.x == 0)
          for (int i = 0; i < c; ++i) Rm[i][c] = Rm[i][c] + cplx{d[2 * i], d[2 * i + 1]};
        grid.sync();
      }
      double nn[1] = {0.0};
      for (long long k = tid; k < n; k += nth) nn[0] += abs2(qc[k]);
      grid_sum(grid, R, nn);
      const double rcc = sqrt(nn[0]);
      if (threadIdx.x == 0) Rm[c][c] = {rcc, 0.0};
      if (rcc > 0.0) {  // an exactly dependent column keeps q = 0 (as Householder's R_cc = 0)
        for (long long k = tid; k < n; k += nth) {
          cplx q = qc[k];
          qc[k] = {q.re / rcc, q.im / rcc};
        }
      }
      grid.sync();
    }
    __syncthreads();
    double dmax = 0.0;
    for (int c = 0; c < kk; ++c) dmax = fmax(dmax, fabs(Rm[c][c].re));
    bool good[kMaxSem];
    bool all_good = true;
    int ng = 0;
    for (int c = 0; c < kk; ++c) {
      double dg = fabs(Rm[c][c].re);
      good[c] = dmax > 0 ? dg >= a.rank_tol * dmax : dg > 0;
      all_good = all_good && good[c];
      ng += good[c];
    }
    if (all_good) {
      // s = R^{-1} Q^H b
      double d[2 * kMaxSem];
#pragma unroll
      for (int i = 0; i < 2 * kMaxSem; ++i) d[i] = 0.0;
      for (long long k = tid; k < n; k += nth) {
        cplx bk = a.b[k];
        for (int i = 0; i < kk; ++i) {
          cplx p = conj(a.Q[(size_t)i * n + k]) * bk;
          d[2 * i] += p.re; d[2 * i + 1] += p.im;
        }
      }
      grid_sum(grid, R, d);
      cplx s[kMaxSem];
      for (int i = kk - 1; i >= 0; --i) {
        cplx t = {d[2 * i], d[2 * i + 1]};
        for (int k2 = i + 1; k2 < kk; ++k2) t = t - Rm[i][k2] * s[k2];
        s[i] = cdiv(t, Rm[i][i]);
      }
      for (long long k = tid; k < n; k += nth) {
        cplx x = {0.0, 0.0}, y = {0.0, 0.0};
        for (int i = 0; i < kk; ++i) {
          cfma(x, a.X[(size_t)keep[i] * n + k], s[i]);
          if (a.ax0) cfma(y, a.Y[(size_t)keep[i] * n + k], s[i]);
        }
        a.x0[k] = x;
        if (a.ax0) a.ax0[k] = y;
      }
      if (tid == 0) { a.out->kept = kk; a.out->fallback = 0; }
      return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int w = 0;
      for (int c = 0; c < kk; ++c)
        if (good[c]) keep[w++] = keep[c];
      nkeep = w;
    }
    __syncthreads();
    if (ng == 0) break;
  }
  for (long long k = tid; k < n; k += nth) {
    a.x0[k] = a.X[k];
    if (a.ax0) a.ax0[k] = a.Y[k];
  }
  if (tid == 0) { a.out->kept = 0; a.out->fallback = 1; }
}

__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_sem(SemArgs a) {
  cg::grid_group grid = cg::this_grid();
  GridRed R{a.partial, 0};
  switch (a.K) {
    case 1: sem_body<1>(grid, R, a); break;
    case 2: sem_body<2>(grid, R, a); break;
    case 3: sem_body<3>(grid, R, a); break;
    default: sem_body<4>(grid, R, a); break;
  }
}

// Batched GEMV y_b = A_b x_b through the TMA ring (regular launch; system
// blockIdx.y, row groups dealt over blockIdx.x).
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_gemv_tma(const cplx* A, const cplx* x,
                                                               cplx* y, long long n) {
  extern __shared__ __align__(128) unsigned char ring_smem[];
  __shared__ uint64_t ring_bar[kNS];
  Ring ring{reinterpret_cast<cplx*>(ring_smem), ring_bar, 0u, 0u};
  ring_init(ring, true);
  const size_t sys = blockIdx.y;
  cplx* ys = y + sys * n;
  long long r0, r1;
  cta_rows(n, r0, r1);
  matvec_rows<1>(ring, A + sys * n * n, n, x + sys * n, r0, r1,
                 [&](long long row0, int nr, cplx (*sum)[1]) {
                   if (threadIdx.x < nr) ys[row0 + threadIdx.x] = sum[threadIdx.x][0];
                 });
}

// Row-balance calibration: one matvec over the current split, all CTAs
// released together (cooperative launch), per-CTA duration recorded.
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_calib(const cplx* A,
                                                                         const cplx* x, cplx* y,
                                                                         long long n,
                                                                         unsigned long long* t) {
  extern __shared__ __align__(128) unsigned char ring_smem[];
  __shared__ uint64_t ring_bar[kNS];
  Ring ring{reinterpret_cast<cplx*>(ring_smem), ring_bar, 0u, 0u};
  ring_init(ring, true);
  long long r0, r1;
  cta_rows(n, r0, r1);
  cg::this_grid().sync();
  const unsigned long long t0 = gtimer();
  // rate mark: time and rows done when the CTA passes half of its rows, i.e.
  // while (nearly) every CTA is still streaming; a finish-time measure would
  // credit the last CTAs with the bandwidth the early finishers released
  long long done = 0;
  const long long half = (r1 - r0) / 2;
  matvec_rows<1>(ring, A, n, x, r0, r1, [&](long long row0, int nr, cplx (*sum)[1]) {
    if (threadIdx.x < nr) y[row0 + threadIdx.x] = sum[threadIdx.x][0];
    if (done < half && done + nr >= half && threadIdx.x == 0) {
      t[gridDim.x + blockIdx.x] = gtimer() - t0;
      t[2 * gridDim.x + blockIdx.x] = (unsigned long long)(done + nr);
    }
    done += nr;
  });
  __syncthreads();
  if (threadIdx.x == 0) t[blockIdx.x] = gtimer() - t0;
}

// Plain batched GEMV y_b = A_b x_b (one launch, `batch` systems of size n).
template <int RR>
__global__ void __launch_bounds__(512) k_gemv_batched(const cplx* A, const cplx* x, cplx* y,
                                                      long long n, int batch) {
  // blockIdx.y = system
  const cplx* Ab = A + (size_t)blockIdx.y * n * n;
  const cplx* xb = x + (size_t)blockIdx.y * n;
  cplx* yb = y + (size_t)blockIdx.y * n;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r0 = gw * RR; r0 < n; r0 += nw * RR) {
    cplx acc[RR];
#pragma unroll
    for (int a = 0; a < RR; ++a) acc[a] = {0.0, 0.0};
    const int nr = (int)min((long long)RR, n - r0);
#pragma unroll 2
    for (long long c = lane; c < n; c += 32) {
      cplx xv = ldg(xb + c);
#pragma unroll
      for (int a = 0; a < RR; ++a)
        if (a < nr) cfma(acc[a], ldc(Ab + (r0 + a) * n + c), xv);
    }
#pragma unroll
    for (int a = 0; a < RR; ++a) {
      warp_sum(acc[a]);
      if (lane == 0 && a < nr) yb[r0 + a] = acc[a];
    }
  }
}

// ---------------------------------------------------------------------
static int g_coop_blocks = 0;

static int coop_grid(const void* fn) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kSolveThreads, kRingBytes);
  if (per < 1) per = 1;
  return sms * per;
}

static int g_solver_limit = 0;  // 0: every co-resident CTA

void set_solver_ctas(int ctas) { g_solver_limit = ctas > 0 ? ctas : 0; }

int solver_grid_blocks() {
  const int m = solver_grid_max();
  return g_solver_limit > 0 && g_solver_limit < m ? g_solver_limit : m;
}

int solver_grid_max() {
  if (g_coop_blocks == 0) {
    int a = coop_grid((const void*)k_gmres), b = coop_grid((const void*)k_sem);
    int c = coop_grid((const void*)k_gmres_mgs), d = coop_grid((const void*)k_gmres_f);
    g_coop_blocks = a < b ? a : b;
    g_coop_blocks = c < g_coop_blocks ? c : g_coop_blocks;
    g_coop_blocks = d < g_coop_blocks ? d : g_coop_blocks;
  }
  return g_coop_blocks;
}

cudaError_t launch_gmres(GmresArgs& args, cudaStream_t s) {
  int G = solver_grid_blocks();
  void* params[] = {&args};
  note_launch();
  const void* fn = args.ortho == 1   ? (const void*)k_gmres_mgs
                   : args.ortho == 2 ? (const void*)k_gmres
                                     : (const void*)k_gmres_f;
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kSolveThreads), params, kRingBytes, s);
}

// Y = A X for K <= 4 columns in one TMA-streamed pass (SEM's products,
// linsolve.py:228).  Regular launch, 1 CTA/SM, full register budget.
template <int K>
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_multi_gemv(const cplx* A, const cplx* X,
                                                                 cplx* Y, long long n) {
  extern __shared__ __align__(128) unsigned char ring_smem[];
  __shared__ uint64_t ring_bar[kNS];
  Ring ring{reinterpret_cast<cplx*>(ring_smem), ring_bar, 0u, 0u};
  ring_init(ring, 16.0 * (double)n * (double)n > 96e6);
  long long r0, r1;
  cta_rows(n, r0, r1);
  auto store = [&](long long row0, int nr, cplx (*sum)[K]) {
    if (threadIdx.x < nr * K) {
      const int row = threadIdx.x / K, k = threadIdx.x % K;
      Y[k * n + row0 + row] = sum[row][k];
    }
  };
  if constexpr (K <= 2) matvec_rows<K>(ring, A, n, X, r0, r1, store);
  else matvec_rows_wide<K>(ring, A, n, X, r0, r1, store);
}

template <int K>
static cudaError_t launch_multi_gemv(const cplx* A, const cplx* X, cplx* Y, long long n,
                                     cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute((const void*)k_multi_gemv<K>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
    attr = true;
  }
  // the solver's CTA budget (the rest of the GPU may be assembling)
  unsigned blocks = (unsigned)solver_grid_blocks();
  EWB_NOTE k_multi_gemv<K><<<blocks, kSolveThreads, kRingBytes, s>>>(A, X, Y, n);
  return cudaGetLastError();
}

cudaError_t launch_sem(SemArgs& args, cudaStream_t s) {
  // Y = A X in one pass over A (K = 3, 4 with the 4-slice layout)
  cudaError_t e;
  switch (args.K) {
    case 1: e = launch_multi_gemv<1>(args.A, args.X, args.Y, args.n, s); break;
    case 2: e = launch_multi_gemv<2>(args.A, args.X, args.Y, args.n, s); break;
    case 3: e = launch_multi_gemv<3>(args.A, args.X, args.Y, args.n, s); break;
    default: e = launch_multi_gemv<4>(args.A, args.X, args.Y, args.n, s); break;
  }
  if (e != cudaSuccess) return e;
  int G = solver_grid_blocks();
  void* params[] = {&args};
  note_launch();
  return cudaLaunchCooperativeKernel((const void*)k_sem, dim3(G), dim3(kSolveThreads), params,
                                     kRingBytes, s);
}

#ifndef EWB_BAL_DAMP
#define EWB_BAL_DAMP 0.7
#endif
constexpr double kBalDamp = EWB_BAL_DAMP;

cudaError_t calibrate_rows(const cplx* A, long long n, int iters, double* stats,
                           cudaStream_t s) {
  const int G = solver_grid_blocks();
  if (G > kMaxBalGrid || n < 2LL * G) return cudaErrorInvalidValue;
  cudaFuncSetAttribute((const void*)k_calib, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kRingBytes);
  cplx *x = nullptr, *y = nullptr;
  unsigned long long* t = nullptr;
  cudaError_t e = cudaMalloc(&x, sizeof(cplx) * n);
  if (!e) e = cudaMalloc(&y, sizeof(cplx) * n);
  if (!e) e = cudaMalloc(&t, sizeof(unsigned long long) * 3 * G);
  if (!e) e = cudaMemsetAsync(x, 0, sizeof(cplx) * n, s);
  std::vector<double> cumw(G + 1), speed(G, 0.0);
  std::vector<unsigned long long> th(3 * G);
  for (int b = 0; b <= G; ++b) cumw[b] = (double)b / G;
  int zero = 0;
  if (!e) e = cudaMemcpyToSymbolAsync(c_bal_g, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, s);
  void* params[] = {(void*)&A, (void*)&x, (void*)&y, (void*)&n, (void*)&t};
  double spread0 = 0.0, spread1 = 0.0, mean0 = 0.0, mean1 = 0.0;
  for (int it = 0; !e && it <= iters; ++it) {
    // two launches per split: the first warms up, the second is measured
    for (int rep = 0; !e && rep < 2; ++rep) {
      note_launch();
      e = cudaLaunchCooperativeKernel((const void*)k_calib, dim3(G), dim3(kSolveThreads), params,
                                      kRingBytes, s);
    }
    if (!e) e = cudaMemcpyAsync(th.data(), t, sizeof(unsigned long long) * 3 * G,
                                cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) break;
    double tmax = 0.0, tmin = 1e30, tsum = 0.0;
    for (int b = 0; b < G; ++b) {
      const double tb = (double)th[b];
      tmax = tb > tmax ? tb : tmax;
      tmin = tb < tmin ? tb : tmin;
      tsum += tb;
    }
    if (it == 0) { spread0 = tmax - tmin; mean0 = tsum / G; }
    spread1 = tmax - tmin;
    mean1 = tsum / G;
    if (it == iters) break;   // last pass only measures the final split
    // damped fixed-point step on the finish times: a CTA that finishes
    // later than the mean gives rows away in proportion (the rates depend
    // on the split through the contention pattern, so no one-shot solve)
    const double tmean = tsum / G;
    double fsum = 0.0;
    for (int b = 0; b < G; ++b) {
      const double f = cumw[b + 1] - cumw[b];
      speed[b] = f * (1.0 + kBalDamp * (tmean - (double)th[b]) / tmean);
      fsum += speed[b];
    }
    double acc = 0.0;
    for (int b = 0; b < G; ++b) {
      cumw[b] = acc;
      acc += speed[b] / fsum;
    }
    cumw[G] = 1.0;
    e = cudaMemcpyToSymbolAsync(c_cumw, cumw.data(), sizeof(double) * (G + 1), 0,
                                cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemcpyToSymbolAsync(c_bal_g, &G, sizeof(int), 0, cudaMemcpyHostToDevice, s);
  }
  if (stats) {
    stats[0] = spread0 * 1e-3; stats[1] = mean0 * 1e-3;   // us, equal split
    stats[2] = spread1 * 1e-3; stats[3] = mean1 * 1e-3;   // us, calibrated split
  }
  cudaStreamSynchronize(s);
  cudaFree(x);
  cudaFree(y);
  cudaFree(t);
  return e;
}

cudaError_t reset_row_balance(cudaStream_t s) {
  int zero = 0;
  return cudaMemcpyToSymbolAsync(c_bal_g, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, s);
}

cudaError_t launch_gemv_batched(const cplx* A, const cplx* x, cplx* y, long long n, int batch,
                                cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute((const void*)k_gemv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRingBytes);
    attr = true;
  }
  long long blocks = sms;
  EWB_NOTE k_gemv_tma<<<dim3((unsigned)blocks, batch), kSolveThreads, kRingBytes, s>>>(A, x, y, n);
  return cudaGetLastError();
}

}  // namespace ewb
