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
EWB_DEBUG_TU(krylov)

// one 512-thread CTA per SM: register cap 65536 / 512 = 128 per thread
// (a 256-thread CTA streamed a pass in 749 us instead of 525 us)
constexpr int kSolveThreads = 512;
constexpr int kSolveMinBlocks = 1;
constexpr int kSolveWarps = kSolveThreads / 32;
constexpr int kMaxRed = 16;  // doubles per grid reduction

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

// ---------------------------------------------------------------------
// TMA (cp.async.bulk) matvec.  Each CTA streams its row blocks through a
// kNS-stage ring of shared-memory tiles (kRR rows x kTC columns), one bulk
// copy per row segment, completion tracked by a transaction-count mbarrier
// per stage.  Thread t owns column t % kTC of every tile (or kCpt columns
// when the tile is wider than the CTA) for kRpt rows; the per-row sums are
// reduced across the CTA at the end of each row block.  kNS x 96 KB =
// 192 KB per SM are in flight with no register cost.
// ---------------------------------------------------------------------
// Ring geometry: 12 rows x 512 columns x 16 B = 96 KB per stage, 2 stages.
// The row segments are 8 KB bulk copies; measured on cfg2 (A/B in one job,
// tools/sweep_time.py): 16 x 256 x 3 (4 KB copies) 3.63 s of solves per
// sweep, 8 x 512 x 3 3.39 s, 12 x 512 x 2 3.31 s, 4 x 1024 x 2-3 (16 KB
// copies, two columns per thread) 3.54 s; cfg4 GEMV 7.04 -> 7.35 TB/s.
// Fewer, larger copies per byte are what the TMA path rewards.
#ifndef EWB_RING_RR
#define EWB_RING_RR 12
#endif
#ifndef EWB_RING_TC
#define EWB_RING_TC 512
#endif
#ifndef EWB_RING_NS
#define EWB_RING_NS 2
#endif
constexpr int kRR = EWB_RING_RR;
constexpr int kTC = EWB_RING_TC;
constexpr int kNS = EWB_RING_NS;
constexpr int kStageElems = kRR * kTC;
constexpr int kRingBytes = kNS * kStageElems * 16;
// Thread mapping of a tile: kTC <= kSolveThreads -> kSlices row slices,
// thread = (slice, column), kRpt rows each; kTC > kSolveThreads -> one slice,
// thread = kCpt columns (col + m kSolveThreads) x all kRR rows.
constexpr int kSlices = kTC <= kSolveThreads ? kSolveThreads / kTC : 1;   // row slices per tile
constexpr int kRpt = kRR / kSlices;              // rows per thread
constexpr int kCpt = kTC <= kSolveThreads ? 1 : kTC / kSolveThreads;      // columns per thread
constexpr int kColSpan = kTC <= kSolveThreads ? kTC : kSolveThreads;      // threads per slice
static_assert((kSolveThreads % kTC == 0 || kTC % kSolveThreads == 0) && kRR % kSlices == 0,
              "tile geometry");

struct Ring {
  cplx* buf;            // dynamic shared memory, kNS stages
  uint64_t* bar;        // kNS mbarriers (static shared)
  unsigned pos;         // stages consumed so far by this CTA (uniform)
  unsigned evict_first; // L2 policy for A: evict_first (A larger than L2) or evict_last
};

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

// xk > 0: the same columns of xk input vectors (X + k n) ride in the stage's
// last xk row slots, so the consumers read x from shared memory.
__device__ __forceinline__ void ring_issue(const Ring& R, unsigned pos, const cplx* A, long long n,
                                           long long row0, int nrows, long long c0, int tc,
                                           const cplx* X = nullptr, int xk = 0) {
  const int b = pos % kNS;
  EWB_DCHECK(nrows >= 1 && nrows + xk <= kRR && tc >= 1 && tc <= kTC && row0 >= 0 &&
                 row0 + nrows <= n && c0 >= 0 && c0 + tc <= n, 101);
  const uint32_t bar = smem_u32(&R.bar[b]);
  const uint32_t bytes = (uint32_t)((nrows + xk) * tc * 16);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  // the policy is made here (issuing thread only) instead of living in
  // registers of every thread across the whole solve
  uint64_t pol;
  if (R.evict_first)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (int r = 0; r < nrows; ++r) {
    const uint32_t dst = smem_u32(R.buf + (size_t)b * kStageElems + r * kTC);
    const cplx* src = A + (row0 + r) * n + c0;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(tc * 16), "r"(bar), "l"(pol)
        : "memory");
  }
  if (xk > 0) {   // x stays in L2 for every CTA and row block: evict_last
    uint64_t polx;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(polx));
    for (int k = 0; k < xk; ++k) {
      const uint32_t dst = smem_u32(R.buf + (size_t)b * kStageElems + (kRR - xk + k) * kTC);
      const cplx* src = X + (long long)k * n + c0;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
          "l"(src), "r"(tc * 16), "r"(bar), "l"(polx)
          : "memory");
    }
  }
}

__device__ __forceinline__ void ring_wait(const Ring& R, unsigned pos) {
  const uint32_t bar = smem_u32(&R.bar[pos % kNS]);
  const uint32_t parity = (pos / kNS) & 1u;
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

constexpr int kMaxDots = 2 * kMaxRestart + 2;

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
__device__ __forceinline__ void cta_rows(long long n, long long& r0, long long& r1) {
  r0 = (long long)blockIdx.x * n / gridDim.x;
  r1 = ((long long)blockIdx.x + 1) * n / gridDim.x;
}

struct NoPre {
  __device__ __forceinline__ void operator()(long long, int) const {}
};
constexpr int kEpiPrefetch = 12;
// pre(row0, nrows) runs kEpiPrefetch tiles before a block's epilogue:
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
    ring_issue(R, R.pos + (unsigned)u, A, n, r0 + rel0, nr, (long long)t * kTC, tc);
  };
  if (threadIdx.x < kNS) s_rel[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int u = 0; u < S && u < kNS; ++u) issue(u);
  }
  const int col = threadIdx.x % kColSpan, slice = threadIdx.x / kColSpan;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  cplx acc[kRpt][K];
#pragma unroll
  for (int r = 0; r < kRpt; ++r)
#pragma unroll
    for (int k = 0; k < K; ++k) acc[r][k] = {0.0, 0.0};
  cplx xn[kCpt][K];  // x for the stage being consumed (prefetched one stage ahead)
#pragma unroll
  for (int m = 0; m < kCpt; ++m)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = col + m * kColSpan;
      xn[m][k] = c < n ? ldg(x + k * n + c) : cplx{0.0, 0.0};
    }
  int q = 0, t = 0;
  long long row0 = r0;
  int nrows = rows / nblk;
  for (int s = 0; s < S; ++s) {
    const long long c0 = (long long)t * kTC;
    const int tc = t == ntile - 1 ? last_tc : kTC;
    cplx xv[kCpt][K];
#pragma unroll
    for (int m = 0; m < kCpt; ++m)
#pragma unroll
      for (int k = 0; k < K; ++k) xv[m][k] = xn[m][k];
    {  // prefetch the next stage's x
      const long long cn = (t == ntile - 1 ? 0 : c0 + kTC) + col;
#pragma unroll
      for (int m = 0; m < kCpt; ++m)
#pragma unroll
        for (int k = 0; k < K; ++k)
          xn[m][k] = cn + m * kColSpan < n ? ldg(x + k * n + cn + m * kColSpan) : cplx{0.0, 0.0};
    }
    if (t == max(0, ntile - 1 - kEpiPrefetch)) pre(row0, nrows);
    const unsigned pos = R.pos + (unsigned)s;
    ring_wait(R, pos);
    {
      const cplx* tile = R.buf + (size_t)(pos % kNS) * kStageElems;
#pragma unroll
      for (int m = 0; m < kCpt; ++m) {
        const int c = col + m * kColSpan;
        if (c < tc) {
#pragma unroll
          for (int r = 0; r < kRpt; ++r) {
            const int row = slice * kRpt + r;
            if (row < nrows) {
              double2 a2 = *reinterpret_cast<const double2*>(tile + row * kTC + c);
              cplx av = {a2.x, a2.y};
#pragma unroll
              for (int k = 0; k < K; ++k) cfma(acc[r][k], av, xv[m][k]);
            }
          }
        }
      }
    }
    __syncwarp();
    int rel_old = -1;
    if ((threadIdx.x & 31) == 0) {
      rel_old = atomicAdd(&s_rel[pos % kNS], 1);
      EWB_DCHECK(rel_old >= 0 && rel_old < kSolveWarps, 102);
    }
    if (rel_old == kSolveWarps - 1) {  // last reader of the slot
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
#ifdef EWB_DEBUG_CHECKS
  __syncthreads();
  if (threadIdx.x < kNS) EWB_DCHECK(s_rel[threadIdx.x] == 0, 103);  // every slot released
#endif
  R.pos += (unsigned)S;
}

// Multi-column matvec (K = 3, 4).  XS = false: kSl = 4 row slices x kRR / 4
// rows; a slice's 128 threads take kTC / 128 columns of every tile and keep
// the next stage's x (kCp x K values) in registers, loaded from global memory
// by every slice.  XS = true (the default for SEM's Y = A X): the stage holds
// kRA = 8 rows of A plus the K x-chunks of the same columns, all brought in by
// the same bulk-copy transaction, 2 row slices x 4 rows x 2 columns per
// thread: x costs no registers, no L2 round trip inside the consumer loop and
// half the replication (measured, tools/sem_time.py).
template <int K, bool XS, typename Epi>
__device__ void matvec_rows_wide(Ring& R, const cplx* __restrict__ A, long long n, const cplx* x,
                            long long r0, long long r1, Epi&& epi) {
  constexpr int kSl = XS ? 2 : 4, kRA = XS ? 8 : kRR, kRw = kRA / kSl;
  constexpr int kCols = kSolveThreads / kSl, kCp = kTC / kCols;
  static_assert(kRA % kSl == 0 && kTC % kCols == 0 && kRA + (XS ? K : 0) <= kRR,
                "matvec_rows_wide layout");
  __shared__ cplx s_red[kSolveWarps][kRw][K];
  __shared__ cplx s_sum[kRA][K];
  __shared__ int s_rel[kNS];  // warps done with each ring slot
  const int rows = (int)(r1 - r0);
  if (rows <= 0) return;
  const int nblk = (rows + kRA - 1) / kRA;
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
               XS ? x : nullptr, XS ? K : 0);
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
  cplx xn[XS ? 1 : kCp][K];  // x of the stage being consumed (XS: one column at a time)
  if (!XS) {
#pragma unroll
    for (int m = 0; m < kCp; ++m)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = col + m * kCols;
        xn[XS ? 0 : m][k] = c < n ? ldg(x + k * n + c) : cplx{0.0, 0.0};
      }
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
          if (XS) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
              double2 x2 = *reinterpret_cast<const double2*>(tile + (kRR - K + k) * kTC + c);
              xn[0][k] = {x2.x, x2.y};
            }
          }
#pragma unroll
          for (int r = 0; r < kRw; ++r) {
            const int row = slice * kRw + r;
            if (row < nrows) {
              double2 a2 = *reinterpret_cast<const double2*>(tile + row * kTC + c);
              cplx av = {a2.x, a2.y};
#pragma unroll
              for (int k = 0; k < K; ++k) cfma(acc[r][k], av, xn[XS ? 0 : m][k]);
            }
          }
        }
      }
    }
    if (!XS) {  // x for the next stage
      const long long cb = (t == ntile - 1 ? 0 : c0 + kTC) + col;
#pragma unroll
      for (int m = 0; m < kCp; ++m)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const long long cn = cb + m * kCols;
          xn[XS ? 0 : m][k] = cn < n ? ldg(x + k * n + cn) : cplx{0.0, 0.0};
        }
    }
    __syncwarp();
    int rel_old = -1;
    if ((threadIdx.x & 31) == 0) {
      rel_old = atomicAdd(&s_rel[pos % kNS], 1);
      EWB_DCHECK(rel_old >= 0 && rel_old < kSolveWarps, 102);
    }
    if (rel_old == kSolveWarps - 1) {  // last reader of the slot
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
      if (threadIdx.x < kRA * K) {
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
#ifdef EWB_DEBUG_CHECKS
  __syncthreads();
  if (threadIdx.x < kNS) EWB_DCHECK(s_rel[threadIdx.x] == 0, 103);  // every slot released
#endif
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

// ---------------------------------------------------------------------
// GMRES with the Arnoldi vector work fused around the matvec: the
// reference's MGS (linsolve.py:150-170) in its one-reduction form
//   h_i = <v_i, w - sum_{l<i} h_l v_l> = d_i - sum_{l<i} <v_i, v_l> h_l,
// d_i = <v_i, w>, i.e. h = (I + L)^{-1} d with L the strictly lower part of
// the basis's Gram matrix (same coefficients up to floating-point
// association), arranged so that an Arnoldi step costs one pass over A
// plus two grid barriers:
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


__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_gmres_f(GmresArgs a) {
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
    if (rnorm / nb <= a.tol) {  // a 0-iteration exit is decided on b - A x0 itself
      rnorm = residual(dpar);
      dpar ^= 1;
      ++n_mv;
    }
  } else if (v2[1] > 0.0) {  // r = b - A x0 (linsolve.py:144)
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
      if (a.W) a.rs[k] = a.r[k];   // the cycle's starting residual
    }
    grid.sync();
    double hprev = beta;
    int used = 0;
    for (int j = 0;; ++j) {
      // ---- matvec + <V_t, w> partials ------------------------------------
      const double sc = 1.0 / hprev;
      for (int t = threadIdx.x; t <= j; t += blockDim.x) s_dacc[t] = {0.0, 0.0};
      __syncthreads();
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
      cplx* part = part_buf(dpar);
      for (int t = threadIdx.x; t <= j; t += blockDim.x)
        part[(size_t)blockIdx.x * kMaxDots + t] = s_dacc[t];
      // Gram rows 1..j-1 (written in earlier steps) staged into the idle
      // ring while other CTAs finish their matvec
      cplx* gsm = scr;
      {
        const int tri = j * (j - 1) / 2;
        if (threadIdx.x == 0) EWB_DCHECK(tri <= kRingBytes / 16, 105);
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
      // ---- d_t and Gram row j; h = (I + L)^{-1} d --------------------------
      {
        // reduce-scatter (CTA b sums value t = b mod G over the CTA partials
        // in a fixed order) + barrier + all-gather: every partial is read
        // once instead of once per CTA
        cplx* fin = reinterpret_cast<cplx*>(a.partial);
        const int cnt = 2 * j + 1;
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
        grid.sync();  // S1b
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) s_dots[t] = fin[t];
        __syncthreads();
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
        }
      }
      // ---- update: u = w - sum_i h_i V_i over [ka, kb) --------------------
      {
        const int nv = j + 1;
        const int nc = max(1, min(nv, kSolveThreads / max(RU, 1)));
        cplx* pu = scr;            // [nc][RU] chunk partials
        cplx* su = scr + nc * RU;  // [RU] u
        if (threadIdx.x == 0) EWB_DCHECK(RU >= 0 && nc * RU + RU <= kRingBytes / 16, 104);
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
      grid.sync();  // S2
      const double hn = sqrt(grid_norm(dpar));
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
      if (threadIdx.x == 0) EWB_DCHECK(used * (used + 1) / 2 <= kRingBytes / 16, 106);
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
    // Cycle end (linsolve.py:200-201).  The restart residual comes from the
    // products this cycle already computed, b - A x_new = r_start - sum_i
    // y_i (A P^{-1} v_i) (no pass over A; equal up to rounding of |A x|).
    // Every exit decision — converged, or out of iterations — is taken on
    // the literal b - A x (one pass), the quantity the reference tests and
    // reports, so final_residual is always the true relative residual.
    bool literal = a.W == nullptr || its >= a.maxiter;
    if (!literal) {
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
      dpar ^= 1;
      literal = rnorm / nb <= a.tol;
    }
    if (literal) {
      rnorm = residual(dpar);
      ++n_mv;
      dpar ^= 1;
    }
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
// SEM (linsolve.py:213-242): Y = A X (passes of up to 4 columns over A),
// QR of Y[:, keep] by classical Gram-Schmidt with one re-orthogonalisation
// (|R_ii| agrees with Householder's to rounding), rank filter
// |R_ii| >= rank_tol * max|R_ii| (<= 2 passes), x0 = X s with R s = Q^H b;
// falls back to the newest column.
// ---------------------------------------------------------------------
__device__ void sem_body(cg::grid_group& grid, GridRed& R, const SemArgs& a) {
  const long long n = a.n, tid = gtid(), nth = gthreads();
  // Y = A X was produced by k_multi_gemv (its own launch: the K-vector
  // matvec needs more registers than this cooperative kernel can give it),
  // or by the matrix-free operator (ewb_sem_from_products)
  __shared__ int keep[kMaxSem];
  __shared__ cplx Rm[kMaxSem][kMaxSem];
  __shared__ int nkeep;
  if (threadIdx.x == 0) {
    nkeep = a.K;
    EWB_DCHECK(a.K >= 1 && a.K <= kMaxSem, 107);
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
  sem_body(grid, R, a);
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

long long ring_cplx_capacity() { return kRingBytes / 16; }

int solver_grid_blocks() {
  const int m = solver_grid_max();
  return g_solver_limit > 0 && g_solver_limit < m ? g_solver_limit : m;
}

int solver_grid_max() {
  if (g_coop_blocks == 0) {
    const int a = coop_grid((const void*)k_sem), b = coop_grid((const void*)k_gmres_f);
    g_coop_blocks = a < b ? a : b;
  }
  return g_coop_blocks;
}

cudaError_t launch_gmres(GmresArgs& args, cudaStream_t s) {
  int G = solver_grid_blocks();
  void* params[] = {&args};
  note_launch();
  return cudaLaunchCooperativeKernel((const void*)k_gmres_f, dim3(G), dim3(kSolveThreads), params, kRingBytes, s);
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
#ifdef EWB_SEM_X_GLOBAL
  constexpr bool kXs = false;
#else
  constexpr bool kXs = kRR >= 8 + K && kTC % (kSolveThreads / 2) == 0;   // x staged in the ring
#endif
  if constexpr (K <= 2) matvec_rows<K>(ring, A, n, X, r0, r1, store);
  else matvec_rows_wide<K, kXs>(ring, A, n, X, r0, r1, store);
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
  // Y = A X in passes of up to 4 columns (K = 3, 4 with the 4-slice layout)
  for (int c0 = 0; c0 < args.K; c0 += 4) {
    const cplx* X = args.X + (size_t)c0 * args.n;
    cplx* Y = args.Y + (size_t)c0 * args.n;
    cudaError_t e;
    switch (args.K - c0 < 4 ? args.K - c0 : 4) {
      case 1: e = launch_multi_gemv<1>(args.A, X, Y, args.n, s); break;
      case 2: e = launch_multi_gemv<2>(args.A, X, Y, args.n, s); break;
      case 3: e = launch_multi_gemv<3>(args.A, X, Y, args.n, s); break;
      default: e = launch_multi_gemv<4>(args.A, X, Y, args.n, s); break;
    }
    if (e != cudaSuccess) return e;
  }
  return launch_sem_products(args, s);
}

cudaError_t launch_sem_products(SemArgs& args, cudaStream_t s) {
  int G = solver_grid_blocks();
  void* params[] = {&args};
  note_launch();
  return cudaLaunchCooperativeKernel((const void*)k_sem, dim3(G), dim3(kSolveThreads), params,
                                     kRingBytes, s);
}

// ---------------------------------------------------------------------
// Operator GMRES (matrix-free seam): the reference's algorithm
// (linsolve.py:107-210) with the operator applied by separate launches and
// every vector, coefficient and decision on the device (OpState).  MGS is
// the reference's sequential form (one grid reduction per projection, the
// update of projection i fused with the dot of projection i+1).
// ---------------------------------------------------------------------
// operator input for vector v: z = P^{-1} v, vt = mask_N z, vu = -mask_D z
__device__ void op_stage_input(const OpArgs& a, const cplx* v, bool precond) {
  const long long n = a.n, tid = gtid(), nth = gthreads();
  const bool pc = precond && a.pinv != nullptr;
  if (!pc && !a.kinds) {   // plain copy (any n)
    for (long long k = tid; k < n; k += nth) {
      a.z[k] = v[k];
      a.vt[k] = v[k];
    }
    return;
  }
  for (long long e = tid; e < n / 3; e += nth) {
    cplx z[3] = {v[3 * e], v[3 * e + 1], v[3 * e + 2]};
    if (pc) {
      const cplx* P = a.pinv + 9 * e;
      cplx o[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {   // einsum('bij,bj->bi') order
        cplx s = P[3 * r] * z[0];
        s = s + P[3 * r + 1] * z[1];
        s = s + P[3 * r + 2] * z[2];
        o[r] = s;
      }
      z[0] = o[0]; z[1] = o[1]; z[2] = o[2];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long k = 3 * e + c;
      a.z[k] = z[c];
      const bool dir = a.kinds && a.kinds[k] == kDirichlet;
      a.vt[k] = dir ? cplx{0.0, 0.0} : z[c];
      if (a.vu) a.vu[k] = dir ? cplx{-z[c].re, -z[c].im} : cplx{0.0, 0.0};
    }
  }
}

// Scalar state: every CTA keeps an identical copy of the head (OpHead) in
// shared memory, modified by its thread 0 only, and block 0 writes it back
// after a grid barrier that follows every CTA's read.

// cycle start from the residual in a.r, |r| = s.rnorm (linsolve.py:153-163)
__device__ void op_start_cycle(cg::grid_group& grid, const OpArgs& a, OpHead& s) {
  const long long n = a.n, tid = gtid(), nth = gthreads();
  const double beta = s.rnorm;
  for (long long k = tid; k < n; k += nth) {
    a.V[k] = {a.r[k].re / beta, a.r[k].im / beta};
    a.rs[k] = a.r[k];
  }
  grid.sync();
  op_stage_input(a, a.V, true);
  __syncthreads();
  if (threadIdx.x == 0) {
    s.m = min(a.restart, a.maxiter - s.its);
    s.j = 0;
    s.used = 0;
    s.in_cycle = 1;
    s.cycle_open = 1;
    if (blockIdx.x == 0) {
      a.st->g[0] = {beta, 0.0};
      for (int k = 1; k <= s.m; ++k) a.st->g[k] = {0.0, 0.0};
    }
  }
  __syncthreads();
}

// exit on the literal residual (linsolve.py:200-205): next apply is A x
__device__ void op_request_literal(const OpArgs& a, OpHead& s) {
  op_stage_input(a, a.x, false);
  __syncthreads();
  if (threadIdx.x == 0) s.lit_pending = 1;
  __syncthreads();
}

__device__ void op_exit(const OpArgs& a, OpHead& s) {
  if (threadIdx.x == 0) {
    s.done = 1;
    s.final_res = s.res;
    s.converged = s.res <= a.tol;
  }
  __syncthreads();
}

__device__ void op_writeback(cg::grid_group& grid, const OpArgs& a, const OpHead& s) {
  grid.sync();   // every CTA has read the old head
  if (blockIdx.x == 0 && threadIdx.x == 0) a.st->h = s;
}

__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_op_begin(OpArgs a) {
  cg::grid_group grid = cg::this_grid();
  GridRed R{a.partial, 0};
  __shared__ OpHead s;
  const long long n = a.n, tid = gtid(), nth = gthreads();
  if (threadIdx.x == 0) memset(&s, 0, sizeof(OpHead));
  __syncthreads();
  double v2[2] = {0.0, 0.0};
  for (long long k = tid; k < n; k += nth) {
    v2[0] += abs2(a.b[k]);
    if (a.has_x0) v2[1] += (a.x[k].re != 0.0 || a.x[k].im != 0.0);
    else a.x[k] = {0.0, 0.0};
  }
  grid_sum(grid, R, v2);
  const double nb = sqrt(v2[0]);
  if (threadIdx.x == 0) s.nb = nb;
  __syncthreads();
  if (nb == 0.0) {   // linsolve.py:136-140
    for (long long k = tid; k < n; k += nth) a.x[k] = {0.0, 0.0};
    if (threadIdx.x == 0) { s.done = 1; s.converged = 1; }
    __syncthreads();
  } else if (v2[1] > 0.0 && !a.ax0) {   // r0 = b - A x0 needs an application
    op_request_literal(a, s);
  } else {
    double q[1] = {0.0};
    for (long long k = tid; k < n; k += nth) {
      const cplx r = v2[1] > 0.0 ? a.b[k] - a.ax0[k] : a.b[k];
      a.r[k] = r;
      q[0] += abs2(r);
    }
    grid_sum(grid, R, q);
    const double rn = sqrt(q[0]), res = rn / nb;
    if (v2[1] > 0.0 && res <= a.tol) {
      op_request_literal(a, s);   // a 0-iteration exit is decided on b - A x0
    } else {
      if (threadIdx.x == 0) {
        s.rnorm = rn; s.res = res; s.init_res = res; s.n_hist = 1;
        if (tid == 0) a.hist[0] = res;
      }
      __syncthreads();
      if (res <= a.tol || a.maxiter <= 0) op_exit(a, s);
      else op_start_cycle(grid, a, s);
    }
  }
  op_writeback(grid, a, s);
}

// r = b - A x from the literal application; exit or restart
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_op_settle(OpArgs a) {
  cg::grid_group grid = cg::this_grid();
  GridRed R{a.partial, 0};
  __shared__ OpHead s;
  if (threadIdx.x == 0) s = a.st->h;
  __syncthreads();
  if (!s.lit_pending) return;   // uniform over the grid
  const long long n = a.n, tid = gtid(), nth = gthreads();
  double q[1] = {0.0};
  for (long long k = tid; k < n; k += nth) {
    const cplx r = a.b[k] - a.w[k];
    a.r[k] = r;
    q[0] += abs2(r);
  }
  grid_sum(grid, R, q);
  const double rn = sqrt(q[0]), res = rn / s.nb;
  if (threadIdx.x == 0) {
    s.rnorm = rn;
    s.res = res;
    s.lit_pending = 0;
    s.applies += 1;
    if (s.n_hist == 0) {   // the initial residual (linsolve.py:144-147)
      s.init_res = res;
      s.n_hist = 1;
      if (tid == 0) a.hist[0] = res;
    }
  }
  __syncthreads();
  if (res <= a.tol || s.its >= a.maxiter) op_exit(a, s);
  else op_start_cycle(grid, a, s);
  op_writeback(grid, a, s);
}

// one Arnoldi step on w = A P^{-1} v_j (linsolve.py:164-194)
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_op_step(OpArgs a) {
  cg::grid_group grid = cg::this_grid();
  GridRed R{a.partial, 0};
  __shared__ OpHead s;
  __shared__ cplx hc[kMaxRestart + 1];            // new Hessenberg column
  __shared__ cplx cs_new, sn_new, gj_new, gj1_new;
  if (threadIdx.x == 0) s = a.st->h;
  __syncthreads();
  if (!s.in_cycle) return;   // uniform over the grid
  const long long n = a.n, tid = gtid(), nth = gthreads();
  const int j = s.j;
  cplx* w = a.r;   // working vector (the cycle's start residual is in a.rs)
  // MGS: h_i = <v_i, w>, w -= h_i v_i; the update of projection i-1 and the
  // dot of projection i share one sweep; the last sweep gives |w|^2
  cplx h = {0.0, 0.0};
  for (int i = 0; i <= j + 1; ++i) {
    double d[2] = {0.0, 0.0};
    const cplx* vi = a.V + (size_t)i * n;
    const cplx* vp = a.V + (size_t)(i > 0 ? i - 1 : 0) * n;
    for (long long k = tid; k < n; k += nth) {
      cplx wk;
      if (i == 0) {
        wk = a.w[k];
        a.W[(size_t)j * n + k] = wk;
      } else {
        wk = w[k] - h * vp[k];
      }
      w[k] = wk;
      if (i <= j) {
        const cplx p = conj(vi[k]) * wk;
        d[0] += p.re; d[1] += p.im;
      } else {
        d[0] += abs2(wk);
      }
    }
    grid_sum(grid, R, d);
    h = i <= j ? cplx{d[0], d[1]} : cplx{sqrt(d[0]), 0.0};
    if (threadIdx.x == 0) hc[i] = h;
  }
  __syncthreads();
  const double hn = hc[j + 1].re;
  if (threadIdx.x == 0) {   // Givens, identical in every CTA
    const OpState* S = a.st;
    for (int i = 0; i < j; ++i) {   // previous rotations on the new column
      const cplx hi = hc[i], hi1 = hc[i + 1];
      hc[i] = S->cs[i] * hi + S->sn[i] * hi1;
      hc[i + 1] = (-conj(S->sn[i])) * hi + conj(S->cs[i]) * hi1;
    }
    const cplx hjj = hc[j], hj1 = hc[j + 1];
    const double ahj = hypot(hjj.re, hjj.im), ahn = hypot(hj1.re, hj1.im);
    const double den = sqrt(ahj * ahj + ahn * ahn);
    cplx c, sn;
    if (den == 0.0) {
      c = {1.0, 0.0}; sn = {0.0, 0.0};
    } else if (hjj.re == 0.0 && hjj.im == 0.0) {
      c = {0.0, 0.0}; sn = {1.0, 0.0};
    } else {
      c = {ahj / den, 0.0};
      const cplx ph = {hjj.re / ahj, hjj.im / ahj};
      const cplx t = ph * conj(hj1);
      sn = {t.re / den, t.im / den};
    }
    hc[j] = c * hjj + sn * hj1;
    hc[j + 1] = {0.0, 0.0};
    const cplx gj = S->g[j];
    cs_new = c;
    sn_new = sn;
    gj1_new = (-conj(sn)) * gj;
    gj_new = c * gj;
    const double est = hypot(gj1_new.re, gj1_new.im) / s.nb;
    if (tid == 0 && s.n_hist < a.hist_cap) a.hist[s.n_hist] = est;
    s.n_hist += 1;
    s.its += 1;
    s.applies += 1;
    s.used = j + 1;
    s.j = j + 1;
    if (est <= a.tol || j + 1 == s.m) s.in_cycle = 0;
  }
  __syncthreads();
  grid.sync();   // every CTA has read cs, sn, g before block 0 updates them
  if (blockIdx.x == 0) {
    OpState* S = a.st;
    for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) S->H[i * kMaxRestart + j] = hc[i];
    if (threadIdx.x == 0) {
      S->cs[j] = cs_new;
      S->sn[j] = sn_new;
      S->g[j] = gj_new;
      S->g[j + 1] = gj1_new;
      S->h = s;
    }
  }
  if (s.in_cycle) {
    cplx* vn = a.V + (size_t)(j + 1) * n;
    if (hn > 0.0)
      for (long long k = tid; k < n; k += nth) vn[k] = {w[k].re / hn, w[k].im / hn};
    grid.sync();
    op_stage_input(a, vn, true);
  }
}

// back substitution, x update, restart residual (linsolve.py:195-201)
__global__ void __launch_bounds__(kSolveThreads, kSolveMinBlocks) k_op_cycle_end(OpArgs a) {
  cg::grid_group grid = cg::this_grid();
  GridRed R{a.partial, 0};
  __shared__ OpHead s;
  __shared__ cplx y[kMaxRestart];
  if (threadIdx.x == 0) s = a.st->h;
  __syncthreads();
  if (!s.cycle_open || s.in_cycle) return;   // uniform over the grid
  const long long n = a.n, tid = gtid(), nth = gthreads();
  const int used = s.used;
  if (threadIdx.x == 0) {
    const OpState* S = a.st;
    for (int i = used - 1; i >= 0; --i) {
      cplx t = S->g[i];
      for (int k = i + 1; k < used; ++k) t = t - S->H[i * kMaxRestart + k] * y[k];
      y[i] = cdiv(t, S->H[i * kMaxRestart + i]);
    }
  }
  __syncthreads();
  // x += P^{-1} (V y) and r = r_start - W y (= b - A x_new up to rounding);
  // unit u = element (3 DOFs, preconditioned) or a single DOF
  const bool pc = a.pinv != nullptr;
  const int per = pc ? 3 : 1;
  double q[1] = {0.0};
  for (long long e = tid; e < n / per; e += nth) {
    cplx u[3];
    for (int c = 0; c < per; ++c) {
      const long long k = per * e + c;
      cplx sv = {0.0, 0.0}, sr = a.rs[k];
      for (int i = 0; i < used; ++i) {
        cfma(sv, a.V[(size_t)i * n + k], y[i]);
        sr = sr - y[i] * a.W[(size_t)i * n + k];
      }
      u[c] = sv;
      a.r[k] = sr;
      q[0] += abs2(sr);
    }
    if (pc) {
      const cplx* P = a.pinv + 9 * e;
#pragma unroll
      for (int r = 0; r < 3; ++r) {   // einsum order, as block_diag_precond
        cplx t = P[3 * r] * u[0];
        t = t + P[3 * r + 1] * u[1];
        t = t + P[3 * r + 2] * u[2];
        a.x[3 * e + r] = a.x[3 * e + r] + t;
      }
    } else {
      a.x[e] = a.x[e] + u[0];
    }
  }
  grid_sum(grid, R, q);   // also orders the x update before the staging below
  const double rn = sqrt(q[0]), res = rn / s.nb;
  if (threadIdx.x == 0) {
    s.cycle_open = 0;
    s.rnorm = rn;
    s.res = res;
  }
  __syncthreads();
  if (res <= a.tol || s.its >= a.maxiter) op_request_literal(a, s);
  else op_start_cycle(grid, a, s);
  op_writeback(grid, a, s);
}

cudaError_t launch_op_gmres(int phase, OpArgs& args, cudaStream_t s) {
  const void* fn = phase == 0 ? (const void*)k_op_begin
                   : phase == 1 ? (const void*)k_op_step
                   : phase == 2 ? (const void*)k_op_cycle_end
                                : (const void*)k_op_settle;
  int G = solver_grid_blocks();
  void* params[] = {&args};
  note_launch();
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kSolveThreads), params, 0, s);
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
