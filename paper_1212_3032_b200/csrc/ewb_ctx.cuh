// Device-resident per-mesh context (the state the reference keeps in its
// Assembler, assembly.py:103-216) and the internal launch interfaces.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ewb_common.cuh"

namespace ewb {

constexpr int kSelfQ = 384;          // 3 sub-triangles x 8 radial x 16 angular
constexpr int kMaxNearLevel = 4;     // quadrature.py:209 (levels 1..4)
constexpr int kWarpsPerBlock = 4;

// Quadrature rule table offsets (device buffer `rules`):
//   bary (Q,3) then w (Q) for gauss3, gauss7, gauss7-sub1..4.
struct RuleRef {
  int off, q;
};

// Structure-of-arrays mesh geometry on the device.
struct Geo {
  int n_e;
  const double *cx, *cy, *cz;        // centroids (collocation points)
  const double *nx, *ny, *nz;        // unit normals
  const double *area, *diam;         // area, diameter (longest edge)
  const double *vx, *vy, *vz;        // corners [3][n_e] each (v0, v1, v2 blocks)
  const double *yfar;                // [3 q][3 comp][n_e] gauss3 field points
  const double *ymid;                // [7 q][3 comp][n_e] gauss7 field points
  const double *wfar, *wmid;         // rule weights (unscaled), 3 and 7
  const double4 *self_pts;           // [n_e][384] (x, y, z, w*area folded)
  const int *near_ptr;               // CSR by row, n_e+1
  const int *near_j;                 // column of each near pair
  const int *near_lvl;               // subdivision level 1..4
  const int *near_row;               // row of each near pair
  const int *near_order;             // launch order of the near pairs (deepest level first)
  const int *mid_ptr;                // CSR by row of the mid (gauss7) pairs, n_e+1
  const int *mid_j;                  // column of each mid pair
  const int *mid_row;                // row of each mid pair
  const double *rules;               // rule tables
  RuleRef sub[kMaxNearLevel + 1];    // sub[L] for L = 1..4
};

// ---------------------------------------------------------------------
// exact tier: numpy's  norm(c_i - c_j, axis=-1) / diam_j  without FMA
// contraction, left-associated sum ((dx^2 + dy^2) + dz^2) — the box meshes
// have hundreds of pairs whose ratio is exactly 4.0.
// ---------------------------------------------------------------------
__device__ __forceinline__ int exact_tier(double xi, double yi, double zi, double xj,
                                          double yj, double zj, double dj) {
  double dx = __dsub_rn(xi, xj), dy = __dsub_rn(yi, yj), dz = __dsub_rn(zi, zj);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  double ratio = __ddiv_rn(__dsqrt_rn(s), dj);
  return ratio < kNearRatio ? 2 : (ratio < kFarRatio ? 1 : 0);
}

// Same decision, cheaply: compare |c_i - c_j|^2 with 16 d_j^2 and 2.25 d_j^2
// (no sqrt, no divide) and take the exact numpy-rounding path above only
// within 1e-12 (relative) of a threshold, where rounding could decide.
// (Measured: faster in the matrix-free N-body kernel, slower in the dense
// k_farmid where the extra branches cost more than the divide they save.)
__device__ __forceinline__ int exact_tier_fast(double xi, double yi, double zi, double xj,
                                               double yj, double zj, double dj) {
  const double dx = xi - xj, dy = yi - yj, dz = zi - zj;
  const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double dj2 = dj * dj;
  const double far2 = kFarRatio * kFarRatio * dj2, near2 = kNearRatio * kNearRatio * dj2;
  constexpr double lo = 1.0 - 1e-12, hi = 1.0 + 1e-12;
  if (d2 > far2 * hi) return 0;
  if (d2 < near2 * lo) return 2;
  if (d2 > near2 * hi && d2 < far2 * lo) return 1;
  return exact_tier(xi, yi, zi, xj, yj, zj, dj);
}

__device__ __forceinline__ void load_corners(const Geo& g, int j, double v[9]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    v[3 * k] = g.vx[k * g.n_e + j];
    v[3 * k + 1] = g.vy[k * g.n_e + j];
    v[3 * k + 2] = g.vz[k * g.n_e + j];
  }
}

template <bool DYN>
struct Phys;
template <>
struct Phys<true> {
  using S = cplx;
  FreqConst fc;
  __device__ __forceinline__ void point(Acc<cplx>& A, double r, double ir, double dx, double dy,
                                        double dz, double dn, double w) const {
    point_dynamic(A, fc, r, ir, dx, dy, dz, dn, w);
  }
  __device__ __forceinline__ double i4pm() const { return fc.inv4pimu; }
  __device__ __forceinline__ double i4p() const { return fc.inv4pi; }
};
template <>
struct Phys<false> {
  using S = double;
  StaticConst sc;
  __device__ __forceinline__ void point(Acc<double>& A, double r, double ir, double dx, double dy,
                                        double dz, double dn, double w) const {
    (void)r;
    point_static(A, sc, ir, dx, dy, dz, dn, w);
  }
  __device__ __forceinline__ double i4pm() const { return sc.inv4pimu; }
  __device__ __forceinline__ double i4p() const { return sc.inv4pi; }
};

__device__ __forceinline__ bool finite(double v) { return isfinite(v); }
__device__ __forceinline__ bool finite(cplx v) { return isfinite(v.re) && isfinite(v.im); }
__device__ __forceinline__ cplx to_c(double v) { return {v, 0.0}; }
__device__ __forceinline__ cplx to_c(cplx v) { return v; }

// Multi-frequency batch: per-frequency constants plus the
// phase step used when the batch is equispaced in Re(omega) with one
// Im(omega) (every exponential-window sweep: omega_k = k dw - i eta).
constexpr int kMaxBatch = 32;
struct FreqBatch {
  FreqConst fc[kMaxBatch];
  int nf;
  int recur;                         // 1: step the phase factors across the batch
  double dks, dkp;                   // Re(ks), Re(kp) step between consecutive members
  double cr2, c4r;                   // ratio - 2, 4 - ratio (ratio = c_p^2 / c_s^2)
};

// Outputs of a multi-frequency system assembly; member f of every array
// starts at f x its per-frequency size.
struct SysBatch {
  const uint8_t* kinds;              // (N,)
  const cplx* p;                     // (nf, N) prescribed values
  cplx* A;                           // (nf, N, N)
  cplx* b;                           // (nf, N)
  cplx* pinv;                        // (nf, n_e, 3, 3)
  int* flags;                        // (nf, 4): [0] non-finite, [1] singular blocks
  cplx* bpart;                       // (nf, n_tiles, N) far b partials
  cplx* bmid;                        // (nf, n_mid, 3)
  cplx* bnear;                       // (nf, n_near, 3)
};

struct Context {
  int n_e = 0;
  int n_near = 0;
  int n_tiles = 0;                   // column tiles of 32
  long long n_far = 0, n_mid = 0;    // off-diagonal pair counts per tier
  long long n_near_lvl[kMaxNearLevel + 1] = {0, 0, 0, 0, 0};
  double lam = 0, mu = 0, rho = 0;
  double min_diam = 0;               // shortest longest-edge (far-pair distance bound)
  int exterior = 0;                  // 1: c + PV int T = I diagonal
  Geo g{};
  // owned device buffers
  std::vector<void*> owned;
  double* rowsums = nullptr;         // [n_e][9] static off-diagonal T row sums
  double* u_sta_self = nullptr;      // [n_e][9]
  double* t_sta_self = nullptr;      // [n_e][9]
  double* diag_base = nullptr;       // [n_e][9] = -rowsums - t_sta_self
  cplx* bpart = nullptr;             // [n_tiles][3 n_e] far/mid b partials
  cplx* bnear = nullptr;             // [n_near][3] near-pair b partials
  double* spart = nullptr;           // [n_tiles][n_e][9] static row-sum partials
  double* snear = nullptr;           // [n_near][9]
  int* flags = nullptr;              // [0] non-finite seen, [1] singular blocks
  // multi-frequency scratch, allocated on first use for nf_cap members
  int nf_cap = 0;
  cplx* bpart_m = nullptr;
  cplx* bmid_m = nullptr;
  cplx* bnear_m = nullptr;
  cudaStream_t stream = nullptr;
};

StaticConst static_const(const Context& c);
FreqConst freq_const(const Context& c, double ore, double oim);

// kernels launched by the C API (ewb_assembly.cu)
cudaError_t setup_context(Context& c, const double* centroids, const double* normals,
                          const double* areas, const double* diameters,
                          const double* corners, const double* gl8, const double* gl16,
                          const double* rules_host, const int* rule_off, const int* rule_q,
                          cudaStream_t s);
cudaError_t launch_static_pass(Context& c, double* t_out, double* u_out, cudaStream_t s);
cudaError_t launch_assemble_tu(Context& c, double ore, double oim, cplx* T, cplx* U,
                               cudaStream_t s);
cudaError_t launch_assemble_system(Context& c, double ore, double oim, const uint8_t* kinds,
                                   const cplx* prescribed, cplx* A, cplx* b, cplx* pinv,
                                   cudaStream_t s);
cudaError_t launch_apply_bcs(const cplx* T, const cplx* U, const uint8_t* kinds,
                             const cplx* p, long long n, cplx* A, cplx* b, cudaStream_t s);
cudaError_t launch_blockdiag_inverse(const cplx* A, long long n, cplx* pinv, int* singular,
                                     cudaStream_t s);
cudaError_t set_exterior(Context& c, int on, cudaStream_t s);
// nf frequencies in one pass over the element pairs (batch buffers: SysBatch)
cudaError_t launch_assemble_system_multi(Context& c, int nf, const double* ore,
                                         const double* oim, const uint8_t* kinds,
                                         const cplx* prescribed, cplx* A, cplx* b, cplx* pinv,
                                         int* flags, cudaStream_t s);

}  // namespace ewb
