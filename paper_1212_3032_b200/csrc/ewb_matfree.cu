// Matrix-free operator application and the pair-kernel microbenchmark.
//
// Matrix-free (north-star item 2; seam: gmres(apply_a=callable),
// linsolve.py:73-77).  For meshes whose dense (N,N) matrix exceeds HBM the
// operator is recomputed in every application:
//     y_k = T vt_k + U vu_k ,   k < K
// which covers A v (vt = mask_N v, vu = -mask_D v; assembly.py:293-294),
// the right-hand side b = U mask_N p - T mask_D p (assembly.py:295-296) and
// the SEM product Y = A X (K columns in one pass, linsolve.py:228).  The
// quadrature ladder, exact tiers, near grading, self rule and rigid-body
// diagonal are the dense assembler's (assembly.py:122-254).
//
// Far/mid pairs use an N-body decomposition: a thread owns a collocation
// row i, a CTA stages 32 column elements at a time (geometry, field points
// and the K input 3-vectors) in shared memory, and every thread applies
// the 3x3 blocks straight from the contraction accumulators, so no block
// is ever stored.  Column chunks (blockIdx.y) write partial results that a
// final pass sums in a fixed order with the near pairs (warp per pair)
// and the self term (warp per element): deterministic, no atomics.
#include <cuda_runtime.h>

#include <type_traits>
#include <vector>

#include "ewb_ctx.cuh"

namespace ewb {
EWB_DEBUG_TU(matfree)

constexpr int kMfTile = 32;
constexpr int kMfMaxK = 5;

// (T v)_a and (U v)_a straight from the accumulators (kernels.py:336-356):
//   U v = (su v - P v) / (4 pi mu)
//   T v = (sa v + n (va . v) + B v + vc (n . v)) / (4 pi)
__device__ __forceinline__ void acc_apply_T(const Acc<cplx>& A, double nx, double ny, double nz,
                                            double c2, const cplx v[3], cplx y[3]) {
  cplx vav = A.va[0] * v[0];
  cfma(vav, A.va[1], v[1]);
  cfma(vav, A.va[2], v[2]);
  cplx nv = nx * v[0] + ny * v[1] + nz * v[2];
  const double n[3] = {nx, ny, nz};
  const int sym[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cplx t = A.sa * v[a];
    t = t + n[a] * vav;
    cfma(t, A.B[sym[a][0]], v[0]);
    cfma(t, A.B[sym[a][1]], v[1]);
    cfma(t, A.B[sym[a][2]], v[2]);
    cfma(t, A.vc[a], nv);
    y[a] = y[a] + c2 * t;
  }
}

__device__ __forceinline__ void acc_apply_U(const Acc<cplx>& A, double c1, const cplx v[3],
                                            cplx y[3]) {
  const int sym[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cplx t = A.su * v[a];
    cplx pv = A.P[sym[a][0]] * v[0];
    cfma(pv, A.P[sym[a][1]], v[1]);
    cfma(pv, A.P[sym[a][2]], v[2]);
    y[a] = y[a] + c1 * (t - pv);
  }
}

struct MfArgs {
  const cplx* vt;       // [K][N]
  const cplx* vu;       // [K][N] or nullptr
  cplx* ypart;          // [nchunk][K][N]
  cplx* ynear;          // [n_near][K][3]
  cplx* y;              // [K][N]
  const uint8_t* kinds; // for the preconditioner blocks (nullable)
  cplx* pinv;           // (n_e,3,3) or nullptr
  const double* diag_base;
  int* flags;
  const int* gate;      // nullable: the application is skipped when *gate == 0
  int K, nchunk, chunk_cols;
  // bit k clear: vt_k (t_mask) / vu_k (u_mask) is known to be zero and its
  // product is skipped (b of an all-Neumann frequency has vt = 0, SEM's
  // columns vu = 0: half the block applies of the K = 5 pass)
  unsigned t_mask, u_mask;
};
#define EWB_MF_GATE \
  if (m.gate && *m.gate == 0) return;

#ifndef EWB_MF_MINB
#define EWB_MF_MINB 3
#endif
#ifndef EWB_MF_QUNROLL
#define EWB_MF_QUNROLL 3
#endif
constexpr int kMfQUnroll = EWB_MF_QUNROLL;
// the accumulator-free K = 1 product needs ~130 registers instead of 168
#ifndef EWB_MF1_MINB
#define EWB_MF1_MINB 4
#endif
// SER = false: no far pair of this application can reach the series branch
// (mf_launch checks |k_s| x the far-pair distance bound, as series_free in
// ewb_assembly.cu); mid pairs always keep the check.
// K >= kMfYsMin: the K x 3 row outputs live in shared memory ([k][a][thread],
// conflict-free 128-bit accesses) instead of 6 K registers per thread: they
// are touched once per PAIR, and beside the 40-word accumulator they made the
// K = 5 pass spill (804 bytes of spill stores in the <5, U> instance).
#ifndef EWB_MF_YS_MIN
#define EWB_MF_YS_MIN 3
#endif
constexpr int kMfYsMin = EWB_MF_YS_MIN;
template <int K, bool USE_U, bool SER>
__global__ void __launch_bounds__(128, (K == 1 && !USE_U) ? EWB_MF1_MINB : EWB_MF_MINB)
    k_mf_farmid(Geo g, Phys<true> ph, MfArgs m) {
  EWB_MF_GATE
  constexpr bool YS = K >= kMfYsMin;
  extern __shared__ __align__(16) unsigned char mf_dyn[];   // YS: K x 3 x 128 complex
  cplx* s_yacc = reinterpret_cast<cplx*>(mf_dyn);
  __shared__ double s_geo[kMfTile][8];        // cx cy cz diam nx ny nz area
  __shared__ double s_y[kMfTile][30];         // 3 far + 7 mid points
  __shared__ cplx s_vt[kMfTile][K][3];
  __shared__ cplx s_vu[USE_U ? kMfTile : 1][K][3];
  const int n = g.n_e;
  const long long N = 3LL * n;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j_begin = blockIdx.y * m.chunk_cols;
  const int j_end = min(n, j_begin + m.chunk_cols);
  const bool row_ok = i < n;
  double xi = 0, yi = 0, zi = 0;
  if (row_ok) { xi = g.cx[i]; yi = g.cy[i]; zi = g.cz[i]; }
  cplx y[YS ? 1 : K][3];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (YS) s_yacc[(k * 3 + a) * 128 + threadIdx.x] = {0.0, 0.0};
      else y[YS ? 0 : k][a] = {0.0, 0.0};
    }
  for (int t0 = j_begin; t0 < j_end; t0 += kMfTile) {
    const int tc = min(kMfTile, j_end - t0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < tc * 38; idx += blockDim.x) {
      int jj = idx / 38, f = idx % 38, j = t0 + jj;
      double v;
      if (f < 8) {
        const double* src[8] = {g.cx, g.cy, g.cz, g.diam, g.nx, g.ny, g.nz, g.area};
        v = src[f][j];
        s_geo[jj][f] = v;
      } else if (f < 17) {
        int q = (f - 8) / 3, c = (f - 8) % 3;
        s_y[jj][f - 8] = g.yfar[(size_t)(3 * q + c) * n + j];
      } else {
        int q = (f - 17) / 3, c = (f - 17) % 3;
        s_y[jj][f - 8] = g.ymid[(size_t)(3 * q + c) * n + j];
      }
    }
    for (int idx = threadIdx.x; idx < tc * K * 3; idx += blockDim.x) {
      int jj = idx / (3 * K), r = idx % (3 * K), k = r / 3, a = r % 3;
      s_vt[jj][k][a] = m.vt[(size_t)k * N + 3 * (t0 + jj) + a];
      if (USE_U) s_vu[jj][k][a] = m.vu[(size_t)k * N + 3 * (t0 + jj) + a];
    }
    __syncthreads();
    if (!row_ok) continue;
    for (int jj = 0; jj < tc; ++jj) {
      const int j = t0 + jj;
      if (j == i) continue;
      const int tier = exact_tier_fast(xi, yi, zi, s_geo[jj][0], s_geo[jj][1], s_geo[jj][2],
                                  s_geo[jj][3]);
      if (tier == 2) continue;
      const double nx = s_geo[jj][4], ny = s_geo[jj][5], nz = s_geo[jj][6], ar = s_geo[jj][7];
      // 1/(4 pi mu) and 1/(4 pi) ride in the weights; series out of line
      const double cu = ar * ph.fc.inv4pimu, ct = ar * ph.fc.inv4pi;
      if constexpr (K == 1 && !USE_U) {
        // GMRES product: each point applied straight to v (no accumulator)
        const cplx v[3] = {s_vt[jj][0][0], s_vt[jj][0][1], s_vt[jj][0][2]};
        cplx nv = nx * v[0];
        axpy(nv, ny, v[1]);
        axpy(nv, nz, v[2]);
        auto point1 = [&](const double* yq, double wq, auto ser) {
          double dx = yq[0] - xi, dy = yq[1] - yi, dz = yq[2] - zi;
          const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
          const double ir = rsqrt(r2);
          const double r = r2 * ir;
          dx *= ir; dy *= ir; dz *= ir;
          const double dn = fma(dz, nz, fma(dy, ny, dx * nx));
          point_apply_T<decltype(ser)::value>(y[0], ph.fc, c_num.far_sw, r, ir, dx, dy, dz, dn,
                                              wq * ir * ir * ct, v, nv, nx, ny, nz);
        };
        if (tier == 0) {
#ifndef EWB_MF_NO_DELTA
          // damping factors of points 1, 2 from point 0's (column-uniform test)
          if (fabs(ph.fc.ks.im) * s_geo[jj][3] <= c_math.delta_max) {
            double r0 = 0, ms0 = 0, mp0 = 0;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const double* yq = &s_y[jj][3 * q];
              double dx = yq[0] - xi, dy = yq[1] - yi, dz = yq[2] - zi;
              const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
              const double ir = rsqrt(r2);
              const double r = r2 * ir;
              dx *= ir; dy *= ir; dz *= ir;
              const double dn = fma(dz, nz, fma(dy, ny, dx * nx));
              double ms, mp;
              if (q == 0) {
                damping_factors<false>(ph.fc, r, 0.0, 0.0, 0.0, ms, mp);
                r0 = r; ms0 = ms; mp0 = mp;
              } else {
                damping_factors<true>(ph.fc, r, r0, ms0, mp0, ms, mp);
              }
              point_apply_T_m<SER>(y[0], ph.fc, c_num.far_sw, r, ir, dx, dy, dz, dn,
                                   g.wfar[q] * ir * ir * ct, v, nv, nx, ny, nz, ms, mp);
            }
            continue;
          }
#endif
#pragma unroll kMfQUnroll
          for (int q = 0; q < 3; ++q)
            point1(&s_y[jj][3 * q], g.wfar[q], std::integral_constant<bool, SER>{});
        } else {
#pragma unroll 1
          for (int q = 0; q < 7; ++q)
            point1(&s_y[jj][9 + 3 * q], g.wmid[q], std::true_type{});
        }
        continue;
      }
      Acc<cplx> acc;
      acc_zero(acc);
      auto point = [&](const double* yq, double wq, auto ser) {
        double dx = yq[0] - xi, dy = yq[1] - yi, dz = yq[2] - zi;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const double ir = rsqrt(r2);
        const double r = r2 * ir;
        dx *= ir; dy *= ir; dz *= ir;
        const double dn = fma(dz, nz, fma(dy, ny, dx * nx));
        const double wi = wq * ir;
        point_dynamic_scaled<decltype(ser)::value>(acc, ph.fc, c_num.far_sw, r, ir, dx, dy, dz, dn,
                                                   wi * cu, wi * ir * ct);
      };
      if (tier == 0) {
#ifndef EWB_MF_NO_DELTA
        if (fabs(ph.fc.ks.im) * s_geo[jj][3] <= c_math.delta_max) {
          double r0 = 0, ms0 = 0, mp0 = 0;
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const double* yq = &s_y[jj][3 * q];
            double dx = yq[0] - xi, dy = yq[1] - yi, dz = yq[2] - zi;
            const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
            const double ir = rsqrt(r2);
            const double r = r2 * ir;
            dx *= ir; dy *= ir; dz *= ir;
            const double dn = fma(dz, nz, fma(dy, ny, dx * nx));
            const double wi = g.wfar[q] * ir;
            double ms, mp;
            if (q == 0) {
              damping_factors<false>(ph.fc, r, 0.0, 0.0, 0.0, ms, mp);
              r0 = r; ms0 = ms; mp0 = mp;
            } else {
              damping_factors<true>(ph.fc, r, r0, ms0, mp0, ms, mp);
            }
            point_dynamic_scaled_m<SER>(acc, ph.fc, c_num.far_sw, r, ir, dx, dy, dz, dn, wi * cu,
                                        wi * ir * ct, ms, mp);
          }
        } else
#endif
        {
#pragma unroll kMfQUnroll
          for (int q = 0; q < 3; ++q)
            point(&s_y[jj][3 * q], g.wfar[q], std::integral_constant<bool, SER>{});
        }
      } else {
#pragma unroll 1
        for (int q = 0; q < 7; ++q) point(&s_y[jj][9 + 3 * q], g.wmid[q], std::true_type{});
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const bool dt = (m.t_mask >> k) & 1u, du = USE_U && ((m.u_mask >> k) & 1u);
        if (YS) {
          if (!dt && !du) continue;
          cplx yk[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double2 v2 = *reinterpret_cast<const double2*>(
                &s_yacc[(k * 3 + a) * 128 + threadIdx.x]);
            yk[a] = {v2.x, v2.y};
          }
          if (dt) acc_apply_T(acc, nx, ny, nz, 1.0, s_vt[jj][k], yk);
          if (du) acc_apply_U(acc, 1.0, s_vu[jj][k], yk);
#pragma unroll
          for (int a = 0; a < 3; ++a)
            *reinterpret_cast<double2*>(&s_yacc[(k * 3 + a) * 128 + threadIdx.x]) =
                make_double2(yk[a].re, yk[a].im);
        } else {
          if (dt) acc_apply_T(acc, nx, ny, nz, 1.0, s_vt[jj][k], y[YS ? 0 : k]);
          if (du) acc_apply_U(acc, 1.0, s_vu[jj][k], y[YS ? 0 : k]);
        }
      }
    }
  }
  if (!row_ok) return;
  cplx* out = m.ypart + (size_t)blockIdx.y * K * N;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a)
      out[(size_t)k * N + 3 * i + a] =
          YS ? s_yacc[(k * 3 + a) * 128 + threadIdx.x] : y[YS ? 0 : k][a];
}

template <int K, bool USE_U>
__global__ void __launch_bounds__(128) k_mf_near(Geo g, Phys<true> ph, MfArgs m, int n_near) {
  EWB_MF_GATE
  const int lane = threadIdx.x & 31;
  const int wp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wp >= n_near) return;
  const int p = g.near_order[wp];   // deepest level first (uniform CTAs)
  const int i = g.near_row[p], j = g.near_j[p], L = g.near_lvl[p];
  EWB_DCHECK(p >= 0 && p < n_near && i >= 0 && i < g.n_e && j >= 0 && j < g.n_e && i != j &&
                 L >= 1 && L <= kMaxNearLevel, 301);
  const long long N = 3LL * g.n_e;
  const double xi = g.cx[i], yi = g.cy[i], zi = g.cz[i];
  const double nx = g.nx[j], ny = g.ny[j], nz = g.nz[j], ar = g.area[j];
  double v[9];
  load_corners(g, j, v);
  const RuleRef rr = g.sub[L];
  const double* bary = g.rules + rr.off;
  const double* wq = bary + 3 * rr.q;
  Acc<cplx> acc;
  acc_zero(acc);
  for (int q = lane; q < rr.q; q += 32) {
    double b0 = bary[3 * q], b1 = bary[3 * q + 1], b2 = bary[3 * q + 2];
    double dx = fma(b2, v[6], fma(b1, v[3], b0 * v[0])) - xi;
    double dy = fma(b2, v[7], fma(b1, v[4], b0 * v[1])) - yi;
    double dz = fma(b2, v[8], fma(b1, v[5], b0 * v[2])) - zi;
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    double ir = rsqrt(r2);  // one MUFU + Newton: replaces sqrt + divide (~1 ulp)
    double r = r2 * ir;
    dx *= ir; dy *= ir; dz *= ir;
    double dn = fma(dz, nz, fma(dy, ny, dx * nx));
    ph.point(acc, r, ir, dx, dy, dz, dn, wq[q] * ar);
  }
  acc_warp_sum(acc);
  if (lane != 0) return;
  for (int k = 0; k < K; ++k) {
    cplx vt[3], yk[3] = {{0, 0}, {0, 0}, {0, 0}};
    if ((m.t_mask >> k) & 1u) {
      for (int a = 0; a < 3; ++a) vt[a] = m.vt[(size_t)k * N + 3 * j + a];
      acc_apply_T(acc, nx, ny, nz, ph.fc.inv4pi, vt, yk);
    }
    if (USE_U && ((m.u_mask >> k) & 1u)) {
      cplx vu[3];
      for (int a = 0; a < 3; ++a) vu[a] = m.vu[(size_t)k * N + 3 * j + a];
      acc_apply_U(acc, ph.fc.inv4pimu, vu, yk);
    }
    for (int a = 0; a < 3; ++a) m.ynear[((size_t)p * K + k) * 3 + a] = yk[a];
  }
}

__device__ bool inv3_mf(const cplx Ain[3][3], cplx Inv[3][3]) {
  cplx M[3][6];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      M[r][c] = Ain[r][c];
      M[r][3 + c] = {r == c ? 1.0 : 0.0, 0.0};
    }
  for (int col = 0; col < 3; ++col) {
    int piv = col;
    double best = fabs(M[col][col].re) + fabs(M[col][col].im);
    for (int r = col + 1; r < 3; ++r) {
      double v = fabs(M[r][col].re) + fabs(M[r][col].im);
      if (v > best) { best = v; piv = r; }
    }
    if (best == 0.0) return false;
    if (piv != col)
      for (int c = 0; c < 6; ++c) { cplx tmp = M[col][c]; M[col][c] = M[piv][c]; M[piv][c] = tmp; }
    cplx inv_p = cdiv(cplx{1.0, 0.0}, M[col][col]);
    for (int c = 0; c < 6; ++c) M[col][c] = M[col][c] * inv_p;
    for (int r = 0; r < 3; ++r) {
      if (r == col) continue;
      cplx f = M[r][col];
      for (int c = 0; c < 6; ++c) M[r][c] = M[r][c] - f * M[col][c];
    }
  }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) Inv[r][c] = M[r][3 + c];
  return true;
}

// Self term + fixed-order final sum:  y_i = sum_chunks + sum_near + D_i v_i.
template <int K, bool USE_U>
__global__ void __launch_bounds__(128) k_mf_self(Geo g, Phys<true> ph, MfArgs m) {
  EWB_MF_GATE
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= g.n_e) return;
  const long long N = 3LL * g.n_e;
  const double xi = g.cx[j], yi = g.cy[j], zi = g.cz[j];
  const double nx = g.nx[j], ny = g.ny[j], nz = g.nz[j];
  Acc<cplx> acc;
  acc_zero(acc);
  const double4* sp = g.self_pts + (size_t)j * kSelfQ;
  for (int q = lane; q < kSelfQ; q += 32) {
    double4 yq = sp[q];
    double dx = yq.x - xi, dy = yq.y - yi, dz = yq.z - zi;
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    double ir = rsqrt(r2);  // one MUFU + Newton: replaces sqrt + divide (~1 ulp)
    double r = r2 * ir;
    dx *= ir; dy *= ir; dz *= ir;
    double dn = fma(dz, nz, fma(dy, ny, dx * nx));
    ph.point(acc, r, ir, dx, dy, dz, dn, yq.w);
  }
  acc_warp_sum(acc);
  // chunk partials: lanes split (k, a, chunk) sums in a fixed order
  cplx part[K][3];
  for (int k = 0; k < K; ++k)
    for (int a = 0; a < 3; ++a) {
      cplx s = {0.0, 0.0};
      for (int c = lane; c < m.nchunk; c += 32) s = s + m.ypart[((size_t)c * K + k) * N + 3 * j + a];
      warp_sum(s);
      part[k][a] = s;
    }
  if (lane != 0) return;
  cplx U[3][3], T[3][3];
  acc_finalize(acc, nx, ny, nz, ph.fc.inv4pimu, ph.fc.inv4pi, U, T);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) T[a][b] = T[a][b] + cplx{m.diag_base[9 * j + 3 * a + b], 0.0};
  bool ok = true;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) ok = ok && finite(U[a][b]) && finite(T[a][b]);
  if (!ok) m.flags[0] = 1;
  for (int k = 0; k < K; ++k) {
    cplx yk[3] = {part[k][0], part[k][1], part[k][2]};
    for (int p = g.near_ptr[j]; p < g.near_ptr[j + 1]; ++p)
      for (int a = 0; a < 3; ++a) yk[a] = yk[a] + m.ynear[((size_t)p * K + k) * 3 + a];
    for (int a = 0; a < 3; ++a) {
      cplx s = {0.0, 0.0};
      for (int b = 0; b < 3; ++b) {
        if ((m.t_mask >> k) & 1u) cfma(s, T[a][b], m.vt[(size_t)k * N + 3 * j + b]);
        if (USE_U && ((m.u_mask >> k) & 1u)) cfma(s, U[a][b], m.vu[(size_t)k * N + 3 * j + b]);
      }
      m.y[(size_t)k * N + 3 * j + a] = yk[a] + s;
    }
  }
  if (m.pinv) {
    cplx Dm[3][3], Inv[3][3];
    for (int c = 0; c < 3; ++c) {
      bool dir = m.kinds && m.kinds[3 * j + c] == kDirichlet;
      for (int a = 0; a < 3; ++a) Dm[a][c] = dir ? -U[a][c] : T[a][c];
    }
    if (!inv3_mf(Dm, Inv)) {
      atomicAdd(m.flags + 1, 1);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Inv[a][b] = {a == b ? 1.0 : 0.0, 0.0};
    }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) m.pinv[9 * j + 3 * a + b] = Inv[a][b];
  }
}

template <int K, bool USE_U>
static cudaError_t mf_launch(Context& c, Phys<true> ph, MfArgs m, cudaStream_t s) {
  const int n = c.n_e;
  dim3 grid((n + 127) / 128, m.nchunk);
  Phys<true> phf = ph;
  phf.fc.sw = kFarSwitch;
  // far pairs: r >= 3 d_j >= 2.9 min d (series_free, ewb_assembly.cu)
  constexpr size_t ys_bytes = K >= kMfYsMin ? sizeof(cplx) * K * 3 * 128 : 0;
  static bool attr = false;
  if (!attr && ys_bytes) {   // static + dynamic shared memory exceeds the 48 KB default
    cudaFuncSetAttribute(k_mf_farmid<K, USE_U, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ys_bytes);
    cudaFuncSetAttribute(k_mf_farmid<K, USE_U, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ys_bytes);
    attr = true;
  }
  if (c.min_diam > 0.0 && ph.fc.ks_abs * (2.9 * c.min_diam) >= kFarSwitch)
    EWB_NOTE k_mf_farmid<K, USE_U, false><<<grid, 128, ys_bytes, s>>>(c.g, phf, m);
  else
    EWB_NOTE k_mf_farmid<K, USE_U, true><<<grid, 128, ys_bytes, s>>>(c.g, phf, m);
  if (c.n_near)
    EWB_NOTE k_mf_near<K, USE_U><<<(c.n_near * 32 + 127) / 128, 128, 0, s>>>(c.g, ph, m, c.n_near);
  EWB_NOTE k_mf_self<K, USE_U><<<(n * 32 + 127) / 128, 128, 0, s>>>(c.g, ph, m);
  return cudaGetLastError();
}

// CTAs the far/mid grid should have, in units of the SM count.  The K = 1
// product runs at 4 CTAs/SM, so the old 148 x 8 CTAs were two waves and a
// 16 %-full third one; measured on the cfg5 application (K = 1 / K = 5, ms,
// A/B in one job): 8 -> 381 / 615, 16 -> 368 / 600, 32 -> 355 / 580,
// 64 -> 349 / 571, 128 -> 348 / 568, 256 -> 346 / 566.
#ifndef EWB_MF_CTAS_PER_SM
#define EWB_MF_CTAS_PER_SM 256
#endif
int mf_chunks(const Context& c) {
  // chunks of >= 256 columns
  int row_blocks = (c.n_e + 127) / 128;
  int want = (148 * EWB_MF_CTAS_PER_SM + row_blocks - 1) / row_blocks;
  int max_chunks = (c.n_e + 255) / 256;
  if (want > max_chunks) want = max_chunks;
  if (want < 1) want = 1;
  if (want > 128) want = 128;
  return want;
}

size_t mf_workspace_bytes(const Context& c, int K) {
  size_t N = 3 * (size_t)c.n_e;
  return sizeof(cplx) * ((size_t)mf_chunks(c) * K * N + (size_t)c.n_near * K * 3 + 16);
}

cudaError_t launch_matfree(Context& c, double ore, double oim, const cplx* vt, const cplx* vu,
                           int K, cplx* y, const uint8_t* kinds, cplx* pinv, void* ws,
                           const int* gate, cudaStream_t s, unsigned t_mask, unsigned u_mask) {
  cudaError_t e = upload_series(s);
  if (e) return e;
  Phys<true> ph{freq_const(c, ore, oim)};
  MfArgs m{};
  m.vt = vt; m.vu = vu; m.y = y; m.kinds = kinds; m.pinv = pinv;
  m.diag_base = c.diag_base; m.flags = c.flags; m.K = K; m.gate = gate;
  m.t_mask = t_mask; m.u_mask = u_mask;
  m.nchunk = mf_chunks(c);
  m.chunk_cols = (c.n_e + m.nchunk - 1) / m.nchunk;
  size_t N = 3 * (size_t)c.n_e;
  m.ypart = (cplx*)ws;
  m.ynear = m.ypart + (size_t)m.nchunk * K * N;
  const bool u = vu != nullptr;
#define EWB_MF(KK)                                              \
  case KK:                                                      \
    return u ? mf_launch<KK, true>(c, ph, m, s) : mf_launch<KK, false>(c, ph, m, s);
  switch (K) {
    EWB_MF(1)
    EWB_MF(2)
    EWB_MF(3)
    EWB_MF(4)
    EWB_MF(5)
    default: return cudaErrorInvalidValue;
  }
#undef EWB_MF
}

// ---------------------------------------------------------------------
// Pair-kernel microbenchmark (BASELINE cfg3): P collocation points x M
// random triangles x F complex frequencies, gauss7 on every pair (no
// ladder), full 3x3 U and T (kernels.py:292-357 via pair_geometry +
// integrated_blocks).  Triangles arrive as corners (M,3,3); normal and
// area follow mesh.py:88-98.
// ---------------------------------------------------------------------
struct TriSoA {
  const double* tri;   // (M, 9)
  long long M;
};

__device__ __forceinline__ void tri_normal_area(const double* v, double& nx, double& ny,
                                                double& nz, double& area) {
  double ax = v[3] - v[0], ay = v[4] - v[1], az = v[5] - v[2];
  double bx = v[6] - v[0], by = v[7] - v[1], bz = v[8] - v[2];
  double cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
  double n2 = sqrt(cx * cx + cy * cy + cz * cz);
  nx = cx / n2; ny = cy / n2; nz = cz / n2;
  area = 0.5 * n2;
}

// full blocks: thread per (point, triangle) for one frequency (blockIdx.y)
__global__ void k_pair_blocks(const double* x, long long P, const double* tri, long long M,
                              const FreqConst* fcs, const double* b7, const double* w7,
                              cplx* u_out, cplx* t_out) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P * M) return;
  const int f = blockIdx.y;
  const long long p = idx / M, m = idx % M;
  const FreqConst fc = fcs[f];
  const double* v = tri + 9 * m;
  double nx, ny, nz, ar;
  tri_normal_area(v, nx, ny, nz, ar);
  const double xi = x[3 * p], yi = x[3 * p + 1], zi = x[3 * p + 2];
  Acc<cplx> acc;
  acc_zero(acc);
  for (int q = 0; q < 7; ++q) {
    double b0 = b7[3 * q], b1 = b7[3 * q + 1], b2 = b7[3 * q + 2];
    double dx = fma(b2, v[6], fma(b1, v[3], b0 * v[0])) - xi;
    double dy = fma(b2, v[7], fma(b1, v[4], b0 * v[1])) - yi;
    double dz = fma(b2, v[8], fma(b1, v[5], b0 * v[2])) - zi;
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    double ir = rsqrt(r2);  // one MUFU + Newton: replaces sqrt + divide (~1 ulp)
    double r = r2 * ir;
    dx *= ir; dy *= ir; dz *= ir;
    double dn = fma(dz, nz, fma(dy, ny, dx * nx));
    point_dynamic(acc, fc, r, ir, dx, dy, dz, dn, w7[q] * ar);
  }
  cplx U[3][3], T[3][3];
  acc_finalize(acc, nx, ny, nz, fc.inv4pimu, fc.inv4pi, U, T);
  size_t base = (((size_t)f * P + p) * M + m) * 9;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      u_out[base + 3 * a + b] = U[a][b];
      t_out[base + 3 * a + b] = T[a][b];
    }
}

// fused reduction: y_U[f][p] = sum_m U(p,m) x_m, y_T likewise.  Thread per
// point, CTA stages 32 triangles (field points, normal, weight*area, x_m)
// in shared memory; blockIdx.y = frequency group, blockIdx.z = triangle chunk.
constexpr int kPkTile = 32;
#ifndef EWB_PK_MINB
#define EWB_PK_MINB 3
#endif
// FC frequencies per thread (blockIdx.y = frequency group): the pair
// geometry of a point (r, 1/r, d, d.n: rsqrt + ~20 FP64 instructions) is
// computed once for the group instead of once per frequency.
template <int FC>
__global__ void __launch_bounds__(128, EWB_PK_MINB) k_pair_reduce(const double* x, long long P,
                                                     const double* tri, long long M,
                                                     const cplx* xv, const FreqConst* fcs, int F,
                                                     const double* b7, const double* w7,
                                                     long long chunk, cplx* part) {
  __shared__ double s_y[kPkTile][21];
  __shared__ double s_n[kPkTile][4];   // nx ny nz area
  __shared__ cplx s_x[kPkTile][3];
  __shared__ FreqConst s_fcs[FC];
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int f0 = blockIdx.y * FC;
  for (int k = threadIdx.x; k < FC * (int)(sizeof(FreqConst) / 8); k += blockDim.x) {
    const int c = k / (int)(sizeof(FreqConst) / 8), w = k % (int)(sizeof(FreqConst) / 8);
    ((double*)&s_fcs[c])[w] = ((const double*)(fcs + min(f0 + c, F - 1)))[w];
  }
  __syncthreads();
  const long long m0 = (long long)blockIdx.z * chunk, m1 = min(M, m0 + chunk);
  const bool ok = p < P;
  const double xi = ok ? x[3 * p] : 0.0, yi = ok ? x[3 * p + 1] : 0.0, zi = ok ? x[3 * p + 2] : 0.0;
  cplx yu[FC][3], yt[FC][3];
#pragma unroll
  for (int c = 0; c < FC; ++c)
#pragma unroll
    for (int a = 0; a < 3; ++a) { yu[c][a] = {0.0, 0.0}; yt[c][a] = {0.0, 0.0}; }
  double w7r[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) w7r[q] = w7[q];
  for (long long t0 = m0; t0 < m1; t0 += kPkTile) {
    const int tc = (int)min((long long)kPkTile, m1 - t0);
    __syncthreads();
    for (int jj = threadIdx.x; jj < tc; jj += blockDim.x) {
      const double* v = tri + 9 * (t0 + jj);
      double vv[9];
      for (int k = 0; k < 9; ++k) vv[k] = v[k];
      double nx, ny, nz, ar;
      tri_normal_area(vv, nx, ny, nz, ar);
      s_n[jj][0] = nx; s_n[jj][1] = ny; s_n[jj][2] = nz; s_n[jj][3] = ar;
      for (int q = 0; q < 7; ++q)
        for (int c = 0; c < 3; ++c)
          s_y[jj][3 * q + c] = fma(b7[3 * q + 2], vv[6 + c], fma(b7[3 * q + 1], vv[3 + c], b7[3 * q] * vv[c]));
      for (int c = 0; c < 3; ++c) s_x[jj][c] = xv[3 * (t0 + jj) + c];
    }
    __syncthreads();
    if (!ok) continue;
    for (int jj = 0; jj < tc; ++jj) {
      const double nx = s_n[jj][0], ny = s_n[jj][1], nz = s_n[jj][2], ar = s_n[jj][3];
      // points applied straight to x_m (no 20-word accumulator); 1/(4 pi mu),
      // 1/(4 pi) folded into the weights; per-frequency constants read from
      // shared memory where used (not held in registers)
      // (material constants: the same in every member of the group)
      const double cu = ar * s_fcs[0].inv4pimu, ct = ar * s_fcs[0].inv4pi;
      const cplx v[3] = {s_x[jj][0], s_x[jj][1], s_x[jj][2]};
      cplx nv = nx * v[0];
      axpy(nv, ny, v[1]);
      axpy(nv, nz, v[2]);
#pragma unroll 1
      for (int q = 0; q < 7; ++q) {
        double dx = s_y[jj][3 * q] - xi, dy = s_y[jj][3 * q + 1] - yi, dz = s_y[jj][3 * q + 2] - zi;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const double ir = rsqrt(r2);
        const double r = r2 * ir;
        dx *= ir; dy *= ir; dz *= ir;
        const double dn = fma(dz, nz, fma(dy, ny, dx * nx));
        const double wi = w7r[q] * ir;
        const double wu = wi * cu, wt = wi * ir * ct;
#pragma unroll
        for (int c = 0; c < FC; ++c) {
          const FreqConst& sf = s_fcs[c];
          FreqConst fc;
          fc.ks = lds_c(&sf.ks); fc.kp = lds_c(&sf.kp);
          fc.tas = lds_c(&sf.tas); fc.tbs = lds_c(&sf.tbs);
          fc.tap = lds_c(&sf.tap); fc.tbp = lds_c(&sf.tbp);
          fc.g2 = lds_c(&sf.g2); fc.ks_abs = lds_d(&sf.ks_abs);
          fc.ratio = lds_d(&sf.ratio);
          point_apply_UT(yu[c], yt[c], fc, lds_d(&sf.sw), r, ir, dx, dy, dz, dn, wu, wt, v, nv,
                         nx, ny, nz);
        }
      }
    }
  }
  if (!ok) return;
#pragma unroll
  for (int c = 0; c < FC; ++c) {
    if (f0 + c >= F) break;
    cplx* o = part + (((size_t)blockIdx.z * F + f0 + c) * P + p) * 6;
    for (int a = 0; a < 3; ++a) { o[a] = yu[c][a]; o[3 + a] = yt[c][a]; }
  }
}

__global__ void k_pair_reduce_final(const cplx* part, int nchunk, int F, long long P, cplx* yu,
                                    cplx* yt) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)F * P * 6) return;
  cplx s = {0.0, 0.0};
  for (int c = 0; c < nchunk; ++c) s = s + part[(size_t)c * F * P * 6 + idx];
  long long fp = idx / 6;
  int a = (int)(idx % 6);
  if (a < 3) yu[fp * 3 + a] = s;
  else yt[fp * 3 + a - 3] = s;
}

cudaError_t launch_pair_blocks(const double* x, long long P, const double* tri, long long M,
                               const FreqConst* fcs_dev, int F, const double* b7, const double* w7,
                               cplx* u, cplx* t, cudaStream_t s) {
  cudaError_t e = upload_series(s);
  if (e) return e;
  dim3 grid((unsigned)((P * M + 127) / 128), F);
  EWB_NOTE k_pair_blocks<<<grid, 128, 0, s>>>(x, P, tri, M, fcs_dev, b7, w7, u, t);
  return cudaGetLastError();
}

cudaError_t launch_pair_reduce(const double* x, long long P, const double* tri, long long M,
                               const cplx* xv, const FreqConst* fcs_dev, int F, const double* b7,
                               const double* w7, cplx* yu, cplx* yt, cplx* part, int nchunk,
                               cudaStream_t s) {
  cudaError_t e = upload_series(s);
  if (e) return e;
  long long chunk = (M + nchunk - 1) / nchunk;
  // frequencies per thread: 2 shares the pair geometry but measured 2.5 %
  // slower on cfg3 (7.41e9 vs 7.60e9 pair-evals/s: 96 bytes of spills and
  // two interleaved phase evaluations at 168 registers), so 1
#ifndef EWB_PK_FC
#define EWB_PK_FC 1
#endif
  constexpr int kFc = EWB_PK_FC;
  dim3 grid((unsigned)((P + 127) / 128), (unsigned)((F + kFc - 1) / kFc), nchunk);
  EWB_NOTE k_pair_reduce<kFc><<<grid, 128, 0, s>>>(x, P, tri, M, xv, fcs_dev, F, b7, w7, chunk,
                                                   part);
  long long tot = (long long)F * P * 6;
  EWB_NOTE k_pair_reduce_final<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(part, nchunk, F, P, yu, yt);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------
// FP64 peak probe: 8 independent DFMA chains per thread (the roofline
// denominator MEASURED_PEAKS.json lacks).
// ---------------------------------------------------------------------
__global__ void k_dfma_probe(long long iters, double* sink) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999999, c = 1e-12;
  for (long long k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) sink[0] = s;
}

cudaError_t fp64_peak_probe(long long iters, int blocks_per_sm, double* tflops, double* ms,
                            cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&sink, 8, s);
  if (e) return e;
  const int threads = 256;
  const int blocks = sms * blocks_per_sm;
  EWB_NOTE k_dfma_probe<<<blocks, threads, 0, s>>>(iters / 8 + 1, sink);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  EWB_NOTE k_dfma_probe<<<blocks, threads, 0, s>>>(iters, sink);
  cudaEventRecord(e1, s);
  e = cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, s);
  if (e) return e;
  double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  *ms = t;
  *tflops = flops / (t * 1e-3) / 1e12;
  return cudaGetLastError();
}

}  // namespace ewb
