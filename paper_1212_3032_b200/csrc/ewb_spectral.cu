// Time reconstruction (transform.py:137-203): conjugate fill of the solved
// half spectrum, frequency-domain window, inverse DFT (x N), imaginary
// residue check, and the e^{+eta n dt} rescale — fused, for every DOF at
// once (the reference does it per probe with pocketfft).
//
// One block per DOF column; thread n produces time sample n as a direct
// DFT sum over the N frequency bins with twiddles from a host-exact table
// in shared memory (N <= 4096; the sweeps use N = 64..256).
#include <cuda_runtime.h>

#include "ewb_common.cuh"

namespace ewb {
EWB_DEBUG_TU(spectral)

__global__ void k_window_idft(const cplx* half, long long n_half, long long D, const double* win,
                              const cplx* tw, double eta_dt, double* out, double* residue) {
  extern __shared__ unsigned char smem[];
  const int N = (int)(2 * (n_half - 1));
  cplx* s_tw = reinterpret_cast<cplx*>(smem);
  cplx* s_v = s_tw + N;
  double* s_red = reinterpret_cast<double*>(s_v + N);
  const long long d = blockIdx.x;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    s_tw[k] = tw[k];
    cplx v;
    if (k < n_half) v = half[(size_t)k * D + d];
    else v = conj(half[(size_t)(N - k) * D + d]);        // conj of the mirror bin
    if (k == 0 || k == n_half - 1) v.im = 0.0;             // real DC / Nyquist
    s_v[k] = {v.re * win[k], v.im * win[k]};
  }
  __syncthreads();
  double max_abs = 0.0, max_im = 0.0;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    cplx s = {0.0, 0.0};
    int idx = 0;
    for (int k = 0; k < N; ++k) {
      cfma(s, s_v[k], s_tw[idx]);
      idx += n;
      if (idx >= N) idx -= N;
    }
    out[(size_t)n * D + d] = s.re * exp(eta_dt * n);
    max_abs = fmax(max_abs, hypot(s.re, s.im));
    max_im = fmax(max_im, fabs(s.im));
  }
  // block max-reduce
  for (int o = 16; o > 0; o >>= 1) {
    max_abs = fmax(max_abs, __shfl_down_sync(0xffffffffu, max_abs, o));
    max_im = fmax(max_im, __shfl_down_sync(0xffffffffu, max_im, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { s_red[2 * wid] = max_abs; s_red[2 * wid + 1] = max_im; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a = fmax(a, s_red[2 * w]); m = fmax(m, s_red[2 * w + 1]); }
    residue[d] = a > 0.0 ? m / a : 0.0;
  }
}

cudaError_t launch_window_idft(const cplx* half, long long n_half, long long D, const double* win,
                               const cplx* tw, double eta_dt, double* out, double* residue,
                               cudaStream_t s) {
  const int N = (int)(2 * (n_half - 1));
  int threads = N < 256 ? ((N + 31) / 32) * 32 : 256;
  size_t smem = (size_t)2 * N * sizeof(cplx) + 2 * 8 * sizeof(double) * 8;
  EWB_NOTE k_window_idft<<<(unsigned)D, threads, smem, s>>>(half, n_half, D, win, tw, eta_dt, out, residue);
  return cudaGetLastError();
}

}  // namespace ewb

namespace ewb {
// device sin/cos/exp of the kernel phases (ewb_common.cuh) on host arguments:
// the accuracy test of fast_sincos / fast_exp against libm (ewb_math_selftest)
__global__ void k_math_selftest(const double* x, long long n, double* s, double* c, double* e) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  fast_sincos(x[i], s + i, c + i);
  e[i] = fast_exp(x[i]);
}

// exp_small (the damping-factor update between the quadrature points of a
// far pair) on host arguments |t| <= 2^-4
__global__ void k_math_selftest_delta(const double* t, long long n, double* e) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) e[i] = exp_small(t[i]);
}

cudaError_t launch_math_selftest_delta(const double* t, long long n, double* e, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  EWB_NOTE k_math_selftest_delta<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(t, n, e);
  return cudaGetLastError();
}

cudaError_t launch_math_selftest(const double* x, long long n, double* s, double* c, double* e,
                                 cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  EWB_NOTE k_math_selftest<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, n, s, c, e);
  return cudaGetLastError();
}
}  // namespace ewb
