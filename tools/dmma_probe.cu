// FP64 pipes on sm_100a: DFMA-only, DMMA-only (mma.sync m8n8k4 f64) and
// both interleaved in one warp, to learn whether DMMA is a separate pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_probe.cu -o tools/dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void probe(double* out, int iters) {
  double x[8], acc[4][2];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
  const double a = 1.0000001, b = 0.9999999;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    if (MODE != 0) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) dmma(acc[k], a + k, b);
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    for (int mode = 0; mode < 3; ++mode) {
      auto k = mode == 0 ? probe<0> : mode == 1 ? probe<1> : probe<2>;
      dim3 grid(sms * 2);
      k<<<grid, threads>>>(out, 10);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<grid, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // per thread per iteration: DFMA 32 x 2 flop; DMMA per warp 8 x (8x8x4 x 2) flop
      double warps = (double)grid.x * threads / 32;
      double f_fma = mode != 1 ? (double)grid.x * threads * iters * 32 * 2 : 0;
      double f_mma = mode != 0 ? warps * iters * 8 * 512.0 : 0;
      printf("threads %4d mode %s: %.3f ms  DFMA %.2f TF  DMMA %.2f TF  total %.2f TF\n", threads,
             mode == 0 ? "dfma" : mode == 1 ? "dmma" : "both", ms, f_fma / ms / 1e9,
             f_mma / ms / 1e9, (f_fma + f_mma) / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
