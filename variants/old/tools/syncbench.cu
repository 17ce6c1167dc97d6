// Grid-barrier cost probe: cooperative kernel doing `iters` grid.sync()s, with
// and without a trivial global write/read between them.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -cudart static \
//      -o tools/libsyncbench.so tools/syncbench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, double* buf, int mode) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (mode == 1 && threadIdx.x == 0) buf[blockIdx.x] = i;
    g.sync();
    if (mode == 1 && threadIdx.x == 0) acc += buf[(blockIdx.x + 1) % gridDim.x];
  }
  if (acc == -1) buf[0] = acc;
}

// hand-rolled barrier: one arrival per CTA (red.release.gpu), spin on a
// generation counter (ld.acquire.gpu)
__device__ __forceinline__ void my_barrier(unsigned* count, volatile unsigned* gen, unsigned nb,
                                           unsigned& local_gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g0 = local_gen;
    unsigned prev;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(count) : "memory");
    if (prev == nb - 1) {
      *count = 0;
      __threadfence();
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
      } while (cur == g0);
    }
  }
  local_gen++;
  __syncthreads();
}

__global__ void k_mybar(int iters, unsigned* ctr, double* buf) {
  unsigned lg = 0;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) buf[blockIdx.x] = i;
    my_barrier(ctr, ctr + 1, gridDim.x, lg);
    if (threadIdx.x == 0) acc += buf[(blockIdx.x + 1) % gridDim.x];
  }
  if (acc == -1) buf[0] = acc;
}

extern "C" int sync_probe(int threads, int blocks, int iters, float* out_us) {
  double* buf;
  unsigned* ctr;
  cudaMalloc(&buf, 8 * 4096);
  cudaMalloc(&ctr, 64);
  cudaMemset(ctr, 0, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    void* args_c[] = {&iters, &buf, &mode};
    void* args_m[] = {&iters, &ctr, &buf};
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      cudaError_t e;
      if (mode < 2)
        e = cudaLaunchCooperativeKernel((void*)k_sync, blocks, threads, args_c, 0, 0);
      else
        e = cudaLaunchCooperativeKernel((void*)k_mybar, blocks, threads, args_m, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      out_us[mode] = ms * 1000.f / iters;
    }
  }
  cudaFree(buf);
  cudaFree(ctr);
  return 0;
}
