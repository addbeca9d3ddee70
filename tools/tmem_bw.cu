// TMEM read-bandwidth probe: W warps per CTA (one CTA per SM, all 512
// columns) repeatedly load 32 lanes x C columns (tcgen05.ld.32x32b.xC) and
// fold the values; reports bytes per SM-cycle.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

template <int WAITEVERY>
__global__ void __launch_bounds__(512, 1) probe(int iters, long long* out, float* sink) {
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase + ((unsigned)(32 * (warp & 3)) << 16);
  float acc = 0.0f;
  __syncthreads();
  const long long c0 = clock64();
  for (int r = 0; r < iters; ++r) {
    uint32_t a[32], b[32];
    const unsigned col = (unsigned)((r * 64 + warp * 32) & 511);
    tmem_ld32_nowait(t + col, a);
    if (WAITEVERY == 1) {
      tmem_ld_wait();
      tmem_regs_ready(a);
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += __uint_as_float(a[e]);
    } else {
      tmem_ld32_nowait(t + ((col + 32) & 511), b);
      tmem_ld_wait();
      tmem_regs_ready(a);
      tmem_regs_ready(b);
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += __uint_as_float(a[e]) + __uint_as_float(b[e]);
    }
  }
  __syncthreads();
  const long long c1 = clock64();
  if (tid == 0) out[blockIdx.x] = c1 - c0;
  sink[blockIdx.x * 512 + tid] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 512 * sizeof(float));
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int mode = 1; mode <= 2; ++mode) {
      if (mode == 1) probe<1><<<148, warps * 32>>>(iters, d, sink);
      else probe<2><<<148, warps * 32>>>(iters, d, sink);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
      long long v;
      cudaMemcpy(&v, d, sizeof(v), cudaMemcpyDeviceToHost);
      const double bytes = (double)iters * warps * 32 * 32 * 4 * mode;
      printf("warps=%2d loads/wait=%d: %.1f B/cycle/SM (%.2f fp32/cycle)\n", warps, mode, bytes / v, bytes / v / 4);
    }
  }
  return 0;
}
