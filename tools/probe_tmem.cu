// TMEM store/load throughput per SM: W warps per CTA, C CTAs per SM, each warp
// looping tcgen05.st.32x32b.x32 (and/or .ld) over its lane quarter, with or
// without a wait per iteration.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc -o tools/probe_tmem tools/probe_tmem.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

template <int MODE>  // 0: st + wait each; 1: st, wait every 4; 2: ld + wait each; 3: st+ld alternate
__global__ void __launch_bounds__(256, 2) tp(int iters, long long* out) {
  __shared__ unsigned tbase;
  const int warp = threadIdx.x >> 5, q = warp & 3;
  if (warp == 0) tmem_alloc(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(warp >> 2) * 64;
  uint32_t r[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) r[e] = threadIdx.x * 32 + e;
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      tmem_st32(t + (it & 1) * 32, r);
      tmem_st_wait();
    } else if (MODE == 1) {
      tmem_st32(t + (it & 1) * 32, r);
      if ((it & 3) == 3) tmem_st_wait();
    } else if (MODE == 2) {
      tmem_ld32_nowait(t + (it & 1) * 32, r);
      tmem_ld_wait();
      tmem_regs_ready(r);
    } else {
      tmem_ld32_nowait(t + (it & 1) * 32, r);
      tmem_ld_wait();
      tmem_regs_ready(r);
#pragma unroll
      for (int e = 0; e < 32; ++e) r[e] += 1;
      tmem_st32(t + 32 - (it & 1) * 32, r);
      tmem_st_wait();
    }
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
  if (r[threadIdx.x & 31] == 0xdeadbeef) out[0] = 0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

template <int MODE>
void run(long long* d, int sms, int ctas) {
  const int iters = 2000;
  tp<MODE><<<sms * ctas, 256>>>(100, d);
  tp<MODE><<<sms * ctas, 256>>>(iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("error\n");
    return;
  }
  long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = 8.0 * ctas * 32 * 32 * 4 * iters;  // 8 warps/CTA x 4 KB per op per SM
  printf("mode %d (%s), %d CTA/SM: %.1f cycles/op/warp, %.0f B/cycle/SM\n", MODE,
         MODE == 0 ? "st+wait" : MODE == 1 ? "st, wait/4" : MODE == 2 ? "ld+wait" : "ld+st",
         ctas, (double)h / iters, bytes * (MODE == 3 ? 2 : 1) / h);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 4096 * sizeof(long long));
  for (int c : {1, 2}) {
    run<0>(d, sms, c);
    run<1>(d, sms, c);
    run<2>(d, sms, c);
    run<3>(d, sms, c);
  }
  return 0;
}
