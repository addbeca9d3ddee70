// Build the pass-1 epilogue up step by step (no MMA) to see which ingredient
// costs the time: 16 warps, 1 CTA/SM, 32-column blocks.
//   bit 0: FMNMX3 block min      bit 1: tcgen05.ld of the block (else registers)
//   bit 2: named barrier per slot (4 warps) per block
//   bit 3: mbarrier test (completed phase) per block
//   bit 4: Kahan fp32 accumulation + rare-path compare
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc -o tools/epi_build tools/epi_build.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int blocks, float* out, long long* cyc) {
  __shared__ unsigned tbase;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, s = warp >> 2, q = warp & 3;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_arrive(&bar);  // phase 0 complete
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(s * 128);
  const unsigned ba = (unsigned)__cvta_generic_to_shared(&bar);
  float sx = 0.f, sxc = 0.f, m1 = 1e30f, inv = 1.0f + 1e-7f * tid, nr = -1000.5f, acc = 0.f;
  const long long c0 = clock64();
  for (int kb = 0; kb < blocks; ++kb) {
    if (MODE & 8) {
      while (!mbar_test_addr(ba, 0u)) {
      }
    }
    uint32_t r[32];
    if (MODE & 2) {
      tmem_ld32_nowait(t + (unsigned)((kb & 3) * 32), r);
      tmem_ld_wait();
      tmem_regs_ready(r);
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(1000.0f + (float)((lane * 7 + e * 13 + kb) & 63));
    }
    if (MODE & 4) asm volatile("bar.sync %0, 128;" ::"r"(1 + s) : "memory");
    float w[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) w[e] = fminf(fabsf(__uint_as_float(r[e])), 2000.0f);
    float mb = 0.f;
    if (MODE & 1) {
      float t11[11];
#pragma unroll
      for (int e = 0; e < 10; ++e) t11[e] = fminf(w[3 * e], fminf(w[3 * e + 1], w[3 * e + 2]));
      t11[10] = fminf(w[30], w[31]);
      mb = fminf(fminf(fminf(t11[0], fminf(t11[1], t11[2])), fminf(t11[3], fminf(t11[4], t11[5]))),
                 fminf(fminf(t11[6], fminf(t11[7], t11[8])), fminf(t11[9], t11[10])));
    }
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 32; ++e) s4[e & 3] += ex2a(-fmaf(w[e], inv, nr));
    const float bs = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    if (MODE & 16) {
      if (mb * inv < m1) m1 = mb * inv;
      const float y = bs - sxc, tt = sx + y;
      sxc = (tt - sx) - y;
      sx = tt;
    } else {
      acc += bs + mb;
    }
  }
  const long long c1 = clock64();
  out[blockIdx.x * 512 + tid] = sx + acc + m1;
  if (tid == 0) cyc[blockIdx.x] = c1 - c0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int M>
void run(float* out, long long* cyc) {
  const int blocks = 2000;
  k<M><<<148, 512>>>(blocks, out, cyc);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("mode %d error\n", M); return; }
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("mode %2d: %.2f ex2/clk/SM, %.0f cycles per block-round\n", M, (double)blocks * 32 * 512 / c,
         (double)c / blocks);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  run<0>(out, cyc);
  run<1>(out, cyc);
  run<2>(out, cyc);
  run<3>(out, cyc);
  run<7>(out, cyc);
  run<15>(out, cyc);
  run<31>(out, cyc);
  run<19>(out, cyc);
  run<4>(out, cyc);
  run<8>(out, cyc);
  return 0;
}
