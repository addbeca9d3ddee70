// Throughput of the pass-1 epilogue instruction mix without TMEM or barriers:
// per 32-value block FMNMX3 tree + 32 x (FFMA, MUFU.EX2, FADD) + Kahan step.
// Reports ex2 per SM-cycle for W warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/epi_rate tools/epi_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void k(int iters, float* out, long long* cyc) {
  float w[32];
  const int tid = threadIdx.x;
#pragma unroll
  for (int e = 0; e < 32; ++e) w[e] = 0.001f * (float)((tid * 37 + e * 11) & 63);
  float sx = 0.0f, sxc = 0.0f, m1 = 1e30f, inv = 1.0f + 1e-7f * tid, nr = -0.5f;
  __syncthreads();
  const long long c0 = clock64();
  for (int r = 0; r < iters; ++r) {
    if (MODE >= 1) {
      float t11[11];
#pragma unroll
      for (int e = 0; e < 10; ++e) t11[e] = fminf(w[3 * e], fminf(w[3 * e + 1], w[3 * e + 2]));
      t11[10] = fminf(w[30], w[31]);
      const float mb = fminf(fminf(fminf(t11[0], fminf(t11[1], t11[2])), fminf(t11[3], fminf(t11[4], t11[5]))),
                             fminf(fminf(t11[6], fminf(t11[7], t11[8])), fminf(t11[9], t11[10])));
      m1 = fminf(m1, mb * inv);
    }
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 32; ++e) s4[e & 3] += ex2a(-fmaf(w[e], inv, nr));
    const float y = ((s4[0] + s4[1]) + (s4[2] + s4[3])) - sxc;
    const float t = sx + y;
    sxc = (t - sx) - y;
    sx = t;
    if (MODE >= 2) {
#pragma unroll
      for (int e = 0; e < 32; ++e) w[e] = __int_as_float(__float_as_int(w[e]) ^ (r & 1));
    }
  }
  const long long c1 = clock64();
  out[blockIdx.x * blockDim.x + tid] = sx + m1;
  if (tid == 0) cyc[blockIdx.x] = c1 - c0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16, 24, 32}) {
      if (mode == 0) k<0><<<148, warps * 32>>>(iters, out, cyc);
      if (mode == 1) k<1><<<148, warps * 32>>>(iters, out, cyc);
      if (mode == 2) k<2><<<148, warps * 32>>>(iters, out, cyc);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      printf("mode %d warps %2d: %.2f ex2/clk/SM\n", mode, warps, (double)iters * 32 * warps * 32 / c);
    }
  return 0;
}
