// Accuracy + throughput probe of the exponential building blocks on the B200:
//   * ex2.approx.ftz.f32 relative error (mean = bias, max) against fp64 exp2
//   * conversion fp64 -> fp32 by integer ops (truncating) vs F2F (RN)
//   * issue rates of MUFU.EX2, F2F.F32.F64, DFMA alone and mixed
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ex2_check tools/ex2_check.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void acc_kernel(double lo, double hi, int n, int mode, double* out) {
  __shared__ double s_sum[256], s_max[256];
  double sum = 0, mx = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d = lo + (hi - lo) * ((double)i + 0.5) / n;  // exact fp64 argument
    float f;
    if (mode == 0) {
      f = (float)d;  // RN conversion
    } else {          // integer truncating conversion + debias (as pgx_grid.cuh)
      const unsigned u = __funnelshift_l(__double2loint(d), __double2hiint(d) - 0x38000000, 3);
      const float a = __uint_as_float(u);  // |d|
      f = -fmaf(a, 5.9604645e-8f, a);
      if (mode == 2) f = -a;  // without the debias
    }
    const double got = (double)ex2a(f);
    const double ref = exp2(d);
    const double rel = (got - ref) / ref;
    sum += rel;
    mx = fmax(mx, fabs(rel));
  }
  s_sum[threadIdx.x] = sum;
  s_max[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, m = 0;
    for (int t = 0; t < 256; ++t) a += s_sum[t], m = fmax(m, s_max[t]);
    atomicAdd(out, a);
    unsigned long long* mp = (unsigned long long*)(out + 1);
    atomicMax(mp, __double_as_longlong(m));
  }
}

template <int MODE>
__global__ void rate_kernel(float* out, int iters) {
  float a = threadIdx.x * 1e-3f - 3.0f, b = a - 1.0f, c = a - 2.0f, d = a - 0.5f;
  double da = a, db = b, dc = c, dd = d;
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0 || MODE == 3) {  // MUFU.EX2
      a = ex2a(a) - 3.0f; b = ex2a(b) - 3.0f; c = ex2a(c) - 3.0f; d = ex2a(d) - 3.0f;
    }
    if (MODE == 1 || MODE == 3) {  // F2F.F32.F64
      a += (float)da; b += (float)db; c += (float)dc; d += (float)dd;
      da += 1e-9; db += 1e-9; dc += 1e-9; dd += 1e-9;
    }
    if (MODE == 2) {  // DFMA
      da = fma(da, 0.999, 1e-3); db = fma(db, 0.999, 1e-3); dc = fma(dc, 0.999, 1e-3);
      dd = fma(dd, 0.999, 1e-3);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + (float)(da + db + dc + dd);
}

int main() {
  double* d_out;
  cudaMalloc(&d_out, 16);
  const char* names[3] = {"F2F(RN)", "int-trunc+debias", "int-trunc"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int r = 0; r < 3; ++r) {
      const double ranges[3][2] = {{-1.0, -0.0}, {-8.0, -1.0}, {-40.0, -8.0}};
      if (mode > 0 && r == 0) continue;  // int conversion needs |d| >= 1 in this probe
      cudaMemset(d_out, 0, 16);
      const int n = 1 << 26;
      acc_kernel<<<1024, 256>>>(ranges[r][0], ranges[r][1], n, mode, d_out);
      double h[2];
      cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
      printf("ex2 %-18s d in [%6.1f,%5.1f]: mean rel err %+.3e  max %.3e\n", names[mode],
             ranges[r][0], ranges[r][1], h[0] / n, h[1]);
    }
  }
  float* buf;
  cudaMalloc(&buf, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  const char* rn[4] = {"MUFU.EX2", "F2F.F32.F64", "DFMA", "EX2+F2F"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) rate_kernel<0><<<148 * 8, 256>>>(buf, iters);
      if (m == 1) rate_kernel<1><<<148 * 8, 256>>>(buf, iters);
      if (m == 2) rate_kernel<2><<<148 * 8, 256>>>(buf, iters);
      if (m == 3) rate_kernel<3><<<148 * 8, 256>>>(buf, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 148.0 * 8 * 256 * iters * 4;
      if (rep) printf("rate %-12s %.3f ms -> %.1f Gop/s (%.2f /clk/SM at 1.965 GHz)\n", rn[m], ms,
                      ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
