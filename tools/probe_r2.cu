// Round-2 probes (B200):
//  (1) tcgen05.mma kind::f16 throughput per SM when C CTAs per SM issue
//      concurrently (M=128, K=16; SS or TS; N = 32..256);
//  (2) epilogue exponential mix per SM (16 warps): scalar FFMA+MUFU+FADD,
//      packed FFMA2/FADD2, and a fraction of the exponentials on the FMA pipe
//      (degree-5 polynomial exp2, Cody-Waite split by the 1.5*2^23 shifter).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc \
//      -o tools/probe_r2 tools/probe_r2.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

template <int N, bool TS, int C>
__global__ void __launch_bounds__(128, C) umma_probe(int iters, long long* out) {
  __shared__ __align__(1024) unsigned char sm[2 * 4096 + 2 * 8192];
  __shared__ uint64_t mbar;
  __shared__ unsigned tbase;
  constexpr unsigned kCols = 512 / C;
  constexpr int NACC = (kCols - 64) / N >= 4 ? 4 : ((kCols - 64) / N >= 2 ? 2 : 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (int)sizeof(sm) / 4; e += 128) reinterpret_cast<unsigned*>(sm)[e] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, kCols);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  constexpr uint32_t idesc = umma_idesc_f16(128, N);
  if (warp == 0) {
    const uint64_t da = umma_desc(sb), db = umma_desc(sb + 2 * 4096);
    long long c0 = clock64();
    for (int r = 0; r < iters; ++r) {
      if (tid == 0) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const unsigned d = t + 64 + (unsigned)((u % NACC) * N);
          if (TS)
            umma_f16_ts(d, t + 16 * (u & 3), db + (uint64_t)((u & 1) * 8192 >> 4), idesc, r > 0 || u >= NACC);
          else
            umma_f16_ss(d, da + (uint64_t)((u & 1) * 4096 >> 4), db + (uint64_t)((u & 1) * 8192 >> 4), idesc,
                        r > 0 || u >= NACC);
        }
      }
      __syncwarp();
    }
    if (tid == 0) umma_commit(&mbar);
    __syncwarp();
    mbar_wait(&mbar, 0);
    if (tid == 0) out[blockIdx.x] = clock64() - c0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, kCols);
}

template <int N, bool TS, int C>
void run_umma(long long* d, int sms) {
  const int iters = 400;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  umma_probe<N, TS, C><<<sms * C, 128>>>(20, d);
  cudaEventRecord(a);
  umma_probe<N, TS, C><<<sms * C, 128>>>(iters, d);
  cudaEventRecord(b);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("umma N=%d TS=%d C=%d: error %s\n", N, TS, C, cudaGetErrorString(cudaGetLastError()));
    return;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long h[1024];
  cudaMemcpy(h, d, sizeof(long long) * sms * C, cudaMemcpyDeviceToHost);
  double mx = 0, avg = 0;
  for (int i = 0; i < sms * C; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    avg += h[i];
  }
  avg /= sms * C;
  const double per_cta = avg / (16.0 * iters);
  // SM-wide: C CTAs each issued 16*iters MMAs in ~max cycles
  printf("umma %s N=%3d CTAs/SM=%d: %6.1f cycles/MMA per CTA, %6.1f cycles/MMA per SM (%.3f ms wall, %.0f TF/s)\n",
         TS ? "TS" : "SS", N, C, per_cta, mx / (16.0 * iters * C), ms,
         2.0 * 128 * N * 16 * 16.0 * iters * sms * C / (ms * 1e-3) / 1e12);
}

// ---------------------------------------------------------------- epilogue mix
__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ void upk(unsigned long long v, float& lo, float& hi) {
  lo = __uint_as_float((unsigned)v);
  hi = __uint_as_float((unsigned)(v >> 32));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// 2^x for a pair, x >= -125 clamped: x = n + f, f in [-0.5, 0.5], p(f) degree 5
__device__ __forceinline__ unsigned long long pexp2(unsigned long long x2) {
  float x0, x1;
  upk(x2, x0, x1);
  x0 = fmaxf(x0, -125.0f);
  x1 = fmaxf(x1, -125.0f);
  x2 = pk(x0, x1);
  const unsigned long long SH = pk(12582912.0f, 12582912.0f), NSH = pk(-12582912.0f, -12582912.0f);
  const unsigned long long t = fadd2(x2, SH);
  const unsigned long long j = fadd2(t, NSH);
  const unsigned long long NEG1 = pk(-1.0f, -1.0f);
  const unsigned long long f = ffma2(j, NEG1, x2);
  // minimax-ish coefficients of 2^f on [-0.5, 0.5]
  unsigned long long p = pk(1.327647129073739e-3f, 1.327647129073739e-3f);
  p = ffma2(p, f, pk(9.675541892647743e-3f, 9.675541892647743e-3f));
  p = ffma2(p, f, pk(5.550713092088699e-2f, 5.550713092088699e-2f));
  p = ffma2(p, f, pk(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = ffma2(p, f, pk(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = ffma2(p, f, pk(1.0000001192092896f, 1.0000001192092896f));
  const unsigned tl = (unsigned)t, th = (unsigned)(t >> 32);
  const unsigned pl = (unsigned)p, ph = (unsigned)(p >> 32);
  unsigned rl, rh;
  rl = pl + (tl << 23);
  rh = ph + (th << 23);
  return ((unsigned long long)rh << 32) | rl;
}

// MODE 0: scalar FFMA + MUFU + FADD; 1: packed FFMA2 + MUFU + FADD2;
// 2: packed with NPOLY of every 32 values through pexp2
template <int MODE, int NPOLY>
__global__ void __launch_bounds__(512, 1) epi_probe(int blocks, float* out, long long* cyc) {
  const int tid = threadIdx.x;
  float v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = -0.37f * e - 1e-3f * tid;
  float inv = 1.0f + 1e-7f * tid, nr = 0.25f;
  float acc = 0.f;
  unsigned long long acc2 = 0ull;
  const long long c0 = clock64();
  for (int kb = 0; kb < blocks; ++kb) {
    if (MODE == 0) {
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 32; ++e) s4[e & 3] += ex2a(fmaf(v[e], inv, nr));
      acc += (s4[0] + s4[1]) + (s4[2] + s4[3]);
    } else {
      const unsigned long long inv2 = pk(inv, inv), nr2 = pk(nr, nr);
      unsigned long long s2[2] = {0ull, 0ull};
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const unsigned long long a = ffma2(pk(v[e], v[e + 1]), inv2, nr2);
        unsigned long long y;
        if (e < NPOLY) {
          y = pexp2(a);
        } else {
          float a0, a1;
          upk(a, a0, a1);
          y = pk(ex2a(a0), ex2a(a1));
        }
        s2[(e >> 1) & 1] = fadd2(s2[(e >> 1) & 1], y);
      }
      acc2 = fadd2(acc2, fadd2(s2[0], s2[1]));
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] += 1e-6f;
  }
  const long long c1 = clock64();
  float a0, a1;
  upk(acc2, a0, a1);
  out[blockIdx.x * 512 + tid] = acc + a0 + a1;
  if (tid == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int MODE, int NPOLY>
void run_epi(float* o, long long* c, int sms) {
  const int blocks = 4000;
  epi_probe<MODE, NPOLY><<<sms, 512>>>(100, o, c);
  epi_probe<MODE, NPOLY><<<sms, 512>>>(blocks, o, c);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("epi error\n");
    return;
  }
  long long h = 0;
  cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const double exps = 512.0 * 32 * blocks;
  printf("epi mode=%d poly=%2d/32: %.2f exp/clk/SM\n", MODE, NPOLY, exps / h);
}

// accuracy of pexp2 against exp2 in double over [-30, 24]
__global__ void acc_probe(double* out) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const float x = -30.0f + 54.0f * tid / (gridDim.x * blockDim.x);
  float y0, y1;
  upk(pexp2(pk(x, x)), y0, y1);
  const double r = (double)y0 / exp2((double)x) - 1.0;
  const double m = (double)ex2a(x) / exp2((double)x) - 1.0;
  out[2 * tid] = r;
  out[2 * tid + 1] = m;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 4096 * sizeof(long long));
  run_umma<32, true, 1>(d, sms);
  run_umma<32, true, 2>(d, sms);
  run_umma<32, true, 4>(d, sms);
  run_umma<32, false, 1>(d, sms);
  run_umma<32, false, 2>(d, sms);
  run_umma<64, false, 1>(d, sms);
  run_umma<64, false, 2>(d, sms);
  run_umma<64, true, 2>(d, sms);
  run_umma<128, false, 1>(d, sms);
  run_umma<128, false, 2>(d, sms);
  run_umma<256, false, 1>(d, sms);
  float* o;
  cudaMalloc(&o, sms * 512 * sizeof(float));
  run_epi<0, 0>(o, d, sms);
  run_epi<1, 0>(o, d, sms);
  run_epi<2, 8>(o, d, sms);
  run_epi<2, 12>(o, d, sms);
  run_epi<2, 16>(o, d, sms);
  run_epi<2, 32>(o, d, sms);
  const int n = 148 * 256;
  double* a;
  cudaMalloc(&a, 2 * n * sizeof(double));
  acc_probe<<<148, 256>>>(a);
  double* h = new double[2 * n];
  cudaMemcpy(h, a, 2 * n * sizeof(double), cudaMemcpyDeviceToHost);
  double mr = 0, mm = 0, br = 0, bm = 0;
  for (int i = 0; i < n; ++i) {
    mr = fmax(mr, fabs(h[2 * i]));
    mm = fmax(mm, fabs(h[2 * i + 1]));
    br += h[2 * i];
    bm += h[2 * i + 1];
  }
  printf("pexp2 max rel err %.3e mean %.3e | ex2.approx max rel %.3e mean %.3e\n", mr, br / n, mm, bm / n);
  return 0;
}
