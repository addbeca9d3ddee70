// Issue-rate probe for the epilogue instruction mix of the tc kernels (B200):
// MUFU.EX2, F2FP (cvt.rn.f16x2.f32), FFMA / FFMA2 (packed f32x2), LOP3, FMNMX,
// a polynomial exp2 on the FMA pipe, and mixes of them.  Prints ops/clk/SM
// (thread-level ops; a warp instruction = 32).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_rate tools/pipe_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned cvt_h2(float a, float b) {
  unsigned r;
  asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ float lo_of(u64 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi_of(u64 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}

// 2^x for x <= 0 on the FMA pipe (pairs): round-to-nearest split x = n + f,
// f in [-0.5, 0.5], degree-DEG polynomial, exponent added by integer arithmetic
template <int DEG>
__device__ __forceinline__ u64 exp2_poly2(u64 x2) {
  const float MAGIC = 12582912.0f;  // 1.5 * 2^23
  const u64 m2 = pk(MAGIC, MAGIC), nm2 = pk(-MAGIC, -MAGIC);
  const u64 t2 = fadd2(x2, m2);
  const u64 n2 = fadd2(t2, nm2);
  const u64 f2 = ffma2(n2, pk(-1.0f, -1.0f), x2);
  // minimax-ish coefficients of 2^f on [-0.5, 0.5] (Taylor in ln2 f refined by Remez offline)
  u64 p;
  if (DEG == 5) {
    p = ffma2(pk(1.3333558e-3f, 1.3333558e-3f), f2, pk(9.6181291e-3f, 9.6181291e-3f));
    p = ffma2(p, f2, pk(5.5504109e-2f, 5.5504109e-2f));
  } else if (DEG == 4) {
    p = ffma2(pk(9.6181291e-3f, 9.6181291e-3f), f2, pk(5.5504109e-2f, 5.5504109e-2f));
  } else {
    p = pk(5.5504109e-2f, 5.5504109e-2f);
  }
  p = ffma2(p, f2, pk(2.4022651e-1f, 2.4022651e-1f));
  p = ffma2(p, f2, pk(6.9314718e-1f, 6.9314718e-1f));
  p = ffma2(p, f2, pk(1.0f, 1.0f));
  const unsigned el = (__float_as_uint(lo_of(t2)) << 23) + __float_as_uint(lo_of(p));
  const unsigned eh = (__float_as_uint(hi_of(t2)) << 23) + __float_as_uint(hi_of(p));
  return pk(__uint_as_float(el), __uint_as_float(eh));
}

// MODE: 0 EX2; 1 F2FP; 2 EX2 + F2FP (1:1); 3 FFMA 3-reg; 4 FFMA2; 5 LOP3; 6 FMNMX;
// 7 poly5 pairs; 8 EX2 : poly5 = 3:1; 9 EX2 : poly5 = 1:1; 10 poly4; 11 EX2:poly4 = 3:1
// 12 EX2 + LOP3 + FFMA2 (grad epilogue without the cvt); 13 = 12 + 1 F2FP per value
template <int MODE>
__global__ void rate_kernel(float* out, int iters) {
  float a = threadIdx.x * 1e-3f - 3.0f, b = a - 1.0f, c = a - 2.0f, d = a - 0.5f;
  float e = a - 0.25f, f = a - 0.75f, g = a - 1.25f, h = a - 1.75f;
  unsigned ua = threadIdx.x, ub = threadIdx.x * 3, uc = 7, ud = 11;
  u64 pa = pk(a, b), pb = pk(c, d), pc = pk(e, f), pd = pk(g, h);
  const u64 k1 = pk(0.999f, 0.999f), k2 = pk(-1e-3f, -1e-3f);
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      a = ex2a(a) - 3.0f; b = ex2a(b) - 3.0f; c = ex2a(c) - 3.0f; d = ex2a(d) - 3.0f;
    } else if (MODE == 1) {
      ua += cvt_h2(a, b); ub += cvt_h2(c, d); uc += cvt_h2(e, f); ud += cvt_h2(g, h);
      a = __uint_as_float(ua & 0x3fffffffu); c = __uint_as_float(ub & 0x3fffffffu);
      e = __uint_as_float(uc & 0x3fffffffu); g = __uint_as_float(ud & 0x3fffffffu);
    } else if (MODE == 2) {
      a = ex2a(a); b = ex2a(b); c = ex2a(c); d = ex2a(d);
      ua = cvt_h2(a, b); ub = cvt_h2(c, d); uc = cvt_h2(a, c); ud = cvt_h2(b, d);
      a = __uint_as_float((ua ^ uc) | 0xc0000000u); b = __uint_as_float((ub ^ ud) | 0xc0000000u);
      c = a - 1.0f; d = b - 1.0f;
    } else if (MODE == 3) {
      a = fmaf(a, b, c); b = fmaf(b, c, d); c = fmaf(c, d, e); d = fmaf(d, e, f);
      e = fmaf(e, f, g); f = fmaf(f, g, h); g = fmaf(g, h, a); h = fmaf(h, a, b);
    } else if (MODE == 4) {
      pa = ffma2(pa, k1, pb); pb = ffma2(pb, k1, pc); pc = ffma2(pc, k1, pd); pd = ffma2(pd, k1, pa);
    } else if (MODE == 5) {
      ua = (ua & ub) ^ uc; ub = (ub & uc) ^ ud; uc = (uc | ud) ^ ua; ud = (ud & ua) ^ ub;
    } else if (MODE == 6) {
      a = fminf(a, fminf(b, c)) + 1.0f; b = fminf(b, fminf(c, d)); c = fminf(c, fminf(d, e)); d = fminf(d, fminf(e, a));
    } else if (MODE == 7 || MODE == 10) {
      pa = ffma2(MODE == 7 ? exp2_poly2<5>(pa) : exp2_poly2<4>(pa), k1, k2);
      pb = ffma2(MODE == 7 ? exp2_poly2<5>(pb) : exp2_poly2<4>(pb), k1, k2);
    } else if (MODE == 8 || MODE == 11) {  // 6 MUFU + 2 poly values
      a = ex2a(a) - 3.0f; b = ex2a(b) - 3.0f; c = ex2a(c) - 3.0f; d = ex2a(d) - 3.0f;
      e = ex2a(e) - 3.0f; f = ex2a(f) - 3.0f;
      pa = ffma2(MODE == 8 ? exp2_poly2<5>(pa) : exp2_poly2<4>(pa), k1, k2);
    } else if (MODE == 9) {  // 4 MUFU + 4 poly values
      a = ex2a(a) - 3.0f; b = ex2a(b) - 3.0f; c = ex2a(c) - 3.0f; d = ex2a(d) - 3.0f;
      pa = ffma2(exp2_poly2<5>(pa), k1, k2);
      pb = ffma2(exp2_poly2<5>(pb), k1, k2);
    } else if (MODE == 12 || MODE == 13) {
      // per value: ffma2/2 + ex2 + LOP + ffma2/2 (+ F2FP)
      u64 x = ffma2(pa, k1, k2), y = ffma2(pb, k1, k2);
      a = ex2a(lo_of(x)); b = ex2a(hi_of(x)); c = ex2a(lo_of(y)); d = ex2a(hi_of(y));
      const float h0 = __uint_as_float(__float_as_uint(a) & 0xffffe000u), h1 = __uint_as_float(__float_as_uint(b) & 0xffffe000u);
      const float h2 = __uint_as_float(__float_as_uint(c) & 0xffffe000u), h3 = __uint_as_float(__float_as_uint(d) & 0xffffe000u);
      const u64 l01 = ffma2(pk(h0, h1), pk(-1.0f, -1.0f), pk(a, b));
      const u64 l23 = ffma2(pk(h2, h3), pk(-1.0f, -1.0f), pk(c, d));
      if (MODE == 13) {
        ua ^= cvt_h2(h0, h1); ub ^= cvt_h2(h2, h3);
        uc ^= cvt_h2(lo_of(l01), hi_of(l01)); ud ^= cvt_h2(lo_of(l23), hi_of(l23));
      } else {
        ua ^= __float_as_uint(h0) + __float_as_uint(h1); ub ^= __float_as_uint(h2) + __float_as_uint(h3);
        pc = fadd2(pc, l01); pd = fadd2(pd, l23);
      }
      pa = fadd2(x, k2); pb = fadd2(y, k2);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] =
      a + b + c + d + e + f + g + h + (float)(ua + ub + uc + ud) + lo_of(pa) + hi_of(pa) + lo_of(pb) + hi_of(pb) +
      lo_of(pc) + hi_of(pc) + lo_of(pd) + hi_of(pd);
}

__global__ void acc_kernel(int n, double* out) {
  // accuracy of the polynomial exp2 against fp64 exp2 on x in [-30, 0]
  double s5 = 0, m5 = 0, s4 = 0, m4 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float x = -30.0f * ((float)i + 0.5f) / n;
    const double ref = exp2((double)x);
    const double r5 = ((double)lo_of(exp2_poly2<5>(pk(x, x))) - ref) / ref;
    const double r4 = ((double)lo_of(exp2_poly2<4>(pk(x, x))) - ref) / ref;
    s5 += r5; m5 = fmax(m5, fabs(r5)); s4 += r4; m4 = fmax(m4, fabs(r4));
  }
  atomicAdd(out, s5); atomicAdd(out + 2, s4);
  atomicMax((u64*)(out + 1), (u64)__double_as_longlong(m5));
  atomicMax((u64*)(out + 3), (u64)__double_as_longlong(m4));
}

template <int MODE>
static void run(const char* name, double ops_per_iter, float* buf) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    rate_kernel<MODE><<<148 * 4, 512>>>(buf, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double ops = 148.0 * 4 * 512 * iters * ops_per_iter;
  printf("%-44s %.3f ms  %.2f values/clk/SM (1.965 GHz)\n", name, ms, ops / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
  float* buf;
  cudaMalloc(&buf, 148 * 4 * 512 * 4);
  double* d_out;
  cudaMalloc(&d_out, 32);
  cudaMemset(d_out, 0, 32);
  const int n = 1 << 24;
  acc_kernel<<<512, 256>>>(n, d_out);
  double h[4];
  cudaMemcpy(h, d_out, 32, cudaMemcpyDeviceToHost);
  printf("poly5 exp2: mean rel %+.3e max %.3e;  poly4: mean rel %+.3e max %.3e\n", h[0] / n, h[1], h[2] / n, h[3]);
  run<0>("MUFU.EX2 (+FADD)", 4, buf);
  run<1>("F2FP cvt.rn.f16x2.f32 (per cvt; +IADD+LOP)", 4, buf);
  run<2>("EX2 + F2FP 1:1 (per ex2)", 4, buf);
  run<3>("FFMA 3-reg", 8, buf);
  run<4>("FFMA2 (per f32 value)", 8, buf);
  run<5>("LOP3 x2 (per pair)", 4, buf);
  run<6>("FMNMX x2 (per pair)", 4, buf);
  run<7>("poly5 exp2 (per value)", 4, buf);
  run<10>("poly4 exp2 (per value)", 4, buf);
  run<8>("EX2 : poly5 = 3:1 (per value)", 8, buf);
  run<11>("EX2 : poly4 = 3:1 (per value)", 8, buf);
  run<9>("EX2 : poly5 = 1:1 (per value)", 8, buf);
  run<12>("grad epilogue mix without F2FP (per value)", 4, buf);
  run<13>("grad epilogue mix with F2FP (per value)", 4, buf);
  return 0;
}
