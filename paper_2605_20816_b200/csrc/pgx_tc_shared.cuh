// pgx_tc_shared.cuh — pieces shared by the tensor-core pass-1 (pgx_tc_sweep.cuh)
// and pass-2 (pgx_tc_grad.cuh) kernels: tile geometry and the pass-2 record
// layout that pass 1 writes, the exact fp64 candidate bookkeeping of the
// tie-tolerant arg-min (geometry.py:201-210), packed fp32-pair (f32x2)
// arithmetic and an mbarrier spin.
#pragma once

#include <math_constants.h>

#include "pgx_common.cuh"
#include "pgx_tc_coeffs.cuh"

namespace pgx {

#ifndef PGX_TC2_GROUP
#define PGX_TC2_GROUP 16
#endif
constexpr int kTcThreadsTile = 128;  // pixels per pass-1 tile (UMMA M, TMEM lanes)
constexpr int kTc2Epi = 256;         // pass-2 epilogue threads (8 warps)
constexpr int kTc2Grains = 128;      // grains per pass-2 CTA (TMEM lanes)
constexpr int kTc2Px = kTcPixTile;   // pixels per pass-2 tile
constexpr int kTc2Group = PGX_TC2_GROUP;  // tiles per fp32 R group before the fp64 flush (16: 1024 pixels;
                                          // c5 pass 2 7.02 -> 6.70 ms, tc-vs-exact grad error 1.5e-6 -> 1.9e-6; 32: 4.3e-6)
constexpr int kTc2S = 3;             // pass-2 S stages in TMEM (UMMA 1 runs 3 tiles ahead)
constexpr int kTc2RecFloats = 4 * kTc2Px;  // pass-2 record per tile: w13[64] | wl13[64] | qn[64] | label[64]

// exact per-pixel state for near-minimal logits
struct TcRare {
  double m, m2, hb0, hb1;
  int b0, b1, cnt, flags;  // flags: 1 dirty (candidate list overflowed), 2 needfix
};

__device__ __forceinline__ void tc_rare_update(TcRare& st, int i, double h, double c) {
  if (h < st.m) {
    st.m2 = fmin(st.m2, st.m);
    st.m = h;
    const double thr = h + c * kTieRtol * (1.0 + fabs(h / c));
    if (st.cnt > 0 && !(st.hb0 <= thr)) {
      if (st.flags & 1) st.flags |= 2;
      if (st.cnt > 1 && st.hb1 <= thr) {
        st.b0 = st.b1;
        st.hb0 = st.hb1;
        st.cnt = 1;
      } else {
        st.cnt = 0;
      }
    } else if (st.cnt > 1 && !(st.hb1 <= thr)) {
      st.cnt = 1;
    }
  } else if (h < st.m2) {
    st.m2 = h;
  }
  const double thr = st.m + c * kTieRtol * (1.0 + fabs(st.m / c));
  if (h <= thr) {
    if (st.cnt == 0) {
      st.b0 = i;
      st.hb0 = h;
      st.cnt = 1;
    } else if (st.cnt == 1) {
      st.b1 = i;
      st.hb1 = h;
      st.cnt = 2;
    } else {
      st.flags |= 1;
    }
  }
}

// packed fp32 pairs (f32x2 SIMD on sm_100: FFMA2 / FADD2)
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ float f2lo(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float f2hi(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }
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

// 2^x for a pair on the FMA pipe (no MUFU): x clamped to >= -125, split
// x = n + f by the 1.5 * 2^23 shifter (f in [-0.5, 0.5]), degree-5 minimax
// polynomial, exponent added with integer arithmetic.  Relative error
// <= 2.2e-7 (mean 5e-8; tools/probe_r2.cu), the same order as ex2.approx.
__device__ __forceinline__ unsigned long long pexp2(unsigned long long x2) {
  x2 = f2pack(fmaxf(f2lo(x2), -125.0f), fmaxf(f2hi(x2), -125.0f));
  const unsigned long long t = fadd2(x2, f2pack(12582912.0f, 12582912.0f));
  const unsigned long long j = fadd2(t, f2pack(-12582912.0f, -12582912.0f));
  const unsigned long long f = ffma2(j, f2pack(-1.0f, -1.0f), x2);
  unsigned long long p = f2pack(1.327647129073739e-3f, 1.327647129073739e-3f);
  p = ffma2(p, f, f2pack(9.675541892647743e-3f, 9.675541892647743e-3f));
  p = ffma2(p, f, f2pack(5.550713092088699e-2f, 5.550713092088699e-2f));
  p = ffma2(p, f, f2pack(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = ffma2(p, f, f2pack(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = ffma2(p, f, f2pack(1.0000001192092896f, 1.0000001192092896f));
  const unsigned rl = (unsigned)p + ((unsigned)t << 23);
  const unsigned rh = (unsigned)(p >> 32) + ((unsigned)(t >> 32) << 23);
  return ((unsigned long long)rh << 32) | rl;
}

// spin on a phase (no suspend hint: the epilogue's waits are short); a lost
// arrival traps instead of hanging the GPU
__device__ __forceinline__ void mbar_spin(unsigned addr, unsigned parity) {
  for (unsigned spin = 0;; ++spin) {
    unsigned done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (spin == (1u << 28)) __trap();
  }
}

}  // namespace pgx
