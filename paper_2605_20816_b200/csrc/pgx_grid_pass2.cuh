// pgx_grid_pass2.cuh — regular-grid pass 2 (grain-major): the gradient
// contraction sum_x (onehot_G(x) - p(x)) eta(x) (objective.py:109-113).
//
// CTA = GT grains x PT = 128/GT pixel lanes over a range of lines.  Per
// 128-pixel segment the per-pixel records (w, q, label, L_j(x_fast) in fp64
// and fp32) are staged in shared memory and read as warp broadcasts.  Per
// logit: the fp64 logit h'', p/2 = 2^(w - h'') by one MUFU.EX2 of the
// RN-converted argument, r/2 = label ? q : -p/2, and R_j += r L_j in fp32.
// R is flushed per segment into fp64 line sums and expanded into the K
// gradient rows per line (fp64, shared memory, one column per thread).
#pragma once

#include "pgx_grid_common.cuh"

namespace pgx {

constexpr int kG2Threads = 128;
constexpr int kG2Seg = 128;

template <int DIM, int D, int GT>
__global__ void __launch_bounds__(kG2Threads) k_grid_pass2(GridParams g) {
  constexpr int J = D + 1;
  constexpr int K = feature_count(DIM, D);
  constexpr int PT = kG2Threads / GT;
  constexpr int XPT = kG2Seg / PT;
  constexpr int JDP = (J + 1) & ~1;      // w, v_1..v_D (fp64)
  constexpr int JFP = (J + 1 + 3) & ~3;  // q, label, vf_1..vf_D (fp32)
  __shared__ __align__(16) double pd[kG2Seg][JDP];
  __shared__ __align__(16) float pf[kG2Seg][JFP];
  __shared__ double lc[K];
  extern __shared__ double acc_s[];  // [K][kG2Threads]

  const int tid = threadIdx.x;
  const int tg = tid % GT, pl = tid / GT;
  const int i = blockIdx.x * GT + tg;
  const bool active = i < g.N;
  const int ic = active ? i : g.N - 1;
  const int64_t l0 = (int64_t)blockIdx.y * g.lines_per_split;
  const int64_t l1 = min((int64_t)g.lines, l0 + g.lines_per_split);
  const unsigned pd_addr = (unsigned)__cvta_generic_to_shared(&pd[0][0]);
  const unsigned pf_addr = (unsigned)__cvta_generic_to_shared(&pf[0][0]);

#pragma unroll
  for (int k = 0; k < K; ++k) acc_s[k * kG2Threads + tid] = 0.0;
  griddep_wait();  // PDL: pass 1's per-pixel records are complete

  for (int64_t line = l0; line < l1; ++line) {
    __syncthreads();
    if (tid == 0) {
      double lcr[K];
      line_factors<DIM, D>(line, g, lcr);
#pragma unroll
      for (int k = 0; k < K; ++k) lc[k] = lcr[k];
    }
    __syncthreads();
    double B[J];
    line_coeffs<DIM, D>(g.theta, g.N, ic, lc, g.c, B);
    double R64[J];
#pragma unroll
    for (int j = 0; j < J; ++j) R64[j] = 0.0;
    const int64_t pline = line * g.side;
    for (int s0 = 0; s0 < g.side; s0 += kG2Seg) {
      __syncthreads();
      {
        const int col = s0 + tid;  // kG2Seg == kG2Threads
        double u[J];
        axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
        pd[tid][0] = g.pix_w[pline + col];
        pf[tid][0] = g.pix_q[pline + col];
        pf[tid][1] = __int_as_float(g.labels[pline + col]);
#pragma unroll
        for (int j = 1; j < J; ++j) {
          pd[tid][j] = u[j];
          pf[tid][j + 1] = (float)u[j];
        }
      }
      __syncthreads();
      float Rf[J];
#pragma unroll
      for (int j = 0; j < J; ++j) Rf[j] = 0.0f;
#pragma unroll 8
      for (int xi = 0; xi < XPT; ++xi) {
        const int x = pl * XPT + xi;
        double rd[JDP];
        float rf[JFP];
#pragma unroll
        for (int j = 0; j < JDP; j += 2) lds_f64x2(pd_addr + (x * JDP + j) * 8, rd[j], rd[j + 1]);
#pragma unroll
        for (int j = 0; j < JFP; j += 4)
          lds_f32x4(pf_addr + (x * JFP + j) * 4, rf[j], rf[j + 1], rf[j + 2], rf[j + 3]);
        double h = B[0];
#pragma unroll
        for (int j = 1; j < J; ++j) h = fma(B[j], rd[j], h);
        const float p2 = ex2_neg(h - rd[0]);                         // p_i / 2, argument >= 1
        const float r = (__float_as_int(rf[1]) == i) ? rf[0] : -p2;  // r / 2: objective.py:110-112
        Rf[0] += r;
#pragma unroll
        for (int j = 1; j < J; ++j) Rf[j] = fmaf(r, rf[j + 1], Rf[j]);
      }
#pragma unroll
      for (int j = 0; j < J; ++j) R64[j] += 2.0 * (double)Rf[j];
    }
    // expand the line sums into the K gradient rows (objective.py:113)
#pragma unroll
    for (int k = 0; k < K; ++k)
      acc_s[k * kG2Threads + tid] =
          fma(lc[k], R64[alpha_of(DIM, D, k, DIM - 1)], acc_s[k * kG2Threads + tid]);
  }
  __syncthreads();
  // fixed-order reduction over the PT pixel lanes of each grain
  if (pl == 0 && active) {
    for (int k = 0; k < K; ++k) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < PT; ++q) a += acc_s[k * kG2Threads + q * GT + tg];
      g.part_g[((int64_t)blockIdx.y * K + k) * g.N + i] = a;
    }
  }
}

}  // namespace pgx
