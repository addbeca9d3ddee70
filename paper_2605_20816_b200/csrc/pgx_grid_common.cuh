// pgx_grid_common.cuh — shared pieces of the regular-grid (separable) path.
//
// On a regular grid every pixel line along the fastest axis shares all other
// coordinates, and the tensor-product basis factorises (basis.py:105-117):
//
//   h_i(x) = sum_k theta_{k,i} eta_k(x) = sum_{j<=d} B_{j,i}(line) L_j(x_fast),
//   B_{j,i}(line) = sum_{k: alpha_fast(k) = j} theta_{k,i} prod_{other axes} L(x_axis)
//
// so a logit costs d+1 fp64 FMAs instead of K = C(d+dim, dim), and the
// gradient contraction sum_x r_i(x) eta_k(x) (objective.py:113) factorises the
// same way: R_{j,i}(line) = sum_{x in line} r_i(x) L_j(x_fast), then
// grad_{k,i} += prod_other L * R_{alpha_fast(k),i}(line).
//
// Units: h'' = h * c with c = log2(e)/eps, so softmax weights are powers of 2.
#pragma once

#include <math_constants.h>

#include "../../include/pgx.h"
#include "pgx_common.cuh"
#include "pgx_general.cuh"

namespace pgx {

// ------------------------------------------------------------ index helpers
__host__ __device__ constexpr int alpha_of(int dim, int D, int k, int axis) {
  int idx = 0;
  for (int t = 0; t <= D; ++t)
    for (int a1 = t; a1 >= 0; --a1) {
      if (dim == 2) {
        if (idx == k) return axis == 0 ? a1 : t - a1;
        ++idx;
      } else {
        for (int a2 = t - a1; a2 >= 0; --a2) {
          if (idx == k) return axis == 0 ? a1 : (axis == 1 ? a2 : t - a1 - a2);
          ++idx;
        }
      }
    }
  return 0;
}

// ------------------------------------------------------------ exponentials
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// a as fp32, round-to-nearest, for 0.5 <= a < 2^127 (a > 0), without F2F:
// F2F.F32.F64 issues on the same pipe as MUFU.EX2 (measured: 15.7 vs 7.4
// results/clk/SM alone vs together), so the conversion is done with integer
// ops: +2^28 on the 64-bit pattern rounds the 29 dropped mantissa bits, the
// exponent is re-biased in the high word (E8 = E11 - 896; no borrow since
// E11 >= 1022) and the funnel shift drops the sign and the (zero) top
// exponent bits.  Three integer ops.
__device__ __forceinline__ float pos_f64_to_f32_rn(double a) {
  const unsigned long long b =
      (unsigned long long)__double_as_longlong(a) + (1ull << 28) - (0x38000000ull << 32);
  return __uint_as_float(__funnelshift_l((unsigned)b, (unsigned)(b >> 32), 3));
}

// 2^-a for a >= 0.5 given in fp64: one MUFU.EX2 (negation is an operand modifier)
__device__ __forceinline__ float ex2_neg(double a) { return ex2_approx(-pos_f64_to_f32_rn(a)); }

__device__ __forceinline__ void lds_f64x2(unsigned addr, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr));
}
__device__ __forceinline__ void lds_f32x4(unsigned addr, float& a, float& b, float& c, float& d) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
               : "r"(addr));
}

// ------------------------------------------------------------ parameters
struct GridParams {
  int64_t P;
  int N;
  int M;           // resolution; side = 2M
  int side;
  int pside;       // tensor-core kernels: side rounded up to a multiple of 128 (padding pixels masked)
  int legendre;
  int R;           // pixels per thread (pass 1)
  int lines;       // number of lines along the fast axis
  int segs;        // pass-1 tiles per line
  const double* __restrict__ theta;  // K x N fp64
  const int32_t* __restrict__ labels;
  double eps;
  double c;        // log2(e) / eps
  double tau_amb;
  // fp32 theta of this evaluation (nullptr: theta is fp64): k_tc_coeffs reads
  // it directly and, on line 0, writes the fp64 copy `theta` for the kernels after it
  const float* __restrict__ theta32;
  // outputs / scratch
  double* pix_m;   // min cost (h units) for the arg-min fix-up
  double* pix_w;   // w: p_i / 2 = 2^(w - h''_i) with w - h'' <= -1
  float* pix_q;    // (1 - p_G) / 2 = sum_{j != G} p_j / 2
  double* part_d;
  long long* part_i;
  int* fix_count;
  int* fix_list;
  // pass 2
  int GT;          // grains per CTA (pass 2)
  int lines_per_split;
  int64_t items_per_split;  // tc pass 2: (line, 64-pixel tile) items per CTA row
  int splits;
  double* part_g;  // [splits][K][N]
  // tensor-core path: per-line coefficient tables (pgx_tc_coeffs.cuh)
  const double* tc_coef;        // [lines][N][J] exact B''
  const unsigned char* tc_img;  // [lines][chunks] UMMA operand images
  const int2* tc_meta;          // [lines][chunks] {sB, bnorm bits}
  int tc_nchunks;
  double* tc_lc;                // [lines][K] line factors (k_tc_coeffs)
  const unsigned char* tc_pix;  // [side / 64] pass-2 pixel operand tiles (k_tc_pix)
  // tensor-core launches over a part of the evaluation (line chunks that
  // overlap pass 1 of one chunk with pass 2 of the previous one)
  int64_t tile_lo, tile_hi;     // pass 1: tiles [tile_lo, tile_hi) of 128 pixels
  int part_off;                 // pass 1: first per-CTA partial slot
  int64_t line_lo;              // pass 2: first line (g.lines = end line)
  int split_off;                // pass 2: first gradient-partial split slot
  float* tc_rec;                // [lines][pside / 64][4][64] pass-2 pixel records
                                // (w13, wl13, qn, label) written by TC pass 1
  // hard-assignment variant of the tensor-core sweep (pgx_assign)
  long long* labels_out;        // 1-based arg-min labels
  float* margin_out;            // top-2 margin (nullable)
};

// Per-line factors: lc[k] = prod over the non-fast axes of u_axis[alpha]
template <int DIM, int D>
__device__ __forceinline__ void line_factors(int64_t line, const GridParams& g,
                                             double lc[feature_count(DIM, D)]) {
  constexpr int K = feature_count(DIM, D);
  double u0[D + 1], u1[D + 1];
  if (DIM == 2) {
    axis_table<D>(axis_coord(line, g.M), g.legendre != 0, u0);
#pragma unroll
    for (int k = 0; k < K; ++k) lc[k] = u0[alpha_of(DIM, D, k, 0)];
  } else {
    axis_table<D>(axis_coord(line / g.side, g.M), g.legendre != 0, u0);
    axis_table<D>(axis_coord(line % g.side, g.M), g.legendre != 0, u1);
#pragma unroll
    for (int k = 0; k < K; ++k)
      lc[k] = __dmul_rn(u0[alpha_of(DIM, D, k, 0)], u1[alpha_of(DIM, D, k, 1)]);
  }
}

// B''_{j,i} = c * sum_{k: alpha_fast(k) = j} theta_{k,i} lc[k]   (fixed order)
template <int DIM, int D, typename T>
__device__ __forceinline__ void line_coeffs(const T* __restrict__ theta, int N, int i,
                                            const double lc[feature_count(DIM, D)], double c,
                                            double B[D + 1]) {
  constexpr int K = feature_count(DIM, D);
#pragma unroll
  for (int j = 0; j <= D; ++j) B[j] = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = alpha_of(DIM, D, k, DIM - 1);
    B[j] = fma((double)__ldg(theta + (int64_t)k * N + i), lc[k], B[j]);  // fp32 theta: exact widening
  }
#pragma unroll
  for (int j = 0; j <= D; ++j) B[j] *= c;
}

// h'' = B_0 + sum_{j>=1} B_j v_j  (L_0 == 1; the fixed fma order every kernel uses)
template <int J>
__device__ __forceinline__ double eval_line(const double* B, const double* v) {
  double h = B[0];
#pragma unroll
  for (int j = 1; j < J; ++j) h = fma(B[j], v[j], h);
  return h;
}

}  // namespace pgx
