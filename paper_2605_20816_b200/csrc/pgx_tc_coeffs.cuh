// pgx_tc_coeffs.cuh — once per evaluation, the per-line grain coefficients of
// the tensor-core path, shared by every CTA that touches the line:
//
//   coef[line][i][j]   exact fp64 B''_{j,i}(line) (c-scaled), for the fp64
//                      re-evaluation of near-minimal logits and the label term;
//   img[line][chunk]   the UMMA operand image of 128 grains: K-major
//                      SWIZZLE_NONE slabs, K pattern [hi, lo, hi] of the
//                      2^sB-scaled fp16 split (pass-1 B operand, pass-2 A);
//   meta[line][chunk]  {sB, max_i sum_j |B''_{j,i}|}.
//
// Without it every pass-1 CTA rebuilt each chunk twice (sweeps A and B) and
// every pass-2 CTA rebuilt its tile per line: K fp64 FMAs + K loads per grain,
// ~30% of pass-1 instructions at c5.
#pragma once

#include "pgx_grid_common.cuh"
#include "pgx_tc_common.cuh"

namespace pgx {

constexpr int kTcCoefChunk = 128;  // grains per image chunk (= pass-1 UMMA N = pass-2 M)

struct TcCoefMeta {
  int sB;       // fp16 scale exponent of the chunk
  float bnorm;  // max over the chunk's grains of sum_j |B''_j|
};

template <int J>
__host__ __device__ constexpr int tc_img_bytes() {
  return tc_ksteps(J) * kTcCoefChunk * 32;
}

template <int DIM, int D>
__global__ void __launch_bounds__(kTcCoefChunk) k_tc_coeffs(GridParams g, double* __restrict__ coef,
                                                            unsigned char* __restrict__ img,
                                                            TcCoefMeta* __restrict__ meta,
                                                            int nchunks) {
  constexpr int J = D + 1;
  constexpr int K = feature_count(DIM, D);
  constexpr int KS = tc_ksteps(J);
  __shared__ double lc[K];
  __shared__ unsigned s_max, s_b1;
  const int tid = threadIdx.x;
  // lines on gridDim.x (3-D grids have side^2 > 65535 of them), chunks on y
  const int chunk = blockIdx.y;
  const int64_t line = blockIdx.x;
  const int i = chunk * kTcCoefChunk + tid;
  if (tid == 0) {
    double lcr[K];
    line_factors<DIM, D>(line, g, lcr);
#pragma unroll
    for (int k = 0; k < K; ++k) lc[k] = lcr[k];
    if (chunk == 0 && g.tc_lc) {
#pragma unroll
      for (int k = 0; k < K; ++k) g.tc_lc[line * K + k] = lcr[k];
    }
    s_max = 0u;
    s_b1 = 0u;
  }
  __syncthreads();
  double B[J];
  if (i < g.N) {
    if (g.theta32) {
      line_coeffs<DIM, D>(g.theta32, g.N, i, lc, g.c, B);
      if (line == 0) {  // the fp64 theta every later kernel reads
        double* th64 = const_cast<double*>(g.theta);
#pragma unroll
        for (int k = 0; k < K; ++k)
          th64[(int64_t)k * g.N + i] = (double)g.theta32[(int64_t)k * g.N + i];
      }
    } else {
      line_coeffs<DIM, D>(g.theta, g.N, i, lc, g.c, B);
    }
    double* out = coef + (line * g.N + i) * J;
#pragma unroll
    for (int j = 0; j < J; ++j) out[j] = B[j];
  } else {
#pragma unroll
    for (int j = 0; j < J; ++j) B[j] = 0.0;
  }
  float bm = 0.0f, b1 = 0.0f;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    bm = fmaxf(bm, (float)fabs(B[j]));
    b1 += (float)fabs(B[j]);
  }
  // non-finite coefficients poison the scale; the passes then flag the pixels
  atomicMax(&s_max, __float_as_uint(isfinite(bm) ? bm : CUDART_INF_F));
  atomicMax(&s_b1, __float_as_uint(isfinite(b1) ? b1 * 1.0000005f : CUDART_INF_F));
  __syncthreads();
  const float chmax = __uint_as_float(s_max);
  const int sB = chmax > 0.0f && chmax < 3e38f ? 13 - ilogbf(chmax) : 0;
  const double scl = ldexp(1.0, sB);
  __half hi[J], lo[J];
#pragma unroll
  for (int j = 0; j < J; ++j) split_f16(B[j] * scl, hi[j], lo[j]);
  unsigned char* dst = img + (line * nchunks + chunk) * (int64_t)tc_img_bytes<J>();
  // row tid: 16 K-elements per slab = two 16-byte core-matrix rows
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    __half row[16];
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const int k = s * 16 + kk;
      const int b = k / J, j = k % J;
      row[kk] = k < 3 * J ? (b == 1 ? lo[j] : hi[j]) : __float2half(0.0f);
    }
    unsigned char* slab = dst + s * (kTcCoefChunk * 32);
    *reinterpret_cast<uint4*>(slab + slab_off(tid, 0)) = *reinterpret_cast<const uint4*>(row);
    *reinterpret_cast<uint4*>(slab + slab_off(tid, 8)) = *reinterpret_cast<const uint4*>(row + 8);
  }
  if (tid == 0) {
    TcCoefMeta m;
    m.sB = sB;
    m.bnorm = __uint_as_float(s_b1);
    meta[line * nchunks + chunk] = m;
  }
}

// The same tables with several lines per CTA, for many features (K > 16): the chunk's
// theta (K x 128) is read once into registers and serves kTcCoefLines lines.  Every
// (line, chunk) CTA re-reading it made k_tc_coeffs L2-read bound at c5 (3 GB of theta
// reads for 1.1 GB of table writes: 0.43 -> 0.35 ms); with few features the one-line
// kernel above is faster (c4: 0.58 vs 0.68 ms), so the launcher picks (tc_coef_lines).
constexpr int kTcCoefLines = 8;
__host__ __device__ constexpr int tc_coef_lines(int dim, int degree) {
  return feature_count(dim, degree) > 16 ? kTcCoefLines : 1;
}

template <int DIM, int D>
__global__ void __launch_bounds__(kTcCoefChunk) k_tc_coeffs_ml(GridParams g, double* __restrict__ coef,
                                                            unsigned char* __restrict__ img,
                                                            TcCoefMeta* __restrict__ meta,
                                                            int nchunks) {
  constexpr int J = D + 1;
  constexpr int K = feature_count(DIM, D);
  constexpr int KS = tc_ksteps(J);
  __shared__ double lc[tc_coef_lines(DIM, D)][K];
  __shared__ unsigned s_max[tc_coef_lines(DIM, D)], s_b1[tc_coef_lines(DIM, D)];
  const int tid = threadIdx.x;
  // line groups on gridDim.x (3-D grids have side^2 > 65535 lines), chunks on y
  const int chunk = blockIdx.y;
  constexpr int LPC = tc_coef_lines(DIM, D);
  const int64_t line0 = (int64_t)blockIdx.x * LPC;
  const int nl = (int)min((int64_t)LPC, (int64_t)g.lines - line0);
  const int i = chunk * kTcCoefChunk + tid;
  if (tid < nl) {
    double lcr[K];
    line_factors<DIM, D>(line0 + tid, g, lcr);
#pragma unroll
    for (int k = 0; k < K; ++k) lc[tid][k] = lcr[k];
    if (chunk == 0 && g.tc_lc) {
#pragma unroll
      for (int k = 0; k < K; ++k) g.tc_lc[(line0 + tid) * K + k] = lcr[k];
    }
    s_max[tid] = 0u;
    s_b1[tid] = 0u;
  }
  // this thread's grain: theta column i, widened exactly when fp32
  double th[K];
  if (i < g.N) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      th[k] = g.theta32 ? (double)__ldg(g.theta32 + (int64_t)k * g.N + i) : __ldg(g.theta + (int64_t)k * g.N + i);
    if (g.theta32 && line0 == 0) {  // the fp64 theta every later kernel reads
      double* th64 = const_cast<double*>(g.theta);
#pragma unroll
      for (int k = 0; k < K; ++k) th64[(int64_t)k * g.N + i] = th[k];
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) th[k] = 0.0;
  }
  __syncthreads();
#pragma unroll 1
  for (int l = 0; l < nl; ++l) {
    // B''_{j,i} = c * sum_{k: alpha_fast(k) = j} theta_{k,i} lc[k]: the order of line_coeffs
    double B[J];
#pragma unroll
    for (int j = 0; j < J; ++j) B[j] = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = alpha_of(DIM, D, k, DIM - 1);
      B[j] = fma(th[k], lc[l][k], B[j]);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) B[j] *= g.c;
    if (i < g.N) {
      double* out = coef + ((line0 + l) * g.N + i) * J;
#pragma unroll
      for (int j = 0; j < J; ++j) out[j] = B[j];
    }
    float bm = 0.0f, b1 = 0.0f;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      bm = fmaxf(bm, (float)fabs(B[j]));
      b1 += (float)fabs(B[j]);
    }
    // non-finite coefficients poison the scale; the passes then flag the pixels
    atomicMax(&s_max[l], __float_as_uint(isfinite(bm) ? bm : CUDART_INF_F));
    atomicMax(&s_b1[l], __float_as_uint(isfinite(b1) ? b1 * 1.0000005f : CUDART_INF_F));
    __syncthreads();
    const float chmax = __uint_as_float(s_max[l]);
    const int sB = chmax > 0.0f && chmax < 3e38f ? 13 - ilogbf(chmax) : 0;
    const double scl = ldexp(1.0, sB);
    __half hi[J], lo[J];
#pragma unroll
    for (int j = 0; j < J; ++j) split_f16(B[j] * scl, hi[j], lo[j]);
    unsigned char* dst = img + ((line0 + l) * nchunks + chunk) * (int64_t)tc_img_bytes<J>();
    // row tid: 16 K-elements per slab = two 16-byte core-matrix rows
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      __half row[16];
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int k = s * 16 + kk;
        const int b = k / J, j = k % J;
        row[kk] = k < 3 * J ? (b == 1 ? lo[j] : hi[j]) : __float2half(0.0f);
      }
      unsigned char* slab = dst + s * (kTcCoefChunk * 32);
      *reinterpret_cast<uint4*>(slab + slab_off(tid, 0)) = *reinterpret_cast<const uint4*>(row);
      *reinterpret_cast<uint4*>(slab + slab_off(tid, 8)) = *reinterpret_cast<const uint4*>(row + 8);
    }
    if (tid == 0) {
      TcCoefMeta m;
      m.sB = sB;
      m.bnorm = __uint_as_float(s_b1[l]);
      meta[(line0 + l) * nchunks + chunk] = m;
    }
  }
}

// ------------------------------------------------------------------ pixel tables
// Pass-2 pixel operands of one 64-pixel tile of the fast axis (they depend on
// the column only, so one table serves every line; built once per problem):
//   [0, KS*2048)          UMMA 1 B: 64 rows (pixels) x K, pattern [hi, hi, lo]
//                         of the 2^10-scaled fp16 split of u_j(x)
//   [KS*2048, +4096)      UMMA 2 B: 32 rows x K = 64 pixels, rows 0-15 = L_hi(j),
//                         rows 16-31 = L_lo(j) (zero-padded j), one 1 KB slab per
//                         16 pixels
constexpr int kTcPixTile = 64;

template <int J>
__host__ __device__ constexpr int tc_pix_bytes() {
  return tc_ksteps(J) * kTcPixTile * 32 + 2 * (kTcPixTile / 16) * 16 * 32;
}

template <int D>
__global__ void __launch_bounds__(kTcPixTile) k_tc_pix(int M, int legendre,
                                                       unsigned char* __restrict__ pix) {
  constexpr int J = D + 1;
  constexpr int KS = tc_ksteps(J);
  const int tid = threadIdx.x;
  const int col = blockIdx.x * kTcPixTile + tid;
  unsigned char* dst = pix + (int64_t)blockIdx.x * tc_pix_bytes<J>();
  double u[J];
  axis_table<D>(axis_coord(col, M), legendre != 0, u);
  __half hi[J], lo[J];
  // (padding columns of a side % 128 != 0 grid: zero operands, so S = 0 and R += 0)
#pragma unroll
  for (int j = 0; j < J; ++j) split_f16(col < 2 * M ? u[j] * 1024.0 : 0.0, hi[j], lo[j]);
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    __half row[16];
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const int k = s * 16 + kk;
      const int b = k / J, j = k % J;
      row[kk] = k < 3 * J ? (b < 2 ? hi[j] : lo[j]) : __float2half(0.0f);
    }
    unsigned char* slab = dst + s * (kTcPixTile * 32);
    *reinterpret_cast<uint4*>(slab + slab_off(tid, 0)) = *reinterpret_cast<const uint4*>(row);
    *reinterpret_cast<uint4*>(slab + slab_off(tid, 8)) = *reinterpret_cast<const uint4*>(row + 8);
  }
  unsigned char* l2 = dst + KS * (kTcPixTile * 32);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    unsigned char* slab = l2 + (tid / 16) * (32 * 32);
    *reinterpret_cast<__half*>(slab + slab_off(j, tid % 16)) = j < J ? hi[j] : __float2half(0.0f);
    *reinterpret_cast<__half*>(slab + slab_off(16 + j, tid % 16)) = j < J ? lo[j] : __float2half(0.0f);
  }
}

// cooperative copy of one coefficient image (KS * 4 KB) into shared memory
template <int J, int NT>
__device__ __forceinline__ void copy_coef_img(unsigned char* dst, const unsigned char* src, int tid) {
  constexpr int n16 = tc_img_bytes<J>() / 16;
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = tid; q < n16; q += NT) d[q] = __ldg(s + q);
}

}  // namespace pgx
