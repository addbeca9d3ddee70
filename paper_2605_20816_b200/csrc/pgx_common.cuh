// pgx_common.cuh — device helpers shared by every pgx kernel.
//
// Coordinates and basis features are regenerated on the device with the same
// IEEE operation sequence as the reference (no FMA contraction), so eta(x) is
// bit-identical to basis.DesignBasis.evaluate (basis.py:105-142) on the grid
// of geometry.make_grid (geometry.py:59-71).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pgx {

constexpr int kMaxDim = 3;
constexpr int kMaxDegree2 = 10;  // 2-D: K <= 66
constexpr int kMaxDegree3 = 4;   // 3-D: K <= 35
constexpr int kMaxK = 66;
constexpr double kTieRtol = 1e-12;  // geometry.py:19

__host__ __device__ constexpr int binom(int n, int k) {
  return k == 0 ? 1 : (n * binom(n - 1, k - 1)) / k;
}
__host__ __device__ constexpr int feature_count(int dim, int degree) {
  return binom(degree + dim, dim);
}

// Multi-index table: alpha[k][j] = exponent of axis j in feature k
// (graded-lex, a1 descending: basis.py:42-48; 3-D: Appendix B of SURVEY.md).
struct AlphaTable {
  int8_t a[kMaxK][3];
};

// Pixel-centre coordinate of 0-based index k on a (2M) axis: -1 + (k+1 - 1/2)/M
// (geometry.py:68), evaluated without contraction.
// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in the
// stream is still running; griddep_wait() blocks until that predecessor has
// completed and its writes are visible. Every kernel launched that way calls
// it before its first global access that depends on (or is read by) the
// predecessor; without the attribute it returns at once.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// lets the dependent grid be scheduled before this grid exits
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ double axis_coord(int64_t k, int m) {
  return __dadd_rn(-1.0, __ddiv_rn(__dsub_rn((double)(k + 1), 0.5), (double)m));
}

// Coordinates of point p: regular grid (row-major, first axis slowest,
// geometry.py:69-70) or an unstructured point list.
template <int DIM>
__device__ __forceinline__ void point_coords(int64_t p, int m, const double* __restrict__ pts,
                                             double x[DIM]) {
  if (m > 0) {
    const int64_t side = 2 * (int64_t)m;
    if (DIM == 2) {
      x[0] = axis_coord(p / side, m);
      x[1] = axis_coord(p % side, m);
    } else {
      x[0] = axis_coord(p / (side * side), m);
      x[1] = axis_coord((p / side) % side, m);
      x[DIM - 1] = axis_coord(p % side, m);
    }
  } else {
#pragma unroll
    for (int j = 0; j < DIM; ++j) x[j] = pts[p * DIM + j];
  }
}

// u[0..D] of one axis: Legendre three-term recurrence (basis.py:128-142) or
// powers (basis.py:120-125), in the reference's exact operation order.
template <int D>
__device__ __forceinline__ void axis_table(double t, bool legendre, double u[D + 1]) {
  u[0] = 1.0;
  if (D >= 1) u[1] = t;
  if (legendre) {
#pragma unroll
    for (int m = 1; m < D; ++m) {
      double a = __dmul_rn(__dmul_rn((double)(2 * m + 1), t), u[m]);
      double b = __dmul_rn((double)m, u[m - 1]);
      u[m + 1] = __ddiv_rn(__dsub_rn(a, b), (double)(m + 1));
    }
  } else {
#pragma unroll
    for (int m = 1; m < D; ++m) u[m + 1] = __dmul_rn(u[m], t);
  }
}

// Full feature vector eta(x), K = C(D+DIM, DIM) entries in graded-lex order.
template <int DIM, int D>
__device__ __forceinline__ void features(const double x[DIM], bool legendre,
                                         double eta[feature_count(DIM, D)]) {
  double u0[D + 1], u1[D + 1];
  axis_table<D>(x[0], legendre, u0);
  axis_table<D>(x[1], legendre, u1);
  if (DIM == 2) {
    int k = 0;
#pragma unroll
    for (int tot = 0; tot <= D; ++tot) {
#pragma unroll
      for (int a1 = tot; a1 >= 0; --a1) eta[k++] = __dmul_rn(u0[a1], u1[tot - a1]);
    }
  } else {
    double u2[D + 1];
    axis_table<D>(x[DIM - 1], legendre, u2);
    int k = 0;
#pragma unroll
    for (int tot = 0; tot <= D; ++tot) {
#pragma unroll
      for (int a1 = tot; a1 >= 0; --a1) {
#pragma unroll
        for (int a2 = tot - a1; a2 >= 0; --a2)
          eta[k++] = __dmul_rn(__dmul_rn(u0[a1], u1[a2]), u2[tot - a1 - a2]);
      }
    }
  }
}

__device__ __forceinline__ double tie_threshold(double m) {
  // geometry.py:208-210, m + TIE_RTOL * (1 + |m|) without contraction
  return __dadd_rn(m, __dmul_rn(kTieRtol, __dadd_rn(1.0, fabs(m))));
}

}  // namespace pgx
