// pgx_design.cuh — the hot path on an explicit (K, P) design matrix: the
// reference's evaluate_objective(theta_values, design_values, labels0, eps)
// form (objective.py:129-165), where the features eta(x) are given as a
// matrix instead of a grid + basis (any K, any features).  Same arithmetic as
// the general exact path (pgx_general.cuh): fp64 logits, fp64 exp/log, the
// tie-tolerant arg-min of geometry.py:201-210, fixed-order partials; the
// design columns are read coalesced (point p of a CTA-wide run at
// design[k P + p]).  K is a runtime value <= KB (the template bucket).
#pragma once

#include "pgx_general.cuh"

namespace pgx {

// feature vector of point p from the design matrix (zeros beyond K)
template <int KB>
__device__ __forceinline__ void design_eta(const double* __restrict__ dsg, int64_t P, int K, int64_t p,
                                           double (&eta)[KB]) {
#pragma unroll
  for (int k = 0; k < KB; ++k) eta[k] = k < K ? __ldg(dsg + (int64_t)k * P + p) : 0.0;
}

// pass 1: logits, online min / log-sum-exp, arg-min and the per-point
// scratch, exactly as k_general_pass1; a point whose 2-entry candidate list
// overflowed is re-scanned here (no fix-up queue: the tail has no features)
template <int KB, bool EVAL>
__global__ void __launch_bounds__(kP1Threads) k_design_pass1(EvalParams prm, const double* __restrict__ dsg,
                                                             int K) {
  __shared__ double th_s[KB][kP1Chunk];
  __shared__ double red_d[kP1Threads];
  __shared__ long long red_i[kP1Threads];
  const int tid = threadIdx.x;
  const int64_t p = (int64_t)blockIdx.x * kP1Threads + tid;
  const bool active = p < prm.P;
  const int N = prm.N;
  double eta[KB];
  int g = -1;
  if (active) {
    design_eta<KB>(dsg, prm.P, K, p, eta);
    if (prm.labels) g = prm.labels[p];
  } else {
#pragma unroll
    for (int k = 0; k < KB; ++k) eta[k] = 0.0;
  }
  ScanState st;
  st.init();
  double thr = CUDART_INF;
  for (int c0 = 0; c0 < N; c0 += kP1Chunk) {
    const int cn = min(kP1Chunk, N - c0);
    __syncthreads();
    for (int idx = tid; idx < KB * kP1Chunk; idx += kP1Threads) {
      const int k = idx / kP1Chunk, j = idx % kP1Chunk;
      th_s[k][j] = (j < cn && k < K) ? prm.theta[(int64_t)k * N + c0 + j] : 0.0;
    }
    __syncthreads();
    if (active) {
      for (int j = 0; j < cn; ++j) {
        double h = 0.0;
#pragma unroll
        for (int k = 0; k < KB; ++k)
          if (k < K) h = fma(th_s[k][j], eta[k], h);
        const int i = c0 + j;
        if (i == g) st.hG = h;
        scan_update<EVAL>(st, thr, i, h, prm.eps);
      }
    }
  }
  double ell = 0.0, e0 = 0.0;
  long long correct = 0, amb = 0, nonfinite = 0;
  if (active) {
    const double margin = st.m2 - st.m1;
    amb = (margin <= prm.tau_amb * (1.0 + fabs(st.m1))) ? 1 : 0;
    if (st.cnt == 0 || st.needfix) {  // exact re-scan: smallest index within the tie tolerance
      const double t2 = tie_threshold(st.m1);
      int best = -1;
      for (int i = 0; i < N && best < 0; ++i) {
        double h = 0.0;
        for (int k = 0; k < K; ++k) h = fma(prm.theta[(int64_t)k * N + i], eta[k], h);
        if (h <= t2) best = i;
      }
      st.b0 = best < 0 ? 0 : best;
    }
    prm.pix_m[p] = st.m1;
    if (EVAL) {
      const double ls = log(st.s);
      prm.pix_ls[p] = ls;
      ell = (st.m1 - st.hG) / prm.eps - ls;  // objective.py:103,106
      e0 = st.hG - st.m1;                    // objective.py:119
      if (!isfinite(ell)) nonfinite = 1;
    }
    correct = (st.b0 == g) ? 1 : 0;
    if (prm.labels_out) prm.labels_out[p] = st.b0 + 1;
    if (prm.margin_out) prm.margin_out[p] = (float)margin;
  }
  const double s_ell = block_sum<kP1Threads>(ell, red_d);
  const double s_e0 = block_sum<kP1Threads>(e0, red_d);
  const long long s_cor = block_sum<kP1Threads>(correct, red_i);
  const long long s_amb = block_sum<kP1Threads>(amb, red_i);
  const long long s_nf = block_sum<kP1Threads>(nonfinite, red_i);
  if (tid == 0) {
    prm.part_d[2 * blockIdx.x + 0] = s_ell;
    prm.part_d[2 * blockIdx.x + 1] = s_e0;
    prm.part_i[4 * blockIdx.x + 0] = s_cor;
    prm.part_i[4 * blockIdx.x + 1] = s_amb;
    prm.part_i[4 * blockIdx.x + 2] = s_nf;
    prm.part_i[4 * blockIdx.x + 3] = 0;
  }
}

// pass 2: grain-major gradient over point splits (objective.py:109-113)
template <int KB>
__global__ void __launch_bounds__(kP2Threads) k_design_pass2(EvalParams prm, const double* __restrict__ dsg,
                                                             int K) {
  __shared__ double eta_s[KB][kP2Chunk];
  __shared__ double m_s[kP2Chunk], ls_s[kP2Chunk];
  __shared__ int lab_s[kP2Chunk];
  const int tid = threadIdx.x;
  const int N = prm.N;
  const int i = blockIdx.x * kP2Threads + tid;
  const bool active = i < N;
  const int y = blockIdx.y;
  const int64_t pb = prm.P * y / prm.splits;
  const int64_t pe = prm.P * (y + 1) / prm.splits;
  double th[KB], acc[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    th[k] = (active && k < K) ? prm.theta[(int64_t)k * N + i] : 0.0;
    acc[k] = 0.0;
  }
  for (int64_t p0 = pb; p0 < pe; p0 += kP2Chunk) {
    const int cn = (int)min((int64_t)kP2Chunk, pe - p0);
    __syncthreads();
    for (int idx = tid; idx < KB * kP2Chunk; idx += kP2Threads) {
      const int k = idx / kP2Chunk, j = idx % kP2Chunk;
      eta_s[k][j] = (j < cn && k < K) ? __ldg(dsg + (int64_t)k * prm.P + p0 + j) : 0.0;
    }
    if (tid < cn) {
      m_s[tid] = prm.pix_m[p0 + tid];
      ls_s[tid] = prm.pix_ls[p0 + tid];
      lab_s[tid] = prm.labels[p0 + tid];
    }
    __syncthreads();
    if (active) {
      for (int j = 0; j < cn; ++j) {
        double h = 0.0;
#pragma unroll
        for (int k = 0; k < KB; ++k)
          if (k < K) h = fma(th[k], eta_s[k][j], h);
        const double e = exp((m_s[j] - h) / prm.eps - ls_s[j]);
        const double r = (lab_s[j] == i) ? 1.0 - e : -e;  // objective.py:110-112
#pragma unroll
        for (int k = 0; k < KB; ++k) acc[k] = fma(r, eta_s[k][j], acc[k]);
      }
    }
  }
  if (active) {
#pragma unroll
    for (int k = 0; k < KB; ++k)
      if (k < K) prm.part_g[((int64_t)y * K + k) * N + i] = acc[k];
  }
}

// dense soft assignment (objective.py:80-87): p[i][x] = exp((m - h_i)/eps) / sum,
// for small problems; one thread per point, features from the grid or the design
template <int KB>
__global__ void __launch_bounds__(128) k_design_soft(EvalParams prm, const double* __restrict__ dsg, int K,
                                                     double* __restrict__ prob) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= prm.P) return;
  double eta[KB];
  design_eta<KB>(dsg, prm.P, K, p, eta);
  const int N = prm.N;
  auto logit = [&](int i) {
    double h = 0.0;
#pragma unroll
    for (int k = 0; k < KB; ++k)
      if (k < K) h = fma(prm.theta[(int64_t)k * N + i], eta[k], h);
    return h;
  };
  double m = CUDART_INF;
  for (int i = 0; i < N; ++i) m = fmin(m, logit(i));
  double s = 0.0;
  for (int i = 0; i < N; ++i) s += exp((m - logit(i)) / prm.eps);
  for (int i = 0; i < N; ++i) prob[(int64_t)i * prm.P + p] = exp((m - logit(i)) / prm.eps) / s;
}

}  // namespace pgx

namespace pgx {

// the same dense soft assignment with features from the grid / point list
template <int DIM, int D>
__global__ void __launch_bounds__(128) k_general_soft(EvalParams prm, double* __restrict__ prob) {
  constexpr int K = feature_count(DIM, D);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= prm.P) return;
  double x[DIM], eta[K];
  point_coords<DIM>(p, prm.M, prm.pts, x);
  features<DIM, D>(x, prm.legendre != 0, eta);
  const int N = prm.N;
  auto logit = [&](int i) {
    double h = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) h = fma(prm.theta[(int64_t)k * N + i], eta[k], h);
    return h;
  };
  double m = CUDART_INF;
  for (int i = 0; i < N; ++i) m = fmin(m, logit(i));
  double s = 0.0;
  for (int i = 0; i < N; ++i) s += exp((m - logit(i)) / prm.eps);
  for (int i = 0; i < N; ++i) prob[(int64_t)i * prm.P + p] = exp((m - logit(i)) / prm.eps) / s;
}

}  // namespace pgx
