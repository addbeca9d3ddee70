// k_lbfgs.cu — device-resident optimiser state for the fit's host loop
// (the reference's L-BFGS two-loop recursion and Wolfe
// line search, optimizer.py:248-318, keep their decisions on the host and see
// only scalars).  The vectors -- the free parameters u = theta[:, :N-1], the
// gradient, the search direction and the (s, y) history -- never leave the GPU:
//   k_lb_point      u_t = u + t d, scattered into the K x N theta the kernels read
//   k_lb_after      packs the gradient of the free columns, g_t . d and |g_t|^2
//   k_lb_two_loop   the whole two-loop recursion in ONE single-CTA kernel
//                   (2 m + 2 dot products and axpys without a launch each)
//   k_lb_accept     s = u_t - u, y = g - g_t, curvature test, history push
// All reductions are single-CTA, fixed-order (deterministic trajectories).
// pgx_api.cu captures point -> pgx_eval kernels -> after into one CUDA graph,
// so a line-search trial is one graph launch and one synchronisation.
#include <cuda_runtime.h>

#include <cstdint>

#include "pgx_launch.cuh"

namespace pgx {

constexpr int kLbThreads = 1024;

// fixed-order block sum of one double per thread (all threads get the result)
__device__ __forceinline__ double lb_block_sum(double v, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();  // (red may still be read from the previous call)
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kLbThreads / 32; ++w) s += red[w];
  return s;
}

__device__ __forceinline__ double lb_dot(const double* a, const double* b, int64_t n, double* red) {
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kLbThreads) acc = fma(a[i], b[i], acc);
  return lb_block_sum(acc, red);
}

// theta[k][i] = u[k (N-1) + i] + t d[...] for i < N-1 (the last column stays 0: gauge)
__global__ void k_lb_point(double* __restrict__ theta, double* __restrict__ ut, const double* __restrict__ u,
                           const double* __restrict__ d, const double* t_ptr, int K, int N) {
  const double t = *t_ptr;  // (mapped pinned host memory: the host writes t, then launches the graph)
  const int64_t n = (int64_t)K * (N - 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double v = d ? fma(t, d[e], u[e]) : u[e];
    ut[e] = v;
    theta[(e / (N - 1)) * N + e % (N - 1)] = v;
  }
}

// gt = grad[:, :N-1]; out[0] = gt . d (0 without d), out[1] = |gt|^2
__global__ void __launch_bounds__(kLbThreads) k_lb_after(const double* __restrict__ grad, double* __restrict__ gt,
                                                         const double* __restrict__ d, double* out, int K, int N) {
  __shared__ double red[kLbThreads / 32];
  const int64_t n = (int64_t)K * (N - 1);
  double sd = 0.0, sg = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += kLbThreads) {
    const double v = grad[(e / (N - 1)) * N + e % (N - 1)];
    gt[e] = v;
    if (d) sd = fma(v, d[e], sd);
    sg = fma(v, v, sg);
  }
  sd = lb_block_sum(sd, red);
  sg = lb_block_sum(sg, red);
  if (threadIdx.x == 0) {
    out[0] = sd;
    out[1] = sg;
  }
}

// state[0] = next ring slot (head), state[1] = pairs held (<= m); ring of m + 1 rows
// mode 0: two-loop (steepest ascent scaled by 1/|g|^2 without history); 1: g / |g|^2; 2: g
__global__ void __launch_bounds__(kLbThreads) k_lb_two_loop(const double* __restrict__ g, double* __restrict__ d,
                                                            const double* __restrict__ S, const double* __restrict__ Y,
                                                            const double* __restrict__ rho, double* alpha,
                                                            const int* state, int m, int64_t n, int mode,
                                                            double* out) {
  __shared__ double red[kLbThreads / 32];
  const int tid = threadIdx.x;
  const int head = state[0], cnt = mode == 0 ? state[1] : 0;
  const int ring = m + 1;
  const double gg = lb_dot(g, g, n, red);
  if (cnt == 0) {
    const double sc = mode == 2 ? 1.0 : 1.0 / gg;
    for (int64_t i = tid; i < n; i += kLbThreads) d[i] = g[i] * sc;
  } else {
    for (int64_t i = tid; i < n; i += kLbThreads) d[i] = g[i];  // q
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {  // newest -> oldest (optimizer.py:256-260)
      const int slot = (head - 1 - j + 2 * ring) % ring;
      const double a = rho[slot] * lb_dot(S + slot * n, d, n, red);
      if (tid == 0) alpha[j] = a;
      const double* y = Y + slot * n;
      for (int64_t i = tid; i < n; i += kLbThreads) d[i] = fma(-a, y[i], d[i]);
      __syncthreads();
    }
    const int newest = (head - 1 + ring) % ring;
    const double sy = lb_dot(S + newest * n, Y + newest * n, n, red);
    const double yy = lb_dot(Y + newest * n, Y + newest * n, n, red);
    const double gamma = sy / yy;  // optimizer.py:261
    for (int64_t i = tid; i < n; i += kLbThreads) d[i] *= gamma;
    __syncthreads();
    for (int j = cnt - 1; j >= 0; --j) {  // oldest -> newest (optimizer.py:262-264)
      const int slot = (head - 1 - j + 2 * ring) % ring;
      const double b = rho[slot] * lb_dot(Y + slot * n, d, n, red);
      const double coef = alpha[j] - b;
      const double* s = S + slot * n;
      for (int64_t i = tid; i < n; i += kLbThreads) d[i] = fma(coef, s[i], d[i]);
      __syncthreads();
    }
  }
  __syncthreads();
  const double slope = lb_dot(g, d, n, red);
  const double dd = lb_dot(d, d, n, red);
  if (tid == 0) {
    out[0] = slope;
    out[1] = dd;
    out[2] = gg;
    out[3] = (double)cnt;
  }
}

// s = ut - u, y = g - gt into the free ring row; pushed when
// s.y > skip sqrt(s.s) sqrt(y.y) (optimizer.py:303-309); then u <- ut, g <- gt
__global__ void __launch_bounds__(kLbThreads) k_lb_accept(double* __restrict__ u, double* __restrict__ g,
                                                          const double* __restrict__ ut, const double* __restrict__ gt,
                                                          double* __restrict__ S, double* __restrict__ Y, double* rho,
                                                          int* state, int m, int64_t n, double skip, int keep_pair,
                                                          double* out) {
  __shared__ double red[kLbThreads / 32];
  const int tid = threadIdx.x;
  const int head = state[0], cnt = state[1];
  double* s = S + head * n;
  double* y = Y + head * n;
  double sy = 0.0, ss = 0.0, yy = 0.0, gg = 0.0, uu = 0.0;
  for (int64_t i = tid; i < n; i += kLbThreads) {
    const double sv = ut[i] - u[i], yv = g[i] - gt[i];
    s[i] = sv;
    y[i] = yv;
    sy = fma(sv, yv, sy);
    ss = fma(sv, sv, ss);
    yy = fma(yv, yv, yy);
    gg = fma(gt[i], gt[i], gg);
    uu = fma(ut[i], ut[i], uu);
    u[i] = ut[i];
    g[i] = gt[i];
  }
  sy = lb_block_sum(sy, red);
  ss = lb_block_sum(ss, red);
  yy = lb_block_sum(yy, red);
  gg = lb_block_sum(gg, red);
  uu = lb_block_sum(uu, red);
  const bool push = keep_pair && sy > skip * sqrt(ss) * sqrt(yy);
  if (tid == 0) {
    if (push) {
      rho[head] = 1.0 / sy;
      state[0] = (head + 1) % (m + 1);
      state[1] = cnt < m ? cnt + 1 : m;
    }
    out[0] = gg;
    out[1] = push ? 1.0 : 0.0;
    out[2] = uu;
    out[3] = sy;
  }
}

void launch_lb_point(double* theta, double* ut, const double* u, const double* d, const double* t_ptr, int K,
                     int N, int sms, cudaStream_t s) {
  const int64_t n = (int64_t)K * (N - 1);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4 * sms);
  k_lb_point<<<blocks, 256, 0, s>>>(theta, ut, u, d, t_ptr, K, N);
}
void launch_lb_after(const double* grad, double* gt, const double* d, double* out, int K, int N,
                     cudaStream_t s) {
  k_lb_after<<<1, kLbThreads, 0, s>>>(grad, gt, d, out, K, N);
}
void launch_lb_two_loop(const double* g, double* d, const double* S, const double* Y, const double* rho,
                        double* alpha, const int* state, int m, int64_t n, int mode, double* out,
                        cudaStream_t s) {
  k_lb_two_loop<<<1, kLbThreads, 0, s>>>(g, d, S, Y, rho, alpha, state, m, n, mode, out);
}
void launch_lb_accept(double* u, double* g, const double* ut, const double* gt, double* S, double* Y,
                      double* rho, int* state, int m, int64_t n, double skip, int keep_pair, double* out,
                      cudaStream_t s) {
  k_lb_accept<<<1, kLbThreads, 0, s>>>(u, g, ut, gt, S, Y, rho, state, m, n, skip, keep_pair, out);
}

}  // namespace pgx
