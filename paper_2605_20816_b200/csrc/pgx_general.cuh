// pgx_general.cuh — the general fp64 CUDA-core path (any point list, any
// supported basis/degree).  It is the reference-faithful restatement of
// objective._chunk_stats (objective.py:97-120) on the device:
//
//   pass 1  (pixel-major, one thread per point): eta(x) in registers, theta
//           staged through shared memory in grain chunks; fp64 logits
//           h_i = theta_i . eta(x); online min / log-sum-exp over grains
//           (objective.py:99-106); tie-tolerant arg-min (geometry.py:201-210)
//           with a 2-entry candidate list and an exact re-scan fallback;
//           per-point (min, log s) scratch for pass 2; fixed-order per-block
//           partials of sum(ell), sum(e0), #correct, #ambiguous, #non-finite.
//   pass 2  (grain-major, split over points): recomputes h, p = exp(z - log s),
//           r = onehot - p and accumulates dtheta_i += r eta(x)
//           (objective.py:109-113) into per-split partials.
//   reduce  fixed-order fp64 reductions (objective.py:123-126,155-165).
//
// The regular-grid fast path (pgx_grid.cuh) and the tensor-core path reuse
// pass-2's contract and the reduce kernels.
#pragma once

#include <math_constants.h>

#include "../../include/pgx.h"
#include "pgx_common.cuh"

namespace pgx {

struct EvalParams {
  int64_t P;
  int N;
  int M;          // grid resolution (0 = unstructured)
  int legendre;   // basis kind
  const double* __restrict__ pts;
  const int32_t* __restrict__ labels;
  const double* __restrict__ theta;  // K x N fp64
  const float* __restrict__ theta32;  // tc grid path: fp32 source converted by k_tc_coeffs
  double eps;
  double inv_eps;
  double tau_amb;
  // per-point scratch
  double* pix_m;
  double* pix_ls;
  // pass-1 per-block partials
  double* part_d;      // [blocks][2]: sum ell, sum e0
  long long* part_i;   // [blocks][4]: correct, ambiguous, nonfinite, (unused)
  int* fix_count;
  int* fix_list;
  long long* fix_correct;  // correct pixels discovered by the fix-up re-scan
  // assign outputs (nullable)
  long long* labels_out;
  float* margin_out;
  // pass 2
  int splits;
  double* part_g;  // [splits][K][N]
};

constexpr int kP1Threads = 128;
constexpr int kP1Chunk = 64;
constexpr int kP2Threads = 128;
constexpr int kP2Chunk = 32;

// Per-point running state of the grain scan.
struct ScanState {
  double m1, m2, s, hG, hb0, hb1;
  int b0, b1, cnt;
  bool dirty, needfix;
  __device__ __forceinline__ void init() {
    m1 = CUDART_INF;
    m2 = CUDART_INF;
    s = 0.0;
    hG = 0.0;
    hb0 = hb1 = 0.0;
    b0 = b1 = -1;
    cnt = 0;
    dirty = needfix = false;
  }
};

// One logit h of grain i.  LSE: online log-sum-exp in fp64 with exact exp.
// The common case (h above the running tie threshold) only touches s and m2.
template <bool LSE>
__device__ __forceinline__ void scan_update(ScanState& st, double& thr, int i, double h,
                                            double eps) {
  if (h <= thr) {
    if (h < st.m1) {
      if (LSE) st.s = st.s * exp((h - st.m1) / eps) + 1.0;
      st.m2 = st.m1;
      st.m1 = h;
      thr = tie_threshold(h);
      // prune candidates that no longer lie within the tie tolerance
      if (st.cnt > 0 && !(st.hb0 <= thr)) {
        if (st.dirty) st.needfix = true;
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
    } else {
      if (LSE) st.s += exp((st.m1 - h) / eps);
      if (h < st.m2) st.m2 = h;
    }
    // h qualifies as a (tie-tolerant) minimiser; keep the two smallest indices
    if (st.cnt == 0) {
      st.b0 = i;
      st.hb0 = h;
      st.cnt = 1;
    } else if (st.cnt == 1) {
      st.b1 = i;
      st.hb1 = h;
      st.cnt = 2;
    } else {
      st.dirty = true;
    }
  } else {
    if (LSE) st.s += exp((st.m1 - h) / eps);
    if (h < st.m2) st.m2 = h;
  }
}

// Fixed-order block reduction (deterministic): tree over kThreads entries.
template <int kThreads, typename T>
__device__ __forceinline__ T block_sum(T v, T* buf) {
  const int tid = threadIdx.x;
  buf[tid] = v;
  __syncthreads();
#pragma unroll
  for (int off = kThreads / 2; off > 0; off >>= 1) {
    if (tid < off) buf[tid] = buf[tid] + buf[tid + off];
    __syncthreads();
  }
  T r = buf[0];
  __syncthreads();
  return r;
}

// Fixed-order block reduction of three fp64 and three integer partials with
// one barrier: warp shuffle trees, then warp 0 folds the per-warp sums in
// warp order (deterministic).  Result valid in thread 0.
template <int kThreads>
__device__ __forceinline__ void block_sum6(double& a, double& b, double& c, long long& x, long long& y,
                                           long long& z) {
  __shared__ double sd[kThreads / 32][3];
  __shared__ long long si[kThreads / 32][3];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
    c += __shfl_xor_sync(0xffffffffu, c, off);
    x += __shfl_xor_sync(0xffffffffu, x, off);
    y += __shfl_xor_sync(0xffffffffu, y, off);
    z += __shfl_xor_sync(0xffffffffu, z, off);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sd[w][0] = a;
    sd[w][1] = b;
    sd[w][2] = c;
    si[w][0] = x;
    si[w][1] = y;
    si[w][2] = z;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = b = c = 0.0;
    x = y = z = 0;
#pragma unroll
    for (int v = 0; v < kThreads / 32; ++v) {
      a += sd[v][0];
      b += sd[v][1];
      c += sd[v][2];
      x += si[v][0];
      y += si[v][1];
      z += si[v][2];
    }
  }
}

// ---------------------------------------------------------------- pass 1
template <int DIM, int D, bool EVAL>
__global__ void __launch_bounds__(kP1Threads) k_general_pass1(EvalParams prm) {
  constexpr int K = feature_count(DIM, D);
  __shared__ double th_s[K][kP1Chunk];
  __shared__ double red_d[kP1Threads];
  __shared__ long long red_i[kP1Threads];

  const int tid = threadIdx.x;
  const int64_t p = (int64_t)blockIdx.x * kP1Threads + tid;
  const bool active = p < prm.P;
  const int N = prm.N;

  double eta[K];
  int g = -1;
  if (active) {
    double x[DIM];
    point_coords<DIM>(p, prm.M, prm.pts, x);
    features<DIM, D>(x, prm.legendre != 0, eta);
    if (prm.labels) g = prm.labels[p];
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) eta[k] = 0.0;
  }

  ScanState st;
  st.init();
  double thr = CUDART_INF;
  for (int c0 = 0; c0 < N; c0 += kP1Chunk) {
    const int cn = min(kP1Chunk, N - c0);
    __syncthreads();
    for (int idx = tid; idx < K * kP1Chunk; idx += kP1Threads) {
      const int k = idx / kP1Chunk, j = idx % kP1Chunk;
      th_s[k][j] = (j < cn) ? prm.theta[(int64_t)k * N + c0 + j] : 0.0;
    }
    __syncthreads();
    if (active) {
      for (int j = 0; j < cn; ++j) {
        double h = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) h = fma(th_s[k][j], eta[k], h);
        const int i = c0 + j;
        if (i == g) st.hG = h;
        scan_update<EVAL>(st, thr, i, h, prm.eps);
      }
    }
  }

  double ell = 0.0, e0 = 0.0;
  long long correct = 0, amb = 0, nonfinite = 0;
  if (active) {
    if (st.cnt == 0) st.needfix = true;
    const double margin = st.m2 - st.m1;
    amb = (margin <= prm.tau_amb * (1.0 + fabs(st.m1))) ? 1 : 0;
    prm.pix_m[p] = st.m1;
    if (EVAL) {
      const double ls = log(st.s);
      prm.pix_ls[p] = ls;
      ell = (st.m1 - st.hG) / prm.eps - ls;  // objective.py:103,106
      e0 = st.hG - st.m1;                    // objective.py:119
      if (!isfinite(ell)) nonfinite = 1;
    }
    if (st.needfix) {
      const int slot = atomicAdd(prm.fix_count, 1);
      prm.fix_list[slot] = (int)p;
    } else {
      correct = (st.b0 == g) ? 1 : 0;
      if (prm.labels_out) prm.labels_out[p] = st.b0 + 1;
    }
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

// Exact arg-min for the (rare) points whose candidate list overflowed:
// smallest index with h <= min + tol (geometry.py:208-210).  h is recomputed
// with the same fma order as pass 1, so it is bit-identical.
template <int DIM, int D>
__global__ void __launch_bounds__(128) k_general_fixup(EvalParams prm) {
  constexpr int K = feature_count(DIM, D);
  const int count = *prm.fix_count;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
    const int64_t p = prm.fix_list[t];
    double x[DIM], eta[K];
    point_coords<DIM>(p, prm.M, prm.pts, x);
    features<DIM, D>(x, prm.legendre != 0, eta);
    const double thr = tie_threshold(prm.pix_m[p]);
    int best = -1;
    for (int i = 0; i < prm.N && best < 0; ++i) {
      double h = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) h = fma(prm.theta[(int64_t)k * prm.N + i], eta[k], h);
      if (h <= thr) best = i;
    }
    if (prm.labels_out) prm.labels_out[p] = best + 1;
    if (prm.labels && best == prm.labels[p]) atomicAdd((unsigned long long*)prm.fix_correct, 1ull);
  }
}

// ---------------------------------------------------------------- pass 2
template <int DIM, int D>
__global__ void __launch_bounds__(kP2Threads) k_general_pass2(EvalParams prm) {
  constexpr int K = feature_count(DIM, D);
  __shared__ double eta_s[K][kP2Chunk];
  __shared__ double m_s[kP2Chunk], ls_s[kP2Chunk];
  __shared__ int lab_s[kP2Chunk];

  const int tid = threadIdx.x;
  const int N = prm.N;
  const int i = blockIdx.x * kP2Threads + tid;
  const bool active = i < N;
  const int y = blockIdx.y;
  const int64_t pb = prm.P * y / prm.splits;
  const int64_t pe = prm.P * (y + 1) / prm.splits;

  double th[K], acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    th[k] = active ? prm.theta[(int64_t)k * N + i] : 0.0;
    acc[k] = 0.0;
  }
  for (int64_t p0 = pb; p0 < pe; p0 += kP2Chunk) {
    const int cn = (int)min((int64_t)kP2Chunk, pe - p0);
    __syncthreads();
    if (tid < cn) {
      const int64_t p = p0 + tid;
      double x[DIM], eta[K];
      point_coords<DIM>(p, prm.M, prm.pts, x);
      features<DIM, D>(x, prm.legendre != 0, eta);
#pragma unroll
      for (int k = 0; k < K; ++k) eta_s[k][tid] = eta[k];
      m_s[tid] = prm.pix_m[p];
      ls_s[tid] = prm.pix_ls[p];
      lab_s[tid] = prm.labels[p];
    }
    __syncthreads();
    if (active) {
      for (int j = 0; j < cn; ++j) {
        double h = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) h = fma(th[k], eta_s[k][j], h);
        const double e = exp((m_s[j] - h) / prm.eps - ls_s[j]);
        const double r = (lab_s[j] == i) ? 1.0 - e : -e;  // objective.py:110-112
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = fma(r, eta_s[k][j], acc[k]);
      }
    }
  }
  if (active) {
#pragma unroll
    for (int k = 0; k < K; ++k) prm.part_g[((int64_t)y * K + k) * N + i] = acc[k];
  }
}

// ---------------------------------------------------------------- reductions
struct ReduceParams {
  int K, N, splits;
  int64_t P;
  double eps, lambda;
  const double* theta;
  const double* part_g;
  double* grad_out;
  int* nonfinite;  // counter
};

// grad = -(sum over splits, fixed order) / (eps P) - lambda theta (free columns)
static __global__ void __launch_bounds__(256) k_reduce_grad(ReduceParams prm) {
  const int64_t KN = (int64_t)prm.K * prm.N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < KN;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < prm.splits; ++s) acc += prm.part_g[s * KN + e];
    double g = -acc / (prm.eps * (double)prm.P);  // objective.py:162
    const int i = (int)(e % prm.N);
    if (prm.lambda != 0.0 && i < prm.N - 1) g -= prm.lambda * prm.theta[e];
    if (!isfinite(g)) atomicAdd(prm.nonfinite, 1);
    prm.grad_out[e] = g;
  }
}

struct FinalParams {
  int blocks1;
  int K, N;
  int64_t P;
  double eps, lambda;
  int want_assign;
  const double* theta;
  const double* part_d;
  const long long* part_i;
  const long long* fix_correct;
  const int* nonfinite_grad;
  void* stats_out;  // pgx_stats layout
};

struct StatsDev {
  double phi, err, e0, n_rescanned;
  long long n_points, n_correct, n_ambiguous, n_nonfinite, flags;
};

static __global__ void __launch_bounds__(256) k_finalize(FinalParams prm) {
  const int tid = threadIdx.x;
  // fixed contiguous partition of the pass-1 partials per thread
  const int per = (prm.blocks1 + 255) / 256;
  const int b0 = tid * per, b1 = min(prm.blocks1, b0 + per);
  double ell = 0.0, e0 = 0.0;
  long long cor = 0, amb = 0, nf = 0;
  for (int b = b0; b < b1; ++b) {
    ell += prm.part_d[2 * b + 0];
    e0 += prm.part_d[2 * b + 1];
    cor += prm.part_i[4 * b + 0];
    amb += prm.part_i[4 * b + 1];
    nf += prm.part_i[4 * b + 2];
  }
  double th2 = 0.0;
  if (prm.lambda != 0.0) {
    const int64_t KN = (int64_t)prm.K * prm.N;
    const int64_t per2 = (KN + 255) / 256;
    for (int64_t e = tid * per2; e < min(KN, (tid + 1) * per2); ++e)
      if (e % prm.N < prm.N - 1) th2 += prm.theta[e] * prm.theta[e];
  }
  block_sum6<256>(ell, e0, th2, cor, amb, nf);
  if (tid == 0) {
    StatsDev* out = reinterpret_cast<StatsDev*>(prm.stats_out);
    const double P = (double)prm.P;
    cor += *prm.fix_correct;
    nf += prm.nonfinite_grad ? *prm.nonfinite_grad : 0;
    double phi = ell / P;  // objective.py:161
    if (prm.lambda != 0.0) phi -= 0.5 * prm.lambda * th2;
    out->phi = phi;
    out->err = prm.want_assign ? 1.0 - (double)cor / P : 0.0;  // objective.py:163
    out->e0 = prm.want_assign ? e0 / P : 0.0;                  // objective.py:164
    out->n_rescanned = 0.0;
    out->n_points = prm.P;
    out->n_correct = cor;
    out->n_ambiguous = amb;
    out->n_nonfinite = nf + (isfinite(phi) ? 0 : 1);
    out->flags = 0;
  }
}

// ---------------------------------------------------------------- fused tail
// One launch after the passes: (1) exact arg-min re-scan of the flagged points
// (grid-stride, rare), (2) fixed-order reduction of the per-split gradient
// partials — 32 entries per CTA, 8 warps over interleaved splits, then a
// fixed smem tree — with the -1/(eps P) scaling and the lambda term, (3) the
// last CTA to finish (atomic ticket) reduces the pass-1 partials into the
// scalars.  Every sum has a fixed order, so results are bit-reproducible.
struct TailParams {
  ReduceParams red;
  FinalParams fin;
  int want_grad;
  int fix_amb;  // the re-scan decides the ambiguity of queued points (grid path)
  unsigned* ticket;
  double* part_th2;  // [gridDim.x] per-CTA partials of ||theta[:, :N-1]||^2
  // fast modes: c = log2(e) / eps (0 = no check); the largest column L1 norm
  // of theta (fp32 bits, atomicMax: order-independent) times c beyond
  // PGX_FAST_RANGE sets PGX_STAT_RANGE
  double range_c;
  unsigned* range_bits;
};

constexpr int kTailThreads = 256;

template <int DIM, int D>
__global__ void __launch_bounds__(kTailThreads) k_tail(EvalParams e, TailParams t) {
  constexpr int K = feature_count(DIM, D);
  __shared__ double sred[8][33];
  __shared__ bool last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  griddep_wait();  // PDL: the passes before this kernel are complete

  // the fix-up count, loaded now so its latency overlaps phase (2)
  const int count = *e.fix_count;

  // (2) gradient: warp w of CTA b owns entries ent = 8 b + w (grid-strided);
  // it also accumulates its entries' share of ||theta[:, :N-1]||^2 for the
  // lambda term (fixed order)
  double th2 = 0.0;
  {
    const ReduceParams& r = t.red;
    const int64_t KN = (int64_t)t.fin.K * t.fin.N;
    const bool lam = t.fin.lambda != 0.0;
    if (t.want_grad || lam) {
      // one warp per entry, lanes over the splits (s = lane mod 32), fixed
      // shuffle tree: many loads in flight, deterministic order
      const int nw = gridDim.x * (kTailThreads / 32);
      for (int64_t ent = (int64_t)blockIdx.x * (kTailThreads / 32) + warp; ent < KN; ent += nw) {
        double a = 0.0;
        if (t.want_grad) {
          // 8 loads in flight per lane (the partials are L2 reads one sector
          // each), summed in split order
          for (int s0 = lane; s0 < r.splits; s0 += 32 * 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int s = s0 + 32 * u;
              v[u] = s < r.splits ? __ldcg(r.part_g + (int64_t)s * KN + ent) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) a += v[u];
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        }
        if (lane == 0) {
          const int i = (int)(ent % t.fin.N);
          const double th = t.fin.theta[ent];
          if (lam && i < t.fin.N - 1) th2 += th * th;
          if (t.want_grad) {
            double gv = -a / (r.eps * (double)r.P);  // objective.py:162
            if (lam && i < r.N - 1) gv -= r.lambda * th;
            if (!isfinite(gv)) atomicAdd(r.nonfinite, 1);
            r.grad_out[ent] = gv;
          }
        }
      }
    }
    // per-CTA partial of the lambda norm: lane 0 of each warp, fixed order
    if (lane == 0) sred[warp][0] = th2;
    __syncthreads();
    if (tid == 0) {
      double s8 = 0.0;
#pragma unroll
      for (int w = 0; w < kTailThreads / 32; ++w) s8 += sred[w][0];
      t.part_th2[blockIdx.x] = s8;
    }
  }

  // (1) exact fp64 re-scan of the queued points: min and runner-up, then the
  // smallest index within the tie tolerance (geometry.py:208-210); for the
  // grid path it also decides the ambiguity of these points (fix_amb).
  // One warp per queued point, lanes over grains (coalesced theta reads).
  const int nwarps = gridDim.x * (kTailThreads / 32);
  for (int q = blockIdx.x * (kTailThreads / 32) + warp; q < count; q += nwarps) {
    const int64_t p = e.fix_list[q];
    double x[DIM], eta[K];
    point_coords<DIM>(p, e.M, e.pts, x);
    features<DIM, D>(x, e.legendre != 0, eta);
    double m = CUDART_INF, m2 = CUDART_INF;
    for (int i = lane; i < e.N; i += 32) {
      double h = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) h = fma(e.theta[(int64_t)k * e.N + i], eta[k], h);
      if (h < m) {
        m2 = m;
        m = h;
      } else if (h < m2) {
        m2 = h;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {  // merge (min, runner-up) pairs
      const double om = __shfl_xor_sync(0xffffffffu, m, off);
      const double om2 = __shfl_xor_sync(0xffffffffu, m2, off);
      const double nm = fmin(m, om);
      m2 = fmin(fmax(m, om), fmin(m2, om2));
      m = nm;
    }
    const double thr = tie_threshold(m);
    int best = 0x7fffffff;
    for (int i = lane; i < e.N; i += 32) {
      double h = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) h = fma(e.theta[(int64_t)k * e.N + i], eta[k], h);
      if (h <= thr) {
        best = i;
        break;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, off));
    if (best == 0x7fffffff) best = 0;
    if (lane == 0) {
      if (e.labels_out) e.labels_out[p] = best + 1;
      if (e.labels && best == e.labels[p]) atomicAdd((unsigned long long*)e.fix_correct, 1ull);
      if (t.fix_amb && (m2 - m) <= e.tau_amb * (1.0 + fabs(m)))
        atomicAdd((unsigned long long*)e.fix_correct + 1, 1ull);
    }
  }

  // (1b) the logit-range bound of the fast modes (pgx.h PGX_STAT_RANGE)
  if (t.range_c > 0.0) {
    float vmax = 0.0f;
    for (int i = blockIdx.x * kTailThreads + tid; i < t.fin.N; i += gridDim.x * kTailThreads) {
      double a = 0.0;
      for (int k = 0; k < t.fin.K; ++k) a += fabs(t.fin.theta[(int64_t)k * t.fin.N + i]);
      vmax = fmaxf(vmax, a <= 3e38 ? (float)a : CUDART_INF_F);  // NaN -> inf
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, off));
    if (lane == 0 && vmax > 0.0f) atomicMax(t.range_bits, __float_as_uint(vmax));
  }

  // (3) last CTA: scalars
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(t.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const FinalParams& prm = t.fin;
  const int per = (prm.blocks1 + kTailThreads - 1) / kTailThreads;
  const int b0 = tid * per, b1 = min(prm.blocks1, b0 + per);
  double ell = 0.0, e0 = 0.0;
  long long cor = 0, amb = 0, nf = 0;
  int n_fix = 0;
  if (tid == 0) {  // the counters, loaded alongside the partials (one round trip, not two)
    cor = *(volatile long long*)prm.fix_correct;
    amb = *((volatile long long*)prm.fix_correct + 1);
    nf = prm.nonfinite_grad ? *(volatile int*)prm.nonfinite_grad : 0;
    n_fix = *(volatile int*)e.fix_count;
  }
#pragma unroll 4
  for (int b = b0; b < b1; ++b) {
    ell += prm.part_d[2 * b + 0];
    e0 += prm.part_d[2 * b + 1];
    cor += prm.part_i[4 * b + 0];
    amb += prm.part_i[4 * b + 1];
    nf += prm.part_i[4 * b + 2];
  }
  th2 = 0.0;
  if (prm.lambda != 0.0) {  // per-CTA partials of phase (2), fixed order
    const int per2 = (gridDim.x + kTailThreads - 1) / kTailThreads;
    for (int q = tid * per2; q < min((int)gridDim.x, (tid + 1) * per2); ++q) th2 += t.part_th2[q];
  }
  block_sum6<kTailThreads>(ell, e0, th2, cor, amb, nf);
  if (tid == 0) {
    StatsDev* out = reinterpret_cast<StatsDev*>(prm.stats_out);
    const double P = (double)prm.P;
    double phi = ell / P;  // objective.py:161
    if (prm.lambda != 0.0) phi -= 0.5 * prm.lambda * th2;
    out->phi = phi;
    out->err = prm.want_assign ? 1.0 - (double)cor / P : 0.0;  // objective.py:163
    out->e0 = prm.want_assign ? e0 / P : 0.0;                  // objective.py:164
    out->n_rescanned = (double)n_fix;  // points re-scanned exactly
    out->n_points = prm.P;
    out->n_correct = cor;
    out->n_ambiguous = amb;
    out->n_nonfinite = nf + (isfinite(phi) ? 0 : 1);
    long long flags = 0;
    if (t.range_c > 0.0) {
      const float rb = __uint_as_float(*(volatile unsigned*)t.range_bits);
      if (!((double)rb * t.range_c <= PGX_FAST_RANGE)) flags |= PGX_STAT_RANGE;
      *t.range_bits = 0u;
    }
    out->flags = flags;
    // re-arm the counters for the next call (stream-ordered)
    *e.fix_count = 0;
    *(long long*)prm.fix_correct = 0;
    *((long long*)prm.fix_correct + 1) = 0;
    if (t.red.nonfinite) *t.red.nonfinite = 0;
    *t.ticket = 0;
  }
}

// theta (fp32 or fp64) -> fp64 working copy
static __global__ void k_theta_to_f64(const void* __restrict__ src, int is_f32, int64_t n,
                               double* __restrict__ dst) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = is_f32 ? (double)static_cast<const float*>(src)[e] : static_cast<const double*>(src)[e];
}

}  // namespace pgx
