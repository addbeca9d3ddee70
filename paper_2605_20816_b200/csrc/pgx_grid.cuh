// pgx_grid.cuh — regular-grid (separable) fp64 path: plan + dispatch.
// Kernels: pgx_grid_pass1.cuh (min / arg-min / log-sum-exp), pgx_grid_pass2.cuh
// (gradient contraction); shared pieces in pgx_grid_common.cuh.
#pragma once

#include <algorithm>

#include "pgx_grid_common.cuh"
#include "pgx_grid_pass1.cuh"
#include "pgx_grid_pass2.cuh"
#include "pgx_tc_pass1.cuh"
#include "pgx_tc_pass2.cuh"

namespace pgx {

struct GridPlan {
  bool enabled = false;
  bool tc = false;  // PGX_PREC_TC: tensor-core pass 1
  int dim = 2, D = 1;
  int R = 1, segs = 1, lines = 0, blocks1 = 0;
  int tcR = 1, tc_segs = 1, tc_blocks = 0;
  int tc2_gtiles = 0, tc2_lps = 1, tc2_splits = 0;  // tensor-core pass 2 (0 = CUDA-core pass 2)
  int part_splits = 0;                             // allocated split slots of part_g
  int tc_nchunks = 0;                              // 128-grain chunks (pgx_tc_coeffs.cuh)
  void* d_tc = nullptr;                            // coef | img | meta
  double* tc_coef = nullptr;
  unsigned char* tc_img = nullptr;
  int2* tc_meta = nullptr;
  void* d_tc_pix = nullptr;                        // pass-2 pixel operand tiles (once per problem)
  unsigned char* tc_pix = nullptr;
  bool tc_pix_ready = false;
  float* tc_rec = nullptr;                         // pass-2 pixel records (aliases pix_w | pix_q)
  double* tc_lc = nullptr;                         // [lines][K] line factors
  int GT = 128, gtiles = 1, splits = 1, lines_per_split = 1;
  int splits_out = 1;
  double* part_out = nullptr;
  void* d_part = nullptr;  // single allocation: part_g | pix_w, pix_q (fp64) or tc_rec (TC)
  double* pix_w = nullptr;
  float* pix_q = nullptr;
  int smem2 = 0;
};

inline void grid_plan_shape(GridPlan& gp, const pgx_desc* d, int sms) {
  gp.enabled = false;
  if (d->resolution <= 0 || d->precision == PGX_PREC_EXACT) return;
  const int side = 2 * d->resolution;
  if (side % 128 != 0) return;  // small grids use the general path
  if (d->dim == 2 && d->degree > 8) return;
  if (d->dim == 3 && d->degree > 4) return;
  gp.enabled = true;
  gp.dim = d->dim;
  gp.D = d->degree;
  gp.lines = (int)(d->n_points / side);
  // pixels per thread: register blocking of the shared B'' loads, bounded by
  // the register file and by the wave count (>= ~6 CTAs per SM when possible)
  const int rmax = d->degree <= 3 ? 4 : (d->degree <= 5 ? 2 : 1);
  int R = std::min(rmax, side / 128);
  while (R > 1 && (int64_t)gp.lines * (side / (128 * R)) < 6 * sms) R /= 2;
  gp.R = R;
  gp.segs = side / (128 * gp.R);
  gp.blocks1 = gp.lines * gp.segs;
  // tensor-core pass 1: <= 2 CTAs per SM (256 TMEM columns each); R tiles of
  // 128 pixels share each chunk's coefficient build
  gp.tc = d->precision == PGX_PREC_TC;
  if (gp.tc) {
    // shared memory per CTA must stay <= ~56 KB for 4 CTAs per SM
    int tr = std::min(tc_ksteps(d->degree + 1) == 1 ? 4 : 2, side / 128);
    while (tr > 1 && (int64_t)gp.lines * (side / (128 * tr)) < 4 * sms) tr /= 2;
    gp.tcR = tr;
    gp.tc_segs = side / (128 * tr);
    gp.tc_blocks = gp.lines * gp.tc_segs;
    gp.blocks1 = gp.tc_blocks;
  }
  const int N = d->n_grains;
  // grains per pass-2 CTA: least padding, larger tile on ties
  gp.GT = 128;
  for (int gt : {64, 32})
    if ((N + gt - 1) / gt * gt < (N + gp.GT - 1) / gp.GT * gp.GT) gp.GT = gt;
  gp.gtiles = (N + gp.GT - 1) / gp.GT;
  const int target = 8 * sms;
  gp.splits = std::max(1, std::min(gp.lines, (target + gp.gtiles - 1) / gp.gtiles));
  gp.lines_per_split = (gp.lines + gp.splits - 1) / gp.splits;
  gp.splits = (gp.lines + gp.lines_per_split - 1) / gp.lines_per_split;
  gp.splits_out = gp.splits;
  const int K = feature_count(d->dim, d->degree);
  gp.smem2 = K * kG2Threads * 8;
  if (gp.tc && side % kTc2Px == 0) {
    // tensor-core pass 2: 128-grain tiles x line ranges, 2 CTAs per SM; the
    // split count minimises waves x lines-per-CTA (ties: fewer splits, so the
    // tail reduces less)
    gp.tc2_gtiles = (N + kTc2Grains - 1) / kTc2Grains;
    const int64_t slots = 2LL * sms;
    int64_t best = -1;
    for (int sp = 1; sp <= std::min(gp.lines, 8 * sms); ++sp) {
      const int lps = (gp.lines + sp - 1) / sp;
      const int spr = (gp.lines + lps - 1) / lps;
      if (spr != sp) continue;
      const int64_t waves = ((int64_t)gp.tc2_gtiles * spr + slots - 1) / slots;
      const int64_t cost = waves * (lps + 1);  // + ~1 line of per-CTA pipeline fill
      if (best < 0 || cost < best) {
        best = cost;
        gp.tc2_lps = lps;
        gp.tc2_splits = spr;
      }
    }
    gp.splits_out = gp.tc2_splits;
    gp.part_splits = std::max(gp.splits, gp.tc2_splits);
  }
}

inline size_t grid_workspace_bytes(const pgx_desc* d, int sms) {
  GridPlan gp;
  grid_plan_shape(gp, d, sms);
  if (!gp.enabled) return 0;
  const int K = feature_count(d->dim, d->degree);
  return (size_t)std::max(gp.splits, gp.part_splits) * K * d->n_grains * 8 + (size_t)d->n_points * 16;
}

inline cudaError_t grid_plan_create(GridPlan& gp, const pgx_desc* d, int sms, size_t& bytes) {
  grid_plan_shape(gp, d, sms);
  if (!gp.enabled) return cudaSuccess;
  const int K = feature_count(d->dim, d->degree);
  const size_t part = (size_t)std::max(gp.splits, gp.part_splits) * K * d->n_grains;
  const size_t n = part * 8 + (size_t)d->n_points * 16 + 256;
  cudaError_t e = cudaMalloc(&gp.d_part, n);
  if (e != cudaSuccess) return e;
  bytes += n;
  gp.part_out = static_cast<double*>(gp.d_part);
  gp.pix_w = gp.part_out + part;
  gp.pix_q = reinterpret_cast<float*>(gp.pix_w + d->n_points);
  if (gp.tc) {
    const int J = d->degree + 1;
    gp.tc_nchunks = (d->n_grains + kTcCoefChunk - 1) / kTcCoefChunk;
    const size_t ncoef = (size_t)gp.lines * d->n_grains * J;
    const size_t nimg = (size_t)gp.lines * gp.tc_nchunks * tc_ksteps(J) * kTcCoefChunk * 32;
    const size_t nmeta = (size_t)gp.lines * gp.tc_nchunks;
    const size_t nlc = (size_t)gp.lines * K;
    const size_t tb = ncoef * 8 + nimg + nmeta * 8 + nlc * 8 + 256;
    e = cudaMalloc(&gp.d_tc, tb);
    if (e != cudaSuccess) return e;
    bytes += tb;
    gp.tc_coef = static_cast<double*>(gp.d_tc);
    gp.tc_img = reinterpret_cast<unsigned char*>(gp.tc_coef + ncoef);
    gp.tc_meta = reinterpret_cast<int2*>(gp.tc_img + nimg);
    gp.tc_lc = reinterpret_cast<double*>(gp.tc_meta + nmeta);
    if (gp.tc2_splits > 0) {
      gp.tc_rec = reinterpret_cast<float*>(gp.pix_w);  // 16 bytes per pixel
      const size_t npix = (size_t)(2 * d->resolution / kTcPixTile) *
                          (tc_ksteps(J) * kTcPixTile * 32 + 2 * (kTcPixTile / 16) * 16 * 32);
      e = cudaMalloc(&gp.d_tc_pix, npix);
      if (e != cudaSuccess) return e;
      bytes += npix;
      gp.tc_pix = static_cast<unsigned char*>(gp.d_tc_pix);
      gp.tc_pix_ready = false;
    }
  }
  return cudaSuccess;
}

template <int DIM, int D>
inline void grid_dispatch_pass1(const GridParams& g, int R, int blocks, cudaStream_t s) {
  if (R == 4)
    k_grid_pass1<DIM, D, 4><<<blocks, kG1Threads, 0, s>>>(g);
  else if (R == 2)
    k_grid_pass1<DIM, D, 2><<<blocks, kG1Threads, 0, s>>>(g);
  else
    k_grid_pass1<DIM, D, 1><<<blocks, kG1Threads, 0, s>>>(g);
}

template <int DIM, int D, int R>
inline void launch_tc_pass1_r(const GridParams& g, int blocks, cudaStream_t s) {
  auto kern = k_tc_pass1<DIM, D, R>;
  // padded so that <= 4 CTAs (4 x 128 TMEM columns) share an SM
  const int smem = std::max(TcP1Smem<D + 1, R>::TOTAL, kTcMinSmem);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  kern<<<blocks, kTcThreads, smem, s>>>(g);
}

template <int DIM, int D>
inline void tc_dispatch_pass1(const GridParams& g, int R, int blocks, cudaStream_t s) {
  if (R == 4)
    launch_tc_pass1_r<DIM, D, 4>(g, blocks, s);
  else if (R == 2)
    launch_tc_pass1_r<DIM, D, 2>(g, blocks, s);
  else
    launch_tc_pass1_r<DIM, D, 1>(g, blocks, s);
}

template <int DIM, int D>
inline void tc_dispatch_coeffs(const GridParams& g, const GridPlan& gp, cudaStream_t s) {
  dim3 grid(gp.tc_nchunks, gp.lines);
  k_tc_coeffs<DIM, D><<<grid, kTcCoefChunk, 0, s>>>(g, gp.tc_coef, gp.tc_img,
                                                    reinterpret_cast<TcCoefMeta*>(gp.tc_meta),
                                                    gp.tc_nchunks);
}

template <int DIM, int D>
inline void tc_dispatch_pix(const GridParams& g, const GridPlan& gp, cudaStream_t s) {
  k_tc_pix<D><<<g.side / kTcPixTile, kTcPixTile, 0, s>>>(g.M, g.legendre, gp.tc_pix);
}

template <int DIM, int D>
inline void tc_dispatch_pass2(const GridParams& g, dim3 grid, cudaStream_t s) {
  auto kern = k_tc_pass2<DIM, D>;
  // padded so that <= 2 CTAs (2 x 256 TMEM columns) share an SM
  const int smem = std::max(TcP2Smem<D + 1>::TOTAL, 80 * 1024);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  kern<<<grid, kTc2Threads, smem, s>>>(g);
}

template <int DIM, int D, int GT>
inline void launch_grid_pass2_gt(const GridParams& g, dim3 grid, int smem, cudaStream_t s) {
  auto kern = k_grid_pass2<DIM, D, GT>;
  static bool configured = false;  // static + dynamic shared memory may exceed 48 KB
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    configured = true;
  }
  kern<<<grid, kG2Threads, smem, s>>>(g);
}

template <int DIM, int D>
inline void grid_dispatch_pass2(const GridParams& g, int GT, dim3 grid, int smem, cudaStream_t s) {
  if (GT == 32)
    launch_grid_pass2_gt<DIM, D, 32>(g, grid, smem, s);
  else if (GT == 64)
    launch_grid_pass2_gt<DIM, D, 64>(g, grid, smem, s);
  else
    launch_grid_pass2_gt<DIM, D, 128>(g, grid, smem, s);
}

#define PGX_GRID_DEG(DIM_, FN, ...)              \
  switch (gp.D) {                                \
    case 0: FN<DIM_, 0>(__VA_ARGS__); break;     \
    case 1: FN<DIM_, 1>(__VA_ARGS__); break;     \
    case 2: FN<DIM_, 2>(__VA_ARGS__); break;     \
    case 3: FN<DIM_, 3>(__VA_ARGS__); break;     \
    case 4: FN<DIM_, 4>(__VA_ARGS__); break;     \
    case 5: FN<DIM_, 5>(__VA_ARGS__); break;     \
    case 6: FN<DIM_, 6>(__VA_ARGS__); break;     \
    case 7: FN<DIM_, 7>(__VA_ARGS__); break;     \
    default: FN<DIM_, 8>(__VA_ARGS__); break;    \
  }
#define PGX_GRID_DEG3(FN, ...)                   \
  switch (gp.D) {                                \
    case 0: FN<3, 0>(__VA_ARGS__); break;        \
    case 1: FN<3, 1>(__VA_ARGS__); break;        \
    case 2: FN<3, 2>(__VA_ARGS__); break;        \
    case 3: FN<3, 3>(__VA_ARGS__); break;        \
    default: FN<3, 4>(__VA_ARGS__); break;       \
  }

struct GridProf {
  void* ctx;
  void (*begin)(void*, const char*);
  void (*end)(void*);
};

inline pgx_status grid_eval(GridPlan& gp, const EvalParams& e, int prec, bool want_grad,
                            cudaStream_t s, int* launches, int* blocks1, const GridProf& prof) {
  (void)prec;
  GridParams g{};
  g.P = e.P;
  g.N = e.N;
  g.M = e.M;
  g.side = 2 * e.M;
  g.legendre = e.legendre;
  g.R = gp.R;
  g.lines = gp.lines;
  g.segs = gp.segs;
  g.theta = e.theta;
  g.labels = e.labels;
  g.eps = e.eps;
  g.c = 1.4426950408889634074 / e.eps;
  g.tau_amb = e.tau_amb;
  g.pix_m = e.pix_m;
  g.pix_w = gp.pix_w;
  g.pix_q = gp.pix_q;
  g.part_d = e.part_d;
  g.part_i = e.part_i;
  g.fix_count = e.fix_count;
  g.fix_list = e.fix_list;
  g.GT = gp.GT;
  g.lines_per_split = gp.lines_per_split;
  g.splits = gp.splits;
  g.part_g = gp.part_out;
  g.tc_coef = gp.tc_coef;
  g.tc_img = gp.tc_img;
  g.tc_meta = gp.tc_meta;
  g.tc_nchunks = gp.tc_nchunks;
  g.tc_pix = gp.tc_pix;
  g.tc_lc = gp.tc_lc;
  g.tc_rec = want_grad ? gp.tc_rec : nullptr;
  if (gp.tc && gp.tc_pix && !gp.tc_pix_ready) {  // once per problem
    if (gp.dim == 2) {
      PGX_GRID_DEG(2, tc_dispatch_pix, g, gp, s)
    } else {
      PGX_GRID_DEG3(tc_dispatch_pix, g, gp, s)
    }
    ++*launches;
    if (cudaPeekAtLastError() != cudaSuccess) return PGX_ERR_CUDA;
    gp.tc_pix_ready = true;
  }
  if (gp.tc) {
    prof.begin(prof.ctx, "tc_coeffs");
    if (gp.dim == 2) {
      PGX_GRID_DEG(2, tc_dispatch_coeffs, g, gp, s)
    } else {
      PGX_GRID_DEG3(tc_dispatch_coeffs, g, gp, s)
    }
    prof.end(prof.ctx);
    ++*launches;
    g.R = gp.tcR;
    g.segs = gp.tc_segs;
    prof.begin(prof.ctx, "tc_pass1");
    if (gp.dim == 2) {
      PGX_GRID_DEG(2, tc_dispatch_pass1, g, gp.tcR, gp.tc_blocks, s)
    } else {
      PGX_GRID_DEG3(tc_dispatch_pass1, g, gp.tcR, gp.tc_blocks, s)
    }
    prof.end(prof.ctx);
    g.R = gp.R;
    g.segs = gp.segs;
  } else {
    prof.begin(prof.ctx, "grid_pass1");
    if (gp.dim == 2) {
      PGX_GRID_DEG(2, grid_dispatch_pass1, g, gp.R, gp.blocks1, s)
    } else {
      PGX_GRID_DEG3(grid_dispatch_pass1, g, gp.R, gp.blocks1, s)
    }
    prof.end(prof.ctx);
  }
  ++*launches;
  *blocks1 = gp.blocks1;
  if (cudaPeekAtLastError() != cudaSuccess) return PGX_ERR_CUDA;
  if (want_grad && gp.tc && gp.tc2_splits > 0) {
    dim3 grid(gp.tc2_gtiles, gp.tc2_splits);
    g.lines_per_split = gp.tc2_lps;
    g.splits = gp.tc2_splits;
    prof.begin(prof.ctx, "tc_pass2");
    if (gp.dim == 2) {
      PGX_GRID_DEG(2, tc_dispatch_pass2, g, grid, s)
    } else {
      PGX_GRID_DEG3(tc_dispatch_pass2, g, grid, s)
    }
    prof.end(prof.ctx);
    ++*launches;
    if (cudaPeekAtLastError() != cudaSuccess) return PGX_ERR_CUDA;
  } else if (want_grad) {
    dim3 grid(gp.gtiles, gp.splits);
    prof.begin(prof.ctx, "grid_pass2");
    if (gp.dim == 2) {
      PGX_GRID_DEG(2, grid_dispatch_pass2, g, gp.GT, grid, gp.smem2, s)
    } else {
      PGX_GRID_DEG3(grid_dispatch_pass2, g, gp.GT, grid, gp.smem2, s)
    }
    prof.end(prof.ctx);
    ++*launches;
    if (cudaPeekAtLastError() != cudaSuccess) return PGX_ERR_CUDA;
  }
  return PGX_OK;
}

}  // namespace pgx
