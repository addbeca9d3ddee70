// pgx_grid_eval.cuh — one evaluation on the regular-grid paths: the launch
// sequence over the kernel families (included by pgx_api.cu only, so the
// k_*.cu units do not implicitly instantiate each other's launchers).
#pragma once

#include "pgx_grid.cuh"
#include "pgx_launch.cuh"

namespace pgx {

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

// the kernels' view of one evaluation / assignment on the plan
inline GridParams grid_params(const GridPlan& gp, const EvalParams& e, bool want_grad) {
  GridParams g{};
  g.P = e.P;
  g.N = e.N;
  g.M = e.M;
  g.side = 2 * e.M;
  g.pside = gp.pside;
  g.legendre = e.legendre;
  g.R = gp.R;
  g.lines = gp.lines;
  g.segs = gp.segs;
  g.theta = e.theta;
  g.labels = e.labels;
  g.eps = e.eps;
  g.c = 1.4426950408889634074 / e.eps;
  g.tau_amb = e.tau_amb;
  g.theta32 = gp.tc ? e.theta32 : nullptr;

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
  g.tile_lo = 0;
  g.tile_hi = (int64_t)gp.lines * (g.pside / kTcThreadsTile);
  g.part_off = 0;
  g.line_lo = 0;
  g.split_off = 0;
  g.labels_out = e.labels_out;
  g.margin_out = e.margin_out;
  return g;
}

// hard assignment on the tensor-core path: coefficient tables + the ASSIGN sweep
inline pgx_status grid_assign(GridPlan& gp, const EvalParams& e, cudaStream_t s, int* launches,
                              int* blocks1, const GridProf& prof) {
  GridParams g = grid_params(gp, e, false);
  prof.begin(prof.ctx, "tc_coeffs");
  if (gp.dim == 2) {
    PGX_GRID_DEG(2, tc_dispatch_coeffs, g, gp, s)
  } else {
    PGX_GRID_DEG3(tc_dispatch_coeffs, g, gp, s)
  }
  prof.end(prof.ctx);
  ++*launches;
  if (cudaPeekAtLastError() != cudaSuccess) return PGX_ERR_CUDA;
  prof.begin(prof.ctx, "tc_assign");
  if (gp.dim == 2) {
    PGX_GRID_DEG(2, tc_dispatch_assign, g, gp.tc_blocks, s)
  } else {
    PGX_GRID_DEG3(tc_dispatch_assign, g, gp.tc_blocks, s)
  }
  prof.end(prof.ctx);
  ++*launches;
  *blocks1 = gp.tc_blocks;
  return cudaPeekAtLastError() == cudaSuccess ? PGX_OK : PGX_ERR_CUDA;
}

inline pgx_status grid_eval(GridPlan& gp, const EvalParams& e, int prec, bool want_grad,
                            cudaStream_t s, int* launches, int* blocks1, const GridProf& prof) {
  (void)prec;
  GridParams g = grid_params(gp, e, want_grad);
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
    // a failed table launch must not leave pass 1 reading stale images
    if (cudaPeekAtLastError() != cudaSuccess) return PGX_ERR_CUDA;
    prof.begin(prof.ctx, "tc_pass1");
    if (gp.dim == 2) {
      PGX_GRID_DEG(2, tc_dispatch_pass1, g, gp.tc_blocks, s)
    } else {
      PGX_GRID_DEG3(tc_dispatch_pass1, g, gp.tc_blocks, s)
    }
    prof.end(prof.ctx);
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
    g.items_per_split = gp.tc2_ips;
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
