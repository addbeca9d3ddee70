// pgx_grid.cuh — regular-grid (separable) fast path.  Placeholder plan until
// the separable kernels land; the general path serves every problem.
#pragma once
#include "../../include/pgx.h"
#include "pgx_general.cuh"

namespace pgx {

struct GridPlan {
  bool enabled = false;
  int splits_out = 1;
  double* part_out = nullptr;
  void* d_part = nullptr;
};

inline size_t grid_workspace_bytes(const pgx_desc*, int) { return 0; }
inline cudaError_t grid_plan_create(GridPlan& g, const pgx_desc*, int, size_t&) {
  g.enabled = false;
  return cudaSuccess;
}
inline pgx_status grid_eval(GridPlan&, const EvalParams&, int, bool, cudaStream_t, int*, int*) {
  return PGX_ERR_CUDA;
}

}  // namespace pgx
