// k_grid1.cu — regular-grid fp64 pass 1; launchers declared in pgx_launch.cuh.
#include "pgx_grid.cuh"
#include "pgx_launch.cuh"

namespace pgx {

template <int DIM, int D>
void grid_dispatch_pass1(const GridParams& g, int R, int blocks, cudaStream_t s) {
  if (R == 4)
    launch_pdl(k_grid_pass1<DIM, D, 4>, dim3(blocks), dim3(kG1Threads), 0, s, g);
  else if (R == 2)
    launch_pdl(k_grid_pass1<DIM, D, 2>, dim3(blocks), dim3(kG1Threads), 0, s, g);
  else
    launch_pdl(k_grid_pass1<DIM, D, 1>, dim3(blocks), dim3(kG1Threads), 0, s, g);
}

#define PGX_I(DIM, D) template void grid_dispatch_pass1<DIM, D>(const GridParams&, int, int, cudaStream_t);
// the build may compile this unit several times, each with a subset
// (build.py: -DPGX_INST_SET=...), so the slow fp64 kernels compile in parallel
#ifndef PGX_INST_SET
#define PGX_INST_SET PGX_INST_GRID
#endif
PGX_INST_SET(PGX_I)

}  // namespace pgx
