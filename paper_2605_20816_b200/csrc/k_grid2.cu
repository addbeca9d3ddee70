// k_grid2.cu — regular-grid fp64 pass 2; launchers declared in pgx_launch.cuh.
#include "pgx_grid.cuh"
#include "pgx_launch.cuh"

namespace pgx {

template <int DIM, int D, int GT>
static void launch_grid_pass2_gt(const GridParams& g, dim3 grid, int smem, cudaStream_t s) {
  auto kern = k_grid_pass2<DIM, D, GT>;
  static DeviceOnce once;  // static + dynamic shared memory may exceed 48 KB
  once.run([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024); });
  launch_pdl(kern, grid, dim3(kG2Threads), smem, s, g);
}

template <int DIM, int D>
void grid_dispatch_pass2(const GridParams& g, int GT, dim3 grid, int smem, cudaStream_t s) {
  if (GT == 32)
    launch_grid_pass2_gt<DIM, D, 32>(g, grid, smem, s);
  else if (GT == 64)
    launch_grid_pass2_gt<DIM, D, 64>(g, grid, smem, s);
  else
    launch_grid_pass2_gt<DIM, D, 128>(g, grid, smem, s);
}

#define PGX_I(DIM, D) template void grid_dispatch_pass2<DIM, D>(const GridParams&, int, dim3, int, cudaStream_t);
// the build may compile this unit several times, each with a subset
// (build.py: -DPGX_INST_SET=...), so the slow fp64 kernels compile in parallel
#ifndef PGX_INST_SET
#define PGX_INST_SET PGX_INST_GRID
#endif
PGX_INST_SET(PGX_I)

}  // namespace pgx
