// k_tc1.cu — tensor-core pass 1 (pgx_tc_sweep.cuh); launcher declared in pgx_launch.cuh.
#include "pgx_grid.cuh"
#include "pgx_launch.cuh"
#include "pgx_tc_sweep.cuh"

namespace pgx {

template <int DIM, int D>
void tc_dispatch_pass1(const GridParams& g, int blocks, cudaStream_t s) {
  auto kern = k_tc_sweep<DIM, D, false>;
  const int smem = SwSmem<D + 1>::TOTAL;
  static DeviceOnce once;
  once.run([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  launch_pdl(kern, dim3(blocks), dim3(kSwThreads), smem, s, g);
}

// the hard-assignment variant of the sweep (pgx_assign on a tensor-core problem)
template <int DIM, int D>
void tc_dispatch_assign(const GridParams& g, int blocks, cudaStream_t s) {
  auto kern = k_tc_sweep<DIM, D, true>;
  const int smem = SwSmem<D + 1>::TOTAL;
  static DeviceOnce once;
  once.run([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  launch_pdl(kern, dim3(blocks), dim3(kSwThreads), smem, s, g);
}

#define PGX_I(DIM, D)                                                                  \
  template void tc_dispatch_pass1<DIM, D>(const GridParams&, int, cudaStream_t);       \
  template void tc_dispatch_assign<DIM, D>(const GridParams&, int, cudaStream_t);
PGX_INST_GRID(PGX_I)

}  // namespace pgx
