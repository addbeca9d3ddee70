// k_tc1.cu — tensor-core pass 1; launchers declared in pgx_launch.cuh.
#include "pgx_grid.cuh"

namespace pgx {

template <int DIM, int D, int R>
static void launch_tc_pass1_r(const GridParams& g, int blocks, cudaStream_t s) {
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
void tc_dispatch_pass1(const GridParams& g, int R, int blocks, cudaStream_t s) {
  if (R == 4)
    launch_tc_pass1_r<DIM, D, 4>(g, blocks, s);
  else if (R == 2)
    launch_tc_pass1_r<DIM, D, 2>(g, blocks, s);
  else
    launch_tc_pass1_r<DIM, D, 1>(g, blocks, s);
}

#define PGX_I(DIM, D) template void tc_dispatch_pass1<DIM, D>(const GridParams&, int, int, cudaStream_t);
PGX_INST_GRID(PGX_I)

}  // namespace pgx
