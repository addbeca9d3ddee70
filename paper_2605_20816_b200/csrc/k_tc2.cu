// k_tc2.cu — tensor-core pass 2 (pgx_tc_grad.cuh) and the per-evaluation operand
// tables (pgx_tc_coeffs.cuh); launchers declared in pgx_launch.cuh.
#include "pgx_grid.cuh"
#include "pgx_tc_grad.cuh"
#include "pgx_launch.cuh"

namespace pgx {

template <int DIM, int D>
void tc_dispatch_coeffs(const GridParams& g, const GridPlan& gp, cudaStream_t s) {
  constexpr int LPC = tc_coef_lines(DIM, D);
  if constexpr (LPC > 1) {
    dim3 grid((gp.lines + LPC - 1) / LPC, gp.tc_nchunks);
    k_tc_coeffs_ml<DIM, D><<<grid, kTcCoefChunk, 0, s>>>(g, gp.tc_coef, gp.tc_img,
                                                         reinterpret_cast<TcCoefMeta*>(gp.tc_meta),
                                                         gp.tc_nchunks);
  } else {
    dim3 grid(gp.lines, gp.tc_nchunks);
    k_tc_coeffs<DIM, D><<<grid, kTcCoefChunk, 0, s>>>(g, gp.tc_coef, gp.tc_img,
                                                      reinterpret_cast<TcCoefMeta*>(gp.tc_meta),
                                                      gp.tc_nchunks);
  }
}

template <int DIM, int D>
void tc_dispatch_pix(const GridParams& g, const GridPlan& gp, cudaStream_t s) {
  k_tc_pix<D><<<g.pside / kTcPixTile, kTcPixTile, 0, s>>>(g.M, g.legendre, gp.tc_pix);
}

template <int DIM, int D>
void tc_dispatch_pass2(const GridParams& g, dim3 grid, cudaStream_t s) {
  auto kern = k_tc_grad<DIM, D>;
  // padded so that <= 2 CTAs (2 x 256 TMEM columns) share an SM
  const int smem = std::max(GdSmem<DIM, D>::TOTAL, 80 * 1024);
  static DeviceOnce once;
  once.run([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  launch_pdl(kern, grid, dim3(kGdThreads), smem, s, g);
}

#define PGX_I(DIM, D) \
  template void tc_dispatch_coeffs<DIM, D>(const GridParams&, const GridPlan&, cudaStream_t); \
  template void tc_dispatch_pix<DIM, D>(const GridParams&, const GridPlan&, cudaStream_t); \
  template void tc_dispatch_pass2<DIM, D>(const GridParams&, dim3, cudaStream_t);
PGX_INST_GRID(PGX_I)

}  // namespace pgx


#ifdef PGX_GD_TRACE
extern "C" int pgx_debug_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, pgx::gd_trace, sizeof(pgx::gd_trace));
}
#endif
