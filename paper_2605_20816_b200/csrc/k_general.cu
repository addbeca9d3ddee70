// k_general.cu — general (any point list) path; launchers declared in
// pgx_launch.cuh.
#include "pgx_launch.cuh"

namespace pgx {

template <int DIM, int D>
void launch_general_pass1(const EvalParams& prm, int blocks, bool eval, cudaStream_t s) {
  if (eval)
    k_general_pass1<DIM, D, true><<<blocks, kP1Threads, 0, s>>>(prm);
  else
    k_general_pass1<DIM, D, false><<<blocks, kP1Threads, 0, s>>>(prm);
}
template <int DIM, int D>
void launch_general_pass2(const EvalParams& prm, int N, int splits, cudaStream_t s) {
  dim3 grid((N + kP2Threads - 1) / kP2Threads, splits);
  k_general_pass2<DIM, D><<<grid, kP2Threads, 0, s>>>(prm);
}

#define PGX_I(DIM, D)                                                                      \
  template void launch_general_pass1<DIM, D>(const EvalParams&, int, bool, cudaStream_t); \
  template void launch_general_pass2<DIM, D>(const EvalParams&, int, int, cudaStream_t);
PGX_INST_GENERAL(PGX_I)

}  // namespace pgx
