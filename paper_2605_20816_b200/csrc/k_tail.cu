// k_tail.cu — the tail kernel (arg-min fix-up, split reduction, finalize);
// launcher declared in pgx_launch.cuh.
#include "pgx_launch.cuh"

namespace pgx {

template <int DIM, int D>
void launch_tail(const EvalParams& prm, const TailParams& tp, int blocks, cudaStream_t s) {
  launch_pdl(k_tail<DIM, D>, dim3(blocks), dim3(kTailThreads), 0, s, prm, tp);
}

#define PGX_I(DIM, D) \
  template void launch_tail<DIM, D>(const EvalParams&, const TailParams&, int, cudaStream_t);
PGX_INST_GENERAL(PGX_I)

}  // namespace pgx
