// k_design.cu — the explicit design-matrix path and the dense soft assignment
// (pgx_design.cuh); launchers declared in pgx_launch.cuh.
#include "pgx_design.cuh"
#include "pgx_launch.cuh"

namespace pgx {

#define PGX_KB_SWITCH(K, FN)          \
  if ((K) <= 8) {                     \
    FN(8);                            \
  } else if ((K) <= 16) {             \
    FN(16);                           \
  } else if ((K) <= 32) {             \
    FN(32);                           \
  } else {                            \
    FN(kMaxK);                        \
  }

void launch_design_pass1(const EvalParams& prm, const double* dsg, int K, int blocks, bool eval,
                         cudaStream_t s) {
#define L1(KB)                                                                            \
  if (eval)                                                                               \
    k_design_pass1<KB, true><<<blocks, kP1Threads, 0, s>>>(prm, dsg, K);                  \
  else                                                                                    \
    k_design_pass1<KB, false><<<blocks, kP1Threads, 0, s>>>(prm, dsg, K);
  PGX_KB_SWITCH(K, L1)
#undef L1
}

void launch_design_pass2(const EvalParams& prm, const double* dsg, int K, int splits, cudaStream_t s) {
  dim3 grid((prm.N + kP2Threads - 1) / kP2Threads, splits);
#define L2(KB) k_design_pass2<KB><<<grid, kP2Threads, 0, s>>>(prm, dsg, K);
  PGX_KB_SWITCH(K, L2)
#undef L2
}

void launch_design_soft(const EvalParams& prm, const double* dsg, int K, double* prob, cudaStream_t s) {
  const int blocks = (int)((prm.P + 127) / 128);
#define L3(KB) k_design_soft<KB><<<blocks, 128, 0, s>>>(prm, dsg, K, prob);
  PGX_KB_SWITCH(K, L3)
#undef L3
}

template <int DIM, int D>
void launch_general_soft(const EvalParams& prm, double* prob, cudaStream_t s) {
  k_general_soft<DIM, D><<<(int)((prm.P + 127) / 128), 128, 0, s>>>(prm, prob);
}

#define PGX_I(DIM, D) template void launch_general_soft<DIM, D>(const EvalParams&, double*, cudaStream_t);
PGX_INST_GENERAL(PGX_I)

}  // namespace pgx
