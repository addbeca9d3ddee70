// pgx_launch.cuh — host-side launchers of every kernel family, declared here
// and defined + explicitly instantiated in one translation unit per family
// (k_*.cu), so the families compile in parallel and pgx_api.cu instantiates
// no kernels itself.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "pgx_general.cuh"
#include "pgx_grid_common.cuh"

namespace pgx {

struct GridPlan;

// PDL on (default) unless PGX_PDL=0
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PGX_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// A per-device one-time action (a kernel's cudaFuncSetAttribute applies to the
// current device only): runs `f` the first time it is called on each device
// ordinal; thread-safe (a racing duplicate call is harmless: the attribute
// set is idempotent).
struct DeviceOnce {
  std::atomic<uint64_t> done{0};
  template <typename F>
  void run(F&& f) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
      (void)cudaGetLastError();
      dev = 0;
    }
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    f();
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
};

// launch `kern` with programmatic stream serialization (the kernel must call
// griddep_wait() before touching its predecessor's data, see pgx_common.cuh)
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  if (pdl_enabled()) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...) == cudaSuccess) return;
    (void)cudaGetLastError();  // not launchable this way: plain launch below
  }
  kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
}

// general (any point list) path + tail: pgx_general.cuh
template <int DIM, int D>
void launch_general_pass1(const EvalParams& prm, int blocks, bool eval, cudaStream_t s);
template <int DIM, int D>
void launch_general_pass2(const EvalParams& prm, int N, int splits, cudaStream_t s);
template <int DIM, int D>
void launch_tail(const EvalParams& prm, const TailParams& tp, int blocks, cudaStream_t s);

// explicit design matrix (any K <= kMaxK) and the dense soft assignment: pgx_design.cuh
void launch_design_pass1(const EvalParams& prm, const double* dsg, int K, int blocks, bool eval,
                         cudaStream_t s);
void launch_design_pass2(const EvalParams& prm, const double* dsg, int K, int splits, cudaStream_t s);
void launch_design_soft(const EvalParams& prm, const double* dsg, int K, double* prob, cudaStream_t s);
template <int DIM, int D>
void launch_general_soft(const EvalParams& prm, double* prob, cudaStream_t s);

// label moments over a problem's resident int32 labels: k_moments.cu
cudaError_t launch_label_moments_i32(int M, int64_t P, const int32_t* labels0, int N,
                                     unsigned long long* out, int* bad, int sms, cudaStream_t s);

// device-resident optimiser vectors (k_lbfgs.cu)
void launch_lb_point(double* theta, double* ut, const double* u, const double* d, const double* t_ptr, int K,
                     int N, int sms, cudaStream_t s);
void launch_lb_after(const double* grad, double* gt, const double* d, double* out, int K, int N,
                     cudaStream_t s);
void launch_lb_two_loop(const double* g, double* d, const double* S, const double* Y, const double* rho,
                        double* alpha, const int* state, int m, int64_t n, int mode, double* out,
                        cudaStream_t s);
void launch_lb_accept(double* u, double* g, const double* ut, const double* gt, double* S, double* Y,
                      double* rho, int* state, int m, int64_t n, double skip, int keep_pair, double* out,
                      cudaStream_t s);

// regular-grid fp64 path: pgx_grid_pass1.cuh, pgx_grid_pass2.cuh
template <int DIM, int D>
void grid_dispatch_pass1(const GridParams& g, int R, int blocks, cudaStream_t s);
template <int DIM, int D>
void grid_dispatch_pass2(const GridParams& g, int GT, dim3 grid, int smem, cudaStream_t s);

// tensor-core path: pgx_tc_coeffs.cuh, pgx_tc_sweep.cuh (pass 1), pgx_tc_grad.cuh (pass 2)
template <int DIM, int D>
void tc_dispatch_coeffs(const GridParams& g, const GridPlan& gp, cudaStream_t s);
template <int DIM, int D>
void tc_dispatch_pix(const GridParams& g, const GridPlan& gp, cudaStream_t s);
template <int DIM, int D>
void tc_dispatch_pass1(const GridParams& g, int blocks, cudaStream_t s);
template <int DIM, int D>
void tc_dispatch_assign(const GridParams& g, int blocks, cudaStream_t s);
template <int DIM, int D>
void tc_dispatch_pass2(const GridParams& g, dim3 grid, cudaStream_t s);

}  // namespace pgx

// explicit instantiation over the degrees each path dispatches
#define PGX_INST_GRID(DECL)                                                         \
  DECL(2, 0) DECL(2, 1) DECL(2, 2) DECL(2, 3) DECL(2, 4) DECL(2, 5) DECL(2, 6) \
  DECL(2, 7) DECL(2, 8) DECL(3, 0) DECL(3, 1) DECL(3, 2) DECL(3, 3) DECL(3, 4)
#define PGX_INST_2D_LO(DECL) DECL(2, 0) DECL(2, 1) DECL(2, 2) DECL(2, 3) DECL(2, 4) DECL(2, 5)
#define PGX_INST_2D_6(DECL) DECL(2, 6)
#define PGX_INST_2D_7(DECL) DECL(2, 7)
#define PGX_INST_2D_8(DECL) DECL(2, 8)
#define PGX_INST_3D_LO(DECL) DECL(3, 0) DECL(3, 1) DECL(3, 2)
#define PGX_INST_3D_3(DECL) DECL(3, 3)
#define PGX_INST_3D_4(DECL) DECL(3, 4)
#define PGX_INST_GENERAL(DECL) PGX_INST_GRID(DECL) DECL(2, 9) DECL(2, 10)
