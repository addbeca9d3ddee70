// k_moments.cu — per-grain label moments of a regular 2-D grid, the input of
// the moment heuristic (heuristics.py:46-73: counts, sums of x and of the
// products x_a x_b per grain, np.bincount over the labels).
//
// On make_grid's grid a coordinate is x = (2k + 1 - 2M) / (2M), so a = 2M x
// is an odd integer: the six sums {1, a1, a2, a1^2, a1 a2, a2^2} per grain are
// exact in int64 (|sum| <= P (2M)^2 < 2^63 for every grid that fits in HBM)
// and order-independent, so integer atomics give bit-reproducible results.
// A warp first merges lanes with equal labels (__match_any_sync: neighbouring
// pixels of a line mostly share their grain), one atomic per distinct label.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/pgx.h"

namespace pgx {

template <typename LabelT>
__global__ void k_label_moments(int M, int64_t P, const LabelT* __restrict__ labels0, int N,
                                unsigned long long* __restrict__ out, int* __restrict__ bad) {
  const int side = 2 * M;
  const unsigned lane = threadIdx.x & 31u;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x; p0 < P; p0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = p0 + threadIdx.x;
    const bool in = p < P;
    int lab = -1;
    long long v[6] = {0, 0, 0, 0, 0, 0};
    if (in) {
      const int64_t l = labels0[p];
      if (l < 0 || l >= N) {
        atomicExch(bad, 1);
      } else {
        lab = (int)l;
        const long long a = 2 * (p / side) + 1 - side, b = 2 * (p % side) + 1 - side;
        v[0] = 1;
        v[1] = a;
        v[2] = b;
        v[3] = a * a;
        v[4] = a * b;
        v[5] = b * b;
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, lab);
    const unsigned leader = __ffs(peers) - 1;
    // sum over the peers with the same label (fixed lane order: exact integers anyway)
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      long long s = 0;
      for (unsigned m = peers; m; m &= m - 1u) s += __shfl_sync(peers, v[q], __ffs(m) - 1);
      v[q] = s;
    }
    if (lab >= 0 && lane == leader)
#pragma unroll
      for (int q = 0; q < 6; ++q) atomicAdd(out + (int64_t)lab * 6 + q, (unsigned long long)v[q]);
  }
}

// Stream-ordered launch over labels already resident on the device (the
// problem handle's int32 copy): zeroes out / bad, then accumulates.
cudaError_t launch_label_moments_i32(int M, int64_t P, const int32_t* labels0, int N,
                                     unsigned long long* out, int* bad, int sms, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, (size_t)N * 6 * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  const int64_t want = (P + 255) / 256;
  const int blocks = (int)(want < 8LL * sms ? want : 8LL * sms);
  k_label_moments<int32_t><<<blocks, 256, 0, s>>>(M, P, labels0, N, out, bad);
  return cudaGetLastError();
}

}  // namespace pgx

namespace {
thread_local std::string g_mom_error;
}

extern "C" const char* pgx_label_moments_error(void) { return g_mom_error.c_str(); }

extern "C" pgx_status pgx_label_moments(int resolution, int64_t n_points, const int64_t* labels0,
                                        int n_grains, int64_t* out) {
  g_mom_error.clear();
  if (resolution <= 0 || n_points != 4LL * resolution * resolution || !labels0 || !out || n_grains < 1) {
    g_mom_error = "pgx_label_moments: needs a regular 2-D grid (n_points = (2 resolution)^2), labels and output";
    return PGX_ERR_INVALID_ARGUMENT;
  }
  int64_t* d_lab = nullptr;
  unsigned long long* d_out = nullptr;
  int* d_bad = nullptr;
  auto fail = [&](cudaError_t e) {
    g_mom_error = std::string("pgx_label_moments: ") + cudaGetErrorString(e);
    cudaFree(d_lab);
    cudaFree(d_out);
    cudaFree(d_bad);
    return e == cudaErrorMemoryAllocation ? PGX_ERR_RESOURCE : PGX_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_lab, n_points * sizeof(int64_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&d_out, (size_t)n_grains * 6 * sizeof(unsigned long long))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&d_bad, sizeof(int))) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpy(d_lab, labels0, n_points * sizeof(int64_t), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e);
  cudaMemset(d_out, 0, (size_t)n_grains * 6 * sizeof(unsigned long long));
  cudaMemset(d_bad, 0, sizeof(int));
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n_points + 255) / 256;
  const int blocks = (int)(want < 8LL * sms ? want : 8LL * sms);
  pgx::k_label_moments<int64_t><<<blocks, 256>>>(resolution, n_points, d_lab, n_grains, d_out, d_bad);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  int bad = 0;
  if ((e = cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpy(out, d_out, (size_t)n_grains * 6 * sizeof(int64_t), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return fail(e);
  cudaFree(d_lab);
  cudaFree(d_out);
  cudaFree(d_bad);
  if (bad) {
    g_mom_error = "pgx_label_moments: labels must lie in [0, n_grains)";
    return PGX_ERR_INVALID_ARGUMENT;
  }
  return PGX_OK;
}
