// Latency of a tcgen05.mma chain: issue NM MMAs (kind::f16, M=128, K=16, N)
// then tcgen05.commit -> mbarrier, and wait for it: cycles from the first
// issue to the observed completion (1 thread, C CTAs per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc -o tools/probe_lat tools/probe_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

template <int N, bool TS, int NM>
__global__ void __launch_bounds__(128, 2) lat(int reps, long long* out) {
  __shared__ __align__(1024) unsigned char sm[2 * 4096 + 2 * 8192];
  __shared__ uint64_t mbar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (int)sizeof(sm) / 4; e += 128) reinterpret_cast<unsigned*>(sm)[e] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  constexpr uint32_t idesc = umma_idesc_f16(128, N);
  long long tot = 0;
  if (warp == 0) {
    const uint64_t da = umma_desc(sb), db = umma_desc(sb + 2 * 4096);
    for (int r = 0; r < reps; ++r) {
      const long long c0 = clock64();
      if (tid == 0) {
#pragma unroll
        for (int u = 0; u < NM; ++u) {
          if (TS)
            umma_f16_ts(t + 128, t + 8 * (u & 3), db, idesc, u > 0);
          else
            umma_f16_ss(t + 128, da, db, idesc, u > 0);
        }
        umma_commit(&mbar);
      }
      __syncwarp();
      mbar_wait(&mbar, (unsigned)r & 1u);
      tot += clock64() - c0;
    }
    if (tid == 0) out[blockIdx.x] = tot / reps;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 256);
}

template <int N, bool TS, int NM>
void run(long long* d, int grid) {
  lat<N, TS, NM><<<grid, 128>>>(200, d);
  long long h = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("error\n");
    return;
  }
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s N=%3d x%2d MMAs + commit -> wait: %6lld cycles (grid %d)\n", TS ? "TS" : "SS", N, NM, h, grid);
}

int main() {
  long long* d;
  cudaMalloc(&d, 4096 * sizeof(long long));
  for (int grid : {1, 296}) {
    run<32, true, 0>(d, grid);
    run<32, true, 1>(d, grid);
    run<32, true, 2>(d, grid);
    run<32, true, 8>(d, grid);
    run<64, false, 2>(d, grid);
    run<64, false, 1>(d, grid);
    run<32, true, 16>(d, grid);
  }
  return 0;
}
