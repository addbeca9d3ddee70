// Producer/consumer mbarrier ping-pong on one SM: 1 producer warp, C consumer
// warps, B buffers.  Producer: wait empty[b] -> (MMA + commit | plain arrive)
// -> full[b]; consumers: wait full[b] -> arrive empty[b].  Cycles per round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc -o tools/pingpong tools/pingpong.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

__global__ void __launch_bounds__(544, 1) k(int nb, int nc, int mode, int rounds, long long* out, int flags) {
  __shared__ __align__(1024) unsigned char sm[8192 + 4096];
  __shared__ uint64_t full[8], empty[8];
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < (int)sizeof(sm) / 4; e += blockDim.x) reinterpret_cast<unsigned*>(sm)[e] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    for (int b = 0; b < 8; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], nc);
    }
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  long long c0 = clock64();
  if (warp == nc) {
    for (int r = 0; r < rounds; ++r) {
      const int b = r % nb;
      mbar_wait(&empty[b], (unsigned)((r / nb) & 1) ^ 1u);
      tc_fence_after();
      if (lane == 0) {
        if (mode == 0) {
          mbar_arrive(&full[b]);
        } else {
          for (int k = 0; k < mode; ++k)
            umma_f16_ss(t + (unsigned)(b * 32), umma_desc(sb), umma_desc(sb + 8192), umma_idesc_f16(128, 32), k > 0);
          umma_commit(&full[b]);
        }
      }
      __syncwarp();
    }
  } else if (warp < nc) {
    for (int r = 0; r < rounds; ++r) {
      const int b = r % nb;
      if (flags & 4)
        mbar_wait_addr((unsigned)__cvta_generic_to_shared(&full[b]), (unsigned)((r / nb) & 1));
      else
        mbar_wait(&full[b], (unsigned)((r / nb) & 1));
      if (!(flags & 2)) tc_fence_after();
      if (!(flags & 1)) {
        uint32_t v[32];
        tmem_ld32_nowait(t + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(b * 32), v);
        tmem_ld_wait();
        tmem_regs_ready(v);
      }
      if (!(flags & 2)) tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
      if (flags & 8) {  // ~1000 cycles of dependent-free work after the release
        float a0 = r, a1 = r + 1, a2 = r + 2, a3 = r + 3;
#pragma unroll 1
        for (int i = 0; i < 64; ++i) {
          a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 1.0001f, 0.5f);
          a2 = fmaf(a2, 1.0001f, 0.5f); a3 = fmaf(a3, 1.0001f, 0.5f);
        }
        if (a0 + a1 + a2 + a3 == 1.2345f) out[1] = 1;
      }
    }
  }
  __syncthreads();
  if (tid == 0) out[0] = (clock64() - c0) / rounds;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int flags : {0, 8})
  for (int mode : {0, 8})
    for (int nc : {16})
      for (int nb : {1, 2, 4, 8}) {
        k<<<1, (nc + 1) * 32>>>(nb, nc, mode, 2000, d, flags);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
        long long v;
        cudaMemcpy(&v, d, 8, cudaMemcpyDeviceToHost);
        printf("flags=%d mmas/round=%d consumers=%2d buffers=%d: %lld cycles/round\n", flags, mode, nc, nb, v);
      }
  return 0;
}
