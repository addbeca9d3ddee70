// Latency probe of the pass-2 tensor-core chain on one SM (clock64 around
// issue -> commit -> mbarrier wait), averaged over many rounds:
//   mode 0: UMMA 1 only      (KS x SS 128x64x16)
//   mode 1: UMMA 2 only      (12 x TS 128x16x16)
//   mode 2: UMMA 2 + UMMA 1  (the producer's per-tile chain)
//   mode 3: UMMA 2 as 4 x TS 128x32x16 + 4 x TS 128x16x16 (hi . [L_hi|L_lo], lo . L_hi)
//   mode 4: 12 x SS 128x16x16 (A from shared memory)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc \
//      -o tools/umma_lat tools/umma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

__global__ void __launch_bounds__(128, 1) probe(int mode, int rounds, long long* out, int pipelined) {
  __shared__ __align__(1024) unsigned char sm[128 * 32 * 4 + 64 * 32 * 2];
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
  if (tid == 0) {
    unsigned phase = 0;
    long long total = 0;
    for (int r = 0; r < rounds + 4; ++r) {
      const long long c0 = clock64();
      if (mode == 0 || mode == 2 || mode == 5) {
        if (mode == 2)
          for (int s = 0; s < 12; ++s)
            umma_f16_ts(t + 128, t + 8 * (s % 8), umma_desc(sb + (s % 4) * 512), umma_idesc_f16(128, 16), s > 0);
        for (int s = 0; s < 2; ++s)
          umma_f16_ss(t, umma_desc(sb + s * 4096), umma_desc(sb + 16384 + s * 2048), umma_idesc_f16(128, 64), s > 0);
      } else if (mode == 1) {
        for (int s = 0; s < 12; ++s)
          umma_f16_ts(t + 128, t + 8 * (s % 8), umma_desc(sb + (s % 4) * 512), umma_idesc_f16(128, 16), s > 0);
      } else if (mode == 3) {
        for (int s = 0; s < 4; ++s)
          umma_f16_ts(t + 128, t + 8 * s, umma_desc(sb + s * 1024), umma_idesc_f16(128, 32), s > 0);
        for (int s = 0; s < 4; ++s)
          umma_f16_ts(t + 160, t + 32 + 8 * s, umma_desc(sb + s * 512), umma_idesc_f16(128, 16), s > 0);
      } else if (mode == 4) {
        for (int s = 0; s < 12; ++s)
          umma_f16_ss(t + 128, umma_desc(sb + (s % 4) * 4096), umma_desc(sb + 16384 + (s % 4) * 512),
                      umma_idesc_f16(128, 16), s > 0);
      }
      if (!pipelined || r == rounds + 3 || r == 3) {
        umma_commit(&mbar);
        mbar_wait(&mbar, phase);
        phase ^= 1u;
      }
      const long long c1 = clock64();
      if (r >= 4) total += c1 - c0;
    }
    out[mode] = total / rounds;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const char* names[] = {"UMMA1 (2 x SS 128x64x16)", "UMMA2 (12 x TS 128x16x16)", "UMMA2 + UMMA1",
                         "UMMA2 as 4 x TS N32 + 4 x TS N16", "12 x SS 128x16x16"};
  for (int pl = 0; pl < 2; ++pl)
  for (int m = 0; m < 5; ++m) {
    probe<<<1, 128>>>(m, 200, d, pl);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("error in mode %d\n", m);
      return 1;
    }
    long long v;
    cudaMemcpy(&v, d + m, sizeof(v), cudaMemcpyDeviceToHost);
    printf("%-12s %-36s %6lld cycles\n", pl ? "throughput" : "latency", names[m], v);
  }
  return 0;
}
