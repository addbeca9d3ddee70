// Throughput probe of tcgen05.mma (kind::f16, M=128, K=16) on one SM: cycles
// per instruction for a given N, A source (SMEM or TMEM) and number of
// independent accumulators the instruction stream rotates over (1 = one
// dependent accumulation chain).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc \
//      -o tools/umma_tput tools/umma_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

template <int N, bool TS, int NACC, bool ACC, int NA = 1>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* out) {
  __shared__ __align__(1024) unsigned char sm[4 * 128 * 32 + 4 * 128 * 32];
  __shared__ uint64_t mbar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (int)sizeof(sm) / 4; e += 128) reinterpret_cast<unsigned*>(sm)[e] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
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
  if (warp == 0) {
    const uint64_t da = umma_desc(sb), db = umma_desc(sb + 4 * 4096);
    long long c0 = 0;
    for (int r = 0; r < iters + 1; ++r) {
      if (r == 1) {
        if (tid == 0) umma_commit(&mbar);
        __syncwarp();
        mbar_wait(&mbar, 0);
        c0 = clock64();
      }
      if (tid == 0) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const unsigned d = t + 256 + (unsigned)((u % NACC) * N) % 256;
          if (TS)
            umma_f16_ts(d, t + 8 * u, db + (uint64_t)((u % NA) * 4096 >> 4), idesc, ACC && (r > 0 || u >= NACC));
          else
            umma_f16_ss(d, da + (uint64_t)((u % NA) * 4096 >> 4), db + (uint64_t)((u % NA) * 4096 >> 4), idesc,
                        ACC && (r > 0 || u >= NACC));
        }
      }
      __syncwarp();
    }
    if (tid == 0) umma_commit(&mbar);
    __syncwarp();
    mbar_wait(&mbar, 1);
    if (tid == 0) out[0] = (clock64() - c0) * 100 / (16 * iters);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 512);
}

template <int N, bool TS>
void run(long long* d) {
  for (int accum = 0; accum < 2; ++accum)
    for (int nacc : {1, 2, 4}) {
      if (nacc * N > 256 && nacc > 1) continue;
      auto k = accum ? (nacc == 1 ? probe<N, TS, 1, true> : nacc == 2 ? probe<N, TS, 2, true> : probe<N, TS, 4, true>)
                     : (nacc == 1 ? probe<N, TS, 1, false> : nacc == 2 ? probe<N, TS, 2, false> : probe<N, TS, 4, false>);
      k<<<1, 128>>>(500, d);
      long long v = 0;
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("error\n");
        return;
      }
      cudaMemcpy(&v, d, sizeof(v), cudaMemcpyDeviceToHost);
      printf("%s N=%3d accumulate=%d accumulators=%d: %6.2f cycles/MMA (%.0f flop/clk)\n",
             TS ? "TS" : "SS", N, accum, nacc, v / 100.0, 2.0 * 128 * N * 16 / (v / 100.0));
    }
}

template <int N, bool TS>
void run_na(long long* d) {
  for (int na : {1, 2, 4}) {
    auto k = na == 1 ? probe<N, TS, 4, true, 1> : na == 2 ? probe<N, TS, 4, true, 2> : probe<N, TS, 4, true, 4>;
    k<<<1, 128>>>(500, d);
    long long v = 0;
    cudaDeviceSynchronize();
    cudaMemcpy(&v, d, sizeof(v), cudaMemcpyDeviceToHost);
    printf("%s N=%3d distinct operand tiles=%d: %6.2f cycles/MMA\n", TS ? "TS" : "SS", N, na, v / 100.0);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  run_na<32, false>(d);
  run_na<64, false>(d);
  run_na<128, false>(d);
  run_na<32, true>(d);
  run_na<64, true>(d);
  return 0;
}
