// tcgen05.mma issue / dependency probe (B200): M=128, K=16, kind::f16, TS or SS.
// W issuing warps per CTA, each rotating over NACC accumulators of N columns;
// C CTAs per SM.  NACC=1 gives the dependent-accumulate interval, large NACC the
// per-thread issue interval; W>1 shows whether several issuing threads of one
// CTA overlap.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc \
//      -o tools/umma_dep tools/umma_dep.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

template <int N, bool TS>
__global__ void __launch_bounds__(128) probe(int iters, int nacc, int W, unsigned cols, long long* out) {
  __shared__ __align__(1024) unsigned char sm[2 * 4096 + 2 * 8192];
  __shared__ uint64_t mbar[4];
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < (int)sizeof(sm) / 4; e += 128) reinterpret_cast<unsigned*>(sm)[e] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, cols);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&mbar[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  constexpr uint32_t idesc = umma_idesc_f16(128, N);
  if (warp < W) {
    const uint64_t da = umma_desc(sb), db = umma_desc(sb + 2 * 4096);
    const long long c0 = clock64();
    if (lane == 0) {
      int a = 0;
      for (int r = 0; r < iters * 16; ++r) {
        const unsigned d = t + 64 + (unsigned)((warp * nacc + a) * N);
        if (TS)
          umma_f16_ts(d, t + 16 * (r & 3), db + (uint64_t)((r & 1) * 8192 >> 4), idesc, r >= nacc);
        else
          umma_f16_ss(d, da + (uint64_t)((r & 1) * 4096 >> 4), db + (uint64_t)((r & 1) * 8192 >> 4), idesc,
                      r >= nacc);
        if (++a == nacc) a = 0;
      }
      umma_commit(&mbar[warp]);
    }
    __syncwarp();
    mbar_wait(&mbar[warp], 0);
    if (lane == 0) out[blockIdx.x * 4 + warp] = clock64() - c0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, cols);
}

template <int N, bool TS>
void run(long long* d, int sms, int C, int nacc, int W) {
  const int iters = 200;
  const unsigned cols = 512 / C;
  if (64 + W * nacc * N > (int)cols) return;
  probe<N, TS><<<sms * C, 128>>>(10, nacc, W, cols, d);
  probe<N, TS><<<sms * C, 128>>>(iters, nacc, W, cols, d);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
    return;
  }
  long long h[148 * 4 * 4];
  cudaMemcpy(h, d, sizeof(long long) * sms * C * 4, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms * C; ++i) avg += h[4 * i];
  avg /= sms * C;
  printf("%s N=%2d CTAs/SM=%d warps=%d nacc=%d: %6.1f clk/MMA per issuing thread, %6.1f per CTA, %6.1f per SM\n",
         TS ? "TS" : "SS", N, C, W, nacc, avg / (16.0 * iters), avg / (16.0 * iters * W), avg / (16.0 * iters * W * C));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 4 * 4 * sizeof(long long));
  for (int C = 1; C <= 2; ++C)
    for (int W = 1; W <= 2; ++W)
      for (int nacc : {1, 2, 4}) {
        run<32, true>(d, 148, C, nacc, W);
        run<64, false>(d, 148, C, nacc, W);
      }
  run<32, true>(d, 148, 1, 6, 2);
  run<32, true>(d, 148, 1, 3, 4);
  return 0;
}
