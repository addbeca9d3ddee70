// What does a thread-side TMEM store cost next to tcgen05.mma traffic? (B200)
// One CTA per SM (C = 1 or 2), 4 epilogue warps + 1 issuer warp, per round:
//   issuer: UMMA 1 (SS) D -> S columns; commit -> bar_s
//   epilogue: wait bar_s; tcgen05.ld S; [tcgen05.st to X]; wait::st; fence; arrive bar_p
//   issuer: wait bar_p; [UMMA 2 (TS) with A = Y]; commit -> bar_d; wait bar_d
// MODE 0: no store            (ld only)
// MODE 1: store over S        (X = S, Y = S: the k_tc_grad scheme)
// MODE 2: store to a separate region, MMA reads it (X = Y = other columns)
// MODE 3: store to a region no MMA touches (X = scratch), MMA reads S
// MODE 4: as 1 but without UMMA 2
// Second part (kb): the issuer streams SS MMAs (N = 32, one accumulator) back to back
// with no hand-shake while the 4 epilogue warps loop ld -> st -> wait::st on columns no
// MMA touches: cycles per ld/st iteration with and without the MMA stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc -o tools/st_hazard tools/st_hazard.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

template <int MODE>
__global__ void __launch_bounds__(160, 2) k(int rounds, long long* out) {
  __shared__ __align__(1024) unsigned char sm[2 * 4096 + 2 * 8192];
  __shared__ uint64_t bar_s, bar_p, bar_d;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < (int)sizeof(sm) / 4; e += 160) reinterpret_cast<unsigned*>(sm)[e] = 0x3c003c00u;
  if (warp == 4) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&bar_s, 1);
    mbar_init(&bar_p, 4);
    mbar_init(&bar_d, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  constexpr uint32_t id1 = umma_idesc_f16(128, 64), id2 = umma_idesc_f16(128, 32);
  const long long c0 = clock64();
  if (warp == 4) {
    if (elect_one()) {
      const uint64_t da = umma_desc(sb), db = umma_desc(sb + 2 * 4096);
      for (int r = 0; r < rounds; ++r) {
        umma_f16_ss(t, da, db, id1, false);
        umma_f16_ss(t, da + (4096 >> 4), db + (8192 >> 4), id1, true);
        umma_commit(&bar_s);
        mbar_wait(&bar_p, r & 1);
        tc_fence_after();
        if (MODE != 4) {
          const unsigned a = MODE == 2 ? t + 64 : t;
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ts(t + 192, a + 8u * (s & 3) + (s >= 4 ? 16u : 0u), db + (uint64_t)((s & 3) * 1024 >> 4), id2,
                        s > 0);
        }
        umma_commit(&bar_d);
        mbar_wait(&bar_d, r & 1);
        tc_fence_after();
      }
    }
    __syncwarp();
  } else {
    const unsigned lane_off = (unsigned)(32 * warp) << 16;
    uint32_t v[32];
    for (int r = 0; r < rounds; ++r) {
      mbar_wait(&bar_s, r & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        tmem_ld32_nowait(t + lane_off + 32u * h, v);
        tmem_ld_wait();
        tmem_regs_ready(v);
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = (v[e] & 0x03ff03ffu) | 0x3c003c00u;
        if (MODE == 1 || MODE == 4) tmem_st32(t + lane_off + 32u * h, v);
        if (MODE == 2) tmem_st32(t + lane_off + 64u + 32u * h, v);
        if (MODE == 3) tmem_st32(t + lane_off + 128u + 32u * h, v);
        if (MODE == 0) asm volatile("" ::"r"(v[0] ^ v[7] ^ v[31]));
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p);
    }
  }
  if (tid == 0) out[blockIdx.x] = clock64() - c0;
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc(t, 256);
}

template <bool MMA, bool ST>
__global__ void __launch_bounds__(160, 2) kb(int rounds, long long* out) {
  __shared__ __align__(1024) unsigned char sm[2 * 4096 + 2 * 8192];
  __shared__ uint64_t bar_d;
  __shared__ unsigned tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < (int)sizeof(sm) / 4; e += 160) reinterpret_cast<unsigned*>(sm)[e] = 0x3c003c00u;
  if (warp == 4) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&bar_d, 1);
    stop = 0;
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  constexpr uint32_t id2 = umma_idesc_f16(128, 32);
  if (warp == 4) {
    if (MMA && elect_one()) {
      const uint64_t da = umma_desc(sb), db = umma_desc(sb + 2 * 4096);
      int n = 0;
      while (!stop) {
#pragma unroll
        for (int s = 0; s < 8; ++s) umma_f16_ss(t + 192, da, db, id2, true);
        if (++n % 8 == 0) {  // bound the queue: wait for the batch every 64 MMAs
          umma_commit(&bar_d);
          mbar_wait(&bar_d, ((n / 8) - 1) & 1);
        }
      }
    }
    __syncwarp();
  } else {
    const unsigned lane_off = (unsigned)(32 * warp) << 16;
    uint32_t v[32];
    const long long c0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      tmem_ld32_nowait(t + lane_off + 32u * (r & 1), v);
      tmem_ld_wait();
      tmem_regs_ready(v);
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] += 1;
      if (ST) {
        tmem_st32(t + lane_off + 64u + 32u * (r & 1), v);
        tmem_st_wait();
      } else {
        asm volatile("" ::"r"(v[0] ^ v[9] ^ v[31]));
      }
    }
    if (lane == 0 && warp == 0) out[blockIdx.x] = clock64() - c0;
    __syncwarp();
    if (tid == 0) stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc(t, 256);
}

template <bool MMA, bool ST>
void runb(long long* d, int ctas) {
  const int rounds = 4000;
  kb<MMA, ST><<<148 * ctas, 160>>>(100, d);
  kb<MMA, ST><<<148 * ctas, 160>>>(rounds, d);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("kb: error %s\n", cudaGetErrorString(cudaGetLastError()));
    return;
  }
  long long h[296];
  cudaMemcpy(h, d, sizeof(long long) * 148 * ctas, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148 * ctas; ++i) avg += h[i];
  printf("ld%s per iteration, MMA stream %s, %d CTA/SM: %.0f cycles\n", ST ? " + st + wait::st" : " only",
         MMA ? "ON " : "off", ctas, avg / (148.0 * ctas) / rounds);
}

template <int MODE>
void run(long long* d, int ctas) {
  const int rounds = 2000;
  k<MODE><<<148 * ctas, 160>>>(50, d);
  k<MODE><<<148 * ctas, 160>>>(rounds, d);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("mode %d: error %s\n", MODE, cudaGetErrorString(cudaGetLastError()));
    return;
  }
  long long h[296];
  cudaMemcpy(h, d, sizeof(long long) * 148 * ctas, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148 * ctas; ++i) avg += h[i];
  printf("mode %d, %d CTA/SM: %.0f cycles per round\n", MODE, ctas, avg / (148.0 * ctas) / rounds);
}

int main() {
  long long* d;
  cudaMalloc(&d, 512 * sizeof(long long));
  for (int c = 1; c <= 2; ++c) {
    run<0>(d, c);
    run<1>(d, c);
    run<2>(d, c);
    run<3>(d, c);
    run<4>(d, c);
  }
  for (int c = 1; c <= 2; ++c) {
    runb<false, false>(d, c);
    runb<true, false>(d, c);
    runb<false, true>(d, c);
    runb<true, true>(d, c);
  }
  return 0;
}
