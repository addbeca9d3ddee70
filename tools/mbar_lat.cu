// mbarrier primitive costs on one SM: a single warp (or W warps on separate
// barriers) loops { arrive; wait(phase) } on a count-1 barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc -o tools/mbar_lat tools/mbar_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

__global__ void k(int mode, int rounds, long long* out) {
  __shared__ uint64_t bar[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 32) mbar_init(&bar[tid], 1);
  fence_mbar_init();
  __syncthreads();
  const long long c0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if (lane == 0) {
      if (mode >= 2)
        asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&bar[warp]))
                     : "memory");
      else
        mbar_arrive(&bar[warp]);
    }
    __syncwarp();
    if (mode == 0 || mode == 2)
      mbar_wait(&bar[warp], (unsigned)(r & 1));
    else if (mode == 4) {
      unsigned done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"((unsigned)__cvta_generic_to_shared(&bar[warp])), "r"((unsigned)(r & 1)) : "memory");
    }
    else
      mbar_wait_addr((unsigned)__cvta_generic_to_shared(&bar[warp]), (unsigned)(r & 1));
  }
  const long long c1 = clock64();
  if (tid == 0) out[0] = (c1 - c0) / rounds;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int mode = 0; mode < 5; ++mode)
    for (int w : {1, 4, 16}) {
      k<<<1, 32 * w>>>(mode, 10000, d);
      cudaDeviceSynchronize();
      long long v;
      cudaMemcpy(&v, d, 8, cudaMemcpyDeviceToHost);
      const char* nm[] = {"release arrive + try_wait", "release arrive + test_wait", "relaxed arrive + try_wait", "relaxed arrive + test_wait", "relaxed arrive + relaxed try_wait"};
      printf("%s warps=%2d: %lld cycles\n", nm[mode], w, v);
    }
  return 0;
}
