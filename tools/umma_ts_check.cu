// Layout/ordering probe for tcgen05.mma with the A operand in TMEM (kind::f16):
//   D[128 x 16] = A[128 x 64] . B[16 x 64]^T, A written to TMEM by tcgen05.st as
//   packed fp16 pairs (column c of lane m = A[m][2c] | A[m][2c+1] << 16).
// Each round: store A, issue 4 TS MMAs into D, then IMMEDIATELY an SS MMA that
// overwrites the A columns with zeros (write-after-read through the in-order
// tensor pipe), commit, check D against the host product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_20816_b200/csrc \
//      -o tools/umma_ts_check tools/umma_ts_check.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "pgx_tc_common.cuh"

using namespace pgx;

__host__ __device__ inline int aval(int m, int k, int r) { return ((m * 7 + k * 3 + r) % 11) - 5; }
__host__ __device__ inline int bval(int n, int k) { return ((n * 5 + k) % 7) - 3; }

__global__ void __launch_bounds__(128, 1) probe(int rounds, float* out) {
  __shared__ __align__(1024) unsigned char sb[4 * 16 * 32];        // B: 4 K slabs x 16 rows
  __shared__ __align__(1024) unsigned char sz[128 * 32 + 64 * 32];  // zero operands for the SS overwrite
  __shared__ uint64_t mbar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 16 * 64; e += 128) {
    const int n = e / 64, k = e % 64;
    *reinterpret_cast<__half*>(sb + (k / 16) * 512 + slab_off(n, k % 16)) = __float2half((float)bval(n, k));
  }
  for (int e = tid; e < (int)sizeof(sz) / 4; e += 128) reinterpret_cast<unsigned*>(sz)[e] = 0u;
  if (warp == 0) tmem_alloc(&tbase, 128);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned t = tbase, lane_off = (unsigned)(warp * 32) << 16;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sb);
  const unsigned zbase = (unsigned)__cvta_generic_to_shared(sz);
  unsigned phase = 0;
  for (int r = 0; r < rounds; ++r) {
    // A row tid into columns [0, 32) as packed pairs
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int k = 2 * (c0 + c);
        const __half2 h = __halves2half2(__float2half((float)aval(tid, k, r)),
                                         __float2half((float)aval(tid, k + 1, r)));
        v[c] = *reinterpret_cast<const uint32_t*>(&h);
      }
      tmem_st16(t + lane_off + c0, v);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      for (int s = 0; s < 4; ++s)
        umma_f16_ts(t + 64, t + s * 8, umma_desc(sbase + s * 512), umma_idesc_f16(128, 16), s > 0);
      // overwrite the A columns right away: S[128 x 64] = 0 . 0^T into columns [0, 64)
      umma_f16_ss(t, umma_desc(zbase), umma_desc(zbase + 128 * 32), umma_idesc_f16(128, 64), false);
      umma_commit(&mbar);
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    tc_fence_after();
    float d[32];
    tmem_ld32(t + lane_off + 64, d);
    for (int n = 0; n < 16; ++n) out[((size_t)r * 128 + tid) * 16 + n] = d[n];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 128);
}

int main() {
  const int rounds = 8;
  float* d_out;
  cudaMalloc(&d_out, sizeof(float) * rounds * 128 * 16);
  probe<<<1, 128>>>(rounds, d_out);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(err));
    return 1;
  }
  static float h[rounds * 128 * 16];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int r = 0; r < rounds; ++r)
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 16; ++n) {
        long ref = 0;
        for (int k = 0; k < 64; ++k) ref += (long)aval(m, k, r) * bval(n, k);
        const float got = h[((size_t)r * 128 + m) * 16 + n];
        if (got != (float)ref) {
          if (bad < 5) printf("r=%d m=%d n=%d got %g ref %ld\n", r, m, n, got, ref);
          ++bad;
        }
      }
  printf("umma_ts_check: %ld mismatches of %d\n", bad, rounds * 128 * 16);
  return bad != 0;
}
