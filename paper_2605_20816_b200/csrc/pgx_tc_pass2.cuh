// pgx_tc_pass2.cuh — PGX_PREC_TC pass 2: the gradient contraction
// sum_x (onehot_G(x) - p(x)) eta(x) (objective.py:109-113) with BOTH
// contractions on the tensor cores (FlashAttention-backward-like, grain-major):
//
//   UMMA 1  S^T[128 grains x 64 px] = B''(line)[grains x 3J] . L(x)[px x 3J]^T
//   epilogue (thread = grain = TMEM lane): p/2 = 2^(w_x - h~''), r/2 = label ?
//           q_x : -p/2, split into fp16 hi/lo, stored as the K-major A operand
//   UMMA 2  R[128 grains x 16] += [r_hi r_hi r_lo] . [L_hi L_lo L_hi]^T
//           (K = 3 x 64 pixels, fp32 accumulate in TMEM)
//
// R is flushed every 4 tiles into fp64 line sums and expanded per line into
// the K gradient rows (fp64 shared memory), as in the CUDA-core grid pass 2.
// CTA: 128 threads, one 128-grain tile, a range of lines; TMEM: 64 + 16
// columns (alloc 128) so 4 CTAs share an SM.
#pragma once

#include "pgx_grid_common.cuh"
#include "pgx_tc_coeffs.cuh"
#include "pgx_tc_common.cuh"

namespace pgx {

constexpr int kTc2Threads = 128;
constexpr int kTc2Px = 64;        // pixels per tile (UMMA 1 N, UMMA 2 K per product)
constexpr int kTc2Flush = 4;      // tiles per fp32 -> fp64 flush of R
constexpr float kTc2RScale = 8192.0f;  // r/2 scaled by 2^13 into the fp16 range

template <int J>
struct TcP2Smem {
  static constexpr int KS = tc_ksteps(J);
  static constexpr int A1 = KS * kTc2Threads * 32;   // B'' operand (128 rows)
  static constexpr int B1 = KS * kTc2Px * 32;        // L operand (64 rows)
  static constexpr int RPART = (kTc2Px / 16) * kTc2Threads * 32;  // r_hi or r_lo (16 KB)
  static constexpr int LPART = (kTc2Px / 16) * 16 * 32;           // L_hi or L_lo (2 KB)
  static constexpr int A1_OFF = 0;
  static constexpr int B1_OFF = A1_OFF + A1;
  static constexpr int RH_OFF = B1_OFF + B1;
  static constexpr int RL_OFF = RH_OFF + RPART;
  static constexpr int LH_OFF = RL_OFF + RPART;
  static constexpr int LL_OFF = LH_OFF + LPART;
  static constexpr int TOTAL = LL_OFF + LPART;
};

template <int DIM, int D>
__global__ void __launch_bounds__(kTc2Threads, 4) k_tc_pass2(GridParams g) {
  constexpr int J = D + 1;
  constexpr int K = feature_count(DIM, D);
  using L = TcP2Smem<J>;
  constexpr int KS = L::KS;
  constexpr uint32_t IDESC1 = umma_idesc_f16(128, kTc2Px);
  constexpr uint32_t IDESC2 = umma_idesc_f16(128, 16);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ double lc[K];
  __shared__ __align__(16) float w_s[kTc2Px], wl_s[kTc2Px], q_s[kTc2Px];
  __shared__ __align__(16) int lab_s[kTc2Px];
  __shared__ uint64_t mbar;
  __shared__ unsigned tmem_base;
  __shared__ unsigned s_bmax;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int i = blockIdx.x * kTc2Threads + tid;  // this thread's grain (TMEM lane)
  const bool active = i < g.N;
  const int64_t l0 = (int64_t)blockIdx.y * g.lines_per_split;
  const int64_t l1 = min((int64_t)g.lines, l0 + g.lines_per_split);

  if (warp == 0) tmem_alloc(&tmem_base, 128);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  // fp64 gradient rows of this thread's grain accumulate in place in part_g
  double* acc = g.part_g + (int64_t)blockIdx.y * K * g.N + (active ? i : 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = tmem_base;
  const unsigned t_s = tmem;        // S^T: columns [0, 64)
  const unsigned t_r = tmem + 64;   // R:   columns [64, 80)
  const unsigned lane_off = (unsigned)(warp * 32) << 16;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  unsigned phase = 0;

  auto sync_tc = [&]() {
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };
  auto wait_mma = [&]() {
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    tc_fence_after();
  };

  for (int64_t line = l0; line < l1; ++line) {
    // ---- per line: the precomputed operand image of this 128-grain tile (A of UMMA 1)
    __syncthreads();
    if (tid == 0) {
      double lcr[K];
      line_factors<DIM, D>(line, g, lcr);
#pragma unroll
      for (int k = 0; k < K; ++k) lc[k] = lcr[k];
    }
    const int64_t ci = line * g.tc_nchunks + blockIdx.x;
    copy_coef_img<J, kTc2Threads>(smem + L::A1_OFF, g.tc_img + ci * tc_img_bytes<J>(), tid);
    const int sB = g.tc_meta[ci].x;
    __syncthreads();
    const float inv = ldexpf(1.0f, -(sB + 10));  // S * inv = h~''
    double R64[J];
#pragma unroll
    for (int j = 0; j < J; ++j) R64[j] = 0.0;
    const int64_t pline = line * g.side;
    const int ntiles = g.side / kTc2Px;

    for (int t = 0; t < ntiles; ++t) {
      // ---- per tile: pixel operands (UMMA 1 B, UMMA 2 B) and per-pixel records
      if (tid < kTc2Px) {
        const int col = t * kTc2Px + tid;
        double u[J];
        axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
        __half hi[J], lo[J];
#pragma unroll
        for (int j = 0; j < J; ++j) split_f16(u[j] * 1024.0, hi[j], lo[j]);
#pragma unroll
        for (int k = 0; k < 16 * KS; ++k) {
          const int b = k / J, j = k % J;
          const __half val = k < 3 * J ? (b < 2 ? hi[j] : lo[j]) : __float2half(0.0f);
          *reinterpret_cast<__half*>(smem + L::B1_OFF + (k / 16) * (kTc2Px * 32) +
                                     slab_off(tid, k % 16)) = val;
        }
        // UMMA 2 B operand: rows j (N = 16), K = pixels
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const __half h = j < J ? hi[j] : __float2half(0.0f);
          const __half l = j < J ? lo[j] : __float2half(0.0f);
          const unsigned off = (tid / 16) * (16 * 32) + slab_off(j, tid % 16);
          *reinterpret_cast<__half*>(smem + L::LH_OFF + off) = h;
          *reinterpret_cast<__half*>(smem + L::LL_OFF + off) = l;
        }
        const double wd = g.pix_w[pline + col];
        w_s[tid] = (float)wd;
        wl_s[tid] = (float)(wd - (double)(float)wd);
        q_s[tid] = g.pix_q[pline + col] * kTc2RScale;
        lab_s[tid] = g.labels[pline + col];
      }
      sync_tc();
      if (tid == 0) {
#pragma unroll
        for (int s = 0; s < KS; ++s)
          umma_f16_ss(t_s, umma_desc(sbase + L::A1_OFF + s * (kTc2Threads * 32)),
                      umma_desc(sbase + L::B1_OFF + s * (kTc2Px * 32)), IDESC1, s > 0);
        umma_commit(&mbar);
      }
      wait_mma();

      // ---- epilogue: r/2 * 2^13 as fp16 hi/lo into the UMMA 2 A operand
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[32];
        tmem_ld32(t_s + lane_off + half * 32, v);
#pragma unroll
        for (int q8 = 0; q8 < 32; q8 += 8) {
          uint32_t ph[4], pl[4];
          float wv[8], wlv[8], qv[8];
          int lv[8];
          {  // per-pixel records of these 8 pixels: 128-bit broadcast loads
            const int x0 = half * 32 + q8;
            *reinterpret_cast<float4*>(wv) = *reinterpret_cast<const float4*>(w_s + x0);
            *reinterpret_cast<float4*>(wv + 4) = *reinterpret_cast<const float4*>(w_s + x0 + 4);
            *reinterpret_cast<float4*>(wlv) = *reinterpret_cast<const float4*>(wl_s + x0);
            *reinterpret_cast<float4*>(wlv + 4) = *reinterpret_cast<const float4*>(wl_s + x0 + 4);
            *reinterpret_cast<float4*>(qv) = *reinterpret_cast<const float4*>(q_s + x0);
            *reinterpret_cast<float4*>(qv + 4) = *reinterpret_cast<const float4*>(q_s + x0 + 4);
            *reinterpret_cast<int4*>(lv) = *reinterpret_cast<const int4*>(lab_s + x0);
            *reinterpret_cast<int4*>(lv + 4) = *reinterpret_cast<const int4*>(lab_s + x0 + 4);
          }
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            float rr[2];
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) {
              const int xe = e + u2;
              const float a = fmaf(v[q8 + xe], inv, -wv[xe]) - wlv[xe];  // h'' - w >= 1
              const float p2 = ex2_approx(13.0f - a);                     // (p/2) 2^13
              rr[u2] = (lv[xe] == i) ? qv[xe] : -p2;
            }
            const __half2 h2 = __floats2half2_rn(rr[0], rr[1]);
            const float2 hf = __half22float2(h2);
            const __half2 l2 = __floats2half2_rn(rr[0] - hf.x, rr[1] - hf.y);
            ph[e / 2] = *reinterpret_cast<const uint32_t*>(&h2);
            pl[e / 2] = *reinterpret_cast<const uint32_t*>(&l2);
          }
          // 8 consecutive pixels (k) of row tid = one 16-byte core-matrix row
          const int x0 = half * 32 + q8;
          const unsigned off = (x0 / 16) * (kTc2Threads * 32) + slab_off(tid, x0 % 16);
          *reinterpret_cast<uint4*>(smem + L::RH_OFF + off) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
          *reinterpret_cast<uint4*>(smem + L::RL_OFF + off) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
        }
      }
      sync_tc();
      if (tid == 0) {
        const bool fresh = (t % kTc2Flush) == 0;
#pragma unroll
        for (int s = 0; s < 3 * (kTc2Px / 16); ++s) {
          const int p = s / (kTc2Px / 16), ks = s % (kTc2Px / 16);
          const unsigned a_off = (p < 2 ? L::RH_OFF : L::RL_OFF) + ks * (kTc2Threads * 32);
          const unsigned b_off = (p == 1 ? L::LL_OFF : L::LH_OFF) + ks * (16 * 32);
          umma_f16_ss(t_r, umma_desc(sbase + a_off), umma_desc(sbase + b_off), IDESC2,
                      !(fresh && s == 0));
        }
        umma_commit(&mbar);
      }
      wait_mma();
      if ((t % kTc2Flush) == kTc2Flush - 1 || t == ntiles - 1) {
        float v[32];
        tmem_ld32(t_r + lane_off, v);
#pragma unroll
        for (int j = 0; j < J; ++j) R64[j] += (double)v[j];
        tc_fence_before();
      }
    }
    // R_j = 2 * sum (r/2) L_j = 2 * acc * 2^-(13 + 10): expand into the K rows
    const double rs = 2.0 / (8192.0 * 1024.0);
    if (active) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double prev = line == l0 ? 0.0 : acc[(int64_t)k * g.N];
        acc[(int64_t)k * g.N] = fma(lc[k], rs * R64[alpha_of(DIM, D, k, DIM - 1)], prev);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

}  // namespace pgx
