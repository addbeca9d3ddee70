// pgx_grid_pass1.cuh — regular-grid pass 1 (pixel-major): per-pixel min,
// arg-min and log-sum-exp over all grains (objective.py:99-106,115-119;
// geometry.py:201-210), fp64 logits, branch-free inner loops.
//
// One CTA = 128 threads x R pixels of one line.  Grains stream through shared
// memory in chunks of 128 whose line coefficients B'' are built cooperatively.
//
//   sweep A (fp32, FMA/ALU pipes): approximate min b1, runner-up b2 and arg-min
//           of h'' with a CTA-wide rounding bound delta;
//   sweep B (fp64 logits): s' = sum_{i != G} 2^(ref - h''_i) with the fixed
//           reference ref = b1 - delta - 1 <= min h'' - 1, so every exponent
//           argument a = h'' - ref is >= 1 (no rescaling, no overflow, a valid
//           domain for the integer RN conversion) and one MUFU.EX2 per logit.
//
// Arg-min: if b2 - b1 exceeds 2 delta + tie tolerance + ambiguity band the
// fp32 arg-min is the exact tie-tolerant arg-min; otherwise the pixel is
// queued for the exact fp64 re-scan of the tail kernel (which also decides
// its ambiguity).  The label term is excluded from s' so that
// 1 - p_G = sum_{j != G} p_j keeps full relative precision.
#pragma once

#include "pgx_grid_common.cuh"

namespace pgx {

constexpr int kG1Threads = 128;
constexpr int kG1Chunk = 128;
constexpr int kG1Flush = 16;  // fp32 partial sums are flushed to fp64 every 16 grains

template <int DIM, int D, int R>
__global__ void __launch_bounds__(kG1Threads) k_grid_pass1(GridParams g) {
  constexpr int J = D + 1;
  constexpr int K = feature_count(DIM, D);
  constexpr int JP = (J + 1) & ~1;  // fp64 coefficient row (pairs)
  constexpr int JF = (J + 3) & ~3;  // fp32 coefficient row (quads)
  __shared__ __align__(16) double B_s[kG1Chunk][JP];
  __shared__ __align__(16) float Bf_s[kG1Chunk][JF];
  __shared__ double lc[K];
  __shared__ double red_d[kG1Threads];
  __shared__ long long red_i[kG1Threads];
  __shared__ unsigned s_bmax;  // max_i sum_j |B''_{j,i}| (float bits, >= 0)
  __shared__ int cta_safe;

  const int tid = threadIdx.x;
  const int64_t line = blockIdx.x / g.segs;
  const int seg = blockIdx.x % g.segs;
  const int64_t pbase = line * g.side + (int64_t)seg * kG1Threads * R;
  const int N = g.N;
  const double c = g.c;
  griddep_wait();               // PDL: theta staged, the previous evaluation complete
  griddep_launch_dependents();  // pass 2 is scheduled once the last wave is resident

  if (tid == 0) {
    double lcr[K];
    line_factors<DIM, D>(line, g, lcr);
#pragma unroll
    for (int k = 0; k < K; ++k) lc[k] = lcr[k];
    s_bmax = 0u;
    cta_safe = 0;
  }
  __syncthreads();

  double v[R][J];
  float vf[R][J];
  int lab[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int col = seg * kG1Threads * R + tid + kG1Threads * r;
    axis_table<D>(axis_coord(col, g.M), g.legendre != 0, v[r]);
#pragma unroll
    for (int j = 0; j < J; ++j) vf[r][j] = (float)v[r][j];
    lab[r] = g.labels[pbase + tid + kG1Threads * r];
  }

  // builds chunk [c0, c0 + cn) of B'' (fp64 and fp32) in shared memory, padded
  // to a multiple of kG1Flush with inert grains (h'' = 1e30: never a minimum,
  // weight 2^-1e30 = 0, never a label)
  auto build_chunk = [&](int c0, int cn, bool fp32_too) {
    __syncthreads();
    const int cpad = (cn + kG1Flush - 1) & ~(kG1Flush - 1);
    if (tid < cn) {
      double B[J];
      line_coeffs<DIM, D>(g.theta, N, c0 + tid, lc, c, B);
      double bsum = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        B_s[tid][j] = B[j];
        if (fp32_too) Bf_s[tid][j] = (float)B[j];
        bsum += fabs(B[j]);
      }
      if (fp32_too) {
        // |h''| <= 2^100 keeps fp32 sweep A finite and the conversion valid
        if (!(bsum < 1e30)) cta_safe = 1;
        else atomicMax(&s_bmax, __float_as_uint((float)bsum));
      }
    } else if (tid < cpad) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        B_s[tid][j] = j == 0 ? 1e30 : 0.0;
        Bf_s[tid][j] = j == 0 ? 1e30f : 0.0f;
      }
    }
    __syncthreads();
  };

  // ---------------------------------------------------------------- sweep A
  float b1[R], b2[R];
  int ib[R];
  double m64[R];  // exact min (SAFE path only)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    b1[r] = CUDART_INF_F;
    b2[r] = CUDART_INF_F;
    ib[r] = 0;
    m64[r] = CUDART_INF;
  }
  const unsigned bf_addr = (unsigned)__cvta_generic_to_shared(&Bf_s[0][0]);
  const unsigned bs_addr = (unsigned)__cvta_generic_to_shared(&B_s[0][0]);
  for (int c0 = 0; c0 < N; c0 += kG1Chunk) {
    const int cn = min(kG1Chunk, N - c0);
    const bool was_safe = cta_safe != 0;
    build_chunk(c0, cn, true);
    if (cta_safe && !was_safe && c0 > 0) {
      c0 = -kG1Chunk;  // extreme coefficients appeared: restart sweep A in fp64
      continue;
    }
    if (!cta_safe) {
      const int cpad = (cn + kG1Flush - 1) & ~(kG1Flush - 1);
      for (int g0 = 0; g0 < cpad; g0 += kG1Flush) {
#pragma unroll
        for (int jj = 0; jj < kG1Flush; ++jj) {
          const int jg = g0 + jj;
          float Bf[JF];
#pragma unroll
          for (int j = 0; j < JF; j += 4)
            lds_f32x4(bf_addr + (jg * JF + j) * 4, Bf[j], Bf[j + 1], Bf[j + 2], Bf[j + 3]);
          const int i = c0 + jg;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float ht = Bf[0];
#pragma unroll
            for (int j = 1; j < J; ++j) ht = fmaf(Bf[j], vf[r][j], ht);
            const bool p = ht < b1[r];
            b2[r] = p ? b1[r] : fminf(b2[r], ht);
            b1[r] = p ? ht : b1[r];
            ib[r] = p ? i : ib[r];
          }
        }
      }
    } else {  // fp64 fallback for extreme or non-finite coefficients
      for (int jg = 0; jg < cn; ++jg) {
        const int i = c0 + jg;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double h = eval_line<J>(B_s[jg], v[r]);
          if (h < m64[r] || i == 0) {
            m64[r] = h;
            ib[r] = i;
          }
        }
      }
    }
  }
  const bool safe = cta_safe != 0;
  // CTA-wide bound of |ht - h''|: fp32 coefficients, basis values and the
  // J-term fma chain (|L_j| <= 1 on [-1,1]); generous factor 2
  const double delta = safe ? 0.0 : 2.0 * (J + 3) * 5.9604644775390625e-08 *
                                         (double)__uint_as_float(s_bmax);

  double ref[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    ref[r] = safe ? m64[r] - 1.0 : (double)b1[r] - delta - 1.0;  // a = h'' - ref >= 1

  // ---------------------------------------------------------------- sweep B
  float sx[R];
  double sx64[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    sx[r] = 0.0f;
    sx64[r] = 0.0;
  }
  for (int c0 = 0; c0 < N; c0 += kG1Chunk) {
    const int cn = min(kG1Chunk, N - c0);
    if (N > kG1Chunk) build_chunk(c0, cn, false);  // single chunk: still resident
    const int cpad = (cn + kG1Flush - 1) & ~(kG1Flush - 1);
    for (int g0 = 0; g0 < cpad; g0 += kG1Flush) {
      const int ge = safe ? min(kG1Flush, cn - g0) : kG1Flush;
      if (!safe) {
#pragma unroll
        for (int jj = 0; jj < kG1Flush; ++jj) {
          const int jg = g0 + jj;
          double B[JP];
#pragma unroll
          for (int j = 0; j < JP; j += 2) lds_f64x2(bs_addr + (jg * JP + j) * 8, B[j], B[j + 1]);
          const int i = c0 + jg;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double h = eval_line<J>(B, v[r]);
            const float e = ex2_neg(h - ref[r]);
            sx[r] += (i != lab[r]) ? e : 0.0f;
          }
        }
      } else {
        for (int jj = 0; jj < ge; ++jj) {
          const int jg = g0 + jj;
          const int i = c0 + jg;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double h = eval_line<J>(B_s[jg], v[r]);
            sx[r] += (i != lab[r]) ? (float)exp2(ref[r] - h) : 0.0f;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        sx64[r] += (double)sx[r];
        sx[r] = 0.0f;
      }
    }
  }

  // ---------------------------------------------------------- per-pixel finish
  double ell = 0.0, e0 = 0.0;
  long long correct = 0, nonfinite = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t p = pbase + tid + kG1Threads * r;
    double Bg[J];
    line_coeffs<DIM, D>(g.theta, N, lab[r], lc, c, Bg);
    const double hG = eval_line<J>(Bg, v[r]);
    line_coeffs<DIM, D>(g.theta, N, ib[r], lc, c, Bg);
    const double hm = eval_line<J>(Bg, v[r]);  // exact h'' of the (approximate) arg-min
    const double aG = hG - ref[r];
    const double eG = exp2(-aG);
    const double s = sx64[r] + eG;
    const double l2s = log2(s);
    const double l = (-aG - l2s) * 0.69314718055994530942;  // log p_G: objective.py:103-106
    ell += l;
    e0 += (hG - hm) / c;                                    // objective.py:119
    if (!isfinite(l)) nonfinite = 1;
    g.pix_w[p] = ref[r] - 1.0 - l2s;           // p_i / 2 = 2^(w - h''_i)
    g.pix_q[p] = (float)(0.5 * sx64[r] / s);  // (1 - p_G) / 2 = sum_{j != G} p_j / 2
    g.pix_m[p] = hm / c;
    // exact arg-min unless the runner-up is within 2 delta + tie + ambiguity band
    const double band = c * fmax(kTieRtol, g.tau_amb) * (1.0 + fabs(hm / c));
    const bool clear = !safe && ((double)b2[r] - (double)b1[r] > 2.0 * delta + band);
    if (!clear) {
      const int slot = atomicAdd(g.fix_count, 1);
      g.fix_list[slot] = (int)p;
    } else {
      correct += (ib[r] == lab[r]) ? 1 : 0;
    }
  }
  const double s_ell = block_sum<kG1Threads>(ell, red_d);
  const double s_e0 = block_sum<kG1Threads>(e0, red_d);
  const long long s_cor = block_sum<kG1Threads>(correct, red_i);
  const long long s_nf = block_sum<kG1Threads>(nonfinite, red_i);
  if (tid == 0) {
    g.part_d[2 * blockIdx.x + 0] = s_ell;
    g.part_d[2 * blockIdx.x + 1] = s_e0;
    g.part_i[4 * blockIdx.x + 0] = s_cor;
    g.part_i[4 * blockIdx.x + 1] = 0;  // ambiguity is decided by the tail re-scan
    g.part_i[4 * blockIdx.x + 2] = s_nf;
    g.part_i[4 * blockIdx.x + 3] = 0;
  }
}

}  // namespace pgx
