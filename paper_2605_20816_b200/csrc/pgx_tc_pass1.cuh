// pgx_tc_pass1.cuh — PGX_PREC_TC pass 1: the logit contraction h'' = L(x_fast)
// B''(line) (objective.py:99) on the 5th-generation tensor cores, the
// log-sum-exp / min / arg-min epilogue on the CUDA cores.
//
// CTA = R tiles of 128 pixels of one line (4 warps; thread = TMEM lane = pixel).
// Grains stream in chunks of 256 = the UMMA N.  Per (chunk, tile) one elected
// thread issues tc_ksteps(J) tcgen05.mma (M=128, N=256, K=16, fp16 in, fp32
// accumulate in TMEM) and commits to an mbarrier; the epilogue reads 32-column
// blocks with tcgen05.ld.  Operands use a 3-product fp16 split (hi*hi + hi*lo
// + lo*hi): logits carry ~fp32 accuracy, bounded by delta = gamma * max|B''|_1.
//
//   sweep A: m~ = min h~'' (one FMNMX per logit);
//   sweep B: s' = sum_{i != G} 2^(ref - h~''_i), ref = m~ - delta - 1, one
//            FFMA + MUFU.EX2 + FADD per logit; logits within 2 delta + tie +
//            ambiguity band of m~ are re-evaluated exactly in fp64 (vote per
//            32-column block) for the exact tie-tolerant arg-min
//            (geometry.py:201-210), min and runner-up.
// The label term is exact (fp64) and excluded from s'.
#pragma once

#include "pgx_grid_common.cuh"
#include "pgx_tc_coeffs.cuh"
#include "pgx_tc_common.cuh"

namespace pgx {

constexpr int kTcThreads = 128;
constexpr int kTcChunk = 128;     // grains per chunk (UMMA N)
constexpr int kTcTmemCols = 128;  // one fp32 accumulator tile: 4 CTAs share an SM's TMEM
constexpr int kTcMinSmem = 46 * 1024;  // keeps residency at <= 4 CTAs per SM

// exact per-pixel state for near-minimal logits (shared memory)
struct TcRare {
  double m, m2, hb0, hb1;
  int b0, b1, cnt, flags;  // flags: 1 dirty (candidate list overflowed), 2 needfix
};

__device__ __forceinline__ void tc_rare_update(TcRare& st, int i, double h, double c) {
  if (h < st.m) {
    st.m2 = fmin(st.m2, st.m);
    st.m = h;
    const double thr = h + c * kTieRtol * (1.0 + fabs(h / c));
    if (st.cnt > 0 && !(st.hb0 <= thr)) {
      if (st.flags & 1) st.flags |= 2;
      if (st.cnt > 1 && st.hb1 <= thr) {
        st.b0 = st.b1;
        st.hb0 = st.hb1;
        st.cnt = 1;
      } else {
        st.cnt = 0;
      }
    } else if (st.cnt > 1 && !(st.hb1 <= thr)) {
      st.cnt = 1;
    }
  } else if (h < st.m2) {
    st.m2 = h;
  }
  const double thr = st.m + c * kTieRtol * (1.0 + fabs(st.m / c));
  if (h <= thr) {
    if (st.cnt == 0) {
      st.b0 = i;
      st.hb0 = h;
      st.cnt = 1;
    } else if (st.cnt == 1) {
      st.b1 = i;
      st.hb1 = h;
      st.cnt = 2;
    } else {
      st.flags |= 1;
    }
  }
}

template <int J, int R>
struct TcP1Smem {
  static constexpr int KS = tc_ksteps(J);
  static constexpr int A_BYTES = R * KS * kTcThreads * 32;
  static constexpr int B_BYTES = KS * kTcChunk * 32;
  static constexpr int BD_BYTES = 0;  // exact B'' is read from the per-line table
  static constexpr int RARE_BYTES = R * kTcThreads * (int)sizeof(TcRare);
  static constexpr int A_OFF = 0;
  static constexpr int B_OFF = A_OFF + A_BYTES;
  static constexpr int BD_OFF = B_OFF + B_BYTES;
  static constexpr int RARE_OFF = BD_OFF + BD_BYTES;
  static constexpr int TOTAL = RARE_OFF + RARE_BYTES;
};

template <int DIM, int D, int R>
__global__ void __launch_bounds__(kTcThreads, 4) k_tc_pass1(GridParams g) {
  constexpr int J = D + 1;
  constexpr int K = feature_count(DIM, D);
  using L = TcP1Smem<J, R>;
  constexpr int KS = L::KS;
  constexpr uint32_t IDESC = umma_idesc_f16(128, kTcChunk);
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* A_s = smem + L::A_OFF;
  unsigned char* B_s = smem + L::B_OFF;
  TcRare* rare = reinterpret_cast<TcRare*>(smem + L::RARE_OFF);  // [R][128]
  __shared__ double lc[K];
  __shared__ uint64_t mbar;
  __shared__ unsigned tmem_base;
  __shared__ unsigned s_bmax;     // max over grains of sum_j |B''_j| (float bits)
  __shared__ double red_d[kTcThreads];
  __shared__ long long red_i[kTcThreads];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t line = blockIdx.x / g.segs;
  const int seg = blockIdx.x % g.segs;
  const int64_t pbase = line * g.side + (int64_t)seg * kTcThreads * R;
  const int N = g.N;
  const double c = g.c;

  if (warp == 0) tmem_alloc(&tmem_base, kTcTmemCols);
  if (tid == 0) {
    double lcr[K];
    line_factors<DIM, D>(line, g, lcr);
#pragma unroll
    for (int k = 0; k < K; ++k) lc[k] = lcr[k];
    mbar_init(&mbar, 1);
    fence_mbar_init();
    s_bmax = 0u;
  }

  // pixel operands: A'[p][k] = 2^10 L_j(x_fast), k = b J + j, blocks [hi, hi, lo]
  int lab[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int col = seg * kTcThreads * R + kTcThreads * r + tid;
    double u[J];
    axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
    __half hi[J], lo[J];
#pragma unroll
    for (int j = 0; j < J; ++j) split_f16(u[j] * 1024.0, hi[j], lo[j]);
#pragma unroll
    for (int k = 0; k < 16 * KS; ++k) {
      const int b = k / J, j = k % J;
      const __half val = k < 3 * J ? (b < 2 ? hi[j] : lo[j]) : __float2half(0.0f);
      *reinterpret_cast<__half*>(A_s + (r * KS + k / 16) * (kTcThreads * 32) +
                                 slab_off(tid, k % 16)) = val;
    }
    lab[r] = g.labels[pbase + kTcThreads * r + tid];
    TcRare& st = rare[r * kTcThreads + tid];
    st.m = CUDART_INF;
    st.m2 = CUDART_INF;
    st.cnt = 0;
    st.flags = 0;
    st.b0 = st.b1 = -1;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = tmem_base;
  const unsigned a_addr = (unsigned)__cvta_generic_to_shared(A_s);
  const unsigned b_addr = (unsigned)__cvta_generic_to_shared(B_s);
  unsigned phase = 0;

  // chunk [c0, c0 + cn): copy the precomputed operand image (pgx_tc_coeffs.cuh)
  // of this line into B_s; returns 2^-(sB + 10) so that D * this = h~''
  const double* coef_line = g.tc_coef + line * (int64_t)N * J;  // exact B'' of this line
  auto build_chunk = [&](int c0, int cn) -> float {
    (void)cn;
    __syncthreads();
    const int64_t ci = line * g.tc_nchunks + c0 / kTcChunk;
    copy_coef_img<J, kTcThreads>(B_s, g.tc_img + ci * tc_img_bytes<J>(), tid);
    const int2 m = g.tc_meta[ci];
    if (tid == 0) atomicMax(&s_bmax, (unsigned)m.y);  // non-negative float bits
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    return ldexpf(1.0f, -(m.x + 10));
  };

  // one UMMA tile: D[128 x 256] = A_r B^T, then wait for the accumulator
  auto mma_tile = [&](int r) {
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < KS; ++s)
        umma_f16_ss(tmem, umma_desc(a_addr + (r * KS + s) * (kTcThreads * 32)),
                    umma_desc(b_addr + s * (kTcChunk * 32)), IDESC, s > 0);
      umma_commit(&mbar);
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    tc_fence_after();
  };
  const unsigned trow = tmem + ((unsigned)(warp * 32) << 16);

  // ---------------------------------------------------------------- sweep A
  // Per-tile state lives in small arrays indexed by the (rolled) tile loop:
  // a few local-memory accesses per tile instead of R copies of the epilogue
  // code (the unrolled version thrashed the instruction cache).
  float mt[R];
#pragma unroll
  for (int r = 0; r < R; ++r) mt[r] = CUDART_INF_F;
  for (int c0 = 0; c0 < N; c0 += kTcChunk) {
    const int cn = min(kTcChunk, N - c0);
    const float inv = build_chunk(c0, cn);
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      mma_tile(r);
      float m0 = CUDART_INF_F, m1 = CUDART_INF_F;
      for (int cb = 0; cb < cn; cb += 32) {
        float v[32];
        tmem_ld32(trow + cb, v);
        if (cb + 32 <= cn) {
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            m0 = fminf(m0, v[q]);
            m1 = fminf(m1, v[q + 1]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (cb + q < cn) m0 = fminf(m0, v[q]);
        }
      }
      mt[r] = fminf(mt[r], fminf(m0, m1) * inv);
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
    }
  }
  const float bnorm = __uint_as_float(s_bmax);
  // |h~'' - h''| <= delta: fp16 split (2^-21 relative per operand pair) plus
  // the fp32 accumulation of 3J products; generous factor 2
  const float delta = 2.0f * (4.7683716e-07f + 3 * J * 5.9604645e-08f) * bnorm + 1e-30f;

  // ---------------------------------------------------------------- sweep B
  float ref[R], athr[R], sx[R];
  double sx64[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    ref[r] = mt[r] - delta - 1.0f;
    const double band = c * fmax(kTieRtol, g.tau_amb) * (1.0 + fabs((double)mt[r] / c));
    athr[r] = 1.0f + 3.0f * delta + (float)band * 1.001f;  // a = h~'' - ref <= athr: candidate
    sx[r] = 0.0f;
    sx64[r] = 0.0;
  }
  for (int c0 = 0; c0 < N; c0 += kTcChunk) {
    const int cn = min(kTcChunk, N - c0);
    const float inv = build_chunk(c0, cn);
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      mma_tile(r);
      const int labc = lab[r] - c0;
      const float refr = ref[r], athrr = athr[r];
      double sxr = sx64[r];
      for (int cb = 0; cb < cn; cb += 32) {
        float v[32];
        tmem_ld32(trow + cb, v);
        const bool full = cb + 32 <= cn;
        const bool lab_here = (unsigned)(labc - cb) < 32u;
        bool cand = false;
        float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // 4 independent FADD chains
        if (full && !__any_sync(0xffffffffu, lab_here)) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float a = fmaf(v[q], inv, -refr);
            cand |= a <= athrr;
            s4[q & 3] += ex2_approx(-a);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float a = fmaf(v[q], inv, -refr);
            const bool ok = cb + q < cn;
            cand |= ok && a <= athrr;
            const float e = ex2_approx(-a);
            s4[q & 3] += (ok && cb + q != labc) ? e : 0.0f;
          }
        }
        sxr += (double)((s4[0] + s4[1]) + (s4[2] + s4[3]));
        if (__any_sync(0xffffffffu, cand)) {
          // exact fp64 re-evaluation of the near-minimal logits: collect the
          // candidate columns as a bit mask (static register indices), then
          // walk the set bits
          unsigned cm = 0u;
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (fmaf(v[q], inv, -refr) <= athrr && cb + q < cn) cm |= 1u << q;
          if (cm) {
            const int col = seg * kTcThreads * R + kTcThreads * r + tid;
            double u[J];
            axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
            TcRare& st = rare[r * kTcThreads + tid];
            while (cm) {
              const int q = __ffs(cm) - 1;
              cm &= cm - 1u;
              tc_rare_update(st, c0 + cb + q,
                             eval_line<J>(coef_line + (int64_t)(c0 + cb + q) * J, u), c);
            }
          }
        }
      }
      sx64[r] = sxr;
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
    }
  }

  // ---------------------------------------------------------- per-pixel finish
  double ell = 0.0, e0 = 0.0;
  long long correct = 0, amb = 0, nonfinite = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int col = seg * kTcThreads * R + kTcThreads * r + tid;
    const int64_t p = pbase + kTcThreads * r + tid;
    double u[J];
    axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
    const double hG = eval_line<J>(coef_line + (int64_t)lab[r] * J, u);  // same bits as the refine
    TcRare& st = rare[r * kTcThreads + tid];
    const double refd = (double)ref[r];
    const double aG = hG - refd;
    const double eG = exp2(-aG);
    const double s = sx64[r] + eG;
    const double l2s = log2(s);
    const double l = (-aG - l2s) * 0.69314718055994530942;  // log p_G: objective.py:103-106
    ell += l;
    if (!isfinite(l) || !(bnorm <= 3e38f)) nonfinite = 1;
    if (g.tc_rec) {  // pass-2 record: p_i/2 * 2^13 = 2^(w13 + wl13 - h~''_i)
      const double w13 = refd - 1.0 - l2s + 13.0;
      const float wh = (float)w13;
      float* rec = g.tc_rec + (line * (g.side / kTcPixTile) + (col >> 6)) * (4 * kTcPixTile) + (col & 63);
      rec[0] = wh;
      rec[kTcPixTile] = (float)(w13 - (double)wh);
      rec[2 * kTcPixTile] = (float)(-4096.0 * sx64[r] / s);  // -(1 - p_G)/2 * 2^13
      reinterpret_cast<int*>(rec)[3 * kTcPixTile] = lab[r];
    }
    const bool found = st.cnt > 0 && !(st.flags & 2);
    const double m = st.cnt > 0 ? st.m : hG;
    g.pix_m[p] = m / c;
    e0 += (hG - m) / c;  // objective.py:119
    if (!found) {
      const int slot = atomicAdd(g.fix_count, 1);
      g.fix_list[slot] = (int)p;
    } else {
      correct += (st.b0 == lab[r]) ? 1 : 0;
      amb += ((st.m2 - st.m) <= c * g.tau_amb * (1.0 + fabs(st.m / c))) ? 1 : 0;
    }
  }
  const double s_ell = block_sum<kTcThreads>(ell, red_d);
  const double s_e0 = block_sum<kTcThreads>(e0, red_d);
  const long long s_cor = block_sum<kTcThreads>(correct, red_i);
  const long long s_amb = block_sum<kTcThreads>(amb, red_i);
  const long long s_nf = block_sum<kTcThreads>(nonfinite, red_i);
  if (tid == 0) {
    g.part_d[2 * blockIdx.x + 0] = s_ell;
    g.part_d[2 * blockIdx.x + 1] = s_e0;
    g.part_i[4 * blockIdx.x + 0] = s_cor;
    g.part_i[4 * blockIdx.x + 1] = s_amb;
    g.part_i[4 * blockIdx.x + 2] = s_nf;
    g.part_i[4 * blockIdx.x + 3] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTcTmemCols);
}

}  // namespace pgx
