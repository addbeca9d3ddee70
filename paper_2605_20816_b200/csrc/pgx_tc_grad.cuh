// pgx_tc_grad.cuh — PGX_PREC_TC pass 2 ("grad"): the gradient contraction
// sum_x (onehot_G(x) - p(x)) eta(x) (objective.py:109-113) with both
// contractions on the tensor cores (FlashAttention-backward-like, grain-major):
//
//   UMMA 1 (SS)  S^T[128 grains x 64 px] = B''(line)[grains x 3J] . L(x)[px x 3J]^T
//   epilogue     thread = grain = TMEM lane: r' = p/2 * 2^13 = 2^(w13 - h~'')
//                (packed FFMA2 argument pairs + MUFU.EX2), or -(1 - p_G)/2 * 2^13
//                on the pixel's label grain (pass-1 record: no cancellation);
//                split exactly into fp16 hi (the fp32 value with its 13 low
//                mantissa bits cleared) + lo (the fp32 remainder) and written
//                back into TMEM over S (packed f16x2)
//   UMMA 2 (TS)  R[128 grains x 32] += r'_hi . [L_hi | L_lo]^T + r'_lo . [L_hi | L_lo]^T
//                (A from TMEM, K = 16 pixels per MMA, 8 MMAs per tile)
//
// Warp specialisation, 320 threads, 2 CTAs per SM:
//   warps 0-7  epilogue: warp w owns TMEM lanes 32 (w % 4) .. (grains); warps
//              0-3 take the even tiles, 4-7 the odd ones (all 64 pixels);
//   warp 8     MMA: one lane issues UMMA 2 of tile n and UMMA 1 of tile n + 3
//              as soon as the epilogue of tile n has written r' (S is
//              triple-buffered in TMEM) -- nothing else on its critical path;
//   warp 9     loader: bulk copies (cp.async.bulk + mbarrier tx counts) of the
//              line's coefficient image (kGdA slots) and each tile's pixel
//              operands and pass-1 records (kGdBuf-deep), refilled as the
//              MMAs reading them complete.
// R alternates between two TMEM accumulators per group of 4 tiles; a finished
// group is flushed into fp64 line sums 3 tiles later (when it is known to be
// complete) and per line expanded into the K gradient rows of the CTA's split
// slot of the partials (fp64; the tail reduces the splits in fixed order).
//
// TMEM (256 columns): S_0..S_2 [0, 192) (64 each), R_a [192, 224), R_b [224, 256).
// Within S_s, pixel half h keeps r'_hi in [32h, 32h + 16) and r'_lo in
// [32h + 16, 32h + 32): only columns its own warps have already read.
#pragma once

#include "pgx_grid_common.cuh"
#include "pgx_tc_coeffs.cuh"
#include "pgx_tc_common.cuh"
#include "pgx_tc_shared.cuh"

namespace pgx {

// pixel-operand + record buffers: the loader warp runs up to kGdBuf items
// ahead of UMMA 2 (hides the L2 bulk-copy latency of several thousand cycles)
constexpr int kGdBuf = 8;
constexpr int kGdA = 3;    // coefficient-image slots (lines in flight)
constexpr int kGdMmaWarp = kTc2Epi / 32, kGdLoadWarp = kGdMmaWarp + 1;
constexpr int kGdThreads = kTc2Epi + 64;  // + MMA warp + loader warp
#ifdef PGX_GD_TRACE
#ifndef PGX_GD_TRACE_X  // the traced CTA
#define PGX_GD_TRACE_X 3
#define PGX_GD_TRACE_Y 5
#endif
// experiment builds only (tools/gd_trace.py): clock64 stamps of one CTA's first 256 items
__device__ long long gd_trace[14][256];
#define GD_STAMP(e, n) \
  do { if (blockIdx.x == PGX_GD_TRACE_X && blockIdx.y == PGX_GD_TRACE_Y && (n) < 256) gd_trace[e][n] = clock64(); } while (0)
#else
#define GD_STAMP(e, n) do { } while (0)
#endif

template <int DIM, int D>
struct GdSmem {
  static constexpr int J = D + 1;
  static constexpr int K = feature_count(DIM, D);
  static constexpr int KS = tc_ksteps(J);
  static constexpr int A1 = KS * kTc2Grains * 32;  // coefficient image (128 rows)
  static constexpr int PIX = tc_pix_bytes<J>();
  static constexpr int REC = kTc2RecFloats * 4;
  static constexpr int A1_OFF = 0;
  static constexpr int PIX_OFF = A1_OFF + kGdA * A1;
  static constexpr int REC_OFF = PIX_OFF + kGdBuf * PIX;
  static constexpr int R_OFF = REC_OFF + kGdBuf * REC;  // fp64 [J][128] line sums
  static constexpr int TOTAL = R_OFF + J * kTc2Grains * 8;
};

// program-ordered variants: a warp issues in order, and MUFU.EX2 (8 cycles per
// warp instruction on its pipe) and F2FP (~5) block the instructions behind
// them, so the epilogue interleaves the exponentials of one pixel pair with
// the conversions of an earlier pair; volatile keeps that order
__device__ __forceinline__ float ex2_ordered(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_h2_ordered(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
#ifndef PGX_GD_FLUSH32
#define PGX_GD_FLUSH32 1  // the L_hi / L_lo halves of an fp32 group sum are added in fp32 (2^-24 relative)
#endif
#ifndef PGX_GD_ILV
#define PGX_GD_ILV 1
#endif

// fp16 pair of two fp32 values, low half = a (the even pixel)
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// Once per line and grain: grad rows += line factors x the line's fp64 sums,
// acc[k N] (the grain's column of its split slot) += lc[k] R_{alpha_fast(k)}.
// Out of line so that its 16-deep load batches do not weigh on the register
// allocation of the tile loop.
template <int DIM, int D>
__device__ __noinline__ void tc_grad_line(double* __restrict__ acc, int N, const double* __restrict__ lcp,
                                          const double* R64, bool first) {
  constexpr int K = feature_count(DIM, D);
  constexpr int J = D + 1;
  const double rs = -2.0 / (8192.0 * 1024.0);  // R_true = -2 R' 2^-(13 + 10): r' = -r
  double r[J];
#pragma unroll
  for (int j = 0; j < J; ++j) r[j] = rs * R64[j * kTc2Grains];
  constexpr int CH = 16;
#pragma unroll
  for (int k0 = 0; k0 < K; k0 += CH) {
    double prev[CH];
#pragma unroll
    for (int k = k0; k < k0 + CH && k < K; ++k) prev[k - k0] = first ? 0.0 : acc[(int64_t)k * N];
#pragma unroll
    for (int k = k0; k < k0 + CH && k < K; ++k)
      acc[(int64_t)k * N] = fma(__ldg(lcp + k), r[alpha_of(DIM, D, k, DIM - 1)], prev[k - k0]);
  }
}

template <int DIM, int D>
__global__ void __launch_bounds__(kGdThreads, 2) k_tc_grad(GridParams g) {
  using L = GdSmem<DIM, D>;
  constexpr int J = L::J;
  constexpr int K = L::K;
  constexpr int KS = L::KS;
  constexpr uint32_t IDESC1 = umma_idesc_f16(128, kTc2Px);
  constexpr uint32_t IDESC2 = umma_idesc_f16(128, 32);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_full[kGdBuf], bar_pf[kGdBuf], bar_a[kGdA], bar_af[kGdA];
  __shared__ uint64_t bar_s[kTc2S], bar_p[kTc2S], bar_end;
  __shared__ unsigned tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gbase = blockIdx.x * kTc2Grains;
  // items (line, tile) of this CTA: [a0, a1) of the launch's line range
  const int ntiles = g.pside / kTc2Px;
  const int gpl = (ntiles + kTc2Group - 1) / kTc2Group;  // R groups per line
  const int64_t a0 = g.line_lo * ntiles + (int64_t)blockIdx.y * g.items_per_split;
  const int64_t a1 = min((int64_t)g.lines * ntiles, a0 + g.items_per_split);
  if (a1 <= a0) return;
  const int nitems = (int)(a1 - a0);
  const int64_t l0 = a0 / ntiles;
  const int t0 = (int)(a0 - l0 * ntiles);
  const int nlines = (int)((a1 - 1) / ntiles - l0 + 1);

  if (warp == kGdMmaWarp) tmem_alloc(&tmem_base, 256);
  if (tid == kTc2Epi) {
    for (int b = 0; b < kGdBuf; ++b) {
      mbar_init(&bar_full[b], 1);
      mbar_init(&bar_pf[b], 1);
    }
    for (int b = 0; b < kGdA; ++b) {
      mbar_init(&bar_a[b], 1);
      mbar_init(&bar_af[b], 1);
    }
    for (int b = 0; b < kTc2S; ++b) {
      mbar_init(&bar_s[b], 1);
      mbar_init(&bar_p[b], 4);  // the four warps of the tile's group
    }
    mbar_init(&bar_end, 1);
    fence_mbar_init();
  }
  {  // zero the fp64 line sums
    double* R = reinterpret_cast<double*>(smem + L::R_OFF);
    for (int e = tid; e < J * kTc2Grains; e += kGdThreads) R[e] = 0.0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();  // PDL: pass 1's records, fix lists and partials are complete
  const unsigned tmem = tmem_base;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  // the (line, tile) of an item, walked incrementally
  struct Cur {
    int n, li, t;
    __device__ __forceinline__ void next(int nt) {
      ++n;
      if (++t == nt) {
        t = 0;
        ++li;
      }
    }
  };
  auto group_last = [&](const Cur& c) {
    return c.t == ntiles - 1 || (c.t & (kTc2Group - 1)) == kTc2Group - 1 || c.n == nitems - 1;
  };
  auto r_col = [&](const Cur& c) {  // R accumulator of the item's group
    return tmem + 192u + 32u * (unsigned)((c.li * gpl + c.t / kTc2Group) & 1);
  };

  if (warp == kGdLoadWarp) {
    // ======================= loader warp: every image and every item's pixel
    // operands + records, in consumption order; a buffer is refilled once the
    // MMAs that read it are complete (commits of the MMA warp)
    if (elect_one()) {
      Cur cl{0, 0, t0};
      int al = 0;  // lines whose coefficient image has been requested
      for (; cl.n < nitems; cl.next(ntiles)) {
        if (cl.n == 0 || cl.t == 0) {  // the line's image (lines ahead as the slots free up)
          for (; al <= cl.li && al < nlines; ++al) {
            const int ab = al % kGdA;
            if (al >= kGdA) mbar_wait_sleep(&bar_af[ab], (unsigned)((al - kGdA) / kGdA) & 1u);
            mbar_arrive_expect_tx(&bar_a[ab], L::A1);
            bulk_g2s(smem + L::A1_OFF + ab * L::A1,
                     g.tc_img + ((l0 + al) * g.tc_nchunks + blockIdx.x) * (int64_t)L::A1, L::A1, &bar_a[ab]);
          }
        }
        const int b = cl.n % kGdBuf;
        if (cl.n >= kGdBuf) mbar_wait_sleep(&bar_pf[b], (unsigned)((cl.n - kGdBuf) / kGdBuf) & 1u);
        mbar_arrive_expect_tx(&bar_full[b], L::PIX + L::REC);
        bulk_g2s(smem + L::PIX_OFF + b * L::PIX, g.tc_pix + (int64_t)cl.t * L::PIX, L::PIX, &bar_full[b]);
        bulk_g2s(smem + L::REC_OFF + b * L::REC,
                 g.tc_rec + ((l0 + cl.li) * ntiles + cl.t) * (int64_t)kTc2RecFloats, L::REC, &bar_full[b]);
      }
    }
    __syncwarp();
  } else if (warp == kGdMmaWarp) {
    // ======================= MMA issuer: ONE thread runs the whole role (no
    // warp-level re-convergence inside the loop), and every tcgen05 operand is
    // derived from warp-uniform values (the TMEM base broadcast by a shuffle),
    // so that each MMA is a single UTCHMMA on uniform registers instead of an
    // elect / broadcast loop: the issuer's per-item time bounds the kernel
    const unsigned tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    const unsigned sbase_u = __shfl_sync(0xffffffffu, sbase, 0);
    if (elect_one()) {
      const uint64_t d_a1 = umma_desc(sbase_u + L::A1_OFF);
      const uint64_t d_pix = umma_desc(sbase_u + L::PIX_OFF);
      Cur cs{0, 0, t0}, cm{0, 0, t0};  // next UMMA 1, next UMMA 2
      int cs_st = 0, cs_b = 0;         // cs.n % kTc2S, cs.n % kGdBuf
      auto issue_s = [&]() {  // UMMA 1 of item cs into S_(n % 3)
        const int ab = cs.li % kGdA;
        if (cs.t == 0 || cs.n == 0) mbar_wait(&bar_a[ab], (unsigned)(cs.li / kGdA) & 1u);
        mbar_wait(&bar_full[cs_b], (unsigned)(cs.n / kGdBuf) & 1u);
        tc_fence_after();
        const uint64_t da = d_a1 + (uint64_t)((ab * L::A1) >> 4);
        const uint64_t db = d_pix + (uint64_t)((cs_b * L::PIX) >> 4);
#pragma unroll
        for (int s = 0; s < KS; ++s)
          umma_f16_ss(tmem_u + 64u * cs_st, da + (uint64_t)((s * kTc2Grains * 32) >> 4),
                      db + (uint64_t)((s * kTc2Px * 32) >> 4), IDESC1, s > 0);
        umma_commit(&bar_s[cs_st]);
        if (cs.t == ntiles - 1 || cs.n == nitems - 1) umma_commit(&bar_af[ab]);  // the line's image is free
        GD_STAMP(4, cs.n);
        cs.next(ntiles);
        if (++cs_st == kTc2S) cs_st = 0;
        if (++cs_b == kGdBuf) cs_b = 0;
      };
      while (cs.n < nitems && cs.n < kTc2S) issue_s();
      int st = 0, b = 0;
      unsigned ph_p = 0;  // phase parity of bar_p[st]: flips each time st wraps
      unsigned rsel = (unsigned)(t0 / kTc2Group) & 1u;  // R accumulator of cm's group (= r_col)
      for (int k = 0; k < nitems; ++k) {
        mbar_wait(&bar_p[st], ph_p);  // r' of item k is in S_st
        tc_fence_after();
        GD_STAMP(2, k);
        {  // UMMA 2: R += [r_hi; r_lo] . [L_hi | L_lo]^T over the 64 pixels
          const unsigned ts = tmem_u + 64u * st;
          const uint64_t dl = d_pix + (uint64_t)((b * L::PIX + KS * (kTc2Px * 32)) >> 4);
          const bool fresh = (cm.t & (kTc2Group - 1)) == 0 || cm.n == 0;  // a group's first item
          auto umma2 = [&](unsigned tr) {
#pragma unroll
            for (int s = 0; s < 2 * (kTc2Px / 16); ++s) {
              const int p = s / (kTc2Px / 16), ks = s % (kTc2Px / 16);
              // pixels [16 ks, 16 ks + 16): half ks / 2, packed columns 8 (ks % 2); p = 1: r_lo
              const unsigned a = ts + 32u * (ks >> 1) + 8u * (ks & 1) + (p == 1 ? 16u : 0u);
              const uint64_t bo = dl + (uint64_t)((ks * 1024) >> 4);
              umma_f16_ts(tr, a, bo, IDESC2, !(fresh && s == 0));
            }
          };
          // (one copy per accumulator: a data-dependent D address costs an
          // elect / broadcast loop per MMA)
          if (rsel)
            umma2(tmem_u + 224u);
          else
            umma2(tmem_u + 192u);
          umma_commit(&bar_pf[b]);  // item k's pixel / record buffer is free once UMMA 2 is done
          if (k == nitems - 1) umma_commit(&bar_end);
          GD_STAMP(3, k);
        }
        cm.next(ntiles);
        if ((cm.t & (kTc2Group - 1)) == 0) rsel ^= 1u;  // the group index grows by one per boundary
        if (cs.n < nitems) issue_s();  // item k + 3 into the S stage item k just released
        if (++st == kTc2S) {
          st = 0;
          ph_p ^= 1u;
        }
        if (++b == kGdBuf) b = 0;
      }
    }
    __syncwarp();
  } else {
    // ======================= epilogue warps: two groups of four (one warp per
    // TMEM lane quarter) take alternate tiles, all 64 pixels each, so that a
    // warp does twice the work per synchronisation and the two groups' waits
    // interleave instead of coinciding
    const int q = warp & 3, grp = warp >> 2;  // lane quarter, tile parity
    const int i = gbase + 32 * q + lane;       // this thread's grain (TMEM lane)
    const int g0w = gbase + 32 * q;            // the warp's first grain
    const unsigned lane_off = (unsigned)(32 * q) << 16;
    // this grain's fp64 line sums [J] in shared memory (stride 128:
    // conflict-free, no registers held across the tile loop); its gradient rows
    // [K] accumulate per line in the CTA's split slot of the partials
    double* acc = g.part_g + (int64_t)(g.split_off + blockIdx.y) * K * g.N + (i < g.N ? i : 0);
    double* R64 = reinterpret_cast<double*>(smem + L::R_OFF) + 32 * q + lane;
    auto flush = [&](const Cur& c) {  // group of item c complete -> fp64; line -> K rows
      uint32_t rv[16], rw[16];
      tmem_ld16_nowait(r_col(c) + lane_off, rv);
      tmem_ld16_nowait(r_col(c) + lane_off + 16u, rw);
      tmem_ld_wait();
      tmem_regs_ready(rv);
      tmem_regs_ready(rw);
#pragma unroll
      for (int j = 0; j < J; ++j)
        R64[j * kTc2Grains] += PGX_GD_FLUSH32 ? (double)(__uint_as_float(rv[j]) + __uint_as_float(rw[j]))
                                              : (double)__uint_as_float(rv[j]) + (double)__uint_as_float(rw[j]);
      if (c.t == ntiles - 1 || c.n == nitems - 1) {  // the line's (or the CTA's) last item
        if (i < g.N) tc_grad_line<DIM, D>(acc, g.N, g.tc_lc + (l0 + c.li) * K, R64, c.li == 0);
#pragma unroll
        for (int j = 0; j < J; ++j) R64[j * kTc2Grains] = 0.0;
      }
    };

    const unsigned sbar_s = (unsigned)__cvta_generic_to_shared(&bar_s[0]);
    const unsigned sbar_f = (unsigned)__cvta_generic_to_shared(&bar_full[0]);
    float inv = 0.0f;
    int li_inv = -1;               // line whose chunk scale `inv` is
    Cur c{0, 0, t0}, cf{0, 0, t0};  // current item; item whose group may be flushed (group 0)
    if (grp == 1) c.next(ntiles);
    for (; c.n < nitems; c.next(ntiles), c.next(ntiles)) {
      if (c.li != li_inv) {
        li_inv = c.li;
        const int sB = __ldg(&g.tc_meta[(l0 + c.li) * g.tc_nchunks + blockIdx.x].x);
        inv = __int_as_float((127 - (sB + 10)) << 23);  // 2^-(sB + 10): S * inv = h~''
      }
      const int st = c.n % kTc2S, b = c.n % kGdBuf;
      const float* rec0 = reinterpret_cast<const float*>(smem + L::REC_OFF + b * L::REC);
      if (q == 0 && lane == 0) GD_STAMP(5, c.n);
      mbar_spin(sbar_s + 8u * st, (unsigned)(c.n / kTc2S) & 1u);
      tc_fence_after();
      if (q == 0 && lane == 0) GD_STAMP(0, c.n);
      if (lane == 0) GD_STAMP(10 + q, c.n);
      // UMMA 1 of this item follows UMMA 2 of item n - 3: the groups ending
      // there are final
      if (grp == 0)
        for (; cf.n + kTc2S <= c.n; cf.next(ntiles))
          if (group_last(cf)) flush(cf);
      mbar_spin(sbar_f + 8u * b, (unsigned)(c.n / kGdBuf) & 1u);  // records visible
      const unsigned long long ninv2 = f2pack(-inv, -inv);
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {  // pixel halves [32 h, 32 h + 32)
        const unsigned ts = tmem + 64u * st + lane_off + 32u * h;
        const float* rec = rec0 + 32 * h;
        uint32_t sv[32];
        tmem_ld32_nowait(ts, sv);
        // label grains of this warp among the half-tile's pixels (rare)
        const int lab_x = reinterpret_cast<const int*>(rec)[3 * kTc2Px + lane];
        const unsigned hit = __ballot_sync(0xffffffffu, (unsigned)(lab_x - g0w) < 32u);
        tmem_ld_wait();
        tmem_regs_ready(sv);
        uint32_t pp[32];  // [0, 16): r'_hi pairs, [16, 32): r'_lo pairs
        // exact split: hi = r' with the 13 low mantissa bits cleared (an fp16
        // value), lo = r' - hi (exact in fp32, |lo| < 2^-10 |r'|) rounded to fp16
        if (PGX_GD_ILV && !hit) {
          // software-pipelined by pixel pairs: exponentials of pair cc, split and
          // conversions of pair cc - LAG
          constexpr int LAG = 3;
          float ra[16], rb[16];
#pragma unroll
          for (int cc = 0; cc < 16 + LAG; ++cc) {
            if (cc < 16) {
              const float2 w2 = *reinterpret_cast<const float2*>(rec + 2 * cc);
              const unsigned long long a01 = ffma2(
                  f2pack(__uint_as_float(sv[2 * cc]), __uint_as_float(sv[2 * cc + 1])), ninv2, f2pack(w2.x, w2.y));
              ra[cc] = ex2_ordered(f2lo(a01));  // p/2 * 2^13 = 2^(13 + w - h~'')
              rb[cc] = ex2_ordered(f2hi(a01));
            }
            if (cc >= LAG) {
              const int c2 = cc - LAG;
              const float h0 = __uint_as_float(__float_as_uint(ra[c2]) & 0xffffe000u);
              const float h1 = __uint_as_float(__float_as_uint(rb[c2]) & 0xffffe000u);
              const unsigned long long lo2 = ffma2(f2pack(h0, h1), f2pack(-1.0f, -1.0f), f2pack(ra[c2], rb[c2]));
              pp[c2] = pack_h2_ordered(h0, h1);
              pp[16 + c2] = pack_h2_ordered(f2lo(lo2), f2hi(lo2));
            }
          }
        } else {
          float rr[32];
#pragma unroll
          for (int x4 = 0; x4 < 32; x4 += 4) {
            const float4 w4 = *reinterpret_cast<const float4*>(rec + x4);
            const unsigned long long a01 =
                ffma2(f2pack(__uint_as_float(sv[x4]), __uint_as_float(sv[x4 + 1])), ninv2, f2pack(w4.x, w4.y));
            const unsigned long long a23 =
                ffma2(f2pack(__uint_as_float(sv[x4 + 2]), __uint_as_float(sv[x4 + 3])), ninv2, f2pack(w4.z, w4.w));
            rr[x4] = ex2_approx(f2lo(a01));  // p/2 * 2^13 = 2^(13 + w - h~'')
            rr[x4 + 1] = ex2_approx(f2hi(a01));
            rr[x4 + 2] = ex2_approx(f2lo(a23));
            rr[x4 + 3] = ex2_approx(f2hi(a23));
          }
          if (hit) {  // label grain: -(1 - p_G)/2 * 2^13 from pass 1 (no cancellation)
            // the pixels of each distinct in-range label at once (a 32-pixel run
            // mostly lies in one grain): one round per distinct label, not per pixel
            const unsigned same = __match_any_sync(0xffffffffu, lab_x);
            unsigned mine = 0u;
            for (unsigned m = hit; m;) {
              const int x = __ffs(m) - 1;
              const unsigned gx = __shfl_sync(0xffffffffu, same, x);
              if (__shfl_sync(0xffffffffu, lab_x, x) == i) mine = gx;
              m &= ~gx;
            }
            if (__any_sync(0xffffffffu, mine != 0u)) {
              const float* qn = rec + 2 * kTc2Px;
#pragma unroll
              for (int x = 0; x < 32; ++x)
                if (mine & (1u << x)) rr[x] = qn[x];
            }
          }
#pragma unroll
          for (int cc = 0; cc < 16; ++cc) {
            const float h0 = __uint_as_float(__float_as_uint(rr[2 * cc]) & 0xffffe000u);
            const float h1 = __uint_as_float(__float_as_uint(rr[2 * cc + 1]) & 0xffffe000u);
            const unsigned long long lo2 =
                ffma2(f2pack(h0, h1), f2pack(-1.0f, -1.0f), f2pack(rr[2 * cc], rr[2 * cc + 1]));
            pp[cc] = pack_h2(h0, h1);
            pp[16 + cc] = pack_h2(f2lo(lo2), f2hi(lo2));
          }
        }
        tmem_st32(ts, pp);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (q == 0 && lane == 0) GD_STAMP(1, c.n);
      if (lane == 0) GD_STAMP(6 + q, c.n);
      if (lane == 0) mbar_arrive(&bar_p[st]);
    }
    // the last groups: complete once the final commit lands
    if (grp == 0) {
      mbar_wait(&bar_end, 0);
      tc_fence_after();
      for (; cf.n < nitems; cf.next(ntiles))
        if (group_last(cf)) flush(cf);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kGdMmaWarp) tmem_dealloc(tmem, 256);
}

}  // namespace pgx
