// pgx_tc_pass2.cuh — PGX_PREC_TC pass 2: the gradient contraction
// sum_x (onehot_G(x) - p(x)) eta(x) (objective.py:109-113) with BOTH
// contractions on the tensor cores (FlashAttention-backward-like, grain-major):
//
//   UMMA 1 (SS)  S^T[128 grains x 64 px] = B''(line)[grains x 3J] . L(x)[px x 3J]^T
//   epilogue     thread = grain = TMEM lane: r' = p/2 * 2^13 = 2^(w13 - h~''),
//                or -(1 - p_G)/2 * 2^13 on the pixel's label grain; split into
//                fp16 hi/lo and written BACK into TMEM over S (packed pairs)
//   UMMA 2 (TS)  R[128 grains x 32] += r'_hi . [L_hi | L_lo]^T + r'_lo . [L_hi | L_lo]^T
//                (A operand from TMEM, K = 2 x 64 pixels, N = 32 = the hi and lo
//                rows of L side by side; columns j and 16 + j are summed in the
//                flush).  8 MMAs per tile: below N = 128 every tcgen05.mma costs
//                a ~54-cycle floor (tools/umma_tput.cu), so the instruction count,
//                not the flops, is what the tensor pipe spends here.
//
// Warp specialisation (FlashAttention-4 style), 288 threads, 2 CTAs per SM:
//   warps 0-7  epilogue: warp w owns TMEM lanes 32 (w % 4) .. (grains) and the
//              pixel half w / 4 of each tile (32 pixels);
//   warp 8     producer: bulk async copies (cp.async.bulk + mbarrier tx counts)
//              of the per-line coefficient image, the tile's pixel operands (one
//              table per problem) and the tile's pass-1 records; issues UMMA 2 of
//              tile n and UMMA 1 of tile n + 3 as soon as the epilogue of tile n
//              has written r' — S is triple-buffered in TMEM, so the tensor core
//              computes logits well ahead of the epilogue's exponentials.
// R alternates between two TMEM accumulators per group of 4 tiles; a finished
// group is flushed into fp64 line sums three tiles later (when it is known to
// be complete) and per line expanded into the K gradient rows.
//
// TMEM (256 columns): S_0..S_2 [0, 192) (64 each), R_a [192, 224), R_b [224, 256).
// Within S_s, pixel half h keeps r'_hi in [32h, 32h + 16) and r'_lo in
// [32h + 16, 32h + 32): only columns its own warps have already read.
#pragma once

#include "pgx_grid_common.cuh"
#include "pgx_tc_coeffs.cuh"
#include "pgx_tc_common.cuh"

namespace pgx {

constexpr int kTc2Epi = 256;              // epilogue threads (8 warps)
constexpr int kTc2Threads = kTc2Epi + 32;  // + producer warp
constexpr int kTc2Grains = 128;           // grains per CTA (TMEM lanes)
constexpr int kTc2Px = kTcPixTile;        // pixels per tile
constexpr int kTc2Group = 4;              // tiles per fp32 R group before the fp64 flush
constexpr int kTc2S = 3;                  // S stages in TMEM (UMMA 1 runs 3 tiles ahead)
constexpr int kTc2Buf = 6;                // tile buffers (pixel operands + records)
constexpr int kTc2RecFloats = 4 * kTc2Px;  // w13[64] | wl13[64] | qn[64] | label[64]

// The exponent 13 + w - h~'' is formed from the fp32-rounded w = (float)w13 and,
// optionally, its fp32 residual wl13 (pass-1 record). The residual is below the
// logit error itself (|w13 - w| <= 2^-24 |w13| against ~2^-22 |h''| for the
// fp16-split logits; measured c1-c5 tc-vs-exact errors unchanged without it,
// tools/tc_err.py), so it is dropped -- one FADD and half the record loads per
// logit -- except in the high-degree 2-D kernels, where the register allocation
// at the 96-register cap came out 2% slower without it (c5).
template <int DIM, int D>
constexpr bool kTc2WithResidual = DIM == 2 && D >= 6;

template <int J>
struct TcP2Smem {
  static constexpr int KS = tc_ksteps(J);
  static constexpr int A1 = KS * kTc2Grains * 32;  // coefficient image (128 rows)
  static constexpr int PIX = tc_pix_bytes<J>();
  static constexpr int REC = kTc2RecFloats * 4;
  static constexpr int A1_OFF = 0;
  static constexpr int PIX_OFF = A1_OFF + 2 * A1;
  static constexpr int REC_OFF = PIX_OFF + kTc2Buf * PIX;
  static constexpr int TOTAL = REC_OFF + kTc2Buf * REC;
};

// (line index, tile) walk over a CTA's items without divisions
struct Tc2Cursor {
  int n = 0, li = 0, t = 0;
  __device__ explicit Tc2Cursor(int t0) : t(t0) {}
  __device__ __forceinline__ void advance(int ntiles) {
    ++n;
    if (++t == ntiles) {
      t = 0;
      ++li;
    }
  }
};

template <int DIM, int D, bool MID>
__global__ void __launch_bounds__(kTc2Threads, 2) k_tc_pass2(GridParams g) {
  constexpr int J = D + 1;
  constexpr int K = feature_count(DIM, D);
  using L = TcP2Smem<J>;
  constexpr int KS = L::KS;
  constexpr uint32_t IDESC1 = umma_idesc_f16(128, kTc2Px);
  constexpr uint32_t IDESC2 = umma_idesc_f16(128, 32);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_full[kTc2Buf], bar_a[2], bar_s[kTc2S], bar_p[kTc2S], bar_end;
  __shared__ unsigned tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gbase = blockIdx.x * kTc2Grains;
  // items (line, tile) [line_lo, lines) x [0, ntiles) of this launch,
  // items_per_split per CTA row; MID: the CTA may start and end mid-line
  // (otherwise items_per_split is a multiple of ntiles and the mid-line
  // bookkeeping compiles away: it costs registers the hot loop needs)
  const int ntiles = g.side / kTc2Px;
  const int gpl = (ntiles + kTc2Group - 1) / kTc2Group;  // R groups per line
  int64_t l0;  // first line (partial when t0 > 0)
  int nitems, nlines, t0 = 0;
  if (MID) {
    const int64_t a0 = g.line_lo * ntiles + (int64_t)blockIdx.y * g.items_per_split;
    const int64_t a1 = min((int64_t)g.lines * ntiles, a0 + g.items_per_split);
    if (a1 <= a0) return;
    nitems = (int)(a1 - a0);
    l0 = a0 / ntiles;
    t0 = (int)(a0 - l0 * ntiles);
    nlines = (int)((a1 - 1) / ntiles - l0 + 1);
  } else {
    const int lps = (int)(g.items_per_split / ntiles);
    l0 = g.line_lo + (int64_t)blockIdx.y * lps;
    nlines = (int)(min((int64_t)g.lines, l0 + lps) - l0);
    nitems = nlines * ntiles;
    if (nitems <= 0) return;
  }

  if (warp == 8) tmem_alloc(&tmem_base, 256);
  if (tid == kTc2Epi) {
    for (int b = 0; b < kTc2Buf; ++b) mbar_init(&bar_full[b], 1);
    for (int b = 0; b < kTc2S; ++b) {
      mbar_init(&bar_s[b], 1);
      mbar_init(&bar_p[b], kTc2Epi / 32);
    }
    mbar_init(&bar_a[0], 1);
    mbar_init(&bar_a[1], 1);
    mbar_init(&bar_end, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();  // PDL: pass 1's records, fix lists and partials are complete
  const unsigned tmem = tmem_base;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  auto group_last = [&](const Tc2Cursor& c) {
    return c.t == ntiles - 1 || c.t % kTc2Group == kTc2Group - 1 || (MID && c.n == nitems - 1);
  };
  auto r_col = [&](const Tc2Cursor& c) {  // R accumulator of the item's group
    return tmem + 192u + 32u * (unsigned)((c.li * gpl + c.t / kTc2Group) & 1);
  };

  if (warp == 8) {
    // ======================= producer / MMA warp: the loop is warp-uniform,
    // one lane issues the copies and the MMAs
    const bool leader = lane == 0;
    const uint64_t d_a1 = umma_desc(sbase + L::A1_OFF);
    const uint64_t d_pix = umma_desc(sbase + L::PIX_OFF);
    Tc2Cursor cl(t0), cs(t0), cm(t0), cw(t0);  // next load, UMMA 1, UMMA 2, completion check
    auto load_next = [&]() {
      const int b = cl.n % kTc2Buf;
      if (leader) {
        mbar_arrive_expect_tx(&bar_full[b], L::PIX + L::REC);
        bulk_g2s(smem + L::PIX_OFF + b * L::PIX, g.tc_pix + (int64_t)cl.t * L::PIX, L::PIX,
                 &bar_full[b]);
        bulk_g2s(smem + L::REC_OFF + b * L::REC,
                 g.tc_rec + ((l0 + cl.li) * ntiles + cl.t) * (int64_t)kTc2RecFloats, L::REC,
                 &bar_full[b]);
      }
      cl.advance(ntiles);
    };
    auto load_coef = [&](int li) {
      const int b = li & 1;
      if (leader) {
        mbar_arrive_expect_tx(&bar_a[b], L::A1);
        bulk_g2s(smem + L::A1_OFF + b * L::A1,
                 g.tc_img + ((l0 + li) * g.tc_nchunks + blockIdx.x) * (int64_t)L::A1, L::A1,
                 &bar_a[b]);
      }
    };
    auto issue_s = [&]() {  // UMMA 1 of item cs into S_(n % 3)
      const int b = cs.n % kTc2Buf, st = cs.n % kTc2S;
      if (cs.t == 0 || (MID && cs.n == 0)) mbar_wait(&bar_a[cs.li & 1], (unsigned)(cs.li >> 1) & 1u);
      mbar_wait(&bar_full[b], (unsigned)(cs.n / kTc2Buf) & 1u);
      tc_fence_after();
      if (leader) {
        const uint64_t da = d_a1 + (uint64_t)(((cs.li & 1) * L::A1) >> 4);
        const uint64_t db = d_pix + (uint64_t)((b * L::PIX) >> 4);
#pragma unroll
        for (int s = 0; s < KS; ++s)
          umma_f16_ss(tmem + 64u * st, da + (uint64_t)((s * kTc2Grains * 32) >> 4),
                      db + (uint64_t)((s * kTc2Px * 32) >> 4), IDESC1, s > 0);
        umma_commit(&bar_s[st]);
      }
      __syncwarp();
      cs.advance(ntiles);
    };
    load_coef(0);
    if (nlines > 1) load_coef(1);
    while (cl.n < nitems && cl.n < kTc2Buf - 1) load_next();
    while (cs.n < nitems && cs.n < kTc2S) issue_s();
    for (int k = 0; k < nitems; ++k) {
      const int st = k % kTc2S, b = k % kTc2Buf;
      mbar_wait(&bar_p[st], (unsigned)(k / kTc2S) & 1u);  // r' of item k is in S_st
      tc_fence_after();
      if (leader) {  // UMMA 2: R += [r_hi; r_lo] . [L_hi | L_lo]^T over the 64 pixels
        const unsigned tr = r_col(cm);
        const unsigned ts = tmem + 64u * st;
        const uint64_t dl = d_pix + (uint64_t)((b * L::PIX + KS * (kTc2Px * 32)) >> 4);
        const bool fresh = cm.t % kTc2Group == 0 || (MID && cm.n == 0);  // a group's first item
#pragma unroll
        for (int s = 0; s < 2 * (kTc2Px / 16); ++s) {
          const int p = s / (kTc2Px / 16), ks = s % (kTc2Px / 16);
          // pixels [16 ks, 16 ks + 16): half ks / 2, packed columns 8 (ks % 2); p = 1: r_lo
          const unsigned a = ts + 32u * (ks >> 1) + 8u * (ks & 1) + (p == 1 ? 16u : 0u);
          const uint64_t bo = dl + (uint64_t)((ks * 1024) >> 4);
          umma_f16_ts(tr, a, bo, IDESC2, !(fresh && s == 0));
        }
      }
      __syncwarp();
      cm.advance(ntiles);
      if (cs.n < nitems)
        issue_s();  // item k + 3 into the S stage item k just released
      else if (k == nitems - 1 && leader)
        umma_commit(&bar_end);
      if (k + 2 < nitems) {
        // UMMA 1 of item k + 2 complete => every MMA issued before it, incl. UMMA 2
        // of item k - 1: its buffer is free; so is a finished line's coefficient image
        mbar_wait(&bar_s[(k + 2) % kTc2S], (unsigned)((k + 2) / kTc2S) & 1u);
        if (cl.n < nitems) load_next();
        for (; cw.n <= k + 2; cw.advance(ntiles))  // every item up to k + 2 is done
          if (cw.t == ntiles - 1 && cw.li + 2 < nlines) load_coef(cw.li + 2);
      }
    }
  } else {
    // ======================= epilogue warps
    const int q = warp & 3, h = warp >> 2;  // lane quarter, pixel half
    const int i = gbase + 32 * q + lane;     // this thread's grain (TMEM lane)
    const bool active = i < g.N;
    const unsigned lane_off = (unsigned)(32 * q) << 16;
    double* acc = g.part_g + (int64_t)(g.split_off + blockIdx.y) * K * g.N + (active ? i : 0);
    const double rs = -2.0 / (8192.0 * 1024.0);  // R_true = -2 acc 2^-(13 + 10): r' = -r
    double R64[J];
#pragma unroll
    for (int j = 0; j < J; ++j) R64[j] = 0.0;
    auto flush = [&](const Tc2Cursor& c) {  // group of item c complete -> fp64; line -> K rows
      uint32_t rv[16], rw[16];
      tmem_ld16_nowait(r_col(c) + lane_off, rv);
      tmem_ld16_nowait(r_col(c) + lane_off + 16u, rw);
      tmem_ld_wait();
      tmem_regs_ready(rv);
      tmem_regs_ready(rw);
#pragma unroll
      for (int j = 0; j < J; ++j)
        R64[j] += (double)__uint_as_float(rv[j]) + (double)__uint_as_float(rw[j]);
      if (c.t == ntiles - 1 || (MID && c.n == nitems - 1)) {  // the line's (or the CTA's) last item
        if (active) {
          const double* lcp = g.tc_lc + (l0 + c.li) * K;  // k_tc_coeffs
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const double prev = c.li == 0 ? 0.0 : acc[(int64_t)k * g.N];
            acc[(int64_t)k * g.N] = fma(lcp[k], rs * R64[alpha_of(DIM, D, k, DIM - 1)], prev);
          }
        }
#pragma unroll
        for (int j = 0; j < J; ++j) R64[j] = 0.0;
      }
    };

    int sB_next = g.tc_meta[l0 * g.tc_nchunks + blockIdx.x].x;
    float inv = 0.0f;
    Tc2Cursor c(t0), cf(t0);  // current item; item whose group may be flushed (lags by kTc2S)
    for (; c.n < nitems; c.advance(ntiles)) {
      if (c.t == 0 || (MID && c.n == 0)) {
        inv = ldexpf(1.0f, -(sB_next + 10));  // S * inv = h~''
        if (c.li + 1 < nlines) sB_next = g.tc_meta[(l0 + c.li + 1) * g.tc_nchunks + blockIdx.x].x;
      }
      const int st = c.n % kTc2S, b = c.n % kTc2Buf;
      const unsigned ts = tmem + 64u * st;
      const float* rec = reinterpret_cast<const float*>(smem + L::REC_OFF + b * L::REC) + 32 * h;
      mbar_wait(&bar_s[st], (unsigned)(c.n / kTc2S) & 1u);
      tc_fence_after();
      // UMMA 1 of this item follows UMMA 2 of item n - 3: that group may be final
      if (c.n >= kTc2S) {
        if (h == 0 && group_last(cf)) flush(cf);
        cf.advance(ntiles);
      }
      uint32_t sv[32];
      tmem_ld32_nowait(ts + lane_off + 32u * h, sv);
      mbar_wait(&bar_full[b], (unsigned)(c.n / kTc2Buf) & 1u);  // records visible
      const int lab_me = reinterpret_cast<const int*>(rec)[3 * kTc2Px + lane];
      const bool lab_warp = __any_sync(0xffffffffu, (unsigned)(lab_me - (gbase + 32 * q)) < 32u);
      tmem_ld_wait();
      tmem_regs_ready(sv);
      float rr[32];
#pragma unroll
      for (int x4 = 0; x4 < 32; x4 += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(rec + x4);
        const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
        if constexpr (!kTc2WithResidual<DIM, D>) {
#pragma unroll
          for (int e = 0; e < 4; ++e)  // p/2 * 2^13 = 2^(13 + w - h~'')
            rr[x4 + e] = ex2_approx(fmaf(-__uint_as_float(sv[x4 + e]), inv, wv[e]));
        } else {
          const float4 l4 = *reinterpret_cast<const float4*>(rec + kTc2Px + x4);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            rr[x4 + e] = ex2_approx(fmaf(-__uint_as_float(sv[x4 + e]), inv, wv[e]) + lv[e]);
        }
      }
      if (lab_warp) {  // label grain: -(1 - p_G)/2 * 2^13 from pass 1 (no cancellation)
        const int* labs = reinterpret_cast<const int*>(rec) + 3 * kTc2Px;
        const float* qn = rec + 2 * kTc2Px;
#pragma unroll
        for (int x = 0; x < 32; ++x)
          if (labs[x] == i) rr[x] = qn[x];
      }
      uint32_t ph[16], pl[16];
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const __half2 h2 = __floats2half2_rn(rr[2 * cc], rr[2 * cc + 1]);
        const float2 hf = __half22float2(h2);
        const __half2 l2 = __floats2half2_rn(rr[2 * cc] - hf.x, rr[2 * cc + 1] - hf.y);
        ph[cc] = *reinterpret_cast<const uint32_t*>(&h2);
        pl[cc] = *reinterpret_cast<const uint32_t*>(&l2);
      }
      tmem_st16(ts + lane_off + 32u * h, ph);
      tmem_st16(ts + lane_off + 32u * h + 16u, pl);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p[st]);
    }
    // the last groups: complete once the final commit lands
    mbar_wait(&bar_end, 0);
    tc_fence_after();
    for (; cf.n < nitems; cf.advance(ntiles))
      if (h == 0 && group_last(cf)) flush(cf);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 256);
}

}  // namespace pgx
