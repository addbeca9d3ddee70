// pgx_tc_sweep.cuh — PGX_PREC_TC pass 1 ("sweep"): the logit contraction
// h'' = L(x_fast) B''(line) (objective.py:99) on the tcgen05 tensor cores and
// ONE streaming pass over the grains per pixel on the CUDA cores: running
// min, online log-sum-exp (objective.py:102-106) and the arg-min bookkeeping
// of geometry.py:201-210.
//
// One persistent CTA per SM, warp-specialised:
//   warps 0-15  epilogue: slot s = warp / 4 owns one 128-pixel tile of the
//               item (thread = TMEM lane = pixel), lane quarter warp % 4, so
//               a slot's four warps sit on the four SM sub-partitions;
//   warp 16     loader: cp.async.bulk of the per-line coefficient images
//               (pgx_tc_coeffs.cuh) into a RING-deep shared-memory ring;
//   warp 17     MMA issuer: one lane issues tcgen05.mma (M = 128 pixels,
//               N = 64 grains, K = 16 tc_ksteps(J), fp16 3-product split,
//               fp32 accumulate) into two TMEM accumulators per slot, each
//               committed to a "full" mbarrier; the slot's warps release a
//               buffer ("free", 4 arrivals) right after loading it.
// TMEM: 4 slots x 2 buffers x 64 columns = 512.  An item is 4 consecutive
// tiles (one line when the side has >= 4 tiles); items are strided over the
// CTAs in a fixed order (deterministic per-CTA partials).  Pixel operands are
// double-buffered per slot: the tile of the next item is written while the
// current one runs.
//
// Epilogue per 64-column block: two tcgen05.ld of 32 columns; per 32 columns
// (h~'' = S * inv, inv = 2^-(sB + 10) of the 128-grain chunk):
//   mb = block min (FMNMX3); the three best 32-column block minima and, for
//   the best two, the columns within 2 delta + tie band of their min (a bit
//   mask) are tracked; s' = sum_{i != G} 2^(ref - h~''_i) with a reference
//   that moves only when the min falls more than kSwStale below it:
//   packed FFMA2 (argument pairs) + MUFU.EX2 + packed FADD2 per logit pair.
// Per pixel at the end: the label term in fp64, the exact fp64 tie-tolerant
// arg-min over the masked columns (a third block as close, or an overflowing
// candidate list, queues the pixel for the tail's exact re-scan), the pass-2
// record and the per-pixel statistics.
#pragma once

#include "pgx_grid_common.cuh"
#include "pgx_tc_coeffs.cuh"
#include "pgx_tc_common.cuh"
#include "pgx_tc_shared.cuh"

namespace pgx {

constexpr int kSwSlots = 4;                      // 128-pixel tiles per item
constexpr int kSwEpiWarps = 4 * kSwSlots;        // 16
constexpr int kSwThreads = 32 * kSwEpiWarps + 64;  // + loader warp + MMA warp
constexpr int kSwCols = 64;                      // grains per MMA block (UMMA N)
constexpr int kSwBufs = 2;                       // accumulators per slot
constexpr int kSwRingMax = 16;                   // coefficient images in flight
constexpr float kSwStale = 24.0f;                // ref may lag the min by this (log2 units)
// pairs (of the 16 per 32-column block) whose exponentials run on the FMA pipe
// (pexp2) instead of MUFU: the sweep is MUFU bound
#ifndef PGX_SW_POLY
#define PGX_SW_POLY 2
#endif

template <int J>
struct SwSmem {
  static constexpr int KS = tc_ksteps(J);
  static constexpr int A_TILE = KS * kTcThreadsTile * 32;  // one 128-row pixel operand
  static constexpr int IMG = tc_img_bytes<J>();
  static constexpr int A_OFF = 0;
  static constexpr int IMG_OFF = A_OFF + 2 * kSwSlots * A_TILE;
  static constexpr int BUDGET = 200 * 1024;
  static constexpr int RING = (BUDGET - IMG_OFF) / IMG < kSwRingMax ? (BUDGET - IMG_OFF) / IMG : kSwRingMax;
  static constexpr int TOTAL = IMG_OFF + RING * IMG;
};

// ASSIGN: the hard-assignment variant (pgx_assign; objective.py:62-77): the
// same sweep without exponentials, label term or pass-2 records; it writes the
// 1-based arg-min label and the top-2 margin per pixel.
// Sides that are not a multiple of 128 run on tiles padded to g.pside: the
// padding pixels ride through the MMAs and barriers, contribute nothing and
// get an all-zero (-inf exponent) pass-2 record.
template <int DIM, int D, bool ASSIGN>
__global__ void __launch_bounds__(kSwThreads, 1) k_tc_sweep(GridParams g) {
  constexpr int J = D + 1;
  using L = SwSmem<J>;
  constexpr int KS = L::KS;
  constexpr int QB = kTcCoefChunk / kSwCols;  // MMA blocks per coefficient image
  constexpr uint32_t IDESC = umma_idesc_f16(128, kSwCols);
  constexpr int W_LOAD = kSwEpiWarps, W_MMA = kSwEpiWarps + 1;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_full[kSwSlots][kSwBufs], bar_free[kSwSlots][kSwBufs];
  __shared__ uint64_t bar_a[kSwSlots][2];
  __shared__ uint64_t bar_img[kSwRingMax], bar_imgfree[kSwRingMax];
  __shared__ unsigned tmem_base;
  __shared__ double red_d[kSwEpiWarps][2];
  __shared__ long long red_i[kSwEpiWarps][3];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = g.N;
  const double c = g.c;
  const int tpl = g.pside / kTcThreadsTile;  // tiles per (padded) line
  const int64_t ntiles = (int64_t)g.lines * tpl;
  const int64_t nitems = (ntiles + kSwSlots - 1) / kSwSlots;
  const int nimg = (N + kTcCoefChunk - 1) / kTcCoefChunk;
  const int nblk = (N + kSwCols - 1) / kSwCols;

  if (warp == W_MMA) tmem_alloc(&tmem_base, 512);
  if (tid == 32 * W_LOAD) {
    for (int s = 0; s < kSwSlots; ++s) {
      for (int b = 0; b < kSwBufs; ++b) {
        mbar_init(&bar_full[s][b], 1);
        mbar_init(&bar_free[s][b], 4);  // the slot's four warps
      }
      mbar_init(&bar_a[s][0], 4);
      mbar_init(&bar_a[s][1], 4);
    }
    for (int r = 0; r < L::RING; ++r) {
      mbar_init(&bar_img[r], 1);
      mbar_init(&bar_imgfree[r], 1);  // the MMA issuer's commit after the image's last MMA
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();  // PDL: the set-up above overlaps the predecessor (k_tc_coeffs)
  const unsigned tmem = tmem_base;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);

  // the distinct lines among an item's tiles: js[s] = image index of slot s
  // within a chunk's group of images; returns the group size
  auto distinct = [&](int64_t it, int (&js)[kSwSlots]) {
    const int64_t t0 = it * kSwSlots;
    int n = 0;
    for (int s = 0; s < kSwSlots; ++s) {
      if (s > 0 && t0 + s < ntiles && (t0 + s) / tpl == (t0 + s - 1) / tpl)
        js[s] = js[s - 1];
      else
        js[s] = t0 + s < ntiles ? n++ : 0;
    }
    return n;
  };

  if (warp == W_LOAD) {
    // ======================== loader: every image of every item, in the MMA
    // issuer's consumption order, into the ring
    int gl = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      int js[kSwSlots];
      const int nl = distinct(it, js);
      for (int ci = 0; ci < nimg; ++ci)
        for (int j = 0; j < nl; ++j, ++gl) {
          const int slot = gl % L::RING;
          mbar_wait_sleep(&bar_imgfree[slot], (unsigned)((gl / L::RING) & 1) ^ 1u);
          if (lane == 0) {
            int s = 0;
            while (js[s] != j) ++s;  // first slot on distinct line j
            const int64_t line = (it * kSwSlots + s) / tpl;
            mbar_arrive_expect_tx(&bar_img[slot], L::IMG);
            bulk_g2s(smem + L::IMG_OFF + slot * L::IMG,
                     g.tc_img + (line * g.tc_nchunks + ci) * (int64_t)L::IMG, L::IMG, &bar_img[slot]);
          }
          __syncwarp();
        }
    }
  } else if (warp == W_MMA) {
    // ======================== MMA issuer (lane 0 issues; the warp walks in step)
    int gc = 0;        // images consumed so far
    unsigned rc = 0;   // 64-column rounds so far (all slots in step)
    int li = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x, ++li) {
      int js[kSwSlots];
      const int nl = distinct(it, js);
      bool act[kSwSlots];
      const int ib = li & 1;
#pragma unroll
      for (int s = 0; s < kSwSlots; ++s) {
        act[s] = it * kSwSlots + s < ntiles;
        if (act[s]) mbar_wait(&bar_a[s][ib], (unsigned)(li >> 1) & 1u);
      }
      for (int ci = 0; ci < nimg; ++ci) {
        for (int j = 0; j < nl; ++j)
          mbar_wait(&bar_img[(gc + j) % L::RING], (unsigned)(((gc + j) / L::RING) & 1));
        tc_fence_after();
        for (int qb = 0; qb < QB && ci * QB + qb < nblk; ++qb, ++rc) {
          const unsigned buf = rc & 1u;
#pragma unroll
          for (int s = 0; s < kSwSlots; ++s) {
            if (!act[s]) continue;
            mbar_wait(&bar_free[s][buf], ((rc >> 1) & 1u) ^ 1u);
            tc_fence_after();
            if (lane == 0) {
              const unsigned a_s = sbase + L::A_OFF + (unsigned)((ib * kSwSlots + s) * L::A_TILE);
              const unsigned b_s = sbase + L::IMG_OFF + (unsigned)(((gc + js[s]) % L::RING) * L::IMG) +
                                   (unsigned)(qb * (kSwCols / 8) * 256);
#pragma unroll
              for (int k = 0; k < KS; ++k)
                umma_f16_ss(tmem + (unsigned)((s * kSwBufs + buf) * kSwCols),
                            umma_desc(a_s + k * (kTcThreadsTile * 32)),
                            umma_desc(b_s + k * (kTcCoefChunk * 32)), IDESC, k > 0);
              umma_commit(&bar_full[s][buf]);
            }
            __syncwarp();
          }
        }
        if (lane == 0)
          for (int j = 0; j < nl; ++j) umma_commit(&bar_imgfree[(gc + j) % L::RING]);
        __syncwarp();
        gc += nl;
      }
    }
  } else {
    // ======================== epilogue: thread = pixel of slot s
    const int s = warp >> 2, q = warp & 3;
    const unsigned lane_off = (unsigned)(32 * q) << 16;
    const int prow = 32 * q + lane;  // row of the slot's 128-pixel tile
    const unsigned t_slot = tmem + lane_off + (unsigned)(s * kSwBufs * kSwCols);
    const unsigned a_full = (unsigned)__cvta_generic_to_shared(&bar_full[s][0]);
    const unsigned a_free = (unsigned)__cvta_generic_to_shared(&bar_free[s][0]);
    double ell = 0.0, e0 = 0.0;
    long long correct = 0, amb = 0, nonfinite = 0;
    unsigned rc = 0;

    // pixel operand row of item it2's tile in buffer ib:
    // A'[p][k] = 2^10 L_j(x_fast), k = b J + j, K blocks [hi, hi, lo]
    auto write_a = [&](int64_t it2, int ib) {
      const int64_t tile = it2 * kSwSlots + s;
      if (tile >= ntiles) return;
      const int col = (int)(tile % tpl) * kTcThreadsTile + prow;
      double u[J];
      axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
      __half hi[J], lo[J];
#pragma unroll
      for (int j = 0; j < J; ++j) split_f16(col < g.side ? u[j] * 1024.0 : 0.0, hi[j], lo[j]);  // padding: 0
      unsigned char* A_s = smem + L::A_OFF + (ib * kSwSlots + s) * L::A_TILE;
#pragma unroll
      for (int k = 0; k < 16 * KS; ++k) {
        const int b = k / J, j = k % J;
        const __half val = k < 3 * J ? (b < 2 ? hi[j] : lo[j]) : __float2half(0.0f);
        *reinterpret_cast<__half*>(A_s + (k / 16) * (kTcThreadsTile * 32) + slab_off(prow, k % 16)) = val;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_a[s][ib]);
    };

    int li = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x, ++li) {
      if (li == 0) write_a(it, 0);
      if (it + gridDim.x < nitems) write_a(it + gridDim.x, (li + 1) & 1);
      const int64_t tile = it * kSwSlots + s;
      if (tile >= ntiles) continue;  // (only in a CTA's last item; no MMA is issued for it)
      const int64_t line = tile / tpl;
      const int col = (int)(tile % tpl) * kTcThreadsTile + prow;
      const bool valid = col < g.side;  // (false on the padding of a side % 128 != 0 grid)
      const int64_t p = line * g.side + col;
      const int lab = valid && g.labels ? g.labels[p] : -1;
      const double* coef_line = g.tc_coef + line * (int64_t)N * J;
      const int2* meta = g.tc_meta + line * g.tc_nchunks;
      float ref = CUDART_INF_F, m1 = CUDART_INF_F, m2b = CUDART_INF_F, m3b = CUDART_INF_F, bmax = 0.0f;
      int b1 = 0, b2 = 0;
      unsigned mask1 = 0u, mask2 = 0u;  // columns of 32-blocks b1, b2 within the candidate window
      float sx = 0.0f, sxc = 0.0f;      // Kahan-compensated sum of the 32-block sums
      float gm1 = CUDART_INF_F, gm2 = CUDART_INF_F;  // ASSIGN + margins: two smallest logits (fp32)
      const bool want_margin = ASSIGN && g.margin_out != nullptr;
      float inv = 0.0f, rinv = 0.0f, dblk = 0.0f;
      const float bandf = (float)(c * fmax(kTieRtol, g.tau_amb)), inv_cf = (float)(1.0 / c);

      // one 32-column block kb (grains 32 kb ..): min bookkeeping + exponentials
      // (w: the block's 32 logits in S units, padding columns already +inf)
      auto block32 = [&](int kb, const float (&w)[32]) {
        float t11[11];
#pragma unroll
        for (int e = 0; e < 10; ++e) t11[e] = fminf(w[3 * e], fminf(w[3 * e + 1], w[3 * e + 2]));
        t11[10] = fminf(w[30], w[31]);
        const float mb = fminf(fminf(fminf(t11[0], fminf(t11[1], t11[2])), fminf(t11[3], fminf(t11[4], t11[5]))),
                               fminf(fminf(t11[6], fminf(t11[7], t11[8])), fminf(t11[9], t11[10])));
        const float mbs = mb * inv;
        if (ASSIGN && want_margin) {  // runner-up for the reported margin: the block's two smallest
          float a = CUDART_INF_F, b = CUDART_INF_F;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float t = fmaxf(a, w[e]);
            a = fminf(a, w[e]);
            b = fminf(b, t);
          }
          const float a1 = a * inv, a2 = b * inv;
          gm2 = fminf(fmaxf(gm1, a1), fminf(gm2, a2));
          gm1 = fminf(gm1, a1);
        }
        if (mbs < m3b) {  // top-3 blocks (rare after the first few)
          if (mbs < m2b) {
            // candidate columns: within 2 delta + tie band of the block min; bit e =
            // sign of thr - w_e (exact, no FTZ), i.e. w_e > thr or +inf padding
            const float thr = (mbs + 2.0f * dblk + bandf * (1.0f + fabsf(mbs) * inv_cf) * 1.001f) * rinv;
            unsigned nm = 0u;
#pragma unroll
            for (int e = 31; e >= 0; --e) nm = __funnelshift_l(__float_as_uint(__fsub_rn(thr, w[e])), nm, 1);
            const unsigned mk = ~nm;
            m3b = m2b;
            if (mbs < m1) {
              m2b = m1;
              b2 = b1;
              mask2 = mask1;
              m1 = mbs;
              b1 = kb;
              mask1 = mk;
            } else {
              m2b = mbs;
              b2 = kb;
              mask2 = mk;
            }
          } else {
            m3b = mbs;
          }
          if (mbs < ref - kSwStale) {  // (also the first block: ref = +inf)
            const float nref = mbs - 1.0f;
            const double f = exp2((double)nref - (double)ref);
            sx = (float)((double)sx * f);
            sxc = (float)((double)sxc * f);
            ref = nref;
          }
        }
        if constexpr (!ASSIGN) {
          const unsigned long long ninv2 = f2pack(-inv, -inv), ref2 = f2pack(ref, ref);
          unsigned long long sa = 0ull, sb = 0ull;
          const int labc = lab - kb * 32;
          // padding columns (+inf) give exact zeros: only a block holding some
          // lane's label column needs the masked loop
          if (!__any_sync(0xffffffffu, (unsigned)labc < 32u)) {
  #pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const unsigned long long a = ffma2(f2pack(w[e], w[e + 1]), ninv2, ref2);
              // (every (16 / PGX_SW_POLY)-th pair on the FMA pipe)
              const bool poly = PGX_SW_POLY > 0 && (e / 2) % (16 / (PGX_SW_POLY > 0 ? PGX_SW_POLY : 1)) == 1;
              const unsigned long long y = poly ? pexp2(a) : f2pack(ex2_approx(f2lo(a)), ex2_approx(f2hi(a)));
              if (e & 2)
                sb = fadd2(sb, y);
              else
                sa = fadd2(sa, y);
            }
          } else {
  #pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const unsigned long long a = ffma2(f2pack(w[e], w[e + 1]), ninv2, ref2);
              const float y0 = ex2_approx(f2lo(a)), y1 = ex2_approx(f2hi(a));
              const unsigned long long y = f2pack(e != labc ? y0 : 0.0f, e + 1 != labc ? y1 : 0.0f);
              if (e & 2)
                sb = fadd2(sb, y);
              else
                sa = fadd2(sa, y);
            }
          }
          const unsigned long long s2 = fadd2(sa, sb);
          const float y = (f2lo(s2) + f2hi(s2)) - sxc;  // Kahan step
          const float t = sx + y;
          sxc = (t - sx) - y;
          sx = t;
        }
      };

#pragma unroll 1
      for (int kb = 0; kb < nblk; ++kb, ++rc) {
        if (kb % QB == 0) {  // scale and error bound of 128-grain chunk kb / QB
          const int2 mt = __ldg(meta + kb / QB);
          rinv = __int_as_float((127 + (mt.x + 10)) << 23);
          inv = __int_as_float((127 - (mt.x + 10)) << 23);  // 2^-(sB + 10): S * inv = h~''
          const float bn = __int_as_float(mt.y);
          bmax = fmaxf(bmax, bn);
          dblk = 2.0f * (4.7683716e-07f + 3 * J * 5.9604645e-08f) * bn + 1e-30f;
        }
        const unsigned buf = rc & 1u;
        mbar_spin(a_full + 8u * buf, (rc >> 1) & 1u);
        tc_fence_after();
        const unsigned taddr = t_slot + buf * kSwCols;
        uint32_t r0[32];
        float w[32];
        tmem_ld32_nowait(taddr, r0);
        tmem_ld_wait();
        tmem_regs_ready(r0);
        const int cn = N - kb * kSwCols;  // valid columns of this block (>= 64 but in the last)
#pragma unroll
        for (int e = 0; e < 32; ++e) w[e] = __uint_as_float(r0[e]);
        if (cn < 32) {  // the last block only: padding grains (zero images) -> +inf
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e >= cn) w[e] = CUDART_INF_F;
        }
        block32(2 * kb, w);
        tmem_ld32_nowait(taddr + 32u, r0);
        tmem_ld_wait();
        tmem_regs_ready(r0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_addr(a_free + 8u * buf);
        if (cn > 32) {
#pragma unroll
          for (int e = 0; e < 32; ++e) w[e] = __uint_as_float(r0[e]);
          if (cn < 64) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e + 32 >= cn) w[e] = CUDART_INF_F;
          }
          block32(2 * kb + 1, w);
        }
      }

      // ------------------------------------------------ per-pixel finish
      if (!valid) {
        if (!ASSIGN && g.tc_rec) {  // r' = 2^(-inf) = 0 for every grain, no label grain
          float* rec = g.tc_rec + (line * (g.pside / kTcPixTile) + (col >> 6)) * (4 * kTcPixTile) + (col & 63);
          rec[0] = -CUDART_INF_F;
          rec[kTcPixTile] = 0.0f;
          rec[2 * kTcPixTile] = 0.0f;
          reinterpret_cast<int*>(rec)[3 * kTcPixTile] = -1;
        }
        continue;
      }
      // |h~'' - h''| <= delta: fp16 split (2^-21 relative per operand pair) plus
      // the fp32 accumulation of 3J products; generous factor 2
      const float delta = 2.0f * (4.7683716e-07f + 3 * J * 5.9604645e-08f) * bmax + 1e-30f;
      const double band = c * fmax(kTieRtol, g.tau_amb) * (1.0 + fabs((double)m1 / c));
      const float wnd = 2.0f * delta + (float)band * 1.001f + 1e-30f;
      double u[J];
      axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
      TcRare st;
      st.m = CUDART_INF;
      st.m2 = CUDART_INF;
      st.cnt = 0;
      st.flags = 0;
      st.b0 = st.b1 = -1;
      // exact fp64 scan of the candidate columns: block b1, and block b2 when
      // its min is as close (in index order: the tie rule picks the smallest)
      const bool two = m2b <= m1 + wnd;
      const int bl = two && b2 < b1 ? b2 : b1, bh = two && b2 < b1 ? b1 : b2;
      const unsigned ml = two && b2 < b1 ? mask2 : mask1, mh = two && b2 < b1 ? mask1 : mask2;
      for (unsigned mk = ml; mk; mk &= mk - 1u) {
        const int i = bl * 32 + __ffs(mk) - 1;
        tc_rare_update(st, i, eval_line<J>(coef_line + (int64_t)i * J, u), c);
      }
      if (two)
        for (unsigned mk = mh; mk; mk &= mk - 1u) {
          const int i = bh * 32 + __ffs(mk) - 1;
          tc_rare_update(st, i, eval_line<J>(coef_line + (int64_t)i * J, u), c);
        }
      // a third block as close (or an overflowing candidate list, or logits
      // beyond the fp32 range): exact re-scan in the tail
      bool found = st.cnt > 0 && !(st.flags & 2) && !(m3b <= m1 + wnd) && bmax <= 3e38f;
      double m2x = st.m2;  // exact runner-up among the candidates (+inf: a single candidate)
      st.m2 = fmin(st.m2, (double)(two ? m3b : m2b) - (double)delta);  // out-of-block runner-up bound
      if (!found && bmax <= 3e38f) {
        // more than two blocks (or more than two columns) within the window -- e.g. every
        // pixel at theta = 0, the default start of a fit: decide here with an exact fp64
        // scan of the line's coefficient table (J FMAs per grain; all lanes of a warp read
        // the same rows) instead of queueing the pixel for the tail's K-term re-scan
        double em = CUDART_INF, em2 = CUDART_INF;
        for (int i = 0; i < N; ++i) {
          const double h = eval_line<J>(coef_line + (int64_t)i * J, u);
          em2 = fmin(em2, fmax(em, h));
          em = fmin(em, h);
        }
        const double thr = em + c * kTieRtol * (1.0 + fabs(em / c));
        int best = 0;
        for (int i = 0; i < N; ++i)
          if (eval_line<J>(coef_line + (int64_t)i * J, u) <= thr) {
            best = i;
            break;
          }
        st.m = em;
        st.m2 = m2x = em2;
        st.b0 = best;
        st.cnt = 1;
        found = true;
      }
      if constexpr (ASSIGN) {
        // (without candidates the tail's re-scan only needs an upper bound of the min)
        const double m = st.cnt > 0 ? st.m : (double)m1 + (double)delta;
        g.pix_m[p] = m / c;
        // exact when the runner-up is a candidate, else its fp32 logit (error <= delta)
        if (g.margin_out) g.margin_out[p] = (float)(fmax(fmin(m2x, (double)gm2) - m, 0.0) / c);
        if (!found) {
          const int slot = atomicAdd(g.fix_count, 1);
          g.fix_list[slot] = (int)p;
        } else {
          g.labels_out[p] = st.b0 + 1;
          correct += (st.b0 == lab) ? 1 : 0;
          amb += ((st.m2 - st.m) <= c * g.tau_amb * (1.0 + fabs(st.m / c))) ? 1 : 0;
        }
      } else {
        const double hG = eval_line<J>(coef_line + (int64_t)lab * J, u);
        const double refd = (double)ref;
        const double aG = hG - refd;
        const double eG = exp2(-aG);
        const double sxd = (double)sx - (double)sxc;
        const double sum = sxd + eG;
        const double l2s = log2(sum);
        const double l = (-aG - l2s) * 0.69314718055994530942;  // log p_G: objective.py:103-106
        ell += l;
        if (!isfinite(l) || !(bmax <= 3e38f)) nonfinite = 1;
        if (g.tc_rec) {  // pass-2 record: p_i/2 * 2^13 = 2^(w13 + wl13 - h~''_i)
          const double w13 = refd - 1.0 - l2s + 13.0;
          const float wh = (float)w13;
          float* rec = g.tc_rec + (line * (g.pside / kTcPixTile) + (col >> 6)) * (4 * kTcPixTile) + (col & 63);
          rec[0] = wh;
          rec[kTcPixTile] = (float)(w13 - (double)wh);
          rec[2 * kTcPixTile] = (float)(-4096.0 * sxd / sum);  // -(1 - p_G)/2 * 2^13
          reinterpret_cast<int*>(rec)[3 * kTcPixTile] = lab;
        }
        const double m = st.cnt > 0 ? st.m : hG;
        g.pix_m[p] = m / c;
        e0 += (hG - m) / c;  // objective.py:119
        if (!found) {
          const int slot = atomicAdd(g.fix_count, 1);
          g.fix_list[slot] = (int)p;
        } else {
          correct += (st.b0 == lab) ? 1 : 0;
          amb += ((st.m2 - st.m) <= c * g.tau_amb * (1.0 + fabs(st.m / c))) ? 1 : 0;
        }
      }
    }
    // per-CTA partials: warp shuffle tree, then warps in fixed order
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ell += __shfl_xor_sync(0xffffffffu, ell, off);
      e0 += __shfl_xor_sync(0xffffffffu, e0, off);
      correct += __shfl_xor_sync(0xffffffffu, correct, off);
      amb += __shfl_xor_sync(0xffffffffu, amb, off);
      nonfinite += __shfl_xor_sync(0xffffffffu, nonfinite, off);
    }
    if (lane == 0) {
      red_d[warp][0] = ell;
      red_d[warp][1] = e0;
      red_i[warp][0] = correct;
      red_i[warp][1] = amb;
      red_i[warp][2] = nonfinite;
    }
  }
  tc_fence_before();
  __syncthreads();
  // PDL: pass 2 is scheduled once every pass-1 CTA is past its main loop
  griddep_launch_dependents();
  if (tid == 0) {
    double s_ell = 0.0, s_e0 = 0.0;
    long long s_cor = 0, s_amb = 0, s_nf = 0;
    for (int w = 0; w < kSwEpiWarps; ++w) {
      s_ell += red_d[w][0];
      s_e0 += red_d[w][1];
      s_cor += red_i[w][0];
      s_amb += red_i[w][1];
      s_nf += red_i[w][2];
    }
    const int64_t b = g.part_off + blockIdx.x;  // partial slot of this CTA
    g.part_d[2 * b + 0] = s_ell;
    g.part_d[2 * b + 1] = s_e0;
    g.part_i[4 * b + 0] = s_cor;
    g.part_i[4 * b + 1] = s_amb;
    g.part_i[4 * b + 2] = s_nf;
    g.part_i[4 * b + 3] = 0;
  }
  if (warp == W_MMA) tmem_dealloc(tmem, 512);
}

}  // namespace pgx
