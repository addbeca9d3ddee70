// pgx_tc_pass1.cuh — PGX_PREC_TC pass 1: the logit contraction h'' = L(x_fast)
// B''(line) (objective.py:99) on the 5th-generation tensor cores and ONE
// streaming sweep over the grains per pixel on the CUDA cores: running min,
// online log-sum-exp (objective.py:102-106) and the arg-min bookkeeping of
// geometry.py:201-210.
//
// Persistent, warp-specialised, kT1CtasPerSm CTAs per SM sharing TMEM:
//   epilogue warps: slot s = warp / 4 is one tile of 128 pixels of a
//               line, lane quarter warp % 4; thread = TMEM lane = pixel;
//   warp 16     producer: bulk async copies of the per-line coefficient
//               images (pgx_tc_coeffs.cuh) into a 3-stage ring, and one lane
//               issuing tcgen05.mma (M = 128 pixels, N = 64 grains, K = 16 *
//               tc_ksteps(J), fp16 3-product split, fp32 accumulate) into a
//               double-buffered accumulator per slot, committed to mbarriers.
// A work item is 4 consecutive tiles (one line when the side has >= 4 tiles,
// else one tile per line — each slot then has its own coefficient image);
// items are strided over the CTAs in a fixed order (deterministic partials).
//
// Epilogue, per 32-column block of one pixel (h~'' = S * inv):
//   mb = block min (FMNMX3); the three best block minima and, for the best
//   two, the columns within 2 delta + tie band of their min (a bit mask) are
//   tracked.  The reference ref of s' = sum_{i != G} 2^(ref - h~''_i) moves
//   only when the min falls more than kT1Stale below it (s' is then rescaled
//   by 2^(ref_old - ref_new)): one FFMA + MUFU.EX2 + FADD per logit.
// Per pixel at the end: the label term in fp64, and the exact
//   fp64 tie-tolerant arg-min / min / runner-up over the masked columns of the
//   best block (and of the second one when its min is that close).  A third
//   block that close (real 3-way cross-block ties) queues the pixel for the
//   exact re-scan of the tail kernel.
#pragma once

#include "pgx_grid_common.cuh"
#include "pgx_tc_coeffs.cuh"
#include "pgx_tc_common.cuh"

namespace pgx {

constexpr int kTcThreadsTile = 128;              // pixels per tile (UMMA M, TMEM lanes)
constexpr int kT1Slots = 2;                      // pixel tiles per item
constexpr int kT1CtasPerSm = 2;                  // independent CTAs per SM (their sync phases interleave)
constexpr int kT1EpiWarps = 4 * kT1Slots;        // 16
constexpr int kT1Threads = 32 * kT1EpiWarps + 32;  // + producer warp
constexpr int kT1Cols = 32;                      // grains per MMA (UMMA N) = one block
constexpr int kT1Bufs = 4;                       // accumulator buffers per slot (TMEM)
constexpr int kT1Ring = 16;                      // coefficient image ring (images in flight)
constexpr float kT1Stale = 24.0f;                // ref may lag the min by this (log2 units)
constexpr int kT1SmemBudget = 100 * 1024;        // per CTA (kT1CtasPerSm share an SM)

// exact per-pixel state for near-minimal logits
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

template <int J>
struct TcP1Smem {
  static constexpr int KS = tc_ksteps(J);
  static constexpr int A_SLOT = KS * kTcThreadsTile * 32;  // one 128-row pixel operand
  static constexpr int IMG = tc_img_bytes<J>();
  static constexpr int A_OFF = 0;
  static constexpr int IMG_OFF = A_OFF + kT1Slots * A_SLOT;
  static constexpr int RING = (kT1SmemBudget - IMG_OFF) / IMG < kT1Ring ? (kT1SmemBudget - IMG_OFF) / IMG : kT1Ring;
  static constexpr int TOTAL = IMG_OFF + RING * IMG;
};

// named barrier of the 4 warps (128 threads) of one slot
__device__ __forceinline__ void slot_sync(int s) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + s) : "memory");
}

template <int DIM, int D>
__global__ void __launch_bounds__(kT1Threads, kT1CtasPerSm) k_tc_pass1(GridParams g) {
  constexpr int J = D + 1;
  using L = TcP1Smem<J>;
  constexpr int KS = L::KS;
  constexpr int QB = kTcCoefChunk / kT1Cols;  // blocks per coefficient image
  constexpr uint32_t IDESC = umma_idesc_f16(128, kT1Cols);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_full[kT1Slots][kT1Bufs];  // MMA of a slot's buffer complete
  __shared__ uint64_t bar_img[kT1Ring], bar_imgfree[kT1Ring];
  __shared__ unsigned tmem_base;
  __shared__ double red_d[kT1EpiWarps][2];
  __shared__ long long red_i[kT1EpiWarps][3];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = g.N;
  const double c = g.c;
  const int tpl = g.side / kTcThreadsTile;  // tiles per line
  // this launch's tiles [tbase, ntiles) (a line range of the evaluation)
  const int64_t tbase = g.tile_lo, ntiles = g.tile_hi;
  const int64_t nitems = (ntiles - tbase + kT1Slots - 1) / kT1Slots;
  const int nimg = (N + kTcCoefChunk - 1) / kTcCoefChunk;
  const int nblk = (N + kT1Cols - 1) / kT1Cols;

  constexpr unsigned kCols = kT1Slots * kT1Bufs * kT1Cols;  // TMEM columns of this CTA
  if (warp == kT1EpiWarps) tmem_alloc(&tmem_base, kCols);
  if (tid == 32 * kT1EpiWarps) {
    for (int s = 0; s < kT1Slots; ++s)
      for (int b = 0; b < kT1Bufs; ++b) mbar_init(&bar_full[s][b], 1);
    for (int b = 0; b < L::RING; ++b) {
      mbar_init(&bar_img[b], 1);
      mbar_init(&bar_imgfree[b], kT1Slots);  // every slot leader releases every image
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();  // PDL: the set-up above overlaps the predecessor (k_tc_coeffs)
  const unsigned tmem = tmem_base;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);

  // the images of a chunk: one per distinct line among the item's tiles;
  // js[s] = index of slot s's image, returns the count
  auto distinct = [&](int64_t it, int (&js)[kT1Slots]) {
    const int64_t t0 = tbase + it * kT1Slots;
    int n = 0;
    for (int s = 0; s < kT1Slots; ++s) {
      if (s > 0 && t0 + s < ntiles && (t0 + s) / tpl == (t0 + s - 1) / tpl)
        js[s] = js[s - 1];
      else
        js[s] = t0 + s < ntiles ? n++ : 0;
    }
    return n;
  };

  if (warp == kT1EpiWarps) {
    // ============================ loader warp: every image of every item of
    // this CTA, in consumption order, into a RING-deep ring; a ring slot is
    // refilled once all four slot leaders released its previous image
    const bool leader = lane == 0;
    int gl = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      int js[kT1Slots];
      const int nl = distinct(it, js);
      for (int ci = 0; ci < nimg; ++ci)
        for (int j = 0; j < nl; ++j, ++gl) {
          const int slot = gl % L::RING;
          mbar_wait_sleep(&bar_imgfree[slot], (unsigned)((gl / L::RING) & 1) ^ 1u);  // sleeps: no issue slots taken from the epilogue
          if (leader) {
            int s = 0;
            while (js[s] != j) ++s;  // first tile slot of distinct line j
            const int64_t line = (tbase + it * kT1Slots + s) / tpl;
            mbar_arrive_expect_tx(&bar_img[slot], L::IMG);
            bulk_g2s(smem + L::IMG_OFF + slot * L::IMG,
                     g.tc_img + (line * g.tc_nchunks + ci) * (int64_t)L::IMG, L::IMG, &bar_img[slot]);
          }
          __syncwarp();
        }
    }
  } else {
    // ============================ epilogue warps: thread = pixel of slot s;
    // the slot's 4 warps meet at a named barrier after every TMEM load and the
    // slot leader (lane 0 of warp 4s) issues the MMA that refills the buffer
    const int s = warp >> 2, q = warp & 3;
    const bool leader = q == 0 && lane == 0;
    const unsigned lane_off = (unsigned)(32 * q) << 16;
    const int prow = 32 * q + lane;  // row of the slot's 128-pixel tile
    const unsigned t_slot = tmem + lane_off + (unsigned)(s * kT1Bufs * kT1Cols);
    const unsigned a_full = (unsigned)__cvta_generic_to_shared(&bar_full[s][0]);
    const unsigned a_slot = sbase + L::A_OFF + (unsigned)(s * KS * (kTcThreadsTile * 32));
    double ell = 0.0, e0 = 0.0;
    long long correct = 0, amb = 0, nonfinite = 0;
    int rc = 0;  // rounds (blocks) of this slot so far: buffer rc % kT1Bufs, phase (rc / kT1Bufs) & 1
    int gc = 0;  // images released so far (leader only; all slots walk the same image sequence)
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      int js[kT1Slots];
      const int nl = distinct(it, js);
      const int64_t tile = tbase + it * kT1Slots + s;
      const bool active = tile < ntiles;
      const int64_t line = active ? tile / tpl : 0;
      const int col = (int)(tile % tpl) * kTcThreadsTile + prow;
      if (active) {  // pixel operand row: A'[p][k] = 2^10 L_j(x_fast), k = b J + j, blocks [hi, hi, lo]
        double u[J];
        axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
        __half hi[J], lo[J];
#pragma unroll
        for (int j = 0; j < J; ++j) split_f16(u[j] * 1024.0, hi[j], lo[j]);
        unsigned char* A_s = smem + L::A_OFF + s * L::A_SLOT;
#pragma unroll
        for (int k = 0; k < 16 * KS; ++k) {
          const int b = k / J, j = k % J;
          const __half val = k < 3 * J ? (b < 2 ? hi[j] : lo[j]) : __float2half(0.0f);
          *reinterpret_cast<__half*>(A_s + (k / 16) * (kTcThreadsTile * 32) + slab_off(prow, k % 16)) = val;
        }
        fence_proxy_async_smem();
      }
      slot_sync(s);
      // leader: MMA of block kb of this item into buffer (rc0 + kb) % kT1Bufs;
      // waits for the chunk's images at its first block, releases them after its last
      const int rc0 = rc;
      auto issue = [&](int kb) {
        const int ci = kb / QB, qb = kb % QB;
        if (qb == 0)
          for (int j = 0; j < nl; ++j)
            mbar_wait(&bar_img[(gc + j) % L::RING], (unsigned)(((gc + j) / L::RING) & 1));
        tc_fence_after();
        const unsigned buf = (unsigned)((rc0 + kb) % kT1Bufs);
        const unsigned bimg = sbase + L::IMG_OFF + (unsigned)(((gc + js[s]) % L::RING) * L::IMG) +
                              (unsigned)(qb * (kT1Cols / 8) * 256);
#pragma unroll
        for (int k = 0; k < KS; ++k)
          umma_f16_ss(tmem + (unsigned)((s * kT1Bufs + buf) * kT1Cols),
                      umma_desc(a_slot + k * (kTcThreadsTile * 32)), umma_desc(bimg + k * (kTcCoefChunk * 32)),
                      IDESC, k > 0);
        umma_commit(&bar_full[s][buf]);
        if (qb == QB - 1 || kb == nblk - 1) {
          for (int j = 0; j < nl; ++j) umma_commit(&bar_imgfree[(gc + j) % L::RING]);
          gc += nl;
        }
      };
      if (!active) {  // empty slot of the last item: release the images, nothing else
        if (leader)
          for (int ci = 0; ci < nimg; ++ci) {
            for (int j = 0; j < nl; ++j) {
              mbar_wait(&bar_img[(gc + j) % L::RING], (unsigned)(((gc + j) / L::RING) & 1));
              mbar_arrive(&bar_imgfree[(gc + j) % L::RING]);
            }
            gc += nl;
          }
        continue;
      }
      if (leader)
        for (int kb = 0; kb < min(kT1Bufs, nblk); ++kb) issue(kb);
      const int64_t p = line * g.side + col;
      const int lab = g.labels[p];
      const double* coef_line = g.tc_coef + line * (int64_t)N * J;
      const int2* meta = g.tc_meta + line * g.tc_nchunks;
      float ref = CUDART_INF_F, m1 = CUDART_INF_F, m2b = CUDART_INF_F, m3b = CUDART_INF_F, bmax = 0.0f;
      int b1 = 0, b2 = 0;
      unsigned mask1 = 0u, mask2 = 0u;  // columns of blocks b1, b2 within the candidate window of their min
      float sx = 0.0f, sxc = 0.0f;  // Kahan-compensated sum of the block sums
      float inv = 0.0f, dblk = 0.0f;
      // candidate window terms in fp32 (a window, widened by 0.1%): no fp64
      // division on the per-block path
      const float bandf = (float)(c * fmax(kTieRtol, g.tau_amb)), inv_cf = (float)(1.0 / c);
      float rinv = 0.0f;  // 1 / inv (exact: powers of two)
      // one 32-grain block: wait, load, refill, min bookkeeping, exponentials
      auto chunk_meta = [&](int ci) {  // scale and error bound of 128-grain chunk ci
        const int2 mt = __ldg(meta + ci);
        rinv = __int_as_float((127 + (mt.x + 10)) << 23);
        inv = __int_as_float((127 - (mt.x + 10)) << 23);  // 2^-(sB + 10): S * inv = h~''
        const float bn = __int_as_float(mt.y);
        bmax = fmaxf(bmax, bn);
        dblk = 2.0f * (4.7683716e-07f + 3 * J * 5.9604645e-08f) * bn + 1e-30f;
      };
      auto block = [&](int kb, int cn) {
        const unsigned buf = (unsigned)(rc % kT1Bufs);
        mbar_wait_addr(a_full + 8u * buf, (unsigned)((rc / kT1Bufs) & 1));
        tc_fence_after();
        uint32_t r0[32];
        tmem_ld32_nowait(t_slot + buf * kT1Cols, r0);
        tmem_ld_wait();
        tmem_regs_ready(r0);
        // the slot's warps meet every second block: buffers of blocks kb - 1 and
        // kb are then free for the refills kb + 3 and kb + 4 (issued 2 and 3
        // blocks before their use); measured c2 -2%, c4/c5 unchanged vs every block
        if (kb & 1) {
          tc_fence_before();
          slot_sync(s);
          if (leader) {
            if (kb + kT1Bufs - 1 < nblk) issue(kb + kT1Bufs - 1);
            if (kb + kT1Bufs < nblk) issue(kb + kT1Bufs);
          }
        }
        ++rc;
        float w[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) w[e] = (cn == 32 || e < cn) ? __uint_as_float(r0[e]) : CUDART_INF_F;
        // block min: FMNMX3 tree
        float t11[11];
#pragma unroll
        for (int e = 0; e < 10; ++e) t11[e] = fminf(w[3 * e], fminf(w[3 * e + 1], w[3 * e + 2]));
        t11[10] = fminf(w[30], w[31]);
        const float mb = fminf(fminf(fminf(t11[0], fminf(t11[1], t11[2])), fminf(t11[3], fminf(t11[4], t11[5]))),
                               fminf(fminf(t11[6], fminf(t11[7], t11[8])), fminf(t11[9], t11[10])));
        const float mbs = mb * inv;
        if (mbs < m3b) {  // top-3 blocks (rare after the first few)
          if (mbs < m2b) {
            // candidate columns of the block: within 2 delta + tie band of its min
            const float thr = (mbs + 2.0f * dblk + bandf * (1.0f + fabsf(mbs) * inv_cf) * 1.001f) * rinv;
            // bit e of nm = sign of thr - w_e (exact: no FTZ, gradual underflow), i.e.
            // w_e > thr or w_e = +inf padding; two instructions per column
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
          if (mbs < ref - kT1Stale) {  // (also the first block: ref = +inf)
            const float nref = mbs - 1.0f;
            const double f = exp2((double)nref - (double)ref);
            sx = (float)((double)sx * f);
            sxc = (float)((double)sxc * f);
            ref = nref;
          }
        }
        const float nr = -ref;
        const int labc = lab - kb * kT1Cols;
        float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // 4 independent FADD chains
        // padding columns (e >= cn) hold +inf: their terms are exactly 0, so only
        // a block holding some lane's label column needs the masked loop
        if (!__any_sync(0xffffffffu, (unsigned)labc < 32u)) {
#pragma unroll
          for (int e = 0; e < 32; ++e) s4[e & 3] += ex2_approx(-fmaf(w[e], inv, nr));
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float x = ex2_approx(-fmaf(w[e], inv, nr));
            s4[e & 3] += e != labc ? x : 0.0f;
          }
        }
        const float y = ((s4[0] + s4[1]) + (s4[2] + s4[3])) - sxc;  // Kahan step
        const float t = sx + y;
        sxc = (t - sx) - y;
        sx = t;
      };
      const int nfull = N / kT1Cols;  // full blocks; a partial one follows if N % 32
      // chunk by chunk (the chunk's scale read once), block by block
#pragma unroll 1
      for (int kb0 = 0; kb0 < nfull; kb0 += QB) {
        chunk_meta(kb0 / QB);
        const int kb1 = min(nfull, kb0 + QB);
#pragma unroll 1
        for (int kb = kb0; kb < kb1; ++kb) block(kb, 32);
      }
      if (nfull < nblk) {
        if (nfull % QB == 0) chunk_meta(nfull / QB);
        block(nfull, N - nfull * kT1Cols);
      }

      // ------------------------------------------------ per-pixel finish
      // |h~'' - h''| <= delta: fp16 split (2^-21 relative per operand pair) plus
      // the fp32 accumulation of 3J products; generous factor 2
      const float delta = 2.0f * (4.7683716e-07f + 3 * J * 5.9604645e-08f) * bmax + 1e-30f;
      const double band = c * fmax(kTieRtol, g.tau_amb) * (1.0 + fabs((double)m1 / c));
      const float wnd = 2.0f * delta + (float)band * 1.001f + 1e-30f;
      double u[J];
      axis_table<D>(axis_coord(col, g.M), g.legendre != 0, u);
      const double hG = eval_line<J>(coef_line + (int64_t)lab * J, u);
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
        const int i = bl * kT1Cols + __ffs(mk) - 1;
        tc_rare_update(st, i, eval_line<J>(coef_line + (int64_t)i * J, u), c);
      }
      if (two)
        for (unsigned mk = mh; mk; mk &= mk - 1u) {
          const int i = bh * kT1Cols + __ffs(mk) - 1;
          tc_rare_update(st, i, eval_line<J>(coef_line + (int64_t)i * J, u), c);
        }
      // a third block as close (or an overflowing candidate list): exact re-scan in the tail
      bool found = st.cnt > 0 && !(st.flags & 2) && !(m3b <= m1 + wnd);
      st.m2 = fmin(st.m2, (double)(two ? m3b : m2b) - (double)delta);  // out-of-block runner-up bound
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
        float* rec = g.tc_rec + (line * (g.side / kTcPixTile) + (col >> 6)) * (4 * kTcPixTile) + (col & 63);
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
  // PDL: pass 2 is scheduled once every pass-1 CTA is past its main loop (it
  // sets up, then waits for this grid to complete)
  griddep_launch_dependents();
  if (tid == 0) {
    double s_ell = 0.0, s_e0 = 0.0;
    long long s_cor = 0, s_amb = 0, s_nf = 0;
    for (int w = 0; w < kT1EpiWarps; ++w) {
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
  if (warp == kT1EpiWarps) tmem_dealloc(tmem, kCols);
}

}  // namespace pgx
