// pgx_grid.cuh — regular-grid (separable) fp64 path: plan + dispatch.
// Kernels: pgx_grid_pass1.cuh (min / arg-min / log-sum-exp), pgx_grid_pass2.cuh
// (gradient contraction); shared pieces in pgx_grid_common.cuh.
#pragma once

#include <algorithm>
#include <cstdlib>

#include "pgx_grid_common.cuh"
#include "pgx_grid_pass1.cuh"
#include "pgx_grid_pass2.cuh"
#include "pgx_tc_shared.cuh"

namespace pgx {

struct GridPlan {
  bool enabled = false;
  bool tc = false;  // PGX_PREC_TC: tensor-core pass 1
  int dim = 2, D = 1;
  int pside = 0;    // tensor-core tiles: side rounded up to a multiple of 128
  int R = 1, segs = 1, lines = 0, blocks1 = 0;
  int tc_blocks = 0;
  int tc2_gtiles = 0, tc2_lps = 1, tc2_splits = 0;  // tensor-core pass 2 (0 = CUDA-core pass 2)
  int64_t tc2_ips = 1;                               // its items per CTA row
  int part_splits = 0;                             // allocated split slots of part_g
  int tc_nchunks = 0;                              // 128-grain chunks (pgx_tc_coeffs.cuh)
  void* d_tc = nullptr;                            // coef | img | meta
  double* tc_coef = nullptr;
  unsigned char* tc_img = nullptr;
  int2* tc_meta = nullptr;
  void* d_tc_pix = nullptr;                        // pass-2 pixel operand tiles (once per problem)
  unsigned char* tc_pix = nullptr;
  bool tc_pix_ready = false;
  float* tc_rec = nullptr;                         // pass-2 pixel records (aliases pix_w | pix_q)
  double* tc_lc = nullptr;                         // [lines][K] line factors
  int GT = 128, gtiles = 1, splits = 1, lines_per_split = 1;
  int splits_out = 1;
  double* part_out = nullptr;
  void* d_part = nullptr;  // single allocation: part_g | pix_w, pix_q (fp64) or tc_rec (TC)
  double* pix_w = nullptr;
  float* pix_q = nullptr;
  int smem2 = 0;
};

// pass-2 line splits over `lines` lines: minimise waves x (lines per CTA + 1)
inline void tc2_splits_for(int lines, int gtiles, int64_t slots, int cap, int& lps_out, int& splits_out) {
  int64_t best = -1;
  lps_out = lines;
  splits_out = 1;
  for (int sp = 1; sp <= std::min(lines, cap); ++sp) {
    const int lps = (lines + sp - 1) / sp;
    const int spr = (lines + lps - 1) / lps;
    if (spr != sp) continue;
    const int64_t waves = ((int64_t)gtiles * spr + slots - 1) / slots;
    const int64_t cost = waves * (lps + 1);  // + ~1 line of per-CTA pipeline fill
    if (best < 0 || cost < best) {
      best = cost;
      lps_out = lps;
      splits_out = spr;
    }
  }
}

// pass-2 item splits (items = (line, 64-pixel tile) pairs, a CTA may start
// and end mid-line): minimise waves x (items per CTA + one line of pipeline fill)
inline void tc2_item_splits_for(int64_t items, int tpl, int gtiles, int64_t slots, int cap,
                                int64_t& ips_out, int& splits_out) {
  int64_t best = -1;
  ips_out = items;
  splits_out = 1;
  for (int sp = 1; sp <= cap && sp <= items; ++sp) {
    const int64_t ips = (items + sp - 1) / sp;
    const int spr = (int)((items + ips - 1) / ips);
    if (spr != sp) continue;
    const int64_t waves = ((int64_t)gtiles * spr + slots - 1) / slots;
    const int64_t cost = waves * (ips + tpl);
    if (best < 0 || cost < best) {
      best = cost;
      ips_out = ips;
      splits_out = spr;
    }
  }
}

inline void grid_plan_shape(GridPlan& gp, const pgx_desc* d, int sms) {
  gp.enabled = false;
  if (d->resolution <= 0 || d->precision == PGX_PREC_EXACT) return;
  const int side = 2 * d->resolution;
  // the fp64 separable kernels need side % 128 == 0; the tensor-core kernels
  // pad any side >= 64 to the next multiple of 128 (masked pixels); smaller
  // grids use the general path
  const bool tc_ok = d->precision == PGX_PREC_TC && side >= 64 && (d->n_grains + 127) / 128 <= 65535;
  if (side % 128 != 0 && !tc_ok) return;
  if (d->dim == 2 && d->degree > 8) return;
  if (d->dim == 3 && d->degree > 4) return;
  gp.enabled = true;
  gp.dim = d->dim;
  gp.D = d->degree;
  gp.lines = (int)(d->n_points / side);
  gp.pside = (side + 127) / 128 * 128;
  // pixels per thread: register blocking of the shared B'' loads, bounded by
  // the register file and by the wave count (>= ~6 CTAs per SM when possible)
  const int rmax = d->degree <= 3 ? 4 : (d->degree <= 5 ? 2 : 1);
  int R = std::max(1, std::min(rmax, side / 128));
  while (R > 1 && (int64_t)gp.lines * (side / (128 * R)) < 6 * sms) R /= 2;
  gp.R = R;
  gp.segs = std::max(1, side / (128 * gp.R));
  gp.blocks1 = gp.lines * gp.segs;
  // (k_tc_coeffs puts the 128-grain chunks on gridDim.y)
  gp.tc = tc_ok;
  if (gp.tc) {
    // tensor-core pass 1 (k_tc_sweep): persistent, one CTA per SM, items of 4 tiles
    const int64_t ntiles = (int64_t)gp.lines * (gp.pside / kTcThreadsTile);
    gp.tc_blocks = (int)std::min<int64_t>((ntiles + 3) / 4, (int64_t)sms);
    gp.blocks1 = gp.tc_blocks;
  }
  const int N = d->n_grains;
  // grains per pass-2 CTA: least padding, larger tile on ties
  gp.GT = 128;
  for (int gt : {64, 32})
    if ((N + gt - 1) / gt * gt < (N + gp.GT - 1) / gp.GT * gp.GT) gp.GT = gt;
  gp.gtiles = (N + gp.GT - 1) / gp.GT;
  const int K = feature_count(d->dim, d->degree);
  // line splits: >= 8 CTAs per SM, up to 32 (small problems are latency
  // bound: more, shorter CTAs fill the SMs) while the per-split gradient
  // partials the tail reduces stay within 32 MB
  {
    const int s8 = std::max(1, std::min(gp.lines, (8 * sms + gp.gtiles - 1) / gp.gtiles));
    const int s32 = std::max(1, std::min(gp.lines, (32 * sms + gp.gtiles - 1) / gp.gtiles));
    const int cap = (int)std::max<int64_t>(1, (32LL << 20) / ((int64_t)K * N * 8));
    gp.splits = std::max(s8, std::min(s32, cap));
  }
  gp.lines_per_split = (gp.lines + gp.splits - 1) / gp.splits;
  gp.splits = (gp.lines + gp.lines_per_split - 1) / gp.lines_per_split;
  gp.splits_out = gp.splits;
  gp.smem2 = K * kG2Threads * 8;
  // (>= 2 tiles per line: two consecutive one-item R groups would reuse an
  // accumulator before its flush)
  if (gp.tc) {  // (pside >= 128: at least two 64-pixel tiles per line)
    // tensor-core pass 2: 128-grain tiles x line ranges, 2 CTAs per SM; the
    // split count minimises waves x lines-per-CTA (ties: fewer splits, so the
    // tail reduces less)
    gp.tc2_gtiles = (N + kTc2Grains - 1) / kTc2Grains;
    // line-aligned CTA ranges unless item-granular ones are >= 5% cheaper
    // (c2: 28 items per CTA instead of 4 lines = 32; the mid-line kernel
    // variant costs registers, measured 3% slower per item at c5)
    const int tpl2 = gp.pside / kTc2Px;
    tc2_splits_for(gp.lines, gp.tc2_gtiles, 2LL * sms, 8 * sms, gp.tc2_lps, gp.tc2_splits);
    int64_t ips = 0;
    int isp = 0;
    tc2_item_splits_for((int64_t)gp.lines * tpl2, tpl2, gp.tc2_gtiles, 2LL * sms, 8 * sms, ips, isp);
    const auto waves = [&](int sp) { return ((int64_t)gp.tc2_gtiles * sp + 2LL * sms - 1) / (2LL * sms); };
    const int64_t cost_line = waves(gp.tc2_splits) * ((int64_t)gp.tc2_lps * tpl2 + tpl2);
    const int64_t cost_item = waves(isp) * (ips + tpl2);
    gp.tc2_ips = (int64_t)gp.tc2_lps * tpl2;
    if (20 * cost_item < 19 * cost_line) {
      gp.tc2_ips = ips;
      gp.tc2_splits = isp;
    }
    gp.splits_out = gp.tc2_splits;
    gp.part_splits = std::max(gp.splits, gp.splits_out);
  }
}

// byte sizes of the plan's allocations (one place: the estimate reported with
// PGX_ERR_RESOURCE is exactly what grid_plan_create asks for)
struct GridBytes {
  size_t part = 0;    // gradient partial slots (doubles)
  size_t main = 0;    // part_g | per-pixel scratch (16 B per pixel)
  size_t ncoef = 0, nimg = 0, nmeta = 0, nlc = 0;
  size_t tc = 0;      // coef | img | meta | line factors (PGX_PREC_TC)
  size_t pix = 0;     // pass-2 pixel operand tiles (PGX_PREC_TC)
  size_t total() const { return main + tc + pix; }
};

inline GridBytes grid_bytes(const GridPlan& gp, const pgx_desc* d) {
  GridBytes b;
  if (!gp.enabled) return b;
  const int K = feature_count(d->dim, d->degree);
  b.part = (size_t)std::max(gp.splits, gp.part_splits) * K * d->n_grains;
  // per-pixel scratch, 16 B per pixel (tensor-core problems: per padded pixel, the pass-2 records)
  const size_t npix = gp.tc ? (size_t)gp.lines * gp.pside : (size_t)d->n_points;
  b.main = b.part * 8 + npix * 16 + 256;
  if (gp.tc) {
    const int J = d->degree + 1;
    const size_t nchunks = (d->n_grains + kTcCoefChunk - 1) / kTcCoefChunk;
    b.ncoef = (size_t)gp.lines * d->n_grains * J;
    b.nimg = (size_t)gp.lines * nchunks * tc_ksteps(J) * kTcCoefChunk * 32;
    b.nmeta = (size_t)gp.lines * nchunks;
    b.nlc = (size_t)gp.lines * K;
    b.tc = b.ncoef * 8 + b.nimg + b.nmeta * 8 + b.nlc * 8 + 256;
    if (gp.tc2_splits > 0)
      b.pix = (size_t)(gp.pside / kTcPixTile) *
              (tc_ksteps(J) * kTcPixTile * 32 + 2 * (kTcPixTile / 16) * 16 * 32);
  }
  return b;
}

inline size_t grid_workspace_bytes(const pgx_desc* d, int sms) {
  GridPlan gp;
  grid_plan_shape(gp, d, sms);
  return grid_bytes(gp, d).total();
}

inline cudaError_t grid_plan_create(GridPlan& gp, const pgx_desc* d, int sms, size_t& bytes) {
  grid_plan_shape(gp, d, sms);
  if (!gp.enabled) return cudaSuccess;
  const GridBytes b = grid_bytes(gp, d);
  cudaError_t e = cudaMalloc(&gp.d_part, b.main);
  if (e != cudaSuccess) return e;
  bytes += b.main;
  gp.part_out = static_cast<double*>(gp.d_part);
  gp.pix_w = gp.part_out + b.part;
  gp.pix_q = reinterpret_cast<float*>(gp.pix_w + (gp.tc ? (size_t)gp.lines * gp.pside : (size_t)d->n_points));
  if (gp.tc) {
    gp.tc_nchunks = (d->n_grains + kTcCoefChunk - 1) / kTcCoefChunk;
    e = cudaMalloc(&gp.d_tc, b.tc);
    if (e != cudaSuccess) return e;
    bytes += b.tc;
    gp.tc_coef = static_cast<double*>(gp.d_tc);
    gp.tc_img = reinterpret_cast<unsigned char*>(gp.tc_coef + b.ncoef);
    gp.tc_meta = reinterpret_cast<int2*>(gp.tc_img + b.nimg);
    gp.tc_lc = reinterpret_cast<double*>(gp.tc_meta + b.nmeta);
    if (gp.tc2_splits > 0) {
      gp.tc_rec = reinterpret_cast<float*>(gp.pix_w);  // 16 bytes per pixel
      e = cudaMalloc(&gp.d_tc_pix, b.pix);
      if (e != cudaSuccess) return e;
      bytes += b.pix;
      gp.tc_pix = static_cast<unsigned char*>(gp.d_tc_pix);
      gp.tc_pix_ready = false;
    }
  }
  return cudaSuccess;
}

inline void grid_plan_destroy(GridPlan& gp) { (void)gp; }

}  // namespace pgx

#include "pgx_launch.cuh"
