// pgx_api.cu — the C ABI (include/pgx.h): problem lifetime, workspace,
// dispatch onto the sm_100a kernels, host<->device staging, error mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pgx.h"
#include "pgx_common.cuh"
#include "pgx_general.cuh"
#include "pgx_grid.cuh"
#include "pgx_grid_eval.cuh"
#include "pgx_launch.cuh"

using namespace pgx;

namespace {

thread_local std::string g_last_error;

pgx_status fail(pgx_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define PGX_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(PGX_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

#define PGX_LAUNCH_CHECK() PGX_CUDA(cudaGetLastError())

int max_degree_for(int dim) { return dim == 2 ? kMaxDegree2 : kMaxDegree3; }

}  // namespace

struct pgx_problem {
  int dim = 2, kind = PGX_BASIS_LEGENDRE, degree = 1, K = 3, N = 2, M = 0, prec = PGX_PREC_FP64;
  int device = 0;
  int sms = 148;
  int64_t P = 0;
  bool has_labels = false;
  cudaStream_t stream = nullptr;
  int last_launches = 0;

  // device buffers owned by the problem
  double* d_points = nullptr;
  double* d_design = nullptr;     // explicit K x P design matrix (pgx_desc.design)
  int32_t* d_labels = nullptr;
  double* d_theta = nullptr;      // K x N fp64 working copy
  void* d_theta_in = nullptr;     // host-theta staging (K x N x 8 bytes)
  double* d_pix_m = nullptr;
  double* d_pix_ls = nullptr;
  int* d_fix_list = nullptr;
  int* d_counters = nullptr;      // [0] fix_count, [1] nonfinite grad
  long long* d_fix_correct = nullptr;
  double* d_part_th2 = nullptr;   // tail: per-CTA lambda-norm partials
  double* d_part_d = nullptr;
  long long* d_part_i = nullptr;
  double* d_part_g = nullptr;
  double* d_grad = nullptr;       // host-mode staging
  pgx_stats* d_stats = nullptr;   // host-mode staging
  long long* d_labels_out = nullptr;
  float* d_margin_out = nullptr;
  unsigned long long* d_moments = nullptr;  // N x 6 label-moment sums + 1 flag word (2-D grids)
  // true between the first launch of a call and its tail launch: a call that
  // failed in between leaves the fix-up / ticket counters armed, and the next
  // call re-zeroes them first (normally the tail's last CTA re-arms them)
  bool counters_dirty = false;
  int blocks1 = 0;   // general pass-1 blocks
  int splits = 1;    // pass-2 point splits
  GridPlan grid;     // regular-grid fast path plan (grid.enabled)
  size_t bytes = 0;

  // kernel-level profiling: event pairs recorded on the stream around launches
  static constexpr int kProfMax = 32;
  bool profiling = false;
  cudaEvent_t prof_ev[2 * kProfMax] = {};
  const char* prof_name[kProfMax] = {};
  int prof_n = 0;
  void prof_reset() { prof_n = 0; }
  void prof_begin(const char* name) {
    if (!profiling || prof_n >= kProfMax) return;
    prof_name[prof_n] = name;
    cudaEventRecord(prof_ev[2 * prof_n], stream);
  }
  void prof_end() {
    if (!profiling || prof_n >= kProfMax) return;
    cudaEventRecord(prof_ev[2 * prof_n + 1], stream);
    ++prof_n;
  }

  template <typename T>
  cudaError_t alloc(T** p, size_t n) {
    bytes += n * sizeof(T);
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(1, n) * sizeof(T));
  }
  void release() {
    void* bufs[] = {d_points, d_design, d_labels, d_theta, d_theta_in, d_pix_m, d_pix_ls, d_fix_list,
                    d_counters, d_fix_correct, d_part_th2, d_part_d, d_part_i, d_part_g, d_grad, d_stats,
                    d_labels_out, d_margin_out, d_moments, grid.d_part, grid.d_tc, grid.d_tc_pix};
    for (void* b : bufs)
      if (b) cudaFree(b);
    grid_plan_destroy(grid);
    for (cudaEvent_t& e : prof_ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

int sm_count(int device) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n;
}

// ------------------------------------------------------------------ dispatch
// (launchers are defined and instantiated in the k_*.cu translation units)
#define PGX_DEG_SWITCH2(FN, ...)                 \
  switch (pb->degree) {                          \
    case 0: FN<2, 0>(__VA_ARGS__); break;        \
    case 1: FN<2, 1>(__VA_ARGS__); break;        \
    case 2: FN<2, 2>(__VA_ARGS__); break;        \
    case 3: FN<2, 3>(__VA_ARGS__); break;        \
    case 4: FN<2, 4>(__VA_ARGS__); break;        \
    case 5: FN<2, 5>(__VA_ARGS__); break;        \
    case 6: FN<2, 6>(__VA_ARGS__); break;        \
    case 7: FN<2, 7>(__VA_ARGS__); break;        \
    case 8: FN<2, 8>(__VA_ARGS__); break;        \
    case 9: FN<2, 9>(__VA_ARGS__); break;        \
    default: FN<2, 10>(__VA_ARGS__); break;      \
  }
#define PGX_DEG_SWITCH3(FN, ...)                 \
  switch (pb->degree) {                          \
    case 0: FN<3, 0>(__VA_ARGS__); break;        \
    case 1: FN<3, 1>(__VA_ARGS__); break;        \
    case 2: FN<3, 2>(__VA_ARGS__); break;        \
    case 3: FN<3, 3>(__VA_ARGS__); break;        \
    default: FN<3, 4>(__VA_ARGS__); break;       \
  }
#define PGX_DISPATCH(FN, ...)                                      \
  do {                                                             \
    if (pb->dim == 2) {                                            \
      PGX_DEG_SWITCH2(FN, __VA_ARGS__)                             \
    } else {                                                       \
      PGX_DEG_SWITCH3(FN, __VA_ARGS__)                             \
    }                                                              \
  } while (0)

EvalParams make_params(pgx_problem* pb, double eps) {
  EvalParams prm{};
  prm.P = pb->P;
  prm.N = pb->N;
  prm.M = pb->M;
  prm.legendre = pb->kind == PGX_BASIS_LEGENDRE;
  prm.pts = pb->d_points;
  prm.labels = pb->has_labels ? pb->d_labels : nullptr;
  prm.theta = pb->d_theta;
  prm.eps = eps;
  prm.inv_eps = 1.0 / eps;
  prm.tau_amb = 1e-10;
  prm.pix_m = pb->d_pix_m;
  prm.pix_ls = pb->d_pix_ls;
  prm.part_d = pb->d_part_d;
  prm.part_i = pb->d_part_i;
  prm.fix_count = pb->d_counters;
  prm.fix_list = pb->d_fix_list;
  prm.fix_correct = pb->d_fix_correct;
  prm.splits = pb->splits;
  prm.part_g = pb->d_part_g;
  return prm;
}

// Device alias of a pinned, mapped host pointer (nullptr for pageable memory).
constexpr size_t kZeroCopyMax = 256 * 1024;
void* host_mapped(void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// theta (host or device, f32 or f64) -> the fp64 pointer the kernels read.
// With `out32` (the tc grid path) an fp32 theta is not converted here: k_tc_coeffs
// reads it and writes the fp64 copy *out (one launch less per evaluation).
pgx_status stage_theta(pgx_problem* pb, const void* theta, uint32_t flags, const double** out,
                       int* launches, const float** out32 = nullptr) {
  const size_t KN = (size_t)pb->K * pb->N;
  const bool f32 = flags & PGX_THETA_F32;
  const bool dev = flags & PGX_DEVICE_PTRS;
  if (!theta) return fail(PGX_ERR_INVALID_ARGUMENT, "theta must not be NULL");
  if (dev && !f32) {
    *out = static_cast<const double*>(theta);
    return PGX_OK;
  }
  const void* src = theta;
  if (!dev) {
    PGX_CUDA(cudaMemcpyAsync(pb->d_theta_in, theta, KN * (f32 ? 4 : 8), cudaMemcpyHostToDevice,
                             pb->stream));
    src = pb->d_theta_in;
    if (!f32) {
      *out = static_cast<const double*>(pb->d_theta_in);
      return PGX_OK;
    }
  }
  if (out32) {
    *out32 = static_cast<const float*>(src);
    *out = pb->d_theta;
    return PGX_OK;
  }
  const int blocks = (int)std::min<size_t>((KN + 255) / 256, 1024);
  k_theta_to_f64<<<blocks, 256, 0, pb->stream>>>(src, 1, (int64_t)KN, pb->d_theta);
  PGX_LAUNCH_CHECK();
  ++*launches;
  *out = pb->d_theta;
  return PGX_OK;
}

pgx_status validate_desc(const pgx_desc* d) {
  if (!d) return fail(PGX_ERR_INVALID_ARGUMENT, "descriptor must not be NULL");
  if (d->design) {  // explicit design matrix: basis and grid fields are ignored
    if (d->design_k < 1 || d->design_k > kMaxK)
      return fail(PGX_ERR_INVALID_ARGUMENT, "design_k must lie in [1, %d], got %d", kMaxK, d->design_k);
    if (d->n_grains < 2) return fail(PGX_ERR_INVALID_ARGUMENT, "a grain map needs at least two grains");
    if (d->n_grains > (1 << 24)) return fail(PGX_ERR_INVALID_ARGUMENT, "n_grains %d too large", d->n_grains);
    if (d->n_points < 1 || d->n_points > ((int64_t)1 << 31) - 1)
      return fail(PGX_ERR_INVALID_ARGUMENT, "n_points out of range");
    return PGX_OK;
  }
  if (d->dim != 2 && d->dim != 3)
    return fail(PGX_ERR_INVALID_ARGUMENT, "dim must be 2 or 3, got %d", d->dim);
  if (d->basis_kind != PGX_BASIS_LEGENDRE && d->basis_kind != PGX_BASIS_MONOMIAL)
    return fail(PGX_ERR_INVALID_ARGUMENT, "unknown basis kind %d", d->basis_kind);
  if (d->degree < 0 || d->degree > max_degree_for(d->dim))
    return fail(PGX_ERR_INVALID_ARGUMENT, "degree %d unsupported for dim %d (max %d)", d->degree,
                d->dim, max_degree_for(d->dim));
  if (d->n_grains < 2)
    return fail(PGX_ERR_INVALID_ARGUMENT, "a grain map needs at least two grains");
  if (d->n_grains > (1 << 24))
    return fail(PGX_ERR_INVALID_ARGUMENT, "n_grains %d too large", d->n_grains);
  if (d->precision < PGX_PREC_EXACT || d->precision > PGX_PREC_TC)
    return fail(PGX_ERR_INVALID_ARGUMENT, "unknown precision mode %d", d->precision);
  if (d->resolution > 0) {
    int64_t side = 2 * (int64_t)d->resolution;
    int64_t expect = side * side * (d->dim == 3 ? side : 1);
    if (d->n_points != expect)
      return fail(PGX_ERR_INVALID_ARGUMENT, "regular grid with M=%d requires %lld points, got %lld",
                  d->resolution, (long long)expect, (long long)d->n_points);
  } else {
    if (d->n_points < 1) return fail(PGX_ERR_INVALID_ARGUMENT, "a grid needs at least one point");
    if (!d->points) return fail(PGX_ERR_INVALID_ARGUMENT, "unstructured grid needs points");
  }
  if (d->n_points > ((int64_t)1 << 31) - 1)
    return fail(PGX_ERR_INVALID_ARGUMENT, "n_points too large");
  return PGX_OK;
}

// pass-2 point splits of the general kernels: up to 4 CTAs per SM and grain
// tile, at least 128 points each (few grains leave most of a CTA's threads
// idle: many short CTAs fill the SMs instead; the tail reduces the splits in
// fixed order)
int general_splits(int64_t P, int tiles, int sms) {
  return std::max(1, std::min<int>(4 * sms / tiles, (int)std::min<int64_t>((P + 127) / 128, 1 << 20)));
}

size_t workspace_estimate(const pgx_desc* d, int sms) {
  const int64_t P = d->n_points;
  const int K = d->design ? d->design_k : feature_count(d->dim, d->degree);
  const int64_t KN = (int64_t)K * d->n_grains;
  const int64_t blocks1 = (P + kP1Threads - 1) / kP1Threads;
  const int tiles = (d->n_grains + kP2Threads - 1) / kP2Threads;
  const int splits = general_splits(P, tiles, sms);
  size_t b = 0;
  b += (d->resolution > 0 ? 0 : (size_t)P * d->dim * 8);
  b += (size_t)P * 4 + (size_t)KN * 8 * 3 + (size_t)P * 8 * 2 + (size_t)P * 4;
  b += (size_t)blocks1 * (16 + 32) + (size_t)splits * KN * 8;
  b += (size_t)P * 12;
  if (d->design)
    b += (size_t)P * K * 8;
  else
    b += grid_workspace_bytes(d, sms);
  return b;
}

}  // namespace

// counters a failed call may have left armed (see pgx_problem::counters_dirty)
static pgx_status rearm_counters(pgx_problem* pb) {
  if (!pb->counters_dirty) return PGX_OK;
  PGX_CUDA(cudaMemsetAsync(pb->d_counters, 0, 4 * sizeof(int), pb->stream));
  PGX_CUDA(cudaMemsetAsync(pb->d_fix_correct, 0, 2 * sizeof(long long), pb->stream));
  pb->counters_dirty = false;
  return PGX_OK;
}

// ====================================================================== ABI
extern "C" {

int pgx_abi_version(void) { return PGX_ABI_VERSION; }

const char* pgx_last_error(void) { return g_last_error.c_str(); }

size_t pgx_workspace_bytes(const pgx_desc* desc) {
  if (validate_desc(desc) != PGX_OK) return 0;
  return workspace_estimate(desc, 148);
}

pgx_status pgx_problem_create(const pgx_desc* desc, pgx_problem** out) {
  g_last_error.clear();
  if (!out) return fail(PGX_ERR_INVALID_ARGUMENT, "out must not be NULL");
  *out = nullptr;
  pgx_status st = validate_desc(desc);
  if (st != PGX_OK) return st;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(PGX_ERR_CUDA, "no CUDA device available (the pgx hot path has no CPU fallback)");
  PGX_CUDA(cudaSetDevice(desc->device));

  pgx_problem* pb = new pgx_problem();
  const bool design = desc->design != nullptr;
  pb->dim = design ? 2 : desc->dim;
  pb->kind = desc->basis_kind;
  pb->degree = design ? 0 : desc->degree;  // (the tail's kernel instantiation only)
  pb->K = design ? desc->design_k : feature_count(desc->dim, desc->degree);
  pb->N = desc->n_grains;
  pb->P = desc->n_points;
  pb->M = design ? -1 : desc->resolution;  // -1: no grid, no point list
  pb->prec = design ? PGX_PREC_EXACT : desc->precision;
  pb->device = desc->device;
  pb->stream = static_cast<cudaStream_t>(desc->stream);
  const int sms = sm_count(desc->device);
  pb->sms = sms;
  const int64_t P = pb->P;
  const int64_t KN = (int64_t)pb->K * pb->N;
  pb->blocks1 = (int)((P + kP1Threads - 1) / kP1Threads);
  const int tiles = (pb->N + kP2Threads - 1) / kP2Threads;
  pb->splits = general_splits(P, tiles, sms);

  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
  };
  if (pb->M == 0) A(pb->alloc(&pb->d_points, (size_t)P * pb->dim));
  if (design) A(pb->alloc(&pb->d_design, (size_t)P * pb->K));
  A(pb->alloc(&pb->d_labels, (size_t)P));
  A(pb->alloc(&pb->d_theta, (size_t)KN));
  A(pb->alloc(reinterpret_cast<double**>(&pb->d_theta_in), (size_t)KN));
  A(pb->alloc(&pb->d_pix_m, (size_t)P));
  A(pb->alloc(&pb->d_pix_ls, (size_t)P));
  A(pb->alloc(&pb->d_fix_list, (size_t)P));
  A(pb->alloc(&pb->d_counters, 4));
  A(pb->alloc(&pb->d_fix_correct, 2));
  A(pb->alloc(&pb->d_part_th2, (size_t)4 * sms + 8));
  A(pb->alloc(&pb->d_part_d, (size_t)pb->blocks1 * 2));
  A(pb->alloc(&pb->d_part_i, (size_t)pb->blocks1 * 4));
  A(pb->alloc(&pb->d_part_g, (size_t)pb->splits * KN));
  A(pb->alloc(&pb->d_grad, (size_t)KN));
  A(pb->alloc(&pb->d_stats, 1));
  A(pb->alloc(&pb->d_labels_out, (size_t)P));
  A(pb->alloc(&pb->d_margin_out, (size_t)P));
  if (pb->M > 0 && pb->dim == 2) A(pb->alloc(&pb->d_moments, (size_t)pb->N * 6 + 1));
  if (e == cudaSuccess && !design) e = grid_plan_create(pb->grid, desc, sms, pb->bytes);
  if (e == cudaSuccess) e = cudaMemset(pb->d_counters, 0, 4 * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(pb->d_fix_correct, 0, 2 * sizeof(long long));
  if (e != cudaSuccess) {
    size_t need = workspace_estimate(desc, sms);
    pb->release();
    delete pb;
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation)
      return fail(PGX_ERR_RESOURCE,
                  "device workspace allocation failed: needs about %zu bytes (P=%lld, K=%d, N=%d)",
                  need, (long long)P, feature_count(desc->dim, desc->degree), desc->n_grains);
    return fail(PGX_ERR_CUDA, "workspace allocation failed: %s", cudaGetErrorString(e));
  }

  // points
  const bool dev_in = desc->mem == PGX_MEM_DEVICE;
  const cudaMemcpyKind kind_in = dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (pb->M == 0) {
    if (!dev_in) {
      // geometry.py:40-43: finite and strictly inside the open cube
      for (int64_t q = 0; q < P * pb->dim; ++q) {
        double v = desc->points[q];
        if (!(v > -1.0 && v < 1.0)) {
          pb->release();
          delete pb;
          return fail(PGX_ERR_INVALID_ARGUMENT,
                      "grid points must be finite and lie strictly inside [-1,1]^%d", desc->dim);
        }
      }
    }
    cudaError_t c = cudaMemcpy(pb->d_points, desc->points, (size_t)P * pb->dim * 8, kind_in);
    if (c != cudaSuccess) {
      pb->release();
      delete pb;
      return fail(PGX_ERR_CUDA, "copying points failed: %s", cudaGetErrorString(c));
    }
  }
  if (design) {
    cudaError_t c = cudaMemcpy(pb->d_design, desc->design, (size_t)P * pb->K * 8, kind_in);
    if (c != cudaSuccess) {
      pb->release();
      delete pb;
      return fail(PGX_ERR_CUDA, "copying the design matrix failed: %s", cudaGetErrorString(c));
    }
  }
  // labels: int64 0-based -> int32 on device, range-checked (geometry.py:96-97)
  if (desc->labels0) {
    std::vector<int64_t> host((size_t)P);
    cudaError_t c =
        cudaMemcpy(host.data(), desc->labels0, (size_t)P * 8,
                   dev_in ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost);
    if (c != cudaSuccess) {
      pb->release();
      delete pb;
      return fail(PGX_ERR_CUDA, "reading labels failed: %s", cudaGetErrorString(c));
    }
    std::vector<int32_t> l32((size_t)P);
    for (int64_t q = 0; q < P; ++q) {
      int64_t v = host[(size_t)q];
      if (v < 0 || v >= pb->N) {
        pb->release();
        delete pb;
        return fail(PGX_ERR_INVALID_ARGUMENT, "labels0 must lie in [0, %d)", pb->N);
      }
      l32[(size_t)q] = (int32_t)v;
    }
    c = cudaMemcpy(pb->d_labels, l32.data(), (size_t)P * 4, cudaMemcpyHostToDevice);
    if (c != cudaSuccess) {
      pb->release();
      delete pb;
      return fail(PGX_ERR_CUDA, "copying labels failed: %s", cudaGetErrorString(c));
    }
    pb->has_labels = true;
  }
  *out = pb;
  return PGX_OK;
}

void pgx_problem_destroy(pgx_problem* pb) {
  if (!pb) return;
  cudaSetDevice(pb->device);
  if (pb->stream) cudaStreamSynchronize(pb->stream);
  pb->release();
  delete pb;
}

pgx_status pgx_set_stream(pgx_problem* pb, void* stream) {
  if (!pb) return fail(PGX_ERR_INVALID_ARGUMENT, "problem must not be NULL");
  pb->stream = static_cast<cudaStream_t>(stream);
  return PGX_OK;
}

size_t pgx_problem_bytes(pgx_problem* pb) { return pb ? pb->bytes : 0; }

pgx_status pgx_problem_label_moments(pgx_problem* pb, uint32_t flags, int64_t* out) {
  g_last_error.clear();
  if (!pb || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "problem and out must not be NULL");
  if (!pb->d_moments || !pb->has_labels)
    return fail(PGX_ERR_INVALID_ARGUMENT,
                "label moments need a regular 2-D grid problem created with labels");
  PGX_CUDA(cudaSetDevice(pb->device));
  int* bad = reinterpret_cast<int*>(pb->d_moments + (size_t)pb->N * 6);
  PGX_CUDA(launch_label_moments_i32(pb->M, pb->P, pb->d_labels, pb->N, pb->d_moments, bad, pb->sms, pb->stream));
  pb->last_launches = 1;
  const size_t nb = (size_t)pb->N * 6 * sizeof(int64_t);
  const bool dev = (flags & PGX_DEVICE_PTRS) != 0;
  PGX_CUDA(cudaMemcpyAsync(out, pb->d_moments, nb, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           pb->stream));
  if (!dev) PGX_CUDA(cudaStreamSynchronize(pb->stream));
  return PGX_OK;  // (labels were range-checked at creation: the flag word cannot be set)
}

int pgx_last_launch_count(pgx_problem* pb) { return pb ? pb->last_launches : 0; }

int pgx_problem_path(pgx_problem* pb) {
  if (!pb || !pb->grid.enabled) return PGX_PATH_GENERAL;
  return pb->grid.tc ? PGX_PATH_GRID_TC : PGX_PATH_GRID_FP64;
}

pgx_status pgx_set_profiling(pgx_problem* pb, int enable) {
  if (!pb) return fail(PGX_ERR_INVALID_ARGUMENT, "problem must not be NULL");
  PGX_CUDA(cudaSetDevice(pb->device));
  if (enable && !pb->prof_ev[0])
    for (cudaEvent_t& e : pb->prof_ev) PGX_CUDA(cudaEventCreate(&e));
  pb->profiling = enable != 0;
  pb->prof_n = 0;
  return PGX_OK;
}

int pgx_profile_count(pgx_problem* pb) { return pb ? pb->prof_n : 0; }

const char* pgx_profile_name(pgx_problem* pb, int i) {
  if (!pb || i < 0 || i >= pb->prof_n) return "";
  return pb->prof_name[i];
}

float pgx_profile_ms(pgx_problem* pb, int i) {
  if (!pb || i < 0 || i >= pb->prof_n) return -1.0f;
  float ms = -1.0f;
  if (cudaEventSynchronize(pb->prof_ev[2 * i + 1]) != cudaSuccess) return -1.0f;
  if (cudaEventElapsedTime(&ms, pb->prof_ev[2 * i], pb->prof_ev[2 * i + 1]) != cudaSuccess)
    return -1.0f;
  return ms;
}

pgx_status pgx_synchronize(pgx_problem* pb) {
  if (!pb) return fail(PGX_ERR_INVALID_ARGUMENT, "problem must not be NULL");
  PGX_CUDA(cudaStreamSynchronize(pb->stream));
  return PGX_OK;
}

static pgx_status eval_impl(pgx_problem* pb, const void* theta, double eps, double lambda,
                            uint32_t flags, double* grad_out, pgx_stats* stats_out, bool force_general);

pgx_status pgx_eval(pgx_problem* pb, const void* theta, double eps, double lambda, uint32_t flags,
                    double* grad_out, pgx_stats* stats_out) {
  g_last_error.clear();
  pgx_status st = eval_impl(pb, theta, eps, lambda, flags, grad_out, stats_out, false);
  if (st == PGX_OK && !(flags & PGX_DEVICE_PTRS) && (stats_out->flags & PGX_STAT_RANGE))
    st = eval_impl(pb, theta, eps, lambda, flags, grad_out, stats_out, true);
  else if (st == PGX_ERR_NUMERICAL && !(flags & PGX_DEVICE_PTRS) && pb->grid.enabled &&
           (stats_out->flags & PGX_STAT_RANGE))
    st = eval_impl(pb, theta, eps, lambda, flags, grad_out, stats_out, true);
  return st;
}

static pgx_status eval_impl(pgx_problem* pb, const void* theta, double eps, double lambda,
                            uint32_t flags, double* grad_out, pgx_stats* stats_out, bool force_general) {
  if (!pb) return fail(PGX_ERR_INVALID_ARGUMENT, "problem must not be NULL");
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(PGX_ERR_INVALID_ARGUMENT, "eps must be positive");
  if (!(lambda >= 0.0) || !std::isfinite(lambda))
    return fail(PGX_ERR_INVALID_ARGUMENT, "lambda must be a finite non-negative number");
  if (!pb->has_labels)
    return fail(PGX_ERR_INVALID_ARGUMENT, "problem was created without labels; only pgx_assign is available");
  const bool want_grad = flags & PGX_WANT_GRAD;
  const bool want_assign = flags & PGX_WANT_ASSIGN;
  const bool dev = flags & PGX_DEVICE_PTRS;
  if (want_grad && !grad_out) return fail(PGX_ERR_INVALID_ARGUMENT, "grad_out must not be NULL");
  if (!stats_out) return fail(PGX_ERR_INVALID_ARGUMENT, "stats_out must not be NULL");
  PGX_CUDA(cudaSetDevice(pb->device));
  cudaStream_t s = pb->stream;
  int launches = 0;
  pb->prof_reset();
  if (rearm_counters(pb) != PGX_OK) return PGX_ERR_CUDA;
  const double* theta64 = nullptr;
  const float* theta32 = nullptr;
  // fast modes check the logit-range bound of pgx.h PGX_STAT_RANGE on the
  // device (tail kernel); with host buffers an out-of-range theta is then
  // re-evaluated on the exact kernels (the general path) before returning
  const bool use_grid = pb->grid.enabled && !force_general;
  const bool fuse32 = use_grid && pb->grid.tc && (flags & PGX_THETA_F32);
  pgx_status st = stage_theta(pb, theta, flags, &theta64, &launches, fuse32 ? &theta32 : nullptr);
  if (st != PGX_OK) return st;

  // counters (fix-up list, non-finite, ticket) are zero here: zeroed at
  // creation and re-armed by the last CTA of the tail kernel.
  EvalParams prm = make_params(pb, eps);
  prm.theta = theta64;
  prm.theta32 = theta32;
  double* grad_dst = dev ? grad_out : pb->d_grad;
  pgx_stats* stats_dst = dev ? stats_out : pb->d_stats;
  // host results in pinned (device-mapped) memory: the tail kernel writes them
  // over the bus directly instead of two small D2H copies (each a few us of
  // DMA latency on the timeline); large gradients keep the copy engine
  bool zero_copy = false;
  if (!dev && (size_t)pb->K * pb->N * 8 <= kZeroCopyMax) {
    void* g_dev = nullptr;
    void* s_dev = host_mapped(stats_out);
    if (want_grad) g_dev = host_mapped(grad_out);
    if (s_dev && (!want_grad || g_dev)) {
      zero_copy = true;
      stats_dst = static_cast<pgx_stats*>(s_dev);
      if (want_grad) grad_dst = static_cast<double*>(g_dev);
    }
  }
  int blocks1 = pb->blocks1;
  pb->counters_dirty = true;  // until the tail (which re-arms them) is enqueued
  if (use_grid) {
    GridProf prof{pb, [](void* c, const char* n) { static_cast<pgx_problem*>(c)->prof_begin(n); },
                  [](void* c) { static_cast<pgx_problem*>(c)->prof_end(); }};
    st = grid_eval(pb->grid, prm, pb->prec, want_grad, s, &launches, &blocks1, prof);
    if (st != PGX_OK) return fail(st, "grid path: %s", cudaGetErrorString(cudaGetLastError()));
    PGX_LAUNCH_CHECK();
  } else if (pb->d_design) {
    pb->prof_begin("design_pass1");
    launch_design_pass1(prm, pb->d_design, pb->K, pb->blocks1, true, s);
    pb->prof_end();
    PGX_LAUNCH_CHECK();
    ++launches;
    if (want_grad) {
      pb->prof_begin("design_pass2");
      launch_design_pass2(prm, pb->d_design, pb->K, pb->splits, s);
      pb->prof_end();
      PGX_LAUNCH_CHECK();
      ++launches;
    }
  } else {
    pb->prof_begin("general_pass1");
    PGX_DISPATCH(launch_general_pass1, prm, pb->blocks1, true, s);
    pb->prof_end();
    PGX_LAUNCH_CHECK();
    ++launches;
    if (want_grad) {
      pb->prof_begin("general_pass2");
      PGX_DISPATCH(launch_general_pass2, prm, pb->N, pb->splits, s);
      pb->prof_end();
      PGX_LAUNCH_CHECK();
      ++launches;
    }
  }
  TailParams tp{};
  tp.want_grad = want_grad;
  tp.fix_amb = use_grid ? 1 : 0;
  tp.ticket = reinterpret_cast<unsigned*>(pb->d_counters + 2);
  tp.part_th2 = pb->d_part_th2;
  tp.range_c = use_grid ? 1.4426950408889634074 / eps : 0.0;
  tp.range_bits = reinterpret_cast<unsigned*>(pb->d_counters + 3);
  ReduceParams& rp = tp.red;
  rp.K = pb->K;
  rp.N = pb->N;
  rp.splits = use_grid ? pb->grid.splits_out : pb->splits;
  rp.P = pb->P;
  rp.eps = eps;
  rp.lambda = lambda;
  rp.theta = theta64;
  rp.part_g = use_grid ? pb->grid.part_out : pb->d_part_g;
  rp.grad_out = grad_dst;
  rp.nonfinite = pb->d_counters + 1;
  FinalParams& fp = tp.fin;
  fp.blocks1 = blocks1;
  fp.K = pb->K;
  fp.N = pb->N;
  fp.P = pb->P;
  fp.eps = eps;
  fp.lambda = lambda;
  fp.want_assign = want_assign;
  fp.theta = theta64;
  fp.part_d = pb->d_part_d;
  fp.part_i = pb->d_part_i;
  fp.fix_correct = pb->d_fix_correct;
  fp.nonfinite_grad = want_grad ? pb->d_counters + 1 : nullptr;
  fp.stats_out = stats_dst;
  const int64_t KN = (int64_t)pb->K * pb->N;
  const int tail_blocks =
      want_grad ? (int)std::min<int64_t>((KN + 7) / 8, 4 * pb->sms) : pb->sms;
  pb->prof_begin("tail");
  PGX_DISPATCH(launch_tail, prm, tp, tail_blocks, s);
  pb->prof_end();
  PGX_LAUNCH_CHECK();
  pb->counters_dirty = false;
  ++launches;
  pb->last_launches = launches;

  if (!dev) {
    if (!zero_copy) {
      if (want_grad)
        PGX_CUDA(cudaMemcpyAsync(grad_out, pb->d_grad, (size_t)pb->K * pb->N * 8,
                                 cudaMemcpyDeviceToHost, s));
      PGX_CUDA(cudaMemcpyAsync(stats_out, pb->d_stats, sizeof(pgx_stats), cudaMemcpyDeviceToHost, s));
    }
    PGX_CUDA(cudaStreamSynchronize(s));
    if (stats_out->n_nonfinite > 0)
      return fail(PGX_ERR_NUMERICAL, "non-finite objective or gradient: phi=%g (%lld non-finite terms)",
                  stats_out->phi, (long long)stats_out->n_nonfinite);
  }
  return PGX_OK;
}

pgx_status pgx_assign(pgx_problem* pb, const void* theta, uint32_t flags, int64_t* labels_out,
                      float* margin_out, pgx_stats* stats_out) {
  g_last_error.clear();
  if (!pb) return fail(PGX_ERR_INVALID_ARGUMENT, "problem must not be NULL");
  if (!labels_out) return fail(PGX_ERR_INVALID_ARGUMENT, "labels_out must not be NULL");
  const bool dev = flags & PGX_DEVICE_PTRS;
  PGX_CUDA(cudaSetDevice(pb->device));
  cudaStream_t s = pb->stream;
  int launches = 0;
  if (rearm_counters(pb) != PGX_OK) return PGX_ERR_CUDA;
  const double* theta64 = nullptr;
  pgx_status st = stage_theta(pb, theta, flags, &theta64, &launches);
  if (st != PGX_OK) return st;
  pb->counters_dirty = true;
  EvalParams prm = make_params(pb, 1.0);
  prm.theta = theta64;
  prm.labels_out = reinterpret_cast<long long*>(dev ? labels_out : (int64_t*)pb->d_labels_out);
  prm.margin_out = margin_out ? (dev ? margin_out : pb->d_margin_out) : nullptr;
  // tensor-core problems assign with the sweep kernel's ASSIGN variant (fp32
  // screening on the tensor cores, exact fp64 decision of every candidate, the
  // tail's exact re-scan for the rest): bit-identical labels, no N x P costs
  const bool use_tc = pb->grid.enabled && pb->grid.tc && !pb->d_design;
  int blocks1 = pb->blocks1;
  pb->prof_reset();
  if (use_tc) {
    GridProf prof{pb, [](void* c, const char* n) { static_cast<pgx_problem*>(c)->prof_begin(n); },
                  [](void* c) { static_cast<pgx_problem*>(c)->prof_end(); }};
    st = grid_assign(pb->grid, prm, s, &launches, &blocks1, prof);
    if (st != PGX_OK) return fail(st, "grid assign: %s", cudaGetErrorString(cudaGetLastError()));
  } else if (pb->d_design) {
    launch_design_pass1(prm, pb->d_design, pb->K, pb->blocks1, false, s);
    ++launches;
  } else {
    pb->prof_begin("general_assign");
    PGX_DISPATCH(launch_general_pass1, prm, pb->blocks1, false, s);
    pb->prof_end();
    ++launches;
  }
  PGX_LAUNCH_CHECK();
  TailParams tp{};
  tp.want_grad = 0;
  tp.fix_amb = use_tc ? 1 : 0;
  tp.ticket = reinterpret_cast<unsigned*>(pb->d_counters + 2);
  tp.part_th2 = pb->d_part_th2;
  FinalParams& fp = tp.fin;
  fp.blocks1 = blocks1;
  fp.K = pb->K;
  fp.N = pb->N;
  fp.P = pb->P;
  fp.eps = 1.0;
  fp.want_assign = 1;
  fp.theta = theta64;
  fp.part_d = pb->d_part_d;
  fp.part_i = pb->d_part_i;
  fp.fix_correct = pb->d_fix_correct;
  fp.stats_out = (stats_out && dev) ? (void*)stats_out : (void*)pb->d_stats;
  PGX_DISPATCH(launch_tail, prm, tp, pb->sms, s);
  PGX_LAUNCH_CHECK();
  pb->counters_dirty = false;
  ++launches;
  pb->last_launches = launches;
  if (!dev) {
    PGX_CUDA(cudaMemcpyAsync(labels_out, pb->d_labels_out, (size_t)pb->P * 8, cudaMemcpyDeviceToHost, s));
    if (margin_out)
      PGX_CUDA(cudaMemcpyAsync(margin_out, pb->d_margin_out, (size_t)pb->P * 4,
                               cudaMemcpyDeviceToHost, s));
    if (stats_out)
      PGX_CUDA(cudaMemcpyAsync(stats_out, pb->d_stats, sizeof(pgx_stats), cudaMemcpyDeviceToHost, s));
    PGX_CUDA(cudaStreamSynchronize(s));
  }
  return PGX_OK;
}

pgx_status pgx_soft_assign(pgx_problem* pb, const void* theta, double eps, uint32_t flags, double* prob_out) {
  g_last_error.clear();
  if (!pb) return fail(PGX_ERR_INVALID_ARGUMENT, "problem must not be NULL");
  if (!prob_out) return fail(PGX_ERR_INVALID_ARGUMENT, "prob_out must not be NULL");
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(PGX_ERR_INVALID_ARGUMENT, "eps must be positive");
  const bool dev = flags & PGX_DEVICE_PTRS;
  PGX_CUDA(cudaSetDevice(pb->device));
  cudaStream_t s = pb->stream;
  int launches = 0;
  const double* theta64 = nullptr;
  pgx_status st = stage_theta(pb, theta, flags, &theta64, &launches);
  if (st != PGX_OK) return st;
  const size_t bytes = (size_t)pb->N * pb->P * 8;
  double* out = prob_out;
  if (!dev) PGX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out), bytes, s));
  EvalParams prm = make_params(pb, eps);
  prm.theta = theta64;
  if (pb->d_design)
    launch_design_soft(prm, pb->d_design, pb->K, out, s);
  else
    PGX_DISPATCH(launch_general_soft, prm, out, s);
  cudaError_t le = cudaGetLastError();
  if (!dev) {
    if (le == cudaSuccess) le = cudaMemcpyAsync(prob_out, out, bytes, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(out, s);
    if (le == cudaSuccess) le = cudaStreamSynchronize(s);
  }
  if (le != cudaSuccess) return fail(PGX_ERR_CUDA, "soft assignment failed: %s", cudaGetErrorString(le));
  pb->last_launches = launches + 1;
  return PGX_OK;
}

// ------------------------------------------------------------------ device-resident optimiser state
// (kernels in k_lbfgs.cu)
struct pgx_lbfgs {
  pgx_problem* pb = nullptr;
  int m = 10;
  int64_t n = 0;  // K (N - 1) free parameters
  double *u = nullptr, *g = nullptr, *ut = nullptr, *gt = nullptr, *d = nullptr;
  double *S = nullptr, *Y = nullptr, *rho = nullptr, *alpha = nullptr;
  double *theta = nullptr, *grad = nullptr;  // K x N, what pgx_eval reads / writes
  int* state = nullptr;                      // {head, count}
  double* host = nullptr;                    // pinned + mapped: [0] t, [2..5] kernel scalars, [8..] pgx_stats
  double* host_dev = nullptr;                // its device alias
  bool have_dir = false;                     // d holds a direction (trial points are u + t d)
  cudaGraphExec_t graph = nullptr;           // point -> pgx_eval -> after, for (eps, lambda, have_dir)
  double g_eps = 0.0, g_lambda = 0.0;
  bool g_dir = false;
  // the legacy default stream cannot be captured: a problem on it runs the
  // optimiser calls on this stream instead (every call synchronises before returning)
  cudaStream_t own_stream = nullptr;
  // accept -> two-loop -> first trial as one graph (pgx_lbfgs_iterate), for (eps, lambda, keep_pair)
  cudaGraphExec_t it_graph = nullptr;
  double it_eps = 0.0, it_lambda = 0.0;
  int it_keep = -1;
  void drop_graph() {
    if (graph) cudaGraphExecDestroy(graph);
    if (it_graph) cudaGraphExecDestroy(it_graph);
    graph = nullptr;
    it_graph = nullptr;
  }
};

namespace {

constexpr int kLbScal = 2, kLbStats = 8;  // offsets (in doubles) inside pgx_lbfgs::host
constexpr int kLbDir = 24, kLbAcc = 28;   // pgx_lbfgs_iterate: direction / accept scalars

// runs the problem on the state's own stream while a call is in progress (see own_stream)
struct LbStream {
  pgx_problem* pb;
  cudaStream_t saved;
  explicit LbStream(pgx_lbfgs* st) : pb(st->pb), saved(st->pb->stream) {
    if (!saved || saved == cudaStreamLegacy) {
      cudaStreamSynchronize(saved);
      pb->stream = st->own_stream;
    }
  }
  ~LbStream() { pb->stream = saved; }
};

// enqueue: theta <- u (+ t d); evaluate; pack the free-column gradient and its dot products
pgx_status lb_enqueue(pgx_lbfgs* st, double eps, double lambda) {
  pgx_problem* pb = st->pb;
  launch_lb_point(st->theta, st->ut, st->u, st->have_dir ? st->d : nullptr, st->host_dev, pb->K, pb->N,
                  pb->sms, pb->stream);
  PGX_LAUNCH_CHECK();
  pgx_status rc = eval_impl(pb, st->theta, eps, lambda, PGX_WANT_GRAD | PGX_WANT_ASSIGN | PGX_DEVICE_PTRS,
                            st->grad, reinterpret_cast<pgx_stats*>(st->host_dev + kLbStats), false);
  if (rc != PGX_OK) return rc;
  launch_lb_after(st->grad, st->gt, st->have_dir ? st->d : nullptr, st->host_dev + kLbScal, pb->K, pb->N,
                  pb->stream);
  PGX_LAUNCH_CHECK();
  return PGX_OK;
}

// one evaluation at u + t d through the captured graph (re-captured when eps,
// lambda or the kind of point changes); out = {phi, g_t.d, err, e0, n_nonfinite, flags, |g_t|^2}
pgx_status lb_evaluate(pgx_lbfgs* st, double t, double eps, double lambda, double* out) {
  pgx_problem* pb = st->pb;
  PGX_CUDA(cudaSetDevice(pb->device));
  static const bool use_graph = [] {
    const char* e = std::getenv("PGX_FIT_GRAPH");
    return !(e && e[0] == '0');
  }();
  st->host[0] = t;
  if (use_graph && !pb->profiling) {
    if (!st->graph || st->g_eps != eps || st->g_lambda != lambda || st->g_dir != st->have_dir) {
      st->drop_graph();
      // (the first evaluation of a problem runs its one-time set-up launches: not captured)
      pgx_status rc = lb_enqueue(st, eps, lambda);
      if (rc != PGX_OK) return rc;
      PGX_CUDA(cudaStreamSynchronize(pb->stream));
      cudaGraph_t gr = nullptr;
      PGX_CUDA(cudaStreamBeginCapture(pb->stream, cudaStreamCaptureModeThreadLocal));
      rc = lb_enqueue(st, eps, lambda);
      cudaError_t ce = cudaStreamEndCapture(pb->stream, &gr);
      if (rc != PGX_OK || ce != cudaSuccess) {
        if (gr) cudaGraphDestroy(gr);
        (void)cudaGetLastError();
        return rc != PGX_OK ? rc : fail(PGX_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
      }
      ce = cudaGraphInstantiate(&st->graph, gr, 0);
      cudaGraphDestroy(gr);
      if (ce != cudaSuccess) return fail(PGX_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
      st->g_eps = eps;
      st->g_lambda = lambda;
      st->g_dir = st->have_dir;
      // (the uncaptured run above already evaluated this point: its results stand)
    } else {
      PGX_CUDA(cudaGraphLaunch(st->graph, pb->stream));
    }
  } else {
    pgx_status rc = lb_enqueue(st, eps, lambda);
    if (rc != PGX_OK) return rc;
  }
  PGX_CUDA(cudaStreamSynchronize(pb->stream));
  const pgx_stats* ps = reinterpret_cast<const pgx_stats*>(st->host + kLbStats);
  out[0] = ps->phi;
  out[1] = st->host[kLbScal];
  out[2] = ps->err;
  out[3] = ps->e0;
  out[4] = (double)ps->n_nonfinite;
  out[5] = (double)ps->flags;
  out[6] = st->host[kLbScal + 1];
  return PGX_OK;
}

}  // namespace

void pgx_lbfgs_destroy(pgx_lbfgs* st) {
  if (!st) return;
  st->drop_graph();
  void* bufs[] = {st->u, st->g, st->ut, st->gt, st->d, st->S, st->Y, st->rho, st->alpha, st->theta, st->grad,
                  st->state};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (st->host) cudaFreeHost(st->host);
  if (st->own_stream) cudaStreamDestroy(st->own_stream);
  delete st;
}

pgx_status pgx_lbfgs_create(pgx_problem* pb, int memory, pgx_lbfgs** out) {
  g_last_error.clear();
  if (!pb || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "problem and out must not be NULL");
  if (memory < 1 || memory > 256) return fail(PGX_ERR_INVALID_ARGUMENT, "memory must lie in 1..256");
  if (!pb->has_labels) return fail(PGX_ERR_INVALID_ARGUMENT, "problem was created without labels");
  PGX_CUDA(cudaSetDevice(pb->device));
  pgx_lbfgs* st = new pgx_lbfgs();
  st->pb = pb;
  st->m = memory;
  st->n = (int64_t)pb->K * (pb->N - 1);
  const size_t n = (size_t)st->n, kn = (size_t)pb->K * pb->N, ring = (size_t)memory + 1;
  cudaError_t e = cudaSuccess;
  auto alloc = [&](double** p, size_t cnt) {
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(1, cnt) * 8);
    if (e == cudaSuccess) e = cudaMemset(*p, 0, std::max<size_t>(1, cnt) * 8);
  };
  alloc(&st->u, n), alloc(&st->g, n), alloc(&st->ut, n), alloc(&st->gt, n), alloc(&st->d, n);
  alloc(&st->S, ring * n), alloc(&st->Y, ring * n), alloc(&st->rho, ring), alloc(&st->alpha, ring);
  alloc(&st->theta, kn), alloc(&st->grad, kn);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&st->state), 2 * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(st->state, 0, 2 * sizeof(int));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st->own_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&st->host), 64 * 8, cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&st->host_dev), st->host, 0);
  if (e != cudaSuccess) {
    pgx_lbfgs_destroy(st);
    return fail(e == cudaErrorMemoryAllocation ? PGX_ERR_RESOURCE : PGX_ERR_CUDA,
                "optimiser state (%zu bytes): %s", (2 * ring + 5) * n * 8 + 2 * kn * 8, cudaGetErrorString(e));
  }
  std::memset(st->host, 0, 64 * 8);
  *out = st;
  return PGX_OK;
}

pgx_status pgx_lbfgs_start(pgx_lbfgs* st, const double* theta, double eps, double lambda, double* out) {
  g_last_error.clear();
  if (!st || !theta || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "state, theta and out must not be NULL");
  LbStream stream_scope(st);
  pgx_problem* pb = st->pb;
  PGX_CUDA(cudaSetDevice(pb->device));
  // u <- the free columns of the host theta (K x N): staged through st->grad
  PGX_CUDA(cudaMemcpyAsync(st->grad, theta, (size_t)pb->K * pb->N * 8, cudaMemcpyHostToDevice, pb->stream));
  launch_lb_after(st->grad, st->u, nullptr, st->host_dev + kLbScal, pb->K, pb->N, pb->stream);
  PGX_LAUNCH_CHECK();
  PGX_CUDA(cudaMemsetAsync(st->state, 0, 2 * sizeof(int), pb->stream));
  PGX_CUDA(cudaMemsetAsync(st->theta, 0, (size_t)pb->K * pb->N * 8, pb->stream));
  st->have_dir = false;
  return pgx_lbfgs_restart(st, eps, lambda, out);
}

pgx_status pgx_lbfgs_restart(pgx_lbfgs* st, double eps, double lambda, double* out) {
  g_last_error.clear();
  if (!st || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "state and out must not be NULL");
  LbStream stream_scope(st);
  pgx_problem* pb = st->pb;
  PGX_CUDA(cudaSetDevice(pb->device));
  PGX_CUDA(cudaMemsetAsync(st->state, 0, 2 * sizeof(int), pb->stream));  // drop the history
  st->have_dir = false;
  pgx_status rc = lb_evaluate(st, 0.0, eps, lambda, out);
  if (rc != PGX_OK) return rc;
  // the evaluated point becomes the current one: g <- g_t (u_t == u)
  PGX_CUDA(cudaMemcpyAsync(st->g, st->gt, (size_t)st->n * 8, cudaMemcpyDeviceToDevice, pb->stream));
  PGX_CUDA(cudaStreamSynchronize(pb->stream));
  return PGX_OK;
}

pgx_status pgx_lbfgs_clear(pgx_lbfgs* st) {
  g_last_error.clear();
  if (!st) return fail(PGX_ERR_INVALID_ARGUMENT, "state must not be NULL");
  LbStream stream_scope(st);
  PGX_CUDA(cudaSetDevice(st->pb->device));
  PGX_CUDA(cudaMemsetAsync(st->state, 0, 2 * sizeof(int), st->pb->stream));
  return PGX_OK;
}

pgx_status pgx_lbfgs_direction(pgx_lbfgs* st, int mode, double* out) {
  g_last_error.clear();
  if (!st || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "state and out must not be NULL");
  LbStream stream_scope(st);
  if (mode < 0 || mode > 2) return fail(PGX_ERR_INVALID_ARGUMENT, "mode must be 0, 1 or 2");
  pgx_problem* pb = st->pb;
  PGX_CUDA(cudaSetDevice(pb->device));
  launch_lb_two_loop(st->g, st->d, st->S, st->Y, st->rho, st->alpha, st->state, st->m, st->n, mode,
                     st->host_dev + kLbScal, pb->stream);
  PGX_LAUNCH_CHECK();
  PGX_CUDA(cudaStreamSynchronize(pb->stream));
  for (int i = 0; i < 4; ++i) out[i] = st->host[kLbScal + i];
  st->have_dir = true;
  return PGX_OK;
}

pgx_status pgx_lbfgs_trial(pgx_lbfgs* st, double t, double eps, double lambda, double* out) {
  g_last_error.clear();
  if (!st || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "state and out must not be NULL");
  LbStream stream_scope(st);
  if (!st->have_dir) return fail(PGX_ERR_INVALID_ARGUMENT, "no search direction: call pgx_lbfgs_direction first");
  return lb_evaluate(st, t, eps, lambda, out);
}

pgx_status pgx_lbfgs_accept(pgx_lbfgs* st, int keep_pair, double* out) {
  g_last_error.clear();
  if (!st || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "state and out must not be NULL");
  LbStream stream_scope(st);
  pgx_problem* pb = st->pb;
  PGX_CUDA(cudaSetDevice(pb->device));
  launch_lb_accept(st->u, st->g, st->ut, st->gt, st->S, st->Y, st->rho, st->state, st->m, st->n, 1e-10,
                   keep_pair, st->host_dev + kLbScal, pb->stream);
  PGX_LAUNCH_CHECK();
  PGX_CUDA(cudaStreamSynchronize(pb->stream));
  for (int i = 0; i < 4; ++i) out[i] = st->host[kLbScal + i];
  return PGX_OK;
}

// One L-BFGS iteration's device work in ONE submission and one synchronisation:
// [accept the last trial (keep_pair >= 0)] -> two-loop direction -> trial at u + t0 d.
// out[0..3] accept scalars (as pgx_lbfgs_accept; zeros without accept),
// out[4..7] direction scalars (as pgx_lbfgs_direction), out[8..14] trial scalars
// (as pgx_lbfgs_trial).  The host then runs its line search from the first trial.
pgx_status pgx_lbfgs_iterate(pgx_lbfgs* st, int keep_pair, double t0, double eps, double lambda, double* out) {
  g_last_error.clear();
  if (!st || !out) return fail(PGX_ERR_INVALID_ARGUMENT, "state and out must not be NULL");
  LbStream stream_scope(st);
  pgx_problem* pb = st->pb;
  PGX_CUDA(cudaSetDevice(pb->device));
  static const bool use_graph = [] {
    const char* e = std::getenv("PGX_FIT_GRAPH");
    return !(e && e[0] == '0');
  }();
  st->host[0] = t0;
  auto enqueue = [&]() -> pgx_status {
    if (keep_pair >= 0) {
      launch_lb_accept(st->u, st->g, st->ut, st->gt, st->S, st->Y, st->rho, st->state, st->m, st->n, 1e-10,
                       keep_pair, st->host_dev + kLbAcc, pb->stream);
      PGX_LAUNCH_CHECK();
    }
    launch_lb_two_loop(st->g, st->d, st->S, st->Y, st->rho, st->alpha, st->state, st->m, st->n, 0,
                       st->host_dev + kLbDir, pb->stream);
    PGX_LAUNCH_CHECK();
    st->have_dir = true;
    return lb_enqueue(st, eps, lambda);
  };
  if (use_graph && !pb->profiling && st->graph) {  // (the plain trial graph exists: set-up launches are done)
    if (!st->it_graph || st->it_eps != eps || st->it_lambda != lambda || st->it_keep != keep_pair) {
      if (st->it_graph) cudaGraphExecDestroy(st->it_graph);
      st->it_graph = nullptr;
      cudaGraph_t gr = nullptr;
      PGX_CUDA(cudaStreamBeginCapture(pb->stream, cudaStreamCaptureModeThreadLocal));
      pgx_status rc = enqueue();
      cudaError_t ce = cudaStreamEndCapture(pb->stream, &gr);
      if (rc != PGX_OK || ce != cudaSuccess) {
        if (gr) cudaGraphDestroy(gr);
        (void)cudaGetLastError();
        return rc != PGX_OK ? rc : fail(PGX_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
      }
      ce = cudaGraphInstantiate(&st->it_graph, gr, 0);
      cudaGraphDestroy(gr);
      if (ce != cudaSuccess) return fail(PGX_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
      st->it_eps = eps;
      st->it_lambda = lambda;
      st->it_keep = keep_pair;
    }
    st->have_dir = true;
    PGX_CUDA(cudaGraphLaunch(st->it_graph, pb->stream));
  } else {
    pgx_status rc = enqueue();
    if (rc != PGX_OK) return rc;
  }
  PGX_CUDA(cudaStreamSynchronize(pb->stream));
  const pgx_stats* ps = reinterpret_cast<const pgx_stats*>(st->host + kLbStats);
  for (int i = 0; i < 4; ++i) out[i] = keep_pair >= 0 ? st->host[kLbAcc + i] : 0.0;
  for (int i = 0; i < 4; ++i) out[4 + i] = st->host[kLbDir + i];
  out[8] = ps->phi;
  out[9] = st->host[kLbScal];
  out[10] = ps->err;
  out[11] = ps->e0;
  out[12] = (double)ps->n_nonfinite;
  out[13] = (double)ps->flags;
  out[14] = st->host[kLbScal + 1];
  return PGX_OK;
}

pgx_status pgx_lbfgs_theta(pgx_lbfgs* st, double* theta_out) {
  g_last_error.clear();
  if (!st || !theta_out) return fail(PGX_ERR_INVALID_ARGUMENT, "state and theta_out must not be NULL");
  LbStream stream_scope(st);
  pgx_problem* pb = st->pb;
  PGX_CUDA(cudaSetDevice(pb->device));
  // theta <- u (the current point, not the last trial)
  const bool dir = st->have_dir;
  st->have_dir = false;
  launch_lb_point(st->theta, st->ut, st->u, nullptr, st->host_dev, pb->K, pb->N, pb->sms, pb->stream);
  st->have_dir = dir;
  PGX_LAUNCH_CHECK();
  PGX_CUDA(cudaMemcpyAsync(theta_out, st->theta, (size_t)pb->K * pb->N * 8, cudaMemcpyDeviceToHost, pb->stream));
  PGX_CUDA(cudaStreamSynchronize(pb->stream));
  return PGX_OK;
}

}  // extern "C"
