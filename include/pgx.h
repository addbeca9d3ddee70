/*
 * pgx.h — C ABI of the B200-native polygrain fit hot path (libpgx.so).
 *
 * This is the drop-in boundary for the reference's in-process NumPy hot path
 * (reference = /root/reference/pkg/src/polygrain):
 *
 *   pgx_problem_create  replaces  basis.assemble_design_matrix   (basis.py:183-193)
 *                       + the per-fit ``labels0 = labels - 1``    (optimizer.py:205-207)
 *                       — no K x P design matrix is ever formed: the grid
 *                       coordinates (geometry.py:59-71) and the Legendre /
 *                       monomial features (basis.py:105-142) are regenerated
 *                       on the device inside the kernels.
 *   pgx_eval            replaces  objective.evaluate_objective    (objective.py:129-165)
 *                       (Phi, grad, err, e0 of one fused evaluation; also the
 *                       bodies of objective() :168-178 and gradient() :181-198)
 *   pgx_assign          replaces  objective.hard_assign           (objective.py:70-77)
 *                       + geometry.argmin_labels                   (geometry.py:201-210)
 *                       without the N x P cost matrix.
 *   pgx_last_error      carries the message of the exception the reference
 *                       would raise (errors.py:4-13).
 *
 * Conventions
 *  - theta is K x N row-major (column i = grain i), exactly ParamMatrix.values
 *    (basis.py:287-327); fp64 by default, fp32 with PGX_THETA_F32.
 *  - labels are 0-based int64, exactly the reference's ``labels0``.
 *  - Without PGX_DEVICE_PTRS every pointer argument is HOST memory: the call
 *    copies theta to the device, runs, copies results back and synchronises.
 *    With PGX_DEVICE_PTRS they are device pointers and the call is enqueued on
 *    the problem's stream without synchronising (CUDA-Graph capturable: no
 *    allocation happens after pgx_problem_create).
 *  - Results are bit-identical run to run (fixed reduction partitions, fp64
 *    final reduction, no floating-point atomics) — the GPU analogue of the
 *    reference's threads == 1 sequential fold (objective.py:155-158).
 *  - Status codes map onto the reference's exceptions:
 *      PGX_ERR_INVALID_ARGUMENT -> ValueError      (objective.py:171-175)
 *      PGX_ERR_RESOURCE         -> ResourceError   (basis.py:185-192)
 *      PGX_ERR_NUMERICAL        -> NumericalError  (optimizer.py:222-226)
 *      PGX_ERR_CUDA             -> RuntimeError
 *  - A handle is used by one host thread at a time.
 */
#ifndef PGX_H
#define PGX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGX_ABI_VERSION 2

typedef enum {
    PGX_OK = 0,
    PGX_ERR_INVALID_ARGUMENT = 1,
    PGX_ERR_RESOURCE = 2,
    PGX_ERR_NUMERICAL = 3,
    PGX_ERR_CUDA = 4
} pgx_status;

/* basis kinds: basis.py:29-31 (MONOMIAL, LEGENDRE) */
enum { PGX_BASIS_MONOMIAL = 0, PGX_BASIS_LEGENDRE = 1 };

/* precision modes (DESIGN.md "Precision modes" states each tolerance) */
enum {
    PGX_PREC_EXACT = 0, /* fp64 logits, fp64 exp/log — reference-faithful     */
    PGX_PREC_FP64 = 1,  /* fp64 logits, fp32 (MUFU) exp of an fp64 argument   */
    PGX_PREC_TC = 2     /* tcgen05 fp16-split logits + fp64 near-min refine   */
};

/* flags for pgx_eval / pgx_assign */
enum {
    PGX_WANT_GRAD = 1u,   /* objective.py:109-113 (want_grad)   */
    PGX_WANT_ASSIGN = 2u, /* objective.py:115-119 (want_assign) */
    PGX_DEVICE_PTRS = 4u, /* pointers are device memory; async on the stream */
    PGX_THETA_F32 = 8u    /* theta is float32 instead of float64 */
};

/* where pgx_desc.points / pgx_desc.labels0 live */
enum { PGX_MEM_HOST = 0, PGX_MEM_DEVICE = 1 };

typedef struct {
    int32_t dim;          /* ambient dimension: 2 (reference) or 3 (extension)  */
    int32_t basis_kind;   /* PGX_BASIS_*                                        */
    int32_t degree;       /* total degree d >= 0; K = C(d+dim, dim)             */
    int32_t n_grains;     /* N >= 2 (geometry.py:94-95)                          */
    int64_t n_points;     /* P >= 1                                             */
    int32_t resolution;   /* M > 0: regular (2M)^dim grid generated on device
                             (geometry.py:59-71); 0: unstructured points       */
    int32_t precision;    /* PGX_PREC_*                                         */
    const double* points; /* n_points x dim row-major when resolution == 0     */
    const int64_t* labels0; /* n_points 0-based labels in [0, N)               */
    int32_t mem;          /* PGX_MEM_HOST or PGX_MEM_DEVICE for points/labels0  */
    int32_t device;       /* CUDA device ordinal                                */
    void* stream;         /* cudaStream_t (NULL = legacy default stream)        */
    /* Explicit design matrix (objective.py:129-132 ``design_values``): when not
     * NULL, design is K x n_points row-major fp64 (K = design_k <= 66, any
     * features), in host or device memory per ``mem``; dim, basis_kind,
     * degree, resolution and points are then ignored.  The exact fp64
     * kernels evaluate it (PGX_PREC_EXACT arithmetic whatever ``precision``). */
    const double* design;
    int32_t design_k;
} pgx_desc;

/* Scalar results of one evaluation (objective.EvalResult, objective.py:90-94,
 * plus the counters the host needs). */
typedef struct {
    double phi;            /* Phi (+ lambda term)                              */
    double err;            /* 1 - n_correct / P           (want_assign)        */
    double e0;             /* mean(h_G - min h)           (want_assign)        */
    double n_rescanned;    /* points whose arg-min needed the exact fp64 re-scan */
    int64_t n_points;      /* P                                                */
    int64_t n_correct;     /* pixels whose tie-tolerant arg-min equals G       */
    int64_t n_ambiguous;   /* pixels whose top-2 margin <= tau (1 + |min|)     */
    int64_t n_nonfinite;   /* non-finite Phi / grad contributions seen         */
    int64_t flags;         /* PGX_STAT_* bits                                  */
} pgx_stats;

/* pgx_stats.flags.  PGX_STAT_RANGE: a fast mode (FP64 / TC) evaluated a theta
 * whose logit range max_i sum_k |theta_ki| / (eps ln 2) exceeds 2^16, beyond
 * which the fp32 / fp16-split logits no longer meet the stated tolerances.
 * With host pointers pgx_eval never returns it: it evaluates such a theta on
 * the exact kernels instead (PGX_PREC_EXACT arithmetic).  With
 * PGX_DEVICE_PTRS the check runs on the device and the caller re-evaluates
 * (the Python device loop does so on a PGX_PREC_EXACT problem). */
enum { PGX_STAT_RANGE = 1 };
#define PGX_FAST_RANGE 65536.0

typedef struct pgx_problem pgx_problem;

int pgx_abi_version(void);

/* Thread-local message of the last failing call ("" if none). */
const char* pgx_last_error(void);

/* Bytes of device workspace pgx_problem_create would allocate. */
size_t pgx_workspace_bytes(const pgx_desc* desc);

pgx_status pgx_problem_create(const pgx_desc* desc, pgx_problem** out);
void pgx_problem_destroy(pgx_problem* problem);

/* Re-targets the stream used by subsequent calls (cudaStream_t). */
pgx_status pgx_set_stream(pgx_problem* problem, void* stream);

/* One fused evaluation: Phi, grad (K x N, fp64, = -(1/(eps P)) sum_x
 * (onehot - softmax) eta, no gauge projection) and the assignment statistics.
 * lambda >= 0 adds -lambda/2 ||theta[:, :N-1]||^2 to Phi and
 * -lambda theta[:, :N-1] to grad (lambda = 0 is the reference). grad_out may
 * be NULL when PGX_WANT_GRAD is not set. Without PGX_DEVICE_PTRS the call is
 * synchronous; host result buffers in pinned (mapped) memory are written by the
 * last kernel directly (up to 256 KB of gradient), pageable ones by copies. */
pgx_status pgx_eval(pgx_problem* problem, const void* theta, double eps, double lambda,
                    uint32_t flags, double* grad_out, pgx_stats* stats_out);

/* Tie-tolerant hard assignment: labels_out[p] = 1-based smallest grain index
 * whose cost is <= min + 1e-12 (1 + |min|); margin_out (nullable) receives the
 * top-2 cost margin; stats_out (nullable) receives n_correct / n_ambiguous. */
pgx_status pgx_assign(pgx_problem* problem, const void* theta, uint32_t flags,
                      int64_t* labels_out, float* margin_out, pgx_stats* stats_out);

/* Dense soft assignment (objective.py:80-87, a small-problem diagnostic):
 * prob_out[i * n_points + x] = exp((min_j h_j(x) - h_i(x)) / eps) / sum_j (...),
 * N x n_points fp64 (host memory unless PGX_DEVICE_PTRS).  eps > 0. */
pgx_status pgx_soft_assign(pgx_problem* problem, const void* theta, double eps, uint32_t flags,
                           double* prob_out);

/* Per-grain label moments of a regular 2-D grid (make_grid(resolution)), the
 * input of the moment heuristic (heuristics.py:46-73, np.bincount of 1, x_a and
 * x_a x_b by label).  out[6 i + q], q = 0..5, receives the exact integer sums of
 * {1, a1, a2, a1^2, a1 a2, a2^2} over the pixels of grain i, where
 * a = 2 resolution x is the odd integer coordinate.  labels0: host, 0-based.
 * Stand-alone (no problem handle); synchronous. */
pgx_status pgx_label_moments(int resolution, int64_t n_points, const int64_t* labels0, int n_grains,
                             int64_t* out);
const char* pgx_label_moments_error(void);

/* The same sums from a problem handle: a regular 2-D grid problem created with
 * labels (its device-resident labels are used: no label upload, no allocation,
 * stream-ordered on the problem's stream).  out: n_grains x 6 int64, host
 * memory (the call then synchronises) or device memory with PGX_DEVICE_PTRS. */
pgx_status pgx_problem_label_moments(pgx_problem* problem, uint32_t flags, int64_t* out);

/* Bytes of device memory the problem actually holds (equals
 * pgx_workspace_bytes of its descriptor up to small per-buffer rounding). */
size_t pgx_problem_bytes(pgx_problem* problem);

/* Which kernel family pgx_eval runs for this problem (fixed at creation):
 * PGX_PATH_GENERAL (fp64 CUDA-core kernels over any point list; the exact
 * mode, and the fallback of the fast modes where the grid paths do not
 * apply), PGX_PATH_GRID_FP64 (separable regular-grid kernels) or
 * PGX_PATH_GRID_TC (tcgen05 regular-grid kernels). */
enum { PGX_PATH_GENERAL = 0, PGX_PATH_GRID_FP64 = 1, PGX_PATH_GRID_TC = 2 };
int pgx_problem_path(pgx_problem* problem);

/* ---- Device-resident optimiser state.
 * The fit loop of the reference (optimizer.py:195-342: L-BFGS two-loop
 * recursion, strong-Wolfe line search, gauge fixing by the zero last column)
 * keeps its decisions on the host; these calls keep its VECTORS on the GPU: the
 * free parameters u = theta[:, :N-1], the gradient, the search direction and
 * the (s, y) history.  Each call returns a handful of scalars.  A line-search
 * trial (u + t d -> theta, pgx_eval, g_t . d) replays one captured CUDA graph.
 * All reductions are fixed-order: identical inputs give identical trajectories.
 *
 * pgx_lbfgs_start   u <- theta[:, :N-1] (theta: K x N fp64, host), history cleared, evaluate:
 *                   out[0..6] = {Phi, 0, err, e0, n_nonfinite, stats flags, |g|^2}
 * pgx_lbfgs_restart re-evaluate the current point at a new eps (annealing); history cleared
 * pgx_lbfgs_direction mode 0: d = two-loop(g) (optimizer.py:253-269; g/|g|^2 without history),
 *                   1: d = g/|g|^2, 2: d = g; out[0..3] = {g.d, |d|^2, |g|^2, pairs used}
 * pgx_lbfgs_trial   evaluate at u + t d: out[0..6] = {Phi, g_t.d, err, e0, n_nonfinite, flags, |g_t|^2}
 * pgx_lbfgs_accept  the LAST trial point becomes current; with keep_pair the pair
 *                   s = u_t - u, y = g - g_t joins the history when
 *                   s.y > 1e-10 |s| |y| (optimizer.py:303-309);
 *                   out[0..3] = {|g|^2, pushed (0/1), |u|^2, s.y}
 * pgx_lbfgs_theta   the current point as a K x N fp64 host matrix (last column zero)
 * pgx_lbfgs_iterate one iteration's device work in ONE submission and synchronisation:
 *                   [accept the last trial when keep_pair >= 0] -> two-loop direction ->
 *                   trial at u + t0 d; out[0..3] accept, out[4..7] direction, out[8..14]
 *                   trial scalars (each laid out as in the single calls) */
typedef struct pgx_lbfgs pgx_lbfgs;
pgx_status pgx_lbfgs_create(pgx_problem* problem, int memory, pgx_lbfgs** out);
void pgx_lbfgs_destroy(pgx_lbfgs* state);
pgx_status pgx_lbfgs_start(pgx_lbfgs* state, const double* theta, double eps, double lambda, double* out);
pgx_status pgx_lbfgs_restart(pgx_lbfgs* state, double eps, double lambda, double* out);
pgx_status pgx_lbfgs_clear(pgx_lbfgs* state);
pgx_status pgx_lbfgs_direction(pgx_lbfgs* state, int mode, double* out);
pgx_status pgx_lbfgs_trial(pgx_lbfgs* state, double t, double eps, double lambda, double* out);
pgx_status pgx_lbfgs_accept(pgx_lbfgs* state, int keep_pair, double* out);
pgx_status pgx_lbfgs_theta(pgx_lbfgs* state, double* theta_out);
pgx_status pgx_lbfgs_iterate(pgx_lbfgs* state, int keep_pair, double t0, double eps, double lambda,
                             double* out);

/* Number of kernel launches the last pgx_eval / pgx_assign enqueued. */
int pgx_last_launch_count(pgx_problem* problem);

/* Kernel-level timing (for bench.py's roofline): when enabled, every kernel
 * a call enqueues is bracketed by CUDA events on the problem's stream. */
pgx_status pgx_set_profiling(pgx_problem* problem, int enable);
/* Number of timed kernels of the last call; name and duration (ms) of the
 * i-th (pgx_profile_ms synchronises on its end event). */
int pgx_profile_count(pgx_problem* problem);
const char* pgx_profile_name(pgx_problem* problem, int i);
float pgx_profile_ms(pgx_problem* problem, int i);

/* Waits for all work enqueued on the problem's stream. */
pgx_status pgx_synchronize(pgx_problem* problem);

#ifdef __cplusplus
}
#endif

#endif /* PGX_H */
