/* A plain C99 consumer of include/pgx.h: what a non-Python host (or a cgo / JNI
 * stub) links against.  Builds a 128 x 128 problem with N = 4 grains (labels =
 * quadrant index), evaluates Phi + gradient + assignment at theta = 0 in the
 * requested precision, and prints the scalars.  At theta = 0 every grain ties:
 * Phi = -log N exactly, the arg-min is grain 1 everywhere (smallest index), so
 * err = 3/4, and the gradient columns sum to zero.
 *   gcc -std=c99 -I include tests/c_abi/abi_smoke.c -L paper_2605_20816_b200/lib -lpgx -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pgx.h"

int main(int argc, char** argv) {
  const int prec = argc > 1 ? atoi(argv[1]) : PGX_PREC_TC;
  const int M = 64, side = 2 * M, N = 4, K = 3;
  int64_t* labels0 = (int64_t*)malloc(sizeof(int64_t) * side * side);
  for (int a = 0; a < side; ++a)
    for (int b = 0; b < side; ++b) labels0[a * side + b] = 2 * (a >= M) + (b >= M);
  pgx_desc d;
  memset(&d, 0, sizeof d);
  d.dim = 2;
  d.basis_kind = PGX_BASIS_LEGENDRE;
  d.degree = 1;
  d.n_grains = N;
  d.n_points = (int64_t)side * side;
  d.resolution = M;
  d.precision = prec;
  d.labels0 = labels0;
  pgx_problem* pb = NULL;
  if (pgx_problem_create(&d, &pb) != PGX_OK) {
    fprintf(stderr, "create failed: %s\n", pgx_last_error());
    return 2;
  }
  double theta[3 * 4] = {0}, grad[3 * 4];
  pgx_stats st;
  if (pgx_eval(pb, theta, 0.05, 0.0, PGX_WANT_GRAD | PGX_WANT_ASSIGN, grad, &st) != PGX_OK) {
    fprintf(stderr, "eval failed: %s\n", pgx_last_error());
    return 3;
  }
  double colsum = 0.0;
  for (int k = 0; k < K; ++k)
    for (int i = 0; i < N; ++i) colsum += (k == 0 ? 1.0 : 0.0) * grad[k * N + i];
  int64_t* lab = (int64_t*)malloc(sizeof(int64_t) * side * side);
  if (pgx_assign(pb, theta, 0, lab, NULL, NULL) != PGX_OK) {
    fprintf(stderr, "assign failed: %s\n", pgx_last_error());
    return 4;
  }
  int64_t ones = 0;
  for (int64_t p = 0; p < d.n_points; ++p) ones += lab[p] == 1;
  printf("abi %d path %d phi %.15g err %.15g row0sum %.3e ones %lld\n", pgx_abi_version(), pgx_problem_path(pb),
         st.phi, st.err, colsum, (long long)ones);
  const int ok = fabs(st.phi + log((double)N)) < 1e-6 && fabs(st.err - 0.75) < 1e-12 && fabs(colsum) < 1e-9 &&
                 ones == d.n_points;
  pgx_problem_destroy(pb);
  free(labels0);
  free(lab);
  return ok ? 0 : 1;
}
