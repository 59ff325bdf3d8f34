/* abi_smoke.c — a plain C host of libfabm.so (include/fabm.h), as a
 * non-Python binding of the reference's solver call would use it: one
 * fabm_solve of the fractional Lorenz system (weights generated on the
 * device), then the CSV of the trajectory through fabm_format_csv.
 * Prints y_N with 17 significant digits and the CSV byte count; with a
 * directory argument also writes states.bin (raw doubles) and traj.csv.
 *   gcc -std=c99 -I include tests/c/abi_smoke.c -L paper_1611_08678_b200 -lfabm -o abi_smoke */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fabm.h"

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 20000;
  fabm_problem p;
  memset(&p, 0, sizeof(p));
  p.alpha = 0.99;
  p.dim = 3;
  p.system = FABM_SYS_LORENZ;
  p.params[0] = 10.0;
  p.params[1] = 28.0;
  p.params[2] = 8.0 / 3.0;
  p.y0[0] = p.y0[1] = p.y0[2] = 1.0;
  fabm_grid g;
  memset(&g, 0, sizeof(g)); /* zero scalars: filled by the library */
  g.n_steps = n;
  g.h = 1e-3;
  double* Y = malloc(sizeof(double) * 3 * (size_t)(n + 1));
  double* F = malloc(sizeof(double) * 3 * (size_t)(n + 1));
  fabm_status st;
  int rc = fabm_solve(&p, &g, FABM_WEIGHTS_ACCURATE, NULL, NULL, NULL, Y, F, &st);
  if (rc != FABM_OK) {
    fprintf(stderr, "fabm_solve: %d %s (step %lld)\n", rc, st.message, (long long)st.step);
    return 1;
  }
  printf("y_N %.17g %.17g %.17g\n", Y[3 * n], Y[3 * n + 1], Y[3 * n + 2]);
  int64_t need = 0;
  rc = fabm_format_csv(Y, NULL, n + 1, 3, g.h, 0, NULL, 0, &need, NULL, &st);
  if (rc != FABM_ERR_CONFIG || need <= 0) {
    fprintf(stderr, "fabm_format_csv size query: %d\n", rc);
    return 1;
  }
  char* out = malloc((size_t)need);
  int64_t got = 0;
  rc = fabm_format_csv(Y, NULL, n + 1, 3, g.h, 0, out, need, &got, NULL, &st);
  if (rc != FABM_OK || got != need) {
    fprintf(stderr, "fabm_format_csv: %d %s\n", rc, st.message);
    return 1;
  }
  printf("csv_bytes %lld\n", (long long)got);
  if (argc > 2) {
    char path[4096];
    snprintf(path, sizeof(path), "%s/states.bin", argv[2]);
    FILE* fh = fopen(path, "wb");
    if (!fh || fwrite(Y, sizeof(double), 3 * (size_t)(n + 1), fh) != 3 * (size_t)(n + 1)) return 1;
    fclose(fh);
    snprintf(path, sizeof(path), "%s/traj.csv", argv[2]);
    fh = fopen(path, "wb");
    if (!fh || fwrite(out, 1, (size_t)got, fh) != (size_t)got) return 1;
    fclose(fh);
  }
  printf("version %s\n", fabm_version());
  free(out);
  free(Y);
  free(F);
  return 0;
}
