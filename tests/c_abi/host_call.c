/* The C-ABI from plain C (C11): what a reference-side binding (cgo, ctypes, a
 * C extension) compiles against.  Built and linked by tests/test_lib.py on the
 * CPU; run on a GPU box it evaluates the config-3 volume term of a few seeded
 * elements from host buffers and prints one checksum. */
#include <stdio.h>
#include <stdlib.h>

#include "sumfac_b200.h"

int main(void) {
  const int64_t E = 3, n = 4, nodes = 64;
  /* GLL D for n = 4 (operators.py:136-152 would build it; any n x n works) */
  const double D[16] = {-3.0, 4.04508497187474, -1.54508497187474, 0.5,
                        -0.809016994374947, 0.0, 1.11803398874989, -0.309016994374947,
                        0.309016994374947, -1.11803398874989, 0.0, 0.809016994374947,
                        -0.5, 1.54508497187474, -4.04508497187474, 3.0};
  double* U = malloc(sizeof(double) * E * 5 * nodes);
  double* R = malloc(sizeof(double) * E * 5 * nodes);
  for (int64_t e = 0; e < E; ++e)
    for (int64_t r = 0; r < nodes; ++r) {
      double rho = 1.0 + 0.01 * (double)((r * 7 + e) % 11), v = 0.05, p = 1.0;
      U[(e * 5 + 0) * nodes + r] = rho;
      U[(e * 5 + 1) * nodes + r] = rho * v;
      U[(e * 5 + 2) * nodes + r] = 0.0;
      U[(e * 5 + 3) * nodes + r] = 0.0;
      U[(e * 5 + 4) * nodes + r] = p / 0.4 + 0.5 * rho * v * v;
    }
  int rc = sfb_euler_volume_cartesian_host(E, n, D, 1.4, 2.0, U, R);
  if (rc != SFB_OK) {
    fprintf(stderr, "sfb_euler_volume_cartesian_host: %d %s\n", rc, sfb_last_error());
    return 1;
  }
  double s = 0.0;
  for (int64_t i = 0; i < E * 5 * nodes; ++i) s += R[i] * R[i];
  printf("ok %d %.17g\n", sfb_version(), s);
  free(U);
  free(R);
  return 0;
}
