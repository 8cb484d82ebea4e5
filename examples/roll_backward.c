/* Minimal C client of the heterodyn ABI: the reference's roll + chain_backward
 * (drivers.cpp:31-99) through the B200 library.  Build:
 *   gcc -O2 -I include examples/roll_backward.c \
 *       -L paper_2605_14526_b200/_lib -lheterodyn_b200 \
 *       -Wl,-rpath,$PWD/paper_2605_14526_b200/_lib -o roll_backward
 * Usage: roll_backward [builtin-scene-name] [frames]
 * Prints the final-state norm and |dL/dq0| for L = 1/2 |q_T|^2. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "heterodyn.h"

static int fail(const char* what) {
  fprintf(stderr, "%s: %s (code %d)\n", what, hd_last_error(), hd_last_error_code());
  return 1;
}

int main(int argc, char** argv) {
  const char* name = argc > 1 ? argv[1] : "cantilever3";
  int frames = argc > 2 ? atoi(argv[2]) : 5;
  hd_scene* scene = hd_scene_builtin(name);
  if (!scene) return fail("hd_scene_builtin");
  hd_sim* sim = hd_sim_create(scene);
  if (!sim) return fail("hd_sim_create");
  int dof = hd_sim_dof_count(sim);
  double* q = malloc(sizeof(double) * dof);
  double* g = malloc(sizeof(double) * dof);
  if (hd_sim_record(sim, 1) != HD_OK) return fail("hd_sim_record");
  for (int f = 0; f < frames; ++f)
    if (hd_sim_step(sim) != HD_OK) return fail("hd_sim_step");
  if (hd_sim_positions(sim, q, dof) != HD_OK) return fail("hd_sim_positions");
  double nq = 0, ng = 0;
  for (int i = 0; i < dof; ++i) nq += q[i] * q[i];
  /* dL/dq_T = q_T for L = 1/2 |q_T|^2 */
  if (hd_sim_backward(sim, NULL, q, NULL, g, NULL, NULL, NULL, NULL, 0) != HD_OK)
    return fail("hd_sim_backward");
  for (int i = 0; i < dof; ++i) ng += g[i] * g[i];
  printf("scene=%s frames=%d iterations=%d |q_T|=%.12e |dL/dq0|=%.12e adjoint_sweeps=%d\n", name, frames,
         hd_sim_last_iterations(sim), sqrt(nq), sqrt(ng), hd_sim_backward_iterations(sim));
  free(q);
  free(g);
  hd_sim_free(sim);
  hd_scene_free(scene);
  return 0;
}
