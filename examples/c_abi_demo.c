/* Plain-C consumer of include/lattdse_c.h (the drop-in boundary).
 * Build: gcc -std=c11 -I include examples/c_abi_demo.c \
 *        -L paper_1808_06357_b200 -llattdse_b200 -Wl,-rpath,$PWD/paper_1808_06357_b200 -o c_abi_demo
 * Run:   ./c_abi_demo            (lattice + CBC + anti-aliasing, CPU only)
 *        ./c_abi_demo --gpu      (also a 64-step Strang propagation on device 0)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lattdse_c.h"

#define CHECK(x)                                                                    \
  do {                                                                              \
    int rc_ = (x);                                                                  \
    if (rc_) {                                                                      \
      fprintf(stderr, "%s -> %d: %s\n", #x, rc_, lattdse_last_error());             \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

int main(int argc, char** argv) {
  int gpu = argc > 1 && strcmp(argv[1], "--gpu") == 0;
  /* reference Fig. 1 lattice: hash from the reference's own lattice.cpp */
  int64_t z55[2] = {1, 34};
  lattdse_lattice* fig1;
  CHECK(lattdse_lattice_rank1(z55, 2, 55, &fig1));
  uint64_t h;
  CHECK(lattdse_lattice_hash(fig1, &h));
  char js[256];
  CHECK(lattdse_lattice_to_json(fig1, js, sizeof js, NULL));
  printf("fig1 hash=0x%016llx json=%s\n", (unsigned long long)h, js);
  if (h != 0xc52fc32f65226f72ULL) return 2;
  /* error mapping: non_divisible_moduli = code 2 */
  int64_t eye[4] = {1, 0, 0, 1}, bad[2] = {4, 8};
  lattdse_lattice* tmp;
  int rc = lattdse_lattice_create(2, 2, eye, bad, &tmp);
  printf("grid(4,8) -> %d (%s)\n", rc, lattdse_last_error());
  if (rc != 2) return 3;

  /* config-0 lattice: prime-n CBC + anti-aliasing norms */
  const int64_t n = 4099;
  int64_t z[2];
  double w[2];
  CHECK(lattdse_cbc_construct(n, 2, z, w));
  lattdse_lattice* lat;
  CHECK(lattdse_lattice_rank1(z, 2, n, &lat));
  uint32_t* norm2 = malloc(sizeof(uint32_t) * n);
  uint32_t mx = 0;
  CHECK(lattdse_aaset_build(lat, -1.0, norm2, NULL, &mx));
  printf("C0 z=(%lld,%lld) max|h|^2=%u\n", (long long)z[0], (long long)z[1], mx);

  if (gpu) {
    double a[2], b[1], c[2];
    int p[2];
    CHECK(lattdse_problem_draw(0x180806357ULL, 2, 1, 0.4, 0.6, 2, a, b, c, p));
    lattdse_problem prob = {0.1, 2, a, b, 1, 0.1, c, p};
    lattdse_solver* s;
    CHECK(lattdse_solver_create_with_norms(lat, norm2, &prob, NULL, &s));
    CHECK(lattdse_solver_set_dt(s, 1.0 / 256));
    CHECK(lattdse_solver_discretize_initial(s));
    CHECK(lattdse_solver_step(s, 64));
    double nrm, en;
    CHECK(lattdse_solver_l2_norm(s, &nrm));
    CHECK(lattdse_solver_energy(s, &en));
    printf("64 Strang steps: |u|-1=%.3e energy=%.12f\n", nrm - 1.0, en);
    lattdse_solver_destroy(s);
    if (fabs(nrm - 1.0) > 1e-12) return 4;
  }
  lattdse_lattice_destroy(lat);
  lattdse_lattice_destroy(fig1);
  free(norm2);
  printf("ok\n");
  return 0;
}
