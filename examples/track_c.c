/* A plain C program using only include/phd.h and libphd.so: a small tracking
 * run (3 targets on CV tracks, position sensor with clutter, the BASELINE cfg-1
 * model), phd_step per scan, printing the extracted estimates against truth.
 * It shows the ABI without Python: parameters, create, population, step,
 * estimates, errors, destroy.  Exit code 0 if every target is tracked within
 * 50 m at the last scan.
 *
 *   cc -O2 -I include examples/track_c.c -L paper_1503_03769_b200/lib -lphd \
 *      -Wl,-rpath,$PWD/paper_1503_03769_b200/lib -lm -o track_c && ./track_c
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "phd.h"

#define NT 3        /* targets */
#define STEPS 25
#define MAXM 64

static uint64_t rng = 88172645463325252ull;
static double urand(void) { /* xorshift64*, uniform (0, 1) */
  rng ^= rng >> 12;
  rng ^= rng << 25;
  rng ^= rng >> 27;
  return ((rng * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0) + 1e-17;
}
static double nrand(void) { return sqrt(-2.0 * log(urand())) * cos(2.0 * M_PI * urand()); }

static int check(phd_ctx* c, phd_status s, const char* what) {
  if (s == PHD_OK) return 0;
  fprintf(stderr, "%s: %s (%s)\n", what, phd_status_str(s), c ? phd_last_error(c) : "");
  return 1;
}

int main(void) {
  phd_params p;
  memset(&p, 0, sizeof p);
  p.abi_version = PHD_ABI_VERSION;
  p.meas = PHD_MEAS_POSITION;
  p.T = 1.0;
  p.sigma_a = 5.0;
  p.p_s = 0.99;
  p.p_d = 0.98;
  p.sigma_z[0] = p.sigma_z[1] = 10.0;
  p.region[0] = -1000.0;
  p.region[1] = 1000.0;
  p.region[2] = -1000.0;
  p.region[3] = 1000.0;
  p.clutter_rate = 10.0;
  p.birth_mass = 0.1;
  p.birth_sigma_v = 10.0;
  p.births_per_step = 200;
  p.particles_per_target = 500;
  p.count_mode = PHD_COUNT_ADAPTIVE;
  p.max_meas = MAXM;
  p.capacity = 1 << 15;
  p.seed = 1;
  p.mode = PHD_MODE_EXACT;

  phd_ctx* c = NULL;
  if (check(NULL, phd_create(&p, 0, 1, NULL, 0, NULL, NULL, &c), "phd_create")) return 2;

  /* initial population: 1500 particles uniform over the region, total mass 1 */
  const int64_t n0 = 1500;
  float* soa = (float*)malloc(sizeof(float) * 4 * n0);
  for (int64_t i = 0; i < n0; ++i) {
    soa[0 * n0 + i] = (float)(-1000.0 + 2000.0 * urand());
    soa[1 * n0 + i] = (float)(40.0 * urand() - 20.0);
    soa[2 * n0 + i] = (float)(-1000.0 + 2000.0 * urand());
    soa[3 * n0 + i] = (float)(40.0 * urand() - 20.0);
  }
  if (check(c, phd_set_particles(c, soa, NULL, n0, n0, 1.0, PHD_STAGE_RESAMPLED), "phd_set_particles")) return 2;

  double tx[NT], tvx[NT], ty[NT], tvy[NT];
  for (int t = 0; t < NT; ++t) {
    tx[t] = -600.0 + 600.0 * t;
    ty[t] = -300.0 + 250.0 * t;
    tvx[t] = 12.0 - 6.0 * t;
    tvy[t] = 8.0;
  }
  float z[MAXM * 2];
  phd_estimate est[MAXM];
  phd_summary sum;
  int n_est = 0;
  for (int k = 1; k <= STEPS; ++k) {
    int M = 0;
    for (int t = 0; t < NT; ++t) {
      tx[t] += tvx[t] + 0.5 * 5.0 * nrand();
      tvx[t] += 5.0 * nrand() * 0.2;
      ty[t] += tvy[t] + 0.5 * 5.0 * nrand();
      tvy[t] += 5.0 * nrand() * 0.2;
      if (urand() < p.p_d) {
        z[2 * M] = (float)(tx[t] + 10.0 * nrand());
        z[2 * M + 1] = (float)(ty[t] + 10.0 * nrand());
        ++M;
      }
    }
    for (int j = 0; j < 10 && M < MAXM; ++j, ++M) { /* clutter */
      z[2 * M] = (float)(-1000.0 + 2000.0 * urand());
      z[2 * M + 1] = (float)(-1000.0 + 2000.0 * urand());
    }
    if (check(c, phd_step(c, k, z, M, est, MAXM, &n_est, &sum), "phd_step")) return 2;
    printf("k=%2d M=%2d W=%6.3f LT=%lld N=%lld estimates:", k, M, sum.W, (long long)sum.LT, (long long)sum.N);
    for (int e = 0; e < n_est; ++e) printf(" (%.0f, %.0f)", est[e].state[0], est[e].state[2]);
    printf("\n");
  }
  /* every target has an estimate within 50 m at the last scan */
  int ok = 1;
  for (int t = 0; t < NT; ++t) {
    double best = 1e30;
    for (int e = 0; e < n_est; ++e) {
      double dx = est[e].state[0] - tx[t], dy = est[e].state[2] - ty[t];
      best = fmin(best, sqrt(dx * dx + dy * dy));
    }
    printf("target %d at (%.0f, %.0f): nearest estimate %.1f m\n", t, tx[t], ty[t], best);
    ok = ok && best < 50.0;
  }
  /* an error case: an update out of order is refused with PHD_ESTATE */
  phd_status st = phd_update(c, z, 1);
  printf("phd_update out of order -> %s\n", phd_status_str(st));
  ok = ok && st == PHD_ESTATE;
  phd_destroy(c);
  free(soa);
  return ok ? 0 : 1;
}
