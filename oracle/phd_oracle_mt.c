/* TEST INFRASTRUCTURE, NOT PRODUCT CODE: the all-core CPU baseline (SURVEY.md
 * §8(d) "Oracle timing": the same oracle loops split over particles with
 * threads and a fixed-order fp64 reduction).  Timing only: orc_normalizers_mt
 * and orc_update_mt compute exactly orc_normalizers / orc_update of
 * phd_oracle.c (the per-particle arithmetic is the same calls; only the fp64
 * sums over particles are split into per-thread partials added in thread
 * order), pinned against them by tests/test_oracle_pins.py. */
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "phd_oracle.h"

typedef struct {
  const orc_model* m;
  int64_t i0, i1;
  const double *x, *vx, *y, *vy, *w, *z, *C;
  int32_t nz;
  double* part;  /* [nz] (normalizers) or [5 nz] (update) */
  double* w_out;
} mt_job;

static void* norm_job(void* arg) {
  mt_job* j = (mt_job*)arg;
  orc_normalizers(j->m, j->i1 - j->i0, j->x + j->i0, j->y + j->i0, j->w + j->i0, j->z, j->nz, j->part);
  return NULL;
}

static void* update_job(void* arg) {
  mt_job* j = (mt_job*)arg;
  orc_update(j->m, j->i1 - j->i0, j->x + j->i0, j->vx + j->i0, j->y + j->i0, j->vy + j->i0, j->w + j->i0, j->z,
             j->nz, j->C, j->w_out + j->i0, j->part);
  return NULL;
}

static void run(int nt, mt_job* jobs, void* (*fn)(void*)) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, fn, &jobs[t]);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(th);
}

void orc_normalizers_mt(const orc_model* m, int64_t n, const double* x, const double* y, const double* w,
                        const double* z, int32_t nz, double* C, int32_t nthreads) {
  int nt = nthreads < 1 ? 1 : nthreads;
  mt_job* jobs = (mt_job*)calloc((size_t)nt, sizeof(mt_job));
  double* part = (double*)calloc((size_t)nt * (size_t)(nz > 0 ? nz : 1), sizeof(double));
  for (int t = 0; t < nt; ++t) {
    jobs[t].m = m;
    jobs[t].i0 = n * t / nt;
    jobs[t].i1 = n * (t + 1) / nt;
    jobs[t].x = x;
    jobs[t].y = y;
    jobs[t].w = w;
    jobs[t].z = z;
    jobs[t].nz = nz;
    jobs[t].part = part + (size_t)t * nz;
  }
  run(nt, jobs, norm_job);
  for (int32_t p = 0; p < nz; ++p) {
    double s = 0.0;
    for (int t = 0; t < nt; ++t) s += part[(size_t)t * nz + p];
    C[p] = s;
  }
  free(part);
  free(jobs);
}

void orc_update_mt(const orc_model* m, int64_t n, const double* x, const double* vx, const double* y,
                   const double* vy, const double* w, const double* z, int32_t nz, const double* C,
                   double* w_out, double* acc, int32_t nthreads) {
  int nt = nthreads < 1 ? 1 : nthreads;
  mt_job* jobs = (mt_job*)calloc((size_t)nt, sizeof(mt_job));
  double* part = (double*)calloc((size_t)nt * 5 * (size_t)(nz > 0 ? nz : 1), sizeof(double));
  for (int t = 0; t < nt; ++t) {
    jobs[t].m = m;
    jobs[t].i0 = n * t / nt;
    jobs[t].i1 = n * (t + 1) / nt;
    jobs[t].x = x;
    jobs[t].vx = vx;
    jobs[t].y = y;
    jobs[t].vy = vy;
    jobs[t].w = w;
    jobs[t].z = z;
    jobs[t].C = C;
    jobs[t].nz = nz;
    jobs[t].part = part + (size_t)t * 5 * nz;
    jobs[t].w_out = w_out;
  }
  run(nt, jobs, update_job);
  for (int32_t q = 0; q < 5 * nz; ++q) {
    double s = 0.0;
    for (int t = 0; t < nt; ++t) s += part[(size_t)t * 5 * nz + q];
    acc[q] = s;
  }
  free(part);
  free(jobs);
}
