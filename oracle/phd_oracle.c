/* oracle/phd_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain single-threaded fp64 reference of one particle-PHD filter step,
 * written from the paper (arXiv 1503.03769; /root/reference/PAPER.md) in the
 * paper's order and notation.  No blocking, fusion or reordering: every sum
 * is a straight loop in index order.  Readings of garbled or silent passages
 * are the ones listed in DESIGN.md §2 (S1..S27 of SURVEY.md §8(c)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
 * reference arm) may load this library.  The CUDA product path never does.
 */
#include "phd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double ORC_PI = 3.14159265358979323846264338327950288;

/* ---------------------------------------------------------------------- */
/* Counter-based noise (DESIGN.md §2 "noise"): Philox4x32-10 (Salmon, Moraes,
 * Dror, Shaw, SC'11).  Each round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 * c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); the key is bumped between rounds. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

double orc_conv23(uint32_t w) { return ((double)(w >> 9) + 0.5) * ldexp(1.0, -23); }

double orc_u52(uint32_t w0, uint32_t w1) {
  return ((double)(w0 >> 6) * ldexp(1.0, 26) + (double)(w1 >> 6) + 0.5) * ldexp(1.0, -52);
}

void orc_box_muller(double u1, double u2, double* n1, double* n2) {
  double rad = sqrt(-2.0 * log(u1));
  *n1 = rad * cos(2.0 * ORC_PI * u2);
  *n2 = rad * sin(2.0 * ORC_PI * u2);
}

static void philox_at(const orc_model* m, uint64_t g, int32_t k, uint32_t stream, uint32_t out[4]) {
  uint32_t ctr[4] = {(uint32_t)g, (uint32_t)k, stream, (uint32_t)(g >> 32)};
  uint32_t key[2] = {(uint32_t)m->seed, (uint32_t)(m->seed >> 32)};
  orc_philox4x32_10(ctr, key, out);
}

/* ---------------------------------------------------------------------- */
/* 0) Initialisation ("t=0: Generate M particles for each group. The
 * number of all particles is N. All these particles are shared with same weights
 * omega_0 = 1/M"), with the reading S23 of SURVEY.md §8(c): the population of
 * n_out particles is index-stratified in y over box = (x0, x1, y0, y1),
 *   y_g = y0 + (y1 - y0) (g + u0) / n_out,  x_g = x0 + (x1 - x0) u1,
 *   (vx, vy) = v_max (2 u2 - 1, 2 u3 - 1),
 * u_c = conv23 of word c of Philox({g, 0, 5, g >> 32}) (stream 5, step 0); every
 * state is rounded to fp32, the precision the filter stores it in.  Particles
 * g_lo .. g_hi-1 are generated (one group or the whole population); their weights
 * share total_mass equally (omega_0 = mass / M), or, with a mass box, equally among
 * the generated particles whose stored (fp32) position lies inside it (closed box),
 * 0 elsewhere.  No particle inside: every weight 0.  Returns the inside count. */
int64_t orc_init_population(const orc_model* m, int64_t n_out, int64_t g_lo, int64_t g_hi, const double box[4],
                            double v_max, double total_mass, const double* mass_box, double* x, double* vx,
                            double* y, double* vy, double* w) {
  int64_t n = g_hi - g_lo, inside = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t g = g_lo + i;
    uint32_t ctr[4] = {(uint32_t)g, 0u, 5u, (uint32_t)((uint64_t)g >> 32)};
    uint32_t key[2] = {(uint32_t)m->seed, (uint32_t)(m->seed >> 32)};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    double u0 = orc_conv23(o[0]), u1 = orc_conv23(o[1]), u2 = orc_conv23(o[2]), u3 = orc_conv23(o[3]);
    y[i] = (double)(float)(box[2] + (box[3] - box[2]) * ((double)g + u0) / (double)n_out);
    x[i] = (double)(float)(box[0] + (box[1] - box[0]) * u1);
    vx[i] = (double)(float)(v_max * (2.0 * u2 - 1.0));
    vy[i] = (double)(float)(v_max * (2.0 * u3 - 1.0));
    if (mass_box && x[i] >= mass_box[0] && x[i] <= mass_box[1] && y[i] >= mass_box[2] && y[i] <= mass_box[3])
      ++inside;
  }
  if (!mass_box) inside = n;
  for (int64_t i = 0; i < n; ++i) {
    int in = !mass_box ||
             (x[i] >= mass_box[0] && x[i] <= mass_box[1] && y[i] >= mass_box[2] && y[i] <= mass_box[3]);
    w[i] = (in && inside > 0) ? (double)(float)(total_mass / (double)inside) : 0.0;
  }
  return inside;
}

/* ---------------------------------------------------------------------- */
/* Models (§4). */

/* kappa_k(z) = lambda_k V u(z), read as the uniform clutter
 * intensity lambda / V over the measurement region, constant in z (S17). */
double orc_kappa(const orc_model* m) {
  double V = (m->region[1] - m->region[0]) * (m->region[3] - m->region[2]);
  return m->clutter_rate / V;
}

/* Wrap an angle difference into (-pi, pi] (S15). */
static double wrap_pi(double d) {
  while (d > ORC_PI) d -= 2.0 * ORC_PI;
  while (d <= -ORC_PI) d += 2.0 * ORC_PI;
  return d;
}

/* g_k(z | x): position sensor z = (x, y) + v, or the range-bearing sensor
 * z = (R, theta) + v, R = sqrt((x-s_x)^2 + (y-s_y)^2),
 * theta = arctan((y-s_y)/(x-s_x)) taken as atan2 with a
 * wrapped residual (S15); v ~ N(0, diag(sigma_z^2)) (S16). */
double orc_likelihood(const orc_model* m, double z0, double z1, double x, double y) {
  double s0 = m->sigma_z[0], s1 = m->sigma_z[1];
  double d0, d1;
  if (m->meas == 0) {
    d0 = z0 - x;
    d1 = z1 - y;
  } else {
    double px = x - m->sensor[0], py = y - m->sensor[1];
    double R = sqrt(px * px + py * py);
    double th = (px == 0.0 && py == 0.0) ? 0.0 : atan2(py, px);
    d0 = z0 - R;
    d1 = wrap_pi(z1 - th);
  }
  double e = d0 * d0 / (2.0 * s0 * s0) + d1 * d1 / (2.0 * s1 * s1);
  return exp(-e) / (2.0 * ORC_PI * s0 * s1);
}

/* ---------------------------------------------------------------------- */
/* N(a; mu, sd^2) on the real line. */
static double normal1(double a, double mu, double sd) {
  double t = (a - mu) / sd;
  return exp(-0.5 * t * t) / (sqrt(2.0 * ORC_PI) * sd);
}

/* 1) Prediction (§2.2 step 1, Eq 5; Algorithm 1).
 * The transition is the CV model x' = F x + G w_k with
 * w_k = sigma_a (n1, n2), n from Box-Muller of Philox({g, k, 1, g>>32}).
 * q_k is the same CV model with noise std s sigma_a (s = proposal_scale; s = 1
 * is the transition prior of S10).  phi_{k|k-1}(x, x') = e_{k|k-1} f(x|x')
 * (no spawning), so Eq 5 gives w~ = p_s f(x|x') / q(x|x') w.  f and q are both
 * carried by the plane x = F x' + G a, so their ratio is the ratio of the noise
 * densities N(a; 0, sigma_a^2 I) / N(a; 0, s^2 sigma_a^2 I) at the drawn a. */
void orc_predict(const orc_model* m, int32_t k, int64_t n, int64_t g0,
                 double* x, double* vx, double* y, double* vy, double* w) {
  double T = m->T;
  double s = m->proposal_scale > 0.0 ? m->proposal_scale : 1.0;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t o[4];
    philox_at(m, (uint64_t)(g0 + i), k, 1u, o);
    double n1, n2;
    orc_box_muller(orc_conv23(o[0]), orc_conv23(o[1]), &n1, &n2);
    double ax = s * m->sigma_a * n1, ay = s * m->sigma_a * n2;
    double ratio = 1.0;
    if (s != 1.0 && m->sigma_a > 0.0) {
      double f = normal1(ax, 0.0, m->sigma_a) * normal1(ay, 0.0, m->sigma_a);
      double q = normal1(ax, 0.0, s * m->sigma_a) * normal1(ay, 0.0, s * m->sigma_a);
      ratio = f / q;
    }
    double x1 = x[i] + T * vx[i] + 0.5 * T * T * ax;
    double vx1 = vx[i] + T * ax;
    double y1 = y[i] + T * vy[i] + 0.5 * T * T * ay;
    double vy1 = vy[i] + T * ay;
    x[i] = x1;
    vx[i] = vx1;
    y[i] = y1;
    vy[i] = vy1;
    w[i] = m->p_s * ratio * w[i];
  }
}

/* Eq 6 (Algorithm 1; Step 1 line 266):
 * J_k births drawn from p_k(.|Z) -- measurement-driven around Z_{k-1} (S10),
 * uniform over the region when no previous measurement exists -- each with
 * weight gamma / J_k (importance ratio read as 1, S10).  Birth b uses
 * measurement b mod M_{k-1} and the four normals of Philox({n_out+b, k, 2, .}).
 * birth_model 2 draws the same way; orc_birth_is_weights then replaces the
 * weights by the full Eq 6 ratio. */
void orc_births(const orc_model* m, int32_t k, int64_t n_out, int64_t J, int64_t b0, int64_t nb,
                const double* zprev, int32_t m_prev,
                double* x, double* vx, double* y, double* vy, double* w) {
  for (int64_t i = 0; i < nb; ++i) {
    int64_t b = b0 + i;
    uint32_t o[4];
    philox_at(m, (uint64_t)(n_out + b), k, 2u, o);
    double u0 = orc_conv23(o[0]), u1 = orc_conv23(o[1]);
    double u2 = orc_conv23(o[2]), u3 = orc_conv23(o[3]);
    double n1, n2, n3, n4;
    orc_box_muller(u0, u1, &n1, &n2);
    orc_box_muller(u2, u3, &n3, &n4);
    if (m->birth_model == 1) {
      /* births from the normal density N(x-bar, Q), Q diagonal */
      x[i] = m->birth_mean[0] + m->birth_std[0] * n1;
      vx[i] = m->birth_mean[1] + m->birth_std[1] * n2;
      y[i] = m->birth_mean[2] + m->birth_std[2] * n3;
      vy[i] = m->birth_mean[3] + m->birth_std[3] * n4;
      w[i] = m->birth_mass / (double)J;
      continue;
    }
    double a, c;
    if (m_prev > 0) {
      const double* z = zprev + 2 * (b % m_prev);
      a = z[0] + m->sigma_z[0] * n1;
      c = z[1] + m->sigma_z[1] * n2;
    } else {
      a = m->region[0] + (m->region[1] - m->region[0]) * u0;
      c = m->region[2] + (m->region[3] - m->region[2]) * u1;
    }
    if (m->meas == 0) {
      x[i] = a;
      y[i] = c;
    } else { /* invert the range-bearing sensor (S27) */
      x[i] = m->sensor[0] + a * cos(c);
      y[i] = m->sensor[1] + a * sin(c);
    }
    vx[i] = m->birth_sigma_v * n3;
    vy[i] = m->birth_sigma_v * n4;
    w[i] = m->birth_mass / (double)J;
  }
}

/* Number of birth indices b in [0, e) with b mod M == c. */
static int64_t count_below(int64_t e, int64_t c, int64_t M) { return e > c ? (e - c - 1) / M + 1 : 0; }

/* Eq 6 with the full importance ratio: w = gamma(x) / (J p_k(x|Z)).
 * gamma(x) = birth_mass N(x; x-bar, Q) over (x, vx, y, vy).
 * p_k is the density the births [blo, blo+J) of this filter are drawn from: birth b
 * takes component c = b mod M_{k-1} deterministically, so p_k is the mixture
 * sum_c (n_c / J) q_c with n_c the number of those births using c (the balance-heuristic
 * estimator, unbiased for any n_c).  q_c = (position law) x N(vx; 0, sv^2) N(vy; 0, sv^2),
 * the position law being
 *   position sensor:      N(x; z_c0, s0^2) N(y; z_c1, s1^2);
 *   range-bearing sensor: (a, c) ~ N(z_c, diag(s0^2, s1^2)) mapped by (a cos c, a sin c),
 *     whose density at (x, y) is the sum over the preimages (r, th) and (-r, th + pi) of
 *     N(a; z_c0, s0^2) N(wrap(c - z_c1); 0, s1^2) / r (Jacobian |a| = r; bearing wrapped
 *     into (-pi, pi], the nearest 2 pi image);
 * with no previous measurements, uniform over the region: 1/V (position) or 1/(V r). */
void orc_birth_is_weights(const orc_model* m, int64_t J, int64_t blo, int64_t nb,
                          const double* zprev, int32_t m_prev, const double* x, const double* vx,
                          const double* y, const double* vy, double* w) {
  double V = (m->region[1] - m->region[0]) * (m->region[3] - m->region[2]);
  for (int64_t i = 0; i < nb; ++i) {
    double r = 0.0, th = 0.0;
    if (m->meas != 0) {
      double px = x[i] - m->sensor[0], py = y[i] - m->sensor[1];
      r = sqrt(px * px + py * py);
      th = (px == 0.0 && py == 0.0) ? 0.0 : atan2(py, px);
    }
    double pos = 0.0;
    if (m_prev > 0) {
      for (int32_t c = 0; c < m_prev; ++c) {
        int64_t n_c = count_below(blo + J, c, m_prev) - count_below(blo, c, m_prev);
        if (n_c == 0) continue;
        const double* z = zprev + 2 * c;
        double q;
        if (m->meas == 0) {
          q = normal1(x[i], z[0], m->sigma_z[0]) * normal1(y[i], z[1], m->sigma_z[1]);
        } else {
          double qa = normal1(r, z[0], m->sigma_z[0]) * normal1(wrap_pi(th - z[1]), 0.0, m->sigma_z[1]);
          double qb = normal1(-r, z[0], m->sigma_z[0]) * normal1(wrap_pi(th + ORC_PI - z[1]), 0.0, m->sigma_z[1]);
          q = (qa + qb) / r;
        }
        pos += (double)n_c / (double)J * q;
      }
    } else {
      pos = m->meas == 0 ? 1.0 / V : 1.0 / (V * r);
    }
    double p = pos * normal1(vx[i], 0.0, m->birth_sigma_v) * normal1(vy[i], 0.0, m->birth_sigma_v);
    double g = m->birth_mass * normal1(x[i], m->birth_mean[0], m->birth_std[0]) *
               normal1(vx[i], m->birth_mean[1], m->birth_std[1]) *
               normal1(y[i], m->birth_mean[2], m->birth_std[2]) *
               normal1(vy[i], m->birth_mean[3], m->birth_std[3]);
    w[i] = p > 0.0 ? g / ((double)J * p) : 0.0;
  }
}

/* ---------------------------------------------------------------------- */
/* 2) Update (§2.2 step 2).
 * Eq 7 / Eq 11: C_k(z) = sum_j psi_{k,z}(x~_j) w~_j, psi = p_D g;
 * the printed "* x~" factor is read as a typo (S2); the sum runs over all
 * particles of all ranks (S3). */
void orc_normalizers(const orc_model* m, int64_t n, const double* x, const double* y,
                     const double* w, const double* z, int32_t nz, double* C) {
  for (int32_t p = 0; p < nz; ++p) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i)
      s += m->p_d * orc_likelihood(m, z[2 * p], z[2 * p + 1], x[i], y[i]) * w[i];
    C[p] = s;
  }
}

/* Eq 8 / Eqs 12-15: w_i = [nu + sum_p psi_p(x_i) / (kappa + C_p)] w~_i with
 * nu = 1 - p_D (S4); G^{i,p} = psi/(kappa+C) (Eq 12), dw^{i,p} = G w~ (Eq 13),
 * dw^{i,0} = nu w~ (Eq 14), w = sum_p dw^{i,p} + dw^{i,0} (Eq 15).
 * A measurement with kappa + C_p = 0 contributes 0.
 * Eq 16: dW_p = sum_i dw^{i,p}; Eq 18 numerators: S_p = sum_i dw^{i,p} x~_i.
 * acc[5p..5p+4] = (dW_p, S_p.x, S_p.vx, S_p.y, S_p.vy). */
void orc_update(const orc_model* m, int64_t n, const double* x, const double* vx,
                const double* y, const double* vy, const double* w,
                const double* z, int32_t nz, const double* C, double* w_out, double* acc) {
  double kappa = orc_kappa(m);
  double nu = 1.0 - m->p_d;
  memset(acc, 0, sizeof(double) * 5 * (size_t)nz);
  for (int64_t i = 0; i < n; ++i) {
    double wi = nu * w[i]; /* Eq 14 sub-weight */
    for (int32_t p = 0; p < nz; ++p) {
      double D = kappa + C[p];
      double G = 0.0;
      if (D != 0.0) G = m->p_d * orc_likelihood(m, z[2 * p], z[2 * p + 1], x[i], y[i]) / D; /* Eq 12 */
      double dw = G * w[i];                                                                  /* Eq 13 */
      wi += dw;                                                                              /* Eq 15 */
      acc[5 * p + 0] += dw;                                                                  /* Eq 16 */
      acc[5 * p + 1] += dw * x[i];
      acc[5 * p + 2] += dw * vx[i];
      acc[5 * p + 3] += dw * y[i];
      acc[5 * p + 4] += dw * vy[i];
    }
    w_out[i] = wi;
  }
}

/* ---------------------------------------------------------------------- */
/* 3) STPHD local estimation.
 * LT = round(sum_i w_i) (line 315; half away from zero, S7; all particles, S6);
 * the LT largest dW_p with their labels (line 319; ties: smaller label, S8;
 * only dW_p > 0 eligible; clamp + flag when LT exceeds them, S8);
 * zeta_l = sum_i w^{i,l} x~_i with w^{i,l} = dw^{i,l} / sum_i dw^{i,l} (Eq 18,
 * Sigma_i restored, S9) = S_l / dW_l.  Undetected mass dW^0 = sum_i nu w~_i
 * (Eq 17) = (1 - p_D) W_pred. */
static const double* g_sort_acc;
static int cmp_label(const void* a, const void* b) {
  int32_t pa = *(const int32_t*)a, pb = *(const int32_t*)b;
  double wa = g_sort_acc[5 * pa], wb = g_sort_acc[5 * pb];
  if (wa > wb) return -1;
  if (wa < wb) return 1;
  return (pa < pb) ? -1 : (pa > pb);
}

int32_t orc_extract(const orc_model* m, int32_t nz, const double* acc, double W, double W_pred,
                    int32_t cap, int32_t* labels, double* states, double* mass,
                    int64_t* LT, int32_t* lt_clamped, double* undetected_mass) {
  int64_t lt = (int64_t)floor(W + 0.5);
  if (lt < 0) lt = 0;
  *LT = lt;
  *undetected_mass = (1.0 - m->p_d) * W_pred;
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nz > 0 ? nz : 1));
  int32_t ne = 0;
  for (int32_t p = 0; p < nz; ++p)
    if (acc[5 * p] > 0.0) idx[ne++] = p;
  g_sort_acc = acc;
  qsort(idx, (size_t)ne, sizeof(int32_t), cmp_label);
  *lt_clamped = (lt > ne) ? 1 : 0;
  int64_t nsel = lt < ne ? lt : ne;
  if (nsel > cap) nsel = cap;
  for (int64_t s = 0; s < nsel; ++s) {
    int32_t p = idx[s];
    double dW = acc[5 * p];
    labels[s] = p;
    mass[s] = dW;
    for (int c = 0; c < 4; ++c) states[4 * s + c] = acc[5 * p + 1 + c] / dW;
  }
  free(idx);
  return (int32_t)nsel;
}

/* ---------------------------------------------------------------------- */
/* 4) Resampling (Algorithm 1; Step 5 line 339):
 * N_k = sum_j w~_j; resample {x~, w~/N_k} into n_out particles, each of weight
 * N_k / n_out (mass preserved, S19).  Scheme: systematic (S18) with one offset
 * U in (0,1) from Philox({0, k, 3, 0}), thresholds t_j = (j + U) N_k / n_out,
 * ancestor(j) = min{ i : B_i > t_j } with B_i the sequential fp64 cumsum. */
double orc_resample_U(uint64_t seed, int32_t k) {
  uint32_t ctr[4] = {0u, (uint32_t)k, 3u, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  orc_philox4x32_10(ctr, key, o);
  return orc_u52(o[0], o[1]);
}

double orc_resample(int64_t n, const double* w, double U, int64_t n_out, int64_t* anc) {
  double W = 0.0;
  for (int64_t i = 0; i < n; ++i) W += w[i];
  if (!(W > 0.0)) {
    for (int64_t j = 0; j < n_out; ++j) anc[j] = (int64_t)((double)j * (double)n / (double)n_out);
    return W;
  }
  int64_t last_pos = n - 1;
  while (last_pos > 0 && !(w[last_pos] > 0.0)) --last_pos;
  int64_t i = 0;
  double B = w[0];
  for (int64_t j = 0; j < n_out; ++j) {
    double t = ((double)j + U) * W / (double)n_out;
    while (i < n - 1 && !(B > t)) {
      ++i;
      B += w[i];
    }
    anc[j] = (B > t) ? i : last_pos;
  }
  return W;
}
