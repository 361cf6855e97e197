/* oracle/phd_oracle.h -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain, slow, single-threaded fp64 CPU reference of the particle PHD filter
 * step (arXiv 1503.03769, §2.2 Eqs 5-8 and §3 Eqs 10-18).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
 * may load it.  It shares no code, header, table or constant with the CUDA
 * library under paper_1503_03769_b200/ (DESIGN.md §3).
 *
 * Parity pins: see tests/test_oracle_pins.py.  Every function below is pinned
 * (Philox vs ATen philox_engine, closed forms, invariants, mpmath brute force,
 * hand-derived resampling cases); none is "parity unpinned".
 */
#ifndef PHD_ORACLE_H
#define PHD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t meas;          /* 0 = position (x, y) sensor, 1 = range-bearing */
  int32_t pad_;
  double T;              /* CV sampling period */
  double sigma_a;        /* std of the CV noise w_k on both axes */
  double p_s;            /* survival probability e_{k|k-1} */
  double p_d;            /* detection probability P_D */
  double sigma_z[2];     /* (sigma_x, sigma_y) or (sigma_r, sigma_theta) */
  double sensor[2];      /* sensor position (s_x, s_y) */
  double region[4];      /* measurement region: z0 in [r0,r1], z1 in [r2,r3] */
  double clutter_rate;   /* lambda: kappa = lambda / V */
  double birth_mass;     /* gamma: total birth mass per step */
  double birth_sigma_v;  /* birth velocity std */
  uint64_t seed;         /* Philox key {lo32, hi32} */
  int32_t birth_model;   /* 0: around Z_{k-1} (S10); 1: N(birth_mean, diag(birth_std^2));
                            2: drawn as 0, weighted by the full Eq 6 ratio gamma(x)/(J p_k(x|Z)) with
                               gamma(x) = birth_mass N(x; birth_mean, diag(birth_std^2)) */
  int32_t pad2_;
  double birth_mean[4];  /* x-bar (x, vx, y, vy) */
  double birth_std[4];   /* sqrt(diag Q) */
  double proposal_scale; /* s: Eq 5 proposal q_k = CV transition with noise std s sigma_a
                            (0 or 1: q_k = transition prior, ratio p_s) */
} orc_model;

/* Philox4x32-10 block cipher; ctr = {c0,c1,c2,c3}, key = {k0,k1}. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* 32-bit word -> uniform in (0,1): ((w >> 9) + 0.5) * 2^-23 (exact). */
double orc_conv23(uint32_t w);
/* two words -> uniform in (0,1) with 52 bits: ((w0>>6)*2^26 + (w1>>6) + 0.5) * 2^-52 (exact). */
double orc_u52(uint32_t w0, uint32_t w1);
/* Box-Muller: n1 = sqrt(-2 ln u1) cos(2 pi u2), n2 = sqrt(-2 ln u1) sin(2 pi u2). */
void orc_box_muller(double u1, double u2, double* n1, double* n2);

/* t = 0 population (reading S23): particles g_lo .. g_hi-1 of n_out,
 * y-stratified over box = (x0, x1, y0, y1), x uniform, v = v_max (2u - 1), u from
 * Philox({g, 0, 5, g>>32}); states rounded to fp32; weights total_mass shared equally
 * (over the particles inside mass_box when given, 0 outside).  Returns the inside count. */
int64_t orc_init_population(const orc_model* m, int64_t n_out, int64_t g_lo, int64_t g_hi, const double box[4],
                            double v_max, double total_mass, const double* mass_box, double* x, double* vx,
                            double* y, double* vy, double* w);

/* kappa(z) = lambda / V, V the area of the measurement region. */
double orc_kappa(const orc_model* m);
/* g(z | x) of the sensor model; (x, y) is the target position. */
double orc_likelihood(const orc_model* m, double z0, double z1, double x, double y);

/* Eq 5 with q = transition prior: survivors at global indices g0 .. g0+n-1 (in place). */
void orc_predict(const orc_model* m, int32_t k, int64_t n, int64_t g0,
                 double* x, double* vx, double* y, double* vy, double* w);
/* Eq 6: births b0 .. b0+nb-1 of J, at global slots n_out + b, drawn around Z_{k-1}. */
void orc_births(const orc_model* m, int32_t k, int64_t n_out, int64_t J, int64_t b0, int64_t nb,
                const double* zprev, int32_t m_prev,
                double* x, double* vx, double* y, double* vy, double* w);
/* Eq 6 importance weights of nb births with states (x, vx, y, vy) (birth_model 2), into w:
 * w_b = gamma(x_b) / (J p_k(x_b | Z_{k-1})), p_k the stratified proposal mixture
 * of the births [blo, blo+J) of this filter (birth b uses component b mod m_prev). */
void orc_birth_is_weights(const orc_model* m, int64_t J, int64_t blo, int64_t nb,
                          const double* zprev, int32_t m_prev, const double* x, const double* vx,
                          const double* y, const double* vy, double* w);
/* Eq 7 / Eq 11: C[p] = sum_i p_D g(z_p | x_i) w_i. */
void orc_normalizers(const orc_model* m, int64_t n, const double* x, const double* y,
                     const double* w, const double* z, int32_t nz, double* C);
/* Eqs 8, 12-16: new weights and STPHD accumulators acc[p] = (dW, Sx, Svx, Sy, Svy). */
void orc_update(const orc_model* m, int64_t n, const double* x, const double* vx,
                const double* y, const double* vy, const double* w,
                const double* z, int32_t nz, const double* C, double* w_out, double* acc);
/* All-core timing variants (oracle/phd_oracle_mt.c): the same loops split over
 * particles across nthreads threads, per-thread partial sums added in thread order. */
void orc_normalizers_mt(const orc_model* m, int64_t n, const double* x, const double* y, const double* w,
                        const double* z, int32_t nz, double* C, int32_t nthreads);
void orc_update_mt(const orc_model* m, int64_t n, const double* x, const double* vx, const double* y,
                   const double* vy, const double* w, const double* z, int32_t nz, const double* C,
                   double* w_out, double* acc, int32_t nthreads);
/* LT = round(W); top-LT labels by (dW desc, label asc); zeta = S/dW.
 * Returns the number of estimates written (<= cap). */
int32_t orc_extract(const orc_model* m, int32_t nz, const double* acc, double W, double W_pred,
                    int32_t cap, int32_t* labels, double* states, double* mass,
                    int64_t* LT, int32_t* lt_clamped, double* undetected_mass);
/* Systematic-resampling offset U = u52(Philox({0,k,3,0}, seed)). */
double orc_resample_U(uint64_t seed, int32_t k);
/* systematic resampling of n weights into n_out offspring.
 * anc[j] = min{ i : B_i > (j + U) W / n_out },  B_i = w_0 + ... + w_i (sequential fp64).
 * Returns W.  W == 0: anc[j] = floor(j n / n_out). */
double orc_resample(int64_t n, const double* w, double U, int64_t n_out, int64_t* anc);

#ifdef __cplusplus
}
#endif
#endif
