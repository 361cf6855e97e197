/* include/phd.h -- C ABI of the B200-native particle PHD filter hot path.
 *
 * Implements one step of the particle PHD filter of arXiv 1503.03769
 * ("Distributed Computation Particle PHD filter"; /root/reference/PAPER.md),
 * sharded over P processes (one per GPU) exactly as the paper partitions
 * particles over processing elements: every rank holds a
 * contiguous block of the global particle array and the full measurement set.
 *
 * Step order (Algorithm 1):
 *   phd_init_population    t = 0: the initial population, once
 *   phd_predict            Eq 5 survivors (CV model PAPER.md:370-388) + Eq 6 births
 *   phd_update             Eq 7/11 normaliser C(z) (all-reduced), Eq 8/12-16 weights
 *                          and STPHD accumulators (all-reduced)
 *   phd_extract            PAPER.md:313-324 LT = round(W), top-LT labels, zeta = S/dW
 *                          (rank 0 = the central unit)
 *   phd_resample_exchange  PAPER.md:177-180, 339-352 systematic resampling, exact
 *                          over the global array, then the particle exchange that
 *                          rebalances the shards
 * or the fused phd_step.  Readings of garbled/silent passages: DESIGN.md §2.
 *
 * Conventions
 *  - Every call returns phd_status; nothing throws across the ABI.  On error
 *    phd_last_error(ctx) holds a one-line message.
 *  - Ownership: the ctx owns its device memory (allocated once in phd_create,
 *    or carved from a caller workspace of phd_workspace_size() bytes that the
 *    caller keeps alive until phd_destroy).  No allocation happens in a step.
 *    With world > 1 (exact mode) phd_create also allocates, outside the
 *    workspace, the particle double buffers that the ranks map into each other
 *    (CUDA IPC) for the fused resample + exchange (2 x 20 bytes x the rank's
 *    capacity).
 *    Host arrays passed in are borrowed for the duration of the call; outputs
 *    are caller-allocated.  Pointers to measurement / particle arrays may be
 *    host or device pointers (copied with cudaMemcpyDefault).
 *  - Streams: all device work is ordered on the ctx stream (the caller's
 *    cudaStream_t passed to phd_create, or the ctx's own).  Calls that return
 *    host data synchronise that stream.  A ctx is not thread-safe.
 *  - Collectives: with world > 1 every call except the getters is collective:
 *    every rank makes the same calls in the same order with the same
 *    non-pointer arguments and the same measurement set.
 *  - Labels are 0-based measurement indices into the array passed to
 *    phd_update (the paper and SPEC use 1..M_k).
 *  - State layout: particle state is SoA fp32 in the paper's component order
 *    (x, vx, y, vy); host arrays "soa4" are [4][n] row-major.
 */
#ifndef PHD_H
#define PHD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHD_ABI_VERSION 3

typedef struct phd_ctx phd_ctx;

typedef enum {
  PHD_OK = 0,
  PHD_EINVAL = 1,     /* invalid argument or parameter (message says which) */
  PHD_ESTATE = 2,     /* call out of order (predict -> update -> [extract] -> resample) */
  PHD_ECAPACITY = 3,  /* particle count exceeds capacity (fixed mode) */
  PHD_EMODEL = 4,     /* non-finite C, D or W detected (a NaN particle makes every C NaN; the gated
                         update counts NaN particles itself, on every rank) */
  PHD_ENOMEM = 5,     /* device allocation failed / workspace too small */
  PHD_ECUDA = 6,      /* CUDA runtime error (message has the CUDA string) */
  PHD_ENCCL = 7,      /* NCCL error or NCCL unavailable for world > 1 */
  PHD_ENODEV = 8      /* no CUDA device */
} phd_status;

typedef enum { PHD_MEAS_POSITION = 0, PHD_MEAS_RANGE_BEARING = 1 } phd_meas_model;
typedef enum { PHD_COUNT_ADAPTIVE = 0, PHD_COUNT_FIXED = 1 } phd_count_mode;
typedef enum { PHD_STAGE_RESAMPLED = 0, PHD_STAGE_PREDICTED = 1 } phd_stage;
/* PHD_MODE_EXACT: global C (all-reduced), exact global systematic resampling with
 *   an order-preserving rebalance -- the single-device particle PHD filter,
 *   P-invariant (north_star hot path).
 * PHD_MODE_DCP: the paper's DCPFPHD (§3, Algorithm 1, Steps 1-6): every
 *   rank is a group with its own population, local C (Eq 11), local estimates
 *   fused at rank 0 by the label vote of Step 4, local resampling to
 *   max(LT_j,1) R (Algorithm 1) and the ring exchange of L particles of
 *   Step 6.  With world = 1 both modes are identical. */
typedef enum { PHD_MODE_EXACT = 0, PHD_MODE_DCP = 1 } phd_mode;

/* Model and sizing parameters (§4 simulation model; values per
 * BASELINE.json configs).  All doubles; the kernels derive fp32 constants. */
typedef struct {
  int32_t abi_version;        /* must be PHD_ABI_VERSION */
  int32_t meas;               /* phd_meas_model */
  double T;                   /* CV sampling period, > 0 */
  double sigma_a;             /* std of the CV process noise w_k, both axes, >= 0 */
  double p_s;                 /* survival probability e_{k|k-1} in [0,1] (Eq 5) */
  double p_d;                 /* detection probability P_D in [0,1] (Eq 4, 8) */
  double sigma_z[2];          /* (sigma_x, sigma_y) or (sigma_r, sigma_theta), > 0 */
  double sensor_xy[2];        /* range-bearing sensor position */
  double region[4];           /* measurement region: position (xmin,xmax,ymin,ymax);
                                 range-bearing (rmin,rmax,thmin,thmax); kappa = lambda/V */
  double clutter_rate;        /* lambda >= 0 */
  double birth_mass;          /* gamma >= 0: total birth mass per step (Eq 6) */
  double birth_sigma_v;       /* birth velocity std >= 0 */
  int64_t births_per_step;    /* J >= 0; J = 0 requires gamma = 0 */
  int64_t particles_per_target; /* R >= 1 (adaptive mode: N_out = max(LT,1) R) */
  int64_t fixed_count;        /* N_out in fixed mode */
  int32_t count_mode;         /* phd_count_mode */
  int32_t max_meas;           /* max M per step, 1..65536 */
  int64_t capacity;           /* max global N = N_out + J */
  uint64_t seed;              /* Philox4x32-10 key {lo32, hi32} */
  int32_t mode;               /* phd_mode */
  int32_t reserved0;          /* must be 0 */
  int64_t exchange_count;     /* DCP ring exchange L per step (0: floor(min_j N_j / 10));
                                 clamped to floor(min_j N_j / 2) */
  int32_t birth_model;        /* 0: births around Z_{k-1} (uniform when none), S10,
                                    weight gamma/J;
                                 1: N(birth_mean, diag(birth_std^2)), gamma/J;
                                 2: drawn as 0, weighted by the full Eq 6 ratio
                                    gamma N(x; birth_mean, Q) / (J p_k(x|Z_{k-1})), p_k the
                                    stratified proposal mixture; needs
                                    birth_sigma_v > 0 and birth_std > 0 */
  int32_t gate_floor;         /* gated update only.  0: exact gating -- a (tile, measurement) pair
                                 is skipped only when every term of it underflows to exactly 0
                                 in the dense kernels (largest possible exponent < -130).
                                 F in [-126, -20]: a pair is skipped when its largest possible
                                 term p_D g w is below 2^F; each C(z) then differs from the dense
                                 one by less than N_global 2^F (absolute; the weights and sums by
                                 correspondingly less), which the caller sizes against its
                                 tolerance (DESIGN.md §5 "Gated update": bench's floor
                                 log2(kappa) - 60 keeps every C within 2^-36 kappa at N <= 2^24).
                                 Other values: PHD_EINVAL. */
  double birth_mean[4];       /* x-bar (x, vx, y, vy) of birth_model 1 */
  double birth_std[4];        /* sqrt(diag Q) of birth_model 1, >= 0 */
  int32_t stphd_all;          /* 0: pass 2 accumulates the STPHD state sums S_l only for the
                                 top-LT index set I, selected right after
                                 pass 1 from dW = C/D and W = (1-pD) W_pred + sum dW; the
                                 accumulators of other labels read 0.  1: for every measurement. */
  int32_t gate;               /* update algorithm (DESIGN.md §5 "Gated update"):
                                 0: dense -- both passes evaluate all N x M pairs;
                                 1: gated, automatic -- particles ordered by measurement-space
                                    cell (a sorted copy; the filter's particle order and hence
                                    resampling are unchanged), tiles of 512 paired only with the
                                    measurements whose largest possible exponent over the tile is
                                    >= -130, i.e. every skipped pass-1 term underflows to exactly
                                    0 in the dense kernels (same non-zero terms, fp64 sums in
                                    another fixed order); a skipped pass-2 term u/(kappa + C) is
                                    below 2^-130/kappa, far below fp32 resolution of any weight.  Runs dense for an update whose candidate
                                    pairs exceed half of N x M or the workspace, or with
                                    N x M < 2^29 in exact mode (the sort would dominate);
                                 2: gated whenever the candidate lists fit the workspace. */
  double proposal_scale;      /* s in (0, 1e3]: Eq 5 proposal q_k = the CV transition with
                                 noise std s sigma_a, survivors weighted p_s f/q
                                 (PAPER.md:148-152); 0 or 1: q_k = transition prior (S10) */
} phd_params;

/* One labelled estimate: label = measurement index, state =
 * zeta = S/dW (x, vx, y, vy), mass = dW (Eq 16). */
typedef struct {
  int32_t label;
  float state[4];
  float mass;
} phd_estimate;

typedef struct {
  double W;               /* sum of updated weights over all ranks (N_k); DCP mode:
                             the mean over the K groups (each group is a full-intensity filter,
                             PAPER.md:221, so the mean, not the sum, estimates the count) */
  double W_pred;          /* sum of predicted weights (DCP: mean over the groups) */
  double undetected_mass; /* dW^0 = (1 - p_D) W_pred (Eq 17) */
  int64_t LT;             /* round half away from zero of W */
  int64_t N;              /* global particle count of this update */
  int64_t N_out;          /* offspring count of the next resample (filled by extract) */
  int32_t M;              /* measurements of this update */
  int32_t n_est;          /* estimates written */
  int32_t lt_clamped;     /* LT exceeded the eligible labels (dW > 0) */
  int32_t count_clamped;  /* adaptive N_out clamped to capacity */
  int32_t zero_mass;      /* W == 0: offspring spread uniformly with weight 0 */
  int32_t near_half;      /* |W - (n + 1/2)| < 1e-4 max(1,W): LT may differ from fp64 */
} phd_summary;

/* ---- version / errors ---------------------------------------------------- */
int32_t phd_abi_version(void);
const char* phd_status_str(phd_status s);
/* Last error message of ctx (never NULL; "" when none). */
const char* phd_last_error(const phd_ctx* ctx);

/* ---- lifecycle ----------------------------------------------------------- */
/* 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it). */
phd_status phd_nccl_unique_id(uint8_t out[128]);
/* Device bytes phd_create needs for these params at this world size. */
phd_status phd_workspace_size(const phd_params* p, int32_t world, size_t* bytes);
/* Create a context on `device` for rank `rank` of `world`.
 * nccl_id: 128-byte id from phd_nccl_unique_id (ignored when world == 1).
 * stream: a cudaStream_t to order work on, or NULL for an own stream.
 * workspace: device pointer of >= phd_workspace_size bytes, or NULL to allocate.
 * Errors: PHD_EINVAL (bad params: sigma <= 0, p outside [0,1], J = 0 with gamma > 0,
 * fixed N_out + J > capacity, max_meas out of range, rank/world), PHD_ENODEV,
 * PHD_ENOMEM, PHD_ENCCL. */
phd_status phd_create(const phd_params* p, int32_t rank, int32_t world, const uint8_t* nccl_id,
                      int32_t device, void* stream, void* workspace, phd_ctx** out);
void phd_destroy(phd_ctx* ctx);

/* In-process rank group: `world` contexts in ONE process (one host thread per
 * rank, possibly all on one GPU) whose collectives are host barriers plus
 * device-to-device copies instead of NCCL.  It runs exactly the multi-rank
 * orchestration of phd_update / phd_resample_exchange and exists to test that
 * path without W GPUs; ranks never wait on one another inside a kernel.  Every
 * rank's calls must be issued concurrently (one thread per rank).
 * world in [1, 16].  The group must outlive its contexts. */
typedef struct phd_group phd_group;
phd_status phd_group_create(int32_t world, phd_group** out);
void phd_group_destroy(phd_group* g);
phd_status phd_create_in_group(const phd_params* p, phd_group* g, int32_t rank, int32_t device, void* stream,
                               void* workspace, phd_ctx** out);

/* Host transport: a multi-process rank group whose collectives run through caller
 * callbacks on HOST buffers (test infrastructure: several processes on one GPU, where
 * NCCL refuses duplicate devices).  Everything else is the product path: the peer-memory
 * window (CUDA IPC handles, all-gathered through allgather_bytes), the fused gather with
 * its P2P stores, the kernels.  Callbacks are synchronous and collective (every rank calls
 * them in the same order): allreduce_f64 sums buf[0..n) over the ranks in rank order, in
 * place; allgather_bytes writes rank r's send[0..bytes) to recv + r * bytes.  They return
 * 0 on success.  The struct is copied; user must outlive the ctx. */
typedef struct {
  void* user;
  int32_t (*allreduce_f64)(void* user, double* buf, size_t n);
  int32_t (*allgather_bytes)(void* user, const void* send, void* recv, size_t bytes);
} phd_host_transport;
phd_status phd_create_with_transport(const phd_params* p, int32_t rank, int32_t world, const phd_host_transport* t,
                                     int32_t device, void* stream, void* workspace, phd_ctx** out);

/* ---- t = 0: the initial population ---------------------------------------
 * PAPER.md:260 ("t=0: Generate M particles for each group. The number of all
 * particles is N. All these particles are shared with same weights omega_0 = 1/M"),
 * with the reading S23 of DESIGN.md §2.  Generates on the device, in this rank's
 * block, the N_out particles of the population (fixed count: fixed_count; adaptive:
 * max(round(total_mass), 1) R clamped to capacity - J, flag count_clamped):
 *   y_g = y0 + (y1 - y0)(g + u0)/N_out   (index-stratified: contiguous rank blocks are y-bands)
 *   x_g = x0 + (x1 - x0) u1,  (vx, vy) = v_max (2 u2 - 1, 2 u3 - 1)
 * with u_c = ((w_c >> 9) + 1/2) 2^-23 of Philox4x32-10 word c at counter
 * (g lo32, 0, 5, g hi32), key = seed; fp64 arithmetic, one rounding to fp32.
 * box = (x0, x1, y0, y1), host array of 4 doubles; NULL: the position region, or
 *   for range-bearing the square of side r_max centred on the sensor.
 * Weights: total_mass / N_out each (omega_0 = 1/M per unit mass); with mass_box
 *   (host, 4 doubles, closed) total_mass / (number of particles whose fp32
 *   position lies inside it, over all ranks) inside and 0 outside; none inside:
 *   all 0.  DCP mode: group j holds block j of the population and its own
 *   total_mass (each group is a full-intensity filter).
 * Stream-ordered, no host synchronisation; collective for world > 1.  The next
 * call must be phd_predict (k = 1: births uniform over the region).
 * Errors: PHD_EINVAL (total_mass or v_max negative / non-finite, empty box),
 * PHD_ECAPACITY (DCP group above capacity). */
phd_status phd_init_population(phd_ctx* ctx, double total_mass, const double* box, const double* mass_box,
                               double v_max);

/* ---- population injection / inspection (parity, checkpoint) ---------------
 * The global particle array at a step is [survivors 0..N_out-1, births
 * N_out..N_out+J-1]; rank r owns the block [floor(r N/W), floor((r+1) N/W)).
 * stage = PHD_STAGE_RESAMPLED: soa4/w are this rank's survivors (the part of its
 *   block below n_global), n_global = global survivor count N_out; the next
 *   call must be phd_predict.  w == NULL: every weight = mass / n_global.
 *   DCP mode: every rank holds its own group; n_global is ignored (= n_local).
 * stage = PHD_STAGE_PREDICTED: soa4/w are this rank's whole block of a
 *   predicted array of n_global particles; the next call must be phd_update.
 * Errors: PHD_EINVAL (n_local does not match the block), PHD_ECAPACITY. */
phd_status phd_set_particles(phd_ctx* ctx, const float* soa4, const float* w, int64_t n_local,
                             int64_t n_global, double mass, int32_t stage);
/* Checkpoint / resume: set the measurement set Z_{k-1} that the next
 * phd_predict(k, NULL) / phd_step draws its births around (the set an update
 * retains; M = 0: none, births uniform).  With phd_set_particles of a saved
 * resampled population this resumes a run exactly (the noise is counter-based:
 * Philox at (slot, k, stream)).  z: host or device [M][2].  Errors: PHD_EINVAL. */
phd_status phd_set_retained_measurements(phd_ctx* ctx, const float* z, int32_t M);
/* Copy this rank's particles (SoA [4][n] and weights) to host; synchronous.
 * n_local receives the count, global_offset the global index of element 0. */
phd_status phd_get_particles(phd_ctx* ctx, float* soa4, float* w, int64_t cap, int64_t* n_local,
                             int64_t* global_offset);

/* ---- the step ------------------------------------------------------------- */
/* Eq 5 + Eq 6 at step k >= 1.  z_prev [M_prev][2] is Z_{k-1} for the births
 * (measurement-driven, S10); NULL = the Z retained by the last
 * phd_update (none yet: births uniform over the region). */
phd_status phd_predict(phd_ctx* ctx, int32_t k, const float* z_prev, int32_t M_prev);
/* Update with Z_k: z [M][2] fp32 (position: (x,y); range-bearing: (r, theta) with
 * theta in [-pi, pi]).  0 <= M <= max_meas. */
phd_status phd_update(phd_ctx* ctx, const float* z, int32_t M);
/* Estimates of the last update (rank 0 fills out[], every rank fills s).
 * Writes min(LT, #eligible, cap) estimates sorted by (mass desc, label asc). */
phd_status phd_extract(phd_ctx* ctx, phd_estimate* out, int32_t cap, int32_t* n_out, phd_summary* s);
/* Systematic resampling of the updated global array into N_out offspring
 * (adaptive: max(LT,1) R clamped to capacity - J; fixed: fixed_count), then
 * the exchange that leaves every rank its block of the next step's array. */
phd_status phd_resample_exchange(phd_ctx* ctx, int32_t k);
/* predict(k, NULL) + update(z, M) + extract + resample_exchange(k), with one host
 * synchronisation (the update's end-of-stage bookkeeping -- rank masses, LT, the
 * non-finite guard -- completes with the extraction's read-back; a PHD_EMODEL of
 * the update is then reported by phd_step after the extraction kernel ran).
 * Results equal those of the four calls. */
phd_status phd_step(phd_ctx* ctx, int32_t k, const float* z, int32_t M, phd_estimate* out,
                    int32_t cap, int32_t* n_out, phd_summary* s);

/* ---- introspection (synchronous; for parity tests and debugging) ---------- */
/* Global C[M] (Eq 7) of the last update, label order. */
phd_status phd_get_normalizers(phd_ctx* ctx, double* C, int32_t cap);
/* Global STPHD accumulators [M][5] = (dW, Sx, Svx, Sy, Svy) (Eqs 16, 18), label order.
 * With stphd_all = 0 the state sums of labels outside the estimated index set are 0. */
phd_status phd_get_accumulators(phd_ctx* ctx, double* acc, int32_t cap);
/* DCP mode: this rank's local (pre-fusion) estimates of the last extract,
 * sorted by (mass desc, label asc); n receives the count. */
phd_status phd_get_local_estimates(phd_ctx* ctx, phd_estimate* out, int32_t cap, int32_t* n);
/* Ancestors (global index into the updated array) of this rank's produced
 * offspring of the last resample, in global offspring order; n = count,
 * first = global offspring index of anc[0]. */
phd_status phd_get_ancestors(phd_ctx* ctx, int32_t* anc, int64_t cap, int64_t* n, int64_t* first);
/* W, U, N_out and the per-rank masses W_r[world] of the last resample. */
phd_status phd_get_resample_meta(phd_ctx* ctx, double* W, double* U, int64_t* N_out, double* W_r);
/* Gated update statistics of the last phd_update (gate != 0): out[0] = 1 if the
 * gated path ran (0: dense), out[1] = candidate entries (tile, measurement),
 * out[2] = (particle, measurement) pairs evaluated (entries x 512 incl. tile padding),
 * out[3] = tiles. */
phd_status phd_get_gate_stats(phd_ctx* ctx, int64_t* out /* [4] */);
/* Particle exchange path of the last resampling: 0 none (world 1, or DCP ring only),
 * 1 send/recv (NCCL grouped send/recv, or device copies in an in-process group),
 * 2 fused gather + exchange over the peer-memory window. */
int32_t phd_exchange_path(const phd_ctx* ctx);
/* Kernel launches issued by this ctx since creation (all streams). */
int64_t phd_launch_count(const phd_ctx* ctx);
/* Device time (ms) of the last update's pass-1 and pass-2 kernels, measured
 * with CUDA events on the ctx stream when timing is enabled. */
phd_status phd_set_timing(phd_ctx* ctx, int32_t enable);
/* CUDA-graph steps of phd_step (one rank, dense update; opt-in with PHD_GRAPH=1): graphs
 * captured (one per launch shape) and replayed so far. */
phd_status phd_get_graph_stats(const phd_ctx* ctx, int64_t* captures, int64_t* replays);
phd_status phd_get_timing(phd_ctx* ctx, float* ms /* [8]: predict, pass1, pass2, update_total,
                                                      extract, resample, exchange, step */);

/* ---- host-only helpers (no device needed; used by the CPU tests) ---------- */
/* Library's own Philox4x32-10 (host build of the device generator). */
void phd_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* The same block cipher as the device code of the filter runs it (the kernels' own
 * Philox, known-answer tests against cuRAND's curand_Philox4x32_10): out[i] =
 * Philox4x32-10(ctr[i], key = {seed lo32, seed hi32}) for i < n.  ctr and out are
 * DEVICE arrays of n x 4 uint32; stream: cudaStream_t (NULL: the legacy stream);
 * synchronous.  Errors: PHD_EINVAL (n < 0, NULL arrays), PHD_ECUDA. */
phd_status phd_philox4x32_10_device(uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out, void* stream);
/* Block [lo, hi) of n items owned by rank (floor(r n / world) bounds). */
phd_status phd_rank_block(int64_t n, int32_t world, int32_t rank, int64_t* lo, int64_t* hi);
/* Resampling bounds: W = sum W_r (rank order), O_r = exclusive prefix,
 * bounds[r] = n(O_r) = clamp(ceil(O_r n_out / W - U), 0, n_out), bounds[world] = n_out.
 * Rank r produces the offspring [bounds[r], bounds[r+1]). */
phd_status phd_resample_bounds(int32_t world, const double* W_r, int64_t n_out, double U,
                               int64_t* bounds, double* W);
/* Exchange plan for `rank`: offspring produced on rank s are [bounds[s], bounds[s+1]);
 * the next step's survivors [0, n_out) are owned per phd_rank_block(n_out + J).
 * send_* / recv_* [world]: element counts and offsets (into the rank's produced
 * range for sends, into its local block for receives). */
phd_status phd_plan_exchange(int32_t world, int32_t rank, const int64_t* bounds, int64_t n_out,
                             int64_t J, int64_t* send_count, int64_t* send_off, int64_t* recv_count,
                             int64_t* recv_off);

#ifdef __cplusplus
}
#endif
#endif /* PHD_H */
