// Internal interface between the C-ABI orchestration (phd_api.cpp) and the
// CUDA kernels (k_*.cu).  Not installed; not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdio>
#include <utility>
#include <algorithm>
#include <stdint.h>

namespace phd {

// Device bounds checks, compiled in only with -DPHD_DEBUG_BOUNDS (a build
// variant for the tests; compute-sanitizer is unavailable on the GPU pool).
#ifdef PHD_DEBUG_BOUNDS
#define PHD_DCHECK(cond)                                                                         \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("PHD_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)threadIdx.x);                                                 \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define PHD_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// ---- programmatic dependent launch (PDL) -------------------------------------
// Every kernel is launched with programmatic stream serialization and starts
// with griddepcontrol.wait, which blocks until the preceding grid has completed
// and its memory is visible -- so the semantics are those of plain stream order,
// but the launch and block scheduling of a kernel overlap the tail of the one
// before it (the step is a chain of ~20-45 kernels, many of them short).
// Right after the wait each kernel signals griddepcontrol.launch_dependents, so the next
// kernel of the chain is launched (its CTAs parked at their own wait) while this one
// runs: one kernel of lookahead.  A dependent grid launches only once every CTA of this
// one has started and signalled, so parked CTAs never hold back this grid's own.
// PHD_PDL=0 in the environment launches without the attribute.
#ifndef PHD_PDL_EARLY
#define PHD_PDL_EARLY 0
#endif
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if PHD_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
#endif
}
bool pdl_enabled();

// CUDA loads kernels lazily (CUDA_MODULE_LOADING=LAZY, the default): the first launch of
// each one pays for loading it, ~0.1 ms, inside whichever step first needs that variant
// (a tile size, a pass-2 instance, ...).  Each kernel file's preload_*() asks for the
// attributes of all its kernels, which loads them; phd_create calls preload_kernels()
// once per device.
template <typename... K>
inline void touch_kernels(K... k) {
  cudaFuncAttributes a;
  int dummy[] = {0, ((void)cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k)), 0)...};
  (void)dummy;
}
void preload_update();
void preload_select();
void preload_extract();
void preload_resample();
void preload_predict();
void preload_gate();
void preload_kernels();  // all of the above, once per device (thread-safe)

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute: set it
// once per (kernel, device) -- and again if a launch needs more -- so that one
// process driving several GPUs can launch the >48 KB kernels on every device.
cudaError_t ensure_max_smem_impl(const void* func, int bytes);
template <typename... KArgs>
inline cudaError_t ensure_max_smem(void (*kernel)(KArgs...), size_t bytes) {
  return ensure_max_smem_impl(reinterpret_cast<const void*>(kernel), (int)bytes);
}
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- tiling constants ----------------------------------------
// measurement slots per lane: 4 or 8 (kernel template), i.e. 128 or 256 per warp
#ifndef PHD_MAX_WARPS_Z
#define PHD_MAX_WARPS_Z 16
#endif
// warps per CTA of the dense passes: up to 16 with 8 slots per lane (one CTA row covers
// 4096 slots: cfg 5's particle records are read once, not once per z-block), 8 with 4
constexpr int kMaxWarpsZ = PHD_MAX_WARPS_Z;
constexpr int kMaxWarpsZ4 = 8;
constexpr int max_warps_z(int zl) { return zl == 8 ? kMaxWarpsZ : kMaxWarpsZ4; }
constexpr int kMinWarpsZ = 2;                   // warps per z-block at least (1 measured no faster at cfg 1/2)
#ifndef PHD_TILE_P
#define PHD_TILE_P 256
#endif
constexpr int kTileP = PHD_TILE_P;              // particles per smem tile
constexpr int kTileSmall = 64;                 // small populations (plan_gp)
constexpr int kFlushTiles = 16;                 // fp32 mid-level -> fp64 every 16 tiles
constexpr int kBlockW = 1024;                   // particles per finalize / scan block
constexpr int kBlockOff = 1024;                 // offspring per gather block

enum Model : int { kPosIso = 0, kPosAniso = 1, kRangeBearing = 2 };

// Per-slot measurement constants, slot-major arrays of length slots_pad.
// position: s0 = -z_x, s1 = -z_y; range-bearing: s0 = -z_r, s1 = -z_theta,
// s2/s3 = -(centre x / y) of z in Cartesian, rep = bearing representation.
struct SlotConsts {
  float* s0;
  float* s1;
  float* s2;
  float* s3;
  float* d;        // 1 / (kappa + C) (fp32, 0 when D == 0)
  int32_t* rep;    // range-bearing: 0 (-pi,pi], 1 [0,2pi), 2 (-2pi,0]
};

// The pass-1 slot layout of one update (slots.cuh): slot -> label map and per-slot constants.
struct BuildSlotsArgs {
  const float* z;            // Z (read); zcopy != nullptr: also copied there (the device-resident
  float* zcopy;              //   Z of the one-sync step: no separate device-to-device copy)
  const int* Mp;             // graph replays: this step's M, else nullptr and M
  int M, model, identity, slots_pad;
  int32_t* slot_label;
  float sx, sy;              // range-bearing sensor position
  SlotConsts sc;
  int* bad;                  // non-finite measurements are counted here
};

struct PassArgs {
  int64_t n;                 // local particles
  int64_t tiles_per_cta;
  int tile;                  // particles per record tile: kTileP or kTileSmall (plan_gp)
  int js_split;              // pass 2: the per-warp state-sum layout may be used (js_layout)
  const float* x;
  const float* vx;
  const float* y;
  const float* vy;
  const float* w;
  const float* rb;           // range-bearing repr [8][rb_stride]
  int64_t rb_stride;
  SlotConsts sc;
  int slots_pad;             // stride of slot-major partials
  float na0, na1;            // -alpha_0, -alpha_1 (log2 units)
  float rbs;                 // range-bearing: sigma_r / sigma_theta (bearing residuals in range units)
  float wscale;              // p_D * c, c = 1 / (2 pi sigma_0 sigma_1)
  double* Cpart;             // [gp][slots_pad]
  double* Apart;             // [gp][4][slots_pad]
  float* P;                  // [zb][P_stride]
  int64_t P_stride;
  const int32_t* js;         // pass 2: state sums for the first *js slot pairs of every lane (nullptr: all)
  float* rec;                // per-particle records of the dense passes [n_pad][record_width] (k_records)
};

// Per-step scalars of a CUDA-graph replay of phd_step (world 1, DESIGN.md §4 "graph
// step"): the host stages k, M, M_prev (copied by the graph's first node); block 0 of
// k_scan_chunks (resample_setup_body) fills the rest from the update's results.
// Kernels read them when handed a DevStep pointer, their by-value arguments otherwise.
struct DevStep {
  int32_t k, M, M_prev, zero_mass;
  int64_t n_out;             // offspring of this step's resampling
  double U, W, scale;        // resampling offset, mass, n_out / W
  float w_off;               // offspring weight W / n_out
  int32_t count_clamped;
};

struct PredictArgs {
  int64_t n_local;           // slots of this rank's block
  int64_t g0;                // global index of local slot 0
  int64_t n_out;             // global survivors (slots g < n_out are survivors)
  int64_t J;                 // births per step
  int32_t k;
  uint64_t seed;
  uint64_t ctr_base;         // Philox counter of local slot i is ctr_base + g0 + i (DCP groups: own space)
  int64_t birth_offset;      // global index of this rank's first birth (measurement choice b mod M)
  float T, sigma_a, p_s;
  float prop_s;              // Eq 5 proposal noise scale s (1: transition prior)
  float w_uniform;           // >= 0: survivors' weight before predict; < 0: read w
  int meas;
  float sigma_z0, sigma_z1, sensor_x, sensor_y;
  float region[4];
  float birth_w, birth_sigma_v;
  int birth_model;           // 0 around Z_{k-1}; 1 N(birth_mean, diag(birth_std^2)); 2 as 0 + Eq 6 ratio
  float birth_mean[4], birth_std[4];
  const float* zprev;        // device [m_prev][2]
  int32_t m_prev;
  float *x, *vx, *y, *vy, *w;
  float* rb;                 // range-bearing repr out (nullptr for position)
  int64_t rb_stride;
  const DevStep* ds;         // graph replay: k and m_prev from here
};

// t = 0 population (reading S23): local slots [0, n_local) hold the
// global particles [g0, g0 + n_local) of a population of n_out.
struct InitArgs {
  int64_t n_local, g0, n_out;
  uint64_t seed;
  double box[4];             // x0, x1, y0, y1 (y-stratified)
  double v_max;
  int has_mbox;              // mass only inside mbox (closed)
  double mbox[4];
  double total_mass;
  double n_norm;             // particles sharing the mass without a mass box (population or DCP group)
  float *x, *vx, *y, *vy, *w;
  double* count;             // particles inside the mass box (fp64 integer sum; all-reduced over ranks)
};
cudaError_t launch_init_population(const InitArgs& a, cudaStream_t s);
// second pass (mass box): w = total_mass / count inside, 0 outside
cudaError_t launch_init_weights(const InitArgs& a, cudaStream_t s);

struct ResampleArgs {
  int64_t n_local;
  int64_t g0;
  const float* w;            // updated weights
  const double* blk_off;     // exclusive prefix of block sums (within its scan chunk)
  double O_r;                // exclusive prefix of the per-rank masses
  double scale;              // n_out / W
  double U;
  int64_t lo, hi;            // bounds[r], bounds[r+1]
  int zero_mass;             // W == 0: particle g gets [ceil(g n_out / N), ceil((g+1) n_out / N))
  int64_t n_upd, n_out;      // N (global particles updated) and n_out, for the zero-mass spread
  const DevStep* ds;         // graph replay: lo = 0, hi = n_out, scale, U, zero_mass from here (world 1)
};

// Eq 6 importance weights of the births (birth_model 2): local slots [i0, i0 + nb)
// hold births of this filter, whose births are [birth_offset, birth_offset + J).
struct BirthISArgs {
  int64_t i0, nb;            // first local birth slot, local birth count
  int64_t J, birth_offset;
  int meas;
  double sigma_z0, sigma_z1, sensor_x, sensor_y;
  double region[4];
  double gamma, birth_sigma_v;
  double birth_mean[4], birth_std[4];
  const float* zprev;
  int32_t m_prev;
  const float *x, *vx, *y, *vy;
  float* w;
};

// ---- launchers (return cudaGetLastError of the launch) -----------------------
cudaError_t launch_predict(const PredictArgs& a, cudaStream_t s);
cudaError_t launch_birth_is(const BirthISArgs& a, cudaStream_t s);
cudaError_t launch_rb_repr(const float* x, const float* y, int64_t n, float sx, float sy, float* rb,
                           int64_t stride, cudaStream_t s);
// pass-1 slot layout + per-slot constants on the device (k_build_slots, k_select.cu)
cudaError_t launch_build_slots(const BuildSlotsArgs& a, cudaStream_t s);
cudaError_t launch_pass(int model, int pass, const PassArgs& a, int gp, int zb, int wz, int zl, cudaStream_t s);
// the dense pass 2 folds 1/D into its terms: its state-sum partials already carry 1/D
bool pass2_sums_scaled();
// floats per particle record of the dense passes; build them (once per update, before pass 1)
int record_width(int model);
// blk != nullptr: also the fp64 block sums of a.w (kBlockW particles per block, k_block_sum's
// order); bs != nullptr: one more block builds the pass-1 slot layout (k_build_slots' work)
cudaError_t launch_records(int model, const PassArgs& a, cudaStream_t s, double* blk = nullptr,
                           const BuildSlotsArgs* bs = nullptr);
int pass_occupancy(int model, int pass, int wz, int zl);

// per-slot constants after C: D = kappa + C, C_lab / D_lab by label, d = 1/D (fp32), non-finite count
struct ZConstArgs {
  const int32_t* slot_label;
  double kappa;
  float* d_slot;
  double* C_lab;
  double* D_lab;
  int* bad;
};
// one slot: D = kappa + C, C_lab / D_lab, d = 1/D (0 for padding or D <= 0), NaN count
__device__ __forceinline__ void zconst_one(const ZConstArgs& zc, int s, double C) {
  const int lab = zc.slot_label[s];
  float d = 0.0f;
  if (lab >= 0) {
    const double D = zc.kappa + C;
    zc.C_lab[lab] = C;
    zc.D_lab[lab] = D;
    if (!isfinite(D)) atomicAdd(zc.bad, 1);
    d = D > 0.0 ? (float)fmin(1.0 / D, 3.0e38) : 0.0f;
  }
  zc.d_slot[s] = d;
}

// (wblk != nullptr: one extra block also writes *wout = sum of wblk[0..nwb), the
// rank's W_pred from the block sums of launch_block_sums, which then rides in C1;
// zc != nullptr, one rank only: the per-slot constants of launch_zconst as well)
cudaError_t launch_reduce_C(const double* Cpart, int gp, int slots_pad, int s0, int s1, double* C_slot,
                            cudaStream_t s, const double* wblk = nullptr, int nwb = 0, double* wout = nullptr,
                            const ZConstArgs* zc = nullptr);
// (wpred != nullptr: a non-finite all-reduced W_pred -- a rank's NaN particles, see the
// gated sort -- is counted in bad too, so every rank reports PHD_EMODEL)
cudaError_t launch_zconst(const double* C_slot, const int32_t* slot_label, int s0, int s1, double kappa,
                          float* d_slot, double* C_lab, double* D_lab, int* bad, cudaStream_t s,
                          const double* wpred = nullptr);
// inv != nullptr (gated update): P is one plane in sorted order, read as P[inv[i]]
cudaError_t launch_finalize(const float* w, const float* P, int64_t P_stride, int zb, int64_t n, float nu,
                            float wscale, float* w_out, double* blk_w, double* blk_wp, cudaStream_t s,
                            const int32_t* inv = nullptr);
cudaError_t launch_reduce_acc(const double* Apart, int gp, int slots_pad, int n_slots, const int32_t* slot_label,
                              const double* C_lab, const double* D_lab, const float* s0, const float* s1, const float* s2,
                              const float* s3, int model, const double* blk_w, const double* blk_wp, int nb,
                              double* acc_lab, double* rank_slots, int rank, int world, int lead,
                              const int32_t* sel_flag, cudaStream_t s, int sums_scaled, double n_local);
// W = sum_{r < count} W[r], W_pred = sum Wp[r]; writes the estimates to est[0..)
// and their count to *count_out (the header entry of the gather block).
cudaError_t launch_extract(const double* acc_lab, int M, const double* W, const double* Wp, int count, double p_d,
                           void* est /*phd_estimate*/, int cap, double* summary /*[8]*/, int32_t* count_out,
                           const double* sel_info /*nullptr or (W_id, LT, ...) of k_select*/,
                           const int32_t* sel_flag /*nullptr or k_select's index-set flags*/, cudaStream_t s, const int* Mp = nullptr, int M_alloc = 0);
cudaError_t launch_ring_pack(float* const* src, float* const* dst, int narr, int64_t L, int64_t n, double v,
                             cudaStream_t s);
cudaError_t launch_ring_unpack(float* const* src, float* const* dst, int narr, int64_t L, int64_t n, double v,
                               cudaStream_t s);
// fused resample + exchange (world > 1, peer-memory window)
constexpr int kMaxPeers = 16;
// Resampling + gather in one kernel (k_resample_gather): the block offsets are
// off(b) = coff[b / kResScanChunk] + loc[b] (k_scan_chunks, fixed association).
constexpr int kResScanChunk = 1024;
struct ResampleGatherArgs {
  ResampleArgs r;            // weights, O_r, scale, U, produced range [lo, hi); r.blk_off = loc
  const double* coff;        // [nchunks + 1] chunk offsets
  const float *x, *vx, *y, *vy;  // predicted states (local)
  float w_off;               // offspring weight W / n_out (graph replay: ds->w_off)
  float *ox, *ovx, *oy, *ovy, *ow;  // local outputs at the produced index (p2p == 0)
  int32_t* anc;              // [produced]: global ancestor
};
// one-sync / graph step (world 1): n_out, U, W, scale, w_off, zero_mass of this step into ds
struct SetupArgs {
  const double* rslots;      // rank slots [W_r | ...] (C2 buffer)
  const double* sel_info;    // (W by the mass identity, LT, ...) of k_select_slots
  int fixed;                 // count mode fixed
  int64_t fixed_count, R, lim;  // N_out (fixed), particles per target, capacity - J (adaptive)
  uint64_t seed;
  int32_t k;                 // the step (> 0), or 0: ds->k (graph replays)
};
// exclusive fp64 scan of nb block masses: loc[b] (within its chunk of kResScanChunk), coff[c]
// (chunk prefix; coff[nchunks] = total); deterministic, one launch (last CTA combines).
// ds != nullptr: the same launch computes the step's resampling scalars (SetupArgs) into ds.
cudaError_t launch_scan_chunks(const double* blk, int nb, double* loc, double* ctot, double* coff, unsigned* counter,
                               cudaStream_t s, const SetupArgs* sa = nullptr, DevStep* ds = nullptr);
struct PeerOut;
cudaError_t launch_resample_gather(const ResampleGatherArgs& a, const PeerOut* po, cudaStream_t s);

// End of a one-sync / graph step (world 1): every result the host reads after the step's
// one synchronisation, stored by one kernel into pinned host memory (mapped, UVA) instead
// of one copy per buffer; the non-finite counters are cleared for the next step.
struct StepOutArgs {
  const double* rslots;                 // rank slots [3 world] -> h_rslots
  int n_rslots;
  double* h_rslots;
  int* bad;                             // non-finite counters [4]: [0..1] -> h_bad, then zeroed
  int32_t* h_bad;
  const double* sel_info;               // [4] -> h_sel (nullptr: none)
  double* h_sel;
  const double* summ;                   // extraction summary [8] -> h_summ
  double* h_summ;
  const void* est;                      // estimates (24 B each), their count at *est_count
  const int32_t* est_count;
  void* h_est;
  int est_cap;                          // at most this many copied
  const DevStep* ds;                    // -> *h_ds (nullptr: none)
  DevStep* h_ds;
};
cudaError_t launch_step_out(const StepOutArgs& a, cudaStream_t s);

struct PeerOut {
  float* dst[kMaxPeers][5];   // owner q's next-step arrays x, vx, y, vy, w (peer pointers)
  int64_t blo[kMaxPeers + 1]; // next-step block partition of N' = n_out + J
  int world;
};
cudaError_t launch_fill(float* p, float v, int64_t n, cudaStream_t s);
cudaError_t launch_philox_kat(uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out, cudaStream_t s);
// label selection before pass 2 (k_select.cu)
cudaError_t launch_block_sums(const float* w, int64_t n, double* blk, cudaStream_t s);  // blk only
cudaError_t launch_select(const double* C_lab, const double* D_lab, int M, const double* W_pred, double p_d,
                          int32_t* sel_flag, double* info, cudaStream_t s);
// k_select + the pass-2 slot layout with its per-slot constants (as k_build_slots) and 1/D
// *js = j | (h << 8): the first j + 1 slot pairs of every lane of the first h warps (global
// warp index, z-block major) and the first j of every other lane carry the state sums
// (j in 0..ZL/2; warp-uniform, so each warp runs the sweep instance of its own count), or
// kJsZBlock | b: every slot of the first b z-blocks does (layout 0: whichever needs fewer
// sum slots; 1 / 2 force the per-lane / whole-z-block layout, for tests: PHD_SUM_LAYOUT)
constexpr int32_t kJsZBlock = 0x10000;
// slot pairs per lane with state sums, for global warp gw, from the per-lane encoding above
__host__ __device__ inline int js_of_warp(int32_t v, int gw) { return (v & 0xFF) + (gw < ((v >> 8) & 0xFF) ? 1 : 0); }
// The per-lane layout for n_sel selected slots over `lanes` lanes of zl slots: jl pairs
// per lane, one more on the lanes of the first n_hi warps -- split only where it saves at
// least a quarter of the lane-uniform layout's sum slots, else lane-uniform.  Returns the
// encoding jl | (n_hi << 8) and the state-sum slots.  The layout depends only on this
// step's data (a resumed run is bitwise the same); which pass-2 instance runs it is a
// host guess (the SPLIT instance costs ~1 % where nothing is split, cfg 5): the non-SPLIT
// instance reads a split encoding as "every slot pair" -- a superset, the same bits.
__host__ __device__ inline int32_t js_layout(int n_sel, int lanes, int zl, bool allow_split, int* sum_slots) {
  int jl = n_sel / (2 * lanes);
  if (jl > zl / 2) jl = zl / 2;
  const int rem = n_sel - 2 * jl * lanes > 0 ? n_sel - 2 * jl * lanes : 0;
  int n_hi = jl < zl / 2 ? (rem + 63) / 64 : 0;
  if (n_hi > 0 && (!allow_split || 4 * (2 * jl * lanes + 64 * n_hi) > 3 * (2 * (jl + 1) * lanes))) {
    jl += 1;  // lane-uniform
    n_hi = 0;
  }
  *sum_slots = 2 * jl * lanes + 64 * n_hi;
  return jl | (n_hi << 8);
}
cudaError_t launch_select_slots(const double* C_lab, const double* D_lab, int M, const double* W_pred, double p_d,
                                int32_t* sel_flag, double* info, const float* z, int model, int zl, int wz,
                                int layout, int slots_pad, int32_t* slot_label, int32_t* js, float sensor_x,
                                float sensor_y, SlotConsts sc, cudaStream_t s, const int* Mp = nullptr, int M_alloc = 0);

// ---- gated update (k_gate.cu, DESIGN.md §5 "Gated update") ------------------
// Particles are ordered by a Morton cell key in measurement space (stable
// counting sort; the filter's own particle order is untouched, the passes read
// a sorted copy), cut into tiles of gate_tp(model), and every tile is paired only with
// the measurements whose largest possible exponent over the tile's bounding box,
//   e_max = -alpha0 dx^2 - alpha1 dy^2 + max_i log2(p_D c w_i),
// is >= kGateLog2Min: every skipped pair has e < -130, so its fp32 term
// 2^e flushes to exactly 0 in the dense kernels too (ex2.approx.ftz).
constexpr int kGateG = 64;            // cells per axis (Morton key of 12 bits)
constexpr int kGateBins = kGateG * kGateG;
// Counting-sort blocks (8 warps each): sort_block(n) items per block, a power of two
// in [kSortBlockMin, kSortBlockMax] giving about kSortBlocks blocks, so small sorts
// still fill the GPU and the 16-bit per-warp counters never overflow.
// One block sums a[0..n) in fixed order (thread t: t, t + blockDim, ..., eight loads
// in flight; then a warp tree and a tree over the warps); thread 0 writes *out.
__device__ __forceinline__ void block_sum_f64(const double* __restrict__ a, int n, double* out) {
  __shared__ double ws_[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  double acc = 0.0;
  for (int k0 = tid; k0 < n; k0 += 8 * nt) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = k0 + r * nt < n ? a[k0 + r * nt] : 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) acc += v[r];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) ws_[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    acc = lane < (nt >> 5) ? ws_[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) *out = acc;
  }
}

constexpr int kSortBlockMin = 2048;
constexpr int kSortBlockMax = 65536;
constexpr int kSortBlocks = 256;
inline int64_t sort_block(int64_t n) {
  int64_t b = kSortBlockMin;
  while (b < kSortBlockMax && b * kSortBlocks < n) b <<= 1;
  return b;
}
// upper bound of the block count for n <= cap items (hist / scan buffers)
inline int64_t sort_blocks_max(int64_t cap) { return (cap + sort_block(cap) - 1) / sort_block(cap) + kSortBlocks + 1; }
constexpr int kSortMaxBins = 4096;    // bins per counting-sort pass (12-bit digits)
// particles per gated tile: 1024 for the position sensor (a cfg 5 tile lies inside one
// 31 m cell either way, so half the tiles and entries for the same candidates), 512 for
// range-bearing ((r, theta) tiles span more cells); kGateTP bounds both (allocation)
#ifndef PHD_GATE_TP_POS
#define PHD_GATE_TP_POS 1024
#endif
constexpr int kGateTP = 1024, kGateTPMin = 512;
__host__ __device__ constexpr int gate_tp(int model) { return model == kRangeBearing ? 512 : PHD_GATE_TP_POS; }
constexpr int kGateChunk = 256;       // candidates staged in shared memory at a time
constexpr float kGateLog2Min = -130.0f;

struct GateGrid {
  float lo0, lo1;                     // grid origin (x, y) or (r, -pi)
  float inv_h0, inv_h1;               // cells per unit
  int wrap1;                          // axis 1 is an angle (range-bearing): cells wrap mod kGateG
  float floor;                        // log2 of the skipped terms' bound: kGateLog2Min (exact) or gate_floor
  int kbuf;                           // candidates the count pass buffers per tile (gate_kbuf)
};

// Sorted copy of the particle block (n_pad = ntiles * gate_tp records of n4 float4):
//   position      (x, y, vx, vy), (lw, 0, 0, 0)
//   range-bearing (r_hi, r_lo, thA hi, thA lo), (thB hi, thB lo, thC hi, thC lo), (x, y, vx, vy), (lw, 0, 0, 0)
// with lw = log2(p_D c w) (-inf for w = 0 and padding).
struct GateSorted {
  float4* rec;
  int n4;
  int32_t* inv;                       // local index -> sorted position
  int* lw_max;                        // max lw over the particles (ordered-int encoding)
  int64_t n;                          // particles sorted (records [n, n_pad) are padding)
  int* bad;                           // += NaN particles (x, y or w): the dense C would be NaN
};

struct GateArgs {
  int64_t n;                          // local particles
  int ntiles;
  int model;
  GateSorted so;
  const int32_t* tstart;              // [ntiles + 1] candidate offsets
  const int32_t* cand;                // [E] candidate labels, tile-major
  SlotConsts sc;                      // identity slot layout (slot = label)
  const int32_t* sel;                 // pass 2: label in the index set I (nullptr: all)
  float na0, na1;
  double* part1;                      // [E] tile sums of u = p_D g w (pass 1)
  float* part2;                       // [E][4] tile sums of the centred state terms (pass 2, selected labels)
  float* Ps;                          // [n_pad] sum_z u d per sorted particle (pass 2)
  int64_t E;                          // candidate entries (bounds checks of the debug build)
  int M;                              // measurements (bounds checks of the debug build)
};

// key + stable counting sort of the local particles; writes the sorted copy, and the fp64
// sums of the predicted w per sort block into blk_wp[0 .. *nblk_out) (fixed order: the
// W_pred that rides with C in the C1 all-reduce; the gated update needs no k_block_sum).
// Launch count added to *launches.
cudaError_t gate_sort_particles(int model, const float* const* A /*x,vx,y,vy,w*/, const float* rb, int64_t rb_stride,
                                int64_t n, int64_t n_pad, float wscale, const GateGrid& grid, int32_t* hist,
                                int32_t* scan_tmp, int32_t* keys /*[n] scratch*/, const GateSorted& so, cudaStream_t s,
                                int64_t* launches, double* blk_wp, int* nblk_out);
// measurements -> grid cells (one CTA): zcell_start[kGateBins + 1], items stable by label
cudaError_t gate_zbin(const float* z, int M, const GateGrid& grid, int32_t* hist, int32_t* scan_tmp,
                      int32_t* zcell_start, int32_t* zcell_items, float2* zcell_z, cudaStream_t s, int64_t* launches);
// per-tile bounding boxes + candidate counts (fill = 0) or labels (fill = 1)
// (fill = 0 also buffers the first kbuf candidates per tile in cbuf [ntiles][kbuf]).  kbuf covers
// max_meas (a tile has at most M candidates) up to 4096, so the fill pass is a copy and never
// enumerates a window again (the long windows of tiles spanning a Morton jump set its duration)
constexpr int kGateKBufMax = 4096;
inline int gate_kbuf(int max_meas) { return std::min(kGateKBufMax, std::max(32, (max_meas + 31) & ~31)); }
cudaError_t gate_tiles(int fill, int model, const GateSorted& so, int ntiles, float na0, float na1,
                       const GateGrid& grid, const int32_t* zcell_start, const int32_t* zcell_items,
                       const float2* zcell_z, int32_t* tcount, const int32_t* tstart, int32_t* cbuf, int32_t* cand,
                       cudaStream_t s, int64_t ecap = 0);  // fill: entries [0, ecap) of cand are written
// exclusive scan of n int32 (in place); out[n] = total.  tmp >= ceil(n / 4096) + 1 ints.
cudaError_t gate_scan(int32_t* a, int64_t n, int32_t* tmp, cudaStream_t s, int64_t* launches);
// stable sort of the E candidate entries by label: mlist = entry indices grouped by
// label (ascending entry within a label), mstart[l] = first position of label l.
cudaError_t gate_sort_entries(const int32_t* cand, int64_t E, int M, int32_t* kbuf, int32_t* vbuf, int32_t* mlist,
                              int32_t* hist, int32_t* scan_tmp, int32_t* mstart, cudaStream_t s, int64_t* launches);
cudaError_t launch_gpass(int pass, const GateArgs& g, cudaStream_t s);
// per-label fixed-order fp64 sums over its entries: pass 1 -> C_slot[l];
// pass 2 -> A[q * slots_pad + l] for labels in I (all with sel == nullptr)
// pass 1 with wblk != nullptr: one extra block writes *wout = sum of wblk[0..nwb) (see launch_reduce_C)
cudaError_t launch_gate_reduce(int pass, const int32_t* mstart, const int32_t* mlist, int M, const double* part1,
                               const float* part2, const int32_t* sel, double* out, int slots_pad, cudaStream_t s,
                               const double* wblk = nullptr, int nwb = 0, double* wout = nullptr,
                               const ZConstArgs* zc = nullptr, const int* poison = nullptr);

}  // namespace phd
