// C-ABI implementation (include/phd.h): context, device memory layout, step
// orchestration on one CUDA stream, NCCL collectives for world > 1.
//
// Per step:
//   predict   k_predict                                     (HBM)
//   update    k_records (+ block sums of w, + the slot layout in one more block) -> k_pass<1> -> k_reduce_C (+ W_pred;
//             one rank: + the per-slot constants) -> [C1 all-reduce -> k_zconst] ->
//             k_select_slots -> k_pass<2> -> k_finalize -> k_reduce_acc -> [C2 all-reduce]
//             -> D2H of the rank masses and flags (gated: k_gate.cu kernels instead)
//   extract   k_extract on rank 0 (the central unit) + D2H of the estimates
//   resample  k_scan_chunks -> k_resample_gather (one rank inside phd_step: k_scan_chunks also
//             computes the resampling scalars; the extraction on a second stream, one host
//             synchronisation per step)
//   exchange  world 1: buffer swap; world > 1: k_resample_gather<true> into the owners'
//             arrays over the peer-memory window + one barrier, or grouped ncclSend/ncclRecv (C3)
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "phd.h"
#include "phd_internal.h"
#include "philox.cuh"

#include <nvtx3/nvToolsExt.h>

using namespace phd;

namespace {

// NVTX range per ABI stage (SURVEY.md §5 tracing): visible in nsys / ncu
// timelines, a no-op without an attached tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr double kLog2e = 1.44269504088896340735992468100189214;
enum Stage { kResampled = 0, kPredicted = 1, kUpdated = 2 };

struct Layout {
  int64_t cap_g = 0, cap_l = 0, cap_off = 0;
  int slots_max = 0, zb_max = 0;
  int64_t part_cap = 0;  // max gp * slots_pad
  int64_t nbw_max = 0, nbo_max = 0;
  size_t total = 0;
  // byte offsets
  size_t o_A[5], o_B[5], o_wn, o_rb, o_rec, o_P, o_Cpart, o_Apart, o_zlab, o_zprev, o_slot, o_s[5], o_rep, o_C, o_Cslot, o_sel, o_selinfo, o_D,
      o_acc, o_blk_w, o_blk_wp, o_blk_off, o_ctot, o_coff, o_counter, o_anc, o_step, o_est, o_gather, o_ring, o_summ, o_bad;
  // gated update (p->gate != 0)
  int64_t g_npad = 0, g_ecap = 0, g_hist = 0, g_scan = 0;
  int g_ntiles = 0, g_nsorted = 0;
  size_t o_gkeys, o_ginv, o_gsorted[13], o_gPs, o_ghist, o_gscan, o_gtstart, o_gcand, o_gk, o_gv, o_gmlist,
      o_gpart1, o_gpart2, o_gmstart, o_gzstart, o_gzitems, o_gzz, o_gcbuf, o_glwmax, o_gA;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

Layout make_layout(const phd_params* p, int world, int sms) {
  Layout L;
  L.cap_g = p->capacity;
  L.cap_l = align_up((size_t)(ceil_div(p->capacity, world) + 1), kBlockW);
  L.cap_off = align_up((size_t)p->capacity, kBlockOff);
  // slots: M labels + up to 3 bearing-class pads + the pass-2 select layout's M + 6;
  // every z-block size (wz * 32 * zl, 256 ... 2048 slots) divides 2048
  L.slots_max = (int)align_up((size_t)p->max_meas + 8, 2048);
  // P planes: one per CTA z-block (smallest: kMinWarpsZ warps x 32 lanes x 4 slots) or group
  L.zb_max = std::max(1, L.slots_max / (kMinWarpsZ * 32 * 4));
  L.part_cap = (int64_t)64 * sms * 256 + 8192;
  L.nbw_max = ceil_div(L.cap_l, kBlockW) + 1;
  L.nbo_max = ceil_div(L.cap_off, kBlockOff) + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  for (int i = 0; i < 5; ++i) L.o_A[i] = take(sizeof(float) * L.cap_l);
  for (int i = 0; i < 5; ++i) L.o_B[i] = take(sizeof(float) * std::max(L.cap_off, L.cap_l));
  L.o_wn = take(sizeof(float) * L.cap_l);
  L.o_rb = take(p->meas == PHD_MEAS_RANGE_BEARING ? sizeof(float) * 8 * L.cap_l : 256);
  L.o_P = take(sizeof(float) * (size_t)L.zb_max * L.cap_l);
  // dense-pass particle records (k_records): [cap_l rounded up to kTileP][record_width]
  L.o_rec = take(sizeof(float) * align_up((size_t)L.cap_l, kTileP) *
                 (p->meas == PHD_MEAS_RANGE_BEARING ? 16 : 8));
  L.o_Cpart = take(sizeof(double) * L.part_cap);
  L.o_Apart = take(sizeof(double) * 4 * L.part_cap);
  L.o_zlab = take(sizeof(float) * 2 * (size_t)(p->max_meas + 1));
  L.o_zprev = take(sizeof(float) * 2 * (size_t)(p->max_meas + 1));
  L.o_slot = take(sizeof(int32_t) * L.slots_max);
  for (int i = 0; i < 5; ++i) L.o_s[i] = take(sizeof(float) * L.slots_max);
  L.o_rep = take(sizeof(int32_t) * L.slots_max);
  L.o_C = take(sizeof(double) * (size_t)(p->max_meas + 1));
  L.o_Cslot = take(sizeof(double) * ((size_t)L.slots_max + 8));  // + W_pred (all-reduced with C)
  L.o_sel = take(sizeof(int32_t) * (size_t)(p->max_meas + 8));
  L.o_selinfo = take(sizeof(double) * 8 + 64);
  L.o_D = take(sizeof(double) * (size_t)(p->max_meas + 1));
  L.o_acc = take(sizeof(double) * (5 * (size_t)p->max_meas + 3 * (size_t)world + 8));
  L.o_ring = take(sizeof(double) * ((size_t)world + 8));
  L.o_blk_w = take(sizeof(double) * L.nbw_max);
  L.o_blk_wp = take(sizeof(double) * L.nbw_max);
  L.o_blk_off = take(sizeof(double) * (L.nbw_max + 1));
  L.o_ctot = take(sizeof(double) * (L.nbw_max / kResScanChunk + 2));
  L.o_coff = take(sizeof(double) * (L.nbw_max / kResScanChunk + 3));
  L.o_counter = take(sizeof(unsigned) * 4);
  L.o_anc = take(sizeof(int32_t) * L.cap_off);
  L.o_step = take(sizeof(DevStep));
  L.o_est = take(sizeof(phd_estimate) * (size_t)(p->max_meas + 1));  // [0] header (count), [1..] estimates
  L.o_gather = take(p->mode == PHD_MODE_DCP ? sizeof(phd_estimate) * (size_t)(p->max_meas + 1) * world : 256);
  L.o_summ = take(sizeof(double) * 16);
  L.o_bad = take(sizeof(int) * 4);
  // gated update buffers (DESIGN.md §5 "Gated update"); 256-byte stubs when gate == 0
  const bool gt = p->gate != 0;
  L.g_npad = align_up((size_t)L.cap_l, kGateTP);
  L.g_ntiles = (int)(L.g_npad / kGateTPMin);  // the most tiles of either tile size
  L.g_ecap = std::max<int64_t>((int64_t)1 << 20, (int64_t)L.g_ntiles * std::min(p->max_meas, 256));
  L.g_hist = std::max<int64_t>((int64_t)kGateBins * sort_blocks_max(L.cap_l),
                               (int64_t)kSortMaxBins * sort_blocks_max(L.g_ecap)) + 1;
  L.g_scan = ceil_div(std::max<int64_t>(L.g_hist, L.g_ntiles + (int64_t)p->max_meas + 2), 4096) + 2;
  L.g_nsorted = p->meas == PHD_MEAS_RANGE_BEARING ? 13 : 5;
  auto gtake = [&](size_t bytes) { return take(gt ? bytes : 256); };
  L.o_gkeys = gtake(sizeof(int32_t) * L.cap_l);
  L.o_ginv = gtake(sizeof(int32_t) * L.cap_l);
  L.o_gsorted[0] = gtake(sizeof(float) * (p->meas == PHD_MEAS_RANGE_BEARING ? 16 : 8) * L.g_npad);
  L.o_gPs = gtake(sizeof(float) * L.g_npad);
  L.o_ghist = gtake(sizeof(int32_t) * L.g_hist);
  L.o_gscan = gtake(sizeof(int32_t) * L.g_scan);
  L.o_gtstart = gtake(sizeof(int32_t) * (L.g_ntiles + 1));
  L.o_gcand = gtake(sizeof(int32_t) * L.g_ecap);
  L.o_gk = gtake(p->max_meas > kSortMaxBins ? sizeof(int32_t) * L.g_ecap : 0);
  L.o_gv = gtake(p->max_meas > kSortMaxBins ? sizeof(int32_t) * L.g_ecap : 0);
  L.o_gmlist = gtake(sizeof(int32_t) * L.g_ecap);
  L.o_gpart1 = gtake(sizeof(double) * L.g_ecap);
  L.o_gpart2 = gtake(sizeof(float) * 4 * L.g_ecap);
  L.o_gmstart = gtake(sizeof(int32_t) * ((size_t)p->max_meas + 2));
  L.o_gzstart = gtake(sizeof(int32_t) * (kGateBins + 1));
  L.o_gzitems = gtake(sizeof(int32_t) * ((size_t)p->max_meas + 1));
  L.o_gzz = gtake(sizeof(float) * 2 * ((size_t)p->max_meas + 1));
  L.o_gcbuf = gtake(sizeof(int32_t) * (size_t)L.g_ntiles * gate_kbuf(p->max_meas));
  L.o_gA = gtake(sizeof(double) * 4 * (size_t)L.slots_max);
  L.o_glwmax = gtake(sizeof(int) * 4);
  L.total = off;
  return L;
}

}  // namespace

struct phd_ctx {
  phd_params p{};
  int rank = 0, world = 1, device = 0, sms = 148;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  char* ws = nullptr;
  bool own_ws = false;
  Layout L;
  Comm* comm = nullptr;
  std::string err;
  int64_t launches = 0;
  int model = kPosIso;
  double kappa = 0.0;
  float na0 = 0, na1 = 0, wscale = 0, nu = 0;
  // device arrays
  float* A[5];   // x, vx, y, vy, w
  float* B[5];   // offspring
  float* wn;
  float* rb;
  float* P;
  float* rec;
  double *Cpart, *Apart;
  float *zlab, *zprev;
  int32_t* slot_label;
  float* s[5];   // s0, s1, s2, s3, d
  int32_t* rep;
  double *C, *D, *acc, *rslots;
  double *blk_w, *blk_wp, *blk_off, *ctot, *coff;
  unsigned* scan_counter;
  int32_t* anc;
  DevStep* dstep;          // graph replays: this step's scalars on the device
  phd_estimate* est;      // gather block: est[0].label = count, est[1..] = estimates
  phd_estimate* gather;   // DCP: every rank's gather block
  phd_estimate* h_gather = nullptr;
  double* ring = nullptr;   // DCP: per-rank offspring counts (one-hot all-reduce)
  std::vector<phd_estimate> local_est;
  bool dcp = false;
  double* summ;
  int* bad;
  // pinned host staging
  double* h_meta = nullptr;  // [16 + 2 world + 2]
  phd_estimate* h_est = nullptr;
  float* h_z = nullptr;
  // step state
  int stage = kResampled;
  bool populated = false;
  int64_t n_out = 0;      // global survivors entering predict
  int64_t N = 0;          // global particles of the predicted/updated array
  int64_t n_local = 0, g0 = 0;
  int64_t n_surv_local = 0;
  int M = 0, n_slots = 0, slots_pad = 0, wz = 2, zl = 4, zb = 0, gp = 0, M_z = -1, tile = kTileP;
  bool bad_clean = false;  // the non-finite counters were cleared by the last k_step_out
  int est_eager = 0;       // estimates k_step_out stores (one-sync step)
  double* C_slot = nullptr;
  int32_t* sel_flag = nullptr;   // k_select: label in the estimated index set I
  double* sel_info = nullptr;    // (W_id, LT, n_eligible, n_sel, ..)
  int32_t* s_lim = nullptr;      // pass 2: state-sum layout (js pairs per lane or kJsZBlock|b; k_select_slots)
  bool select = false;           // this update selected I before pass 2
  int m_prev_ext = -1;   // >= 0: zprev holds an explicit Z_{k-1} of this size
  double W = 0, W_pred = 0;
  int64_t LT = 0;
  int64_t N_all = 0;      // particles updated over all ranks
  std::vector<double> Wr, Wpr;
  int bad_flag = 0;
  int near_half = 0;
  // resample
  double U_last = 0, W_last = 0;
  int64_t N_out_last = 0, prod_first = 0, prod_n = 0;
  int count_clamped = 0, zero_mass = 0;
  int64_t ring_L = 0;
  // fused resample + exchange over the peer-memory window (world > 1, exact mode)
  int p2p_state = 0;                       // 0 not set up yet, 1 active, -1 unavailable (send/recv exchange)
  bool p2p_live = false;                   // A currently points into pbuf
  // phd_step: the update's host bookkeeping waits for the extraction's synchronisation
  bool defer_update_sync = false, update_pending = false;
  float* pbuf[2] = {nullptr, nullptr};     // this rank's two particle buffers [5][cap_l] (A / B alternate)
  std::vector<float*> peer_buf;            // [world][2]: every rank's pbuf[0], pbuf[1]
  int par = 0;                             // A = pbuf[par] once live; all ranks flip together
  // gated update
  GateSorted gso{};
  GateGrid ggrid{};
  int32_t *gkeys = nullptr, *ghist = nullptr, *gscan = nullptr, *gtstart = nullptr, *gcand = nullptr, *gk = nullptr,
          *gv = nullptr, *gmlist = nullptr, *gmstart = nullptr, *gzstart = nullptr,
          *gzitems = nullptr, *gcbuf = nullptr;
  float2* gzz = nullptr;
  float *gPs = nullptr, *gpart2 = nullptr;
  double *gpart1 = nullptr, *gA = nullptr;
  bool gated = false;            // the last update ran the gated path
  int64_t g_entries = 0, g_tiles = 0;
  int g_nwb = 0;  // predicted-w block sums written by the particle sort (gated W_pred)
  // CUDA-graph steps (world 1, dense): phd_step replays a captured graph per launch shape
  bool capturing = false;                  // the step's calls are being stream-captured
  bool dev_scalars = false;                // one-sync step: resampling scalars on the device,
                                           // extraction on st2 overlapping the resampling
  cudaStream_t st2 = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaEvent_t ev_plan = nullptr;  // the gate plan's candidate total has reached the host
  bool graph_off = false;                  // disabled (PHD_GRAPH=0, or a capture failed)
  struct GraphEntry {
    int64_t key[8];
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  int32_t* h_stepin = nullptr;             // pinned: k, M, M_prev of the next replay
  DevStep* h_stepout = nullptr;            // pinned: the replay's resampling scalars
  double* hd_meta = nullptr;               // device aliases of h_meta, h_est, h_stepout
  phd_estimate* hd_est = nullptr;
  DevStep* hd_stepout = nullptr;
  int64_t graph_captures = 0, graph_replays = 0;
  // timing
  bool timing = false;
  cudaEvent_t ev[16] = {};
  float t_ms[8] = {};
};

// ---------------------------------------------------------------------------
namespace {

phd_status fail(phd_ctx* c, phd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define CU(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return fail(c, PHD_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                       \
  } while (0)
#define KL(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    ++c->launches;                                                                                \
    if (e_ != cudaSuccess) return fail(c, PHD_ECUDA, "launch %s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define COMM(call)                                                                                \
  do {                                                                                            \
    std::string e_ = (call);                                                                      \
    if (!e_.empty()) return fail(c, PHD_ENCCL, "%s", e_.c_str());                                 \
  } while (0)

void block_of(int64_t n, int world, int rank, int64_t* lo, int64_t* hi) {
  *lo = (int64_t)((__int128)n * rank / world);
  *hi = (int64_t)((__int128)n * (rank + 1) / world);
}

int64_t n_of_host(double B, double scale, double U, int64_t n_out) {
  volatile double t = B * scale;  // no contraction: same IEEE ops as the device __dmul_rn/__dsub_rn
  volatile double t2 = t - U;
  double c = std::ceil((double)t2);
  if (c <= 0.0) return 0;
  if (c >= (double)n_out) return n_out;
  return (int64_t)c;
}

phd_status validate(const phd_params* p, int world, phd_ctx* c) {
  if (!p) return fail(c, PHD_EINVAL, "params is NULL");
  if (p->abi_version != PHD_ABI_VERSION) return fail(c, PHD_EINVAL, "abi_version %d != %d", p->abi_version, PHD_ABI_VERSION);
  if (p->meas != PHD_MEAS_POSITION && p->meas != PHD_MEAS_RANGE_BEARING) return fail(c, PHD_EINVAL, "meas model %d", p->meas);
  if (!(p->T > 0)) return fail(c, PHD_EINVAL, "T must be > 0");
  if (!(p->sigma_a >= 0)) return fail(c, PHD_EINVAL, "sigma_a must be >= 0");
  if (!(p->p_s >= 0 && p->p_s <= 1)) return fail(c, PHD_EINVAL, "p_s outside [0,1]");
  if (!(p->p_d >= 0 && p->p_d <= 1)) return fail(c, PHD_EINVAL, "p_d outside [0,1]");
  if (!(p->sigma_z[0] > 0 && p->sigma_z[1] > 0)) return fail(c, PHD_EINVAL, "sigma_z must be > 0");
  if (!(p->region[1] > p->region[0] && p->region[3] > p->region[2])) return fail(c, PHD_EINVAL, "empty region");
  if (!(p->clutter_rate >= 0)) return fail(c, PHD_EINVAL, "clutter_rate must be >= 0");
  if (!(p->birth_mass >= 0 && p->birth_sigma_v >= 0)) return fail(c, PHD_EINVAL, "birth params must be >= 0");
  if (p->births_per_step < 0) return fail(c, PHD_EINVAL, "births_per_step < 0");
  if (p->births_per_step == 0 && p->birth_mass > 0) return fail(c, PHD_EINVAL, "J = 0 with gamma > 0 (SPEC.md:161)");
  if (p->max_meas < 1 || p->max_meas > 8192) return fail(c, PHD_EINVAL, "max_meas must be in [1, 8192]");
  if (p->capacity < 1 || p->capacity > ((int64_t)1 << 31) - 1) return fail(c, PHD_EINVAL, "capacity must be in [1, 2^31)");
  if (p->count_mode == PHD_COUNT_FIXED) {
    if (p->fixed_count < 1) return fail(c, PHD_EINVAL, "fixed_count must be >= 1");
    if (p->fixed_count + p->births_per_step > p->capacity) return fail(c, PHD_EINVAL, "fixed N_out + J > capacity");
  } else if (p->count_mode == PHD_COUNT_ADAPTIVE) {
    if (p->particles_per_target < 1) return fail(c, PHD_EINVAL, "particles_per_target must be >= 1");
    if (p->particles_per_target + p->births_per_step > p->capacity) return fail(c, PHD_EINVAL, "R + J > capacity");
  } else {
    return fail(c, PHD_EINVAL, "count_mode %d", p->count_mode);
  }
  if (p->mode != PHD_MODE_EXACT && p->mode != PHD_MODE_DCP) return fail(c, PHD_EINVAL, "mode %d", p->mode);
  if (p->reserved0 != 0) return fail(c, PHD_EINVAL, "reserved0 must be 0");
  if (p->exchange_count < 0) return fail(c, PHD_EINVAL, "exchange_count < 0");
  if (p->birth_model < 0 || p->birth_model > 2) return fail(c, PHD_EINVAL, "birth_model %d", p->birth_model);
  if (p->birth_model == 2) {
    if (!(p->birth_sigma_v > 0)) return fail(c, PHD_EINVAL, "birth_model 2 needs birth_sigma_v > 0");
    for (int i = 0; i < 4; ++i)
      if (!(p->birth_std[i] > 0)) return fail(c, PHD_EINVAL, "birth_model 2 needs birth_std > 0");
    if (p->meas == PHD_MEAS_RANGE_BEARING && p->region[0] < 0)
      return fail(c, PHD_EINVAL, "birth_model 2 needs a range region with rmin >= 0");
  }
  if (!(p->proposal_scale >= 0 && p->proposal_scale <= 1e3)) return fail(c, PHD_EINVAL, "proposal_scale outside [0, 1e3]");
  if (p->gate_floor != 0 && (p->gate_floor < -126 || p->gate_floor > -20))
    return fail(c, PHD_EINVAL, "gate_floor %d: 0 (exact) or in [-126, -20]", p->gate_floor);
  if (p->gate < 0 || p->gate > 2) return fail(c, PHD_EINVAL, "gate must be 0, 1 or 2");
  if (p->stphd_all != 0 && p->stphd_all != 1) return fail(c, PHD_EINVAL, "stphd_all must be 0 or 1");
  for (int i = 0; i < 4; ++i)
    if (!(p->birth_std[i] >= 0)) return fail(c, PHD_EINVAL, "birth_std must be >= 0");
  if (world < 1) return fail(c, PHD_EINVAL, "world < 1");
  return PHD_OK;
}

template <class T>
T* at(char* base, size_t off) {
  return reinterpret_cast<T*>(base + off);
}

void timing_record(phd_ctx* c, int i) {
  if (c->timing) cudaEventRecord(c->ev[i], c->st);
}

// DCP: the births of group `rank` are the block [jlo, jhi) of the J births (Step 1).
void group_births(const phd_ctx* c, int64_t* jlo, int64_t* jhi) {
  block_of(c->p.births_per_step, c->world, c->rank, jlo, jhi);
}

uint64_t dcp_space(const phd_ctx* c) { return ((uint64_t)0x40000000u << 32) | (uint64_t)c->rank; }

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

int32_t phd_abi_version(void) { return PHD_ABI_VERSION; }

const char* phd_status_str(phd_status s) {
  switch (s) {
    case PHD_OK: return "ok";
    case PHD_EINVAL: return "invalid argument";
    case PHD_ESTATE: return "call out of order";
    case PHD_ECAPACITY: return "capacity exceeded";
    case PHD_EMODEL: return "non-finite model quantity";
    case PHD_ENOMEM: return "out of device memory";
    case PHD_ECUDA: return "CUDA error";
    case PHD_ENCCL: return "NCCL error";
    case PHD_ENODEV: return "no CUDA device";
  }
  return "unknown status";
}

const char* phd_last_error(const phd_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void phd_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  U4 o = philox10(U4{ctr[0], ctr[1], ctr[2], ctr[3]}, key[0], key[1]);
  out[0] = o.x;
  out[1] = o.y;
  out[2] = o.z;
  out[3] = o.w;
}

phd_status phd_philox4x32_10_device(uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out, void* stream) {
  if (n < 0 || (n > 0 && (!ctr || !out))) return PHD_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (launch_philox_kat(seed, ctr, n, out, s) != cudaSuccess) return PHD_ECUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? PHD_OK : PHD_ECUDA;
}

phd_status phd_rank_block(int64_t n, int32_t world, int32_t rank, int64_t* lo, int64_t* hi) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi) return PHD_EINVAL;
  block_of(n, world, rank, lo, hi);
  return PHD_OK;
}

phd_status phd_resample_bounds(int32_t world, const double* W_r, int64_t n_out, double U, int64_t* bounds,
                               double* W_out) {
  if (world < 1 || !W_r || !bounds || n_out < 0) return PHD_EINVAL;
  double W = 0.0;
  for (int r = 0; r < world; ++r) W += W_r[r];
  if (W_out) *W_out = W;
  if (!(W > 0.0)) return PHD_EINVAL;
  double scale = (double)n_out / W;
  double O = 0.0;
  for (int r = 0; r < world; ++r) {
    bounds[r] = r == 0 ? 0 : n_of_host(O, scale, U, n_out);
    O += W_r[r];
  }
  bounds[world] = n_out;
  return PHD_OK;
}

phd_status phd_plan_exchange(int32_t world, int32_t rank, const int64_t* bounds, int64_t n_out, int64_t J,
                             int64_t* send_count, int64_t* send_off, int64_t* recv_count, int64_t* recv_off) {
  if (world < 1 || rank < 0 || rank >= world || !bounds) return PHD_EINVAL;
  int64_t Nn = n_out + J;
  for (int q = 0; q < world; ++q) {
    int64_t lo, hi;
    block_of(Nn, world, q, &lo, &hi);
    int64_t a = std::min(lo, n_out), b = std::min(hi, n_out);
    // what rank sends to q
    int64_t s0 = std::max(bounds[rank], a), s1 = std::min(bounds[rank + 1], b);
    send_count[q] = std::max<int64_t>(0, s1 - s0);
    send_off[q] = send_count[q] ? s0 - bounds[rank] : 0;
  }
  int64_t mlo, mhi;
  block_of(Nn, world, rank, &mlo, &mhi);
  int64_t a = std::min(mlo, n_out), b = std::min(mhi, n_out);
  for (int q = 0; q < world; ++q) {
    int64_t r0 = std::max(bounds[q], a), r1 = std::min(bounds[q + 1], b);
    recv_count[q] = std::max<int64_t>(0, r1 - r0);
    recv_off[q] = recv_count[q] ? r0 - mlo : 0;
  }
  return PHD_OK;
}

phd_status phd_nccl_unique_id(uint8_t out[128]) { return nccl_unique_id(out) ? PHD_OK : PHD_ENCCL; }

struct phd_group {
  LocalGroup* g;
};

phd_status phd_group_create(int32_t world, phd_group** out) {
  if (!out || world < 1 || world > 16) return PHD_EINVAL;
  *out = new phd_group{local_group_create(world)};
  return PHD_OK;
}

void phd_group_destroy(phd_group* g) {
  if (!g) return;
  local_group_destroy(g->g);
  delete g;
}

phd_status phd_workspace_size(const phd_params* p, int32_t world, size_t* bytes) {
  phd_status s = validate(p, world, nullptr);
  if (s != PHD_OK) return s;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  *bytes = make_layout(p, world, sms).total;
  return PHD_OK;
}

static phd_status create_impl(const phd_params* p, int32_t rank, int32_t world, const uint8_t* nccl_id,
                              phd_group* group, int32_t device, void* stream, void* workspace, phd_ctx** out,
                              const phd_host_transport* ht = nullptr) {
  if (!out) return PHD_EINVAL;
  *out = nullptr;
  phd_ctx* c = new phd_ctx();
  phd_status s = validate(p, world, c);
  if (s == PHD_OK && (rank < 0 || rank >= world)) s = fail(c, PHD_EINVAL, "rank %d of world %d", rank, world);
  if (s != PHD_OK) {
    fprintf(stderr, "phd_create: %s\n", c->err.c_str());
    delete c;
    return s;
  }
  c->p = *p;
  c->rank = rank;
  c->world = world;
  c->device = device;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    delete c;
    return PHD_ENODEV;
  }
  auto bail = [&](phd_status st) {
    fprintf(stderr, "phd_create: %s\n", c->err.c_str());
    phd_destroy(c);
    return st;
  };
#define CUB(call)                                                                              \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return bail(fail(c, PHD_ECUDA, "%s: %s", #call, cudaGetErrorString(e_))); \
  } while (0)
  CUB(cudaSetDevice(device));
  CUB(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
  preload_kernels();  // no lazy kernel loading inside a step (first use of a variant)
  if (stream) {
    c->st = (cudaStream_t)stream;
  } else {
    CUB(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  c->L = make_layout(p, world, c->sms);
  if (workspace) {
    c->ws = (char*)workspace;
  } else {
    cudaError_t e = cudaMalloc(&c->ws, c->L.total);
    if (e != cudaSuccess) return bail(fail(c, PHD_ENOMEM, "cudaMalloc(%zu): %s", c->L.total, cudaGetErrorString(e)));
    c->own_ws = true;
  }
  const Layout& L = c->L;
  for (int i = 0; i < 5; ++i) {
    c->A[i] = at<float>(c->ws, L.o_A[i]);
    c->B[i] = at<float>(c->ws, L.o_B[i]);
    c->s[i] = at<float>(c->ws, L.o_s[i]);
  }
  c->wn = at<float>(c->ws, L.o_wn);
  c->rb = p->meas == PHD_MEAS_RANGE_BEARING ? at<float>(c->ws, L.o_rb) : nullptr;
  c->P = at<float>(c->ws, L.o_P);
  c->rec = at<float>(c->ws, L.o_rec);
  c->Cpart = at<double>(c->ws, L.o_Cpart);
  c->Apart = at<double>(c->ws, L.o_Apart);
  c->zlab = at<float>(c->ws, L.o_zlab);
  c->zprev = at<float>(c->ws, L.o_zprev);
  c->slot_label = at<int32_t>(c->ws, L.o_slot);
  c->rep = at<int32_t>(c->ws, L.o_rep);
  c->C = at<double>(c->ws, L.o_C);
  c->C_slot = at<double>(c->ws, L.o_Cslot);
  c->sel_flag = at<int32_t>(c->ws, L.o_sel);
  c->sel_info = at<double>(c->ws, L.o_selinfo);
  c->s_lim = reinterpret_cast<int32_t*>(c->sel_info + 6);
  c->D = at<double>(c->ws, L.o_D);
  // C2 buffer: the rank slots [W_r | W_pred_r | N_r] (3 per rank) first, at a fixed
  // offset, then the label accumulators [M][5] -- one contiguous all-reduce of 3W + 5M
  c->rslots = at<double>(c->ws, L.o_acc);
  c->acc = c->rslots + align_up((size_t)3 * world, 4);
  c->blk_w = at<double>(c->ws, L.o_blk_w);
  c->blk_wp = at<double>(c->ws, L.o_blk_wp);
  c->blk_off = at<double>(c->ws, L.o_blk_off);
  c->ctot = at<double>(c->ws, L.o_ctot);
  c->coff = at<double>(c->ws, L.o_coff);
  c->scan_counter = at<unsigned>(c->ws, L.o_counter);
  c->dstep = at<DevStep>(c->ws, L.o_step);
  c->anc = at<int32_t>(c->ws, L.o_anc);
  c->est = at<phd_estimate>(c->ws, L.o_est);
  c->gather = at<phd_estimate>(c->ws, L.o_gather);
  c->ring = at<double>(c->ws, L.o_ring);
  c->dcp = p->mode == PHD_MODE_DCP;
  c->summ = at<double>(c->ws, L.o_summ);
  c->bad = at<int>(c->ws, L.o_bad);
  if (p->gate != 0) {
    c->gso.inv = at<int32_t>(c->ws, L.o_ginv);
    c->gkeys = at<int32_t>(c->ws, L.o_gkeys);
    c->gso.rec = at<float4>(c->ws, L.o_gsorted[0]);
    c->gso.n4 = p->meas == PHD_MEAS_RANGE_BEARING ? 4 : 2;
    c->gso.lw_max = at<int>(c->ws, L.o_glwmax);
    c->gPs = at<float>(c->ws, L.o_gPs);
    c->ghist = at<int32_t>(c->ws, L.o_ghist);
    c->gscan = at<int32_t>(c->ws, L.o_gscan);
    c->gtstart = at<int32_t>(c->ws, L.o_gtstart);
    c->gcand = at<int32_t>(c->ws, L.o_gcand);
    c->gk = at<int32_t>(c->ws, L.o_gk);
    c->gv = at<int32_t>(c->ws, L.o_gv);
    c->gmlist = at<int32_t>(c->ws, L.o_gmlist);
    c->gpart1 = at<double>(c->ws, L.o_gpart1);
    c->gpart2 = at<float>(c->ws, L.o_gpart2);
    c->gmstart = at<int32_t>(c->ws, L.o_gmstart);
    c->gzstart = at<int32_t>(c->ws, L.o_gzstart);
    c->gzitems = at<int32_t>(c->ws, L.o_gzitems);
    c->gzz = at<float2>(c->ws, L.o_gzz);
    c->gcbuf = at<int32_t>(c->ws, L.o_gcbuf);
    c->gA = at<double>(c->ws, L.o_gA);
    if (p->meas == PHD_MEAS_RANGE_BEARING) {
      c->ggrid.lo0 = (float)p->region[0];
      c->ggrid.inv_h0 = (float)(kGateG / (p->region[1] - p->region[0]));
      c->ggrid.lo1 = (float)-kPi;
      c->ggrid.inv_h1 = (float)(kGateG / (2.0 * kPi));
      c->ggrid.wrap1 = 1;
      c->ggrid.floor = p->gate_floor != 0 ? (float)p->gate_floor : kGateLog2Min;
      c->ggrid.kbuf = gate_kbuf(p->max_meas);
    } else {
      c->ggrid.lo0 = (float)p->region[0];
      c->ggrid.inv_h0 = (float)(kGateG / (p->region[1] - p->region[0]));
      c->ggrid.lo1 = (float)p->region[2];
      c->ggrid.inv_h1 = (float)(kGateG / (p->region[3] - p->region[2]));
      c->ggrid.wrap1 = 0;
      c->ggrid.floor = p->gate_floor != 0 ? (float)p->gate_floor : kGateLog2Min;
      c->ggrid.kbuf = gate_kbuf(p->max_meas);
    }
  }
  CUB(cudaMallocHost(&c->h_meta, sizeof(double) * (48 + 4 * world)));
  CUB(cudaMallocHost(&c->h_est, sizeof(phd_estimate) * (p->max_meas + 1)));
  if (c->dcp) CUB(cudaMallocHost(&c->h_gather, sizeof(phd_estimate) * (p->max_meas + 1) * world));
  CUB(cudaMallocHost(&c->h_z, sizeof(float) * 2 * (p->max_meas + 1)));
  CUB(cudaMallocHost(&c->h_stepin, sizeof(int32_t) * 4));
  CUB(cudaMallocHost(&c->h_stepout, sizeof(DevStep)));
  // device aliases of the pinned result buffers k_step_out stores into (UVA: the same
  // addresses on this platform; asked for, not assumed)
  CUB(cudaHostGetDevicePointer((void**)&c->hd_meta, c->h_meta, 0));
  CUB(cudaHostGetDevicePointer((void**)&c->hd_est, c->h_est, 0));
  CUB(cudaHostGetDevicePointer((void**)&c->hd_stepout, c->h_stepout, 0));
  for (int i = 0; i < 16; ++i) CUB(cudaEventCreate(&c->ev[i]));
  CUB(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
  CUB(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
  CUB(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
  CUB(cudaEventCreateWithFlags(&c->ev_plan, cudaEventDisableTiming));
  // derived model constants (fp32 for the pair kernels, fp64 for kappa)
  double s0 = p->sigma_z[0], s1 = p->sigma_z[1];
  bool rbm = p->meas == PHD_MEAS_RANGE_BEARING;
  c->model = rbm ? kRangeBearing : (s0 == s1 ? kPosIso : kPosAniso);
  c->na0 = (float)(-kLog2e / (2.0 * s0 * s0));
  c->na1 = (float)(-kLog2e / (2.0 * s1 * s1));
  c->wscale = (float)(p->p_d / (2.0 * kPi * s0 * s1));
  c->nu = (float)(1.0 - p->p_d);
  c->kappa = p->clutter_rate / ((p->region[1] - p->region[0]) * (p->region[3] - p->region[2]));
  c->Wr.assign(world, 0.0);
  c->Wpr.assign(world, 0.0);
  if (world > 1) {
    std::string e;
    if (group) {
      c->comm = make_local_comm(group->g, rank, device, &e);
    } else if (ht) {
      HostTransport t{ht->user, reinterpret_cast<int (*)(void*, double*, size_t)>(ht->allreduce_f64),
                      reinterpret_cast<int (*)(void*, const void*, void*, size_t)>(ht->allgather_bytes)};
      c->comm = make_host_comm(t, world, rank, &e);
    } else {
      if (!nccl_id) return bail(fail(c, PHD_EINVAL, "nccl_id required for world > 1"));
      c->comm = make_nccl_comm(nccl_id, world, rank, &e);
    }
    if (!c->comm) return bail(fail(c, PHD_ENCCL, "%s", e.c_str()));
  }
  CUB(cudaMemsetAsync(c->ws, 0, L.total, c->st));
  {
    // particle double buffers of the peer-memory window (world > 1, exact mode), mapped
    // by the other ranks at the first resampling (p2p_setup); allocated here so that no
    // step allocates.  A failed allocation just keeps the send/recv exchange.
    const char* xch = getenv("PHD_EXCHANGE");
    if (world > 1 && !c->dcp && world <= kMaxPeers && !(xch && strcmp(xch, "nccl") == 0)) {
      const size_t bytes = sizeof(float) * 5 * (size_t)L.cap_l;
      for (int b = 0; b < 2; ++b) {
        if (cudaMalloc(&c->pbuf[b], bytes) != cudaSuccess) {
          c->pbuf[b] = nullptr;
          cudaGetLastError();
        } else {
          CUB(cudaMemsetAsync(c->pbuf[b], 0, bytes, c->st));
        }
      }
    }
  }
  CUB(cudaStreamSynchronize(c->st));

#undef CUB
  *out = c;
  return PHD_OK;
}

phd_status phd_create(const phd_params* p, int32_t rank, int32_t world, const uint8_t* nccl_id, int32_t device,
                      void* stream, void* workspace, phd_ctx** out) {
  return create_impl(p, rank, world, nccl_id, nullptr, device, stream, workspace, out);
}

phd_status phd_create_with_transport(const phd_params* p, int32_t rank, int32_t world, const phd_host_transport* t,
                                     int32_t device, void* stream, void* workspace, phd_ctx** out) {
  if (!t) return PHD_EINVAL;
  return create_impl(p, rank, world, nullptr, nullptr, device, stream, workspace, out, t);
}

phd_status phd_create_in_group(const phd_params* p, phd_group* g, int32_t rank, int32_t device, void* stream,
                               void* workspace, phd_ctx** out) {
  if (!g) return PHD_EINVAL;
  return create_impl(p, rank, local_group_world(g->g), nullptr, g, device, stream, workspace, out);
}

void phd_destroy(phd_ctx* c) {
  if (!c) return;
  if (c->st) cudaStreamSynchronize(c->st);
  delete c->comm;
  for (int b = 0; b < 2; ++b)
    if (c->pbuf[b]) cudaFree(c->pbuf[b]);
  for (int i = 0; i < 16; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->ev_plan) cudaEventDestroy(c->ev_plan);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->own_ws && c->ws) cudaFree(c->ws);
  if (c->h_meta) cudaFreeHost(c->h_meta);
  if (c->h_est) cudaFreeHost(c->h_est);
  if (c->h_gather) cudaFreeHost(c->h_gather);
  if (c->h_z) cudaFreeHost(c->h_z);
  if (c->h_stepin) cudaFreeHost(c->h_stepin);
  if (c->h_stepout) cudaFreeHost(c->h_stepout);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  delete c;
}

int64_t phd_launch_count(const phd_ctx* c) { return c ? c->launches : 0; }

int32_t phd_exchange_path(const phd_ctx* c) {
  if (!c || c->world <= 1 || c->dcp) return 0;
  return c->p2p_state == 1 ? 2 : 1;
}

phd_status phd_set_timing(phd_ctx* c, int32_t enable) {
  if (!c) return PHD_EINVAL;
  c->timing = enable != 0;
  return PHD_OK;
}

phd_status phd_get_timing(phd_ctx* c, float* ms) {
  if (!c || !ms) return PHD_EINVAL;
  cudaSetDevice(c->device);
  CU(cudaStreamSynchronize(c->st));
  for (int i = 0; i < 8; ++i) ms[i] = c->t_ms[i];
  return PHD_OK;
}

// ---------------------------------------------------------------------------
phd_status phd_set_particles(phd_ctx* c, const float* soa4, const float* w, int64_t n_local, int64_t n_global,
                             double mass, int32_t stage) {
  if (!c || !soa4) return PHD_EINVAL;
  cudaSetDevice(c->device);
  c->err.clear();
  int64_t J = c->p.births_per_step;
  int64_t lo = 0, hi = 0;
  if (c->dcp) {
    // every rank is a group with its own population (n_global ignored)
    int64_t jlo, jhi;
    group_births(c, &jlo, &jhi);
    n_global = n_local;
    int64_t need = stage == PHD_STAGE_PREDICTED ? n_local : n_local + (jhi - jlo);
    if (n_local < 0 || need > c->L.cap_l - 1) return fail(c, PHD_ECAPACITY, "group size %lld exceeds capacity", (long long)need);
    hi = n_local;
  } else {
    int64_t Nblk = stage == PHD_STAGE_PREDICTED ? n_global : n_global + J;
    if (n_global < 0 || Nblk > c->p.capacity) return fail(c, PHD_ECAPACITY, "n_global %lld exceeds capacity", (long long)n_global);
    block_of(Nblk, c->world, c->rank, &lo, &hi);
    int64_t expect = stage == PHD_STAGE_PREDICTED ? hi - lo : std::max<int64_t>(0, std::min(hi, n_global) - std::min(lo, n_global));
    if (n_local != expect)
      return fail(c, PHD_EINVAL, "n_local %lld != %lld (rank block of %lld)", (long long)n_local, (long long)expect, (long long)Nblk);
  }
  for (int i = 0; i < 4; ++i)
    CU(cudaMemcpyAsync(c->A[i], soa4 + (size_t)i * n_local, sizeof(float) * n_local, cudaMemcpyDefault, c->st));
  if (w) {
    CU(cudaMemcpyAsync(c->A[4], w, sizeof(float) * n_local, cudaMemcpyDefault, c->st));
  } else {
    KL(launch_fill(c->A[4], (float)(n_global > 0 ? mass / (double)n_global : 0.0), n_local, c->st));
  }
  if (stage == PHD_STAGE_PREDICTED) {
    c->N = n_global;
    c->n_out = n_global;
    c->n_local = n_local;
    c->g0 = lo;
    if (c->rb) KL(launch_rb_repr(c->A[0], c->A[2], n_local, (float)c->p.sensor_xy[0], (float)c->p.sensor_xy[1], c->rb, c->L.cap_l, c->st));
    c->stage = kPredicted;
  } else {
    c->n_out = n_global;
    c->n_surv_local = n_local;
    c->stage = kResampled;
  }
  c->populated = true;
  CU(cudaStreamSynchronize(c->st));
  return PHD_OK;
}

phd_status phd_init_population(phd_ctx* c, double total_mass, const double* box, const double* mass_box,
                               double v_max) {
  NvtxRange nvtx_("phd_init_population");
  if (!c) return PHD_EINVAL;
  cudaSetDevice(c->device);
  c->err.clear();
  if (!(total_mass >= 0.0) || !std::isfinite(total_mass)) return fail(c, PHD_EINVAL, "total_mass must be finite and >= 0");
  if (!(v_max >= 0.0) || !std::isfinite(v_max)) return fail(c, PHD_EINVAL, "v_max must be finite and >= 0");
  double b[4];
  if (box) {
    for (int i = 0; i < 4; ++i) b[i] = box[i];
  } else if (c->p.meas == PHD_MEAS_POSITION) {
    for (int i = 0; i < 4; ++i) b[i] = c->p.region[i];
  } else {  // range-bearing: the Cartesian square of side r_max centred on the sensor (S27)
    const double h = 0.5 * c->p.region[1];
    b[0] = c->p.sensor_xy[0] - h;
    b[1] = c->p.sensor_xy[0] + h;
    b[2] = c->p.sensor_xy[1] - h;
    b[3] = c->p.sensor_xy[1] + h;
  }
  for (int i = 0; i < 4; ++i)
    if (!std::isfinite(b[i]) || (mass_box && std::isnan(mass_box[i]))) return fail(c, PHD_EINVAL, "non-finite box");
  if (!(b[1] > b[0] && b[3] > b[2])) return fail(c, PHD_EINVAL, "empty box");
  // population size: N_out of the count mode (adaptive: max(round(m0), 1) R, clamped as next_count)
  int64_t n_out;
  int clamped = 0;
  if (c->p.count_mode == PHD_COUNT_FIXED) {
    n_out = c->p.fixed_count;
  } else {
    const int64_t m0 = std::max<int64_t>(1, (int64_t)std::floor(total_mass + 0.5));
    n_out = m0 * c->p.particles_per_target;
    const int64_t lim = c->p.capacity - c->p.births_per_step;
    if (m0 > lim / c->p.particles_per_target || n_out > lim) {
      n_out = lim;
      clamped = 1;
    }
  }
  InitArgs a{};
  int64_t lo, hi;
  if (c->dcp) {  // group j holds block j of the population, with its own mass (omega_0 = 1/M per group)
    block_of(n_out, c->world, c->rank, &lo, &hi);
    int64_t jlo, jhi;
    group_births(c, &jlo, &jhi);
    if ((hi - lo) + (jhi - jlo) > c->L.cap_l - 1) return fail(c, PHD_ECAPACITY, "group size exceeds capacity");
  } else {
    block_of(n_out + c->p.births_per_step, c->world, c->rank, &lo, &hi);
    lo = std::min(lo, n_out);
    hi = std::min(hi, n_out);
  }
  a.n_local = hi - lo;
  a.g0 = lo;
  a.n_out = n_out;
  a.seed = c->p.seed;
  for (int i = 0; i < 4; ++i) a.box[i] = b[i];
  a.v_max = v_max;
  a.has_mbox = mass_box != nullptr;
  if (mass_box)
    for (int i = 0; i < 4; ++i) a.mbox[i] = mass_box[i];
  a.total_mass = total_mass;
  a.n_norm = c->dcp ? (double)(hi - lo) : (double)n_out;
  a.x = c->A[0];
  a.vx = c->A[1];
  a.y = c->A[2];
  a.vy = c->A[3];
  a.w = c->A[4];
  a.count = c->ring;  // scratch (the DCP ring counts are rewritten at every resampling)
  if (a.has_mbox) CU(cudaMemsetAsync(a.count, 0, sizeof(double), c->st));
  KL(launch_init_population(a, c->st));
  if (a.has_mbox) {
    if (c->world > 1 && !c->dcp) COMM(c->comm->allreduce_f64(a.count, 1, c->st));
    KL(launch_init_weights(a, c->st));
  }
  c->n_out = c->dcp ? hi - lo : n_out;
  c->n_surv_local = hi - lo;
  c->count_clamped = clamped;
  c->M_z = -1;  // t = 0: no Z_{k-1}, the first births are uniform over the region
  c->stage = kResampled;
  c->populated = true;
  return PHD_OK;
}

phd_status phd_set_retained_measurements(phd_ctx* c, const float* z, int32_t M) {
  if (!c) return PHD_EINVAL;
  cudaSetDevice(c->device);
  c->err.clear();
  if (M < 0 || M > c->p.max_meas) return fail(c, PHD_EINVAL, "M = %d outside [0, max_meas = %d]", M, c->p.max_meas);
  if (M > 0 && !z) return fail(c, PHD_EINVAL, "z is NULL");
  if (M > 0) {
    CU(cudaMemcpyAsync(c->zlab, z, sizeof(float) * 2 * M, cudaMemcpyDefault, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  c->M_z = M;
  return PHD_OK;
}

phd_status phd_get_particles(phd_ctx* c, float* soa4, float* w, int64_t cap, int64_t* n_local, int64_t* global_offset) {
  if (!c) return PHD_EINVAL;
  cudaSetDevice(c->device);
  int64_t n, g0;
  if (c->stage == kResampled) {
    int64_t lo = 0, hi;
    if (!c->dcp) block_of(c->n_out + c->p.births_per_step, c->world, c->rank, &lo, &hi);
    n = c->n_surv_local;
    g0 = lo;
  } else {
    n = c->n_local;
    g0 = c->g0;
  }
  if (n_local) *n_local = n;
  if (global_offset) *global_offset = g0;
  if (cap < n) return fail(c, PHD_EINVAL, "cap %lld < %lld", (long long)cap, (long long)n);
  if (soa4)
    for (int i = 0; i < 4; ++i) CU(cudaMemcpyAsync(soa4 + (size_t)i * n, c->A[i], sizeof(float) * n, cudaMemcpyDeviceToHost, c->st));
  if (w) CU(cudaMemcpyAsync(w, c->stage == kUpdated ? c->wn : c->A[4], sizeof(float) * n, cudaMemcpyDeviceToHost, c->st));
  CU(cudaStreamSynchronize(c->st));
  return PHD_OK;
}

phd_status phd_predict(phd_ctx* c, int32_t k, const float* z_prev, int32_t M_prev) {
  NvtxRange nvtx_("phd_predict");
  if (!c) return PHD_EINVAL;
  cudaSetDevice(c->device);
  c->err.clear();
  if (!c->populated || c->stage != kResampled) return fail(c, PHD_ESTATE, "phd_predict needs a resampled population");
  if (k < 1) return fail(c, PHD_EINVAL, "k must be >= 1");
  if (z_prev && (M_prev < 0 || M_prev > c->p.max_meas)) return fail(c, PHD_EINVAL, "M_prev %d out of range", M_prev);
  timing_record(c, 0);
  const float* zp = nullptr;
  int mp = 0;
  if (z_prev) {
    if (M_prev > 0) CU(cudaMemcpyAsync(c->zprev, z_prev, sizeof(float) * 2 * M_prev, cudaMemcpyDefault, c->st));
    zp = c->zprev;
    mp = M_prev;
  } else if (c->M_z >= 0) {
    zp = c->zlab;  // Z retained by the last update
    mp = c->M_z;
  }
  int64_t J = c->p.births_per_step;
  PredictArgs a{};
  if (c->dcp) {
    // group-local array [survivors, births of this group]; own Philox counter space
    int64_t jlo, jhi;
    group_births(c, &jlo, &jhi);
    c->N = c->n_out + (jhi - jlo);
    c->g0 = 0;
    c->n_local = c->N;
    if (c->N > c->L.cap_l - 1) return fail(c, PHD_ECAPACITY, "group size %lld exceeds capacity", (long long)c->N);
    a.ctr_base = c->world > 1 ? ((uint64_t)(0x40000000u + (uint32_t)c->rank)) << 32 : 0;  // c3 = 0x40000000 + j
    a.birth_offset = jlo;
    a.J = jhi - jlo;
  } else {
    c->N = c->n_out + J;
    block_of(c->N, c->world, c->rank, &c->g0, &c->n_local);
    c->n_local -= c->g0;
    a.ctr_base = 0;
    a.birth_offset = 0;
    a.J = J;
  }
  a.n_local = c->n_local;
  a.g0 = c->g0;
  a.n_out = c->n_out;
  a.k = k;
  a.seed = c->p.seed;
  a.T = (float)c->p.T;
  const double prop_s = c->p.proposal_scale > 0 ? c->p.proposal_scale : 1.0;
  a.sigma_a = (float)(prop_s * c->p.sigma_a);  // the proposal's noise std (Eq 5)
  a.prop_s = (float)prop_s;
  a.p_s = (float)c->p.p_s;
  a.w_uniform = -1.0f;
  a.meas = c->p.meas;
  a.sigma_z0 = (float)c->p.sigma_z[0];
  a.sigma_z1 = (float)c->p.sigma_z[1];
  a.sensor_x = (float)c->p.sensor_xy[0];
  a.sensor_y = (float)c->p.sensor_xy[1];
  for (int i = 0; i < 4; ++i) a.region[i] = (float)c->p.region[i];
  // Eq 6 weight gamma / J_k; a DCP group is a full-intensity PHD filter with its own J_k births
  a.birth_w = a.J > 0 ? (float)(c->p.birth_mass / (double)a.J) : 0.0f;
  a.birth_sigma_v = (float)c->p.birth_sigma_v;
  a.birth_model = c->p.birth_model;
  for (int i = 0; i < 4; ++i) {
    a.birth_mean[i] = (float)c->p.birth_mean[i];
    a.birth_std[i] = (float)c->p.birth_std[i];
  }
  a.zprev = zp;
  a.m_prev = mp;
  if (c->capturing) {  // graph replay: k and M_{k-1} from the device step block, Z_{k-1} in zlab
    a.zprev = c->zlab;
    a.ds = c->dstep;
  }
  a.x = c->A[0];
  a.vx = c->A[1];
  a.y = c->A[2];
  a.vy = c->A[3];
  a.w = c->A[4];
  a.rb = c->rb;
  a.rb_stride = c->L.cap_l;
  KL(launch_predict(a, c->st));
  if (c->p.birth_model == 2) {
    // Eq 6 importance weights of this rank's births (slots with global index >= n_out)
    BirthISArgs b{};
    b.i0 = std::max<int64_t>(0, a.n_out - a.g0);
    b.nb = std::max<int64_t>(0, a.n_local - b.i0);
    b.J = a.J;
    b.birth_offset = a.birth_offset;
    b.meas = c->p.meas;
    b.sigma_z0 = c->p.sigma_z[0];
    b.sigma_z1 = c->p.sigma_z[1];
    b.sensor_x = c->p.sensor_xy[0];
    b.sensor_y = c->p.sensor_xy[1];
    for (int i = 0; i < 4; ++i) {
      b.region[i] = c->p.region[i];
      b.birth_mean[i] = c->p.birth_mean[i];
      b.birth_std[i] = c->p.birth_std[i];
    }
    b.gamma = c->p.birth_mass;
    b.birth_sigma_v = c->p.birth_sigma_v;
    b.zprev = zp;
    b.m_prev = mp;
    b.x = a.x;
    b.vx = a.vx;
    b.y = a.y;
    b.vy = a.vy;
    b.w = a.w;
    if (b.nb > 0) KL(launch_birth_is(b, c->st));
  }
  timing_record(c, 1);
  c->stage = kPredicted;
  return PHD_OK;
}

// Slot layout parameters of the dense passes: a function of M only (the slot -> label map
// itself is built on the device by k_build_slots).  Range-bearing: measurements grouped by
// bearing class with pair padding (<= M + 3 slots), room for the pass-2 layout (M + 6).
static phd_status build_slots(phd_ctx* c, int M) {
  int n = M;
  if (c->model == kRangeBearing && M > 0) n = M + 6;
  c->n_slots = n;
  {
  // slots per lane: 8 (halves the per-particle overheads) unless it pads much more than 4;
  // warps per CTA: the fewest padded slots among {the warps needed, 8, 4, 2} (ties: more
  // warps).  Padding slots cost full pair work: cfg 4 (M ~ 3000) pads to 4096 slots with
  // 8 warps but 3072 with 4 (update 6.06 -> 5.79 ms measured)
  int best_zl = 4, best_wz = 2, best_zb = 1;
  int64_t best_pad = -1;
  for (int zl : {8, 4}) {
    const int64_t per_warp = 32 * zl;
    const int need = (int)std::min<int64_t>(max_warps_z(zl), std::max<int64_t>(kMinWarpsZ, ceil_div(std::max(n, 1), per_warp)));
    int wz_z = need;
    int64_t pad_z = -1;
    for (int cand : {need, 16, 8, 4, 2}) {
      const int wz = std::min(max_warps_z(zl), std::max(kMinWarpsZ, cand));
      const int64_t pad = ceil_div(std::max(n, 1), (int64_t)wz * per_warp) * wz * per_warp;
      if (pad_z < 0 || pad < pad_z || (pad == pad_z && wz > wz_z)) {
        pad_z = pad;
        wz_z = wz;
      }
    }
    if (best_pad < 0 || pad_z < best_pad - std::max(n, 16) / 16) {
      best_pad = pad_z;
      best_zl = zl;
      best_wz = wz_z;
      best_zb = (int)ceil_div(std::max(n, 1), (int64_t)wz_z * per_warp);
    }
  }
  if (const char* fz = getenv("PHD_FORCE_ZL")) {  // tuning experiments only
    int zl = atoi(fz);
    if (zl == 4 || zl == 8) {
      best_zl = zl;
      best_wz = (int)std::min<int64_t>(max_warps_z(zl), std::max<int64_t>(kMinWarpsZ, ceil_div(std::max(n, 1), 32 * zl)));
      best_zb = (int)ceil_div(std::max(n, 1), (int64_t)best_wz * 32 * zl);
      best_pad = (int64_t)best_zb * best_wz * 32 * zl;
    }
  }
  c->zl = best_zl;
  c->wz = best_wz;
  c->zb = M > 0 ? best_zb : 0;
  c->slots_pad = (int)best_pad;
  }
  // the P planes and the slot arrays are sized for the worst layout (make_layout)
  if (c->slots_pad > c->L.slots_max || c->zb > c->L.zb_max)
    return fail(c, PHD_ECAPACITY, "slot layout %d slots / %d z-blocks exceeds %d / %d", c->slots_pad, c->zb,
                c->L.slots_max, c->L.zb_max);
  return PHD_OK;
}

// Gated update (DESIGN.md §5 "Gated update"): identity slot layout (slot = label).
static void gate_slots(phd_ctx* c, int M) {
  c->n_slots = M;
  c->slots_pad = std::max(2, (M + 1) & ~1);
  c->zl = 4;
  c->wz = kMinWarpsZ;
  c->zb = M > 0 ? 1 : 0;
}

// Sort the particles by cell, bin Z_k, count every tile's candidates; decide
// (collectively for world > 1: every rank must use the same slot layout).
static phd_status gate_plan(phd_ctx* c, int M, int64_t n, bool* use) {
  *use = false;
  const int tp = gate_tp(c->model);
  const int64_t npad = ceil_div(n, tp) * tp;
  const int ntiles = (int)(npad / tp);
  const float* A[5] = {c->A[0], c->A[1], c->A[2], c->A[3], c->A[4]};
  c->gso.n = n;
  c->gso.bad = c->bad;
  CU(gate_sort_particles(c->model, A, c->rb, c->L.cap_l, n, npad, c->wscale, c->ggrid, c->ghist, c->gscan,
                         c->gkeys, c->gso, c->st, &c->launches, c->blk_wp, &c->g_nwb));
  CU(gate_zbin(c->zlab, M, c->ggrid, c->ghist, c->gscan, c->gzstart, c->gzitems, c->gzz, c->st, &c->launches));
  int64_t tot = 0;
  if (ntiles > 0) {
    KL(gate_tiles(0, c->model, c->gso, ntiles, c->na0, c->na1, c->ggrid, c->gzstart, c->gzitems, c->gzz, c->gtstart,
                  nullptr, c->gcbuf, nullptr, c->st));
    CU(gate_scan(c->gtstart, ntiles, c->gscan, c->st, &c->launches));
    int32_t* h = reinterpret_cast<int32_t*>(c->h_meta + 3 * c->world + 40);
    CU(cudaMemcpyAsync(h, c->gtstart + ntiles, sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
    CU(cudaEventRecord(c->ev_plan, c->st));
    // the candidate fill runs while the host waits for the total (bounded by the workspace;
    // unused if the update then runs dense)
    KL(gate_tiles(1, c->model, c->gso, ntiles, c->na0, c->na1, c->ggrid, c->gzstart, c->gzitems, c->gzz, nullptr,
                  c->gtstart, c->gcbuf, c->gcand, c->st, c->L.g_ecap));
    CU(cudaEventSynchronize(c->ev_plan));
    tot = *h;
  }
  c->g_entries = tot;
  c->g_tiles = ntiles;
  const bool fits = tot <= c->L.g_ecap;
  // gate = 1 runs dense when the candidates are most of the pairs
  const bool pays = (double)tot * tp <= 0.5 * (double)n * (double)M;
  double veto = (fits && (c->p.gate == 2 || pays)) ? 0.0 : 1.0;
  if (c->world > 1) {
    double* d = c->C_slot;  // scratch: rewritten by the update
    c->h_meta[3 * c->world + 44] = veto;
    CU(cudaMemcpyAsync(d, c->h_meta + 3 * c->world + 44, sizeof(double), cudaMemcpyHostToDevice, c->st));
    COMM(c->comm->allreduce_f64(d, 1, c->st));
    CU(cudaMemcpyAsync(c->h_meta + 3 * c->world + 44, d, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    veto = c->h_meta[3 * c->world + 44];
  }
  *use = veto == 0.0;
  return PHD_OK;
}

static phd_status update_finish(phd_ctx* c);

// particle-CTA count and record-tile size of the dense passes: one wave of resident CTAs
// over the z-blocks; small populations (fewer than two CTAs' worth of kTileP tiles per
// SM) take kTileSmall tiles so that they still fill the SMs (measured: cfg 2, 8 tiles of
// 256, passes 37 -> 21 us with 64; cfg 3 keeps 256; PHD_TILE=64|256 forces a size)
static int plan_gp(phd_ctx* c, int64_t n) {
  int occ = std::min(pass_occupancy(c->model, 1, c->wz, c->zl), pass_occupancy(c->model, 2, c->wz, c->zl));
  occ = std::max(1, occ);
  int64_t want = std::max<int64_t>(1, (int64_t)occ * c->sms / std::max(1, c->zb));
  int tile = kTileP;
  const char* e = getenv("PHD_TILE");
  if (e && *e) {
    if (atoi(e) == kTileSmall) tile = kTileSmall;
  } else if (ceil_div(n, kTileP) * std::max(1, c->zb) < 2 * (int64_t)c->sms) {
    tile = kTileSmall;
  }
  c->tile = tile;
  const int64_t tiles = ceil_div(n, tile);
  int64_t cap_gp = std::max<int64_t>(1, c->L.part_cap / c->slots_pad);
  int gp = (int)std::min<int64_t>(std::min(want, cap_gp), tiles);
  int64_t tpc = ceil_div(tiles, gp);
  return (int)ceil_div(tiles, tpc);
}
// pass-2 state-sum layout: 0 automatic, 1 per-lane slot pairs, 2 whole z-blocks (PHD_SUM_LAYOUT, tests)
static int sum_layout() {
  const char* e = getenv("PHD_SUM_LAYOUT");
  if (e && strcmp(e, "lane") == 0) return 1;
  if (e && strcmp(e, "zblock") == 0) return 2;
  return 0;
}
constexpr int64_t kEstEager = 256;  // estimates copied with the summary inside phd_step

phd_status phd_update(phd_ctx* c, const float* z, int32_t M) {
  NvtxRange nvtx_("phd_update");
  if (!c) return PHD_EINVAL;
  cudaSetDevice(c->device);
  c->err.clear();
  if (c->stage != kPredicted) return fail(c, PHD_ESTATE, "phd_update needs a predicted population");
  if (M < 0 || M > c->p.max_meas) return fail(c, PHD_EINVAL, "M = %d outside [0, max_meas = %d]", M, c->p.max_meas);
  if (M > 0 && !z) return fail(c, PHD_EINVAL, "z is NULL");
  timing_record(c, 2);
  c->M = M;
  // gate = 1 skips the gated path for small updates (< 2^29 pairs, where the cell
  // sort and candidate lists cost more than the dense passes: measured at cfg 3,
  // 6.8e7 pairs, 0.28 ms dense vs 0.50 ms gated).  N is global in exact mode, so
  // every rank takes the same branch; DCP groups always plan (collectively).
  const bool small = c->p.gate == 1 && !c->dcp && (double)c->N * (double)M < 536870912.0;
  // the candidate offsets are an int32 scan: at most M candidates per tile, so a
  // capacity whose tiles x M could exceed INT32_MAX runs dense (same on every rank)
  const bool fits32 = (double)c->L.g_ntiles * (double)M <= (double)INT32_MAX;
  const bool try_gate = c->p.gate != 0 && M > 0 && !small && fits32;
  // one-sync step with a device-resident Z and no gate plan (which reads zlab): the slot
  // layout kernel reads Z where it is and leaves the copy in zlab (one launch, no copy)
  const float* z_slots = c->zlab;
  float* z_copy = nullptr;
  if (M > 0 && c->capturing) {
    // graph replay: Z_k staged by the host in the pinned h_z (after predict read Z_{k-1})
    CU(cudaMemcpyAsync(c->zlab, c->h_z, sizeof(float) * 2 * c->p.max_meas, cudaMemcpyHostToDevice, c->st));
  } else if (M > 0) {
    cudaPointerAttributes pa{};
    bool dev = cudaPointerGetAttributes(&pa, z) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    if (dev && c->dev_scalars && !try_gate) {
      z_slots = z;
      z_copy = c->zlab;
    } else if (dev) {  // device-resident Z stays on the device (the slot layout is built there)
      CU(cudaMemcpyAsync(c->zlab, z, sizeof(float) * 2 * M, cudaMemcpyDeviceToDevice, c->st));
    } else {
      memcpy(c->h_z, z, sizeof(float) * 2 * M);
      CU(cudaMemcpyAsync(c->zlab, c->h_z, sizeof(float) * 2 * M, cudaMemcpyHostToDevice, c->st));
    }
  }
  c->M_z = M;
  const int64_t n = c->n_local;
  bool gated = false;
  // non-finite counters (k_zconst: C/D; the gated sort: NaN particles), before any of them
  // runs; a one-sync step finds them cleared by the previous step's k_step_out
  if (!(c->dev_scalars && !c->capturing && c->bad_clean)) CU(cudaMemsetAsync(c->bad, 0, sizeof(int) * 4, c->st));
  c->bad_clean = false;
  if (try_gate) {
    phd_status st = gate_plan(c, M, n, &gated);
    if (st != PHD_OK) return st;
  }
  c->gated = gated;
  if (gated) {
    gate_slots(c, M);
  } else {
    phd_status st = build_slots(c, M);
    if (st != PHD_OK) return st;
  }
  BuildSlotsArgs bsa{};
  if (M > 0) {  // slot -> label map and per-slot constants, on the device
    SlotConsts sc{c->s[0], c->s[1], c->s[2], c->s[3], c->s[4], c->rep};
    bsa.z = z_slots;
    bsa.zcopy = z_copy;
    bsa.Mp = c->capturing ? &c->dstep->M : nullptr;
    bsa.M = M;
    bsa.model = c->model;
    bsa.identity = gated ? 1 : 0;
    bsa.slots_pad = c->slots_pad;
    bsa.slot_label = c->slot_label;
    bsa.sx = (float)c->p.sensor_xy[0];
    bsa.sy = (float)c->p.sensor_xy[1];
    bsa.sc = sc;
    bsa.bad = c->bad;
  }
  const int gp = M > 0 && n > 0 && !gated ? plan_gp(c, n) : 0;
  // the dense update builds the slot layout in one more block of the records kernel (one
  // launch fewer); the gated update (and an empty population) launches it on its own
  if (M > 0 && gp <= 0) KL(launch_build_slots(bsa, c->st));
  c->gp = gp;
  PassArgs pa{};
  pa.n = n;
  pa.tile = gp > 0 ? c->tile : kTileP;
  pa.tiles_per_cta = gp > 0 ? ceil_div(ceil_div(n, pa.tile), gp) : 0;
  pa.x = c->A[0];
  pa.vx = c->A[1];
  pa.y = c->A[2];
  pa.vy = c->A[3];
  pa.w = c->A[4];
  pa.rb = c->rb;
  pa.rb_stride = c->L.cap_l;
  pa.sc = SlotConsts{c->s[0], c->s[1], c->s[2], c->s[3], c->s[4], c->rep};
  pa.slots_pad = c->slots_pad;
  pa.na0 = c->na0;
  pa.na1 = c->na1;
  pa.rbs = (float)(c->p.sigma_z[0] / c->p.sigma_z[1]);
  pa.wscale = c->wscale;
  pa.Cpart = c->Cpart;
  pa.Apart = c->Apart;
  pa.P = c->P;
  pa.P_stride = c->L.cap_l;
  pa.rec = c->rec;
  c->select = M > 0 && c->p.stphd_all == 0;
  pa.js = nullptr;
  if (M > 0 && gated) {
    // candidate lists, entries grouped by label, then the two gated passes
    const int ntiles = (int)c->g_tiles;  // (the candidate fill ran in gate_plan)
    CU(gate_sort_entries(c->gcand, c->g_entries, M, c->gk, c->gv, c->gmlist, c->ghist, c->gscan, c->gmstart, c->st,
                         &c->launches));
    GateArgs ga{};
    ga.n = n;
    ga.ntiles = ntiles;
    ga.model = c->model;
    ga.so = c->gso;
    ga.tstart = c->gtstart;
    ga.cand = c->gcand;
    ga.sc = pa.sc;
    ga.sel = nullptr;
    ga.na0 = c->na0;
    ga.na1 = c->na1;
    ga.part1 = c->gpart1;
    ga.part2 = c->gpart2;
    ga.Ps = c->gPs;
    ga.E = c->g_entries;
    ga.M = M;
    timing_record(c, 3);
    if (ntiles > 0) KL(launch_gpass(1, ga, c->st));
    timing_record(c, 4);
    // W_pred's block sums: written by the particle sort (c->g_nwb blocks of its own)
    const bool c_final = c->world == 1 || c->dcp;  // else the constants follow the C1 all-reduce
    const ZConstArgs zc{c->slot_label, c->kappa, c->s[4], c->C, c->D, c->bad};
    KL(launch_gate_reduce(1, c->gmstart, c->gmlist, M, c->gpart1, nullptr, nullptr, c->C_slot, c->slots_pad, c->st,
                          c->blk_wp, c->g_nwb, c->C_slot + c->slots_pad, c_final ? &zc : nullptr,
                          c->bad));
    if (!c_final) {
      COMM(c->comm->allreduce_f64(c->C_slot, (size_t)c->slots_pad + 1, c->st));
      KL(launch_zconst(c->C_slot, c->slot_label, 0, c->slots_pad, c->kappa, c->s[4], c->C, c->D, c->bad, c->st,
                       c->C_slot + c->slots_pad));
    }
    if (c->select) {
      KL(launch_select(c->C, c->D, M, c->C_slot + c->slots_pad, c->p.p_d, c->sel_flag, c->sel_info, c->st));
      ga.sel = c->sel_flag;
    }
    timing_record(c, 5);
    if (ntiles > 0) KL(launch_gpass(2, ga, c->st));
    timing_record(c, 6);
    KL(launch_gate_reduce(2, c->gmstart, c->gmlist, M, nullptr, c->gpart2, ga.sel, c->gA, c->slots_pad, c->st));
  } else if (M > 0) {
    // the records also carry the fp64 block sums of the predicted w (W_pred, which rides with
    // C in the C1 all-reduce: element slots_pad)
    if (gp > 0) KL(launch_records(c->model, pa, c->st, c->blk_wp, &bsa));
    timing_record(c, 3);
    if (gp > 0) KL(launch_pass(c->model, 1, pa, gp, c->zb, c->wz, c->zl, c->st));
    timing_record(c, 4);
    if (gp <= 0) KL(launch_block_sums(c->A[4], n, c->blk_wp, c->st));
    // one rank (or a DCP group): C is final after the reduction, which then also writes
    // the per-slot constants; otherwise they follow the C1 all-reduce
    const bool c_final = c->world == 1 || c->dcp;
    const ZConstArgs zc{c->slot_label, c->kappa, c->s[4], c->C, c->D, c->bad};
    KL(launch_reduce_C(c->Cpart, gp, c->slots_pad, 0, c->slots_pad, c->C_slot, c->st, c->blk_wp,
                       (int)ceil_div(n, kBlockW), c->C_slot + c->slots_pad, c_final ? &zc : nullptr));
    if (!c_final) {
      COMM(c->comm->allreduce_f64(c->C_slot, (size_t)c->slots_pad + 1, c->st));
      KL(launch_zconst(c->C_slot, c->slot_label, 0, c->slots_pad, c->kappa, c->s[4], c->C, c->D, c->bad, c->st,
                       c->C_slot + c->slots_pad));
    }
    if (c->select) {
      // index set I from dW = C/D and the mass identity; pass-2 slot layout with I first
      SlotConsts sc2{c->s[0], c->s[1], c->s[2], c->s[3], c->s[4], c->rep};
      // pass 2's SPLIT instance when the per-warp state-sum layout is expected, from the
      // previous step's LT (a guess for speed only: the layout is the select kernel's, from
      // this step's data, and either instance computes its bits -- js_layout)
      int ss_uniform, ss_split;
      const int lanes = c->slots_pad / c->zl;
      const int n_est = (int)std::min<int64_t>(c->LT > 0 ? c->LT : M / 4, M);
      js_layout(n_est, lanes, c->zl, false, &ss_uniform);
      js_layout(n_est, lanes, c->zl, true, &ss_split);
      pa.js_split = ss_split < ss_uniform ? 1 : 0;
      const char* jse = getenv("PHD_JS_SPLIT");  // tests: force either instance
      if (jse && (jse[0] == '0' || jse[0] == '1')) pa.js_split = jse[0] - '0';
      KL(launch_select_slots(c->C, c->D, M, c->C_slot + c->slots_pad, c->p.p_d, c->sel_flag, c->sel_info, c->zlab,
                             c->model, c->zl, c->wz, sum_layout(), c->slots_pad, c->slot_label, c->s_lim,
                             (float)c->p.sensor_xy[0], (float)c->p.sensor_xy[1], sc2, c->st,
                             c->capturing ? &c->dstep->M : nullptr, c->p.max_meas));
      pa.js = c->s_lim;
    }
    timing_record(c, 5);
    if (gp > 0) KL(launch_pass(c->model, 2, pa, gp, c->zb, c->wz, c->zl, c->st));
    timing_record(c, 6);
  } else {
    timing_record(c, 3);
    timing_record(c, 4);
    timing_record(c, 5);
    timing_record(c, 6);
  }
  int nbw = (int)ceil_div(n, kBlockW);
  if (n > 0 && gated)
    KL(launch_finalize(c->A[4], c->gPs, 0, M > 0 ? 1 : 0, n, c->nu, c->wscale, c->wn, c->blk_w, c->blk_wp, c->st,
                       c->gso.inv));
  else if (n > 0)
    KL(launch_finalize(c->A[4], c->P, c->L.cap_l, M > 0 && gp > 0 ? c->zb : 0, n, c->nu, c->wscale, c->wn, c->blk_w, c->blk_wp, c->st));
  double* rank_slots = c->rslots;
  KL(launch_reduce_acc(gated ? c->gA : c->Apart, gated ? 1 : gp, c->slots_pad, M > 0 ? c->slots_pad : 0, c->slot_label, c->C, c->D, c->s[0],
                       c->s[1], c->s[2], c->s[3], c->model, c->blk_w, c->blk_wp, nbw, c->acc, rank_slots, c->rank,
                       c->world, c->dcp || c->rank == 0 ? 1 : 0, c->select ? c->sel_flag : nullptr, c->st,
                       pass2_sums_scaled() ? 1 : 0, (double)n));
  // rank slots [W_r | W_pred_r | N_r] (3 per rank), written by k_reduce_acc's last block
  if (c->world > 1) {
    if (c->dcp)  // groups keep their own accumulators; only the per-group masses are shared
      COMM(c->comm->allreduce_f64(rank_slots, (size_t)(3 * c->world), c->st));
    else
      COMM(c->comm->allreduce_f64(c->rslots, (size_t)(c->acc - c->rslots) + 5 * (size_t)M, c->st));
  }
  if (!c->dev_scalars) {  // one-sync / graph step: k_step_out stores them at the end of the step
    CU(cudaMemcpyAsync(c->h_meta, rank_slots, sizeof(double) * 3 * c->world, cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(c->h_meta + 3 * c->world, c->bad, sizeof(int) * 2, cudaMemcpyDeviceToHost, c->st));
    if (c->select)
      CU(cudaMemcpyAsync(c->h_meta + 3 * c->world + 32, c->sel_info, sizeof(double) * 4, cudaMemcpyDeviceToHost, c->st));
  }
  timing_record(c, 7);
  if (c->defer_update_sync) {  // phd_step: finished by phd_extract after its one synchronisation
    c->update_pending = true;
    c->stage = kUpdated;
    return PHD_OK;
  }
  CU(cudaStreamSynchronize(c->st));
  return update_finish(c);
}

// Host side of the end of an update, once its D2H copies (rank masses, NaN flags,
// index-set meta) have completed.
static phd_status update_finish(phd_ctx* c) {
  c->update_pending = false;
  c->W = 0.0;
  c->W_pred = 0.0;
  c->N_all = 0;
  for (int r = 0; r < c->world; ++r) {
    c->Wr[r] = c->h_meta[r];
    c->Wpr[r] = c->h_meta[c->world + r];
    c->W += c->Wr[r];
    c->W_pred += c->Wpr[r];
    c->N_all += (int64_t)c->h_meta[2 * c->world + r];
  }
  if (c->dcp) {
    // every group is a full-intensity PHD filter: the summary reports the
    // mean over the K groups; each group resamples from its own W_r (next_count_dcp)
    c->W /= c->world;
    c->W_pred /= c->world;
  }
  c->bad_flag = reinterpret_cast<int*>(c->h_meta + 3 * c->world)[0];
  double Wsel = c->W;
  if (c->select && !c->dcp) Wsel = c->h_meta[3 * c->world + 32];  // W by the mass identity (k_select)
  c->LT = (int64_t)std::floor(Wsel + 0.5);
  if (c->select && !c->dcp) c->LT = (int64_t)c->h_meta[3 * c->world + 33];
  if (c->LT < 0) c->LT = 0;
  double frac = Wsel - std::floor(Wsel);
  c->near_half = std::fabs(frac - 0.5) < 1e-4 * std::max(1.0, Wsel);
  c->stage = kUpdated;
  if (c->timing) {
    cudaEventElapsedTime(&c->t_ms[0], c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&c->t_ms[1], c->ev[3], c->ev[4]);
    cudaEventElapsedTime(&c->t_ms[2], c->ev[5], c->ev[6]);
    cudaEventElapsedTime(&c->t_ms[3], c->ev[2], c->ev[7]);
  }
  if (c->bad_flag || !std::isfinite(c->W) || !std::isfinite(c->W_pred))
    return fail(c, PHD_EMODEL, "non-finite C/D/W (bad=%d, W=%g)", c->bad_flag, c->W);
  return PHD_OK;
}

static int64_t next_count(phd_ctx* c, int* clamped) {
  *clamped = 0;
  if (c->p.count_mode == PHD_COUNT_FIXED) return c->p.fixed_count;
  int64_t want = std::max<int64_t>(c->LT, 1) * c->p.particles_per_target;
  int64_t lim = c->p.capacity - c->p.births_per_step;
  if (want > lim) {
    *clamped = 1;
    want = lim;
  }
  return want;
}

static int64_t next_count_dcp(phd_ctx* c, int* clamped) {
  // Algorithm 1: the group resamples into N_k(j) R_k = max(LT_j, 1) R particles
  // (fixed-count configs: the group's block of N_out)
  *clamped = 0;
  if (c->p.count_mode == PHD_COUNT_FIXED) {
    int64_t lo, hi;
    block_of(c->p.fixed_count, c->world, c->rank, &lo, &hi);
    return hi - lo;
  }
  int64_t jlo, jhi;
  group_births(c, &jlo, &jhi);
  int64_t LT = (int64_t)std::floor(c->Wr[c->rank] + 0.5);
  int64_t want = std::max<int64_t>(LT, 1) * c->p.particles_per_target;
  int64_t lim = c->L.cap_l - 1 - (jhi - jlo);
  if (want > lim) {
    *clamped = 1;
    want = lim;
  }
  return want;
}

// Step 4: keep a label reported by more than half of the groups,
// state = mean of the supporters' states (fp64), mass = mean of their dW.  Labels ascending.
static int fuse_estimates(phd_ctx* c, phd_estimate* out, int cap) {
  const int cap1 = c->p.max_meas + 1;
  std::vector<int> cnt(c->p.max_meas, 0);
  std::vector<double> acc((size_t)c->p.max_meas * 5, 0.0);
  for (int r = 0; r < c->world; ++r) {
    const phd_estimate* blk = c->h_gather + (size_t)r * cap1;
    int n = blk[0].label;
    for (int i = 0; i < n; ++i) {
      const phd_estimate& e = blk[1 + i];
      if (e.label < 0 || e.label >= c->p.max_meas) continue;
      cnt[e.label] += 1;
      for (int q = 0; q < 4; ++q) acc[5 * (size_t)e.label + q] += (double)e.state[q];
      acc[5 * (size_t)e.label + 4] += (double)e.mass;
    }
  }
  int k = 0;
  for (int l = 0; l < c->p.max_meas && k < cap; ++l) {
    if (2 * cnt[l] <= c->world) continue;
    phd_estimate e;
    e.label = l;
    for (int q = 0; q < 4; ++q) e.state[q] = (float)(acc[5 * (size_t)l + q] / cnt[l]);
    e.mass = (float)(acc[5 * (size_t)l + 4] / cnt[l]);
    if (out) out[k] = e;
    ++k;
  }
  return k;
}

phd_status phd_extract(phd_ctx* c, phd_estimate* out, int32_t cap, int32_t* n_out, phd_summary* s) {
  NvtxRange nvtx_("phd_extract");
  if (!c) return PHD_EINVAL;
  cudaSetDevice(c->device);
  c->err.clear();
  if (c->stage != kUpdated) return fail(c, PHD_ESTATE, "phd_extract needs an updated population");
  int nest = 0;
  int lt_clamped = 0;
  double* rank_slots = c->rslots;
  double* smh = c->h_meta + 3 * c->world + 4;
  if (c->dcp) {
    // every group extracts locally (Step 3); the CU (rank 0) fuses (Step 4)
    timing_record(c, 8);
    const int capd = c->p.max_meas;
    KL(launch_extract(c->acc, c->M, rank_slots + c->rank, rank_slots + c->world + c->rank, 1, c->p.p_d, c->est + 1,
                      capd, c->summ, &c->est[0].label, c->select ? c->sel_info : nullptr, nullptr, c->st));
    CU(cudaMemcpyAsync(smh, c->summ, sizeof(double) * 8, cudaMemcpyDeviceToHost, c->st));
    if (c->world > 1)
      COMM(c->comm->allgather_bytes(c->est, c->gather, sizeof(phd_estimate) * (size_t)(c->p.max_meas + 1), c->st));
    CU(cudaStreamSynchronize(c->st));
    if (c->update_pending) {
      phd_status st = update_finish(c);
      if (st != PHD_OK) return st;
    }
    const int nloc = (int)smh[5];
    lt_clamped = (int)smh[6];
    c->local_est.resize(nloc);
    if (nloc > 0)
      CU(cudaMemcpyAsync(c->local_est.data(), c->est + 1, sizeof(phd_estimate) * nloc, cudaMemcpyDeviceToHost, c->st));
    if (c->rank == 0) {
      if (c->world > 1) {
        CU(cudaMemcpyAsync(c->h_gather, c->gather, sizeof(phd_estimate) * (size_t)(c->p.max_meas + 1) * c->world,
                           cudaMemcpyDeviceToHost, c->st));
      } else {
        CU(cudaMemcpyAsync(c->h_gather, c->est, sizeof(phd_estimate) * (size_t)(c->p.max_meas + 1),
                           cudaMemcpyDeviceToHost, c->st));
      }
    }
    CU(cudaStreamSynchronize(c->st));
    if (c->rank == 0) nest = fuse_estimates(c, out, std::max(0, cap));
    timing_record(c, 9);
    if (c->timing) cudaEventElapsedTime(&c->t_ms[4], c->ev[8], c->ev[9]);
  } else if (c->rank == 0) {
    timing_record(c, 8);
    int capd = std::max(0, std::min(cap, c->p.max_meas));
    // one-sync step: the extraction runs on st2, overlapping the resampling (it reads the
    // accumulators only); the resampling joins it before the step's synchronisation
    cudaStream_t es = c->st;
    if (c->dev_scalars) {
      CU(cudaEventRecord(c->fork_ev, c->st));
      CU(cudaStreamWaitEvent(c->st2, c->fork_ev, 0));
      es = c->st2;
    }
    KL(launch_extract(c->acc, c->M, rank_slots, rank_slots + c->world, c->world, c->p.p_d, c->est + 1, capd, c->summ,
                      &c->est[0].label, c->select ? c->sel_info : nullptr, c->select ? c->sel_flag : nullptr,
                      es, c->capturing ? &c->dstep->M : nullptr, c->p.max_meas));
    if (!c->dev_scalars) CU(cudaMemcpyAsync(smh, c->summ, sizeof(double) * 8, cudaMemcpyDeviceToHost, es));
    // the estimate count is min(LT, eligible, cap) <= min(LT, cap): copy that many with the
    // summary, so the extraction costs one synchronisation
    // (inside phd_step LT is not on the host yet: copy up to kEstEager estimates, the
    // rest, if any, after the synchronisation)
    const int64_t ncopy = (!out && !c->dev_scalars) ? 0
                          : c->update_pending ? std::min<int64_t>(kEstEager, capd)
                                              : std::min<int64_t>(std::max<int64_t>(c->LT, 0), capd);
    if (c->dev_scalars) {  // one-sync step: k_step_out stores summary + estimates; step_finish
      c->est_eager = (int)ncopy;
      CU(cudaEventRecord(c->join_ev, c->st2));
      return PHD_OK;
    }
    if (ncopy > 0)
      CU(cudaMemcpyAsync(c->h_est, c->est + 1, sizeof(phd_estimate) * ncopy, cudaMemcpyDeviceToHost, es));
    CU(cudaStreamSynchronize(c->st));
    if (c->update_pending) {
      phd_status st = update_finish(c);
      if (st != PHD_OK) return st;
    }
    nest = (int)smh[5];
    lt_clamped = (int)smh[6];
    if (nest > ncopy && out) {  // more estimates than the eager copy (phd_step, LT > kEstEager)
      CU(cudaMemcpyAsync(c->h_est + ncopy, c->est + 1 + ncopy, sizeof(phd_estimate) * (nest - ncopy),
                         cudaMemcpyDeviceToHost, c->st));
      CU(cudaStreamSynchronize(c->st));
    }
    if (nest > 0 && out) memcpy(out, c->h_est, sizeof(phd_estimate) * nest);
    timing_record(c, 9);
    if (c->timing) cudaEventElapsedTime(&c->t_ms[4], c->ev[8], c->ev[9]);
  } else if (c->update_pending) {  // ranks other than the CU: only the update's bookkeeping
    CU(cudaStreamSynchronize(c->st));
    phd_status st = update_finish(c);
    if (st != PHD_OK) return st;
  }
  if (n_out) *n_out = nest;
  if (s) {
    int clamped;
    s->W = c->W;
    s->W_pred = c->W_pred;
    s->undetected_mass = (1.0 - c->p.p_d) * c->W_pred;
    s->LT = c->LT;
    s->N = c->dcp ? c->N_all : c->N;
    s->N_out = c->dcp ? next_count_dcp(c, &clamped) : next_count(c, &clamped);
    s->M = c->M;
    s->n_est = nest;
    s->lt_clamped = lt_clamped;
    s->count_clamped = clamped;
    s->zero_mass = !(c->W > 0.0);
    s->near_half = c->near_half;
  }
  return PHD_OK;
}

phd_status phd_get_local_estimates(phd_ctx* c, phd_estimate* out, int32_t cap, int32_t* n) {
  if (!c) return PHD_EINVAL;
  int k = (int)std::min<size_t>(c->local_est.size(), (size_t)std::max(0, cap));
  if (n) *n = (int32_t)c->local_est.size();
  if (out && k > 0) memcpy(out, c->local_est.data(), sizeof(phd_estimate) * k);
  return PHD_OK;
}

// Peer-memory window for the fused resample + exchange, shared at
// the first multi-rank resampling (a collective point: the ranks of an in-process
// group are created one after another, but step in parallel).  The particle double
// buffers are library allocations (phd_create) every rank maps; any failure (no
// IPC / peer access, PHD_EXCHANGE=nccl) keeps the send/recv exchange.
static phd_status p2p_setup(phd_ctx* c) {
  const char* xch = getenv("PHD_EXCHANGE");
  if (c->world <= 1 || c->dcp || c->world > kMaxPeers || (xch && strcmp(xch, "nccl") == 0)) {
    c->p2p_state = -1;
    return PHD_OK;
  }
  const bool ok = c->pbuf[0] && c->pbuf[1];  // allocated by phd_create
  std::vector<void*> all;
  void* loc[2] = {c->pbuf[0], c->pbuf[1]};
  // collective on every rank; a rank without buffers fails IPC and the verdict falls back everywhere
  std::string e = c->comm->share_buffers(loc, 2, &all, c->st);
  if (e.empty() && ok) {
    c->p2p_state = 1;
    c->peer_buf.resize((size_t)c->world * 2);
    for (size_t i = 0; i < all.size(); ++i) c->peer_buf[i] = (float*)all[i];
  } else {
    for (int b = 0; b < 2; ++b)
      if (c->pbuf[b]) cudaFree(c->pbuf[b]);
    c->pbuf[0] = c->pbuf[1] = nullptr;
    cudaGetLastError();
    c->p2p_state = -1;
  }
  CU(cudaStreamSynchronize(c->st));
  return PHD_OK;
}

static ResampleGatherArgs rg_args(phd_ctx* c, const ResampleArgs& ra, float w_off) {
  ResampleGatherArgs g{};
  g.r = ra;
  g.coff = c->coff;
  g.x = c->A[0];
  g.vx = c->A[1];
  g.y = c->A[2];
  g.vy = c->A[3];
  g.w_off = w_off;
  g.ox = c->B[0];
  g.ovx = c->B[1];
  g.oy = c->B[2];
  g.ovy = c->B[3];
  g.ow = c->B[4];
  g.anc = c->anc;
  return g;
}

phd_status phd_resample_exchange(phd_ctx* c, int32_t k) {
  NvtxRange nvtx_("phd_resample_exchange");
  if (!c) return PHD_EINVAL;
  cudaSetDevice(c->device);
  c->err.clear();
  if (c->stage != kUpdated) return fail(c, PHD_ESTATE, "phd_resample_exchange needs an updated population");
  if (c->dev_scalars) {
    // one-sync / graph step (world 1, exact): n_out, U, W, zero mass of this step are
    // computed on the device from the update's results (resample_setup_body in k_scan_chunks), read back after
    // the step's synchronisation
    SetupArgs sa{};
    sa.rslots = c->rslots;
    sa.sel_info = c->select ? c->sel_info : nullptr;
    sa.fixed = c->p.count_mode == PHD_COUNT_FIXED;
    sa.fixed_count = c->p.fixed_count;
    sa.R = c->p.particles_per_target;
    sa.lim = c->p.capacity - c->p.births_per_step;
    sa.seed = c->p.seed;
    sa.k = c->capturing ? 0 : k;  // graph replays: k from the staged step block
    const int64_t n = c->n_local;
    KL(launch_scan_chunks(c->blk_w, (int)ceil_div(n, kBlockW), c->blk_off, c->ctot, c->coff, c->scan_counter, c->st,
                          &sa, c->dstep));
    ResampleArgs ra{};
    ra.n_local = n;
    ra.g0 = 0;
    ra.w = c->wn;
    ra.blk_off = c->blk_off;
    ra.n_upd = c->N;
    ra.ds = c->dstep;
    KL(launch_resample_gather(rg_args(c, ra, 0.0f), nullptr, c->st));
    if (c->rank == 0) CU(cudaStreamWaitEvent(c->st, c->join_ev, 0));  // the extraction on st2
    // everything the host reads after the step's synchronisation, by one kernel
    StepOutArgs so{};
    so.rslots = c->rslots;
    so.n_rslots = 3 * c->world;
    so.h_rslots = c->hd_meta;
    so.bad = c->bad;
    so.h_bad = reinterpret_cast<int32_t*>(c->hd_meta + 3 * c->world);
    so.sel_info = c->select ? c->sel_info : nullptr;
    so.h_sel = c->hd_meta + 3 * c->world + 32;
    so.summ = c->summ;
    so.h_summ = c->hd_meta + 3 * c->world + 4;
    so.est = c->est + 1;
    so.est_count = c->rank == 0 ? &c->est[0].label : nullptr;
    so.h_est = c->hd_est;
    so.est_cap = c->est_eager;
    so.ds = c->dstep;
    so.h_ds = c->hd_stepout;
    KL(launch_step_out(so, c->st));
    c->bad_clean = true;
    return PHD_OK;
  }
  timing_record(c, 10);
  int clamped = 0;
  const int64_t n_out = c->dcp ? next_count_dcp(c, &clamped) : next_count(c, &clamped);
  c->count_clamped = clamped;
  const int64_t J = c->p.births_per_step;
  // systematic-resampling offset: one U shared by all ranks (exact mode); one per group (DCP, K > 1)
  U4 o = (c->dcp && c->world > 1) ? philox_at(c->p.seed, dcp_space(c), (uint32_t)k, 3u)
                                  : philox_at(c->p.seed, 0, (uint32_t)k, 3u);
  const double U = u52(o.x, o.y);
  const double W = c->dcp ? c->Wr[c->rank] : c->W;
  c->zero_mass = !(W > 0.0);
  std::vector<int64_t> bounds(c->world + 1);
  double O_r = 0.0;
  int64_t lo, hi;
  if (c->dcp) {
    // local resampling of the group (Step 5)
    lo = 0;
    hi = n_out;
  } else {
    if (!c->zero_mass) {
      phd_resample_bounds(c->world, c->Wr.data(), n_out, U, bounds.data(), nullptr);
    } else {
      // W == 0: offspring j copies particle floor(j N / n_out), produced by its owner
      for (int r = 0; r <= c->world; ++r) {
        int64_t blo, bhi;
        block_of(c->N, c->world, std::min(r, c->world - 1), &blo, &bhi);
        int64_t g = r == c->world ? c->N : blo;
        bounds[r] = (int64_t)(((__int128)g * n_out + c->N - 1) / c->N);
      }
      bounds[c->world] = n_out;
    }
    lo = bounds[c->rank];
    hi = bounds[c->rank + 1];
    for (int r = 0; r < c->rank; ++r) O_r += c->Wr[r];
  }
  const int64_t nprod = hi - lo;
  const float w_off = n_out > 0 ? (float)(W / (double)n_out) : 0.0f;
  const int64_t n = c->n_local;
  const int nbw = (int)ceil_div(n, kBlockW);
  // systematic resampling + gather in one kernel (k_resample_gather); zero mass: the
  // deterministic spread (offspring j copies particle floor(j N / n_out), weight 0)
  ResampleArgs ra{};
  ra.n_local = n;
  ra.g0 = c->g0;
  ra.w = c->wn;
  ra.blk_off = c->blk_off;
  ra.O_r = O_r;
  ra.scale = c->zero_mass ? 0.0 : (double)n_out / W;
  ra.U = U;
  ra.lo = lo;
  ra.hi = hi;
  ra.zero_mass = c->zero_mass ? 1 : 0;
  ra.n_upd = c->dcp ? c->n_local : c->N;
  ra.n_out = n_out;
  if (!c->zero_mass && nprod > 0)
    KL(launch_scan_chunks(c->blk_w, nbw, c->blk_off, c->ctot, c->coff, c->scan_counter, c->st));
  if (!c->dcp && c->world > 1 && c->p2p_state == 0) {
    phd_status st = p2p_setup(c);
    if (st != PHD_OK) return st;
  }
  const int dst_b = c->p2p_live ? 1 - c->par : 0;  // the buffer that becomes A on every rank
  if (c->p2p_state == 1 && !c->dcp) {
    // fused gather + exchange: offspring stored straight into their owners' next-step
    // arrays, then one collective barrier
    PeerOut po{};
    po.world = c->world;
    for (int q = 0; q < c->world; ++q) {
      int64_t blo, bhi;
      block_of(n_out + J, c->world, q, &blo, &bhi);
      po.blo[q] = blo;
      float* base = c->peer_buf[(size_t)q * 2 + dst_b];
      for (int i = 0; i < 5; ++i) po.dst[q][i] = base + (size_t)i * c->L.cap_l;
    }
    po.blo[c->world] = n_out + J;
    if (nprod > 0) KL(launch_resample_gather(rg_args(c, ra, w_off), &po, c->st));
  } else {
    if (nprod > 0) KL(launch_resample_gather(rg_args(c, ra, w_off), nullptr, c->st));
  }
  timing_record(c, 11);
  // exchange: the next step's survivors [0, n_out) are block-partitioned over N' = n_out + J
  if (c->dcp) {
    for (int i = 0; i < 5; ++i) std::swap(c->A[i], c->B[i]);
    c->n_surv_local = n_out;
    if (c->world > 1) {
      // Step 6 ring exchange: L particles to rank+1, refill the same
      // slots from rank-1 (swap semantics); L is common to all groups
      for (int r = 0; r < c->world; ++r) c->h_meta[3 * c->world + 20 + r] = r == c->rank ? (double)n_out : 0.0;
      CU(cudaMemcpyAsync(c->ring, c->h_meta + 3 * c->world + 20, sizeof(double) * c->world, cudaMemcpyHostToDevice,
                         c->st));
      COMM(c->comm->allreduce_f64(c->ring, (size_t)c->world, c->st));
      CU(cudaMemcpyAsync(c->h_meta + 3 * c->world + 20, c->ring, sizeof(double) * c->world, cudaMemcpyDeviceToHost,
                         c->st));
      CU(cudaStreamSynchronize(c->st));
      int64_t n_min = INT64_MAX;
      for (int r = 0; r < c->world; ++r) n_min = std::min<int64_t>(n_min, (int64_t)c->h_meta[3 * c->world + 20 + r]);
      int64_t L = c->p.exchange_count > 0 ? c->p.exchange_count : n_min / 10;
      L = std::min<int64_t>(L, n_min / 2);
      c->ring_L = L;
      if (L > 0) {
        U4 v4 = philox_at(c->p.seed, dcp_space(c), (uint32_t)k, 4u);
        const double v = u52(v4.x, v4.y);
        float* sendb[5];
        float* recvb[5];
        for (int i = 0; i < 5; ++i) {
          sendb[i] = c->B[i];
          recvb[i] = c->B[i] + L;
        }
        KL(launch_ring_pack(c->A, sendb, 5, L, n_out, v, c->st));
        ExchangePlan plan;
        plan.send_count.assign(c->world, 0);
        plan.send_off.assign(c->world, 0);
        plan.recv_count.assign(c->world, 0);
        plan.recv_off.assign(c->world, 0);
        plan.send_count[(c->rank + 1) % c->world] = L;
        plan.recv_count[(c->rank + c->world - 1) % c->world] = L;
        COMM(c->comm->exchange(sendb, recvb, 5, plan, c->st));
        KL(launch_ring_unpack(recvb, c->A, 5, L, n_out, v, c->st));
      }
    }
  } else if (c->world == 1) {
    for (int i = 0; i < 5; ++i) std::swap(c->A[i], c->B[i]);
    c->n_surv_local = n_out;
  } else if (c->p2p_state == 1) {
    // every rank's stores into the peers' next-step arrays are complete once all ranks
    // pass this stream-ordered barrier (a one-element all-reduce); then every rank's A
    // is its buffer dst_b, B the other one
    c->h_meta[3 * c->world + 46] = 0.0;
    CU(cudaMemcpyAsync(c->ring, c->h_meta + 3 * c->world + 46, sizeof(double), cudaMemcpyHostToDevice, c->st));
    COMM(c->comm->allreduce_f64(c->ring, 1, c->st));
    for (int i = 0; i < 5; ++i) {
      c->A[i] = c->pbuf[dst_b] + (size_t)i * c->L.cap_l;
      c->B[i] = c->pbuf[1 - dst_b] + (size_t)i * c->L.cap_l;
    }
    c->par = dst_b;
    c->p2p_live = true;
    int64_t blo, bhi;
    block_of(n_out + J, c->world, c->rank, &blo, &bhi);
    c->n_surv_local = std::max<int64_t>(0, std::min(bhi, n_out) - std::min(blo, n_out));
  } else {
    std::vector<int64_t> sc(c->world), so(c->world), rc(c->world), ro(c->world);
    phd_plan_exchange(c->world, c->rank, bounds.data(), n_out, J, sc.data(), so.data(), rc.data(), ro.data());
    // local part first (device copy), then the grouped peer transfers (C3)
    if (sc[c->rank] > 0)
      for (int i = 0; i < 5; ++i)
        CU(cudaMemcpyAsync(c->A[i] + ro[c->rank], c->B[i] + so[c->rank], sizeof(float) * sc[c->rank],
                           cudaMemcpyDeviceToDevice, c->st));
    ExchangePlan plan{sc, so, rc, ro};
    COMM(c->comm->exchange(c->B, c->A, 5, plan, c->st));
    int64_t blo, bhi;
    block_of(n_out + J, c->world, c->rank, &blo, &bhi);
    c->n_surv_local = std::max<int64_t>(0, std::min(bhi, n_out) - std::min(blo, n_out));
  }
  timing_record(c, 12);
  if (c->timing) {
    cudaEventSynchronize(c->ev[12]);
    cudaEventElapsedTime(&c->t_ms[5], c->ev[10], c->ev[11]);
    cudaEventElapsedTime(&c->t_ms[6], c->ev[11], c->ev[12]);
  }
  c->U_last = U;
  c->W_last = W;
  c->N_out_last = n_out;
  c->prod_first = lo;
  c->prod_n = nprod;
  c->n_out = n_out;
  c->stage = kResampled;
  return PHD_OK;
}

// ---------------------------------------------------------------------------
// Graph steps (DESIGN.md §4 "graph step"): with one rank, a dense update and nothing
// that needs the host mid-step, phd_step replays a CUDA graph of its whole kernel chain
// (predict, the dense update, extraction, resampling) -- one launch and one host
// synchronisation instead of ~15 launches.  The per-step scalars (k, M, M_{k-1}) are
// staged in pinned memory and copied by the graph's first node; the resampling
// count, offset and mass are computed on the device (resample_setup_body in k_scan_chunks); graphs are
// cached per launch shape (particle count, slot layout, particle buffer), so a
// configuration replays a handful of graphs.
static bool graph_eligible(const phd_ctx* c, int M) {
  // opt-in (PHD_GRAPH=1): measured slower than the eager launches with programmatic
  // dependent launch on B200 (cfg 3: 0.214 vs 0.189 ms back to back; cfg 2 0.186 vs
  // 0.127 ms, whose adaptive count keeps changing the launch shape): the small steps are
  // GPU-bound, not launch-bound
  const char* ge = getenv("PHD_GRAPH");
  const bool env_off = !(ge && ge[0] == '1');
  if (env_off || c->graph_off || c->world != 1 || c->dcp || c->timing || M <= 0) return false;
  if (c->p.birth_model == 2 || c->stage != kResampled || !c->populated) return false;
  if (c->p.gate == 2) return false;
  if (c->p.gate == 1 && (double)(c->n_out + c->p.births_per_step) * (double)M >= 536870912.0) return false;
  return true;
}

// host state of the calls a replay stands for (phd_predict / phd_update up to the sync)
static void graph_host_state(phd_ctx* c, int M) {
  c->N = c->n_out + c->p.births_per_step;
  c->g0 = 0;
  c->n_local = c->N;
  c->M = M;
  c->M_z = M;
  c->gated = false;
  c->select = c->p.stphd_all == 0;
  c->update_pending = true;
  c->stage = kUpdated;
}

// host side of a one-sync (or graph) step after its synchronisation: the update's
// bookkeeping, the estimates, the resampling scalars the device computed
static phd_status step_finish(phd_ctx* c, phd_estimate* out, int32_t cap, int32_t* n_out, phd_summary* s) {
  phd_status st = update_finish(c);
  if (st != PHD_OK) return st;
  const double* smh = c->h_meta + 3 * c->world + 4;
  const int capd = std::max(0, std::min(cap, c->p.max_meas));
  const int64_t ncopy = out ? std::min<int64_t>(kEstEager, capd) : 0;
  const int nest = (int)smh[5];
  const int lt_clamped = (int)smh[6];
  if (nest > ncopy && out) {
    CU(cudaMemcpyAsync(c->h_est + ncopy, c->est + 1 + ncopy, sizeof(phd_estimate) * (nest - ncopy),
                       cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  if (nest > 0 && out) memcpy(out, c->h_est, sizeof(phd_estimate) * nest);
  const DevStep d = *c->h_stepout;
  int clamped = 0;
  const int64_t want = next_count(c, &clamped);
  if (want != d.n_out) return fail(c, PHD_ECUDA, "graph step: device n_out %lld != %lld", (long long)d.n_out, (long long)want);
  c->count_clamped = clamped;
  c->zero_mass = d.zero_mass;
  c->U_last = d.U;
  c->W_last = d.W;
  c->N_out_last = d.n_out;
  c->prod_first = 0;
  c->prod_n = d.n_out;
  for (int i = 0; i < 5; ++i) std::swap(c->A[i], c->B[i]);
  c->n_surv_local = d.n_out;
  c->n_out = d.n_out;
  c->stage = kResampled;
  if (n_out) *n_out = nest;
  if (s) {
    s->W = c->W;
    s->W_pred = c->W_pred;
    s->undetected_mass = (1.0 - c->p.p_d) * c->W_pred;
    s->LT = c->LT;
    s->N = c->N;
    s->N_out = d.n_out;
    s->M = c->M;
    s->n_est = nest;
    s->lt_clamped = lt_clamped;
    s->count_clamped = clamped;
    s->zero_mass = !(c->W > 0.0);
    s->near_half = c->near_half;
  }
  return PHD_OK;
}

static phd_status step_graph(phd_ctx* c, int32_t k, const float* z, int32_t M, phd_estimate* out, int32_t cap,
                             int32_t* n_out, phd_summary* s) {
  // launch shape: particle count, slot layout and CTA count of the passes, buffers
  const int64_t N = c->n_out + c->p.births_per_step;
  if (N > c->L.cap_l - 1) return fail(c, PHD_ECAPACITY, "N %lld exceeds capacity", (long long)N);
  phd_status st = build_slots(c, M);
  if (st != PHD_OK) return st;
  const int gp = plan_gp(c, N);
  const int64_t key[8] = {c->n_out, (int64_t)(uintptr_t)c->A[0], c->zl | ((int64_t)c->tile << 8), c->wz, c->zb, c->slots_pad, gp,
                          std::min(cap, c->p.max_meas) > 0 ? 1 : 0};
  // stage this step's inputs: Z_k, (k, M, M_{k-1}), this rank's particle count
  cudaPointerAttributes pa{};
  const bool dev = cudaPointerGetAttributes(&pa, z) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
  cudaGetLastError();
  if (dev) {
    CU(cudaMemcpyAsync(c->h_z, z, sizeof(float) * 2 * M, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
  } else {
    memcpy(c->h_z, z, sizeof(float) * 2 * M);
  }
  c->h_stepin[0] = k;
  c->h_stepin[1] = M;
  c->h_stepin[2] = std::max(c->M_z, 0);
  c->h_meta[3 * c->world + 16] = (double)N;
  cudaGraphExec_t exec = nullptr;
  for (auto& g : c->graphs)
    if (std::equal(key, key + 8, g.key)) exec = g.exec;
  if (!exec) {
    // capture the calls of one step (they run as stream-ordered work only: no host syncs)
    const int64_t launches0 = c->launches;
    c->capturing = true;
    c->dev_scalars = true;
    c->defer_update_sync = true;
    cudaError_t e = cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      e = cudaMemcpyAsync(c->dstep, c->h_stepin, sizeof(int32_t) * 3, cudaMemcpyHostToDevice, c->st);
      if (e == cudaSuccess) st = phd_predict(c, k, nullptr, 0);
      if (e == cudaSuccess && st == PHD_OK) st = phd_update(c, c->h_z, M);
      if (e == cudaSuccess && st == PHD_OK) st = phd_extract(c, out, cap, n_out, s);
      if (e == cudaSuccess && st == PHD_OK) st = phd_resample_exchange(c, k);
      cudaGraph_t graph = nullptr;
      cudaError_t e2 = cudaStreamEndCapture(c->st, &graph);
      if (e == cudaSuccess) e = e2;
      if (e == cudaSuccess && st == PHD_OK) e = cudaGraphInstantiate(&exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
    }
    c->capturing = false;
    c->dev_scalars = false;
    c->defer_update_sync = false;
    c->launches = launches0;
    if (e != cudaSuccess || st != PHD_OK || !exec) {
      cudaGetLastError();
      if (exec) cudaGraphExecDestroy(exec);
      c->graph_off = true;  // eager from now on
      c->stage = kResampled;
      return PHD_ENODEV;    // caller retries eagerly
    }
    if (c->graphs.size() >= 32) {
      cudaGraphExecDestroy(c->graphs.front().exec);
      c->graphs.erase(c->graphs.begin());
    }
    phd_ctx::GraphEntry ge;
    std::copy(key, key + 8, ge.key);
    ge.exec = exec;
    c->graphs.push_back(ge);
    ++c->graph_captures;
  }
  graph_host_state(c, M);
  c->gp = gp;
  CU(cudaGraphLaunch(exec, c->st));
  CU(cudaStreamSynchronize(c->st));
  ++c->graph_replays;
  c->launches += 14;  // the kernels of the captured chain (predict ... resample gather)
  return step_finish(c, out, cap, n_out, s);
}

// One-sync step (world 1, exact mode): the resampling count / offset / mass are computed
// on the device (resample_setup_body in k_scan_chunks), so predict -> update -> [extraction on st2 |
// resampling] run without the host in between and the step synchronises once, at its end.
static phd_status step_onesync(phd_ctx* c, int32_t k, const float* z, int32_t M, phd_estimate* out, int32_t cap,
                               int32_t* n_out, phd_summary* s) {
  c->dev_scalars = true;  // (k, M, M_prev) reach the kernels as arguments: no staged step block
  c->defer_update_sync = true;
  phd_status st = phd_predict(c, k, nullptr, 0);
  if (st == PHD_OK) st = phd_update(c, z, M);
  if (st == PHD_OK) st = phd_extract(c, out, cap, n_out, s);
  if (st == PHD_OK) st = phd_resample_exchange(c, k);
  c->dev_scalars = false;
  c->defer_update_sync = false;
  if (st != PHD_OK) {
    cudaStreamSynchronize(c->st2);
    cudaStreamSynchronize(c->st);
    return st;
  }
  CU(cudaStreamSynchronize(c->st));
  return step_finish(c, out, cap, n_out, s);
}

phd_status phd_step(phd_ctx* c, int32_t k, const float* z, int32_t M, phd_estimate* out, int32_t cap, int32_t* n_out,
                    phd_summary* s) {
  NvtxRange nvtx_("phd_step");
  if (!c) return PHD_EINVAL;
  const bool args_ok = k >= 1 && M >= 0 && M <= c->p.max_meas && (M == 0 || z);
  if (args_ok && graph_eligible(c, M)) {
    cudaSetDevice(c->device);
    c->err.clear();
    phd_status st = step_graph(c, k, z, M, out, cap, n_out, s);
    if (st != PHD_ENODEV) return st;  // PHD_ENODEV: the capture failed, run the step eagerly
  }
  if (args_ok && c->world == 1 && !c->dcp && !c->timing && c->populated && c->stage == kResampled &&
      !(getenv("PHD_ONESYNC") && getenv("PHD_ONESYNC")[0] == '0')) {
    cudaSetDevice(c->device);
    c->err.clear();
    return step_onesync(c, k, z, M, out, cap, n_out, s);
  }
  timing_record(c, 13);
  phd_status st = phd_predict(c, k, nullptr, 0);
  if (st != PHD_OK) return st;
  // one host synchronisation for update + extraction: the update's bookkeeping (masses,
  // LT, the non-finite guard) completes inside phd_extract
  c->defer_update_sync = true;
  st = phd_update(c, z, M);
  c->defer_update_sync = false;
  if (st != PHD_OK) return st;
  st = phd_extract(c, out, cap, n_out, s);
  if (st != PHD_OK) return st;
  st = phd_resample_exchange(c, k);
  timing_record(c, 14);
  if (c->timing) {
    cudaEventSynchronize(c->ev[14]);
    cudaEventElapsedTime(&c->t_ms[7], c->ev[13], c->ev[14]);
  }
  return st;
}

phd_status phd_get_graph_stats(const phd_ctx* c, int64_t* captures, int64_t* replays) {
  if (!c) return PHD_EINVAL;
  if (captures) *captures = c->graph_captures;
  if (replays) *replays = c->graph_replays;
  return PHD_OK;
}

phd_status phd_get_gate_stats(phd_ctx* c, int64_t* out) {
  if (!c || !out) return PHD_EINVAL;
  out[0] = c->gated ? 1 : 0;
  out[1] = c->g_entries;
  out[2] = c->g_entries * gate_tp(c->model);
  out[3] = c->g_tiles;
  return PHD_OK;
}

phd_status phd_get_normalizers(phd_ctx* c, double* C, int32_t cap) {
  if (!c || !C) return PHD_EINVAL;
  cudaSetDevice(c->device);
  if (c->stage != kUpdated) return fail(c, PHD_ESTATE, "no update yet");
  if (cap < c->M) return fail(c, PHD_EINVAL, "cap < M");
  if (c->M > 0) CU(cudaMemcpyAsync(C, c->C, sizeof(double) * c->M, cudaMemcpyDeviceToHost, c->st));
  CU(cudaStreamSynchronize(c->st));
  return PHD_OK;
}

phd_status phd_get_accumulators(phd_ctx* c, double* acc, int32_t cap) {
  if (!c || !acc) return PHD_EINVAL;
  cudaSetDevice(c->device);
  if (c->stage != kUpdated) return fail(c, PHD_ESTATE, "no update yet");
  if (cap < c->M) return fail(c, PHD_EINVAL, "cap < M");
  if (c->M > 0) CU(cudaMemcpyAsync(acc, c->acc, sizeof(double) * 5 * c->M, cudaMemcpyDeviceToHost, c->st));
  CU(cudaStreamSynchronize(c->st));
  return PHD_OK;
}

phd_status phd_get_ancestors(phd_ctx* c, int32_t* anc, int64_t cap, int64_t* n, int64_t* first) {
  if (!c || !anc) return PHD_EINVAL;
  cudaSetDevice(c->device);
  if (n) *n = c->prod_n;
  if (first) *first = c->prod_first;
  if (cap < c->prod_n) return fail(c, PHD_EINVAL, "cap < produced");
  if (c->prod_n > 0) CU(cudaMemcpyAsync(anc, c->anc, sizeof(int32_t) * c->prod_n, cudaMemcpyDeviceToHost, c->st));
  CU(cudaStreamSynchronize(c->st));
  return PHD_OK;
}

phd_status phd_get_resample_meta(phd_ctx* c, double* W, double* U, int64_t* N_out, double* W_r) {
  if (!c) return PHD_EINVAL;
  if (W) *W = c->W_last;
  if (U) *U = c->U_last;
  if (N_out) *N_out = c->N_out_last;
  if (W_r)
    for (int r = 0; r < c->world; ++r) W_r[r] = c->Wr[r];
  return PHD_OK;
}

}  // extern "C"
