// Systematic resampling (Algorithm 1; Step 5 line
// 339), exact over the global particle array and executed rank-locally
// (DESIGN.md §4): rank r scans its own updated weights in fp64 starting at
// O_r = sum_{s<r} W_s; particle i receives the offspring
//   [n(B_{i-1}), n(B_i)),  n(B) = clamp(ceil(B n_out / W - U), 0, n_out),
// pinned so that the ranks' ranges tile [0, n_out) exactly.  Offspring are
// produced in global order by a mark + max-scan + gather pass (HBM-bound).
#include "phd_internal.h"
#include "philox.cuh"

#include <algorithm>

namespace phd {

__device__ __forceinline__ int64_t n_of(double B, double scale, double U, int64_t lo, int64_t hi) {
  double t = __dsub_rn(__dmul_rn(B, scale), U);
  double c = ceil(t);
  int64_t n = c <= (double)lo ? lo : (c >= (double)hi ? hi : (int64_t)c);
  return n;
}

// Graph replay (world 1): this step's resampling scalars from the update's results, in
// the host's arithmetic (phd_resample_exchange / next_count): n_out (fixed, or
// max(LT, 1) R clamped to capacity - J), U = u52(Philox(0, k, 3, 0)), W = W_0 (the rank's
// updated mass), scale = n_out / W, w_off = W / n_out; zero mass when !(W > 0).
__device__ __forceinline__ void resample_setup_body(const SetupArgs& a, DevStep* ds) {
  int64_t n_out = a.fixed_count;
  int clamped = 0;
  const double W = a.rslots[0];
  if (!a.fixed) {
    int64_t LT = a.sel_info ? (int64_t)a.sel_info[1] : (int64_t)floor(W + 0.5);
    if (LT < 0) LT = 0;
    n_out = (LT > 1 ? LT : 1) * a.R;
    if (n_out > a.lim) {
      n_out = a.lim;
      clamped = 1;
    }
  }
  const U4 o = philox_at(a.seed, 0, (uint32_t)(a.k > 0 ? a.k : ds->k), 3u);
  ds->n_out = n_out;
  ds->count_clamped = clamped;
  ds->U = u52(o.x, o.y);
  ds->W = W;
  ds->zero_mass = !(W > 0.0);
  ds->scale = W > 0.0 ? (double)n_out / W : 0.0;
  ds->w_off = n_out > 0 ? (float)(W / (double)n_out) : 0.0f;
}

// Multi-CTA exclusive scan of the block masses, deterministic: CTA c scans its chunk of
// kResScanChunk (warp shuffles, then the warp totals: a fixed tree), writes the local
// exclusive prefixes and its chunk total; the last CTA to finish (atomic ticket) adds the
// chunk totals in order.  Readers form off(b) = coff[b / kResScanChunk] + loc[b].
// ds != nullptr (one-sync / graph step): block 0 also computes the step's resampling
// scalars (resample_setup_body; one launch fewer).
__global__ void __launch_bounds__(1024) k_scan_chunks(const double* __restrict__ blk, int nb, double* loc,
                                                      double* ctot, double* coff, unsigned* counter,
                                                      const SetupArgs sa, DevStep* ds) {
  pdl_wait();
  if (ds != nullptr && blockIdx.x == 0 && threadIdx.x == 0) resample_setup_body(sa, ds);
  __shared__ double ws[33];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = blockIdx.x * kResScanChunk + tid;
  const double v = i < nb ? blk[i] : 0.0;
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double x = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const double prev = __shfl_up_sync(0xffffffffu, x, 1);
    ws[lane] = lane > 0 ? prev : 0.0;
    if (lane == 31) ws[32] = x;
  }
  __syncthreads();
  const double prevl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (i < nb) loc[i] = lane > 0 ? ws[warp] + prevl : ws[warp];
  if (tid == 0) {
    ctot[blockIdx.x] = ws[32];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && tid == 0) {
    __threadfence();
    double acc = 0.0;
    for (unsigned c = 0; c < gridDim.x; ++c) {
      const double t = __ldcg(ctot + c);
      coff[c] = acc;
      acc += t;
    }
    coff[gridDim.x] = acc;
    *counter = 0u;  // ready for the next scan
  }
}

cudaError_t launch_scan_chunks(const double* blk, int nb, double* loc, double* ctot, double* coff, unsigned* counter,
                               cudaStream_t s, const SetupArgs* sa, DevStep* ds) {
  if (nb <= 0 && ds == nullptr) return cudaSuccess;
  const unsigned grid = (unsigned)std::max<int64_t>(1, ((int64_t)nb + kResScanChunk - 1) / kResScanChunk);
  pdl_launch(k_scan_chunks, grid, kResScanChunk, 0, s, blk, std::max(nb, 0), loc, ctot, coff, counter,
             sa ? *sa : SetupArgs{}, ds);
  return cudaGetLastError();
}

// kMP particles per thread of the resampling kernel (the per-thread scans and bounds
// are amortised over them).
constexpr int kMP = 8, kMT = kBlockW / kMP;
// small populations (fewer than kGatherSmall blocks): kGatherR x kMT threads per block
// place the offspring (latency: more gathers in flight per SM)
constexpr int kGatherR = 4, kGatherSmall = 4 * 148;

// zero mass: particle g (of N updated) gets the offspring [ceil(g n_out / N), ...), i.e.
// offspring j copies particle floor(j N / n_out), with weight 0
__device__ __forceinline__ int64_t n_spread(int64_t g, int64_t n_out, int64_t N) {
  return (g * n_out + N - 1) / N;
}
// Systematic resampling and the offspring gather in one pass: per block
// of kBlockW particles the offspring bounds n(B_i) (the fp64 formula and pinning above),
// all kBlockW upper bounds in shared memory; then every offspring k of the block finds
// its particle by binary search over those bounds (balanced whatever the weights) and
// copies its state (coalesced writes at consecutive produced indices).  Reads w + state
// (20 B) per particle, writes state + w + ancestor (24 B) per offspring; no marks, no
// memsets, no max-scan.
template <bool P2P>
__global__ void __launch_bounds__(kMT * kGatherR) k_resample_gather(const ResampleGatherArgs g, const PeerOut po) {
  pdl_wait();
  ResampleArgs a = g.r;
  float w_off = g.w_off;
  if (a.ds != nullptr) {  // graph replay (world 1): this step's values from the device
    a.lo = 0;
    a.hi = a.ds->n_out;
    a.n_out = a.ds->n_out;
    a.scale = a.ds->scale;
    a.U = a.ds->U;
    a.zero_mass = a.ds->zero_mass;
    w_off = a.ds->w_off;
  }
  __shared__ double wsum[kMT / 32];
  __shared__ int wmax[kMT / 32];
  __shared__ int hb[kBlockW];
  // the first kMT threads own kMP particles each (bounds); all blockDim.x threads (kMT, or
  // kGatherR kMT for small populations: more offspring in flight) place offspring
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  const bool owner = tid < kMT;  // warp-uniform
  const int64_t b = blockIdx.x;
  const int64_t base = b * kBlockW;
  const int64_t nb = (a.n_local + kBlockW - 1) / kBlockW;
  // block bounds from off(b) = coff[b / kResScanChunk] + loc[b] (every reader forms the same bits)
  auto off = [&](int64_t bb) { return g.coff[bb / kResScanChunk] + a.blk_off[bb]; };
  const double Eb = a.O_r + (a.zero_mass ? 0.0 : off(b));
  const int64_t gb = a.g0 + base;  // global index of the block's first particle
  const int64_t nEb = (b == 0) ? a.lo
                      : (a.zero_mass ? n_spread(gb, a.n_out, a.n_upd) : n_of(Eb, a.scale, a.U, a.lo, a.hi));
  const int64_t nEb1 = (b == nb - 1) ? a.hi
                       : (a.zero_mass ? n_spread(gb + kBlockW, a.n_out, a.n_upd)
                                      : n_of(a.O_r + off(b + 1), a.scale, a.U, a.lo, a.hi));
  double w4[kMP];
  double tsum = 0.0, incl = 0.0;
  if (owner) {
    if (base + kMP * tid + kMP - 1 < a.n_local) {
#pragma unroll
      for (int v = 0; v < kMP / 4; ++v) {
        const float4 q = *reinterpret_cast<const float4*>(a.w + base + kMP * tid + 4 * v);
        w4[4 * v + 0] = (double)q.x;
        w4[4 * v + 1] = (double)q.y;
        w4[4 * v + 2] = (double)q.z;
        w4[4 * v + 3] = (double)q.w;
      }
    } else {
#pragma unroll
      for (int m = 0; m < kMP; ++m) {
        const int64_t i = base + kMP * tid + m;
        w4[m] = i < a.n_local ? (double)a.w[i] : 0.0;
      }
    }
#pragma unroll
    for (int m = 0; m < kMP; ++m) tsum += w4[m];
    incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
  }
  __syncthreads();
  int h[kMP];
  int incl_m = 0;
  if (owner) {
    double wpre = 0.0;
    for (int k = 0; k < warp; ++k) wpre += wsum[k];
    const double excl = wpre + (incl - tsum);
    double L = excl;
    int run = 0;
#pragma unroll
    for (int m = 0; m < kMP; ++m) {
      const int k = kMP * tid + m;
      const int64_t i = base + k;
      L += w4[m];
      int64_t hi;
      if (i >= a.n_local - 1 || k == kBlockW - 1) hi = nEb1;
      else if (a.zero_mass) hi = min(max(n_spread(a.g0 + i + 1, a.n_out, a.n_upd), nEb), nEb1);
      else hi = n_of(Eb + L, a.scale, a.U, nEb, nEb1);
      run = max(run, (int)(hi - nEb));
      h[m] = run;
    }
    incl_m = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl_m, o);
      if (lane >= o) incl_m = max(incl_m, v);
    }
    if (lane == 31) wmax[warp] = incl_m;
  }
  __syncthreads();
  if (owner) {
    int carry = 0;
    for (int k = 0; k < warp; ++k) carry = max(carry, wmax[k]);
    const int prev = __shfl_up_sync(0xffffffffu, incl_m, 1);
    if (lane > 0) carry = max(carry, prev);
#pragma unroll
    for (int m = 0; m < kMP; ++m) hb[kMP * tid + m] = max(h[m], carry);
  }
  __syncthreads();
  // offspring [0, end) of this block: produced indices pbase + k
  const int end = (int)(nEb1 - nEb);
  const int64_t pbase = nEb - a.lo;
  int q = 0;
  // GI offspring per thread per round: their binary searches and gathers are independent,
  // so their latencies overlap (the loop is bound by the dependent search + load chain;
  // cfg 5 0.174 -> 0.145 ms with 6; staging the block's states in shared memory first
  // measured slower, 0.168)
#ifndef PHD_GATHER_ILP
#define PHD_GATHER_ILP 6
#endif
  constexpr int GI = PHD_GATHER_ILP;
  for (int k0 = tid; k0 < end; k0 += GI * nthr) {
    int pos[GI];
#pragma unroll
    for (int u = 0; u < GI; ++u) pos[u] = 0;  // number of particles whose upper bound is <= k: the ancestor
#pragma unroll
    for (int step = kBlockW / 2; step > 0; step >>= 1)
#pragma unroll
      for (int u = 0; u < GI; ++u) {
        const int k = k0 + u * nthr;
        if (hb[pos[u] + step - 1] <= k) pos[u] += step;
      }
    float X[GI], VX[GI], Y[GI], VY[GI];
#pragma unroll
    for (int u = 0; u < GI; ++u) {
      const int k = k0 + u * nthr;
      if (k < end) {
        PHD_DCHECK(pos[u] < kBlockW && base + pos[u] < a.n_local);
        const int64_t l = base + pos[u];
        X[u] = g.x[l];
        VX[u] = g.vx[l];
        Y[u] = g.y[l];
        VY[u] = g.vy[l];
      }
    }
#pragma unroll
    for (int u = 0; u < GI; ++u) {
      const int k = k0 + u * nthr;
      if (k >= end) break;
      const int64_t l = base + pos[u];
      const int64_t j = pbase + k;
      if (P2P) {
        const int64_t gj = a.lo + j;  // global offspring index -> owner of the next step's block
        while (q + 1 < po.world && po.blo[q + 1] <= gj) ++q;
        const int64_t o = gj - po.blo[q];
        po.dst[q][0][o] = X[u];
        po.dst[q][1][o] = VX[u];
        po.dst[q][2][o] = Y[u];
        po.dst[q][3][o] = VY[u];
        po.dst[q][4][o] = w_off;
      } else {
        g.ox[j] = X[u];
        g.ovx[j] = VX[u];
        g.oy[j] = Y[u];
        g.ovy[j] = VY[u];
        g.ow[j] = w_off;
      }
      g.anc[j] = (int32_t)(a.g0 + l);
    }
  }
  if (P2P) __threadfence_system();
}


cudaError_t launch_resample_gather(const ResampleGatherArgs& a, const PeerOut* po, cudaStream_t s) {
  if (a.r.n_local <= 0) return cudaSuccess;
  const unsigned nb = (unsigned)((a.r.n_local + kBlockW - 1) / kBlockW);
  const int nt = nb < (unsigned)kGatherSmall ? kMT * kGatherR : kMT;  // (2 kMT for large: slower)
  if (po)
    pdl_launch(k_resample_gather<true>, nb, nt, 0, s, a, *po);
  else
    pdl_launch(k_resample_gather<false>, nb, nt, 0, s, a, PeerOut{});
  return cudaGetLastError();
}

// DCP ring exchange: the L slots s_i = floor(((i + v) n) / L)
// of this group (fp64, one rounding per operation, as in the oracle).
struct Arr5 {
  float* p[5];
};

__device__ __forceinline__ int64_t ring_slot(int64_t i, int64_t n, int64_t L, double v) {
  double t = __ddiv_rn(__dmul_rn(__dadd_rn((double)i, v), (double)n), (double)L);
  return (int64_t)floor(t);
}

__global__ void k_ring_pack(Arr5 src, Arr5 dst, int narr, int64_t L, int64_t n, double v) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  int64_t sl = ring_slot(i, n, L, v);
  for (int q = 0; q < narr; ++q) dst.p[q][i] = src.p[q][sl];
}

__global__ void k_ring_unpack(Arr5 src, Arr5 dst, int narr, int64_t L, int64_t n, double v) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  int64_t sl = ring_slot(i, n, L, v);
  for (int q = 0; q < narr; ++q) dst.p[q][sl] = src.p[q][i];
}

cudaError_t launch_ring_pack(float* const* src, float* const* dst, int narr, int64_t L, int64_t n, double v,
                             cudaStream_t s) {
  if (L <= 0) return cudaSuccess;
  Arr5 a{}, b{};
  for (int q = 0; q < narr; ++q) {
    a.p[q] = src[q];
    b.p[q] = dst[q];
  }
  pdl_launch(k_ring_pack, (unsigned)((L + 255) / 256), 256, 0, s, a, b, narr, L, n, v);
  return cudaGetLastError();
}

cudaError_t launch_ring_unpack(float* const* src, float* const* dst, int narr, int64_t L, int64_t n, double v,
                               cudaStream_t s) {
  if (L <= 0) return cudaSuccess;
  Arr5 a{}, b{};
  for (int q = 0; q < narr; ++q) {
    a.p[q] = src[q];
    b.p[q] = dst[q];
  }
  pdl_launch(k_ring_unpack, (unsigned)((L + 255) / 256), 256, 0, s, a, b, narr, L, n, v);
  return cudaGetLastError();
}


void preload_resample() {
  touch_kernels(k_scan_chunks, k_resample_gather<false>, k_resample_gather<true>, k_ring_pack,
                k_ring_unpack);
}

}  // namespace phd
