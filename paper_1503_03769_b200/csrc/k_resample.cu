// Systematic resampling (Algorithm 1; Step 5 line
// 339), exact over the global particle array and executed rank-locally
// (DESIGN.md §4): rank r scans its own updated weights in fp64 starting at
// O_r = sum_{s<r} W_s; particle i receives the offspring
//   [n(B_{i-1}), n(B_i)),  n(B) = clamp(ceil(B n_out / W - U), 0, n_out),
// pinned so that the ranks' ranges tile [0, n_out) exactly.  Offspring are
// produced in global order by a mark + max-scan + gather pass (HBM-bound).
#include "phd_internal.h"

namespace phd {

__device__ __forceinline__ int64_t n_of(double B, double scale, double U, int64_t lo, int64_t hi) {
  double t = __dsub_rn(__dmul_rn(B, scale), U);
  double c = ceil(t);
  int64_t n = c <= (double)lo ? lo : (c >= (double)hi ? hi : (int64_t)c);
  return n;
}

// One-CTA exclusive scan of a long array (1024 threads): tiles of 4096 loaded
// coalesced into shared memory, each thread folds 4 consecutive elements, a warp
// shuffle scan and a scan of the 32 warp totals give the offsets, the tile is
// written back coalesced, and the carry moves to the next tile.  Fixed order
// (deterministic); Op is associative (fp64 add in this order, or int max).
constexpr int kCtaScanTile = 4096;

template <class T, class Op>
__device__ __forceinline__ T cta_exclusive_scan(const T* in, T* out, int n, T ident, Op op, T* sm, T* ws) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T carry = ident;
  if (n <= 1024) {  // one element per thread, no shared-memory staging
    const T v = tid < n ? in[tid] : ident;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = op(y, incl);
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      T x = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = op(y, x);
      }
      const T prev = __shfl_up_sync(0xffffffffu, x, 1);
      ws[lane] = lane > 0 ? prev : ident;
      if (lane == 31) ws[32] = x;
    }
    __syncthreads();
    const T prevl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (tid < n) out[tid] = lane > 0 ? op(ws[warp], prevl) : ws[warp];
    return ws[32];
  }
  for (int t0 = 0; t0 < n; t0 += kCtaScanTile) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = t0 + r * 1024 + tid;
      sm[r * 1024 + tid] = i < n ? in[i] : ident;
    }
    __syncthreads();
    T v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = sm[4 * tid + k];
    T tot = v[0];
#pragma unroll
    for (int k = 1; k < 4; ++k) tot = op(tot, v[k]);
    T incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = op(y, incl);
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const T x0 = ws[lane];
      T x = x0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = op(y, x);
      }
      const T prev = __shfl_up_sync(0xffffffffu, x, 1);
      ws[lane] = lane > 0 ? op(carry, prev) : carry;  // exclusive warp offsets incl. the carry
      if (lane == 31) ws[32] = op(carry, x);          // carry after this tile
    }
    __syncthreads();
    const T prevl = __shfl_up_sync(0xffffffffu, incl, 1);  // exclusive within the warp
    T run = lane > 0 ? op(ws[warp], prevl) : ws[warp];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      sm[4 * tid + k] = run;
      run = op(run, v[k]);
    }
    carry = ws[32];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = t0 + r * 1024 + tid;
      if (i < n) out[i] = sm[r * 1024 + tid];
    }
    __syncthreads();
  }
  return carry;
}

struct AddF64 {
  __device__ __forceinline__ double operator()(double a, double b) const { return a + b; }
};
struct MaxI32 {
  __device__ __forceinline__ int operator()(int a, int b) const { return max(a, b); }
};

// Exclusive fp64 scan of the per-block masses (one CTA; fixed order); off[nb] = total.
__global__ void __launch_bounds__(1024) k_scan_blocks(const double* __restrict__ blk, int nb, double* off) {
  pdl_wait();
  __shared__ double sm[kCtaScanTile];
  __shared__ double ws[33];
  const double tot = cta_exclusive_scan(blk, off, nb, 0.0, AddF64{}, sm, ws);
  if (threadIdx.x == 0) off[nb] = tot;
}

// Multi-CTA exclusive scan of the block masses, deterministic: CTA c scans its chunk of
// kResScanChunk (warp shuffles, then the warp totals: a fixed tree), writes the local
// exclusive prefixes and its chunk total; the last CTA to finish (atomic ticket) adds the
// chunk totals in order.  Readers form off(b) = coff[b / kResScanChunk] + loc[b].
__global__ void __launch_bounds__(1024) k_scan_chunks(const double* __restrict__ blk, int nb, double* loc,
                                                      double* ctot, double* coff, unsigned* counter) {
  pdl_wait();
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
                               cudaStream_t s) {
  if (nb <= 0) return cudaSuccess;
  pdl_launch(k_scan_chunks, (unsigned)((nb + kResScanChunk - 1) / kResScanChunk), kResScanChunk, 0, s, blk, nb, loc, ctot, coff,
             counter);
  return cudaGetLastError();
}

cudaError_t launch_scan_blocks(const double* blk, int nb, double* blk_off, cudaStream_t s) {
  pdl_launch(k_scan_blocks, 1, 1024, 0, s, blk, nb, blk_off);
  return cudaGetLastError();
}

// Per block of kBlockW particles: local fp64 inclusive prefix, offspring ranges,
// and a mark at the first offspring of every particle with a non-empty range.
// kMP particles per thread (the per-thread scans and bounds are amortised over them).
constexpr int kMP = 8, kMT = kBlockW / kMP;
__global__ void __launch_bounds__(kMT) k_resample_mark(const ResampleArgs a) {
  pdl_wait();
  __shared__ double wsum[kMT / 32];
  __shared__ int his[kMT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.x;
  const int64_t base = b * kBlockW;
  const int64_t nb = (a.n_local + kBlockW - 1) / kBlockW;
  double w4[kMP];
  double tsum = 0.0;
  if (base + kMP * tid + kMP - 1 < a.n_local) {  // 16-byte loads (base is a multiple of kBlockW)
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
      int64_t i = base + kMP * tid + m;
      w4[m] = i < a.n_local ? (double)a.w[i] : 0.0;
    }
  }
#pragma unroll
  for (int m = 0; m < kMP; ++m) tsum += w4[m];
  // block exclusive scan of thread sums: warp shuffle + smem over warps
  double incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  double wpre = 0.0;
  for (int k = 0; k < warp; ++k) wpre += wsum[k];
  double excl = wpre + (incl - tsum);
  // block bounds
  const double Eb = a.O_r + a.blk_off[b];
  const int64_t nEb = (b == 0) ? a.lo : n_of(Eb, a.scale, a.U, a.lo, a.hi);
  const int64_t nEb1 = (b == nb - 1) ? a.hi : n_of(a.O_r + a.blk_off[b + 1], a.scale, a.U, a.lo, a.hi);
  // raw upper bounds, clamped into [n(E_b), n(E_{b+1})]; the block's last particle
  // (and the rank's last) is pinned to n(E_{b+1}); a block-wide running max makes
  // the bounds non-decreasing so the ranges [his[k-1], his[k]) tile the block's
  // offspring exactly (rounding of the fp64 partial sums cannot create gaps or
  // overlaps).
  // offspring bounds as 32-bit offsets from n(E_b) (a rank produces < 2^31 offspring)
  __shared__ int wmax[kMT / 32];
  double L = excl;
  int run = 0;
  int h[kMP];
#pragma unroll
  for (int m = 0; m < kMP; ++m) {
    int k = kMP * tid + m;
    int64_t i = base + k;
    L += w4[m];
    int64_t hi;
    if (i >= a.n_local - 1 || k == kBlockW - 1) hi = nEb1;
    else hi = n_of(Eb + L, a.scale, a.U, nEb, nEb1);
    run = max(run, (int)(hi - nEb));
    h[m] = run;
  }
  int incl_m = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl_m, o);
    if (lane >= o) incl_m = max(incl_m, v);
  }
  if (lane == 31) wmax[warp] = incl_m;
  __syncthreads();
  int carry = 0;
  for (int k = 0; k < warp; ++k) carry = max(carry, wmax[k]);
  const int prev = __shfl_up_sync(0xffffffffu, incl_m, 1);
  if (lane > 0) carry = max(carry, prev);
#pragma unroll
  for (int m = 0; m < kMP; ++m) h[m] = max(h[m], carry);
  his[tid] = h[kMP - 1];  // each thread's last bound: the next thread's first lower bound
  __syncthreads();
  int lo = tid == 0 ? 0 : his[tid - 1];
  const int end = (int)(nEb1 - nEb);
#pragma unroll
  for (int m = 0; m < kMP; ++m) {
    const int64_t i = base + kMP * tid + m;
    if (i >= a.n_local) break;
    if (h[m] > lo) {
      const int64_t p = nEb + lo - a.lo;  // first offspring, local produced index
      a.marks[p] = (int32_t)(a.g0 + i);
      // the ranges tile the offspring, so the block's next mark (if any) sits at h[m]:
      // this mark is the block's last in its offspring block iff that position is
      // past the block's range or in another offspring block -> max per offspring
      // block (integer atomicMax: order-independent, k_scan_max then scans it)
      if (h[m] == end || (p + (h[m] - lo)) / kBlockOff != p / kBlockOff)
        atomicMax(&a.bmax[p / kBlockOff], (int32_t)(a.g0 + i));
    }
    lo = h[m];
  }
}

cudaError_t launch_resample_mark(const ResampleArgs& a, cudaStream_t s) {
  if (a.n_local <= 0) return cudaSuccess;
  unsigned nb = (unsigned)((a.n_local + kBlockW - 1) / kBlockW);
  pdl_launch(k_resample_mark, nb, kMT, 0, s, a);
  return cudaGetLastError();
}

// Systematic resampling and the offspring gather in one pass: per block
// of kBlockW particles the bounds of k_resample_mark (same fp64 formula and pinning),
// all kBlockW upper bounds in shared memory; then every offspring k of the block finds
// its particle by binary search over those bounds (balanced whatever the weights) and
// copies its state (coalesced writes at consecutive produced indices).  Reads w + state
// (20 B) per particle, writes state + w + ancestor (24 B) per offspring; no marks, no
// memsets, no max-scan.
template <bool P2P>
__global__ void __launch_bounds__(kMT) k_resample_gather(const ResampleGatherArgs g, const PeerOut po) {
  pdl_wait();
  const ResampleArgs& a = g.r;
  __shared__ double wsum[kMT / 32];
  __shared__ int wmax[kMT / 32];
  __shared__ int hb[kBlockW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.x;
  const int64_t base = b * kBlockW;
  const int64_t nb = (a.n_local + kBlockW - 1) / kBlockW;
  double w4[kMP];
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
  double tsum = 0.0;
#pragma unroll
  for (int m = 0; m < kMP; ++m) tsum += w4[m];
  double incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  double wpre = 0.0;
  for (int k = 0; k < warp; ++k) wpre += wsum[k];
  const double excl = wpre + (incl - tsum);
  // block bounds from off(b) = coff[b / kResScanChunk] + loc[b] (every reader forms the same bits)
  auto off = [&](int64_t bb) { return g.coff[bb / kResScanChunk] + a.blk_off[bb]; };
  const double Eb = a.O_r + off(b);
  const int64_t nEb = (b == 0) ? a.lo : n_of(Eb, a.scale, a.U, a.lo, a.hi);
  const int64_t nEb1 = (b == nb - 1) ? a.hi : n_of(a.O_r + off(b + 1), a.scale, a.U, a.lo, a.hi);
  double L = excl;
  int run = 0;
  int h[kMP];
#pragma unroll
  for (int m = 0; m < kMP; ++m) {
    const int k = kMP * tid + m;
    const int64_t i = base + k;
    L += w4[m];
    int64_t hi;
    if (i >= a.n_local - 1 || k == kBlockW - 1) hi = nEb1;
    else hi = n_of(Eb + L, a.scale, a.U, nEb, nEb1);
    run = max(run, (int)(hi - nEb));
    h[m] = run;
  }
  int incl_m = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl_m, o);
    if (lane >= o) incl_m = max(incl_m, v);
  }
  if (lane == 31) wmax[warp] = incl_m;
  __syncthreads();
  int carry = 0;
  for (int k = 0; k < warp; ++k) carry = max(carry, wmax[k]);
  const int prev = __shfl_up_sync(0xffffffffu, incl_m, 1);
  if (lane > 0) carry = max(carry, prev);
#pragma unroll
  for (int m = 0; m < kMP; ++m) hb[kMP * tid + m] = max(h[m], carry);
  __syncthreads();
  // offspring [0, end) of this block: produced indices pbase + k
  const int end = (int)(nEb1 - nEb);
  const int64_t pbase = nEb - a.lo;
  int q = 0;
  for (int k = tid; k < end; k += kMT) {
    int pos = 0;  // number of particles whose upper bound is <= k: the ancestor
#pragma unroll
    for (int step = kBlockW / 2; step > 0; step >>= 1)
      if (hb[pos + step - 1] <= k) pos += step;
    PHD_DCHECK(pos < kBlockW && base + pos < a.n_local);
    const int64_t l = base + pos;
    const int64_t j = pbase + k;
    const float X = g.x[l], VX = g.vx[l], Y = g.y[l], VY = g.vy[l];
    if (P2P) {
      const int64_t gj = a.lo + j;  // global offspring index -> owner of the next step's block
      while (q + 1 < po.world && po.blo[q + 1] <= gj) ++q;
      const int64_t o = gj - po.blo[q];
      po.dst[q][0][o] = X;
      po.dst[q][1][o] = VX;
      po.dst[q][2][o] = Y;
      po.dst[q][3][o] = VY;
      po.dst[q][4][o] = g.w_off;
    } else {
      g.ox[j] = X;
      g.ovx[j] = VX;
      g.oy[j] = Y;
      g.ovy[j] = VY;
      g.ow[j] = g.w_off;
    }
    g.anc[j] = (int32_t)(a.g0 + l);
  }
  if (P2P) __threadfence_system();
}

cudaError_t launch_resample_gather(const ResampleGatherArgs& a, const PeerOut* po, cudaStream_t s) {
  if (a.r.n_local <= 0) return cudaSuccess;
  const unsigned nb = (unsigned)((a.r.n_local + kBlockW - 1) / kBlockW);
  if (po)
    pdl_launch(k_resample_gather<true>, nb, kMT, 0, s, a, *po);
  else
    pdl_launch(k_resample_gather<false>, nb, kMT, 0, s, a, PeerOut{});
  return cudaGetLastError();
}

__device__ __forceinline__ int warp_max_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = max(v, u);
  }
  return v;
}

// In place: bmax[b] <- max(bmax[0..b-1]) (exclusive; -1 for b = 0).
__global__ void __launch_bounds__(1024) k_scan_max(int32_t* bmax, int nb) {
  pdl_wait();
  __shared__ int sm[kCtaScanTile];
  __shared__ int ws[33];
  cta_exclusive_scan(bmax, bmax, nb, -1, MaxI32{}, sm, ws);
}

cudaError_t launch_scan_max(int32_t* bmax, int nb, cudaStream_t s) {
  if (nb <= 0) return cudaSuccess;
  pdl_launch(k_scan_max, 1, 1024, 0, s, bmax, nb);
  return cudaGetLastError();
}

// Offspring j (local produced index): ancestor = running max of the marks;
// copy the ancestor's state, set the offspring weight W / n_out.
__global__ void __launch_bounds__(256) k_gather(const int32_t* __restrict__ marks, const int32_t* __restrict__ bex,
                                                int64_t n, int64_t g0, const float* __restrict__ x,
                                                const float* __restrict__ vx, const float* __restrict__ y,
                                                const float* __restrict__ vy, float w_off, float* ox, float* ovx,
                                                float* oy, float* ovy, float* ow, int32_t* anc, int zero_mass,
                                                int64_t first, int64_t n_upd, int64_t n_out) {
  pdl_wait();
  __shared__ int wm[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kBlockOff;
  int a4[4];
  if (zero_mass) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int64_t j = base + 4 * tid + r;
      a4[r] = (int)(((first + j) * n_upd) / n_out);
    }
  } else {
    int m = -1;
    const int64_t j0 = base + 4 * tid;
    if (j0 + 3 < n) {  // 16-byte load (base is a multiple of kBlockOff)
      const int4 q = *reinterpret_cast<const int4*>(marks + j0);
      a4[0] = q.x;
      a4[1] = q.y;
      a4[2] = q.z;
      a4[3] = q.w;
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) a4[r] = j0 + r < n ? marks[j0 + r] : -1;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      m = max(m, a4[r]);
      a4[r] = m;  // thread-local inclusive running max
    }
    int incl = warp_max_scan(m, lane);
    if (lane == 31) wm[warp] = incl;
    __syncthreads();
    int carry = bex[blockIdx.x];
    for (int k = 0; k < warp; ++k) carry = max(carry, wm[k]);
    int prev = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane > 0) carry = max(carry, prev);
#pragma unroll
    for (int r = 0; r < 4; ++r) a4[r] = max(a4[r], carry);
  }
  const int64_t j0 = base + 4 * tid;
  if (j0 + 3 < n) {  // 16-byte stores of four consecutive offspring
    float4 X, VX, Y, VY;
    float* px = &X.x;
    float* pvx = &VX.x;
    float* py = &Y.x;
    float* pvy = &VY.x;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t l = (int64_t)a4[r] - g0;
      px[r] = __ldg(x + l);
      pvx[r] = __ldg(vx + l);
      py[r] = __ldg(y + l);
      pvy[r] = __ldg(vy + l);
    }
    *reinterpret_cast<float4*>(ox + j0) = X;
    *reinterpret_cast<float4*>(ovx + j0) = VX;
    *reinterpret_cast<float4*>(oy + j0) = Y;
    *reinterpret_cast<float4*>(ovy + j0) = VY;
    *reinterpret_cast<float4*>(ow + j0) = make_float4(w_off, w_off, w_off, w_off);
    *reinterpret_cast<int4*>(anc + j0) = make_int4(a4[0], a4[1], a4[2], a4[3]);
    return;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int64_t j = j0 + r;
    if (j >= n) break;
    int64_t l = (int64_t)a4[r] - g0;
    ox[j] = x[l];
    ovx[j] = vx[l];
    oy[j] = y[l];
    ovy[j] = vy[l];
    ow[j] = w_off;
    anc[j] = a4[r];
  }
}

cudaError_t launch_gather(const int32_t* marks, const int32_t* bmax_excl, int64_t n, int64_t g0, const float* x,
                          const float* vx, const float* y, const float* vy, float w_off, float* ox, float* ovx,
                          float* oy, float* ovy, float* ow, int32_t* anc, int zero_mass, int64_t first,
                          int64_t n_global_upd, int64_t n_out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pdl_launch(k_gather, (unsigned)((n + kBlockOff - 1) / kBlockOff), 256, 0, s, 
      marks, bmax_excl, n, g0, x, vx, y, vy, w_off, ox, ovx, oy, ovy, ow, anc, zero_mass, first, n_global_upd, n_out);
  return cudaGetLastError();
}

// Fused resample + exchange: offspring g = first + j goes straight
// to its owner q of the next step's block partition (blo), at local slot
// g - blo[q], stored through the peer-memory window (NVLink P2P for one process
// per GPU).  Consecutive offspring have consecutive destinations, so the remote
// stores of a warp coalesce.  The caller's collective barrier after this kernel
// orders the stores before any rank reads its next-step array.
__global__ void __launch_bounds__(256) k_gather_p2p(const int32_t* __restrict__ marks, const int32_t* __restrict__ bex,
                                                    int64_t n, int64_t g0, const float* __restrict__ x,
                                                    const float* __restrict__ vx, const float* __restrict__ y,
                                                    const float* __restrict__ vy, float w_off, const PeerOut po,
                                                    int32_t* anc, int zero_mass, int64_t first, int64_t n_upd,
                                                    int64_t n_out) {
  pdl_wait();
  __shared__ int wm[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kBlockOff;
  int a4[4];
  if (zero_mass) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int64_t j = base + 4 * tid + r;
      a4[r] = (int)(((first + j) * n_upd) / n_out);
    }
  } else {
    int m = -1;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int64_t j = base + 4 * tid + r;
      a4[r] = j < n ? marks[j] : -1;
      m = max(m, a4[r]);
      a4[r] = m;
    }
    int incl = warp_max_scan(m, lane);
    if (lane == 31) wm[warp] = incl;
    __syncthreads();
    int carry = bex[blockIdx.x];
    for (int k = 0; k < warp; ++k) carry = max(carry, wm[k]);
    int prev = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane > 0) carry = max(carry, prev);
#pragma unroll
    for (int r = 0; r < 4; ++r) a4[r] = max(a4[r], carry);
  }
  int q = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t j = base + 4 * tid + r;
    if (j >= n) break;
    const int64_t g = first + j;
    while (q + 1 < po.world && po.blo[q + 1] <= g) ++q;
    const int64_t off = g - po.blo[q];
    const int64_t l = (int64_t)a4[r] - g0;
    po.dst[q][0][off] = x[l];
    po.dst[q][1][off] = vx[l];
    po.dst[q][2][off] = y[l];
    po.dst[q][3][off] = vy[l];
    po.dst[q][4][off] = w_off;
    anc[j] = a4[r];
  }
  __threadfence_system();
}

cudaError_t launch_gather_p2p(const int32_t* marks, const int32_t* bmax_excl, int64_t n, int64_t g0, const float* x,
                              const float* vx, const float* y, const float* vy, float w_off, const PeerOut& po,
                              int32_t* anc, int zero_mass, int64_t first, int64_t n_global_upd, int64_t n_out,
                              cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pdl_launch(k_gather_p2p, (unsigned)((n + kBlockOff - 1) / kBlockOff), 256, 0, s, 
      marks, bmax_excl, n, g0, x, vx, y, vy, w_off, po, anc, zero_mass, first, n_global_upd, n_out);
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

}  // namespace phd
