// Gated particle x measurement update (SURVEY.md §8(f) NEXT-2 "measurement
// gating by spatial binning"; DESIGN.md §5 "Gated update").
//
// The dense passes (k_update.cu) evaluate every (particle, measurement) pair,
// although at these configs almost all terms p_D g(z|x) w underflow: with
// sigma = 10 m a term is below 2^-126 (and flushed to exactly 0 by
// ex2.approx.ftz) once |x - z| exceeds ~120 m.  This path computes the same
// non-zero terms and skips only pairs whose exponent is provably below -130:
//
//   1. k_gate_keys + counting sort: each particle gets the Morton key of its
//      64 x 64 cell in measurement space ((x, y), or (r, theta) for the
//      range-bearing sensor); a stable counting sort orders the particle
//      indices by cell, and k_gate_gather writes a sorted copy of the state
//      (the filter's own particle order, which defines resampling, is untouched).
//   2. k_gate_zbin: measurements binned into the same cells (one CTA).
//   3. k_gate_tiles: per tile of kGateTP sorted particles, the bounding box and
//      max log2(p_D c w); a measurement is a candidate of the tile iff
//         e_max = -alpha0 dx^2 - alpha1 dy^2 + max_i log2(p_D c w_i) >= -130
//      with (dx, dy) its distance to the box (wrapped in bearing).  Every term
//      of a non-candidate pair has e <= e_max < -130 (fp32 rounding of the
//      kernels' exponent is ~1e-4 here), so it is exactly 0 in the dense path.
//   4. k_gpass<1>: CTA per tile, two particles per thread (f32x2), candidates
//      broadcast from shared memory; the same per-pair arithmetic as the dense
//      pass (pair_math.cuh), so every term is bitwise the dense kernel's.  Tile
//      sums per candidate: warp tree (transposed butterfly), fp64 across warps.
//   5. the entries (tile, candidate) are stably sorted by label and k_gate_reduce
//      sums each label's tile partials in entry order (fp64, warp tree):
//      deterministic, no atomics on floating point.
//   6. k_gpass<2>: weights (sum_z u d_z per particle, complete inside the CTA)
//      and the centred STPHD state sums for candidates in the index set I.
#include "phd_internal.h"
#include "pair_math.cuh"

namespace phd {

namespace {

constexpr float kPi = 3.14159265358979323846f;
constexpr float kTwoPi = 6.28318530717958647692f;

__device__ __forceinline__ uint32_t spread6(uint32_t v) {
  v &= 63u;
  v = (v | (v << 4)) & 0x0F0Fu;
  v = (v | (v << 2)) & 0x3333u;
  v = (v | (v << 1)) & 0x5555u;
  return v;
}
__device__ __forceinline__ int morton(int c0, int c1) { return (int)(spread6((uint32_t)c0) | (spread6((uint32_t)c1) << 1)); }

// unclamped cell coordinate (monotone in v: one rounded subtract, one rounded multiply)
__device__ __forceinline__ int cell_raw(float v, float lo, float inv_h) {
  float t = __fmul_rn(__fsub_rn(v, lo), inv_h);
  t = fminf(fmaxf(t, -1.0e6f), 1.0e6f);  // NaN -> -1e6 (fmaxf), inf clamped
  return (int)floorf(t);
}
__device__ __forceinline__ int clampc(int c) { return min(max(c, 0), kGateG - 1); }
__device__ __forceinline__ int wrapc(int c) { return ((c % kGateG) + kGateG) % kGateG; }

__device__ __forceinline__ int cell_key(float v0, float v1, const GateGrid& g) {
  int c0 = clampc(cell_raw(v0, g.lo0, g.inv_h0));
  int c1 = cell_raw(v1, g.lo1, g.inv_h1);
  c1 = g.wrap1 ? wrapc(c1) : clampc(c1);
  return morton(c0, c1);
}

// distance from v to [a, b]
__device__ __forceinline__ float dist_iv(float v, float a, float b) { return fmaxf(0.0f, fmaxf(a - v, v - b)); }
// distance from the angle v (any real, e.g. fp32(pi) > pi) to the arc [a, b]
// (a <= b); 0 when the arc covers the circle.  Slightly under-estimated (1e-5).
__device__ __forceinline__ float dist_arc(float v, float a, float b) {
  const float len = b - a;
  float t = v - a;
  t -= kTwoPi * floorf(t / kTwoPi);  // angle from a to v, in [0, 2 pi]
  if (len >= kTwoPi || t <= len) return 0.0f;
  return fmaxf(0.0f, fminf(t - len, kTwoPi - t) - 1e-5f);
}

// ---------------------------------------------------------------------------
// int32 exclusive scan (chunks of 4096 = 1024 threads x 4)
constexpr int kScanChunk = 4096;

__device__ __forceinline__ int block_excl_scan_1024(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = sh[lane];
    int t = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sh[lane] = t - s;
    if (lane == 31) sh[32] = t;
  }
  __syncthreads();
  int r = x - v + sh[warp];
  *total = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) k_scan_sum(const int32_t* __restrict__ a, int64_t n, int32_t* csum) {
  __shared__ int sh[33];
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * 4;
  int s = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (base + r < n) s += a[base + r];
  int tot;
  block_excl_scan_1024(s, sh, &tot);
  if (threadIdx.x == 0) csum[blockIdx.x] = tot;
}

// one CTA: exclusive scan of csum[0..nc), csum[nc] = total, *total_out = total
__global__ void __launch_bounds__(1024) k_scan_top(int32_t* csum, int nc, int32_t* total_out) {
  __shared__ int sh[33];
  int carry = 0;
  for (int b = 0; b < nc; b += 1024) {
    int i = b + threadIdx.x;
    int v = i < nc ? csum[i] : 0;
    int tot;
    int e = block_excl_scan_1024(v, sh, &tot);
    if (i < nc) csum[i] = e + carry;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    csum[nc] = carry;
    if (total_out) *total_out = carry;
  }
}

__global__ void __launch_bounds__(1024) k_scan_apply(int32_t* a, int64_t n, const int32_t* __restrict__ csum) {
  __shared__ int sh[33];
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * 4;
  int v[4];
  int s = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    v[r] = base + r < n ? a[base + r] : 0;
    s += v[r];
  }
  int tot;
  int e = block_excl_scan_1024(s, sh, &tot) + csum[blockIdx.x];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (base + r < n) a[base + r] = e;
    e += v[r];
  }
}

// ---------------------------------------------------------------------------
// Stable counting sort pass on bits [shift, shift + log2 nbins) of keys.
// hist is bin-major, hist[bin * nblk + blk], so its exclusive scan is the
// first output position of every (bin, block): stable across blocks; within a
// block one warp walks the keys in order (match_any ranks equal bins).
__global__ void __launch_bounds__(256) k_csort_hist(const int32_t* __restrict__ keys, int64_t n, int shift, int nbins,
                                                    int nblk, int32_t* hist) {
  __shared__ int h[kSortMaxBins];
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * kSortBlock;
  const int64_t i1 = min(n, i0 + kSortBlock);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) atomicAdd(&h[(keys[i] >> shift) & (nbins - 1)], 1);
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) hist[(int64_t)b * nblk + blockIdx.x] = h[b];
}

__global__ void __launch_bounds__(32) k_csort_scatter(const int32_t* __restrict__ keys, const int32_t* __restrict__ vals,
                                                      int64_t n, int shift, int nbins, int nblk,
                                                      const int32_t* __restrict__ hs, int32_t* out_keys,
                                                      int32_t* out_vals) {
  __shared__ int cnt[kSortMaxBins];
  const int lane = threadIdx.x;
  for (int b = lane; b < nbins; b += 32) cnt[b] = hs[(int64_t)b * nblk + blockIdx.x];
  __syncwarp();
  const int64_t i0 = (int64_t)blockIdx.x * kSortBlock;
  const int64_t i1 = min(n, i0 + kSortBlock);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = i0; base < i1; base += 32) {
    const int64_t i = base + lane;
    const bool ok = i < i1;
    const int key = ok ? keys[i] : 0;
    const int bin = ok ? ((key >> shift) & (nbins - 1)) : kSortMaxBins + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    int pos = 0;
    if (ok) pos = cnt[bin] + __popc(peers & lt);
    __syncwarp();
    if (ok) {
      if (lane == __ffs(peers) - 1) cnt[bin] += __popc(peers);
      if (out_keys) out_keys[pos] = key;
      out_vals[pos] = vals ? vals[i] : (int32_t)i;
    }
    __syncwarp();
  }
}

cudaError_t csort_pass(const int32_t* keys, const int32_t* vals, int64_t n, int shift, int nbins, int32_t* hist,
                       int32_t* scan_tmp, int32_t* out_keys, int32_t* out_vals, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  const int nblk = (int)((n + kSortBlock - 1) / kSortBlock);
  k_csort_hist<<<nblk, 256, 0, s>>>(keys, n, shift, nbins, nblk, hist);
  ++*launches;
  cudaError_t e = gate_scan(hist, (int64_t)nbins * nblk, scan_tmp, s, launches);
  if (e != cudaSuccess) return e;
  k_csort_scatter<<<nblk, 32, 0, s>>>(keys, vals, n, shift, nbins, nblk, hist, out_keys, out_vals);
  ++*launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// particle keys: position (x, y); range-bearing (r_hi, thetaA_hi)
__global__ void k_gate_keys(int model, const float* __restrict__ a0, const float* __restrict__ a1, int64_t n,
                            GateGrid g, int32_t* keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = cell_key(a0[i], a1[i], g);
}

struct GatherSrc {
  const float* c[8];
  const float *x, *y, *vx, *vy, *w;
};

// sorted copy; padding positions [n, n_pad) get zero state and lw = -inf
__global__ void k_gate_gather(int model, GatherSrc src, int64_t n, int64_t n_pad, float wscale, GateSorted so) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pad) return;
  const bool rb = model == kRangeBearing;
  if (p < n) {
    const int i = so.perm[p];
    if (rb) {
#pragma unroll
      for (int c = 0; c < 8; ++c) so.c[c][p] = src.c[c][i];
    }
    so.x[p] = src.x[i];
    so.y[p] = src.y[i];
    so.vx[p] = src.vx[i];
    so.vy[p] = src.vy[i];
    so.lw[p] = log2f(src.w[i] * wscale);  // the dense TileLoader's exact expression
    so.inv[i] = (int32_t)p;
  } else {
    if (rb) {
#pragma unroll
      for (int c = 0; c < 8; ++c) so.c[c][p] = 0.0f;
    }
    so.x[p] = 0.0f;
    so.y[p] = 0.0f;
    so.vx[p] = 0.0f;
    so.vy[p] = 0.0f;
    so.lw[p] = -INFINITY;
  }
}

// ---------------------------------------------------------------------------
// measurements -> cells (one CTA of 1024): zcell_start[kGateBins + 1], items
// stable by label within a cell (warp 0 walks the labels in order)
__global__ void __launch_bounds__(1024) k_gate_zbin(const float* __restrict__ z, int M, GateGrid g,
                                                    int32_t* zkey, int32_t* zcell_start, int32_t* zcell_items) {
  __shared__ int h[kGateBins];
  __shared__ int sh[33];
  for (int b = threadIdx.x; b < kGateBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (int l = threadIdx.x; l < M; l += blockDim.x) {
    int k = cell_key(z[2 * l], z[2 * l + 1], g);
    zkey[l] = k;
    atomicAdd(&h[k], 1);
  }
  __syncthreads();
  // exclusive scan of 4096 bins (4 per thread)
  int v[4], s = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    v[r] = h[threadIdx.x * 4 + r];
    s += v[r];
  }
  int tot;
  int e = block_excl_scan_1024(s, sh, &tot);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    zcell_start[threadIdx.x * 4 + r] = e;
    h[threadIdx.x * 4 + r] = e;
    e += v[r];
  }
  if (threadIdx.x == 0) zcell_start[kGateBins] = tot;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const unsigned lt = (1u << lane) - 1u;
    for (int b = 0; b < M; b += 32) {
      int l = b + lane;
      bool ok = l < M;
      int k = ok ? zkey[l] : kGateBins + lane;
      unsigned peers = __match_any_sync(0xffffffffu, k);
      int pos = ok ? h[k] + __popc(peers & lt) : 0;
      __syncwarp();
      if (ok) {
        if (lane == __ffs(peers) - 1) h[k] += __popc(peers);
        zcell_items[pos] = l;
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// per tile (one warp): bounding box in measurement space, max log2(p_D c w),
// then the candidates: cells of the window in rounds of 32 (lane = cell),
// measurements of a cell in item order; FILL writes them at tstart[t] in
// (round, lane, item) order -- deterministic.
template <bool FILL>
__global__ void __launch_bounds__(256) k_gate_tiles(int model, const float* __restrict__ c0, const float* __restrict__ c1,
                                                    const float* __restrict__ lw, int ntiles, float na0, float na1,
                                                    GateGrid g, const int32_t* __restrict__ zcell_start,
                                                    const int32_t* __restrict__ zcell_items,
                                                    const float* __restrict__ z, int32_t* tcount,
                                                    const int32_t* __restrict__ tstart, int32_t* cand) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  const int64_t p0 = (int64_t)t * kGateTP;
  float b0 = INFINITY, b1 = -INFINITY, e0 = INFINITY, e1 = -INFINITY, lm = -INFINITY;
  for (int j = lane; j < kGateTP; j += 32) {
    const float l = lw[p0 + j];
    if (l > -INFINITY) {  // zero-weight particles and padding contribute nothing
      const float v0 = c0[p0 + j], v1 = c1[p0 + j];
      b0 = fminf(b0, v0);
      b1 = fmaxf(b1, v0);
      e0 = fminf(e0, v1);
      e1 = fmaxf(e1, v1);
      lm = fmaxf(lm, l);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    b0 = fminf(b0, __shfl_xor_sync(0xffffffffu, b0, o));
    b1 = fmaxf(b1, __shfl_xor_sync(0xffffffffu, b1, o));
    e0 = fminf(e0, __shfl_xor_sync(0xffffffffu, e0, o));
    e1 = fmaxf(e1, __shfl_xor_sync(0xffffffffu, e1, o));
    lm = fmaxf(lm, __shfl_xor_sync(0xffffffffu, lm, o));
  }
  const float budget = lm - kGateLog2Min;  // e_max >= -130  <=>  alpha0 dx^2 + alpha1 dy^2 <= budget
  int total = 0;
  int out = FILL ? tstart[t] : 0;
  if (budget > 0.0f && isfinite(b0) && isfinite(e0) && isfinite(b1) && isfinite(e1)) {
    const float R0 = sqrtf(budget / -na0) * 1.0001f + 1e-3f;
    const float R1 = sqrtf(budget / -na1) * 1.0001f + 1e-6f;
    const int x0 = clampc(cell_raw(b0 - R0, g.lo0, g.inv_h0)), x1 = clampc(cell_raw(b1 + R0, g.lo0, g.inv_h0));
    int y0, y1;
    if (g.wrap1) {
      y0 = cell_raw(e0 - R1, g.lo1, g.inv_h1) - 1;
      y1 = cell_raw(e1 + R1, g.lo1, g.inv_h1) + 1;
      if (y1 - y0 + 1 >= kGateG) {
        y0 = 0;
        y1 = kGateG - 1;
      }
    } else {
      y0 = clampc(cell_raw(e0 - R1, g.lo1, g.inv_h1));
      y1 = clampc(cell_raw(e1 + R1, g.lo1, g.inv_h1));
    }
    const int nx = x1 - x0 + 1, ny = y1 - y0 + 1;
    const int nc = nx * ny;
    for (int r = 0; r < nc; r += 32) {
      const int ci = r + lane;
      int cnt = 0, j0 = 0, j1 = 0;
      if (ci < nc) {
        const int cx = x0 + ci % nx;
        int cy = y0 + ci / nx;
        if (g.wrap1) cy = wrapc(cy);
        const int key = morton(cx, cy);
        j0 = zcell_start[key];
        j1 = zcell_start[key + 1];
        for (int j = j0; j < j1; ++j) {
          const int l = zcell_items[j];
          const float z0 = z[2 * l], z1 = z[2 * l + 1];
          const float dx = dist_iv(z0, b0, b1);
          const float dy = g.wrap1 ? dist_arc(z1, e0, e1) : dist_iv(z1, e0, e1);
          const float em = fmaf(na0, dx * dx, fmaf(na1, dy * dy, lm));
          if (em >= kGateLog2Min) ++cnt;
        }
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (FILL && cnt > 0) {
        int w = out + incl - cnt;
        for (int j = j0; j < j1; ++j) {
          const int l = zcell_items[j];
          const float z0 = z[2 * l], z1 = z[2 * l + 1];
          const float dx = dist_iv(z0, b0, b1);
          const float dy = g.wrap1 ? dist_arc(z1, e0, e1) : dist_iv(z1, e0, e1);
          const float em = fmaf(na0, dx * dx, fmaf(na1, dy * dy, lm));
          if (em >= kGateLog2Min) cand[w++] = l;
        }
      }
      const int rt = __shfl_sync(0xffffffffu, incl, 31);
      out += rt;
      total += rt;
    }
  }
  if (!FILL && lane == 0) tcount[t] = total;
}

// per-label entry counts (integer atomics: order-independent)
__global__ void k_gate_count_labels(const int32_t* __restrict__ cand, int64_t E, int32_t* cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) atomicAdd(&cnt[cand[e]], 1);
}

__global__ void k_zero_i32(int32_t* a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = 0;
}

// ---------------------------------------------------------------------------
// The gated passes.  Tile t = sorted particles [t*512, t*512 + 512); thread
// tid holds particles tid and tid + 256 as one f32x2 pair.
template <int MODEL>
struct GPart {
  float2 X, Y, LW;            // position: x, y (residual coordinates); all: Cartesian x, y for pass 2
  float2 R_hi, R_lo, T_hi[3], T_lo[3];  // range-bearing representation
  float2 VX, VY;
};

template <int MODEL, int PASS>
__global__ void __launch_bounds__(256, 3) k_gpass(const GateArgs g) {
  constexpr bool RB = MODEL == kRangeBearing;
  __shared__ float2 zn[kGateChunk];          // (-z0, -z1)
  __shared__ float zd[kGateChunk];           // 1 / (kappa + C)          (pass 2)
  __shared__ int zr[kGateChunk];             // bearing representation   (range-bearing)
  __shared__ float2 zc[kGateChunk];          // -(Cartesian centre)      (range-bearing, pass 2)
  __shared__ int zi[kGateChunk];             // chunk-local entry index  (pass 2: selected first)
  __shared__ int wcnt[9];
  __shared__ float wpart[8][kGateChunk];     // pass 1: per-warp candidate sums
  __shared__ float4 wq[PASS == 2 ? 8 : 1][PASS == 2 ? kGateChunk : 1];  // pass 2: per-warp state sums

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = blockIdx.x;
  const int64_t pa = (int64_t)t * kGateTP + tid, pb = pa + 256;
  const float2 na0 = f2(g.na0, g.na0), na1 = f2(g.na1, g.na1);
  GPart<MODEL> P;
  P.LW = f2(g.so.lw[pa], g.so.lw[pb]);
  if (RB) {
    P.R_hi = f2(g.so.c[0][pa], g.so.c[0][pb]);
    P.R_lo = f2(g.so.c[1][pa], g.so.c[1][pb]);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      P.T_hi[r] = f2(g.so.c[2 + 2 * r][pa], g.so.c[2 + 2 * r][pb]);
      P.T_lo[r] = f2(g.so.c[3 + 2 * r][pa], g.so.c[3 + 2 * r][pb]);
    }
  }
  if (!RB || PASS == 2) {
    P.X = f2(g.so.x[pa], g.so.x[pb]);
    P.Y = f2(g.so.y[pa], g.so.y[pb]);
  }
  if (PASS == 2) {
    P.VX = f2(g.so.vx[pa], g.so.vx[pb]);
    P.VY = f2(g.so.vy[pa], g.so.vy[pb]);
  }
  const int e0 = g.tstart[t];
  const int K = g.tstart[t + 1] - e0;
  float2 pacc = f2(0.0f, 0.0f);

  // u = p_D g(z_k | x) w for the thread's two particles (bitwise the dense term)
  auto term = [&](int k, float2& d0, float2& d1) -> float2 {
    const float2 nz = zn[k];
    if (RB) {
      const int rep = zr[k];
      const float2 th = rep == 0 ? P.T_hi[0] : (rep == 1 ? P.T_hi[1] : P.T_hi[2]);
      const float2 tl = rep == 0 ? P.T_lo[0] : (rep == 1 ? P.T_lo[1] : P.T_lo[2]);
      d0 = __fadd2_rn(__fadd2_rn(P.R_hi, f2(nz.x, nz.x)), P.R_lo);  // (r_hi - z_r) + r_lo
      d1 = __fadd2_rn(__fadd2_rn(th, f2(nz.y, nz.y)), tl);          // (th_hi - z_th) + th_lo
    } else {
      d0 = __fadd2_rn(P.X, f2(nz.x, nz.x));  // x - z_x
      d1 = __fadd2_rn(P.Y, f2(nz.y, nz.y));  // y - z_y
    }
    return ex2v(expo<MODEL>(d0, d1, na0, na1, P.LW));
  };

  for (int cb = 0; cb < K; cb += kGateChunk) {
    const int cl = min(kGateChunk, K - cb);
    const int cl8 = (cl + 7) & ~7;
    __syncthreads();  // previous chunk fully consumed
    int nsel = 0;
    if (PASS == 1) {
      if (tid < cl8) {
        if (tid < cl) {
          const int l = g.cand[e0 + cb + tid];
          zn[tid] = f2(g.sc.s0[l], g.sc.s1[l]);
          if (RB) zr[tid] = g.sc.rep[l];
        } else {
          zn[tid] = f2(-1e30f, -1e30f);  // sentinel: every term exactly 0
          if (RB) zr[tid] = 0;
        }
      }
    } else {
      // stable partition: labels in I first (their state sums are reduced), then the rest
      int l = -1, fl = 0;
      if (tid < cl) {
        l = g.cand[e0 + cb + tid];
        fl = g.sel == nullptr ? 1 : (g.sel[l] != 0);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, fl);
      if (lane == 0) wcnt[warp] = __popc(bal);
      __syncthreads();
      if (tid == 0) {
        int s = 0;
        for (int w = 0; w < 8; ++w) {
          const int c = wcnt[w];
          wcnt[w] = s;
          s += c;
        }
        wcnt[8] = s;
      }
      __syncthreads();
      nsel = wcnt[8];
      if (tid < cl) {
        const int before = wcnt[warp] + __popc(bal & ((1u << lane) - 1u));
        const int pos = fl ? before : nsel + (tid - before);
        zn[pos] = f2(g.sc.s0[l], g.sc.s1[l]);
        zd[pos] = g.sc.d[l];
        zi[pos] = tid;
        if (RB) {
          zr[pos] = g.sc.rep[l];
          zc[pos] = f2(g.sc.s2[l], g.sc.s3[l]);
        }
      }
    }
    __syncthreads();

    if (PASS == 1) {
      for (int k8 = 0; k8 < cl8; k8 += 8) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float2 d0, d1;
          const float2 u = term(k8 + j, d0, d1);
          v[j] = u.x + u.y;
        }
        const float r = transpose_reduce8(v, lane);
        if ((lane & 3) == 0) wpart[warp][k8 + (lane >> 2)] = r;
      }
      __syncthreads();
      if (tid < cl) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += (double)wpart[w][tid];
        g.part1[e0 + cb + tid] = s;
      }
    } else {
      // selected candidates, two at a time: weights + the four centred state sums
      for (int k = 0; k < nsel; k += 2) {
        float v[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kk = k + h;
          if (kk < nsel) {
            float2 d0, d1;
            const float2 u = term(kk, d0, d1);
            pacc = __ffma2_rn(u, f2(zd[kk], zd[kk]), pacc);
            if (RB) {
              const float2 c = zc[kk];
              d0 = __fadd2_rn(P.X, f2(c.x, c.x));  // x - centre_x
              d1 = __fadd2_rn(P.Y, f2(c.y, c.y));  // y - centre_y
            }
            const float2 a0 = __fmul2_rn(u, d0), a1 = __fmul2_rn(u, P.VX);
            const float2 a2 = __fmul2_rn(u, d1), a3 = __fmul2_rn(u, P.VY);
            v[4 * h + 0] = a0.x + a0.y;
            v[4 * h + 1] = a1.x + a1.y;
            v[4 * h + 2] = a2.x + a2.y;
            v[4 * h + 3] = a3.x + a3.y;
          } else {
            v[4 * h + 0] = v[4 * h + 1] = v[4 * h + 2] = v[4 * h + 3] = 0.0f;
          }
        }
        const float r = transpose_reduce8(v, lane);
        const int q = lane >> 2;  // value index 0..7: candidate k + q / 4, quantity q % 4
        if ((lane & 3) == 0 && k + (q >> 2) < nsel) reinterpret_cast<float*>(&wq[warp][k + (q >> 2)])[q & 3] = r;
      }
      // the rest: weights only
#pragma unroll 4
      for (int k = nsel; k < cl; ++k) {
        float2 d0, d1;
        const float2 u = term(k, d0, d1);
        pacc = __ffma2_rn(u, f2(zd[k], zd[k]), pacc);
      }
      __syncthreads();
      if (tid < nsel) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const float4 a = wq[w][tid];
          s0 += (double)a.x;
          s1 += (double)a.y;
          s2 += (double)a.z;
          s3 += (double)a.w;
        }
        reinterpret_cast<float4*>(g.part2)[e0 + cb + zi[tid]] = make_float4((float)s0, (float)s1, (float)s2, (float)s3);
      }
    }
  }
  if (PASS == 2) {
    g.Ps[pa] = pacc.x;
    g.Ps[pb] = pacc.y;
  }
}

// one warp per label: fixed-order fp64 sum of its entries (lane-strided + xor tree)
template <int PASS>
__global__ void __launch_bounds__(256) k_gate_reduce(const int32_t* __restrict__ mstart, const int32_t* __restrict__ mlist,
                                                     int M, const double* __restrict__ part1,
                                                     const float4* __restrict__ part2, const int32_t* __restrict__ sel,
                                                     double* out, int slots_pad) {
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (l >= slots_pad) return;
  const bool live = l < M && (PASS == 1 || sel == nullptr || sel[l] != 0);
  const int j0 = live ? mstart[l] : 0, j1 = live ? mstart[l + 1] : 0;
  if (PASS == 1) {
    double s = 0.0;
    for (int j = j0 + lane; j < j1; j += 32) s += part1[mlist[j]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[l] = s;
  } else {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = j0 + lane; j < j1; j += 32) {
      const float4 a = part2[mlist[j]];
      s[0] += (double)a.x;
      s[1] += (double)a.y;
      s[2] += (double)a.z;
      s[3] += (double)a.w;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) out[(int64_t)q * slots_pad + l] = s[q];
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
cudaError_t gate_scan(int32_t* a, int64_t n, int32_t* tmp, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  const int nc = (int)((n + kScanChunk - 1) / kScanChunk);
  k_scan_sum<<<nc, 1024, 0, s>>>(a, n, tmp);
  k_scan_top<<<1, 1024, 0, s>>>(tmp, nc, a + n);
  k_scan_apply<<<nc, 1024, 0, s>>>(a, n, tmp);
  *launches += 3;
  return cudaGetLastError();
}

cudaError_t gate_sort_particles(int model, const float* const* A, const float* rb, int64_t rb_stride, int64_t n,
                                int64_t n_pad, float wscale, const GateGrid& grid, int32_t* keys, int32_t* hist,
                                int32_t* scan_tmp, const GateSorted& so, cudaStream_t s, int64_t* launches) {
  const bool rbm = model == kRangeBearing;
  if (n > 0) {
    const float* a0 = rbm ? rb : A[0];
    const float* a1 = rbm ? rb + 2 * rb_stride : A[2];
    k_gate_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(model, a0, a1, n, grid, keys);
    ++*launches;
    cudaError_t e = csort_pass(keys, nullptr, n, 0, kGateBins, hist, scan_tmp, nullptr, so.perm, s, launches);
    if (e != cudaSuccess) return e;
  }
  GatherSrc src{};
  for (int c = 0; c < 8; ++c) src.c[c] = rbm ? rb + c * rb_stride : nullptr;
  src.x = A[0];
  src.vx = A[1];
  src.y = A[2];
  src.vy = A[3];
  src.w = A[4];
  if (n_pad > 0) {
    k_gate_gather<<<(unsigned)((n_pad + 255) / 256), 256, 0, s>>>(model, src, n, n_pad, wscale, so);
    ++*launches;
  }
  return cudaGetLastError();
}

cudaError_t gate_zbin(const float* z, int M, const GateGrid& grid, int32_t* zkey, int32_t* zcell_start,
                      int32_t* zcell_items, cudaStream_t s) {
  k_gate_zbin<<<1, 1024, 0, s>>>(z, M, grid, zkey, zcell_start, zcell_items);
  return cudaGetLastError();
}

cudaError_t gate_tiles(int fill, int model, const GateSorted& so, int ntiles, float na0, float na1, const GateGrid& grid,
                       const int32_t* zcell_start, const int32_t* zcell_items, const float* z_lab, int32_t* tcount,
                       const int32_t* tstart, int32_t* cand, cudaStream_t s) {
  if (ntiles <= 0) return cudaSuccess;
  const bool rbm = model == kRangeBearing;
  const float* c0 = rbm ? so.c[0] : so.x;
  const float* c1 = rbm ? so.c[2] : so.y;
  const unsigned blocks = (unsigned)((ntiles + 7) / 8);
  if (fill)
    k_gate_tiles<true><<<blocks, 256, 0, s>>>(model, c0, c1, so.lw, ntiles, na0, na1, grid, zcell_start, zcell_items,
                                              z_lab, tcount, tstart, cand);
  else
    k_gate_tiles<false><<<blocks, 256, 0, s>>>(model, c0, c1, so.lw, ntiles, na0, na1, grid, zcell_start, zcell_items,
                                               z_lab, tcount, tstart, cand);
  return cudaGetLastError();
}

cudaError_t gate_sort_entries(const int32_t* cand, int64_t E, int M, int32_t* kbuf, int32_t* vbuf, int32_t* mlist,
                              int32_t* hist, int32_t* scan_tmp, int32_t* mstart, cudaStream_t s, int64_t* launches) {
  // mstart: per-label counts, exclusive scan (mstart[M] = E)
  k_zero_i32<<<(M + 256) / 256, 256, 0, s>>>(mstart, M + 1);
  ++*launches;
  if (E > 0) {
    k_gate_count_labels<<<(unsigned)((E + 255) / 256), 256, 0, s>>>(cand, E, mstart);
    ++*launches;
  }
  cudaError_t e = gate_scan(mstart, M, scan_tmp, s, launches);
  if (e != cudaSuccess || E <= 0) return e;
  // LSD passes of 12 bits over the label
  int bits = 1;
  while ((1 << bits) < M) ++bits;
  if (bits <= 12) {
    return csort_pass(cand, nullptr, E, 0, 1 << bits, hist, scan_tmp, nullptr, mlist, s, launches);
  }
  e = csort_pass(cand, nullptr, E, 0, kSortMaxBins, hist, scan_tmp, kbuf, vbuf, s, launches);
  if (e != cudaSuccess) return e;
  return csort_pass(kbuf, vbuf, E, 12, 1 << (bits - 12), hist, scan_tmp, nullptr, mlist, s, launches);
}

template <int MODEL>
static cudaError_t gpass_m(int pass, const GateArgs& g, cudaStream_t s) {
  if (pass == 1)
    k_gpass<MODEL, 1><<<g.ntiles, 256, 0, s>>>(g);
  else
    k_gpass<MODEL, 2><<<g.ntiles, 256, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_gpass(int pass, const GateArgs& g, cudaStream_t s) {
  if (g.ntiles <= 0) return cudaSuccess;
  if (g.model == kPosIso) return gpass_m<kPosIso>(pass, g, s);
  if (g.model == kPosAniso) return gpass_m<kPosAniso>(pass, g, s);
  return gpass_m<kRangeBearing>(pass, g, s);
}

cudaError_t launch_gate_reduce(int pass, const int32_t* mstart, const int32_t* mlist, int M, const double* part1,
                               const float* part2, const int32_t* sel, double* out, int slots_pad, cudaStream_t s) {
  if (slots_pad <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((slots_pad + 7) / 8);
  if (pass == 1)
    k_gate_reduce<1><<<blocks, 256, 0, s>>>(mstart, mlist, M, part1, nullptr, nullptr, out, slots_pad);
  else
    k_gate_reduce<2><<<blocks, 256, 0, s>>>(mstart, mlist, M, nullptr, reinterpret_cast<const float4*>(part2), sel,
                                            out, slots_pad);
  return cudaGetLastError();
}

}  // namespace phd
