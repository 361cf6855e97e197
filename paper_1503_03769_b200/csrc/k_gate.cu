// Gated particle x measurement update (SURVEY.md §8(f) NEXT-2 "measurement
// gating by spatial binning"; DESIGN.md §5 "Gated update").
//
// The dense passes (k_update.cu) evaluate every (particle, measurement) pair,
// although at these configs almost all terms p_D g(z|x) w underflow: with
// sigma = 10 m a term is below 2^-126 (and flushed to exactly 0 by
// ex2.approx.ftz) once |x - z| exceeds ~120 m.  This path computes the same
// non-zero terms and skips only pairs whose exponent is provably below -130:
//
//   1. k_ms_hist<KeyCell> + gate_scan + k_psort_scatter: each particle gets the
//      Morton key of its 64 x 64 cell in measurement space ((x, y), or (r, theta)
//      for the range-bearing sensor); a stable counting sort writes every particle
//      as one whole record (state + log2(p_D c w)) to its sorted slot and inv[i]
//      (the filter's own particle order, which defines resampling, is untouched).
//      NaN particles are counted here (the dense C would be NaN).
//   2. gate_zbin: measurements binned into the same cells (the same counting sort).
//   3. k_gate_count / k_gate_fill (tile_enum): per tile of gate_tp sorted particles,
//      the bounding box and max log2(p_D c w); a measurement is a candidate of the
//      tile iff
//         e_max = -alpha0 dx^2 - alpha1 dy^2 + max_i log2(p_D c w_i) >= -130
//      with (dx, dy) its distance to the box (wrapped in bearing).  Every term
//      of a non-candidate pair has e <= e_max < -130 (fp32 rounding of the
//      kernels' exponent is ~1e-4 here), so it is exactly 0 in the dense path.
//   4. k_gpass<1>: CTA per tile, four particles per thread (2 x f32x2), candidates
//      broadcast from shared memory; the same per-pair arithmetic as the dense
//      pass (pair_math.cuh), so every term is bitwise the dense pass 2's.  Tile
//      sums per candidate: warp tree (transposed butterfly), fp64 across warps.
//   5. the entries (tile, candidate) are stably sorted by label and k_gate_reduce
//      sums each label's tile partials in entry order (fp64, warp tree):
//      deterministic, no atomics on floating point.
//   6. k_gpass<2>: weights (sum_z u d_z per particle, complete inside the CTA)
//      and the centred STPHD state sums for candidates in the index set I.
#include "phd_internal.h"

#include <type_traits>
#include "pair_math.cuh"

#include <algorithm>

namespace phd {

namespace {

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

// Lanes of the warp holding the same digit d, among the lanes with ok set: one
// ballot per key bit (MATCH.ANY has a much lower throughput; ballots over only
// the bits that vary in the warp, found with REDUX, measured slower still).
template <int NBITS>
__device__ __forceinline__ unsigned match_digit(int d, bool ok) {
  unsigned m = __ballot_sync(0xffffffffu, ok);
#pragma unroll
  for (int b = 0; b < NBITS; ++b) {
    const bool bit = (d >> b) & 1;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}
__device__ __forceinline__ unsigned match_digit_rt(int d, bool ok, int nbits) {
  unsigned m = __ballot_sync(0xffffffffu, ok);
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (d >> b) & 1;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

// The same peer mask as match_digit, faster for rows of one digit (cell keys of
// particles in ancestor order are clustered): the first lane's digit is peeled
// off by a broadcast and one ballot, the remaining lanes (rows with more distinct
// digits) go through the per-bit ballots.  Warp-uniform control flow.
template <int NBITS>
__device__ __forceinline__ unsigned match_digit_peel(int d, bool ok) {
  constexpr int kPeel = 1;  // measured: 1 / 2 / 3 peels 0.295 / 0.301 / 0.311 ms at cfg 5 (0.322 none)
  const int lane = threadIdx.x & 31;
  unsigned rem = __ballot_sync(0xffffffffu, ok);
  unsigned peers = 0u;
#pragma unroll
  for (int it = 0; it < kPeel; ++it) {
    if (rem == 0u) break;  // uniform
    const int dl = __shfl_sync(0xffffffffu, d, __ffs(rem) - 1);
    const bool mine = ((rem >> lane) & 1u) && d == dl;
    const unsigned m = __ballot_sync(0xffffffffu, mine);
    if (mine) peers = m;
    rem &= ~m;
  }
  if (rem != 0u) {  // uniform
    const bool in = (rem >> lane) & 1u;
    const unsigned m = match_digit<NBITS>(d, in);
    if (in) peers = m;
  }
  return peers;
}

// float <-> int with the same order (for integer atomicMax on floats)
__device__ __forceinline__ int f2ord(float f) {
  const int b = __float_as_int(f);
  return b >= 0 ? b : b ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord2f(int o) { return __int_as_float(o >= 0 ? o : o ^ 0x7FFFFFFF); }

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
  pdl_wait();
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
  pdl_wait();
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
  pdl_wait();
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
// Stable counting sort pass (deterministic; no floating point involved).
// hist is bin-major, hist[bin * nblk + blk], so its exclusive scan gives the
// first output position of every (bin, block).  A CTA of kMsWarps warps owns
// per_blk consecutive items, warp w the w-th slice; per-warp 16-bit
// sub-histograms in shared memory give each warp its offset inside the
// block's run of a bin, and the warp then walks its slice in order, ranking
// equal bins with match_any.  Keys come from a functor: the digit of an int
// array, or a particle's measurement-space cell.
constexpr int kMsWarps = 8;
constexpr int kMsRows = 8;  // rows of 32 items whose loads are issued together

struct KeyArr {
  const int32_t* k;
  int shift, mask;
  __device__ __forceinline__ int digit(int32_t raw) const { return (raw >> shift) & mask; }
  __device__ __forceinline__ int32_t raw(int64_t i) const { return __ldg(k + i); }
};
struct KeyCell {
  const float* a0;
  const float* a1;
  GateGrid g;
  __device__ __forceinline__ int digit(int32_t raw) const { return raw; }
  __device__ __forceinline__ int32_t raw(int64_t i) const { return cell_key(__ldg(a0 + i), __ldg(a1 + i), g); }
};

struct KeyZ {  // measurement l = (z[2l], z[2l+1]) -> its cell
  const float* z;
  GateGrid g;
  __device__ __forceinline__ int digit(int32_t raw) const { return raw; }
  __device__ __forceinline__ int32_t raw(int64_t i) const { return cell_key(__ldg(z + 2 * i), __ldg(z + 2 * i + 1), g); }
};

template <class KF>
__global__ void __launch_bounds__(1024) k_ms_hist(KF kf, int64_t n, int64_t per_blk, int nbins, int nblk, int32_t* hist,
                                                 int32_t* keys_out = nullptr) {
  pdl_wait();
  __shared__ int h[kSortMaxBins];
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * per_blk;
  const int64_t i1 = min(n, i0 + per_blk);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const int32_t raw = kf.raw(i);
    if (keys_out) keys_out[i] = raw;  // the particle sort keeps its cell keys for the ranking pass
    atomicAdd(&h[kf.digit(raw)], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) hist[(int64_t)b * nblk + blockIdx.x] = h[b];
}

// smem: wh[kMsWarps][nbins / 2] packed 16-bit counters, base[nbins]
template <class KF>
__global__ void __launch_bounds__(256) k_ms_scatter(KF kf, int64_t n, int64_t per_blk, int nbins, int nblk,
                                                    const int32_t* __restrict__ hs, const int32_t* __restrict__ vals,
                                                    int32_t* out_keys, int32_t* out_vals) {
  pdl_wait();
  extern __shared__ uint32_t sm[];
  const int nw = nbins >> 1;  // nbins even
  uint32_t* wh = sm;
  int* base = reinterpret_cast<int*>(sm + kMsWarps * nw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < kMsWarps * nw; j += blockDim.x) wh[j] = 0u;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * per_blk;
  const int64_t i1 = min(n, i0 + per_blk);
  const int64_t pw = per_blk / kMsWarps;
  const int64_t w0 = min(i1, i0 + warp * pw), w1 = min(i1, w0 + pw);
  uint32_t* my = wh + warp * nw;
  // 1. per-warp sub-histograms
  for (int64_t b0 = w0; b0 < w1; b0 += 32 * kMsRows) {
    int32_t raw[kMsRows];
#pragma unroll
    for (int r = 0; r < kMsRows; ++r) raw[r] = kf.raw(min(b0 + r * 32 + lane, w1 - 1));
#pragma unroll
    for (int r = 0; r < kMsRows; ++r)
      if (b0 + r * 32 + lane < w1) {
        const int d = kf.digit(raw[r]);
        atomicAdd(&my[d >> 1], 1u << (16 * (d & 1)));
      }
  }
  __syncthreads();
  // 2. exclusive prefix over the warps of every bin; block offsets of the bins
  for (int j = tid; j < nw; j += blockDim.x) {
    uint32_t run = 0u;
#pragma unroll
    for (int w = 0; w < kMsWarps; ++w) {
      const uint32_t c = wh[w * nw + j];
      wh[w * nw + j] = run;
      run += c;  // the two 16-bit halves never carry: per-block counts < 65536
    }
    base[2 * j] = hs[(int64_t)(2 * j) * nblk + blockIdx.x];
    base[2 * j + 1] = hs[(int64_t)(2 * j + 1) * nblk + blockIdx.x];
  }
  __syncthreads();
  // 3. stable ranking of the warp's slice
  const unsigned lt = (1u << lane) - 1u;
  int nbits = 1;
  while ((1 << nbits) < nbins) ++nbits;
  for (int64_t b0 = w0; b0 < w1; b0 += 32 * kMsRows) {
    int32_t raw[kMsRows];
    int32_t val[kMsRows];
#pragma unroll
    for (int r = 0; r < kMsRows; ++r) {
      const int64_t i = min(b0 + r * 32 + lane, w1 - 1);
      raw[r] = kf.raw(i);
      val[r] = vals ? __ldg(vals + i) : (int32_t)(b0 + r * 32 + lane);
    }
#pragma unroll
    for (int r = 0; r < kMsRows; ++r) {
      const bool ok = b0 + r * 32 + lane < w1;
      const int d = ok ? kf.digit(raw[r]) : 0;
      const unsigned peers = match_digit_rt(d, ok, nbits);
      int pos = 0;
      if (ok) pos = base[d] + (int)((my[d >> 1] >> (16 * (d & 1))) & 0xFFFFu) + __popc(peers & lt);
      __syncwarp();
      if (ok) {
        if (lane == __ffs(peers) - 1) atomicAdd(&my[d >> 1], (uint32_t)__popc(peers) << (16 * (d & 1)));
        PHD_DCHECK(pos >= 0 && pos < n);
        if (out_keys) out_keys[pos] = raw[r];
        out_vals[pos] = val[r];
      }
      __syncwarp();
    }
  }
}

template <class KF>
cudaError_t ms_pass(KF kf, const int32_t* vals, int64_t n, int64_t per_blk, int nbins, int32_t* hist,
                    int32_t* scan_tmp, int32_t* out_keys, int32_t* out_vals, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  nbins = std::max(2, nbins);
  const int nblk = (int)((n + per_blk - 1) / per_blk);
  const size_t smem = sizeof(uint32_t) * (size_t)kMsWarps * (nbins / 2) + sizeof(int) * (size_t)nbins;
  ensure_max_smem(k_ms_scatter<KF>, sizeof(uint32_t) * kMsWarps * (kSortMaxBins / 2) + sizeof(int) * kSortMaxBins);
  pdl_launch(k_ms_hist<KF>, nblk, 256, 0, s, kf, n, per_blk, nbins, nblk, hist, nullptr);
  ++*launches;
  cudaError_t e = gate_scan(hist, (int64_t)nbins * nblk, scan_tmp, s, launches);
  if (e != cudaSuccess) return e;
  pdl_launch(k_ms_scatter<KF>, nblk, 256, smem, s, kf, n, per_blk, nbins, nblk, hist, vals, out_keys, out_vals);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t csort_pass(const int32_t* keys, const int32_t* vals, int64_t n, int shift, int nbins, int32_t* hist,
                       int32_t* scan_tmp, int32_t* out_keys, int32_t* out_vals, cudaStream_t s, int64_t* launches) {
  KeyArr kf{keys, shift, std::max(2, nbins) - 1};
  return ms_pass(kf, vals, n, sort_block(n), nbins, hist, scan_tmp, out_keys, out_vals, s, launches);
}

// ---------------------------------------------------------------------------
// Particle sort.  k_ms_hist<KeyCell> counts the cells; k_psort_scatter ranks
// each particle stably (as k_ms_scatter) and writes it, read coalesced in the
// filter's order, as one whole record to its sorted slot: 32 bytes (position)
// or 64 bytes (range-bearing), i.e. full sectors, never partial-sector writes;
// inv[i] = sorted slot is written coalesced.
struct GatherSrc {
  const float* c[8];
  const float *x, *y, *vx, *vy, *w;
};

// padding records [n, n_pad): zero state, lw = -inf
__global__ void k_psort_pad(int64_t n, int64_t n_pad, GateSorted so) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) *so.lw_max = f2ord(-INFINITY);  // reset before the scatter's max
  const int64_t p = n + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pad) return;
  float4* r = so.rec + p * so.n4;
  for (int k = 0; k < so.n4 - 1; ++k) r[k] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  r[so.n4 - 1] = make_float4(-INFINITY, 0.0f, 0.0f, 0.0f);
}

// one 256-bit store (STG.E.ENL2.256, sm_100) of two float4: a whole 32-byte sector
__device__ __forceinline__ void st_v8(float4* dst, float4 a, float4 b) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(a.x), "f"(a.y), "f"(a.z),
               "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}

// ps_warps(MODEL) warps per CTA, their 16-bit sub-histograms (8 KB each) + 16 KB of bases in
// shared memory.  Position: 16 (one CTA per SM, 144 KB; cfg 5 ranking 345 -> 325 us, gated
// step 2.03 -> 2.00 ms); range-bearing keeps 8 (cfg 4 +1 % with 16); 12 and 24 were slower.
#ifndef PHD_PSORT_WARPS
#define PHD_PSORT_WARPS 16
#endif
__host__ __device__ constexpr int ps_warps(int model) { return model == kRangeBearing ? 8 : PHD_PSORT_WARPS; }
template <int MODEL, int kPsWarps = ps_warps(MODEL)>
__global__ void __launch_bounds__(kPsWarps * 32) k_psort_scatter(GatherSrc src, const int32_t* __restrict__ keys, int64_t n,
                                                       int64_t per_blk, int nblk, const int32_t* __restrict__ hs,
                                                       float wscale, GateSorted so, double* blk_wp) {
  pdl_wait();
  constexpr bool RB = MODEL == kRangeBearing;
  constexpr int N4 = RB ? 4 : 2;
  constexpr int ROWS = RB ? 2 : 4;
  constexpr int nw = kGateBins / 2;
  extern __shared__ uint32_t sm[];
  uint32_t* wh = sm;
  int* base = reinterpret_cast<int*>(sm + kPsWarps * nw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < kPsWarps * nw; j += blockDim.x) wh[j] = 0u;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * per_blk;
  const int64_t i1 = min(n, i0 + per_blk);
  const int64_t pw = per_blk / kPsWarps;  // the last warp also takes the remainder
  const int64_t w0 = min(i1, i0 + warp * pw), w1 = warp == kPsWarps - 1 ? i1 : min(i1, w0 + pw);
  uint32_t* my = wh + warp * nw;
  // 1. per-warp sub-histograms
  for (int64_t b0 = w0; b0 < w1; b0 += 32 * kMsRows) {
    int32_t key[kMsRows];
#pragma unroll
    for (int r = 0; r < kMsRows; ++r) key[r] = __ldg(keys + min(b0 + r * 32 + lane, w1 - 1));
#pragma unroll
    for (int r = 0; r < kMsRows; ++r)
      if (b0 + r * 32 + lane < w1) atomicAdd(&my[key[r] >> 1], 1u << (16 * (key[r] & 1)));
  }
  __syncthreads();
  // 2. exclusive prefix over the warps of every cell; block offsets
  for (int j = tid; j < nw; j += blockDim.x) {
    uint32_t run = 0u;
#pragma unroll
    for (int w = 0; w < kPsWarps; ++w) {
      const uint32_t c = wh[w * nw + j];
      wh[w * nw + j] = run;
      run += c;
    }
    base[2 * j] = hs[(int64_t)(2 * j) * nblk + blockIdx.x];
    base[2 * j + 1] = hs[(int64_t)(2 * j + 1) * nblk + blockIdx.x];
  }
  __syncthreads();
  // 3. rank and write the records (and the max of lw, for the tile kernels' fast path)
  const unsigned lt = (1u << lane) - 1u;
  float lwm = -INFINITY;
  double wsum = 0.0;  // predicted w of this lane's items (W_pred block sum below)
  bool nanp = false;  // clamped duplicates of the last item repeat a real item: no false flag
  for (int64_t b0 = w0; b0 < w1; b0 += 32 * ROWS) {
    float4 q[ROWS][N4];
    float wr[ROWS];
    int kr[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int64_t i = min(b0 + r * 32 + lane, w1 - 1);
      kr[r] = __ldg(keys + i);
      if (RB) {
        q[r][0] = make_float4(__ldg(src.c[0] + i), __ldg(src.c[1] + i), __ldg(src.c[2] + i), __ldg(src.c[3] + i));
        q[r][1] = make_float4(__ldg(src.c[4] + i), __ldg(src.c[5] + i), __ldg(src.c[6] + i), __ldg(src.c[7] + i));
      }
      q[r][N4 - 2] = make_float4(__ldg(src.x + i), __ldg(src.y + i), __ldg(src.vx + i), __ldg(src.vy + i));
      wr[r] = __ldg(src.w + i);
      q[r][N4 - 1] = make_float4(log2f(wr[r] * wscale), 0.0f, 0.0f, 0.0f);  // the dense records' expression (k_records)
      lwm = fmaxf(lwm, q[r][N4 - 1].x);  // clamped duplicates of the last item do not change the max
      // a NaN particle makes every dense term NaN (C, D non-finite -> PHD_EMODEL); the
      // gated path might not evaluate it, so it is flagged here (one atomic per warp at the end)
      const float4 st = q[r][N4 - 2];
      nanp |= isnan(st.x) | isnan(st.y) | isnan(q[r][N4 - 1].x);
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int64_t i = b0 + r * 32 + lane;
      const bool ok = i < w1;
      if (ok) wsum += (double)wr[r];  // this lane's items in order
      const int d = ok ? kr[r] : 0;
      // the one-digit fast path pays for clustered cells (position sensor: 0.322 -> 0.295 ms at
      // cfg 5); range-bearing rows in (r, theta) cells are less uniform (cfg 4: +2 %)
      const unsigned peers = RB ? match_digit<12>(d, ok) : match_digit_peel<12>(d, ok);
      int pos = 0;
      if (ok) pos = base[d] + (int)((my[d >> 1] >> (16 * (d & 1))) & 0xFFFFu) + __popc(peers & lt);
      __syncwarp();
      if (ok) {
        if (lane == __ffs(peers) - 1) atomicAdd(&my[d >> 1], (uint32_t)__popc(peers) << (16 * (d & 1)));
        PHD_DCHECK(pos >= 0 && pos < n && d >= 0 && d < kGateBins);
        float4* dst = so.rec + (int64_t)pos * N4;
#pragma unroll
        for (int k = 0; k < N4; k += 2) st_v8(dst + k, q[r][k], q[r][k + 1]);
        so.inv[i] = pos;
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lwm = fmaxf(lwm, __shfl_xor_sync(0xffffffffu, lwm, o));
  if (lane == 0 && w0 < w1) atomicMax(so.lw_max, f2ord(lwm));
  if (__any_sync(0xffffffffu, nanp) && lane == 0) atomicAdd(so.bad, 1);
  if (blk_wp != nullptr) {  // fixed order: lanes' sums by xor tree, the warps in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    __shared__ double wpart[kPsWarps];
    if (lane == 0) wpart[warp] = wsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < kPsWarps; ++k) t += wpart[k];
      blk_wp[blockIdx.x] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// per tile (one warp): bounding box in measurement space, max log2(p_D c w),
// then the candidates: cells of the window in rounds of 32 (lane = cell),
// measurements of a cell in item order, written in (round, lane, item) order
// -- deterministic.  The count pass also keeps the first kbuf (gate_kbuf) candidates
// of every tile, so the fill pass copies them instead of enumerating again.

// the tile kernels' view of the sorted records: c0, c1 (measurement-space
// coordinates) and lw of record p at [p * stride]
struct RecView {
  const float* c0;
  const float* c1;
  const float* lw;
  int stride;
  int64_t n;             // particles (records [n, n_pad) are padding)
  const int* lw_max;     // ordered-int encoding of max lw over all particles (k_psort_scatter)
  int tp;                // particles per tile (gate_tp)
};


// window enumeration switches to a scan of all M binned measurements when the window has more
// than M / kGateDirectRatio cells (0 = never, A/B builds)
#ifndef PHD_GATE_DIRECT
#define PHD_GATE_DIRECT 1
#endif
#ifndef PHD_BOX_UNROLL
#define PHD_BOX_UNROLL 8
#endif
constexpr int kBoxUnroll = PHD_BOX_UNROLL;
#ifndef PHD_GATE_DIRECT_RATIO
#define PHD_GATE_DIRECT_RATIO 8
#endif
constexpr int kGateDirectRatio = PHD_GATE_DIRECT_RATIO;

__device__ __forceinline__ int tile_enum(int t, const RecView& rv, float na0, float na1, const GateGrid& g,
                                         const int32_t* __restrict__ zcell_start, const int32_t* __restrict__ zcell_items,
                                         const float2* __restrict__ zcell_z, int32_t* dst, int cap) {
  const int lane = threadIdx.x & 31;
  const int tp = rv.tp;
  const int64_t p0 = (int64_t)t * tp;
  float b0 = INFINITY, b1 = -INFINITY, e0 = INFINITY, e1 = -INFINITY, lm = -INFINITY;
  // Fast path: a full tile whose first and last particles share an interior cell holds
  // only particles of that cell (the tiles are in cell-key order), so the cell's box
  // (a little widened against the fp32 rounding of the cell index) and the global
  // max of log2(p_D c w) bound the tile conservatively: never fewer candidates.
  bool fast = false;
  if (p0 + tp <= rv.n) {
    const int64_t oa = p0 * rv.stride, ob = (p0 + tp - 1) * rv.stride;
    const int ax = cell_raw(__ldg(rv.c0 + oa), g.lo0, g.inv_h0), ay = cell_raw(__ldg(rv.c1 + oa), g.lo1, g.inv_h1);
    const int bx = cell_raw(__ldg(rv.c0 + ob), g.lo0, g.inv_h0), by = cell_raw(__ldg(rv.c1 + ob), g.lo1, g.inv_h1);
    if (ax == bx && ay == by && ax > 0 && ax < kGateG - 1 && ay > 0 && ay < kGateG - 1) {
      fast = true;
      const float w0 = 1.0f / g.inv_h0, w1 = 1.0f / g.inv_h1;
      b0 = g.lo0 + ((float)ax - 0.01f) * w0;
      b1 = g.lo0 + ((float)ax + 1.01f) * w0;
      e0 = g.lo1 + ((float)ay - 0.01f) * w1;
      e1 = g.lo1 + ((float)ay + 1.01f) * w1;
      lm = ord2f(__ldg(rv.lw_max));
    }
  }
#pragma unroll kBoxUnroll
  for (int j = lane; j < (fast ? 0 : tp); j += 32) {  // (the box loads of several rows in flight)
    const int64_t o = (p0 + j) * rv.stride;
    const float l = __ldg(rv.lw + o);
    const float v0 = __ldg(rv.c0 + o), v1 = __ldg(rv.c1 + o);
    // zero-weight particles, padding and non-finite coordinates (whose dense terms
    // are 0, or NaN and flagged by the sort) do not widen the box
    if (l > -INFINITY && isfinite(v0) && isfinite(v1)) {
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
  const float budget = lm - g.floor;  // e_max >= floor  <=>  alpha0 dx^2 + alpha1 dy^2 <= budget
  int total = 0;
  if (!(budget > 0.0f && isfinite(b0) && isfinite(e0) && isfinite(b1) && isfinite(e1))) return 0;
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
  // lane = cell of the round; the cell's item range of the next round is loaded
  // ahead, and the first kStash items' labels with their coordinates, so a round
  // costs about one dependent load (long windows: tiles spanning a Morton jump).
  // (Four rounds per iteration with all loads in flight measured slower: 72
  // registers, fewer resident warps.)
  auto cell_range = [&](int ci, int& j0, int& j1) {
    j0 = j1 = 0;
    if (ci < nc) {
      const int cx = x0 + ci % nx;
      int cy = y0 + ci / nx;
      if (g.wrap1) cy = wrapc(cy);
      const int key = morton(cx, cy);
      PHD_DCHECK(key >= 0 && key < kGateBins);
      j0 = zcell_start[key];
      j1 = zcell_start[key + 1];
    }
  };
  auto passes = [&](float2 zz) {
    const float dx = dist_iv(zz.x, b0, b1);
    const float dy = g.wrap1 ? dist_arc(zz.y, e0, e1) : dist_iv(zz.y, e0, e1);
    return fmaf(na0, dx * dx, fmaf(na1, dy * dy, lm)) >= g.floor;
  };
  // long windows (tiles spanning a Morton jump cover a large part of the grid): scan every
  // binned measurement in cell order instead, four rounds of 32 with their loads in flight
  // (no dependent cell-range loads); the same test, so the same candidate set
  const int Mz = __ldg(zcell_start + kGateBins);
  if (PHD_GATE_DIRECT && nc * kGateDirectRatio > Mz) {
    for (int r0 = 0; r0 < Mz; r0 += 128) {
      float2 zz[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = r0 + 32 * u + lane;
        zz[u] = j < Mz ? zcell_z[j] : make_float2(INFINITY, INFINITY);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = r0 + 32 * u + lane;
        const bool ok = j < Mz && passes(zz[u]);
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int w = total + __popc(bal & ((1u << lane) - 1u));
        if (ok && dst != nullptr && w < cap) dst[w] = zcell_items[j];
        total += __popc(bal);
      }
    }
    return total;
  }
  constexpr int kStash = 4;
  int j0n, j1n;
  cell_range(lane, j0n, j1n);
  for (int r = 0; r < nc; r += 32) {
    const int j0 = j0n, j1 = j1n;
    if (r + 32 < nc) cell_range(r + 32 + lane, j0n, j1n);
    int cnt = 0;
    unsigned pbits = 0u;
    int it[kStash];
#pragma unroll
    for (int q = 0; q < kStash; ++q) {
      it[q] = -1;
      if (j0 + q < j1) {
        const float2 zz = zcell_z[j0 + q];
        if (dst != nullptr) it[q] = zcell_items[j0 + q];
        if (passes(zz)) {
          pbits |= 1u << q;
          ++cnt;
        }
      }
    }
    for (int j = j0 + kStash; j < j1; ++j) cnt += passes(zcell_z[j]);  // crowded cells
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (cnt > 0 && dst != nullptr) {
      int w = total + incl - cnt;
#pragma unroll
      for (int q = 0; q < kStash; ++q)
        if (((pbits >> q) & 1u) && w < cap) dst[w++] = it[q];
      for (int j = j0 + kStash; j < j1 && w < cap; ++j)
        if (passes(zcell_z[j])) {
          PHD_DCHECK(w < cap);
          dst[w++] = zcell_items[j];
        }
    }
    total += __shfl_sync(0xffffffffu, incl, 31);
  }
  return total;
}

// count pass: tcount[t] and the first kbuf candidates in cbuf[t][.]
__global__ void __launch_bounds__(256) k_gate_count(const RecView rv, int ntiles, float na0, float na1,
                                                    GateGrid g, const int32_t* __restrict__ zcell_start,
                                                    const int32_t* __restrict__ zcell_items,
                                                    const float2* __restrict__ zcell_z, int32_t* tcount, int32_t* cbuf) {
  pdl_wait();
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  const int total = tile_enum(t, rv, na0, na1, g, zcell_start, zcell_items, zcell_z,
                              cbuf + (int64_t)t * g.kbuf, g.kbuf);
  if ((threadIdx.x & 31) == 0) tcount[t] = total;
}

// fill pass: copy the buffered candidates to cand[tstart[t]..]; tiles with more
// than kbuf candidates enumerate again
__global__ void __launch_bounds__(256) k_gate_fill(const RecView rv, int ntiles, float na0, float na1,
                                                   GateGrid g, const int32_t* __restrict__ zcell_start,
                                                   const int32_t* __restrict__ zcell_items,
                                                   const float2* __restrict__ zcell_z, const int32_t* __restrict__ tstart,
                                                   const int32_t* __restrict__ cbuf, int32_t* cand, int64_t ecap) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  const int e0 = tstart[t], K = tstart[t + 1] - e0;
  // launched before the host has checked the total against the workspace: entries past
  // ecap are not written (the update then runs dense and ignores cand)
  const int64_t room = ecap - (int64_t)e0;
  const int Kw = room <= 0 ? 0 : (room < (int64_t)K ? (int)room : K);
  if (K <= g.kbuf) {
    for (int j = lane; j < Kw; j += 32) cand[e0 + j] = cbuf[(int64_t)t * g.kbuf + j];
  } else if (Kw > 0) {
    tile_enum(t, rv, na0, na1, g, zcell_start, zcell_items, zcell_z, cand + e0, Kw);
  }
}

// per-label entry counts (integer atomics: order-independent)
__global__ void k_gate_count_labels(const int32_t* __restrict__ cand, int64_t E, int32_t* cnt) {
  pdl_wait();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) atomicAdd(&cnt[cand[e]], 1);
}

__global__ void k_mstart_from_hist(const int32_t* __restrict__ hs, int nblk, int M, int32_t E, int32_t* mstart) {
  pdl_wait();
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < M) mstart[l] = hs[(int64_t)l * nblk];
  if (l == M) mstart[M] = E;
}

__global__ void k_zero_i32(int32_t* a, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = 0;
}

// ---------------------------------------------------------------------------
// The gated passes.  Tile t = sorted particles [t*TP, t*TP + TP); a CTA of
// TP / (2 NPAIR) threads, thread tid holds 2 NPAIR particles as NPAIR f32x2 pairs
// h = 0, 1: (tid + 256 h, tid + 128 + 256 h).  Per candidate the thread sums
// its four terms before the cross-lane reduction.

template <int MODEL>
struct GPair {
  float2 X, Y, LW;                        // Cartesian x, y; log2(p_D c w)
  float2 R_hi, R_lo, T_hi[3], T_lo[3];    // range-bearing representation
  float2 VX, VY;
};

#ifndef PHD_GPASS2_MINB
#define PHD_GPASS2_MINB 8
#endif
// (resident CTAs per SM scale with 512 / TP: the same threads per SM for both tile sizes)
template <int MODEL, int PASS, int NPAIR, int TP = gate_tp(MODEL)>
__global__ void __launch_bounds__(TP / (2 * NPAIR),
                                  ((MODEL == kRangeBearing && PASS == 2) ? 5 : (PASS == 2 ? PHD_GPASS2_MINB : 8)) * 512 / TP)
    k_gpass(const GateArgs g) {
  pdl_wait();
  constexpr bool RB = MODEL == kRangeBearing;
  constexpr int THREADS = TP / (2 * NPAIR);  // particle pairs (tid + 2 THREADS h, + THREADS) per thread
  constexpr int WARPS = THREADS / 32;
  // + 2: pass 2 pads an odd selected count with one sentinel candidate
  __shared__ float2 zn[kGateChunk + 2];      // (-z0, -z1)
  __shared__ float zd[kGateChunk + 2];       // 1 / (kappa + C)          (pass 2)
  __shared__ int zr[kGateChunk + 2];         // bearing representation   (range-bearing)
  __shared__ float2 zc[kGateChunk + 2];      // -(Cartesian centre)      (range-bearing, pass 2)
  __shared__ int zi[kGateChunk + 2];         // chunk-local entry index  (pass 2: selected first)
  __shared__ unsigned gmask[kGateChunk / 32];  // pass 2: "in I" ballot per 32 candidates
  __shared__ float wpart[PASS == 1 ? WARPS : 1][PASS == 1 ? kGateChunk : 1];   // pass 1: per-warp sums
  __shared__ float4 wq[PASS == 2 ? WARPS : 1][PASS == 2 ? kGateChunk + 2 : 1];     // pass 2: per-warp state sums

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = blockIdx.x;
  const float2 na0 = f2(g.na0, g.na0), na1 = f2(g.na1, g.na1);
  GPair<MODEL> P[NPAIR];
  constexpr int N4 = RB ? 4 : 2;
#pragma unroll
  for (int h = 0; h < NPAIR; ++h) {
    const int64_t pa = (int64_t)t * TP + 2 * THREADS * h + tid, pb = pa + THREADS;
    const float4* ra = g.so.rec + pa * N4;
    const float4* rbp = g.so.rec + pb * N4;
    P[h].LW = f2(__ldg(ra + N4 - 1).x, __ldg(rbp + N4 - 1).x);
    if (RB) {
      const float4 a0 = __ldg(ra), b0 = __ldg(rbp), a1 = __ldg(ra + 1), b1 = __ldg(rbp + 1);
      P[h].R_hi = f2(a0.x, b0.x);
      P[h].R_lo = f2(a0.y, b0.y);
      P[h].T_hi[0] = f2(a0.z, b0.z);
      P[h].T_lo[0] = f2(a0.w, b0.w);
      P[h].T_hi[1] = f2(a1.x, b1.x);
      P[h].T_lo[1] = f2(a1.y, b1.y);
      P[h].T_hi[2] = f2(a1.z, b1.z);
      P[h].T_lo[2] = f2(a1.w, b1.w);
    }
    if (!RB || PASS == 2) {
      const float4 a = __ldg(ra + N4 - 2), b = __ldg(rbp + N4 - 2);
      P[h].X = f2(a.x, b.x);
      P[h].Y = f2(a.y, b.y);
      P[h].VX = f2(a.z, b.z);
      P[h].VY = f2(a.w, b.w);
    }
  }
  const int e0 = g.tstart[t];
  const int K = g.tstart[t + 1] - e0;
  float2 pacc[NPAIR];
#pragma unroll
  for (int h = 0; h < NPAIR; ++h) pacc[h] = f2(0.0f, 0.0f);

  // u = p_D g(z_k | x) w for pair h (bitwise the dense kernel's term)
  auto term = [&](int k, int h, float2& d0, float2& d1) -> float2 {
    const float2 nz = zn[k];
    if (RB) {
      const int rep = zr[k];
      const float2 th = rep == 0 ? P[h].T_hi[0] : (rep == 1 ? P[h].T_hi[1] : P[h].T_hi[2]);
      const float2 tl = rep == 0 ? P[h].T_lo[0] : (rep == 1 ? P[h].T_lo[1] : P[h].T_lo[2]);
      d0 = __fadd2_rn(__fadd2_rn(P[h].R_hi, f2(nz.x, nz.x)), P[h].R_lo);  // (r_hi - z_r) + r_lo
      d1 = __fadd2_rn(__fadd2_rn(th, f2(nz.y, nz.y)), tl);                // (th_hi - z_th) + th_lo
    } else {
      d0 = __fadd2_rn(P[h].X, f2(nz.x, nz.x));  // x - z_x
      d1 = __fadd2_rn(P[h].Y, f2(nz.y, nz.y));  // y - z_y
    }
    return ex2v(expo<MODEL>(d0, d1, na0, na1, P[h].LW));
  };
  // pass 2 with 1/D folded into the exponent (zd = log2(d)/na0): u d = p_D g w / (kappa + C),
  // bitwise the dense pass 2's term
  auto term_fold = [&](int k, int h, float2& d0, float2& d1) -> float2 {
    const float2 nz = zn[k];
    if (RB) {
      const int rep = zr[k];
      const float2 th = rep == 0 ? P[h].T_hi[0] : (rep == 1 ? P[h].T_hi[1] : P[h].T_hi[2]);
      const float2 tl = rep == 0 ? P[h].T_lo[0] : (rep == 1 ? P[h].T_lo[1] : P[h].T_lo[2]);
      d0 = __fadd2_rn(__fadd2_rn(P[h].R_hi, f2(nz.x, nz.x)), P[h].R_lo);
      d1 = __fadd2_rn(__fadd2_rn(th, f2(nz.y, nz.y)), tl);
    } else {
      d0 = __fadd2_rn(P[h].X, f2(nz.x, nz.x));
      d1 = __fadd2_rn(P[h].Y, f2(nz.y, nz.y));
    }
    return ex2v(expo_fold<MODEL>(d0, d1, na0, na1, P[h].LW, f2(zd[k], zd[k])));
  };
  constexpr bool FOLD = PHD_FOLD_D != 0;

  for (int cb = 0; cb < K; cb += kGateChunk) {
    const int cl = min(kGateChunk, K - cb);
    const int cl8 = (cl + 7) & ~7;
    __syncthreads();  // previous chunk fully consumed
    int nsel = 0, base_sel_unpadded = 0;
    if (PASS == 1) {
      for (int k = tid; k < cl8; k += THREADS) {
        if (k < cl) {
          PHD_DCHECK(e0 + cb + k < g.E);
          const int l = g.cand[e0 + cb + k];
          PHD_DCHECK(l >= 0 && l < g.M);
          zn[k] = f2(g.sc.s0[l], g.sc.s1[l]);
          if (RB) zr[k] = g.sc.rep[l];
        } else {
          zn[k] = f2(-1e30f, -1e30f);  // sentinel: every term exactly 0
          if (RB) zr[k] = 0;
        }
      }
    } else {
      // stable partition: labels in I first (their state sums are reduced), then the
      // rest.  One sweep of ballots (candidate k = tid + THREADS i lies in 32-group
      // k >> 5, owned by one warp), one barrier, then every candidate's position from the
      // group masks: selected ones at their rank among the selected, the others after
      // the (pair-padded) selected block at their rank among the unselected.
      for (int k = tid; k < ((cl + 31) & ~31); k += THREADS) {
        int fl = 0;
        if (k < cl) {
          const int l = g.cand[e0 + cb + k];
          fl = g.sel == nullptr ? 1 : (g.sel[l] != 0);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, fl);
        if (lane == 0) gmask[k >> 5] = bal;
      }
      __syncthreads();
      const int ng = (cl + 31) >> 5;
      for (int q = 0; q < ng; ++q) nsel += __popc(gmask[q]);
      base_sel_unpadded = nsel;
      const int nsel2 = (nsel + 1) & ~1;
      for (int k = tid; k < cl; k += THREADS) {
        const int grp = k >> 5;
        const unsigned m = gmask[grp];
        int before = __popc(m & ((1u << (k & 31)) - 1u));
        for (int q = 0; q < grp; ++q) before += __popc(gmask[q]);
        const bool s = (m >> (k & 31)) & 1u;
        const int pos = s ? before : nsel2 + (k - before);
        PHD_DCHECK(pos < kGateChunk + 2);
        const int l = g.cand[e0 + cb + k];
        PHD_DCHECK(l >= 0 && l < g.M);
        zi[pos] = k;
        zn[pos] = f2(g.sc.s0[l], g.sc.s1[l]);
        zd[pos] = FOLD ? log2f(g.sc.d[l]) / g.na0 : g.sc.d[l];  // fold: d = 0 -> +inf
        if (RB) {
          zr[pos] = g.sc.rep[l];
          zc[pos] = f2(g.sc.s2[l], g.sc.s3[l]);
        }
      }
      if (tid == 0 && nsel2 > nsel) {  // sentinel: every term exactly 0, zi = -1 (never written)
        zi[nsel] = -1;
        zn[nsel] = f2(-1e30f, -1e30f);
        zd[nsel] = FOLD ? INFINITY : 0.0f;
        if (RB) {
          zr[nsel] = 0;
          zc[nsel] = f2(0.0f, 0.0f);
        }
      }
      nsel = nsel2;
    }
    __syncthreads();

    if (PASS == 1) {
      // groups of 8 candidates per transposed reduction; the last, partial group skips the
      // padding candidates' terms (exactly 0) instead of evaluating them (CTA-uniform branch)
      auto group8 = [&](int k8, auto tail_tag) {
        constexpr bool TAIL = decltype(tail_tag)::value;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (TAIL && k8 + j >= cl) {
            v[j] = 0.0f;
            continue;
          }
          float2 d0, d1;
          float2 u = __fadd2_rn(term(k8 + j, 0, d0, d1), term(k8 + j, 1, d0, d1));
          if (NPAIR == 4) u = __fadd2_rn(u, __fadd2_rn(term(k8 + j, 2, d0, d1), term(k8 + j, 3, d0, d1)));
          v[j] = u.x + u.y;
        }
        const float r = transpose_reduce8(v, lane);
        if ((lane & 3) == 0) {
          PHD_DCHECK(k8 + (lane >> 2) < kGateChunk);
          wpart[warp][k8 + (lane >> 2)] = r;
        }
      };
      const int cfull = cl & ~7;
      for (int k8 = 0; k8 < cfull; k8 += 8) group8(k8, std::false_type{});
      if (cfull < cl) group8(cfull, std::true_type{});
      __syncthreads();
      for (int k = tid; k < cl; k += THREADS) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) sum += (double)wpart[w][k];
        PHD_DCHECK(e0 + cb + k < g.E);
        g.part1[e0 + cb + k] = sum;
      }
    } else {
      // selected candidates, two at a time: weights + the four centred state sums; an odd
      // count's last pair skips its sentinel's terms (exactly 0) instead of evaluating them
      auto pair2 = [&](int k, auto tail_tag) {
        constexpr bool TAIL = decltype(tail_tag)::value;
        float v[8];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int kk = k + hh;
          if (TAIL && hh == 1) {
            v[4] = v[5] = v[6] = v[7] = 0.0f;
          } else {
            float2 a0 = f2(0.0f, 0.0f), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
            for (int h = 0; h < NPAIR; ++h) {
              float2 d0, d1;
              float2 u;
              if (FOLD) {
                u = term_fold(kk, h, d0, d1);
                pacc[h] = __fadd2_rn(pacc[h], u);
              } else {
                u = term(kk, h, d0, d1);
                pacc[h] = __ffma2_rn(u, f2(zd[kk], zd[kk]), pacc[h]);
              }
              if (RB) {
                const float2 c = zc[kk];
                d0 = __fadd2_rn(P[h].X, f2(c.x, c.x));  // x - centre_x
                d1 = __fadd2_rn(P[h].Y, f2(c.y, c.y));  // y - centre_y
              }
              a0 = __ffma2_rn(u, d0, a0);
              a1 = __ffma2_rn(u, P[h].VX, a1);
              a2 = __ffma2_rn(u, d1, a2);
              a3 = __ffma2_rn(u, P[h].VY, a3);
            }
            v[4 * hh + 0] = a0.x + a0.y;
            v[4 * hh + 1] = a1.x + a1.y;
            v[4 * hh + 2] = a2.x + a2.y;
            v[4 * hh + 3] = a3.x + a3.y;
          }
        }
        const float r = transpose_reduce8(v, lane);
        const int q = lane >> 2;  // value index 0..7: candidate k + q / 4, quantity q % 4
        if ((lane & 3) == 0) {
          PHD_DCHECK(k + (q >> 2) < kGateChunk + 2);
          reinterpret_cast<float*>(&wq[warp][k + (q >> 2)])[q & 3] = r;
        }
      };
      const int npf = base_sel_unpadded & ~1;  // full pairs of selected candidates
      for (int k = 0; k < npf; k += 2) pair2(k, std::false_type{});
      if (nsel > npf) pair2(npf, std::true_type{});
      // the rest: weights only
      const int kend = cl + (nsel - base_sel_unpadded);
#pragma unroll 2
      for (int k = nsel; k < kend; ++k) {
        const float2 dk = f2(zd[k], zd[k]);
#pragma unroll
        for (int h = 0; h < NPAIR; ++h) {
          float2 d0, d1;
          if (FOLD)
            pacc[h] = __fadd2_rn(pacc[h], term_fold(k, h, d0, d1));
          else
            pacc[h] = __ffma2_rn(term(k, h, d0, d1), dk, pacc[h]);
        }
      }
      __syncthreads();
      for (int k = tid; k < nsel; k += THREADS) {
        if (zi[k] < 0) continue;  // sentinel
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
          const float4 a = wq[w][k];
          s0 += (double)a.x;
          s1 += (double)a.y;
          s2 += (double)a.z;
          s3 += (double)a.w;
        }
        PHD_DCHECK(zi[k] < cl && e0 + cb + zi[k] < g.E);
        reinterpret_cast<float4*>(g.part2)[e0 + cb + zi[k]] = make_float4((float)s0, (float)s1, (float)s2, (float)s3);
      }
    }
  }
  if (PASS == 2) {
#pragma unroll
    for (int h = 0; h < NPAIR; ++h) {
      const int64_t pa = (int64_t)t * TP + 2 * THREADS * h + tid;
      PHD_DCHECK(pa + THREADS < (int64_t)g.ntiles * TP);
      g.Ps[pa] = pacc[h].x;
      g.Ps[pa + THREADS] = pacc[h].y;
    }
  }
}

// one warp per label: fixed-order fp64 sum of its entries (lane-strided + xor tree)
constexpr int kGR = 8;
template <int PASS>
__global__ void __launch_bounds__(256) k_gate_reduce(const int32_t* __restrict__ mstart, const int32_t* __restrict__ mlist,
                                                     int M, const double* __restrict__ part1,
                                                     const float4* __restrict__ part2, const int32_t* __restrict__ sel,
                                                     double* out, int slots_pad, const double* __restrict__ wblk,
                                                     int nwb, double* wout, ZConstArgs zc, const int* poison) {
  pdl_wait();
  if (PASS == 1 && wblk != nullptr && blockIdx.x == gridDim.x - 1) {  // the rank's W_pred (rides in C1)
    block_sum_f64(wblk, nwb, wout);
    // NaN particles (counted by the sort): poison W_pred so that every rank sees a
    // non-finite W_pred after C1 and reports PHD_EMODEL, as the dense path's NaN C does
    if (threadIdx.x == 0 && poison != nullptr && *poison != 0) *wout = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (l >= slots_pad) return;
  const bool live = l < M && (PASS == 1 || sel == nullptr || sel[l] != 0);
  const int j0 = live ? mstart[l] : 0, j1 = live ? mstart[l + 1] : 0;
  if (PASS == 1) {
    double s = 0.0;
    // kGR entries per lane per round: index loads, then partial loads, in flight
    for (int j = j0 + lane; j < j1; j += 32 * kGR) {
      int e[kGR];
#pragma unroll
      for (int r = 0; r < kGR; ++r) e[r] = j + 32 * r < j1 ? mlist[j + 32 * r] : -1;
      double v[kGR];
#pragma unroll
      for (int r = 0; r < kGR; ++r) {
        PHD_DCHECK(e[r] < mstart[M]);
        v[r] = e[r] >= 0 ? part1[e[r]] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < kGR; ++r) s += v[r];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      out[l] = s;
      if (zc.slot_label) zconst_one(zc, l, s);  // one rank: C is final here
    }
  } else {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = j0 + lane; j < j1; j += 32 * kGR) {
      int e[kGR];
#pragma unroll
      for (int r = 0; r < kGR; ++r) e[r] = j + 32 * r < j1 ? mlist[j + 32 * r] : -1;
      float4 v[kGR];
#pragma unroll
      for (int r = 0; r < kGR; ++r) v[r] = e[r] >= 0 ? part2[e[r]] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int r = 0; r < kGR; ++r) {
        s[0] += (double)v[r].x;
        s[1] += (double)v[r].y;
        s[2] += (double)v[r].z;
        s[3] += (double)v[r].w;
      }
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
  pdl_launch(k_scan_sum, nc, 1024, 0, s, a, n, tmp);
  pdl_launch(k_scan_top, 1, 1024, 0, s, tmp, nc, a + n);
  pdl_launch(k_scan_apply, nc, 1024, 0, s, a, n, tmp);
  *launches += 3;
  return cudaGetLastError();
}

cudaError_t gate_sort_particles(int model, const float* const* A, const float* rb, int64_t rb_stride, int64_t n,
                                int64_t n_pad, float wscale, const GateGrid& grid, int32_t* hist, int32_t* scan_tmp,
                                int32_t* keys, const GateSorted& so, cudaStream_t s, int64_t* launches, double* blk_wp,
                                int* nblk_out) {
  *nblk_out = 0;
  const bool rbm = model == kRangeBearing;
  // always launched: it also resets the lw max
  pdl_launch(k_psort_pad, (unsigned)std::max<int64_t>(1, (n_pad - n + 255) / 256), 256, 0, s, n, n_pad, so);
  ++*launches;
  if (n <= 0) return cudaGetLastError();
  KeyCell kf{rbm ? rb : A[0], rbm ? rb + 2 * rb_stride : A[2], grid};
  GatherSrc src{};
  for (int c = 0; c < 8; ++c) src.c[c] = rbm ? rb + c * rb_stride : nullptr;
  src.x = A[0];
  src.vx = A[1];
  src.y = A[2];
  src.vy = A[3];
  src.w = A[4];
  const int64_t per_blk = sort_block(n);
  const int nblk = (int)((n + per_blk - 1) / per_blk);
  *nblk_out = nblk;
  const int psw = ps_warps(rbm ? kRangeBearing : kPosIso);
  const size_t smem = sizeof(uint32_t) * (size_t)psw * (kGateBins / 2) + sizeof(int) * (size_t)kGateBins;
  ensure_max_smem(k_psort_scatter<kRangeBearing>,
                  sizeof(uint32_t) * (size_t)ps_warps(kRangeBearing) * (kGateBins / 2) + sizeof(int) * (size_t)kGateBins);
  ensure_max_smem(k_psort_scatter<kPosIso>,
                  sizeof(uint32_t) * (size_t)ps_warps(kPosIso) * (kGateBins / 2) + sizeof(int) * (size_t)kGateBins);
#ifndef PHD_CELL_HIST_THREADS
#define PHD_CELL_HIST_THREADS 1024
#endif
  // 1024 threads per 64 K-particle block: the cell histogram is latency-bound on its loads
  pdl_launch(k_ms_hist<KeyCell>, nblk, PHD_CELL_HIST_THREADS, 0, s, kf, n, per_blk, kGateBins, nblk, hist, keys);
  ++*launches;
  cudaError_t e = gate_scan(hist, (int64_t)kGateBins * nblk, scan_tmp, s, launches);
  if (e != cudaSuccess) return e;
  if (rbm)
    pdl_launch(k_psort_scatter<kRangeBearing>, nblk, psw * 32, smem, s, src, keys, n, per_blk, nblk, hist, wscale,
               so, blk_wp);
  else
    pdl_launch(k_psort_scatter<kPosIso>, nblk, psw * 32, smem, s, src, keys, n, per_blk, nblk, hist, wscale, so,
               blk_wp);
  ++*launches;
  return cudaGetLastError();
}

// measurement bins by the same stable counting sort (multi-warp; the single-CTA
// k_gate_zbin took ~40 us at M = 4096): zcell_items = labels by cell, zcell_start
// = the scanned histogram's first column, zcell_z = coordinates in cell order
__global__ void k_zbin_finish(const int32_t* __restrict__ hs, int nblk, const float* __restrict__ z,
                              const int32_t* __restrict__ items, int M, int32_t* zcell_start, float2* zcell_z) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kGateBins) zcell_start[i] = hs[(int64_t)i * nblk];
  if (i == kGateBins) zcell_start[kGateBins] = M;
  if (i < M) {
    const int l = items[i];
    zcell_z[i] = make_float2(z[2 * l], z[2 * l + 1]);
  }
}

cudaError_t gate_zbin(const float* z, int M, const GateGrid& grid, int32_t* hist, int32_t* scan_tmp,
                      int32_t* zcell_start, int32_t* zcell_items, float2* zcell_z, cudaStream_t s, int64_t* launches) {
  if (M <= 0) return cudaSuccess;
  KeyZ kf{z, grid};
  const int64_t per_blk = sort_block(M);
  const int nblk = (int)((M + per_blk - 1) / per_blk);
  cudaError_t e = ms_pass(kf, nullptr, M, per_blk, kGateBins, hist, scan_tmp, nullptr, zcell_items, s, launches);
  if (e != cudaSuccess) return e;
  const int nt = std::max(M, kGateBins + 1);
  pdl_launch(k_zbin_finish, (nt + 255) / 256, 256, 0, s, hist, nblk, z, zcell_items, M, zcell_start, zcell_z);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t gate_tiles(int fill, int model, const GateSorted& so, int ntiles, float na0, float na1, const GateGrid& grid,
                       const int32_t* zcell_start, const int32_t* zcell_items, const float2* zcell_z, int32_t* tcount,
                       const int32_t* tstart, int32_t* cbuf, int32_t* cand, cudaStream_t s, int64_t ecap) {
  if (ntiles <= 0) return cudaSuccess;
  const bool rbm = model == kRangeBearing;
  const float* f = reinterpret_cast<const float*>(so.rec);
  RecView rv{f, f + (rbm ? 2 : 1), f + 4 * (so.n4 - 1), 4 * so.n4, so.n, so.lw_max, gate_tp(model)};
  const unsigned blocks = (unsigned)((ntiles + 7) / 8);
  if (fill)
    pdl_launch(k_gate_fill, blocks, 256, 0, s, rv, ntiles, na0, na1, grid, zcell_start, zcell_items, zcell_z, tstart, cbuf,
               cand, ecap);
  else
    pdl_launch(k_gate_count, blocks, 256, 0, s, rv, ntiles, na0, na1, grid, zcell_start, zcell_items, zcell_z, tcount, cbuf);
  return cudaGetLastError();
}

cudaError_t gate_sort_entries(const int32_t* cand, int64_t E, int M, int32_t* kbuf, int32_t* vbuf, int32_t* mlist,
                              int32_t* hist, int32_t* scan_tmp, int32_t* mstart, cudaStream_t s, int64_t* launches) {
  int bits = 1;
  while ((1 << bits) < M) ++bits;
  if (bits <= 12 && E > 0) {
    // one pass: the scanned histogram's first column is the label offsets
    cudaError_t e = csort_pass(cand, nullptr, E, 0, 1 << bits, hist, scan_tmp, nullptr, mlist, s, launches);
    if (e != cudaSuccess) return e;
    const int nblk = (int)((E + sort_block(E) - 1) / sort_block(E));
    pdl_launch(k_mstart_from_hist, (M + 256) / 256, 256, 0, s, hist, nblk, M, (int32_t)E, mstart);
    ++*launches;
    return cudaGetLastError();
  }
  // mstart: per-label counts (integer atomics), exclusive scan (mstart[M] = E)
  pdl_launch(k_zero_i32, (M + 256) / 256, 256, 0, s, mstart, M + 1);
  ++*launches;
  if (E > 0) {
    pdl_launch(k_gate_count_labels, (unsigned)((E + 255) / 256), 256, 0, s, cand, E, mstart);
    ++*launches;
  }
  cudaError_t e = gate_scan(mstart, M, scan_tmp, s, launches);
  if (e != cudaSuccess || E <= 0) return e;
  // two LSD passes of 12 + (bits - 12) bits over the label
  e = csort_pass(cand, nullptr, E, 0, kSortMaxBins, hist, scan_tmp, kbuf, vbuf, s, launches);
  if (e != cudaSuccess) return e;
  return csort_pass(kbuf, vbuf, E, 12, 1 << (bits - 12), hist, scan_tmp, nullptr, mlist, s, launches);
}

#ifndef PHD_GATE_NPAIR1_POS
#define PHD_GATE_NPAIR1_POS 2
#endif
#ifndef PHD_GATE_NPAIR_POS
#define PHD_GATE_NPAIR_POS 4
#endif
template <int MODEL>
static cudaError_t gpass_m(int pass, const GateArgs& g, cudaStream_t s) {
  // pass 2, position: 8 particles per thread (64 threads per tile); range-bearing
  // holds 8 representation registers per pair: 4 particles per thread (128 threads)
  // (measured at cfg 5: pass 2 0.73 -> 0.64 ms with 8 particles per thread, pass 1
  // 0.42 -> 0.44 ms, so pass 1 keeps 4)
  constexpr int NP2 = MODEL == kRangeBearing ? 2 : PHD_GATE_NPAIR_POS;
  constexpr int NP1 = MODEL == kRangeBearing ? 2 : PHD_GATE_NPAIR1_POS;
  if (pass == 1)
    pdl_launch(k_gpass<MODEL, 1, NP1>, g.ntiles, gate_tp(MODEL) / (2 * NP1), 0, s, g);
  else
    pdl_launch(k_gpass<MODEL, 2, NP2>, g.ntiles, gate_tp(MODEL) / (2 * NP2), 0, s, g);
  return cudaGetLastError();
}

cudaError_t launch_gpass(int pass, const GateArgs& g, cudaStream_t s) {
  if (g.ntiles <= 0) return cudaSuccess;
  if (g.model == kPosIso) return gpass_m<kPosIso>(pass, g, s);
  if (g.model == kPosAniso) return gpass_m<kPosAniso>(pass, g, s);
  return gpass_m<kRangeBearing>(pass, g, s);
}

cudaError_t launch_gate_reduce(int pass, const int32_t* mstart, const int32_t* mlist, int M, const double* part1,
                               const float* part2, const int32_t* sel, double* out, int slots_pad, cudaStream_t s,
                               const double* wblk, int nwb, double* wout, const ZConstArgs* zc, const int* poison) {
  if (pass != 1) wblk = nullptr;
  const ZConstArgs z = zc && pass == 1 ? *zc : ZConstArgs{};
  const unsigned blocks = (unsigned)((std::max(slots_pad, 0) + 7) / 8 + (wblk ? 1 : 0));
  if (blocks == 0) return cudaSuccess;
  if (pass == 1)
    pdl_launch(k_gate_reduce<1>, blocks, 256, 0, s, mstart, mlist, M, part1, nullptr, nullptr, out, slots_pad, wblk,
               nwb, wout, z, poison);
  else
    pdl_launch(k_gate_reduce<2>, blocks, 256, 0, s, mstart, mlist, M, nullptr, reinterpret_cast<const float4*>(part2), sel,
                                            out, slots_pad, nullptr, 0, nullptr, z, nullptr);
  return cudaGetLastError();
}


void preload_gate() {
  touch_kernels(k_scan_sum, k_scan_top, k_scan_apply, k_ms_hist<KeyCell>, k_ms_hist<KeyArr>, k_ms_hist<KeyZ>,
                k_ms_scatter<KeyArr>, k_ms_scatter<KeyZ>, k_psort_pad, k_psort_scatter<kPosIso>,
                k_psort_scatter<kRangeBearing>, k_gate_count, k_gate_fill, k_gate_count_labels, k_mstart_from_hist,
                k_zero_i32, k_gate_reduce<1>, k_gate_reduce<2>, k_zbin_finish);
  touch_kernels(k_gpass<kPosIso, 1, PHD_GATE_NPAIR1_POS>, k_gpass<kPosIso, 2, PHD_GATE_NPAIR_POS>, k_gpass<kPosAniso, 1, PHD_GATE_NPAIR1_POS>,
                k_gpass<kPosAniso, 2, PHD_GATE_NPAIR_POS>, k_gpass<kRangeBearing, 1, 2>, k_gpass<kRangeBearing, 2, 2>);
}

}  // namespace phd
