// Prediction step (§2.2 step 1): Eq 5 survivors with the CV model
// and Eq 6 births (measurement-driven, S10).
// One thread per particle slot of this rank's block; SoA fp32 in/out, HBM-bound
// (20 B read + 20 B written per survivor; 20 B written per birth; +32 B of
// range-bearing representation when that sensor is used).
#include "phd_internal.h"
#include "philox.cuh"

namespace phd {

// Per-particle range-bearing representation, computed once in fp64 and split
// into fp32 hi + lo (DESIGN.md §5 "seam-free residual"):
// [0] r_hi [1] r_lo [2,3] thetaA in (-pi,pi] [4,5] thetaB in [0,2pi) [6,7] thetaC in (-2pi,0].
__device__ __forceinline__ void rb_repr(float xf, float yf, float sx, float sy, float* rb, int64_t stride,
                                        int64_t i) {
  const double two_pi = 6.283185307179586476925286766559;
  double px = (double)xf - (double)sx, py = (double)yf - (double)sy;
  double r = sqrt(px * px + py * py);
  double th = (px == 0.0 && py == 0.0) ? 0.0 : atan2(py, px);
  double thB = th < 0.0 ? th + two_pi : th;
  double thC = th > 0.0 ? th - two_pi : th;
  float rh = (float)r, ah = (float)th, bh = (float)thB, ch = (float)thC;
  rb[0 * stride + i] = rh;
  rb[1 * stride + i] = (float)(r - (double)rh);
  rb[2 * stride + i] = ah;
  rb[3 * stride + i] = (float)(th - (double)ah);
  rb[4 * stride + i] = bh;
  rb[5 * stride + i] = (float)(thB - (double)bh);
  rb[6 * stride + i] = ch;
  rb[7 * stride + i] = (float)(thC - (double)ch);
}

__global__ void __launch_bounds__(256) k_predict(const PredictArgs a) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_local) return;
  int64_t g = a.g0 + i;
  float x, vx, y, vy, w;
  if (g < a.n_out) {
    // Eq 5: x~ ~ f(.|x) (q = transition prior), w~ = e_{k|k-1} w.
    U4 o = philox_at(a.seed, a.ctr_base + (uint64_t)g, (uint32_t)a.k, 1u);
    float u1 = u01(o.x), u2 = u01(o.y);
    float rad = sqrtf(-2.0f * logf(u1));
    float sn, cs;
    sincospif(2.0f * u2, &sn, &cs);
    float ax = a.sigma_a * (rad * cs), ay = a.sigma_a * (rad * sn);
    float hT2 = 0.5f * a.T * a.T;
    x = a.x[i];
    vx = a.vx[i];
    y = a.y[i];
    vy = a.vy[i];
    w = a.w_uniform >= 0.0f ? a.w_uniform : a.w[i];
    x = x + a.T * vx + hT2 * ax;
    vx = vx + a.T * ax;
    y = y + a.T * vy + hT2 * ay;
    vy = vy + a.T * ay;
    w = a.p_s * w;
  } else {
    // Eq 6: birth b ~ p_k(.|Z_{k-1}) with weight gamma / J_k.
    int64_t b = g - a.n_out;
    U4 o = philox_at(a.seed, a.ctr_base + (uint64_t)g, (uint32_t)a.k, 2u);
    float u0 = u01(o.x), u1 = u01(o.y), u2 = u01(o.z), u3 = u01(o.w);
    float r01 = sqrtf(-2.0f * logf(u0)), r23 = sqrtf(-2.0f * logf(u2));
    float s1, c1, s2, c2;
    sincospif(2.0f * u1, &s1, &c1);
    sincospif(2.0f * u3, &s2, &c2);
    float n1 = r01 * c1, n2 = r01 * s1, n3 = r23 * c2, n4 = r23 * s2;
    float p0, p1;
    if (a.birth_model == 1) {
      // birth intensity N(x-bar, Q), Q diagonal
      a.x[i] = a.birth_mean[0] + a.birth_std[0] * n1;
      a.vx[i] = a.birth_mean[1] + a.birth_std[1] * n2;
      a.y[i] = a.birth_mean[2] + a.birth_std[2] * n3;
      a.vy[i] = a.birth_mean[3] + a.birth_std[3] * n4;
      a.w[i] = a.birth_w;
      if (a.rb) rb_repr(a.x[i], a.y[i], a.sensor_x, a.sensor_y, a.rb, a.rb_stride, i);
      return;
    }
    if (a.m_prev > 0) {
      int64_t m = (a.birth_offset + b) % a.m_prev;
      p0 = a.zprev[2 * m] + a.sigma_z0 * n1;
      p1 = a.zprev[2 * m + 1] + a.sigma_z1 * n2;
    } else {
      p0 = a.region[0] + (a.region[1] - a.region[0]) * u0;
      p1 = a.region[2] + (a.region[3] - a.region[2]) * u1;
    }
    if (a.meas == 0) {
      x = p0;
      y = p1;
    } else {
      float sp, cp;
      sincosf(p1, &sp, &cp);
      x = a.sensor_x + p0 * cp;
      y = a.sensor_y + p0 * sp;
    }
    vx = a.birth_sigma_v * n3;
    vy = a.birth_sigma_v * n4;
    w = a.birth_w;
  }
  a.x[i] = x;
  a.vx[i] = vx;
  a.y[i] = y;
  a.vy[i] = vy;
  a.w[i] = w;
  if (a.rb) rb_repr(x, y, a.sensor_x, a.sensor_y, a.rb, a.rb_stride, i);
}

__global__ void __launch_bounds__(256) k_rb_repr(const float* __restrict__ x, const float* __restrict__ y,
                                                 int64_t n, float sx, float sy, float* rb, int64_t stride) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rb_repr(x[i], y[i], sx, sy, rb, stride, i);
}

__global__ void k_fill(float* p, float v, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

cudaError_t launch_predict(const PredictArgs& a, cudaStream_t s) {
  if (a.n_local <= 0) return cudaSuccess;
  int64_t blocks = (a.n_local + 255) / 256;
  k_predict<<<(unsigned)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_rb_repr(const float* x, const float* y, int64_t n, float sx, float sy, float* rb,
                           int64_t stride, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_rb_repr<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, y, n, sx, sy, rb, stride);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* p, float v, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_fill<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, v, n);
  return cudaGetLastError();
}

}  // namespace phd

// ---------------------------------------------------------------------------
// In-process rank-group all-reduce (LocalComm, test transport): dst = sum over
// ranks in rank order of srcs[r] (all buffers device-visible).
#include "comm.h"

namespace phd {

struct RankPtrs {
  const double* p[16];
};

__global__ void k_sum_ranks(RankPtrs ptrs, int world, double* dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += ptrs.p[r][i];
  dst[i] = s;
}

cudaError_t launch_sum_ranks(const double* const* srcs, int world, double* dst, size_t n, cudaStream_t s) {
  if (world > 16) return cudaErrorInvalidValue;
  RankPtrs rp{};
  for (int r = 0; r < world; ++r) rp.p[r] = srcs[r];
  k_sum_ranks<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rp, world, dst, n);
  return cudaGetLastError();
}

}  // namespace phd
