// Prediction step (§2.2 step 1): Eq 5 survivors with the CV model
// and Eq 6 births (measurement-driven, S10), plus the
// Eq 6 importance weights of birth_model 2 (k_birth_is).
// SoA fp32 in/out, HBM-bound (20 B read + 20 B written per survivor; 20 B written
// per birth; +32 B of range-bearing representation when that sensor is used): four
// survivors per thread with float4 loads/stores for large position-sensor
// populations, one slot per thread otherwise (k_predict<VEC>).
#include "phd_internal.h"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include "philox.cuh"

namespace phd {

cudaError_t ensure_max_smem_impl(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[std::make_pair(func, dev)];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

void preload_kernels() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert(dev).second) return;
  preload_predict();
  preload_update();
  preload_select();
  preload_extract();
  preload_resample();
  preload_gate();
  cudaGetLastError();  // attribute queries never leave an error behind
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("PHD_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

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

// Eq 5 for one survivor: x~ ~ q(.|x), the CV model with noise std s sigma_a
// (a.sigma_a holds s sigma_a), w~ = e_{k|k-1} f/q w.  f/q is the ratio of the noise
// densities at the drawn a = s sigma_a n; with n1^2 + n2^2 = -2 ln u1 (Box-Muller
// radius) it is s^2 u1^(s^2 - 1), and 1 for s = 1 (transition prior).  Explicit
// roundings, so the vector and scalar paths give the same bits.
__device__ __forceinline__ void survivor(const PredictArgs& a, int64_t g, float& x, float& vx, float& y, float& vy,
                                         float& w) {
  U4 o = philox_at(a.seed, a.ctr_base + (uint64_t)g, (uint32_t)(a.ds ? a.ds->k : a.k), 1u);
  float u1 = u01(o.x), u2 = u01(o.y);
  float rad = sqrtf(-2.0f * logf(u1));
  float sn, cs;
  sincospif(2.0f * u2, &sn, &cs);
  const float ax = __fmul_rn(a.sigma_a, __fmul_rn(rad, cs)), ay = __fmul_rn(a.sigma_a, __fmul_rn(rad, sn));
  const float hT2 = 0.5f * a.T * a.T;
  x = __fmaf_rn(hT2, ax, __fmaf_rn(a.T, vx, x));
  vx = __fmaf_rn(a.T, ax, vx);
  y = __fmaf_rn(hT2, ay, __fmaf_rn(a.T, vy, y));
  vy = __fmaf_rn(a.T, ay, vy);
  w = __fmul_rn(a.p_s, w);
  if (a.prop_s != 1.0f) {
    const float s2 = a.prop_s * a.prop_s;
    w = __fmul_rn(w, s2 * exp2f((s2 - 1.0f) * log2f(u1)));
  }
}

// One slot (survivor or birth), scalar loads and stores.
__device__ __forceinline__ void predict_one(const PredictArgs& a, int64_t i) {
  int64_t g = a.g0 + i;
  float x, vx, y, vy, w;
  if (g < a.n_out) {
    x = a.x[i];
    vx = a.vx[i];
    y = a.y[i];
    vy = a.vy[i];
    w = a.w_uniform >= 0.0f ? a.w_uniform : a.w[i];
    survivor(a, g, x, vx, y, vy, w);
  } else {
    // Eq 6: birth b ~ p_k(.|Z_{k-1}) with weight gamma / J_k.
    int64_t b = g - a.n_out;
    U4 o = philox_at(a.seed, a.ctr_base + (uint64_t)g, (uint32_t)(a.ds ? a.ds->k : a.k), 2u);
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
    const int m_prev = a.ds ? a.ds->M_prev : a.m_prev;
    if (m_prev > 0) {
      int64_t m = (a.birth_offset + b) % m_prev;
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

// Large position-sensor populations: four consecutive slots per thread, float4
// loads and stores of the SoA arrays when all four are survivors (the local arrays
// are 16-byte aligned), the scalar path for births and the tail.  Range-bearing and
// small populations: one slot per thread (the fp64 representation dominates the
// range-bearing case; four per thread measured slower there).
template <bool VEC>
__global__ void __launch_bounds__(256) k_predict(const PredictArgs a) {
  pdl_wait();
  if (!VEC) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.n_local) predict_one(a, i);
    return;
  }
  const int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (i0 >= a.n_local) return;
  if (i0 + 3 < a.n_local && a.g0 + i0 + 3 < a.n_out) {
    float4 X = *reinterpret_cast<const float4*>(a.x + i0);
    float4 VX = *reinterpret_cast<const float4*>(a.vx + i0);
    float4 Y = *reinterpret_cast<const float4*>(a.y + i0);
    float4 VY = *reinterpret_cast<const float4*>(a.vy + i0);
    float4 W = a.w_uniform >= 0.0f ? make_float4(a.w_uniform, a.w_uniform, a.w_uniform, a.w_uniform)
                                   : *reinterpret_cast<const float4*>(a.w + i0);
    const int64_t g = a.g0 + i0;
    survivor(a, g, X.x, VX.x, Y.x, VY.x, W.x);
    survivor(a, g + 1, X.y, VX.y, Y.y, VY.y, W.y);
    survivor(a, g + 2, X.z, VX.z, Y.z, VY.z, W.z);
    survivor(a, g + 3, X.w, VX.w, Y.w, VY.w, W.w);
    *reinterpret_cast<float4*>(a.x + i0) = X;
    *reinterpret_cast<float4*>(a.vx + i0) = VX;
    *reinterpret_cast<float4*>(a.y + i0) = Y;
    *reinterpret_cast<float4*>(a.vy + i0) = VY;
    *reinterpret_cast<float4*>(a.w + i0) = W;
    return;
  }
  for (int q = 0; q < 4; ++q)
    if (i0 + q < a.n_local) predict_one(a, i0 + q);
}

// Eq 6 with the full ratio (birth_model 2):
//   w_b = gamma N(x_b; x-bar, Q) / (J p_k(x_b | Z_{k-1})),
//   p_k(x) = sum_c (n_c / J) q_c(pos) N(vx; 0, sv^2) N(vy; 0, sv^2),
// n_c = #{b in [birth_offset, birth_offset + J) : b mod M' = c} (the births take
// component b mod M' deterministically: a stratified mixture).  q_c is the
// proposal's position law: N(z_c, diag(s0^2, s1^2)) for the position sensor; for
// range-bearing the image of N(z_c, .) under (a, c) -> (a cos c, a sin c), whose
// density at (x, y) sums the preimages (r, th) and (-r, th + pi), each divided by
// the Jacobian r.  No previous set: uniform, 1/V or 1/(V r).
// One thread per birth; components staged through shared memory with their
// mixture weights.  Residuals and exponents in fp64, the exponential by
// ex2.approx of the fp32-rounded exponent (relative error <= |E| 2^-24 + 2 ulp),
// the mixture sum in fp64.  J M' terms per step: cold (births only).
constexpr int kISChunk = 1024;

__device__ __forceinline__ double wrap_pi_d(double d) {
  const double pi = 3.141592653589793238462643383279503, two_pi = 6.283185307179586476925286766559;
  d = fmod(d, two_pi);
  if (d > pi) d -= two_pi;
  if (d <= -pi) d += two_pi;
  return d;
}

__device__ __forceinline__ int64_t count_below(int64_t e, int64_t c, int64_t M) {
  return e > c ? (e - c - 1) / M + 1 : 0;
}

__device__ __forceinline__ double ex2d(double e) {  // 2^e via MUFU on the fp32-rounded exponent
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"((float)e));
  return (double)y;
}

__global__ void __launch_bounds__(256) k_birth_is(const BirthISArgs a) {
  pdl_wait();
  __shared__ double zc0[kISChunk], zc1[kISChunk], wc[kISChunk];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < a.nb;
  const double log2e = 1.4426950408889634073599246810019;
  const double pi = 3.141592653589793238462643383279503;
  double x = 0, vx = 0, y = 0, vy = 0, r = 0, th = 0;
  if (live) {
    const int64_t i = a.i0 + t;
    x = a.x[i];
    vx = a.vx[i];
    y = a.y[i];
    vy = a.vy[i];
    if (a.meas != 0) {
      const double px = x - a.sensor_x, py = y - a.sensor_y;
      r = sqrt(px * px + py * py);
      th = (px == 0.0 && py == 0.0) ? 0.0 : atan2(py, px);
    }
  }
  // -log2 e / (2 s^2) per axis
  const double k0 = -log2e / (2.0 * a.sigma_z0 * a.sigma_z0), k1 = -log2e / (2.0 * a.sigma_z1 * a.sigma_z1);
  double pos = 0.0;
  if (a.m_prev > 0) {
    for (int c0 = 0; c0 < a.m_prev; c0 += kISChunk) {
      const int nc = min(kISChunk, a.m_prev - c0);
      __syncthreads();
      for (int q = threadIdx.x; q < nc; q += blockDim.x) {
        const int64_t c = c0 + q;
        zc0[q] = a.zprev[2 * c];
        zc1[q] = a.zprev[2 * c + 1];
        const int64_t n_c = count_below(a.birth_offset + a.J, c, a.m_prev) - count_below(a.birth_offset, c, a.m_prev);
        wc[q] = (double)n_c / (double)a.J;
      }
      __syncthreads();
      if (live) {
        if (a.meas == 0) {
          for (int q = 0; q < nc; ++q) {
            const double d0 = x - zc0[q], d1 = y - zc1[q];
            pos += wc[q] * ex2d(k0 * d0 * d0 + k1 * d1 * d1);
          }
        } else {
          for (int q = 0; q < nc; ++q) {
            const double da = r - zc0[q], db = -r - zc0[q];
            const double ta = wrap_pi_d(th - zc1[q]), tb = wrap_pi_d(th + pi - zc1[q]);
            pos += wc[q] * (ex2d(k0 * da * da + k1 * ta * ta) + ex2d(k0 * db * db + k1 * tb * tb));
          }
        }
      }
    }
    pos *= 1.0 / (2.0 * pi * a.sigma_z0 * a.sigma_z1);
    if (a.meas != 0) pos = r > 0.0 ? pos / r : 0.0;
  } else {
    const double V = (a.region[1] - a.region[0]) * (a.region[3] - a.region[2]);
    pos = a.meas == 0 ? 1.0 / V : (r > 0.0 ? 1.0 / (V * r) : 0.0);
  }
  if (!live) return;
  const double sv = a.birth_sigma_v;
  // log of the velocity factor of p_k and of gamma(x) / gamma; 2 pi factors explicit
  const double lpv = -(vx * vx + vy * vy) / (2.0 * sv * sv) - log(2.0 * pi * sv * sv);
  const double st[4] = {x, vx, y, vy};
  double lg = -2.0 * log(2.0 * pi);
  for (int d = 0; d < 4; ++d) {
    const double u = (st[d] - a.birth_mean[d]) / a.birth_std[d];
    lg += -0.5 * u * u - log(a.birth_std[d]);
  }
  double w = 0.0;
  if (pos > 0.0) w = a.gamma / (double)a.J * exp(lg - lpv - log(pos));
  a.w[a.i0 + t] = (float)w;
}

cudaError_t launch_birth_is(const BirthISArgs& a, cudaStream_t s) {
  if (a.nb <= 0) return cudaSuccess;
  pdl_launch(k_birth_is, (unsigned)((a.nb + 255) / 256), 256, 0, s, a);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_rb_repr(const float* __restrict__ x, const float* __restrict__ y,
                                                 int64_t n, float sx, float sy, float* rb, int64_t stride) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rb_repr(x[i], y[i], sx, sy, rb, stride, i);
}

// ---------------------------------------------------------------------------
// t = 0 population ("Generate M particles for each group ... same weights
// omega_0 = 1/M"; reading S23): particle g is y-stratified over the box,
//   y = y0 + (y1 - y0)(g + u0)/n_out,  x = x0 + (x1 - x0) u1,  v = v_max (2 u2 - 1, 2 u3 - 1),
// u_c = word c of Philox({g, 0, 5, g >> 32}); fp64 with explicit IEEE roundings (no
// contraction) then one rounding to fp32, so the states are bitwise the oracle's.
// HBM-bound: 20 B written per particle.
__device__ __forceinline__ bool in_box(float x, float y, const double* b) {
  const double xd = x, yd = y;
  return xd >= b[0] && xd <= b[1] && yd >= b[2] && yd <= b[3];
}

__global__ void __launch_bounds__(256) k_init_population(const InitArgs a) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int cnt = 0;
  const float wu = a.has_mbox ? 0.0f : __double2float_rn(__ddiv_rn(a.total_mass, a.n_norm));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_local; i += stride) {
    const int64_t g = a.g0 + i;
    const U4 o = philox_at(a.seed, (uint64_t)g, 0u, 5u);
    const double u0 = u01(o.x), u1 = u01(o.y), u2 = u01(o.z), u3 = u01(o.w);
    const double y = __dadd_rn(a.box[2], __ddiv_rn(__dmul_rn(__dsub_rn(a.box[3], a.box[2]), __dadd_rn((double)g, u0)),
                                                   (double)a.n_out));
    const double x = __dadd_rn(a.box[0], __dmul_rn(__dsub_rn(a.box[1], a.box[0]), u1));
    const double vx = __dmul_rn(a.v_max, __dsub_rn(__dmul_rn(2.0, u2), 1.0));
    const double vy = __dmul_rn(a.v_max, __dsub_rn(__dmul_rn(2.0, u3), 1.0));
    const float xf = __double2float_rn(x), yf = __double2float_rn(y);
    a.x[i] = xf;
    a.vx[i] = __double2float_rn(vx);
    a.y[i] = yf;
    a.vy[i] = __double2float_rn(vy);
    if (a.has_mbox) {
      cnt += in_box(xf, yf, a.mbox) ? 1 : 0;
    } else {
      a.w[i] = wu;
    }
  }
  if (a.has_mbox) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt > 0) atomicAdd(a.count, (double)cnt);  // integers: exact in any order
  }
}

__global__ void __launch_bounds__(256) k_init_weights(const InitArgs a) {
  pdl_wait();
  const double c = *a.count;
  const float wv = c > 0.0 ? __double2float_rn(__ddiv_rn(a.total_mass, c)) : 0.0f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_local; i += stride)
    a.w[i] = in_box(a.x[i], a.y[i], a.mbox) ? wv : 0.0f;
}

static unsigned init_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

cudaError_t launch_init_population(const InitArgs& a, cudaStream_t s) {
  if (a.n_local <= 0) return cudaSuccess;
  pdl_launch(k_init_population, init_grid(a.n_local), 256, 0, s, a);
  return cudaGetLastError();
}

cudaError_t launch_init_weights(const InitArgs& a, cudaStream_t s) {
  if (a.n_local <= 0) return cudaSuccess;
  pdl_launch(k_init_weights, init_grid(a.n_local), 256, 0, s, a);
  return cudaGetLastError();
}

// Known-answer hook: the kernels' Philox (philox.cuh) on n device counters.
__global__ void k_philox_kat(uint64_t seed, const uint4* __restrict__ ctr, int64_t n, uint4* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 c = ctr[i];
  const U4 o = philox10(U4{c.x, c.y, c.z, c.w}, (uint32_t)seed, (uint32_t)(seed >> 32));
  out[i] = make_uint4(o.x, o.y, o.z, o.w);
}

cudaError_t launch_philox_kat(uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_philox_kat<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(seed, reinterpret_cast<const uint4*>(ctr), n,
                                                           reinterpret_cast<uint4*>(out));
  return cudaGetLastError();
}

__global__ void k_fill(float* p, float v, int64_t n) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

cudaError_t launch_predict(const PredictArgs& a, cudaStream_t s) {
  if (a.n_local <= 0) return cudaSuccess;
  // four slots per thread only when that still fills the GPU (cfg 3, 1.1e5 slots:
  // 4.2 us scalar vs 6.8 us; cfg 5, 1.7e7: 135 vs 108 us)
  if (a.rb || a.n_local < (int64_t)1 << 21) {
    pdl_launch(k_predict<false>, (unsigned)((a.n_local + 255) / 256), 256, 0, s, a);
  } else {
    pdl_launch(k_predict<true>, (unsigned)((a.n_local + 1023) / 1024), 256, 0, s, a);  // four slots per thread
  }
  return cudaGetLastError();
}

cudaError_t launch_rb_repr(const float* x, const float* y, int64_t n, float sx, float sy, float* rb,
                           int64_t stride, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pdl_launch(k_rb_repr, (unsigned)((n + 255) / 256), 256, 0, s, x, y, n, sx, sy, rb, stride);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* p, float v, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pdl_launch(k_fill, (unsigned)((n + 255) / 256), 256, 0, s, p, v, n);
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
  pdl_wait();
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
  pdl_launch(k_sum_ranks, (unsigned)((n + 255) / 256), 256, 0, s, rp, world, dst, n);
  return cudaGetLastError();
}


void preload_predict() {
  touch_kernels(k_predict<false>, k_predict<true>, k_birth_is, k_rb_repr, k_init_population, k_init_weights,
                k_philox_kat, k_fill, k_sum_ranks);
}

}  // namespace phd
