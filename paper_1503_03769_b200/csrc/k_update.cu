// The fused two-pass particle x measurement update (§2.2 step 2,
// Eqs 7-8; §3 Eqs 10-16).  Never materialises the N x M likelihood matrix.
//
// Tiling: measurement-stationary.  A CTA owns wz x 32 x ZL
// measurement slots (each lane ZL = 8 slots = four f32x2 pairs in registers);
// particles stream through shared memory in tiles of 64 and are broadcast to
// every lane.  Per (particle, slot) pair the lane evaluates the likelihood with
// packed FFMA2/FADD2/FMUL2 and one MUFU.EX2:
//   both:    u = 2^(-alpha q + log2(p_D c w_i)) = p_D g(z_s|x_i) w_i (ex2.approx.ftz)
//   pass 1:  C_s += u                                                      (Eq 7)
//   pass 2:  P_i += u d_s, d_s = 1/(kappa + C_s);  S'_s += u (x_i - z_s), u vx_i, ...
//            (Eqs 8, 12-16; dW_s = C_s/D_s)
// Per-slot sums accumulate in fp32 over one tile (64 particles), then in fp64
// in shared memory (DESIGN.md §5 "accumulation precision").  Per-particle sums Pe_i are reduced across lanes with a
// transposed butterfly and across warps through shared memory, giving one
// fp32 partial per (particle, z-block).  Cross-CTA sums are fp64 in fixed order.
#include "phd_internal.h"

#include <atomic>
#include "pair_math.cuh"
#include "bulk.cuh"
#include "slots.cuh"

#include <algorithm>
#include <type_traits>

#ifndef PHD_FIN_STAGE
#define PHD_FIN_STAGE 1
#endif

#ifndef PHD_PP_UNROLL1
#define PHD_PP_UNROLL1 8
#endif
#ifndef PHD_PP_UNROLL2
#define PHD_PP_UNROLL2 8
#endif

// pass 1: evaluate exp2 of the last slot pair with the FFMA2 polynomial on every
// PHD_EMU_PERIOD-th particle (0 = never); the rest go to MUFU.EX2
#ifndef PHD_EMU_PERIOD
#define PHD_EMU_PERIOD 4
#endif

namespace phd {

// particles unrolled per lane in the pair loop (pass 1 / pass 2; measured on B200)
constexpr int kPPUnroll1 = PHD_PP_UNROLL1;
constexpr int kPPUnroll2 = PHD_PP_UNROLL2;

// range-bearing pass 1 carries 8 FP32x2 per slot pair against 2 MUFU (balanced pipes): half
// the offload (measured cfg 4 pass 1 1.80 -> 1.76 ms; position keeps 1/16: 15.3 vs 15.7 ms)
#ifndef PHD_EMU_PERIOD_RB
#define PHD_EMU_PERIOD_RB 8
#endif
constexpr int kEmuPeriod = PHD_EMU_PERIOD;
constexpr int kEmuPeriodRB = PHD_EMU_PERIOD_RB;
constexpr bool kFoldD = PHD_FOLD_D != 0;

// 2^x for a pair on the FMA pipe (MUFU offload):
// x = j + r with j = rint(x) by the 1.5*2^23 shifter, |r| <= 1/2, 2^r by a
// degree-5 polynomial (relative error <= 3.2e-7 including fp32 Horner rounding,
// tools/fit_exp2_poly.py; MUFU.EX2 is ~2 ulp), exponent j added to the bits.
// x is clamped to -127, where the result is +0 exactly; for x in (-127, -126)
// it returns a value below 2^-126 that ex2.approx.ftz would flush to 0.
__device__ __forceinline__ float2 ex2_poly(float2 x) {
  constexpr float kShift = 12582912.0f;  // 1.5 * 2^23
  x = f2(fmaxf(x.x, -127.0f), fmaxf(x.y, -127.0f));
  const float2 t = __fadd2_rn(x, f2(kShift, kShift));
  const float2 mj = __fadd2_rn(f2(kShift, kShift), f2(-t.x, -t.y));  // -j, exact
  const float2 r = __fadd2_rn(x, mj);                                // exact
  float2 p = __ffma2_rn(f2(1.2943478e-3f, 1.2943478e-3f), r, f2(9.6695982e-3f, 9.6695982e-3f));
  p = __ffma2_rn(p, r, f2(5.5516288e-2f, 5.5516288e-2f));
  p = __ffma2_rn(p, r, f2(2.4022245e-1f, 2.4022245e-1f));
  p = __ffma2_rn(p, r, f2(6.9314647e-1f, 6.9314647e-1f));
  p = __ffma2_rn(p, r, f2(1.0f, 1.0f));
  return f2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
            __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Particle records of the dense passes (floats, multiple of 4), built once per update
// in global memory by k_records and streamed into shared memory by bulk copies.  Scalars,
// read as broadcast f32x2 operands (FADD2 Rd, Ra.F32, Rb.F32x2):
//   position (8):        x, y, lw, 0 | vx, vy, 0, 0
//   range-bearing (16):  r_hi, r_lo, lw, 0 | thA hi, lo, thB hi, lo | thC hi, lo, x, y | vx, vy, 0, 0
// with lw = log2(p_D c w); the bearing representation c of a slot pair sits at 4 + 2c, its
// lo part pre-scaled by s = sigma_r / sigma_theta (the dense kernels measure the bearing
// residual in range units, see residual()).
template <int MODEL>
struct GRec {
  static constexpr bool RB = MODEL == kRangeBearing;
  static constexpr int WIDTH = RB ? 16 : 8;
  static constexpr int LW = 2;
  static constexpr int XY = RB ? 10 : 0;
  static constexpr int V = RB ? 12 : 4;
};

#ifndef PHD_PASS_STAGES
#define PHD_PASS_STAGES 2
#endif
constexpr int kPassStages = PHD_PASS_STAGES;  // record tiles in flight per CTA (bulk copies)
// fp32 runs of the per-slot sums before they are added in fp64 (DESIGN.md §5 "accumulation
// precision"): at most 128 particles, whatever the tile size
#ifndef PHD_FLUSH_P
#define PHD_FLUSH_P 128
#endif
constexpr int kFlushP = PHD_FLUSH_P < kTileP ? PHD_FLUSH_P : kTileP;

// Per-lane measurement constants for its NP slot pairs.
template <int MODEL, int PASS, int NP, bool FOLD = false, int JS = NP>
struct LaneZ {
  float2 n0[NP], n1[NP];  // -z components
  float2 d[NP];           // pass 2: 1/(kappa + C), or with FOLD c = log2(1/(kappa + C)) / na0
  float2 c0[NP], c1[NP];  // -(Cartesian centre) (range-bearing, pass 2)
  int roff[NP];           // bearing-representation offset in the record (range-bearing)

  __device__ __forceinline__ void load(const PassArgs& a, int slot0) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      int s = slot0 + 2 * j;
      n0[j] = f2(a.sc.s0[s], a.sc.s0[s + 1]);
      n1[j] = f2(a.sc.s1[s], a.sc.s1[s + 1]);
      if (PASS == 2) {
        d[j] = f2(a.sc.d[s], a.sc.d[s + 1]);
        if (FOLD) d[j] = f2(log2f(d[j].x) / a.na0, log2f(d[j].y) / a.na0);  // d = 0: +inf
      }
      if (MODEL == kRangeBearing) {
        roff[j] = 4 + 2 * a.sc.rep[s];
        if (PASS == 2 && j < JS) {  // the centres are used by the state sums only
          c0[j] = f2(a.sc.s2[s], a.sc.s2[s + 1]);
          c1[j] = f2(a.sc.s3[s], a.sc.s3[s + 1]);
        }
      }
    }
  }
};

// Residuals (d0, d1) of the lane's slot pair j against the broadcast particle.
// P = the record's first float4: (x, y, lw, 0) or (r_hi, r_lo, lw, 0).  Range-bearing: the
// bearing residual is returned in range units, d1 = s (th_hi - z_th) + s th_lo with
// s = sigma_r / sigma_theta (one FFMA2; s th_lo from the record), so the exponent is the
// isotropic alpha_r (d0^2 + d1^2) -- one FMUL2 fewer per slot pair than two coefficients.
// The residual th_hi - z_th is exact and the FFMA rounds once (as the FADD it replaces).
template <int MODEL, int PASS, int NP, bool FOLD, int JS>
__device__ __forceinline__ void residual(const float* rec, const float4& P, const LaneZ<MODEL, PASS, NP, FOLD, JS>& z,
                                         int j, float2& d0, float2& d1, float2 s) {
  if (MODEL == kRangeBearing) {
    const float2 T = *reinterpret_cast<const float2*>(rec + z.roff[j]);  // (th_hi, s th_lo) of the pair's class
    d0 = __fadd2_rn(__fadd2_rn(f2(P.x, P.x), z.n0[j]), f2(P.y, P.y));   // (r_hi - z_r) + r_lo
    d1 = __ffma2_rn(__fadd2_rn(f2(T.x, T.x), z.n1[j]), s, f2(T.y, T.y)); // s (th_hi - z_th) + s th_lo
  } else {
    d0 = __fadd2_rn(f2(P.x, P.x), z.n0[j]);  // x - z_x
    d1 = __fadd2_rn(f2(P.y, P.y), z.n1[j]);  // y - z_y
  }
}

// ZL = measurement slots per lane (4 or 8); the CTA covers wz * 32 * ZL slots.
#ifndef PHD_PASS_MINB8
#define PHD_PASS_MINB8 2
#endif
#ifndef PHD_PASS1_MINB8
#define PHD_PASS1_MINB8 2
#endif
template <int MODEL, int PASS, int ZL, int TILE, bool SPLIT>
__global__ void __launch_bounds__(max_warps_z(ZL) * 32,
                                  ZL == 8 ? (kMaxWarpsZ > 8 ? 1 : (PASS == 1 ? PHD_PASS1_MINB8 : PHD_PASS_MINB8)) : 3)
    k_pass(const PassArgs a) {
  pdl_wait();
  using L = GRec<MODEL>;
  constexpr int NQ = PASS == 1 ? 1 : 4;  // pass 2: S'x, Svx, S'y, Svy (dW = C/D from pass 1)
  constexpr int NP = ZL / 2;
  constexpr int tile = TILE;  // particles per smem tile: kTileP, or kTileSmall (plan_gp)
  const uint32_t kTileBytes = sizeof(float) * tile * L::WIDTH;
  const int chunk = tile < kFlushP ? tile : kFlushP;
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t mbar[kPassStages];
  const int nthr = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, wz = nthr >> 5;
  float* recs = smem;                                            // [kPassStages][tile][WIDTH]
  float* psum = recs + kPassStages * tile * L::WIDTH;             // [2][wz][tile] (pass 2)
  // fp64 accumulators per lane slot in shared memory, [NQ*ZL][nthr] (conflict-free)
  double* out64 = reinterpret_cast<double*>(psum + (PASS == 2 ? 2 * wz * tile : 0));

  const int zb = blockIdx.y;
  const int slot0 = (zb * wz + warp) * (32 * ZL) + lane * ZL;
  // pass 2: state sums for the first js slot pairs of every lane (the index set I sits there)
  int js = 0;
  if (PASS == 2) {
    const int v = a.js == nullptr ? NP : *a.js;
    // kJsZBlock | b: all slot pairs of the first b z-blocks (CTA-uniform), none elsewhere
    // SPLIT (pass 2 of a per-warp layout, js_layout): the count of this warp
    js = (v & kJsZBlock) ? (zb < (v & (kJsZBlock - 1)) ? NP : 0)
                         : (SPLIT ? min(js_of_warp(v, zb * wz + warp), NP) : min(v, NP));
  }
  // one instance of the whole sweep per JS (pass 2: state sums for the first JS slot pairs
  // of every lane, where the index set I lives), so that each instance holds only the
  // per-lane constants it uses
  auto run = [&](auto js_tag) {
    constexpr int JS = decltype(js_tag)::value;
    constexpr bool FOLD = PASS == 2 && kFoldD;
    LaneZ<MODEL, PASS, NP, FOLD, JS> z;
    z.load(a, slot0);
    const float2 na0 = f2(a.na0, a.na0), na1 = f2(a.na1, a.na1), rbs = f2(a.rbs, a.rbs);
    // exponent form: range-bearing residuals are both in range units (residual()), so the
    // isotropic form with alpha_r applies
    constexpr int EM = MODEL == kRangeBearing ? kPosIso : MODEL;

    float2 in[NQ][NP];
  #pragma unroll
    for (int q = 0; q < NQ; ++q)
  #pragma unroll
      for (int j = 0; j < NP; ++j) in[q][j] = f2(0.0f, 0.0f);
  #pragma unroll
    for (int q = 0; q < NQ * ZL; ++q) out64[q * nthr + tid] = 0.0;

    const int64_t ntiles = (a.n + tile - 1) / tile;
    const int64_t t_begin = (int64_t)blockIdx.x * a.tiles_per_cta;
    const int64_t t_end = min(t_begin + a.tiles_per_cta, ntiles);

    // record tiles stream into shared memory by bulk copies (one thread issues them), a
    // tile of `tile` records per stage; the records of padding slots past n are zero with
    // log2(p_D c w) = -inf, so every term of theirs is exactly 0
    if (tid == 0) {
  #pragma unroll
      for (int s = 0; s < kPassStages; ++s) mbar_init(&mbar[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
  #pragma unroll
      for (int s = 0; s < kPassStages; ++s)
        if (t_begin + s < t_end) {
          mbar_arrive_expect_tx(&mbar[s], kTileBytes);
          bulk_g2s(recs + s * tile * L::WIDTH, a.rec + (t_begin + s) * tile * L::WIDTH, kTileBytes, &mbar[s]);
        }
    }

    for (int64_t t = t_begin; t < t_end; ++t) {
      const int it = (int)(t - t_begin);
      const int buf = it & 1;                   // psum double buffer
      const int stage = it % kPassStages;
      mbar_wait(&mbar[stage], (uint32_t)((it / kPassStages) & 1));
      const float* rb = recs + stage * tile * L::WIDTH;
      // per-slot sums of <= kFlushP particles in fp32 -> fp64; pass 2 only for the js
      // slot pairs that carry state sums (the F2F conversions share the XU pipe with EX2)
      auto flush64 = [&]() {
  #pragma unroll
        for (int q = 0; q < NQ; ++q)
  #pragma unroll
          for (int j = 0; j < NP; ++j) {
            if (PASS == 2 && j >= js) continue;
            out64[(q * ZL + 2 * j) * nthr + tid] += (double)in[q][j].x;
            out64[(q * ZL + 2 * j + 1) * nthr + tid] += (double)in[q][j].y;
            in[q][j] = f2(0.0f, 0.0f);
          }
      };

      // pass 2: state sums only in the first JS slot pairs of each lane, where the
      // index set I lives (uniform over the warp; one instance of the loop per JS)
  #pragma unroll 1
      for (int c0 = 0; c0 < tile; c0 += chunk) {
  #pragma unroll 1
      for (int p0 = c0; p0 < c0 + chunk; p0 += 8) {
        float pe[8];
  #pragma unroll(PASS == 1 ? kPPUnroll1 : kPPUnroll2)
        for (int pp = 0; pp < 8; ++pp) {
          const float* rec = rb + (p0 + pp) * L::WIDTH;
          const float4 P = *reinterpret_cast<const float4*>(rec);
          const float2 wv = f2(P.z, P.z);  // log2(p_D c w), both passes
          float2 pacc = f2(0.0f, 0.0f), pacc1 = f2(0.0f, 0.0f);
  #pragma unroll
          for (int j = 0; j < NP; ++j) {
            float2 d0, d1;
            residual(rec, P, z, j, d0, d1, rbs);
            if (PASS == 1) {
              // u = p_D g w = 2^(-alpha q + log2(p_D c w)), flushed to zero below 2^-126
              // exactly as in pass 2 (the same exponent bits; the polynomial-offloaded
              // terms differ from MUFU.EX2 by <= 3.2e-7 relative)
              const float2 e = expo<EM>(d0, d1, na0, na1, wv);
              constexpr int EP = MODEL == kRangeBearing ? kEmuPeriodRB : kEmuPeriod;
              const bool emu = EP > 0 && j == NP - 1 && pp % (EP > 0 ? EP : 1) == 0;
              in[0][j] = __fadd2_rn(in[0][j], emu ? ex2_poly(e) : ex2v(e));
            } else if (FOLD) {
              // u = p_D g w / (kappa + C_s): two interleaved FADD2 chains over the slot pairs
              const float2 u = ex2v(expo_fold<EM>(d0, d1, na0, na1, wv, z.d[j]));
              if (j == 0) pacc = u;
              else if (j == 1) pacc1 = u;
              else if (j & 1) pacc1 = __fadd2_rn(pacc1, u);
              else pacc = __fadd2_rn(pacc, u);
              if (j < JS && MODEL == kRangeBearing) {
                const float2 XY = *reinterpret_cast<const float2*>(rec + L::XY);
                d0 = __fadd2_rn(f2(XY.x, XY.x), z.c0[j]);  // x - centre_x
                d1 = __fadd2_rn(f2(XY.y, XY.y), z.c1[j]);  // y - centre_y
              }
              if (j < JS) {
                const float2 V = *reinterpret_cast<const float2*>(rec + L::V);
                in[0][j] = __ffma2_rn(u, d0, in[0][j]);
                in[1][j] = __ffma2_rn(u, f2(V.x, V.x), in[1][j]);
                in[2][j] = __ffma2_rn(u, d1, in[2][j]);
                in[3][j] = __ffma2_rn(u, f2(V.y, V.y), in[3][j]);
              }
            } else {
              const float2 u = ex2v(expo<EM>(d0, d1, na0, na1, wv));  // u = p_D g w
              pacc = __ffma2_rn(u, z.d[j], pacc);
              if (j < JS && MODEL == kRangeBearing) {
                const float2 XY = *reinterpret_cast<const float2*>(rec + L::XY);
                d0 = __fadd2_rn(f2(XY.x, XY.x), z.c0[j]);  // x - centre_x
                d1 = __fadd2_rn(f2(XY.y, XY.y), z.c1[j]);  // y - centre_y
              }
              if (j < JS) {
                const float2 V = *reinterpret_cast<const float2*>(rec + L::V);
                in[0][j] = __ffma2_rn(u, d0, in[0][j]);
                in[1][j] = __ffma2_rn(u, f2(V.x, V.x), in[1][j]);
                in[2][j] = __ffma2_rn(u, d1, in[2][j]);
                in[3][j] = __ffma2_rn(u, f2(V.y, V.y), in[3][j]);
              }
            }
          }
          if (FOLD && NP > 1) pacc = __fadd2_rn(pacc, pacc1);
          pe[pp] = pacc.x + pacc.y;
        }
        if (PASS == 2) {
          float s = transpose_reduce8(pe, lane);
          if ((lane & 3) == 0) psum[(buf * wz + warp) * tile + p0 + (lane >> 2)] = s;
        }
      }
      flush64();
      }
      __syncthreads();
      // every thread is done with this stage's records: refill it with tile t + kPassStages
      if (tid == 0 && t + kPassStages < t_end) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&mbar[stage], kTileBytes);
        bulk_g2s(recs + stage * tile * L::WIDTH, a.rec + (t + kPassStages) * tile * L::WIDTH, kTileBytes,
                 &mbar[stage]);
      }

      if (PASS == 2) {
        // per-particle partial over this CTA's slots: fixed-order sum over warps
        for (int p = tid; p < tile; p += nthr) {
          int64_t i = t * tile + p;
          if (i < a.n) {
            float s = 0.0f;
            for (int w2 = 0; w2 < wz; ++w2) s += psum[(buf * wz + w2) * tile + p];
            a.P[(int64_t)zb * a.P_stride + i] = s;
          }
        }
      }
    }
    const int64_t base = (int64_t)blockIdx.x * NQ * a.slots_pad;
    double* dst = PASS == 1 ? a.Cpart : a.Apart;
  #pragma unroll
    for (int q = 0; q < NQ; ++q)
  #pragma unroll
      for (int m = 0; m < ZL; ++m) dst[base + (int64_t)q * a.slots_pad + slot0 + m] = out64[(q * ZL + m) * nthr + tid];
  };
  if (PASS == 1 || js >= NP) run(std::integral_constant<int, NP>{});
  else if (js == 0) run(std::integral_constant<int, 0>{});
  else if (js == 1) run(std::integral_constant<int, 1>{});
  else if (NP > 2 && js == 2) run(std::integral_constant<int, (NP > 2 ? 2 : 1)>{});
  else run(std::integral_constant<int, (NP > 3 ? 3 : 1)>{});
}

template <int MODEL, int PASS, int ZL>
static size_t pass_smem(int wz, int tile) {
  using L = GRec<MODEL>;
  size_t b = sizeof(float) * kPassStages * tile * L::WIDTH;
  if (PASS == 2) b += sizeof(float) * 2 * wz * tile;
  b += sizeof(double) * (PASS == 1 ? 1 : 4) * ZL * wz * 32;
  return b;
}

template <int MODEL, int PASS, int ZL, int TILE, bool SPLIT>
static void set_attr() {
  ensure_max_smem(k_pass<MODEL, PASS, ZL, TILE, SPLIT>, pass_smem<MODEL, PASS, ZL>(max_warps_z(ZL), TILE));
}

// the tile size is a template parameter (a runtime tile costs 4.5% in cfg 5's pass 2)
template <int MODEL, int PASS, int ZL, int TILE, bool SPLIT>
static cudaError_t launch_tile(const PassArgs& a, int gp, int zb, int wz, cudaStream_t s) {
  set_attr<MODEL, PASS, ZL, TILE, SPLIT>();
  dim3 grid((unsigned)gp, (unsigned)zb);
  pdl_launch(k_pass<MODEL, PASS, ZL, TILE, SPLIT>, grid, wz * 32, pass_smem<MODEL, PASS, ZL>(wz, TILE), s, a);
  return cudaGetLastError();
}

template <int MODEL, int PASS, int ZL, int TILE>
static cudaError_t launch_split(const PassArgs& a, int gp, int zb, int wz, cudaStream_t s) {
  if (PASS == 2 && a.js_split) return launch_tile<MODEL, PASS, ZL, TILE, PASS == 2>(a, gp, zb, wz, s);
  return launch_tile<MODEL, PASS, ZL, TILE, false>(a, gp, zb, wz, s);
}

template <int MODEL, int PASS, int ZL>
static cudaError_t launch_one(const PassArgs& a, int gp, int zb, int wz, cudaStream_t s) {
  if (a.tile == kTileSmall) return launch_split<MODEL, PASS, ZL, kTileSmall>(a, gp, zb, wz, s);
  if (a.tile != kTileP) return cudaErrorInvalidValue;
  return launch_split<MODEL, PASS, ZL, kTileP>(a, gp, zb, wz, s);
}

template <int MODEL, int ZL>
static cudaError_t launch_m(int pass, const PassArgs& a, int gp, int zb, int wz, cudaStream_t s) {
  return pass == 1 ? launch_one<MODEL, 1, ZL>(a, gp, zb, wz, s) : launch_one<MODEL, 2, ZL>(a, gp, zb, wz, s);
}

template <int ZL>
static cudaError_t launch_z(int model, int pass, const PassArgs& a, int gp, int zb, int wz, cudaStream_t s) {
  if (model == kPosIso) return launch_m<kPosIso, ZL>(pass, a, gp, zb, wz, s);
  if (model == kPosAniso) return launch_m<kPosAniso, ZL>(pass, a, gp, zb, wz, s);
  return launch_m<kRangeBearing, ZL>(pass, a, gp, zb, wz, s);
}

bool pass2_sums_scaled() { return kFoldD; }

#ifndef PHD_REC_THREADS
#define PHD_REC_THREADS 1024
#endif
constexpr int kRecThreads = PHD_REC_THREADS;  // >= 256 (the block sums' threads)

// Per-particle records of the dense passes (GRec), once per update: HBM-bound, 20 B read
// and 32 B written per particle (range-bearing: 52 B read, 64 B written).  One float4 of
// the record per thread, so that a warp's stores are contiguous.  Slots [n, n_pad) get
// zero records with lw = -inf (their terms are exactly 0).  Block b covers the particles
// [b kBlockW, (b + 1) kBlockW) and, with blk != nullptr, also writes their fp64 weight sum
// blk[b] in k_block_sum's order (one launch fewer; the same bits).
template <int MODEL>
__global__ void __launch_bounds__(kRecThreads) k_records(const PassArgs a, int64_t n_pad, double* blk,
                                                         const BuildSlotsArgs bs) {
  pdl_wait();
  if (bs.slot_label != nullptr && blockIdx.x == gridDim.x - 1) {  // the slot layout's block
    build_slots_body(bs);
    return;
  }
  constexpr int Q = GRec<MODEL>::WIDTH / 4;  // float4 per record
  float4* out = reinterpret_cast<float4*>(a.rec);
  const int64_t base = (int64_t)blockIdx.x * kBlockW;
  const int64_t f0 = base * Q, f1 = min(n_pad, base + kBlockW) * Q;
  for (int64_t f = f0 + threadIdx.x; f < f1; f += blockDim.x) {
    const int64_t i = f / Q;
    const int q = (int)(f % Q);
    const bool ok = i < a.n;
    float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (MODEL == kRangeBearing) {
      if (q == 0) {
        v = ok ? make_float4(a.rb[i], a.rb[a.rb_stride + i], log2f(a.w[i] * a.wscale), 0.0f)
               : make_float4(0.0f, 0.0f, -INFINITY, 0.0f);
      } else if (ok && q == 1) {
        v = make_float4(a.rb[2 * a.rb_stride + i], a.rbs * a.rb[3 * a.rb_stride + i], a.rb[4 * a.rb_stride + i],
                        a.rbs * a.rb[5 * a.rb_stride + i]);
      } else if (ok && q == 2) {
        v = make_float4(a.rb[6 * a.rb_stride + i], a.rbs * a.rb[7 * a.rb_stride + i], a.x[i], a.y[i]);
      } else if (ok) {
        v = make_float4(a.vx[i], a.vy[i], 0.0f, 0.0f);
      }
    } else {
      if (q == 0)
        v = ok ? make_float4(a.x[i], a.y[i], log2f(a.w[i] * a.wscale), 0.0f) : make_float4(0.0f, 0.0f, -INFINITY, 0.0f);
      else if (ok)
        v = make_float4(a.vx[i], a.vy[i], 0.0f, 0.0f);
    }
    out[f] = v;
  }
  if (blk != nullptr && base < a.n) {  // block-uniform; the first 256 threads, k_block_sum's order
    __shared__ double sw[8];
    const int tid = threadIdx.x;
    double s = 0.0;
    if (tid < 256) {
#pragma unroll
      for (int r = 0; r < kBlockW / 256; ++r) {
        const int64_t i = base + r * 256 + tid;
        if (i < a.n) s += (double)a.w[i];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((tid & 31) == 0) sw[tid >> 5] = s;
    }
    __syncthreads();
    if (tid == 0) {
      double x = 0.0;
      for (int k = 0; k < 8; ++k) x += sw[k];
      blk[blockIdx.x] = x;
    }
  }
}

int record_width(int model) { return model == kRangeBearing ? GRec<kRangeBearing>::WIDTH : GRec<kPosIso>::WIDTH; }

cudaError_t launch_records(int model, const PassArgs& a, cudaStream_t s, double* blk, const BuildSlotsArgs* bs) {
  const int64_t n_pad = (a.n + kTileP - 1) / kTileP * kTileP;
  if (n_pad <= 0 && bs == nullptr) return cudaSuccess;
  static_assert(kBlockW == 4 * 256, "k_records' block sums follow k_block_sum's order");
  const BuildSlotsArgs b = bs ? *bs : BuildSlotsArgs{};
  const unsigned grid = (unsigned)((std::max<int64_t>(n_pad, 0) + kBlockW - 1) / kBlockW) + (bs ? 1u : 0u);
  if (model == kRangeBearing)
    pdl_launch(k_records<kRangeBearing>, grid, kRecThreads, 0, s, a, n_pad, blk, b);
  else
    pdl_launch(k_records<kPosIso>, grid, kRecThreads, 0, s, a, n_pad, blk, b);
  return cudaGetLastError();
}

cudaError_t launch_pass(int model, int pass, const PassArgs& a, int gp, int zb, int wz, int zl, cudaStream_t s) {
  if (gp <= 0 || zb <= 0) return cudaSuccess;
  return zl == 8 ? launch_z<8>(model, pass, a, gp, zb, wz, s) : launch_z<4>(model, pass, a, gp, zb, wz, s);
}

template <int MODEL, int PASS, int ZL>
static int occ_one(int wz) {
  set_attr<MODEL, PASS, ZL, kTileP, false>();
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_pass<MODEL, PASS, ZL, kTileP, false>, wz * 32,
                                                pass_smem<MODEL, PASS, ZL>(wz, kTileP));
  return n;
}

template <int ZL>
static int occ_z(int model, int pass, int wz) {
  if (model == kPosIso) return pass == 1 ? occ_one<kPosIso, 1, ZL>(wz) : occ_one<kPosIso, 2, ZL>(wz);
  if (model == kPosAniso) return pass == 1 ? occ_one<kPosAniso, 1, ZL>(wz) : occ_one<kPosAniso, 2, ZL>(wz);
  return pass == 1 ? occ_one<kRangeBearing, 1, ZL>(wz) : occ_one<kRangeBearing, 2, ZL>(wz);
}

// cached per (device, model, pass, zl, wz): asked once, not every update (a runtime call
// per query costs host time on the small configs' critical path)
int pass_occupancy(int model, int pass, int wz, int zl) {
  static std::atomic<int> cache[16][3][2][2][kMaxWarpsZ + 1];
  int dev = 0;
  cudaGetDevice(&dev);
  const bool cacheable = dev >= 0 && dev < 16 && model >= 0 && model < 3 && (pass == 1 || pass == 2) &&
                         wz >= 0 && wz <= kMaxWarpsZ;
  if (cacheable) {
    const int v = cache[dev][model][pass - 1][zl == 8][wz].load(std::memory_order_relaxed);
    if (v > 0) return v;
  }
  const int v = zl == 8 ? occ_z<8>(model, pass, wz) : occ_z<4>(model, pass, wz);
  if (cacheable && v > 0) cache[dev][model][pass - 1][zl == 8][wz].store(v, std::memory_order_relaxed);
  return v;
}

// C_slot[s] = sum over particle-CTAs (fixed order) of the pass-1 partials (fp64),
// for the slot range [s0, s1) (one measurement group).
// zc != nullptr (one rank: no all-reduce between): also the per-slot constants of k_zconst.
__global__ void k_reduce_C(const double* __restrict__ Cpart, int gp, int slots_pad, int s0, int s1,
                           double* C_slot, const double* __restrict__ wblk, int nwb, double* wout, ZConstArgs zc) {
  pdl_wait();
  if (wblk != nullptr && blockIdx.x == gridDim.x - 1) {  // the rank's W_pred (rides in C1)
    block_sum_f64(wblk, nwb, wout);
    return;
  }
  // one warp per slot, lanes over the particle-CTA partials, fixed-order xor tree
  const int lane = threadIdx.x & 31;
  int s = s0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= s1) return;
  double c = 0.0;
  // batches of 8 predicated loads in flight per lane (the partials were just written:
  // L2-latency bound); the sum keeps the order b = lane, lane + 32, ... (+0 is exact)
  for (int b0 = lane; b0 < gp; b0 += 32 * 8) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int b = b0 + 32 * r;
      v[r] = b < gp ? Cpart[(int64_t)b * slots_pad + s] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) c += v[r];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) {
    C_slot[s] = c;
    if (zc.slot_label) zconst_one(zc, s, c);
  }
}

cudaError_t launch_reduce_C(const double* Cpart, int gp, int slots_pad, int s0, int s1, double* C_slot,
                            cudaStream_t s, const double* wblk, int nwb, double* wout, const ZConstArgs* zc) {
  const int blocks = (std::max(s1 - s0, 0) + 7) / 8 + (wblk ? 1 : 0);
  if (blocks == 0) return cudaSuccess;
  const ZConstArgs z = zc ? *zc : ZConstArgs{};
  pdl_launch(k_reduce_C, blocks, 256, 0, s, Cpart, gp, slots_pad, s0, s1, C_slot, wblk, nwb, wout, z);
  return cudaGetLastError();
}

// For slots [s0, s1) of one group, with C_slot global (after the C1 all-reduce):
// D = kappa + C, per-slot d = 1/D as fp32 (0 when D == 0 or padding), and the
// label-order copies C_lab, D_lab used by the STPHD reduction and the getters.
__global__ void k_zconst(const double* __restrict__ C_slot, int s0, int s1, ZConstArgs zc,
                         const double* __restrict__ wpred) {
  pdl_wait();
  if (wpred != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && !isfinite(*wpred)) atomicAdd(zc.bad, 1);
  int s = s0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= s1) return;
  zconst_one(zc, s, C_slot[s]);
}

cudaError_t launch_zconst(const double* C_slot, const int32_t* slot_label, int s0, int s1, double kappa,
                          float* d_slot, double* C_lab, double* D_lab, int* bad, cudaStream_t s,
                          const double* wpred) {
  if (s1 <= s0) return cudaSuccess;
  ZConstArgs zc{slot_label, kappa, d_slot, C_lab, D_lab, bad};
  pdl_launch(k_zconst, (s1 - s0 + 255) / 256, 256, 0, s, C_slot, s0, s1, zc, wpred);
  return cudaGetLastError();
}

// w'_i = w_i [ (1 - p_D) + p_D c sum_zb P[zb][i] ]  (Eq 8 / Eq 15); fp64 block sums
// of w' and of the predicted w (blocks of kBlockW particles, fixed tree order).
__global__ void __launch_bounds__(256) k_finalize(const float* __restrict__ w, const float* __restrict__ P,
                                                  int64_t P_stride, int zb, int64_t n, float nu, float wscale,
                                                  float* w_out, double* blk_w, double* blk_wp,
                                                  const int32_t* __restrict__ inv) {
  pdl_wait();
  __shared__ double sw[8], swp[8];
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kBlockW;
  double a = 0.0, b = 0.0;
  constexpr int R = kBlockW / 256;
  if (PHD_FIN_STAGE && inv != nullptr && base + kBlockW <= n) {
    // gated update, full block: the R index loads, then the R gathers of P through inv, in
    // flight together (the gather is the latency chain of this kernel)
    float wi[R], s[R];
    int32_t j[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      j[r] = inv[base + r * 256 + tid];
      wi[r] = w[base + r * 256 + tid];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = zb > 0 ? P[j[r]] : 0.0f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float wn = wi[r] * nu + s[r];
      w_out[base + r * 256 + tid] = wn;
      a += (double)wn;
      b += (double)wi[r];
    }
  } else {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int64_t i = base + r * 256 + tid;
    if (i < n) {
      float wi = w[i];
      float s = 0.0f;
      if (inv) {
        if (zb > 0) s = P[inv[i]];  // gated update: one plane in sorted order
      } else {
        for (int k = 0; k < zb; ++k) s += P[(int64_t)k * P_stride + i];
      }
      float wn = wi * nu + s;  // P carries p_D c w (pass 2 folds log2 w into the exponent)
      w_out[i] = wn;
      a += (double)wn;
      b += (double)wi;
    }
  }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((tid & 31) == 0) {
    sw[tid >> 5] = a;
    swp[tid >> 5] = b;
  }
  __syncthreads();
  if (tid == 0) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < 8; ++k) {
      x += sw[k];
      y += swp[k];
    }
    blk_w[blockIdx.x] = x;
    blk_wp[blockIdx.x] = y;
  }
}

cudaError_t launch_finalize(const float* w, const float* P, int64_t P_stride, int zb, int64_t n, float nu,
                             float wscale, float* w_out, double* blk_w, double* blk_wp, cudaStream_t s,
                             const int32_t* inv) {
  if (n <= 0) return cudaSuccess;
  unsigned nb = (unsigned)((n + kBlockW - 1) / kBlockW);
  pdl_launch(k_finalize, nb, 256, 0, s, w, P, P_stride, zb, n, nu, wscale, w_out, blk_w, blk_wp, inv);
  return cudaGetLastError();
}

#ifndef PHD_RACC_UNROLL
#define PHD_RACC_UNROLL 4
#endif
constexpr int kRaccUnroll = PHD_RACC_UNROLL;

// STPHD accumulators in label order (Eqs 16, 18):
//   dW = C / D  (Eq 16 summed over i is exactly C_p/(kappa + C_p), the north_star identity),
//   Sx = A0 / D + cx dW,  Svx = A1 / D,  Sy = A2 / D + cy dW,  Svy = A3 / D
// with (cx, cy) the centre the kernel subtracted (the measurement itself for
// the position sensor).  The last CTA reduces the per-block masses into this
// rank's W_r and W_pred_r and writes them into the all-reduce buffer.
__global__ void k_reduce_acc(const double* __restrict__ Apart, int gp, int slots_pad, int n_slots,
                             const int32_t* __restrict__ slot_label, const double* __restrict__ C_lab,
                             const double* __restrict__ D_lab, const float* __restrict__ s0,
                             const float* __restrict__ s1, const float* __restrict__ s2,
                             const float* __restrict__ s3, int model, const double* __restrict__ blk_w,
                             const double* __restrict__ blk_wp, int nb, double* acc_lab, double* rank_slots,
                             int rank, int world, int lead, const int32_t* __restrict__ sel_flag,
                             int sums_scaled, double n_local) {
  pdl_wait();
  if (blockIdx.x == gridDim.x - 1) {
    __shared__ double sa[256], sb[256];
    double a = 0.0, b = 0.0;
    // eight loads of each array in flight per round (one round trip each, not one
    // per element); the sums keep the element order k = tid, tid + 256, ...
    for (int k0 = threadIdx.x; k0 < nb; k0 += 8 * (int)blockDim.x) {
      double va[8], vb[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int k = k0 + r * (int)blockDim.x;
        va[r] = k < nb ? blk_w[k] : 0.0;
        vb[r] = k < nb ? blk_wp[k] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        a += va[r];
        b += vb[r];
      }
    }
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) {
        sa[threadIdx.x] += sa[threadIdx.x + o];
        sb[threadIdx.x] += sb[threadIdx.x + o];
      }
      __syncthreads();
    }
    for (int r = threadIdx.x; r < 3 * world; r += blockDim.x) rank_slots[r] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      rank_slots[rank] = sa[0];
      rank_slots[world + rank] = sb[0];
      rank_slots[2 * world + rank] = n_local;  // N_r (the all-reduce sums N)
    }
    return;
  }
  // one warp per slot: lanes stride over the particle-CTA partials, fixed-order
  // xor tree (deterministic); the last block handles the rank masses above
  const int lane = threadIdx.x & 31;
  int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= n_slots) return;
  int lab = slot_label[s];
  if (lab < 0) return;
  // state sums outside the index set I were not accumulated: their partials are not read
  const bool sums = sel_flag == nullptr || sel_flag[lab] != 0;
  double A[4] = {0, 0, 0, 0};
  // batches of kRaccUnroll x 4 predicated loads in flight per lane (L2-latency bound: the
  // partials were just written by pass 2); the sums keep the order b = lane, lane + 32, ...
  for (int b0 = sums ? lane : gp; b0 < gp; b0 += 32 * kRaccUnroll) {
    double v[kRaccUnroll][4];
#pragma unroll
    for (int r = 0; r < kRaccUnroll; ++r) {
      const int b = b0 + 32 * r;
      const double* p = Apart + (int64_t)b * 4 * slots_pad + s;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[r][q] = b < gp ? p[(int64_t)q * slots_pad] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < kRaccUnroll; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) A[q] += v[r][q];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) A[q] += __shfl_xor_sync(0xffffffffu, A[q], o);
  if (lane != 0) return;
  double D = D_lab[lab];
  double inv = D > 0.0 ? 1.0 / D : 0.0;
  double cx, cy;
  if (model == kRangeBearing) {
    cx = -(double)s2[s];
    cy = -(double)s3[s];
  } else {
    cx = -(double)s0[s];
    cy = -(double)s1[s];
  }
  // C (hence dW) is already global: only rank 0 contributes the dW and centre
  // terms, every rank its own centred partial sums (the C2 all-reduce adds them).
  double dW = lead ? C_lab[lab] * inv : 0.0;
  double* o = acc_lab + 5 * (int64_t)lab;
  if (!sums) {
    o[0] = dW;
    o[1] = o[2] = o[3] = o[4] = 0.0;
    return;
  }
  // sums_scaled: the dense pass 2 folded 1/D into its terms (expo_fold)
  const double sc = sums_scaled ? 1.0 : inv;
  o[0] = dW;
  o[1] = A[0] * sc + cx * dW;
  o[2] = A[1] * sc;
  o[3] = A[2] * sc + cy * dW;
  o[4] = A[3] * sc;
}

cudaError_t launch_reduce_acc(const double* Apart, int gp, int slots_pad, int n_slots, const int32_t* slot_label,
                              const double* C_lab, const double* D_lab, const float* s0, const float* s1,
                              const float* s2, const float* s3, int model, const double* blk_w, const double* blk_wp,
                              int nb, double* acc_lab, double* rank_slots, int rank, int world, int lead,
                              const int32_t* sel_flag, cudaStream_t s, int sums_scaled, double n_local) {
  int blocks = (n_slots + 7) / 8 + 1;  // 8 slots (warps) per block + the rank-mass block
  pdl_launch(k_reduce_acc, blocks, 256, 0, s, Apart, gp, slots_pad, n_slots, slot_label, C_lab, D_lab, s0, s1, s2, s3, model,
                                      blk_w, blk_wp, nb, acc_lab, rank_slots, rank, world, lead, sel_flag, sums_scaled,
             n_local);
  return cudaGetLastError();
}


template <int MODEL>
static void preload_model() {
  touch_kernels(k_pass<MODEL, 1, 4, kTileP, false>, k_pass<MODEL, 1, 4, kTileSmall, false>,
                k_pass<MODEL, 1, 8, kTileP, false>, k_pass<MODEL, 1, 8, kTileSmall, false>,
                k_pass<MODEL, 2, 4, kTileP, false>, k_pass<MODEL, 2, 4, kTileSmall, false>,
                k_pass<MODEL, 2, 8, kTileP, false>, k_pass<MODEL, 2, 8, kTileSmall, false>,
                k_pass<MODEL, 2, 4, kTileP, true>, k_pass<MODEL, 2, 4, kTileSmall, true>,
                k_pass<MODEL, 2, 8, kTileP, true>, k_pass<MODEL, 2, 8, kTileSmall, true>);
}
void preload_update() {
  preload_model<kPosIso>();
  preload_model<kPosAniso>();
  preload_model<kRangeBearing>();
  touch_kernels(k_records<kPosIso>, k_records<kRangeBearing>, k_reduce_C, k_zconst, k_finalize, k_reduce_acc);
}

}  // namespace phd
