// STPHD label selection before pass 2.
//
// After pass 1 the normalisers C are global, so every quantity the extraction
// needs is already known except the state sums:
//   dW_l = C_l / (kappa + C_l)            (Eq 16 summed over particles, exactly)
//   W    = (1 - p_D) W_pred + sum_l dW_l   (the mass identity of Eqs 8 / 15)
//   LT   = round(W), index set I = the LT largest dW (dW desc, label asc).
// Pass 2 then accumulates the weighted-state sums S_l (Eq 18) only for l in I
// -- the labels whose states the paper estimates -- in a
// slot layout that puts I first (on every lane's first slot pairs, or on whole
// z-blocks), so the choice is warp- or CTA-uniform.
#include "phd_internal.h"
#include "slots.cuh"
#include "topk.cuh"

#include <algorithm>

namespace phd {

// fp64 block sums of w (kBlockW per block); the rank total is summed by an extra
// block of the C reduction (block_sum_f64) so that it rides in the C1 all-reduce.
__global__ void __launch_bounds__(256) k_block_sum(const float* __restrict__ w, int64_t n, double* blk) {
  pdl_wait();
  __shared__ double sw[8];
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kBlockW;
  double a = 0.0;
#pragma unroll
  for (int r = 0; r < kBlockW / 256; ++r) {
    int64_t i = base + r * 256 + tid;
    if (i < n) a += (double)w[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((tid & 31) == 0) sw[tid >> 5] = a;
  __syncthreads();
  if (tid == 0) {
    double x = 0.0;
    for (int k = 0; k < 8; ++k) x += sw[k];
    blk[blockIdx.x] = x;
  }
}

cudaError_t launch_block_sums(const float* w, int64_t n, double* blk, cudaStream_t s) {
  int nb = (int)((n + kBlockW - 1) / kBlockW);
  if (nb > 0) pdl_launch(k_block_sum, nb, 256, 0, s, w, n, blk);
  return cudaGetLastError();
}

// One CTA.  sel_flag[l] = 1 for l in I; info = (W_id, LT, n_eligible, n_sel).
// I = the n_sel largest dW (ties: lowest labels), by radix select (topk.cuh).
__device__ __forceinline__ void select_body(const double* __restrict__ C_lab, const double* __restrict__ D_lab,
                                            int M, const double* __restrict__ W_pred, double p_d, int32_t* sel_flag,
                                            double* info, unsigned long long* kw) {
  __shared__ TopkShared sh;
  __shared__ double red[32];
  __shared__ int n_elig, snsel;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) n_elig = 0;
  __syncthreads();
  double part = 0.0;
  int cnt = 0;
  for (int i = tid; i < M; i += nthr) {
    const double D = D_lab[i];
    const double dW = C_lab[i] * (D > 0.0 ? 1.0 / D : 0.0);  // same arithmetic as k_reduce_acc
    part += dW;
    sel_flag[i] = 0;
    kw[i] = dW > 0.0 ? (unsigned long long)__double_as_longlong(dW) : 0ull;
    cnt += dW > 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  if (cnt) atomicAdd(&n_elig, cnt);
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < (nthr >> 5); ++w) sum += red[w];
    const double W = (1.0 - p_d) * (*W_pred) + sum;
    long long LT = (long long)floor(W + 0.5);
    if (LT < 0) LT = 0;
    const long long nsel = LT < n_elig ? LT : n_elig;
    snsel = (int)nsel;
    info[0] = W;
    info[1] = (double)LT;
    info[2] = (double)n_elig;
    info[3] = (double)nsel;
  }
  __syncthreads();
  const int nsel = snsel;
  if (nsel <= 0) return;  // uniform over the CTA
  unsigned long long T, mask;
  int keq;
  topk_threshold(kw, M, nsel, sh, &T, &keq, &mask);
  int carry = 0;
  for (int r = 0; r < M; r += nthr) {
    const int i = r + tid;
    const unsigned long long key = i < M ? kw[i] : 0ull;
    const bool eq = i < M && key != 0ull && (key & mask) == T;
    int tot;
    const int before = carry + topk_round_scan(eq, sh, &tot);
    if (i < M && key != 0ull && ((key & mask) > T || (eq && before < keq))) sel_flag[i] = 1;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kTopkThreads) k_select(const double* __restrict__ C_lab,
                                                         const double* __restrict__ D_lab, int M,
                                                         const double* __restrict__ W_pred, double p_d,
                                                         int32_t* sel_flag, double* info) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char sm[];
  select_body(C_lab, D_lab, M, W_pred, p_d, sel_flag, info, reinterpret_cast<unsigned long long*>(sm));
}

cudaError_t launch_select(const double* C_lab, const double* D_lab, int M, const double* W_pred, double p_d,
                          int32_t* sel_flag, double* info, cudaStream_t s) {
  size_t smem = (size_t)std::max(M, 1) * sizeof(unsigned long long);
  ensure_max_smem(k_select, 8192 * 8);
  pdl_launch(k_select, 1, topk_block(M), smem, s, C_lab, D_lab, M, W_pred, p_d, sel_flag, info);
  return cudaGetLastError();
}

// Pass-2 slot layout (one CTA).  Sequence = [selected labels | unselected labels],
// each part grouped by bearing class (range-bearing) and padded to even counts so
// that every f32x2 slot pair is class-homogeneous; labels ascending inside.  The
// sequence fills first the "state-sum" slots -- the first 2 jl slots of every lane and
// two more on every lane of the first n_hi warps, just enough for the selected labels
// (a lane-uniform count wasted up to a pair per lane: cfg 4, 1000 of 3100 labels
// selected, summed on 50 % of the slot pairs instead of 31 %) -- then the remaining slots.
// *js_out = jl | (n_hi << 8).
// Sequence position p -> slot.  The state-sum region: lanes of the first n_hi warps hold
// 2 (jl + 1) sequence slots each, the other lanes 2 jl (lane-major inside a lane); then the
// rest fills the remaining zl - 2 js(lane) slots of every lane in lane order.  jl < 0:
// whole-z-block layout (the sequence in slot order).
__device__ __forceinline__ int seq_slot(int p, int lanes, int zl, int jl, int n_hi) {
  if (jl < 0) return p;
  const int jh = jl + 1, lh = 32 * n_hi;  // lanes with jh pairs
  const int s_hi = 2 * jh * lh, n_s = s_hi + 2 * jl * (lanes - lh);
  if (p < n_s) {
    if (p < s_hi) return (p / (2 * jh)) * zl + p % (2 * jh);
    const int q = p - s_hi;
    return (lh + q / (2 * jl)) * zl + q % (2 * jl);
  }
  int q = p - n_s;
  const int rh = zl - 2 * jh, rl = zl - 2 * jl;
  if (rh > 0 && q < rh * lh) return (q / rh) * zl + 2 * jh + q % rh;
  q -= rh * lh;
  return (lh + q / rl) * zl + 2 * jl + q % rl;
}

__device__ __forceinline__ void slots2_body(const float* __restrict__ z, const int32_t* sel_flag, int M, int model,
                                            int zl, int wz, int layout, int slots_pad, int32_t* slot_label,
                                            int32_t* js_out, float sx, float sy, const SlotConsts& sc,
                                            const double* __restrict__ D_lab) {
  // categories 0-2: selected labels of bearing class 0, 1, 2; 3-5: the unselected ones
  // (position sensor: class 0 only).  Every thread owns a contiguous run of labels: one
  // counting pass, one block-wide scan of the six counts, one placement pass.
  constexpr int NC = 6;
  __shared__ int wsum[32][NC];
  __shared__ int cat_start[NC + 1];
  __shared__ int s_js, s_nhi;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x, nw = nthr >> 5;
  const int per = (M + nthr - 1) / nthr;
  const float hp = 1.57079632679489662f;
  const int lanes = slots_pad / zl;
  const bool rb = model == kRangeBearing;

  for (int s = tid; s < slots_pad; s += nthr) slot_label[s] = -1;
  auto cat_of = [&](int l) {
    int cls = 0;
    if (rb) {
      const float t = z[2 * l + 1];
      cls = t > hp ? 1 : (t < -hp ? 2 : 0);
    }
    return (sel_flag[l] != 0 ? 0 : 3) + cls;
  };
  int cnt[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) cnt[c] = 0;
  for (int q = 0; q < per; ++q) {
    const int l = tid * per + q;
    if (l >= M) break;
    const int c = cat_of(l);
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) cnt[cc] += c == cc;
  }
  // exclusive prefix of every count over the threads (warp shuffles, then the warp totals)
  int excl[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    int incl = cnt[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    excl[c] = incl - cnt[c];
    if (lane == 31) wsum[warp][c] = incl;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int v = lane < nw ? wsum[lane][c] : 0;
      int inc2 = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc2, o);
        if (lane >= o) inc2 += u;
      }
      if (lane < nw) wsum[lane][c] = inc2 - v;
      const int tot = __shfl_sync(0xffffffffu, inc2, 31);
      if (lane == 0) cat_start[c + 1] = tot;  // category total for now
    }
    if (lane == 0) {
      // category offsets in the sequence, each category padded to an even count
      // (range-bearing: class-homogeneous f32x2 slot pairs)
      int base = 0;
      for (int c = 0; c < NC; ++c) {
        const int tot = cat_start[c + 1];
        cat_start[c] = base;
        base += tot + (rb && (tot & 1) ? 1 : 0);
      }
      cat_start[NC] = base;
      // state-sum layout: js slot pairs on every lane, or whole z-blocks (CTA-uniform)
      // when that needs fewer state-sum slots: *js_out = kJsZBlock | zb_sum
      // per lane: jl slot pairs, one more on the lanes of the first n_hi warps (warp-
      // uniform), just enough for the n_sel selected slots (js_layout)
      const int n_sel = cat_start[3];
      int sum_slots;
      const int32_t enc = js_layout(n_sel, lanes, zl, true, &sum_slots);
      const int jl = enc & 0xFF, n_hi = (enc >> 8) & 0xFF;
      const int spz = wz * 32 * zl;
      const int zb_sum = (n_sel + spz - 1) / spz;
      if (layout == 2 || (layout == 0 && zb_sum * spz < sum_slots)) {
        *js_out = kJsZBlock | zb_sum;
        s_js = -1;
        s_nhi = 0;
      } else {
        *js_out = jl | (n_hi << 8);
        s_js = jl;
        s_nhi = n_hi;
      }
    }
  }
  __syncthreads();
  const int js = s_js, n_hi = s_nhi;
  int pos[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) pos[c] = cat_start[c] + wsum[warp][c] + excl[c];
  for (int q = 0; q < per; ++q) {
    const int l = tid * per + q;
    if (l >= M) break;
    const int c = cat_of(l);
    int p = 0;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
      if (c == cc) p = pos[cc]++;
    slot_label[seq_slot(p, lanes, zl, js, n_hi)] = l;
  }
  __syncthreads();
  // per-slot constants of the new layout (as k_build_slots) and d = 1/D (as k_zconst):
  // padding slots get the sentinel that makes every term exactly 0
  for (int s = tid; s < slots_pad; s += nthr) {
    const int lab = slot_label[s];
    float s0 = -1e30f, s1 = -1e30f, s2 = 0.0f, s3 = 0.0f, d = 0.0f;
    int rep = 0;
    if (lab >= 0) {
      const float z0 = z[2 * lab], z1 = z[2 * lab + 1];
      s0 = -z0;
      s1 = -z1;
      if (model == kRangeBearing) {
        rep = (z1 > hp) ? 1 : ((z1 < -hp) ? 2 : 0);
        float sn, cs;
        sincosf(z1, &sn, &cs);
        s2 = -(sx + z0 * cs);
        s3 = -(sy + z0 * sn);
      }
      const double D = D_lab[lab];
      d = D > 0.0 ? (float)fmin(1.0 / D, 3.0e38) : 0.0f;
    }
    sc.s0[s] = s0;
    sc.s1[s] = s1;
    if (sc.s2) {
      sc.s2[s] = s2;
      sc.s3[s] = s3;
    }
    if (sc.rep) sc.rep[s] = rep;
    sc.d[s] = d;
  }
}

// Pass-1 slot layout on the device (slots.cuh), one CTA.
__global__ void __launch_bounds__(kTopkThreads) k_build_slots(const BuildSlotsArgs a) {
  pdl_wait();
  build_slots_body(a);
}

cudaError_t launch_build_slots(const BuildSlotsArgs& a, cudaStream_t s) {
  if (a.slots_pad <= 0) return cudaSuccess;
  pdl_launch(k_build_slots, 1, topk_block(a.Mp ? a.slots_pad : a.M), 0, s, a);
  return cudaGetLastError();
}

// Dense path: the index set and the pass-2 layout in one CTA (one launch).
__global__ void __launch_bounds__(kTopkThreads) k_select_slots(const double* __restrict__ C_lab,
                                                               const double* __restrict__ D_lab, int M_arg,
                                                               const int* Mp,
                                                               const double* __restrict__ W_pred, double p_d,
                                                               int32_t* sel_flag, double* info,
                                                               const float* __restrict__ z, int model, int zl,
                                                               int wz, int layout, int slots_pad, int32_t* slot_label,
                                                               int32_t* js_out, float sx, float sy, SlotConsts sc) {
  pdl_wait();
  const int M = Mp ? *Mp : M_arg;  // graph replays: this step's M (shared memory sized for max_meas)
  extern __shared__ __align__(16) unsigned char sm[];
  select_body(C_lab, D_lab, M, W_pred, p_d, sel_flag, info, reinterpret_cast<unsigned long long*>(sm));
  __syncthreads();  // sel_flag (global) complete and visible to the CTA
  slots2_body(z, sel_flag, M, model, zl, wz, layout, slots_pad, slot_label, js_out, sx, sy, sc, D_lab);
}

cudaError_t launch_select_slots(const double* C_lab, const double* D_lab, int M, const double* W_pred, double p_d,
                                int32_t* sel_flag, double* info, const float* z, int model, int zl, int wz,
                                int layout, int slots_pad, int32_t* slot_label, int32_t* js, float sensor_x,
                                float sensor_y, SlotConsts sc, cudaStream_t s, const int* Mp, int M_alloc) {
  size_t smem = (size_t)std::max(Mp ? M_alloc : M, 1) * sizeof(unsigned long long);
  ensure_max_smem(k_select_slots, 8192 * 8);
  pdl_launch(k_select_slots, 1, topk_block(std::max(Mp ? M_alloc : M, slots_pad / 4)), smem, s, C_lab, D_lab, M, Mp, W_pred, p_d, sel_flag, info, z, model, zl,
             wz, layout, slots_pad, slot_label, js, sensor_x, sensor_y, sc);
  return cudaGetLastError();
}


void preload_select() { touch_kernels(k_block_sum, k_select, k_select_slots, k_build_slots); }

}  // namespace phd
