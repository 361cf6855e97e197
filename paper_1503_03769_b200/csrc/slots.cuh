// Pass-1 slot layout body (one CTA), shared by k_build_slots (k_select.cu) and the
// records kernel's extra block (k_update.cu, dense path: one launch fewer).
#pragma once
#include "phd_internal.h"

namespace phd {

// Pass-1 slot layout on the device (one CTA; replaces the host layout and its copy):
// identity (position sensor, gated path: slot = label), or, range-bearing, the labels
// grouped by bearing class 0, 1, 2 (label order inside, every class padded to an even
// count so each f32x2 slot pair is class-homogeneous); slots past the sequence are
// padding (-1).  Then the per-slot constants.  M from *Mp when given
// (graph replays), else M.
__device__ __forceinline__ void build_slots_body(const BuildSlotsArgs& a) {
  const float* __restrict__ z = a.z;
  const int* Mp = a.Mp;
  const int M_arg = a.M;
  const int model = a.model, identity = a.identity, slots_pad = a.slots_pad;
  int32_t* slot_label = a.slot_label;
  const float sx = a.sx, sy = a.sy;
  const SlotConsts& sc = a.sc;
  int* bad = a.bad;
  float* zcopy = a.zcopy;
  __shared__ int wsum[32];
  __shared__ int base_s;
  const int M = Mp ? *Mp : M_arg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  if (zcopy)  // later kernels read Z from zcopy; this one reads the source
    for (int i = tid; i < 2 * M; i += nthr) zcopy[i] = z[i];
  const float hp = 1.57079632679489662f;
  if (identity || model != kRangeBearing) {
    for (int s = tid; s < slots_pad; s += nthr) slot_label[s] = s < M ? s : -1;
  } else {
    const int per = (M + nthr - 1) / nthr;
    for (int s = tid; s < slots_pad; s += nthr) slot_label[s] = -1;
    if (tid == 0) base_s = 0;
    __syncthreads();
    for (int cls_want = 0; cls_want < 3; ++cls_want) {
      int c = 0;
      for (int q = 0; q < per; ++q) {
        const int l = tid * per + q;
        if (l >= M) break;
        const float t = z[2 * l + 1];
        const int cls = t > hp ? 1 : (t < -hp ? 2 : 0);
        c += cls == cls_want;
      }
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const int v = lane < nthr / 32 ? wsum[lane] : 0;
        int inc2 = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, inc2, o);
          if (lane >= o) inc2 += u;
        }
        if (lane < nthr / 32) wsum[lane] = inc2 - v;
      }
      __syncthreads();
      int pos = base_s + wsum[warp] + (incl - c);
      for (int q = 0; q < per; ++q) {
        const int l = tid * per + q;
        if (l >= M) break;
        const float t = z[2 * l + 1];
        const int cls = t > hp ? 1 : (t < -hp ? 2 : 0);
        if (cls == cls_want) slot_label[pos++] = l;
      }
      __syncthreads();
      if (tid == nthr - 1) {
        int total = base_s + wsum[warp] + incl;
        base_s = total + (total & 1);  // pair padding (slot stays -1)
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int s = tid; s < slots_pad; s += nthr) {
    const int lab = slot_label[s];
    float s0 = -1e30f, s1 = -1e30f, s2 = 0.0f, s3 = 0.0f;
    int rep = 0;
    if (lab >= 0) {
      const float z0 = z[2 * lab], z1 = z[2 * lab + 1];
      // a NaN measurement makes its dense C NaN (PHD_EMODEL); counted here because the
      // gated update may give it no candidate at all
      if (bad != nullptr && (z0 != z0 || z1 != z1)) atomicAdd(bad, 1);
      s0 = -z0;
      s1 = -z1;
      if (model == kRangeBearing) {
        rep = (z1 > hp) ? 1 : ((z1 < -hp) ? 2 : 0);
        float sn, cs;
        sincosf(z1, &sn, &cs);
        s2 = -(sx + z0 * cs);
        s3 = -(sy + z0 * sn);
      }
    }
    sc.s0[s] = s0;
    sc.s1[s] = s1;
    if (sc.s2) {
      sc.s2[s] = s2;
      sc.s3[s] = s3;
    }
    if (sc.rep) sc.rep[s] = rep;
    sc.d[s] = 0.0f;
  }
}

}  // namespace phd
