// STPHD local estimation on the central unit (rank 0):
// W = sum_r W_r, LT = round(W) (half away from zero, S7), labels with
// dW > 0 sorted by (dW desc, label asc) (S8), zeta_l = S_l / dW_l (Eq 18, S9),
// undetected mass (1 - p_D) W_pred (Eq 17).  One CTA; bitonic sort in shared
// memory over the next power of two >= M (M <= 8192).
#include "phd_internal.h"

namespace phd {

struct EstOut {
  int32_t label;
  float state[4];
  float mass;
};

__device__ __forceinline__ bool before(double wa, int la, double wb, int lb) {
  return wa > wb || (wa == wb && la < lb);
}

__global__ void __launch_bounds__(1024) k_extract(const double* __restrict__ acc, int M, int n2,
                                                  const double* __restrict__ Wv, const double* __restrict__ Wpv,
                                                  int count, double p_d, EstOut* est, int cap, double* summary,
                                                  int32_t* count_out, const double* sel_info) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* kw = reinterpret_cast<double*>(sm);
  int* kl = reinterpret_cast<int*>(kw + n2);
  __shared__ int n_elig;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (tid == 0) n_elig = 0;
  __syncthreads();
  int cnt = 0;
  for (int i = tid; i < n2; i += nthr) {
    double w = -1.0;
    if (i < M) {
      w = acc[5 * (int64_t)i];
      if (w > 0.0) ++cnt; else w = -1.0;
    }
    kw[i] = w;
    kl[i] = i;
  }
  if (cnt) atomicAdd(&n_elig, cnt);
  __syncthreads();
  // bitonic sort, order = before()
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < n2; i += nthr) {
        int p = i ^ j;
        if (p > i) {
          bool up = (i & k) == 0;
          double wi = kw[i], wp = kw[p];
          int li = kl[i], lp = kl[p];
          bool swap = up ? before(wp, lp, wi, li) : before(wi, li, wp, lp);
          if (swap) {
            kw[i] = wp;
            kw[p] = wi;
            kl[i] = lp;
            kl[p] = li;
          }
        }
      }
      __syncthreads();
    }
  }
  __shared__ int snsel;
  if (tid == 0) {
    double W = 0.0, Wp = 0.0;
    for (int r = 0; r < count; ++r) {
      W += Wv[r];
      Wp += Wpv[r];
    }
    long long LT = (long long)floor(W + 0.5);
    if (sel_info) LT = (long long)sel_info[1];  // the index set of k_select (mass identity W)
    if (LT < 0) LT = 0;
    long long nsel = LT < n_elig ? LT : n_elig;
    if (nsel > cap) nsel = cap;
    snsel = (int)nsel;
    double frac = W - floor(W);
    summary[0] = W;
    summary[1] = Wp;
    summary[2] = (1.0 - p_d) * Wp;
    summary[3] = (double)LT;
    summary[4] = (double)n_elig;
    summary[5] = (double)nsel;
    summary[6] = LT > n_elig ? 1.0 : 0.0;
    summary[7] = fabs(frac - 0.5) < 1e-4 * fmax(1.0, W) ? 1.0 : 0.0;
    if (count_out) *count_out = (int32_t)nsel;
  }
  __syncthreads();
  for (int s = tid; s < snsel; s += nthr) {
    int l = kl[s];
    const double* a = acc + 5 * (int64_t)l;
    double dW = a[0];
    EstOut e;
    e.label = l;
    e.mass = (float)dW;
    for (int c = 0; c < 4; ++c) e.state[c] = (float)(a[1 + c] / dW);
    est[s] = e;
  }
}

cudaError_t launch_extract(const double* acc_lab, int M, const double* W, const double* Wp, int count, double p_d,
                           void* est, int cap, double* summary, int32_t* count_out, const double* sel_info,
                           cudaStream_t s) {
  int n2 = 1;
  while (n2 < M) n2 <<= 1;
  size_t smem = (size_t)n2 * (sizeof(double) + sizeof(int));
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_extract, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 12);
    attr_set = true;
  }
  k_extract<<<1, 1024, smem, s>>>(acc_lab, M, n2, W, Wp, count, p_d, reinterpret_cast<EstOut*>(est), cap, summary,
                                  count_out, sel_info);
  return cudaGetLastError();
}

}  // namespace phd
