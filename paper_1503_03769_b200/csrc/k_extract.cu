// STPHD local estimation on the central unit (rank 0):
// W = sum_r W_r, LT = round(W) (half away from zero, S7), labels with
// dW > 0 sorted by (dW desc, label asc) (S8), zeta_l = S_l / dW_l (Eq 18, S9),
// undetected mass (1 - p_D) W_pred (Eq 17).  One CTA: radix select of the
// top-LT labels, bitonic sort of those (M <= 8192).
#include "phd_internal.h"
#include "topk.cuh"

#include <algorithm>

namespace phd {

struct EstOut {
  int32_t label;
  float state[4];
  float mass;
};

__device__ __forceinline__ bool before(double wa, int la, double wb, int lb) {
  return wa > wb || (wa == wb && la < lb);
}

// One CTA.  The n_sel = min(LT, eligible, cap) largest dW are found by radix
// select (topk.cuh), compacted in label order, then bitonic-sorted by (dW desc,
// label asc) -- n_sel (~ the target count) instead of all M labels.
__global__ void __launch_bounds__(kTopkThreads) k_extract(const double* __restrict__ acc, int M_arg, const int* Mp,
                                                          const double* __restrict__ Wv, const double* __restrict__ Wpv,
                                                          int count, double p_d, EstOut* est, int cap, double* summary,
                                                          int32_t* count_out, const double* sel_info,
                                                          const int32_t* __restrict__ sel_flag) {
  pdl_wait();
  const int M = Mp ? *Mp : M_arg;  // graph replays: this step's M (shared memory sized for max_meas)
  extern __shared__ __align__(16) unsigned char sm[];
  const int n2m = M <= 1 ? 1 : 1 << (32 - __clz(M - 1));  // next power of two >= M
  unsigned long long* kw = reinterpret_cast<unsigned long long*>(sm);
  double* cw = reinterpret_cast<double*>(kw + M);
  int* cl = reinterpret_cast<int*>(cw + n2m);
  __shared__ TopkShared sh;
  __shared__ int n_elig, snsel;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (tid == 0) n_elig = 0;
  __syncthreads();
  int cnt = 0;
  for (int i = tid; i < M; i += nthr) {
    const double w = acc[5 * (int64_t)i];
    kw[i] = w > 0.0 ? (unsigned long long)__double_as_longlong(w) : 0ull;
    cnt += w > 0.0;
  }
  if (cnt) atomicAdd(&n_elig, cnt);
  __syncthreads();
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
  const int nsel = snsel;
  if (nsel <= 0) return;
  // the index set I of k_select is exactly this top-nsel set when nsel is its size
  // (same keys: k_select and k_reduce_acc compute dW = C (1/D) alike): compact it
  // instead of selecting again
  const bool use_sel = sel_flag != nullptr && sel_info != nullptr && (double)nsel == sel_info[3];
  unsigned long long T = 0ull, mask = ~0ull;
  int keq = 0;
  if (!use_sel) topk_threshold(kw, M, nsel, sh, &T, &keq, &mask);
  // compact the selected labels in label order
  int carry = 0, carry_eq = 0;
  for (int r = 0; r < M; r += nthr) {
    const int i = r + tid;
    const unsigned long long key = i < M ? kw[i] : 0ull;
    const bool eq = !use_sel && i < M && key != 0ull && (key & mask) == T;
    int tot_eq;
    const int before_eq = carry_eq + topk_round_scan(eq, sh, &tot_eq);
    const bool take =
        i < M && (use_sel ? sel_flag[i] != 0 : key != 0ull && ((key & mask) > T || (eq && before_eq < keq)));
    int tot;
    const int pos = carry + topk_round_scan(take, sh, &tot);
    if (take) {
      cw[pos] = __longlong_as_double((long long)key);
      cl[pos] = i;
    }
    carry += tot;
    carry_eq += tot_eq;
  }
  int n2 = 1;
  while (n2 < nsel) n2 <<= 1;
  for (int i = nsel + tid; i < n2; i += nthr) {
    cw[i] = -1.0;
    cl[i] = 0x7fffffff;
  }
  __syncthreads();
  if (n2 <= nthr) {
    // one element per thread in registers: partner exchanges by shuffle for
    // j < 32, through shared memory above (labels are unique: before() is strict)
    double w = tid < n2 ? cw[tid] : -1.0;
    int l = tid < n2 ? cl[tid] : 0x7fffffff;
    for (int k = 2; k <= n2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        double pw;
        int pl;
        if (j >= 32) {
          __syncthreads();
          if (tid < n2) {
            cw[tid] = w;
            cl[tid] = l;
          }
          __syncthreads();
          pw = tid < n2 ? cw[tid ^ j] : -1.0;
          pl = tid < n2 ? cl[tid ^ j] : 0x7fffffff;
        } else {
          pw = __shfl_xor_sync(0xffffffffu, w, j);
          pl = __shfl_xor_sync(0xffffffffu, l, j);
        }
        const bool want_first = ((tid & j) == 0) == ((tid & k) == 0);
        const bool take = want_first ? before(pw, pl, w, l) : before(w, l, pw, pl);
        if (take && tid < n2) {
          w = pw;
          l = pl;
        }
      }
    }
    __syncthreads();
    if (tid < n2) {
      cw[tid] = w;
      cl[tid] = l;
    }
    __syncthreads();
  } else
  // bitonic sort of the n_sel selected in shared memory, order = before()
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < n2; i += nthr) {
        int p = i ^ j;
        if (p > i) {
          bool up = (i & k) == 0;
          double wi = cw[i], wp = cw[p];
          int li = cl[i], lp = cl[p];
          bool swap = up ? before(wp, lp, wi, li) : before(wi, li, wp, lp);
          if (swap) {
            cw[i] = wp;
            cw[p] = wi;
            cl[i] = lp;
            cl[p] = li;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int s = tid; s < nsel; s += nthr) {
    int l = cl[s];
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
                           const int32_t* sel_flag, cudaStream_t s, const int* Mp, int M_alloc) {
  const int Ms = Mp ? M_alloc : M;  // shared memory for the largest M the launch may see
  int n2 = 1;
  while (n2 < Ms) n2 <<= 1;
  size_t smem = (size_t)std::max(Ms, 1) * sizeof(unsigned long long) + (size_t)n2 * (sizeof(double) + sizeof(int));
  ensure_max_smem(k_extract, 8192 * 20);
  pdl_launch(k_extract, 1, topk_block(Ms), smem, s, acc_lab, M, Mp, W, Wp, count, p_d, reinterpret_cast<EstOut*>(est), cap,
             summary, count_out, sel_info, sel_flag);
  return cudaGetLastError();
}

// One CTA: the step's host-visible results into pinned host memory (StepOutArgs; UVA
// maps cudaMallocHost memory, so the host pointers are device pointers).  Stores only;
// the host reads them after the stream synchronisation that follows.
__global__ void __launch_bounds__(256) k_step_out(const StepOutArgs a) {
  pdl_wait();
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int i = tid; i < a.n_rslots; i += nthr) a.h_rslots[i] = a.rslots[i];
  if (tid < 2) a.h_bad[tid] = a.bad[tid];
  if (a.sel_info && tid < 4) a.h_sel[tid] = a.sel_info[tid];
  if (tid < 8) a.h_summ[tid] = a.summ[tid];
  // the estimates: 6 words each, as many as the extraction wrote (<= est_cap)
  const int n = a.est_count ? min(max(*a.est_count, 0), a.est_cap) : 0;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(a.est);
  uint32_t* dst = reinterpret_cast<uint32_t*>(a.h_est);
  for (int i = tid; i < 6 * n; i += nthr) dst[i] = src[i];
  if (a.ds) {
    const uint32_t* d0 = reinterpret_cast<const uint32_t*>(a.ds);
    uint32_t* d1 = reinterpret_cast<uint32_t*>(a.h_ds);
    for (int i = tid; i < (int)(sizeof(DevStep) / 4); i += nthr) d1[i] = d0[i];
  }
  __syncthreads();  // every thread has read bad before it is cleared
  if (tid < 4) a.bad[tid] = 0;
}

cudaError_t launch_step_out(const StepOutArgs& a, cudaStream_t s) {
  static_assert(sizeof(EstOut) == 24, "estimate layout");
  pdl_launch(k_step_out, 1, 256, 0, s, a);
  return cudaGetLastError();
}


void preload_extract() { touch_kernels(k_extract, k_step_out); }

}  // namespace phd
