// Block-wide top-K selection for the STPHD index set (reading
// S8: order (dW desc, label asc), only dW > 0 eligible).  One CTA of 1024
// threads, M <= 8192 keys in shared memory.  Keys are the fp64 bits of dW >= 0
// (monotone in dW); 0 marks an ineligible label.  A most-significant-digit
// radix select (up to 8 passes of 8 bits) finds the K-th largest key T and how many
// keys equal to T are taken (the lowest labels first), replacing a full bitonic
// sort of all M labels.  It stops early once the digit bucket holding the K-th key
// holds exactly the keys still to take: then T is that bucket's prefix, compared
// under the returned mask, and every nonzero key matching it is taken.
#pragma once
#include <stdint.h>
#include <stdlib.h>

namespace phd {

constexpr int kTopkThreads = 1024;

// Block size of the one-CTA label kernels for M labels: one label per thread up to
// kTopkThreads, at least 128 threads (fewer warps: cheaper barriers for small M).
// PHD_TOPK_THREADS forces a size (A/B runs).
inline int topk_block(int M) {
  static const int forced = [] {
    const char* e = getenv("PHD_TOPK_THREADS");
    return e && *e ? atoi(e) : 0;
  }();
  if (forced >= 32 && forced <= kTopkThreads && forced % 32 == 0) return forced;
  int t = (M + 127) / 128 * 128;
  return t < 128 ? 128 : (t > kTopkThreads ? kTopkThreads : t);
}

struct TopkShared {
  int hist[256];
  int wsum[32];
  unsigned long long prefix;
  int k;
  int carry;
  int done;
};

// T = K-th largest nonzero key of kw[0..M) under *mask_out (the top bits examined),
// keq = number of nonzero keys with (key & mask) == T among the K taken (every nonzero
// key with (key & mask) > T is taken).  Requires 1 <= K <= #nonzero keys.
__device__ inline void topk_threshold(const unsigned long long* kw, int M, int K, TopkShared& sh,
                                      unsigned long long* T, int* keq, unsigned long long* mask_out) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    sh.prefix = 0ull;
    sh.k = K;
    sh.done = 0;
  }
  unsigned long long mask = 0ull;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) sh.hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sh.prefix;
    for (int i = tid; i < M; i += blockDim.x) {
      const unsigned long long key = kw[i];
      if (key != 0ull && (key & mask) == prefix) atomicAdd(&sh.hist[(int)((key >> shift) & 255ull)], 1);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l holds the 8 digits 255 - 8l .. 248 - 8l (descending)
      int c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = sh.hist[255 - 8 * lane - j];
        s += c[j];
      }
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int k = sh.k;
      __syncwarp();  // every lane has read k before the owning lane rewrites it
      const int before = incl - s;
      const bool mine = before < k && k <= incl;
      if (mine) {
        int cum = before;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + c[j] >= k) {
            sh.prefix = prefix | ((unsigned long long)(255 - 8 * lane - j) << shift);
            sh.k = k - cum;
            sh.done = cum + c[j] == k;  // the bucket holds exactly the keys still to take
            break;
          }
          cum += c[j];
        }
      }
    }
    mask |= 255ull << shift;
    __syncthreads();
    if (sh.done) break;  // uniform: read after the barrier
  }
  *T = sh.prefix;
  *keq = sh.k;
  *mask_out = mask;
  __syncthreads();
}

// Exclusive prefix count of flag over the index order i = r * blockDim + tid
// (round r); returns the count before i; sh.carry is advanced by the caller's
// rounds.  All threads of the block must call it the same number of times.
__device__ inline int topk_round_scan(bool flag, TopkShared& sh, int* round_total) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) sh.wsum[warp] = __popc(bal);
  __syncthreads();
  int off = 0, tot = 0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) {
    const int c = sh.wsum[w];
    if (w < warp) off += c;
    tot += c;
  }
  __syncthreads();
  *round_total = tot;
  return off + __popc(bal & ((1u << lane) - 1u));
}

}  // namespace phd
