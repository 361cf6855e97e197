// Counter-based noise for the CUDA path: Philox4x32-10 (Salmon et al., SC'11),
// host+device.  This is the product's own implementation; the oracle has an
// independent one.  Counter convention ("noise"):
// ctr = (g lo32, k, stream, g hi32), key = (seed lo32, seed hi32); streams:
// 1 predict, 2 birth, 3 resample offset U.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PHD_HD __host__ __device__ __forceinline__
#else
#define PHD_HD inline
#endif

namespace phd {

struct U4 { uint32_t x, y, z, w; };

PHD_HD void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if defined(__CUDA_ARCH__)
  hi = __umulhi(a, b);
  lo = a * b;
#else
  uint64_t p = (uint64_t)a * (uint64_t)b;
  hi = (uint32_t)(p >> 32);
  lo = (uint32_t)p;
#endif
}

PHD_HD U4 philox10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2511F53u, c.x, hi0, lo0);
    mulhilo(0xCD9E8D57u, c.z, hi1, lo1);
    U4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

PHD_HD U4 philox_at(uint64_t seed, uint64_t g, uint32_t k, uint32_t stream) {
  U4 c{(uint32_t)g, k, stream, (uint32_t)(g >> 32)};
  return philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
}

// ((w >> 9) + 0.5) * 2^-23: exact in fp32, in [2^-24, 1 - 2^-24].
PHD_HD float u01(uint32_t w) { return ((float)(w >> 9) + 0.5f) * 1.1920928955078125e-07f; }

// ((w0 >> 6) 2^26 + (w1 >> 6) + 0.5) 2^-52: exact in fp64.
PHD_HD double u52(uint32_t w0, uint32_t w1) {
  return ((double)(w0 >> 6) * 67108864.0 + (double)(w1 >> 6) + 0.5) * 2.220446049250313080847263336181640625e-16;
}

}  // namespace phd
