// Pipe-throughput microbenchmark for the B200 roofline of the PHD update
// kernels (FP32 scalar FFMA, packed FFMA2/FADD2/FMUL2, MUFU.EX2, F2F+DADD).
// Prints ops per SM per SM-clock. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ float ex2f(float x) {
  float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}

__global__ void k_ffma(float* out, float a, float b, long long* cyc) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3f + c;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = fmaf(v[c], a, b);
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 3-register FFMA (multiplier in a register that varies) to avoid imm-form
__global__ void k_ffma3(float* out, const float* ab, long long* cyc) {
  float a = ab[threadIdx.x & 31], b = ab[32 + (threadIdx.x & 31)];
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3f + c;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = fmaf(v[c], a, b);
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, const float* ab, long long* cyc) {
  float2 a = make_float2(ab[threadIdx.x & 31], ab[(threadIdx.x + 1) & 31]);
  float2 b = make_float2(ab[32 + (threadIdx.x & 31)], ab[32 + ((threadIdx.x + 3) & 31)]);
  float2 v[CH];
  for (int c = 0; c < CH; ++c) v[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __ffma2_rn(v[c], a, b);
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c].x + v[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_fadd2(float* out, const float* ab, long long* cyc) {
  float2 a = make_float2(ab[threadIdx.x & 31], ab[(threadIdx.x + 1) & 31]);
  float2 v[CH];
  for (int c = 0; c < CH; ++c) v[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __fadd2_rn(v[c], a);
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c].x + v[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2(float* out, long long* cyc) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = 0.5f + threadIdx.x * 1e-4f + c * 1e-3f;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = ex2f(-v[c]);
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// mixed: 1 EX2 + 3 FFMA2 per element pair (the pass-1 shape: 6 FP32 ops + 2 EX2 per 2 pairs)
__global__ void k_mix13(float* out, const float* ab, long long* cyc) {
  float2 a = make_float2(ab[threadIdx.x & 31], ab[(threadIdx.x + 1) & 31]);
  float2 b = make_float2(ab[32 + (threadIdx.x & 31)], -ab[32 + ((threadIdx.x + 3) & 31)]);
  float2 v[CH];
  for (int c = 0; c < CH; ++c) v[c] = make_float2(0.3f + c * 1e-3f, 0.4f + threadIdx.x * 1e-5f);
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      float2 t = __ffma2_rn(v[c], a, b);
      t = __ffma2_rn(t, a, b);
      t = __ffma2_rn(t, a, b);
      v[c].x = ex2f(-fabsf(t.x));
      v[c].y = ex2f(-fabsf(t.y));
    }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c].x + v[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_f2f_dadd(float* out, long long* cyc) {
  float v[CH]; double acc[CH];
  for (int c = 0; c < CH; ++c) { v[c] = threadIdx.x * 1e-3f + c; acc[c] = 0; }
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) { acc[c] += (double)v[c]; v[c] += 1.0f; }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// mixed packed + scalar FP32: does the lite FMA pipe run scalar FFMA while the
// heavy pipe runs FFMA2?  RATIO scalar chains per packed chain.
template <int NS>
__global__ void k_mix_ffma2_scalar(float* out, const float* ab, long long* cyc) {
  float2 a = make_float2(ab[threadIdx.x & 31], ab[(threadIdx.x + 1) & 31]);
  float2 b = make_float2(ab[32 + (threadIdx.x & 31)], ab[32 + ((threadIdx.x + 3) & 31)]);
  float as = ab[(threadIdx.x + 5) & 31], bs = ab[32 + ((threadIdx.x + 7) & 31)];
  float2 v[CH];
  float w[CH * NS];
  for (int c = 0; c < CH; ++c) v[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  for (int c = 0; c < CH * NS; ++c) w[c] = threadIdx.x * 2e-3f + c;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __ffma2_rn(v[c], a, b);
#pragma unroll
    for (int c = 0; c < CH * NS; ++c) w[c] = fmaf(w[c], as, bs);
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c].x + v[c].y;
  for (int c = 0; c < CH * NS; ++c) s += w[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0; cudaDeviceProp p; CHK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f}\n", p.name, sms, clk_khz / 1e3);
  const int threads = 256;
  float *out, *ab; long long* cyc;
  int blocks_list[] = {sms * 4, sms * 8};
  CHK(cudaMalloc(&out, sizeof(float) * sms * 8 * threads));
  CHK(cudaMalloc(&cyc, sizeof(long long) * sms * 8));
  CHK(cudaMalloc(&ab, sizeof(float) * 64));
  float hab[64]; for (int i = 0; i < 64; ++i) hab[i] = 0.999f - i * 1e-5f;
  CHK(cudaMemcpy(ab, hab, sizeof(hab), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"ffma_imm", "ffma_3reg", "ffma2", "fadd2", "ex2", "mix_3ffma2_2ex2", "f2f_dadd",
                         "ffma2+1scalar", "ffma2+2scalar"};
  // fp32 lane-ops per chain step
  double ops_per[] = {1, 1, 2, 2, 1, 2, 1, 3, 4};
  for (int bi = 0; bi < 2; ++bi) {
    int blocks = blocks_list[bi];
    for (int k = 0; k < 9; ++k) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        switch (k) {
          case 0: k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-4f, cyc); break;
          case 1: k_ffma3<<<blocks, threads>>>(out, ab, cyc); break;
          case 2: k_ffma2<<<blocks, threads>>>(out, ab, cyc); break;
          case 3: k_fadd2<<<blocks, threads>>>(out, ab, cyc); break;
          case 4: k_ex2<<<blocks, threads>>>(out, cyc); break;
          case 5: k_mix13<<<blocks, threads>>>(out, ab, cyc); break;
          case 6: k_f2f_dadd<<<blocks, threads>>>(out, cyc); break;
          case 7: k_mix_ffma2_scalar<1><<<blocks, threads>>>(out, ab, cyc); break;
          case 8: k_mix_ffma2_scalar<2><<<blocks, threads>>>(out, ab, cyc); break;
        }
        cudaEventRecord(e1); CHK(cudaEventSynchronize(e1)); CHK(cudaGetLastError());
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long hc[2048]; CHK(cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
        long long mx = 0; double mean = 0;
        for (int i = 0; i < blocks; ++i) { if (hc[i] > mx) mx = hc[i]; mean += hc[i]; }
        mean /= blocks;
        double total = (double)blocks * threads * ITERS * CH;  // chain steps
        double per_s = total / (ms * 1e-3);
        // SM-clock estimate: the per-block cycle count over the kernel time, assuming
        // blocks/sms/occupancy waves; report ops/SM/clk using event time and nominal max clock too
        double eff_mhz = 0;
        int waves = 1;  // with <=8 blocks/SM of 256 threads all are resident (2048 thr/SM)
        eff_mhz = mx / (ms * 1e-3) / 1e6 * waves;
        double ops_clk_sm = per_s / (sms * eff_mhz * 1e6);
        if (rep == 2)
          printf("{\"kernel\": \"%s\", \"blocks\": %d, \"ms\": %.4f, \"steps_per_s\": %.4e, \"eff_sm_mhz\": %.0f, "
                 "\"instr_per_clk_per_sm\": %.2f, \"fp32_lane_ops_per_clk_per_sm\": %.2f, \"mean_cyc\": %.0f, \"max_cyc\": %lld}\n",
                 names[k], blocks, ms, per_s, eff_mhz, ops_clk_sm, ops_clk_sm * ops_per[k], mean, mx);
      }
    }
  }
  return 0;
}
