// Register-file read cost of packed FP32 on sm_100a: FFMA2/FADD2 with 2 or 3
// distinct 64-bit register operands (no operand-reuse), vs scalar FFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rfread rfread.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 8;

// acc_c = fma(a_c, b_c, acc_c): three distinct register pairs per instruction
__global__ void k_ffma2_3(float* out, const float* in) {
  float2 a[CH], b[CH], acc[CH];
  for (int c = 0; c < CH; ++c) {
    a[c] = make_float2(in[c], in[c + 8]);
    b[c] = make_float2(in[c + 16], in[c + 24]);
    acc[c] = make_float2(threadIdx.x * 1e-6f, c);
  }
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(a[c], b[c], acc[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// acc_c = fma(a, b_c, acc_c): a shared (reuse-cache candidate)
__global__ void k_ffma2_2(float* out, const float* in) {
  float2 a = make_float2(in[0], in[1]), b[CH], acc[CH];
  for (int c = 0; c < CH; ++c) {
    b[c] = make_float2(in[c + 16], in[c + 24]);
    acc[c] = make_float2(threadIdx.x * 1e-6f, c);
  }
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(a, b[c], acc[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// acc_c = acc_c + b_c (two distinct pairs)
__global__ void k_fadd2_2(float* out, const float* in) {
  float2 b[CH], acc[CH];
  for (int c = 0; c < CH; ++c) {
    b[c] = make_float2(in[c + 16] * 1e-3f, in[c + 24] * 1e-3f);
    acc[c] = make_float2(threadIdx.x * 1e-6f, c);
  }
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __fadd2_rn(acc[c], b[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// scalar acc_c = fma(a_c, b_c, acc_c) (three distinct registers)
__global__ void k_ffma_3(float* out, const float* in) {
  float a[2 * CH], b[2 * CH], acc[2 * CH];
  for (int c = 0; c < 2 * CH; ++c) {
    a[c] = in[c];
    b[c] = in[c + 16];
    acc[c] = threadIdx.x * 1e-6f + c;
  }
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < 2 * CH; ++c) acc[c] = fmaf(a[c], b[c], acc[c]);
  float s = 0;
  for (int c = 0; c < 2 * CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// scalar acc_c = fma(a, b_c, acc_c) (a shared)
__global__ void k_ffma_2(float* out, const float* in) {
  float a = in[0], b[2 * CH], acc[2 * CH];
  for (int c = 0; c < 2 * CH; ++c) {
    b[c] = in[c + 16];
    acc[c] = threadIdx.x * 1e-6f + c;
  }
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < 2 * CH; ++c) acc[c] = fmaf(a, b[c], acc[c]);
  float s = 0;
  for (int c = 0; c < 2 * CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  float *out, *in;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  cudaMalloc(&in, sizeof(float) * 64);
  float h[64];
  for (int i = 0; i < 64; ++i) h[i] = 0.9999f - i * 1e-6f;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"ffma2_3distinct", "ffma2_2distinct", "fadd2_2distinct", "ffma_3distinct", "ffma_2distinct"};
  double lane_ops[] = {2.0 * CH, 2.0 * CH, 2.0 * CH, 2.0 * CH, 2.0 * CH};  // fp32 lane-ops per thread-iteration
  double instr[] = {CH, CH, CH, 2.0 * CH, 2.0 * CH};
  int blocks = sms * 8;
  for (int k = 0; k < 5; ++k) {
    float best = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      switch (k) {
        case 0: k_ffma2_3<<<blocks, 256>>>(out, in); break;
        case 1: k_ffma2_2<<<blocks, 256>>>(out, in); break;
        case 2: k_fadd2_2<<<blocks, 256>>>(out, in); break;
        case 3: k_ffma_3<<<blocks, 256>>>(out, in); break;
        case 4: k_ffma_2<<<blocks, 256>>>(out, in); break;
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    double threads = (double)blocks * 256 * ITERS;
    double ops = threads * lane_ops[k] / (best * 1e-3);
    double ins = threads * instr[k] / 32 / (best * 1e-3);
    // per SM per cycle at 1965 MHz (the clock during these runs; see the clocks file)
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"fp32_lane_ops_per_s\": %.4e, \"lane_ops_per_clk_sm_at_1965\": %.1f, "
           "\"warp_instr_per_clk_smsp_at_1965\": %.3f}\n",
           names[k], best, ops, ops / (sms * 1.965e9), ins / (sms * 4 * 1.965e9));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
