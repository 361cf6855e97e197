// Known-answer reference for the device Philox: cuRAND's curand_Philox4x32_10 (an
// implementation independent of this repo), on counters read from a binary file.
//   curand_philox_kat <seed> <in.bin: n x 4 uint32> <out.bin: n x 4 uint32>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <curand_kernel.h>

__global__ void kat(unsigned long long seed, const uint4* c, int n, uint4* o) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = curand_Philox4x32_10(c[i], make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
}

int main(int argc, char** argv) {
  if (argc != 4) return 2;
  unsigned long long seed = strtoull(argv[1], nullptr, 10);
  FILE* f = fopen(argv[2], "rb");
  if (!f) return 3;
  std::vector<uint4> h;
  uint4 v;
  while (fread(&v, sizeof v, 1, f) == 1) h.push_back(v);
  fclose(f);
  int n = (int)h.size();
  uint4 *dc, *dout;
  cudaMalloc(&dc, sizeof(uint4) * n);
  cudaMalloc(&dout, sizeof(uint4) * n);
  cudaMemcpy(dc, h.data(), sizeof(uint4) * n, cudaMemcpyHostToDevice);
  kat<<<(n + 255) / 256, 256>>>(seed, dc, n, dout);
  std::vector<uint4> o(n);
  if (cudaMemcpy(o.data(), dout, sizeof(uint4) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 4;
  f = fopen(argv[3], "wb");
  fwrite(o.data(), sizeof(uint4), n, f);
  fclose(f);
  return 0;
}
