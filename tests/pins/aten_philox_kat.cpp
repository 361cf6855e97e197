// Known-answer helper: prints Philox4x32-10 outputs from ATen's header-only
// at::philox_engine (torch/include/ATen/core/PhiloxRNGEngine.h), an
// implementation independent of oracle/phd_oracle.c.  Reads lines
// "seed subsequence offset" from stdin, prints the 4 output words.
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cinttypes>
int main() {
  unsigned long long seed, sub, off;
  while (std::scanf("%llu %llu %llu", &seed, &sub, &off) == 3) {
    at::philox_engine e(seed, sub, off);
    uint32_t a = e(), b = e(), c = e(), d = e();
    std::printf("%u %u %u %u\n", a, b, c, d);
  }
  return 0;
}
