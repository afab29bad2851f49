// div_check.cu -- exhaustive check (all 2^32 fp32 inputs) that division by a constant c computed as
//   q0 = RN(x * rc), r = fma(-q0, c, x), q = fma(r, rc, q0)        (rc = RN(1 / c)), for 2^-100 <= |x| <= 2^100
// equals the IEEE quotient RN(x / c) bit for bit (NaNs compared as NaN). Used to justify env.cu's
// div_const for the transition model's constant divisors: both sides then agree with the
// oracle's plain x / c.      build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/div_check.cu
#include <cstdio>
#include <cstdint>
#include <cmath>

__global__ void k_check(float c, float rc, unsigned long long* bad, unsigned* first) {
  const uint64_t n = 1ull << 32;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((uint32_t)i);
    const float ref = __fdiv_rn(x, c);
    const float q0 = __fmul_rn(x, rc);
    const float r = __fmaf_rn(-q0, c, x);
    const float q = __fmaf_rn(r, rc, q0);
    const float ax = fabsf(x);
    const bool in_range = ax >= 0x1p-100f && ax <= 0x1p100f;  // div_const's fast-path domain
    const bool same = !in_range || (__float_as_uint(ref) == __float_as_uint(q));
    if (!same) {
      if (atomicAdd(bad, 1ull) < 4) first[atomicAdd(first + 8, 1u) & 7] = (uint32_t)i;
    }
  }
}

int main() {
  const float cs[] = {0.05f, 30.0f, 1.7f, 0.5f, 2.0f, 0.25f, 0.02f};
  unsigned long long* bad;
  unsigned* first;
  cudaMalloc(&bad, 8);
  cudaMalloc(&first, 64);
  for (float c : cs) {
    const float rc = (float)(1.0 / (double)c);
    cudaMemset(bad, 0, 8);
    cudaMemset(first, 0, 64);
    k_check<<<148 * 8, 256>>>(c, rc, bad, first);
    unsigned long long hb = 0;
    unsigned hf[16];
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hf, first, 64, cudaMemcpyDeviceToHost);
    printf("c = %.9g rc = %.9g: %llu mismatches of 2^32", c, rc, hb);
    for (unsigned k = 0; k < (hb < 4 ? hb : 4); ++k) {
      float x;
      memcpy(&x, &hf[k], 4);
      printf("  [x = %.9g (0x%08x)]", x, hf[k]);
    }
    printf("\n");
  }
  return 0;
}
