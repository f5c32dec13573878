// Exhaustive check (all 2^32 fp32 bit patterns) that the 3-op sequence
//   q0 = a * 0.2f;  r = fma(-q0, 5, a);  q = fma(r, 0.2f, q0)
// returns the correctly rounded a / 5 (IEEE, __fdiv_rn) — the division used
// by kernel_stencil.cu.  NaN results compare as NaN.
#include <cstdio>
#include <cstdint>
__global__ void check(unsigned long long* bad, unsigned* first) {  // first: up to 8 mismatching inputs
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (1ull << 32); i += (uint64_t)gridDim.x * blockDim.x) {
    const float a = __uint_as_float((uint32_t)i);
    const float q0 = __fmul_rn(a, 0.2f);
    const float r = __fmaf_rn(-q0, 5.0f, a);
    const float q = __fmaf_rn(r, 0.2f, q0);
    const float ref = __fdiv_rn(a, 5.0f);
    const bool same = (__float_as_uint(q) == __float_as_uint(ref)) || (q != q && ref != ref);
    if (!same) { const unsigned long long k = atomicAdd(bad, 1ull); if (k < 8) first[k] = (uint32_t)i; }
  }
}
int main() {
  unsigned long long* bad; unsigned* first;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&first, 32);
  *bad = 0; *first = 0;
  check<<<148 * 16, 256>>>(bad, first);
  cudaDeviceSynchronize();
  printf("mismatches %llu\n", *bad);
  for (unsigned long long k = 0; k < *bad && k < 8; ++k) printf("  0x%08x (%g)\n", first[k], (double)__builtin_bit_cast(float, first[k]));
  return 0;
}
