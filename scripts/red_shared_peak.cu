// Microbenchmark: throughput of red.shared.add.u32 with conflict-free,
// lane-private addresses (the C4 histogram's update pattern: PRMT-formed
// offsets bin << 8 | lane << 2 -> bank = lane), all SMs, 3 CTAs x 8 warps per SM.  Reports updates/s and
// updates per clock per SM (the C4 roofline denominator).
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(256) red_kernel(unsigned* sink, int iters) {
  extern __shared__ unsigned cnt[];  // [256 bins][64 words]; lanes use words 0..31
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  const uint32_t base0 = (uint32_t)__cvta_generic_to_shared(cnt);  // [256 bins][64 words], lane-private column
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // one LCG step per 4 bins (the kernel: one LDS.128 per 16)
      x = x * 1664525u + 1013904223u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t off = __byte_perm(x, 4u * lane, 0x5504u | (j << 4));  // bin << 8 | lane << 2
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base0 + off) : "memory");
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(sink, cnt[lane]);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* sink; cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(red_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int per_sm = 3, iters = 4096;
  red_kernel<<<sms * per_sm, 256, 65536>>>(sink, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  red_kernel<<<sms * per_sm, 256, 65536>>>(sink, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double ups = (double)sms * per_sm * 256 * iters * 16 / (ms * 1e-3);
  printf("red.shared.add.u32 lane-private: %.3e updates/s = %.2f /clk/SM at the %.0f MHz nominal clock (%d SMs)\n",
         ups, ups / sms / (clk * 1e3), clk / 1e3, sms);
  return 0;
}
