// Device implementation of the inputs/gen.py counter-based stream.
// Input generation only: no method arithmetic lives here (see include/hpar_inputs.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include "hpar_inputs.h"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int KIND>
__global__ void fill_kernel(uint64_t seed, uint64_t begin, int64_t n, void* dst, const double* cdf) {
  const uint64_t base = seed * (1ull << 40) + begin;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    const uint64_t z = splitmix64(base + (uint64_t)e);
    if (KIND == 0) {
      ((int32_t*)dst)[e] = (int32_t)(uint32_t)(z & 0xFFFFFFFFull);
    } else if (KIND == 1) {
      ((float*)dst)[e] = (float)((double)(z >> 40) * 0x1p-24);
    } else if (KIND == 2) {
      ((uint8_t*)dst)[e] = (uint8_t)(z >> 56);
    } else {
      const double u = (double)(z >> 11) * 0x1p-53;
      int lo = 0, hi = 256;  // first index with cdf[idx] > u  (== searchsorted right)
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
      }
      ((uint8_t*)dst)[e] = (uint8_t)(lo > 255 ? 255 : lo);
    }
  }
}

template <int KIND>
int launch(uint64_t seed, uint64_t begin, int64_t n, void* dst, const double* cdf, void* stream) {
  if (n <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  fill_kernel<KIND><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(seed, begin, n, dst, cdf);
  return (int)cudaGetLastError();
}

}  // namespace

extern "C" {
int hpar_inputs_fill_i32(uint64_t seed, uint64_t begin, int64_t n, int32_t* dst, void* stream) {
  return launch<0>(seed, begin, n, dst, nullptr, stream);
}
int hpar_inputs_fill_f32(uint64_t seed, uint64_t begin, int64_t n, float* dst, void* stream) {
  return launch<1>(seed, begin, n, dst, nullptr, stream);
}
int hpar_inputs_fill_u8(uint64_t seed, uint64_t begin, int64_t n, uint8_t* dst, void* stream) {
  return launch<2>(seed, begin, n, dst, nullptr, stream);
}
int hpar_inputs_fill_u8_cdf(uint64_t seed, uint64_t begin, int64_t n, const double* cdf256,
                            uint8_t* dst, void* stream) {
  return launch<3>(seed, begin, n, dst, cdf256, stream);
}
}
