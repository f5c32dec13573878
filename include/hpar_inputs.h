/* hpar_inputs.h — seeded synthetic input generator (device side).
 *
 * NOT part of the method: this library only fills device buffers with the
 * counter-based stream that inputs/gen.py defines on the host (DESIGN.md,
 * "Input recipe").  It exists because the full-size
 * workloads (2^32 bytes for config 4, 2^34 fp32 for config 5) cannot be
 * generated on the host and copied in reasonable time.  It contains no
 * partitioning and no reduction arithmetic, and the product library
 * (libhpar.so) does not link it.
 *
 *   z(seed, i) = splitmix64(seed * 2^40 + i)      (Stafford-13 finaliser)
 *   int32 = low 32 bits of z;  fp32 = (z >> 40) * 2^-24;  uint8 = z >> 56
 *
 * All calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  `dst` is a caller-owned device pointer holding `n`
 * elements; element e receives z(seed, begin + e).  Return 0 on success,
 * otherwise the cudaError_t of the failed launch.
 */
#ifndef HPAR_INPUTS_H
#define HPAR_INPUTS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

int hpar_inputs_fill_i32(uint64_t seed, uint64_t begin, int64_t n, int32_t* dst, void* stream);
int hpar_inputs_fill_f32(uint64_t seed, uint64_t begin, int64_t n, float* dst, void* stream);
int hpar_inputs_fill_u8(uint64_t seed, uint64_t begin, int64_t n, uint8_t* dst, void* stream);
/* Skewed bytes: symbol = number of cdf[] entries <= u, u = (z >> 11) * 2^-53,
 * clamped to 255; `cdf256` is a device array of 256 doubles (ascending). */
int hpar_inputs_fill_u8_cdf(uint64_t seed, uint64_t begin, int64_t n, const double* cdf256,
                            uint8_t* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif
