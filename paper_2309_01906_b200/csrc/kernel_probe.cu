// kernel_probe.cu — level barrier visibility probe (§8(a) A10, verify only).
//
// The §3.7 fallback pattern generalised to a level: in every
// round each task writes f(round, its id) into its slot, the LEVEL BARRIER
// runs, then each task reads all of its siblings' slots and folds them
// ("every lane gets 36" is the 8-lane case).  The kernel does NOT
// judge the folds itself: every task adds its per-round folds into
// folds[task] (mod 2^64) and the caller compares them with the oracle's
// group folds (tests/test_gpu_parity.py).  The barriers are the ones the hot
// path uses:
//     lane level : __syncwarp
//     warp level : bar.sync
//     CTA level  : barrier.cluster arrive.release / wait.acquire over DSMEM
// Slots are double-buffered by round parity so that one barrier per round
// suffices (a slot is rewritten only after the next barrier).
//
// Negative control (HPAR_PROBE_NO_BARRIER): the level barrier is left out
// and sibling k delays its write by (k + 1) * delay_ns (spin on
// %globaltimer), so a missing barrier is observable: readers fold stale
// slots and the caller sees folds differing from the oracle's.  (Divergent
// lanes reconverge at the end of the delay branch, which is why the lane
// level's control may still fold correctly; compute-sanitizer racecheck is
// the evidence there.)
#include <cuda_runtime.h>
#include <stdint.h>
#include "level_primitives.cuh"
#include "hpar.h"

namespace hpar {
namespace {

__device__ __forceinline__ unsigned long long probe_val(int round, uint64_t id) {
  return fp_mix(((uint64_t)round << 40) ^ id);
}

__device__ __forceinline__ void spin_ns(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

__global__ void probe_kernel(int level, int rounds, int no_barrier, uint32_t delay_ns,
                             unsigned long long* folds) {
  __shared__ unsigned long long lane_slot[2][32][32];  // [parity][warp][lane]
  __shared__ unsigned long long warp_slot[2][32];
  __shared__ unsigned long long cta_slot[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const uint32_t crank = cluster_ctarank(), K = cluster_nctarank();
  const uint64_t cta_id = blockIdx.x;
  for (int i = threadIdx.x; i < 2 * 32 * 32; i += blockDim.x) (&lane_slot[0][0][0])[i] = 0;
  for (int i = threadIdx.x; i < 2 * 32; i += blockDim.x) (&warp_slot[0][0])[i] = 0;
  if (threadIdx.x < 2) cta_slot[threadIdx.x] = 0;
  __syncthreads();
  cluster_sync_all();
  unsigned long long acc = 0;
  for (int r = 0; r < rounds; ++r) {
    const int p = r & 1;
    if (level == HPAR_LANE) {
      const uint64_t base = ((uint64_t)blockIdx.x * W + warp) * 32;
      if (no_barrier && delay_ns) spin_ns((uint64_t)(lane + 1) * delay_ns);
      lane_slot[p][warp][lane] = probe_val(r, base + lane);
      if (!no_barrier) __syncwarp();
      unsigned long long got = 0;
      for (int j = 0; j < 32; ++j) got += ((volatile unsigned long long*)lane_slot[p][warp])[j];
      acc += got;
    } else if (level == HPAR_WARP) {
      const uint64_t base = (uint64_t)blockIdx.x * W;
      if (lane == 0) {
        if (no_barrier && delay_ns) spin_ns((uint64_t)(warp + 1) * delay_ns);
        warp_slot[p][warp] = probe_val(r, base + warp);
      }
      if (!no_barrier) __syncthreads();
      if (lane == 0) {
        unsigned long long got = 0;
        for (int j = 0; j < W; ++j) got += ((volatile unsigned long long*)warp_slot[p])[j];
        acc += got;
      }
    } else {  // HPAR_CTA: siblings are the CTAs of the cluster
      if (threadIdx.x == 0) {
        if (no_barrier && delay_ns) spin_ns((uint64_t)(crank + 1) * delay_ns);
        cta_slot[p] = probe_val(r, cta_id);
      }
      if (!no_barrier) {
        cluster_arrive_release();
        cluster_wait_acquire();
      }
      if (threadIdx.x == 0) {
        unsigned long long got = 0;
        for (uint32_t k = 0; k < K; ++k) got += ld_cluster_u64(mapa(smem_addr(&cta_slot[p]), k));
        acc += got;
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a sibling may still read its slots
  if (!folds) return;
  if (level == HPAR_LANE) folds[(uint64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
  else if (level == HPAR_WARP && lane == 0) folds[(uint64_t)blockIdx.x * W + warp] = acc;
  else if (level == HPAR_CTA && threadIdx.x == 0) folds[cta_id] = acc;
}

}  // namespace

cudaError_t launch_probe(int level, int64_t C, int K, int W, int rounds, int no_barrier, uint32_t delay_ns,
                         unsigned long long* folds, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * K));
  cfg.blockDim = dim3((unsigned)(W * 32));
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, probe_kernel, level, rounds, no_barrier, delay_ns, folds);
}

}  // namespace hpar
