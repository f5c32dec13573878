// kernel_probe.cu — level barrier + visibility probe (§8(a) A10).
//
// The §3.7 fallback pattern generalised to a level: every task
// writes f(round, its id) into its slot, the LEVEL BARRIER runs, then every
// task reads all of its siblings' slots and folds them ("every lane
// gets 36" is the 8-lane case).  A task whose fold differs from the value
// the siblings wrote counts as a mismatch: 0 mismatches = the barrier gives
// rendezvous + visibility.  The barriers are the ones the hot path uses:
//     lane level : __syncwarp
//     warp level : bar.sync
//     CTA level  : barrier.cluster arrive.release / wait.acquire over DSMEM
// Slots are double-buffered by round parity so that one barrier per round
// suffices (a slot is rewritten only after the next barrier).
#include <cuda_runtime.h>
#include <stdint.h>
#include "level_primitives.cuh"
#include "hpar.h"

namespace hpar {
namespace {

__device__ __forceinline__ unsigned long long probe_val(int round, uint64_t id) {
  return fp_mix(((uint64_t)round << 40) ^ id);
}

__global__ void probe_kernel(int level, int rounds, unsigned long long* mismatches) {
  __shared__ unsigned long long lane_slot[2][32][32];  // [parity][warp][lane]
  __shared__ unsigned long long warp_slot[2][32];
  __shared__ unsigned long long cta_slot[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const uint32_t crank = cluster_ctarank(), K = cluster_nctarank();
  const uint64_t cta_id = blockIdx.x;
  unsigned long long bad = 0;
  for (int r = 0; r < rounds; ++r) {
    const int p = r & 1;
    if (level == HPAR_LANE) {
      const uint64_t base = ((uint64_t)blockIdx.x * W + warp) * 32;
      lane_slot[p][warp][lane] = probe_val(r, base + lane);
      __syncwarp();
      unsigned long long got = 0, want = 0;
      for (int j = 0; j < 32; ++j) {
        got += ((volatile unsigned long long*)lane_slot[p][warp])[j];
        want += probe_val(r, base + j);
      }
      bad += (got != want);
    } else if (level == HPAR_WARP) {
      const uint64_t base = (uint64_t)blockIdx.x * W;
      if (lane == 0) warp_slot[p][warp] = probe_val(r, base + warp);
      __syncthreads();
      if (lane == 0) {
        unsigned long long got = 0, want = 0;
        for (int j = 0; j < W; ++j) {
          got += ((volatile unsigned long long*)warp_slot[p])[j];
          want += probe_val(r, base + j);
        }
        bad += (got != want);
      }
    } else {  // HPAR_CTA: siblings are the CTAs of the cluster
      const uint64_t base = cta_id - crank;
      if (threadIdx.x == 0) cta_slot[p] = probe_val(r, cta_id);
      cluster_arrive_release();
      cluster_wait_acquire();
      if (threadIdx.x == 0) {
        unsigned long long got = 0, want = 0;
        for (uint32_t k = 0; k < K; ++k) {
          got += ld_cluster_u64(mapa(smem_addr(&cta_slot[p]), k));
          want += probe_val(r, base + k);
        }
        bad += (got != want);
      }
    }
  }
  if (level == HPAR_CTA) cluster_sync_all();
  if (bad && mismatches) atomicAdd(mismatches, bad);
}

}  // namespace

cudaError_t launch_probe(int level, int64_t C, int K, int W, int rounds, unsigned long long* mismatches,
                         cudaStream_t s) {
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
  return cudaLaunchKernelEx(&cfg, probe_kernel, level, rounds, mismatches);
}

}  // namespace hpar
