// node_fused.cuh — the node level inside the kernel (the
// paper's missing level above the GPU).
//
// The CTA that folds this GPU's result (the last arriver of the grid
// ticket) stores it into slot [parity][my rank] of EVERY rank's symmetric
// buffer (NVLink loads/stores through NCCL's LSA pointers), the same CTAs of
// all GPUs meet at one NCCL LSA barrier (acq_rel), and each then folds the
// G slots of its own buffer in ascending rank order — the GPU level's static
// block order, so ordered ops (AFFINE) stay ordered.  Two slot halves
// alternate between calls: a rank reusing a half has passed the next call's
// barrier, which every rank reaches only after reading the half.
#pragma once
#include <nccl_device.h>

#include "level_primitives.cuh"
#include "plan.h"

namespace hpar {

__device__ __forceinline__ size_t node_slot_off(const NestArgs& a, int nranks, int rank) {
  return ((size_t)a.node_parity * nranks + rank) * (size_t)a.node_slot;
}

// All threads of the CTA call it; `tot` is meaningful in thread 0 on entry
// (this GPU's result) and on return (the node's result).
template <int OP, typename Acc>
__device__ void node_fold_scalar(const NestArgs& a, Acc& tot) {
  const ncclDevComm& dc = *(const ncclDevComm*)a.node_dc;
  ncclWindow_t win = (ncclWindow_t)a.node_win;
  if (threadIdx.x == 0)
    for (int p = 0; p < dc.lsaSize; ++p) *(Acc*)ncclGetLsaPointer(win, node_slot_off(a, dc.nRanks, dc.rank), p) = tot;
  {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
  if (threadIdx.x == 0) {
    Acc r = OpT<OP, Acc>::identity();
    for (int g = 0; g < dc.nRanks; ++g) r = OpT<OP, Acc>::combine(r, *(const Acc*)ncclGetLocalPointer(win, node_slot_off(a, dc.nRanks, g)));
    tot = r;
  }
}

// 256 u64 bins: thread t owns bins t, t + blockDim.x, ... (tot[] holds them).
template <int NB>
__device__ void node_fold_bins(const NestArgs& a, unsigned long long (&tot)[NB]) {
  const ncclDevComm& dc = *(const ncclDevComm*)a.node_dc;
  ncclWindow_t win = (ncclWindow_t)a.node_win;
  for (int p = 0; p < dc.lsaSize; ++p) {
    unsigned long long* dst = (unsigned long long*)ncclGetLsaPointer(win, node_slot_off(a, dc.nRanks, dc.rank), p);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int bin = threadIdx.x + j * blockDim.x;
      if (bin < 256) dst[bin] = tot[j];
    }
  }
  {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int bin = threadIdx.x + j * blockDim.x;
    if (bin >= 256) continue;
    unsigned long long r = 0;
    for (int g = 0; g < dc.nRanks; ++g)
      r += ((const unsigned long long*)ncclGetLocalPointer(win, node_slot_off(a, dc.nRanks, g)))[bin];
    tot[j] = r;
  }
}

}  // namespace hpar
