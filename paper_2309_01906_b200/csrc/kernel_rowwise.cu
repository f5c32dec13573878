// kernel_rowwise.cu — fused 4-level row-wise nest reduction (config 2).
//
// Nest shape (SURVEY §8(a) A3, §8(c) reading #13):
//     GPU      static        loop 0 (rows; host: rank shard)
//     cluster  static        loop 0: a contiguous block of rows per cluster
//     CTA      static        loop 1: a contiguous block of n1/K columns
//     warp     static(128)   loop 1
//     lane     static(4)     loop 1
// One result per row (keyed by loop 0): the row owner is the cluster, whose
// CTAs, warps and lanes combine every row.
//
// B200 design (per cluster, per row):
//   * each CTA's producer warp streams its n1/K-column segment of the row
//     with one 1-D TMA bulk copy into an S-stage smem ring (full/empty
//     mbarriers), L2 evict-first;
//   * lane level: each lane sums its float4s (fp32 pairwise, fp64 across);
//     lane -> warp: ordered SHFL tree (fp64);
//   * warp -> CTA -> cluster: every warp's lane 0 pushes its warp partial
//     with st.async into the LEADER CTA's slot ring over DSMEM; the store
//     itself completes the leader's per-row mbarrier (complete_tx), so the
//     warp- and CTA-level barriers are transaction barriers with no
//     bar.sync / barrier.cluster in the row loop;
//   * a combiner warp in the leader CTA waits the row's mbarrier, folds the
//     K*W warp partials in ascending order (CTA partials, then the row),
//     writes the row and frees the slot by arriving remotely on every CTA's
//     slot-empty mbarrier.
// Slots are a ring of R rows, so the combine of row j overlaps the loads of
// rows j+1 .. j+S.  The only cluster barriers are at start-up and exit.
#include <cuda_runtime.h>
#include <stdint.h>
#include "fused_common.cuh"

namespace hpar {
namespace {

constexpr int kStages = 6;   // TMA ring depth (rows in flight per CTA)
constexpr int kSlots = 8;    // DSMEM row-slot ring depth in the leader
constexpr int kMaxPush = 32; // K*W <= 32 warp partials per row

template <bool VERIFY>
__global__ void __launch_bounds__(1024, 1) rowwise_kernel(const __grid_constant__ NestArgs a, int W, int qcols) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ __align__(8) uint64_t row_full[kSlots], slot_empty[kSlots];
  __shared__ __align__(8) double slot[kSlots][kMaxPush];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K;
  const uint32_t crank = cluster_ctarank();
  const int64_t c = blockIdx.x / K;
  // cluster c's block of rows (static over C clusters)
  const int64_t q = a.n0 / a.C, r = a.n0 % a.C;
  const int64_t row0 = c * q + (c < r ? c : r);
  const int64_t nrows = q + (c < r ? 1 : 0);
  const int64_t col0 = (int64_t)crank * qcols;
  const float* x = (const float*)a.in;
  const uint32_t seg_bytes = (uint32_t)qcols * 4;
  const int npush = K * W;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&row_full[s], 1);   // armed by the combiner with expect_tx
      mbar_init(&slot_empty[s], 1); // one remote arrive from the leader's combiner
    }
    fence_mbarrier_init_cluster();
  }
  cluster_sync_all();  // barriers of every CTA initialised before any remote use

  if (warp == W) {
    // ------------------------------ producer warp: TMA row segments ----
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int64_t j = 0; j < nrows; ++j) {
        const int s = (int)(j % kStages);
        if (j >= kStages) mbar_wait(&empty[s], (uint32_t)(((j / kStages) - 1) & 1));
        mbar_arrive_expect_tx(&full[s], seg_bytes);
        bulk_g2s(dsm + (size_t)s * seg_bytes, x + (row0 + j) * a.ld + col0, seg_bytes, &full[s], pol);
      }
    }
  } else if (warp == W + 1) {
    // ------------------------------ combiner warp (leader CTA only) ----
    if (crank == 0) {
      for (int64_t j = 0; j < nrows; ++j) {
        const int s = (int)(j % kSlots);
        const uint32_t ph = (uint32_t)((j / kSlots) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&row_full[s], (uint32_t)(npush * 8));
        mbar_wait_cluster(&row_full[s], ph);
        double v = lane < npush ? slot[s][lane] : 0.0;
        // warp partials -> CTA partials (lanes k*W), ordered
        v = shfl_tree<OP_SUM, double>(v, 1, W);
        if (VERIFY && (a.verify & V_PARTIALS) && lane < npush && (lane % W) == 0)
          export_slot<double>(a, S_CTA, (row0 + j) * K + lane / W, v);
        // CTA partials -> row (cluster), ordered
        v = shfl_tree<OP_SUM, double>(v, W, K);
        if (lane == 0) {
          const int64_t row = row0 + j;
          if (a.out_dtype == DT_F32) ((float*)a.out)[row] = (float)v;
          else ((double*)a.out)[row] = v;
        }
        __syncwarp();
        // free the slot in every CTA of the cluster
        if (lane < K) mbar_arrive_cluster(mapa(smem_addr(&slot_empty[s]), (uint32_t)lane));
      }
    }
  } else {
    // ------------------------------ W consumer warps --------------------
    const int nvec = qcols / 4;
    const uint32_t leader_slot_base = mapa(smem_addr(&slot[0][0]), 0);
    const uint32_t leader_full_base = mapa(smem_addr(&row_full[0]), 0);
    const int push_idx = (int)crank * W + warp;
    const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + (int64_t)blockIdx.x * W * 32 + threadIdx.x;
    for (int64_t j = 0; j < nrows; ++j) {
      const int s = (int)(j % kStages);
      mbar_wait(&full[s], (uint32_t)((j / kStages) & 1));
      const float4* st = (const float4*)(dsm + (size_t)s * seg_bytes);
      double acc = 0.0;
      for (int f = warp * 32 + lane; f < nvec; f += W * 32) {
        const float4 v = st[f];
        acc += (double)((v.x + v.y) + (v.z + v.w));
        if constexpr (VERIFY) {
          for (int e = 0; e < 4; ++e) {
            const int64_t it = (row0 + j) * a.n1 + col0 + 4 * f + e;
            if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // stage consumed
      if constexpr (VERIFY) {
        if (a.verify & V_PARTIALS)
          export_slot<double>(a, S_LANE_IN, (row0 + j) * (int64_t)(npush * 32) + push_idx * 32 + lane, acc);
      }
      acc = warp_fold<OP_SUM>(acc);
      if (lane == 0) {
        if constexpr (VERIFY) {
          if (a.verify & V_PARTIALS) export_slot<double>(a, S_WARP, (row0 + j) * npush + push_idx, acc);
        }
        const int ss = (int)(j % kSlots);
        if (j >= kSlots) mbar_wait_cluster(&slot_empty[ss], (uint32_t)(((j / kSlots) - 1) & 1));
        st_async_u64(leader_slot_base + (uint32_t)((ss * kMaxPush + push_idx) * 8),
                     leader_full_base + (uint32_t)(ss * 8), (unsigned long long)__double_as_longlong(acc));
      }
      __syncwarp();
    }
  }
  // every CTA stays until the leader has consumed all pushes and freed slots
  cluster_sync_all();
}

template <bool V>
cudaError_t launch_t(const NestArgs& a, int W, int qcols, cudaStream_t s) {
  auto kern = rowwise_kernel<V>;
  const size_t smem = (size_t)kStages * qcols * 4;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.C * a.K));
  cfg.blockDim = dim3((unsigned)((W + 2) * 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, W, qcols);
}

bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

}  // namespace

bool rowwise_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 2 || !a.keyed || a.offsets) { *why = "not a dense keyed 2-loop nest"; return false; }
  if (a.op != OP_SUM || a.in_dtype != DT_F32) { *why = "rowwise kernel: f32 sum only"; return false; }
  if (a.verify & V_FINGERPRINT) { *why = "fingerprints not produced by the rowwise kernel"; return false; }
  if (a.lane_w != 1) { *why = "lane partition"; return false; }
  LevelView v = device_levels(a);
  if (v.n != 4) { *why = "needs cluster, CTA, warp, lane levels"; return false; }
  const DevLevel *c = v.l[0], *k = v.l[1], *w = v.l[2], *l = v.l[3];
  if (!is_level(c, S_CLUSTER) || !is_level(k, S_CTA) || !is_level(w, S_WARP) || !is_level(l, S_LANE)) {
    *why = "levels not cluster/CTA/warp/lane";
    return false;
  }
  if (c->loop != 0 || c->sched != SCHED_STATIC) { *why = "rows must be static over clusters"; return false; }
  if (k->loop != 1 || k->sched != SCHED_STATIC) { *why = "columns must be static over CTAs"; return false; }
  if (w->loop != 1 || w->sched != SCHED_STATIC_CHUNK || w->chunk != 128) { *why = "warp static(128)"; return false; }
  if (l->loop != 1 || l->sched != SCHED_STATIC_CHUNK || l->chunk != 4) { *why = "lane static(4)"; return false; }
  const int64_t K = a.K, W = a.radix[S_WARP];
  if (!pow2(K) || !pow2(W) || K * W > kMaxPush) { *why = "K, W powers of two with K*W <= 32"; return false; }
  if (a.n1 % (4 * K) != 0 || a.ld % 4 != 0 || ((uintptr_t)a.in & 15)) { *why = "alignment"; return false; }
  if ((a.n1 / K) * 4 * kStages > 200 * 1024) { *why = "row segment too large for the smem ring"; return false; }
  if (a.n1 == 0) { *why = "empty rows"; return false; }
  return true;
}

cudaError_t launch_rowwise(const NestArgs& a, int W, cudaStream_t s, const char** name) {
  *name = "rowwise_tma_dsmem";
  const int qcols = (int)(a.n1 / a.K);
  return a.verify ? launch_t<true>(a, W, qcols, s) : launch_t<false>(a, W, qcols, s);
}

}  // namespace hpar
