// kernel_hist.cu — level-scoped 256-bin histogram (config 4).
//
// Nest shape (flat, uint8; V = 16 bytes per lane vector):
//     GPU      static            (host: rank shard)
//     cluster  static(K*tile)
//     CTA      static(tile)
//     warp     static(512)       (32 lanes x 16 B)
//     lane     static(16)
// Privatisation per level:
//     warp    : its own 256 u32 bins in shared memory (lanes increment them
//               with shared-memory atomics — lanes have no private bins)
//     CTA     : sum of its warps' bins (ascending warp), bar.sync
//     cluster : reduce-scatter over DSMEM — CTA k owns bins [256k/K, 256(k+1)/K)
//               and sums them over the K CTAs (ascending), barrier.cluster
//     GPU     : u64 cluster partials + single-pass ticket; the last cluster
//               folds them in ascending cluster order
//     node    : ncclAllReduce of 256 u64 (runtime.cpp)
// Input stream: producer warp + 1-D TMA bulk ring as in kernel_flat.cu.
#include <cuda_runtime.h>
#include <stdint.h>
#include "fused_common.cuh"

namespace hpar {
namespace {

constexpr int kStages = 4;

template <bool VERIFY>
__global__ void __launch_bounds__(1024, 1) hist_kernel(const __grid_constant__ NestArgs a, int W, int tile) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t wbins[16][256];
  __shared__ uint32_t cbins[256];
  __shared__ int s_flag;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = a.n0;
  const int64_t ntiles = (n + tile - 1) / tile;
  const int64_t nblocks = gridDim.x;
  const int64_t b = blockIdx.x;
  const int64_t my_tiles = (b < ntiles) ? (ntiles - 1 - b) / nblocks + 1 : 0;
  const uint8_t* x = (const uint8_t*)a.in;
  const int K = a.K;
  const uint32_t crank = cluster_ctarank();
  const int64_t cl = blockIdx.x / K;

  for (int i = threadIdx.x; i < W * 256; i += blockDim.x) (&wbins[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    fence_mbarrier_init_cluster();
  }
  __syncthreads();

  if (warp == W) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int64_t j = 0; j < my_tiles; ++j) {
        const int s = (int)(j % kStages);
        if (j >= kStages) mbar_wait(&empty[s], (uint32_t)(((j / kStages) - 1) & 1));
        const int64_t base = (j * nblocks + b) * tile;
        const int64_t len = (n - base < tile) ? (n - base) : tile;
        const uint32_t bytes = (uint32_t)(len & ~(int64_t)15);
        mbar_arrive_expect_tx(&full[s], bytes);
        if (bytes) bulk_g2s(dsm + (size_t)s * tile, x + base, bytes, &full[s], pol);
      }
    }
  } else {
    uint32_t* mybins = wbins[warp];
    const int nvec = tile / 16;
    const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + b * W * 32 + threadIdx.x;
    for (int64_t j = 0; j < my_tiles; ++j) {
      const int s = (int)(j % kStages);
      const int64_t base = (j * nblocks + b) * tile;
      const int64_t len = (n - base < tile) ? (n - base) : tile;
      mbar_wait(&full[s], (uint32_t)((j / kStages) & 1));
      const unsigned char* st = dsm + (size_t)s * tile;
      if (len == tile) {
#pragma unroll 2
        for (int f = warp * 32 + lane; f < nvec; f += W * 32) {
          const uint4 v = ((const uint4*)st)[f];
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            atomicAdd(&mybins[w4[k] & 0xFF], 1u);
            atomicAdd(&mybins[(w4[k] >> 8) & 0xFF], 1u);
            atomicAdd(&mybins[(w4[k] >> 16) & 0xFF], 1u);
            atomicAdd(&mybins[w4[k] >> 24], 1u);
          }
          if constexpr (VERIFY) {
            for (int e = 0; e < 16; ++e) {
              const int64_t it = base + 16 * f + e;
              if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
            }
          }
        }
      } else {
        const int64_t in_smem = len & ~(int64_t)15;
        for (int f = warp * 32 + lane; f < nvec; f += W * 32) {
          for (int e = 0; e < 16; ++e) {
            const int64_t off = 16 * (int64_t)f + e;
            if (off >= len) break;
            const uint8_t byte = off < in_smem ? st[off] : x[base + off];
            atomicAdd(&mybins[byte], 1u);
            if constexpr (VERIFY) {
              if (a.verify & V_COVERAGE) { a.owner[base + off] = leaf; atomicAdd(&a.count[base + off], 1u); }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncwarp();
  __syncthreads();
  // warp -> CTA (ascending warp), export warp partials
  unsigned long long* parts = (unsigned long long*)a.cluster_partials;
  for (int bin = threadIdx.x; bin < 256; bin += blockDim.x) {
    uint32_t sacc = 0;
    for (int w = 0; w < W; ++w) {
      sacc += wbins[w][bin];
      if (VERIFY && (a.verify & V_PARTIALS)) {
        for (int l = 0; l < a.nlev; ++l)
          if (a.lv[l].slast == S_WARP && a.partials[l])
            ((unsigned long long*)a.partials[l])[((int64_t)blockIdx.x * W + w) * 256 + bin] = wbins[w][bin];
      }
    }
    cbins[bin] = sacc;
    if (VERIFY && (a.verify & V_PARTIALS)) {
      for (int l = 0; l < a.nlev; ++l)
        if (a.lv[l].slast == S_CTA && a.partials[l])
          ((unsigned long long*)a.partials[l])[(int64_t)blockIdx.x * 256 + bin] = sacc;
    }
  }
  cluster_sync_all();
  // CTA -> cluster: reduce-scatter over DSMEM, CTA k owns a bin range
  {
    const int lo = (int)(256 * crank / K), hi = (int)(256 * (crank + 1) / K);
    for (int bin = lo + threadIdx.x; bin < hi; bin += blockDim.x) {
      unsigned long long sacc = 0;
      for (int k = 0; k < K; ++k) {
        uint32_t v;
        asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(mapa(smem_addr(&cbins[bin]), (uint32_t)k)));
        sacc += v;
      }
      parts[cl * 256 + bin] = sacc;
      if (VERIFY && (a.verify & V_PARTIALS)) {
        for (int l = 0; l < a.nlev; ++l)
          if (a.lv[l].slast == S_CLUSTER && a.partials[l]) ((unsigned long long*)a.partials[l])[cl * 256 + bin] = sacc;
      }
    }
  }
  __threadfence();
  cluster_sync_all();  // the whole cluster partial is written (and siblings done reading my bins)
  // cluster -> GPU: single pass; the leader CTA takes the ticket
  if (crank == 0) {
    if (threadIdx.x == 0) {
      const unsigned t = atomicAdd(a.grid_ticket, 1u);
      s_flag = (t == (unsigned)(a.C - 1));
      if (s_flag) __threadfence();
    }
    __syncthreads();
    if (s_flag) {
      for (int bin = threadIdx.x; bin < 256; bin += blockDim.x) {
        unsigned long long tot = 0;
        for (int64_t c = 0; c < a.C; ++c) tot += ((volatile unsigned long long*)parts)[c * 256 + bin];
        ((unsigned long long*)a.out)[bin] = tot;
        if (VERIFY && (a.verify & V_PARTIALS)) {
          for (int l = 0; l < a.nlev; ++l)
            if (a.lv[l].slast == S_GPU && a.partials[l]) ((unsigned long long*)a.partials[l])[bin] = tot;
        }
      }
      if (threadIdx.x == 0) *a.grid_ticket = 0u;
    }
  }
}

template <bool V>
cudaError_t launch_t(const NestArgs& a, int W, int tile, cudaStream_t s) {
  auto kern = hist_kernel<V>;
  const size_t smem = (size_t)kStages * tile;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.C * a.K));
  cfg.blockDim = dim3((unsigned)((W + 1) * 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, W, tile);
}

}  // namespace

bool hist_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 1 || a.keyed || a.op != OP_HIST || a.in_dtype != DT_U8) { *why = "flat u8 hist"; return false; }
  if (((uintptr_t)a.in & 15) != 0) { *why = "input not 16-byte aligned"; return false; }
  if (a.verify & V_FINGERPRINT) { *why = "fingerprints not produced by the hist kernel"; return false; }
  if (a.lane_w != 1) { *why = "lane partition"; return false; }
  LevelView v = device_levels(a);
  if (v.n != 4) { *why = "needs cluster, CTA, warp, lane levels"; return false; }
  const DevLevel *c = v.l[0], *k = v.l[1], *w = v.l[2], *l = v.l[3];
  if (!is_level(c, S_CLUSTER) || !is_level(k, S_CTA) || !is_level(w, S_WARP) || !is_level(l, S_LANE)) {
    *why = "levels not cluster/CTA/warp/lane";
    return false;
  }
  const int64_t W = a.radix[S_WARP], tile = k->chunk;
  if (l->sched != SCHED_STATIC_CHUNK || l->chunk != 16) { *why = "lane static(16)"; return false; }
  if (w->sched != SCHED_STATIC_CHUNK || w->chunk != 512) { *why = "warp static(512)"; return false; }
  if (k->sched != SCHED_STATIC_CHUNK || tile % (512 * W) != 0 || tile > 32768) { *why = "CTA static(tile)"; return false; }
  if (c->sched != SCHED_STATIC_CHUNK || c->chunk != a.K * tile) { *why = "cluster static(K*tile)"; return false; }
  if (W > 16) { *why = "W <= 16 (warp bins)"; return false; }
  return true;
}

cudaError_t launch_hist(const NestArgs& a, int W, cudaStream_t s, const char** name) {
  *name = "hist256_tma";
  const int tile = (int)device_levels(a).l[1]->chunk;
  return a.verify ? launch_t<true>(a, W, tile, s) : launch_t<false>(a, W, tile, s);
}

}  // namespace hpar
