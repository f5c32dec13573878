// kernel_hist.cu — level-scoped 256-bin histogram (config 4).
//
// Nest shape (flat, uint8; V = 16 bytes per lane vector):
//     GPU      static            (host: rank shard)
//     cluster  static(K*tile)
//     CTA      static(tile)
//     warp     static(512)       (32 lanes x 16 B)
//     lane     static(16)
// Privatisation per level:
//     lane    : its own 256 u32 counters.  Warps 2p and 2p+1 share a 64 KiB
//               region laid out [bin][warp & 1][lane] (256-byte bin rows), so
//               lane l always hits bank l: no bank conflicts and no two lanes
//               on one address, whatever the data (skewed or all-zero inputs
//               cost the same).  A counter's offset in the region is
//               bin << 8 | (warp & 1) << 7 | lane << 2: ONE byte permute
//               (PRMT) of the data word with the lane's column gives it, so an
//               increment is PRMT + one fire-and-forget shared atomic
//               (red.shared, no return value).  With W > 6 consumer warps
//               (the timed geometry: W = 8) the pairs share R = 2 regions
//               round robin: pair p uses region p mod R, so a counter sums
//               the same lane column of W / (2R) warps.  The atomics keep
//               that exact; the lane and warp levels are then folded inside
//               the shared counters and not materialised, which is why
//               lane / warp partials (verify) require private regions.
//     warp    : sum of its 32 lanes' counters (rotated reads, conflict-free)
//     CTA     : sum of its warps' bins (ascending warp), bar.sync
//     cluster : reduce-scatter over DSMEM — CTA k owns bins [256k/K, 256(k+1)/K)
//               and sums them over the K CTAs (ascending), barrier.cluster
//     GPU     : u64 cluster partials + single-pass ticket; the last cluster
//               folds them in ascending cluster order
//     node    : ncclAllReduce of 256 u64 (runtime.cpp)
// Input stream: producer warp + 1-D TMA bulk ring as in kernel_flat.cu.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <algorithm>
#include <type_traits>
#include "fused_common.cuh"

namespace hpar {
namespace {

constexpr int kStages = 8;  // TMA ring stages at most (fewer when the lane tables leave less room)
constexpr int kSmemBudget = 227 * 1024 - 8 * 1024;  // dynamic smem next to the static arrays
constexpr int kMaxW = 16;  // consumer warps (private tables: W <= 6, 3 x 64 KiB regions)
constexpr int kMaxPrivW = 6;
constexpr int kRegion = 65536;  // lane tables of a warp pair
// ring stage stride: a misaligned input copies one more 16-byte granule per tile
__host__ __device__ __forceinline__ int ring_stride(int tile, uint32_t mis) { return mis ? tile + 16 : tile; }
__host__ __device__ __forceinline__ int ring_stages(int R, int stride) {
  const int room = (kSmemBudget - R * kRegion) / stride;
  return room < kStages ? room : kStages;
}
// offset of counter (bin, lane) of `warp` inside its pair's region, in words
__device__ __forceinline__ int tab_word(int bin, int warp, int lane) { return bin * 64 + (warp & 1) * 32 + lane; }

__device__ __forceinline__ void inc_shared(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}

// Verify only, shared lane-table regions (R < pairs): the lane and warp
// levels are folded inside the shared counters, so their partials are built
// here instead — every byte a lane counts is also added to its lane's and its
// warp's partial bins in global memory (u64 atomics; exact, slow, verify
// runs only).  Layout as the tables' export: [CTA*W*32 + warp*32 + lane][256]
// and [CTA*W + warp][256].
template <bool VERIFY>
struct InnerDirect {
  unsigned long long* lanep = nullptr;
  unsigned long long* warpp = nullptr;
  __device__ __forceinline__ InnerDirect(const NestArgs& a, int W, int R) {
    if constexpr (VERIFY) {
      if (!(a.verify & V_PARTIALS) || R == (W + 1) / 2) return;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int lv = 0; lv < a.nlev; ++lv) {
        if (!a.partials[lv]) continue;
        if (a.lv[lv].slast == S_LANE_IN)
          lanep = (unsigned long long*)a.partials[lv] + ((int64_t)blockIdx.x * W * 32 + warp * 32 + lane) * 256;
        if (a.lv[lv].slast == S_WARP) warpp = (unsigned long long*)a.partials[lv] + ((int64_t)blockIdx.x * W + warp) * 256;
      }
      // the bins start at zero (each lane clears its own row and an eighth of
      // its warp's; the warp's lanes meet before any count is added)
      for (int k = 0; k < 256; ++k)
        if (lanep) lanep[k] = 0ull;
      for (int k = lane; k < 256; k += 32)
        if (warpp) warpp[k] = 0ull;
      __syncwarp();
    }
  }
  __device__ __forceinline__ void add(uint32_t byte) const {
    if constexpr (VERIFY) {
      if (lanep) atomicAdd(lanep + byte, 1ull);
      if (warpp) atomicAdd(warpp + byte, 1ull);
    }
  }
};

// lane -> warp -> CTA -> cluster -> GPU (-> node) of the per-lane tables,
// shared by the TMA-ring and register-streaming kernels.  `counts`: the R
// lane-table regions; `wbins`: W x 256 u32 scratch; the caller has synced the
// CTA after the stream.  Lane / warp partials come from the tables only when
// every warp pair has its own region (R == pairs); with shared regions the
// verify stream adds them to the partial arrays directly (see inner_direct).
template <bool VERIFY>
__device__ __forceinline__ void hist_climb(const NestArgs& a, int W, int R, const uint32_t* counts,
                                           uint32_t (*wbins)[256], uint32_t* cbins, int& s_flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K;
  const uint32_t crank = cluster_ctarank();
  const int64_t cl = blockIdx.x / K;
  const bool tab_inner = R == (W + 1) / 2;  // lane / warp levels materialised in the tables
  // lane -> warp: warp w sums the 32 lane columns of its table; lane l owns
  // bins l, l+32, ...; rotated column order keeps the reads conflict-free.
  // With shared regions the first 2R warps read the (region, column) tables
  // and the others contribute zero bins.
  if (warp < W && warp >= 2 * R) {
    for (int bin = lane; bin < 256; bin += 32) wbins[warp][bin] = 0;
  } else if (warp < W) {
    const uint32_t* tab = counts + (size_t)(warp >> 1) * (kRegion / 4);
    for (int bin = lane; bin < 256; bin += 32) {
      uint32_t sacc = 0;
      for (int k = 0; k < 32; ++k) {
        const int l = (k + lane) & 31;
        const uint32_t v = tab[tab_word(bin, warp, l)];
        sacc += v;
        if (VERIFY && (a.verify & V_PARTIALS) && tab_inner) {
          for (int lv = 0; lv < a.nlev; ++lv)
            if (a.lv[lv].slast == S_LANE_IN && a.partials[lv])
              ((unsigned long long*)a.partials[lv])[((int64_t)blockIdx.x * W * 32 + warp * 32 + l) * 256 + bin] = v;
        }
      }
      wbins[warp][bin] = sacc;
      if (VERIFY && (a.verify & V_PARTIALS) && tab_inner) {
        for (int lv = 0; lv < a.nlev; ++lv)
          if (a.lv[lv].slast == S_WARP && a.partials[lv])
            ((unsigned long long*)a.partials[lv])[((int64_t)blockIdx.x * W + warp) * 256 + bin] = sacc;
      }
    }
  }
  __syncthreads();
  // warp -> CTA (ascending warp)
  unsigned long long* parts = (unsigned long long*)a.cluster_partials;
  for (int bin = threadIdx.x; bin < 256; bin += blockDim.x) {
    uint32_t sacc = 0;
    for (int w = 0; w < W; ++w) sacc += wbins[w][bin];
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
      constexpr int NB = 4;  // bins per thread (blockDim.x >= 64)
      unsigned long long tot[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int bin = threadIdx.x + j * blockDim.x;
        tot[j] = 0;
        if (bin >= 256) continue;
        for (int64_t c = 0; c < a.C; ++c) tot[j] += ((volatile unsigned long long*)parts)[c * 256 + bin];
        if (VERIFY && (a.verify & V_PARTIALS)) {
          for (int l = 0; l < a.nlev; ++l)
            if (a.lv[l].slast == S_GPU && a.partials[l]) ((unsigned long long*)a.partials[l])[bin] = tot[j];
        }
      }
      if (a.node_dc) node_fold_bins<NB>(a, tot);  // the node level in-kernel (f1)
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int bin = threadIdx.x + j * blockDim.x;
        if (bin < 256) ((unsigned long long*)a.out)[bin] = tot[j];
      }
      if (threadIdx.x == 0) *a.grid_ticket = 0u;
    }
  }
}

// VPL: 16-byte vectors per lane per tile (tile == 512*W*VPL), 0 = generic
template <bool VERIFY, int VPL>
// R = lane-table regions: (W+1)/2 (every warp pair its own region: the
// lane and warp levels materialised, required for VERIFY) or fewer, shared
// round robin by the pairs (the atomics make sharing exact; the warp level is
// then folded into the shared counters and not materialised)
__global__ void __launch_bounds__(1024, 1) hist_kernel(const __grid_constant__ NestArgs a, int W, int tile, int nst, int R) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
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
  const uint32_t mis = (uint32_t)((uintptr_t)x & 15);  // misaligned input: byte path (P:252 peel)
  const int stride = ring_stride(tile, mis);
  const uint32_t crank = cluster_ctarank();
  const int64_t cl = blockIdx.x / K;
  // dynamic smem: the lane-table regions first (their shared addresses are
  // link-time constants, so a region base folds into the atomic's immediate
  // offset), then the TMA ring
  uint32_t* counts = (uint32_t*)dsm;  // [R][256][2][32]
  unsigned char* ring = dsm + (size_t)R * kRegion;
  // the warp bins reuse the ring once the stream is consumed (nst >= 2 tiles
  // of >= 512 W bytes >= W x 256 u32)
  uint32_t(*wbins)[256] = (uint32_t(*)[256])ring;

  for (int i = threadIdx.x; i < R * (kRegion / 4); i += blockDim.x) counts[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    fence_mbarrier_init_cluster();
  }
  __syncthreads();

  if (warp == W) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int64_t j = 0; j < my_tiles; ++j) {
        if (j >= nst) mbar_wait(&empty[s], ph ^ 1);
        const int64_t base = (j * nblocks + b) * tile;
        const int64_t len = (n - base < tile) ? (n - base) : tile;
        // misaligned input: copy the enclosing 16-byte granules (never past
        // the granule of a valid byte); the tile's bytes then start at `mis`
        const uint32_t bytes = mis ? (uint32_t)((len + mis + 15) & ~(int64_t)15) : (uint32_t)(len & ~(int64_t)15);
        mbar_arrive_expect_tx(&full[s], bytes);
        if (bytes) bulk_g2s(ring + (size_t)s * stride, x + base - mis, bytes, &full[s], pol);
        if (++s == nst) { s = 0; ph ^= 1; }
      }
    }
  } else {
   // the pair's region (a compile-time constant per PAIR instance) and this
   // lane's column (byte 0 of every counter offset; PRMT puts the data byte
   // in byte 1): an increment is PRMT + RED [reg + imm]
   auto consume = [&](auto pair_c) {
    constexpr int PAIR = decltype(pair_c)::value;
    const uint32_t region = smem_addr(dsm) + (uint32_t)PAIR * kRegion;
    const uint32_t col = (uint32_t)((warp & 1) * 128 + lane * 4);
#define HPAR_INC(w, k) inc_shared(region + __byte_perm((w), col, 0x5504u | ((k) << 4)))
    const int nvec = tile / 16;
    const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + b * W * 32 + threadIdx.x;
    unsigned long long fpo = 0, fpw = 0, fpn = 0;  // verify: coverage fingerprints
    InnerDirect<VERIFY> inner(a, W, R);
    auto visit = [&](int64_t it, uint32_t byte) {  // verify bookkeeping of one iteration (byte) of this lane
      if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
      if (a.verify & V_FINGERPRINT) {
        const uint64_t g = a.global_begin + (uint64_t)it;
        fpo += fp_mix(g); fpw += fp_mix2(g, (uint64_t)leaf); fpn += 1;
      }
      inner.add(byte);
    };
    int s = 0;
    uint32_t ph = 0;
    for (int64_t j = 0; j < my_tiles; ++j) {
      const int64_t base = (j * nblocks + b) * tile;
      const int64_t len = (n - base < tile) ? (n - base) : tile;
      mbar_wait(&full[s], ph);
      const unsigned char* st = ring + (size_t)s * stride + mis;
      if (len == tile && VPL > 0 && !mis) {
        // all of this lane's vectors of the tile first (ILP over the smem
        // latency), then the increments
        uint4 vv[VPL > 0 ? VPL : 1];
#pragma unroll
        for (int q = 0; q < VPL; ++q) vv[q] = ((const uint4*)st)[(q * W + warp) * 32 + lane];
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const uint32_t w4[4] = {vv[q].x, vv[q].y, vv[q].z, vv[q].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t w = w4[k];
            HPAR_INC(w, 0);
            HPAR_INC(w, 1);
            HPAR_INC(w, 2);
            HPAR_INC(w, 3);
          }
        }
        if constexpr (VERIFY) {
          for (int f = warp * 32 + lane; f < nvec; f += W * 32)
            for (int e = 0; e < 16; ++e) visit(base + 16 * f + e, st[16 * f + e]);
        }
      } else if (len == tile && !mis) {
#pragma unroll 2
        for (int f = warp * 32 + lane; f < nvec; f += W * 32) {
          const uint4 v = ((const uint4*)st)[f];
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t w = w4[k];
            HPAR_INC(w, 0);
            HPAR_INC(w, 1);
            HPAR_INC(w, 2);
            HPAR_INC(w, 3);
          }
          if constexpr (VERIFY) {
            for (int e = 0; e < 16; ++e) visit(base + 16 * f + e, st[16 * f + e]);
          }
        }
      } else {
        const int64_t in_smem = mis ? len : (len & ~(int64_t)15);
        for (int f = warp * 32 + lane; f < nvec; f += W * 32) {
          for (int e = 0; e < 16; ++e) {
            const int64_t off = 16 * (int64_t)f + e;
            if (off >= len) break;
            const uint32_t byte = off < in_smem ? st[off] : x[base + off];
            inc_shared(region + col + (byte << 8));
            if constexpr (VERIFY) visit(base + off, byte);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == nst) { s = 0; ph ^= 1; }
    }
    if constexpr (VERIFY) {
      if (a.verify & V_FINGERPRINT) {
        atomicAdd(&a.fp[0], fpo);
        atomicAdd(&a.fp[1], fpw);
        atomicAdd(&a.fp[2], fpn);
      }
    }
   };
    switch ((warp >> 1) % R) {
      case 0: consume(std::integral_constant<int, 0>()); break;
      case 1: consume(std::integral_constant<int, 1>()); break;
      default: consume(std::integral_constant<int, 2>()); break;
    }
  }
  __syncwarp();
  __syncthreads();
#undef HPAR_INC
  hist_climb<VERIFY>(a, W, R, counts, wbins, cbins, s_flag);
}

template <bool V, int VPL>
cudaError_t launch_t(const NestArgs& a, int W, int tile, int R, cudaStream_t s) {
  auto kern = hist_kernel<V, VPL>;
  const int stride = ring_stride(tile, (uint32_t)((uintptr_t)a.in & 15));
  const int nst = ring_stages(R, stride);
  const size_t smem = (size_t)nst * stride + (size_t)R * kRegion;
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
  return cudaLaunchKernelEx(&cfg, kern, a, W, tile, nst, R);
}

}  // namespace

// lane or warp partials requested: those levels must be materialised
static bool inner_partials(const NestArgs& a) {
  if (!(a.verify & V_PARTIALS)) return false;
  for (int l = 0; l < a.nlev; ++l)
    if ((a.lv[l].slast == S_LANE_IN || a.lv[l].slast == S_WARP) && a.partials[l]) return true;
  return false;
}

// lane-table regions: private per warp pair when lane / warp partials are
// requested (or W <= 6 and HPAR_C4_REGIONS unset), else
// min(HPAR_C4_REGIONS or 2, pairs): two 64 KiB regions leave room for a
// 5-stage ring of 16 KiB tiles (W = 8: 0.69 ms vs 0.78 ms with one region
// and 1.25 ms with three, whose ring is 2 stages deep; scripts/sweep_hist2.sh)
static int hist_regions(const NestArgs& a, int W) {
  const int pairs = (W + 1) / 2;
  static int knob = -2;
  if (knob == -2) knob = getenv("HPAR_C4_REGIONS") ? atoi(getenv("HPAR_C4_REGIONS")) : -1;
  if (inner_partials(a) && W <= kMaxPrivW) return pairs;  // the tables hold the lane / warp levels
  int r = knob > 0 ? knob : (W <= kMaxPrivW ? pairs : 2);
  if (r > 3) r = 3;
  return r < pairs ? r : pairs;
}

bool hist_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 1 || a.keyed || a.op != OP_HIST || a.in_dtype != DT_U8) { *why = "flat u8 hist"; return false; }
  if (a.lane_w != 1) { *why = "lane partition"; return false; }
  // the flat shape in any spelling (separate or collapsed cluster..CTA and
  // warp..lane levels), lane chunks of 16 bytes
  int64_t tile, V;
  if (!flat_nest_shape(a, why, &tile, &V)) return false;
  const int64_t W = a.radix[S_WARP];
  if (V != 16) { *why = "lane static(16) (warp static(512))"; return false; }
  if (tile % (512 * W) != 0 || tile > 32768) { *why = "CTA static(tile), a multiple of 512*W, <= 32 KiB"; return false; }
  const int R = hist_regions(a, (int)W);
  if (W > kMaxW || ring_stages(R, (int)tile + 16) < 2) {
    *why = "W <= 16 consumer warps";
    return false;
  }
  return true;
}

cudaError_t launch_hist(const NestArgs& a, int W, cudaStream_t s, const char** name) {
  *name = "hist256_lanepriv_tma";
  int64_t tile64 = 0, v64 = 0;
  const char* why;
  if (!flat_nest_shape(a, &why, &tile64, &v64)) return cudaErrorInvalidValue;
  const int tile = (int)tile64;
  const int vpl = (tile % (512 * W) == 0) ? tile / (512 * W) : 0;
  const int R = hist_regions(a, W);
  if (a.verify) {
    switch (vpl) {
      case 2: return launch_t<true, 2>(a, W, tile, R, s);
      case 4: return launch_t<true, 4>(a, W, tile, R, s);
      case 8: return launch_t<true, 8>(a, W, tile, R, s);
      default: return launch_t<true, 0>(a, W, tile, R, s);
    }
  }
  switch (vpl) {
    case 1: return launch_t<false, 1>(a, W, tile, R, s);
    case 2: return launch_t<false, 2>(a, W, tile, R, s);
    case 3: return launch_t<false, 3>(a, W, tile, R, s);
    case 4: return launch_t<false, 4>(a, W, tile, R, s);
    case 8: return launch_t<false, 8>(a, W, tile, R, s);
    case 16: return launch_t<false, 16>(a, W, tile, R, s);
    default: return launch_t<false, 0>(a, W, tile, R, s);
  }
}

}  // namespace hpar
