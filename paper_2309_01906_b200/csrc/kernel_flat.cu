// kernel_flat.cu — fused flat nest reduction (configs 1 (flat form), 5).
//
// The nest shape it implements (the coalesced default):
//     GPU      static            (host: rank shard, §8(a) A2)
//     cluster  static(K*tile)    over the GPU's list
//     CTA      static(tile)      over the cluster's list
//     warp     static(32*V)      over the CTA's list        (V = 4 elements = 16 B)
//     lane     static(V)         over the warp's list
// Composed, CTA b = c*K + k owns global tiles  m*(C*K) + b  (m = 0, 1, ...)
// and lane l of warp w reads, inside each tile, the 16-byte vectors
// (r*W + w)*32 + l: exactly the owner map the oracle computes for this nest.
//
// B200 design: persistent grid of C clusters x K CTAs; one producer warp per
// CTA streams the CTA's tiles with 1-D TMA bulk copies (cp.async.bulk,
// L2 evict-first) into an S-stage shared-memory ring guarded by full/empty
// mbarriers; W consumer warps read their vectors with LDS.128 and accumulate
// (fp32 pairwise inside a vector, fp64 across vectors: §8(c) reading #6).
// The lane -> warp -> CTA -> cluster -> GPU combine runs once at the end
// (fused_common.cuh).  No GPU-scope fence inside the stream loop.
// Also served: fp32 / int32 / fp64 / int64 inputs with SUM / MIN / MAX, the
// ordered AFFINE op over int64 (every fold ascends, so the result is the
// nest's fold), and inputs 4 / 8 / 12 bytes off a 16-byte granule (MIS: the
// ring takes each tile's enclosing granules; lanes shift by the offset).
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include "fused_common.cuh"

namespace hpar {

namespace {

constexpr int kStages = 4;

// ring stage stride: a misaligned input (4, 8 or 12 bytes past a 16-byte
// granule) copies the enclosing granules, one more than the aligned tile
__host__ __device__ __forceinline__ uint32_t stage_stride(uint32_t tile_bytes, bool mis) {
  return mis ? tile_bytes + 16 : tile_bytes;
}

template <typename In, typename Acc, int OP, bool VERIFY, bool MIS, int V = 4>
__global__ void __launch_bounds__(1024, 1) flat_tma_kernel(const __grid_constant__ NestArgs a, int W,
                                                            int tile) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ ClimbSmem<Acc> csm;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = a.n0;
  const int64_t ntiles = (n + tile - 1) / tile;
  const int64_t nblocks = (int64_t)gridDim.x;
  const int64_t b = blockIdx.x;
  const int64_t my_tiles = (b < ntiles) ? (ntiles - 1 - b) / nblocks + 1 : 0;
  const In* x = (const In*)a.in;
  const uint32_t tile_bytes = (uint32_t)tile * sizeof(In);
  // misaligned input (P:252's peel, done by the copy): the ring holds the
  // granules enclosing each tile, whose elements then start at byte `mis`
  const uint32_t mis = MIS ? (uint32_t)((uintptr_t)x & 15) : 0u;
  const uint32_t stride = stage_stride(tile_bytes, MIS);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    fence_mbarrier_init_cluster();
  }
  __syncthreads();

  Acc acc = OpT<OP, Acc>::identity();
  if (warp == W) {
    // ---------------- producer warp: TMA bulk stream of the CTA's tiles ----
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int64_t j = 0; j < my_tiles; ++j) {
        const int s = (int)(j % kStages);
        if (j >= kStages) mbar_wait(&empty[s], (uint32_t)(((j / kStages) - 1) & 1));
        const int64_t t = j * nblocks + b;
        const int64_t base = t * tile;
        const int64_t len = (n - base < tile) ? (n - base) : tile;
        // TMA: multiple of 16 B; a misaligned tile takes its enclosing
        // granules (never past the granule of a valid element)
        const uint32_t bytes = MIS ? (uint32_t)((len * (int64_t)sizeof(In) + mis + 15) & ~(int64_t)15)
                                   : (uint32_t)((len * sizeof(In)) & ~(int64_t)15);
        mbar_arrive_expect_tx(&full[s], bytes);
        if (bytes)
          bulk_g2s(dsm + (size_t)s * stride, (const unsigned char*)(x + base) - mis, bytes, &full[s], pol);
      }
    }
  } else {
    // ---------------- W consumer warps ----------------------------------
    const int vec_per_tile = tile / V;  // lane chunks of V elements
    const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + b * W * 32 + threadIdx.x;
    unsigned long long fpo = 0, fpw = 0, fpn = 0;
    for (int64_t j = 0; j < my_tiles; ++j) {
      const int s = (int)(j % kStages);
      const int64_t t = j * nblocks + b;
      const int64_t base = t * tile;
      const int64_t len = (n - base < tile) ? (n - base) : tile;
      mbar_wait(&full[s], (uint32_t)((j / kStages) & 1));
      const In* st = (const In*)(dsm + (size_t)s * stride + mis);
      if (len == tile) {
        if constexpr (V != 4) {
          // lane static(1) / static(2): scalar shared loads of the lane's
          // chunk (fp32 sums pairwise inside a chunk, fp64 across)
#pragma unroll 4
          for (int f = warp * 32 + lane; f < vec_per_tile; f += W * 32) {
            In e[V];
#pragma unroll
            for (int q = 0; q < V; ++q) e[q] = st[V * f + q];
            if constexpr (OP == OP_SUM && std::is_same<In, float>::value) {
              float ps = e[0];
#pragma unroll
              for (int q = 1; q < V; ++q) ps += e[q];
              acc += (double)ps;
            } else {
              Acc c = ElemT<OP, Acc, In>::make(e[0]);
#pragma unroll
              for (int q = 1; q < V; ++q) c = OpT<OP, Acc>::combine(c, ElemT<OP, Acc, In>::make(e[q]));
              acc = OpT<OP, Acc>::combine(acc, c);
            }
            if constexpr (VERIFY) {
              for (int q = 0; q < V; ++q) {
                const int64_t it = base + V * f + q;
                if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
                if (a.verify & V_FINGERPRINT) {
                  const uint64_t g2 = a.global_begin + (uint64_t)it;
                  fpo += fp_mix(g2); fpw += fp_mix2(g2, (uint64_t)leaf); fpn += 1;
                }
              }
            }
          }
        } else if constexpr (sizeof(In) == 4 && MIS) {
          // two aligned LDS.128 per vector (conflict-free) and a uniform
          // shift: the same four elements, the same arithmetic as below
          using V = typename std::conditional<std::is_floating_point<In>::value, float4, int4>::type;
          const V* g = (const V*)(dsm + (size_t)s * stride);
          const uint32_t m4 = mis / 4;
#pragma unroll 4
          for (int f = warp * 32 + lane; f < vec_per_tile; f += W * 32) {
            const V v = shift4(g[f], g[f + 1], m4);
            if constexpr (OP == OP_SUM) {
              if constexpr (std::is_floating_point<Acc>::value) {
                acc += (double)((v.x + v.y) + (v.z + v.w));
              } else {
                acc += (long long)v.x + (long long)v.y + (long long)v.z + (long long)v.w;
              }
            } else {
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(v.x));
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(v.y));
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(v.z));
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(v.w));
            }
            if constexpr (VERIFY) {
              for (int q = 0; q < 4; ++q) {
                const int64_t it = base + 4 * f + q;
                if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
                if (a.verify & V_FINGERPRINT) {
                  const uint64_t g2 = a.global_begin + (uint64_t)it;
                  fpo += fp_mix(g2); fpw += fp_mix2(g2, (uint64_t)leaf); fpn += 1;
                }
              }
            }
          }
        } else if constexpr (sizeof(In) == 8) {
          // 8-byte elements: a lane's 4 elements are 32 bytes, two aligned
          // LDS.128 (three when the input sits 8 bytes off a granule)
          using V = typename std::conditional<std::is_floating_point<In>::value, double2, longlong2>::type;
          const V* g = (const V*)(dsm + (size_t)s * stride);
#pragma unroll 2
          for (int f = warp * 32 + lane; f < vec_per_tile; f += W * 32) {
            V lo, hi;
            if constexpr (MIS) {
              const V a0 = g[2 * f], a1 = g[2 * f + 1], a2 = g[2 * f + 2];
              lo.x = a0.y; lo.y = a1.x; hi.x = a1.y; hi.y = a2.x;
            } else {
              lo = g[2 * f];
              hi = g[2 * f + 1];
            }
            if constexpr (OP == OP_SUM) {
              acc += (lo.x + lo.y) + (hi.x + hi.y);  // integers: two's complement, wraps mod 2^64
            } else {
              // a tree over the four (associative: the same result as the
              // in-order fold, also for the ordered AFFINE op) keeps the
              // dependent chain on acc to one combine per vector
              using E = ElemT<OP, Acc, In>;
              using O = OpT<OP, Acc>;
              acc = O::combine(acc, O::combine(O::combine(E::make(lo.x), E::make(lo.y)),
                                               O::combine(E::make(hi.x), E::make(hi.y))));
            }
            if constexpr (VERIFY) {
              for (int q = 0; q < 4; ++q) {
                const int64_t it = base + 4 * f + q;
                if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
                if (a.verify & V_FINGERPRINT) {
                  const uint64_t g2 = a.global_begin + (uint64_t)it;
                  fpo += fp_mix(g2); fpw += fp_mix2(g2, (uint64_t)leaf); fpn += 1;
                }
              }
            }
          }
        } else if constexpr (sizeof(In) == 4) {
#pragma unroll 4
          for (int f = warp * 32 + lane; f < vec_per_tile; f += W * 32) {
            if constexpr (OP == OP_SUM) {
              if constexpr (std::is_floating_point<Acc>::value) {  // fp32 pairwise, then fp64
                const float4 v = ((const float4*)st)[f];
                acc += (double)((v.x + v.y) + (v.z + v.w));
              } else {
                const int4 v = ((const int4*)st)[f];
                acc += (long long)v.x + (long long)v.y + (long long)v.z + (long long)v.w;
              }
            } else {
              const In* e = st + 4 * f;
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[0]));
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[1]));
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[2]));
              acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[3]));
            }
            if constexpr (VERIFY) {
              for (int q = 0; q < 4; ++q) {
                const int64_t it = base + 4 * f + q;
                if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
                if (a.verify & V_FINGERPRINT) {
                  const uint64_t g = a.global_begin + (uint64_t)it;
                  fpo += fp_mix(g); fpw += fp_mix2(g, (uint64_t)leaf); fpn += 1;
                }
              }
            }
          }
        }
      } else {
        // ragged last tile: bulk part from smem, the < 16 B tail from global
        const int64_t in_smem = MIS ? len : (len * (int64_t)sizeof(In)) / 16 * 16 / (int64_t)sizeof(In);
        for (int f = warp * 32 + lane; f < vec_per_tile; f += W * 32) {
          for (int q = 0; q < V; ++q) {
            const int64_t off = V * (int64_t)f + q;
            if (off >= len) break;
            const In e = (off < in_smem) ? st[off] : x[base + off];
            acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e));
            if constexpr (VERIFY) {
              const int64_t it = base + off;
              if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
              if (a.verify & V_FINGERPRINT) {
                const uint64_t g = a.global_begin + (uint64_t)it;
                fpo += fp_mix(g); fpw += fp_mix2(g, (uint64_t)leaf); fpn += 1;
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if constexpr (VERIFY) {
      if (a.verify & V_FINGERPRINT) {
        atomicAdd(&a.fp[0], fpo);
        atomicAdd(&a.fp[1], fpw);
        atomicAdd(&a.fp[2], fpn);
      }
    }
  }
  __syncwarp();
  fused_total_climb<OP, Acc>(a, acc, W, csm);
}

int g_flat_tile = 4096;

template <typename In, typename Acc, int OP, bool VERIFY, bool MIS, int V>
cudaError_t launch_t(const NestArgs& a, int W, int tile, cudaStream_t s) {
  auto kern = flat_tma_kernel<In, Acc, OP, VERIFY, MIS, V>;
  const size_t smem = (size_t)kStages * stage_stride((uint32_t)(tile * sizeof(In)), MIS);
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

template <typename In, typename Acc, int OP>
cudaError_t launch_v(const NestArgs& a, int W, int tile, cudaStream_t s) {
  int64_t tile_unused, v64 = 4;
  const char* why;
  flat_nest_shape(a, &why, &tile_unused, &v64);
  const int v = (int)v64;  // the lane chunk: 1, 2 or 4
  const bool mis = ((uintptr_t)a.in & 15) != 0;
  auto go = [&](auto v_c) -> cudaError_t {
    constexpr int VV = decltype(v_c)::value;
    if (mis)
      return a.verify ? launch_t<In, Acc, OP, true, true, VV>(a, W, tile, s) : launch_t<In, Acc, OP, false, true, VV>(a, W, tile, s);
    return a.verify ? launch_t<In, Acc, OP, true, false, VV>(a, W, tile, s) : launch_t<In, Acc, OP, false, false, VV>(a, W, tile, s);
  };
  if (v == 1) return go(std::integral_constant<int, 1>());
  if (v == 2) return go(std::integral_constant<int, 2>());
  return go(std::integral_constant<int, 4>());
}

}  // namespace

// Does the nest have the coalesced flat shape (and the call suit the kernel)?
bool flat_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 1 || a.keyed) { *why = "not a flat total"; return false; }
  if (a.op == OP_HIST) { *why = "sum/min/max/affine only"; return false; }
  if (a.op == OP_AFFINE && a.in_dtype != DT_I64) { *why = "affine: int64 input"; return false; }
  if (a.in_dtype != DT_F32 && a.in_dtype != DT_I32 && a.in_dtype != DT_F64 && a.in_dtype != DT_I64) {
    *why = "dtype";
    return false;
  }
  const int64_t esz = (a.in_dtype == DT_F64 || a.in_dtype == DT_I64) ? 8 : 4;
  if (((uintptr_t)a.in & (esz - 1)) != 0) { *why = "input not element-aligned"; return false; }
  if (a.lane_w != 1) { *why = "lane partition"; return false; }
  int64_t tile, V;
  if (!flat_nest_shape(a, why, &tile, &V)) return false;
  if (V != 1 && V != 2 && V != 4) { *why = "lane chunk must be 1, 2 or 4"; return false; }
  const int64_t W = a.radix[S_WARP];
  if (tile % (32 * V * W) != 0 || tile * esz > 32768) {
    *why = "tile must be a multiple of 32*V*W, <= 32 KiB";
    return false;
  }
  if (W > 31) { *why = "W > 31 (one producer warp is added)"; return false; }
  return true;
}

cudaError_t launch_flat(const NestArgs& a, int W, cudaStream_t s, const char** name) {
  int64_t tile64 = 0, v64 = 0;
  const char* why;
  if (!flat_nest_shape(a, &why, &tile64, &v64)) return cudaErrorInvalidValue;
  const int tile = (int)tile64;
  *name = "flat_tma";
  if (a.in_dtype == DT_F32) {
    if (a.op == OP_SUM) return launch_v<float, double, OP_SUM>(a, W, tile, s);
    if (a.op == OP_MIN) return launch_v<float, double, OP_MIN>(a, W, tile, s);
    if (a.op == OP_MAX) return launch_v<float, double, OP_MAX>(a, W, tile, s);
  } else if (a.in_dtype == DT_F64) {
    if (a.op == OP_SUM) return launch_v<double, double, OP_SUM>(a, W, tile, s);
    if (a.op == OP_MIN) return launch_v<double, double, OP_MIN>(a, W, tile, s);
    if (a.op == OP_MAX) return launch_v<double, double, OP_MAX>(a, W, tile, s);
  } else if (a.in_dtype == DT_I64) {
    if (a.op == OP_SUM) return launch_v<long long, long long, OP_SUM>(a, W, tile, s);
    if (a.op == OP_AFFINE) return launch_v<long long, Aff, OP_AFFINE>(a, W, tile, s);
    if (a.op == OP_MIN) return launch_v<long long, long long, OP_MIN>(a, W, tile, s);
    if (a.op == OP_MAX) return launch_v<long long, long long, OP_MAX>(a, W, tile, s);
  } else {
    if (a.op == OP_SUM) return launch_v<int32_t, long long, OP_SUM>(a, W, tile, s);
    if (a.op == OP_MIN) return launch_v<int32_t, long long, OP_MIN>(a, W, tile, s);
    if (a.op == OP_MAX) return launch_v<int32_t, long long, OP_MAX>(a, W, tile, s);
  }
  return cudaErrorInvalidValue;
}

// clusters of K CTAs of the flat kernel (W consumer warps + the producer,
// the 4-stage ring of g_flat_tile fp32) that fit on the device at once
// (cudaOccupancyMaxActiveClusters: counts SMs, per-SM residency and the GPC
// placement of clusters).  0 on error.
int flat_max_active_clusters(int K, int W) {
  auto kern = flat_tma_kernel<float, double, OP_SUM, false, false>;
  const size_t smem = (size_t)kStages * g_flat_tile * 4;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (K > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)K);
  cfg.blockDim = dim3((unsigned)((W + 1) * 32));
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return 0;
  return n;
}

int flat_resident_ctas_per_sm(int W) {
  int n = 0;
  auto kern = flat_tma_kernel<float, double, OP_SUM, false, false>;
  const size_t smem = (size_t)kStages * g_flat_tile * 4;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 2;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, (W + 1) * 32, smem) != cudaSuccess || n < 1) return 2;
  return n;
}

}  // namespace hpar
