// kernel_rowwise.cu — fused 4-level row-wise nest reduction (config 2).
//
// Nest shape (SURVEY §8(a) A3, §8(c) reading #13):
//     GPU      static        loop 0 (rows; host: rank shard)
//     cluster  static        loop 0: a contiguous block of rows per cluster
//     CTA      static        loop 1: a contiguous block of n1/K columns
//     warp     static(128)   loop 1
//     lane     static(4)     loop 1
// One result per row (keyed by loop 0): the row owner is the cluster, whose
// CTAs, warps and lanes combine every row.  SUM / MIN / MAX over
// fp32 (the config-2 case, fp32 lane/warp tree), fp64, int32 and int64
// (64-bit partials, 8-byte DSMEM slots).
//
// B200 design (per cluster, per row):
//   * each CTA's producer warp streams its n1/K-column segment of the row
//     with one 1-D TMA bulk copy into an S-stage smem ring (full/empty
//     mbarriers), L2 evict-first;
//   * lane level: each lane sums its NV float4s in fp32; lane -> warp: xor
//     butterfly (lane 0 receives exactly the ordered tree
//     ((x0+x1)+(x2+x3))+..., §8(c) reading #4) in fp32 — a warp's share of a
//     row is 128*NV elements, so the worst-case relative error of a warp
//     partial is (4*NV + 4) u <= 2.2e-6 for NV <= 8 (reading #6);
//   * warp -> CTA -> cluster: every warp's lane 0 pushes its warp partial with
//     st.async into the LEADER CTA's slot ring over DSMEM; the store itself
//     completes the leader's per-row mbarrier (complete_tx): the warp- and
//     CTA-level barriers are transaction barriers, no bar.sync or
//     barrier.cluster in the row loop;
//   * a combiner warp in the leader CTA folds 32/(K*W) rows per pass in fp64
//     (warp partials -> CTA partials -> row, ascending), writes the rows and
//     frees their slots with relaxed remote arrives on every CTA's
//     slot-empty mbarrier (a .release arrive would cost a MEMBAR.ALL.GPU).
// The slot ring holds kSlots rows, so combining row j overlaps the loads of
// rows j+1 .. j+S.  Cluster barriers only at start-up and exit.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <type_traits>
#include "fused_common.cuh"

namespace hpar {
namespace {

constexpr int kMaxStages = 16;  // TMA ring depth bound (rows in flight per CTA)
constexpr int kSlots = 16;      // DSMEM row-slot ring depth in the leader
constexpr int kMaxPush = 32;    // K*W <= 32 warp partials per row


// NV (fp32 sums): float4 vectors per lane per row (qcols == 128*W*NV);
// 0 = generic loop; -1 = ragged rows: any n1, ld and element-aligned input.
// Then the CTAs' column blocks follow the static partition (the first
// n1 % K CTAs take one column more), a CTA's segment of a row may start
// anywhere in a 16-byte granule, so the producer copies the enclosing
// granules and the lanes shift by the row's offset (load_quad).
bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// the lane chunk V of the columns' warp / lane part — warp static(32V) +
// lane static(V), or one collapsed warp..lane level static(V) (the same
// chunk -> thread map) — or -1
int rowwise_lane_chunk(const NestArgs& a) {
  LevelView v = device_levels(a);
  int64_t V = -1;
  if (v.n == 4) {
    const DevLevel *w = v.l[2], *l = v.l[3];
    if (!is_level(w, S_WARP) || !is_level(l, S_LANE) || w->loop != 1 || l->loop != 1) return -1;
    if (w->sched != SCHED_STATIC_CHUNK || l->sched != SCHED_STATIC_CHUNK || w->chunk != 32 * l->chunk) return -1;
    V = l->chunk;
  } else if (v.n == 3) {
    const DevLevel* t = v.l[2];
    if (t->sfirst != S_WARP || t->slast != S_LANE_IN || t->loop != 1 || t->sched != SCHED_STATIC_CHUNK) return -1;
    V = t->chunk;
  }
  return (V == 1 || V == 2 || V == 4) ? (int)V : -1;
}

int elem_bytes(const NestArgs& a) { return (a.in_dtype == DT_F64 || a.in_dtype == DT_I64) ? 8 : 4; }

// rows the aligned path cannot copy whole: n1 not a multiple of 4K, or rows
// (ld, the base pointer) off 16-byte boundaries
bool rowwise_ragged(const NestArgs& a) {
  const int64_t esz = elem_bytes(a);
  return a.n1 % (4 * a.K) != 0 || (a.ld * esz) % 16 != 0 || ((uintptr_t)a.in & 15) != 0;
}

// ring-stage stride in bytes: the aligned path's n1/K columns; a ragged
// segment of up to ceil(n1/K) columns starting anywhere in a granule needs
// one granule more
int64_t rowwise_stage_bytes(const NestArgs& a) {
  const int64_t esz = elem_bytes(a);
  if (!rowwise_ragged(a)) return a.n1 / a.K * esz;
  const int64_t qmax = (a.n1 + a.K - 1) / a.K;
  // the lanes read whole 16-byte granules: a 4-element vector spans
  // esz / 4 granules plus one for the shift, so the last (partial) vector
  // reaches granule (esz / 4) * ceil(qmax / 4) — allocate through it
  return ((qmax + 3) / 4 * (esz / 4) + 1) * 16;
}

// Element and partial types.  In: the input element; P: the lane / warp
// partial and the DSMEM slot (fp32 for fp32 sums — the fp32 tree of reading
// #4 — else the 64-bit accumulator); X: the combiner's and the exported
// partials' type (fp64 for floating point, int64 for integers).
template <typename In, int OP> struct RwX { using T = long long; };
template <int OP> struct RwX<float, OP> { using T = double; };
template <int OP> struct RwX<double, OP> { using T = double; };
template <> struct RwX<long long, OP_AFFINE> { using T = Aff; };  // the ordered op (NEXT f2)
template <typename In, int OP>
using RwP = typename std::conditional<std::is_same<In, float>::value && OP == OP_SUM, float,
                                      typename RwX<In, OP>::T>::type;

// xor shuffles that also move the 16-byte ordered accumulator; lane 0's
// butterfly combines (own, higher lanes) at every step: the ordered tree
template <typename T>
__device__ __forceinline__ T shfl_xor_t(T v, int off) { return __shfl_xor_sync(0xffffffffu, v, off); }
template <>
__device__ __forceinline__ Aff shfl_xor_t<Aff>(Aff v, int off) {
  return Aff{__shfl_xor_sync(0xffffffffu, v.a, off), __shfl_xor_sync(0xffffffffu, v.b, off)};
}

// the four elements of lane vector f (elements 4f .. 4f+3 of the CTA's
// block), from a ring stage whose data start `mis` bytes into its first
// 16-byte granule (0 unless ragged)
template <typename In, bool RAG>
__device__ __forceinline__ void load_quad(const unsigned char* stage, int f, uint32_t mis, In (&e)[4]) {
  if constexpr (sizeof(In) == 4) {
    using V = typename std::conditional<std::is_floating_point<In>::value, float4, int4>::type;
    const V* g = (const V*)stage;
    V t = g[f];
    if (RAG && mis) t = shift4(t, g[f + 1], mis >> 2);
    e[0] = t.x; e[1] = t.y; e[2] = t.z; e[3] = t.w;
  } else {
    using V = typename std::conditional<std::is_floating_point<In>::value, double2, longlong2>::type;
    const V* g = (const V*)stage;
    if (RAG && mis) {
      const V a0 = g[2 * f], a1 = g[2 * f + 1], a2 = g[2 * f + 2];
      e[0] = a0.y; e[1] = a1.x; e[2] = a1.y; e[3] = a2.x;
    } else {
      const V lo = g[2 * f], hi = g[2 * f + 1];
      e[0] = lo.x; e[1] = lo.y; e[2] = hi.x; e[3] = hi.y;
    }
  }
}

__device__ __forceinline__ void st_async_part(uint32_t addr, uint32_t bar, float v) {
  st_async_u32(addr, bar, __float_as_uint(v));
}
__device__ __forceinline__ void st_async_part(uint32_t addr, uint32_t bar, double v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async_part(uint32_t addr, uint32_t bar, long long v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr), "l"(v),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async_part(uint32_t addr, uint32_t bar, Aff v) {  // two 8-byte transactions
  st_async_part(addr, bar, (long long)v.a);
  st_async_part(addr + 8, bar, (long long)v.b);
}

template <typename X>
__device__ __forceinline__ void store_row(const NestArgs& a, int64_t row, X v) {
  if constexpr (std::is_same<X, Aff>::value) {
    ((Aff*)a.out)[row] = v;  // u64 [rows][2]
    return;
  } else
  switch (a.out_dtype) {
    case DT_F32: ((float*)a.out)[row] = (float)v; break;
    case DT_F64: ((double*)a.out)[row] = (double)v; break;
    default: ((long long*)a.out)[row] = (long long)v; break;
  }
}

template <typename In, int OP, bool VERIFY, int NV, int V = 4>
__global__ void __launch_bounds__(1024, 1)
    rowwise_kernel(const __grid_constant__ NestArgs a, int W, int qcols, int kStages, int stage_bytes) {
  using P = RwP<In, OP>;
  using X = typename RwX<In, OP>::T;
  constexpr bool F32SUM = std::is_same<P, float>::value;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ __align__(8) uint64_t row_full[kSlots], slot_empty[kSlots];
  __shared__ __align__(8) P slot[kSlots][kMaxPush];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K;
  const uint32_t crank = cluster_ctarank();
  const int64_t c = blockIdx.x / K;
  // cluster c's block of rows (static over C clusters)
  const int64_t q = a.n0 / a.C, r = a.n0 % a.C;
  const int64_t row0 = c * q + (c < r ? c : r);
  const uint32_t nrows = (uint32_t)(q + (c < r ? 1 : 0));
  const int64_t q1 = a.n1 / K, r1 = a.n1 % K;
  const int64_t col0 = NV < 0 ? (int64_t)crank * q1 + ((int64_t)crank < r1 ? crank : r1) : (int64_t)crank * qcols;
  const int lenk = NV < 0 ? (int)(q1 + ((int64_t)crank < r1 ? 1 : 0)) : qcols;  // this CTA's columns
  const In* x = (const In*)a.in;
  const uint32_t seg_bytes = (uint32_t)stage_bytes;
  const int npush = K * W;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&row_full[s], 1);    // armed by the combiner with expect_tx
      mbar_init(&slot_empty[s], 1);  // one remote arrive from the leader's combiner
    }
    fence_mbarrier_init_cluster();
  }
  cluster_sync_all();  // every CTA's barriers initialised before any remote use

  if (warp == W) {
    // ------------------------------ producer warp: TMA row segments ----
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const In* src = x + row0 * a.ld + col0;
      int s = 0;
      uint32_t ph = 0;
      for (uint32_t j = 0; j < nrows; ++j) {
        if (j >= (uint32_t)kStages) mbar_wait(&empty[s], ph ^ 1);
        if constexpr (NV < 0) {
          // the granules enclosing this row's segment (never past the
          // granule of a valid element)
          const uint32_t mis = (uint32_t)((uintptr_t)src & 15);
          const uint32_t bytes = lenk ? (uint32_t)((lenk * (uint32_t)sizeof(In) + mis + 15) & ~15u) : 0u;
          mbar_arrive_expect_tx(&full[s], bytes);
          if (bytes) bulk_g2s(dsm + (size_t)s * seg_bytes, (const unsigned char*)src - mis, bytes, &full[s], pol);
        } else {
          mbar_arrive_expect_tx(&full[s], seg_bytes);
          bulk_g2s(dsm + (size_t)s * seg_bytes, src, seg_bytes, &full[s], pol);
        }
        src += a.ld;
        if (++s == kStages) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == W + 1) {
    // ------------------------------ combiner warp (leader CTA only) ----
    if (crank == 0) {
      // rows per pass: at most the slot ring's depth (K*W = 1 would give 32
      // lanes 32 rows on 16 slots: two rows per slot in one pass)
      const int rpp = 32 / npush < kSlots ? 32 / npush : kSlots;
      const int g = lane / npush;          // this lane's row within the pass
      const int e = lane % npush;          // warp partial index within the row
      for (uint32_t j0 = 0; j0 < nrows; j0 += rpp) {
        const uint32_t j = j0 + g;
        const bool live = g < rpp && j < nrows;
        const int s = (int)(j % kSlots);
        X v = OpT<OP, X>::identity();
        if (live) {
          if (e == 0) mbar_arrive_expect_tx(&row_full[s], (uint32_t)(npush * sizeof(P)));
          mbar_wait_cluster(&row_full[s], (j / kSlots) & 1);
          v = (X)slot[s][e];
        }
        // warp partials -> CTA partials (every W lanes), ordered
        for (int off = 1; off < W; off <<= 1) v = OpT<OP, X>::combine(v, shfl_xor_t(v, off));
        if (VERIFY && live && (a.verify & V_PARTIALS) && (e % W) == 0)
          export_slot<X>(a, S_CTA, (row0 + j) * K + e / W, v);
        // CTA partials -> row (cluster), ordered
        for (int off = W; off < npush; off <<= 1) v = OpT<OP, X>::combine(v, shfl_xor_t(v, off));
        if (live && e == 0) store_row<X>(a, row0 + j, v);
        // free the slot in every CTA of the cluster (relaxed: it orders only
        // the slot reads above, which the shuffles have consumed)
        if (live && e < K) mbar_arrive_cluster_relaxed(mapa(smem_addr(&slot_empty[s]), (uint32_t)e));
      }
    }
  } else {
    // ------------------------------ W consumer warps --------------------
    const int nvec = NV < 0 ? (lenk + V - 1) / V : qcols / V;  // lane chunks of V columns
    const uint32_t leader_slot_base = mapa(smem_addr(&slot[0][0]), 0);
    const uint32_t leader_full_base = mapa(smem_addr(&row_full[0]), 0);
    const int push_idx = (int)crank * W + warp;
    const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + (int64_t)blockIdx.x * W * 32 + threadIdx.x;
    int s = 0, ss = 0;
    uint32_t ph = 0, sph = 0;
    for (uint32_t j = 0; j < nrows; ++j) {
      mbar_wait(&full[s], ph);
      const unsigned char* stage = dsm + (size_t)s * seg_bytes;
      P acc = OpT<OP, P>::identity();
      if constexpr (V != 4) {
        // lane static(1) / static(2): scalar shared loads of the chunk from
        // the row segment's first element (ragged: `mis` bytes into the
        // copied granules); a partial last chunk gets identities
        const uint32_t mis = NV < 0 ? (uint32_t)(((uintptr_t)(x + (row0 + j) * a.ld + col0)) & 15) : 0u;
        const In* se = (const In*)(stage + mis);
        for (int f = warp * 32 + lane; f < nvec; f += W * 32) {
          P t[V];
#pragma unroll
          for (int k = 0; k < V; ++k)
            t[k] = (NV >= 0 || V * f + k < lenk) ? ElemT<OP, P, In>::make(se[V * f + k]) : OpT<OP, P>::identity();
          if constexpr (OP == OP_SUM) {
            P ps = t[0];
#pragma unroll
            for (int k = 1; k < V; ++k) ps += t[k];
            acc += ps;
          } else {
#pragma unroll
            for (int k = 0; k < V; ++k) acc = OpT<OP, P>::combine(acc, t[k]);
          }
        }
      } else if constexpr (NV > 0 && F32SUM) {
        const float4* st = (const float4*)stage;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const float4 t = st[(v * W + warp) * 32 + lane];
          acc += (t.x + t.y) + (t.z + t.w);
        }
      } else {
        const uint32_t mis = NV < 0 ? (uint32_t)(((uintptr_t)(x + (row0 + j) * a.ld + col0)) & 15) : 0u;
        for (int f = warp * 32 + lane; f < nvec; f += W * 32) {
          In e[4];
          load_quad<In, (NV < 0)>(stage, f, mis, e);
          P t[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) t[k] = ElemT<OP, P, In>::make(e[k]);
          if constexpr (NV < 0) {
            const int rem = lenk - 4 * f;  // the last vector may be partial: identities keep the tree's order
#pragma unroll
            for (int k = 1; k < 4; ++k)
              if (rem <= k) t[k] = OpT<OP, P>::identity();
          }
          if constexpr (OP == OP_SUM) {
            acc += (t[0] + t[1]) + (t[2] + t[3]);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = OpT<OP, P>::combine(acc, t[k]);
          }
        }
      }
      if constexpr (VERIFY) {
        for (int f = warp * 32 + lane; f < nvec; f += W * 32)
          for (int e = 0; e < V && V * f + e < lenk; ++e) {
            const int64_t it = (row0 + j) * a.n1 + col0 + V * f + e;
            if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // stage consumed
      if (++s == kStages) { s = 0; ph ^= 1; }
      if constexpr (VERIFY) {
        if (a.verify & V_PARTIALS)
          export_slot<X>(a, S_LANE_IN, (row0 + j) * (int64_t)(npush * 32) + push_idx * 32 + lane, (X)acc);
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) acc = OpT<OP, P>::combine(acc, shfl_xor_t(acc, off));
      if (lane == 0) {
        if constexpr (VERIFY) {
          if (a.verify & V_PARTIALS) export_slot<X>(a, S_WARP, (row0 + j) * npush + push_idx, (X)acc);
        }
        if (j >= (uint32_t)kSlots) mbar_wait_relaxed_cluster(&slot_empty[ss], sph ^ 1);
        st_async_part(leader_slot_base + (uint32_t)((ss * kMaxPush + push_idx) * sizeof(P)),
                      leader_full_base + (uint32_t)(ss * 8), acc);
      }
      if (++ss == kSlots) { ss = 0; sph ^= 1; }
    }
  }
  // reconverge the warp (producer / combiner lanes ran alone) before the
  // blocking cluster barrier, so an idle lane never starves a working one
  __syncwarp();
  // every CTA stays until the leader has consumed all pushes and freed slots
  cluster_sync_all();
}

template <typename In, int OP, bool V, int NV, int LV = 4>
cudaError_t launch_t(const NestArgs& a, int W, int qcols, int stages, int stage_bytes, cudaStream_t s) {
  auto kern = rowwise_kernel<In, OP, V, NV, LV>;
  const size_t smem = (size_t)stages * stage_bytes;
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
  return cudaLaunchKernelEx(&cfg, kern, a, W, qcols, stages, stage_bytes);
}

template <typename In, int OP, bool V>
cudaError_t launch_nv(const NestArgs& a, int W, int qcols, int stages, int stage_bytes, cudaStream_t s) {
  const int lv = rowwise_lane_chunk(a);  // the lane chunk: 1, 2 or 4
  if (lv == 1)
    return rowwise_ragged(a) ? launch_t<In, OP, V, -1, 1>(a, W, qcols, stages, stage_bytes, s)
                             : launch_t<In, OP, V, 0, 1>(a, W, qcols, stages, stage_bytes, s);
  if (lv == 2)
    return rowwise_ragged(a) ? launch_t<In, OP, V, -1, 2>(a, W, qcols, stages, stage_bytes, s)
                             : launch_t<In, OP, V, 0, 2>(a, W, qcols, stages, stage_bytes, s);
  if (rowwise_ragged(a)) return launch_t<In, OP, V, -1>(a, W, qcols, stages, stage_bytes, s);
  if constexpr (std::is_same<In, float>::value && OP == OP_SUM) {
    const int nv = (qcols % (128 * W) == 0) ? qcols / (128 * W) : 0;
    switch (nv) {
      case 1: return launch_t<In, OP, V, 1>(a, W, qcols, stages, stage_bytes, s);
      case 2: return launch_t<In, OP, V, 2>(a, W, qcols, stages, stage_bytes, s);
      case 4: return launch_t<In, OP, V, 4>(a, W, qcols, stages, stage_bytes, s);
      case 8: return launch_t<In, OP, V, 8>(a, W, qcols, stages, stage_bytes, s);
      default: break;
    }
  }
  return launch_t<In, OP, V, 0>(a, W, qcols, stages, stage_bytes, s);
}

template <typename In>
cudaError_t launch_op(const NestArgs& a, int W, int qcols, int stages, int stage_bytes, cudaStream_t s) {
  const bool v = a.verify != 0;
  switch (a.op) {
    case OP_SUM: return v ? launch_nv<In, OP_SUM, true>(a, W, qcols, stages, stage_bytes, s)
                          : launch_nv<In, OP_SUM, false>(a, W, qcols, stages, stage_bytes, s);
    case OP_MIN: return v ? launch_nv<In, OP_MIN, true>(a, W, qcols, stages, stage_bytes, s)
                          : launch_nv<In, OP_MIN, false>(a, W, qcols, stages, stage_bytes, s);
    case OP_MAX: return v ? launch_nv<In, OP_MAX, true>(a, W, qcols, stages, stage_bytes, s)
                          : launch_nv<In, OP_MAX, false>(a, W, qcols, stages, stage_bytes, s);
    case OP_AFFINE:
      if constexpr (std::is_same<In, long long>::value)
        return v ? launch_nv<In, OP_AFFINE, true>(a, W, qcols, stages, stage_bytes, s)
                 : launch_nv<In, OP_AFFINE, false>(a, W, qcols, stages, stage_bytes, s);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

int rowwise_stages(int stage_bytes) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("HPAR_RW_STAGES");
    env = e ? atoi(e) : -1;
  }
  // default: ~16 KiB of row segments in flight per CTA; many small CTAs keep
  // more bytes in flight per SM than few deep ones (measured)
  int st = (env >= 2 && env <= kMaxStages) ? env : (int)(16384 / (size_t)stage_bytes);
  if (st < 2) st = 2;
  if (st > kMaxStages) st = kMaxStages;
  while (st > 2 && (size_t)st * stage_bytes > 200 * 1024) --st;
  return st;
}

}  // namespace

bool rowwise_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 2 || !a.keyed || a.offsets) { *why = "not a dense keyed 2-loop nest"; return false; }
  if (a.op != OP_SUM && a.op != OP_MIN && a.op != OP_MAX && a.op != OP_AFFINE) {
    *why = "rowwise kernel: sum / min / max / affine";
    return false;
  }
  if (a.op == OP_AFFINE && a.in_dtype != DT_I64) { *why = "affine: int64 input"; return false; }
  if (a.in_dtype != DT_F32 && a.in_dtype != DT_F64 && a.in_dtype != DT_I32 && a.in_dtype != DT_I64) {
    *why = "rowwise kernel: dtype";
    return false;
  }
  if (a.verify & V_FINGERPRINT) { *why = "fingerprints not produced by the rowwise kernel"; return false; }
  if (a.lane_w != 1) { *why = "lane partition"; return false; }
  LevelView v = device_levels(a);
  if (v.n != 4 && v.n != 3) { *why = "needs cluster, CTA, warp + lane (or warp..lane) levels"; return false; }
  const DevLevel *c = v.l[0], *k = v.l[1];
  if (!is_level(c, S_CLUSTER) || !is_level(k, S_CTA)) { *why = "levels not cluster / CTA"; return false; }
  if (c->loop != 0 || c->sched != SCHED_STATIC) { *why = "rows must be static over clusters"; return false; }
  if (k->loop != 1 || k->sched != SCHED_STATIC) { *why = "columns must be static over CTAs"; return false; }
  if (rowwise_lane_chunk(a) < 0) {
    *why = "columns over warps / lanes: warp static(32V) + lane static(V), or warp..lane static(V), V = 1|2|4";
    return false;
  }
  const int64_t K = a.K, W = a.radix[S_WARP];
  if (!pow2(K) || !pow2(W) || K * W > kMaxPush || W > 30) { *why = "K, W powers of two, K*W <= 32"; return false; }
  if (((uintptr_t)a.in & (elem_bytes(a) - 1)) || a.ld < a.n1) { *why = "input not element-aligned or ld < n1"; return false; }
  if (rowwise_stage_bytes(a) * 2 > 200 * 1024) { *why = "row segment too large for the smem ring"; return false; }
  if (a.n1 == 0) { *why = "empty rows"; return false; }
  return true;
}

cudaError_t launch_rowwise(const NestArgs& a, int W, cudaStream_t s, const char** name) {
  *name = "rowwise_tma_dsmem";
  const int qcols = (int)(a.n1 / a.K);  // the aligned path's columns per CTA
  const int sb = (int)rowwise_stage_bytes(a);
  const int st = rowwise_stages(sb);
  switch (a.in_dtype) {
    case DT_F32: return launch_op<float>(a, W, qcols, st, sb, s);
    case DT_F64: return launch_op<double>(a, W, qcols, st, sb, s);
    case DT_I32: return launch_op<int32_t>(a, W, qcols, st, sb, s);
    case DT_I64: return launch_op<long long>(a, W, qcols, st, sb, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hpar
