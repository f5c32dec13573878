// kernel_stencil.cu — one 5-point Jacobi step inside a sibling's packed
// buffer (the §4 ghost-map workload).
//
// Levels: the device level's map (hpar_map_*: each GPU holds its
// to-section, ghost surface included, and writes back its from-section) is
// host-side; this kernel is everything below it:
//   CTA   static(1) over the 2-D tiles of the from-section (persistent grid,
//         round robin).  Each tile arrives as ONE 2-D TMA box with a 1-cell
//         ghost ring — the §4 map one level down ("supporting the map
//         clause for lower-level memories such as block-shared memory"):
//         to = tile + ghosts (rows -1..TY, cols -4..TX+3 for 16-byte
//         alignment), from = the tile.  Cells outside the to-section buffer
//         are zero-filled by the TMA unit (never used: they lie beyond the
//         parent array's boundary, where cells copy through).
//   warp  static over tile rows (TY / 8 per warp; TY = 64 by default)
//   lane  static(4) over tile columns (one float4 per lane and row)
// Arithmetic (exact parity with oracle/ghostmap.py): each interior cell is
// ((((c + n) + s) + w) + e) / 5 in IEEE fp32 (__fadd_rn, and a division by
// 5 that is correctly rounded for every input, see div5); parent-boundary
// cells copy.  Tiles without boundary or section edges take a branch-free
// path.  Stores use the default L2 policy (st.global.cs measured 1.5% slower).  4-stage TMA ring and ONE CTA per SM (the ring's 144 KiB
// leaves room for no second CTA): three boxes are in flight while one is
// computed.  148 deep read streams beat 444 shallow ones (3 CTAs x 2
// stages: 0.411 vs 0.343 ms; an L2 prefetch of boxes further ahead made it
// slower still): the 2-D box rows land on DRAM pages more orderly.
// Measured alternatives (scripts/sweep_stencil*.sh): TY = 16 / 32 / 128,
// 2-6 stages, 1-3 CTAs per SM, L2 promotion off, per-CTA column strips.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "hpar.h"
#include "level_primitives.cuh"

namespace hpar {
namespace {

constexpr int TX = 128;       // tile columns: 32 lanes x 4
constexpr int BX = TX + 8;    // TMA box columns: 4 left (16-byte alignment of the tile) + 4 right
constexpr int THREADS = 256;  // 8 warps, TY / 8 rows each
template <int TY, int NST>
struct Geo {
  static constexpr int BY = TY + 2;                                // TMA box rows (1 ghost row each side)
  static constexpr int STAGE = ((BY * BX * 4 + 127) / 128) * 128;  // bytes per ring stage (128-byte aligned)
  static constexpr int RPW = TY / 8;                               // rows per warp
};

struct StParams {
  float* out;
  int64_t ld;
  int fr0, fc0;       // from-section origin, local coordinates
  int nrows, ncols;   // from-section extent
  int ca0;            // tiling column origin (fc0 rounded down to 4)
  int tiles_x, tiles_y, ntiles;
  int64_t gr0, gc0;   // global coordinates of local (0, 0) = to.off
  int64_t R, C;       // parent extents
  int dbg;            // (timing knob HPAR_ST_DEBUG) bit 1: no ghost ring in the box, bit 2: no stores -- results wrong; bit 4: streaming (.cs) stores instead of default-policy ones
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

// a / 5 correctly rounded (== __fdiv_rn(a, 5.0f), verified for all 2^32
// inputs by scripts/div5_exhaustive.cu): q0 = RN(a * RN(1/5)), the remainder
// a - 5 q0 is exact by FMA, one correction step; ±0 and ±inf take q0 (the
// only inputs where the correction differs: sign of zero, inf - inf).
__device__ __forceinline__ float div5(float a) {
  const float q0 = __fmul_rn(a, 0.2f);
  const float r = __fmaf_rn(-q0, 5.0f, a);
  const float q = __fmaf_rn(r, 0.2f, q0);
  return (a == 0.0f || fabsf(a) == __int_as_float(0x7f800000)) ? q0 : q;
}
__device__ __forceinline__ float avg5(float c, float n, float s, float w, float e) {
  return div5(__fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(c, n), s), w), e));
}

template <int TY, int NST>
__global__ void __launch_bounds__(THREADS) stencil5_kernel(const __grid_constant__ CUtensorMap tmap,
                                                            const StParams p) {
  using Gm = Geo<TY, NST>;
  constexpr int BY = Gm::BY, STAGE = Gm::STAGE, RPW = Gm::RPW;
  extern __shared__ __align__(128) unsigned char st_smem[];
  __shared__ uint64_t bar[NST];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
    fence_mbarrier_init_cluster();
  }
  __syncthreads();
  // tiles in row-major order, round robin over the persistent CTAs: the tiles
  // in flight at any time form a few contiguous row bands (sequential HBM
  // traffic; walking column strips per CTA measured 35% slower)
  auto issue = [&](int t, int s) {
    const int ty = t / p.tiles_x, tx = t - ty * p.tiles_x;
    mbar_arrive_expect_tx(&bar[s], (p.dbg & 1) ? (uint32_t)(TY * TX * 4) : (uint32_t)(BY * BX * 4));
    tma_load_2d(st_smem + s * STAGE, &tmap, p.ca0 + tx * TX - ((p.dbg & 1) ? 0 : 4), p.fr0 + ty * TY - ((p.dbg & 1) ? 0 : 1), &bar[s]);
  };
  int it = 0;
  if (tid == 0 && (int)blockIdx.x < p.ntiles) issue(blockIdx.x, 0);
  const bool vec_ok = (p.ld & 3) == 0;
  // prologue: the first NST - 1 tiles of this CTA
  if (tid == 0)
    for (int j = 1; j < NST - 1; ++j)
      if ((int)blockIdx.x + j * (int)gridDim.x < p.ntiles) issue(blockIdx.x + j * gridDim.x, j);
  for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
    const int s = it % NST;
    // the stage of tile it + NST - 1 was released by the barrier that ended tile it - 1
    const int tn = t + (NST - 1) * (int)gridDim.x;
    if (tid == 0 && tn < p.ntiles) issue(tn, (it + NST - 1) % NST);
    mbar_wait(&bar[s], (unsigned)((it / NST) & 1));
    const float* S = (const float*)(st_smem + s * STAGE);
    const int ty = t / p.tiles_x, tx = t - ty * p.tiles_x;
    const int y0 = p.fr0 + ty * TY, xb = p.ca0 + tx * TX;  // local coordinates of the tile's (0, 0)
    const int col = 4 * lane;
    const int64_t gx0 = p.gc0 + xb + col;  // global column of this lane's first cell
    bool colb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) colb[i] = (gx0 + i == 0) || (gx0 + i == p.C - 1);
    const int lx = xb + col;  // local column of this lane's first cell
    const bool cols_full = lx >= p.fc0 && lx + 4 <= p.fc0 + p.ncols;
    float4 nr = *(const float4*)(S + (RPW * warp) * BX + col + 4);
    float4 cr = *(const float4*)(S + (RPW * warp + 1) * BX + col + 4);
    // interior tile (the common case): inside `from`, no parent-boundary cell
    const int64_t gy0 = p.gr0 + y0, gxt = p.gc0 + xb;
    const bool interior = vec_ok && y0 + TY <= p.fr0 + p.nrows && xb >= p.fc0 && xb + TX <= p.fc0 + p.ncols &&
                          gy0 > 0 && gy0 + TY < p.R && gxt > 0 && gxt + TX < p.C;
    if (interior) {
      float* dst = p.out + (int64_t)(y0 + RPW * warp) * p.ld + lx;
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        const int r = RPW * warp + k;
        const float4 sr = *(const float4*)(S + (r + 2) * BX + col + 4);
        float left = __shfl_up_sync(0xffffffffu, cr.w, 1);
        float right = __shfl_down_sync(0xffffffffu, cr.x, 1);
        if (lane == 0) left = S[(r + 1) * BX + 3];
        if (lane == 31) right = S[(r + 1) * BX + 4 + TX];
        float4 o;
        o.x = avg5(cr.x, nr.x, sr.x, left, cr.y);
        o.y = avg5(cr.y, nr.y, sr.y, cr.x, cr.z);
        o.z = avg5(cr.z, nr.z, sr.z, cr.y, cr.w);
        o.w = avg5(cr.w, nr.w, sr.w, cr.z, right);
        if (!(p.dbg & 2)) {
          if (p.dbg & 4) __stcs((float4*)dst, o);
          else *(float4*)dst = o;
        }
        dst += p.ld;
        nr = cr;
        cr = sr;
      }
      __syncthreads();  // stage s is free again
      continue;
    }
#pragma unroll
    for (int k = 0; k < RPW; ++k) {
      const int r = RPW * warp + k;  // tile row; smem row r + 1
      const float4 sr = *(const float4*)(S + (r + 2) * BX + col + 4);
      float left = __shfl_up_sync(0xffffffffu, cr.w, 1);
      float right = __shfl_down_sync(0xffffffffu, cr.x, 1);
      if (lane == 0) left = S[(r + 1) * BX + 3];
      if (lane == 31) right = S[(r + 1) * BX + 4 + TX];
      const int ly = y0 + r;
      const int64_t gy = p.gr0 + ly;
      const bool rowb = (gy == 0) || (gy == p.R - 1);
      float4 o;
      o.x = (rowb || colb[0]) ? cr.x : avg5(cr.x, nr.x, sr.x, left, cr.y);
      o.y = (rowb || colb[1]) ? cr.y : avg5(cr.y, nr.y, sr.y, cr.x, cr.z);
      o.z = (rowb || colb[2]) ? cr.z : avg5(cr.z, nr.z, sr.z, cr.y, cr.w);
      o.w = (rowb || colb[3]) ? cr.w : avg5(cr.w, nr.w, sr.w, cr.z, right);
      if (ly < p.fr0 + p.nrows) {
        float* dst = p.out + (int64_t)ly * p.ld + lx;
        if (cols_full && vec_ok) {
          *(float4*)dst = o;
        } else {
          const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (lx + i >= p.fc0 && lx + i < p.fc0 + p.ncols) dst[i] = ov[i];
        }
      }
      nr = cr;
      cr = sr;
    }
    __syncthreads();  // stage s is free again
  }
}

// Register-streaming variant (HPAR_ST_IMPL=1): work unit = a 128-column
// strip x RB rows of the from-section; warp static(1) over the units
// (round robin over all warps of the persistent grid, units numbered band
// by band so the warps in flight cover contiguous memory); lane static(4)
// over the strip's columns.  A warp walks down its strip: rows arrive as
// coalesced 16-byte loads PF rows ahead into a register ring, north / centre
// / south slide in registers, west / east through SHFL (lanes 0 / 31 load
// the strip's halo column).  No shared memory: many warps per SM keep the
// loads in flight.  Same arithmetic and boundary rules as the tiled kernel.
template <int RB, int PF, int V>
__global__ void __launch_bounds__(THREADS) stencil5_rows_kernel(const float* __restrict__ in, const StParams p,
                                                                int strips, int nunits, int len0, int len1) {
  constexpr int SW = TX * V;  // strip width: V float4 per lane and row, float4 j of lane l at 4 (32 j + l)
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (THREADS / 32);
  const int64_t gw = (int64_t)blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
  for (int64_t u = gw; u < nunits; u += nw) {
    const int band = (int)(u / strips), strip = (int)(u - (int64_t)band * strips);
    const int y0 = p.fr0 + band * RB;
    const int yend = min(y0 + RB, p.fr0 + p.nrows);
    const int xs = p.ca0 + strip * SW;
    const int64_t gy0 = p.gr0 + y0, gxt = p.gc0 + xs;
    const bool interior = yend == y0 + RB && xs >= p.fc0 && xs + SW <= p.fc0 + p.ncols && y0 >= 1 &&
                          y0 + RB < len0 && xs >= 1 && xs + SW < len1 && gy0 > 0 && gy0 + RB < p.R && gxt > 0 &&
                          gxt + SW < p.C;
    if (interior) {
      const int lx = xs + 4 * lane;
      const float* src = in + (int64_t)(y0 - 1) * p.ld + lx;
      float* dst = p.out + (int64_t)y0 * p.ld + lx;
      const float* hs = in + (int64_t)y0 * p.ld + (lane == 0 ? xs - 1 : xs + SW);  // halo column of row y0
      float4 nr[V], cr[V];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        nr[j] = __ldg((const float4*)(src + TX * j));
        cr[j] = __ldg((const float4*)(src + p.ld + TX * j));
      }
      src += 2 * p.ld;
#pragma unroll 1
      for (int r = 0; r < RB; r += PF) {
        float4 sr[PF][V];
        float hv[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k)
#pragma unroll
          for (int j = 0; j < V; ++j) sr[k][j] = __ldg((const float4*)(src + (int64_t)k * p.ld + TX * j));
#pragma unroll
        for (int k = 0; k < PF; ++k) hv[k] = (lane == 0 || lane == 31) ? __ldg(hs + (int64_t)k * p.ld) : 0.f;
        src += (int64_t)PF * p.ld;
        hs += (int64_t)PF * p.ld;
#pragma unroll
        for (int k = 0; k < PF; ++k) {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            float left = __shfl_up_sync(0xffffffffu, cr[j].w, 1);
            float right = __shfl_down_sync(0xffffffffu, cr[j].x, 1);
            const float lw = j > 0 ? __shfl_sync(0xffffffffu, cr[j > 0 ? j - 1 : 0].w, 31) : hv[k];
            const float re = j < V - 1 ? __shfl_sync(0xffffffffu, cr[j < V - 1 ? j + 1 : 0].x, 0) : hv[k];
            if (lane == 0) left = lw;
            if (lane == 31) right = re;
            float4 o;
            o.x = avg5(cr[j].x, nr[j].x, sr[k][j].x, left, cr[j].y);
            o.y = avg5(cr[j].y, nr[j].y, sr[k][j].y, cr[j].x, cr[j].z);
            o.z = avg5(cr[j].z, nr[j].z, sr[k][j].z, cr[j].y, cr[j].w);
            o.w = avg5(cr[j].w, nr[j].w, sr[k][j].w, cr[j].z, right);
            *(float4*)(dst + TX * j) = o;
          }
          dst += p.ld;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            nr[j] = cr[j];
            cr[j] = sr[k][j];
          }
        }
      }
      continue;
    }
    for (int sub = 0; sub < V; ++sub) {
    const int xb = xs + TX * sub;
    const int lx = xb + 4 * lane;
    // general unit: predicated loads (cells outside the buffer read as 0 and
    // are never used), parent-boundary cells copy, writes only inside `from`
    const bool in_cols = lx + 3 < p.ld;
    auto ld4 = [&](int y) -> float4 {
      if (y < 0 || y >= len0 || !in_cols) return make_float4(0.f, 0.f, 0.f, 0.f);
      return __ldg((const float4*)(in + (int64_t)y * p.ld + lx));
    };
    auto ld1 = [&](int y, int x) -> float {
      if (y < 0 || y >= len0 || x < 0 || x >= (int)p.ld) return 0.f;
      return __ldg(in + (int64_t)y * p.ld + x);
    };
    const int64_t gx0 = p.gc0 + lx;
    bool colb[4], colin[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      colb[i] = (gx0 + i == 0) || (gx0 + i == p.C - 1);
      colin[i] = lx + i >= p.fc0 && lx + i < p.fc0 + p.ncols;
    }
    float4 nr = ld4(y0 - 1), cr = ld4(y0);
    for (int y = y0; y < yend; ++y) {
      const float4 sr = ld4(y + 1);
      const float hv = ld1(y, lane == 0 ? xb - 1 : xb + TX);
      float left = __shfl_up_sync(0xffffffffu, cr.w, 1);
      float right = __shfl_down_sync(0xffffffffu, cr.x, 1);
      if (lane == 0) left = hv;
      if (lane == 31) right = hv;
      const int64_t gy = p.gr0 + y;
      const bool rowb = (gy == 0) || (gy == p.R - 1);
      float4 o;
      o.x = (rowb || colb[0]) ? cr.x : avg5(cr.x, nr.x, sr.x, left, cr.y);
      o.y = (rowb || colb[1]) ? cr.y : avg5(cr.y, nr.y, sr.y, cr.x, cr.z);
      o.z = (rowb || colb[2]) ? cr.z : avg5(cr.z, nr.z, sr.z, cr.y, cr.w);
      o.w = (rowb || colb[3]) ? cr.w : avg5(cr.w, nr.w, sr.w, cr.z, right);
      float* dst = p.out + (int64_t)y * p.ld + lx;
      if (colin[0] && colin[3] && in_cols) {
        *(float4*)dst = o;
      } else {
        const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (colin[i]) dst[i] = ov[i];
      }
      nr = cr;
      cr = sr;
    }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  return fn;
}

}  // namespace

template <int TY, int NST>
cudaError_t launch_ty(const CUtensorMap& map, const StParams& p0, int sm_count, cudaStream_t s) {
  StParams p = p0;
  p.tiles_y = (p.nrows + TY - 1) / TY;
  p.ntiles = p.tiles_x * p.tiles_y;
  const int smem = NST * Geo<TY, NST>::STAGE;
  cudaError_t e = cudaFuncSetAttribute(stencil5_kernel<TY, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stencil5_kernel<TY, NST>, THREADS, smem);
  if (e != cudaSuccess) return e;
  int grid = sm_count * (per_sm > 0 ? per_sm : 1);
  if (const char* g = getenv("HPAR_ST_CPS")) grid = sm_count * atoi(g);  // (experiment) CTAs per SM
  if (grid > p.ntiles) grid = p.ntiles;
  if (grid < 1) return cudaSuccess;
  stencil5_kernel<TY, NST><<<grid, THREADS, smem, s>>>(map, p);
  return cudaGetLastError();
}

cudaError_t launch_stencil5(const hpar_stencil_desc& d, int device, int sm_count, cudaStream_t s, const char** why) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) {
    *why = "cuTensorMapEncodeTiled unavailable";
    return cudaErrorNotSupported;
  }
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)d.to.len[1], (cuuint64_t)d.to.len[0]};
  const cuuint64_t strides[1] = {(cuuint64_t)d.ld * 4};
  static int ty_knob = -1, l2p = -1;
  if (ty_knob < 0) ty_knob = getenv("HPAR_ST_TY") ? atoi(getenv("HPAR_ST_TY")) : 64;
  if (l2p < 0) l2p = getenv("HPAR_ST_L2P") ? atoi(getenv("HPAR_ST_L2P")) : 256;
  const int TYv = (ty_knob == 64) ? 64 : (ty_knob == 16 ? 16 : 32);
  static int dbg = -1;
  if (dbg < 0) dbg = getenv("HPAR_ST_DEBUG") ? atoi(getenv("HPAR_ST_DEBUG")) : 0;
  const cuuint32_t box[2] = {(dbg & 1) ? (cuuint32_t)TX : (cuuint32_t)BX, (cuuint32_t)(TYv + ((dbg & 1) ? 0 : 2))};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)d.in, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          l2p == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                   : (l2p == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B),
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    *why = "cuTensorMapEncodeTiled rejected the buffer layout";
    return cudaErrorInvalidValue;
  }
  StParams p;
  p.out = d.out;
  p.ld = d.ld;
  p.fr0 = (int)(d.from.off[0] - d.to.off[0]);
  p.fc0 = (int)(d.from.off[1] - d.to.off[1]);
  p.nrows = (int)d.from.len[0];
  p.ncols = (int)d.from.len[1];
  p.ca0 = p.fc0 & ~3;
  p.tiles_x = (p.fc0 + p.ncols - p.ca0 + TX - 1) / TX;
  p.gr0 = d.to.off[0];
  p.gc0 = d.to.off[1];
  p.R = d.extent[0];
  p.C = d.extent[1];
  p.dbg = dbg;
  (void)device;
  static int impl = -1;
  if (impl < 0) impl = getenv("HPAR_ST_IMPL") ? atoi(getenv("HPAR_ST_IMPL")) : 0;
  if (impl == 1 && (d.ld & 3) == 0) {
    static int vk = -1, pfk = -1, rbk = -1;
    if (vk < 0) vk = getenv("HPAR_ST_V") ? atoi(getenv("HPAR_ST_V")) : 1;
    if (pfk < 0) pfk = getenv("HPAR_ST_PF") ? atoi(getenv("HPAR_ST_PF")) : 4;
    if (rbk < 0) rbk = getenv("HPAR_ST_RB") ? atoi(getenv("HPAR_ST_RB")) : 32;
    auto go = [&](auto kern, int RB, int V) -> cudaError_t {
      const int SW = TX * V;
      const int strips = (p.fc0 + p.ncols - p.ca0 + SW - 1) / SW;
      const int nunits = ((p.nrows + RB - 1) / RB) * strips;
      int per_sm = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, 0);
      if (e != cudaSuccess) return e;
      int64_t grid = (int64_t)sm_count * (per_sm > 0 ? per_sm : 1);
      const int64_t need = (nunits + THREADS / 32 - 1) / (THREADS / 32);
      if (grid > need) grid = need;
      if (grid < 1) return cudaSuccess;
      kern<<<(unsigned)grid, THREADS, 0, s>>>(d.in, p, strips, nunits, (int)d.to.len[0], (int)d.to.len[1]);
      return cudaGetLastError();
    };
    if (vk == 4) return pfk >= 2 ? go(stencil5_rows_kernel<32, 2, 4>, 32, 4) : go(stencil5_rows_kernel<32, 1, 4>, 32, 4);
    if (vk == 2) return pfk >= 4 ? go(stencil5_rows_kernel<32, 4, 2>, 32, 2) : go(stencil5_rows_kernel<32, 2, 2>, 32, 2);
    if (rbk == 64) return pfk >= 8 ? go(stencil5_rows_kernel<64, 8, 1>, 64, 1) : go(stencil5_rows_kernel<64, 4, 1>, 64, 1);
    return pfk >= 8 ? go(stencil5_rows_kernel<32, 8, 1>, 32, 1) : go(stencil5_rows_kernel<32, 4, 1>, 32, 1);
  }
  // ring depth: TY = 64 takes 4 stages (144 KiB: one CTA per SM — fewer, deeper
  // read streams; 3 CTAs x 2 stages measured 0.411 vs 0.343 ms)
  static int nst_knob = -1;
  if (nst_knob < 0) nst_knob = getenv("HPAR_ST_NST") ? atoi(getenv("HPAR_ST_NST")) : (TYv == 64 ? 4 : 2);
  if (TYv == 16) return nst_knob >= 4 ? launch_ty<16, 4>(map, p, sm_count, s)
                                      : (nst_knob == 3 ? launch_ty<16, 3>(map, p, sm_count, s) : launch_ty<16, 2>(map, p, sm_count, s));
  if (TYv == 64)
    return nst_knob >= 4 ? launch_ty<64, 4>(map, p, sm_count, s)
         : nst_knob == 3 ? launch_ty<64, 3>(map, p, sm_count, s) : launch_ty<64, 2>(map, p, sm_count, s);
  return nst_knob >= 4 ? launch_ty<32, 4>(map, p, sm_count, s)
                       : (nst_knob == 3 ? launch_ty<32, 3>(map, p, sm_count, s) : launch_ty<32, 2>(map, p, sm_count, s));
}

}  // namespace hpar
