// kernel_segrows.cu — the collapsed CSR nest (config-3 shape) for the ops and
// dtypes the fp32-sum kernel (kernel_segmented.cu) does not take: SUM / MIN /
// MAX over fp32 (MIN/MAX), fp64, int32, int64 values.
//
// Nest shape (the same as kernel_segmented.cu, reading #14):
//     GPU                  static          loop 0 (rows; host: rank shard)
//     cluster..warp        dynamic(256)    loop 0: blocks of 256 rows claimed by warps
//     lane                 static(LPL)     loop 2: the block's collapsed (row, nonzero) list
// Rows longer than 4096 nonzeros are re-bound by length class to
// dynamic(4096) chunks over all warps of the grid (P:244-253 chunking).
//
// B200 design: no exact-prefix trick exists for MIN/MAX or for fp64 values,
// so a window of 32·LPL positions is reduced as a segmented reduction:
//   pass A   one lane per row starting in the window sets its head bit;
//   lane     each lane folds its LPL values left to right, restarting at
//            heads (the values are loaded straight from global: LPL scalar
//            loads per lane, whole 128-byte lines per warp);
//   warp     a segmented Hillis-Steele scan of the lanes' open folds gives
//            each lane the fold entering it since the last head;
//   pass B   one lane per row overlapping the window reads its part at its
//            last position and completes or carries it.
// Long rows go to a list (row, start, length, first chunk; one packed
// 64-bit atomic both numbers the entry and reserves its chunks, so chunk
// numbers ascend with entries) and a second launch reduces their chunks over
// all warps; the last chunk of a row (acq_rel ticket) folds the chunk
// partials in ascending order.  Deterministic: every fold has a fixed order.
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <type_traits>
#include "fused_common.cuh"

namespace hpar {
namespace {

constexpr int SR_RB = 256;          // rows per block claim (the nest's dynamic(256))
constexpr int64_t SR_LONG = 4096;   // longer rows are chunked over the grid
#ifndef SR_CHUNK_LEN
#define SR_CHUNK_LEN 4096  // 4096: -1.5% vs 16384 (8192 between; scripts/segrows_ab.sh)
#endif
constexpr int64_t SR_CHUNK = SR_CHUNK_LEN;  // positions per long-row chunk
constexpr int SR_WARPS = 8;         // warps per CTA (the nest's W)
#ifndef SR_MINB
#define SR_MINB 3                   // min resident CTAs (register budget: 80; 1 and 4 measured slower)
#endif
#ifndef SR_PF_L2
#define SR_PF_L2 0                  // prefetch into L2 instead of L1 (A/B knob)
#endif
#ifndef SR_PF
#define SR_PF 2                     // windows ahead the lanes prefetch into L1
#endif

struct SREntry {
  long long row, start, len, cbase;
};

struct SegRowsWS {
  unsigned long long* hdr;  // [0] block ticket, [1] (entries << 40) | chunks, [2] chunk ticket
  SREntry* ent;
  int* cmap;                // chunk -> entry
  void* part;               // chunk partials (X)
  unsigned* done;           // per entry: chunks finished (self-resetting)
  int64_t cap_ent, cap_chunks;
};

template <typename In, int OP>
struct SrX {
  using T = typename std::conditional<std::is_floating_point<In>::value, double, long long>::type;
};
template <>
struct SrX<long long, OP_AFFINE> {  // the ordered op (NEXT f2): every fold below is order-preserving
  using T = Aff;
};
template <typename T>
__device__ __forceinline__ T shfl_up_t(T v, int off) { return __shfl_up_sync(0xffffffffu, v, off); }
template <>
__device__ __forceinline__ Aff shfl_up_t<Aff>(Aff v, int off) {
  return Aff{__shfl_up_sync(0xffffffffu, v.a, off), __shfl_up_sync(0xffffffffu, v.b, off)};
}
template <typename T>
__device__ __forceinline__ T shfl_idx_t(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
template <>
__device__ __forceinline__ Aff shfl_idx_t<Aff>(Aff v, int src) {
  return Aff{__shfl_sync(0xffffffffu, v.a, src), __shfl_sync(0xffffffffu, v.b, src)};
}

template <typename X>
__device__ __forceinline__ void sr_store(const NestArgs& a, int64_t row, X v) {
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

// a 16-byte granule as 16 / sizeof(In) elements
template <typename In>
__device__ __forceinline__ void gran_elems(const int4 r, In (&e)[16 / sizeof(In)]) {
  if constexpr (sizeof(In) == 4) {
    const int w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if constexpr (std::is_floating_point<In>::value) e[t] = __int_as_float(w[t]);
      else e[t] = (In)w[t];
    }
  } else {
    const long long lo = (long long)(unsigned)r.x | ((long long)r.y << 32);
    const long long hi = (long long)(unsigned)r.z | ((long long)r.w << 32);
    if constexpr (std::is_floating_point<In>::value) {
      e[0] = __longlong_as_double(lo);
      e[1] = __longlong_as_double(hi);
    } else {
      e[0] = (In)lo;
      e[1] = (In)hi;
    }
  }
}

// the window fold type: fp64 / int64 sums, the affine pair; fp32 MIN/MAX
// stay fp32 (exact)
template <typename In, int OP>
using SrFold = typename std::conditional<std::is_same<In, float>::value && OP != OP_SUM, float,
                                         typename SrX<In, OP>::T>::type;

template <typename In, int OP, int LPL, bool VERIFY>
__global__ void __launch_bounds__(SR_WARPS * 32, SR_MINB) segrows_blocks(const __grid_constant__ NestArgs a, SegRowsWS ws) {
  using X = SrFold<In, OP>;
  using O = OpT<OP, X>;
  using E = ElemT<OP, X, In>;
  constexpr int WIN = 32 * LPL;
  // dynamic: per warp the block's offsets, then the window's folds (padded:
  // lane-major rows of LPL + 1 values, conflict-free)
  extern __shared__ __align__(16) unsigned char sr_dsm[];
  __shared__ X s_cin[SR_WARPS][32];
  __shared__ int s_fh[SR_WARPS][32];
  __shared__ unsigned s_hb[SR_WARPS][WIN / 32];
  __shared__ unsigned s_long[SR_WARPS][SR_RB / 32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const In* x = (const In*)a.in;
  constexpr int VEC = 16 / (int)sizeof(In);
  const bool vec = ((uintptr_t)x & 15) == 0;  // granule loads; else scalar
  const int64_t R = a.n0;
  const int64_t nblocks = (R + SR_RB - 1) / SR_RB;
  long long* off = (long long*)sr_dsm + (size_t)warp * (SR_RB + 1);
  X* S = (X*)((long long*)sr_dsm + (size_t)SR_WARPS * (SR_RB + 1)) + (size_t)warp * 32 * (LPL + 1);  // 8-byte aligned
  const int64_t leaf0 = (int64_t)a.rank * a.threads_per_gpu + ((int64_t)blockIdx.x * SR_WARPS + warp) * 32;
  auto cover = [&](int64_t p, int64_t who) {
    if constexpr (VERIFY) {
      if (a.verify & V_COVERAGE) {
        a.owner[p] = who;
        atomicAdd(&a.count[p], 1u);
      }
    }
  };

  for (;;) {
    long long blk = 0;
    if (lane == 0) blk = (long long)atomicAdd(&ws.hdr[0], 1ull);
    blk = __shfl_sync(0xffffffffu, blk, 0);
    if (blk >= nblocks) break;
    const int64_t r0 = blk * SR_RB;
    const int nr = (int)((R - r0 < SR_RB) ? (R - r0) : SR_RB);
    __syncwarp();
    for (int i = lane; i <= nr; i += 32) off[i] = a.offsets[r0 + i];
    __syncwarp();
    // long rows: list them (the second launch reduces them), mark them
#pragma unroll
    for (int k = 0; k < SR_RB / 32; ++k) {
      const int i = 32 * k + lane;
      const long long len = i < nr ? off[i + 1] - off[i] : 0;
      const bool lg = len > SR_LONG;
      if (lg) {
        const unsigned long long nch = (unsigned long long)((len + SR_CHUNK - 1) / SR_CHUNK);
        const unsigned long long old = atomicAdd(&ws.hdr[1], (1ull << 40) + nch);
        const long long e = (long long)(old >> 40), cb = (long long)(old & ((1ull << 40) - 1));
        // capacity by construction: every entry holds > SR_LONG nonzeros and
        // every chunk >= 1, so entries <= nnz / SR_LONG and chunks <= nnz /
        // SR_CHUNK + entries, both below the workspace's caps (the guard only
        // keeps a corrupted offsets array from writing out of bounds)
        if (e < ws.cap_ent && cb + (long long)nch <= ws.cap_chunks) {
          ws.ent[e] = SREntry{r0 + i, off[i], len, cb};
          for (unsigned long long j = 0; j < nch; ++j) ws.cmap[cb + j] = (int)e;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, lg);
      if (lane == 0) s_long[warp][k] = m;
    }
    __syncwarp();
    // first row >= i whose long bit equals `want` (nr if none): 8 mask words
    auto next_row = [&](int i, bool want) -> int {
      for (int k = i >> 5; k < SR_RB / 32; ++k) {
        unsigned m = want ? s_long[warp][k] : ~s_long[warp][k];
        if (k == (i >> 5)) m &= 0xffffffffu << (i & 31);
        if (m) {
          const int r = 32 * k + __ffs(m) - 1;
          return r < nr ? r : nr;
        }
      }
      return nr;
    };
    // runs of consecutive short rows, window by window
    int rc = 0;
    while (rc < nr) {
      rc = next_row(rc, false);
      if (rc >= nr) break;
      const int re = next_row(rc, true);
      const long long P0 = off[rc], P1 = off[re];
      int rcur = rc;
      X carry = O::identity();
      // windows from the granule holding P0 (positions before P0 and past
      // the run are the identity); a lane's LPL values are whole granules
      for (long long w = vec ? (P0 & ~(long long)(VEC - 1)) : P0; w < P1; w += WIN) {
        const long long we = (w + WIN < P1) ? w + WIN : P1;
        X v[LPL];
        if (vec) {
#pragma unroll
          for (int g = 0; g < LPL / VEC; ++g) {
            const long long q0 = w + LPL * lane + g * VEC;
            In e[VEC];
            if (q0 < we) gran_elems<In>(__ldg((const int4*)x + q0 / VEC), e);  // a granule holding a valid element
            // a later window's line of this lane into L1, in flight while
            // this window is reduced (one prefetch per lane covers its run)
            if (g == 0 && q0 + SR_PF * WIN < P1) {
#if SR_PF_L2
              asm volatile("prefetch.global.L2 [%0];" ::"l"(x + q0 + SR_PF * WIN));
#else
              asm volatile("prefetch.global.L1 [%0];" ::"l"(x + q0 + SR_PF * WIN));
#endif
            }
#pragma unroll
            for (int t = 0; t < VEC; ++t) {
              const long long q = q0 + t;
              v[g * VEC + t] = (q >= P0 && q < we) ? E::make(e[t]) : O::identity();
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < LPL; ++k) {
            const long long q = w + LPL * lane + k;
            v[k] = q < we ? E::make(__ldg(x + q)) : O::identity();
          }
        }
        // pass A: row heads (empty rows mark the next row's head: harmless)
        if (lane < WIN / 32) s_hb[warp][lane] = 0u;
        __syncwarp();
        for (int r = rcur;; r += 32) {
          const int i = r + lane;
          const long long s_ = off[i < re ? i : re];
          const bool in = i < re && s_ < we;
          if (in && s_ >= w) atomicOr(&s_hb[warp][(s_ - w) >> 5], 1u << ((s_ - w) & 31));
          if (__ballot_sync(0xffffffffu, in) != 0xffffffffu) break;
        }
        __syncwarp();
        const unsigned hbits = (LPL == 16) ? (s_hb[warp][lane >> 1] >> ((lane & 1) * 16)) & 0xFFFFu
                                           : (s_hb[warp][lane >> 2] >> ((lane & 3) * 8)) & 0xFFu;
        // lane: segmented folds, restarted at heads
        X run = O::identity();
#pragma unroll
        for (int k = 0; k < LPL; ++k) {
          run = ((hbits >> k) & 1u) ? v[k] : O::combine(run, v[k]);
          S[lane * (LPL + 1) + k] = run;
        }
        // warp: segmented scan of the open folds (lane l folds in lanes
        // (last head lane <= l, l-1]; Hillis-Steele, combine at step o iff
        // o <= the distance to that lane)
        const unsigned Hm = __ballot_sync(0xffffffffu, hbits != 0u);
        const unsigned upto = Hm & (0xffffffffu >> (31 - lane));
        const int lim = upto ? lane - (31 - __clz(upto)) : lane;
        X y = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const X t = shfl_up_t(y, o);
          if (o <= lim) y = O::combine(t, y);
        }
        X cin = shfl_up_t(y, 1);
        if (lane == 0) cin = O::identity();
        s_cin[warp][lane] = cin;
        s_fh[warp][lane] = hbits ? __ffs(hbits) - 1 : LPL;
        __syncwarp();
        // pass B: one lane per row overlapping the window
        int r = rcur;
        for (;;) {
          const int i = r + lane;
          const long long s_ = off[i < re ? i : re];
          const long long e_ = off[i + 1 < re ? i + 1 : re];
          const bool valid = i < re && s_ < we;
          const int sc = (int)min(max(s_ - w, 0ll), (long long)WIN);
          const int ec = (int)min(max(e_ - w, (long long)sc), (long long)WIN);
          X val = O::identity();
          if (valid && ec > sc) {
            const int q = ec - 1, L = q / LPL, k = q % LPL;
            val = S[L * (LPL + 1) + k];
            if (k < s_fh[warp][L]) val = O::combine(s_cin[warp][L], val);
          }
          if (valid && s_ < w) val = O::combine(carry, val);  // the row open from the previous window
          const bool complete = valid && e_ <= we;
          if (complete) sr_store<X>(a, r0 + i, val);
          if constexpr (VERIFY) {
            if (valid)
              for (int qq = sc; qq < ec; ++qq) cover(w + qq, leaf0 + qq / LPL);
          }
          const unsigned vm = __ballot_sync(0xffffffffu, valid);
          const unsigned cm = __ballot_sync(0xffffffffu, complete);
          const int cnt = __popc(vm);
          if (cnt == 0) break;
          if (!((cm >> (cnt - 1)) & 1u)) {  // the last overlapping row continues
            carry = shfl_idx_t(val, cnt - 1);
            rcur = r + cnt - 1;
            break;
          }
          r += cnt;
          rcur = r;
          carry = O::identity();
          if (cnt < 32) break;
        }
        __syncwarp();
      }
      // rows left are empty (start == the run's end): the identity
      for (int i = rcur + lane; i < re; i += 32) sr_store<X>(a, r0 + i, O::identity());
      rc = re;
    }
  }
}

// Long rows: chunks of SR_CHUNK positions over all warps; the last chunk of a
// row folds the row's chunk partials in ascending order.
template <typename In, int OP, bool VERIFY>
__global__ void __launch_bounds__(SR_WARPS * 32) segrows_long(const __grid_constant__ NestArgs a, SegRowsWS ws) {
  using X = typename SrX<In, OP>::T;
  using O = OpT<OP, X>;
  using E = ElemT<OP, X, In>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const In* x = (const In*)a.in;
  X* part = (X*)ws.part;
  const unsigned long long packed = *(volatile unsigned long long*)&ws.hdr[1];
  const long long nch = (long long)(packed & ((1ull << 40) - 1));
  const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + ((int64_t)blockIdx.x * SR_WARPS + warp) * 32 + lane;
  for (;;) {
    long long k = 0;
    if (lane == 0) k = (long long)atomicAdd(&ws.hdr[2], 1ull);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= nch) break;
    const int e = ws.cmap[k];
    const SREntry en = ws.ent[e];
    const long long j = k - en.cbase;
    const long long p0 = en.start + j * SR_CHUNK;
    const long long p1 = (en.start + en.len < p0 + SR_CHUNK) ? en.start + en.len : p0 + SR_CHUNK;
    X acc = O::identity();
    if constexpr (OP == OP_AFFINE) {
      // order-preserving: lane l folds the l-th contiguous 32nd of the chunk
      // in order, the warp fold then composes the lanes in ascending order
      const long long per = (p1 - p0 + 31) / 32;
      const long long b = p0 + lane * per, e_ = (b + per < p1) ? b + per : p1;
      for (long long p = b; p < e_; ++p) acc = O::combine(acc, E::make(__ldg(x + p)));
    } else if (((uintptr_t)x & 15) == 0) {
      // granules g0 .. g1 round-robin over the lanes, 4 in flight per lane;
      // elements outside [p0, p1) are the identity
      constexpr int VEC = 16 / (int)sizeof(In);
      const long long g0 = p0 / VEC, g1 = (p1 + VEC - 1) / VEC;
      X a4[4] = {O::identity(), O::identity(), O::identity(), O::identity()};
      for (long long gb = g0 + lane; gb < g1; gb += 128) {
        In e[4][VEC];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (gb + 32 * u < g1) gran_elems<In>(__ldg((const int4*)x + gb + 32 * u), e[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int t = 0; t < VEC; ++t) {
            const long long q = (gb + 32 * u) * VEC + t;
            if (gb + 32 * u < g1 && q >= p0 && q < p1) a4[u] = O::combine(a4[u], E::make(e[u][t]));
          }
        }
      }
      acc = O::combine(O::combine(a4[0], a4[1]), O::combine(a4[2], a4[3]));
    } else {
      for (long long p = p0 + lane; p < p1; p += 32) acc = O::combine(acc, E::make(__ldg(x + p)));
    }
    if constexpr (VERIFY) {
      if (a.verify & V_COVERAGE) {
        // the positions this lane folded (contiguous for the ordered op)
        const long long per = OP == OP_AFFINE ? (p1 - p0 + 31) / 32 : 1;
        const long long b = OP == OP_AFFINE ? p0 + lane * per : p0 + lane;
        const long long e_ = OP == OP_AFFINE ? ((b + per < p1) ? b + per : p1) : p1;
        for (long long q = b; q < e_; q += OP == OP_AFFINE ? 1 : 32) {
          a.owner[q] = leaf;
          atomicAdd(&a.count[q], 1u);
        }
      }
    }
    acc = warp_fold<OP>(acc);
    const long long nchr = (en.len + SR_CHUNK - 1) / SR_CHUNK;
    unsigned t = 0;
    if (lane == 0) {
      part[k] = acc;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(&ws.done[e]) : "memory");
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((long long)t == nchr - 1) {  // the row's last chunk: ordered fold of its partials
      __threadfence();
      const long long per = (nchr + 31) / 32;
      X v = O::identity();
      for (long long q = lane * per; q < (lane + 1) * per && q < nchr; ++q)
        v = O::combine(v, ld_volatile(part + en.cbase + q));
      v = warp_fold<OP>(v);
      if (lane == 0) {
        sr_store<X>(a, en.row, v);
        ws.done[e] = 0u;  // self-reset for the next call
      }
    }
  }
}

template <typename In, int OP, int LPL, bool V>
cudaError_t launch_blocks(const NestArgs& a, const SegRowsWS& ws, int grid, cudaStream_t s) {
  auto kern = segrows_blocks<In, OP, LPL, V>;
  const size_t smem = (size_t)SR_WARPS * ((SR_RB + 1) * 8 + 32 * (LPL + 1) * sizeof(SrFold<In, OP>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, SR_WARPS * 32, smem, s>>>(a, ws);
  return cudaGetLastError();
}

template <typename In, int OP, bool V>
cudaError_t launch_t(const NestArgs& a, const SegRowsWS& ws, int lpl, int grid_a, int grid_b, cudaStream_t s) {
  cudaError_t e = lpl == 16 ? launch_blocks<In, OP, 16, V>(a, ws, grid_a, s) : launch_blocks<In, OP, 8, V>(a, ws, grid_a, s);
  if (e != cudaSuccess) return e;
  segrows_long<In, OP, V><<<grid_b, SR_WARPS * 32, 0, s>>>(a, ws);
  return cudaGetLastError();
}

template <typename In>
cudaError_t launch_op(const NestArgs& a, const SegRowsWS& ws, int lpl, int ga, int gb, cudaStream_t s) {
  const bool v = a.verify != 0;
  switch (a.op) {
    case OP_SUM: return v ? launch_t<In, OP_SUM, true>(a, ws, lpl, ga, gb, s) : launch_t<In, OP_SUM, false>(a, ws, lpl, ga, gb, s);
    case OP_MIN: return v ? launch_t<In, OP_MIN, true>(a, ws, lpl, ga, gb, s) : launch_t<In, OP_MIN, false>(a, ws, lpl, ga, gb, s);
    case OP_MAX: return v ? launch_t<In, OP_MAX, true>(a, ws, lpl, ga, gb, s) : launch_t<In, OP_MAX, false>(a, ws, lpl, ga, gb, s);
    case OP_AFFINE:
      if constexpr (std::is_same<In, long long>::value)
        return v ? launch_t<In, OP_AFFINE, true>(a, ws, lpl, ga, gb, s) : launch_t<In, OP_AFFINE, false>(a, ws, lpl, ga, gb, s);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

int64_t sr_cap_ent(int64_t nnz) { return nnz / SR_LONG + 64; }
int64_t sr_cap_chunks(int64_t nnz) { return nnz / SR_CHUNK + nnz / SR_LONG + 64; }

}  // namespace

// workspace bytes for nnz nonzeros (header, entries, chunk map, partials, tickets)
size_t segrows_ws_bytes(int64_t nnz) {
  return 64 + (size_t)sr_cap_ent(nnz) * (sizeof(SREntry) + 4) + (size_t)sr_cap_chunks(nnz) * (4 + 16) + 256;
}

bool segrows_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 2 || !a.keyed || !a.offsets) { *why = "not a keyed CSR nest"; return false; }
  if (a.op != OP_SUM && a.op != OP_MIN && a.op != OP_MAX && a.op != OP_AFFINE) {
    *why = "CSR rows: sum / min / max / affine";
    return false;
  }
  if (a.op == OP_AFFINE && a.in_dtype != DT_I64) { *why = "affine: int64 input"; return false; }
  if (a.in_dtype != DT_F32 && a.in_dtype != DT_F64 && a.in_dtype != DT_I32 && a.in_dtype != DT_I64) {
    *why = "CSR rows: dtype";
    return false;
  }
  if (a.verify & (V_FINGERPRINT | V_PARTIALS)) { *why = "CSR rows: coverage verify only"; return false; }
  LevelView v = device_levels(a);
  if (v.n != 2) { *why = "needs [cluster..warp dynamic(256) rows] [lane static(8|16) positions]"; return false; }
  const DevLevel *t = v.l[0], *l = v.l[1];
  if (t->sfirst != S_CLUSTER || t->slast != S_WARP || t->sched != SCHED_DYNAMIC || t->chunk != SR_RB || t->loop != 0) {
    *why = "teams-warps level must be dynamic(256) over rows";
    return false;
  }
  if (!is_level(l, S_LANE) || l->sched != SCHED_STATIC_CHUNK || (l->chunk != 8 && l->chunk != 16) || l->loop != 2) {
    *why = "lane level must be static(8) or static(16) over the collapsed nonzeros (loop 2)";
    return false;
  }
  if (a.radix[S_WARP] != SR_WARPS) { *why = "W must be 8"; return false; }
  const int esz = (a.in_dtype == DT_F64 || a.in_dtype == DT_I64) ? 8 : 4;
  if (((uintptr_t)a.in & (esz - 1)) != 0) { *why = "values not element-aligned"; return false; }
  return true;
}

// ws: segrows_ws_bytes(ws_nnz) device bytes, zeroed once at allocation (the
// per-entry tickets self-reset; the header is cleared here every call)
cudaError_t launch_segrows(const NestArgs& a, void* wsbuf, int64_t ws_nnz, cudaStream_t s, const char** name) {
  *name = "segrows_csr";
  unsigned char* p = (unsigned char*)wsbuf;
  SegRowsWS ws;
  ws.hdr = (unsigned long long*)p;
  p += 64;
  ws.cap_ent = sr_cap_ent(ws_nnz);
  ws.cap_chunks = sr_cap_chunks(ws_nnz);
  ws.ent = (SREntry*)p;
  p += ws.cap_ent * sizeof(SREntry);
  ws.part = p;
  p += ws.cap_chunks * 16;  // up to the 16-byte affine pair
  ws.done = (unsigned*)p;
  p += ws.cap_ent * 4;
  ws.cmap = (int*)p;
  cudaError_t e = cudaMemsetAsync(ws.hdr, 0, 64, s);
  if (e != cudaSuccess) return e;
  const int lpl = (int)device_levels(a).l[1]->chunk;
  // the nest's C x K CTAs of W = 8 warps (owner ids stay within the GPU's
  // threads); persistent, so residency is not required
  const int64_t nblocks = (a.n0 + SR_RB - 1) / SR_RB;
  const int64_t ctas = a.C * a.K;
  const int64_t want_a = (nblocks + SR_WARPS - 1) / SR_WARPS;
  const int ga = (int)std::max<int64_t>(1, std::min<int64_t>(want_a, ctas));
  const int gb = (int)std::max<int64_t>(1, ctas);
  switch (a.in_dtype) {
    case DT_F32: return launch_op<float>(a, ws, lpl, ga, gb, s);
    case DT_F64: return launch_op<double>(a, ws, lpl, ga, gb, s);
    case DT_I32: return launch_op<int32_t>(a, ws, lpl, ga, gb, s);
    case DT_I64: return launch_op<long long>(a, ws, lpl, ga, gb, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hpar
