// kernel_segmented.cu — CSR segmented reduction with dynamic per-level
// chunking and length-class level selection (config 3).
//
// Nest (what this kernel executes; SURVEY §8(c) reading #14):
//   GPU            static over rows                     (host: rank shard)
//   cluster..warp  dynamic(RB) over rows: every warp of the GPU is a sibling
//                  (collapsed level, flags = ∩ -> dynamic, atomic); a warp
//                  claims blocks of RB consecutive rows (two ticket levels:
//                  CTA chunks of CB blocks from the GPU, blocks from the CTA)
//   lane           static(LPL) over the block's nonzeros (loop 2 = the
//                  collapsed (row, nonzero) space), LPL = 16 (or 8): a warp
//                  step covers a window of WIN = 32 * LPL nonzeros
// Length class -> level (P:344-359 versioning; P:140 grainedness): a row
// longer than LONG nonzeros is not reduced by its block's warp; it is split
// into segments of SEG nonzeros published in a GPU queue (one 32-byte entry
// each, release/acquire), any warp serves them once it has no block left,
// and the LAST segment of a row to finish folds the row's segment partials
// in ascending order (single-pass, wait-free: warps have no grid barrier).
// Blocks never share a row, so the other rows need no cross-warp fix-up.
//
// Inside a block (per warp): windows are copied by TMA (one 1-D bulk copy
// per window, lane 0 issues) into a D-deep shared-memory ring; windows lying
// inside a long row are never fetched.  Per window the lanes build the fp64
// exclusive prefix E of the window at even positions (lane-local pair sums
// + warp scan); then one lane per row overlapping the window reads the
// row's part as E[end] - E[start] (an odd end adds its one value) plus the
// carry of a row open from the previous window.  Those differences are
// EXACT when the window's nonzero magnitudes span at most EXACT_BINADES
// binades: every value is then a multiple of the smallest one's ulp and each
// prefix sum of <= 512 of them fits 53 bits.  The guard takes min |v| over
// the whole window as a float, so an explicit zero (or the zero fill past
// the array end) counts as binade 0 and sends the window to the direct path
// (conservative; -2.7% time against skipping zeros, same box).  A window failing that guard
// (or holding Inf/NaN) takes the direct path: each row lane adds its
// nonzeros in order in fp64.  Row results are staged in shared memory and
// flushed with coalesced stores.  Results are deterministic.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <mutex>
#include <type_traits>
#include "fused_common.cuh"

#ifndef HPAR_SEG_LEN
#define HPAR_SEG_LEN 16384
#endif
#ifndef HPAR_SEG_FMIN
#define HPAR_SEG_FMIN 1
#endif
namespace hpar {
namespace {

#ifndef SEG_SPEC
#define SEG_SPEC 1  // compute the window prefix before the exactness guard resolves (0.8% faster; A/B knob)
#endif
#ifndef SEG_ABL
#define SEG_ABL 0  // timing ablations only (wrong results): 1 = no window prefix, 2 = no row steps
#endif
constexpr int RB = 256;            // rows per block claim
constexpr int64_t LONG = 4096;     // a row with more nonzeros is split (default; HPAR_SEG_LONG)
constexpr int64_t SPLIT_MIN = 256;  // smallest split threshold the queue is sized for
constexpr int64_t SEG = HPAR_SEG_LEN;  // nonzeros per long-row segment at full size (16384: -1.5% vs 8192, 32768 +0.5%, 65536 +6%)
constexpr int64_t SEG_MIN = 4096;      // the shortest segment the host may pick (small shards; the queue is sized for it)
constexpr int WARPS = 8;           // warps per CTA (all workers)
// kernel variants: LPL = nonzeros per lane per window (the nest's lane
// static(LPL), 8 or 16), WIN = 32 * LPL per window, D = TMA ring depth
constexpr int CB = 8;              // row blocks per CTA claim (CTA-level dynamic chunk)
constexpr int NSB = 8;             // ring of claimed CTA chunks
constexpr int NL = 32;             // long rows per block whose windows are skipped
constexpr int EXACT_BINADES = 20;  // 9 (<= 512 terms) + 24 (fp32 significand) + 20 = 53

struct CtaSmem {
  unsigned int ctr;            // warp-level ticket over the CTA's chunk list
  int pad;
  long long sblock[NSB];       // CTA chunk j (mod NSB) -> GPU chunk index
  volatile int tag[NSB];       // j + 1 once sblock[j % NSB] is published
};

// One long-row segment in the GPU queue (32 bytes).  `row` is written last
// (release); -1 = not yet published.  The segment's partial slot is its
// queue index q; its row's first segment is q - k (the row's ticket slot).
struct SegEntry {
  long long row;
  long long b;  // first nonzero
  int len;      // nonzeros
  int k;        // index within the row
  int ns;       // segments of the row
  int pad;
};
static_assert(sizeof(SegEntry) == 32, "queue entry layout");

struct SegWS {
  unsigned long long* block_ticket;  // next row block chunk
  unsigned long long* q_tail;        // long-row segments appended
  unsigned long long* q_head;        // long-row segments claimed
  unsigned long long* blocks_done;   // row blocks finished
  unsigned long long* warps_done;    // CTAs exited (the last one resets)
  SegEntry* q;                       // the segment queue
  double* partials;                  // per segment partial sums (by queue index)
  unsigned int* tickets;             // per long row (at its first segment): segments done
  int64_t q_cap;
  unsigned long long* dbg_t;  // debug timestamps (6 per warp) or NULL
};
__device__ __forceinline__ long long ld_acquire_s64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned atom_add_acq_rel_u32(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <typename RT, int LPL, int D>
struct alignas(1024) WarpSmem {  // 1 KiB: a swizzled TMA box needs 1 KiB-aligned slots
  static constexpr int WIN = 32 * LPL;
  float ring[D][WIN];            // window ring (TMA destinations)
  double E[32 * (LPL / 2 + 1) + 2];  // exact path: window exclusive prefix at even positions
                                     // q, at q / 2 + q / LPL (one pad per lane: conflict-free);
                                     // fp32 path: the window's segmented sums S[WIN] (swizzled
                                     // 16-byte chunks) + float2 (carry-in, first head) per lane
  int32_t off[RB + 4];           // the block's RB+1 offsets relative to base
  RT res[RB];                    // the block's row results, flushed coalesced
  unsigned int lmask[RB / 32];   // long rows of the block (bit per row): never flushed here
  int32_t lrange[NL][2];         // the first NL long rows: [start, end) relative to base
  int32_t slot_wr[D];            // window position (relative to base) held by each slot
  uint64_t bar[D];               // ring slot "full" barriers
  uint64_t bar2[2];              // the two extra slots of the deep segment ring (D == 2)
  uint32_t hb[WIN / 32];         // SEGF32: row heads of the current window (bit per position)
};
static_assert(RB == 256, "the flush gives each lane 8 consecutive rows");
static_assert(sizeof(WarpSmem<float, 16, 3>) % 16 == 0 && sizeof(WarpSmem<double, 8, 4>) % 16 == 0, "TMA alignment");

// E at an even window position q (0 <= q <= WIN)
template <int LPL, typename W>
__device__ __forceinline__ double e_even(const W& sm, int q) {
  return sm.E[(q >> 1) + q / LPL];
}

// index of window position q inside a ring slot (SWZ: 128-byte swizzle)
template <bool SWZ>
__device__ __forceinline__ int ring_pos(int q) {
  if constexpr (SWZ) return (q & ~31) | ((((q >> 2) & 7) ^ ((q >> 5) & 7)) << 2) | (q & 3);
  else return q;
}

PFN_cuTensorMapEncodeTiled_v12000 seg_encode_fn() {
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

__device__ __forceinline__ float max_nan_abs(float m, float v) {  // max(m, |v|), NaN propagating
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(m), "f"(fabsf(v)));
  return r;
}

// SWZ: block windows arrive as ONE 2-D TMA box [16 rows][32 floats] with
// the 128-byte swizzle (16-byte chunk c of box row r stored at c ^ (r & 7)),
// so the lanes' 64-byte runs load without bank conflicts; the array's last
// partial 32-float row is read directly (limT below).
template <bool VERIFY, bool OUT_F32, int LPL, int D, bool SWZ = false, bool SEGF32 = false, int MINB = 3>
__global__ void __launch_bounds__(WARPS * 32, MINB) segmented_kernel(const __grid_constant__ NestArgs a, SegWS ws, int dbg, int long_min, int cb,
                                                               int seg, const __grid_constant__ CUtensorMap tmx) {
  using RT = typename std::conditional<OUT_F32, float, double>::type;
  constexpr int WIN = 32 * LPL;
  static_assert(!SWZ || LPL == 16, "swizzled windows: 16 rows of 32 floats");
  extern __shared__ __align__(128) unsigned char seg_dsm_raw[];
  __shared__ CtaSmem cs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* seg_dsm = seg_dsm_raw + ((1024u - (smem_addr(seg_dsm_raw) & 1023u)) & 1023u);
  WarpSmem<RT, LPL, D>& sm = ((WarpSmem<RT, LPL, D>*)seg_dsm)[warp];
  if (threadIdx.x == 0) cs.ctr = 0;
  if (threadIdx.x < NSB) cs.tag[threadIdx.x] = 0;
  if (lane < D) mbar_init(&sm.bar[lane], 1);
  if (lane < 2) mbar_init(&sm.bar2[lane], 1);
  for (int i = lane; i < D * WIN; i += 32) (&sm.ring[0][0])[i] = 0.f;  // defined bytes beyond partial copies
  fence_mbarrier_init_cluster();
  fence_proxy_async_shared();
  __syncthreads();
  const int64_t* offs = a.offsets;
  const float* x = (const float*)a.in;
  const int64_t R = a.n0;
  const int64_t nnz_all = a.n1;
  const int64_t nblocks = (R + RB - 1) / RB;
  const int64_t leaf0 = (int64_t)a.rank * a.threads_per_gpu + (int64_t)blockIdx.x * WARPS * 32 + warp * 32;
  const int64_t leaf = leaf0 + lane;
  auto write_row = [&](int64_t r, double v) {
    if constexpr (OUT_F32) ((float*)a.out)[r] = (float)v;
    else ((double*)a.out)[r] = v;
  };
  auto cover_by = [&](int64_t p, int64_t who) {
    if constexpr (VERIFY) {
      if (a.verify & V_COVERAGE) {
        a.owner[p - a.in_shift] = who;
        atomicAdd(&a.count[p - a.in_shift], 1u);
      }
    }
  };
  const int64_t gwarp = (int64_t)blockIdx.x * WARPS + warp;
  if (ws.dbg_t && lane == 0) ws.dbg_t[6 * gwarp] = gtimer();
  const uint64_t pol = policy_evict_first();

  // ------------------------------------------------ phase 1: row blocks ----
  // Software pipeline per warp: the claim of block j+2 and the offsets of
  // block j+1 are in flight while block j is reduced; windows are fetched up
  // to D ahead.  Two-level dynamic chunking: a warp takes the next block of
  // its CTA's chunk list from a shared-memory ticket; the warp that opens
  // chunk j claims it from the GPU ticket (CB blocks at a time).
  const int64_t nchunks = (nblocks + cb - 1) / cb;
  auto claim = [&]() -> unsigned long long {
    long long blk = 0;
    if (lane == 0) {
      const unsigned v = atomicAdd(&cs.ctr, 1u);
      const unsigned j = v / (unsigned)cb, sub = v % (unsigned)cb;
      if (sub == 0) {
        cs.sblock[j % NSB] = (long long)atomicAdd(ws.block_ticket, 1ull);
        __threadfence_block();
        cs.tag[j % NSB] = (int)(j + 1);
      } else {
        while (cs.tag[j % NSB] != (int)(j + 1)) __nanosleep(32);
        __threadfence_block();
      }
      const long long g = ((volatile long long*)cs.sblock)[j % NSB];
      blk = (g < nchunks) ? g * cb + sub : (long long)nblocks + 1;
    }
    return (unsigned long long)__shfl_sync(0xffffffffu, blk, 0);
  };
  int64_t offr[(RB + 1 + 31) / 32];
  auto load_offs = [&](unsigned long long ub) {
    const int64_t rb0 = (int64_t)ub * RB;
    const int64_t nrb = (R - rb0 < RB) ? (R - rb0) : RB;
#pragma unroll
    for (int k = 0; k < (RB + 1 + 31) / 32; ++k) {
      const int i = lane + 32 * k;
      offr[k] = ((int64_t)ub < nblocks && i <= nrb) ? offs[rb0 + i] : 0;
    }
  };
  unsigned long long my_blocks = 0;  // added to blocks_done once, when this warp leaves phase 1
  bool published = false;            // this lane appended long-row segments to the queue
  unsigned iseq = 0, cseq = 0;       // ring: windows issued / consumed by this warp
  unsigned phases = 0;               // parity bit per ring slot
  const int64_t nnz4 = nnz_all & ~(int64_t)3;
  auto ring_wait = [&]() -> int {  // next issued window: its slot, once landed
    const int s = (int)(cseq % D);
    mbar_wait(&sm.bar[s], (phases >> s) & 1u);
    phases ^= 1u << s;
    ++cseq;
    return s;
  };
  // One published long-row segment: its nonzeros stream through the ring
  // (fp32 per lane and window, fp64 across); the row's LAST segment to
  // finish folds the segment partials in ascending order.
  // DEEP (after the warp's blocks, D == 2): 4 window slots — the ring plus
  // the then idle prefix and offsets/results areas — so a segment keeps 3
  // windows (6 KiB) in flight instead of 1.
  auto do_segment = [&](unsigned long long q, auto deep_c) {
    constexpr bool DEEP = decltype(deep_c)::value && D == 2;
    constexpr int NS = DEEP ? 4 : D;
    auto slot_ptr = [&](int s) -> float* {  // DEEP: ring 0, 1, then E, then off + res (2064 contiguous bytes)
      if constexpr (DEEP) return s == 0 ? &sm.ring[0][0] : s == 1 ? &sm.ring[1][0] : s == 2 ? (float*)&sm.E[0] : (float*)&sm.off[0];
      else return &sm.ring[s][0];
    };
    auto slot_bar = [&](int s) -> uint64_t* { return s < D ? &sm.bar[s] : &sm.bar2[s - D]; };
    long long row = -1, b = 0;
    int len = 0, k = 0, ns = 0;
    if (lane == 0) {
      SegEntry& en = ws.q[q];
      while ((row = ld_acquire_s64(&en.row)) < 0) __nanosleep(32);
      b = en.b;
      len = en.len;
      k = en.k;
      ns = en.ns;
      en.row = -1;  // self-reset for the next call
    }
    row = __shfl_sync(0xffffffffu, row, 0);
    b = __shfl_sync(0xffffffffu, b, 0);
    len = __shfl_sync(0xffffffffu, len, 0);
    k = __shfl_sync(0xffffffffu, k, 0);
    ns = __shfl_sync(0xffffffffu, ns, 0);
    const int64_t pb = (int64_t)q - k;
    const int64_t e = b + len;
    const int64_t sb = b & ~(int64_t)3;  // 16-byte aligned origin; positions below relative to it
    const int n = (dbg & 1) ? 0 : (int)(e - sb);
    const int64_t e4 = (e + 3) & ~(int64_t)3;
    const int c4 = (int)((e4 < nnz4 ? e4 : nnz4) - sb);  // copied by TMA; beyond: the array's tail
    const int bo = (int)(b - sb);
    // windows are issued and consumed in order: window i sits at i * WIN and
    // in slot i % NS (own counters; every slot's barrier parity in `phases`)
    int ni = 0, nc = 0;
    auto seg_issue = [&](int w) {
      const int s = ni % NS;
      if (lane == 0) {
        const int m = (c4 - w < WIN) ? c4 - w : WIN;
        if (m > 0) {
          mbar_arrive_expect_tx(slot_bar(s), (uint32_t)m * 4u);
          bulk_g2s(slot_ptr(s), x + sb + w, (uint32_t)m * 4u, slot_bar(s), pol);
        } else {
          mbar_arrive(slot_bar(s));
        }
      }
      ++ni;
    };
    if constexpr (DEEP) {
      // the extra slots alias E / off, last written by generic-proxy stores
      // in phase 1: order those writes before the async-proxy (TMA) writes
      fence_proxy_async_shared();
      __syncwarp();
    }
    int iw = 0;
    for (int d = 0; d < NS && iw < n; ++d, iw += WIN) seg_issue(iw);
    double acc = 0.0;
    while (nc != ni) {
      const int s = nc % NS;
      mbar_wait(slot_bar(s), (phases >> s) & 1u);
      phases ^= 1u << s;
      const int wr = nc * WIN;
      ++nc;
      const float* slot = slot_ptr(s);
      // a segment is one sum: lane l takes float4 chunks l, l + 32, ... of
      // the window (consecutive lanes, consecutive 16 bytes: no conflicts)
      float v[LPL];
#pragma unroll
      for (int j = 0; j < LPL / 4; ++j) {
        const float4 t = *(const float4*)&slot[4 * (32 * j + lane)];
        v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
      }
      auto pos = [&](int j) { return wr + 4 * (32 * (j >> 2) + lane) + (j & 3); };
      if (wr == 0 || wr + WIN > n) {  // segment edges; the array's unaligned tail
#pragma unroll
        for (int j = 0; j < LPL; ++j) {
          const int q2 = pos(j);
          if (q2 >= c4 && q2 < n) v[j] = x[sb + q2];
          if (q2 < bo || q2 >= n) v[j] = 0.f;
        }
      }
      float t4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) t4[j] = (v[4 * j] + v[4 * j + 1]) + (v[4 * j + 2] + v[4 * j + 3]);
      acc += (double)((t4[0] + t4[1]) + (t4[2] + t4[3]));
      if constexpr (VERIFY) {
        for (int j = 0; j < LPL; ++j)
          if (pos(j) >= bo && pos(j) < n) cover_by(sb + pos(j), leaf);
      }
      __syncwarp();  // slot s is free again
      if (iw < n) {
        seg_issue(iw);
        iw += WIN;
      }
    }
    acc = warp_fold<OP_SUM>(acc);
    unsigned t = 0;
    if (lane == 0) {
      __stcg(&ws.partials[q], acc);
      t = atom_add_acq_rel_u32(&ws.tickets[pb], 1u);  // release my partial
    }
    if ((int)__shfl_sync(0xffffffffu, t, 0) == ns - 1) {
      // last segment of the row: the ordered fold, ascending from 0 as a
      // sequential loop would add, but the partials are loaded 32 at a time
      // by the lanes (one L2 round trip per 32 instead of one per partial)
      __threadfence();  // every lane's loads after lane 0's acquire
      double tot = 0.0;
      for (int j0 = 0; j0 < ns; j0 += 32) {
        const double pj = (j0 + lane < ns) ? __ldcg(&ws.partials[pb + j0 + lane]) : 0.0;
        const int m = (ns - j0 < 32) ? ns - j0 : 32;
        for (int l = 0; l < m; ++l) tot += __shfl_sync(0xffffffffu, pj, l);
      }
      if (lane == 0) {
        write_row(row, tot);
        ws.tickets[pb] = 0u;
      }
    }
  };
  // Long-row segments interleave with the row blocks: each warp holds one
  // claimed queue ticket and serves it between blocks once it is published.
  constexpr unsigned long long NONE = ~0ull;
  unsigned long long myq = NONE;
  auto claim_seg = [&]() {
    if (myq == NONE) {
      unsigned long long q = 0;
      if (lane == 0) q = atomicAdd(ws.q_head, 1ull);
      myq = __shfl_sync(0xffffffffu, q, 0);
    }
  };
  unsigned long long u = claim();
  load_offs(u);
  // cross-block prefetch (SWZ path): once a block has no window left to
  // issue, the next block's first window goes into the free ring slot, so
  // the pipeline does not drain at every block boundary
  unsigned pre_next = 0;  // windows already issued for the next block (0..2)
  while ((int64_t)u < nblocks) {
    const unsigned pre_here = pre_next;
    pre_next = 0;
    const unsigned long long u1 = claim();
    const int64_t r0 = (int64_t)u * RB;
    const int nr = (int)((R - r0 < RB) ? (R - r0) : RB);
    // window origin: 64-byte aligned; positions below are 32-bit, relative to
    // it (nnz < 2^31 per rank)
    const int64_t base = __shfl_sync(0xffffffffu, offr[0], 0) & ~(int64_t)31;  // a whole 128-byte row
#pragma unroll
    for (int k = 0; k < (RB + 1 + 31) / 32; ++k) {
      const int i = lane + 32 * k;
      if (i <= nr) sm.off[i] = (int)(offr[k] - base);
    }
#pragma unroll
    for (int k = 0; k < (int)(RB * sizeof(RT)) / 16 / 32; ++k)
      ((float4*)sm.res)[lane + 32 * k] = make_float4(0.f, 0.f, 0.f, 0.f);  // empty rows stay 0
    __syncwarp();
    load_offs(u1);  // next block's offsets, in flight during this block
    const int p0 = sm.off[0], p1 = sm.off[nr];
    // long rows: enqueue their segments, mark them, list the first NL.  A
    // block spanning <= long_min nonzeros cannot hold one: skip the scan
    int nl = 0;
    const bool may_long = p1 - p0 > long_min;
    if (!may_long && lane < RB / 32) sm.lmask[lane] = 0u;
#pragma unroll
    for (int k = 0; k < RB / 32 && may_long; ++k) {
      const int i = lane + 32 * k;
      bool lg = false;
      int s_ = 0, e_ = 0;
      if (i < nr) {
        s_ = sm.off[i];
        e_ = sm.off[i + 1];
        lg = e_ - s_ > long_min;
        if (lg) {
          const int len = e_ - s_;
          const int ns = (len + seg - 1) / seg;
          const unsigned long long q = atomicAdd(ws.q_tail, (unsigned long long)ns);
          published = true;
          for (int j = 0; j < ns; ++j) {
            SegEntry& en = ws.q[q + j];
            en.b = base + s_ + (int64_t)j * seg;
            en.len = (len - j * seg < seg) ? len - j * seg : seg;
            en.k = j;
            en.ns = ns;
          }
          fence_acq_rel_gpu();  // entries before their publication
          for (int j = 0; j < ns; ++j) *(volatile long long*)&ws.q[q + j].row = r0 + i;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, lg);
      if (lane == 0) sm.lmask[k] = m;
      if (lg) {
        const int at = nl + __popc(m & ((1u << lane) - 1u));
        if (at < NL) {
          sm.lrange[at][0] = s_;
          sm.lrange[at][1] = e_;
        }
      }
      nl += __popc(m);
    }
    nl = nl < NL ? nl : NL;
    __syncwarp();

    // window fetch: bytes up to p1 (rounded to 16) but never past the last
    // whole 16 bytes of the array; the <= 3 nonzeros beyond are loaded directly
    const int64_t lim64 = nnz_all - base;
    const int lim = lim64 > 0x7FFFFFF0 ? 0x7FFFFFF0 : (int)lim64;
    const int lim4 = SWZ ? lim & ~31 : lim & ~3;  // positions past lim4 are read directly
    const int p1c = ((p1 + 3) & ~3) < lim4 ? ((p1 + 3) & ~3) : lim4;
    int li = 0;  // issuer's cursor over the long-row list
    auto skip = [&](int w) -> int {  // first window at or after w not inside a long row
      while (li < nl) {
        const int ls = sm.lrange[li][0], le = sm.lrange[li][1];
        if (le <= w) {
          ++li;
        } else if (ls <= w && w + WIN <= le) {
          w = le & ~(WIN - 1);
        } else {
          break;
        }
      }
      return w;
    };
    auto issue = [&](int w) {
      const int s = (int)(iseq % D);
      if (lane == 0) {
        sm.slot_wr[s] = w;
        if constexpr (SWZ) {  // rows past the array's last whole row arrive as zeros
          mbar_arrive_expect_tx(&sm.bar[s], (uint32_t)WIN * 4u);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                  "r"(smem_addr(&sm.ring[s][0])), "l"(&tmx), "r"(0), "r"((int)((base + w) >> 5)), "r"(smem_addr(&sm.bar[s]))
              : "memory");
        } else {
          const int n = (p1c - w < WIN) ? p1c - w : WIN;
          if (n > 0) {
            mbar_arrive_expect_tx(&sm.bar[s], (uint32_t)n * 4u);
            bulk_g2s(&sm.ring[s][0], x + base + w, (uint32_t)n * 4u, &sm.bar[s], pol);
          } else {
            mbar_arrive(&sm.bar[s]);
          }
        }
      }
      ++iseq;
    };
    // the next block's first window, into a free slot (its rows are not known
    // yet, so it is window 0 even if that lies inside a long row: then it is
    // consumed as a partial window of that row, whose result is never flushed)
    const int64_t base_next = __shfl_sync(0xffffffffu, offr[0], 0) & ~(int64_t)31;
    // (not with the between-blocks segment serving knob, dbg & 4, whose segments reuse the ring from slot 0)
    const bool can_pre = SWZ && (dbg & (64 | 4)) == 0 && (int64_t)u1 < nblocks;
    const unsigned xb_max = (dbg & 32) ? 1u : 2u;  // next-block windows issued ahead (knob: HPAR_SEG_DEBUG bit 32 = 1)
    auto issue_next = [&]() {
      if constexpr (SWZ) {
        const int s = (int)(iseq % D);
        const int w = (int)pre_next * WIN;
        if (lane == 0) {
          sm.slot_wr[s] = w;
          mbar_arrive_expect_tx(&sm.bar[s], (uint32_t)WIN * 4u);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                  "r"(smem_addr(&sm.ring[s][0])), "l"(&tmx), "r"(0), "r"((int)((base_next + w) >> 5)), "r"(smem_addr(&sm.bar[s]))
              : "memory");
        }
        ++iseq;
        ++pre_next;
      }
    };
    int iw = (dbg & 2) ? p1 : skip((int)pre_here * WIN);
    for (int d = (int)pre_here; d < D && iw < p1; ++d) {
      issue(iw);
      iw = skip(iw + WIN);
    }
    if (can_pre && iw >= p1 && iseq - cseq < (unsigned)D) issue_next();
    int rcur = 0;        // first row overlapping the next window
    double carry = 0.0;  // row rcur's sum before the next window
    while (cseq != iseq - pre_next) {
      const int s = (int)(cseq % D);
      mbar_wait(&sm.bar[s], (phases >> s) & 1u);
      phases ^= 1u << s;
      ++cseq;
      const int wr = sm.slot_wr[s];
      const int wend = wr + WIN;
      const int p = wr + LPL * lane;
      float v[LPL];
#pragma unroll
      for (int j = 0; j < LPL / 4; ++j) {
        // SWZ: lane l's run is box row l / 2, chunks (l & 1) * 4 + j, stored
        // at chunk ^ (row & 7)
        const int off4 = SWZ ? (lane >> 1) * 32 + ((((lane & 1) * 4 + j) ^ ((lane >> 1) & 7)) << 2) : LPL * lane + 4 * j;
        const float4 t = *(const float4*)&sm.ring[s][off4];
        v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
      }
      // Positions outside [p0, p1) hold neighbours' (or stale) values: no row
      // range covers them, so they cancel in every E difference once E is
      // exact; the guard below sees them too (conservative).  The array's
      // unaligned tail (< 4 nonzeros past the last whole 16 bytes) is read
      // directly.
      if (wend > lim4 && p1 > lim4) {
#pragma unroll
        for (int k = 0; k < LPL; ++k) {
          const int q = p + k;
          if (q >= lim4 && q < p1) v[k] = x[base + q];
        }
      }
      if constexpr (SEGF32) {
        // fp32 range guard: a window holding a finite |v| >= 2^119 could
        // overflow a 512-term fp32 sum that fp64 would not; such (rare)
        // windows take the in-order fp64 loop per row below instead
        float amx = 0.f;
#pragma unroll
        for (int k = 0; k < LPL; ++k) amx = fmaxf(amx, fabsf(v[k]));  // NaN ignored, Inf counted
        const bool big = __any_sync(0xffffffffu, amx >= 0x1p119f && amx <= 3.402823466e38f);
        // ---- pass A: row heads.  Every row starting inside the window marks
        // its first position (empty rows and the block end mark harmlessly:
        // a head only restarts a running sum).
        if (lane < WIN / 32) sm.hb[lane] = 0u;
        __syncwarp();
        for (int r = rcur;; r += 32) {
          const int i = r + lane;
          const int s_ = sm.off[i < nr ? i : nr];
          const bool in = i <= nr && s_ < wend;
          if (in && s_ >= wr) atomicOr(&sm.hb[(s_ - wr) >> 5], 1u << ((s_ - wr) & 31));
          if (__ballot_sync(0xffffffffu, in) != 0xffffffffu) break;
        }
        __syncwarp();
        static_assert(!SEGF32 || (LPL == 16 && SWZ), "fp32 segmented windows: 16 positions per lane, swizzled boxes");
        const unsigned hbits = (sm.hb[lane >> 1] >> ((lane & 1) * 16)) & 0xFFFFu;
        // ---- lane-local segmented sums (fp32, restart at every head)
        float S[LPL];
        float run = 0.f;
#pragma unroll
        for (int k = 0; k < LPL; ++k) {
          run = ((hbits >> k) & 1u) ? v[k] : run + v[k];
          S[k] = run;
        }
        // ---- warp segmented scan of the lanes' open sums: lane l adds the
        // sum of lanes (start_l, l-1] where start_l is the last lane <= l
        // holding a head (Hillis-Steele, add at step o iff o <= lim)
        const unsigned Hm = __ballot_sync(0xffffffffu, hbits != 0u);
        const unsigned upto = Hm & (0xffffffffu >> (31 - lane));  // heads in lanes [0, l]
        const int lim = upto ? lane - (31 - __clz(upto)) : lane;
        float y = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float t = __shfl_up_sync(0xffffffffu, y, o);
          if (o <= lim) y += t;
        }
        float cin = __shfl_up_sync(0xffffffffu, y, 1);  // the open sum entering this lane
        if (lane == 0) cin = 0.f;
        const int fh = hbits ? __ffs(hbits) - 1 : LPL;  // positions before it continue cin
        // ---- publish S (conflict-free: 16-byte chunk j of lane l stored at
        // j ^ ((l >> 1) & 3)).  Not in place of the values: the ring slot is
        // a TMA destination, and ordering generic writes before its refill
        // (fence.proxy.async per window) measured 3% slower.
        float* sS = (float*)&sm.E[0];
        float2* sCF = (float2*)(sS + WIN);
#pragma unroll
        for (int j = 0; j < LPL / 4; ++j)
          *(float4*)&sS[LPL * lane + ((j ^ ((lane >> 1) & 3)) << 2)] = make_float4(S[4 * j], S[4 * j + 1], S[4 * j + 2], S[4 * j + 3]);
        sCF[lane] = make_float2(cin, __int_as_float(fh));
        __syncwarp();
        // ---- pass B: one lane per row overlapping the window; a row's part
        // of the window is the segmented sum at its last position here
        int r = rcur;
        for (;;) {
          const int i = r + lane;
          const int s_ = sm.off[i < nr ? i : nr];
          const int e_ = sm.off[i + 1 < nr ? i + 1 : nr];
          const bool valid = i < nr && s_ < wend;
          const int sc = min(max(s_ - wr, 0), WIN);
          const int ec = min(max(e_ - wr, sc), WIN);
          const int q = ec > sc ? ec - 1 : 0;
          const int L = q / LPL, k = q % LPL;
          const float2 cf = sCF[L];
          float part = sS[LPL * L + (((k >> 2) ^ ((L >> 1) & 3)) << 2) + (k & 3)];
          if (k < __float_as_int(cf.y)) part += cf.x;
          double val = ec > sc ? (double)part : 0.0;
          if (big) {  // in-order fp64 over the row's part of the window
            val = 0.0;
            if (valid)
              for (int qq = sc; qq < ec; ++qq)
                val += (double)((wr + qq >= lim4) ? x[base + wr + qq] : sm.ring[s][ring_pos<SWZ>(qq)]);
          }
          if (s_ < wr) val += carry;  // the row open from the previous window
          const bool complete = valid && e_ <= wend;
          if (complete) sm.res[i] = (RT)val;  // a long row's slot is never flushed
          if constexpr (VERIFY) {
            if (valid && !((sm.lmask[i >> 5] >> (i & 31)) & 1u))
              for (int qq = sc; qq < ec; ++qq) cover_by(base + wr + qq, leaf0 + qq / LPL);
          }
          const unsigned vm = __ballot_sync(0xffffffffu, valid);
          const unsigned cm = __ballot_sync(0xffffffffu, complete);
          const int cnt = __popc(vm);
          if (cnt == 0) break;
          if (!((cm >> (cnt - 1)) & 1u)) {  // the last overlapping row continues
            carry = __shfl_sync(0xffffffffu, val, cnt - 1);
            rcur = r + cnt - 1;
            break;
          }
          r += cnt;
          rcur = r;
          carry = 0.0;
          if (cnt < 32) break;
        }
        __syncwarp();  // S and ring slot s are free again
        if (iw < p1) {
          issue(iw);
          iw = skip(iw + WIN);
        } else if (can_pre && pre_next < xb_max) {
          issue_next();
        }
      } else {
      // exactness guard: binade span of the window's nonzero magnitudes
      float amax = 0.f;
#if HPAR_SEG_FMIN
      // min |v| as a float (3-input FMNMX): a zero makes emin = 0, so a window
      // holding an explicit zero takes the in-order path (CSR values are
      // nonzeros; the exact path stays exact either way)
      float amin = __int_as_float(0x7f800000);
#pragma unroll
      for (int k = 0; k < LPL; ++k) {
        amax = max_nan_abs(amax, v[k]);
        amin = fminf(amin, fabsf(v[k]));
      }
      const unsigned gmax = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));
      const unsigned gmin = __reduce_min_sync(0xffffffffu, __float_as_uint(amin));
      const int emax = (int)(gmax >> 23), emin = (int)(gmin >> 23);
#else
      unsigned umin = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < LPL; ++k) {
        amax = max_nan_abs(amax, v[k]);
        const unsigned t = __float_as_uint(v[k]) * 2u - 1u;  // |v| bits << 1, minus 1: zero -> max
        umin = t < umin ? t : umin;
      }
      const unsigned gmax = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));
      const unsigned gmin = __reduce_min_sync(0xffffffffu, umin);
      const int emax = (int)(gmax >> 23), emin = (int)((gmin + 1u) >> 24);
#endif
      const bool exact = emax < 255 && emax - emin <= EXACT_BINADES;
      // the prefix does not wait for the guard's two warp reductions
      // (SEG_SPEC: computed for every window; non-exact windows ignore it)
      if ((SEG_SPEC || exact) && !(SEG_ABL & 1)) {
        // lane-local prefix at even positions: pair sums, then their prefix
        // in two independent halves (short dependency chains)
        double c[LPL / 2];  // c[j] = v[0] + ... + v[2j+1]
#pragma unroll
        for (int j = 0; j < LPL / 2; ++j) c[j] = (double)v[2 * j] + (double)v[2 * j + 1];
#pragma unroll
        for (int j = 1; j < LPL / 4; ++j) {
          c[j] += c[j - 1];
          c[LPL / 4 + j] += c[LPL / 4 + j - 1];
        }
#pragma unroll
        for (int j = LPL / 4; j < LPL / 2; ++j) c[j] += c[LPL / 4 - 1];
        double incl = c[LPL / 2 - 1];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        double ex = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) ex = 0.0;
        double* el = &sm.E[(LPL / 2 + 1) * lane];
        el[0] = ex;
#pragma unroll
        for (int k = 1; k < LPL / 2; ++k) el[k] = ex + c[k - 1];
        if (lane == 31) sm.E[32 * (LPL / 2 + 1)] = incl;
        __syncwarp();
      }
      // one lane per row overlapping the window, 32 rows per step.  Straight-
      // line per lane: indices are clamped and results selected, so lanes
      // past the window's rows compute a discarded value instead of branching.
      const bool tail_win = wend > lim4;  // the array's unaligned tail is not in the ring
      int r = rcur;
      for (; !(SEG_ABL & 2);) {
        const int i = r + lane;
        const int s_ = sm.off[i < nr ? i : nr];
        const int e_ = sm.off[i + 1 < nr ? i + 1 : nr];
        const bool valid = i < nr && s_ < wend;
        // clamped: a long row whose windows were skipped may end before wr
        const int sc = min(max(s_ - wr, 0), WIN);
        const int ec = min(max(e_ - wr, sc), WIN);
        double val = 0.0;
        if (exact) {
          // an odd end / start adds the one value before it
          float ve = sm.ring[s][ring_pos<SWZ>(ec > 0 ? ec - 1 : 0)];
          float vs = sm.ring[s][ring_pos<SWZ>(sc > 0 ? sc - 1 : 0)];
          if (tail_win) {
            if (ec > 0 && wr + ec - 1 >= lim4) ve = x[base + wr + ec - 1];
            if (sc > 0 && wr + sc - 1 >= lim4) vs = x[base + wr + sc - 1];
          }
          val = (e_even<LPL>(sm, ec & ~1) - e_even<LPL>(sm, sc & ~1)) +
                ((double)((ec & 1) ? ve : 0.f) - (double)((sc & 1) ? vs : 0.f));
        } else if (valid) {
          for (int q = sc; q < ec; ++q) val += (double)((wr + q >= lim4) ? x[base + wr + q] : sm.ring[s][ring_pos<SWZ>(q)]);
        }
        if (s_ < wr) val += carry;  // the row open from the previous window
        const bool complete = valid && e_ <= wend;
        if (complete) sm.res[i] = (RT)val;  // a long row's slot is never flushed
        if constexpr (VERIFY) {
          if (valid && !((sm.lmask[i >> 5] >> (i & 31)) & 1u))
            for (int q = sc; q < ec; ++q) cover_by(base + wr + q, leaf0 + q / LPL);
        }
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        const unsigned cm = __ballot_sync(0xffffffffu, complete);
        const int cnt = __popc(vm);
        if (cnt == 0) break;
        if (!((cm >> (cnt - 1)) & 1u)) {  // the last overlapping row continues
          carry = __shfl_sync(0xffffffffu, val, cnt - 1);
          rcur = r + cnt - 1;
          break;
        }
        r += cnt;
        rcur = r;
        carry = 0.0;
        if (cnt < 32) break;
      }
      __syncwarp();  // E and ring slot s are free again
      if (iw < p1) {
        issue(iw);
        iw = skip(iw + WIN);
      } else if (can_pre && pre_next < xb_max) {
        issue_next();
      }
      }  // exact fp64-prefix windows
    }
    // flush: lane l writes rows 8l..8l+7 (long rows excluded)
    {
      const int rl = 8 * lane;
      const unsigned lm = (sm.lmask[lane >> 2] >> ((lane & 3) * 8)) & 0xFFu;
      RT* o = (RT*)a.out + r0 + rl;
      if (rl + 8 <= nr && lm == 0 && ((uintptr_t)a.out & 15) == 0) {
#pragma unroll
        for (int q = 0; q < (int)(8 * sizeof(RT)) / 16; ++q) ((float4*)o)[q] = ((const float4*)(sm.res + rl))[q];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (rl + j < nr && !((lm >> j) & 1u)) o[j] = sm.res[rl + j];
      }
    }
    __syncwarp();
    ++my_blocks;
    u = u1;
    if (dbg & 4) {  // (knob) serve published segments between blocks
      for (;;) {
        unsigned long long head = 0, tail = 0;
        if (lane == 0) {
          tail = *(volatile unsigned long long*)ws.q_tail;
          head = *(volatile unsigned long long*)ws.q_head;
        }
        tail = __shfl_sync(0xffffffffu, tail, 0);
        head = __shfl_sync(0xffffffffu, head, 0);
        if (myq == NONE && head < tail) claim_seg();
        if (myq == NONE || myq >= tail) break;
        do_segment(myq, std::false_type());
        myq = NONE;
      }
    }
  }

  // release: this warp's q_tail appends are visible before its blocks count
  // (readers rely on q_tail being final once blocks_done == nblocks); a warp
  // that appended nothing has nothing to order and counts relaxed
  if (__any_sync(0xffffffffu, published)) {
    if (lane == 0)
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ws.blocks_done), "l"(my_blocks) : "memory");
  } else if (lane == 0) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(ws.blocks_done), "l"(my_blocks) : "memory");
  }

  if (ws.dbg_t && lane == 0) ws.dbg_t[6 * gwarp + 1] = gtimer();
  // ------------------------------- phase 2: the remaining long-row segments ----
  // Claim a ticket only while the queue looks non-empty; a ticket that lost
  // the race waits for its entry.  Leave once every block is done (no entry
  // can appear any more) and the queue is drained.  Idle polling backs off.
  unsigned nap = 32;
  const unsigned nap_max = (dbg >> 8) ? (unsigned)(dbg >> 8) : 2048u;  // (knob: HPAR_SEG_DEBUG bits 8+)
  unsigned long long dbg_nseg = 0, dbg_tseg = 0, dbg_tdone = 0;
  for (;;) {
    unsigned long long head = 0, tail = 0, done = 0;
    if (lane == 0) {
      tail = *(volatile unsigned long long*)ws.q_tail;
      head = *(volatile unsigned long long*)ws.q_head;
      done = (unsigned long long)ld_acquire_s64((const long long*)ws.blocks_done);
    }
    tail = __shfl_sync(0xffffffffu, tail, 0);
    head = __shfl_sync(0xffffffffu, head, 0);
    done = __shfl_sync(0xffffffffu, done, 0);
    if (myq == NONE && head < tail) claim_seg();
    if (myq != NONE && myq < tail) {
      const unsigned long long t0 = ws.dbg_t ? gtimer() : 0;
      do_segment(myq, std::true_type());  // after the blocks: deep ring
      if (ws.dbg_t) { ++dbg_nseg; dbg_tseg += gtimer() - t0; }
      myq = NONE;
      nap = 32;
      continue;
    }
    if ((int64_t)done >= nblocks) {
      if (ws.dbg_t && !dbg_tdone) dbg_tdone = gtimer();
      // every entry is published before blocks_done counts its block (the
      // acquire above orders these re-reads after it)
      if (lane == 0) {
        tail = *(volatile unsigned long long*)ws.q_tail;
        head = *(volatile unsigned long long*)ws.q_head;
      }
      tail = __shfl_sync(0xffffffffu, tail, 0);
      head = __shfl_sync(0xffffffffu, head, 0);
      if (myq != NONE ? myq < tail : head < tail) continue;
      break;
    }
    __nanosleep(nap);
    nap = nap < nap_max ? 2 * nap : nap_max;
  }

  if (ws.dbg_t && lane == 0) ws.dbg_t[6 * gwarp + 2] = gtimer();
  if (ws.dbg_t && lane == 0) { ws.dbg_t[6 * gwarp + 3] = dbg_nseg; ws.dbg_t[6 * gwarp + 4] = dbg_tseg; ws.dbg_t[6 * gwarp + 5] = dbg_tdone; }
  // --------------------------------------------- exit: last CTA resets ----
  // one arrival per CTA: the barrier orders the CTA's warps' counter updates
  // before thread 0's acq_rel (release is cumulative), and the last CTA sees
  // every CTA's updates before it resets them
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long w;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(w) : "l"(ws.warps_done) : "memory");
    if ((int64_t)w == (int64_t)gridDim.x - 1) {
      *ws.block_ticket = 0ull;
      *ws.q_tail = 0ull;
      *ws.q_head = 0ull;
      *ws.blocks_done = 0ull;
      __threadfence();
      *ws.warps_done = 0ull;
    }
  }
}

}  // namespace

// workspace layout inside the caller-provided buffer
// upper bound on long-row segments: sum of ceil(len/SEG) over rows longer than LONG
static int64_t max_segments(int64_t nnz) { return nnz / SEG_MIN + nnz / SPLIT_MIN + 64; }

size_t segmented_ws_bytes(int64_t nnz) {
  return 64 * 8 + (size_t)max_segments(nnz) * (sizeof(SegEntry) + 8 + 4) + 4096;
}
// byte offset and length of the queue (initialised to all-ones: row = -1 = empty)
void segmented_ws_qrow(int64_t nnz, size_t* off, size_t* len) {
  *off = 64 * 8;
  *len = (size_t)max_segments(nnz) * sizeof(SegEntry);
}

bool segmented_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 2 || !a.keyed || !a.offsets) { *why = "not a keyed CSR nest"; return false; }
  if (a.op != OP_SUM || a.in_dtype != DT_F32) { *why = "segmented kernel: f32 sum only"; return false; }
  if (a.verify & (V_FINGERPRINT | V_PARTIALS)) { *why = "segmented kernel: coverage verify only"; return false; }
  LevelView v = device_levels(a);
  if (v.n != 2) { *why = "needs [cluster..warp dynamic(RB) rows] [lane static(4) positions]"; return false; }
  const DevLevel *t = v.l[0], *l = v.l[1];
  if (t->sfirst != S_CLUSTER || t->slast != S_WARP || t->sched != SCHED_DYNAMIC || t->chunk != RB || t->loop != 0) {
    *why = "teams-warps level must be dynamic(256) over rows";
    return false;
  }
  if (!is_level(l, S_LANE) || l->sched != SCHED_STATIC_CHUNK || (l->chunk != 8 && l->chunk != 16) || l->loop != 2) {
    *why = "lane level must be static(8) or static(16) over the collapsed nonzeros (loop 2)";
    return false;
  }
  if (a.radix[S_WARP] != WARPS) { *why = "W must be 8"; return false; }
  // positions inside a block of RB rows are 32-bit, relative to the block's
  // window origin; the array itself is addressed in 64 bits (tensor-map
  // coordinates in rows of 32 values: nnz < 2^36).  Below 2^31 nonzeros no
  // block can overflow; above, the caller's row-length bound must prove it.
  // (the launch checks the block spans at >= 2^31 nonzeros: segmented_span_ok)
  if (a.n1 >= (1ll << 36) - 64) { *why = "nnz per rank must be < 2^36"; return false; }
  if (((uintptr_t)a.in & 3) != 0) { *why = "values not element-aligned"; return false; }
  return true;
}

// the largest span (nonzeros) of a block of RB rows
__global__ void block_span_kernel(const int64_t* __restrict__ off, int64_t R, unsigned long long* span) {
  const int64_t nb = (R + RB - 1) / RB;
  unsigned long long m = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = (b + 1) * RB < R ? (b + 1) * RB : R;
    const unsigned long long d = (unsigned long long)(off[e] - off[b * RB]);
    m = d > m ? d : m;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(span, m);
}

// Positions inside a row block are 32-bit: below 2^31 nonzeros per rank no
// block can overflow; above, either the caller's row-length bound proves it
// (max_inner * RB < 2^31) or a check kernel measures the block spans, which
// needs one host synchronisation (not possible while a graph is captured).
// `scratch`: 8 device bytes.  Sets *ok; returns a CUDA error or success.
cudaError_t segmented_span_ok(const NestArgs& a, unsigned long long* scratch, cudaStream_t s, bool* ok,
                              bool* needs_sync) {
  constexpr long long kLim = 0x7FFFFF00ll;
  *needs_sync = false;
  *ok = true;
  if (a.n1 < 0x7FFFFFF0 || (a.max_inner > 0 && a.max_inner * RB < kLim)) return cudaSuccess;
  *needs_sync = true;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &cs);
  if (e != cudaSuccess) return e;
  if (cs != cudaStreamCaptureStatusNone) {
    *ok = false;
    return cudaSuccess;
  }
  unsigned long long h = 0;
  if ((e = cudaMemsetAsync(scratch, 0, 8, s)) != cudaSuccess) return e;
  const int64_t nb = (a.n0 + RB - 1) / RB;
  const int grid = (int)((nb + 255) / 256 < 4 * 148 ? (nb + 255) / 256 : 4 * 148);
  if (grid > 0) block_span_kernel<<<grid, 256, 0, s>>>(a.offsets, a.n0, scratch);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(&h, scratch, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  *ok = (long long)h < kLim;
  return cudaSuccess;
}

// offsets + shift into the workspace copy (misaligned values, below)
__global__ void shift_offsets_kernel(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                                     int32_t shift) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] + shift;
}

cudaError_t launch_segmented(const NestArgs& a_call, void* wsbuf, int64_t nnz, int64_t* off_ws, cudaStream_t s,
                             const char** name) {
  *name = "segmented_csr";
  // values off a 16-byte boundary (a slice of a tensor): the kernel sees the
  // array from the granule boundary before them — in_shift more elements —
  // and reads offsets + in_shift from a workspace copy, so TMA windows and the
  // tensor map stay aligned and the aligned call's kernel is untouched; the
  // elements before the first row belong to no row; coverage is written at
  // position - in_shift
  NestArgs a = a_call;
  a.in_shift = (int32_t)(((uintptr_t)a_call.in & 15) / 4);
  if (a.in_shift) {
    if (!off_ws) return cudaErrorInvalidValue;
    a.in = (const float*)a_call.in - a.in_shift;
    a.n1 = a_call.n1 + a.in_shift;
    const int64_t n = a.n0 + 1;
    const int grid = (int)((n + 255) / 256 < 4 * 148 ? (n + 255) / 256 : 4 * 148);
    shift_offsets_kernel<<<grid, 256, 0, s>>>(a_call.offsets, off_ws, n, a.in_shift);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    a.offsets = off_ws;
  }
  const int64_t maxseg = max_segments(nnz);
  unsigned char* p = (unsigned char*)wsbuf;
  SegWS ws;
  ws.block_ticket = (unsigned long long*)p;
  ws.q_tail = ws.block_ticket + 1;
  ws.q_head = ws.block_ticket + 2;
  ws.blocks_done = ws.block_ticket + 3;
  ws.warps_done = ws.block_ticket + 4;
  p += 64 * 8;
  ws.q = (SegEntry*)p;
  p += maxseg * sizeof(SegEntry);
  ws.partials = (double*)p;
  p += maxseg * 8;
  ws.tickets = (unsigned int*)p;
  ws.q_cap = maxseg;
  ws.dbg_t = nullptr;
  // process-wide debug buffer and tensor-map cache: guarded, and the debug
  // buffer regrows when a call has more warps than the last
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static unsigned long long* dbg_buf = nullptr;
  static int64_t dbg_warps = 0;
  const bool times = getenv("HPAR_SEG_TIMES") != nullptr;
  const int64_t nwarps = a.C * a.K * WARPS;
  if (times) {
    if (nwarps > dbg_warps) {
      cudaFree(dbg_buf);
      dbg_buf = nullptr;
      dbg_warps = 0;
      if (cudaMalloc(&dbg_buf, nwarps * 6 * 8) == cudaSuccess) dbg_warps = nwarps;
    }
    ws.dbg_t = dbg_buf;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.C * a.K));
  cfg.blockDim = dim3(WARPS * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool f32 = a.out_dtype == DT_F32;
  // the values as a [nnz / 32][32] fp32 tensor for the swizzled window boxes
  // (the last partial row is read directly by the kernel)
  static CUtensorMap tmx;
  static const void* tmx_ptr = nullptr;
  static int64_t tmx_rows = -1;
  bool tmx_ok = false;
  {
    const int64_t rows32 = a.n1 / 32;
    if (rows32 >= 1 && rows32 < (1ll << 31) && ((uintptr_t)a.in & 15) == 0) {
      if (tmx_ptr == a.in && tmx_rows == rows32) {
        tmx_ok = true;
      } else if (PFN_cuTensorMapEncodeTiled_v12000 enc = seg_encode_fn()) {
        const cuuint64_t dims[2] = {32, (cuuint64_t)rows32};
        const cuuint64_t strides[1] = {128};
        const cuuint32_t box[2] = {32, 16};
        const cuuint32_t estr[2] = {1, 1};
        if (enc(&tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)a.in, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
          tmx_ptr = a.in;
          tmx_rows = rows32;
          tmx_ok = true;
        }
      }
    }
  }
  static int swz_knob = -1;
  if (swz_knob < 0) swz_knob = getenv("HPAR_SEG_SWZ") ? atoi(getenv("HPAR_SEG_SWZ")) : 1;
  if (!swz_knob) tmx_ok = false;
  auto pick = [&](auto kern, size_t warp_smem) -> cudaError_t {
    cfg.dynamicSmemBytes = WARPS * warp_smem + 1024;  // + alignment of the 1 KiB-aligned warp areas
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)cfg.dynamicSmemBytes);
    if (e != cudaSuccess) return e;
    // every CTA must be co-resident (no CTA may start after others exit):
    // clamp the grid to the clusters that fit at once
    int fit = 0;
    e = cudaOccupancyMaxActiveClusters(&fit, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (fit > 0 && (int64_t)fit < a.C) cfg.gridDim = dim3((unsigned)(fit * a.K));
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("HPAR_SEG_DEBUG") ? atoi(getenv("HPAR_SEG_DEBUG")) : 0;
    static int lmin = -1;
    if (lmin < 0) lmin = getenv("HPAR_SEG_LONG") ? atoi(getenv("HPAR_SEG_LONG")) : (int)LONG;
    if (lmin < (int)SPLIT_MIN) lmin = (int)SPLIT_MIN;  // the queue is sized for rows > SPLIT_MIN
    static int cbk = -1;
    if (cbk < 0) cbk = getenv("HPAR_SEG_CB") ? atoi(getenv("HPAR_SEG_CB")) : CB;
    if (cbk < 1) cbk = 1;
    // segment length: SEG at full size (2^28 nonzeros), halved per halving of
    // the shard down to SEG_MIN (scripts/sweep_seglen.sh: 16384 / 8192 / 4096
    // best at 1 / 2 / 4-8 GPUs' shards; HPAR_SEG_LEN_RT overrides)
    static int segk = -1;
    if (segk < 0) segk = getenv("HPAR_SEG_LEN_RT") ? atoi(getenv("HPAR_SEG_LEN_RT")) : 0;
    int seg = (int)SEG;
    if (segk >= (int)SEG_MIN) {
      seg = segk;
    } else {
      for (int64_t n = a.n1; seg > (int)SEG_MIN && n <= (1ll << 27); n *= 2) seg /= 2;
    }
    return cudaLaunchKernelEx(&cfg, kern, a, ws, dbg, lmin, cbk, seg, tmx);
  };
  // variant: LPL from the nest's lane chunk; ring depth D (HPAR_SEG_D knob)
  const int lpl = device_levels(a).l[1]->chunk;
  static int dknob = -1;
  if (dknob < 0) dknob = getenv("HPAR_SEG_D") ? atoi(getenv("HPAR_SEG_D")) : 0;
  static int f32seg = -1;  // (knob) 1 = fp32 segmented windows (DESIGN §6 (l), (q))
  if (f32seg < 0) f32seg = getenv("HPAR_SEG_F32") ? atoi(getenv("HPAR_SEG_F32")) : 0;
  auto launch_v = [&](auto lpl_c, auto d_c) -> cudaError_t {
    constexpr int L = decltype(lpl_c)::value, DD = decltype(d_c)::value;
    if constexpr (L == 16 && DD == 2) {
      if (tmx_ok && f32seg) {  // fp32 segmented windows (knob)
        if (a.verify)
          return f32 ? pick(segmented_kernel<true, true, L, DD, true, true>, sizeof(WarpSmem<float, L, DD>))
                     : pick(segmented_kernel<true, false, L, DD, true, true>, sizeof(WarpSmem<double, L, DD>));
        return f32 ? pick(segmented_kernel<false, true, L, DD, true, true>, sizeof(WarpSmem<float, L, DD>))
                   : pick(segmented_kernel<false, false, L, DD, true, true>, sizeof(WarpSmem<double, L, DD>));
      }
      if (tmx_ok) {
        if (a.verify)
          return f32 ? pick(segmented_kernel<true, true, L, DD, true>, sizeof(WarpSmem<float, L, DD>))
                     : pick(segmented_kernel<true, false, L, DD, true>, sizeof(WarpSmem<double, L, DD>));
        return f32 ? pick(segmented_kernel<false, true, L, DD, true>, sizeof(WarpSmem<float, L, DD>))
                   : pick(segmented_kernel<false, false, L, DD, true>, sizeof(WarpSmem<double, L, DD>));
      }
    }
    if (a.verify)
      return f32 ? pick(segmented_kernel<true, true, L, DD>, sizeof(WarpSmem<float, L, DD>))
                 : pick(segmented_kernel<true, false, L, DD>, sizeof(WarpSmem<double, L, DD>));
    return f32 ? pick(segmented_kernel<false, true, L, DD>, sizeof(WarpSmem<float, L, DD>))
               : pick(segmented_kernel<false, false, L, DD>, sizeof(WarpSmem<double, L, DD>));
  };
  using I8 = std::integral_constant<int, 8>;
  using I16 = std::integral_constant<int, 16>;
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  using I4 = std::integral_constant<int, 4>;
  cudaError_t er;
  if (lpl == 16) er = (dknob == 3) ? launch_v(I16(), I3()) : launch_v(I16(), I2());
  else er = (dknob == 3) ? launch_v(I8(), I3()) : launch_v(I8(), I4());
  if (times && er == cudaSuccess) {  // debug only: per-warp phase times
    cudaStreamSynchronize(s);
    const int64_t nwarps = (int64_t)cfg.gridDim.x * WARPS;
    unsigned long long* h = (unsigned long long*)malloc(nwarps * 48);
    cudaMemcpy(h, dbg_buf, nwarps * 48, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, tmax = 0;
    for (int64_t w = 0; w < nwarps; ++w) { if (h[6 * w] < t0) t0 = h[6 * w]; if (h[6 * w + 2] > tmax) tmax = h[6 * w + 2]; }
    double s1 = 0, s2 = 0, st = 0, p1max = 0, p1min = 1e30, nseg = 0, tseg = 0, tdone = 0, tdmin = 1e30;
    for (int64_t w = 0; w < nwarps; ++w) {
      const double a0 = (h[6 * w] - t0) * 1e-3, a1 = (h[6 * w + 1] - t0) * 1e-3, a2 = (h[6 * w + 2] - t0) * 1e-3;
      st += a0; s1 += a1; s2 += a2; if (a1 > p1max) p1max = a1; if (a1 < p1min) p1min = a1;
      nseg += h[6 * w + 3]; tseg += h[6 * w + 4] * 1e-3;
      const double td = h[6 * w + 5] ? (h[6 * w + 5] - t0) * 1e-3 : 0; tdone += td; if (td > 0 && td < tdmin) tdmin = td;
    }
    fprintf(stderr, "seg times (us): start avg %.1f | phase1 end avg %.1f min %.1f max %.1f | exit avg %.1f max %.1f"
            " | phase2 segs/warp %.2f, us/seg %.2f, all-blocks-done seen avg %.1f min %.1f\n",
            st / nwarps, s1 / nwarps, p1min, p1max, s2 / nwarps, (tmax - t0) * 1e-3, nseg / nwarps, tseg / (nseg > 0 ? nseg : 1), tdone / nwarps, tdmin);
    {  // phase-1 end percentiles
      double* e1 = (double*)malloc(nwarps * sizeof(double));
      for (int64_t w = 0; w < nwarps; ++w) e1[w] = (h[6 * w + 1] - t0) * 1e-3;
      std::sort(e1, e1 + nwarps);
      fprintf(stderr, "seg phase1 end percentiles (us): p10 %.1f p50 %.1f p90 %.1f p99 %.1f p99.9 %.1f\n", e1[nwarps / 10],
              e1[nwarps / 2], e1[nwarps * 9 / 10], e1[nwarps * 99 / 100], e1[nwarps * 999 / 1000]);
      free(e1);
    }
    free(h);
  }
  return er;
}

}  // namespace hpar
