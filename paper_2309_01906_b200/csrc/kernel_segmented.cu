// kernel_segmented.cu — CSR segmented reduction with dynamic per-level
// chunking and length-class level selection (config 3).
//
// Nest (what this kernel executes; SURVEY §8(c) reading #14):
//   GPU            static over rows                     (host: rank shard)
//   cluster..warp  dynamic(RB) over rows: every warp of the GPU is a sibling
//                  (collapsed level, flags = ∩ -> dynamic, atomic); a warp
//                  claims blocks of RB consecutive rows from a GPU ticket
//   lane           static(4) over the block's nonzeros, in 16-byte vectors
//                  of the values array (window of 128 nonzeros per warp step)
// Length class -> level (P:344-359 versioning; P:140 grainedness): a row
// longer than L nonzeros is not reduced by its block's warp; it is split into
// segments of S nonzeros that any warp claims from a GPU queue, and the LAST
// segment to finish folds the row's segment partials in ascending order
// (single-pass, wait-free: warps have no grid barrier).  Blocks never share a
// row, so short/medium rows need no cross-warp fix-up.
//
// Inside a block (per warp): the block's RB+1 offsets are staged in shared
// memory; row starts are marked as heads in a per-warp table; each 128-wide
// window is reduced with a segmented warp scan (lane -> warp level), fp32
// inside a window, fp64 carries across windows and for long-row segments.
// Empty rows write 0.  Results are deterministic (fixed trees and orders).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include "fused_common.cuh"

namespace hpar {
namespace {

constexpr int RB = 256;         // rows per block claim
constexpr int64_t LONG = 1024;  // a row with more nonzeros is split
constexpr int64_t SEG = 8192;   // nonzeros per long-row segment
constexpr int WARPS = 8;        // warps per CTA (all workers)
constexpr int NV = 2;           // 16-byte vectors per lane per window
constexpr int WIN = 128 * NV;   // nonzeros per window (lane l: 4*NV contiguous at 4*NV*l)
constexpr int LPL = 4 * NV;     // nonzeros per lane per window
constexpr int D = 4;            // window prefetch depth (cp.async ring)
constexpr int LBIT = 1 << 30;   // row-id flag: a long row (its nonzeros are phase 2's)
constexpr int CB = 32;          // row blocks per CTA claim (CTA-level dynamic chunk)
constexpr int NSB = 8;          // ring of claimed CTA chunks

struct CtaSmem {
  unsigned int ctr;            // warp-level ticket over the CTA's chunk list
  int pad;
  long long sblock[NSB];       // CTA chunk j (mod NSB) -> GPU chunk index
  volatile int tag[NSB];       // j + 1 once sblock[j % NSB] is published
};

struct SegWS {
  unsigned long long* block_ticket;  // next row block
  unsigned long long* q_tail;        // long-row segments appended
  unsigned long long* q_head;        // long-row segments claimed
  unsigned long long* blocks_done;   // row blocks finished
  unsigned long long* warps_done;    // warps exited (last one resets)
  unsigned long long* part_next;     // partial slots allocated
  int64_t* q_row;                    // segment -> row (-1: not yet published)
  int32_t* q_seg;                    // segment -> index within the row
  int64_t* q_pbase;                  // segment -> first partial slot of its row
  double* partials;                  // per segment partial sums
  unsigned int* tickets;             // per long row (at its pbase): segments done
  int64_t q_cap;
};

struct WarpSmem {
  float4 ring[D][NV][32];  // window ring: slot, vector, lane
  int32_t head[WIN];       // window head table: (block row + 1) | LBIT if long, 0 = none
  int64_t off[RB + 2];     // the block's RB+1 offsets (+1 pad keeps 16-byte alignment)
};

// 16-byte async global -> shared copy; bytes beyond src_bytes are zero-filled
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Warp segmented inclusive scan of (row, value): row >= 0 marks a lane whose
// segment starts in it (its last head); value = its trailing sum.
__device__ __forceinline__ void seg_scan(int& row, float& v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int r2 = __shfl_up_sync(0xffffffffu, row, off);
    const float v2 = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off && row < 0) {
      row = r2;
      v += v2;
    }
  }
}

template <bool VERIFY, bool OUT_F32>
__global__ void __launch_bounds__(WARPS * 32) segmented_kernel(const __grid_constant__ NestArgs a, SegWS ws, int dbg) {
  extern __shared__ __align__(16) unsigned char seg_dsm[];
  __shared__ CtaSmem cs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem& sm = ((WarpSmem*)seg_dsm)[warp];
  if (threadIdx.x == 0) cs.ctr = 0;
  if (threadIdx.x < NSB) cs.tag[threadIdx.x] = 0;
  __syncthreads();
  const int64_t* offs = a.offsets;
  const float* x = (const float*)a.in;
  const int64_t R = a.n0;
  const int64_t nnz_all = a.n1;
  const int64_t nblocks = (R + RB - 1) / RB;
  const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + (int64_t)blockIdx.x * WARPS * 32 + threadIdx.x;
  auto write_row = [&](int64_t r, double v) {
    if constexpr (OUT_F32) ((float*)a.out)[r] = (float)v;
    else ((double*)a.out)[r] = v;
  };
  auto cover = [&](int64_t p) {
    if constexpr (VERIFY) {
      if (a.verify & V_COVERAGE) {
        a.owner[p] = leaf;
        atomicAdd(&a.count[p], 1u);
      }
    }
  };
  for (int i = lane; i < WIN; i += 32) sm.head[i] = 0;
  __syncwarp();

  // ------------------------------------------------ phase 1: row blocks ----
  // Software pipeline per warp: the claim of block j+2 and the offsets of
  // block j+1 are in flight while block j is reduced; windows are copied
  // D ahead with cp.async into the warp's shared-memory ring.
  // Two-level dynamic chunking: a warp takes the next block of its CTA's
  // chunk list from a shared-memory ticket; the warp that opens chunk j
  // claims it from the GPU ticket (CB blocks at a time) and publishes it.
  const int64_t nchunks = (nblocks + CB - 1) / CB;
  auto claim = [&]() -> unsigned long long {
    long long blk = 0;
    if (lane == 0) {
      const unsigned v = atomicAdd(&cs.ctr, 1u);
      const unsigned j = v / CB, sub = v % CB;
      if (sub == 0) {
        cs.sblock[j % NSB] = (long long)atomicAdd(ws.block_ticket, 1ull);
        __threadfence_block();
        cs.tag[j % NSB] = (int)(j + 1);
      } else {
        while (cs.tag[j % NSB] != (int)(j + 1)) __nanosleep(32);
        __threadfence_block();
      }
      const long long g = ((volatile long long*)cs.sblock)[j % NSB];
      blk = (g < nchunks) ? g * CB + sub : (long long)nblocks + 1;
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
  auto load4 = [&](int64_t p, int64_t lo, int64_t hi) -> float4 {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p >= lo && p + 3 < hi) {
      t = ld_stream_f4((const float4*)(x + p));
    } else if (p + 3 >= lo && p < hi) {
      if (p >= lo && p < hi) t.x = x[p];
      if (p + 1 >= lo && p + 1 < hi) t.y = x[p + 1];
      if (p + 2 >= lo && p + 2 < hi) t.z = x[p + 2];
      if (p + 3 >= lo && p + 3 < hi) t.w = x[p + 3];
    }
    return t;
  };
  unsigned long long my_blocks = 0;  // added to blocks_done once, when this warp leaves phase 1
  unsigned long long u = claim();
  load_offs(u);
  while ((int64_t)u < nblocks) {
    const unsigned long long u1 = claim();
    const int64_t r0 = (int64_t)u * RB;
    const int nr = (int)((R - r0 < RB) ? (R - r0) : RB);
#pragma unroll
    for (int k = 0; k < (RB + 1 + 31) / 32; ++k) {
      const int i = lane + 32 * k;
      if (i <= nr) sm.off[i] = offr[k];
    }
    __syncwarp();
    load_offs(u1);  // next block's offsets, in flight during this block
    const int64_t P0 = sm.off[0], P1 = sm.off[nr];
    // long rows: enqueue their segments; empty rows: 0
    bool my_long = false;
    for (int i = lane; i < nr; i += 32) {
      const int64_t len = sm.off[i + 1] - sm.off[i];
      if (len == 0) write_row(r0 + i, 0.0);
      if (len > LONG) {
        my_long = true;
        const int64_t ns = (len + SEG - 1) / SEG;
        const unsigned long long q = atomicAdd(ws.q_tail, (unsigned long long)ns);
        const unsigned long long pb = atomicAdd(ws.part_next, (unsigned long long)ns);
        for (int64_t k = 0; k < ns; ++k) {
          ws.q_seg[q + k] = (int32_t)k;
          ws.q_pbase[q + k] = (int64_t)pb;
        }
        __threadfence();  // entries before their publication
        for (int64_t k = 0; k < ns; ++k) *(volatile int64_t*)&ws.q_row[q + k] = r0 + i;
      }
    }
    const bool had_long = __any_sync(0xffffffffu, my_long);
    // windows of WIN nonzeros, 16-byte aligned.  Every non-empty row starting
    // in a window is a head; long rows are heads too (they close the previous
    // row) but carry LBIT and are never written here.  Positions inside the
    // window loop are 32-bit, relative to `base` (nnz < 2^31 per rank).
    const int64_t base = P0 & ~(int64_t)15;
    const float* xb = x + base;
    const int p0 = (int)(P0 - base), p1 = (int)(P1 - base);
    const int64_t lim64 = nnz_all - base;
    const int lim = lim64 > 0x7FFFFFF0 ? 0x7FFFFFF0 : (int)lim64;  // readable nonzeros from base
    auto issue = [&](int wr, int slot) {  // copy window at relative position wr
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int p = wr + LPL * lane + 4 * v;
        const int bytes = (p + 4 <= lim) ? 16 : (p < lim ? (lim - p) * 4 : 0);
        cp_async16(&sm.ring[slot][v][lane], xb + (bytes ? p : 0), bytes);
      }
      cp_async_commit();
    };
    int cur = 0;           // next block row whose start is not yet marked
    int open_row = -1;     // (block row | LBIT) of the open segment, -1: none
    double carry = 0.0;    // fp64 sum of the open row before this window
    int slot = 0;
#pragma unroll
    for (int i = 0; i < D; ++i) issue(WIN * i, i);
    for (int wr = (dbg & 2) ? p1 : 0; wr < p1; wr += WIN) {
      // inside a long row with no head ahead in this window: skip to the window
      // holding the next row start (the long row's nonzeros are phase 2's)
      if (open_row >= 0 && (open_row & LBIT)) {
        const int nxt = (cur < nr) ? (int)(sm.off[cur] - base) : p1;
        if (nxt >= wr + WIN) {
          wr = (nxt / WIN) * WIN;
          if (wr >= p1) break;
          cp_async_wait<0>();
          slot = 0;
#pragma unroll
          for (int i = 0; i < D; ++i) issue(wr + WIN * i, i);
        }
      }
      const int wend = wr + WIN;
      // mark heads: non-empty rows starting in [wr, wend)
      while (cur < nr && (int)(sm.off[cur] - base) < wend) {
        const int i = cur + lane;
        bool in = false;
        if (i < nr) {
          const int s_ = (int)(sm.off[i] - base), e_ = (int)(sm.off[i + 1] - base);
          in = s_ < wend;
          if (in && e_ > s_) sm.head[s_ - wr] = (i + 1) | ((e_ - s_ > LONG) ? LBIT : 0);
        }
        cur += __popc(__ballot_sync(0xffffffffu, in));
      }
      __syncwarp();
      // this lane's LPL nonzeros (copied D windows ago); refill the slot
      const int p = wr + LPL * lane;
      cp_async_wait<D - 1>();
      float v[LPL];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const float4 t = sm.ring[slot][q][lane];
        v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
      }
      issue(wr + WIN * D, slot);
      slot = (slot + 1 == D) ? 0 : slot + 1;
      if (p < p0 || p + LPL > p1) {
#pragma unroll
        for (int k = 0; k < LPL; ++k)
          if (p + k < p0 || p + k >= p1) v[k] = 0.f;  // neighbours' nonzeros
      }
      int h[LPL];
#pragma unroll
      for (int q = 0; q < LPL / 4; ++q) {
        const int4 hq = *(const int4*)&sm.head[LPL * lane + 4 * q];
        h[4 * q] = hq.x; h[4 * q + 1] = hq.y; h[4 * q + 2] = hq.z; h[4 * q + 3] = hq.w;
        *(int4*)&sm.head[LPL * lane + 4 * q] = make_int4(0, 0, 0, 0);
      }
      // lane-local segmented sums (branch-free); rows entirely inside the
      // lane are written when their successor's head is met
      float pre = 0.f;   // before the first head: belongs to the open row
      float tail = 0.f;  // from the last head on
      int last = -1;     // (block row | LBIT) of the last head in this lane
#pragma unroll
      for (int k = 0; k < LPL; ++k) {
        const bool hk = h[k] != 0;
        if (hk && last >= 0 && !(last & LBIT)) write_row(r0 + last, (double)tail);
        last = hk ? h[k] - 1 : last;
        tail = hk ? 0.f : tail;
        const bool in_open = last < 0;
        pre = in_open ? pre + v[k] : pre;
        tail = in_open ? tail : tail + v[k];
      }
      // lane -> warp: segmented scan of (last head row, trailing value)
      int srow = last;
      float sval = (last >= 0) ? tail : pre;
      seg_scan(srow, sval);
      int erow = __shfl_up_sync(0xffffffffu, srow, 1);
      float eval = __shfl_up_sync(0xffffffffu, sval, 1);
      if (lane == 0) { erow = -1; eval = 0.f; }
      const int prev = (erow >= 0) ? erow : open_row;  // row of the nonzeros before the first head
      // the row open before this lane's first head ends there
      if (last >= 0 && prev >= 0 && !(prev & LBIT)) {
        const double tot = (erow >= 0) ? (double)(eval + pre) : carry + (double)eval + (double)pre;
        write_row(r0 + prev, tot);
      }
      if constexpr (VERIFY) {
        int row = prev;
#pragma unroll
        for (int k = 0; k < LPL; ++k) {
          if (h[k]) row = h[k] - 1;
          if (p + k >= p0 && p + k < p1 && row >= 0 && !(row & LBIT)) cover(base + p + k);
        }
      }
      // window end: the trailing open segment carries into the next window
      const int trow = __shfl_sync(0xffffffffu, srow, 31);
      const float tval = __shfl_sync(0xffffffffu, sval, 31);
      if (trow >= 0) {
        open_row = trow;
        carry = (double)tval;
      } else {
        carry += (double)tval;
      }
    }
    cp_async_wait<0>();  // the ring is reused by the next block
    // the last open row of the block ends at P1
    if (lane == 0 && open_row >= 0 && !(open_row & LBIT)) write_row(r0 + open_row, carry);
    __syncwarp();
    if (had_long && lane == 0) __threadfence();  // queue entries visible before blocks_done says so
    ++my_blocks;
    u = u1;
  }

  if (lane == 0) {
    __threadfence();
    atomicAdd(ws.blocks_done, my_blocks);
  }

  // -------------------------------------------- phase 2: long-row segments ----
  for (;;) {
    unsigned long long q = 0;
    if (lane == 0) q = atomicAdd(ws.q_head, 1ull);
    q = __shfl_sync(0xffffffffu, q, 0);
    // wait until segment q exists, or until no segment can appear any more
    bool have = false;
    for (;;) {
      unsigned long long tail = 0, done = 0;
      if (lane == 0) {
        tail = *(volatile unsigned long long*)ws.q_tail;
        done = *(volatile unsigned long long*)ws.blocks_done;
      }
      tail = __shfl_sync(0xffffffffu, tail, 0);
      done = __shfl_sync(0xffffffffu, done, 0);
      if (q < tail) { have = true; break; }
      if ((int64_t)done >= nblocks) {
        __threadfence();
        if (lane == 0) tail = *(volatile unsigned long long*)ws.q_tail;
        tail = __shfl_sync(0xffffffffu, tail, 0);
        have = q < tail;
        break;
      }
      __nanosleep(200);
    }
    if (!have) break;
    int64_t row = -1;
    if (lane == 0) {
      while ((row = *(volatile int64_t*)&ws.q_row[q]) < 0) __nanosleep(64);
      ws.q_row[q] = -1;  // self-reset for the next call
    }
    row = __shfl_sync(0xffffffffu, row, 0);
    __threadfence();
    const int32_t k = *(volatile int32_t*)&ws.q_seg[q];
    const int64_t pb = *(volatile int64_t*)&ws.q_pbase[q];
    const int64_t s0 = offs[row], e0 = offs[row + 1];
    const int64_t ns = (e0 - s0 + SEG - 1) / SEG;
    const int64_t b = s0 + (int64_t)k * SEG;
    const int64_t e = (b + SEG < e0) ? b + SEG : e0;
    double acc = 0.0;
    {
      constexpr int D2 = 8;
      int64_t wb = (dbg & 1) ? e : (b & ~(int64_t)3);
      for (; wb < e; wb += 128 * D2) {
        float4 t[D2];
#pragma unroll
        for (int i = 0; i < D2; ++i) t[i] = load4(wb + 128 * i + 4 * lane, b, e);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < D2; ++i) s += (t[i].x + t[i].y) + (t[i].z + t[i].w);
        acc += (double)s;
        if constexpr (VERIFY) {
          for (int i = 0; i < D2; ++i)
            for (int j = 0; j < 4; ++j) {
              const int64_t pp = wb + 128 * i + 4 * lane + j;
              if (pp >= b && pp < e) cover(pp);
            }
        }
      }
    }
    acc = warp_fold<OP_SUM>(acc);
    if (lane == 0) {
      ws.partials[pb + k] = acc;
      __threadfence();
      const unsigned t = atomicAdd(&ws.tickets[pb], 1u);
      if ((int64_t)t == ns - 1) {  // last segment of the row: ordered fold
        __threadfence();
        double tot = 0.0;
        for (int64_t j = 0; j < ns; ++j) tot += *(volatile double*)&ws.partials[pb + j];
        write_row(row, tot);
        ws.tickets[pb] = 0u;
      }
    }
  }

  // --------------------------------------------- exit: last warp resets ----
  if (lane == 0) {
    __threadfence();
    const unsigned long long w = atomicAdd(ws.warps_done, 1ull);
    if ((int64_t)w == (int64_t)gridDim.x * WARPS - 1) {
      *ws.block_ticket = 0ull;
      *ws.q_tail = 0ull;
      *ws.q_head = 0ull;
      *ws.blocks_done = 0ull;
      *ws.part_next = 0ull;
      __threadfence();
      *ws.warps_done = 0ull;
    }
  }
}

}  // namespace

// workspace layout inside the caller-provided buffer
// upper bound on long-row segments: sum of ceil(len/SEG) over rows longer than LONG
static int64_t max_segments(int64_t nnz) { return nnz / SEG + nnz / LONG + 64; }

size_t segmented_ws_bytes(int64_t nnz) {
  return 64 * 8 + (size_t)max_segments(nnz) * (8 + 8 + 8 + 4 + 4) + 4096;
}
// byte offset and length of the q_row array (initialised to -1 = empty)
void segmented_ws_qrow(int64_t nnz, size_t* off, size_t* len) {
  *off = 64 * 8;
  *len = (size_t)max_segments(nnz) * 8;
}

bool segmented_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 2 || !a.keyed || !a.offsets) { *why = "not a keyed CSR nest"; return false; }
  if (a.op != OP_SUM || a.in_dtype != DT_F32) { *why = "segmented kernel: f32 sum only"; return false; }
  if (a.verify & (V_FINGERPRINT | V_PARTIALS)) { *why = "segmented kernel: coverage verify only"; return false; }
  LevelView v = device_levels(a);
  if (v.n != 2) { *why = "needs [cluster..warp dynamic(RB) rows] [lane static(4) positions]"; return false; }
  const DevLevel *t = v.l[0], *l = v.l[1];
  if (t->sfirst != S_CLUSTER || t->slast != S_WARP || t->sched != SCHED_DYNAMIC || t->chunk != RB || t->loop != 0) {
    *why = "teams-warps level must be dynamic(128) over rows";
    return false;
  }
  if (!is_level(l, S_LANE) || l->sched != SCHED_STATIC_CHUNK || l->chunk != 4 * NV || l->loop != 2) {
    *why = "lane level must be static(8) over the collapsed nonzeros (loop 2)";
    return false;
  }
  if (a.radix[S_WARP] != WARPS) { *why = "W must be 8"; return false; }
  if (a.n1 >= 0x7FFFFFF0) { *why = "nnz per rank must be < 2^31 (32-bit window positions)"; return false; }
  if (((uintptr_t)a.in & 15) != 0) { *why = "values not 16-byte aligned"; return false; }
  return true;
}

cudaError_t launch_segmented(const NestArgs& a, void* wsbuf, int64_t nnz, cudaStream_t s, const char** name) {
  *name = "segmented_csr";
  const int64_t maxseg = max_segments(nnz);
  unsigned char* p = (unsigned char*)wsbuf;
  SegWS ws;
  ws.block_ticket = (unsigned long long*)p;
  ws.q_tail = ws.block_ticket + 1;
  ws.q_head = ws.block_ticket + 2;
  ws.blocks_done = ws.block_ticket + 3;
  ws.warps_done = ws.block_ticket + 4;
  ws.part_next = ws.block_ticket + 5;
  p += 64 * 8;
  ws.q_row = (int64_t*)p;
  p += maxseg * 8;
  ws.q_pbase = (int64_t*)p;
  p += maxseg * 8;
  ws.partials = (double*)p;
  p += maxseg * 8;
  ws.q_seg = (int32_t*)p;
  p += maxseg * 4;
  ws.tickets = (unsigned int*)p;
  ws.q_cap = maxseg;
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
  cfg.dynamicSmemBytes = WARPS * sizeof(WarpSmem);
  auto pick = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)cfg.dynamicSmemBytes);
    if (e != cudaSuccess) return e;
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("HPAR_SEG_DEBUG") ? atoi(getenv("HPAR_SEG_DEBUG")) : 0;
    return cudaLaunchKernelEx(&cfg, kern, a, ws, dbg);
  };
  const bool f32 = a.out_dtype == DT_F32;
  if (a.verify) return f32 ? pick(segmented_kernel<true, true>) : pick(segmented_kernel<true, false>);
  return f32 ? pick(segmented_kernel<false, true>) : pick(segmented_kernel<false, false>);
}

}  // namespace hpar
