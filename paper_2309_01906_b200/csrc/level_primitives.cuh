// level_primitives.cuh — per-level partition, barrier and combine primitives
// of the B200 hierarchy (sm_100a), used by every kernel of libhpar.so.
//
//  lane    : __syncwarp barrier, SHFL trees (K1/K4)
//  warp    : shared-memory slots + bar.sync ("fallback using memory
//            one level up")
//  CTA     : DSMEM (st.shared::cluster / st.async + mbarrier) + split
//            barrier.cluster (P:406-413, P:613 distributed shared memory)
//  cluster : no barrier; single-pass ticket combine through L2
//
// All trees are ORDER-PRESERVING: the lower-index sibling is always the left
// operand (§8(c) reading #4), so non-commutative associative ops fold in
// ascending task order and sums are run-to-run deterministic.
#pragma once
#ifndef HPAR_TICKET_ACQREL
#define HPAR_TICKET_ACQREL 1
#endif
#include <cuda_runtime.h>
#include <stdint.h>
#include "plan.h"

namespace hpar {

// ---------------------------------------------------------------- ops ----
template <int OP, typename Acc>
struct OpT;

template <typename Acc>
struct OpT<OP_SUM, Acc> {
  __device__ __forceinline__ static Acc identity() { return Acc(0); }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) { return a + b; }
};
template <>
struct OpT<OP_MIN, double> {
  __device__ __forceinline__ static double identity() { return __longlong_as_double(0x7FF0000000000000ll); }
  __device__ __forceinline__ static double combine(double a, double b) { return b < a ? b : a; }
};
template <>
struct OpT<OP_MAX, double> {
  __device__ __forceinline__ static double identity() { return __longlong_as_double(0xFFF0000000000000ll); }
  __device__ __forceinline__ static double combine(double a, double b) { return b > a ? b : a; }
};
template <>
struct OpT<OP_MIN, float> {
  __device__ __forceinline__ static float identity() { return __int_as_float(0x7F800000); }
  __device__ __forceinline__ static float combine(float a, float b) { return b < a ? b : a; }
};
template <>
struct OpT<OP_MAX, float> {
  __device__ __forceinline__ static float identity() { return __int_as_float(0xFF800000); }
  __device__ __forceinline__ static float combine(float a, float b) { return b > a ? b : a; }
};
template <>
struct OpT<OP_MIN, long long> {
  __device__ __forceinline__ static long long identity() { return 0x7FFFFFFFFFFFFFFFll; }
  __device__ __forceinline__ static long long combine(long long a, long long b) { return b < a ? b : a; }
};
template <>
struct OpT<OP_MAX, long long> {
  __device__ __forceinline__ static long long identity() { return (long long)0x8000000000000000ull; }
  __device__ __forceinline__ static long long combine(long long a, long long b) { return b > a ? b : a; }
};

// Ordered user-defined operator: element x is the affine map
// y -> a*y + b (mod 2^64) with a = 2x+1, b = x*x; combine(L, R) applies L then
// R.  Associative, not commutative: only order-preserving trees are correct.
struct Aff {
  unsigned long long a, b;
};
template <>
struct OpT<OP_AFFINE, Aff> {
  __device__ __forceinline__ static Aff identity() { return Aff{1ull, 0ull}; }
  __device__ __forceinline__ static Aff combine(Aff l, Aff r) { return Aff{r.a * l.a, r.a * l.b + r.b}; }
};
// input element -> accumulator
template <int OP, typename Acc, typename In>
struct ElemT {
  __device__ __forceinline__ static Acc make(In x) { return (Acc)x; }
};
template <typename In>
struct ElemT<OP_AFFINE, Aff, In> {
  __device__ __forceinline__ static Aff make(In x) {
    const unsigned long long v = (unsigned long long)x;
    return Aff{2ull * v + 1ull, v * v};
  }
};

// shuffles that also move the 16-byte ordered accumulator
template <typename T>
__device__ __forceinline__ T shfl_down_t(unsigned mask, T v, int off, int width = 32) {
  return __shfl_down_sync(mask, v, off, width);
}
template <>
__device__ __forceinline__ Aff shfl_down_t<Aff>(unsigned mask, Aff v, int off, int width) {
  return Aff{__shfl_down_sync(mask, v.a, off, width), __shfl_down_sync(mask, v.b, off, width)};
}
// L2-coherent read of a value another CTA published (after a fence + ticket)
template <typename T>
__device__ __forceinline__ T ld_volatile(const T* p) {
  return *(const volatile T*)p;
}
template <>
__device__ __forceinline__ Aff ld_volatile<Aff>(const Aff* p) {
  const volatile unsigned long long* q = (const volatile unsigned long long*)p;
  return Aff{q[0], q[1]};
}

// --------------------------------------------------- lane level: shuffle ----
// Order-preserving tree over `count` consecutive groups of `stride` lanes:
// after the call the first lane of every block of stride*count lanes holds
// the ordered fold of its block's group values (groups held at lanes that
// are multiples of `stride`).  `count` and `stride` are powers of two.
template <int OP, typename Acc>
__device__ __forceinline__ Acc shfl_tree(Acc v, int stride, int count) {
  const int lane = threadIdx.x & 31;
  for (int off = stride; off < stride * count; off <<= 1) {
    Acc other = shfl_down_t(0xffffffffu, v, off);
    if ((lane & (2 * off - 1)) == 0) v = OpT<OP, Acc>::combine(v, other);
  }
  return v;
}

// Full-warp ordered fold (stride 1, 32 lanes): result in lane 0.
template <int OP, typename Acc>
__device__ __forceinline__ Acc warp_fold(Acc v) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Acc other = shfl_down_t(0xffffffffu, v, off);
    if ((threadIdx.x & (2 * off - 1)) == 0) v = OpT<OP, Acc>::combine(v, other);
  }
  return v;
}

// ------------------------------------------------- cluster / DSMEM PTX ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// Map a local shared::cta address to the same variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u64(uint32_t addr, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
// store an accumulator (8 or 16 bytes) to a shared::cluster address
template <typename Acc>
__device__ __forceinline__ void st_cluster_acc(uint32_t addr, const Acc& v) {
  static_assert(sizeof(Acc) % 8 == 0, "accumulators are whole 8-byte words");
  const unsigned long long* w = (const unsigned long long*)&v;
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Acc) / 8); ++i) st_cluster_u64(addr + 8 * i, w[i]);
}
__device__ __forceinline__ unsigned long long ld_cluster_u64(uint32_t addr) {
  unsigned long long v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}
// Split cluster barrier.  arrive.release / wait.acquire order the DSMEM
// stores before the barrier with the loads after it.  The .relaxed arrive
// carries no memory ordering (used where mbarrier transactions carry it).
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  cluster_arrive_release();
  cluster_wait_acquire();
}

// ------------------------------------------------------------ mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbarrier_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// Arrive on the mbarrier at shared::cluster address `remote` (another CTA).
// The .release form compiles to MEMBAR.ALL.GPU + arrive on sm_100a; use it
// only when prior global/shared WRITES must be visible to the waiter.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t remote) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// Relaxed remote arrive (no fence): for "slot free" signals that only order
// earlier READS, which are complete once their values were consumed.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t remote) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Acquire at cluster scope: for barriers completed by remote st.async / arrives.
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait_relaxed_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_relaxed_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_relaxed_cluster(bar, parity)) {
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
// st.async: 8-byte store into another CTA's shared memory that signals the
// destination CTA's mbarrier (complete_tx of 8 bytes) when it lands.
__device__ __forceinline__ void st_async_u64(uint32_t remote_addr, uint32_t remote_bar, unsigned long long v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];" ::"r"(remote_addr),
               "l"(v), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void st_async_u32(uint32_t remote_addr, uint32_t remote_bar, uint32_t v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(remote_addr),
               "r"(v), "r"(remote_bar)
               : "memory");
}

// --------------------------------------------------------------- TMA ----
// 1-D bulk copy global -> this CTA's shared memory, completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_addr(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------- streaming loads ----
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_stream_i4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------- grid level: single pass ----
// Cluster -> GPU combine (§8(a) A8).  Clusters have no barrier, so
// the combine is wait-free: each cluster publishes its partial, bumps a
// ticket, and the last arriver folds all partials in ascending cluster order.
// Returns true in the (whole) CTA that arrived last.  Must be called by all
// threads of the CTA (uniform); `my` is read from thread 0.
template <typename Acc>
__device__ __forceinline__ bool grid_arrive(Acc my, Acc* partials, unsigned int* ticket, int64_t c, int64_t C,
                                            int* s_flag) {
  if (threadIdx.x == 0) {
    partials[c] = my;
#if HPAR_TICKET_ACQREL
    // one acq_rel RMW: releases this partial, acquires the others' for the
    // last arriver (its CTA reads them after the bar.sync below)
    unsigned int t;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
    *s_flag = (t == (unsigned int)(C - 1)) ? 1 : 0;
#else
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    *s_flag = (t == (unsigned int)(C - 1)) ? 1 : 0;
    if (*s_flag) __threadfence();
#endif
  }
  __syncthreads();
  return *s_flag != 0;
}

// Ordered fold of partials[0..C) by all threads of one CTA: thread i folds a
// contiguous block, then an ordered tree over the threads.  Result returned
// in thread 0.  `s_warp` holds >= 32 accumulators of shared memory.
template <int OP, typename Acc>
__device__ Acc block_fold_ordered(const Acc* partials, int64_t C, Acc* s_warp) {
  const int nthr = blockDim.x;
  const int64_t per = (C + nthr - 1) / nthr;
  const int64_t b = (int64_t)threadIdx.x * per;
  const int64_t e = (b + per < C) ? b + per : C;
  Acc v = OpT<OP, Acc>::identity();
  for (int64_t i = b; i < e; ++i) v = OpT<OP, Acc>::combine(v, ld_volatile(partials + i));
  v = warp_fold<OP>(v);
  const int w = threadIdx.x >> 5, nw = nthr >> 5;
  if ((threadIdx.x & 31) == 0) s_warp[w] = v;
  __syncthreads();
  Acc r = OpT<OP, Acc>::identity();
  if (threadIdx.x == 0) {
    for (int k = 0; k < nw; ++k) r = OpT<OP, Acc>::combine(r, s_warp[k]);
  }
  __syncthreads();
  return r;
}

// ------------------------------------------------- verify fingerprints ----
__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xFF51AFD7ED558CCDull;
  z ^= z >> 33;
  z *= 0xC4CEB9FE1A85EC53ull;
  z ^= z >> 33;
  return z;
}
__device__ __forceinline__ uint64_t fp_mix(uint64_t i) { return fmix64(i * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull); }
__device__ __forceinline__ uint64_t fp_mix2(uint64_t i, uint64_t o) {
  return fmix64(fp_mix(i) ^ (o * 0xD6E8FEB86659FD93ull));
}

// --------------------------------------------------- partition (own) ----
// Closed forms of S:337 for the device: number of positions of a parent
// list of length n that child t of T owns, and the parent position of the
// child's j-th owned position.
__device__ __forceinline__ int64_t own_count(int sched, int64_t chunk, int64_t n, int64_t T, int64_t t) {
  if (sched == SCHED_STATIC) {
    const int64_t q = n / T, r = n % T;
    return q + (t < r ? 1 : 0);
  }
  if (sched == SCHED_NONE) return t < n ? 1 : 0;
  // static(c) / dynamic modelled as static(c)
  const int64_t nch = (n + chunk - 1) / chunk;
  if (t >= nch) return 0;
  const int64_t mine = (nch - 1 - t) / T + 1;  // chunks t, t+T, ... < nch
  int64_t cnt = mine * chunk;
  const int64_t last = nch - 1;
  if ((last % T) == t) cnt -= nch * chunk - n;  // last chunk may be short
  return cnt;
}
__device__ __forceinline__ int64_t own_map(int sched, int64_t chunk, int64_t n, int64_t T, int64_t t, int64_t j) {
  if (sched == SCHED_STATIC) {
    const int64_t q = n / T, r = n % T;
    return t * q + (t < r ? t : r) + j;
  }
  if (sched == SCHED_NONE) return t;
  return (j / chunk) * (chunk * T) + t * chunk + (j % chunk);
}

}  // namespace hpar
