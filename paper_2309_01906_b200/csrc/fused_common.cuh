// fused_common.cuh — helpers shared by the fused (nest-shape specialised)
// kernels: level-structure matching and the end-of-kernel combine climb.
#pragma once
#ifndef HPAR_CLIMB_RELAXED_EXIT
#define HPAR_CLIMB_RELAXED_EXIT 1
#endif
#include "level_primitives.cuh"
#include "node_fused.cuh"
#include "plan.h"

namespace hpar {

// The device-visible levels of a nest (the host-applied GPU level dropped).
struct LevelView {
  int n;
  const DevLevel* l[kMaxLev];
  int idx[kMaxLev];
};
inline LevelView device_levels(const NestArgs& a) {
  LevelView v;
  v.n = 0;
  for (int i = 0; i < a.nlev; ++i) {
    if (a.lv[i].host_applied) continue;
    v.l[v.n] = &a.lv[i];
    v.idx[v.n] = i;
    ++v.n;
  }
  return v;
}
// level bound to exactly one hardware level (lane: both lane slots)
inline bool is_level(const DevLevel* L, int hw_slot) {
  if (hw_slot == S_LANE) return L->sfirst == S_LANE && L->slast == S_LANE_IN;
  return L->sfirst == hw_slot && L->slast == hw_slot;
}

// The flat shape in any of its equivalent spellings: the upper part is
// cluster static(K*tile) + CTA static(tile), or one collapsed cluster..CTA
// level static(tile) (the same tile -> CTA map: tile m*(C*K) + c*K + k); the
// lower part is warp static(32V) + lane static(V), or one collapsed
// warp..lane level static(V) (the same chunk -> thread map).  Sets tile, V
// (the flat and histogram kernels check V).
inline bool flat_nest_shape(const NestArgs& a, const char** why, int64_t* tile_out, int64_t* v_out) {
  LevelView v = device_levels(a);
  int i = 0;
  int64_t tile = -1, lv = -1;
  auto sc = [](const DevLevel* L) { return L->sched == SCHED_STATIC_CHUNK; };
  if (i < v.n && v.l[i]->sfirst == S_CLUSTER && v.l[i]->slast == S_CTA && sc(v.l[i])) {
    tile = v.l[i]->chunk;
    i += 1;
  } else if (i + 1 < v.n && is_level(v.l[i], S_CLUSTER) && is_level(v.l[i + 1], S_CTA) && sc(v.l[i]) &&
             sc(v.l[i + 1])) {
    tile = v.l[i + 1]->chunk;
    if (v.l[i]->chunk != a.K * tile) { *why = "cluster must be static(K*tile)"; return false; }
    i += 2;
  } else {
    *why = "upper levels not cluster static(K*tile) + CTA static(tile) (or cluster..CTA static(tile))";
    return false;
  }
  if (i < v.n && v.l[i]->sfirst == S_WARP && v.l[i]->slast == S_LANE_IN && sc(v.l[i])) {
    lv = v.l[i]->chunk;
    i += 1;
  } else if (i + 1 < v.n && is_level(v.l[i], S_WARP) && is_level(v.l[i + 1], S_LANE) && sc(v.l[i]) &&
             sc(v.l[i + 1])) {
    lv = v.l[i + 1]->chunk;
    if (v.l[i]->chunk != 32 * lv) { *why = "warp must be static(32*lane chunk)"; return false; }
    i += 2;
  } else {
    *why = "lower levels not warp static(32V) + lane static(V) (or warp..lane static(V))";
    return false;
  }
  if (i != v.n) { *why = "extra levels"; return false; }
  *tile_out = tile;
  *v_out = lv;
  return true;
}

// Write the partial of the task at `slot` to every nest level whose last
// slot is `slot` (verify mode).  `index` = task id below the GPU.
// elements m4 .. m4+3 of the 8-element concatenation (a, b), m4 in 1..3
// (warp-uniform): a lane's 4-element vector when the copied granules start
// m4 elements before the data (misaligned inputs, ragged rows)
template <typename V>
__device__ __forceinline__ V shift4(const V& a, const V& b, uint32_t m4) {
  V r;
  if (m4 == 1) { r.x = a.y; r.y = a.z; r.z = a.w; r.w = b.x; }
  else if (m4 == 2) { r.x = a.z; r.y = a.w; r.z = b.x; r.w = b.y; }
  else { r.x = a.w; r.y = b.x; r.z = b.y; r.w = b.z; }
  return r;
}

template <typename Acc>
__device__ __forceinline__ void export_slot(const NestArgs& a, int slot, int64_t index, Acc v) {
  if (!(a.verify & V_PARTIALS)) return;
  for (int l = 0; l < a.nlev; ++l)
    if (a.lv[l].slast == slot && a.partials[l]) ((Acc*)a.partials[l])[index] = v;
}

// Shared memory for the climb.
template <typename Acc>
struct ClimbSmem {
  Acc warp[33];
  Acc cta[16];
  int flag;
};

// End-of-kernel TOTAL combine for the fused kernels (no lane partition):
// lane -> warp (SHFL) -> CTA (smem, named barrier over the W consumer warps)
// -> cluster (DSMEM + barrier.cluster) -> GPU (single-pass ticket).
// Called by ALL threads of the CTA (consumers and any producer warp, which
// passes the identity and is not part of the named barrier).  Writes the GPU
// total to a.out and resets the ticket.  `W` = consumer warps.
template <int OP, typename Acc>
__device__ void fused_total_climb(const NestArgs& a, Acc v, int W, ClimbSmem<Acc>& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool consumer = warp < W;
  const uint32_t rank = cluster_ctarank();
  const int64_t cl = blockIdx.x / a.K;
  if (consumer) {
    export_slot<Acc>(a, S_LANE_IN, (int64_t)blockIdx.x * W * 32 + threadIdx.x, v);
    v = warp_fold<OP>(v);
    if (lane == 0) {
      sh.warp[warp] = v;
      export_slot<Acc>(a, S_WARP, (int64_t)blockIdx.x * W + warp, v);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(W * 32) : "memory");
    if (threadIdx.x == 0) {
      Acc r = OpT<OP, Acc>::identity();
      for (int w = 0; w < W; ++w) r = OpT<OP, Acc>::combine(r, sh.warp[w]);
      v = r;
      export_slot<Acc>(a, S_CTA, (int64_t)blockIdx.x, v);
      st_cluster_acc(mapa(smem_addr(&sh.cta[rank]), 0), v);
    }
  }
  cluster_sync_all();
  Acc cluster_v = OpT<OP, Acc>::identity();
  if (rank == 0 && threadIdx.x == 0) {
    for (int k = 0; k < a.K; ++k) cluster_v = OpT<OP, Acc>::combine(cluster_v, sh.cta[k]);
    export_slot<Acc>(a, S_CLUSTER, cl, cluster_v);
  }
  if (rank == 0) {
    Acc* parts = (Acc*)a.cluster_partials;
    if (grid_arrive<Acc>(cluster_v, parts, a.grid_ticket, cl, a.C, &sh.flag)) {
      Acc tot = block_fold_ordered<OP, Acc>(parts, a.C, sh.warp);
      if (threadIdx.x == 0) export_slot<Acc>(a, S_GPU, 0, tot);
      if (a.node_dc) node_fold_scalar<OP, Acc>(a, tot);  // the node level in-kernel (f1)
      if (threadIdx.x == 0) {
        *(Acc*)a.out = tot;
        *a.grid_ticket = 0u;
      }
    }
  }
#if HPAR_CLIMB_RELAXED_EXIT
  // no data crosses this barrier (the siblings' DSMEM stores were ordered by
  // the first one): execution-only, no release fence
  cluster_arrive_relaxed();
  asm volatile("barrier.cluster.wait;" ::: "memory");
#else
  cluster_sync_all();  // keep the leader's shared memory alive for its siblings
#endif
}

}  // namespace hpar
