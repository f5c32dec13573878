// kernel_generic.cu — the generic nest interpreter (sm_100a).
//
// Executes ANY nest that hpar_nest_create accepts: per-level static /
// static(c) / none / dynamic(c) partitioning, collapsed
// and partitioned levels, one or two loops bound to
// arbitrary levels, one total or one result per outer iteration,
// plus the verify outputs (coverage, per-level partials, fingerprints).
//
// One launch = the whole nest (SPMD mode): grid = C clusters of K
// CTAs of W warps.  Every thread is a leaf task; its ids at every nest level
// are the mixed-radix digits of (rank, cluster, CTA-in-cluster, warp, lane).
// Iterations are enumerated by composing the closed forms of own() level by
// level (level_primitives.cuh), and combined bottom-up with the level
// primitives: SHFL (lane), smem + bar.sync (warp), DSMEM + barrier.cluster
// (CTA), single-pass ticket (cluster).  The fused streaming kernels in
// kernel_flat.cu / kernel_rowwise.cu are this kernel specialised to one nest
// shape; this one trades speed for generality.
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include "level_primitives.cuh"
#include "node_fused.cuh"
#include "plan.h"

namespace hpar {
namespace {

// A refinement chain: the levels bound to one loop, in nest order.
struct Chain {
  int m;
  int sched[kMaxLev];
  int64_t chunk[kMaxLev], T[kMaxLev], t[kMaxLev];
};

__device__ __forceinline__ void chain_lens(const Chain& ch, int lo, int hi, int64_t n, int64_t* lens) {
  lens[lo] = n;
  for (int k = lo; k < hi; ++k) lens[k + 1] = own_count(ch.sched[k], ch.chunk[k], lens[k], ch.T[k], ch.t[k]);
}
// map position j of the list after level hi-1 up to the list before level lo
__device__ __forceinline__ int64_t chain_map(const Chain& ch, int lo, int hi, const int64_t* lens, int64_t j) {
  for (int k = hi - 1; k >= lo; --k) j = own_map(ch.sched[k], ch.chunk[k], lens[k], ch.T[k], ch.t[k], j);
  return j;
}

// chain_map plus the run length: positions j .. j+run-1 of the list after
// level hi-1 map to consecutive positions of the list before level lo (every
// level keeps them inside one of its chunks / its block), so an iteration
// loop maps once per run and then steps by one — the same visit order.
__device__ __forceinline__ int64_t chain_map_run(const Chain& ch, int lo, int hi, const int64_t* lens, int64_t j,
                                                 int64_t* run) {
  int64_t r = lens[hi] - j;
  for (int k = hi - 1; k >= lo; --k) {
    const int s = ch.sched[k];
    if (s == SCHED_STATIC) {
      const int64_t left = lens[k + 1] - j;
      r = left < r ? left : r;
    } else if (s == SCHED_NONE) {
      r = 1;
    } else {
      const int64_t c = ch.chunk[k];
      const int64_t left = c - j % c;
      r = left < r ? left : r;
    }
    j = own_map(s, ch.chunk[k], lens[k], ch.T[k], ch.t[k], j);
  }
  *run = r > 0 ? r : 1;
  return j;
}

template <typename Acc>
struct Shared {
  Acc warp[2][32];
  Acc cta[2][16];
  unsigned long long claim[2];
  int flag;
};

template <typename In, typename Acc, int OP>
struct Generic {
  const NestArgs& a;
  Shared<Acc>& sh;
  int64_t dig[S_NSLOTS];
  int64_t leaf;
  int parity;      // double-buffer index of the climb slots (per row)
  int claim_par;   // double-buffer index of the claim broadcast
  uint32_t cta_rank;
  unsigned long long fp_once, fp_owner, fp_n;

  __device__ Generic(const NestArgs& args, Shared<Acc>& s) : a(args), sh(s) {
    const int lane = threadIdx.x & 31;
    cta_rank = cluster_ctarank();
    dig[S_GPU] = a.rank;
    dig[S_CLUSTER] = blockIdx.x / a.K;
    dig[S_CTA] = cta_rank;
    dig[S_WARP] = threadIdx.x >> 5;
    dig[S_LANE] = lane / a.lane_w;
    dig[S_LANE_IN] = lane % a.lane_w;
    leaf = (int64_t)a.rank * a.threads_per_gpu + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    parity = 0;
    claim_par = 0;
    fp_once = fp_owner = fp_n = 0;
  }

  __device__ int64_t task_local_id(int lv) const {
    int64_t id = 0;
    for (int s = a.lv[lv].sfirst; s <= a.lv[lv].slast; ++s) id = id * a.radix[s] + dig[s];
    return id;
  }
  // id over slots [lo, hi] (mixed radix)
  __device__ int64_t ids_over(int lo, int hi) const {
    int64_t id = 0;
    for (int s = lo; s <= hi; ++s) id = id * a.radix[s] + dig[s];
    return id;
  }
  __device__ int64_t radix_over(int lo, int hi) const {
    int64_t r = 1;
    for (int s = lo; s <= hi; ++s) r *= a.radix[s];
    return r;
  }
  __device__ bool is_rep_below(int slot) const {  // all digits after `slot` are zero
    for (int s = slot + 1; s < S_NSLOTS; ++s)
      if (dig[s] != 0) return false;
    return true;
  }

  __device__ void build_chain(int loop, Chain& ch, int* dyn_pos) const {
    ch.m = 0;
    *dyn_pos = -1;
    for (int l = 0; l < a.nlev; ++l) {
      const DevLevel& L = a.lv[l];
      if (L.loop != loop || L.host_applied) continue;
      if (l == a.dyn_level) *dyn_pos = ch.m;
      ch.sched[ch.m] = L.sched;
      ch.chunk[ch.m] = L.chunk > 0 ? L.chunk : 1;
      ch.T[ch.m] = L.T;
      ch.t[ch.m] = task_local_id(l);
      ++ch.m;
    }
  }

  // ---- dynamic claim, broadcast within the dynamic level's task --------
  __device__ unsigned long long claim(unsigned long long* ticket, int scope_slot) {
    unsigned long long v = 0;
    if (scope_slot == S_WARP) {
      if ((threadIdx.x & 31) == 0) v = atomicAdd(ticket, 1ull);
      v = __shfl_sync(0xffffffffu, v, 0);
    } else if (scope_slot == S_CTA) {
      if (threadIdx.x == 0) sh.claim[claim_par] = atomicAdd(ticket, 1ull);
      __syncthreads();
      v = sh.claim[claim_par];
      claim_par ^= 1;
    } else {  // S_CLUSTER
      if (cta_rank == 0 && threadIdx.x == 0) sh.claim[claim_par] = atomicAdd(ticket, 1ull);
      cluster_sync_all();
      v = (cta_rank == 0) ? sh.claim[claim_par] : ld_cluster_u64(mapa(smem_addr(&sh.claim[claim_par]), 0));
      claim_par ^= 1;
    }
    return v;
  }

  __device__ __forceinline__ Acc load(int64_t i, int64_t j) const {
    const In* x = (const In*)a.in;
    if (a.nloops == 1) return ElemT<OP, Acc, In>::make(x[i]);
    if (a.offsets) return ElemT<OP, Acc, In>::make(x[a.offsets[i] + j]);
    return ElemT<OP, Acc, In>::make(x[i * a.ld + j]);
  }
  __device__ __forceinline__ int64_t iter_index(int64_t i, int64_t j) const {
    if (a.nloops == 1) return i;
    if (a.offsets) return a.offsets[i] + j;
    return i * a.n1 + j;
  }
  __device__ __forceinline__ void record(int64_t it) {
    if (a.verify & V_COVERAGE) {
      a.owner[it] = leaf;
      atomicAdd(&a.count[it], 1u);
    }
    if (a.verify & V_FINGERPRINT) {
      const uint64_t g = a.global_begin + (uint64_t)it;
      fp_once += fp_mix(g);
      fp_owner += fp_mix2(g, (uint64_t)leaf);
      fp_n += 1;
    }
  }
  __device__ __forceinline__ int64_t row_len(int64_t i) const {
    if (a.nloops == 1) return 1;
    if (a.offsets) return a.offsets[i + 1] - a.offsets[i];
    return a.n1;
  }

  // inner loop (loop 1) of row i: purely per thread (no dynamic levels)
  __device__ Acc inner(const Chain& c1, int64_t i, Acc acc) {
    int64_t lens[kMaxLev + 1];
    chain_lens(c1, 0, c1.m, row_len(i), lens);
    const int64_t cnt = lens[c1.m];
    for (int64_t q = 0; q < cnt;) {
      int64_t run;
      const int64_t j0 = chain_map_run(c1, 0, c1.m, lens, q, &run);
      for (int64_t u = 0; u < run; ++u) {
        acc = OpT<OP, Acc>::combine(acc, load(i, j0 + u));
        record(iter_index(i, j0 + u));
      }
      q += run;
    }
    return acc;
  }

  __device__ void export_partial(int lv, int64_t index, Acc v) const {
    if ((a.verify & V_PARTIALS) && a.partials[lv]) ((Acc*)a.partials[lv])[index] = v;
  }

  // Combine the per-thread values up through slots (from, down to stop+1]:
  // after the call the representative of the task at slot `stop` holds the
  // ordered fold.  keyed_row >= 0: keyed-mode exports for that row.
  __device__ Acc climb(Acc v, int stop, int64_t keyed_row) {
    const int lane = threadIdx.x & 31;
    auto exports = [&](int slot, Acc val) {
      if (!(a.verify & V_PARTIALS)) return;
      if (!is_rep_below(slot)) return;
      for (int l = 0; l < a.nlev; ++l) {
        if (a.lv[l].slast != slot || !a.partials[l]) continue;
        if (keyed_row >= 0) {
          if (l < a.first_inner) continue;
          const int64_t per = radix_over(a.owner_slot + 1, slot);
          export_partial(l, keyed_row * per + ids_over(a.owner_slot + 1, slot), val);
        } else {
          export_partial(l, slot >= S_CLUSTER ? ids_over(S_CLUSTER, slot) : 0, val);
        }
      }
    };
    exports(S_LANE_IN, v);
    // step LANE_IN -> LANE (partition groups of w lanes)
    if (stop < S_LANE_IN && a.lane_w > 1) {
      const unsigned grp = (a.lane_w == 32) ? 0xffffffffu
                                             : (((1u << a.lane_w) - 1u) << ((lane / a.lane_w) * a.lane_w));
      for (int off = 1; off < a.lane_w; off <<= 1) {
        Acc o = shfl_down_t(grp, v, off, a.lane_w);
        if (((lane % a.lane_w) & (2 * off - 1)) == 0) v = OpT<OP, Acc>::combine(v, o);
      }
    }
    if (stop < S_LANE_IN) exports(S_LANE, v);
    // step LANE -> WARP
    if (stop < S_LANE) {
      v = shfl_tree<OP>(v, a.lane_w, 32 / a.lane_w);
      exports(S_WARP, v);
    }
    // step WARP -> CTA (smem slots + bar.sync: P:308-323 fallback one level up)
    if (stop < S_WARP) {
      if (lane == 0) sh.warp[parity][threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x == 0) {
        Acc r = OpT<OP, Acc>::identity();
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = OpT<OP, Acc>::combine(r, sh.warp[parity][w]);
        v = r;
      }
      exports(S_CTA, v);
    }
    // step CTA -> CLUSTER (DSMEM slots in the leader CTA + cluster barrier)
    if (stop < S_CTA) {
      if (threadIdx.x == 0) st_cluster_acc(mapa(smem_addr(&sh.cta[parity][cta_rank]), 0), v);
      cluster_sync_all();
      if (cta_rank == 0 && threadIdx.x == 0) {
        Acc r = OpT<OP, Acc>::identity();
        for (int k = 0; k < a.K; ++k) r = OpT<OP, Acc>::combine(r, sh.cta[parity][k]);
        v = r;
      }
      exports(S_CLUSTER, v);
    }
    parity ^= 1;
    return v;
  }

  __device__ void write_row(int64_t i, Acc v) const {
    if constexpr (std::is_arithmetic<Acc>::value) {
      if (a.out_dtype == DT_F32) {
        ((float*)a.out)[i] = (float)v;
        return;
      }
    }
    ((Acc*)a.out)[i] = v;
  }

  __device__ void run() {
    Chain c0, c1;
    int dyn0 = -1, dyn1 = -1;
    build_chain(0, c0, &dyn0);
    build_chain(1, c1, &dyn1);
    int64_t lens[kMaxLev + 1];
    const bool keyed = a.keyed != 0;
    Acc acc = OpT<OP, Acc>::identity();

    auto visit_row = [&](int64_t i) {
      if (!keyed) {
        if (a.nloops == 1) {
          acc = OpT<OP, Acc>::combine(acc, load(i, 0));
          record(i);
        } else {
          acc = inner(c1, i, acc);
        }
      } else {
        Acc r = inner(c1, i, OpT<OP, Acc>::identity());
        r = climb(r, a.owner_slot, i);
        if (is_rep_below(a.owner_slot)) write_row(i, r);
      }
    };

    if (dyn0 < 0) {
      chain_lens(c0, 0, c0.m, a.n0, lens);
      const int64_t cnt = lens[c0.m];
      for (int64_t q = 0; q < cnt;) {
        int64_t run;
        const int64_t i0 = chain_map_run(c0, 0, c0.m, lens, q, &run);
        for (int64_t u = 0; u < run; ++u) visit_row(i0 + u);
        q += run;
      }
    } else {
      // levels above the dynamic one are static: their list is fixed
      chain_lens(c0, 0, dyn0, a.n0, lens);
      const int64_t n_up = lens[dyn0];
      const int64_t c = c0.chunk[dyn0];
      const int64_t nch = (n_up + c - 1) / c;
      const DevLevel& D = a.lv[a.dyn_level];
      const int64_t slot = ids_over(S_CLUSTER, D.sfirst - 1);  // parent task (below the GPU)
      unsigned long long* ticket = a.dyn_tickets + slot;
      int64_t lensl[kMaxLev + 1];
      for (;;) {
        const int64_t m = (int64_t)claim(ticket, D.slast);
        if (m >= nch) break;
        const int64_t len_m = (n_up - m * c < c) ? (n_up - m * c) : c;
        chain_lens(c0, dyn0 + 1, c0.m, len_m, lensl);
        const int64_t cnt = lensl[c0.m];
        for (int64_t q = 0; q < cnt;) {
          int64_t run1, run2;
          const int64_t p = chain_map_run(c0, dyn0 + 1, c0.m, lensl, q, &run1) + m * c;
          const int64_t i0 = chain_map_run(c0, 0, dyn0, lens, p, &run2);
          const int64_t run = run1 < run2 ? run1 : run2;
          for (int64_t u = 0; u < run; ++u) visit_row(i0 + u);
          q += run;
        }
      }
    }

    if (a.verify & V_FINGERPRINT) {
      atomicAdd(&a.fp[0], fp_once);
      atomicAdd(&a.fp[1], fp_owner);
      atomicAdd(&a.fp[2], fp_n);
    }

    if (!keyed) acc = climb(acc, S_GPU, -1);
    // grid level: single-pass ticket (cluster -> GPU), also resets the tickets.
    // The leader arrives for its whole cluster, so every CTA of the cluster
    // must be done (no more claims) first: in keyed mode no climb has synced
    // the cluster yet.
    if (keyed) cluster_sync_all();
    __syncthreads();
    const bool leader_cta = (cta_rank == 0);
    if (leader_cta) {
      const int64_t cl = blockIdx.x / a.K;
      Acc* parts = (Acc*)a.cluster_partials;
      if (grid_arrive<Acc>(acc, parts, a.grid_ticket, cl, a.C, &sh.flag)) {
        Acc tot = block_fold_ordered<OP, Acc>(parts, a.C, &sh.warp[0][0]);
        if (threadIdx.x == 0 && !keyed && (a.verify & V_PARTIALS)) {
          for (int l = 0; l < a.nlev; ++l)
            if (a.lv[l].slast == S_GPU && a.partials[l]) ((Acc*)a.partials[l])[0] = tot;
        }
        if (!keyed && a.node_dc) node_fold_scalar<OP, Acc>(a, tot);  // the node level in-kernel (f1)
        if (threadIdx.x == 0) {
          if (!keyed) *(Acc*)a.out = tot;
          *a.grid_ticket = 0u;
        }
        for (int64_t s = threadIdx.x; s < a.dyn_slots; s += blockDim.x) a.dyn_tickets[s] = 0ull;
      }
    }
    // no CTA may leave while a sibling can still read its shared memory
    cluster_sync_all();
  }
};

template <typename In, typename Acc, int OP>
__global__ void __launch_bounds__(1024) generic_nest_kernel(const __grid_constant__ NestArgs args) {
  __shared__ Shared<Acc> sh;
  Generic<In, Acc, OP> g(args, sh);
  g.run();
}

}  // namespace

// ------------------------------------------------------------ launcher ----
template <typename In, typename Acc, int OP>
static cudaError_t launch_t(const NestArgs& a, int threads, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.C * a.K));
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, generic_nest_kernel<In, Acc, OP>, a);
}

cudaError_t launch_generic(const NestArgs& a, int threads, cudaStream_t s) {
  const int dt = a.in_dtype, op = a.op;
#define HPAR_G(IN, ACC)                                                   \
  if (op == OP_SUM) return launch_t<IN, ACC, OP_SUM>(a, threads, s);      \
  if (op == OP_MIN) return launch_t<IN, ACC, OP_MIN>(a, threads, s);      \
  if (op == OP_MAX) return launch_t<IN, ACC, OP_MAX>(a, threads, s);
  if (dt == DT_I32) { HPAR_G(int32_t, long long) }
  if (dt == DT_I64) { HPAR_G(long long, long long) }
  if (dt == DT_F32) { HPAR_G(float, double) }
  if (dt == DT_F64) { HPAR_G(double, double) }
#undef HPAR_G
  if (op == OP_AFFINE && dt == DT_I64) return launch_t<long long, Aff, OP_AFFINE>(a, threads, s);
  return cudaErrorInvalidValue;
}

// node level of an ordered op: fold the G per-rank results (gathered by
// ncclAllGather in rank order) in ascending rank order
__global__ void affine_rank_fold_kernel(const Aff* in, int G, Aff* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    Aff v = OpT<OP_AFFINE, Aff>::identity();
    for (int g = 0; g < G; ++g) v = OpT<OP_AFFINE, Aff>::combine(v, in[g]);
    *out = v;
  }
}
cudaError_t launch_affine_rank_fold(const void* gathered, int G, void* out, cudaStream_t s) {
  affine_rank_fold_kernel<<<1, 32, 0, s>>>((const Aff*)gathered, G, (Aff*)out);
  return cudaGetLastError();
}

}  // namespace hpar
