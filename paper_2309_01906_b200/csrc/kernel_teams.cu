// kernel_teams.cu — the two-level "teams x threads" nest (config 1).
//
// Nest shape (SURVEY §8(c) reading #15; PAPER P:152 level(devices,teams,threads)):
//     GPU                static        loop 0 (rows; host: rank shard)
//     teams  = cluster..CTA  static    loop 0: a contiguous block of rows per CTA
//     threads = warp..lane   static(c) loop 1: chunks of c columns round-robin
//                                      over the W*32 threads of the CTA
// This is the paper's 2-level example (outer loop over the outer
// level, inner loop over the inner level, both started once: SPMD mode
// P:238-240).  The generic interpreter computes the same ownership by
// composing own() per element; here the closed forms are inlined: thread j
// owns columns (i*NT + j)*c + [0, c) of every row of its team.  Combine:
// lane -> warp -> CTA -> cluster -> GPU (fused_common.cuh), node via NCCL.
#include <cuda_runtime.h>
#include <stdint.h>
#include "fused_common.cuh"

namespace hpar {
namespace {

template <typename In, typename Acc, int OP, bool VERIFY>
__global__ void __launch_bounds__(1024) teams_kernel(const __grid_constant__ NestArgs a, int W, int chunk) {
  __shared__ ClimbSmem<Acc> csm;
  const int64_t T = (int64_t)gridDim.x;           // teams on this GPU
  const int64_t t = blockIdx.x;
  const int64_t q = a.n0 / T, r = a.n0 % T;       // static block of rows over teams
  const int64_t row0 = t * q + (t < r ? t : r);
  const int64_t nrow = q + (t < r ? 1 : 0);
  const int NT = W * 32;
  const int j = threadIdx.x;
  const In* x = (const In*)a.in;
  const int64_t leaf = (int64_t)a.rank * a.threads_per_gpu + t * NT + j;
  Acc acc = OpT<OP, Acc>::identity();
  // one 16-byte chunk per thread and row (the C1 shape, n1 == 4 NT): a team
  // with several rows issues up to 8 rows' loads before it combines them
  const bool one_vec = !VERIFY && sizeof(In) == 4 && chunk == 4 && a.n1 == (int64_t)NT * 4 &&
                       (((uintptr_t)x) & 15) == 0 && (a.ld & 3) == 0;
  if (one_vec) {
    constexpr int G = 8;
    for (int64_t row = row0; row < row0 + nrow; row += G) {
      int4 v[G];
#pragma unroll
      for (int k = 0; k < G; ++k)
        v[k] = (row + k < row0 + nrow) ? __ldg((const int4*)(x + (row + k) * a.ld) + j) : make_int4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < G; ++k) {
        if (row + k < row0 + nrow) {
          const In* e = (const In*)&v[k];
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[0]));
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[1]));
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[2]));
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[3]));
        }
      }
    }
  }
  for (int64_t row = one_vec ? row0 + nrow : row0; row < row0 + nrow; ++row) {
    const In* xr = x + row * a.ld;
    for (int64_t base = (int64_t)j * chunk; base < a.n1; base += (int64_t)NT * chunk) {
      const int64_t end = (base + chunk < a.n1) ? base + chunk : a.n1;
      if (chunk == 4 && sizeof(In) == 4 && end - base == 4 && ((((uintptr_t)(xr + base)) & 15) == 0)) {
        if constexpr (sizeof(In) == 4) {
          const int4 v = *(const int4*)(xr + base);
          const In* e = (const In*)&v;
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[0]));
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[1]));
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[2]));
          acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(e[3]));
        }
      } else {
        for (int64_t col = base; col < end; ++col) acc = OpT<OP, Acc>::combine(acc, ElemT<OP, Acc, In>::make(xr[col]));
      }
      if constexpr (VERIFY) {
        for (int64_t col = base; col < end; ++col) {
          const int64_t it = row * a.n1 + col;
          if (a.verify & V_COVERAGE) { a.owner[it] = leaf; atomicAdd(&a.count[it], 1u); }
          if (a.verify & V_FINGERPRINT) {
            const uint64_t g = a.global_begin + (uint64_t)it;
            atomicAdd(&a.fp[0], (unsigned long long)fp_mix(g));
            atomicAdd(&a.fp[1], (unsigned long long)fp_mix2(g, (uint64_t)leaf));
            atomicAdd(&a.fp[2], 1ull);
          }
        }
      }
    }
  }
  fused_total_climb<OP, Acc>(a, acc, W, csm);
}

template <typename In, typename Acc, int OP>
cudaError_t launch_t(const NestArgs& a, int W, int chunk, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.C * a.K));
  cfg.blockDim = dim3((unsigned)(W * 32));
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.verify) return cudaLaunchKernelEx(&cfg, teams_kernel<In, Acc, OP, true>, a, W, chunk);
  return cudaLaunchKernelEx(&cfg, teams_kernel<In, Acc, OP, false>, a, W, chunk);
}

}  // namespace

bool teams_matches(const NestArgs& a, const char** why) {
  if (a.nloops != 2 || a.keyed || a.offsets) { *why = "not a dense 2-loop total"; return false; }
  if (a.op == OP_HIST) { *why = "sum/min/max/affine only"; return false; }
  if (a.op == OP_AFFINE && a.in_dtype != DT_I64) { *why = "affine: int64 input"; return false; }
  if (a.lane_w != 1) { *why = "lane partition"; return false; }
  LevelView v = device_levels(a);
  if (v.n != 2) { *why = "needs teams and threads levels"; return false; }
  const DevLevel *tm = v.l[0], *th = v.l[1];
  if (tm->sfirst != S_CLUSTER || tm->slast != S_CTA || tm->loop != 0 || tm->sched != SCHED_STATIC) {
    *why = "teams (cluster..CTA) must be static over loop 0";
    return false;
  }
  if (th->sfirst != S_WARP || th->slast != S_LANE_IN || th->loop != 1 ||
      !(th->sched == SCHED_STATIC_CHUNK && th->chunk >= 1)) {
    *why = "threads (warp..lane) must be static(c) over loop 1";
    return false;
  }
  if (a.radix[S_WARP] > 31) { *why = "W"; return false; }
  return true;
}

cudaError_t launch_teams(const NestArgs& a, int W, cudaStream_t s, const char** name) {
  *name = "teams_threads";
  const int chunk = (int)device_levels(a).l[1]->chunk;
  switch (a.in_dtype) {
    case DT_I32:
      if (a.op == OP_SUM) return launch_t<int32_t, long long, OP_SUM>(a, W, chunk, s);
      if (a.op == OP_MIN) return launch_t<int32_t, long long, OP_MIN>(a, W, chunk, s);
      return launch_t<int32_t, long long, OP_MAX>(a, W, chunk, s);
    case DT_F32:
      if (a.op == OP_SUM) return launch_t<float, double, OP_SUM>(a, W, chunk, s);
      if (a.op == OP_MIN) return launch_t<float, double, OP_MIN>(a, W, chunk, s);
      return launch_t<float, double, OP_MAX>(a, W, chunk, s);
    case DT_I64:
      if (a.op == OP_SUM) return launch_t<long long, long long, OP_SUM>(a, W, chunk, s);
      if (a.op == OP_AFFINE) return launch_t<long long, Aff, OP_AFFINE>(a, W, chunk, s);
      if (a.op == OP_MIN) return launch_t<long long, long long, OP_MIN>(a, W, chunk, s);
      return launch_t<long long, long long, OP_MAX>(a, W, chunk, s);
    default:
      if (a.op == OP_SUM) return launch_t<double, double, OP_SUM>(a, W, chunk, s);
      if (a.op == OP_MIN) return launch_t<double, double, OP_MIN>(a, W, chunk, s);
      return launch_t<double, double, OP_MAX>(a, W, chunk, s);
  }
}

}  // namespace hpar
