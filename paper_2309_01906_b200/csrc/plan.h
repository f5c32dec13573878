// plan.h — resolved-nest structures shared by the host runtime and the
// kernels of libhpar.so (internal; not part of the C ABI).
#pragma once
#include <stdint.h>

namespace hpar {

// Digit slots of a leaf task's mixed-radix id, outermost first.  The lane
// level is always represented by two slots (outer slice, inner slice of the
// lanes(w) partition); without a partition the inner slot has
// radix 1 and the outer slot radix 32.
enum Slot { S_GPU = 0, S_CLUSTER = 1, S_CTA = 2, S_WARP = 3, S_LANE = 4, S_LANE_IN = 5, S_NSLOTS = 6 };

constexpr int kMaxLev = 8;

enum Sched { SCHED_STATIC = 0, SCHED_STATIC_CHUNK = 1, SCHED_DYNAMIC = 2, SCHED_NONE = 3 };
enum Op { OP_SUM = 0, OP_MIN = 1, OP_MAX = 2, OP_HIST = 3, OP_AFFINE = 4 };
enum DType { DT_I32 = 0, DT_I64 = 1, DT_F32 = 2, DT_F64 = 3, DT_U8 = 4, DT_U64 = 5 };
enum Verify { V_COVERAGE = 1, V_PARTIALS = 2, V_FINGERPRINT = 4 };

struct DevLevel {
  int32_t sched;
  int32_t loop;
  int64_t chunk;
  int64_t T;            // tasks per parent (product of the slot radices)
  int32_t sfirst;       // first digit slot
  int32_t slast;        // last digit slot
  int32_t host_applied; // the GPU level: refinement applied by sharding on the host
  int32_t pad;
};

// Everything a kernel needs about the nest and the call.
struct NestArgs {
  int32_t nlev;
  int32_t rank;
  int64_t radix[S_NSLOTS];
  int32_t lane_w;           // lanes per inner slice (1 = no partition)
  int32_t K;                // CTAs per cluster
  int64_t C;                // clusters in the launch
  int64_t threads_per_gpu;  // C*K*W*32
  DevLevel lv[kMaxLev];

  // the call
  int32_t op, in_dtype, nloops, keyed, out_dtype, verify;
  const void* in;
  int64_t n0;               // local extent of loop 0 (this rank's shard)
  int64_t n1, ld;
  const int64_t* offsets;
  void* out;
  void* partials[kMaxLev];
  int64_t* owner;
  uint32_t* count;
  unsigned long long* fp;
  uint64_t global_begin;

  // keyed mode: loop-0 levels are [0, first_inner); the row owner's last slot
  int32_t first_inner;
  int32_t owner_slot;

  // dynamic schedules (generic kernel: at most one level, on loop 0)
  int32_t dyn_level;        // nest level index or -1
  int32_t in_shift;         // segmented kernel: `in` moved back this many elements to a 16-byte
                            // boundary; offsets are read + in_shift (0 otherwise)
  unsigned long long* dyn_tickets;
  int64_t dyn_slots;

  // workspace (self-resetting)
  unsigned int* grid_ticket;
  void* cluster_partials;   // C accumulators (or C x 256 bins)
  int32_t* error_flag;

  // fused node level (NEXT f1; node_fused.cuh): the CTA that produces this
  // GPU's total stores it in every rank's symmetric slot [parity][rank],
  // meets the other GPUs at an NCCL LSA barrier and folds the slots in rank
  // order.  node_dc == NULL: the host enqueues NCCL instead.
  const void* node_dc;    // ncclDevComm (device copy)
  void* node_win;         // ncclWindow_t of the slot buffer
  int32_t node_parity;    // which half of the slot buffer this call uses
  int32_t node_slot;      // bytes per rank slot

  int64_t max_inner;      // CSR: the caller's bound on a row's length (0 = not given)
};

}  // namespace hpar
