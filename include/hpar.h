/* hpar.h — C ABI of the B200-native hierarchical nested-parallel reduction
 * library (libhpar.so), after "Generalizing Hierarchical Parallelism"
 * (M. Kruse, arXiv 2309.01906).  Citations: P:<line> = PAPER.md,
 * S:<line> = SPEC.md of the reference; §8 = SURVEY.md §8.
 *
 * The library executes a nested parallel/worksharing loop nest whose levels
 * are bound to the B200 hierarchy  node -> GPU -> cluster -> CTA -> warp ->
 * lane  ("parallel level(...)"), with per-level iteration
 * partitioning, level-scoped barriers and
 * the level-by-level reduction tree ("on each level, one of the
 * tasks collects the results from all sibling tasks").
 *
 * LEVEL CONVENTION (§8 reading #1).  A level named X has tasks that are X's,
 * as in the paper's `parallel level(warps)` printing one line per warp
 * (P:106-118).  Its `num` is the number of X per parent and its property
 * flags (Table 2) say what SIBLING X's can do together.
 *
 * GENERAL CONVENTIONS.
 *  - Every call returns hpar_status: 0 = OK, < 0 = error.  The text of the
 *    last error of the calling thread is hpar_last_error(); it names the
 *    level or argument at fault.  Validation happens before
 *    any launch: errors are diagnosed, never undefined behaviour (S:338,
 *    S:393).
 *  - `stream` arguments are cudaStream_t values passed as void* (NULL = the
 *    legacy default stream).  Calls that take a stream are asynchronous:
 *    they enqueue work and return; device faults surface at the caller's
 *    next synchronisation.
 *  - The caller owns every buffer it passes (device pointers, e.g. torch
 *    tensors), the stream and a borrowed NCCL communicator; the library
 *    never frees them.  A nest owns a small device workspace (tickets,
 *    cluster partials) that it allocates at creation and frees at destroy.
 *  - A nest must not be used from two streams concurrently (a run
 *    handle is single-user); distinct nests are independent.  Query results
 *    are immutable.
 */
#ifndef HPAR_H
#define HPAR_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HPAR_OK = 0,
  HPAR_E_INVALID = -1,     /* malformed argument / nest (e.g. non-contiguous collapse) */
  HPAR_E_CAPABILITY = -2,  /* level lacks a Table-2 property the request needs   */
  HPAR_E_SCHEDULE = -3,    /* schedule(none) with more iterations than tasks     */
  HPAR_E_PARTITION = -4,   /* partition width does not divide num, or < 1           */
  HPAR_E_UNSUPPORTED = -5, /* valid in the model but not implemented by this library           */
  HPAR_E_CUDA = -6,        /* CUDA runtime error (text carries cudaGetErrorString)             */
  HPAR_E_NCCL = -7,        /* NCCL error (text carries ncclGetErrorString / last error)        */
  HPAR_E_NOMEM = -8        /* allocation failure                                                */
} hpar_status;

/* Hardware levels of one 8xB200 node, outermost first (Fig. 1 analogue,
 * P:517-599; B200 instance per §8(a) A0). */
typedef enum {
  HPAR_NODE = 0,    /* the box (root, 1 task)                         */
  HPAR_GPU = 1,     /* one B200 per rank; siblings = ranks of the comm */
  HPAR_CLUSTER = 2, /* thread-block cluster                */
  HPAR_CTA = 3,     /* CTA ("CUDA block")                       */
  HPAR_WARP = 4,    /* warp                                    */
  HPAR_LANE = 5,    /* warp lane ("CUDA thread")                */
  HPAR_NLEVELS = 6
} hpar_level;

/* Table 2 level properties as flag bits. */
enum {
  HPAR_P_BARRIER = 1 << 0,
  HPAR_P_CRITICAL = 1 << 1,
  HPAR_P_ATOMIC = 1 << 2,
  HPAR_P_SHUFFLE = 1 << 3,
  HPAR_P_OVERSUB = 1 << 4,   /* "oversubcribable" (sic)          */
  HPAR_P_DYNAMIC = 1 << 5,   /* nonstatic schedules allowed      */
  HPAR_P_LOCKSTEP = 1 << 6,
  HPAR_P_PROGRESS = 1 << 7,
  HPAR_P_GLOBALMEM = 1 << 8,
  HPAR_P_LOCALMEM = 1 << 9,  /* memory shared by the siblings            */
  HPAR_P_GROUPMEM = 1 << 10, /* memory private to each sibling           */
  HPAR_P_CACHE = 1 << 11
};

/* One row of the level table (Table 2 per level). */
typedef struct {
  int32_t level;           /* hpar_level                                              */
  uint32_t props;          /* HPAR_P_* flags of the siblings at this level            */
  char name[16];           /* "node", "gpu", "cluster", "cta", "warp", "lane"         */
  int64_t num;             /* tasks per parent running in parallel (resident), num(c) */
  int64_t max_num;         /* launch limit per parent (oversubscription bound)        */
  uint64_t localmem_bytes; /* memory shared by the siblings (Table 2 localmem)        */
  uint64_t groupmem_bytes; /* memory private to each task (Table 2 groupmem)          */
  double grainedness;      /* relative task duration: SM cycles of one
                              combine/synchronisation step among the siblings —
                              measured on B200 for cluster / CTA / warp / lane
                              (1495 / 623 / 59 / 30, scripts/grain_probe.cu),
                              estimates for GPU (NCCL, ~2e4) and node (1e6)      */
} hpar_level_info;

/* A device description.  hpar_device_describe() fills it from the CUDA
 * runtime; callers may also pass a synthetic one (host-only validation). */
typedef struct {
  int32_t sm_count;
  int32_t max_threads_per_sm;
  int32_t max_blocks_per_sm;
  int32_t warp_size;
  int64_t smem_per_block_optin; /* bytes */
  int64_t smem_per_sm;          /* bytes */
  int64_t l2_bytes;
  int64_t hbm_bytes;
  int32_t cc_major, cc_minor;
  int32_t cluster_launch;       /* 1 if clusters are supported                  */
  int32_t max_cluster_size;     /* portable cluster limit (8)                   */
} hpar_device_desc;

/* Fill *out from cudaGetDeviceProperties(device). */
hpar_status hpar_device_describe(int32_t device, hpar_device_desc* out);

/* Pure host: the B200 level table for a device description and geometry
 * (nranks GPUs, K CTAs per cluster, W warps per CTA, C resident clusters;
 * 0 = defaults K=2, W=8, C=derived from the description).  Writes
 * HPAR_NLEVELS rows to out[] and *nlevels = HPAR_NLEVELS. */
hpar_status hpar_hierarchy_describe(const hpar_device_desc* dev, int32_t nranks, int32_t cluster_dim,
                                    int32_t warps_per_cta, int64_t clusters,
                                    hpar_level_info out[HPAR_NLEVELS], int32_t* nlevels);

/* §8(a) A0: the level table of `device`, with the GPU level's num = the size
 * of `nccl_comm` (ncclCommCount of an ncclComm_t borrowed from the caller;
 * NULL = 1 GPU) and the cluster level's num = cudaOccupancyMaxActiveClusters
 * of the flat streaming kernel in the default geometry (K = 2 CTAs of W = 8
 * consumer warps + 1 producer warp, 64 KiB ring): the clusters that can run
 * at once (P:139 num), GPC placement included.  Also the default C of
 * hpar_nest_create (one wave of co-resident clusters). */
hpar_status hpar_hierarchy_query(int32_t device, void* nccl_comm, hpar_level_info out[HPAR_NLEVELS],
                                 int32_t* nlevels);

/* ---- nests --------------------------------------------------------------
 * A nest is an ordered list of nest levels, outermost first (the nested
 * `parallel level(...)` constructs of P:104-118 with their worksharing
 * `for`).  Each nest level
 *  - binds a contiguous range of hardware levels [first, last] (first < last
 *    = collapsed level: num = product, flags = intersection);
 *    consecutive nest levels must be contiguous and the last one must end at
 *    HPAR_LANE.  Hardware levels above the first nest level run 1 task.
 *  - may partition its last hardware level: width > 0 splits it into an outer
 *    slice of num/width tasks (this nest level) and an inner slice of `width`
 *    tasks that the NEXT nest level must start with (P:327-340 `lanes(16)`;
 *    S:93-101).  Only HPAR_LANE may be partitioned by this library.
 *  - workshares loop `loop` (0 = outer, 1 = inner; P:215-225 bind_ancestor)
 *    with `schedule`:
 *      STATIC        contiguous blocks, sizes differ by <= 1, earlier larger;
 *      STATIC_CHUNK  chunks of `chunk` positions round-robin;
 *      DYNAMIC       chunks of `chunk` claimed from an atomic ticket shared by
 *                    the siblings (only where Table-2 `dynamic` holds);
 *      NONE          task t runs iteration t, tasks >= n are masked; n > T is
 *                    HPAR_E_SCHEDULE.
 *    A level refines its parent's local list of that loop (the list of
 *    positions the parent task owns, in order).
 *  - fanout: tasks per parent; 0 = derived from the geometry.  A nonzero
 *    fanout on a range containing HPAR_CLUSTER fixes the cluster count C.
 */
typedef enum {
  HPAR_SCHED_STATIC = 0,
  HPAR_SCHED_STATIC_CHUNK = 1,
  HPAR_SCHED_DYNAMIC = 2,
  HPAR_SCHED_NONE = 3
} hpar_schedule;

typedef struct {
  int32_t first, last; /* hardware level range, HPAR_GPU <= first <= last <= HPAR_LANE */
  int32_t schedule;    /* hpar_schedule                                                  */
  int32_t loop;        /* 0 or 1; 2 = the collapsed (row, nonzero) space of a CSR
                          nest (the fused CSR kernels, reading #14) */
  int64_t chunk;       /* STATIC_CHUNK / DYNAMIC chunk (>= 1)                            */
  int64_t fanout;      /* tasks per parent; 0 = derived                                  */
  int32_t width;       /* partition width of `last`, 0 = none                            */
  int32_t reserved;
} hpar_nest_level;

#define HPAR_MAX_NEST 8

typedef struct {
  int32_t device;        /* CUDA ordinal; -1 = describe-only (no CUDA calls)       */
  int32_t rank, nranks;  /* used when nccl_comm == NULL (single GPU: 0 / 1)         */
  int32_t cluster_dim;   /* K CTAs per cluster; 0 = 2                               */
  int32_t warps_per_cta; /* W; 0 = 8                                                */
  int32_t flags;         /* HPAR_NEST_* options                                     */
  int64_t clusters;      /* C; 0 = derived (resident clusters)                      */
  void* nccl_comm;       /* borrowed ncclComm_t for the GPU level, or NULL          */
  const hpar_device_desc* desc; /* required when device == -1                       */
} hpar_nest_config;

/* flags: HPAR_NEST_NODE_FUSED — the node level runs inside
 * the kernel instead of as a host-enqueued ncclAllReduce: the CTA that folds
 * a GPU's total stores it into every rank's symmetric slot (NCCL LSA pointers
 * over NVLink), all GPUs meet at one NCCL LSA barrier, and each folds the
 * slots in rank order (so ordered ops stay ordered).  Needs nccl_comm; nest
 * creation and destruction become COLLECTIVE over the communicator (NCCL
 * window registration and device-communicator creation); all ranks must be
 * in one NVLink domain (else HPAR_E_CAPABILITY); NCCL >= 2.28 (else
 * HPAR_E_NCCL).  Applies to total-mode calls; keyed calls have no node
 * level. */
#define HPAR_NEST_NODE_FUSED 1
/* HPAR_NEST_NODE_ALWAYS: run the host-enqueued node level (ncclAllReduce /
 * the ordered ops' allgather + rank fold) and the GPU-level barrier's NCCL
 * rendezvous even when the communicator has ONE rank, where they are
 * identities — so the collective path executes on a one-GPU box.  Needs
 * nccl_comm.  A diagnostic / test option; results are unchanged. */
#define HPAR_NEST_NODE_ALWAYS 2

typedef struct hpar_nest* hpar_nest_t;

/* Resolved nest: the geometry and per-nest-level tasks and flags. */
typedef struct {
  int64_t G, C, K, W;               /* GPUs, clusters, CTAs/cluster, warps/CTA             */
  int32_t rank;
  int32_t nlevels;
  int32_t lane_width;               /* lane partition width, 0 = none                      */
  int32_t reserved;
  int64_t tasks[HPAR_MAX_NEST];     /* tasks per parent of every nest level (T)            */
  int64_t total[HPAR_MAX_NEST];     /* tasks of every nest level on this node             */
  uint32_t props[HPAR_MAX_NEST];    /* collapsed Table-2 flags of every nest level         */
  int64_t threads_per_gpu;          /* C*K*W*32 = leaf tasks per GPU                       */
} hpar_nest_info_t;

/* §8(a) A1.  Validate and resolve the nest, allocate its workspace.
 * Errors: HPAR_E_INVALID (range, contiguity, loop, fanout mismatch, nest
 * without the GPU level while nranks > 1), HPAR_E_CAPABILITY (DYNAMIC on a
 * level without `dynamic`), HPAR_E_PARTITION (width does not divide
 * the level's num), HPAR_E_UNSUPPORTED, HPAR_E_CUDA, HPAR_E_NCCL. */
hpar_status hpar_nest_create(const hpar_nest_level* levels, int32_t nlevels, const hpar_nest_config* cfg,
                             hpar_nest_t* out);
hpar_status hpar_nest_destroy(hpar_nest_t nest);
hpar_status hpar_nest_info(hpar_nest_t nest, hpar_nest_info_t* out);

/* §8(a) A2: the rank's shard of the outermost loop under the GPU level's
 * static-block schedule: [*begin, *begin + *count) of [0, n0). */
hpar_status hpar_shard_range(hpar_nest_t nest, int64_t n0, int32_t rank, int64_t* begin, int64_t* count);

/* ---- the hot path ---------------------------------------------------- */
/* HPAR_OP_AFFINE: an ordered, non-commutative user-defined operator (
 * S:377).  int64 element x is the affine map y -> a*y + b (mod 2^64)
 * with a = 2x+1, b = x*x; the fold composes the maps in ascending iteration
 * order (left operand applied first), i.e. it runs the linear recurrence
 * y <- a_i*y + b_i.  Result: uint64[2] = (A, B) of the composed map (per
 * row when keyed; out_dtype HPAR_U64).  Node level: the per-rank maps are
 * gathered and folded in rank order (never an NCCL reduction).  Served by
 * the generic kernel (all trees are order-preserving). */
typedef enum { HPAR_OP_SUM = 0, HPAR_OP_MIN = 1, HPAR_OP_MAX = 2, HPAR_OP_HIST256 = 3, HPAR_OP_AFFINE = 4 } hpar_op;
typedef enum { HPAR_I32 = 0, HPAR_I64 = 1, HPAR_F32 = 2, HPAR_F64 = 3, HPAR_U8 = 4, HPAR_U64 = 5 } hpar_dtype;

enum { HPAR_VERIFY_COVERAGE = 1, HPAR_VERIFY_PARTIALS = 2, HPAR_VERIFY_FINGERPRINT = 4 };
enum { HPAR_LOCAL_N0_EMPTY = -1 };  /* hpar_reduce_desc.local_n0: an empty caller-sharded shard */

typedef struct {
  int32_t op;            /* hpar_op                                                        */
  int32_t in_dtype;      /* I32 / I64 / F32 / F64 (SUM, MIN, MAX); U8 (HIST256)             */
  int32_t nloops;        /* 1: flat loop over n0; 2: loop 0 (rows) x loop 1 (columns)       */
  int32_t keyed;         /* 0: one total (folded up to the node level);
                            1: one result per loop-0 iteration (row-wise / CSR)            */
  const void* in;        /* device; this rank's shard: flat [n0_local], dense rows
                            [n0_local][ld], or CSR values.  Element-aligned is enough: a
                            pointer off a 16-byte boundary (a tensor slice) keeps the fused
                            kernels (enclosing-granule TMA copies; CSR: offsets + shift in
                            a workspace copy), reading never past the granule of a valid
                            element                                                        */
  int64_t n0;            /* GLOBAL extent of loop 0 (sharded over the GPU level)           */
  int64_t n1;            /* dense extent of loop 1; CSR: the number of values
                            (offsets[n0_local]), or 0 = read it from the device (one
                            host synchronisation per call; not inside graph capture)   */
  int64_t ld;            /* dense row stride in elements (>= n1)                            */
  const int64_t* offsets;/* CSR: device int64 [n0_local + 1], local row offsets, or NULL  */
  int64_t max_inner;     /* CSR: max row length (required with schedule NONE on loop 1, and
                            by the fused CSR kernel at >= 2^31 nonzeros per rank, where
                            max_inner * 256 < 2^31 must hold; 0 = not given)                */
  void* out;             /* device.  keyed == 0: accumulator scalar (SUM i32/i64 -> int64,
                            f32/f64 -> double; MIN/MAX same types) or uint64[256] bins;
                            valid on EVERY rank after the stream completes (the node level
                            is an allreduce).  keyed == 1: n0_local results of
                            out_dtype                                                      */
  int32_t out_dtype;     /* keyed results: HPAR_F32 (rounded once from fp64) or HPAR_F64,
                            HPAR_I64 for integer inputs                                   */
  int32_t verify;        /* 0 in timed runs; HPAR_VERIFY_* bits                            */
  void* level_partials[HPAR_MAX_NEST]; /* verify: per nest level, accumulator type;
                            total mode: [total tasks of the level on this GPU] indexed by
                            the task's mixed-radix id below the GPU level (the GPU level
                            itself: 1 entry, this rank); keyed mode: inner (loop-1) levels,
                            [n0_local][tasks per row owner]                               */
  int64_t* coverage_owner;  /* verify: per local iteration, leaf task id (global)          */
  uint32_t* coverage_count; /* verify: per local iteration, visit count (caller zeroes)    */
  uint64_t* fingerprint;    /* verify: uint64[3] += {F_once, F_owner, iterations}         */
  uint64_t global_begin;    /* global index of this rank's first iteration (fingerprints) */
  int64_t local_n0;         /* CSR only: this rank's row count when the caller shards rows
                               by nonzeros (hpar_shard_range_csr); 0 = not caller-sharded
                               (the GPU level's static block of n0); HPAR_LOCAL_N0_EMPTY
                               (-1) = this rank's caller-sharded shard has no rows: the
                               call validates and returns HPAR_OK without a launch (keyed
                               results have no node-level collective)                     */
} hpar_reduce_desc;

/* §8(e) C3: nnz-balanced contiguous row shards of a CSR matrix over
 * `nranks` GPUs — the GPU level's static block weighted by nonzeros.  Rank g
 * gets rows [b_g, b_{g+1}) with b_g = the first row whose start offset is
 * >= ceil(g * nnz / nranks) (b_0 = 0, b_nranks = rows), so every shard holds
 * nnz / nranks nonzeros up to one row.  `offsets`: HOST int64 [rows + 1],
 * nondecreasing from 0.  Pure host. */
hpar_status hpar_shard_range_csr(const int64_t* offsets, int64_t rows, int32_t nranks, int32_t rank,
                                 int64_t* begin, int64_t* count);

/* §8(a) A2-A9: execute the nest over the loop(s) in `desc` and reduce.
 * One launch of a kernel specialisation picked by the planner (the generic
 * nest interpreter, or a fused streaming kernel when the nest matches its
 * shape: flat, teams x threads, row-wise, histogram, CSR fp32 sums, CSR
 * other ops / dtypes — hpar_last_kernel names it), followed on the same
 * stream by one ncclAllReduce at the node level when the GPU level has more
 * than one rank (total mode; ordered ops: allgather + rank-order fold).  A
 * CSR call at >= 2^31 nonzeros per rank without a proving max_inner first
 * measures its row-block spans (one host synchronisation).  Errors:
 * HPAR_E_INVALID (pointers, sizes, alignment of verify buffers),
 * HPAR_E_SCHEDULE (schedule NONE overflow), HPAR_E_UNSUPPORTED (op/dtype),
 * HPAR_E_CAPABILITY (keyed results whose combine would need a barrier the
 * levels lack), HPAR_E_CUDA, HPAR_E_NCCL.  Empty loops yield the identity. */
hpar_status hpar_parallel_for_reduce(hpar_nest_t nest, const hpar_reduce_desc* desc, void* stream);

/* §8(a) A10: a host-level barrier among the sibling tasks of hardware level
 * `level`, enqueued on `stream`.
 *   HPAR_GPU:     a cross-rank rendezvous on the stream (a 1-int NCCL
 *                 allreduce over the nest's communicator; no-op with 1 rank).
 *   HPAR_CLUSTER: HPAR_E_CAPABILITY — clusters have no barrier (P:178 read
 *                 as "does not support"; S:348 diagnose, never UB).
 *   HPAR_CTA / HPAR_WARP / HPAR_LANE / HPAR_NODE: HPAR_OK, nothing enqueued.
 *                 Between two calls every task of these levels has finished
 *                 and its writes are visible at the kernel boundary, which
 *                 stream order already provides; INSIDE a
 *                 call these levels synchronise with __syncwarp / bar.sync /
 *                 barrier.cluster (probed by hpar_barrier_probe).
 * Errors: HPAR_E_INVALID (NULL nest, bad level, describe-only nest),
 * HPAR_E_CAPABILITY, HPAR_E_NCCL. */
hpar_status hpar_barrier(hpar_nest_t nest, int32_t level, void* stream);

/* Verify call for the in-kernel level barriers (§8(c) #5; the §3.7 fallback
 * pattern P:308-323, generalised by S:360 "every lane gets 36").  Launches
 * the nest's C clusters x K CTAs x W warps; for `rounds` rounds every task of
 * `level` (HPAR_CTA: each CTA; HPAR_WARP: each warp; HPAR_LANE: each lane)
 * writes fp_mix((round << 40) ^ id) to its slot — id = the task's linear id
 * on the GPU (CTA: blockIdx; warp: blockIdx * W + warp; lane: blockIdx *
 * 32 W + thread) — the level's barrier runs, and the task adds the sum of
 * its siblings' slots (mod 2^64) to a running fold.  folds[task] (device
 * uint64, C*K / C*K*W / C*K*W*32 entries, caller-owned) receives the fold
 * over all rounds; the caller compares it with the group sums computed
 * independently (the oracle's fp_mix).  flags HPAR_PROBE_NO_BARRIER: the
 * negative control — the barrier is omitted and sibling k delays its write
 * by (k+1) * delay_ns, so readers fold stale slots.  Errors:
 * HPAR_E_CAPABILITY (HPAR_CLUSTER), HPAR_E_INVALID, HPAR_E_CUDA. */
enum { HPAR_PROBE_NO_BARRIER = 1 };
hpar_status hpar_barrier_probe(hpar_nest_t nest, int32_t level, int32_t rounds, uint32_t flags, uint32_t delay_ns,
                               uint64_t* folds, void* stream);

/* ---- property-based level selection (§3.2-3.3) --------------
 * A construct `parallel sync(demand) reserve(sync(reserve))` asks for levels
 * by the Table-2 properties it needs instead of naming them.  Constructs are
 * given outermost first; each takes a contiguous run of the still-unassigned
 * hardware levels starting at the first one (levels are never skipped), the
 * LONGEST run whose collapsed flags (intersection) contain `demand`
 * while the remaining levels can still serve the inner constructs (maximal
 * fan-out: "would use all available parallelism"; SPEC policy S:283).
 * `reserve` additionally requires the levels left to the inner constructs
 * to satisfy it.  The innermost construct must end at the lane
 * level.  Output: one hpar_nest_level per construct (first/last filled,
 * schedule/loop/chunk copied), ready for hpar_nest_create.
 * Errors: HPAR_E_CAPABILITY when no assignment satisfies the demands
 * ("unsatisfiable sync demand"), HPAR_E_INVALID on bad arguments. */
typedef struct {
  uint32_t demand;   /* HPAR_P_* flags the construct needs (0 = sync())       */
  uint32_t reserve;  /* flags the levels left to inner constructs must offer  */
  int32_t schedule;  /* copied to the nest level                               */
  int32_t loop;
  int64_t chunk;
} hpar_sync_construct;

hpar_status hpar_nest_resolve(const hpar_sync_construct* constructs, int32_t n, const hpar_level_info* table,
                              hpar_nest_level* out);

/* Portable level aliases: "devices" = gpu, "teams" =
 * cluster..cta, "threads" = warp..lane, "simd" = lane, plus the hardware
 * level names.  Writes the hardware range of `name`. */
hpar_status hpar_level_alias(const char* name, int32_t* first, int32_t* last);

/* ---- hierarchical memory: ghost maps (§4) --
 * A construct at one level maps one array section per sibling d:
 *   map(to(d):   A[off_r : len_r][off_c : len_c])   what d holds, ghosts incl.
 *   map(from(d): A[off_r : len_r][off_c : len_c])   what d writes back
 * per dimension offset = mul * coord + add, coord = (d / grid_cols,
 * d % grid_cols) — the paper's `(d/2)*511 : 513` form; sections are
 * offset:length (OpenMP array sections).  The to-sections may overlap (the
 * ghost surface); the from-sections "must have unique sources"
 * (P:383).  All host-side and pure (no device work). */
typedef struct {
  int64_t mul, add, len;
} hpar_map_dim;
typedef struct {
  int64_t extent[2];     /* parent array rows, cols                       */
  int32_t siblings;      /* S                                              */
  int32_t grid_cols;     /* sibling grid width (coords of d above)         */
  hpar_map_dim to[2];    /* rows, cols                                     */
  hpar_map_dim from[2];  /* rows, cols                                     */
} hpar_map_spec;
typedef struct {
  int64_t off[2]; /* first row, first col (global coordinates) */
  int64_t len[2]; /* rows, cols                                */
} hpar_rect;

/* Sections of sibling d (0 <= d < siblings), else HPAR_E_INVALID. */
hpar_status hpar_map_sections(const hpar_map_spec* m, int32_t d, hpar_rect* to, hpar_rect* from);

/* positive lengths; every section inside the array; from(d)
 * inside to(d); from-sections pairwise disjoint.  Returns HPAR_E_INVALID on
 * the first violation; for an overlap, `where` (if non-NULL) receives
 * {row, col, sibling_a, sibling_b} of the first shared element in row-major
 * order (a < b).  O(S^2) rectangle tests, no per-element work. */
hpar_status hpar_map_validate(const hpar_map_spec* m, int64_t where[4]);

/* Halo exchange list of sibling d (device-level ghost refresh): for every
 * other sibling e in ascending order, first the rectangle to(d) ∩ from(e)
 * that d receives from e (send = 0), then to(e) ∩ from(d) that d sends to e
 * (send = 1); empty intersections are omitted.  Writes min(cap, total)
 * entries to `out` (may be NULL when cap = 0) and the total to *n. */
typedef struct {
  int32_t peer;
  int32_t send;
  hpar_rect rect; /* global coordinates */
} hpar_halo;
hpar_status hpar_map_exchange_plan(const hpar_map_spec* m, int32_t d, hpar_halo* out, int32_t cap, int32_t* n);

/* One 5-point stencil step inside a sibling's packed buffer (§4's stencil
 * workload).  Every cell of `from` becomes
 *   ((((c + north) + south) + west) + east) / 5      (fp32, in that order)
 * except cells on the parent array's boundary (row 0 / extent[0]-1, col 0 /
 * extent[1]-1), which copy through.  Reads `in`, writes `out`; both hold the
 * to-section row-major (to.len[0] rows, pitch `ld` floats, ld >= to.len[1],
 * ld % 4 == 0, 16-byte aligned) on the nest's device; cells of `out` outside
 * `from` are not written.  The kernel tiles `from` over the CTAs (static,
 * persistent); a CTA's tile arrives by a 2-D TMA box with a 1-cell ghost
 * ring — the same map one level down (block-shared memory).
 * Errors: HPAR_E_INVALID (from ⊄ to, a non-boundary from cell whose
 * neighbour lies outside to, layout/alignment), HPAR_E_CUDA. */
typedef struct {
  const float* in;
  float* out;
  int64_t ld;
  hpar_rect to;
  hpar_rect from;
  int64_t extent[2];
} hpar_stencil_desc;
hpar_status hpar_stencil5(hpar_nest_t nest, const hpar_stencil_desc* desc, void* stream);

/* Ghost refresh at the device level over the nest's NCCL communicator
 * (rank = sibling; needs siblings == nranks): every rectangle of this
 * rank's exchange plan goes through a packed staging buffer with
 * ncclSend/ncclRecv in one NCCL group on `stream`.  One rank: no-op.
 * `buf` = this rank's to-section buffer (pitch ld floats). */
hpar_status hpar_map_exchange(hpar_nest_t nest, const hpar_map_spec* m, float* buf, int64_t ld, void* stream);

/* The same refresh among S sibling buffers on ONE device (tests, replicas):
 * bufs[d] = sibling d's to-section buffer (pitch ld floats); 2-D
 * device-to-device copies on `stream`. */
hpar_status hpar_map_exchange_local(const hpar_map_spec* m, float* const* bufs, int64_t ld, void* stream);

/* Thread-local text of the last error ("" if none). */
const char* hpar_last_error(void);
/* Name of the kernel specialisation the last hpar_parallel_for_reduce on
 * this nest launched ("generic", "flat_tma", ...). */
const char* hpar_last_kernel(hpar_nest_t nest);
/* Library version string. */
const char* hpar_version(void);

#ifdef __cplusplus
}
#endif
#endif
