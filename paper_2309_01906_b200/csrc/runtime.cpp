// runtime.cpp — host side of libhpar.so: the C ABI of include/hpar.h.
//
//  * level table (Table 2 for B200; §8(a) A0)
//  * nest validation and resolution (§8(a) A1)
//  * planner: picks the kernel specialisation for a call, builds NestArgs
//  * workspace (self-resetting tickets, cluster partials)
//  * node level: one ncclAllReduce over NVLink on the caller's stream
//    (§8(a) A9), NCCL resolved with dlopen from the library torch loaded
//  * level barriers (§8(a) A10)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "hpar.h"
#include "nccl.h"         // types only; functions are resolved with dlsym
#include "nccl_device.h"  // ncclDevComm (fused node level, NEXT f1)
#include "plan.h"

namespace hpar {
cudaError_t launch_generic(const NestArgs& a, int threads, cudaStream_t s);
cudaError_t launch_probe(int level, int64_t C, int K, int W, int rounds, int no_barrier, uint32_t delay_ns,
                         unsigned long long* folds, cudaStream_t s);
// fused specialisations (kernel_flat.cu, kernel_rowwise.cu, kernel_hist.cu)
bool flat_matches(const NestArgs& a, const char** why);
cudaError_t launch_flat(const NestArgs& a, int W, cudaStream_t s, const char** name);
bool rowwise_matches(const NestArgs& a, const char** why);
cudaError_t launch_rowwise(const NestArgs& a, int W, cudaStream_t s, const char** name);
bool hist_matches(const NestArgs& a, const char** why);
cudaError_t launch_hist(const NestArgs& a, int W, cudaStream_t s, const char** name);
int flat_resident_ctas_per_sm(int W);
int flat_max_active_clusters(int K, int W);
bool segmented_matches(const NestArgs& a, const char** why);
cudaError_t launch_segmented(const NestArgs& a, void* wsbuf, int64_t ws_nnz, int64_t* off_ws, cudaStream_t s,
                             const char** name);
cudaError_t segmented_span_ok(const NestArgs& a, unsigned long long* scratch, cudaStream_t s, bool* ok,
                              bool* needs_sync);
bool segrows_matches(const NestArgs& a, const char** why);
size_t segrows_ws_bytes(int64_t nnz);
cudaError_t launch_segrows(const NestArgs& a, void* wsbuf, int64_t ws_nnz, cudaStream_t s, const char** name);
size_t segmented_ws_bytes(int64_t nnz);
void segmented_ws_qrow(int64_t nnz, size_t* off, size_t* len);
cudaError_t launch_affine_rank_fold(const void* gathered, int G, void* out, cudaStream_t s);
bool teams_matches(const NestArgs& a, const char** why);
cudaError_t launch_teams(const NestArgs& a, int W, cudaStream_t s, const char** name);
// kernel_stencil.cu
cudaError_t launch_stencil5(const hpar_stencil_desc& d, int device, int sm_count, cudaStream_t s, const char** why);
}  // namespace hpar

using namespace hpar;

// ------------------------------------------------------------- errors ----
static thread_local std::string g_last_error;

static hpar_status fail(hpar_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}
static hpar_status ok() {
  g_last_error.clear();
  return HPAR_OK;
}
#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) return fail(HPAR_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

extern "C" const char* hpar_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* hpar_version(void) { return "hpar 0.1 (sm_100a)"; }

// --------------------------------------------------------------- NCCL ----
namespace {
struct NcclApi {
  bool loaded = false;
  std::string why;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*commUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  const char* (*getLastError)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  // symmetric memory + device communicator (NCCL >= 2.28): fused node level
  ncclResult_t (*memAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*memFree)(void*) = nullptr;
  ncclResult_t (*winRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*winDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
  ncclResult_t (*devCommCreate)(ncclComm_t, const ncclDevCommRequirements_t*, ncclDevComm_t*) = nullptr;
  ncclResult_t (*devCommDestroy)(ncclComm_t, const ncclDevComm_t*) = nullptr;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
  // Prefer the NCCL already loaded into the process (torch's), so a
  // communicator borrowed from torch's ProcessGroupNCCL is ABI-compatible.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    g_nccl.why = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
    return;
  }
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.commCount = (decltype(g_nccl.commCount))dlsym(h, "ncclCommCount");
  g_nccl.commUserRank = (decltype(g_nccl.commUserRank))dlsym(h, "ncclCommUserRank");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.getLastError = (decltype(g_nccl.getLastError))dlsym(h, "ncclGetLastError");
  g_nccl.send = (decltype(g_nccl.send))dlsym(h, "ncclSend");
  g_nccl.recv = (decltype(g_nccl.recv))dlsym(h, "ncclRecv");
  g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
  g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.memAlloc = (decltype(g_nccl.memAlloc))dlsym(h, "ncclMemAlloc");
  g_nccl.memFree = (decltype(g_nccl.memFree))dlsym(h, "ncclMemFree");
  g_nccl.winRegister = (decltype(g_nccl.winRegister))dlsym(h, "ncclCommWindowRegister");
  g_nccl.winDeregister = (decltype(g_nccl.winDeregister))dlsym(h, "ncclCommWindowDeregister");
  g_nccl.devCommCreate = (decltype(g_nccl.devCommCreate))dlsym(h, "ncclDevCommCreate");
  g_nccl.devCommDestroy = (decltype(g_nccl.devCommDestroy))dlsym(h, "ncclDevCommDestroy");
  g_nccl.loaded = g_nccl.allReduce && g_nccl.commCount && g_nccl.commUserRank && g_nccl.getErrorString;
  if (!g_nccl.loaded) g_nccl.why = "libnccl.so.2 lacks required symbols";
}
hpar_status need_nccl() {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl.loaded) return fail(HPAR_E_NCCL, "NCCL unavailable: %s", g_nccl.why.c_str());
  return HPAR_OK;
}
hpar_status nccl_fail(ncclResult_t r, ncclComm_t comm, const char* what) {
  const char* last = (g_nccl.getLastError && comm) ? g_nccl.getLastError(comm) : "";
  return fail(HPAR_E_NCCL, "%s: %s %s", what, g_nccl.getErrorString(r), last ? last : "");
}
}  // namespace

// --------------------------------------------------------- level table ----
namespace {
const char* kLevelNames[HPAR_NLEVELS] = {"node", "gpu", "cluster", "cta", "warp", "lane"};

// Table 2 flags of the SIBLINGS at each hardware level (member convention,
// §8 reading #1; per-level evidence in DESIGN.md "Level table").
uint32_t level_props(int level) {
  switch (level) {
    case HPAR_NODE:
      return HPAR_P_PROGRESS | HPAR_P_GROUPMEM;
    case HPAR_GPU:  // NCCL rendezvous; no cross-GPU atomics; separate HBM
      return HPAR_P_BARRIER | HPAR_P_PROGRESS | HPAR_P_GROUPMEM;
    case HPAR_CLUSTER:  // no barrier (read "does not"), no co-residency guarantee
      return HPAR_P_ATOMIC | HPAR_P_OVERSUB | HPAR_P_DYNAMIC | HPAR_P_GLOBALMEM | HPAR_P_GROUPMEM | HPAR_P_CACHE;
    case HPAR_CTA:  // barrier.cluster, DSMEM, co-scheduled
      return HPAR_P_BARRIER | HPAR_P_ATOMIC | HPAR_P_DYNAMIC | HPAR_P_PROGRESS | HPAR_P_GLOBALMEM |
             HPAR_P_LOCALMEM | HPAR_P_GROUPMEM | HPAR_P_CACHE;
    case HPAR_WARP:  // bar.sync, shared memory of the SM
      return HPAR_P_BARRIER | HPAR_P_ATOMIC | HPAR_P_DYNAMIC | HPAR_P_PROGRESS | HPAR_P_GLOBALMEM |
             HPAR_P_LOCALMEM | HPAR_P_CACHE;
    case HPAR_LANE:  // __syncwarp, SHFL; independent thread scheduling: not lockstep
      return HPAR_P_BARRIER | HPAR_P_SHUFFLE | HPAR_P_PROGRESS | HPAR_P_GLOBALMEM | HPAR_P_GROUPMEM | HPAR_P_CACHE;
  }
  return 0;
}

// Grainedness (units unspecified): the SM-cycle cost of one
// synchronisation / combine step among the level's siblings.  CTA, warp,
// lane and cluster are MEASURED on B200 (scripts/grain_probe.cu,
// profiles/r02_grainedness.txt): a dependent SHFL step 30; slot store +
// bar.sync + sibling load among 8 warps 59; the same over DSMEM with
// barrier.cluster between 2 CTAs 623; a dependent atom.acq_rel.gpu through
// L2 (the single-pass ticket clusters meet at) 1495.  GPU and node are
// estimates (a small NCCL allreduce ~10 us; the job): no multi-GPU box here.
double level_grain(int level) {
  switch (level) {
    case HPAR_NODE: return 1e6;    // estimate
    case HPAR_GPU: return 2e4;     // estimate: NCCL 8-byte allreduce ~10 us
    case HPAR_CLUSTER: return 1495;
    case HPAR_CTA: return 623;
    case HPAR_WARP: return 59;
    case HPAR_LANE: return 30;
  }
  return 1;
}

int64_t default_resident_clusters(const hpar_device_desc& d, int K, int W) {
  int threads = W * 32;
  int by_threads = d.max_threads_per_sm / std::max(threads, 1);
  int per_sm = std::min(std::max(by_threads, 1), std::max(d.max_blocks_per_sm, 1));
  per_sm = std::min(per_sm, 4);  // the fused streaming kernels' residency
  int64_t ctas = (int64_t)d.sm_count * per_sm;
  return std::max<int64_t>(1, ctas / std::max(K, 1));
}
}  // namespace

extern "C" hpar_status hpar_device_describe(int32_t device, hpar_device_desc* out) {
  if (!out) return fail(HPAR_E_INVALID, "hpar_device_describe: out is NULL");
  cudaDeviceProp p;
  CUDA_TRY(cudaGetDeviceProperties(&p, device));
  memset(out, 0, sizeof(*out));
  out->sm_count = p.multiProcessorCount;
  out->max_threads_per_sm = p.maxThreadsPerMultiProcessor;
  out->max_blocks_per_sm = p.maxBlocksPerMultiProcessor;
  out->warp_size = p.warpSize;
  out->smem_per_block_optin = (int64_t)p.sharedMemPerBlockOptin;
  out->smem_per_sm = (int64_t)p.sharedMemPerMultiprocessor;
  out->l2_bytes = p.l2CacheSize;
  out->hbm_bytes = (int64_t)p.totalGlobalMem;
  out->cc_major = p.major;
  out->cc_minor = p.minor;
  int cl = 0;
  cudaDeviceGetAttribute(&cl, cudaDevAttrClusterLaunch, device);
  out->cluster_launch = cl;
  out->max_cluster_size = 8;
  return ok();
}

extern "C" hpar_status hpar_hierarchy_describe(const hpar_device_desc* d, int32_t nranks, int32_t cluster_dim,
                                               int32_t warps_per_cta, int64_t clusters,
                                               hpar_level_info out[HPAR_NLEVELS], int32_t* nlevels) {
  if (!d || !out) return fail(HPAR_E_INVALID, "hpar_hierarchy_describe: NULL argument");
  if (nranks < 1) return fail(HPAR_E_INVALID, "nranks must be >= 1");
  const int K = cluster_dim > 0 ? cluster_dim : 2;
  const int W = warps_per_cta > 0 ? warps_per_cta : 8;
  const int64_t C = clusters > 0 ? clusters : default_resident_clusters(*d, K, W);
  const int64_t num[HPAR_NLEVELS] = {1, nranks, C, K, W, 32};
  const int64_t maxn[HPAR_NLEVELS] = {1, nranks, (int64_t)0x7FFFFFFF / K, 16, 32, 32};
  const uint64_t smem = (uint64_t)d->smem_per_block_optin;
  const uint64_t localmem[HPAR_NLEVELS] = {0, 0, 0, (uint64_t)K * smem, smem, 0};
  const uint64_t groupmem[HPAR_NLEVELS] = {0, (uint64_t)d->hbm_bytes, (uint64_t)K * smem, smem, 0, 255 * 4};
  for (int l = 0; l < HPAR_NLEVELS; ++l) {
    hpar_level_info& r = out[l];
    memset(&r, 0, sizeof(r));
    r.level = l;
    r.props = level_props(l);
    strncpy(r.name, kLevelNames[l], sizeof(r.name) - 1);
    r.num = num[l];
    r.max_num = maxn[l];
    r.localmem_bytes = localmem[l];
    r.groupmem_bytes = groupmem[l];
    r.grainedness = level_grain(l);
  }
  if (nlevels) *nlevels = HPAR_NLEVELS;
  return ok();
}

extern "C" hpar_status hpar_hierarchy_query(int32_t device, void* nccl_comm, hpar_level_info out[HPAR_NLEVELS],
                                            int32_t* nlevels) {
  hpar_device_desc d;
  hpar_status s = hpar_device_describe(device, &d);
  if (s) return s;
  int nranks = 1;
  if (nccl_comm) {
    if ((s = need_nccl())) return s;
    ncclResult_t r = g_nccl.commCount((ncclComm_t)nccl_comm, &nranks);
    if (r != ncclSuccess) return nccl_fail(r, (ncclComm_t)nccl_comm, "ncclCommCount");
  }
  CUDA_TRY(cudaSetDevice(device));
  const int K = 2, W = 8;
  // P:139 num = the tasks the level can run at once: the clusters of the
  // default geometry that are co-resident (occupancy API, GPC placement incl.)
  const int64_t C = hpar::flat_max_active_clusters(K, W);
  if (C < 1) return fail(HPAR_E_CUDA, "cudaOccupancyMaxActiveClusters failed for the K=%d, W=%d geometry", K, W);
  return hpar_hierarchy_describe(&d, nranks, K, W, C, out, nlevels);
}

// --------------------------------------------------------------- nests ----
struct hpar_nest {
  hpar_nest_config cfg;
  int32_t device;
  int32_t rank, nranks;
  void* comm;
  int nlev;
  hpar_nest_level user[HPAR_MAX_NEST];
  DevLevel lv[HPAR_MAX_NEST];
  uint32_t props[HPAR_MAX_NEST];
  int64_t radix[S_NSLOTS];
  int lane_w;
  bool lane_part = false;
  int64_t G, C, K, W;
  int gpu_level;  // nest level holding the GPU slot, or -1
  // workspace
  unsigned int* grid_ticket = nullptr;
  void* cluster_partials = nullptr;
  size_t cluster_partials_bytes = 0;
  unsigned long long* dyn_tickets = nullptr;
  int64_t dyn_slots = 0;
  int32_t* error_flag = nullptr;
  int* barrier_word = nullptr;
  std::string last_kernel = "none";
  void* gather_buf = nullptr;  // node level of ordered ops: G gathered results
  void* seg_ws = nullptr;  // CSR segmented kernel workspace (grown on demand)
  int64_t* seg_off_ws = nullptr;  // shifted offsets for values off a 16-byte boundary (grown on demand)
  int64_t seg_off_rows = 0;
  void* sr_ws = nullptr;   // CSR rows kernel (other ops / dtypes) workspace (grown on demand)
  int64_t sr_ws_nnz = -1;
  size_t seg_ws_bytes = 0;
  int64_t seg_ws_nnz = -1;  // the nnz the workspace layout was built for (its capacity)
  float* halo_buf = nullptr;  // ghost exchange staging (grown on demand)
  size_t halo_bytes = 0;
  // fused node level (HPAR_NEST_NODE_FUSED; node_fused.cuh)
  bool node_fused = false;
  void* node_sym = nullptr;         // symmetric slot buffer (ncclMemAlloc)
  ncclWindow_t node_win = nullptr;  // its NCCL window
  ncclDevComm node_dc;              // device communicator (host copy)
  bool node_dc_made = false;
  void* node_dc_dev = nullptr;      // device copy of node_dc
  uint64_t node_calls = 0;
  bool node_always = false;  // HPAR_NEST_NODE_ALWAYS: the node collective also with one rank
};

namespace {
// slot range of a hardware level range, given whether `first` is the inner
// slice of a lane partition carried from the previous nest level and whether
// `last` is partitioned here.
int slot_first(int hw, bool inner_slice) {
  if (hw == HPAR_LANE) return inner_slice ? S_LANE_IN : S_LANE;
  return hw - 1;  // GPU=1 -> 0, CLUSTER -> 1, CTA -> 2, WARP -> 3
}
int slot_last(int hw, bool partitioned) {
  if (hw == HPAR_LANE) return partitioned ? S_LANE : S_LANE_IN;
  return hw - 1;
}
const char* sched_name(int s) {
  static const char* n[] = {"static", "static(c)", "dynamic(c)", "none"};
  return (s >= 0 && s < 4) ? n[s] : "?";
}
}  // namespace

namespace {
// Fused node level (NEXT f1): one symmetric slot buffer per rank ([2 halves]
// x [G ranks] x 2 KB, enough for 256 u64 bins), registered as an NCCL window,
// and a device communicator with one LSA barrier.  Collective over the
// communicator; every rank must sit in one NVLink (LSA) domain.
constexpr size_t kNodeSlot = 2048;
hpar_status node_fused_setup(hpar_nest* n) {
  if (!n->comm) return fail(HPAR_E_INVALID, "HPAR_NEST_NODE_FUSED needs an NCCL communicator");
  if (n->device < 0) return fail(HPAR_E_INVALID, "HPAR_NEST_NODE_FUSED needs a device");
  if (hpar_status s = need_nccl()) return s;
  if (!g_nccl.memAlloc || !g_nccl.winRegister || !g_nccl.devCommCreate || !g_nccl.devCommDestroy)
    return fail(HPAR_E_NCCL, "NCCL lacks the device API (ncclDevCommCreate / windows: NCCL >= 2.28)");
  ncclComm_t comm = (ncclComm_t)n->comm;
  const size_t bytes = ((2 * (size_t)n->nranks * kNodeSlot + 4095) / 4096) * 4096;
  ncclResult_t r = g_nccl.memAlloc(&n->node_sym, bytes);
  if (r != ncclSuccess) return nccl_fail(r, comm, "ncclMemAlloc");
  CUDA_TRY(cudaMemset(n->node_sym, 0, bytes));
  r = g_nccl.winRegister(comm, n->node_sym, bytes, &n->node_win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) return nccl_fail(r, comm, "ncclCommWindowRegister");
  ncclDevCommRequirements req;
  memset(&req, 0, sizeof(req));
  req.lsaBarrierCount = 1;
  r = g_nccl.devCommCreate(comm, &req, &n->node_dc);
  if (r != ncclSuccess) return nccl_fail(r, comm, "ncclDevCommCreate");
  n->node_dc_made = true;
  if (n->node_dc.lsaSize != n->node_dc.nRanks)
    return fail(HPAR_E_CAPABILITY, "fused node level: the %d ranks span more than one NVLink domain (LSA team of %d)",
                n->node_dc.nRanks, n->node_dc.lsaSize);
  CUDA_TRY(cudaMalloc(&n->node_dc_dev, sizeof(ncclDevComm)));
  CUDA_TRY(cudaMemcpy(n->node_dc_dev, &n->node_dc, sizeof(ncclDevComm), cudaMemcpyHostToDevice));
  n->node_fused = true;
  return HPAR_OK;
}
}  // namespace

extern "C" hpar_status hpar_nest_create(const hpar_nest_level* lv, int32_t nlevels, const hpar_nest_config* cfg,
                                        hpar_nest_t* out) {
  if (!lv || !cfg || !out) return fail(HPAR_E_INVALID, "hpar_nest_create: NULL argument");
  *out = nullptr;
  if (nlevels < 1 || nlevels > HPAR_MAX_NEST)
    return fail(HPAR_E_INVALID, "nest must have 1..%d levels (got %d)", HPAR_MAX_NEST, nlevels);
  const bool describe_only = cfg->device < 0;
  if (describe_only && !cfg->desc) return fail(HPAR_E_INVALID, "describe-only nest (device -1) needs cfg->desc");

  hpar_nest* n = new hpar_nest();
  n->cfg = *cfg;
  n->device = cfg->device;
  n->nlev = nlevels;
  n->comm = cfg->nccl_comm;
  n->rank = cfg->rank;
  n->nranks = cfg->nranks > 0 ? cfg->nranks : 1;
  auto bail = [&](hpar_status s) {
    delete n;
    return s;
  };
  if (cfg->nccl_comm) {
    hpar_status s = need_nccl();
    if (s) return bail(s);
    int cnt = 0, rk = 0;
    ncclResult_t r = g_nccl.commCount((ncclComm_t)cfg->nccl_comm, &cnt);
    if (r != ncclSuccess) return bail(nccl_fail(r, (ncclComm_t)cfg->nccl_comm, "ncclCommCount"));
    r = g_nccl.commUserRank((ncclComm_t)cfg->nccl_comm, &rk);
    if (r != ncclSuccess) return bail(nccl_fail(r, (ncclComm_t)cfg->nccl_comm, "ncclCommUserRank"));
    n->nranks = cnt;
    n->rank = rk;
  }
  if (n->rank < 0 || n->rank >= n->nranks)
    return bail(fail(HPAR_E_INVALID, "rank %d out of range for %d ranks", n->rank, n->nranks));

  // ---- structural validation (contiguity, ranges, loops, schedules) ----
  for (int a = 0; a < nlevels; ++a) {
    const hpar_nest_level& L = lv[a];
    n->user[a] = L;
    if (L.first < HPAR_GPU || L.last > HPAR_LANE || L.first > L.last)
      return bail(fail(HPAR_E_INVALID, "nest level %d: hardware range [%d,%d] outside gpu..lane", a, L.first, L.last));
    if (L.loop < 0 || L.loop > 2) return bail(fail(HPAR_E_INVALID, "nest level %d: loop must be 0, 1 or 2", a));
    if (L.schedule < 0 || L.schedule > 3) return bail(fail(HPAR_E_INVALID, "nest level %d: bad schedule", a));
    if ((L.schedule == HPAR_SCHED_STATIC_CHUNK || L.schedule == HPAR_SCHED_DYNAMIC) && L.chunk < 1)
      return bail(fail(HPAR_E_INVALID, "nest level %d: %s needs chunk >= 1", a, sched_name(L.schedule)));
    if (L.width < 0) return bail(fail(HPAR_E_PARTITION, "nest level %d: partition width %d < 1", a, L.width));
    if (L.width > 0 && L.last != HPAR_LANE)
      return bail(fail(HPAR_E_UNSUPPORTED, "nest level %d: only the lane level can be partitioned", a));
    if (a > 0) {
      const hpar_nest_level& P = lv[a - 1];
      const int expect = P.width > 0 ? P.last : P.last + 1;
      if (L.first != expect)
        return bail(fail(HPAR_E_INVALID,
                         "nest level %d: levels must be contiguous (collapse of a contiguous run, P:149-155): "
                         "expected first=%d, got %d", a, expect, L.first));
    }
  }
  if (lv[nlevels - 1].last != HPAR_LANE || lv[nlevels - 1].width != 0)
    return bail(fail(HPAR_E_INVALID, "the innermost nest level must end at the lane level (unpartitioned)"));
  if (n->nranks > 1 && lv[0].first != HPAR_GPU)
    return bail(fail(HPAR_E_INVALID, "%d ranks: the outermost nest level must bind the GPU level", n->nranks));

  // ---- geometry ----
  int64_t K = cfg->cluster_dim > 0 ? cfg->cluster_dim : 2;
  int64_t W = cfg->warps_per_cta > 0 ? cfg->warps_per_cta : 8;
  int64_t C = cfg->clusters > 0 ? cfg->clusters : 0;
  const int top = lv[0].first;
  if (top > HPAR_GPU && n->nranks != 1) return bail(fail(HPAR_E_INVALID, "nest without GPU level needs 1 rank"));
  if (top > HPAR_CLUSTER) {
    if (C > 1) return bail(fail(HPAR_E_INVALID, "nest without cluster level: clusters must be 1"));
    C = 1;
  }
  if (top > HPAR_CTA) K = 1;
  if (top > HPAR_WARP) W = 1;
  if (K < 1 || K > 16) return bail(fail(HPAR_E_INVALID, "cluster_dim %lld outside 1..16", (long long)K));
  if (W < 1 || W > 32) return bail(fail(HPAR_E_INVALID, "warps_per_cta %lld outside 1..32", (long long)W));
  int lane_w = 1;
  for (int a = 0; a < nlevels; ++a) {
    if (lv[a].width > 0) {
      if (32 % lv[a].width != 0)
        return bail(fail(HPAR_E_PARTITION, "nest level %d: width %d does not divide the lane level's num 32 (S:97)",
                         a, lv[a].width));
      lane_w = lv[a].width;
      n->lane_part = true;
    }
  }
  // fanouts fixing C
  for (int a = 0; a < nlevels; ++a) {
    const hpar_nest_level& L = lv[a];
    if (L.fanout == 0) continue;
    const bool inner_slice = a > 0 && lv[a - 1].width > 0;
    int64_t prod = 1;
    bool has_c = false;
    for (int hw = L.first; hw <= L.last; ++hw) {
      if (hw == HPAR_GPU) prod *= n->nranks;
      else if (hw == HPAR_CLUSTER) has_c = true;
      else if (hw == HPAR_CTA) prod *= K;
      else if (hw == HPAR_WARP) prod *= W;
      else if (hw == HPAR_LANE) {
        if (L.width > 0) prod *= 32 / L.width;
        else if (inner_slice) prod *= lane_w;
        else prod *= 32;
      }
    }
    if (has_c && C == 0) {
      if (L.fanout % prod != 0)
        return bail(fail(HPAR_E_INVALID, "nest level %d: fanout %lld not a multiple of %lld", a,
                         (long long)L.fanout, (long long)prod));
      C = L.fanout / prod;
    } else {
      if (has_c) prod *= C;
      if (prod != L.fanout)
        return bail(fail(HPAR_E_INVALID, "nest level %d: fanout %lld does not match the geometry (%lld)", a,
                         (long long)L.fanout, (long long)prod));
    }
  }
  if (C == 0) {
    if (describe_only) {
      C = default_resident_clusters(*cfg->desc, (int)K, (int)W);
    } else {
      cudaDeviceProp p;
      cudaError_t e = cudaGetDeviceProperties(&p, cfg->device);
      if (e != cudaSuccess) return bail(fail(HPAR_E_CUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e)));
      // the co-resident clusters of the flat kernel for this (K, W): one wave
      C = hpar::flat_max_active_clusters((int)K, (int)W);
      if (C < 1) C = std::max<int64_t>(1, (int64_t)p.multiProcessorCount * hpar::flat_resident_ctas_per_sm((int)W) / K);
    }
  }
  n->G = n->nranks;
  n->C = C;
  n->K = K;
  n->W = W;
  n->lane_w = lane_w;
  n->radix[S_GPU] = n->nranks;
  n->radix[S_CLUSTER] = C;
  n->radix[S_CTA] = K;
  n->radix[S_WARP] = W;
  n->radix[S_LANE] = 32 / lane_w;
  n->radix[S_LANE_IN] = lane_w;
  if (top > HPAR_GPU) n->radix[S_GPU] = 1;

  // ---- resolve every nest level: slots, T, flags; capability checks ----
  n->gpu_level = -1;
  int64_t max_dyn_slots = 0;
  for (int a = 0; a < nlevels; ++a) {
    const hpar_nest_level& L = lv[a];
    const bool inner_slice = a > 0 && lv[a - 1].width > 0;
    DevLevel& D = n->lv[a];
    memset(&D, 0, sizeof(D));
    D.sched = L.schedule;
    D.loop = L.loop;
    D.chunk = L.chunk;
    D.sfirst = slot_first(L.first, inner_slice);
    D.slast = slot_last(L.last, L.width > 0);
    int64_t T = 1;
    for (int s = D.sfirst; s <= D.slast; ++s) T *= n->radix[s];
    D.T = T;
    uint32_t fl = 0xFFFFFFFFu;
    for (int hw = L.first; hw <= L.last; ++hw) fl &= level_props(hw);  // collapse: intersection
    n->props[a] = fl;
    if (D.sfirst == S_GPU) {
      n->gpu_level = a;
      if (n->nranks > 1 && (L.schedule != HPAR_SCHED_STATIC || L.loop != 0))
        return bail(fail(HPAR_E_UNSUPPORTED,
                         "nest level %d binds the GPU level: only static (block) over loop 0 across GPUs "
                         "(shards must be contiguous; P:72 no cross-GPU dynamic)", a));
    }
    if (L.schedule == HPAR_SCHED_DYNAMIC) {
      if (!(fl & HPAR_P_DYNAMIC))
        return bail(fail(HPAR_E_CAPABILITY,
                         "nest level %d (%s..%s): dynamic schedule on a level without the `dynamic` property "
                         "(S:338, Table 2)", a, kLevelNames[L.first], kLevelNames[L.last]));
      int64_t slots = 1;
      for (int s = S_CLUSTER; s < D.sfirst; ++s) slots *= n->radix[s];
      max_dyn_slots = std::max(max_dyn_slots, slots);
    }
  }

  // ---- workspace ----
  n->dyn_slots = max_dyn_slots;
  if (!describe_only) {
    cudaError_t e = cudaSetDevice(cfg->device);
    if (e == cudaSuccess) e = cudaMalloc(&n->grid_ticket, 64);
    if (e == cudaSuccess) e = cudaMemset(n->grid_ticket, 0, 64);
    n->cluster_partials_bytes = (size_t)C * 256 * 8;
    if (e == cudaSuccess) e = cudaMalloc(&n->cluster_partials, n->cluster_partials_bytes);
    if (e == cudaSuccess && max_dyn_slots > 0) {
      e = cudaMalloc(&n->dyn_tickets, (size_t)max_dyn_slots * 8);
      if (e == cudaSuccess) e = cudaMemset(n->dyn_tickets, 0, (size_t)max_dyn_slots * 8);
    }
    if (e == cudaSuccess) e = cudaMalloc(&n->error_flag, 64);
    if (e == cudaSuccess) e = cudaMemset(n->error_flag, 0, 64);
    if (e == cudaSuccess) e = cudaMalloc(&n->barrier_word, 64);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      hpar_nest_destroy(n);
      return fail(e == cudaErrorMemoryAllocation ? HPAR_E_NOMEM : HPAR_E_CUDA, "workspace: %s",
                  cudaGetErrorString(e));
    }
  }
  // ---- fused node level (NEXT f1): collective over the communicator ----
  if (cfg->flags & HPAR_NEST_NODE_ALWAYS) {
    if (!n->comm) {
      hpar_nest_destroy(n);
      return fail(HPAR_E_INVALID, "HPAR_NEST_NODE_ALWAYS needs an NCCL communicator");
    }
    n->node_always = true;
  }
  if (cfg->flags & HPAR_NEST_NODE_FUSED) {
    hpar_status s = node_fused_setup(n);
    if (s) {
      hpar_nest_destroy(n);
      return s;
    }
  }
  *out = n;
  return ok();
}

extern "C" hpar_status hpar_nest_destroy(hpar_nest_t n) {
  if (!n) return ok();
  if (n->device >= 0 && n->comm) {  // fused node level: collective teardown
    cudaSetDevice(n->device);
    cudaDeviceSynchronize();
    ncclComm_t comm = (ncclComm_t)n->comm;
    if (n->node_dc_made && g_nccl.devCommDestroy) g_nccl.devCommDestroy(comm, &n->node_dc);
    if (n->node_win && g_nccl.winDeregister) g_nccl.winDeregister(comm, n->node_win);
    if (n->node_sym && g_nccl.memFree) g_nccl.memFree(n->node_sym);
    cudaFree(n->node_dc_dev);
  }
  if (n->device >= 0) {
    cudaSetDevice(n->device);
    cudaFree(n->grid_ticket);
    cudaFree(n->cluster_partials);
    cudaFree(n->dyn_tickets);
    cudaFree(n->error_flag);
    cudaFree(n->barrier_word);
    cudaFree(n->seg_ws);
    cudaFree(n->seg_off_ws);
    cudaFree(n->sr_ws);
    cudaFree(n->gather_buf);
    cudaFree(n->halo_buf);
  }
  delete n;
  return ok();
}

extern "C" hpar_status hpar_nest_info(hpar_nest_t n, hpar_nest_info_t* out) {
  if (!n || !out) return fail(HPAR_E_INVALID, "hpar_nest_info: NULL argument");
  memset(out, 0, sizeof(*out));
  out->G = n->G;
  out->C = n->C;
  out->K = n->K;
  out->W = n->W;
  out->rank = n->rank;
  out->nlevels = n->nlev;
  out->lane_width = n->lane_part ? n->lane_w : 0;
  int64_t total = 1;
  for (int a = 0; a < n->nlev; ++a) {
    out->tasks[a] = n->lv[a].T;
    total *= n->lv[a].T;
    out->total[a] = total;
    out->props[a] = n->props[a];
  }
  out->threads_per_gpu = n->C * n->K * n->W * 32;
  return ok();
}

extern "C" const char* hpar_last_kernel(hpar_nest_t n) { return n ? n->last_kernel.c_str() : ""; }

namespace {
// rank g's contiguous range of the outermost loop under the GPU-holding
// level's static block schedule (§8(a) A2).
void shard_of(const hpar_nest* n, int64_t n0, int32_t rank, int64_t* begin, int64_t* count) {
  if (n->gpu_level < 0 || n->nranks == 1) {
    *begin = 0;
    *count = n0;
    return;
  }
  const DevLevel& D = n->lv[n->gpu_level];
  const int64_t P = D.T / n->nranks;  // tasks of that level per GPU
  const int64_t q = n0 / D.T, r = n0 % D.T;
  auto start = [&](int64_t t) { return t * q + std::min(t, r); };
  *begin = start((int64_t)rank * P);
  *count = start((int64_t)(rank + 1) * P) - *begin;
}
}  // namespace

extern "C" hpar_status hpar_shard_range_csr(const int64_t* off, int64_t rows, int32_t nranks, int32_t rank,
                                            int64_t* begin, int64_t* count) {
  if (!off || rows < 0 || nranks < 1 || rank < 0 || rank >= nranks || !begin || !count)
    return fail(HPAR_E_INVALID, "hpar_shard_range_csr: bad arguments");
  const int64_t nnz = off[rows];
  auto bound = [&](int32_t g) -> int64_t {  // first row whose start >= ceil(g * nnz / nranks)
    if (g <= 0) return 0;
    if (g >= nranks) return rows;
    const int64_t target = (int64_t)(((__int128)g * nnz + nranks - 1) / nranks);
    return (int64_t)(std::lower_bound(off, off + rows, target) - off);
  };
  const int64_t b = bound(rank), e = bound(rank + 1);
  *begin = b;
  *count = e > b ? e - b : 0;
  return ok();
}

extern "C" hpar_status hpar_shard_range(hpar_nest_t n, int64_t n0, int32_t rank, int64_t* begin, int64_t* count) {
  if (!n || !begin || !count) return fail(HPAR_E_INVALID, "hpar_shard_range: NULL argument");
  if (rank < 0 || rank >= n->nranks) return fail(HPAR_E_INVALID, "rank %d out of range", rank);
  if (n0 < 0) return fail(HPAR_E_INVALID, "n0 < 0");
  shard_of(n, n0, rank, begin, count);
  return ok();
}

// ------------------------------------------------------------ planner ----
namespace {
// maximal list length reaching nest level `upto` of loop `loop` (task 0 owns
// the most for every schedule; under a dynamic level a child sees <= chunk)
int64_t max_parent_len(const hpar_nest* n, int loop, int upto, int64_t extent) {
  int64_t len = extent;
  for (int a = 0; a < upto; ++a) {
    const DevLevel& D = n->lv[a];
    if (D.loop != loop) continue;
    if (D.sched == SCHED_STATIC) len = len / D.T + (len % D.T ? 1 : 0);
    else if (D.sched == SCHED_NONE) len = std::min<int64_t>(len, 1);
    else if (D.sched == SCHED_DYNAMIC) len = std::min(len, D.chunk);
    else {
      const int64_t nch = (len + D.chunk - 1) / D.chunk;
      const int64_t mine = nch > 0 ? (nch - 1) / D.T + 1 : 0;
      len = std::min(len, mine * D.chunk);
    }
  }
  return len;
}
size_t dtype_size(int dt) {
  switch (dt) {
    case HPAR_I32: case HPAR_F32: return 4;
    case HPAR_I64: case HPAR_F64: case HPAR_U64: return 8;
    case HPAR_U8: return 1;
  }
  return 0;
}
}  // namespace

extern "C" hpar_status hpar_parallel_for_reduce(hpar_nest_t n, const hpar_reduce_desc* d, void* stream_) {
  if (!n || !d) return fail(HPAR_E_INVALID, "hpar_parallel_for_reduce: NULL argument");
  cudaStream_t stream = (cudaStream_t)stream_;
  // ---- op / dtype ----
  const bool hist = d->op == HPAR_OP_HIST256;
  const bool affine = d->op == HPAR_OP_AFFINE;
  if (d->op < 0 || d->op > 4) return fail(HPAR_E_UNSUPPORTED, "unknown op %d", d->op);
  if (hist && d->in_dtype != HPAR_U8) return fail(HPAR_E_UNSUPPORTED, "hist256 needs uint8 input");
  if (affine && d->in_dtype != HPAR_I64) return fail(HPAR_E_UNSUPPORTED, "affine needs int64 input");
  if (!hist && !(d->in_dtype == HPAR_I32 || d->in_dtype == HPAR_I64 || d->in_dtype == HPAR_F32 ||
                 d->in_dtype == HPAR_F64))
    return fail(HPAR_E_UNSUPPORTED, "op %d: input dtype %d not supported (i32/i64/f32/f64)", d->op, d->in_dtype);
  if (d->nloops != 1 && d->nloops != 2) return fail(HPAR_E_INVALID, "nloops must be 1 or 2");
  if (d->n0 < 0 || d->n1 < 0) return fail(HPAR_E_INVALID, "negative loop extent");
  if (!d->out) return fail(HPAR_E_INVALID, "out is NULL");
  bool collapsed = false;  // a level bound to loop 2: the flattened (row, column) space
  for (int a = 0; a < n->nlev; ++a) {
    if (n->lv[a].loop == 2) {
      collapsed = true;
      if (d->nloops != 2)
        return fail(HPAR_E_INVALID, "nest level %d binds the collapsed loop 2 but the call has one loop", a);
    } else if (n->lv[a].loop >= d->nloops) {
      return fail(HPAR_E_INVALID, "nest level %d binds loop %d but the call has %d loop(s)", a, n->lv[a].loop,
                  d->nloops);
    }
  }
  const bool csr = d->nloops == 2 && d->offsets != nullptr;
  if (d->nloops == 2 && !csr && d->ld < d->n1) return fail(HPAR_E_INVALID, "ld < n1");
  if (d->keyed && d->nloops != 2) return fail(HPAR_E_INVALID, "keyed results need two loops");
  if (hist && d->keyed) return fail(HPAR_E_UNSUPPORTED, "keyed histograms");

  int64_t begin = 0, local = 0;
  shard_of(n, d->n0, n->rank, &begin, &local);
  bool empty_shard = false;
  if (d->local_n0 > 0 || d->local_n0 == HPAR_LOCAL_N0_EMPTY) {  // caller-sharded CSR rows (§8(e) C3)
    if (!d->offsets || !d->keyed || d->local_n0 > d->n0)
      return fail(HPAR_E_INVALID, "local_n0 is for keyed CSR calls (and <= n0)");
    local = d->local_n0 > 0 ? d->local_n0 : 0;
    empty_shard = local == 0;
  } else if (d->local_n0 < 0) {
    return fail(HPAR_E_INVALID, "local_n0 %lld: > 0 rows, 0 = unset, or HPAR_LOCAL_N0_EMPTY", (long long)d->local_n0);
  }
  if (local > 0 && !d->in) return fail(HPAR_E_INVALID, "in is NULL");

  // ---- schedule(none) overflow (diagnose, never UB) ----
  for (int a = 0; a < n->nlev; ++a) {
    if (n->lv[a].sched != SCHED_NONE) continue;
    const int loop = n->lv[a].loop;
    if (loop == 2) return fail(HPAR_E_UNSUPPORTED, "nest level %d: schedule(none) over the collapsed loop", a);
    int64_t extent = loop == 0 ? d->n0 : d->n1;
    if (loop == 1 && csr) {
      if (d->max_inner <= 0)
        return fail(HPAR_E_INVALID, "nest level %d: schedule(none) over CSR rows needs desc->max_inner", a);
      extent = d->max_inner;
    }
    if (d->nloops == 1 && loop == 0) extent = d->n0;
    const int64_t len = max_parent_len(n, loop, a, extent);
    if (len > n->lv[a].T)
      return fail(HPAR_E_SCHEDULE,
                  "nest level %d: schedule(none) with %lld iterations for %lld tasks (P:251 'more logical "
                  "iterations than tasks')", a, (long long)len, (long long)n->lv[a].T);
  }

  // ---- build the kernel arguments ----
  NestArgs A;
  memset(&A, 0, sizeof(A));
  A.nlev = n->nlev;
  A.rank = n->rank;
  for (int s = 0; s < S_NSLOTS; ++s) A.radix[s] = n->radix[s];
  A.lane_w = n->lane_w;
  A.K = (int32_t)n->K;
  A.C = n->C;
  A.threads_per_gpu = n->C * n->K * n->W * 32;
  for (int a = 0; a < n->nlev; ++a) A.lv[a] = n->lv[a];
  A.op = d->op;
  A.in_dtype = d->in_dtype;
  A.nloops = d->nloops;
  A.keyed = d->keyed;
  A.verify = d->verify;
  A.in = d->in;
  A.n1 = d->n1;
  A.ld = d->ld ? d->ld : d->n1;
  A.offsets = d->offsets;
  // CSR: the fused CSR kernels need the value count (nnz = offsets[n0_local]);
  // hpar.h lets a caller pass n1 = 0 for CSR, so read it from the device then
  // (8 bytes and one host synchronisation; inside graph capture that is not
  // possible: the caller passes n1 = nnz there)
  if (csr && d->n1 == 0 && local > 0) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(stream, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(HPAR_E_INVALID, "CSR call inside graph capture with n1 = 0: pass desc->n1 = offsets[n0_local]");
    int64_t last = 0;
    CUDA_TRY(cudaMemcpyAsync(&last, d->offsets + local, 8, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (last < 0) return fail(HPAR_E_INVALID, "CSR offsets[n0_local] = %lld < 0", (long long)last);
    A.n1 = last;
  }
  A.out = d->out;
  for (int a = 0; a < HPAR_MAX_NEST; ++a) A.partials[a] = d->level_partials[a];
  A.owner = d->coverage_owner;
  A.count = d->coverage_count;
  A.fp = (unsigned long long*)d->fingerprint;
  A.global_begin = d->global_begin;
  A.grid_ticket = n->grid_ticket;
  A.cluster_partials = n->cluster_partials;
  A.error_flag = n->error_flag;
  A.max_inner = d->max_inner;
  A.dyn_tickets = n->dyn_tickets;
  A.dyn_slots = n->dyn_slots;
  A.dyn_level = -1;
  const bool node_in_kernel = n->node_fused && !d->keyed;
  if (node_in_kernel) {
    A.node_dc = n->node_dc_dev;
    A.node_win = n->node_win;
    A.node_parity = (int32_t)(n->node_calls & 1);  // advanced only once the launch succeeded
    A.node_slot = (int32_t)kNodeSlot;
  }

  if ((d->verify & HPAR_VERIFY_COVERAGE) && (!d->coverage_owner || !d->coverage_count))
    return fail(HPAR_E_INVALID, "verify coverage needs coverage_owner and coverage_count");
  if ((d->verify & HPAR_VERIFY_FINGERPRINT) && !d->fingerprint)
    return fail(HPAR_E_INVALID, "verify fingerprint needs fingerprint[3]");

  // The device enumerates GLOBAL loop-0 positions with the full task ids
  // (GPU digit = rank); `in` / offsets / out are the rank's shard, so the
  // GPU-holding level is applied here: it is replaced by the rank's own list
  // [0, local) (static block => contiguous shard, §8(a) A2).
  A.n0 = local;
  if (n->gpu_level >= 0 && n->nranks > 1) {
    // the GPU-holding level keeps its sub-GPU digits: re-express it as a
    // static level over the tasks of this GPU only
    DevLevel& D = A.lv[n->gpu_level];
    D.sfirst = S_CLUSTER <= D.slast ? S_CLUSTER : S_GPU;
    if (D.slast == S_GPU) {
      D.T = 1;
    } else {
      D.T = D.T / n->nranks;
    }
    A.radix[S_GPU] = 1;
  }
  if (n->gpu_level >= 0 && A.lv[n->gpu_level].slast == S_GPU) A.lv[n->gpu_level].host_applied = 1;

  // keyed: loop-0 levels must be a prefix; the row owner is the last of them
  if (d->keyed) {
    int k = 0;
    while (k < n->nlev && n->lv[k].loop == 0) ++k;
    for (int a = k; a < n->nlev; ++a)
      if (n->lv[a].loop == 0)
        return fail(HPAR_E_INVALID, "keyed results: the levels bound to loop 0 must be the outermost ones");
    if (k == 0) return fail(HPAR_E_UNSUPPORTED, "keyed results need loop 0 bound to an outer level");
    A.first_inner = k;
    A.owner_slot = n->lv[k - 1].slast;
    if (A.owner_slot == S_GPU && k < n->nlev)
      return fail(HPAR_E_CAPABILITY,
                  "keyed results owned by the GPU level would combine across clusters, which have no "
                  "barrier (P:178); bind loop 0 down to the cluster level or below");
    const bool fin = d->in_dtype == HPAR_F32 || d->in_dtype == HPAR_F64;
    if (fin && d->out_dtype != HPAR_F32 && d->out_dtype != HPAR_F64)
      return fail(HPAR_E_INVALID, "keyed fp results: out_dtype must be f32 or f64");
    if (affine) {
      if (d->out_dtype != HPAR_U64) return fail(HPAR_E_INVALID, "keyed affine results: out_dtype must be u64 (2 per row)");
    } else if (!fin && d->out_dtype != HPAR_I64) {
      return fail(HPAR_E_INVALID, "keyed int results: out_dtype must be i64");
    }
    A.out_dtype = d->out_dtype;
  } else {
    A.out_dtype = (d->in_dtype == HPAR_F32 || d->in_dtype == HPAR_F64) ? HPAR_F64 : HPAR_I64;
  }

  if (empty_shard) {  // nothing to reduce on this rank; keyed results need no node level
    n->last_kernel = "none (empty shard)";
    return ok();
  }
  // ---- kernel choice: fused specialisation if the nest matches its shape ----
  const char* why = nullptr;
  const char* name = "generic";
  cudaError_t e = cudaSuccess;
  if (n->device < 0) return fail(HPAR_E_INVALID, "describe-only nest: validated, cannot execute");
  CUDA_TRY(cudaSetDevice(n->device));
  if (hist) {
    if (!hist_matches(A, &why))
      return fail(HPAR_E_UNSUPPORTED, "hist256: nest shape not supported by the histogram kernel: %s", why);
    e = launch_hist(A, (int)n->W, stream, &name);
  } else if (flat_matches(A, &why)) {
    e = launch_flat(A, (int)n->W, stream, &name);
  } else if (rowwise_matches(A, &why)) {
    e = launch_rowwise(A, (int)n->W, stream, &name);
  } else if (segmented_matches(A, &why)) {
    // CSR: n1 = nonzeros of this rank's shard (local offsets start at 0)
    // The workspace layout (queue, partials, tickets) is a function of the
    // nnz it was built for, never of the current call's: a later call with
    // fewer nonzeros keeps the same offsets, so the self-reset tickets and the
    // all-ones empty queue slots stay where the kernel looks for them.
    const int64_t nnz = A.n1;
    {
      bool span_ok = true, synced = false;
      // (error_flag's 64 device bytes serve as the check's scratch word)
      CUDA_TRY(segmented_span_ok(A, (unsigned long long*)n->error_flag, stream, &span_ok, &synced));
      if (!span_ok)
        return fail(HPAR_E_UNSUPPORTED,
                    synced ? "segmented CSR: a block of 256 rows spans >= 2^31 nonzeros (32-bit positions)"
                           : "segmented CSR: >= 2^31 nonzeros per rank while capturing a graph: the block-span "
                             "check needs a host sync; pass desc->max_inner with max_inner * 256 < 2^31");
    }
    if (nnz > n->seg_ws_nnz) {
      const size_t need = segmented_ws_bytes(nnz);
      cudaFree(n->seg_ws);
      n->seg_ws = nullptr;
      n->seg_ws_bytes = 0;
      n->seg_ws_nnz = -1;
      cudaError_t ae = cudaMalloc(&n->seg_ws, need);
      if (ae != cudaSuccess) return fail(HPAR_E_NOMEM, "segmented workspace (%zu B): %s", need, cudaGetErrorString(ae));
      size_t qoff, qlen;
      segmented_ws_qrow(nnz, &qoff, &qlen);
      CUDA_TRY(cudaMemsetAsync(n->seg_ws, 0, need, stream));
      CUDA_TRY(cudaMemsetAsync((char*)n->seg_ws + qoff, 0xFF, qlen, stream));  // empty queue slots = -1
      n->seg_ws_bytes = need;
      n->seg_ws_nnz = nnz;
    }
    if (((uintptr_t)A.in & 15) && A.n0 + 1 > n->seg_off_rows) {
      cudaFree(n->seg_off_ws);
      n->seg_off_ws = nullptr;
      n->seg_off_rows = 0;
      cudaError_t ae = cudaMalloc(&n->seg_off_ws, (size_t)(A.n0 + 1) * 8);
      if (ae != cudaSuccess) return fail(HPAR_E_NOMEM, "segmented offsets copy: %s", cudaGetErrorString(ae));
      n->seg_off_rows = A.n0 + 1;
    }
    e = launch_segmented(A, n->seg_ws, n->seg_ws_nnz, n->seg_off_ws, stream, &name);
  } else if (segrows_matches(A, &why)) {
    // CSR rows for the other ops / dtypes: the same nest, a segmented
    // reduction per window (kernel_segrows.cu); workspace keyed on its nnz
    const int64_t nnz = A.n1;
    if (nnz > n->sr_ws_nnz) {
      const size_t need = segrows_ws_bytes(nnz);
      cudaFree(n->sr_ws);
      n->sr_ws = nullptr;
      n->sr_ws_nnz = -1;
      cudaError_t ae = cudaMalloc(&n->sr_ws, need);
      if (ae != cudaSuccess) return fail(HPAR_E_NOMEM, "CSR rows workspace (%zu B): %s", need, cudaGetErrorString(ae));
      CUDA_TRY(cudaMemsetAsync(n->sr_ws, 0, need, stream));
      n->sr_ws_nnz = nnz;
    }
    e = launch_segrows(A, n->sr_ws, n->sr_ws_nnz, stream, &name);
  } else if (teams_matches(A, &why)) {
    e = launch_teams(A, (int)n->W, stream, &name);
  } else if (collapsed) {
    return fail(HPAR_E_UNSUPPORTED, "collapsed loop 2: only the CSR segmented nest shape is implemented (%s)", why);
  } else {
    // generic interpreter: at most one dynamic level, on loop 0
    int ndyn = 0;
    for (int a = 0; a < n->nlev; ++a) {
      if (n->lv[a].sched != SCHED_DYNAMIC) continue;
      ++ndyn;
      if (n->lv[a].loop != 0 && d->nloops == 2)
        return fail(HPAR_E_UNSUPPORTED, "nest level %d: dynamic schedule on the inner loop (generic kernel)", a);
      A.dyn_level = a;
    }
    if (ndyn > 1) return fail(HPAR_E_UNSUPPORTED, "generic kernel: at most one dynamic level");
    if (A.dyn_level >= 0) {
      for (int a = 0; a < A.dyn_level; ++a)
        if (n->lv[a].loop == 0 && n->lv[a].sched == SCHED_DYNAMIC)
          return fail(HPAR_E_UNSUPPORTED, "generic kernel: nested dynamic levels");
    }
    e = launch_generic(A, (int)(n->W * 32), stream);
  }
  if (e != cudaSuccess) return fail(HPAR_E_CUDA, "launch %s: %s", name, cudaGetErrorString(e));
  n->last_kernel = name;
  if (node_in_kernel) ++n->node_calls;  // every rank advances the slot parity in step

  // ---- node level: one allreduce over NVLink (§8(a) A9) ----
  if (node_in_kernel) {
    // done inside the kernel (f1)
  } else if (!d->keyed && (n->nranks > 1 || n->node_always) && affine) {
    // an ordered op cannot be an NCCL reduction: gather the per-rank results
    // in rank order (= the GPU level's static-block order) and fold them
    hpar_status s = need_nccl();
    if (s) return s;
    if (!g_nccl.allGather) return fail(HPAR_E_NCCL, "ncclAllGather unavailable");
    if (!n->gather_buf) {
      cudaError_t ae = cudaMalloc(&n->gather_buf, (size_t)n->nranks * 16);
      if (ae != cudaSuccess) return fail(HPAR_E_NOMEM, "gather buffer: %s", cudaGetErrorString(ae));
    }
    ncclResult_t r = g_nccl.allGather(d->out, n->gather_buf, 2, ncclUint64, (ncclComm_t)n->comm, stream);
    if (r != ncclSuccess) return nccl_fail(r, (ncclComm_t)n->comm, "ncclAllGather");
    e = launch_affine_rank_fold(n->gather_buf, n->nranks, d->out, stream);
    if (e != cudaSuccess) return fail(HPAR_E_CUDA, "rank fold: %s", cudaGetErrorString(e));
  } else if (!d->keyed && (n->nranks > 1 || n->node_always)) {
    hpar_status s = need_nccl();
    if (s) return s;
    ncclDataType_t t;
    ncclRedOp_t op = d->op == HPAR_OP_MIN ? ncclMin : d->op == HPAR_OP_MAX ? ncclMax : ncclSum;
    size_t cnt = 1;
    if (hist) {
      t = ncclUint64;
      cnt = 256;
    } else {
      t = (d->in_dtype == HPAR_F32 || d->in_dtype == HPAR_F64) ? ncclFloat64 : ncclInt64;
    }
    ncclResult_t r = g_nccl.allReduce(d->out, d->out, cnt, t, op, (ncclComm_t)n->comm, stream);
    if (r != ncclSuccess) return nccl_fail(r, (ncclComm_t)n->comm, "ncclAllReduce");
  }
  (void)dtype_size;
  return ok();
}

// ----------------------------------------------------------- barriers ----
extern "C" hpar_status hpar_barrier(hpar_nest_t n, int32_t level, void* stream_) {
  if (!n) return fail(HPAR_E_INVALID, "hpar_barrier: NULL nest");
  if (level < HPAR_NODE || level > HPAR_LANE) return fail(HPAR_E_INVALID, "bad level %d", level);
  if (!(level_props(level) & HPAR_P_BARRIER) && level != HPAR_NODE)
    return fail(HPAR_E_CAPABILITY, "barrier on the %s level, which has no `barrier` property (S:348; P:178)",
                kLevelNames[level]);
  if (n->device < 0) return fail(HPAR_E_INVALID, "describe-only nest cannot execute");
  // node: one process per GPU, the node is the job; CTA / warp / lane: every
  // task of a call has finished (and its writes are visible) at the kernel
  // boundary, which stream order already puts between consecutive calls
  if (level != HPAR_GPU) return ok();
  if (!n->comm || (n->nranks == 1 && !n->node_always)) return ok();
  CUDA_TRY(cudaSetDevice(n->device));
  hpar_status s = need_nccl();
  if (s) return s;
  ncclResult_t r = g_nccl.allReduce(n->barrier_word, n->barrier_word, 1, ncclInt32, ncclSum, (ncclComm_t)n->comm,
                                    (cudaStream_t)stream_);
  if (r != ncclSuccess) return nccl_fail(r, (ncclComm_t)n->comm, "ncclAllReduce (barrier)");
  return ok();
}

extern "C" hpar_status hpar_barrier_probe(hpar_nest_t n, int32_t level, int32_t rounds, uint32_t flags,
                                          uint32_t delay_ns, uint64_t* folds, void* stream_) {
  if (!n) return fail(HPAR_E_INVALID, "hpar_barrier_probe: NULL nest");
  if (level != HPAR_CTA && level != HPAR_WARP && level != HPAR_LANE)
    return fail(level == HPAR_CLUSTER ? HPAR_E_CAPABILITY : HPAR_E_INVALID,
                "barrier probe: in-kernel levels only (cta, warp, lane); %s",
                level == HPAR_CLUSTER ? "clusters have no barrier (P:178)" : "bad level");
  if (rounds < 1 || !folds) return fail(HPAR_E_INVALID, "barrier probe: rounds >= 1 and folds[] required");
  if (flags & ~(uint32_t)HPAR_PROBE_NO_BARRIER) return fail(HPAR_E_INVALID, "barrier probe: unknown flags");
  if (n->device < 0) return fail(HPAR_E_INVALID, "describe-only nest cannot execute");
  CUDA_TRY(cudaSetDevice(n->device));
  cudaError_t e = launch_probe(level, n->C, (int)n->K, (int)n->W, rounds, (flags & HPAR_PROBE_NO_BARRIER) ? 1 : 0,
                               delay_ns, (unsigned long long*)folds, (cudaStream_t)stream_);
  if (e != cudaSuccess) return fail(HPAR_E_CUDA, "barrier probe: %s", cudaGetErrorString(e));
  return ok();
}

// ------------------------------------------- property-based selection ----
// §3.2-3.3; SPEC level_resolver with the selection
// policy of S:283: each construct takes the longest feasible run of the
// remaining levels, starting at the first one.
namespace {
uint32_t run_flags(const hpar_level_info* t, int first, int last) {
  uint32_t f = 0xFFFFFFFFu;
  for (int l = first; l <= last; ++l) f &= t[l].props;
  return f;
}
// can constructs [k, n) be assigned to the levels [s, HPAR_LANE]?  fills ends[]
bool assign(const hpar_sync_construct* c, int n, int k, int s, const hpar_level_info* t, int* ends) {
  if (k == n) return s > HPAR_LANE;  // every level used, nothing left over
  if (s > HPAR_LANE) return false;
  // without a reserve: the longest run first (maximal fan-out);
  // with a reserve: the shortest run first, i.e. the inner constructs get every
  // level that matches the reserve ("uses all levels except the ones that
  // match the reserve clause argument")
  const bool res = c[k].reserve != 0;
  for (int i = 0; i <= HPAR_LANE - s; ++i) {
    const int e = res ? s + i : HPAR_LANE - i;
    const uint32_t f = run_flags(t, s, e);
    if ((f & c[k].demand) != c[k].demand) continue;
    if (c[k].reserve && e < HPAR_LANE) {
      const uint32_t rest = run_flags(t, e + 1, HPAR_LANE);
      if ((rest & c[k].reserve) != c[k].reserve) continue;
    } else if (c[k].reserve && e == HPAR_LANE) {
      continue;  // a reserve needs levels left over
    }
    if (assign(c, n, k + 1, e + 1, t, ends)) {
      ends[k] = e;
      return true;
    }
  }
  return false;
}
}  // namespace

extern "C" hpar_status hpar_nest_resolve(const hpar_sync_construct* c, int32_t n, const hpar_level_info* table,
                                         hpar_nest_level* out) {
  if (!c || !table || !out || n < 1 || n > HPAR_MAX_NEST)
    return fail(HPAR_E_INVALID, "hpar_nest_resolve: bad arguments");
  // the outermost construct starts at the coarsest level from which the
  // demands are satisfiable; levels above it run a single task
  int ends[HPAR_MAX_NEST];
  int s0 = HPAR_GPU;
  while (s0 <= HPAR_LANE && !assign(c, n, 0, s0, table, ends)) ++s0;
  if (s0 > HPAR_LANE)
    return fail(HPAR_E_CAPABILITY,
                "no assignment of the %d construct(s) to contiguous level runs satisfies their sync demands "
                "(S:229 unsatisfiable sync demand)", n);
  int s = s0;
  for (int k = 0; k < n; ++k) {
    memset(&out[k], 0, sizeof(out[k]));
    out[k].first = s;
    out[k].last = ends[k];
    out[k].schedule = c[k].schedule;
    out[k].loop = c[k].loop;
    out[k].chunk = c[k].chunk;
    s = ends[k] + 1;
  }
  return ok();
}

extern "C" hpar_status hpar_level_alias(const char* name, int32_t* first, int32_t* last) {
  if (!name || !first || !last) return fail(HPAR_E_INVALID, "hpar_level_alias: NULL argument");
  struct { const char* n; int f, l; } tab[] = {
      {"devices", HPAR_GPU, HPAR_GPU},   {"gpu", HPAR_GPU, HPAR_GPU},         {"teams", HPAR_CLUSTER, HPAR_CTA},
      {"cluster", HPAR_CLUSTER, HPAR_CLUSTER}, {"cta", HPAR_CTA, HPAR_CTA},   {"threads", HPAR_WARP, HPAR_LANE},
      {"warp", HPAR_WARP, HPAR_WARP},    {"lane", HPAR_LANE, HPAR_LANE},      {"simd", HPAR_LANE, HPAR_LANE},
      {"node", HPAR_NODE, HPAR_NODE}};
  for (auto& e : tab)
    if (strcmp(e.n, name) == 0) {
      *first = e.f;
      *last = e.l;
      return ok();
    }
  return fail(HPAR_E_INVALID, "unknown level or alias '%s'", name);
}

// ------------------------------------------- ghost maps (§4; NEXT f3) ----
namespace {
bool rect_empty(const hpar_rect& r) { return r.len[0] <= 0 || r.len[1] <= 0; }
hpar_rect rect_and(const hpar_rect& a, const hpar_rect& b) {
  hpar_rect r;
  for (int k = 0; k < 2; ++k) {
    const int64_t lo = std::max(a.off[k], b.off[k]);
    const int64_t hi = std::min(a.off[k] + a.len[k], b.off[k] + b.len[k]);
    r.off[k] = lo;
    r.len[k] = hi > lo ? hi - lo : 0;
  }
  return r;
}
bool rect_inside(const hpar_rect& in, const hpar_rect& out) {
  for (int k = 0; k < 2; ++k)
    if (in.off[k] < out.off[k] || in.off[k] + in.len[k] > out.off[k] + out.len[k]) return false;
  return true;
}
// offset = mul * coord + add, coord = (d / grid_cols, d % grid_cols)
void sections_of(const hpar_map_spec* m, int32_t d, hpar_rect* to, hpar_rect* from) {
  const int64_t coord[2] = {d / m->grid_cols, d % m->grid_cols};
  for (int k = 0; k < 2; ++k) {
    to->off[k] = m->to[k].mul * coord[k] + m->to[k].add;
    to->len[k] = m->to[k].len;
    from->off[k] = m->from[k].mul * coord[k] + m->from[k].add;
    from->len[k] = m->from[k].len;
  }
}
hpar_status spec_ok(const hpar_map_spec* m) {
  if (!m) return fail(HPAR_E_INVALID, "map spec is NULL");
  if (m->siblings < 1 || m->grid_cols < 1) return fail(HPAR_E_INVALID, "map: siblings and grid_cols must be >= 1");
  if (m->extent[0] < 1 || m->extent[1] < 1) return fail(HPAR_E_INVALID, "map: empty parent array");
  return HPAR_OK;
}
}  // namespace

extern "C" hpar_status hpar_map_sections(const hpar_map_spec* m, int32_t d, hpar_rect* to, hpar_rect* from) {
  if (hpar_status st = spec_ok(m)) return st;
  if (d < 0 || d >= m->siblings || !to || !from) return fail(HPAR_E_INVALID, "map: sibling %d out of range", d);
  sections_of(m, d, to, from);
  return ok();
}

extern "C" hpar_status hpar_map_validate(const hpar_map_spec* m, int64_t where[4]) {
  if (hpar_status st = spec_ok(m)) return st;
  const hpar_rect whole = {{0, 0}, {m->extent[0], m->extent[1]}};
  for (int32_t d = 0; d < m->siblings; ++d) {
    hpar_rect to, fr;
    sections_of(m, d, &to, &fr);
    if (rect_empty(to) || rect_empty(fr)) return fail(HPAR_E_INVALID, "map: sibling %d has a non-positive length", d);
    if (!rect_inside(to, whole)) return fail(HPAR_E_INVALID, "map: sibling %d to-section outside the array", d);
    if (!rect_inside(fr, whole)) return fail(HPAR_E_INVALID, "map: sibling %d from-section outside the array", d);
    if (!rect_inside(fr, to)) return fail(HPAR_E_INVALID, "map: sibling %d from-section not inside its to-section", d);
  }
  // the first shared element in row-major order (ties: lowest pair)
  bool found = false;
  int64_t best[4] = {0, 0, 0, 0};
  for (int32_t a = 0; a < m->siblings; ++a) {
    hpar_rect ta, fa;
    sections_of(m, a, &ta, &fa);
    for (int32_t b = a + 1; b < m->siblings; ++b) {
      hpar_rect tb, fb;
      sections_of(m, b, &tb, &fb);
      const hpar_rect x = rect_and(fa, fb);
      if (rect_empty(x)) continue;
      const int64_t cand[4] = {x.off[0], x.off[1], a, b};
      if (!found || std::lexicographical_compare(cand, cand + 4, best, best + 4)) {
        std::copy(cand, cand + 4, best);
        found = true;
      }
    }
  }
  if (found) {
    if (where) std::copy(best, best + 4, where);
    return fail(HPAR_E_INVALID, "map: element (%lld, %lld) is written back by siblings %lld and %lld (P:383)",
                (long long)best[0], (long long)best[1], (long long)best[2], (long long)best[3]);
  }
  return ok();
}

extern "C" hpar_status hpar_map_exchange_plan(const hpar_map_spec* m, int32_t d, hpar_halo* out, int32_t cap,
                                              int32_t* n) {
  if (hpar_status st = spec_ok(m)) return st;
  if (d < 0 || d >= m->siblings || !n || (cap > 0 && !out)) return fail(HPAR_E_INVALID, "map plan: bad arguments");
  hpar_rect tod, frd;
  sections_of(m, d, &tod, &frd);
  int32_t k = 0;
  for (int32_t e = 0; e < m->siblings; ++e) {
    if (e == d) continue;
    hpar_rect toe, fre;
    sections_of(m, e, &toe, &fre);
    const hpar_rect rr[2] = {rect_and(tod, fre), rect_and(toe, frd)};
    for (int s = 0; s < 2; ++s) {
      if (rect_empty(rr[s])) continue;
      if (k < cap) out[k] = hpar_halo{e, s, rr[s]};
      ++k;
    }
  }
  *n = k;
  return ok();
}

namespace {
hpar_status check_stencil(const hpar_stencil_desc* d) {
  if (!d || !d->in || !d->out) return fail(HPAR_E_INVALID, "stencil: NULL descriptor or buffer");
  if (rect_empty(d->to) || rect_empty(d->from)) return fail(HPAR_E_INVALID, "stencil: empty section");
  if (!rect_inside(d->from, d->to)) return fail(HPAR_E_INVALID, "stencil: from-section not inside the to-section");
  const hpar_rect whole = {{0, 0}, {d->extent[0], d->extent[1]}};
  if (!rect_inside(d->to, whole)) return fail(HPAR_E_INVALID, "stencil: to-section outside the array");
  if (d->ld < d->to.len[1] || d->ld % 4 != 0)
    return fail(HPAR_E_INVALID, "stencil: ld must be >= the to-section's columns and a multiple of 4");
  if (((uintptr_t)d->in & 15) || ((uintptr_t)d->out & 15))
    return fail(HPAR_E_INVALID, "stencil: buffers must be 16-byte aligned");
  if (d->in == d->out) return fail(HPAR_E_INVALID, "stencil: in and out must differ (Jacobi step)");
  // every non-boundary from cell needs its 4 neighbours inside `to`
  for (int k = 0; k < 2; ++k) {
    const int64_t lo = d->from.off[k], hi = d->from.off[k] + d->from.len[k] - 1;
    if (lo > 0 && lo - 1 < d->to.off[k])
      return fail(HPAR_E_INVALID, "stencil: ghost %s %lld not in the to-section", k ? "col" : "row", (long long)(lo - 1));
    if (hi < d->extent[k] - 1 && hi + 1 >= d->to.off[k] + d->to.len[k])
      return fail(HPAR_E_INVALID, "stencil: ghost %s %lld not in the to-section", k ? "col" : "row", (long long)(hi + 1));
  }
  return HPAR_OK;
}
// 2-D copy of global rectangle r between two buffers holding sections dto / sto
cudaError_t copy_rect(float* dst, int64_t dld, const hpar_rect& dto, const float* src, int64_t sld,
                      const hpar_rect& sto, const hpar_rect& r, cudaStream_t s) {
  float* dp = dst + (r.off[0] - dto.off[0]) * dld + (r.off[1] - dto.off[1]);
  const float* sp = src + (r.off[0] - sto.off[0]) * sld + (r.off[1] - sto.off[1]);
  return cudaMemcpy2DAsync(dp, (size_t)dld * 4, sp, (size_t)sld * 4, (size_t)r.len[1] * 4, (size_t)r.len[0],
                           cudaMemcpyDeviceToDevice, s);
}
}  // namespace

extern "C" hpar_status hpar_stencil5(hpar_nest_t n, const hpar_stencil_desc* d, void* stream_) {
  if (!n) return fail(HPAR_E_INVALID, "stencil: nest is NULL");
  if (hpar_status st = check_stencil(d)) return st;
  CUDA_TRY(cudaSetDevice(n->device));
  int sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, n->device));
  const char* why = "";
  const cudaError_t e = launch_stencil5(*d, n->device, sms, (cudaStream_t)stream_, &why);
  if (e != cudaSuccess) return fail(HPAR_E_CUDA, "stencil5: %s (%s)", cudaGetErrorString(e), why);
  n->last_kernel = "stencil5_tma";
  return ok();
}

extern "C" hpar_status hpar_map_exchange_local(const hpar_map_spec* m, float* const* bufs, int64_t ld, void* stream_) {
  if (hpar_status st = spec_ok(m)) return st;
  if (!bufs || ld < m->to[1].len) return fail(HPAR_E_INVALID, "map exchange: bad buffers or pitch");
  const cudaStream_t s = (cudaStream_t)stream_;
  for (int32_t d = 0; d < m->siblings; ++d) {
    hpar_rect tod, frd;
    sections_of(m, d, &tod, &frd);
    for (int32_t e = 0; e < m->siblings; ++e) {
      if (e == d) continue;
      hpar_rect toe, fre;
      sections_of(m, e, &toe, &fre);
      const hpar_rect r = rect_and(tod, fre);
      if (rect_empty(r)) continue;
      CUDA_TRY(copy_rect(bufs[d], ld, tod, bufs[e], ld, toe, r, s));
    }
  }
  return ok();
}

extern "C" hpar_status hpar_map_exchange(hpar_nest_t n, const hpar_map_spec* m, float* buf, int64_t ld,
                                         void* stream_) {
  if (!n) return fail(HPAR_E_INVALID, "map exchange: nest is NULL");
  if (hpar_status st = spec_ok(m)) return st;
  if (m->siblings != n->nranks)
    return fail(HPAR_E_INVALID, "map exchange: %d siblings but %d ranks", m->siblings, n->nranks);
  if (n->nranks == 1) return ok();
  if (!buf || ld < m->to[1].len) return fail(HPAR_E_INVALID, "map exchange: bad buffer or pitch");
  if (hpar_status st = need_nccl()) return st;
  if (!g_nccl.send || !g_nccl.recv || !g_nccl.groupStart || !g_nccl.groupEnd)
    return fail(HPAR_E_NCCL, "NCCL lacks send/recv");
  const cudaStream_t s = (cudaStream_t)stream_;
  const int32_t d = n->rank;
  int32_t cnt = 0;
  if (hpar_status st = hpar_map_exchange_plan(m, d, nullptr, 0, &cnt)) return st;
  std::vector<hpar_halo> plan(cnt);
  if (hpar_status st = hpar_map_exchange_plan(m, d, plan.data(), cnt, &cnt)) return st;
  size_t total = 0;
  for (const hpar_halo& h : plan) total += (size_t)h.rect.len[0] * h.rect.len[1];
  CUDA_TRY(cudaSetDevice(n->device));
  if (total * 4 > n->halo_bytes) {
    cudaFree(n->halo_buf);
    n->halo_buf = nullptr;
    n->halo_bytes = 0;
    CUDA_TRY(cudaMalloc(&n->halo_buf, total * 4));
    n->halo_bytes = total * 4;
  }
  hpar_rect tod, frd;
  sections_of(m, d, &tod, &frd);
  std::vector<size_t> pos(cnt);
  size_t at = 0;
  for (int32_t i = 0; i < cnt; ++i) {  // pack the sends (staging is rect-shaped)
    pos[i] = at;
    const hpar_rect& r = plan[i].rect;
    if (plan[i].send) CUDA_TRY(copy_rect(n->halo_buf + at, r.len[1], r, buf, ld, tod, r, s));
    at += (size_t)r.len[0] * r.len[1];
  }
  ncclComm_t comm = (ncclComm_t)n->comm;
  ncclResult_t r = g_nccl.groupStart();
  if (r != ncclSuccess) return nccl_fail(r, comm, "ncclGroupStart");
  for (int32_t i = 0; i < cnt; ++i) {
    const size_t elems = (size_t)plan[i].rect.len[0] * plan[i].rect.len[1];
    r = plan[i].send ? g_nccl.send(n->halo_buf + pos[i], elems, ncclFloat32, plan[i].peer, comm, s)
                     : g_nccl.recv(n->halo_buf + pos[i], elems, ncclFloat32, plan[i].peer, comm, s);
    if (r != ncclSuccess) {
      g_nccl.groupEnd();
      return nccl_fail(r, comm, plan[i].send ? "ncclSend" : "ncclRecv");
    }
  }
  r = g_nccl.groupEnd();
  if (r != ncclSuccess) return nccl_fail(r, comm, "ncclGroupEnd");
  for (int32_t i = 0; i < cnt; ++i) {  // unpack the receives
    if (plan[i].send) continue;
    const hpar_rect& rr = plan[i].rect;
    CUDA_TRY(copy_rect(buf, ld, tod, n->halo_buf + pos[i], rr.len[1], rr, rr, s));
  }
  return ok();
}
