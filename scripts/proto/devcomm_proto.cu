// Prototype (single process, 1 rank): NCCL 2.28 device API plumbing for the
// fused node level (NEXT f1): symmetric window + LSA stores + LSA barrier.
#include <cstdio>
#include <nccl.h>
#include <nccl_device.h>
#include <cuda_runtime.h>

#define CK(x) do { auto r = (x); if (r != 0) { printf("%s failed: %d line %d\n", #x, (int)r, __LINE__); return 1; } } while (0)

__global__ void k(ncclDevComm dc, ncclWindow_t win, double v, double* out) {
  // one CTA: thread 0 stores v into every LSA peer's slot [rank]
  if (threadIdx.x == 0) {
    for (int p = 0; p < dc.lsaSize; ++p) {
      double* slot = (double*)ncclGetLsaPointer(win, sizeof(double) * dc.rank, p);
      *slot = v;
    }
  }
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  if (threadIdx.x == 0) {
    double* mine = (double*)ncclGetLocalPointer(win, 0);
    double t = 0;
    for (int r = 0; r < dc.nRanks; ++r) t += mine[r];
    *out = t;
  }
}

int main() {
  ncclUniqueId id; CK(ncclGetUniqueId(&id));
  ncclComm_t comm; CK(ncclCommInitRank(&comm, 1, id, 0));
  void* buf = nullptr; CK(ncclMemAlloc(&buf, 4096));
  ncclWindow_t win; CK(ncclCommWindowRegister(comm, buf, 4096, &win, NCCL_WIN_COLL_SYMMETRIC));
  ncclDevCommRequirements req = {};
  req.lsaBarrierCount = 1;
  ncclDevComm dc; CK(ncclDevCommCreate(comm, &req, &dc));
  double* out; cudaMalloc(&out, 8);
  k<<<1, 128>>>(dc, win, 3.5, out);
  CK(cudaDeviceSynchronize());
  double h = 0; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("ok: rank %d nranks %d lsa %d/%d -> %g\n", dc.rank, dc.nRanks, dc.lsaRank, dc.lsaSize, h);
  CK(ncclDevCommDestroy(comm, &dc));
  CK(ncclCommWindowDeregister(comm, win));
  CK(ncclMemFree(buf));
  CK(ncclCommDestroy(comm));
  return 0;
}
