// Microbenchmark: the synchronisation cost of each in-GPU level of the B200
// hierarchy, in SM cycles — the "grainedness" column of the level table
// (runtime.cpp level_grain).  One cluster of 2 CTAs x 8 warps per
// measurement, clock64() around N dependent repetitions:
//   lane    : a dependent SHFL chain (one lane-level combine step)
//   warp    : one combine step among 8 warps: store a slot, bar.sync, read
//             a sibling's slot (the value feeds the next step)
//   CTA     : the same over DSMEM: store, barrier.cluster arrive.release +
//             wait.acquire, read the sibling CTA's slot (2 CTAs)
//   cluster : a dependent chain of atom.acq_rel.gpu on one global word (the
//             single-pass ticket clusters meet at; they have no barrier)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/grain scripts/grain_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe(long long* out, unsigned* word, int n) {
  const int lane = threadIdx.x & 31;
  long long t0, t1;
  // lane level
  unsigned v = threadIdx.x;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
  t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / n;
  // warp level: slot store, bar.sync, sibling slot load (double-buffered)
  __shared__ volatile unsigned slot[2][8];
  __shared__ unsigned cslot[2];
  const int warp = threadIdx.x >> 5;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (lane == 0) slot[i & 1][warp] = v;
    __syncthreads();
    v += slot[i & 1][(warp + 1) & 7];
  }
  t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (t1 - t0) / n;
  // CTA level: slot store, cluster barrier, the sibling CTA's slot over DSMEM
  unsigned rank, sib;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  cluster_sync();
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == 0) cslot[i & 1] = v;
    cluster_sync();
    uint32_t local = (uint32_t)__cvta_generic_to_shared(&cslot[i & 1]), remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank ^ 1u));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(sib) : "r"(remote) : "memory");
    v += sib;
  }
  t1 = clock64();
  cluster_sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2] = (t1 - t0) / n;
  // cluster level: dependent acq_rel atomics through L2
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned r = 0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(word), "r"(r & 1u) : "memory");
    }
    t1 = clock64();
    out[3] = (t1 - t0) / n;
  }
  if (v == 0xdeadbeef && lane == 0) out[4] = v;
}

__global__ void empty_kernel() {}

int main() {
  long long* out;
  unsigned* word;
  cudaMalloc(&out, 8 * sizeof(long long));
  cudaMalloc(&word, 4);
  cudaMemset(word, 0, 4);
  probe<<<2, 256>>>(out, word, 16);
  probe<<<2, 256>>>(out, word, 4096);
  long long h[8] = {0};
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  // kernel boundary (what a host-level barrier among clusters costs): back-to-back
  // empty launches in a CUDA graph, device time per launch
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 1000; ++i) empty_kernel<<<148, 32, 0, s>>>();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("lane    (dependent SHFL step)            : %lld cycles\n", h[0]);
  printf("warp    (slot + bar.sync + load, 8 warps) : %lld cycles\n", h[1]);
  printf("CTA     (slot + cluster barrier + DSMEM)  : %lld cycles\n", h[2]);
  printf("cluster (dependent atom.acq_rel.gpu)      : %lld cycles\n", h[3]);
  printf("kernel boundary (graph of empty launches) : %.2f us = %.0f cycles at %d MHz\n", ms * 1e3 / 1000,
         ms * 1e3 / 1000 * clk / 1e3, clk / 1000);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
