// Can a 15-CTA cluster (227 KB smem each) run concurrently with a persistent
// 133-CTA kernel (228 KB smem each) on the other SMs?  Both spin ~200 us;
// concurrent -> total ~200 us, serialised -> ~400 us.  Also records the SM
// ids the cluster landed on.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__global__ void __launch_bounds__(512, 1) big(long long spin, unsigned* ids) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) { ids[blockIdx.x] = smid(); sm[0] = 1; }
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}
__global__ void __launch_bounds__(512, 1) clus(long long spin, unsigned* ids) {
  extern __shared__ char sm[];
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) { ids[blockIdx.x] = smid(); sm[0] = 1; }
  cl.sync();
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  cl.sync();
}
int main() {
  unsigned *dbig, *dcl; cudaMalloc(&dbig, 4096); cudaMalloc(&dcl, 4096);
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(clus, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(clus, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int lo, hi; cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t sa, sb; cudaStreamCreateWithPriority(&sa, cudaStreamNonBlocking, hi); cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, lo);
  const long long spin = 400000;  // ~200 us at 1.965 GHz
  for (int order = 0; order < 2; ++order) for (int nbig : {133, 128, 120, 112}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    cudaStreamWaitEvent(sa, e0); cudaStreamWaitEvent(sb, e0);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(15); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 227 * 1024; cfg.stream = sa;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 15; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (order == 0) { cudaLaunchKernelEx(&cfg, clus, spin, dcl); big<<<nbig, 512, 227 * 1024, sb>>>(spin, dbig); }
    else { big<<<nbig, 512, 227 * 1024, sb>>>(spin, dbig); cudaLaunchKernelEx(&cfg, clus, spin, dcl); }
    cudaEvent_t ea, eb; cudaEventCreate(&ea); cudaEventCreate(&eb); cudaEventRecord(ea, sa); cudaEventRecord(eb, sb);
    cudaStreamWaitEvent(0, ea); cudaStreamWaitEvent(0, eb); cudaEventRecord(e1, 0);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned ids[16]; cudaMemcpy(ids, dcl, 60, cudaMemcpyDeviceToHost);
    printf("order=%s nbig=%d: %.1f us (%s) cluster SMs:", order ? "big-first" : "cluster-first", nbig, ms * 1e3, cudaGetErrorString(err));
    for (int i = 0; i < 15; ++i) printf(" %u", ids[i]);
    printf("\n");
  }
  // both gated by the same event (a short kernel before it): big enqueued first
  // on the low-priority stream, the cluster on the high-priority one
  for (int rep = 0; rep < 4; ++rep) for (int nbig : {133, 120}) {
    cudaEvent_t e0, e1, eg; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreateWithFlags(&eg, cudaEventDisableTiming);
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    big<<<1, 32, 16, 0>>>(20000, dbig + 512);  // ~10 us gate
    cudaEventRecord(eg, 0);
    cudaStreamWaitEvent(sa, eg); cudaStreamWaitEvent(sb, eg);
    big<<<nbig, 512, 227 * 1024, sb>>>(spin, dbig);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(15); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 227 * 1024; cfg.stream = sa;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 15; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, clus, spin, dcl);
    cudaEvent_t ea, eb; cudaEventCreate(&ea); cudaEventCreate(&eb); cudaEventRecord(ea, sa); cudaEventRecord(eb, sb);
    cudaStreamWaitEvent(0, ea); cudaStreamWaitEvent(0, eb); cudaEventRecord(e1, 0);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("gated, big enqueued first (low prio), cluster high prio, nbig=%d: %.1f us\n", nbig, ms * 1e3);
  }
  int ncl = 0; cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(15); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 227 * 1024;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 15; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaOccupancyMaxActiveClusters(&ncl, clus, &cfg);
  printf("max active 15-CTA clusters (empty GPU): %d\n", ncl);
}
