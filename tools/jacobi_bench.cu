// Microbenchmark: cost of named barriers, fp64 rsqrt and a Jacobi-like round
// on 128 threads (diagnostics for the core-SVD kernel).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void bsync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__global__ void k_bar(long long* out, int iters) {
  __shared__ double sm[256];
  if (threadIdx.x >= 128) { __syncthreads(); return; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bsync();
  long long t1 = clock64();
  double x = threadIdx.x + 1.0;
  for (int i = 0; i < iters; ++i) x = rsqrt(x + 1.0);
  long long t2 = clock64();
  double y = threadIdx.x;
  for (int i = 0; i < iters; ++i) { sm[threadIdx.x] = y; bsync(); y = sm[(threadIdx.x + 1) & 127] * 0.5 + 1.0; bsync(); }
  long long t3 = clock64();
  double z = threadIdx.x;
  for (int i = 0; i < iters; ++i) z = fma(z, 0.999, 1.0);
  long long t4 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters; out[3] = (t4 - t3) / iters; out[4] = (long long)(x + y + z); }
  __syncthreads();
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[5];
  for (int nt : {128, 512}) {
    k_bar<<<1, nt>>>(d, 1000); cudaDeviceSynchronize();
    k_bar<<<1, nt>>>(d, 1000); cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    printf("threads=%d: bar.sync(128)=%lld cyc, dp rsqrt chain=%lld cyc, sts+bar+lds+bar=%lld cyc, dfma chain=%lld cyc\n", nt, h[0], h[1], h[2], h[3]);
  }
  return 0;
}
