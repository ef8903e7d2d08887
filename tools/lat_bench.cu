// Latency microbenchmarks on B200 (diagnostics): dependent chains of
// LDS.64, STS+LDS round trip, SHFL (double), DFMA, rsqrt(double), F2F.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, int iters, double seed) {
  __shared__ double sm[1024];
  __shared__ int si[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = (i + 1) % 1024; si[i] = (i * 7 + 1) % 1024; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  long long t0, t1;
  double x = seed; int p = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) p = si[p];
  t1 = clock64(); out[0] = (t1 - t0) / iters;
  double d = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = sm[(int)d];
  t1 = clock64(); out[1] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { sm[threadIdx.x] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] + 1.0; __syncwarp(); }
  t1 = clock64(); out[2] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); out[3] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1.0);
  t1 = clock64(); out[4] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x + 2.0);
  t1 = clock64(); out[5] = (t1 - t0) / iters;
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { f = (float)((double)f * 1.0001); }
  t1 = clock64(); out[6] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * 1.0000001;
  t1 = clock64(); out[7] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = x + 1e-300; __syncwarp(); }
  t1 = clock64(); out[8] = (t1 - t0) / iters;
  out[9] = (long long)(x + d + p + f);
}
int main() {
  long long* d; cudaMalloc(&d, 128); long long h[10];
  k<<<1, 128>>>(d, 1000, 1.5); cudaDeviceSynchronize();
  k<<<1, 128>>>(d, 1000, 1.5); cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
  printf("LDS.32 chain %lld | LDS.64 chain %lld | STS+syncwarp+LDS %lld | SHFL f64 %lld | DFMA %lld | rsqrt f64 %lld | F2F f32<->f64 %lld | DMUL %lld | DADD+syncwarp %lld cycles\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
  return 0;
}
