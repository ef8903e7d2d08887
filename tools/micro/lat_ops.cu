// Dependent-chain latency and single-warp throughput (cycles/op) of the ops
// in the small-eigensolver round (volatile PTX so nothing is hoisted).
#include <cstdio>
#define N 64
__global__ void k(long long* out, double x0, float f0) {
  double x = x0 + threadIdx.x * 1e-30, y = x + 1, z = x + 2, w = x + 3;
  float f = f0;
  long long t0, t1;
  int o = 0;
#define T0 asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
#define T1(reg) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory"); out[o++] = t1 - t0;
  T0 for (int i = 0; i < N; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(x) : "d"(y)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(y)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(y)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("{.reg .b32 lo, hi; mov.b64 {lo,hi}, %0; shfl.sync.idx.b32 lo, lo, 1, 31, -1; shfl.sync.idx.b32 hi, hi, 1, 31, -1; mov.b64 %0, {lo,hi};}" : "+d"(x)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("{.reg .f32 t; cvt.rn.f32.f64 t, %0; cvt.f64.f32 %0, t;}" : "+d"(x)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("sqrt.approx.f32 %0, %0;" : "+f"(f)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("shfl.sync.idx.b32 %0, %0, 1, 31, -1;" : "+f"(f)); T1()
  // throughput: 4 independent chains
  T0 for (int i = 0; i < N; ++i) asm volatile("fma.rn.f64 %0, %0, %4, %4; fma.rn.f64 %1, %1, %4, %4; fma.rn.f64 %2, %2, %4, %4; fma.rn.f64 %3, %3, %4, %4;" : "+d"(x), "+d"(y), "+d"(z), "+d"(w) : "d"(x0)); T1()
  T0 for (int i = 0; i < N; ++i) asm volatile("{.reg .b32 a,b,c,d; mov.b64 {a,b}, %0; mov.b64 {c,d}, %1; shfl.sync.idx.b32 a, a, 1, 31, -1; shfl.sync.idx.b32 b, b, 1, 31, -1; shfl.sync.idx.b32 c, c, 1, 31, -1; shfl.sync.idx.b32 d, d, 1, 31, -1; mov.b64 %0, {a,b}; mov.b64 %1, {c,d};}" : "+d"(x), "+d"(y)); T1()
  out[15] = (long long)(x + y + z + w + f);
}
int main() {
  long long* d; cudaMalloc(&d, 128);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 32>>>(d, 1.5, 1.5f);
  cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA lat", "DMUL lat", "DADD lat", "SHFL f64 (2 SHFL) lat", "F2F d->f->d lat", "RSQ64H lat", "SQRT f32 lat", "RCP f32 lat", "SHFL b32 lat",
                      "DFMA 4-indep (per DFMA)", "SHFL 4-indep (per SHFL)"};
  for (int i = 0; i < 11; ++i) printf("%-26s %6.1f cyc\n", nm[i], h[i] / (double)N / (i >= 9 ? 4 : 1));
}
