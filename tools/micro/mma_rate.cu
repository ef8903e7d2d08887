// Throughput of the legacy warp-level tensor path (mma.sync) on sm_100a:
// tf32 m16n8k8 and m16n8k4, bf16 m16n8k16, and FFMA2 for scale.  Each warp
// runs `chains` independent accumulators; the grid is 148 x warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_tf32_k8(float* out, int iters, unsigned seed) {
  unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[CH][4];
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int CH>
__global__ void k_tf32_k4(float* out, int iters, unsigned seed) {
  unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3, b0 = a0 * 11;
  float c[CH][4];
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(b0));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int CH>
__global__ void k_bf16(float* out, int iters, unsigned seed) {
  unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[CH][4];
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int CH>
__global__ void k_ffma2(float* out, int iters, unsigned seed) {
  float2 a = make_float2(threadIdx.x * 1e-3f, seed * 1e-9f), b = make_float2(0.999f, 1.0001f);
  float2 c[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j] = make_float2(j, j + 1);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) c[j] = __ffma2_rn(a, c[j], b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j].x + c[j].y;
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <typename K>
static void run(const char* name, K kern, int warps, int iters, double fma_per_inst, int chains) {
  float* out;
  cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<148, warps * 32>>>(out, iters, 1);
  cudaEventRecord(e0);
  kern<<<148, warps * 32>>>(out, iters, 2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double inst = 148.0 * warps * iters * chains;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-10s warps/SM %2d chains %d: %.3f ms  %.2f warp-inst/clk/SM  %.0f FMA/clk/SM  %.1f TFMA/s\n", name, warps,
         chains, ms, inst / 148.0 / cyc, inst * fma_per_inst / 148.0 / cyc, inst * fma_per_inst / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  const int it = 20000;
  for (int w : {4, 8, 16, 32}) {
    run("tf32k8", k_tf32_k8<1>, w, it, 16 * 8 * 8, 1);
    run("tf32k8", k_tf32_k8<4>, w, it / 4, 16 * 8 * 8, 4);
    run("tf32k4", k_tf32_k4<4>, w, it / 4, 16 * 8 * 4, 4);
    run("bf16k16", k_bf16<4>, w, it / 4, 16 * 8 * 16, 4);
    run("ffma2", k_ffma2<8>, w, it, 64, 8);
  }
  return 0;
}
