// Memory-side ceiling of the strip kernels' tile fill: a persistent grid
// reads tiles of W positions x NL sampled rows (row length N floats, rows
// drawn at random from a 40 GB matrix) with 16-byte cp.async into a
// double-buffered shared stage, no compute.  Reports GB/s for W = 32..256.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strip_fill strip_fill.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int W>
__global__ void __launch_bounds__(512, 1) fill(const float* __restrict__ D, long long ld, const int* rows, int nl,
                                               int ntiles, float* sink) {
  extern __shared__ float st[];
  const int chunks = W / 4;
  const int per = nl * chunks;
  float acc = 0.f;
  int buf = 0;
  auto issue = [&](int t, int b) {
    float* s = st + (size_t)b * nl * W;
    for (int e = threadIdx.x; e < per; e += blockDim.x) {
      const int L = e / chunks, ch = e - L * chunks;
      cp16(s + L * W + 4 * ch, D + (long long)rows[L] * ld + (long long)t * W + 4 * ch);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int t = blockIdx.x;
  if (t < ntiles) issue(t, 0);
  for (; t < ntiles; t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) {
      issue(tn, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    acc += st[(size_t)buf * nl * W + threadIdx.x];
    __syncthreads();
    buf ^= 1;
  }
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

template <int W>
void run(const float* D, long long ld, const int* rows, int nl, long long n2, float* sink, int sms, int nt = 512) {
  const int ntiles = (int)(n2 / W);
  const size_t smem = (size_t)2 * nl * W * 4;
  if (smem > 227 * 1024) { printf("W=%d: stage too big\n", W); return; }
  cudaFuncSetAttribute(fill<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  fill<W><<<sms, nt, smem>>>(D, ld, rows, nl, ntiles, sink);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) fill<W><<<sms, nt, smem>>>(D, ld, rows, nl, ntiles, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = 5.0 * nl * (double)ntiles * W * 4;
  printf("threads %3d lines %3d W=%3d (%4d B/row): %.1f us per pass, %.0f GB/s (%s)\n", nt, nl, W, W * 4, ms * 1e3 / 5, bytes / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long long n1 = 100000, n2 = 100000;
  float* D; cudaMalloc(&D, n1 * n2 * 4);
  cudaMemset(D, 0, n1 * n2 * 4);
  const int nl = 461;
  std::vector<int> h(nl);
  srand(7);
  std::vector<int> all(n1);
  for (int i = 0; i < n1; ++i) all[i] = i;
  for (int i = 0; i < nl; ++i) std::swap(all[i], all[i + rand() % (n1 - i)]);
  for (int i = 0; i < nl; ++i) h[i] = all[i];
  std::sort(h.begin(), h.end());
  int* rows; cudaMalloc(&rows, nl * 4);
  cudaMemcpy(rows, h.data(), nl * 4, cudaMemcpyHostToDevice);
  float* sink; cudaMalloc(&sink, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<32>(D, n2, rows, nl, n2, sink, sms);
  run<32>(D, n2, rows, nl, n2, sink, sms, 32);
  run<32>(D, n2, rows, nl, n2, sink, sms, 128);
  run<32>(D, n2, rows, nl / 2, n2, sink, sms);
  run<64>(D, n2, rows, nl / 2, n2, sink, sms);
  run<128>(D, n2, rows, nl / 4, n2, sink, sms);
  run<256>(D, n2, rows, nl / 8, n2, sink, sms);
  return 0;
}
