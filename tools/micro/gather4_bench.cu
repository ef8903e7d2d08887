// Microbenchmark (diagnostics): filling a [lines x 64] fp32 shared stage with
// rows gathered from a row-major matrix, TMA tile::gather4 vs 16-byte
// cp.async.  148 persistent CTAs, double-buffered, 232 random sorted rows
// per CTA-tile, positions walk the row in 64-element tiles.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

constexpr int TX = 64, NL = 232;
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) k_gather4(const __grid_constant__ CUtensorMap tm, const int* rows, int n2,
                                                    int tiles, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* stage = reinterpret_cast<float*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * NL * TX * 4);
  __shared__ int li[NL];
  for (int i = threadIdx.x; i < NL; i += blockDim.x) li[i] = rows[i];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i, int st) {
    const int t = blockIdx.x + i * gridDim.x;
    if (t >= tiles) return;
    const int x0 = t * TX;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[st])), "r"(NL * TX * 4) : "memory");
    __syncwarp();
    if (threadIdx.x < 32) {
      for (int g = threadIdx.x; g < NL / 4; g += 32) {
        float* dst = stage + (size_t)st * NL * TX + (size_t)g * 4 * TX;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(s32(dst)), "l"(&tm), "r"(s32(&bar[st])),
            "r"(x0), "r"(li[4 * g]), "r"(li[4 * g + 1]), "r"(li[4 * g + 2]), "r"(li[4 * g + 3])
            : "memory");
      }
    }
  };
  issue(0, 0);
  issue(1, 1);
  float acc = 0.f;
  uint32_t ph[2] = {0, 0};
  for (int i = 0;; ++i) {
    const int t = blockIdx.x + i * gridDim.x;
    if (t >= tiles) break;
    const int st = i & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(s32(&bar[st])), "r"(ph[st]) : "memory");
    ph[st] ^= 1;
    const float* sg = stage + (size_t)st * NL * TX;
    for (int e = threadIdx.x; e < NL * TX; e += blockDim.x) acc += sg[e];
    __syncthreads();
    issue(i + 2, st);
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void __launch_bounds__(512, 1) k_cpasync(const float* D, int64_t ldd, const int* rows, int n2, int tiles,
                                                    float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* stage = reinterpret_cast<float*>(sm);
  __shared__ const float* lp[NL];
  for (int i = threadIdx.x; i < NL; i += blockDim.x) lp[i] = D + (int64_t)rows[i] * ldd;
  __syncthreads();
  const int ch = threadIdx.x & 15, l0 = threadIdx.x >> 4;  // 16 chunks per line, 32 lines per pass
  auto issue = [&](int i, int st) {
    const int t = blockIdx.x + i * gridDim.x;
    if (t < tiles) {
      const int x0 = t * TX;
      uint32_t dst = s32(stage + (size_t)st * NL * TX) + (l0 * TX + ch * 4) * 4;
      for (int ln = l0; ln < NL; ln += 32, dst += 32 * TX * 4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(lp[ln] + x0 + ch * 4) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0, 0);
  issue(1, 1);
  float acc = 0.f;
  for (int i = 0;; ++i) {
    const int t = blockIdx.x + i * gridDim.x;
    if (t >= tiles) break;
    const int st = i & 1;
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const float* sg = stage + (size_t)st * NL * TX;
    for (int e = threadIdx.x; e < NL * TX; e += blockDim.x) acc += sg[e];
    __syncthreads();
    issue(i + 2, st);
  }
  if (acc == 12345.f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int64_t n1 = 100000, n2 = 100000;
  float* D; cudaMalloc(&D, n1 * n2 * 4); cudaMemset(D, 0, n1 * n2 * 4);
  std::vector<int> h(NL); srand(1);
  for (auto& x : h) x = rand() % n1;
  std::sort(h.begin(), h.end());
  int* rows; cudaMalloc(&rows, NL * 4); cudaMemcpy(rows, h.data(), NL * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4);
  EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)n2, (cuuint64_t)n1};
  cuuint64_t strides[1] = {(cuuint64_t)n2 * 4};
  cuuint32_t box[2] = {TX, 1}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  const int tiles = (int)((n2 + TX - 1) / TX) * 2;  // two strips' worth
  size_t smem = 2 * NL * TX * 4 + 64;
  cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(a); k_gather4<<<148, 512, smem>>>(tm, rows, (int)n2, tiles, out); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)tiles * NL * TX * 4;
    printf("gather4: %.1f us, %.0f GB/s (%s)\n", ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a); k_cpasync<<<148, 512, smem>>>(D, n2, rows, (int)n2, tiles, out); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("cp.async16: %.1f us, %.0f GB/s (%s)\n", ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
