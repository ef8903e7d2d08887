// Diagnostics: validates the tcgen05 (tf32) operand layouts and descriptors
// of paper_2010_07422_b200/csrc/umma.cuh on the B200 against a host
// reference, and reports how the tensor core converts fp32 inputs to tf32
// (truncation or rounding).  One CTA of 128 threads per test.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_2010_07422_b200/csrc tools/micro/umma_probe.cu -o tools/micro/umma_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#include "umma.cuh"

using namespace ircur::umma;

struct Probe {
  const float* A; const float* B;  // A: M x K row-major, B: N x K row-major (host semantics)
  float* D;                        // 128 lanes x 64 cols dump
  int test;
};

__device__ __forceinline__ uint32_t kmaj_off(int row, int k, int lbo, int sbo) {
  return (row / 8) * sbo + (k / 4) * lbo + (row % 8) * 16 + (k % 4) * 4;
}
__device__ __forceinline__ uint32_t mnmaj_off(int mn, int k, int lbo, int sbo) {
  return (mn / 32) * lbo + (k / 8) * sbo + (k % 8) * 128 + ((((mn % 32) / 4) ^ (k % 8)) * 16) + (mn % 4) * 4;
}

__device__ __forceinline__ uint32_t kmaj_sw128_off(int row, int k, int sbo) {
  return (row / 8) * sbo + (row % 8) * 128 + (((k / 4) ^ (row % 8)) * 16) + (k % 4) * 4;
}
__device__ __forceinline__ uint32_t mnmaj_il_off(int mn, int k, int lbo, int sbo) {
  return (mn / 4) * sbo + (k / 8) * lbo + (k % 8) * 16 + (mn % 4) * 4;
}

__global__ void __launch_bounds__(128, 1) probe_kernel(Probe p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, w = tid >> 5;
  // swizzled layouts are defined on absolute shared addresses: align the
  // operand base to 1 KB (static shared variables precede the dynamic ones)
  unsigned char* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  unsigned char* sa = base;           // 32 KB
  unsigned char* sb = base + 32768;   // 32 KB
  if (w == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) { bar_init(&bar, 1); bar_init_fence(); }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = tbase;
  const uint32_t lane_off = (uint32_t)(32 * w) << 16;
  int M = 128, N = 64, K = 8;
  uint32_t idesc = 0;
  if (p.test == 1) {  // SS, both K-major interleave
    M = 128; N = 64; K = 8;
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      *reinterpret_cast<float*>(sa + kmaj_off(m, k, 128, 256)) = p.A[m * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + kmaj_off(n, k, 128, 256)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 0, 0);
  } else if (p.test == 2) {  // A in TMEM (cols 128..159), B MN-major SW128 (N contiguous)
    M = 128; N = 64; K = 32;
    float v[16];
    for (int h = 0; h < 2; ++h) {
      for (int i = 0; i < 16; ++i) v[i] = p.A[tid * K + 16 * h + i];
      st16(T + lane_off + 128 + 16 * h, v);
    }
    st_wait();
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + mnmaj_off(n, k, 1024, 2048)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 0, 1);
  } else if (p.test == 3) {  // A MN-major SW128 (M contiguous), B K-major interleave, N = 32, K = 16
    M = 128; N = 32; K = 16;
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      *reinterpret_cast<float*>(sa + mnmaj_off(m, k, 1024, 4096)) = p.A[m * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + kmaj_off(n, k, 128, 512)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 1, 0);
  } else if (p.test == 5) {  // A in TMEM, B K-major interleave, K = 32
    M = 128; N = 64; K = 32;
    float v[16];
    for (int h = 0; h < 2; ++h) {
      for (int i = 0; i < 16; ++i) v[i] = p.A[tid * K + 16 * h + i];
      st16(T + lane_off + 128 + 16 * h, v);
    }
    st_wait();
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + kmaj_off(n, k, 128, 1024)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 0, 0);
  } else if (p.test == 6) {  // A K-major interleave, B MN-major SW128, K = 32
    M = 128; N = 64; K = 32;
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      *reinterpret_cast<float*>(sa + kmaj_off(m, k, 128, 1024)) = p.A[m * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + mnmaj_off(n, k, 1024, 2048)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 0, 1);
  } else if (p.test == 7) {  // A K-major SW128 (K = 32 = one 128 B row), B K-major interleave
    M = 128; N = 64; K = 32;
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      *reinterpret_cast<float*>(sa + kmaj_sw128_off(m, k, 1024)) = p.A[m * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + kmaj_off(n, k, 128, 1024)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 0, 0);
  } else if (p.test == 8 || p.test == 10) {  // A K-major interleave, B MN-major interleave
    M = 128; N = 64; K = 32;
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      *reinterpret_cast<float*>(sa + kmaj_off(m, k, 128, 1024)) = p.A[m * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      // core matrices: 4 MN x 8 K (128 B); MN cores 128 B apart, K groups 2048 B apart
      *reinterpret_cast<float*>(sb + mnmaj_il_off(n, k, 2048, 128)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 0, 1);
  } else if (p.test == 9) {  // test 6 data, descriptor LBO/SBO swapped
    M = 128; N = 64; K = 32;
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      *reinterpret_cast<float*>(sa + kmaj_off(m, k, 128, 1024)) = p.A[m * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + mnmaj_off(n, k, 1024, 2048)) = p.B[n * K + k];
    }
    idesc = idesc_tf32(M, N, 0, 1);
  } else if (p.test == 4) {  // M = 64 layout probe: SS K-major, N = 16, K = 8
    M = 64; N = 16; K = 8;
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      *reinterpret_cast<float*>(sa + kmaj_off(m, k, 128, 256)) = p.A[m * K + k];
    }
    for (int e = tid; e < N * K; e += 128) {
      const int n = e / K, k = e % K;
      *reinterpret_cast<float*>(sb + kmaj_off(n, k, 128, 256)) = p.B[n * K + k];
    }
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = -777.f;  // sentinel in all 128 lanes
    st16(T + lane_off, v);
    st_wait();
    idesc = idesc_tf32(M, N, 0, 0);
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    if (p.test == 1 || p.test == 4) {
      mma_ss(T, smem_desc(a0, 128, 256, kSwizzleNone), smem_desc(b0, 128, 256, kSwizzleNone), idesc, false);
    } else if (p.test == 2) {
      for (int s = 0; s < 4; ++s)
        mma_ts(T, T + 128 + 8 * s, smem_desc(b0 + s * 2048, 1024, 2048, kSwizzle128), idesc, s > 0);
    } else if (p.test == 5) {
      for (int s = 0; s < 4; ++s)
        mma_ts(T, T + 128 + 8 * s, smem_desc(b0 + s * 256, 128, 1024, kSwizzleNone), idesc, s > 0);
    } else if (p.test == 6) {
      for (int s = 0; s < 4; ++s)
        mma_ss(T, smem_desc(a0 + s * 256, 128, 1024, kSwizzleNone), smem_desc(b0 + s * 2048, 1024, 2048, kSwizzle128),
               idesc, s > 0);
    } else if (p.test == 7) {
      for (int s = 0; s < 4; ++s)
        mma_ss(T, smem_desc(a0 + s * 32, 16, 1024, kSwizzle128), smem_desc(b0 + s * 256, 128, 1024, kSwizzleNone),
               idesc, s > 0);
    } else if (p.test == 8) {  // interleave: LBO = K-group stride, SBO = MN-core stride
      for (int s = 0; s < 4; ++s)
        mma_ss(T, smem_desc(a0 + s * 256, 128, 1024, kSwizzleNone), smem_desc(b0 + s * 2048, 2048, 128, kSwizzleNone),
               idesc, s > 0);
    } else if (p.test == 10) {  // interleave, the other reading of LBO / SBO
      for (int s = 0; s < 4; ++s)
        mma_ss(T, smem_desc(a0 + s * 256, 128, 1024, kSwizzleNone), smem_desc(b0 + s * 2048, 128, 2048, kSwizzleNone),
               idesc, s > 0);
    } else if (p.test == 9) {
      for (int s = 0; s < 4; ++s)
        mma_ss(T, smem_desc(a0 + s * 256, 128, 1024, kSwizzleNone), smem_desc(b0 + s * 2048, 2048, 1024, kSwizzle128),
               idesc, s > 0);
    } else if (p.test == 3) {
      for (int s = 0; s < 2; ++s)
        mma_ss(T, smem_desc(a0 + s * 4096, 1024, 4096, kSwizzle128),
               smem_desc(b0 + s * 256, 128, 512, kSwizzleNone), idesc, s > 0);
    }
    commit(&bar);
  }
  bar_wait(&bar, 0);
  fence_after();
  float v[16];
  for (int c0 = 0; c0 < 64; c0 += 16) {
    ld16(T + lane_off + c0, v);
    ld_wait();
    for (int i = 0; i < 16; ++i) p.D[tid * 64 + c0 + i] = v[i];
  }
  fence_before();
  __syncthreads();
  if (w == 0) tmem_free(T, 256);
}

static float trunc_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static float round_tf32(float x) {  // nearest, ties away (cvt.rna.tf32.f32)
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  const int M = 128, K = 32, N = 64;
  std::vector<float> A(M * K), B(N * K), D(128 * 64);
  srand(1);
  for (auto& x : A) x = (float)(rand() / (double)RAND_MAX * 2 - 1) * (1 + (rand() % 7));
  for (auto& x : B) x = (float)(rand() / (double)RAND_MAX * 2 - 1);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  int fails = 0;
  for (int test = 1; test <= 10; ++test) {
    int m = 128, n = 64, k = 8;
    if (test == 2 || test >= 5) k = 32;
    if (test == 3) { n = 32; k = 16; }
    if (test == 4) { m = 64; n = 16; k = 8; }
    std::vector<float> a(m * k), b(n * k);
    for (int i = 0; i < m * k; ++i) a[i] = A[i];
    for (int i = 0; i < n * k; ++i) b[i] = B[i];
    cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    Probe p{dA, dB, dD, test};
    probe_kernel<<<1, 128, 65536 + 1024>>>(p);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("test %d: CUDA error %s\n", test, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    if (test == 4) {  // where did row i of the M = 64 result land?
      int found = 0;
      for (int i = 0; i < m; ++i) {
        double want = 0;
        for (int q = 0; q < k; ++q) want += (double)trunc_tf32(a[i * k + q]) * trunc_tf32(b[0 * k + q]);
        for (int lane = 0; lane < 128; ++lane)
          if (fabs(D[lane * 64 + 0] - want) <= 1e-4 * (1 + fabs(want))) {
            if (i < 20 || i % 16 == 15) printf("  M=64 row %d -> lane %d\n", i, lane);
            ++found;
            break;
          }
      }
      int sentinel = 0;
      for (int lane = 0; lane < 128; ++lane) sentinel += D[lane * 64] == -777.f;
      printf("test 4 (M=64): %d/%d rows located, %d lanes untouched\n", found, m, sentinel);
      continue;
    }
    double et = 0, er = 0, ex = 0, mag = 0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        double wt = 0, wr = 0, wx = 0;
        for (int q = 0; q < k; ++q) {
          wt += (double)trunc_tf32(a[i * k + q]) * trunc_tf32(b[j * k + q]);
          wr += (double)round_tf32(a[i * k + q]) * round_tf32(b[j * k + q]);
          wx += (double)a[i * k + q] * b[j * k + q];
        }
        const double g = D[i * 64 + j];
        et = fmax(et, fabs(g - wt));
        er = fmax(er, fabs(g - wr));
        ex = fmax(ex, fabs(g - wx));
        mag = fmax(mag, fabs(wx));
      }
    const bool ok = et <= 1e-5 * mag || er <= 1e-5 * mag;
    fails += !ok;
    printf("test %d: max|D - trunc| %.3e  max|D - round| %.3e  max|D - exact| %.3e  (|D| %.2e) %s\n", test, et,
           er, ex, mag, ok ? "OK" : "FAIL");
  }
  printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
  return fails != 0;
}
