// Isolated timing of ircur::jacobi_eig (diagnostics): whole eig and the
// two phases of one Jacobi round, with and without idle warps parked at a
// block barrier.
#include <cstdio>
#include "../paper_2010_07422_b200/csrc/kernels_svd.cu"
using namespace ircur;
__global__ void k_iso(int kk, int reps, long long* out, double* outlam) {
  extern __shared__ __align__(16) double sm[];
  Sm S;
  S.L = svd_layout(64, 64, kk, 1);
  const SvdLayout& L = S.L;
  S.H = sm + L.oH; S.H2 = sm + L.oH2; S.Z = sm + L.oZ; S.T = sm + L.oT; S.Lc = sm + L.oLc;
  S.cs = sm + L.oCs; S.lam = sm + L.oLam; S.ws = sm + L.oW;
  S.flags = reinterpret_cast<int*>(sm + L.oW + kKMax); S.ptab = reinterpret_cast<int*>(sm + L.oPt);
  long long tot = 0, tround = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (threadIdx.x < kEigNT) {
      for (int e = threadIdx.x; e < kk * kk; e += kEigNT) {
        const int i = e / kk, j = e - i * kk;
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        S.H[i * L.HL + j] = (i == j) ? (double)(kk - i) * 10.0 : 1.0 / (1.0 + lo + 2.0 * hi);
      }
      eig_sync();
      long long t0 = clock64();
      jacobi_eig(S, kk, 4e-16, 30, nullptr);
      tot += clock64() - t0;
      // bare round skeleton: params-like chain + barrier + update-like loop + barrier
      t0 = clock64();
      for (int it = 0; it < 100; ++it) {
        if (threadIdx.x < kk) { double x = S.H[threadIdx.x * L.HL + threadIdx.x]; S.cs[threadIdx.x] = rsqrt(x * x + 1.0); }
        eig_sync();
        for (int e = threadIdx.x; e < kk * kk; e += kEigNT) S.H2[e] = S.cs[e % kk] * S.H[e];
        eig_sync();
      }
      tround += (clock64() - t0) / 100;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = tot / reps; out[1] = tround / reps; for (int i = 0; i < kk; ++i) outlam[i] = S.lam[i]; }
}
int main() {
  long long* d; double* dl; cudaMalloc(&d, 64); cudaMalloc(&dl, 32 * 8);
  cudaFuncSetAttribute(k_iso, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nt : {128, 512}) for (int kk : {4, 10, 20}) {
    size_t smem = svd_smem_bytes(64, 64, kk, 1);
    k_iso<<<1, nt, smem>>>(kk, 20, d, dl);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2]; double lam[32]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); cudaMemcpy(lam, dl, kk * 8, cudaMemcpyDeviceToHost);
    printf("threads=%d kk=%d: %lld cycles per dense eig, %lld cycles per bare round (%s) lam0=%.6f\n", nt, kk, h[0], h[1], cudaGetErrorString(e), lam[0]);
  }
  return 0;
}
