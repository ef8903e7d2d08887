// Isolated timing of ircur::jacobi_eig (diagnostics).
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
  long long dbg[16] = {0};
  long long tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (threadIdx.x < kEigNT) {
      for (int e = threadIdx.x; e < kk * kk; e += kEigNT) {
        const int i = e / kk, j = e - i * kk;
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        S.H[i * L.HL + j] = (i == j) ? (double)(kk - i) * 10.0 : 1.0 / (1.0 + lo + 2.0 * hi);
      }
      eig_sync();
      long long t0 = clock64();
      jacobi_eig(S, kk, 4e-16, nullptr);
      tot += clock64() - t0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = tot / reps; for (int i = 0; i < kk; ++i) outlam[i] = S.lam[i]; }
}
int main() {
  long long* d; double* dl; cudaMalloc(&d, 64); cudaMalloc(&dl, 32 * 8);
  cudaFuncSetAttribute(k_iso, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int kk : {4, 10, 20, 32}) {
    size_t smem = svd_smem_bytes(64, 64, kk, 1);
    k_iso<<<1, 512, smem>>>(kk, 20, d, dl);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; double lam[32]; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); cudaMemcpy(lam, dl, kk * 8, cudaMemcpyDeviceToHost);
    printf("kk=%d: %lld cycles per dense eig (err=%s) lam0=%.6f lamlast=%.6f\n", kk, h, cudaGetErrorString(e), lam[0], lam[kk-1]);
  }
  return 0;
}
