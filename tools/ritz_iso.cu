// Isolated timing of the core-SVD small dense routines (diagnostics):
// jacobi_eig, cholesky_warp and ritz_small on one CTA, test matrices with a
// known structure.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ritz_iso.cu
#include <cstdio>
#include "../paper_2010_07422_b200/csrc/kernels_svd.cu"
using namespace ircur;
__global__ void k_iso(int kk, int reps, int nearly_diag, long long* out, double* outlam) {
  extern __shared__ __align__(16) double sm[];
  Sm S;
  S.L = svd_layout(64, 64, kk, 1);
  const SvdLayout& L = S.L;
  S.H = sm + L.oH; S.H2 = sm + L.oH2; S.Z = sm + L.oZ; S.T = sm + L.oT; S.Lc = sm + L.oLc;
  S.cs = sm + L.oCs; S.lam = sm + L.oLam; S.ws = sm + L.oW; S.rout = sm + L.oRout;
  S.flags = reinterpret_cast<int*>(sm + L.oW + kKMax); S.ptab = reinterpret_cast<int*>(sm + L.oPt);
  __shared__ long long dbg[16];
  if (threadIdx.x < 16) dbg[threadIdx.x] = 0;
  long long tj = 0, tc = 0, tr = 0;
  double* Hp = S.rout;          // kk x kk
  double* M = S.rout + kk * kk; // kk x kk
  for (int rep = 0; rep < reps; ++rep) {
    if (threadIdx.x < kEigNT) {
      for (int e = threadIdx.x; e < kk * kk; e += kEigNT) {
        const int i = e / kk, j = e - i * kk;
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        const double off = nearly_diag ? 1e-4 : 1.0;
        S.H[i * L.HL + j] = (i == j) ? (double)(kk - i) * 10.0 : off / (1.0 + lo + 2.0 * hi);
        Hp[i * kk + j] = S.H[i * L.HL + j];
        M[i * kk + j] = (i == j) ? 1.0 + 1e-3 * i : 1e-3 / (1.0 + i + j);
      }
      eig_sync();
      long long t0 = clock64();
      jacobi_eig(S, kk, 4e-16, 30, dbg);
      long long t1 = clock64();
      cholesky_warp(M, S.Lc, L.HL, kk, S.flags + 1);
      long long t2 = clock64();
      ritz_small(S, kk, Hp, M, 4e-16, 2, dbg);
      long long t3 = clock64();
      tj += t1 - t0; tc += t2 - t1; tr += t3 - t2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = tj / reps; out[1] = tc / reps; out[2] = tr / reps;
    out[3] = dbg[8] / reps; out[4] = dbg[9] / reps; out[5] = dbg[10] / reps; out[6] = dbg[13];
    out[7] = dbg[11]; out[8] = dbg[12]; out[9] = dbg[15]; out[10] = dbg[6];
    for (int i = 0; i < kk; ++i) outlam[i] = S.lam[i];
  }
}
int main() {
  long long* d; double* dl; cudaMalloc(&d, 256); cudaMalloc(&dl, 32 * 8);
  cudaFuncSetAttribute(k_iso, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nd : {0, 1}) for (int nt : {128, 512}) for (int kk : {10, 20, 32}) {
    size_t smem = svd_smem_bytes(64, 64, kk, 1);
    k_iso<<<1, nt, smem>>>(kk, 10, nd, d, dl);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[11]; double lam[32];
    cudaMemcpy(h, d, 88, cudaMemcpyDeviceToHost); cudaMemcpy(lam, dl, kk * 8, cudaMemcpyDeviceToHost);
    printf("nearly_diag=%d threads=%d kk=%d: jacobi(30)=%lld chol=%lld ritz(2 sweeps)=%lld [chol %lld solves %lld jac %lld, sweeps %lld/10] (%s) lam0=%.6f\n",
           nd, nt, kk, h[0], h[1], h[2], h[3], h[4], h[5], h[6], cudaGetErrorString(e), lam[0]);
    const double nr = (double)h[6] * (kk + (kk & 1) - 1);
    printf("   per round: param %.0f  bar1 %.0f  elements %.0f  bar2 %.0f cycles\n", h[7] / nr, h[8] / nr, h[9] / nr, h[10] / nr);
  }
  return 0;
}
