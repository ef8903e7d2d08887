// Host-visible launcher declarations for the IRCUR kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "kernels_iter.cuh"

namespace ircur {

// Function attributes (dynamic shared memory above 48 KB, non-portable
// cluster sizes) are stored per device context, so they are set once per
// (kernel, device): `mask` is the kernel's static bitmask of devices done.
// Two threads racing here both set the attribute, which is idempotent.
template <typename SetFn>
inline cudaError_t attr_once(std::atomic<unsigned long long>& mask, SetFn&& set) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = set();
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <typename K>
inline cudaError_t smem_attr_once(std::atomic<unsigned long long>& mask, K* kern, int bytes,
                                  bool nonportable_cluster = false) {
  return attr_once(mask, [&] {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess || !nonportable_cluster) return e;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  });
}

struct u128 {
  uint64_t lo, hi;
};

// Core SVD/pinv arguments (kernels_svd.cu).
struct SvdArgs {
  const double* U; int ldu;       // m x n core (row-major)
  const double* G; int ldg;       // n x n Gram scratch (written by gram_kernel)
  int m, n, r, kk;
  const void* warm; int warm_ld; int warm_cols;  // n x warm_cols start block (storage type) or null
  double* W; double* sigma; double* V; double* inv;  // fp64 outputs: m x r, r, n x r, r
  void* Wr; void* PI; void* VS; void* QJ;            // storage-type strip inputs: m x r, m x r, n x r, n x r
  double* scratch;                // 3 x n x 32 doubles (double-buffered block + Ritz block X)
  const int* done;
  int* steps_out;
  double tol; int maxsteps;       // Ritz residual target: max(tol, tol_scale * e_{k-1}) * lambda_1
  int sweeps;                     // Jacobi sweeps per intermediate Rayleigh-Ritz step
  double jac_thr;                 // Jacobi off-diagonal threshold (relative) of those steps
  double tol_scale; const double* prev_err;  // e_{k-1} on the device (null at k = 0)
  uint64_t salt;
  long long* dbg;                 // optional per-phase clock64 totals (8)
  int small_reg;                  // register-resident kk x kk kernels (svd_small_reg.cuh) when kk allows
};

struct GenArgs {
  void* D; int dtype; int64_t ldd; int64_t n1, n2, row0, nrows; int rank;
  const double* W; const double* V;
  double alpha, amp_a;
  u128 st0, inc;
  double* blk_max; long long* blk_qsum;
  int stats_only;
};

template <typename T> cudaError_t launch_core(const CoreArgs<T>& a, int R, cudaStream_t st);
template <typename T> size_t strips_smem_bytes(int maxl, int R);
template <typename T> int strips_pick_cluster(int nk_max, int R);
template <typename T>
cudaError_t launch_strips(const StripsArgs<T>& a, int R, int cs, int num_sms, int* ncta_out, cudaStream_t st);
int strips_tx();
// fp32 two-group kernel (kernels_strips2.cu); cudaErrorNotSupported when the
// sampled lines do not fit its shared-memory stage
cudaError_t launch_strips2(const StripsArgs<float>& a, int R, int num_sms, int* ncta_out, cudaStream_t st);
size_t strips2_smem_bytes(int maxl, int R);
// fp32 64-position single-stage kernel (kernels_strips3.cu); NotSupported when the lines do not fit
cudaError_t launch_strips3(const StripsArgs<float>& a, int R, int num_sms, int* ncta_out, cudaStream_t st);
cudaError_t launch_sampled_factors(const SampledArgs& a, int R, cudaStream_t st);
size_t strips3_smem_bytes(int maxl, int R);
// the fp32 strip launch of `a` runs strips3_kernel (what the sampled-factor
// kernel reproduces bitwise)
bool strips3_selected(const StripsArgs<float>& a, int R);
// fp32 tensor-core kernel (kernels_strips5.cu): 4-CTA clusters, 128-position
// tiles; NotSupported outside its envelope (r <= 10, <= 512 lines, aligned
// line segments, kStripFull)
cudaError_t launch_strips5(const StripsArgs<float>& a, int R, int num_sms, int* ncta_out, cudaStream_t st);
bool strips5_supported(const StripsArgs<float>& a, int R);
// the fp32 strip launch of `a` runs strips5_kernel
bool strips5_selected(const StripsArgs<float>& a, int R);
// fp32 warp-level tensor-core kernel (kernels_strips6.cu): mma.sync tf32,
// 32-position tiles, one CTA per SM; NotSupported outside its envelope
// (r <= 10, <= 512 lines, aligned line segments, kStripFull)
cudaError_t launch_strips6(const StripsArgs<float>& a, int R, int num_sms, int* ncta_out, cudaStream_t st);
bool strips6_supported(const StripsArgs<float>& a, int R);
size_t strips6_smem_bytes(int maxl);
bool strips6_selected(const StripsArgs<float>& a, int R);
// a tensor-core strip kernel (strips5 or strips6) runs for `a`: its factor
// sums are not the FFMA chains the sampled-factor kernel reproduces
inline bool strips_tc_selected(const StripsArgs<float>& a, int R) {
  return strips5_selected(a, R) || strips6_selected(a, R);
}
extern std::atomic<int> g_last_strips_kernel;  // diagnostics (ircur_debug_counter 2)
extern std::atomic<int> g_last_strips3_tc;     // the last strips3 launch's residual ran on tcgen05 (counter 4)
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st);
// ---- batched problems (ircur_batched_run): device arrays of per-problem arguments
template <typename T>
cudaError_t launch_core_batched(const CoreArgs<T>* d_args, int n, int max_total, int R, cudaStream_t st);
cudaError_t launch_finalize_batched(const FinalizeArgs* d_args, int n, cudaStream_t st);
template <typename T>
cudaError_t launch_svd_batched(const SvdArgs* d_args, int n, int max_n, int cs, size_t smem, bool reg,
                               cudaStream_t st);
bool svd_reg_path(const SvdArgs& a);
void set_draw_threads_for_thread(int n);  // draws.cu: per-thread draw parallelism (0 = default)  // the svd_kernel<T, true> instantiation runs (kk <= 8)
// min_row_positions: the narrowest row strip of the batch (the residual
// arithmetic is chosen as launch_strips3 chooses it for a problem of that width)
cudaError_t launch_strips3_batched(const StripsArgs<float>* d_args, int n, int ctas, int maxl, int R,
                                   int min_row_positions, cudaStream_t st);
template <typename T> cudaError_t launch_writeout(const WriteoutArgs<T>& a, int R, cudaStream_t st);
template <typename T, typename O>
cudaError_t launch_materialize(const T* Pt, int64_t ldp, const T* Qt, int64_t ldq, int64_t nloc,
                               int64_t n2, O* L, int64_t ldl, int R, cudaStream_t st);
template <typename T>
cudaError_t launch_prep(const T* D, int64_t ldd, int64_t nloc, int64_t n2, T* Dt, int64_t ldt,
                        unsigned long long* maxbits, int* nonfinite, int num_sms, cudaStream_t st);
template <typename T>
cudaError_t launch_prep_select(const T* D, int64_t ldd, int64_t nloc, int64_t n2, const int* colsel, T* Dt,
                               int64_t ldt, unsigned long long* maxbits, int* nonfinite, int num_sms,
                               cudaStream_t st);
// columns cols[0, ncols) of the row-major D into lines [slot0, slot0 + ncols) of Dt (kernels_prep.cu)
template <typename T>
cudaError_t launch_gather_cols(const T* D, int64_t ldd, int64_t nloc, const int* cols, int ncols, T* Dt,
                               int64_t ldt, int64_t slot0, cudaStream_t st);
template <typename T>
cudaError_t launch_slab_sq(const T* D, int64_t ldd, int64_t row0, int64_t nloc, int64_t n2,
                           const int* I, int mI, const int* J, int nJ, int nb_rows, int nb_cols,
                           double* partials, const T* Dt, int64_t ldt, const int* Jline, cudaStream_t st);
// batched prep pass + slab norms (ircur_batch_prepare_many): one entry per problem
struct PrepBatchArg {
  const void* D; int64_t ldd, nloc, n2, row0;
  void* Dt; int64_t ldt;          // column-major copy (modes 1, 2)
  const int* colsel;              // mode 2: column -> copy line (or -1)
  int mode;                       // 0 scan only, 1 full column-major copy, 2 sampled columns
  unsigned long long* maxbits; int* nonfinite;
  // slab norms of set 0 (ircur_slab_sqnorms_async's geometry)
  const int* I; int mI; const int* J; int nJ; const int* Jline; int use_dt;
  int nb_rows, nb_cols; double* partials;
};
// init, prep pass per mode, slab norms and the gather of n x {max|D|,
// non-finite, rows_sq, cols_sq} into d_res; h_args: a host copy of d_args
template <typename T>
cudaError_t launch_prep_batched(const PrepBatchArg* d_args, const PrepBatchArg* h_args, int n, double* d_res,
                                cudaStream_t st);
size_t svd_smem_bytes(int n, int m, int kk, int cs);
int svd_pick_cluster(int n, int m, int kk);
template <typename T> cudaError_t launch_svd(const SvdArgs& a, int cs, cudaStream_t st,
                                             cudaEvent_t after_gram = nullptr);
cudaError_t launch_gen(const GenArgs& a, int64_t* nblocks_out, cudaStream_t st);
int64_t gen_blocks(int64_t nrows, int64_t n2);

}  // namespace ircur
