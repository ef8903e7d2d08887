// Per-iteration kernels of the IRCUR hot path (declarations + arg structs).
#pragma once
#include "ircur_common.cuh"

namespace ircur {

// ------------------------------------------------------------------ core
// U = (D - T_zeta(D - L_k))(I, J) in fp64, plus the compact gathers
// Pold_I (|I| x R) = P_k(I,:) and Qold_J (|J| x R) = Q_k(:,J)^T used by the
// strip kernels.  Mirrors solver.py:375-382 restricted to I x J.
template <typename T>
struct CoreArgs {
  const T* D; int64_t ldd; int64_t row0;      // local rows [row0, row0+nloc)
  const int* I; int mI;                        // local sampled rows (global ids)
  const int* J; int nJ;
  const T* Pt; int64_t ldp;                    // P_k^T  (R x nloc)
  const T* Qt; int64_t ldq;                    // Q_k^T  (R x n2)
  T zt;
  double* U; int ldu;                          // mI x nJ (rows start at upos0)
  int upos0;                                   // position of the first local row inside I (row sharding)
  T* PoldI; T* QoldJ;                          // mI x R, nJ x R
  int* rowmap; int* colmap;                    // position -> index maps (set here, cleared by finalize)
  const int* done;
  // presampled: PoldI / QoldJ already hold P(I,:), Q(:,J) (sampled_factors_kernel
  // of the previous iteration), read instead of gathering from Pt / Qt.
  // verify: gather from Pt / Qt as usual but count entries that differ from
  // what PoldI / QoldJ already hold (a check of the sampled kernel).
  int presampled; int verify; unsigned* mismatches;
};

// ---------------------------------------------------------------- strips
// One "strip" = a set of sampled lines (rows I of D, or columns J of D read
// from the column-major copy) times every position along the other axis.
// For each entry: l = <lineA[k], Bold[:,x]>, c = d - T_zeta(d - l)
// (Phase I+II), the new factor Fnew[:,x] = sum_k lineW[k] c[k][x] (Q = W^T R
// or P = C V Sigma^+), then the residual c - <lineRes[k], Fnew[:,x]> whose
// squared norm, with ||d||^2, feeds e_k (solver.py:393-400).
template <typename T>
struct StripDesc {
  const T* src; int64_t line_stride; int64_t pos_stride;
  int bulk_ok;                                 // line segments are 16B aligned: TMA bulk copies
  const int* lines; int line_off; int nk;      // element (k, x) = src[(lines[k]-line_off)*line_stride + x*pos_stride]
  int npos;
  const T* lineA; const T* lineW; const T* lineRes;  // nk x R each
  const T* Bold; int64_t ldb;                  // R x npos (padded ld, 16B aligned rows)
  T* Fnew; int64_t ldf;                        // R x npos
  const int* omap;                             // npos: index into otherF, or -1
  const T* otherF;                             // (other set size) x R
  int tiles;                                   // ceil(npos / TX)
  // kStripFull: Phase I/II + factor + override + residual in one pass.
  // Row sharding splits the row strip in two launches around the all-reduce
  // of Q: kStripPartial writes the un-overridden local partial sums
  // (Fnew = sum over the local lines), kStripFinish re-thresholds the tile,
  // takes Fnew from Fsrc (the all-reduced sums), applies the override and
  // accumulates the residual.
  int mode;
  const T* Fsrc; int64_t ldfs;                 // kStripFinish only: R x npos
  // the core U = (D - S)(I, J): entry (line k, position with omap e) at
  // U[k * u_ls + e * u_ps] (strips5: the I x J entries of the strips)
  const double* U; int64_t u_ls, u_ps;
};
constexpr int kStripFull = 0, kStripPartial = 1, kStripFinish = 2;

template <typename T>
struct StripsArgs {
  StripDesc<T> s[2];                           // [0] row strip, [1] column strip
  T zt;
  int maxl;                                    // max lines per CTA (smem sizing)
  double* partials;                            // per CTA: {den, res}
  const int* done;
  long long* dbg;                              // optional per-phase clock64 totals (CTA 0, thread 0)
  int tc_ok;                                   // the tensor-core kernel may run (the loop's eps is above its floor)
};

// ------------------------------------------------------- sampled factors
// One strip restricted to a list of positions (kernels_sampled.cu): element
// (line k, position x = pos[p] - pos_off) = src[(lines[k] - line_off) *
// line_stride + x * pos_stride]; B(:, x) = B[t * ldb + x]; out: npos x R.
struct SampledStrip {
  const float* src; int64_t line_stride; int64_t pos_stride;
  const int* lines; int line_off; int nk;
  const float* lineA; const float* lineW;      // nk x R
  const float* B; int64_t ldb;
  const int* pos; int pos_off; int npos;
  const int* omap; const float* otherF;         // override: position -> index of the other set
  float* out;
  int zero_override;                           // row-sharded partial sums: overridden positions give 0 (rank > 0)
};
struct SampledArgs {
  SampledStrip s[2];                            // [0] Q(:, J_{k+1}), [1] P(I_{k+1}, :)
  float zt;
  const int* done;
};

// ------------------------------------------------------------- finalize
struct FinalizeArgs {
  const double* partials; int ncta_rows; int ncta_cols;  // ncta_rows = strip CTAs, 4 sums each
  int k; double eps; int max_iter;
  double* errors; int* done; int* iters; int* converged;
  volatile int* host_done; volatile int* host_iters;   // mapped pinned memory (may be null)
  const int* I; int mI; const int* J; int nJ; int64_t row0;
  int* rowmap; int* colmap;                    // cleared back to -1 for this iteration's sets
  double* sums_out;                            // non-null: only reduce the partials into 4 sums here
};

// --------------------------------------------------------------- writeout
template <typename T>
struct WriteoutArgs {
  const T* D; int64_t ldd; int64_t row0; int64_t nloc; int64_t n2;
  const int* I; int mI; const int* J; int nJ;
  const T* Pt; int64_t ldp; const T* Qt; int64_t ldq;
  T zt;
  double* C; double* R; double* Srows; double* Scols;   // device fp64, any may be null
};

}  // namespace ircur
