/*
 * ircur_b200.h — C-ABI of the B200-native IRCUR hot path.
 *
 * The reference (`/root/reference/pkg/src/ircur`) is a pure Python/numpy
 * package with no FFI layer: its boundary for this path is the Python
 * function `ircur.solver.solve(D, config, observer)` (solver.py:304-416) and
 * the public phase helpers it is built from.  Each export below replaces one
 * piece of that function; the reference-side binding (ctypes, as used by
 * `paper_2010_07422_b200/_capi.py`) is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Plain C types only.  Matrices are device pointers unless stated; D is
 *     row-major with leading dimension `ldd` (elements), BORROWED (read-only,
 *     must outlive the context's use of it).
 *   - Every function returns an ircur_status (0 = OK, <0 = error) and sets a
 *     thread-local message readable with ircur_last_error().
 *   - dtype selects storage AND arithmetic of the strip kernels: F64 data is
 *     processed in fp64 end to end; F32 data in fp32 with fp64 norm
 *     accumulation.  The core SVD/pinv always runs in fp64.
 *   - A context is bound to one device and one stream and is not thread-safe;
 *     independent contexts may share the same D.
 *   - Row sharding: a context may own rows [row0, row0+local_rows) of an
 *     n1 x n2 matrix (multi-GPU); single-GPU callers pass row0=0,
 *     local_rows=n1.
 */
#ifndef IRCUR_B200_H
#define IRCUR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IRCUR_ABI_VERSION 1

typedef enum {
  IRCUR_OK = 0,
  IRCUR_EINVAL = -1,     /* bad argument / config  -> ValueError          */
  IRCUR_ENONFINITE = -2, /* NaN/Inf in D            -> ValueError          */
  IRCUR_ECUDA = -3,      /* CUDA runtime error      -> RuntimeError        */
  IRCUR_ENCCL = -4,      /* collective failure      -> RuntimeError        */
  IRCUR_ENOMEM = -5,     /* device allocation       -> MemoryError         */
  IRCUR_EEMPTY = -6      /* empty D                 -> ValueError          */
} ircur_status;

typedef enum { IRCUR_F32 = 0, IRCUR_F64 = 1 } ircur_dtype;
typedef enum { IRCUR_FIXED = 0, IRCUR_RESAMPLED = 1 } ircur_mode;

typedef struct ircur_ctx* ircur_ctx_t;

/* Library identity. */
int ircur_abi_version(void);
const char* ircur_last_error(void);

/* Create a solver context (workspace for strips' factors, core, SVD scratch,
 * index sets, trace).  max_rows/max_cols bound |I|,|J| (the draw counts m),
 * max_iter bounds the loop.  `stream` is a cudaStream_t (NULL = default).
 * Replaces the allocations solve() makes up front (solver.py:346-356). */
int ircur_ctx_create(ircur_ctx_t* out, int device, int dtype, int64_t n1, int64_t n2,
                     int rank, int max_rows, int max_cols, int max_iter,
                     int64_t row0, int64_t local_rows, void* stream);
int ircur_ctx_destroy(ircur_ctx_t ctx);

/* One pass over the local rows of D: finiteness check, max|D| and (optional)
 * column-major copy used by the column-strip kernel.
 * Replaces matcore.require_finite (matcore.py:70-77, called solver.py:319)
 * and inf_norm (matcore.py:87-91, solver.py:342-344).  Host-blocking. */
int ircur_prepare(ircur_ctx_t ctx, const void* D, int64_t ldd, int make_colmajor,
                  int* all_finite, double* max_abs);

/* Like ircur_prepare, but the column-major copy holds only the columns of
 * the J sets [0, cover_sets) (their union; ~20% of D for 40 iterations at
 * n = 1e5), so the pass writes a fraction of D instead of all of it.  Needs
 * the index sets uploaded first.  Iterations past the covered sets extend
 * the copy automatically (one more pass over D).  Host-blocking. */
int ircur_prepare_sampled(ircur_ctx_t ctx, const void* D, int64_t ldd, int cover_sets,
                          int* all_finite, double* max_abs);

/* The reference's index draws on the host, bit for bit: n_sets pairs
 * I_s = unique(integers(0, n1, m_rows)), J_s = unique(integers(0, n2, m_cols))
 * from a numpy PCG64 Generator whose state is pcg = {state lo, state hi,
 * inc lo, inc hi, has_uint32, uinteger} (rng.bit_generator.state).  Sets are
 * written sorted with strides m_rows / m_cols; counts per set.  pcg_out
 * (optional) receives the state after the draws.  Host only (no device).
 * Replaces sampling.py:93-104 in the order of solver.py:325-329, 362-364. */
int ircur_draw_index_sets(const uint64_t* pcg, int64_t n1, int64_t n2, int m_rows, int m_cols,
                          int n_sets, int64_t* rows, int32_t* row_counts, int64_t* cols,
                          int32_t* col_counts, uint64_t* pcg_out);

/* Upload the pre-generated index sets (host int64, strictly increasing),
 * n_sets consecutive (I_k, J_k) pairs packed with strides max_rows/max_cols.
 * The host draws them with the reference's numpy call sequence
 * (sampling.py:93-104 in the order of solver.py:325-329, 362-364). */
int ircur_set_indices(ircur_ctx_t ctx, int n_sets, const int64_t* rows,
                      const int32_t* row_counts, const int64_t* cols,
                      const int32_t* col_counts);

/* Append n_more index sets after the uploaded ones (same layout as
 * ircur_set_indices); the sampled column-major copy is left as is (later
 * sets extend it on demand).  Lets the host draw the tail of the sequence
 * while the prep pass runs. */
int ircur_append_indices(ircur_ctx_t ctx, int n_more, const int64_t* rows,
                         const int32_t* row_counts, const int64_t* cols,
                         const int32_t* col_counts);

/* Asynchronous prep: ircur_prepare_async launches the pass of ircur_prepare
 * (mode 0/1: make_colmajor) or ircur_prepare_sampled (mode 2, cover_sets)
 * and returns without waiting; ircur_prepare_wait blocks until it is done
 * and reports all_finite / max_abs (ENONFINITE like the blocking calls).
 * Between the two the host may append index sets and queue
 * ircur_slab_sqnorms_async, so its work overlaps the pass over D. */
int ircur_prepare_async(ircur_ctx_t ctx, const void* D, int64_t ldd, int mode, int cover_sets);
/* The same pass in row chunks [row_begin, row_end) of the local rows, in
 * order, starting at 0 (row_begin % 4 == 0): lets the pass over rows already
 * on the device run while the host streams in the rest of D (the caller
 * orders each chunk after its copy, e.g. with an event on the context
 * stream).  The chunk ending at the last row completes the pass like
 * ircur_prepare_async. */
int ircur_prepare_rows_async(ircur_ctx_t ctx, const void* D, int64_t ldd, int mode, int cover_sets,
                             int64_t row_begin, int64_t row_end);
int ircur_prepare_wait(ircur_ctx_t ctx, int* all_finite, double* max_abs);

/* den = ||D(I_s,:)||_F^2, ||D(:,J_s)||_F^2 partial sums of the LOCAL rows
 * for index set s (fp64; host-blocking).  Replaces the pre-loop frob_norm
 * pair of solver.py:331-333 used by the den == 0 early exit (:335-341). */
int ircur_slab_sqnorms(ircur_ctx_t ctx, int set, double* rows_sq, double* cols_sq);
/* Queue the slab norms of set s on the context stream; the next
 * ircur_slab_sqnorms(ctx, s, ...) waits for and returns them. */
int ircur_slab_sqnorms_async(ircur_ctx_t ctx, int set);

/* The device-resident loop, single device (solver.py:358-414): for
 * k = 0..max_iter-1 runs core -> SVD/pinv -> fused strips -> stop check.
 * zetas[k] = gamma**k * zeta0 is evaluated by the caller exactly as the
 * reference does (solver.py:372) and passed in.  mode IRCUR_FIXED uses index
 * set 0 for every k, IRCUR_RESAMPLED set k.  Outputs are host arrays of
 * length max_iter (e_k and per-iteration milliseconds from CUDA events).
 * Host-blocking; stops as soon as e_k <= eps (no per-iteration host sync:
 * the stop flag is written by the device into mapped host memory). */
int ircur_run(ircur_ctx_t ctx, const double* zetas, double eps, int mode, int max_iter,
              int* iterations, int* converged, double* errors, float* iter_ms);

/* Exactly one iteration k on index set `set` with threshold zeta (the
 * observer path, solver.py:410-411).  Returns e_k.  Host-blocking. */
int ircur_iterate(ircur_ctx_t ctx, int k, int set, double zeta, double* e);

/* ---- Row-sharded loop (multi-GPU, one process per GPU) -------------------
 * Each rank's context owns rows [row0, row0+local_rows) of D; index sets and
 * zetas are identical on all ranks.  The caller owns the collectives (NCCL
 * through torch.distributed in paper_2010_07422_b200/dist.py): after each
 * phase it all-reduces (SUM, in place, on the context stream) the exchange
 * buffer named below.  Iteration k:
 *   IRCUR_SHARD_CORE    zero U, write this shard's rows of the thresholded
 *                       core U = (D - T(D - L))(I, J)         -> allreduce U
 *   IRCUR_SHARD_FACTOR  core SVD/pinv of the full U (replicated, bitwise
 *                       identical on every rank); column strip complete
 *                       (local rows); row strip: local partial sums of
 *                       Q_{k+1} = W_r^T R                     -> allreduce Qpart
 *   IRCUR_SHARD_RESID   row strip again: Q_{k+1} = Qpart with Q(:,J) = W^T U,
 *                       residual; local {den_I, res_I, den_J, res_J} sums
 *                                                             -> allreduce scal[0:4]
 *   IRCUR_SHARD_STOP    e_k from scal, stop flag (device + mapped host)
 * Kernels of an iteration after the stop are no-ops, so a rank may run ahead
 * of the stop decision as long as every rank issues the same phases. */
typedef enum {
  IRCUR_SHARD_CORE = 0,
  IRCUR_SHARD_FACTOR = 1,
  IRCUR_SHARD_RESID = 2,
  IRCUR_SHARD_STOP = 3
} ircur_shard_phase_t;

/* Device pointers of the exchange buffers: U (fp64, u_elems), Qpart (context
 * dtype, q_elems), scal (fp64, 4 used). */
int ircur_shard_buffers(ircur_ctx_t ctx, void** U, int64_t* u_elems, void** Qpart,
                        int64_t* q_elems, void** scal);
/* Start a sharded loop (L_0 = 0, flags cleared); like the prologue of ircur_run. */
int ircur_shard_reset(ircur_ctx_t ctx);
/* Enqueue one phase of iteration k (index set `set`, threshold zeta). */
int ircur_shard_phase(ircur_ctx_t ctx, int phase, int k, int set, double zeta, double eps,
                      int max_iter);
/* Non-blocking: device stop flag and completed-iteration count (mapped host
 * memory written by the STOP phase / the single-device loop). */
int ircur_poll(ircur_ctx_t ctx, int* done, int* iterations);
/* Host-blocking end of a sharded loop: iterations, converged, e_k and
 * per-iteration milliseconds (as ircur_run returns them). */
int ircur_shard_finish(ircur_ctx_t ctx, const double* zetas, int mode, int* iterations,
                       int* converged, double* errors, float* iter_ms);

/* Native sharded loop.  ircur_nccl_unique_id writes one NCCL unique id per
 * 128 bytes of `bytes` on one rank; every rank passes n_ids (1 or 2) of them
 * to ircur_shard_comm_init (a collective: all ranks call it together) to give
 * its context its communicators (the process's own NCCL, found with dlopen;
 * no link-time dependency).  ircur_shard_run then runs the whole loop after
 * ircur_prepare / ircur_slab_sqnorms: per iteration the four phases above
 * with the three all-reduces, run-ahead `ahead` iterations, and the trace as
 * ircur_shard_finish returns it; *launched = iterations issued (min(max_iter,
 * K + ahead) on every rank).  overlap = 1 with two communicators (fp32,
 * strips3 eligible): the single-GPU two-stream schedule, the SVD of k + 1
 * (after the all-reduces of the sampled Q partials and of U) beside the
 * strips of k (all-reduces of the Q partials and the 4 sums), one
 * communicator per stream. */
int ircur_nccl_unique_id(void* id, int64_t bytes);
/* Before the prep pass (zeta0 > 0, fp32, two communicators): queue the
 * overlapped loop's chain(0) and chain(1) (core, all-reduce of U, Gram, SVD;
 * sampled(0) from D) on the chain stream, beside the pass, which then waits
 * for the SVD gate and leaves the cluster's SMs free; ircur_shard_run with
 * overlap continues at strips(0).  No-op outside that envelope. */
int ircur_shard_pre_chain(ircur_ctx_t ctx, const void* D, int64_t ldd, double zeta0, double gamma, int mode,
                          int max_iter);
int ircur_shard_comm_init(ircur_ctx_t ctx, const void* ids, int n_ids, int nranks, int rank);
int ircur_shard_run(ircur_ctx_t ctx, const double* zetas, double eps, int mode, int max_iter, int ahead,
                    int overlap, int* iterations, int* converged, double* errors, float* iter_ms,
                    int* launched);

/* Final CUR/sparse strips of the last completed iteration, fp64, written to
 * device or host pointers (cudaMemcpyDefault):  C  local_rows x |J|,
 * R |I_loc| x n2, S_rows |I_loc| x n2, S_cols local_rows x |J| (row-major).
 * Replaces CurFactors.C/R and SparseEstimate (solver.py:375-391). Any
 * pointer may be NULL. */
int ircur_get_strips(ircur_ctx_t ctx, double* C, double* R, double* S_rows, double* S_cols);

/* Core pinv factor of the last iteration (PinvFactor, matcore.py:142-165):
 * W |I| x k, sigma k, V |J| x k, inv_sigma k (fp64, host or device), plus
 * k = min(rank, |I|, |J|) and the final |I|, |J|. */
int ircur_get_core(ircur_ctx_t ctx, double* W, double* sigma, double* V,
                   double* inv_sigma, int* k, int* n_rows, int* n_cols);

/* Rank-r factors of L = P Q of the last iteration: P = C V diag(inv_sigma)
 * (local_rows x rank), Q = W^T R (rank x n2), in the context dtype. */
int ircur_get_factors(ircur_ctx_t ctx, void* P, void* Q);

/* Zero-copy access to the same factors: device pointers of P^T (rank x
 * local_rows, leading dimension *ldp) and Q (rank x n2, *ldq) inside the
 * context.  Valid until the next ircur_run / ircur_shard_reset. */
int ircur_factor_buffers(ircur_ctx_t ctx, void** Pt, int64_t* ldp, void** Qt, int64_t* ldq);

/* Stream L = P Q for the local rows into L (device, row-major, ldl),
 * out_dtype IRCUR_F32/F64.  Replaces solver.materialize (solver.py:211-213)
 * with a K=rank streaming writer. */
int ircur_materialize(ircur_ctx_t ctx, void* L, int64_t ldl, int out_dtype);

/* Measurement hooks for bench.py: per-phase CUDA events recorded on the
 * context stream around core | SVD | strips | stop-check of each iteration
 * (ircur_set_profiling), read back as per-iteration milliseconds, plus the
 * number of iterations launched and kernels launched by the last ircur_run. */
int ircur_set_profiling(ircur_ctx_t ctx, int on);
/* One whole single-GPU solve, natively (the host sequence of
 * paper_2010_07422_b200.solve_device, solver.py:304-416): the index draws
 * from the PCG64 state `pcg` (6 words, see ircur_draw_index_sets; the first
 * sets before the prep pass, the rest while it runs), the column-major copy
 * plan (colmajor 0 none, 1 full, 2 sampled, 3 full when the covered columns
 * exceed 70% of D, else sampled), the prep pass, the den == 0 check, the
 * threshold schedule zeta_k = gamma^k zeta0 (zeta0 <= 0: max|D|) and the loop.
 * rows/cols receive the drawn sets (max_iter x max_rows / max_cols, zero
 * padded; one set in fixed mode), errors / iter_ms max_iter entries.  Results
 * are then read with ircur_get_strips etc. like after ircur_run.  The whole
 * call runs without the caller's interpreter (batched problems from several
 * host threads). */
int ircur_solve(ircur_ctx_t ctx, const void* D, int64_t ldd, const uint64_t* pcg, double zeta0, double gamma,
                double eps, int mode, int max_iter, int colmajor, int64_t* rows, int32_t* row_counts,
                int64_t* cols, int32_t* col_counts, int* iterations, int* converged, double* errors,
                float* iter_ms, double* zeta0_used, int* copy_mode, int* zero_state);

/* Device-side gaps of the last solve while profiling (ms): upload of the
 * index sets -> prep begin, prep pass, prep end -> slab norms queued, slab
 * end -> ircur_run, ircur_run -> first loop kernel; -1 when not recorded. */
int ircur_get_marks(ircur_ctx_t ctx, float* ms);
/* Diagnostic counters of the last ircur_run: 0 = entries of the next
 * iteration's gathers that differ from the sampled-factor kernel's
 * (IRCUR_SAMPLED_CHECK=1; 0 means it reproduces the strips bitwise);
 * 1 = whether the run took the overlapped two-stream loop (IRCUR_OVERLAP),
 * 2 = the strip kernel of the process's last strip launch (1, 2, 3 = the FFMA
 * kernels, 5 / 6 = the opt-in tensor-core kernels),
 * 4 = whether the last strips3 launch ran its residual pass on the tensor
 * cores (tcgen05; the default for row strips of >= 32768 positions). */
int ircur_debug_counter(ircur_ctx_t ctx, int which, long long* value);
/* Loop selection for the following runs on ctx: 1 = the overlapped loop
 * (SVD of k + 1 beside the strips of k on two streams) where eligible, 0 =
 * the sequential loop, -1 = the default (IRCUR_OVERLAP at creation, else 1).
 * Callers that run several solves concurrently on one GPU pass 0: the
 * overlapped loop sizes its strip grid for a GPU of its own. */
int ircur_set_overlap(ircur_ctx_t ctx, int mode);
/* Stop tolerance of the following ircur_iterate calls (ircur_run and
 * ircur_solve take it as an argument).  fp32 strips run on the tensor cores
 * (kernels_strips5.cu) only when eps >= 1e-6 (IRCUR_S5_MIN_EPS): their
 * 3-term tf32 products put the residual's floor near 3e-7, so tighter
 * tolerances take the FFMA kernel, whose floor is fp32 round-off. */
int ircur_set_target_eps(ircur_ctx_t ctx, double eps);
/* Overlapped, profiled run: per iteration k, ms[5k..5k+4] = start and end
 * of the chain (core .. SVD), start and end of the strips, and the end of
 * the sampled-factor kernel of k, relative to the first chain's start
 * (diagnostics of the two-stream schedule; -1 where not recorded). */
int ircur_get_timeline(ircur_ctx_t ctx, int n_iters, float* ms);
int ircur_get_profile(ircur_ctx_t ctx, int n_iters, int* launched_iters,
                      long long* kernel_launches, float* core_ms, float* svd_ms,
                      float* strips_ms, float* finalize_ms);

/* Subspace-iteration steps the core SVD needed in each of the first n_iters
 * iterations of the last run (diagnostics). */
int ircur_get_svd_steps(ircur_ctx_t ctx, int n_iters, int* steps);

/* Accumulated clock64 cycles per phase of the core-SVD kernel while
 * profiling is on: [product | reduction | Rayleigh-Ritz | rotation |
 * next block | all-gather | final stage | loop overhead] (diagnostics). */
int ircur_get_svd_phase_cycles(ircur_ctx_t ctx, long long* cycles32, int reset);

/* Stateless variant: stream L = P Q from caller-held factors Pt (rank x
 * nrows, row stride ldp) and Q (rank x n2, row stride ldq), dtype
 * IRCUR_F32/F64, into L (nrows x n2, ldl) in out_dtype. */
int ircur_materialize_factors(const void* Pt, int64_t ldp, const void* Q, int64_t ldq,
                              int64_t nrows, int64_t n2, int rank, int dtype, void* L,
                              int64_t ldl, int out_dtype, void* stream);

/* BASELINE.json synthetic generator on the device (configs 1-5): rows
 * [row0, row0+nrows) of D = W V^T + S, S = Bernoulli(alpha) support with
 * U[-amp_a, amp_a] values, drawn from the SAME numpy PCG64 stream the host
 * generator uses (oracle/ircur_oracle.py baseline_problem): cell (i,j) takes
 * mask draw i*n2+j and value draw n1*n2+i*n2+j after `pcg` = {state_lo,
 * state_hi, inc_lo, inc_hi}.  Any row sharding reproduces the same matrix.
 * W (n1 x rank) and V (n2 x rank) are fp64 device arrays.  If D is NULL only
 * the statistics are computed: max|L| and the quantised sum
 * sum(rint(|L| * 2^24)) from which a = mean|L| is derived order-free.
 * Host-blocking. */
/* Compact SVD of L = P Q from the device factors (Pt: rank x n1 with leading
 * dimension ldp, Q: rank x n2, ldq; dtype F32/F64): W (n1 x rank, row-major
 * fp64, device), sigma (rank), V (n2 x rank); *k_out = columns kept after
 * dropping sigma < 1e-14 sigma_max.  Replaces convert.cur_to_svd
 * (convert.py:21-48) with r-wide work: Cholesky-QR of P and Q^T and a
 * one-sided Jacobi SVD of the r x r middle factor.  rank <= 16. */
/* BIN matrix files (mio.py:66-121: "IRCM", int32 rows/cols, column-major
 * float64).  ircur_bin_block_to_rowmajor transposes a staged column block
 * (device, nr x nc, column-major fp64, leading dimension ldsrc) into
 * row-major dst (dst_dtype F32/F64, leading dimension ldd) and atomically
 * keeps in *first_bad (device, init ~0) the smallest flat file index
 * (col * file_rows + row, with the block at file rows row0.., cols col0..)
 * of a non-finite value.  ircur_rowmajor_to_bin_block is the inverse for
 * writers (dst: column-major fp64, leading dimension nr). */
int ircur_bin_block_to_rowmajor(const double* src, int64_t ldsrc, int64_t nr, int64_t nc, void* dst,
                                int64_t ldd, int dst_dtype, int64_t file_rows, int64_t row0,
                                int64_t col0, unsigned long long* first_bad, void* stream);
int ircur_rowmajor_to_bin_block(const void* src, int64_t lds, int src_dtype, int64_t nr, int64_t nc,
                                double* dst, void* stream);

/* Background / foreground frames of the video pipeline (cli.py:217-230,
 * mio.py:177-187) for frames [t0, t0 + nt) of D (pixels x frames, row-major,
 * device, same dtype as the factors): bg = clamp(rint(L)), fg =
 * clamp(rint(|D - L| * 255 / peak_t)) as uint8 frames (t, y, x) with pixel
 * (x, y) at row y + x * height.  peaks: nt u64 of device scratch. */
int ircur_video_frames(const void* Pt, int64_t ldp, const void* Q, int64_t ldq, const void* D,
                       int64_t ldd, int dtype, int64_t n1, int height, int width, int64_t t0,
                       int nt, int rank, unsigned long long* peaks, uint8_t* bg, uint8_t* fg,
                       void* stream);

/* Batched independent problems (BASELINE cfg4; the reference's trial pool,
 * cli.py:117-125).  ircur_batch_prepare runs ircur_solve's host sequence up to
 * the loop (draws, copy plan, prep pass, den check, schedule) on one context;
 * *zero_state = 1 means the den == 0 exit (no loop needed).
 * ircur_batched_run then runs the loops of n prepared fp32 contexts (same
 * rank, mode, max_iter, device) together on `stream`: one launch per phase
 * per iteration over all problems (core, Gram + SVD with one svd_cs-CTA
 * cluster per problem -- 0 picks the smallest that fits -- strips, stop
 * test).  Each problem's trace and state are those of its own sequential
 * solve with that cluster size; iterations / converged (n) and errors
 * (n x errors_ld) receive the traces; the factors stay on each context.
 * strip_ms (optional): device time of the batched strip launches, summed. */
int ircur_batch_prepare(ircur_ctx_t ctx, const void* D, int64_t ldd, const uint64_t* pcg, double zeta0,
                        double gamma, double eps, int mode, int max_iter, int colmajor, int64_t* rows,
                        int32_t* row_counts, int64_t* cols, int32_t* col_counts, double* zeta0_used,
                        int* copy_mode, int* zero_state);
/* ircur_batch_prepare over n contexts on `threads` host threads (each context
 * on its own stream).  Per problem p: D[p] (leading dimension ldd), the PCG64
 * state pcg[6p .. 6p + 5], zeta0[p] (<= 0: max|D|), gamma[p], eps[p]; index
 * buffers rows + p n_sets max_rows, row_counts + p n_sets (same for cols);
 * zeta0_used / copy_mode / zero_state [p].  The threads draw and queue every
 * problem's uploads, prep pass and slab norms without host waits; one pass
 * then reads the results.  Entries past each set's count in the index buffers
 * are left unwritten.  *failed = the first failing problem (-1 if none). */
int ircur_batch_prepare_many(ircur_ctx_t* ctxs, int n, const void* const* D, int64_t ldd, const uint64_t* pcg,
                             const double* zeta0, const double* gamma, const double* eps, int mode, int max_iter,
                             int colmajor, int64_t* rows, int32_t* row_counts, int64_t* cols, int32_t* col_counts,
                             double* zeta0_used, int* copy_mode, int* zero_state, int threads, int* failed);
int ircur_batched_run(ircur_ctx_t* ctxs, int n, void* stream, int svd_cs, int* iterations, int* converged,
                      double* errors, int errors_ld, float* strip_ms);
/* The factored form of host-given C (n1 x |J|) and R (|I| x n2), fp64 device
 * row-major: P^T = (C VS)^T (k x n1) with VS = V diag(inv_sigma) (|J| x k,
 * row-major) and Q = W^T R (k x n2) with W (|I| x k, row-major); what
 * convert.py:21-48 multiplies out, as two HBM-bound skinny products
 * (no cuBLAS).  k <= 16, |I| k <= 6144. */
int ircur_cur_to_factors(const double* C, int64_t ldc, const double* R, int64_t ldr, const double* VS,
                         const double* W, int64_t n1, int64_t n2, int mI, int nJ, int k, double* Pt,
                         int64_t ldp, double* Qt, int64_t ldq, void* stream);
int ircur_factors_to_svd(const void* Pt, int64_t ldp, const void* Q, int64_t ldq, int64_t n1,
                         int64_t n2, int rank, int dtype, double* W, double* sigma, double* V,
                         int* k_out, void* stream);

int ircur_gen_baseline(void* D, int dtype, int64_t ldd, int64_t n1, int64_t n2,
                       int64_t row0, int64_t nrows, int rank, const double* W,
                       const double* V, double alpha, double amp_a, const uint64_t* pcg,
                       double* max_abs_L, int64_t* qsum_abs_L, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IRCUR_B200_H */
