/*
 * randutv.h -- C ABI of the B200-native randUTV hot path.
 *
 * randUTV (Martinsson, Quintana-Ortí, Heavner, arXiv 1703.00998) factors a
 * dense fp64 m x n matrix as  A = U T V^T  with U, V orthogonal and T upper
 * triangular (Eq. eq:defUTVpre), one block of b columns per
 * step, following the efficient algorithm of Fig. fig:randUTV
 * (PAPER.md:919-989).  Every step of the computation runs in the library's
 * own sm_100a CUDA kernels.
 *
 * Conventions shared by every entry point
 *   - Matrices are fp64 (double), COLUMN-MAJOR: element (i, j) of a matrix
 *     with leading dimension ld is p[i + j*ld].
 *   - Pointers may be CUDA device pointers or host pointers, as stated per
 *     function.  The caller owns every buffer; the library never frees them.
 *   - ``stream`` arguments are cudaStream_t values passed as void*; NULL means
 *     cudaStreamPerThread.  Functions returning after completion say so.
 *   - Return value (LAPACK ``info`` style): 0 = success; -k = argument k
 *     (1-based, in the order of randutv_factor's parameter list) is invalid;
 *     RANDUTV_ERR_* (> 0) below otherwise.  randutv_strerror() names them.
 *   - The library keeps one cached device workspace (and one staging buffer
 *     for host-buffer calls) per device, grown on demand.  Host threads
 *     serialise on a mutex while they enqueue, and on the device every call's
 *     work is ordered after the previous call's on the same device (the call's
 *     stream first waits on an event recorded at the end of the previous
 *     call), so concurrent calls from several threads or streams never share
 *     the cached workspace at the same time.  Each device's kernel attributes
 *     are set on first use on that device.
 */
#ifndef RANDUTV_H
#define RANDUTV_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RANDUTV_API __attribute__((visibility("default")))
#else
#define RANDUTV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RANDUTV_OK 0
#define RANDUTV_ERR_NONFINITE 1   /* A holds NaN or Inf                */
#define RANDUTV_ERR_CUDA 2        /* a CUDA runtime error                             */
#define RANDUTV_ERR_NOMEM 3       /* device allocation failed                         */
#define RANDUTV_ERR_NCCL 4        /* NCCL error, or a collective timed out (multi-GPU) */
#define RANDUTV_ERR_UNSUPPORTED 5 /* shape outside this build                         */

#define RANDUTV_MAX_B 512

/* Options of randutv_factor_ex.  Zero-initialise, then set what you need. */
typedef struct randutv_opts {
  void* stream;           /* cudaStream_t to enqueue on (NULL: per-thread stream)          */
  double tol;             /* > 0: stop after a step once ||T(I3,J3)||_F <= tol ||A||_F       */
  int32_t no_reortho;     /* 0 (default): re-orthonormalise Y before every X Y in the power
                             loop (R5); 1: plain power loop      */
  int32_t qr_mode;        /* 0 (default): panel QRs by CholeskyQR2 + Householder
                             reconstruction, column-by-column Householder as the fallback
                             for ill-conditioned panels (R20); 1: Householder only */
  void* workspace;        /* optional caller device workspace (NULL: library cache)        */
  size_t workspace_bytes; /* its size; must be >= randutv_workspace_size_ex(...)           */
  int32_t oversample;     /* p >= 0: over-sampled sketch (Remark remark:positivep,
                             PAPER.md:1124-1142; Fig. fig:stepUTVoversampling): G has
                             b + p_i columns, p_i = min(p, n_i - b), and QR(Y) acts on the
                             b dominant left singular vectors of the extended Y.  0 = the
                             paper's Fig. fig:randUTV.  b + p <= RANDUTV_MAX_B.  Honoured by
                             every factorization entry point incl. randutv_factor_dist */
  int32_t reserved1;
} randutv_opts;

/* Diagnostics filled by randutv_factor_ex (may be NULL). */
typedef struct randutv_info {
  int64_t k_done;       /* columns processed: n for a full factorisation                 */
  int32_t steps;        /* randomised steps taken (the ``if`` branch of P:939)           */
  int32_t final_block;  /* 1 if the final SVD block (``else`` branch) ran         */
  int32_t max_sweeps;   /* most Jacobi sweeps any small SVD needed                       */
  int32_t qr_fallbacks; /* panel QRs / re-orthonormalisations that took the Householder
                           fallback (qr_mode 0)                                           */
  double trailing_fro;  /* ||T(k_done+1:m, k_done+1:n)||_F (0 for a full factorisation)  */
  double a_fro;         /* ||A||_F                                                        */
} randutv_info;

/*
 * randutv_factor -- A = U T V^T  (Fig. fig:randUTV).
 *
 *  1 m, 2 n    sizes >= 1.  m < n (fat) follows the Remark "The case m < n"
 *              (PAPER.md:905-915): the final block is reduced by a QR of its rows
 *              and then k_done = m (single-GPU entry points; randutv_factor_dist
 *              needs n <= m)
 *  3 A         m x n input, leading dimension 4 lda >= m.  Read only.  Host or
 *              device memory.  May alias T when lda == m (in-place).
 *  5 b         block size, 1 <= b <= RANDUTV_MAX_B
 *  6 q         power-iteration steps, q >= 0
 *  7 seed      Philox key of the Gaussian sketches G (R2)
 *  8 k_stop    0 = full factorisation; > 0 = stop before the first step whose
 *              offset b(i-1) >= k_stop (so k_done = b*ceil(k_stop/b))
 *  9 U         m x m output (ld = m) or NULL
 * 10 T         m x n output (ld = m), required.  On return T is upper
 *              triangular with exact zeros below the diagonal over the
 *              processed columns; each processed b x b diagonal block is
 *              diagonal, non-negative and non-increasing.
 * 11 V         n x n output (ld = n) or NULL.  U and V must both be given or
 *              both be NULL; NULL selects the paper's "no orthonormal
 *              matrices" mode.
 * U, T, V must all be host or all be device memory.  Host buffers are staged
 * through device memory inside the call (a T-only call on a page-locked T
 * streams T's finished column blocks back while the factorization goes on).
 * Returns after completion; on an error return the contents of U, T, V are
 * undefined (T may be partly written), A is never modified unless T aliases it.
 */
RANDUTV_API int randutv_factor(int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int32_t q, uint64_t seed,
                   int64_t k_stop, double* U, double* T, double* V);

/* As randutv_factor, with options and diagnostics.  Device pointers are
 * processed on opts->stream.  The host waits on that stream: once after
 * validating A (non-finite scan); once per randomized step in qr_mode 0 for
 * the sketch side's CholeskyQR decisions (an event after QR(Y), read while the
 * P = T W_v GEMM runs); once per step when opts->tol > 0 (early-stop test);
 * once after the loop for the column panels' CholeskyQR decisions; and once at
 * the end when info != NULL.  The small SVDs and folds after the loop are
 * enqueued only, so with info == NULL the call returns before they complete
 * (synchronise opts->stream before reading T).  With host buffers it returns
 * after completion. */
RANDUTV_API int randutv_factor_ex(const randutv_opts* opts, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b,
                      int32_t q, uint64_t seed, int64_t k_stop, double* U, double* T, double* V,
                      randutv_info* info);

/* Device workspace bytes randutv_factor_ex needs for this shape
 * (with_uv != 0: U and V requested). */
RANDUTV_API size_t randutv_workspace_size(int64_t m, int64_t n, int64_t b, int32_t q, int32_t with_uv);
/* The same with over-sampling p (randutv_opts.oversample). */
RANDUTV_API size_t randutv_workspace_size_ex(int64_t m, int64_t n, int64_t b, int32_t q, int32_t with_uv,
                                             int32_t oversample);

RANDUTV_API const char* randutv_strerror(int code);
RANDUTV_API const char* randutv_version(void);

/* ---------------------------------------------------------------------------
 * Component entry points (device pointers only, asynchronous on ``stream``).
 * They expose the kernels the factorisation is built from so that each can be
 * checked against the oracle on the same bytes.
 * ------------------------------------------------------------------------ */

/* G (rows x cols, ld ldg) = the step's Gaussian test matrix, PAPER.md:941:
 * Philox4x32-10 with key (lo32 seed, hi32 seed), counter (row/2, col, step,
 * purpose), Box-Muller (R2). */
RANDUTV_API int randutv_gaussian(double* G, int64_t ldg, int64_t rows, int64_t cols, uint64_t seed, uint32_t step,
                     uint32_t purpose, void* stream);

/* C = alpha op(A) op(B) + beta C on the FP64 tensor cores (DMMA).
 * transa/transb: 0 = N, 1 = T.  op(A) is M x K, op(B) K x N, C M x N. */
RANDUTV_API int randutv_dgemm(int32_t transa, int32_t transb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream);

/* Unpivoted Householder QR of the m x b panel in V (ld ldv, m >= b), in place
 * (dlarfg sign convention, R3).  On return V holds
 * the explicit unit-lower-trapezoidal reflectors, R (b x b, ld ldr) the upper
 * triangular factor with zeros below, tau[b] the scalars and Tw (b x b, ld
 * ldt) the forward compact-WY factor: H_1...H_b = I - V Tw V^T. */
RANDUTV_API int randutv_panel_qr(int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
                     double* Tw, int64_t ldt, void* stream);

/* randutv_panel_qr with the algorithm chosen: mode 0 = CholeskyQR2 of the panel
 * followed by the Householder reconstruction of Ballard et al. (same V, R, tau,
 * Tw in exact arithmetic; R20), falling back to mode 1 when the panel
 * is too ill-conditioned (then *fallback = 1, else 0; fallback may be NULL);
 * mode 1 = column-by-column Householder (cluster leaf kernel + DMMA updates).
 * Synchronises ``stream`` once in mode 0 (the fallback decision).  10 mode. */
RANDUTV_API int randutv_panel_qr_ex(int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
                        double* Tw, int64_t ldt, int32_t mode, int32_t* fallback, void* stream);

/* Batched SVD of ``batch`` k x k matrices: R_i at R + i*strideR
 * (ld ldr) = Us_i diag(D_i) Vs_i^T, D_i >= 0 non-increasing.  D is batch x k,
 * Us and Vs are batch consecutive k x k blocks (ld k).  sweeps (may be NULL)
 * receives the Jacobi sweep count per matrix. */
RANDUTV_API int randutv_small_svd_batched(int32_t batch, int32_t k, const double* R, int64_t ldr, int64_t strideR, double* D,
                              double* Us, double* Vs, int32_t* sweeps, void* stream);

/* Randomized SVD (Remark remark:RSVD; NEXT row 3 of
 * SURVEY.md §8(f)): A (m x n, device, ld lda) ~ U diag(D) V^T with U (m x b,
 * ld ldu) and V (n x b, ld ldv) orthonormal, D (b, non-increasing) -- device
 * outputs.  G is the step-0 Philox draw of randutv_factor (m x (b+p),
 * p = opts->oversample); Y = (A^T A)^q A^T G with opts->no_reortho honoured;
 * Q = orth(Y) by the panel QR (opts->qr_mode); B = A Q = Q_B R_B; R_B = Us D Vs^T;
 * U = Q_B Us(:,1:b), V = Q Vs(:,1:b).  Requires b + p <= min(m, n) and
 * <= RANDUTV_MAX_B.  Asynchronous on opts->stream except for the panel QRs'
 * fallback decisions.  Errors: -1 opts, -2 m, -3 n, -4 A, -5 lda, -6 b (+p),
 * -7 q, -9 U/ldu, -11 D, -12 V/ldv. */
RANDUTV_API int randutv_rsvd(const randutv_opts* opts, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b,
                             int32_t q, uint64_t seed, double* U, int64_t ldu, double* D, double* V, int64_t ldv);

/* ---------------------------------------------------------------------------
 * Multi-GPU.  A and T are distributed in 1-D
 * block-cyclic column blocks of width b: global column block j (columns
 * j*b .. min((j+1)b, n)-1) lives on rank j mod nranks; a rank stores its blocks
 * in increasing j, contiguously, as an m x n_loc column-major matrix
 * (n_loc = randutv_dist_local_cols).  Per step the ranks exchange, through the
 * communicator: the b x b Grams of the CholeskyQR steps, Z = X Y (m_i x b),
 * the top b x b block of Q1, P = T(:,J) W_v (m x b) (allreduce), and the
 * panel's (W_u, T_u, R11) (broadcast from the owner of the block).
 * ------------------------------------------------------------------------ */
#define RANDUTV_NCCL_ID_BYTES 128
typedef struct randutv_comm randutv_comm;

/* 128-byte NCCL unique id (rank 0 creates it; the caller distributes it, e.g.
 * with torch.distributed).  NCCL is loaded at run time (the process's
 * libnccl.so.2, e.g. torch's); RANDUTV_ERR_NCCL if unavailable. */
RANDUTV_API int randutv_nccl_unique_id(void* id_out);
/* NCCL communicator for ``rank`` of ``nranks`` on the current CUDA device
 * (collective: every rank must call it).  Released by randutv_comm_destroy.
 * Failure handling: every host wait of randutv_factor_dist polls
 * ncclCommGetAsyncError; an asynchronous error, or a wait longer than
 * RANDUTV_NCCL_TIMEOUT_S seconds (read at creation, default 600) -- e.g. a peer
 * that died -- aborts the communicator (ncclCommAbort) and the call returns
 * RANDUTV_ERR_NCCL; later calls on an aborted communicator return
 * RANDUTV_ERR_NCCL at once (destroy it and create a new one). */
RANDUTV_API int randutv_comm_init_nccl(int32_t nranks, int32_t rank, const void* id, randutv_comm** out);
/* Loopback communicator: this process drives all ``nranks`` ranks on the
 * current device, each with its own shard; collectives are device copies/sums
 * in fixed rank order between bulk-synchronous phases (no kernel waits on
 * another rank).  It checks the distributed arithmetic on one GPU. */
RANDUTV_API int randutv_comm_init_loopback(int32_t nranks, randutv_comm** out);
RANDUTV_API int randutv_comm_destroy(randutv_comm* comm);
/* Collectives issued on ``comm`` since its creation (one per call of the
 * factorization, whatever the number of local ranks) and their payload per
 * rank in bytes: [0] allreduce, [1] broadcast, [2] allgather (either pointer
 * may be NULL).  Returns 0, or RANDUTV_ERR_NCCL if the communicator was
 * aborted. */
RANDUTV_API int randutv_comm_stats(const randutv_comm* comm, long long* counts, long long* bytes);
/* Ranks driven by this process: returns their count (1 for NCCL, nranks for
 * loopback), writes the world size and up to max_ranks rank ids. */
RANDUTV_API int randutv_comm_local_ranks(const randutv_comm* comm, int32_t* world, int32_t* ranks_out,
                                         int32_t max_ranks);
/* Host-only layout queries (no GPU): local column count of ``rank`` and the
 * global column of a rank's local column; -1 on invalid arguments. */
RANDUTV_API int64_t randutv_dist_local_cols(int64_t n, int64_t b, int32_t rank, int32_t nranks);
RANDUTV_API int64_t randutv_dist_global_col(int64_t local_col, int64_t b, int32_t rank, int32_t nranks);

/* Distributed randutv_factor_ex (PAPER.md:919-989 on 1-D column shards).
 *  A_loc[l], T_loc[l]  device shards (m x n_loc, ld lda_loc[l] / ldt_loc[l] >= m)
 *                      of the l-th rank this process drives
 *                      (randutv_comm_local_ranks order).  T_loc may alias A_loc.
 *  U_loc[l], V_loc[l]  NULL (both) for the paper's "no orthonormal matrices"
 *                      mode, else the rank's shards of
 *                      U (m x randutv_dist_local_cols(m, b, ...), ld ldu >= m)
 *                      and V (n x n_loc, ld ldv >= n) in the same block-cyclic
 *                      column layout (U's column block j <-> T's row block j).
 *                      They are formed by backward accumulation (P:951, 958,
 *                      967, 969): W_u is broadcast by the panel owner anyway,
 *                      W_v's row pieces are allgathered once per step at the end.
 * All ranks must pass identical m, n, b, q, seed, k_stop and options.  On
 * return each shard holds that rank's columns of U, T, V; info is identical on
 * all ranks.  Fat inputs (n > m) as on one GPU (Remark "The case m < n"): the
 * final m_i x n_i block's transpose is allgathered and factored redundantly.
 * Errors: -1 opts, -2 comm, -3 m, -4 n,
 * -5 A_loc/lda_loc, -7 b, -8 q, -10 k_stop, -12 U_loc/ldu_loc, -13
 * T_loc/ldt_loc, -16 V_loc/ldv_loc (or only one of U/V given), -1 also for
 * b + opts->oversample > RANDUTV_MAX_B; RANDUTV_ERR_NCCL on a failed
 * collective.  Over-sampling (opts->oversample = p > 0, Remark
 * remark:positivep): the b + p_i column sketch is row-distributed like Y; its
 * projection Z = Q U_R(:, 1:b) is computed redundantly on every rank from the
 * allgathered sketch (Householder QR + Jacobi SVD of R).  Synchronises the stream as randutv_factor_ex does. */
RANDUTV_API int randutv_factor_dist(const randutv_opts* opts, randutv_comm* comm, int64_t m, int64_t n,
                                    const double* const* A_loc, const int64_t* lda_loc, int64_t b, int32_t q,
                                    uint64_t seed, int64_t k_stop, double* const* U_loc, const int64_t* ldu_loc,
                                    double* const* T_loc, const int64_t* ldt_loc, double* const* V_loc,
                                    const int64_t* ldv_loc, randutv_info* info);

/* ---------------------------------------------------------------------------
 * Instrumentation (used by bench.py).
 * ------------------------------------------------------------------------ */

/* Total kernel launches issued by this library since it was loaded. */
RANDUTV_API long long randutv_launch_count(void);

/* Between begin and end every kernel launch is bracketed by CUDA events on its
 * stream.  end synchronises the device and returns, per kernel class, the
 * summed event time in ms, the summed algorithmic flops (2MNK for GEMMs, 0
 * otherwise) and the launch count.  Arrays hold RANDUTV_PROFILE_CLASSES
 * entries (may be NULL); unused trailing classes are zero.  Class names:
 * randutv_profile_class_name(i) (NULL past the last class). */
#define RANDUTV_PROFILE_CLASSES 16
RANDUTV_API int randutv_profile_begin(void);
RANDUTV_API int randutv_profile_end(double* ms, double* flops, long long* launches);
RANDUTV_API const char* randutv_profile_class_name(int cls);
/* Per-launch timeline of the last profile_begin/end window: 4 doubles per
 * launch (class, stream slot numbered by first use, start ms, end ms relative
 * to profile_begin).  Writes up to max_launches entries; returns the count. */
RANDUTV_API long long randutv_profile_timeline(double* out, long long max_launches);

#ifdef __cplusplus
}
#endif

#endif /* RANDUTV_H */
