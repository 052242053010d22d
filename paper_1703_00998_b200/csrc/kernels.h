// Internal host-side launchers of the randUTV sm_100a kernels (not the C-ABI;
// see include/randutv.h for that).  All matrices fp64 column-major, device
// pointers, asynchronous on the given stream.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace rutv {

int num_sms();

// Device-side ordering of C-ABI calls (driver.cu): every call's stream first
// waits for the end of the previous call's work on the same device (the cached
// workspaces and shared side streams are reused), and records that end.
void call_order_begin(cudaStream_t st);
void call_order_end(cudaStream_t st) noexcept;

// ---- prof.cu: launch counting and optional per-class event timing ---------
// Kernel classes of the profiler.  GEMMs are attributed to the role the
// driver is in (set_gemm_role); K_GEMM means "the current role".
enum KClass {
  C_GEMM_SKETCH = 0, C_GEMM_RIGHT = 1, C_GEMM_LEFT = 2, C_GEMM_QR = 3, C_GEMM_OTHER = 4,
  C_QR_LEAF = 5, C_QR_SMALL = 6, C_SVD = 7, C_MISC = 8, K_NCLASS = 9,
  K_GEMM = -1, K_QR = C_QR_LEAF, K_SVD = C_SVD, K_MISC = C_MISC
};
int set_gemm_role(int role);  // returns the previous role
struct GemmRole {
  int prev;
  explicit GemmRole(int r) : prev(set_gemm_role(r)) {}
  ~GemmRole() { set_gemm_role(prev); }
};
void count_launch(int cls, int n = 1);
long long launches_total();
void launches_by_class(long long* out);  // K_NCLASS counters
bool prof_active();                      // per-launch event timing on (randutv_profile_begin)
struct ProfScope {
  ProfScope(cudaStream_t st, int cls, double flops);
  ~ProfScope();
  cudaStream_t st_;
  int cls_;
  double flops_;
  void* a_;
};
void prof_begin();
void prof_end(double* ms, double* flops, long long* counts);
// per-launch timeline of the last profile: 4 doubles per launch
// (class, stream slot in order of first use, start ms, end ms from prof_begin)
const std::vector<double>& prof_timeline();

// ---- gemm.cu -------------------------------------------------------------
// C = alpha op(A) op(B) + beta C.  ``part`` (part_elems doubles) is the split-K
// scratch; force_splits > 0 overrides the split heuristic.
// b_upper: op(B) is upper triangular (only k <= j contributes to column j; TRMM).
void poison_workspace(void* p, size_t bytes, cudaStream_t st);  // test hook (driver.cu)
void dgemm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
           int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, double* part,
           size_t part_elems, int force_splits = 0, bool b_upper = false, bool c_upper = false);
// op(A) op(B) with the K range split: partial products at part + z*M*N (ld M),
// z < returned split count; no reduction (the caller sums in fixed order).
int dgemm_partials(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* part, size_t part_elems);
int gemm_choose_splits(int64_t M, int64_t N, int64_t K, size_t part_elems);

// ---- misc.cu ---------------------------------------------------------------
void scale_matrix(cudaStream_t st, int64_t m, int64_t n, double beta, double* C, int64_t ldc);
void copy_matrix(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* D, int64_t ldd);
void set_identity(cudaStream_t st, int64_t m, int64_t n, double* D, int64_t ldd);  // D = I (m x n)
// D (n x m) = S^T for an m x n S
void transpose_matrix(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* D, int64_t ldd);
void set_zero(cudaStream_t st, int64_t m, int64_t n, double* D, int64_t ldd);
// D(0:b, 0:b) = R (b x b), D(b:m, 0:b) = 0 -- the panel column block after its QR
void put_r_panel(cudaStream_t st, int64_t m, int64_t b, const double* R, int64_t ldr, double* D, int64_t ldd);
// Copy S -> D (may alias when equal), accumulate sum of squares and a
// non-finite flag.  out2[0] = ||S||_F^2 (deterministic two-pass), flag[0] != 0 if any
// entry is NaN/Inf.  ``scratch`` needs 4096 doubles.
void copy_norm_check(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* D,
                     int64_t ldd, double* scratch, double* out2, int* flag);
// sum of squares of an m x n block into out2[0] (deterministic).
void fro2(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* scratch, double* out2);
// Philox4x32-10 Gaussian block (R2).
void gaussian_fill(cudaStream_t st, double* G, int64_t ldg, int64_t rows, int64_t cols, uint64_t seed,
                   uint32_t step, uint32_t purpose);
// D = diag(d) on a k x k block (exact zeros off the diagonal) below which rows
// [k, m) of the same columns are zeroed.
void write_diag_block(cudaStream_t st, int64_t m, int64_t k, const double* d, double* D, int64_t ldd);

// ---- smallmat.cu: b x b cluster kernels of the CholeskyQR2 panel QR --------
struct SmallWork {
  int bp;  // b padded to a multiple of 32; every matrix below is bp x bp, ld bp
  double *W1, *R1, *R1i, *W2, *R2, *R2i, *F, *Li, *Ui, *M, *US;
  double* S;      // bp signs
  double* stats;  // [bad, min diag R1, max diag R1]
  int* flag;      // 0: reconstruction valid
};
int small_pad(int64_t b);
size_t small_work_elems(int64_t b);
SmallWork carve_small(double* base, int64_t b);
// W1 (Gram, b x b valid) -> R1, R1i = R1^-1; stats.
void small_chol_inv(cudaStream_t st, int64_t b, const SmallWork& w);
// W2 = Q1^T Q1 -> second pass + Householder reconstruction: writes R (b x b,
// ld ldr), tau, Tw (ld ldt), w.M = R2^-1 U~^-1 and w.F (L strictly below), w.flag.
// side (optional): T_w, tau and R_h are formed on it (forked after the LU with
// ev_fork); the caller must wait for ev_join before using them.
void small_recon(cudaStream_t st, int64_t b, const SmallWork& w, const double* Q1, int64_t ldq, double* R,
                 int64_t ldr, double* tau, double* Tw, int64_t ldt, double* part, size_t part_elems,
                 cudaStream_t side = nullptr, cudaEvent_t ev_fork = nullptr, cudaEvent_t ev_join = nullptr,
                 double dev_max = 0.5);
// orth_tol for panels whose R factor is kept (see QrWork::orth_tol)
constexpr double kRFactorOrthTol = 1e-7;
// V(0:b, 0:b) <- unit lower L from w.F
void small_put_unit_lower(cudaStream_t st, int64_t b, const SmallWork& w, double* V, int64_t ldv);

// ---- qr.cu -----------------------------------------------------------------
struct QrWork {
  double* part;      // split-K scratch for the inner GEMMs
  size_t part_elems;
  double* sfull;     // b_leaf x b   (V_l^T [V_prev | V_l | A_rest])
  double* s2;        // b_leaf x b
  double* z;         // b x b_leaf
  double* q1 = nullptr;  // m x b scratch of the CholeskyQR2 path (capacity q1_elems)
  size_t q1_elems = 0;
  double* small = nullptr;  // small_work_elems(b) doubles
  int mode = 0;             // 0: CholeskyQR2 + reconstruction, Householder fallback; 1: Householder only
  // CholeskyQR2 accepted while max|Q1^T Q1 - I| <= orth_tol: 0.5 where only the
  // span is used (QR(Y): kappa up to ~1e7); kRFactorOrthTol where R enters T
  // (column panels, final blocks: kappa <~ 3e4, R backward stable to O(u))
  double orth_tol = 0.5;
  int* fallbacks = nullptr; // host counter of fallbacks taken (may be null)
  // Optimistic mode (no host synchronisation): the CholeskyQR results are used
  // unconditionally and each decision flag goes to dev_flags[*flag_count]++;
  // the caller checks them once at the end and redoes the factorization in the
  // synchronous mode if any is raised.
  int* dev_flags = nullptr;
  int* flag_count = nullptr;  // host counter (slots used)
  int flag_cap = 0;
  // panel_qr only: when set, the panel is read from `in` (ld ldin) instead of
  // V (V is then output only; the Householder fallback copies in -> V first)
  const double* in = nullptr;
  int64_t ldin = 0;
};
// writes flag = (stats[0] != 0 || stats[2] > kappa_max * stats[1]) (CholeskyQR re-orthonormalization test)
void reortho_flag(cudaStream_t st, const double* stats, double kappa_max, int* flag);
size_t qr_work_elems(int64_t b);
// Q = thin orthonormal basis of span(Y) with Y = Q R, R upper triangular (the
// re-orthonormalisation of the power loop, R5): CholeskyQR when the
// Gram is well conditioned, Householder (panel_qr + thin_q) otherwise.  Y may
// be overwritten.
int reortho(cudaStream_t st, int64_t m, int64_t b, double* Y, int64_t ldy, double* Q, int64_t ldq, double* tmp_bb,
            double* Tmp_bb, double* tau, const QrWork& w);
// The same CholeskyQR re-orthonormalisation with its triangular factor
// applied AFTER the next product of the power loop (R26):
//   Z = X (Y R^-1) = (X Y) R^-1,
// so that X Y runs concurrently with the Gram and the Cholesky (optimistic
// mode only: begin returns false -- nothing enqueued -- otherwise).
// begin (stream hs): G = Y^T Y, R, R^-1 and the kappa decision flag in the
// next dev_flags slot; apply (stream st, after begin's work): Z = Zp R^-1
// (rows x b TRMM).  w.part must be scratch no concurrent GEMM uses.
bool reortho_defer_begin(cudaStream_t hs, int64_t m, int64_t b, const double* Y, int64_t ldy, const QrWork& w);
void reortho_defer_apply(cudaStream_t st, int64_t rows, int64_t b, const double* Zp, int64_t ldzp, double* Z,
                         int64_t ldz, const QrWork& w);
// Householder QR of the m x b panel held in V (ld ldv), in place:
// on exit V is the explicit unit-lower-trapezoidal reflector matrix, R (b x b,
// ld ldr) the upper-triangular factor (zeros below), tau[b] the reflector
// scalars and Tw (b x b, ld ldt) the forward compact-WY factor:
// H_1 ... H_b = I - V Tw V^T.  LAPACK dlarfg sign convention (R3).
int panel_qr(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
             double* Tw, int64_t ldt, const QrWork& w);
// panel_qr's CholeskyQR2 path in two parts, for callers that overlap the
// reconstruction with work needing only Q1 = V R1^-1 (optimistic mode only:
// begin returns false -- nothing enqueued -- when that path is unavailable).
// begin: G1 = V^T V, R1, Q1 -> w.q1 (m x b, ld m).  finish: second pass +
// reconstruction, exactly panel_qr's outputs (V = W, R, tau, Tw), the decision
// flag in the next dev_flags slot; afterwards W(b:m, :) = -Q1(b:m, :) M with
// M = panel_qr_M(w, b, &ldm) (valid until the next panel QR on this workspace).
bool panel_qr_begin(cudaStream_t st, int64_t m, int64_t b, const double* V, int64_t ldv, const QrWork& w);
void panel_qr_finish(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr,
                     double* tau, double* Tw, int64_t ldt, const QrWork& w);
const double* panel_qr_M(const QrWork& w, int64_t b, int64_t* ldm);
// Q1 = (I - V Tw V^T)[:, :b] (thin explicit Q), written to Q (m x b).
void thin_q(cudaStream_t st, int64_t m, int64_t b, const double* V, int64_t ldv, const double* Tw, int64_t ldt,
            double* Q, int64_t ldq, double* tmp_bb, double* part, size_t part_elems);
int qr_max_rows();

// ---- jacobi.cu -------------------------------------------------------------
// Batched one-sided Jacobi SVD of ``batch`` k x k matrices R_i (R_i at
// R + i*strideR, ld ldr):  R_i = Us_i diag(D_i) Vs_i^T, D_i non-increasing.
// Works on B = R_i^T.  work needs 2*batch*k*k doubles.
size_t jacobi_work_elems(int batch, int k);
// true when a k x k SVD runs as one cluster launch without host synchronisation
bool jacobi_single_launch(int k);
void jacobi_svd_batched(cudaStream_t st, int batch, int k, const double* R, int64_t ldr, int64_t strideR,
                        double* D, double* Us, double* Vs, double* work, int* sweeps_out);
// Incremental form of jacobi_svd_batched for 1 < k <= 256 (jacobi_incremental):
// begin (B = R^T, W = I), any number of jacobi_sweeps launches of up to
// nsweeps sweeps each (no-ops once converged), end (remaining sweeps +
// D, Us, Vs).  Lets the caller place the sweeps where SMs are idle.
bool jacobi_incremental(int k);
void jacobi_begin(cudaStream_t st, int batch, int k, const double* R, int64_t ldr, int64_t strideR, double* work);
void jacobi_sweeps(cudaStream_t st, int batch, int k, double* work, int nsweeps);
void jacobi_end(cudaStream_t st, int batch, int k, double* work, double* D, double* Us, double* Vs, int* sweeps_out);

}  // namespace rutv
