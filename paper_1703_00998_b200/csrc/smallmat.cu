// b x b kernels of the GEMM-based panel QR (qr.cu, R20):
//
//   CholeskyQR2 of a tall panel A (m x b):  G1 = A^T A = R1^T R1,
//   Q1 = A R1^-1,  G2 = Q1^T Q1 = R2^T R2,  Q = Q1 R2^-1,  R = R2 R1,
// followed by the Householder reconstruction of Ballard et al. ("Reconstructing
// Householder vectors from tall-skinny QR", 2015): with S = diag(+-1) chosen
// column by column so that every pivot has modulus >= 1,
//   S - Q(0:b,:) = L U~   (LU without pivoting, L unit lower, U~ upper),
//   W = [L; -Q(b:m,:) U~^-1],  T_w = U~ S L^-T,  R_h = S R,  tau_j = (T_w)_jj,
// which are, in exact arithmetic, exactly the reflectors, compact-WY factor,
// tau and R of LAPACK's Householder QR (dlarfg sign convention, R3)
// -- the convention is fixed by the uniqueness of A = (I - W T W^T)[R_h; 0]
// with W unit lower trapezoidal and 1 <= tau_j <= 2.
//
// The b x b factorizations run on ONE thread-block cluster of SC CTAs: the
// matrices live in global memory (L2-resident, <= 2 MB), split in 32 x 32
// tiles; every block step factors the 32 x 32 diagonal tile in registers of one
// warp (redundantly in every CTA, so no broadcast is needed), then the CTAs
// share the row/column-panel and trailing-update tiles (DMMA m8n8k4 on shared
// memory tiles) with a cluster barrier between phases.  The matrices are
// padded to bp = 32*ceil(b/32) with identity (Grams) or zeros (Q block), which
// leaves the b x b results unchanged.
#include <cooperative_groups.h>

#include <algorithm>
#include <mutex>
#include <vector>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

// phase timestamps for tools/small_prof.cu / tools/chol_bench.cu (compiled out in the library)
#ifndef SMALL_MARK
#define SMALL_MARK(id)
#endif
#ifndef DSM_MARK
#define DSM_MARK(cta, id)
#endif
#ifndef LU_MARK
#define LU_MARK(cta, id)
#endif

namespace rutv {

namespace {
constexpr int TS = 32;    // tile size
constexpr int SLD = 36;   // smem tile stride (== 4 mod 16 doubles: conflict-free DMMA fragments)
constexpr int SNT = 256;  // threads per CTA
#ifndef RUTV_SMALL_SC
#define RUTV_SMALL_SC 8
#endif
constexpr int SC = RUTV_SMALL_SC;  // CTAs per cluster
constexpr int TSZ = TS * SLD;

struct SmallSm {
  double a[TSZ], b[TSZ], c[TSZ];    // operand / intermediate tiles
  double d[TSZ], di[TSZ], dit[TSZ];  // diagonal factor, its inverse (L^-1 for LU), transposed inverse
  double e[TSZ];                     // U~^-1 of the diagonal tile (LU)
  double aug[TS * 97];               // row-major augmented elimination work area [32][96] (+1 pad)
  double piv[TS];
  double sgn[TS];
  double rowbuf[2][96];  // pivot row of the current column step (double-buffered)
  double colbuf[2][TS];  // pivot column of the current column step
  double dmin, dmax;
  unsigned long long devbits;  // cluster max |G2 - I| (bit pattern of a non-negative double)
  int bad;
};

struct TRef {
  const double* p;  // stored tile's (0,0) element
  int ld;
  int tr;           // op(X) = tr ? stored^T : stored
};

__device__ __forceinline__ double* tile_ptr(double* M, int ld, int i, int j) {
  return M + i * TS + size_t(j) * TS * ld;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cluster_barrier(cg::cluster_group& cl) {
  __threadfence();
  cl.sync();
}

// 32x32 tile global -> registers (4 elements per thread; L2 only, the data
// was written by other CTAs of the cluster)
__device__ __forceinline__ void tile_ld(double (&v)[4], const TRef& t) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5;
    v[u] = __ldcg(t.p + r + size_t(c) * t.ld);
  }
}
// registers -> shared tile holding op(X) column-major (stride SLD)
__device__ __forceinline__ void tile_st(double* s, const double (&v)[4], int tr) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5;
    if (tr) s[r * SLD + c] = v[u];
    else s[c * SLD + r] = v[u];
  }
}
__device__ __forceinline__ void tile_load_sync(double* s, const TRef& t) {
  double v[4];
  tile_ld(v, t);
  tile_st(s, v, t.tr);
  __syncthreads();
}

// acc += sA * sB (32x32x32; warp w owns rows 8(w&3).., columns 16(w>>2)..)
__device__ __forceinline__ void tile_mma(double (&acc)[2][2], const double* sA, const double* sB) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int fr = (w & 3) * 8, fc = (w >> 2) * 16;
#pragma unroll
  for (int k4 = 0; k4 < 8; ++k4) {
    const double a = sA[(k4 * 4 + t) * SLD + fr + g];
    const double b0 = sB[(fc + g) * SLD + k4 * 4 + t];
    const double b1 = sB[(fc + 8 + g) * SLD + k4 * 4 + t];
    dmma(acc[0], a, b0);
    dmma(acc[1], a, b1);
  }
}

__device__ __forceinline__ void acc_zero(double (&acc)[2][2]) {
  acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.0;
}

// visit the accumulator elements: f(row, col, value) in tile coordinates
template <class F>
__device__ __forceinline__ void acc_each(const double (&acc)[2][2], F f) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int fr = (w & 3) * 8, fc = (w >> 2) * 16;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) f(fr + g, fc + 8 * j + 2 * t + e, acc[j][e]);
}

__device__ __forceinline__ void acc_to_smem(const double (&acc)[2][2], double* s) {
  acc_each(acc, [&](int r, int c, double v) { s[c * SLD + r] = v; });
  __syncthreads();
}
__device__ __forceinline__ void acc_to_global(const double (&acc)[2][2], double* g, int ld, double scale) {
  acc_each(acc, [&](int r, int c, double v) { g[r + size_t(c) * ld] = scale * v; });
}

// g(tile) -= acc, with every load issued before the first store (the
// compiler cannot hoist loads over possibly-aliasing stores itself)
__device__ __forceinline__ void acc_sub_global(const double (&acc)[2][2], double* g, int ld) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gg = lane >> 2, t = lane & 3;
  const int fr = (w & 3) * 8, fc = (w >> 2) * 16;
  double old[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) old[j][e] = __ldcg(g + (fr + gg) + size_t(fc + 8 * j + 2 * t + e) * ld);
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) g[(fr + gg) + size_t(fc + 8 * j + 2 * t + e) * ld] = old[j][e] - acc[j][e];
}

// acc = sum_{q < np} op(A_q) op(B_q), operands streamed through s.a / s.b with
// a one-deep register prefetch.
template <class GP>
__device__ void tile_sum(double (&acc)[2][2], int np, GP gp, SmallSm& s) {
  acc_zero(acc);
  if (np <= 0) return;
  double va[4], vb[4];
  TRef A, B;
  gp(0, A, B);
  tile_ld(va, A);
  tile_ld(vb, B);
  for (int q = 0; q < np; ++q) {
    __syncthreads();
    tile_st(s.a, va, A.tr);
    tile_st(s.b, vb, B.tr);
    __syncthreads();
    if (q + 1 < np) {
      gp(q + 1, A, B);
      tile_ld(va, A);
      tile_ld(vb, B);
    }
    tile_mma(acc, s.a, s.b);
  }
  __syncthreads();
}

// ---- 32x32 diagonal-tile kernels, whole CTA, one barrier per column ---------
// (Measured on B200: the per-column chain -- pivot, reciprocal, update,
// barrier -- costs ~0.3 us; variants with one warp, shifted registers or
// per-thread 8x8 blocks were slower because the FP64 issue rate of one warp
// (~2.4 cycles per DFMA) or redundant per-warp work dominates.)
//
// Cholesky + inverse by elimination on the augmented [G | I] (row-major, ld 65):
// after the 32 column steps the left block holds U = Dg L^T (G = L Dg L^T) and
// the right block L^-1, so R = Dg^{1/2} L^T and R^-1 = L^-T Dg^{-1/2}.
// In: G tile (column-major in s.d, upper triangle read).  Out: s.d = R (zeros
// below), s.di = R^-1, s.dit = R^-T.  Non-positive / non-finite pivots of valid
// columns set s.bad (and are replaced by 1).
// 1/x for finite x != 0: MUFU seed + two Newton steps (~1 ulp; the division
// routine's slow-path checks sat on the per-column critical path)
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// publish row k and column k (k < 32) of a register-resident augmented
// matrix (thread owns row i, columns j0 .. j0 + N - 1) for the next column step
// The row buffer is stored permuted: the 16-byte chunk jj/2 of the 8 column
// groups are adjacent, so the 8 lanes of a row reading (or writing) their
// chunk touch 128 contiguous bytes (the natural layout's 64- or 96-byte
// stride between groups made every 16-byte access a 4-way bank conflict:
// 484 -> 326 cycles per column step, tools/scratch/stepbench.cu)
template <int N>
__device__ __forceinline__ int rb_pos(int j) {
  const int g = j / N, jj = j % N;
  return (jj >> 1) * 16 + g * 2 + (jj & 1);
}
template <int N>
__device__ __forceinline__ void aug_publish(SmallSm& s, const double (&a)[N], int i, int j0, int k, int buf) {
  (void)j0;
  if (i == k) {
#pragma unroll
    for (int jj = 0; jj < N; jj += 2)
      *reinterpret_cast<double2*>(&s.rowbuf[buf][(jj >> 1) * 16 + (threadIdx.x & 7) * 2]) =
          make_double2(a[jj], a[jj + 1]);
  }
  // owner of column k: j0 = N (k / N); k is an unrolled loop index at every
  // call site, so a[k % N] is a static register
  if ((threadIdx.x & 7) == k / N) s.colbuf[buf][i] = a[k % N];
}

__device__ __noinline__ void cta_chol_inv(SmallSm& s, int gcol0, int b) {
  constexpr int LD = 65;
  double* A = s.aug;
  const int tid = threadIdx.x;
  // thread t owns row i = t / 8, columns 8 (t % 8) .. +7 of [G | I] in
  // registers for all 32 column steps; per step only the pivot row and column
  // go through shared memory (published by their owners, double-buffered), so
  // a step is one barrier, ~6 shared loads and 8 FMAs per thread
  const int i = tid >> 3, j0 = (tid & 7) * 8;
  double a[8];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = j0 + jj;
    a[jj] = (j < TS) ? s.d[max(i, j) * SLD + min(i, j)] : ((j - TS == i) ? 1.0 : 0.0);
  }
  aug_publish(s, a, i, j0, 0, 0);
  __syncthreads();
#pragma unroll  // k - j0 must be a compile-time register index in aug_publish
  for (int k = 0; k < TS; ++k) {
    const int buf = k & 1;
    double p = s.rowbuf[buf][rb_pos<8>(k)];
    if (!(p > 0.0) || !isfinite(p)) p = 1.0;  // flagged below from the stored pivot
    if (i > k) {
      const double l = s.colbuf[buf][i] * frcp(p);
      double r[8];
#pragma unroll
      for (int jj = 0; jj < 8; jj += 2) {
        const double2 t = *reinterpret_cast<const double2*>(&s.rowbuf[buf][(jj >> 1) * 16 + (tid & 7) * 2]);
        r[jj] = t.x;
        r[jj + 1] = t.y;
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (j0 + jj > k) a[jj] = fma(-l, r[jj], a[jj]);
    }
    if (k + 1 < TS) aug_publish(s, a, i, j0, k + 1, buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) A[i * LD + j0 + jj] = a[jj];
  __syncthreads();
  if (tid < TS) {  // warp 0: pivots, their reciprocals, breakdown flag, min / max
    double p = A[tid * LD + tid];
    const bool ok = (p > 0.0) && isfinite(p);
    if (!ok) p = 1.0;
    const double d = sqrt(p);
    s.piv[tid] = d;
    s.c[tid] = frcp(d);
    const bool valid = gcol0 + tid < b;
    if (valid && !ok) atomicOr(&s.bad, 1);
    double mn = valid ? d : DBL_MAX, mx = valid ? d : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (tid == 0) {
      s.dmin = fmin(s.dmin, mn);
      s.dmax = fmax(s.dmax, mx);
    }
  }
  __syncthreads();
  const double* rd = s.c;
  for (int e = tid; e < TS * TS; e += SNT) {
    const int i = e & 31, j = e >> 5;  // (row i, col j), column-major outputs
    s.d[j * SLD + i] = (i <= j) ? A[i * LD + j] * rd[i] : 0.0;
    const double ri = (i <= j) ? A[j * LD + TS + i] * rd[j] : 0.0;  // R^-1(i,j) = L^-1(j,i)/d_j
    s.di[j * SLD + i] = ri;
    s.dit[i * SLD + j] = ri;
  }
  __syncthreads();
}

// The same factorisation with 2 x 2 block pivots: 16 double steps instead of 32
// column steps (one barrier, one reciprocal per two columns).  At double step
// k (even) every row i > k+1 is updated at once from the current rows k and k+1,
//   row_i -= [a_ik, a_i,k+1] P^-1 [row_k; row_k+1],  P = [[a_kk, a_k,k+1], [a_k+1,k, a_k+1,k+1]],
// which in exact arithmetic is column steps k and k+1 (the Schur complement of
// P is what the two single steps leave); a final pass eliminates a_k+1,k
// inside each pair (row_k+1 -= a_k+1,k / a_kk row_k), after which the left
// block is U = D L^T and the right block L^-1 exactly as for cta_chol_inv, and
// the same epilogue follows.  rb: [2 buffers][2 rows][64] (permuted like
// rowbuf), cb: [2][2][32] (the pivot columns).  A non-positive / non-finite
// pivot block is replaced by the identity and flagged from the final pivots.
__device__ __noinline__ void cta_chol_inv2(SmallSm& s, double* rb, double* cb, int gcol0, int b) {
  constexpr int LD = 65;
  double* A = s.aug;
  const int tid = threadIdx.x;
  const int i = tid >> 3, g = tid & 7, j0 = g * 8;
  double a[8];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = j0 + jj;
    a[jj] = (j < TS) ? s.d[max(i, j) * SLD + min(i, j)] : ((j - TS == i) ? 1.0 : 0.0);
  }
  auto pub = [&](int k, int buf) {  // rows k, k+1 and columns k, k+1 for double step k
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (i == k + h) {
#pragma unroll
        for (int jj = 0; jj < 8; jj += 2)
          *reinterpret_cast<double2*>(&rb[(buf * 2 + h) * 64 + (jj >> 1) * 16 + g * 2]) = make_double2(a[jj], a[jj + 1]);
      }
      if (g == (k + h) / 8) cb[(buf * 2 + h) * 32 + i] = a[(k + h) % 8];
    }
  };
  pub(0, 0);
  __syncthreads();
#pragma unroll  // (k + h) % 8 must be a compile-time register index
  for (int k = 0; k < TS; k += 2) {
    const int buf = (k >> 1) & 1;
    const double* r0 = rb + (buf * 2 + 0) * 64;
    const double* r1 = rb + (buf * 2 + 1) * 64;
    if (i > k + 1) {
      const double p00 = r0[rb_pos<8>(k)], p01 = r0[rb_pos<8>(k + 1)];
      const double p10 = r1[rb_pos<8>(k)], p11 = r1[rb_pos<8>(k + 1)];
      const double x0 = cb[(buf * 2 + 0) * 32 + i], x1 = cb[(buf * 2 + 1) * 32 + i];
      const double det = fma(p00, p11, -p01 * p10);
      double c0, c1;
      if (p00 > 0.0 && det > 0.0 && isfinite(det)) {
        const double id = frcp(det);
        c0 = fma(x0, p11, -x1 * p10) * id;
        c1 = fma(x1, p00, -x0 * p01) * id;
      } else {
        c0 = x0;
        c1 = x1;
      }
      double v0[8], v1[8];
#pragma unroll
      for (int jj = 0; jj < 8; jj += 2) {
        const double2 t0 = *reinterpret_cast<const double2*>(&r0[(jj >> 1) * 16 + g * 2]);
        const double2 t1 = *reinterpret_cast<const double2*>(&r1[(jj >> 1) * 16 + g * 2]);
        v0[jj] = t0.x; v0[jj + 1] = t0.y;
        v1[jj] = t1.x; v1[jj + 1] = t1.y;
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (j0 + jj > k + 1) a[jj] = fma(-c1, v1[jj], fma(-c0, v0[jj], a[jj]));
    }
    if (k + 2 < TS) pub(k + 2, buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) A[i * LD + j0 + jj] = a[jj];
  __syncthreads();
  // within each pair: row k+1 -= (a_k+1,k / a_kk) row k, columns > k (both halves)
  if (i & 1) {
    const int k = i - 1;
    double pk = A[k * LD + k];
    if (!(pk > 0.0) || !isfinite(pk)) pk = 1.0;  // flagged from the stored pivot below
    const double l = A[i * LD + k] * frcp(pk);
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = j0 + jj;
      if (j > k) a[jj] = fma(-l, A[k * LD + j], a[jj]);
    }
  }
  __syncthreads();
  if (i & 1) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) A[i * LD + j0 + jj] = a[jj];
  }
  __syncthreads();
  if (tid < TS) {  // warp 0: pivots, their reciprocals, breakdown flag, min / max (as cta_chol_inv)
    double p = A[tid * LD + tid];
    const bool ok = (p > 0.0) && isfinite(p);
    if (!ok) p = 1.0;
    const double d = sqrt(p);
    s.piv[tid] = d;
    s.c[tid] = frcp(d);
    const bool valid = gcol0 + tid < b;
    if (valid && !ok) atomicOr(&s.bad, 1);
    double mn = valid ? d : DBL_MAX, mx = valid ? d : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (tid == 0) {
      s.dmin = fmin(s.dmin, mn);
      s.dmax = fmax(s.dmax, mx);
    }
  }
  __syncthreads();
  const double* rd = s.c;
  for (int e = tid; e < TS * TS; e += SNT) {
    const int i = e & 31, j = e >> 5;  // (row i, col j), column-major outputs
    s.d[j * SLD + i] = (i <= j) ? A[i * LD + j] * rd[i] : 0.0;
    const double ri = (i <= j) ? A[j * LD + TS + i] * rd[j] : 0.0;  // R^-1(i,j) = L^-1(j,i)/d_j
    s.di[j * SLD + i] = ri;
    s.dit[i * SLD + j] = ri;
  }
  __syncthreads();
}

// Sign-modified LU (Householder reconstruction: when column k becomes the
// pivot, s_k = (a_kk <= 0 ? -1 : +1) is added, |pivot| = |a_kk| + 1 >= 1) by
// elimination on [F | I | I] (row-major, ld 97): the middle block becomes L^-1;
// the right block runs the forward elimination of U~^T with the rows of U~ as
// they become final, giving E' with E' U~^T = diag(piv), so U~^-1 = E'^T diag(piv)^-1.
// In: F tile (column-major in s.d).  Out: s.d = L (strict lower) \ U~, s.di =
// L^-1, s.e = U~^-1, s.sgn.
template <class SM>
__device__ __noinline__ void cta_lu_sign_inv(SM& s) {
  constexpr int LD = 97;
  double* A = s.aug;
  const int tid = threadIdx.x;
  // register-resident rows: thread t owns row i = t / 8 and, in each of the
  // three 32-column regions of [F | I | I], the 4 columns 4 (t % 8) .. +3, so
  // the kind of update of a register is known at compile time.  Row buffer
  // position of column j (region r, c = j mod 32, group c / 4, q = c mod 4):
  // chunk 2r + q/2 of 16 doubles (8 groups x 2), conflict-free 16-byte access.
  const int i = tid >> 3, g = tid & 7;
  auto pos = [](int j) { const int r = j >> 5, c = j & 31, q = c & 3; return (2 * r + (q >> 1)) * 16 + (c >> 2) * 2 + (q & 1); };
  double a[12];  // a[4 r + q] = A(i, 32 r + 4 g + q)
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = 4 * g + q;
      a[4 * r + q] = (r == 0) ? s.d[c * SLD + i] : (c == i ? 1.0 : 0.0);
    }
  auto publish = [&](int k, int buf) {  // row k, column k (region 0) for the next step
    if (i == k) {
#pragma unroll
      for (int h = 0; h < 6; ++h)
        *reinterpret_cast<double2*>(&s.rowbuf[buf][h * 16 + g * 2]) = make_double2(a[2 * h], a[2 * h + 1]);
    }
    if (g == (k >> 2)) s.colbuf[buf][i] = a[k & 3];
  };
  publish(0, 0);
  __syncthreads();
#pragma unroll  // k & 3 must be a compile-time register index
  for (int k = 0; k < TS; ++k) {
    const int buf = k & 1;
    const double av = s.rowbuf[buf][pos(k)];
    const double sg = (av <= 0.0) ? -1.0 : 1.0;
    const double pv = av + sg;
    if (tid == 0) {
      s.sgn[k] = sg;
      s.piv[k] = pv;
    }
    if (i > k) {
      const double invp = frcp(pv);
      const double l = s.colbuf[buf][i] * invp;         // F and L^-1 regions: A(i,k) / pivot
      const double lu = s.rowbuf[buf][pos(i)] * invp;   // U~^T region: A(k,i) / pivot
      double rv[12];
#pragma unroll
      for (int h = 0; h < 6; ++h) {
        const double2 t = *reinterpret_cast<const double2*>(&s.rowbuf[buf][h * 16 + g * 2]);
        rv[2 * h] = t.x;
        rv[2 * h + 1] = t.y;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (4 * g + q > k) a[q] = fma(-l, rv[q], a[q]);
        a[4 + q] = fma(-l, rv[4 + q], a[4 + q]);
        a[8 + q] = fma(-lu, rv[8 + q], a[8 + q]);
      }
    }
    if (k + 1 < TS) publish(k + 1, buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) A[i * LD + 32 * r + 4 * g + q] = a[4 * r + q];
  __syncthreads();
  if (tid < TS) s.c[tid] = frcp(s.piv[tid]);
  __syncthreads();
  const double* rp = s.c;
  for (int e = tid; e < TS * TS; e += SNT) {
    const int i = e & 31, j = e >> 5;
    const double pj = s.piv[j];
    s.d[j * SLD + i] = (i > j) ? A[i * LD + j] * rp[j] : ((i == j) ? pj : A[i * LD + j]);
    s.di[j * SLD + i] = (i >= j) ? A[i * LD + TS + j] : 0.0;
    s.e[j * SLD + i] = (i <= j) ? A[j * LD + 2 * TS + i] * rp[j] : 0.0;
  }
  __syncthreads();
}

struct SmallDims {
  int b, bp, nb;
};

__device__ __forceinline__ void copy_tile_smem_to_global(const double* s, double* g, int ld) {
  for (int e = threadIdx.x; e < TS * TS; e += SNT) {
    const int r = e & 31, c = e >> 5;
    g[r + size_t(c) * ld] = s[c * SLD + r];
  }
}


// decode the q-th upper-triangular tile (i, j), lo <= i <= j < nb
__device__ __forceinline__ void upper_pair(int q, int lo, int nb, int& i, int& j) {
  i = lo;
  while (q >= nb - i) {
    q -= nb - i;
    ++i;
  }
  j = i + q;
}

// Blocked right-looking Cholesky with the inverse of the factor built along:
// W (bp x bp, updated in place) = R^T R;  R, Ri = R^-1 (upper, zero lower tiles
// written by the caller's init).  Stats into s.bad / s.dmin / s.dmax.
__device__ void chol_inv_dev(cg::cluster_group& cl, const SmallDims& d, double* W, double* R, double* Ri,
                             SmallSm& s) {
  const int C = (int)cl.num_blocks(), cta = (int)cl.block_rank();
  const int bp = d.bp, nb = d.nb;
  for (int p = 0; p < nb; ++p) {
    SMALL_MARK(0);
    tile_load_sync(s.d, TRef{tile_ptr(W, bp, p, p), bp, 0});
    SMALL_MARK(1);
    cta_chol_inv(s, p * TS, d.b);
    SMALL_MARK(2);
    if (cta == 0) {
      copy_tile_smem_to_global(s.d, tile_ptr(R, bp, p, p), bp);
      copy_tile_smem_to_global(s.di, tile_ptr(Ri, bp, p, p), bp);
    }
    // phase A: R(p, j) = D^-T W(p, j) (j > p);  Ri(k, p) = -(sum_l Ri(k,l) R(l,p)) D^-1 (k < p)
    const int nrow = nb - 1 - p;
    for (int task = cta; task < nb - 1; task += C) {
      double acc[2][2];
      if (task < nrow) {
        const int j = p + 1 + task;
        tile_load_sync(s.a, TRef{tile_ptr(W, bp, p, j), bp, 0});
        acc_zero(acc);
        tile_mma(acc, s.dit, s.a);
        acc_to_global(acc, tile_ptr(R, bp, p, j), bp, 1.0);
      } else {
        const int k = task - nrow;
        tile_sum(acc, p - k, [&](int q, TRef& A, TRef& B) {
          const int l = k + q;
          A = TRef{tile_ptr(Ri, bp, k, l), bp, 0};
          B = TRef{tile_ptr(R, bp, l, p), bp, 0};
        }, s);
        acc_to_smem(acc, s.c);
        acc_zero(acc);
        tile_mma(acc, s.c, s.di);
        acc_to_global(acc, tile_ptr(Ri, bp, k, p), bp, -1.0);
      }
      __syncthreads();
    }
    SMALL_MARK(3);
    cluster_barrier(cl);
    SMALL_MARK(4);
    // phase B: W(i, j) -= R(p, i)^T R(p, j), p < i <= j
    const int nt = nrow * (nrow + 1) / 2;
    for (int task = cta; task < nt; task += C) {
      int i, j;
      upper_pair(task, p + 1, nb, i, j);
      double acc[2][2];
      SMALL_MARK(7);
      tile_sum(acc, 1, [&](int, TRef& A, TRef& B) {
        A = TRef{tile_ptr(R, bp, p, i), bp, 1};
        B = TRef{tile_ptr(R, bp, p, j), bp, 0};
      }, s);
      SMALL_MARK(8);
      acc_sub_global(acc, tile_ptr(W, bp, i, j), bp);
      __syncthreads();
      SMALL_MARK(9);
    }
    SMALL_MARK(5);
    cluster_barrier(cl);
  }
}

// Blocked right-looking sign-modified LU of F (in place: L \ U~), with
// Li = L^-1 and Ui = U~^-1 built along, and the signs into S (bp).
__device__ void lu_sign_inv_dev(cg::cluster_group& cl, const SmallDims& d, double* F, double* Li, double* Ui,
                                double* S, SmallSm& s) {
  const int C = (int)cl.num_blocks(), cta = (int)cl.block_rank();
  const int bp = d.bp, nb = d.nb;
  for (int p = 0; p < nb; ++p) {
    SMALL_MARK(0);
    tile_load_sync(s.d, TRef{tile_ptr(F, bp, p, p), bp, 0});
    SMALL_MARK(1);
    cta_lu_sign_inv(s);
    SMALL_MARK(2);
    if (cta == 0) {
      copy_tile_smem_to_global(s.d, tile_ptr(F, bp, p, p), bp);
      copy_tile_smem_to_global(s.di, tile_ptr(Li, bp, p, p), bp);
      copy_tile_smem_to_global(s.e, tile_ptr(Ui, bp, p, p), bp);
      if (threadIdx.x < TS) S[p * TS + threadIdx.x] = s.sgn[threadIdx.x];
    }
    const int nr = nb - 1 - p;
    for (int task = cta; task < 2 * (nb - 1); task += C) {
      double acc[2][2];
      if (task < nr) {  // U~(p, j) = L_pp^-1 F(p, j)
        const int j = p + 1 + task;
        tile_load_sync(s.a, TRef{tile_ptr(F, bp, p, j), bp, 0});
        acc_zero(acc);
        tile_mma(acc, s.di, s.a);
        acc_to_global(acc, tile_ptr(F, bp, p, j), bp, 1.0);
      } else if (task < 2 * nr) {  // L(i, p) = F(i, p) U~_pp^-1
        const int i = p + 1 + (task - nr);
        tile_load_sync(s.a, TRef{tile_ptr(F, bp, i, p), bp, 0});
        acc_zero(acc);
        tile_mma(acc, s.a, s.e);
        acc_to_global(acc, tile_ptr(F, bp, i, p), bp, 1.0);
      } else if (task < 2 * nr + p) {  // Ui(k, p) = -(sum_l Ui(k,l) U~(l,p)) U~_pp^-1
        const int k = task - 2 * nr;
        tile_sum(acc, p - k, [&](int q, TRef& A, TRef& B) {
          const int l = k + q;
          A = TRef{tile_ptr(Ui, bp, k, l), bp, 0};
          B = TRef{tile_ptr(F, bp, l, p), bp, 0};
        }, s);
        acc_to_smem(acc, s.c);
        acc_zero(acc);
        tile_mma(acc, s.c, s.e);
        acc_to_global(acc, tile_ptr(Ui, bp, k, p), bp, -1.0);
      } else {  // Li(p, k) = -L_pp^-1 (sum_l L(p,l) Li(l,k))
        const int k = task - 2 * nr - p;
        tile_sum(acc, p - k, [&](int q, TRef& A, TRef& B) {
          const int l = k + q;
          A = TRef{tile_ptr(F, bp, p, l), bp, 0};
          B = TRef{tile_ptr(Li, bp, l, k), bp, 0};
        }, s);
        acc_to_smem(acc, s.c);
        acc_zero(acc);
        tile_mma(acc, s.di, s.c);
        acc_to_global(acc, tile_ptr(Li, bp, p, k), bp, -1.0);
      }
      __syncthreads();
    }
    SMALL_MARK(3);
    cluster_barrier(cl);
    SMALL_MARK(4);
    const int nt = nr * nr;
    for (int task = cta; task < nt; task += C) {
      const int i = p + 1 + task % nr, j = p + 1 + task / nr;
      double acc[2][2];
      tile_sum(acc, 1, [&](int, TRef& A, TRef& B) {
        A = TRef{tile_ptr(F, bp, i, p), bp, 0};
        B = TRef{tile_ptr(F, bp, p, j), bp, 0};
      }, s);
      acc_sub_global(acc, tile_ptr(F, bp, i, j), bp);
      __syncthreads();
    }
    SMALL_MARK(5);
    cluster_barrier(cl);
  }
}

__device__ void init_stats(SmallSm& s) {
  if (threadIdx.x == 0) {
    s.bad = 0;
    s.devbits = 0ull;
    s.dmin = DBL_MAX;
    s.dmax = 0.0;
  }
  __syncthreads();
}

// Identity padding of a Gram written by the GEMM into W (b x b valid, ld bp);
// zero the strictly-lower tiles of the listed upper-triangular outputs.
__device__ void init_gram_and_zero(cg::cluster_group& cl, const SmallDims& d, double* W, double* const* zl, int nzl) {
  const int C = (int)cl.num_blocks(), cta = (int)cl.block_rank();
  const int bp = d.bp, b = d.b;
  for (int c = cta; c < bp; c += C)  // column-strided: no 64-bit division per element
    for (int r = threadIdx.x, e = c * bp + threadIdx.x; r < bp; r += SNT, e += SNT) {
    if (r >= b || c >= b) W[e] = (r == c) ? 1.0 : 0.0;
    const int ti = r / TS, tj = c / TS;
    if (ti > tj)
      for (int z = 0; z < nzl; ++z) zl[z][e] = 0.0;
  }
}

// kernel 1: Cholesky + inverse of the Gram G1 = A^T A.
// stats[0] = breakdown (0/1), stats[1] = min diag R, stats[2] = max diag R.
__global__ void __launch_bounds__(SNT, 1)
chol_inv_k(SmallDims d, double* __restrict__ W, double* __restrict__ R, double* __restrict__ Ri,
           double* __restrict__ stats) {
  pdl_begin();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double sm_raw[];
  SmallSm& s = *reinterpret_cast<SmallSm*>(sm_raw);
  init_stats(s);
  double* zl[2] = {R, Ri};
  init_gram_and_zero(cl, d, W, zl, 2);
  cluster_barrier(cl);
  chol_inv_dev(cl, d, W, R, Ri, s);
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    stats[0] = s.bad ? 1.0 : 0.0;
    stats[1] = s.dmin;
    stats[2] = s.dmax;
  }
}

// ---- Cholesky + inverse with the matrix resident in distributed shared memory
// One cluster of nb = bp/32 CTAs (b <= 256); CTA j owns tile column j: the
// Gram / R tiles (i, j), i <= j, and the tiles (i, j), i >= j, of E = R^-T (the
// right half of the elimination on [G | I], which ends as L^-1 = R^-T).  Tiles
// never leave shared memory until the end; other CTAs' tiles are read through
// DSMEM.  Instead of one cluster barrier per phase, readiness is tracked per
// producer with two counters in its shared memory (polled remotely):
//   diag_done: R_jj, R_jj^-T of CTA j are final;
//   row_done = p + 1: R(p, j) of CTA j is final.
// CTA j: for p < j: R(p, j) = R_pp^-T G(p, j) (R_pp^-T read from CTA p), publish,
// then G(i, j) -= R(p, i)^T R(p, j) for p < i <= j (R(p, i) read from CTA i) --
// the diagonal tile first; then factor its own diagonal tile (cta_chol_inv) and
// publish; then its column of E: for p >= j, E(p, j) = R_pp^-T E(p, j) and
// E(i, j) -= R(p, i)^T E(p, j) for i > p.  The critical path per block step is
// the diagonal factorisation plus one flag hop and two 32x32x32 products, with
// no cluster-wide barrier and no L2 round trip.
#ifndef RUTV_CHOL_2X2
#define RUTV_CHOL_2X2 1
#endif
constexpr bool kChol2x2 = RUTV_CHOL_2X2;  // 2 x 2 block pivots in the diagonal tiles (cta_chol_inv2)

struct CholDsm {
  double t[9][TSZ];            // column j: G/R tiles i = 0..j at t[i]; E tiles i = j..nb-1 at t[i + 1]
  double rb[2 * 2 * 64];       // pivot rows of cta_chol_inv2 (double-buffered pairs)
  double cb[2 * 2 * 32];       // pivot columns
  volatile int diag_done;
  volatile int row_done;
  unsigned long long dmin_bits, dmax_bits;  // cluster-wide min / max of diag R (CTA 0)
  int bad;                                  // cluster-wide breakdown flag (CTA 0)
};

__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }

// wait until *remote >= target (thread 0 spins; the CTA then proceeds)
__device__ __forceinline__ void wait_flag(const volatile int* remote, int target) {
  if (threadIdx.x == 0) {
    while (*remote < target) {
    }
    fence_cluster();
  }
  __syncthreads();
}

__device__ __forceinline__ void publish(volatile int* flag, int value) {
  __syncthreads();  // every thread's writes of the tile are done
  if (threadIdx.x == 0) {
    fence_cluster();
    *flag = value;
  }
}

// remote (generic, DSMEM) tile -> local tile, optionally transposed
__device__ __forceinline__ void tile_copy(double* dst, const double* src, bool tr) {
  double v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5;
    v[u] = src[c * SLD + r];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5;
    if (tr) dst[r * SLD + c] = v[u];
    else dst[c * SLD + r] = v[u];
  }
}

// t -= acc (the thread's accumulator elements)
__device__ __forceinline__ void acc_sub_smem(const double (&acc)[2][2], double* t) {
  acc_each(acc, [&](int r, int c, double v) { t[c * SLD + r] -= v; });
}

__global__ void __launch_bounds__(SNT, 1)
chol_inv_dsm_k(SmallDims d, const double* __restrict__ W, double* __restrict__ R, double* __restrict__ Ri,
               double* __restrict__ stats) {
  pdl_begin();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double sm_raw[];
  SmallSm& s = *reinterpret_cast<SmallSm*>(sm_raw);
  CholDsm& q = *reinterpret_cast<CholDsm*>(sm_raw + (sizeof(SmallSm) + 15) / 8 / 2 * 2);
  const int j = (int)cl.block_rank(), nb = d.nb, bp = d.bp, b = d.b;
  auto G = [&](int i) { return q.t[i]; };       // tile (i, j), i <= j
  auto E = [&](int i) { return q.t[i + 1]; };   // tile (i, j), i >= j
  auto remote = [&](int rank) { return cl.map_shared_rank(&q, rank); };
  // ---- load column j of the Gram (identity padding beyond b), E(:, j) = [0; I; 0]
  if (threadIdx.x == 0) {
    q.diag_done = 0;
    q.row_done = 0;
    q.bad = 0;
    q.dmin_bits = __double_as_longlong(DBL_MAX);
    q.dmax_bits = 0ull;
  }
  init_stats(s);
  for (int i = 0; i <= j; ++i) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5, gr = i * TS + r, gc = j * TS + c;
      v[u] = (gr < b && gc < b) ? __ldcg(W + gr + size_t(gc) * bp) : (gr == gc ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5;
      G(i)[c * SLD + r] = v[u];
    }
  }
  for (int i = j; i < nb; ++i)
    for (int e = threadIdx.x; e < TS * TS; e += SNT) {
      const int r = e & 31, c = e >> 5;
      E(i)[c * SLD + r] = (i == j && r == c) ? 1.0 : 0.0;
    }
  cl.sync();  // every CTA's flags are initialised before anyone polls them
  DSM_MARK(j, 0);
  double acc[2][2];
  // ---- Cholesky steps p < j on column j
  for (int p = 0; p < j; ++p) {
    CholDsm* rp = remote(p);
    wait_flag(&rp->diag_done, 1);
    tile_copy(s.a, cl.map_shared_rank(s.dit, p), false);  // R_pp^-T
    __syncthreads();
    acc_zero(acc);
    tile_mma(acc, s.a, G(p));
    __syncthreads();
    acc_each(acc, [&](int r, int c, double v) { G(p)[c * SLD + r] = v; });  // R(p, j)
    publish(&q.row_done, p + 1);
    __syncthreads();
    // trailing update of column j, the diagonal tile (needed soonest by this CTA) first
    for (int ii = 0; ii < j - p; ++ii) {
      const int i = (ii == 0) ? j : p + ii;
      if (i == j) {
        tile_copy(s.b, G(p), true);  // R(p, j)^T
      } else {
        CholDsm* ri = remote(i);
        wait_flag(&ri->row_done, p + 1);
        tile_copy(s.b, ri->t[p], true);  // R(p, i)^T
      }
      __syncthreads();
      acc_zero(acc);
      tile_mma(acc, s.b, G(p));
      acc_sub_smem(acc, G(i));
      __syncthreads();
    }
  }
  // ---- diagonal tile j
  DSM_MARK(j, 1);
  for (int e = threadIdx.x; e < TS * TS; e += SNT) {
    const int r = e & 31, c = e >> 5;
    s.d[c * SLD + r] = G(j)[c * SLD + r];
  }
  __syncthreads();
  if (kChol2x2) cta_chol_inv2(s, q.rb, q.cb, j * TS, b);  // s.d = R_jj, s.di = R_jj^-1, s.dit = R_jj^-T
  else cta_chol_inv(s, j * TS, b);
  DSM_MARK(j, 2);
  for (int e = threadIdx.x; e < TS * TS; e += SNT) {
    const int r = e & 31, c = e >> 5;
    G(j)[c * SLD + r] = s.d[c * SLD + r];
    E(j)[c * SLD + r] = s.dit[c * SLD + r];  // E(j, j) = R_jj^-T I
  }
  publish(&q.diag_done, 1);
  if (threadIdx.x == 0) {  // stats into CTA 0 (non-negative doubles order like their bits)
    CholDsm* r0 = remote(0);
    if (s.bad) atomicOr(&r0->bad, 1);
    atomicMin(&r0->dmin_bits, (unsigned long long)__double_as_longlong(s.dmin));
    atomicMax(&r0->dmax_bits, (unsigned long long)__double_as_longlong(s.dmax));
  }
  // ---- column j of E = R^-T: steps p >= j
  for (int p = j; p < nb; ++p) {
    if (p > j) {
      CholDsm* rp = remote(p);
      wait_flag(&rp->diag_done, 1);
      tile_copy(s.a, cl.map_shared_rank(s.dit, p), false);  // R_pp^-T
      __syncthreads();
      acc_zero(acc);
      tile_mma(acc, s.a, E(p));
      __syncthreads();
      acc_each(acc, [&](int r, int c, double v) { E(p)[c * SLD + r] = v; });
      __syncthreads();
    }
    for (int i = p + 1; i < nb; ++i) {  // E(i, j) -= R(p, i)^T E(p, j)
      CholDsm* ri = remote(i);
      wait_flag(&ri->row_done, p + 1);
      tile_copy(s.b, ri->t[p], true);
      __syncthreads();
      acc_zero(acc);
      tile_mma(acc, s.b, E(p));
      acc_sub_smem(acc, E(i));
      __syncthreads();
    }
  }
  DSM_MARK(j, 3);
  // ---- outputs: R column j (zeros below the diagonal tile), Ri row block j = E(:, j)^T
  for (int i = 0; i < nb; ++i)
    for (int e = threadIdx.x; e < TS * TS; e += SNT) {
      const int r = e & 31, c = e >> 5;
      R[(i * TS + r) + size_t(j * TS + c) * bp] = (i <= j) ? G(i)[c * SLD + r] : 0.0;
      Ri[(j * TS + r) + size_t(i * TS + c) * bp] = (i >= j) ? E(i)[r * SLD + c] : 0.0;
    }
  cl.sync();  // no CTA exits while another may still read its shared memory
  DSM_MARK(j, 4);
  if (j == 0 && threadIdx.x == 0) {
    stats[0] = q.bad ? 1.0 : 0.0;
    stats[1] = __longlong_as_double((long long)q.dmin_bits);
    stats[2] = __longlong_as_double((long long)q.dmax_bits);
  }
}

// ---- sign-modified LU with L^-1 and U~^-1, resident in distributed shared
// memory (the reconstruction's LU, recon_lu_k's outputs), b <= 256: one
// cluster of nb CTAs, CTA j owns column j of F (becoming L \ U~), column j of
// E1 = L^-1 and column k2 = nb-1-j of E2 = U~^-T (forward elimination of
// U~^T; the two E columns of a CTA hold nb + 1 tiles together).  Right-looking
// at tile level with per-producer counters instead of cluster barriers:
//   diag_done: CTA j's diagonal tile is factored (s.di = L_jj^-1, s.e = U~_jj^-1);
//   urow_done = p + 1: U~(p, j) = L_pp^-1 F(p, j) is final in CTA j;
//   lcol_done = i: L(i', j) = F(i', j) U~_jj^-1 is final for i' <= i.
// The critical path per block step is the diagonal tile's factorisation plus
// one flag hop and three 32x32x32 products.
struct LuSm {
  double d[TSZ], di[TSZ], e[TSZ];  // the diagonal tile: in F, out L \ U~, L^-1, U~^-1 (cta_lu_sign_inv)
  double a[TSZ], b[TSZ];           // operand staging
  double aug[TS * 97];
  double piv[TS];
  double sgn[TS];
  double c[TS];
  double rowbuf[2][96];
  double colbuf[2][TS];
  double f[8][TSZ];     // column j of F
  double x[9][TSZ];     // E1(i, j), i >= j at x[i - j]; E2(i, k2), i >= k2 at x[nb - j + i - k2]
  volatile int diag_done, urow_done, lcol_done;
};

__global__ void __launch_bounds__(SNT, 1)
lu_dsm_k(SmallDims dd, double* __restrict__ F, double* __restrict__ Li, double* __restrict__ Ui,
         double* __restrict__ S, double* __restrict__ US) {
  pdl_begin();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double sm_raw[];
  LuSm& q = *reinterpret_cast<LuSm*>(sm_raw);
  const int j = (int)cl.block_rank(), nb = dd.nb, bp = dd.bp, k2 = nb - 1 - j;
  auto E1 = [&](int i) { return q.x[i - j]; };             // i >= j
  auto E2 = [&](int i) { return q.x[nb - j + i - k2]; };   // i >= k2
  auto remote = [&](int rank) { return cl.map_shared_rank(&q, rank); };
  if (threadIdx.x == 0) {
    q.diag_done = 0;
    q.urow_done = 0;
    q.lcol_done = j;
  }
  for (int i = 0; i < nb; ++i) {  // column j of F (zero-padded by recon_r2_k), E columns = [0; I; 0]
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5;
      v[u] = __ldcg(F + (i * TS + r) + size_t(j * TS + c) * bp);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * SNT, r = e & 31, c = e >> 5;
      q.f[i][c * SLD + r] = v[u];
    }
  }
  for (int t = 0; t <= nb; ++t)
    for (int e = threadIdx.x; e < TS * TS; e += SNT) {
      const int r = e & 31, c = e >> 5;
      q.x[t][c * SLD + r] = ((t == 0 || t == nb - j) && r == c) ? 1.0 : 0.0;  // E1(j, j) = I, E2(k2, k2) = I
    }
  cl.sync();
  LU_MARK(j, 0);
  double acc[2][2];
  // E2(p, k2) = U~_pp^-T E2(p, k2);  E2(i, k2) -= U~(p, i)^T E2(p, k2), i > p
  int e2_next = k2;  // next E2 step of this CTA
  auto e2_step = [&](int p) {
    LuSm* rp = remote(p);
    if (p != j) wait_flag(&rp->diag_done, 1);
    tile_copy(q.a, rp->e, true);  // U~_pp^-T
    __syncthreads();
    acc_zero(acc);
    tile_mma(acc, q.a, E2(p));
    __syncthreads();
    acc_each(acc, [&](int r, int c, double v) { E2(p)[c * SLD + r] = v; });
    __syncthreads();
    for (int i = p + 1; i < nb; ++i) {
      LuSm* ri = remote(i);
      if (i != j) wait_flag(&ri->urow_done, p + 1);
      tile_copy(q.b, ri->f[p], true);  // U~(p, i)^T
      __syncthreads();
      acc_zero(acc);
      tile_mma(acc, q.b, E2(p));
      acc_sub_smem(acc, E2(i));
      __syncthreads();
    }
    e2_next = p + 1;
  };
  // ---- phase 1: the LU steps p < j on column j
  for (int p = 0; p < j; ++p) {
    LuSm* rp = remote(p);
    wait_flag(&rp->diag_done, 1);
    tile_copy(q.a, rp->di, false);  // L_pp^-1
    __syncthreads();
    acc_zero(acc);
    tile_mma(acc, q.a, q.f[p]);
    __syncthreads();
    acc_each(acc, [&](int r, int c, double v) { q.f[p][c * SLD + r] = v; });  // U~(p, j)
    publish(&q.urow_done, p + 1);
    __syncthreads();
    // F(i, j) -= L(i, p) U~(p, j); at the last step before the diagonal only
    // the diagonal tile (the rest follows the diagonal factorisation)
    const int iend = (p == j - 1) ? j + 1 : nb;
    for (int i = p + 1; i < iend; ++i) {
      wait_flag(&rp->lcol_done, i);
      tile_copy(q.b, rp->f[i], false);
      __syncthreads();
      acc_zero(acc);
      tile_mma(acc, q.b, q.f[p]);
      acc_sub_smem(acc, q.f[i]);
      __syncthreads();
    }
    // this CTA waits for the next diagonal anyway: advance its E2 column
    // (its own U~(p, j) is final; the other columns' are published early)
    if (p < j - 1 && p >= k2 && e2_next == p) e2_step(p);
  }
  // ---- the diagonal tile j, then L(i, j) = F(i, j) U~_jj^-1 for i > j
  for (int e = threadIdx.x; e < TS * TS; e += SNT) {
    const int r = e & 31, c = e >> 5;
    q.d[c * SLD + r] = q.f[j][c * SLD + r];
  }
  __syncthreads();
  cta_lu_sign_inv(q);  // q.d = L_jj \ U~_jj (pivots on the diagonal), q.di = L_jj^-1, q.e = U~_jj^-1, q.sgn
  for (int e = threadIdx.x; e < TS * TS; e += SNT) {
    const int r = e & 31, c = e >> 5;
    q.f[j][c * SLD + r] = q.d[c * SLD + r];
  }
  publish(&q.diag_done, 1);
  LU_MARK(j, 2);
  __syncthreads();
  for (int i = j + 1; i < nb; ++i) {
    if (j > 0) {  // the deferred update of step j - 1 on tile (i, j)
      LuSm* rp = remote(j - 1);
      wait_flag(&rp->lcol_done, i);
      tile_copy(q.b, rp->f[i], false);
      __syncthreads();
      acc_zero(acc);
      tile_mma(acc, q.b, q.f[j - 1]);
      acc_sub_smem(acc, q.f[i]);
      __syncthreads();
    }
    acc_zero(acc);
    tile_mma(acc, q.f[i], q.e);  // L(i, j) = F(i, j) U~_jj^-1
    __syncthreads();
    acc_each(acc, [&](int r, int c, double v) { q.f[i][c * SLD + r] = v; });
    publish(&q.lcol_done, i);
    __syncthreads();
  }
  LU_MARK(j, 3);
  // ---- phases 2 and 3: E1 column j (steps p >= j), E2 column k2 (steps p >= k2)
  for (int p = 0; p < nb; ++p) {
    if (p >= j) {  // E1(p, j) = L_pp^-1 E1(p, j);  E1(i, j) -= L(i, p) E1(p, j), i > p
      LuSm* rp = remote(p);
      if (p > j) {
        wait_flag(&rp->diag_done, 1);
        tile_copy(q.a, rp->di, false);
      } else {
        tile_copy(q.a, q.di, false);
      }
      __syncthreads();
      acc_zero(acc);
      tile_mma(acc, q.a, E1(p));
      __syncthreads();
      acc_each(acc, [&](int r, int c, double v) { E1(p)[c * SLD + r] = v; });
      __syncthreads();
      for (int i = p + 1; i < nb; ++i) {
        wait_flag(&rp->lcol_done, i);
        tile_copy(q.b, rp->f[i], false);  // L(i, p)
        __syncthreads();
        acc_zero(acc);
        tile_mma(acc, q.b, E1(p));
        acc_sub_smem(acc, E1(i));
        __syncthreads();
      }
    }
    if (p >= e2_next) e2_step(p);
  }
  // ---- outputs: F = L \ U~ (column j), Li column j, Ui row block k2 = E2(:, k2)^T, S, US = U~ S
  if (threadIdx.x < TS) S[j * TS + threadIdx.x] = q.sgn[threadIdx.x];
  for (int i = 0; i < nb; ++i)
    for (int e = threadIdx.x; e < TS * TS; e += SNT) {
      const int r = e & 31, c = e >> 5, gr = i * TS + r, gc = j * TS + c;
      const double fv = q.f[i][c * SLD + r];
      F[gr + size_t(gc) * bp] = fv;
      Li[gr + size_t(gc) * bp] = (i >= j) ? E1(i)[c * SLD + r] : 0.0;
      US[gr + size_t(gc) * bp] = (gr <= gc) ? fv * q.sgn[c] : 0.0;
      Ui[(k2 * TS + r) + size_t(i * TS + c) * bp] = (i >= k2) ? E2(i)[r * SLD + c] : 0.0;
    }
  cl.sync();  // no CTA exits while another may still read its shared memory
  LU_MARK(j, 5);
}

struct ReconArgs {
  SmallDims d;
  double* W2;        // Gram of Q1 (b x b valid, ld bp), destroyed
  const double* R1;  // first-pass factor (bp x bp)
  const double* Q1;  // Q1 (ld ldq), its top b x b block is read
  int64_t ldq;
  double *R2, *R2i, *F, *Li, *Ui, *M, *US, *S;  // bp x bp workspaces (S: bp)
  const double* stats1;                          // chol_inv_k stats of the first pass
  double* Rh;                                    // out: R of the panel (b x b, ld ldr)
  int64_t ldr;
  double* Tw;                                    // out: compact-WY T (b x b, ld ldt)
  int64_t ldt;
  double* tau;                                   // out: b
  int* flag;                                     // out: 0 = reconstruction valid
  double dev_max;                                // max |G2 - I| accepted
};

// kernel 2a: second CholeskyQR pass (R2, R2^-1) and the validity flag.
// Also zero-pads F (written by the b x b GEMM F = -Q(0:b,:) R2^-1 next) and
// zeroes the strictly-lower tiles of R2, R2^-1.
__global__ void __launch_bounds__(SNT, 1) recon_r2_k(ReconArgs a) {
  pdl_begin();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double sm_raw[];
  SmallSm& s = *reinterpret_cast<SmallSm*>(sm_raw);
  __shared__ double devred[SNT / 32];
  const SmallDims d = a.d;
  const int C = (int)cl.num_blocks(), cta = (int)cl.block_rank();
  const int bp = d.bp, b = d.b;
  init_stats(s);
  cl.sync();  // every CTA's stats are initialised before any remote update
  // ---- deviation of G2 from I (before padding), padding, zero lower tiles.
  // This CTA's columns c = cta, cta + C, ... are walked in batches of 16
  // elements per thread with every load of a batch issued before its stores
  // (a load-store-load chain through possibly aliasing pointers serialised ~32
  // L2 round trips per thread: 30-65 us per launch)
  const int per_cta = ((bp - cta + C - 1) / C) * bp;
  {
    double dev = 0.0;
    for (int base = 0; base < per_cta; base += 16 * SNT) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = base + u * SNT + threadIdx.x, cc = idx / bp, r = idx - cc * bp, c = cta + cc * C;
        v[u] = (idx < per_cta && r < b && c < b && r <= c) ? __ldcg(a.W2 + c * bp + r) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = base + u * SNT + threadIdx.x, cc = idx / bp, r = idx - cc * bp, c = cta + cc * C;
        if (idx >= per_cta) continue;
        const int e = c * bp + r;
        if (r < b && c < b) {  // the upper triangle (the Gram GEMM writes only that)
          const double dv = (r <= c) ? v[u] - (r == c ? 1.0 : 0.0) : 0.0;
          dev = fmax(dev, isfinite(dv) ? fabs(dv) : 1e300);
        } else {
          a.W2[e] = (r == c) ? 1.0 : 0.0;
          a.F[e] = 0.0;
        }
        if (r / TS > c / TS) {
          a.R2[e] = 0.0;
          a.R2i[e] = 0.0;
        }
      }
    }
    for (int o = 16; o; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    if ((threadIdx.x & 31) == 0) devred[threadIdx.x >> 5] = dev;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int w = 0; w < SNT / 32; ++w) m = fmax(m, devred[w]);
      if (!(m <= a.dev_max)) atomicOr(cl.map_shared_rank(&s.bad, 0), 1);
      // non-negative doubles order like their bit patterns (NaN/inf were mapped to 1e300)
      atomicMax(cl.map_shared_rank(&s.devbits, 0), (unsigned long long)__double_as_longlong(m));
    }
    __syncthreads();
  }
  cluster_barrier(cl);
  // ---- G2 = Q1^T Q1 = I + E: when b max|E| <= 1e-8 the factor and its inverse
  // are, to O((b max|E|)^2) <= 1e-16,
  //   R2 = I + U(E),  R2^-1 = I - U(E),  U(E) = striu(E) + diag(E)/2
  // (R2^T R2 = I + U + U^T + O(E^2) = I + E), so the 8-step Cholesky is skipped.
  const double devmax = __longlong_as_double((long long)*cl.map_shared_rank(&s.devbits, 0));
  if (double(b) * devmax <= 1e-8) {
    for (int base = 0; base < per_cta; base += 16 * SNT) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = base + u * SNT + threadIdx.x, cc = idx / bp, r = idx - cc * bp, c = cta + cc * C;
        v[u] = (idx < per_cta && r < b && c < b && r <= c) ? __ldcg(a.W2 + c * bp + r) - (r == c ? 1.0 : 0.0)
                                                            : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = base + u * SNT + threadIdx.x, cc = idx / bp, r = idx - cc * bp, c = cta + cc * C;
        if (idx >= per_cta) continue;
        const int e = c * bp + r;
        const double uu = (r < c) ? v[u] : (r == c ? 0.5 * v[u] : 0.0);
        a.R2[e] = (r == c ? 1.0 : 0.0) + uu;
        a.R2i[e] = (r == c ? 1.0 : 0.0) - uu;
      }
    }
  } else {
    chol_inv_dev(cl, d, a.W2, a.R2, a.R2i, s);
  }
  cl.sync();
  if (cta == 0 && threadIdx.x == 0) {
    const bool bad1 = a.stats1[0] != 0.0;
    *a.flag = (bad1 || s.bad) ? 1 : 0;
  }
}

// kernel 2b: sign-modified LU of F (padded bp x bp, F = -Q(0:b,:) R2^-1) with
// L^-1, U~^-1 built along; then US = U~ S.  Zeroes the tiles of Li above and
// of Ui / US below the diagonal first.
__global__ void __launch_bounds__(SNT, 1) recon_lu_k(ReconArgs a) {
  pdl_begin();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double sm_raw[];
  SmallSm& s = *reinterpret_cast<SmallSm*>(sm_raw);
  const SmallDims d = a.d;
  const int C = (int)cl.num_blocks(), cta = (int)cl.block_rank();
  const int bp = d.bp;
  for (int c = cta; c < bp; c += C)  // column-strided: no 64-bit division per element
    for (int r = threadIdx.x, e = c * bp + threadIdx.x; r < bp; r += SNT, e += SNT) {
    if (r / TS > c / TS) {
      a.Ui[e] = 0.0;
      a.US[e] = 0.0;
    }
    if (r / TS < c / TS) a.Li[e] = 0.0;
  }
  cluster_barrier(cl);
  lu_sign_inv_dev(cl, d, a.F, a.Li, a.Ui, a.S, s);
  const int per_cta = ((bp - cta + C - 1) / C) * bp;  // batched as in recon_r2_k: loads before stores
  for (int base = 0; base < per_cta; base += 16 * SNT) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = base + u * SNT + threadIdx.x, cc = idx / bp, r = idx - cc * bp, c = cta + cc * C;
      v[u] = (idx < per_cta && r <= c) ? __ldcg(a.F + c * bp + r) * __ldcg(a.S + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = base + u * SNT + threadIdx.x, cc = idx / bp, r = idx - cc * bp, c = cta + cc * C;
      if (idx < per_cta && r / TS <= c / TS) a.US[c * bp + r] = v[u];
    }
  }
}

// kernel 2c (any grid): tau = diag(T_w), R_h = S (R2 R1) (upper), zeros below
// the diagonal of R_h and T_w.
__global__ void recon_finish_k(int b, int bp, const double* __restrict__ S, const double* __restrict__ RR,
                               double* __restrict__ Rh, int64_t ldr, double* __restrict__ Tw, int64_t ldt,
                               double* __restrict__ tau) {
  pdl_begin();
  for (int c = blockIdx.x; c < b; c += gridDim.x)
    for (int r = threadIdx.x; r < b; r += blockDim.x) {
    Rh[r + c * ldr] = (r <= c) ? S[r] * RR[r + int64_t(c) * bp] : 0.0;
    if (r > c) Tw[r + c * ldt] = 0.0;
    if (r == c) tau[r] = Tw[r + c * ldt];
  }
}

// V(0:b, 0:b) <- unit lower L (strict lower part of F, ld bp)
__global__ void put_unit_lower_k(int b, const double* __restrict__ F, int bp, double* __restrict__ V, int64_t ldv) {
  pdl_begin();
  for (int c = blockIdx.x; c < b; c += gridDim.x)
    for (int r = threadIdx.x; r < b; r += blockDim.x) {
    V[r + c * ldv] = (r > c) ? F[r + int64_t(c) * bp] : (r == c ? 1.0 : 0.0);
  }
}

size_t chol_dsm_smem() { return (sizeof(SmallSm) + 15) / 16 * 16 + sizeof(CholDsm); }

template <class K, class... Args>
void launch_cluster_smem(K kern, cudaStream_t st, int C, size_t smem, Args... args) {
  static SmemAttrPerDevice attr;
  attr.ensure(kern, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(SNT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  RUTV_CK(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <class K, class... Args>
void launch_cluster(K kern, cudaStream_t st, int C, Args... args) {
  // one attribute call per kernel (several kernels share the type K)
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;  // (kernel, device)
  const size_t smem = sizeof(SmallSm);
  {
    std::lock_guard<std::mutex> lock(mu);
    const std::pair<const void*, int> key((const void*)kern, current_device());
    if (std::find(done.begin(), done.end(), key) == done.end()) {
      RUTV_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      done.push_back(key);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(SNT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  RUTV_CK(cudaLaunchKernelEx(&cfg, kern, args...));
}
}  // namespace

int small_pad(int64_t b) { return (int)cdiv(b, TS) * TS; }

size_t small_work_elems(int64_t b) {
  const size_t bp = size_t(small_pad(b));
  return size_t(14) * bp * bp + 2 * bp + 64;
}

SmallWork carve_small(double* base, int64_t b) {
  const size_t bp = size_t(small_pad(b)), q = bp * bp;
  SmallWork w;
  w.bp = (int)bp;
  double* p = base;
  w.W1 = p; p += q;
  w.R1 = p; p += q;
  w.R1i = p; p += q;
  w.W2 = p; p += q;
  w.R2 = p; p += q;
  w.R2i = p; p += q;
  w.F = p; p += q;
  w.Li = p; p += q;
  w.Ui = p; p += q;
  w.M = p; p += q;
  w.US = p; p += q;
  w.S = p; p += bp;
  w.stats = p; p += 16;
  w.flag = reinterpret_cast<int*>(p); p += 16;
  return w;
}

void small_chol_inv(cudaStream_t st, int64_t b, const SmallWork& w) {
  SmallDims d{(int)b, w.bp, w.bp / TS};
  ProfScope _p(st, C_QR_SMALL, 0.0);
  count_launch(C_QR_SMALL);
  static const bool legacy = getenv("RANDUTV_CHOL_L2") != nullptr;  // experiment: the L2-resident kernel
  if (d.nb <= 8 && !legacy) {
    launch_cluster_smem(chol_inv_dsm_k, st, d.nb, chol_dsm_smem(), d, (const double*)w.W1, w.R1, w.R1i, w.stats);
  } else {
    launch_cluster(chol_inv_k, st, SC, d, w.W1, w.R1, w.R1i, w.stats);
  }
}

void small_recon(cudaStream_t st, int64_t b, const SmallWork& w, const double* Q1, int64_t ldq, double* R,
                 int64_t ldr, double* tau, double* Tw, int64_t ldt, double* part, size_t part_elems,
                 cudaStream_t side, cudaEvent_t ev_fork, cudaEvent_t ev_join, double dev_max) {
  ReconArgs a;
  a.d = SmallDims{(int)b, w.bp, w.bp / TS};
  a.W2 = w.W2;
  a.R1 = w.R1;
  a.Q1 = Q1;
  a.ldq = ldq;
  a.R2 = w.R2;
  a.R2i = w.R2i;
  a.F = w.F;
  a.Li = w.Li;
  a.Ui = w.Ui;
  a.M = w.M;
  a.US = w.US;
  a.S = w.S;
  a.stats1 = w.stats;
  a.Rh = R;
  a.ldr = ldr;
  a.Tw = Tw;
  a.ldt = ldt;
  a.tau = tau;
  a.flag = w.flag;
  a.dev_max = dev_max;
  const int bp = w.bp;
  {
    ProfScope _p(st, C_QR_SMALL, 0.0);
    count_launch(C_QR_SMALL);
    launch_cluster(recon_r2_k, st, SC, a);
  }
  // the b x b products run GPU-wide (upper-triangular right operands: TRMM)
  dgemm(st, false, false, b, b, b, -1.0, Q1, ldq, w.R2i, bp, 0.0, w.F, bp, part, part_elems, 0, true);  // F
  {
    ProfScope _p(st, C_QR_SMALL, 0.0);
    count_launch(C_QR_SMALL);
    static const bool legacy = getenv("RANDUTV_LU_L2") != nullptr;  // experiment: the L2-resident kernel
    if (a.d.nb <= 8 && !legacy)
      launch_cluster_smem(lu_dsm_k, st, a.d.nb, sizeof(LuSm), a.d, a.F, a.Li, a.Ui, a.S, a.US);
    else
      launch_cluster(recon_lu_k, st, SC, a);
  }
  // M (needed next by W = -Q1(b:) M) stays on st; T_w, tau and R_h are not
  // needed until after the caller's W GEMM, so with a side stream they are
  // formed concurrently with it (unsplit GEMMs: the split-K scratch is st's)
  cudaStream_t ts = side ? side : st;
  if (side) {
    RUTV_CK(cudaEventRecord(ev_fork, st));
    RUTV_CK(cudaStreamWaitEvent(side, ev_fork, 0));
  }
  double* tpart = side ? nullptr : part;
  const size_t tpe = side ? 0 : part_elems;
  dgemm(st, false, false, b, b, b, 1.0, w.R2i, bp, w.Ui, bp, 0.0, w.M, bp, part, part_elems, 0, true);  // M = R2^-1 U~^-1
  dgemm(ts, false, true, b, b, b, 1.0, w.US, bp, w.Li, bp, 0.0, Tw, ldt, tpart, tpe, 0, true);     // T = US Li^T
  dgemm(ts, false, false, b, b, b, 1.0, w.R2, bp, w.R1, bp, 0.0, w.W2, bp, tpart, tpe, 0, true);   // R2 R1 (W2 is free)
  {
    ProfScope _p(ts, C_QR_SMALL, 0.0);
    count_launch(C_QR_SMALL);
    launch_k(recon_finish_k, dim3((int)std::min<int64_t>(b, 256)), dim3(256), 0, ts, (int)b, bp, w.S, w.W2, R, ldr, Tw,
                                                                                    ldt, tau);
    RUTV_LAUNCH_CK();
  }
  if (side) RUTV_CK(cudaEventRecord(ev_join, side));
}

void small_put_unit_lower(cudaStream_t st, int64_t b, const SmallWork& w, double* V, int64_t ldv) {
  ProfScope _p(st, K_MISC, 0.0);
  count_launch(K_MISC);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(b * b, 256), 512));
  launch_k(put_unit_lower_k, dim3(blocks), dim3(256), 0, st, (int)b, w.F, w.bp, V, ldv);
  RUTV_LAUNCH_CK();
}

}  // namespace rutv
