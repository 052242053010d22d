// Batched one-sided (Hestenes) Jacobi SVD of the b x b blocks R_11 of every
// step (PAPER.md:964 ``svd(R(1:b,1:b))``) and of the final block.
//
// run on B = R^T (QR-preconditioned, 11-15
// sweeps).  B W -> columns mutually orthogonal; then
//     R = Us diag(D) Vs^T  with  Us = W(:, perm),  Vs = B(:, perm) / D.
// Block-cyclic ordering: the k columns are split into nb blocks of kb columns;
// one launch per tournament round pairs the blocks, each CTA loads a block pair
// of B and W (2 kb columns, <= 128 KB) into shared memory and performs one
// cyclic sweep over all its column pairs (round-robin, one warp per pair).
// A sweep with no rotation (|gamma| <= tol sqrt(alpha beta), tol = k eps)
// marks the matrix converged and later launches exit immediately.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <vector>

namespace rutv {

namespace {
constexpr int JNT = 256;
constexpr int MAX_SWEEPS = 40;

struct JacobiDesc {
  int k, kb, nb;  // matrix order, block width, number of blocks (even)
};

__global__ void jacobi_init_k(int batch, int k, const double* __restrict__ R, int64_t ldr, int64_t strideR,
                              double* __restrict__ Bw, double* __restrict__ Wm, int* __restrict__ counts) {
  const int mat = blockIdx.y;
  const double* Ri = R + int64_t(mat) * strideR;
  double* B = Bw + int64_t(mat) * k * k;
  double* W = Wm + int64_t(mat) * k * k;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < int64_t(k) * k;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int r = int(idx % k), c = int(idx / k);
    B[idx] = Ri[c + int64_t(r) * ldr];  // B = R^T
    W[idx] = (r == c) ? 1.0 : 0.0;
  }
  if (blockIdx.x == 0)
    for (int s = threadIdx.x; s <= MAX_SWEEPS; s += blockDim.x) counts[mat * (MAX_SWEEPS + 1) + s] = (s == 0);
}

__device__ __forceinline__ void rr_pair(int nplayers, int round, int i, int& p, int& q) {
  // circle method over nplayers (even): player nplayers-1 fixed
  const int n1 = nplayers - 1;
  if (i == 0) {
    p = round % n1;
    q = n1;
  } else {
    p = (round + i) % n1;
    q = (round - i + n1) % n1;
  }
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
}

// One block-pair operation for tournament round ``round`` of sweep ``sweep``.
__global__ void __launch_bounds__(JNT)
jacobi_round_k(JacobiDesc d, int sweep, int round, double* __restrict__ Bw, double* __restrict__ Wm,
               int* __restrict__ counts, double tol) {
  extern __shared__ __align__(16) double js[];
  const int mat = blockIdx.y;
  int* cnt = counts + mat * (MAX_SWEEPS + 1);
  if (cnt[sweep] == 0) return;  // previous sweep did no rotation: converged
  const int k = d.k, kb = d.kb;
  int bp, bq;
  rr_pair(d.nb, round, blockIdx.x, bp, bq);
  double* B = Bw + int64_t(mat) * k * k;
  double* W = Wm + int64_t(mat) * k * k;
  const int ncol = 2 * kb;
  double* sB = js;                     // [ncol][k]
  double* sW = js + size_t(ncol) * k;  // [ncol][k]
  // column c of the pair -> global column
  auto gcol = [&](int c) { return (c < kb) ? bp * kb + c : bq * kb + (c - kb); };
  for (int idx = threadIdx.x; idx < ncol * k; idx += JNT) {
    int c = idx / k, r = idx % k;
    int g = gcol(c);
    bool ok = g < k;
    sB[idx] = ok ? B[r + int64_t(g) * k] : 0.0;
    sW[idx] = ok ? W[r + int64_t(g) * k] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int rotations = 0;
  for (int rnd = 0; rnd < ncol - 1; ++rnd) {
    for (int pi = warp; pi < kb; pi += JNT / 32) {
      int p, q;
      rr_pair(ncol, rnd, pi, p, q);
      if (gcol(p) >= k || gcol(q) >= k) continue;
      double* bp_ = sB + size_t(p) * k;
      double* bq_ = sB + size_t(q) * k;
      double al = 0.0, be = 0.0, ga = 0.0;
      for (int r = lane; r < k; r += 32) {
        double x = bp_[r], y = bq_[r];
        al = fma(x, x, al);
        be = fma(y, y, be);
        ga = fma(x, y, ga);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      if (ga != 0.0 && fabs(ga) > tol * sqrt(al) * sqrt(be)) {
        double zeta = (be - al) / (2.0 * ga);
        double t = (fabs(zeta) > 1e150) ? 0.5 / zeta
                                        : copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        double c = 1.0 / sqrt(fma(t, t, 1.0));
        double s = c * t;
        double* wp = sW + size_t(p) * k;
        double* wq = sW + size_t(q) * k;
        for (int r = lane; r < k; r += 32) {
          double x = bp_[r], y = bq_[r];
          bp_[r] = c * x - s * y;
          bq_[r] = s * x + c * y;
          double u = wp[r], v = wq[r];
          wp[r] = c * u - s * v;
          wq[r] = s * u + c * v;
        }
        if (lane == 0) ++rotations;
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < ncol * k; idx += JNT) {
    int c = idx / k, r = idx % k;
    int g = gcol(c);
    if (g < k) {
      B[r + int64_t(g) * k] = sB[idx];
      W[r + int64_t(g) * k] = sW[idx];
    }
  }
  if (lane == 0 && rotations) atomicAdd(&cnt[sweep + 1], rotations);
}

// sigma_j = ||B(:,j)||, sort descending, Us = W(:,perm), Vs = B(:,perm)/sigma.
__global__ void __launch_bounds__(JNT)
jacobi_finalize_k(int k, const double* __restrict__ Bw, const double* __restrict__ Wm, double* __restrict__ D,
                  double* __restrict__ Us, double* __restrict__ Vs, const int* __restrict__ counts,
                  int* __restrict__ sweeps_out) {
  extern __shared__ __align__(16) double fs[];
  double* sig = fs;                           // k
  int* rank = reinterpret_cast<int*>(fs + k);  // k
  const int mat = blockIdx.x;
  const double* B = Bw + int64_t(mat) * k * k;
  const double* W = Wm + int64_t(mat) * k * k;
  double* Di = D + int64_t(mat) * k;
  double* Ui = Us + int64_t(mat) * k * k;
  double* Vi = Vs + int64_t(mat) * k * k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < k; j += JNT / 32) {
    double s = 0.0;
    for (int r = lane; r < k; r += 32) s = fma(B[r + int64_t(j) * k], B[r + int64_t(j) * k], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sig[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += JNT) {
    int rk = 0;
    double sj = sig[j];
    for (int i = 0; i < k; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
    rank[j] = rk;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < k * k; idx += JNT) {
    int r = idx % k, j = idx / k;
    int dst = rank[j];
    double s = sig[j];
    Ui[r + int64_t(dst) * k] = W[idx];
    Vi[r + int64_t(dst) * k] = (s > 1e-290) ? B[idx] / s : 0.0;
  }
  for (int j = threadIdx.x; j < k; j += JNT) Di[rank[j]] = sig[j];
  __syncthreads();
  // complete Vs for (numerically) zero singular values: Gram-Schmidt against e_c
  int nz = 0;
  for (int j = 0; j < k; ++j) nz += (sig[j] <= 1e-290);
  __syncthreads();
  if (nz == 0) {
    if (threadIdx.x == 0 && sweeps_out) {
      int s = 0;
      while (s < MAX_SWEEPS && counts[mat * (MAX_SWEEPS + 1) + s + 1] > 0) ++s;
      sweeps_out[mat] = s + 1;
    }
    return;
  }
  double* x = fs;  // reuse: k doubles (sig no longer needed)
  __shared__ double red[JNT / 32];
  int cand = 0;
  for (int slot = k - nz; slot < k; ++slot) {
    for (;; ++cand) {
      for (int r = threadIdx.x; r < k; r += JNT) x[r] = (r == cand) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int c = 0; c < slot; ++c) {
          const double* v = Vi + int64_t(c) * k;
          double s = 0.0;
          for (int r = threadIdx.x; r < k; r += JNT) s = fma(v[r], x[r], s);
          for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) red[warp] = s;
          __syncthreads();
          double tot = 0.0;
          for (int w2 = 0; w2 < JNT / 32; ++w2) tot += red[w2];
          for (int r = threadIdx.x; r < k; r += JNT) x[r] -= tot * v[r];
          __syncthreads();
        }
      }
      double s = 0.0;
      for (int r = threadIdx.x; r < k; r += JNT) s = fma(x[r], x[r], s);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      double tot = 0.0;
      for (int w2 = 0; w2 < JNT / 32; ++w2) tot += red[w2];
      __syncthreads();
      if (tot > 0.25) {
        double inv = 1.0 / sqrt(tot);
        for (int r = threadIdx.x; r < k; r += JNT) Vi[r + int64_t(slot) * k] = x[r] * inv;
        __syncthreads();
        ++cand;
        break;
      }
    }
  }
  if (threadIdx.x == 0 && sweeps_out) {
    int s = 0;
    while (s < MAX_SWEEPS && counts[mat * (MAX_SWEEPS + 1) + s + 1] > 0) ++s;
    sweeps_out[mat] = s + 1;
  }
}

JacobiDesc make_desc(int k) {
  JacobiDesc d;
  // 2 kb columns of B and W in shared memory: 32 kb k bytes <= ~200 KB
  int kb = 16;
  while (kb > 1 && size_t(32) * kb * k > 200 * 1024) kb /= 2;
  d.k = k;
  d.kb = kb;
  d.nb = (int)cdiv(k, kb);
  if (d.nb % 2) d.nb += 1;
  if (d.nb < 2) d.nb = 2;
  return d;
}
}  // namespace

size_t jacobi_work_elems(int batch, int k) { return size_t(2) * batch * k * k + size_t(batch) * (MAX_SWEEPS + 1); }

void jacobi_svd_batched(cudaStream_t st, int batch, int k, const double* R, int64_t ldr, int64_t strideR,
                        double* D, double* Us, double* Vs, double* work, int* sweeps_out) {
  if (batch <= 0 || k <= 0) return;
  JacobiDesc d = make_desc(k);
  double* Bw = work;
  double* Wm = work + size_t(batch) * k * k;
  int* counts = reinterpret_cast<int*>(work + size_t(2) * batch * k * k);
  {
    dim3 g((unsigned)std::min<int64_t>(cdiv(int64_t(k) * k, 256), 64), batch);
    { ProfScope _p(st, K_SVD, 0.0); count_launch(K_SVD); jacobi_init_k<<<g, 256, 0, st>>>(batch, k, R, ldr, strideR, Bw, Wm, counts); }
    RUTV_LAUNCH_CK();
  }
  const size_t smem = size_t(2) * 2 * d.kb * k * sizeof(double);
  static size_t attr_smem = 0;
  if (smem > 48 * 1024 && smem > attr_smem) {
    RUTV_CK(cudaFuncSetAttribute(jacobi_round_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_smem = smem;
  }
  const double tol = double(k) * DBL_EPSILON;
  if (k > 1) {
    // Sweeps are launched in chunks; between chunks the host reads the
    // per-matrix rotation counts once (one sync) and stops when all converged.
    int sweep = 0;
    int chunk = 8;
    std::vector<int> h(size_t(batch) * (MAX_SWEEPS + 1));
    while (sweep < MAX_SWEEPS) {
      int end = std::min(MAX_SWEEPS, sweep + chunk);
      for (; sweep < end; ++sweep) {
        for (int round = 0; round < d.nb - 1; ++round) {
          dim3 g(d.nb / 2, batch);
          { ProfScope _p(st, K_SVD, 0.0); count_launch(K_SVD); jacobi_round_k<<<g, JNT, smem, st>>>(d, sweep, round, Bw, Wm, counts, tol); }
          RUTV_LAUNCH_CK();
        }
      }
      RUTV_CK(cudaMemcpyAsync(h.data(), counts, sizeof(int) * h.size(), cudaMemcpyDeviceToHost, st));
      RUTV_CK(cudaStreamSynchronize(st));
      bool all = true;
      for (int b = 0; b < batch; ++b) all &= (h[size_t(b) * (MAX_SWEEPS + 1) + sweep] == 0);
      if (all) break;
      chunk = 2;
    }
  }
  const size_t fsmem = size_t(k) * (sizeof(double) + sizeof(int)) + 16;
  static size_t attr_f = 0;
  if (fsmem > 48 * 1024 && fsmem > attr_f) {
    RUTV_CK(cudaFuncSetAttribute(jacobi_finalize_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
    attr_f = fsmem;
  }
  { ProfScope _p(st, K_SVD, 0.0); count_launch(K_SVD); jacobi_finalize_k<<<batch, JNT, fsmem, st>>>(k, Bw, Wm, D, Us, Vs, counts, sweeps_out); }
  RUTV_LAUNCH_CK();
}

}  // namespace rutv
