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
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <vector>

namespace cg = cooperative_groups;

namespace rutv {

namespace {
constexpr int JNT = 512;
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

// One cyclic sweep over all column pairs of a block pair held in shared
// memory (sB, sW: ncol columns of length k <= 32*EPL), one warp per pair and
// round.  Each lane keeps its EPL elements of the two columns in registers
// (fully unrolled: the loads, the dot product and the W loads are issued
// back to back).  Column norms are computed once and then tracked with
// Rutishauser's exact update (alpha' = alpha - t gamma, beta' = beta + t
// gamma), so a pair costs a single warp reduction.  Returns this warp's
// rotation count.
template <int EPL>
__device__ int pair_sweep(double* sB, double* sW, double* nrm, int k, int ncol, int kb, int bp, int bq, double tol) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  auto valid = [&](int c) { return ((c < kb) ? bp * kb + c : bq * kb + (c - kb)) < k; };
  for (int c = warp; c < ncol; c += nw) {
    const double* x = sB + size_t(c) * k;
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const int r = lane + 32 * e;
      const double v = (r < k) ? x[r] : 0.0;
      s = fma(v, v, s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) nrm[c] = s;
  }
  __syncthreads();
  int rotations = 0;
  for (int rnd = 0; rnd < ncol - 1; ++rnd) {
    for (int pi = warp; pi < ncol / 2; pi += nw) {
      int p, q;
      rr_pair(ncol, rnd, pi, p, q);
      if (!valid(p) || !valid(q)) continue;
      double* bp_ = sB + size_t(p) * k;
      double* bq_ = sB + size_t(q) * k;
      double x[EPL], y[EPL];
      double ga = 0.0;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const int r = lane + 32 * e;
        x[e] = (r < k) ? bp_[r] : 0.0;
        y[e] = (r < k) ? bq_[r] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < EPL; ++e) ga = fma(x[e], y[e], ga);
#pragma unroll
      for (int o = 16; o; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
      const double al = nrm[p], be = nrm[q];
      if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
        double* wp = sW + size_t(p) * k;
        double* wq = sW + size_t(q) * k;
        constexpr int EPW = EPL <= 8 ? EPL : 1;  // W elements preloaded (register budget at 512 threads)
        double u[EPW], v[EPW];
        if constexpr (EPL <= 8) {
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            const int r = lane + 32 * e;
            u[e] = (r < k) ? wp[r] : 0.0;
            v[e] = (r < k) ? wq[r] : 0.0;
          }
        }
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (fabs(zeta) > 1e150) ? 0.5 / zeta
                                              : copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = rsqrt(fma(t, t, 1.0));
        const double s = c * t;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int r = lane + 32 * e;
          if (r < k) {
            bp_[r] = c * x[e] - s * y[e];
            bq_[r] = s * x[e] + c * y[e];
            const double uu = (EPL <= 8) ? u[e < EPW ? e : 0] : wp[r];
            const double vv = (EPL <= 8) ? v[e < EPW ? e : 0] : wq[r];
            wp[r] = c * uu - s * vv;
            wq[r] = s * uu + c * vv;
          }
        }
        if (lane == 0) {
          nrm[p] = al - t * ga;
          nrm[q] = be + t * ga;
          ++rotations;
        }
      }
    }
    __syncthreads();
  }
  return rotations;
}

__device__ __forceinline__ int pair_sweep_any(double* sB, double* sW, double* nrm, int k, int ncol, int kb, int bp,
                                              int bq, double tol) {
  if (k <= 32) return pair_sweep<1>(sB, sW, nrm, k, ncol, kb, bp, bq, tol);
  if (k <= 64) return pair_sweep<2>(sB, sW, nrm, k, ncol, kb, bp, bq, tol);
  if (k <= 128) return pair_sweep<4>(sB, sW, nrm, k, ncol, kb, bp, bq, tol);
  if (k <= 256) return pair_sweep<8>(sB, sW, nrm, k, ncol, kb, bp, bq, tol);
  return pair_sweep<16>(sB, sW, nrm, k, ncol, kb, bp, bq, tol);  // k <= 512 (larger k: see jacobi_svd_batched)
}

__device__ void load_pair(double* sB, double* sW, const double* B, const double* W, int k, int kb, int bp, int bq) {
  const int ncol = 2 * kb;
  for (int idx = threadIdx.x; idx < ncol * k; idx += blockDim.x) {
    int c = idx / k, r = idx % k;
    int g = (c < kb) ? bp * kb + c : bq * kb + (c - kb);
    bool ok = g < k;
    sB[idx] = ok ? __ldcg(B + r + int64_t(g) * k) : 0.0;
    sW[idx] = ok ? __ldcg(W + r + int64_t(g) * k) : 0.0;
  }
}

__device__ void store_pair(const double* sB, const double* sW, double* B, double* W, int k, int kb, int bp, int bq) {
  const int ncol = 2 * kb;
  for (int idx = threadIdx.x; idx < ncol * k; idx += blockDim.x) {
    int c = idx / k, r = idx % k;
    int g = (c < kb) ? bp * kb + c : bq * kb + (c - kb);
    if (g < k) {
      __stcg(B + r + int64_t(g) * k, sB[idx]);
      __stcg(W + r + int64_t(g) * k, sW[idx]);
    }
  }
}

// One block-pair operation for tournament round ``round`` of sweep ``sweep``
// (one launch per round; used when a matrix's blocks do not fit one cluster).
__global__ void __launch_bounds__(JNT)
jacobi_round_k(JacobiDesc d, int sweep, int round, double* __restrict__ Bw, double* __restrict__ Wm,
               int* __restrict__ counts, double tol) {
  extern __shared__ __align__(16) double js[];
  __shared__ double nrm[64];
  const int mat = blockIdx.y;
  int* cnt = counts + mat * (MAX_SWEEPS + 1);
  if (cnt[sweep] == 0) return;  // previous sweep did no rotation: converged
  const int k = d.k, kb = d.kb;
  int bp, bq;
  rr_pair(d.nb, round, blockIdx.x, bp, bq);
  double* B = Bw + int64_t(mat) * k * k;
  double* W = Wm + int64_t(mat) * k * k;
  double* sB = js;
  double* sW = js + size_t(2 * kb) * k;
  load_pair(sB, sW, B, W, k, kb, bp, bq);
  __syncthreads();
  int rot = pair_sweep_any(sB, sW, nrm, k, 2 * kb, kb, bp, bq, tol);
  store_pair(sB, sW, B, W, k, kb, bp, bq);
  if ((threadIdx.x & 31) == 0 && rot) atomicAdd(&cnt[sweep + 1], rot);
}

// Whole Jacobi SVD of one matrix per cluster (nb/2 CTAs, one block pair
// each): the tournament rounds and the sweeps run inside the kernel, with a
// cluster barrier between rounds (columns move between CTAs through L2) and a
// cluster-wide rotation count deciding convergence.
__global__ void __launch_bounds__(JNT)
jacobi_cluster_k(JacobiDesc d, double* __restrict__ Bw, double* __restrict__ Wm, int* __restrict__ counts,
                 double tol) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double js[];
  __shared__ double nrm[64];
  __shared__ int rot_sm;
  const int mat = blockIdx.y;
  const int cta = (int)cluster.block_rank();
  int* cnt = counts + mat * (MAX_SWEEPS + 1);
  const int k = d.k, kb = d.kb;
  double* B = Bw + int64_t(mat) * k * k;
  double* W = Wm + int64_t(mat) * k * k;
  double* sB = js;
  double* sW = js + size_t(2 * kb) * k;
  for (int sweep = 0; sweep < MAX_SWEEPS; ++sweep) {
    if (threadIdx.x == 0) rot_sm = 0;
    __syncthreads();
    int rot = 0;
    for (int round = 0; round < d.nb - 1; ++round) {
      int bp, bq;
      rr_pair(d.nb, round, cta, bp, bq);
      load_pair(sB, sW, B, W, k, kb, bp, bq);
      __syncthreads();
      rot += pair_sweep_any(sB, sW, nrm, k, 2 * kb, kb, bp, bq, tol);
      store_pair(sB, sW, B, W, k, kb, bp, bq);
      __threadfence();
      cluster.sync();
    }
    if ((threadIdx.x & 31) == 0 && rot) atomicAdd(&rot_sm, rot);
    __syncthreads();
    if (threadIdx.x == 0 && rot_sm) atomicAdd(&cnt[sweep + 1], rot_sm);
    __threadfence();
    cluster.sync();
    const int total = atomicAdd(&cnt[sweep + 1], 0);
    if (total == 0) break;
  }
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

constexpr int MAX_CLUSTER = 8;

JacobiDesc make_desc(int k) {
  JacobiDesc d;
  // 2 kb columns of B and W in shared memory: 32 kb k bytes <= ~200 KB.  One
  // warp rotates one column pair per sub-round; a sub-round's latency grows
  // with the warps contending for the FP64 pipe, while the number of
  // sequential sub-rounds per sweep (~2k) does not depend on kb, so prefer
  // narrow blocks (kb = 8: 8 warps) as long as the matrix fits one cluster.
  int kb = 16;
  while (kb > 1 && size_t(32) * kb * k > 200 * 1024) kb /= 2;
  // (kb = 8 on a 16-CTA cluster for k = 256 was measured: 25 % lower latency
  // per matrix but 2x the SMs per matrix -- slower overall as a side stream)
  d.k = k;
  d.kb = kb;
  d.nb = (int)cdiv(k, kb);
  if (d.nb % 2) d.nb += 1;
  if (d.nb < 2) d.nb = 2;
  return d;
}
}  // namespace

bool jacobi_single_launch(int k) {
  JacobiDesc d = make_desc(k);
  return k > 1 && d.nb / 2 <= MAX_CLUSTER;
}

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
  const double tol = double(k) * DBL_EPSILON;
  const int csize = d.nb / 2;
  if (k > 1 && csize <= MAX_CLUSTER) {
    // one cluster per matrix runs every round and sweep in-kernel
    static size_t attr_c = 0;
    if (smem > attr_c) {
      RUTV_CK(cudaFuncSetAttribute(jacobi_cluster_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      RUTV_CK(cudaFuncSetAttribute(jacobi_cluster_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr_c = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize, batch, 1);
    cfg.blockDim = dim3(32 * d.kb, 1, 1);  // one warp per column pair of a block pair
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope _p(st, K_SVD, 0.0);
    count_launch(K_SVD);
    RUTV_CK(cudaLaunchKernelEx(&cfg, jacobi_cluster_k, d, Bw, Wm, counts, tol));
  } else if (k > 1) {
    static size_t attr_smem = 0;
    if (smem > 48 * 1024 && smem > attr_smem) {
      RUTV_CK(cudaFuncSetAttribute(jacobi_round_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_smem = smem;
    }
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
