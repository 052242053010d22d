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

// Workspace layout: one slot per matrix, [B (k^2) | W (k^2) | rotation counts
// per sweep (MAX_SWEEPS + 1 ints), next-sweep index (1 int)] padded to
// jslot(k) = jacobi_work_elems(1, k) doubles; matrix mat of a launch whose
// work pointer is ``work`` sits at work + mat jslot(k).  A range of matrices
// [s0, s1) of a larger workspace is therefore itself a valid batch at
// work + s0 jslot(k), whatever batch sizes began / advanced / finish it (the
// incremental SVDs of the driver begin one matrix per step and sweep ranges).
__host__ __device__ __forceinline__ int64_t jslot(int k) { return 2 * int64_t(k) * k + (MAX_SWEEPS + 2); }
struct JSlot {
  double* B;
  double* W;
  int* cnt;   // cnt[s]: rotations in sweep s - 1 (cnt[0] = 1)
  int* next;  // next sweep to run, -1 once converged
};
__device__ __forceinline__ JSlot jslot_of(double* work, int k, int mat) {
  double* B = work + int64_t(mat) * jslot(k);
  int* cnt = reinterpret_cast<int*>(B + 2 * int64_t(k) * k);
  return {B, B + int64_t(k) * k, cnt, cnt + MAX_SWEEPS + 1};
}

__global__ void jacobi_init_k(int k, const double* __restrict__ R, int64_t ldr, int64_t strideR,
                              double* __restrict__ work) {
  pdl_begin();
  const int mat = blockIdx.y;
  const double* Ri = R + int64_t(mat) * strideR;
  const JSlot js = jslot_of(work, k, mat);
  double* B = js.B;
  double* W = js.W;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < int64_t(k) * k;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int r = int(idx % k), c = int(idx / k);
    B[idx] = Ri[c + int64_t(r) * ldr];  // B = R^T
    W[idx] = (r == c) ? 1.0 : 0.0;
  }
  if (blockIdx.x == 0) {
    for (int s = threadIdx.x; s <= MAX_SWEEPS; s += blockDim.x) js.cnt[s] = (s == 0);
    if (threadIdx.x == 0) *js.next = 0;  // next sweep (-1: converged)
  }
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
jacobi_round_k(JacobiDesc d, int sweep, int round, double* __restrict__ work, double tol) {
  pdl_begin();
  extern __shared__ __align__(16) double js[];
  __shared__ double nrm[64];
  const int mat = blockIdx.y;
  const JSlot slot = jslot_of(work, d.k, mat);
  int* cnt = slot.cnt;
  if (cnt[sweep] == 0) return;  // previous sweep did no rotation: converged
  const int k = d.k, kb = d.kb;
  int bp, bq;
  rr_pair(d.nb, round, blockIdx.x, bp, bq);
  double* B = slot.B;
  double* W = slot.W;
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
jacobi_cluster_k(JacobiDesc d, double* __restrict__ work, double tol) {
  pdl_begin();
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double js[];
  __shared__ double nrm[64];
  __shared__ int rot_sm;
  const int mat = blockIdx.y;
  const int cta = (int)cluster.block_rank();
  const JSlot slot = jslot_of(work, d.k, mat);
  int* cnt = slot.cnt;
  const int k = d.k, kb = d.kb;
  double* B = slot.B;
  double* W = slot.W;
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

// ---- k <= 256: cross-pair block ordering, one register-resident column per warp
//
// Same tournament over blocks of 16 columns as jacobi_cluster_k, but a round
// visits only the 256 CROSS pairs of its block pair (16 sub-rounds, pair
// (w, (w + sh) mod 16)), and the within-block pairs are visited once per sweep
// (round 0, all blocks at once): every column pair exactly once per sweep, as
// in a cyclic sweep, instead of the within-block pairs once per round (1.8x
// the pair visits; simulated on the c3 R11 blocks: same sweep count).  Warp w
// keeps column w of the first block (B and W) in registers for the whole
// round; the second block lives in shared memory and each of its columns is
// read, rotated and written back by one warp per sub-round.  Column norms are
// recomputed for every pair (alpha, beta, gamma in one fused warp reduction):
// on the c3 blocks (150 singular values within 1e-10 of each other) the
// tracked norms of Rutishauser's update cost extra sweeps.
// Lane l holds rows 64e + 2l + {0, 1} (e < EPL/2): 16-byte shared accesses.
template <int EPL>
struct JacCol {
  double v[EPL];
};

template <int EPL>
__device__ __forceinline__ void jc_lds(JacCol<EPL>& c, const double* col, int lane) {
#pragma unroll
  for (int e = 0; e < EPL / 2; ++e) {
    const double2 t = *reinterpret_cast<const double2*>(col + 64 * e + 2 * lane);
    c.v[2 * e] = t.x;
    c.v[2 * e + 1] = t.y;
  }
}
template <int EPL>
__device__ __forceinline__ void jc_sts(double* col, const JacCol<EPL>& c, int lane) {
#pragma unroll
  for (int e = 0; e < EPL / 2; ++e)
    *reinterpret_cast<double2*>(col + 64 * e + 2 * lane) = make_double2(c.v[2 * e], c.v[2 * e + 1]);
}

// 1/x for x > 0 normal: MUFU seed + two Newton steps (relative error ~1e-16;
// the rotation stays orthogonal to rounding whatever the accuracy of t, since
// c = (1 + t^2)^-1/2 and s = c t)
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// rotate (x, y) so that x^T y = 0; returns 1 if a rotation was applied.
// alpha, beta, gamma by one transposed warp reduction (lane L ends with the
// total of value L & 3); t = 2 gamma sgn(d) / (|d| + sqrt(d^2 + 4 gamma^2)),
// d = beta - alpha -- the classical t = sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)),
// zeta = d / (2 gamma), with one reciprocal and no overflow for small gamma.
template <int EPL, bool FAST>
__device__ __forceinline__ int jc_rotate(JacCol<EPL>& xb, JacCol<EPL>& yb, JacCol<EPL>& xw, JacCol<EPL>& yw,
                                         double tol) {
  const int lane = threadIdx.x & 31;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    v[0] = fma(xb.v[e], xb.v[e], v[0]);
    v[1] = fma(yb.v[e], yb.v[e], v[1]);
    v[2] = fma(xb.v[e], yb.v[e], v[2]);
  }
  {  // 4 values x 32 lanes: 2 transposed levels, then 3 plain levels
    const bool u2 = (lane & 2) != 0;
    double s0 = u2 ? v[0] : v[2], s1 = u2 ? v[1] : v[3];
    double k0 = u2 ? v[2] : v[0], k1 = u2 ? v[3] : v[1];
    k0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    k1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    const bool u1 = (lane & 1) != 0;
    double s = u1 ? k0 : k1, k = u1 ? k1 : k0;
    k += __shfl_xor_sync(0xffffffffu, s, 1);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    v[0] = k;
  }
  const double al = __shfl_sync(0xffffffffu, v[0], 0);
  const double be = __shfl_sync(0xffffffffu, v[0], 1);
  const double ga = __shfl_sync(0xffffffffu, v[0], 2);
  // FAST: the threshold test squared (no IEEE sqrt on the dependent chain)
  if constexpr (FAST) {
    if (!(ga != 0.0 && ga * ga > (tol * tol) * (al * be))) return 0;
  } else {
    if (!(ga != 0.0 && fabs(ga) > tol * sqrt(al * be))) return 0;
  }
  const double d = be - al, g2 = 2.0 * ga;
  const double h = fma(d, d, g2 * g2);
  const double root = h * rsqrt(h);
  const double t = (d >= 0.0 ? g2 : -g2) * rcp_fast(fabs(d) + root);
  const double c = rsqrt(fma(t, t, 1.0));
  const double s = c * t;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const double x = xb.v[e], y = yb.v[e];
    xb.v[e] = c * x - s * y;
    yb.v[e] = s * x + c * y;
    const double u = xw.v[e], w = yw.v[e];
    xw.v[e] = c * u - s * w;
    yw.v[e] = s * u + c * w;
  }
  return 1;
}

template <int EPL, bool FAST>
__global__ void __launch_bounds__(JNT)
jacobi_cluster2_k(JacobiDesc d, double* __restrict__ work, double tol, int max_sweeps, int pair_load) {
  pdl_begin();
  constexpr int KB = 16, KP = 32 * EPL;  // block width, padded column length
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double js[];
  double* sB = js;  // [2 KB][KP]: block p (cols 0..15), block q (16..31)
  double* sW = js + 2 * KB * KP;
  __shared__ int rot_sm;
  const int mat = blockIdx.y;
  const int cta = (int)cluster.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const JSlot slot = jslot_of(work, d.k, mat);
  int* cnt = slot.cnt;
  const int k = d.k;
  double* B = slot.B;
  double* W = slot.W;
  // global <-> shared for one block (16 columns, zero padding beyond k)
  // (16-byte accesses when k is even: a column pair of rows r, r+1 is aligned)
  const bool vec = (k & 1) == 0;
  auto load_block = [&](int blk, int slot) {
    if (vec) {
      for (int idx = threadIdx.x; idx < KB * KP / 2; idx += JNT) {
        const int c = idx / (KP / 2), r = 2 * (idx % (KP / 2)), g = blk * KB + c;
        const bool ok = g < k && r < k;  // k even: r < k implies r + 1 < k
        double2 vb = make_double2(0.0, 0.0), vw = vb;
        if (ok) {
          vb = __ldcg(reinterpret_cast<const double2*>(B + r + int64_t(g) * k));
          vw = __ldcg(reinterpret_cast<const double2*>(W + r + int64_t(g) * k));
        }
        *reinterpret_cast<double2*>(sB + (slot * KB + c) * KP + r) = vb;
        *reinterpret_cast<double2*>(sW + (slot * KB + c) * KP + r) = vw;
      }
      return;
    }
    for (int idx = threadIdx.x; idx < KB * KP; idx += JNT) {
      const int c = idx / KP, r = idx % KP, g = blk * KB + c;
      const bool ok = g < k && r < k;
      sB[(slot * KB + c) * KP + r] = ok ? __ldcg(B + r + int64_t(g) * k) : 0.0;
      sW[(slot * KB + c) * KP + r] = ok ? __ldcg(W + r + int64_t(g) * k) : 0.0;
    }
  };
  // both blocks of a round at once, every load issued before the first shared
  // store (one L2 round trip instead of one per loop iteration: ncu showed
  // long-scoreboard stalls at ~12 % of the issue cycles)
  auto load_pair = [&](int bp, int bq) {
    if (!vec) {
      load_block(bp, 0);
      load_block(bq, 1);
      return;
    }
    constexpr int IT = (KB * KP / 2 + JNT - 1) / JNT;  // double2 per thread per block
    double2 vb[2][IT], vw[2][IT];
#pragma unroll
    for (int sl = 0; sl < 2; ++sl)
#pragma unroll
      for (int u = 0; u < IT; ++u) {
        const int idx = threadIdx.x + u * JNT;
        const int c = idx / (KP / 2), r = 2 * (idx % (KP / 2)), g = (sl ? bq : bp) * KB + c;
        const bool ok = idx < KB * KP / 2 && g < k && r < k;
        vb[sl][u] = vw[sl][u] = make_double2(0.0, 0.0);
        if (ok) {
          vb[sl][u] = __ldcg(reinterpret_cast<const double2*>(B + r + int64_t(g) * k));
          vw[sl][u] = __ldcg(reinterpret_cast<const double2*>(W + r + int64_t(g) * k));
        }
      }
#pragma unroll
    for (int sl = 0; sl < 2; ++sl)
#pragma unroll
      for (int u = 0; u < IT; ++u) {
        const int idx = threadIdx.x + u * JNT;
        if (idx < KB * KP / 2) {
          const int c = idx / (KP / 2), r = 2 * (idx % (KP / 2));
          *reinterpret_cast<double2*>(sB + (sl * KB + c) * KP + r) = vb[sl][u];
          *reinterpret_cast<double2*>(sW + (sl * KB + c) * KP + r) = vw[sl][u];
        }
      }
  };
  auto store_block = [&](int blk, int slot) {
    if (vec) {
      for (int idx = threadIdx.x; idx < KB * KP / 2; idx += JNT) {
        const int c = idx / (KP / 2), r = 2 * (idx % (KP / 2)), g = blk * KB + c;
        if (g < k && r < k) {
          __stcg(reinterpret_cast<double2*>(B + r + int64_t(g) * k),
                 *reinterpret_cast<const double2*>(sB + (slot * KB + c) * KP + r));
          __stcg(reinterpret_cast<double2*>(W + r + int64_t(g) * k),
                 *reinterpret_cast<const double2*>(sW + (slot * KB + c) * KP + r));
        }
      }
      return;
    }
    for (int idx = threadIdx.x; idx < KB * KP; idx += JNT) {
      const int c = idx / KP, r = idx % KP, g = blk * KB + c;
      if (g < k && r < k) {
        __stcg(B + r + int64_t(g) * k, sB[(slot * KB + c) * KP + r]);
        __stcg(W + r + int64_t(g) * k, sW[(slot * KB + c) * KP + r]);
      }
    }
  };
  // resumable: up to max_sweeps sweeps from the stored next-sweep index
  // (-1 once a sweep made no rotation)
  int* next = slot.next;
  const int s0 = __ldcg(next);
  if (s0 < 0) return;
  const int s1 = min(MAX_SWEEPS, s0 + max_sweeps);
  int sweep = s0;
  bool converged = false;
  for (; sweep < s1; ++sweep) {
    if (threadIdx.x == 0) rot_sm = 0;
    int rot = 0;
    for (int round = 0; round < d.nb - 1; ++round) {
      int bp, bq;
      rr_pair(d.nb, round, cta, bp, bq);
      if (pair_load & 1) {
        load_pair(bp, bq);
      } else {
        load_block(bp, 0);
        load_block(bq, 1);
      }
      __syncthreads();
      if (round == 0) {
        // within-block pairs of both blocks: warp w -> block w / 8, pair w % 8
        const int slot = warp >> 3, pi = warp & 7;
        for (int sr = 0; sr < KB - 1; ++sr) {
          int p, q;
          rr_pair(KB, sr, pi, p, q);
          double* cbp = sB + (slot * KB + p) * KP;
          double* cbq = sB + (slot * KB + q) * KP;
          double* cwp = sW + (slot * KB + p) * KP;
          double* cwq = sW + (slot * KB + q) * KP;
          JacCol<EPL> xb, yb, xw, yw;
          jc_lds(xb, cbp, lane);
          jc_lds(yb, cbq, lane);
          jc_lds(xw, cwp, lane);
          jc_lds(yw, cwq, lane);
          if (jc_rotate<EPL, FAST>(xb, yb, xw, yw, tol)) {
            jc_sts(cbp, xb, lane);
            jc_sts(cbq, yb, lane);
            jc_sts(cwp, xw, lane);
            jc_sts(cwq, yw, lane);
            ++rot;
          }
          __syncthreads();
        }
      }
      // cross pairs: warp w holds column w of block p and meets column
      // (w + sh) mod 16 of block q in sub-round sh.  (A per-column flag
      // handoff between neighbouring warps instead of the barrier was
      // measured: no faster.)
      JacCol<EPL> xb, xw;
      jc_lds(xb, sB + warp * KP, lane);
      jc_lds(xw, sW + warp * KP, lane);
      for (int sh = 0; sh < KB; ++sh) {
        const int q = KB + ((warp + sh) & (KB - 1));
        double* cbq = sB + q * KP;
        double* cwq = sW + q * KP;
        JacCol<EPL> yb, yw;
        jc_lds(yb, cbq, lane);
        jc_lds(yw, cwq, lane);
        if (jc_rotate<EPL, FAST>(xb, yb, xw, yw, tol)) {
          jc_sts(cbq, yb, lane);
          jc_sts(cwq, yw, lane);
          ++rot;
        }
        __syncthreads();
      }
      jc_sts(sB + warp * KP, xb, lane);
      jc_sts(sW + warp * KP, xw, lane);
      __syncthreads();
      store_block(bp, 0);
      store_block(bq, 1);
      // the cluster barrier is a release / acquire at cluster scope: it orders
      // these global stores before the other CTAs' loads of the next round
      // (the extra GPU-scope fence cost ~5 % of the issue stalls, ncu)
      if (!(pair_load & 2)) __threadfence();
      cluster.sync();
    }
    if (lane == 0 && rot) atomicAdd(&rot_sm, rot);
    __syncthreads();
    if (threadIdx.x == 0 && rot_sm) atomicAdd(&cnt[sweep + 1], rot_sm);
    __threadfence();
    cluster.sync();
    const int total = atomicAdd(&cnt[sweep + 1], 0);
    if (total == 0) {
      converged = true;
      break;
    }
  }
  cluster.sync();  // every CTA has read the next-sweep index
  if (cta == 0 && threadIdx.x == 0) *next = (converged || sweep >= MAX_SWEEPS) ? -1 : sweep;
}

// sigma_j = ||B(:,j)||, sort descending, Us = W(:,perm), Vs = B(:,perm) / sigma.
__global__ void __launch_bounds__(JNT)
jacobi_finalize_k(int k, double* __restrict__ work, double* __restrict__ D, double* __restrict__ Us,
                  double* __restrict__ Vs, int* __restrict__ sweeps_out) {
  pdl_begin();
  extern __shared__ __align__(16) double fs[];
  double* sig = fs;                           // k
  int* rank = reinterpret_cast<int*>(fs + k);  // k
  const int mat = blockIdx.x;
  const JSlot slot = jslot_of(work, k, mat);
  const double* B = slot.B;
  const double* W = slot.W;
  const int* cnt = slot.cnt;
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
      while (s < MAX_SWEEPS && cnt[s + 1] > 0) ++s;
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
    while (s < MAX_SWEEPS && cnt[s + 1] > 0) ++s;
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

// per matrix: B and W (k x k each) and MAX_SWEEPS + 2 int slots (sweep counts,
// next-sweep index) padded to MAX_SWEEPS + 2 doubles -- an even count, so that
// jacobi_work_elems(j0, k) = j0 jslot(k) is a 16-byte aligned offset for any j0
// (callers carve sub-batches starting at matrix j0; the k-even block I/O is 16-byte)
static_assert((MAX_SWEEPS + 2) % 2 == 0, "16-byte aligned sub-batch offsets");
size_t jacobi_work_elems(int batch, int k) { return size_t(batch) * size_t(jslot(k)); }

namespace {
// up to max_sweeps sweeps of jacobi_cluster2_k on every matrix of the batch
void launch_c2(cudaStream_t st, int batch, int k, double* work, int max_sweeps) {
  // RANDUTV_EXP_NO_SWEEPS=1: timing experiment only (skips the sweeps: wrong results)
  static const bool exp_skip = getenv("RANDUTV_EXP_NO_SWEEPS") && atoi(getenv("RANDUTV_EXP_NO_SWEEPS"));
  if (exp_skip) return;
  JacobiDesc d = make_desc(k);
  const int csize = d.nb / 2;
  const double tol = double(k) * DBL_EPSILON;
  const int epl = k <= 64 ? 2 : (k <= 128 ? 4 : 8);
  const size_t smem2 = size_t(2) * 2 * 16 * 32 * epl * sizeof(double);
  // the squared threshold test (bitwise the same rotations, no IEEE sqrt on the
  // sub-round's dependent chain): k = 256 single matrix 5.85 -> 5.41 ms, c3
  // 250.4 -> 249.1 ms; for k <= 128 (c2) it measured 0.45 ms slower in the
  // factorization (ptxas spills the EPL = 4 variant), so k > 128 only.
  // RANDUTV_JACOBI_FASTROT=0 / 1: A/B switch
  static const int fast_env = [] {
    const char* e = getenv("RANDUTV_JACOBI_FASTROT");
    return e ? atoi(e) : -1;
  }();
  const bool fast = fast_env < 0 ? epl == 8 : fast_env != 0;
  using KernT = void (*)(JacobiDesc, double*, double, int, int);
  // bit 0: load_pair, bit 1: no per-round GPU-scope fence (RANDUTV_JACOBI_PAIRLOAD: A/B switch)
  static const int pair_load = [] {
    const char* e = getenv("RANDUTV_JACOBI_PAIRLOAD");
    return e ? atoi(e) : 3;
  }();
  KernT kern = fast ? (epl == 2 ? jacobi_cluster2_k<2, true> : (epl == 4 ? jacobi_cluster2_k<4, true> : jacobi_cluster2_k<8, true>))
                    : (epl == 2 ? jacobi_cluster2_k<2, false> : (epl == 4 ? jacobi_cluster2_k<4, false> : jacobi_cluster2_k<8, false>));
  static OncePerDevice attr2[6];
  const int ai = (epl == 2 ? 0 : (epl == 4 ? 1 : 2)) + (fast ? 3 : 0);
  attr2[ai]([&] { RUTV_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2)); });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize, batch, 1);
  cfg.blockDim = dim3(JNT, 1, 1);
  cfg.dynamicSmemBytes = smem2;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  ProfScope _p(st, K_SVD, 0.0);
  count_launch(K_SVD);
  RUTV_CK(cudaLaunchKernelEx(&cfg, kern, d, work, tol, max_sweeps, pair_load));
}

void launch_init(cudaStream_t st, int batch, int k, const double* R, int64_t ldr, int64_t strideR, double* work) {
  dim3 g((unsigned)std::min<int64_t>(cdiv(int64_t(k) * k, 256), 64), batch);
  ProfScope _p(st, K_SVD, 0.0);
  count_launch(K_SVD);
  launch_k(jacobi_init_k, dim3(g), dim3(256), 0, st, k, R, ldr, strideR, work);
  RUTV_LAUNCH_CK();
}

void launch_finalize(cudaStream_t st, int batch, int k, double* work, double* D, double* Us, double* Vs,
                     int* sweeps_out) {
  const size_t fsmem = size_t(k) * (sizeof(double) + sizeof(int)) + 16;
  static SmemAttrPerDevice attr_f;
  if (fsmem > 48 * 1024) attr_f.ensure(jacobi_finalize_k, fsmem);
  { ProfScope _p(st, K_SVD, 0.0); count_launch(K_SVD); launch_k(jacobi_finalize_k, dim3(batch), dim3(JNT), fsmem, st, k, work, D, Us, Vs, sweeps_out); }
  RUTV_LAUNCH_CK();
}
}  // namespace

bool jacobi_incremental(int k) { return k > 1 && k <= 256 && make_desc(k).kb == 16; }

void jacobi_begin(cudaStream_t st, int batch, int k, const double* R, int64_t ldr, int64_t strideR, double* work) {
  if (batch <= 0) return;
  launch_init(st, batch, k, R, ldr, strideR, work);
}
void jacobi_sweeps(cudaStream_t st, int batch, int k, double* work, int nsweeps) {
  if (batch <= 0) return;
  launch_c2(st, batch, k, work, nsweeps);
}
void jacobi_end(cudaStream_t st, int batch, int k, double* work, double* D, double* Us, double* Vs,
                int* sweeps_out) {
  if (batch <= 0) return;
  launch_c2(st, batch, k, work, MAX_SWEEPS);  // the remaining sweeps, if any
  launch_finalize(st, batch, k, work, D, Us, Vs, sweeps_out);
}

void jacobi_svd_batched(cudaStream_t st, int batch, int k, const double* R, int64_t ldr, int64_t strideR,
                        double* D, double* Us, double* Vs, double* work, int* sweeps_out) {
  if (batch <= 0 || k <= 0) return;
  JacobiDesc d = make_desc(k);
  launch_init(st, batch, k, R, ldr, strideR, work);
  const size_t smem = size_t(2) * 2 * d.kb * k * sizeof(double);
  const double tol = double(k) * DBL_EPSILON;
  const int csize = d.nb / 2;
  if (jacobi_incremental(k)) {
    launch_c2(st, batch, k, work, MAX_SWEEPS);
  } else if (k > 1 && csize <= MAX_CLUSTER) {

    // one cluster per matrix runs every round and sweep in-kernel
    static SmemAttrPerDevice attr_c;
    attr_c.ensure(jacobi_cluster_k, smem, true);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize, batch, 1);
    cfg.blockDim = dim3(32 * d.kb, 1, 1);  // one warp per column pair of a block pair
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    ProfScope _p(st, K_SVD, 0.0);
    count_launch(K_SVD);
    RUTV_CK(cudaLaunchKernelEx(&cfg, jacobi_cluster_k, d, work, tol));
  } else if (k > 1) {
    static SmemAttrPerDevice attr_r;
    if (smem > 48 * 1024) attr_r.ensure(jacobi_round_k, smem);
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
          { ProfScope _p(st, K_SVD, 0.0); count_launch(K_SVD); launch_k(jacobi_round_k, dim3(g), dim3(JNT), smem, st, d, sweep, round, work, tol); }
          RUTV_LAUNCH_CK();
        }
      }
      // the rotation counts of every matrix: MAX_SWEEPS + 1 ints at the end of each slot
      RUTV_CK(cudaMemcpy2DAsync(h.data(), sizeof(int) * (MAX_SWEEPS + 1), work + 2 * int64_t(k) * k,
                                sizeof(double) * size_t(jslot(k)), sizeof(int) * (MAX_SWEEPS + 1), batch,
                                cudaMemcpyDeviceToHost, st));
      RUTV_CK(cudaStreamSynchronize(st));
      bool all = true;
      for (int b = 0; b < batch; ++b) all &= (h[size_t(b) * (MAX_SWEEPS + 1) + sweep] == 0);
      if (all) break;
      chunk = 2;
    }
  }
  launch_finalize(st, batch, k, work, D, Us, Vs, sweeps_out);
}

}  // namespace rutv
