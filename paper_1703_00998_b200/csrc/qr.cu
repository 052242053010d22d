// Householder QR of tall-thin panels (§2.4, used at P:949
// for QR(Y) and P:957 for the column panel), producing the compact-WY factor
// in-kernel (the T factor of Joffrain et al. 2006, cited at PAPER.md:351).
//
// Blocked right-looking scheme over leaves of W columns:
//   leaf:   one thread-block CLUSTER (<= 16 CTAs on one GPC) holds the m x W
//           leaf in registers (each thread owns up to RPT rows), and computes
//           the W reflectors one column at a time.  Per column a single
//           reduction  d_k = sum_{r>j} x_r a_{r,k}  (k = 0..W-1) gives at once
//           ||x||^2 (k = j), the update coefficients (k > j) and the T-factor
//           inner products V(:,k)^T v_j (k < j); CTAs exchange their partial
//           vectors through distributed shared memory with one cluster barrier
//           per column (double-buffered slots).
//   update: the rest of the panel and the off-diagonal T blocks are DMMA
//           GEMMs over the whole GPU (gemm.cu):
//             S = V_l^T V[j0:, 0:b]                   (one GEMM, two uses)
//             V[j0:, rest] -= V_l (T_l^T S_rest)
//             Tw[0:j0, l]   = -Tw[0:j0,0:j0] S_prev^T T_l
// Reflector convention: LAPACK dlarfg (R3):
//   beta = -copysign(sqrt(alpha^2 + ||x||^2), alpha), tau = (beta - alpha)/beta,
//   v = [1; x / (alpha - beta)], tau = 0 when ||x|| = 0.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace cg = cooperative_groups;

namespace rutv {

namespace {
constexpr int QR_NT = 256;
constexpr int QR_WARPS = QR_NT / 32;
constexpr int QR_MAX_CLUSTER = 16;

// In-warp transpose-reduction of W values: afterwards lane L holds the warp
// total of value (L & (W-1)) in v[0].
template <int W>
__device__ __forceinline__ double warp_transpose_reduce(double (&v)[W], int lane) {
#pragma unroll
  for (int o = W / 2; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      double send = upper ? v[i] : v[i + o];
      double keep = upper ? v[i + o] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double r = v[0];
#pragma unroll
  for (int o = W; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

struct LeafSmem {
  // W <= 32
  double red[QR_WARPS][32];
  double part[2][QR_MAX_CLUSTER][32];  // partial d_k pushed by every CTA (double-buffered by column parity)
  double rowv[2][32];   // the diagonal row's values (pushed by its owner CTA)
  double rowl[32];      // owner's local copy before the push
  double tot[32];
  double rowj[32];
  double wk[32];
  double tl[32][33];    // leaf T factor
  double scal, beta, tau;
};

template <int W, int RPT>
__global__ void __launch_bounds__(QR_NT, 1)
leaf_qr_kernel(int64_t m, int64_t j0, int wj, double* __restrict__ V, int64_t ldv, double* __restrict__ R,
               int64_t ldr, double* __restrict__ tau, double* __restrict__ Tw, int64_t ldt) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ LeafSmem sm;
  const int C = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rows = m - j0;                // active rows (relative row r <-> global j0 + r)
  const int64_t rpc = (rows + C - 1) / C;      // rows per CTA
  const int64_t rbeg = int64_t(crank) * rpc;
  const int64_t rend = min(rows, rbeg + rpc);

  // rows above the leaf's diagonal block are finished R entries of these columns
  if (crank == 0) {
    for (int64_t idx = tid; idx < j0 * wj; idx += QR_NT) {
      int64_t r = idx % j0, k = idx / j0;
      double* vp = V + r + (j0 + k) * ldv;
      R[r + (j0 + k) * ldr] = *vp;
      *vp = 0.0;
    }
  }

  double a[RPT][W];
  int64_t rr[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    rr[i] = rbeg + tid + int64_t(i) * QR_NT;
    const bool ok = rr[i] < rend;
#pragma unroll
    for (int k = 0; k < W; ++k) a[i][k] = (ok && k < wj) ? V[(j0 + rr[i]) + (j0 + k) * ldv] : 0.0;
    if (!ok) rr[i] = -1;
  }
  if (tid < 32)
    for (int k = 0; k < 33; ++k) sm.tl[tid][k] = 0.0;

  // The column loop is NOT unrolled (an unrolled W-column body thrashed the
  // instruction cache: ncu r01 showed 'no_instructions' as the top stall).
  // Register arrays are indexed only by compile-time k; the runtime column j
  // enters through selects.
#pragma unroll 1
  for (int j = 0; j < wj; ++j) {
    const int buf = j & 1;
    // ---- phase A: partial inner products over own rows strictly below row j
    double x[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      double xi = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k) xi = (k == j) ? a[i][k] : xi;
      x[i] = (rr[i] > j) ? xi : 0.0;
    }
    double d[W];
#pragma unroll
    for (int k = 0; k < W; ++k) d[k] = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int k = 0; k < W; ++k) d[k] = fma(x[i], a[i][k], d[k]);
    double wsum = warp_transpose_reduce<W>(d, lane);
    if (lane < W) sm.red[warp][lane] = wsum;
    // the owner of relative row j stages that row locally
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (rr[i] == j) {
#pragma unroll
        for (int k = 0; k < W; ++k) sm.rowl[k] = a[i][k];
      }
    __syncthreads();
    // push this CTA's partial (and, from the owner, row j) into every CTA's
    // slots: remote stores are fire-and-forget, the reads below are local
    const int owner = (int)(int64_t(j) / rpc);
    if (tid < W) {
      double s = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < QR_WARPS; ++w2) s += sm.red[w2][tid];
      const double rv = sm.rowl[tid];
      for (int c = 0; c < C; ++c) {
        *cluster.map_shared_rank(&sm.part[buf][crank][tid], c) = s;
        if (crank == owner) *cluster.map_shared_rank(&sm.rowv[buf][tid], c) = rv;
      }
    }
    cluster.sync();
    // ---- phase B: cluster-wide totals (fixed rank order -> identical on all CTAs)
    if (warp == 0) {
      double tot = 0.0, rowj = 0.0;
      if (lane < W) {
        for (int c = 0; c < C; ++c) tot += sm.part[buf][c][lane];
        rowj = sm.rowv[buf][lane];
      }
      const double alpha = __shfl_sync(0xffffffffu, rowj, j);
      const double xnorm2 = __shfl_sync(0xffffffffu, tot, j);
      double tau_j = 0.0, beta = alpha, scal = 0.0;
      if (xnorm2 > 0.0) {
        double nrm = sqrt(fma(alpha, alpha, xnorm2));
        beta = -copysign(nrm, alpha);
        tau_j = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      // lane k: t_k = V(:,k)^T v_j (k < j) or the update coefficient (k > j)
      const double tk = fma(scal, tot, rowj);
      if (lane < W) sm.wk[lane] = (lane > j && lane < wj) ? tau_j * tk : 0.0;
      // T(0:j, j) = -tau_j T(0:j, 0:j) t
      double tsum = 0.0;
      for (int c = 0; c < j; ++c) {
        double tc = __shfl_sync(0xffffffffu, tk, c);
        if (lane <= c) tsum = fma(sm.tl[lane][c], tc, tsum);
      }
      if (lane < j) sm.tl[lane][j] = -tau_j * tsum;
      if (lane == 0) {
        sm.tl[j][j] = tau_j;
        sm.scal = scal;
        sm.beta = beta;
        sm.tau = tau_j;
      }
    }
    __syncthreads();
    // ---- phase C: apply H_j to own rows (coef = v_r below row j, 1 on row j), store v_j
    const double scal = sm.scal, beta = sm.beta;
    double wk[W];
#pragma unroll
    for (int k = 0; k < W; ++k) wk[k] = sm.wk[k];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const double v = scal * x[i];
      const double coef = (rr[i] > j) ? v : ((rr[i] == j) ? 1.0 : 0.0);
      const double newj = (rr[i] > j) ? v : beta;
      const bool setj = rr[i] >= j;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        double t = fma(-coef, wk[k], a[i][k]);
        a[i][k] = (k == j) ? (setj ? newj : a[i][k]) : t;
      }
    }
    if (crank == 0 && tid == 0) tau[j0 + j] = sm.tau;
  }
  // ---- write back: V explicit (unit lower trapezoidal), R upper
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    if (rr[i] < 0) continue;
    const int64_t r = rr[i], gr = j0 + r;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      if (k >= wj) break;
      double* vp = V + gr + (j0 + k) * ldv;
      if (r < k) {
        R[gr + (j0 + k) * ldr] = a[i][k];
        *vp = 0.0;
      } else if (r == k) {
        R[gr + (j0 + k) * ldr] = a[i][k];
        *vp = 1.0;
      } else {
        *vp = a[i][k];
      }
    }
  }
  if (crank == 0) {
    for (int idx = tid; idx < wj * wj; idx += QR_NT) {
      int r = idx % wj, k = idx / wj;
      Tw[(j0 + r) + (j0 + k) * ldt] = (r <= k) ? sm.tl[r][k] : 0.0;
    }
  }
  cluster.sync();  // keep DSMEM alive until every CTA is done reading
}

template <int W, int RPT>
void launch_leaf(cudaStream_t st, int C, int64_t m, int64_t j0, int wj, double* V, int64_t ldv, double* R,
                 int64_t ldr, double* tau, double* Tw, int64_t ldt) {
  static bool attr = false;
  auto kern = leaf_qr_kernel<W, RPT>;
  if (!attr) {
    RUTV_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(QR_NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ProfScope _p(st, K_QR, 0.0);
  count_launch(K_QR);
  RUTV_CK(cudaLaunchKernelEx(&cfg, kern, m, j0, wj, V, ldv, R, ldr, tau, Tw, ldt));
}

// O = T_l^T (sum_z part_z),  part_z = wj x b split-K partials of V_l^T V[j0:, 0:b].
// One CTA per 32 columns; the split sum runs in fixed order (deterministic).
__global__ void __launch_bounds__(256)
qr_small_k(int wj, int64_t b, int splits, const double* __restrict__ part, const double* __restrict__ Tl,
           int64_t ldt, double* __restrict__ O) {
  __shared__ double sS[32][33];
  __shared__ double sT[32][33];
  const int tid = threadIdx.x;
  const int64_t c0 = int64_t(blockIdx.x) * 32;
  const int64_t slice = int64_t(wj) * b;
  for (int idx = tid; idx < 32 * 32; idx += 256) {
    int k = idx % 32, c = idx / 32;
    double s = 0.0;
    if (k < wj && c0 + c < b)
      for (int z = 0; z < splits; ++z) s += part[int64_t(z) * slice + k + (c0 + c) * wj];
    sS[k][c] = s;
    sT[k][c] = (k < wj && c < wj) ? Tl[k + int64_t(c) * ldt] : 0.0;
  }
  __syncthreads();
  for (int idx = tid; idx < 32 * 32; idx += 256) {
    int i = idx % 32, c = idx / 32;
    if (i >= wj || c0 + c >= b) continue;
    double s = 0.0;
    for (int k = 0; k <= i && k < wj; ++k) s = fma(sT[k][i], sS[k][c], s);  // T_l upper triangular
    O[i + (c0 + c) * wj] = s;
  }
}

// zero the strictly-lower part of the b x b R and the whole Tw before a panel
__global__ void zero_lower_k(int64_t b, double* R, int64_t ldr) {
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < b * b; idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = idx % b, c = idx / b;
    if (r > c) R[r + c * ldr] = 0.0;
  }
}
}  // namespace

int qr_max_rows() { return QR_MAX_CLUSTER * QR_NT * 16; }

size_t qr_work_elems(int64_t b) { return size_t(3) * 32 * size_t(b) + 1024; }

int panel_qr(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
             double* Tw, int64_t ldt, const QrWork& w) {
  if (b <= 0) return OK;
  if (m < b) return ERR_UNSUPPORTED;
  int W, RPT;
  const int64_t cap = int64_t(QR_MAX_CLUSTER) * QR_NT;
  if (m <= cap * 2) { W = 32; RPT = 2; }
  else if (m <= cap * 4) { W = 16; RPT = 4; }
  else if (m <= cap * 8) { W = 8; RPT = 8; }
  else if (m <= cap * 16) { W = 4; RPT = 16; }
  else return ERR_UNSUPPORTED;
  const int C = (int)std::max<int64_t>(1, std::min<int64_t>(QR_MAX_CLUSTER, cdiv(m, int64_t(QR_NT) * RPT)));
  set_zero(st, b, b, Tw, ldt);
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); }
  zero_lower_k<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(b * b, 256), 1024)), 256, 0, st>>>(b, R, ldr);
  RUTV_LAUNCH_CK();
  for (int64_t j0 = 0; j0 < b; j0 += W) {
    const int wj = (int)std::min<int64_t>(W, b - j0);
    const int64_t rows = m - j0;
    const int Cj = (int)std::max<int64_t>(1, std::min<int64_t>(C, cdiv(rows, int64_t(QR_NT) * RPT)));
    switch (W) {
      case 32: launch_leaf<32, 2>(st, Cj, m, j0, wj, V, ldv, R, ldr, tau, Tw, ldt); break;
      case 16: launch_leaf<16, 4>(st, Cj, m, j0, wj, V, ldv, R, ldr, tau, Tw, ldt); break;
      case 8: launch_leaf<8, 8>(st, Cj, m, j0, wj, V, ldv, R, ldr, tau, Tw, ldt); break;
      default: launch_leaf<4, 16>(st, Cj, m, j0, wj, V, ldv, R, ldr, tau, Tw, ldt); break;
    }
    const int64_t rest = b - j0 - wj;
    if (rest == 0 && j0 == 0) continue;
    const double* Vl = V + j0 + j0 * ldv;
    const double* Tl = Tw + j0 + j0 * ldt;
    // S = V_l^T V[j0:, 0:b] as split-K partials; O = T_l^T S  (wj x b)
    const int splits = dgemm_partials(st, true, false, wj, b, rows, Vl, ldv, V + j0, ldv, w.part, w.part_elems);
    {
      ProfScope _p(st, K_QR, 0.0);
      count_launch(K_QR);
      qr_small_k<<<(unsigned)cdiv(b, 32), 256, 0, st>>>(wj, b, splits, w.part, Tl, ldt, w.sfull);
      RUTV_LAUNCH_CK();
    }
    if (rest > 0)  // V[j0:, j0+wj:b] -= V_l O(:, j0+wj:b)
      dgemm(st, false, false, rows, rest, wj, -1.0, Vl, ldv, w.sfull + (j0 + wj) * wj, wj, 1.0,
            V + j0 + (j0 + wj) * ldv, ldv, w.part, w.part_elems);
    if (j0 > 0)    // Tw[0:j0, j0:j0+wj] = -Tw[0:j0, 0:j0] O(:, 0:j0)^T
      dgemm(st, false, true, j0, wj, j0, -1.0, Tw, ldt, w.sfull, wj, 0.0, Tw + j0 * ldt, ldt, w.part, w.part_elems);
  }
  return OK;
}

void thin_q(cudaStream_t st, int64_t m, int64_t b, const double* V, int64_t ldv, const double* Tw, int64_t ldt,
            double* Q, int64_t ldq, double* tmp_bb, double* part, size_t part_elems) {
  // tmp = Tw V1^T (V1 = V[0:b, 0:b]);  Q = E - V tmp
  dgemm(st, false, true, b, b, b, 1.0, Tw, ldt, V, ldv, 0.0, tmp_bb, b, part, part_elems);
  set_identity(st, m, b, Q, ldq);
  dgemm(st, false, false, m, b, b, -1.0, V, ldv, tmp_bb, b, 1.0, Q, ldq, part, part_elems);
}

}  // namespace rutv
