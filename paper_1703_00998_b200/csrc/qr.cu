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
  double red[QR_WARPS][32];
  double part[2][QR_MAX_CLUSTER][32];  // partial d_s pushed by every CTA (double-buffered by column parity)
  double rowv[2][32];                  // the diagonal row's values (pushed by its owner CTA)
  double rowl[32];                     // owner's local copy before the push
  double w[32];                        // update coefficients of the current reflector
  double taus[32];
  double scal, beta;
};

// Stride (doubles) of the per-CTA copy of the finished reflectors in shared
// memory; == 4 (mod 16) so the DMMA fragment loads of the Gram are conflict free.
template <int W>
__host__ __device__ constexpr int vstride() { return W == 4 ? 4 : W + 4; }

template <int W, int RPT>
constexpr size_t leaf_dyn_smem() {
  return size_t(QR_NT) * RPT * vstride<W>() * sizeof(double);
}
// dynamic smem: the reflector copy, reused afterwards for the Gram reduction
// (8 warp partials + 16 cluster slots of 32x32, and the 2 x 32x33 T work area)
template <int W, int RPT>
constexpr size_t leaf_smem_bytes() {
  constexpr size_t red = sizeof(double) * (size_t(QR_WARPS) * 1024 + size_t(QR_MAX_CLUSTER) * 1024);
  return leaf_dyn_smem<W, RPT>() > red ? leaf_dyn_smem<W, RPT>() : red;
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Leaf factorization of W (<= 32) columns on a cluster of C CTAs.
//
// Register layout: thread t of CTA c owns relative rows rbeg_c + t + i*QR_NT
// (i < RPT) and keeps them in a[i][s], where slot s holds leaf column j + s at
// column step j: the reflector update writes slot s from slot s+1
// (a <- a - coef w shifted by one), so the current column is always slot 0 and
// no runtime register indexing or select chain is needed.  Each finished
// column is streamed out (V explicit, R above the diagonal) and copied to
// shared memory; the leaf T factor is formed at the end from the Gram
// V_l^T V_l (DMMA over each CTA's rows + one cluster reduction) with the dlarft
// recurrence T(0:j,j) = -tau_j T(0:j,0:j) (V^T v_j)(0:j).
template <int W, int RPT>
__global__ void __launch_bounds__(QR_NT, 1)
leaf_qr_kernel(int64_t m, int64_t j0, int wj, double* __restrict__ V, int64_t ldv, double* __restrict__ R,
               int64_t ldr, double* __restrict__ tau, double* __restrict__ Tw, int64_t ldt) {
  pdl_begin();
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ LeafSmem sm;
  extern __shared__ __align__(16) double vsm[];  // [QR_NT*RPT rows][vstride]
  constexpr int SV = vstride<W>();
  const int C = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rows = m - j0;                // active rows (relative row r <-> global j0 + r)
  const int64_t rpc = (rows + C - 1) / C;      // rows per CTA
  const int64_t rbeg = int64_t(crank) * rpc;
  const int64_t rend = min(rows, rbeg + rpc);
  const int nloc = (int)(rend > rbeg ? rend - rbeg : 0);

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
    for (int s = 0; s < W; ++s) a[i][s] = (ok && s < wj) ? V[(j0 + rr[i]) + (j0 + s) * ldv] : 0.0;
    if (!ok) rr[i] = -1;
  }

  // dots for column 0: d_s = sum_{r > 0} a_{r,0} a_{r,s}
  double d[W];
#pragma unroll
  for (int s = 0; s < W; ++s) d[s] = 0.0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const double x = (rr[i] > 0) ? a[i][0] : 0.0;
#pragma unroll
    for (int s = 0; s < W; ++s) d[s] = fma(x, a[i][s], d[s]);
  }

#pragma unroll 1
  for (int j = 0; j < wj; ++j) {
    const int buf = j & 1;
    // ---- reduce d over the CTA (warp transpose-reduce, then across warps)
    double wsum = warp_transpose_reduce<W>(d, lane);
    if (lane < W) sm.red[warp][lane] = wsum;
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (rr[i] == j) {
#pragma unroll
        for (int s = 0; s < W; ++s) sm.rowl[s] = a[i][s];
      }
    __syncthreads();
    // ---- push this CTA's partial (and, from the owner, row j) into every CTA
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
    // ---- scalars of H_j (every CTA, same fixed-order sums -> identical values)
    if (warp == 0) {
      double tot = 0.0, rowj = 0.0;
      if (lane < W) {
        double pv[QR_MAX_CLUSTER];
#pragma unroll
        for (int c = 0; c < QR_MAX_CLUSTER; ++c) pv[c] = (c < C) ? sm.part[buf][c][lane] : 0.0;
#pragma unroll
        for (int c = 0; c < QR_MAX_CLUSTER; ++c) tot += pv[c];
        rowj = sm.rowv[buf][lane];
      }
      const double alpha = __shfl_sync(0xffffffffu, rowj, 0);
      const double xnorm2 = __shfl_sync(0xffffffffu, tot, 0);
      double tau_j = 0.0, beta = alpha, scal = 0.0;
      if (xnorm2 > 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, xnorm2));
        beta = -copysign(nrm, alpha);
        tau_j = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      // slot s >= 1 (column j+s): w_s = tau_j v_j^T a_{:,j+s}
      if (lane < W) sm.w[lane] = (lane >= 1 && j + lane < wj) ? tau_j * fma(scal, tot, rowj) : 0.0;
      if (lane == 0) {
        sm.taus[j] = tau_j;
        sm.scal = scal;
        sm.beta = beta;
      }
    }
    __syncthreads();
    // ---- apply H_j to own rows (shifting slots by one), emit column j,
    //      and accumulate the dots of column j+1
    const double scal = sm.scal, beta = sm.beta;
    double coef[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      coef[i] = 0.0;
      if (rr[i] < 0) continue;
      const int64_t r = rr[i];
      const double xj = a[i][0];
      const double v = scal * xj;
      coef[i] = (r > j) ? v : ((r == j) ? 1.0 : 0.0);
      double* vp = V + (j0 + r) + (j0 + j) * ldv;
      if (r <= j) {
        R[(j0 + r) + (j0 + j) * ldr] = (r == j) ? beta : xj;
        *vp = (r == j) ? 1.0 : 0.0;
      } else {
        *vp = v;
      }
      vsm[(tid + i * QR_NT) * SV + j] = (r > j) ? v : ((r == j) ? 1.0 : 0.0);
    }
#pragma unroll
    for (int s = 0; s < W - 1; ++s) {
      const double ws = sm.w[s + 1];
#pragma unroll
      for (int i = 0; i < RPT; ++i) a[i][s] = fma(-coef[i], ws, a[i][s + 1]);
    }
#pragma unroll
    for (int s = 0; s < W; ++s) d[s] = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      a[i][W - 1] = 0.0;
      const double x = (rr[i] > j + 1) ? a[i][0] : 0.0;
#pragma unroll
      for (int s = 0; s < W - 1; ++s) d[s] = fma(x, a[i][s], d[s]);
    }
  }

  // ---- leaf T factor from the Gram G = V_l^T V_l of the stored reflectors
  // zero the unused columns of the local copy (wj < W) and rows beyond nloc
  for (int idx = tid; idx < QR_NT * RPT; idx += QR_NT) {
    for (int c = wj; c < W; ++c) vsm[idx * SV + c] = 0.0;
    if (idx >= nloc)
      for (int c = 0; c < wj; ++c) vsm[idx * SV + c] = 0.0;
  }
  __syncthreads();
  constexpr int NTL = (W + 7) / 8;  // 8x8 tiles per dimension
  double g[NTL][NTL][2];
#pragma unroll
  for (int p = 0; p < NTL; ++p)
#pragma unroll
    for (int q = 0; q < NTL; ++q) g[p][q][0] = g[p][q][1] = 0.0;
  {
    const int gq = lane >> 2, tq = lane & 3;
    const int nslot = QR_NT * RPT;            // local rows (padded with zeros)
    const int per_warp = nslot / QR_WARPS;    // multiple of 4
    for (int k0 = warp * per_warp; k0 < (warp + 1) * per_warp; k0 += 4) {
      const double* rowp = vsm + (k0 + tq) * SV;
      double af[NTL];
#pragma unroll
      for (int p = 0; p < NTL; ++p) af[p] = (p * 8 + gq < W) ? rowp[p * 8 + gq] : 0.0;
#pragma unroll
      for (int p = 0; p < NTL; ++p)
#pragma unroll
        for (int q = 0; q < NTL; ++q) dmma884(g[p][q], af[p], af[q]);
    }
  }
  __syncthreads();  // every warp is done with vsm: reuse it for the reduction
  double* gw = vsm;                                 // [QR_WARPS][32*32]
  {
    const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
    for (int p = 0; p < NTL; ++p)
#pragma unroll
      for (int q = 0; q < NTL; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = p * 8 + gq, col = q * 8 + 2 * tq + e;
          gw[warp * 1024 + row * 32 + col] = g[p][q][e];
        }
  }
  __syncthreads();
  cluster.sync();  // rank 0's reduction area (its vsm tail) is free of readers
  double* slots = vsm + QR_WARPS * 1024;           // rank 0: [C][32*32]
  for (int idx = tid; idx < W * W; idx += QR_NT) {
    const int row = idx / W, col = idx % W;
    double s = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < QR_WARPS; ++w2) s += gw[w2 * 1024 + row * 32 + col];
    *cluster.map_shared_rank(&slots[crank * 1024 + row * 32 + col], 0) = s;
  }
  cluster.sync();
  if (crank == 0) {
    double* G = gw;  // [32][33] reuse
    for (int idx = tid; idx < W * W; idx += QR_NT) {
      const int row = idx / W, col = idx % W;
      double s = 0.0;
      for (int c = 0; c < C; ++c) s += slots[c * 1024 + row * 32 + col];
      G[row * 33 + col] = s;
    }
    __syncthreads();
    // T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j); T stored over G's upper triangle
    double* Tm = gw + 32 * 33;  // [32][33]
    if (warp == 0) {
      for (int j = 0; j < wj; ++j) {
        const double tau_j = sm.taus[j];
        double s = 0.0;
        if (lane < j)
          for (int c = lane; c < j; ++c) s = fma(Tm[lane * 33 + c], G[c * 33 + j], s);
        __syncwarp();
        if (lane < 32) Tm[lane * 33 + j] = (lane < j) ? -tau_j * s : (lane == j ? tau_j : 0.0);
        __syncwarp();
      }
    }
    __syncthreads();
    for (int idx = tid; idx < wj * wj; idx += QR_NT) {
      const int r = idx % wj, k = idx / wj;
      Tw[(j0 + r) + (j0 + k) * ldt] = (r <= k) ? Tm[r * 33 + k] : 0.0;
    }
    for (int j = tid; j < wj; j += QR_NT) tau[j0 + j] = sm.taus[j];
  }
}

template <int W, int RPT>
void launch_leaf(cudaStream_t st, int C, int64_t m, int64_t j0, int wj, double* V, int64_t ldv, double* R,
                 int64_t ldr, double* tau, double* Tw, int64_t ldt) {
  static OncePerDevice attr;
  auto kern = leaf_qr_kernel<W, RPT>;
  attr([&] {
    RUTV_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RUTV_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leaf_smem_bytes<W, RPT>()));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(QR_NT, 1, 1);
  cfg.dynamicSmemBytes = leaf_smem_bytes<W, RPT>();
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
  ProfScope _p(st, K_QR, 0.0);
  count_launch(K_QR);
  RUTV_CK(cudaLaunchKernelEx(&cfg, kern, m, j0, wj, V, ldv, R, ldr, tau, Tw, ldt));
}

// O = T_l^T S, S = sum_z part_z with part_z the b x wj split-K partials of
// S^T = V[j0:, 0:b]^T V_l (ld b).  4 columns of S per CTA; the split sum is
// spread over 8 thread groups and combined in fixed order (deterministic).
__global__ void __launch_bounds__(256)
qr_small_k(int wj, int64_t b, int splits, const double* __restrict__ part, const double* __restrict__ Tl,
           int64_t ldt, double* __restrict__ O) {
  pdl_begin();
  __shared__ double sS[32][5];
  __shared__ double sT[32][33];
  __shared__ double red[8][4 * 32 + 1];
  const int tid = threadIdx.x;
  const int64_t c0 = int64_t(blockIdx.x) * 4;  // 4 columns (of S) per CTA
  const int64_t slice = int64_t(wj) * b;
  {
    // thread (g = tid / 32, e = tid % 32): element (c = e % 4 + ..) -- lanes map
    // to (column c0 + e/8 .. ) pairs so that loads of one split are contiguous
    const int g = tid >> 5, e = tid & 31;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (e < wj) {
      for (int z = g; z < splits; z += 8) {
        const double* pz = part + int64_t(z) * slice + int64_t(e) * b + c0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c0 + c < b) acc[c] += pz[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) red[g][c * 32 + e] = acc[c];
  }
  for (int idx = tid; idx < 32 * 32; idx += 256) {
    int k = idx % 32, c = idx / 32;
    sT[k][c] = (k < wj && c < wj) ? Tl[k + int64_t(c) * ldt] : 0.0;
  }
  __syncthreads();
  if (tid < 128) {
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) s += red[g][tid];
    sS[tid % 32][tid / 32] = s;
  }
  __syncthreads();
  if (tid < 128) {
    int i = tid % 32, c = tid / 32;
    if (i < wj && c0 + c < b) {
      double s = 0.0;
      for (int k = 0; k <= i; ++k) s = fma(sT[k][i], sS[k][c], s);  // T_l upper triangular
      O[i + (c0 + c) * wj] = s;
    }
  }
}

// zero the strictly-lower part of the b x b R and the whole Tw before a panel
__global__ void zero_lower_k(int64_t b, double* R, int64_t ldr) {
  pdl_begin();
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < b * b; idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = idx % b, c = idx / b;
    if (r > c) R[r + c * ldr] = 0.0;
  }
}
}  // namespace

namespace {
__global__ void reortho_flag_k(const double* stats, double kappa_max, int* flag) {
  pdl_begin();
  if (threadIdx.x == 0) *flag = !(stats[0] == 0.0 && stats[2] <= kappa_max * stats[1]);
}
}  // namespace

void reortho_flag(cudaStream_t st, const double* stats, double kappa_max, int* flag) {
  ProfScope _p(st, K_MISC, 0.0);
  count_launch(K_MISC);
  launch_k(reortho_flag_k, dim3(1), dim3(32), 0, st, stats, kappa_max, flag);
  RUTV_LAUNCH_CK();
}

int qr_max_rows() { return QR_MAX_CLUSTER * QR_NT * 16; }

size_t qr_work_elems(int64_t b) { return size_t(3) * 32 * size_t(b) + 1024; }

namespace {
int panel_qr_tsqr(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
                  double* Tw, int64_t ldt, const QrWork& w);

int panel_qr_hh(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
                double* Tw, int64_t ldt, const QrWork& w) {
  if (m > qr_max_rows()) return panel_qr_tsqr(st, m, b, V, ldv, R, ldr, tau, Tw, ldt, w);
  GemmRole role(C_GEMM_QR);
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
  launch_k(zero_lower_k, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(b * b, 256), 1024))), dim3(256), 0, st, b, R, ldr);
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
    // S^T = V[j0:, 0:b]^T V_l (b x wj, skinny tile) as split-K partials; O = T_l^T S  (wj x b)
    const int splits = dgemm_partials(st, true, false, b, wj, rows, V + j0, ldv, Vl, ldv, w.part, w.part_elems);
    {
      ProfScope _p(st, C_QR_SMALL, 0.0);
      count_launch(C_QR_SMALL);
      launch_k(qr_small_k, dim3((unsigned)cdiv(b, 4)), dim3(256), 0, st, wj, b, splits, w.part, Tl, ldt, w.sfull);
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

int read_flag_sync(cudaStream_t st, const int* dflag);

// Householder QR of a panel taller than the cluster leaf kernel holds
// (m > qr_max_rows()): TSQR + Householder reconstruction (Ballard et al. 2015,
// the TSQR-HR variant; the same reconstruction as the CholeskyQR2 path, R20).
//   1. row chunks of h <= 8192 rows: Householder QR each (leaf kernel), keep
//      R_i stacked in S (nc b x b) and the chunk's thin Q_i (into w.q1);
//   2. Householder QR of the stack S = Q_s R, thin Q_s;
//   3. Q = blockdiag(Q_i) Q_s (m x b, orthonormal to rounding whatever the
//      rank or conditioning of the panel);
//   4. the reconstruction with Q as "Q1" and R as "R1" (G2 = Q^T Q = I to
//      rounding, so its second pass is the first-order closed form): W, T_w,
//      tau and R_h = S R -- in exact arithmetic exactly the reflectors of the
//      column-by-column Householder QR (R3).
// Needs w.q1 (m x b) and w.small; stack height nc b <= qr_max_rows().
int panel_qr_tsqr(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
                  double* Tw, int64_t ldt, const QrWork& w) {
  if (!w.q1 || !w.small || size_t(m) * b > w.q1_elems || b > 512) return ERR_UNSUPPORTED;
  constexpr int64_t kChunk = 8192;
  const int64_t nc = cdiv(m, kChunk);
  const int64_t h = cdiv(m, nc);     // balanced chunks of h or h - 1 >= b rows
  const int64_t hs = nc * b;         // stack height
  if (hs > qr_max_rows() || h - 1 < b) return ERR_UNSUPPORTED;
  const size_t stack = size_t(hs) * b;
  if (w.part_elems < 2 * stack + (size_t(1) << 20)) return ERR_UNSUPPORTED;
  GemmRole role(C_GEMM_QR);
  QrWork ws = w;                     // the stack S and Q_s at the tail of the split-K scratch
  ws.part_elems = w.part_elems - 2 * stack;
  double* S = w.part + ws.part_elems;
  double* Qs = S + stack;
  SmallWork sw = carve_small(w.small, b);
  const int bp = sw.bp;
  double* tmp = sw.W1;               // b x b scratch (the Gram slot is unused on this path)
  for (int64_t i = 0; i < nc; ++i) { // 1. chunk QRs, R_i -> S(i b : i b + b, :)
    const int64_t r0 = i * h, hi = std::min(h, m - r0);
    int rc = panel_qr_hh(st, hi, b, V + r0, ldv, S + i * b, hs, tau, Tw, ldt, ws);
    if (rc != OK) return rc;
    thin_q(st, hi, b, V + r0, ldv, Tw, ldt, w.q1 + r0, m, tmp, ws.part, ws.part_elems);
  }
  int rc = panel_qr_hh(st, hs, b, S, hs, R, ldr, tau, Tw, ldt, ws);  // 2. S = Q_s R
  if (rc != OK) return rc;
  thin_q(st, hs, b, S, hs, Tw, ldt, Qs, hs, tmp, ws.part, ws.part_elems);
  for (int64_t i = 0; i < nc; ++i) { // 3. Q = blockdiag(Q_i) Q_s -> V, then -> q1
    const int64_t r0 = i * h, hi = std::min(h, m - r0);
    dgemm(st, false, false, hi, b, b, 1.0, w.q1 + r0, m, Qs + i * b, hs, 0.0, V + r0, ldv, ws.part, ws.part_elems);
  }
  copy_matrix(st, m, b, V, ldv, w.q1, m);
  // 4. reconstruction: R1 := R (identity-padded), no first-pass breakdown
  set_identity(st, bp, bp, sw.R1, bp);
  copy_matrix(st, b, b, R, ldr, sw.R1, bp);
  RUTV_CK(cudaMemsetAsync(sw.stats, 0, sizeof(double), st));
  dgemm(st, true, false, b, b, m, 1.0, w.q1, m, w.q1, m, 0.0, sw.W2, bp, ws.part, ws.part_elems, 0, false, true);
  small_recon(st, b, sw, w.q1, m, R, ldr, tau, Tw, ldt, ws.part, ws.part_elems, nullptr, nullptr, nullptr, 0.5);
  if (read_flag_sync(st, sw.flag) != 0) return ERR_UNSUPPORTED;  // Q not orthonormal: cannot happen short of NaN
  dgemm(st, false, false, m - b, b, b, -1.0, w.q1 + b, m, sw.M, bp, 0.0, V + b, ldv, ws.part, ws.part_elems, 0, true);
  small_put_unit_lower(st, b, sw, V, ldv);
  return OK;
}

int read_flag_sync(cudaStream_t st, const int* dflag) {
  int h = 0;
  RUTV_CK(cudaMemcpyAsync(&h, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RUTV_CK(cudaStreamSynchronize(st));
  return h;
}

void read_stats_sync(cudaStream_t st, const double* dstats, double (&h)[3]) {
  RUTV_CK(cudaMemcpyAsync(h, dstats, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  RUTV_CK(cudaStreamSynchronize(st));
}

// kappa(R1) estimated by its diagonal: CholeskyQR's loss of orthogonality
// ~ kappa^2 eps stays <= 1e-8 -- ample for a basis of the power loop
constexpr double kReorthoKappaMax = 1e4;

bool cholqr_ok(const QrWork& w, int64_t m, int64_t b) {
  return w.mode == 0 && w.q1 && w.small && size_t(m) * b <= w.q1_elems && b <= 512;
}
}  // namespace

// Householder QR of an m x b panel (see kernels.h).  Default path: CholeskyQR2
// + Householder reconstruction (smallmat.cu, R20) -- four GEMMs over
// the panel and two cluster kernels -- with the column-by-column Householder
// kernel as the fallback when the panel is too ill-conditioned for CholeskyQR2
// (Cholesky breakdown or ||Q1^T Q1 - I||_max > 1/2, i.e. kappa >~ 1e7).
// highest-priority helper stream (per device) for the reconstruction's
// T_w / R_h products, and its fork / join events
cudaStream_t recon_side_stream() {
  static cudaStream_t streams[64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (!streams[dev]) {
    int least = 0, greatest = 0;
    RUTV_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    RUTV_CK(cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, greatest));
  }
  return streams[dev];
}
cudaEvent_t recon_event(int which) {
  static cudaEvent_t evs[2][64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (!evs[which][dev]) RUTV_CK(cudaEventCreateWithFlags(&evs[which][dev], cudaEventDisableTiming));
  return evs[which][dev];
}

int panel_qr(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
             double* Tw, int64_t ldt, const QrWork& w) {
  if (b <= 0) return OK;
  if (m < b) return ERR_UNSUPPORTED;
  const double* A0 = w.in ? w.in : V;  // the panel (read by the first CholeskyQR pass only)
  const int64_t lda0 = w.in ? w.ldin : ldv;
  if (cholqr_ok(w, m, b)) {
    GemmRole role(C_GEMM_QR);
    SmallWork sw = carve_small(w.small, b);
    const int bp = sw.bp;
    dgemm(st, true, false, b, b, m, 1.0, A0, lda0, A0, lda0, 0.0, sw.W1, bp, w.part, w.part_elems, 0, false, true);  // G1 (upper)
    small_chol_inv(st, b, sw);                                                                          // R1, R1^-1
    dgemm(st, false, false, m, b, b, 1.0, A0, lda0, sw.R1i, bp, 0.0, w.q1, m, w.part, w.part_elems, 0, true);  // Q1
    dgemm(st, true, false, b, b, m, 1.0, w.q1, m, w.q1, m, 0.0, sw.W2, bp, w.part, w.part_elems, 0, false, true);  // G2
    const bool optimistic = w.dev_flags && w.flag_count && *w.flag_count < w.flag_cap;
    if (optimistic) sw.flag = w.dev_flags + (*w.flag_count)++;
    cudaStream_t rs = recon_side_stream();
    cudaEvent_t ef = recon_event(0), ej = recon_event(1);
    small_recon(st, b, sw, w.q1, m, R, ldr, tau, Tw, ldt, w.part, w.part_elems, rs, ef, ej, w.orth_tol);
    const bool ok = optimistic || read_flag_sync(st, sw.flag) == 0;
    if (ok) {
      if (m > b)  // W(b:m, :) = -Q1(b:m, :) R2^-1 U~^-1
        dgemm(st, false, false, m - b, b, b, -1.0, w.q1 + b, m, sw.M, bp, 0.0, V + b, ldv, w.part, w.part_elems, 0,
              true);
      small_put_unit_lower(st, b, sw, V, ldv);
    }
    RUTV_CK(cudaStreamWaitEvent(st, ej, 0));  // T_w, tau, R_h
    if (ok) return OK;
    if (w.fallbacks) ++*w.fallbacks;
  }
  if (w.in) copy_matrix(st, m, b, w.in, w.ldin, V, ldv);  // the Householder path works in place
  return panel_qr_hh(st, m, b, V, ldv, R, ldr, tau, Tw, ldt, w);
}

bool panel_qr_begin(cudaStream_t st, int64_t m, int64_t b, const double* V, int64_t ldv, const QrWork& w) {
  if (b <= 0 || m < b || !cholqr_ok(w, m, b)) return false;
  if (!(w.dev_flags && w.flag_count && *w.flag_count < w.flag_cap)) return false;  // optimistic mode only
  GemmRole role(C_GEMM_QR);
  SmallWork sw = carve_small(w.small, b);
  const int bp = sw.bp;
  dgemm(st, true, false, b, b, m, 1.0, V, ldv, V, ldv, 0.0, sw.W1, bp, w.part, w.part_elems, 0, false, true);  // G1 (upper)
  small_chol_inv(st, b, sw);                                                                          // R1, R1^-1
  dgemm(st, false, false, m, b, b, 1.0, V, ldv, sw.R1i, bp, 0.0, w.q1, m, w.part, w.part_elems, 0, true);  // Q1
  return true;
}

void panel_qr_finish(cudaStream_t st, int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr,
                     double* tau, double* Tw, int64_t ldt, const QrWork& w) {
  GemmRole role(C_GEMM_QR);
  SmallWork sw = carve_small(w.small, b);
  const int bp = sw.bp;
  dgemm(st, true, false, b, b, m, 1.0, w.q1, m, w.q1, m, 0.0, sw.W2, bp, w.part, w.part_elems, 0, false, true);  // G2
  sw.flag = w.dev_flags + (*w.flag_count)++;
  cudaStream_t rs = recon_side_stream();
  cudaEvent_t ef = recon_event(0), ej = recon_event(1);
  small_recon(st, b, sw, w.q1, m, R, ldr, tau, Tw, ldt, w.part, w.part_elems, rs, ef, ej, w.orth_tol);
  if (m > b)  // W(b:m, :) = -Q1(b:m, :) R2^-1 U~^-1
    dgemm(st, false, false, m - b, b, b, -1.0, w.q1 + b, m, sw.M, bp, 0.0, V + b, ldv, w.part, w.part_elems, 0, true);
  small_put_unit_lower(st, b, sw, V, ldv);
  RUTV_CK(cudaStreamWaitEvent(st, ej, 0));  // T_w, tau, R_h
}

const double* panel_qr_M(const QrWork& w, int64_t b, int64_t* ldm) {
  SmallWork sw = carve_small(w.small, b);
  *ldm = sw.bp;
  return sw.M;
}

int reortho(cudaStream_t st, int64_t m, int64_t b, double* Y, int64_t ldy, double* Q, int64_t ldq, double* tmp_bb,
            double* Tmp_bb, double* tau, const QrWork& w) {
  if (cholqr_ok(w, m, b)) {
    GemmRole role(C_GEMM_QR);
    SmallWork sw = carve_small(w.small, b);
    const int bp = sw.bp;
    dgemm(st, true, false, b, b, m, 1.0, Y, ldy, Y, ldy, 0.0, sw.W1, bp, w.part, w.part_elems, 0, false, true);
    small_chol_inv(st, b, sw);
    constexpr double kKappaMax = kReorthoKappaMax;
    bool ok;
    if (w.dev_flags && w.flag_count && *w.flag_count < w.flag_cap) {
      reortho_flag(st, sw.stats, kKappaMax, w.dev_flags + (*w.flag_count)++);
      ok = true;
    } else {
      double h[3];
      read_stats_sync(st, sw.stats, h);
      ok = h[0] == 0.0 && h[2] <= kKappaMax * h[1];
    }
    if (ok) {
      dgemm(st, false, false, m, b, b, 1.0, Y, ldy, sw.R1i, bp, 0.0, Q, ldq, w.part, w.part_elems, 0, true);
      return OK;
    }
    if (w.fallbacks) ++*w.fallbacks;
  }
  int rc = panel_qr_hh(st, m, b, Y, ldy, tmp_bb, b, tau, Tmp_bb, b, w);
  if (rc != OK) return rc;
  thin_q(st, m, b, Y, ldy, Tmp_bb, b, Q, ldq, tmp_bb, w.part, w.part_elems);
  return OK;
}

bool reortho_defer_begin(cudaStream_t hs, int64_t m, int64_t b, const double* Y, int64_t ldy, const QrWork& w) {
  if (!cholqr_ok(w, m, b) || !(w.dev_flags && w.flag_count && *w.flag_count < w.flag_cap)) return false;
  GemmRole role(C_GEMM_QR);
  SmallWork sw = carve_small(w.small, b);
  dgemm(hs, true, false, b, b, m, 1.0, Y, ldy, Y, ldy, 0.0, sw.W1, sw.bp, w.part, w.part_elems, 0, false, true);
  small_chol_inv(hs, b, sw);
  reortho_flag(hs, sw.stats, kReorthoKappaMax, w.dev_flags + (*w.flag_count)++);
  return true;
}

void reortho_defer_apply(cudaStream_t st, int64_t rows, int64_t b, const double* Zp, int64_t ldzp, double* Z,
                         int64_t ldz, const QrWork& w) {
  GemmRole role(C_GEMM_QR);
  SmallWork sw = carve_small(w.small, b);
  dgemm(st, false, false, rows, b, b, 1.0, Zp, ldzp, sw.R1i, sw.bp, 0.0, Z, ldz, w.part, w.part_elems, 0, true);
}

void thin_q(cudaStream_t st, int64_t m, int64_t b, const double* V, int64_t ldv, const double* Tw, int64_t ldt,
            double* Q, int64_t ldq, double* tmp_bb, double* part, size_t part_elems) {
  GemmRole role(C_GEMM_QR);
  // tmp = Tw V1^T (V1 = V[0:b, 0:b]);  Q = E - V tmp
  dgemm(st, false, true, b, b, b, 1.0, Tw, ldt, V, ldv, 0.0, tmp_bb, b, part, part_elems);
  set_identity(st, m, b, Q, ldq);
  dgemm(st, false, false, m, b, b, -1.0, V, ldv, tmp_bb, b, 1.0, Q, ldq, part, part_elems);
}

}  // namespace rutv
