// Cholesky + inverse of a b x b Gram (the CholeskyQR2 first pass): the
// DSMEM-resident cluster kernel (chol_inv_dsm_k) against the L2-resident one
// (chol_inv_k) on the same input -- max differences of R, R^-1, stats, and
// the time per launch (CUDA events, 50 launches each).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/chol_bench \
//        tools/chol_bench.cu paper_1703_00998_b200/csrc/{prof,gemm,misc}.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ unsigned long long g_mark[8][8];
#define DSM_MARK(cta, id)                                             \
  do {                                                                \
    if (threadIdx.x == 0) {                                           \
      unsigned long long t_;                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));          \
      g_mark[(cta)][(id)] = t_;                                       \
    }                                                                 \
  } while (0)
#include "../paper_1703_00998_b200/csrc/smallmat.cu"

int main(int argc, char** argv) {
  const int b = argc > 1 ? atoi(argv[1]) : 256;
  const double cond = argc > 2 ? atof(argv[2]) : 1e3;
  const int bp = rutv::small_pad(b);
  const rutv::SmallDims d{b, bp, bp / 32};
  std::vector<double> G(size_t(bp) * bp, 0.0);
  // G = X^T X with X = Q diag(s) (random orthogonal-ish via Gram-Schmidt-free scaling): SPD, kappa ~ cond^2
  std::vector<double> X(size_t(b) * b);
  srand(7);
  for (int j = 0; j < b; ++j) {
    const double sc = pow(cond, -double(j) / std::max(b - 1, 1));
    for (int i = 0; i < b; ++i) X[i + size_t(j) * b] = sc * ((rand() / (double)RAND_MAX) - 0.5);
  }
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) {
      double s = 0;
      for (int k = 0; k < b; ++k) s += X[k + size_t(i) * b] * X[k + size_t(j) * b];
      G[i + size_t(j) * bp] = s;
    }
  double *W, *R1, *Ri1, *R2, *Ri2, *st;
  cudaMalloc(&W, G.size() * 8);
  cudaMalloc(&R1, G.size() * 8);
  cudaMalloc(&Ri1, G.size() * 8);
  cudaMalloc(&R2, G.size() * 8);
  cudaMalloc(&Ri2, G.size() * 8);
  cudaMalloc(&st, 64 * 8);
  cudaMemcpy(W, G.data(), G.size() * 8, cudaMemcpyHostToDevice);
  auto old_k = [&]() { rutv::launch_cluster(rutv::chol_inv_k, 0, rutv::SC, d, W, R1, Ri1, st); };
  auto new_k = [&]() {
    rutv::launch_cluster_smem(rutv::chol_inv_dsm_k, 0, d.nb, rutv::chol_dsm_smem(), d, (const double*)W, R2, Ri2,
                              st + 8);
  };
  // old kernel updates W in place: run it on a copy
  double* W0;
  cudaMalloc(&W0, G.size() * 8);
  cudaMemcpy(W0, G.data(), G.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(W, W0, G.size() * 8, cudaMemcpyDeviceToDevice);
  old_k();
  cudaMemcpy(W, W0, G.size() * 8, cudaMemcpyDeviceToDevice);
  new_k();
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<double> a(G.size()), bb(G.size()), c(G.size()), dd(G.size()), s(16);
  cudaMemcpy(a.data(), R1, G.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(bb.data(), R2, G.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), Ri1, G.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(dd.data(), Ri2, G.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(s.data(), st, 16 * 8, cudaMemcpyDeviceToHost);
  double dr = 0, di = 0, nr = 0, ni = 0;
  for (size_t k = 0; k < a.size(); ++k) {
    dr = std::max(dr, fabs(a[k] - bb[k]));
    di = std::max(di, fabs(c[k] - dd[k]));
    nr = std::max(nr, fabs(a[k]));
    ni = std::max(ni, fabs(c[k]));
  }
  // residual of the new R: ||R^T R - G|| / ||G||, and ||R Ri - I||
  double res = 0, gn = 0, inv = 0;
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) {
      double t = 0, u = 0;
      for (int k = 0; k < bp; ++k) {
        t += bb[k + size_t(i) * bp] * bb[k + size_t(j) * bp];
        u += bb[i + size_t(k) * bp] * dd[k + size_t(j) * bp];
      }
      res = std::max(res, fabs(t - G[i + size_t(j) * bp]));
      gn = std::max(gn, fabs(G[i + size_t(j) * bp]));
      inv = std::max(inv, fabs(u - (i == j ? 1.0 : 0.0)));
    }
  printf("b=%d cond=%.1e  max|R_new-R_old|/max|R| %.2e  max|Ri_new-Ri_old|/max|Ri| %.2e  |R^T R-G|/|G| %.2e  |R Ri-I| %.2e\n",
         b, cond, dr / nr, di / ni, res / gn, inv);
  printf("stats old [%g %g %g] new [%g %g %g]\n", s[0], s[1], s[2], s[8], s[9], s[10]);
  {  // per-CTA phase stamps of the last new-kernel launch (ns from CTA 0's start)
    unsigned long long mk[8][8];
    cudaMemcpy(W, W0, G.size() * 8, cudaMemcpyDeviceToDevice);
    new_k();
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(mk, g_mark, sizeof(mk));
    const unsigned long long t0 = mk[0][0];
    for (int c = 0; c < d.nb; ++c)
      printf("  cta %d: start %6.2f  diag %6.2f -> %6.2f  E done %6.2f  end %6.2f us\n", c, (mk[c][0] - t0) * 1e-3,
             (mk[c][1] - t0) * 1e-3, (mk[c][2] - t0) * 1e-3, (mk[c][3] - t0) * 1e-3, (mk[c][4] - t0) * 1e-3);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int which = 0; which < 2; ++which) {
    for (int w = 0; w < 5; ++w) {
      cudaMemcpy(W, W0, G.size() * 8, cudaMemcpyDeviceToDevice);
      which ? new_k() : old_k();
    }
    float tot = 0;
    for (int r = 0; r < 50; ++r) {
      cudaMemcpy(W, W0, G.size() * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      which ? new_k() : old_k();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    printf("%s: %.1f us per launch\n", which ? "chol_inv_dsm_k" : "chol_inv_k   ", 1e3 * tot / 50);
  }
  return 0;
}
