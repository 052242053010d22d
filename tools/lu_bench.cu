// The reconstruction's sign-modified LU (with L^-1, U~^-1, S, U~ S): the
// DSMEM-resident cluster kernel (lu_dsm_k) against the L2-resident one
// (recon_lu_k) on the same F -- max differences of every output and the time
// per launch (CUDA events, 50 launches each), plus per-CTA phase stamps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/lu_bench \
//        tools/lu_bench.cu paper_1703_00998_b200/csrc/{prof,gemm,misc}.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ unsigned long long g_lmark[8][8];
#define LU_MARK(cta, id)                                              \
  do {                                                                \
    if (threadIdx.x == 0) {                                           \
      unsigned long long t_;                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));          \
      g_lmark[(cta)][(id)] = t_;                                      \
    }                                                                 \
  } while (0)
#include "../paper_1703_00998_b200/csrc/smallmat.cu"

int main(int argc, char** argv) {
  const int b = argc > 1 ? atoi(argv[1]) : 256;
  const int bp = rutv::small_pad(b);
  const rutv::SmallDims d{b, bp, bp / 32};
  // F = -Q(0:b,:) R2^-1 of a random orthonormal Q: entries of modulus < 1, zero padding
  std::vector<double> F(size_t(bp) * bp, 0.0);
  srand(11);
  for (int j = 0; j < b; ++j)
    for (int i = 0; i < b; ++i) F[i + size_t(j) * bp] = ((rand() / (double)RAND_MAX) - 0.5) * 0.6;
  size_t q = size_t(bp) * bp;
  double* ws;
  cudaMalloc(&ws, 16 * q * 8);
  double *F0 = ws, *F1 = ws + q, *F2 = ws + 2 * q, *Li1 = ws + 3 * q, *Li2 = ws + 4 * q, *Ui1 = ws + 5 * q,
         *Ui2 = ws + 6 * q, *US1 = ws + 7 * q, *US2 = ws + 8 * q, *S1 = ws + 9 * q, *S2 = ws + 10 * q;
  cudaMemcpy(F0, F.data(), q * 8, cudaMemcpyHostToDevice);
  rutv::ReconArgs a{};
  a.d = d;
  auto old_k = [&]() {
    cudaMemcpy(F1, F0, q * 8, cudaMemcpyDeviceToDevice);
    a.F = F1; a.Li = Li1; a.Ui = Ui1; a.US = US1; a.S = S1;
    rutv::launch_cluster(rutv::recon_lu_k, 0, rutv::SC, a);
  };
  auto new_k = [&]() {
    cudaMemcpy(F2, F0, q * 8, cudaMemcpyDeviceToDevice);
    rutv::launch_cluster_smem(rutv::lu_dsm_k, 0, d.nb, sizeof(rutv::LuSm), d, F2, Li2, Ui2, S2, US2);
  };
  old_k();
  new_k();
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  auto cmp = [&](const char* nm, double* x, double* y, size_t n) {
    std::vector<double> hx(n), hy(n);
    cudaMemcpy(hx.data(), x, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hy.data(), y, n * 8, cudaMemcpyDeviceToHost);
    double dm = 0, nm_ = 0;
    for (size_t k = 0; k < n; ++k) { dm = std::max(dm, fabs(hx[k] - hy[k])); nm_ = std::max(nm_, fabs(hx[k])); }
    printf("  %-3s max|new-old| %.2e (max|old| %.2e)\n", nm, dm, nm_);
  };
  printf("b=%d\n", b);
  cmp("F", F1, F2, q); cmp("Li", Li1, Li2, q); cmp("Ui", Ui1, Ui2, q); cmp("US", US1, US2, q); cmp("S", S1, S2, bp);
  {
    unsigned long long mk[8][8];
    new_k();
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(mk, g_lmark, sizeof(mk));
    const unsigned long long t0 = mk[0][0];
    for (int c = 0; c < d.nb; ++c)
      printf("  cta %d: diag %6.2f -> %6.2f  Lcol %6.2f  E done %6.2f  end %6.2f us\n", c, (mk[c][1] - t0) * 1e-3,
             (mk[c][2] - t0) * 1e-3, (mk[c][3] - t0) * 1e-3, (mk[c][4] - t0) * 1e-3, (mk[c][5] - t0) * 1e-3);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int which = 0; which < 2; ++which) {
    for (int w = 0; w < 5; ++w) which ? new_k() : old_k();
    float tot = 0;
    for (int r = 0; r < 50; ++r) {
      cudaMemcpy(which ? F2 : F1, F0, q * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      if (which) rutv::launch_cluster_smem(rutv::lu_dsm_k, 0, d.nb, sizeof(rutv::LuSm), d, F2, Li2, Ui2, S2, US2);
      else { a.F = F1; rutv::launch_cluster(rutv::recon_lu_k, 0, rutv::SC, a); }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    printf("%s: %.1f us per launch\n", which ? "lu_dsm_k  " : "recon_lu_k", 1e3 * tot / 50);
  }
  return 0;
}
