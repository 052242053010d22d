// Phase timing of the b x b cluster kernels (smallmat.cu) with %globaltimer
// stamps from CTA 0 / thread 0: build with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/small_prof \
//        tools/small_prof.cu paper_1703_00998_b200/csrc/{prof,gemm,misc}.cu
// and run on the GPU: prints, per block step, the ns spent in each phase.
#include <cstdio>
#include <vector>
__device__ unsigned long long g_ts[4096];
__device__ int g_nts;
__device__ long long g_clk[2048];
#define SMALL_MARK(id)                                                              \
  do {                                                                              \
    if (threadIdx.x == 0 && cooperative_groups::this_cluster().block_rank() == 0) { \
      unsigned long long t;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                         \
      int n = g_nts;                                                                \
      if (n < 2048) { g_ts[2 * n] = (id); g_ts[2 * n + 1] = t; g_clk[n] = clock64(); g_nts = n + 1; } \
    }                                                                               \
  } while (0)
#include "../paper_1703_00998_b200/csrc/smallmat.cu"

int main(int argc, char** argv) {
  const int b = argc > 1 ? atoi(argv[1]) : 256;
  const size_t bp = rutv::small_pad(b);
  double* ws;
  cudaMalloc(&ws, rutv::small_work_elems(b) * sizeof(double));
  rutv::SmallWork w = rutv::carve_small(ws, b);
  std::vector<double> G(size_t(b) * b);
  // G = X^T X + b I for a random X: well-conditioned SPD
  std::vector<double> X(size_t(b) * b);
  for (auto& x : X) x = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) {
      double s = (i == j) ? b : 0.0;
      for (int k = 0; k < b; ++k) s += X[k + i * b] * X[k + j * b];
      G[i + j * b] = s;
    }
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy2D(w.W1, bp * 8, G.data(), b * 8, b * 8, b, cudaMemcpyHostToDevice);
    int zero = 0;
    cudaMemcpyToSymbol(g_nts, &zero, sizeof(int));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    if (argc > 2) {  // LU of a diagonally dominant F (recon_lu_k)
      std::vector<double> F(bp * bp, 0.0);
      for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) F[i + j * bp] = (i == j ? 3.0 : 0.0) + ((rand() / (double)RAND_MAX) - 0.5) / b;
      cudaMemcpy(w.F, F.data(), F.size() * 8, cudaMemcpyHostToDevice);
      rutv::ReconArgs a{};
      a.d = rutv::SmallDims{b, (int)bp, (int)bp / 32};
      a.F = w.F; a.Li = w.Li; a.Ui = w.Ui; a.US = w.US; a.S = w.S;
      rutv::launch_cluster(rutv::recon_lu_k, 0, rutv::SC, a);
    } else {
      rutv::small_chol_inv(0, b, w);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int n;
    cudaMemcpyFromSymbol(&n, g_nts, sizeof(int));
    std::vector<unsigned long long> ts(2 * n);
    cudaMemcpyFromSymbol(ts.data(), g_ts, sizeof(unsigned long long) * 2 * n);
    printf("b=%d chol_inv_k %.1f us, %d marks (err=%s)\n", b, ms * 1e3, n, cudaGetErrorString(cudaGetLastError()));
    if (rep == 2) {
      double acc[32] = {0};
      std::vector<long long> ck(n);
      cudaMemcpyFromSymbol(ck.data(), g_clk, sizeof(long long) * n);
      for (int i = 0; i < n && i < 24; ++i)
        printf("    mark %llu at %llu ns, %lld cycles\n", ts[2 * i], ts[2 * i + 1] - ts[1], ck[i] - ck[0]);
      for (int i = 1; i < n; ++i) acc[ts[2 * (i - 1)]] += double(ts[2 * i + 1] - ts[2 * i - 1]);
      const char* nm[] = {"load diag", "diag loop", "phase A", "barrier A", "phase B", "barrier B", "diag out", "B: tile_sum", "B: rmw", "B: next", "d:8x8 fact", "d:write", "d:panels", "d:trail"};
      for (int k = 0; k < 14; ++k) printf("  %-12s %8.1f us total\n", nm[k], acc[k] / 1e3);
    }
  }
  return 0;
}
