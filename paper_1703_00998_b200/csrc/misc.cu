// Memory-bound helpers: copies, identity/zero fills, Frobenius norms with a
// non-finite scan (input validation), the Philox Gaussian draw.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>
#include "philox.cuh"

#include <algorithm>

namespace rutv {

namespace {
constexpr int TB = 256;

inline int grid_for(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, TB), int64_t(num_sms()) * 16));
}

__global__ void scale_k(int64_t m, int64_t n, double beta, double* C, int64_t ldc) {
  pdl_begin();
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
      C[i + j * ldc] = beta == 0.0 ? 0.0 : beta * C[i + j * ldc];
}

// D(r, c) = r < b ? R(r, c) : 0, r < m, c < b
__global__ void put_r_panel_k(int64_t m, int64_t b, const double* __restrict__ R, int64_t ldr, double* __restrict__ D,
                              int64_t ldd) {
  pdl_begin();
  for (int64_t c = blockIdx.y; c < b; c += gridDim.y)
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x)
      D[r + c * ldd] = r < b ? R[r + c * ldr] : 0.0;
}

__global__ void copy_k(int64_t m, int64_t n, const double* __restrict__ S, int64_t lds, double* __restrict__ D,
                       int64_t ldd) {
  pdl_begin();
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
      D[i + j * ldd] = S[i + j * lds];
}

// D (n x m) = S^T (S m x n); 32x32 smem tiles, coalesced both ways
__global__ void transpose_k(int64_t m, int64_t n, const double* __restrict__ S, int64_t lds, double* __restrict__ D,
                            int64_t ldd) {
  pdl_begin();
  __shared__ double t[32][33];
  const int64_t i0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    t[r][threadIdx.x] = (i < m && j < n) ? S[i + j * lds] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;  // D(j, i) = S(i, j)
    if (i < m && j < n) D[j + i * ldd] = t[threadIdx.x][r];
  }
}

__global__ void ident_k(int64_t m, int64_t n, double* D, int64_t ldd, double diagv) {
  pdl_begin();
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
      D[i + j * ldd] = (i == j) ? diagv : 0.0;
}

// Per-block partial sums of squares (fixed partition -> deterministic).
__global__ void norm_partial_k(int64_t m, int64_t n, const double* __restrict__ S, int64_t lds,
                               double* __restrict__ D, int64_t ldd, double* partials, int* flag) {
  pdl_begin();
  __shared__ double red[TB / 32];
  double acc = 0.0;
  int bad = 0;
  // column-strided (fixed partition: deterministic; no 64-bit division per element)
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x)
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      double v = S[i + j * lds];
      if (D) D[i + j * ldd] = v;
      if (!isfinite(v)) bad = 1;
      acc = fma(v, v, acc);
    }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  if (bad && flag) atomicOr(flag, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < TB / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

// fixed-order (deterministic) sum of the partials: strided per thread, then a
// shared-memory tree (one 256-thread block)
__global__ void norm_final_k(int nparts, const double* partials, double* out2) {
  pdl_begin();
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 256) s += partials[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out2[0] = red[0];
}

__global__ void gaussian_k(double* G, int64_t ldg, int64_t rows, int64_t cols, uint32_t k0, uint32_t k1,
                           uint32_t step, uint32_t purpose) {
  pdl_begin();
  const int64_t npairs = (rows + 1) / 2;
  const int64_t total = npairs * cols;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t p = idx % npairs, c = idx / npairs;
    double g0, g1;
    philox_gaussian_pair(uint32_t(p), uint32_t(c), step, purpose, k0, k1, g0, g1);
    G[2 * p + c * ldg] = g0;
    if (2 * p + 1 < rows) G[2 * p + 1 + c * ldg] = g1;
  }
}

__global__ void diag_block_k(int64_t m, int64_t k, const double* d, double* D, int64_t ldd) {
  pdl_begin();
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y)
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
      D[i + j * ldd] = (i == j) ? d[j] : 0.0;
}

dim3 grid2(int64_t m, int64_t n) {
  int gx = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(m, TB), 64));
  int gy = (int)std::max<int64_t>(1, std::min<int64_t>(n, 4096));
  return dim3(gx, gy);
}
}  // namespace

void scale_matrix(cudaStream_t st, int64_t m, int64_t n, double beta, double* C, int64_t ldc) {
  if (m <= 0 || n <= 0) return;
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(scale_k, dim3(grid2(m, n)), dim3(TB), 0, st, m, n, beta, C, ldc); }
  RUTV_LAUNCH_CK();
}

void copy_matrix(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* D, int64_t ldd) {
  if (m <= 0 || n <= 0 || S == D) return;
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(copy_k, dim3(grid2(m, n)), dim3(TB), 0, st, m, n, S, lds, D, ldd); }
  RUTV_LAUNCH_CK();
}

void transpose_matrix(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* D, int64_t ldd) {
  if (m <= 0 || n <= 0) return;
  dim3 g((unsigned)cdiv(m, 32), (unsigned)cdiv(n, 32));
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(transpose_k, dim3(g), dim3(dim3(32, 8)), 0, st, m, n, S, lds, D, ldd); }
  RUTV_LAUNCH_CK();
}

void set_identity(cudaStream_t st, int64_t m, int64_t n, double* D, int64_t ldd) {
  if (m <= 0 || n <= 0) return;
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(ident_k, dim3(grid2(m, n)), dim3(TB), 0, st, m, n, D, ldd, 1.0); }
  RUTV_LAUNCH_CK();
}

void set_zero(cudaStream_t st, int64_t m, int64_t n, double* D, int64_t ldd) {
  if (m <= 0 || n <= 0) return;
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(ident_k, dim3(grid2(m, n)), dim3(TB), 0, st, m, n, D, ldd, 0.0); }
  RUTV_LAUNCH_CK();
}

void put_r_panel(cudaStream_t st, int64_t m, int64_t b, const double* R, int64_t ldr, double* D, int64_t ldd) {
  if (m <= 0 || b <= 0) return;
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(put_r_panel_k, dim3(grid2(m, b)), dim3(TB), 0, st, m, b, R, ldr, D, ldd); }
  RUTV_LAUNCH_CK();
}

void copy_norm_check(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* D,
                     int64_t ldd, double* scratch, double* out2, int* flag) {
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(n, 4096));
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(norm_partial_k, dim3(blocks), dim3(TB), 0, st, m, n, S, lds, (D == S) ? nullptr : D, ldd, scratch, flag); }
  RUTV_LAUNCH_CK();
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(norm_final_k, dim3(1), dim3(256), 0, st, blocks, scratch, out2); }
  RUTV_LAUNCH_CK();
}

void fro2(cudaStream_t st, int64_t m, int64_t n, const double* S, int64_t lds, double* scratch, double* out2) {
  if (m <= 0 || n <= 0) {
    RUTV_CK(cudaMemsetAsync(out2, 0, sizeof(double), st));
    return;
  }
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(n, 4096));
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(norm_partial_k, dim3(blocks), dim3(TB), 0, st, m, n, S, lds, nullptr, 0, scratch, nullptr); }
  RUTV_LAUNCH_CK();
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(norm_final_k, dim3(1), dim3(256), 0, st, blocks, scratch, out2); }
  RUTV_LAUNCH_CK();
}

void gaussian_fill(cudaStream_t st, double* G, int64_t ldg, int64_t rows, int64_t cols, uint64_t seed,
                   uint32_t step, uint32_t purpose) {
  if (rows <= 0 || cols <= 0) return;
  int64_t total = ((rows + 1) / 2) * cols;
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(gaussian_k, dim3(grid_for(total)), dim3(TB), 0, st, G, ldg, rows, cols, uint32_t(seed & 0xffffffffu),
                                             uint32_t(seed >> 32), step, purpose); }
  RUTV_LAUNCH_CK();
}

void write_diag_block(cudaStream_t st, int64_t m, int64_t k, const double* d, double* D, int64_t ldd) {
  if (m <= 0 || k <= 0) return;
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(diag_block_k, dim3(grid2(m, k)), dim3(TB), 0, st, m, k, d, D, ldd); }
  RUTV_LAUNCH_CK();
}

// Test hook (an initcheck substitute: compute-sanitizer is not available on
// the GPU pool): RANDUTV_POISON_WORKSPACE=1 fills the workspace with NaN bit
// patterns before each factorization, so a read of workspace memory that was
// never written shows up as NaN in the results.
void poison_workspace(void* p, size_t bytes, cudaStream_t st) {
  if (p && bytes && getenv("RANDUTV_POISON_WORKSPACE")) RUTV_CK(cudaMemsetAsync(p, 0xFF, bytes, st));
}

}  // namespace rutv
