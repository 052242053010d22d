// FP64 ceiling microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64).
// Prints achieved TFLOP/s for each; used to pick the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma884_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = 0; c1[c] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x * 1e-9 + k * 1e-3;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 0.999 - k * 1e-3;
  double c[CHAINS][4];
#pragma unroll
  for (int q = 0; q < CHAINS; ++q) for (int r = 0; r < 4; ++r) c[q][r] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < CHAINS; ++q)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < CHAINS; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"smem_optin\":%zu,\"l2\":%d,\"clock_khz\":%d,\"regs_per_sm\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.l2CacheSize, clk, p.regsPerMultiprocessor);
  double* out; CK(cudaMalloc(&out, 8));
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb;
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      float ms = time_it([&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
      double fl = 2.0 * 8 * iters * (double)blocks * threads;
      printf("{\"kernel\":\"dfma\",\"wpb\":%d,\"bps\":%d,\"tflops\":%.3f}\n", wpb, bps, fl / ms / 1e9);
      ms = time_it([&] { dmma884_loop<8><<<blocks, threads>>>(out, iters); });
      fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * wpb;
      printf("{\"kernel\":\"dmma_m8n8k4\",\"wpb\":%d,\"bps\":%d,\"tflops\":%.3f}\n", wpb, bps, fl / ms / 1e9);
      ms = time_it([&] { dmma16816_loop<4><<<blocks, threads>>>(out, iters / 4); });
      fl = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * blocks * wpb;
      printf("{\"kernel\":\"dmma_m16n8k16\",\"wpb\":%d,\"bps\":%d,\"tflops\":%.3f}\n", wpb, bps, fl / ms / 1e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
