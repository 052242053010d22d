// Shared device/host helpers of the randUTV sm_100a path.
// Column-major fp64 everywhere: element (i, j) of a matrix with leading
// dimension ld lives at p[i + j * ld].
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace rutv {

// Error codes mirror include/randutv.h.
enum : int {
  OK = 0,
  ERR_NONFINITE = 1,
  ERR_CUDA = 2,
  ERR_NOMEM = 3,
  ERR_NCCL = 4,
  ERR_UNSUPPORTED = 5,
};

struct CudaError {
  cudaError_t e;
  const char* where;
};

#define RUTV_CK(x)                                                    \
  do {                                                                \
    cudaError_t _e = (x);                                             \
    if (_e != cudaSuccess) throw ::rutv::CudaError{_e, #x};          \
  } while (0)

#define RUTV_LAUNCH_CK() RUTV_CK(cudaGetLastError())

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Bump allocator over one device workspace block (256-byte aligned slices).
struct Arena {
  char* base = nullptr;
  size_t size = 0, off = 0;
  bool dry = false;  // dry run: only accumulate the size
  template <typename T>
  T* take(size_t count) {
    size_t bytes = ((count * sizeof(T)) + 255) & ~size_t(255);
    size_t o = off;
    off += bytes;
    if (dry) return nullptr;
    if (off > size) throw CudaError{cudaErrorMemoryAllocation, "arena overflow"};
    return reinterpret_cast<T*>(base + o);
  }
};

}  // namespace rutv
