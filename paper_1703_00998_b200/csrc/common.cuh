// Shared device/host helpers of the randUTV sm_100a path.
// Column-major fp64 everywhere: element (i, j) of a matrix with leading
// dimension ld lives at p[i + j * ld].
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>

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

constexpr int kMaxDevices = 64;

// Programmatic dependent launch (PDL).  Every kernel of the library begins
// with pdl_begin(): it waits until the previous kernel of its stream has
// completed and its writes are visible (griddepcontrol.wait -- a no-op when
// the kernel was not launched as a programmatic dependent), then lets the next
// kernel of the stream be launched (griddepcontrol.launch_dependents, effective
// once every CTA of this grid has started).  Launched through launch_k with
// programmatic stream serialisation, a dependent kernel's launch and CTA
// scheduling overlap the end of its predecessor instead of following its
// completion -- the per-kernel gap of the latency-bound chains.  Nothing runs
// before the wait, so ordering and visibility are those of plain stream order.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_on();         // false with RANDUTV_NO_PDL set (prof.cu)
long long pdl_max_ctas();  // largest grid launched as a programmatic dependent (prof.cu)

template <class K, class... Args>
void launch_k(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // only grids of at most one wave: a dependent grid's CTAs are scheduled
  // early and wait, and a many-wave grid would hold SMs that the side streams'
  // GEMMs use meanwhile (c3 251.6 -> 257.1 ms with PDL on every launch)
  const long long ctas = (long long)grid.x * grid.y * grid.z;
  cfg.numAttrs = (pdl_on() && ctas <= pdl_max_ctas()) ? 1 : 0;
  RUTV_CK(cudaLaunchKernelEx(&cfg, kern, args...));
}

inline int current_device() {
  int d = 0;
  RUTV_CK(cudaGetDevice(&d));
  if (d < 0 || d >= kMaxDevices) throw CudaError{cudaErrorInvalidDevice, "device index >= 64"};
  return d;
}

// cudaFuncSetAttribute acts on the current device only: run a kernel's
// attribute setup once per device (bit d of the mask = done on device d).
struct OncePerDevice {
  std::atomic<unsigned long long> mask{0};
  std::mutex mu;
  template <class F>
  void operator()(F&& f) {
    const unsigned long long bit = 1ull << current_device();
    if (mask.load(std::memory_order_acquire) & bit) return;
    std::lock_guard<std::mutex> lock(mu);
    if (mask.load(std::memory_order_relaxed) & bit) return;
    f();
    mask.fetch_or(bit, std::memory_order_release);
  }
};

// Raise a kernel's dynamic shared-memory limit to >= bytes on the current
// device (tracked per device; a larger later request raises it again).
struct SmemAttrPerDevice {
  std::mutex mu;
  size_t set[kMaxDevices] = {};
  template <class K>
  void ensure(K kern, size_t bytes, bool nonportable_cluster = false) {
    std::lock_guard<std::mutex> lock(mu);
    size_t& s = set[current_device()];
    if (bytes <= s) return;
    RUTV_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    if (nonportable_cluster) RUTV_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    s = bytes;
  }
};

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
