// Launch accounting and optional per-kernel-class CUDA-event timing.
// bench.py uses it to report gpu_launches and the dominant kernel's achieved
// throughput (roofline); it is off unless randutv_profile_begin() was called.
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rutv {

namespace {
std::atomic<long long> g_launches[K_NCLASS];
struct Rec {
  int cls;
  cudaEvent_t a, b;
  double flops;
  cudaStream_t st;
};
cudaEvent_t g_t0 = nullptr;  // timeline origin (recorded at prof_begin on the legacy stream)
std::vector<double> g_tl;     // [cls, stream slot, start ms, end ms] per launch of the last profile
std::vector<cudaStream_t> g_streams;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
size_t g_pool_used = 0;

cudaEvent_t take_event() {
  if (g_pool_used == g_pool.size()) {
    cudaEvent_t e;
    RUTV_CK(cudaEventCreate(&e));
    g_pool.push_back(e);
  }
  return g_pool[g_pool_used++];
}
}  // namespace

namespace {
int g_role = C_GEMM_OTHER;
}

int set_gemm_role(int role) {
  int prev = g_role;
  g_role = role;
  return prev;
}

static inline int resolve(int cls) { return cls == K_GEMM ? g_role : cls; }

void count_launch(int cls, int n) { g_launches[resolve(cls)].fetch_add(n, std::memory_order_relaxed); }

void launches_by_class(long long* out) {
  for (int i = 0; i < K_NCLASS; ++i) out[i] = g_launches[i].load();
}

bool prof_active() { return g_on; }

bool pdl_on() {
  static const bool on = getenv("RANDUTV_NO_PDL") == nullptr;
  return on;
}

long long pdl_max_ctas() {  // one wave of the current device (RANDUTV_PDL_MAX_CTAS: experiments)
  static const long long env = getenv("RANDUTV_PDL_MAX_CTAS") ? atoll(getenv("RANDUTV_PDL_MAX_CTAS")) : -1;
  return env >= 0 ? env : (long long)num_sms();
}

long long launches_total() {
  long long s = 0;
  for (int i = 0; i < K_NCLASS; ++i) s += g_launches[i].load();
  return s;
}

ProfScope::ProfScope(cudaStream_t st, int cls, double flops)
    : st_(st), cls_(resolve(cls)), flops_(flops), a_(nullptr) {
  if (!g_on) return;
  a_ = take_event();
  RUTV_CK(cudaEventRecord((cudaEvent_t)a_, st_));
}

ProfScope::~ProfScope() {
  if (!g_on || !a_) return;
  cudaEvent_t b = take_event();
  cudaEventRecord(b, st_);
  g_recs.push_back(Rec{cls_, (cudaEvent_t)a_, b, flops_, st_});
}

void prof_begin() {
  g_on = true;
  g_recs.clear();
  g_pool_used = 0;
  RUTV_CK(cudaDeviceSynchronize());
  if (!g_t0) RUTV_CK(cudaEventCreate(&g_t0));
  RUTV_CK(cudaEventRecord(g_t0, 0));
}

const std::vector<double>& prof_timeline() { return g_tl; }

void prof_end(double* ms, double* flops, long long* counts) {
  RUTV_CK(cudaDeviceSynchronize());
  for (int c = 0; c < K_NCLASS; ++c) {
    ms[c] = 0.0;
    flops[c] = 0.0;
    counts[c] = 0;
  }
  g_tl.clear();
  g_streams.clear();
  for (auto& r : g_recs) {
    float t = 0.f, t0 = 0.f;
    RUTV_CK(cudaEventElapsedTime(&t, r.a, r.b));
    RUTV_CK(cudaEventElapsedTime(&t0, g_t0, r.a));
    ms[r.cls] += t;
    flops[r.cls] += r.flops;
    counts[r.cls] += 1;
    size_t slot = 0;
    while (slot < g_streams.size() && g_streams[slot] != r.st) ++slot;
    if (slot == g_streams.size()) g_streams.push_back(r.st);
    g_tl.insert(g_tl.end(), {double(r.cls), double(slot), double(t0), double(t0 + t)});
  }
  g_on = false;
  g_recs.clear();
  g_pool_used = 0;
}

}  // namespace rutv
