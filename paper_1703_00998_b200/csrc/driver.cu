// Host driver of the blocked randUTV (Fig. fig:randUTV) and
// the C ABI of include/randutv.h.  The driver only enqueues kernels; every
// arithmetic step runs on the GPU.
//
// Per randomized step i (offset r0 = b(i-1), X = T(r0:m, r0:n)):
//   G = Philox Gaussian (m_i x b)
//   Y = X^T G;  q x { [Y <- thinQ(Y)]; Z = X Y; Y = X^T Z }        P:942-945 (+R5)
//   (W_v, T_v) = householder(Y)
//   T(:, r0:n) -= ((T(:, r0:n) W_v) T_v) W_v^T   (all m rows)     P:950 (R6)
//   (W_u, T_u, R11) = householder(T(r0:m, J2))
//   C = T(r0:m, J3):  C -= W_u ((C^T W_u) T_u)^T
//   T(I2, J2) = R11, T(I3, J2) = 0
// The b x b SVDs and their folds act only on rows I2 / columns J2,
// which later steps never touch, and left/right multiplications commute, so
// they are deferred and batched after the loop (SURVEY §0 finding 3,
// DESIGN.md R13).  U and V are formed, when requested, by backward
// accumulation of the stored reflectors: U = U_1...U_s blockdiag(Us_i).
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/randutv.h"
#include "common.cuh"
#include "kernels.h"

using namespace rutv;

namespace {

constexpr int kYFlags = 16;  // per-step sketch-side CholeskyQR decision slots (reorthos, QR(Y))

// Host threads serialise on g_mu while they enqueue; on the device, every
// call's work is ordered after the previous call's on the same device (the
// cached workspace and the shared side streams / events are reused), see
// CallOrder.  Cached buffers are kept per device.
std::mutex g_mu;
struct DevState {
  void* ws = nullptr;      // cached workspace (calls without opts.workspace)
  size_t ws_bytes = 0;
  void* stage = nullptr;   // device staging for host-buffer calls
  size_t stage_bytes = 0;
  cudaEvent_t last = nullptr;  // recorded at the end of the previous call's work
};
DevState g_dev[kMaxDevices];

DevState& dev_state() { return g_dev[current_device()]; }
}  // namespace

void rutv::call_order_begin(cudaStream_t st) {
  DevState& d = dev_state();
  if (d.last) RUTV_CK(cudaStreamWaitEvent(st, d.last, 0));
}

void rutv::call_order_end(cudaStream_t st) noexcept {
  DevState& d = g_dev[std::max(0, std::min(kMaxDevices - 1, [] { int v = 0; cudaGetDevice(&v); return v; }()))];
  if (!d.last && cudaEventCreateWithFlags(&d.last, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    d.last = nullptr;
    return;
  }
  if (cudaEventRecord(d.last, st) != cudaSuccess) cudaGetLastError();
}

namespace {

// Scope of one C-ABI call on stream st: st first waits for everything the
// previous call on this device enqueued (on any stream: all of them are joined
// into that call's stream before it records `last`), and at scope exit `last`
// is re-recorded on st.  Two threads, or two user streams, therefore never run
// on the same cached workspace at once.
struct CallOrder {
  cudaStream_t st;
  explicit CallOrder(cudaStream_t s) : st(s) { call_order_begin(st); }
  ~CallOrder() { call_order_end(st); }
};

struct Plan {
  int64_t m, n, b;
  int64_t ovs = 0;    // over-sampling p (Remark remark:positivep); sketch width bs = b + p
  int q;
  bool uv;
  int64_t s;          // loop bound min(ceil(m/b), ceil(n/b))
  int64_t nrand;      // number of randomized steps possible
  // offsets (doubles) of per-step reflector slots when uv
  std::vector<size_t> off_v, off_u;
  size_t elems_v = 0, elems_u = 0;
};

Plan make_plan(int64_t m, int64_t n, int64_t b, int q, bool uv, int64_t ovs = 0) {
  Plan p;
  p.m = m; p.n = n; p.b = b; p.q = q; p.uv = uv; p.ovs = ovs;
  p.s = std::min(cdiv(m, b), cdiv(n, b));
  p.nrand = 0;
  for (int64_t i = 1; i <= p.s; ++i)
    if (b * i < m && b * i < n) p.nrand = i;
  if (uv) {
    for (int64_t i = 1; i <= p.s; ++i) {
      int64_t r0 = b * (i - 1);
      p.off_v.push_back(p.elems_v);
      p.off_u.push_back(p.elems_u);
      p.elems_v += size_t(n - r0) * b;
      p.elems_u += size_t(m - r0) * b;
    }
  }
  return p;
}

struct Work {
  double *G, *Y, *Y2, *P, *P2, *Vu, *Wt, *Wt2, *tau, *Rtmp, *Ttmp;
  double *WG, *H;  // look-ahead sketch: [W_u | G'] (m x (b + bs)), H = W_u^T G' (b x bs)
  double* Zp;            // X Y before the deferred R^-1 of the power loop (m x bs, R26)
  double *Pbig, *part2;  // P_big = T(:, J3) Q1(b:, :) (m x b) and its split-K scratch (side stream)
  double *LT, *MT;       // L T_v, M T_v (b x b): the P2 assembly's right factors (read on two streams)
  size_t part2_elems;
  double *Qo, *Ro, *Do, *Uso, *Vso, *jworko;  // over-sampling: thin Q, R, SVD of R (width b + p)
  double *Tv, *Tu, *Rall, *Dall, *Usall, *Vsall, *jwork;
  double *Rfin, *Dfin, *Usfin, *Vsfin, *jworkf;
  double *Wv_all, *Wu_all;
  double *fold, *part, *nrm, *scal;
  int* flag;
  int* sweeps;
  int* qflags;    // optimistic CholeskyQR decision flags
  int qflags_cap;
  size_t part_elems;
  QrWork qw;
};

Work carve(Arena& ar, const Plan& p) {
  Work w{};
  const int64_t m = p.m, n = p.n, b = p.b, mx = std::max(m, n);
  const int64_t sb = std::max<int64_t>(p.nrand, 1);
  const int64_t bs = b + p.ovs;  // sketch width
  w.G = ar.take<double>(size_t(m) * bs);
  // [Wt | Y] contiguous (ld n): the fused left-apply / next-sketch GEMM
  // C^T [W_u | G'] writes C^T W_u into Wt and C^T G' into Y in one launch
  w.Wt = ar.take<double>(size_t(n) * (b + bs));
  w.Y = w.Wt + size_t(n) * b;
  w.Y2 = ar.take<double>(size_t(n) * bs);
  w.WG = ar.take<double>(size_t(m) * (b + bs));
  w.H = ar.take<double>(size_t(b) * bs);
  if (p.ovs > 0) {
    w.Qo = ar.take<double>(size_t(n) * bs);
    w.Ro = ar.take<double>(size_t(bs) * bs);
    w.Do = ar.take<double>(size_t(bs));
    w.Uso = ar.take<double>(size_t(bs) * bs);
    w.Vso = ar.take<double>(size_t(bs) * bs);
    w.jworko = ar.take<double>(jacobi_work_elems(1, (int)bs));
  }
  w.Zp = ar.take<double>(size_t(m) * bs);
  w.P = ar.take<double>(size_t(m) * b);
  w.P2 = ar.take<double>(size_t(m) * b);
  w.Pbig = ar.take<double>(size_t(m) * b);
  w.LT = ar.take<double>(size_t(b) * b);
  w.MT = ar.take<double>(size_t(b) * b);
  w.part2_elems = size_t(8) * m * b + size_t(148) * 32 * 1024;
  w.part2 = ar.take<double>(w.part2_elems);
  w.Vu = w.WG;  // W_u (T-only mode) in the first b columns of [W_u | G']
  w.Wt2 = ar.take<double>(size_t(n) * b);
  w.tau = ar.take<double>(size_t(bs));
  w.Rtmp = ar.take<double>(size_t(bs) * bs);
  w.Ttmp = ar.take<double>(size_t(bs) * bs);
  w.Tv = ar.take<double>(size_t(sb) * b * b);
  w.Tu = ar.take<double>(size_t(sb + 1) * b * b);
  w.Rall = ar.take<double>(size_t(sb) * b * b);
  w.Dall = ar.take<double>(size_t(sb) * b);
  w.Usall = ar.take<double>(size_t(sb) * b * b);
  w.Vsall = ar.take<double>(size_t(sb) * b * b);
  w.jwork = ar.take<double>(jacobi_work_elems((int)sb, (int)b));
  w.Rfin = ar.take<double>(size_t(b) * b);
  w.Dfin = ar.take<double>(size_t(b));
  w.Usfin = ar.take<double>(size_t(b) * b);
  w.Vsfin = ar.take<double>(size_t(b) * b);
  w.jworkf = ar.take<double>(jacobi_work_elems(1, (int)b));
  if (p.uv) {
    w.Wv_all = ar.take<double>(p.elems_v);
    w.Wu_all = ar.take<double>(p.elems_u);
  }
  w.fold = ar.take<double>(size_t(mx) * b);
  w.part_elems = size_t(12) * mx * bs + size_t(148) * 32 * 1024;
  w.part = ar.take<double>(w.part_elems);
  w.qw.part = w.part;
  w.qw.part_elems = w.part_elems;
  w.qw.sfull = ar.take<double>(size_t(32) * bs);
  w.qw.s2 = ar.take<double>(size_t(32) * bs);
  w.qw.z = ar.take<double>(size_t(32) * bs);
  w.qw.q1_elems = size_t(mx) * bs;
  w.qw.q1 = ar.take<double>(w.qw.q1_elems);
  w.qw.small = ar.take<double>(small_work_elems(bs));
  w.nrm = ar.take<double>(8192);
  w.scal = ar.take<double>(16);
  w.flag = ar.take<int>(16);
  w.sweeps = ar.take<int>(size_t(sb) + 16);
  // panel-QR decisions (one per step + final block) and, after them, one
  // step's sketch-side decisions (reorthos, over-sampling QR, QR(Y))
  w.qflags_cap = int((p.q + 3) * std::max<int64_t>(p.nrand, 1) + 8);  // + the sketch side's, deferred in graph mode
  w.qflags = ar.take<int>(size_t(w.qflags_cap) + kYFlags);
  return w;
}

size_t workspace_bytes(const Plan& p) {
  Arena ar;
  ar.dry = true;
  carve(ar, p);
  return ar.off + 4096;
}

enum MemKind { MEM_DEVICE, MEM_HOST };

MemKind mem_kind(const void* ptr) {
  if (!ptr) return MEM_DEVICE;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return MEM_HOST;
  }
  return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? MEM_DEVICE : MEM_HOST;
}

void dg(const Work& w, cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
        const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  dgemm(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, w.part, w.part_elems);
}

// Low-priority side stream per device for work off the critical path (the
// deferred b x b SVDs): its kernels fill the SMs the latency-bound panel-QR
// kernels leave idle, and the block scheduler prefers the main stream's CTAs.
// which = 0: deferred SVD chunks; 1: trailing right-apply updates; 2: D2H copies of final T blocks;
// 3: the last SVD chunk after the loop (concurrent with the end of the previous one).
cudaStream_t side_stream(int which = 0) {
  static cudaStream_t streams[4][64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[which][dev]) {
    int least = 0, greatest = 0;
    RUTV_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    RUTV_CK(cudaStreamCreateWithPriority(&streams[which][dev], cudaStreamNonBlocking, least));
  }
  return streams[which][dev];
}

// Two reusable events per device for the fork/join of the right-apply overlap.
// highest-priority stream of this device: the latency-bound panel QR that runs
// concurrently with the side-stream trailing update.  The caller's stream and
// the side streams share the default (lowest) priority, so without it the
// update's CTAs, queued first, kept the panel-QR GEMMs off the SMs (timeline:
// the 10000 x 256 panel Gram took 1.56 ms instead of 0.05 ms).
cudaStream_t priority_stream() {
  static cudaStream_t streams[64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) {
    int least = 0, greatest = 0;
    RUTV_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    RUTV_CK(cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, greatest));
  }
  return streams[dev];
}

// The factorization's critical path runs on an internal stream one priority
// level above the default (joined to the caller's stream at entry and exit):
// its kernels -- the latency-bound CholeskyQR chains in particular -- are then
// scheduled ahead of the default-priority side streams' GEMM CTAs they
// overlap (the look-ahead left update), and behind the panel QR's.
cudaStream_t crit_stream() {
  static cudaStream_t streams[64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) {
    int least = 0, greatest = 0;
    RUTV_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    RUTV_CK(cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, std::max(greatest, least - 1)));
  }
  return streams[dev];
}

cudaEvent_t overlap_event(int which) {
  static cudaEvent_t evs[16][64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (!evs[which][dev]) RUTV_CK(cudaEventCreateWithFlags(&evs[which][dev], cudaEventDisableTiming));
  return evs[which][dev];
}

int check_qr(int rc) {
  if (rc != OK) throw rc;
  return rc;
}

// ---- CUDA-graph replay of a repeated factorization -------------------------
// With U/V or T-only on device buffers, no early-stop tolerance and the
// optimistic CholeskyQR decisions, the whole enqueue after the non-finite
// scan (the loop, the batched SVDs, folds, final block, U/V formation) makes
// no host decision that depends on data: the launch sequence is a function of
// the arguments only.  A call repeated with the same arguments (same shape,
// pointers, seed, options and workspace) is captured once into a CUDA graph
// (on its second occurrence) and replayed from then on: ~2500 launches become
// one graph launch, which removes the per-launch host and front-end latency
// from the dependent kernel chains (small configs are launch-bound).
struct GraphKey {
  int dev;
  int64_t m, n, lda, b, k_stop;
  int q;
  uint64_t seed;
  const void *A, *U, *T, *V, *ws;
  size_t ws_bytes;
  int no_reortho, qr_mode, oversample;
  bool same(const GraphKey& o) const {
    return dev == o.dev && m == o.m && n == o.n && lda == o.lda && b == o.b && k_stop == o.k_stop && q == o.q &&
           seed == o.seed && A == o.A && U == o.U && T == o.T && V == o.V && ws == o.ws && ws_bytes == o.ws_bytes &&
           no_reortho == o.no_reortho && qr_mode == o.qr_mode && oversample == o.oversample;
  }
};
struct GraphEntry {
  GraphKey key{};
  int seen = 0;                      // eager runs with this key
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaEvent_t> evs;      // events recorded inside the graph (kept alive with it)
  long long launches[K_NCLASS] = {};  // kernels per replay, by class (gpu_launches accounting)
  int64_t steps = 0, k_done = 0;
  bool final_block = false;
  int nflags = 0;
};
std::vector<GraphEntry> g_graphs;  // most recent last; at most kMaxGraphs
constexpr size_t kMaxGraphs = 8;

void drop_graph(GraphEntry& e) {
  if (e.exec) cudaGraphExecDestroy(e.exec);
  for (cudaEvent_t ev : e.evs) cudaEventDestroy(ev);
  e.exec = nullptr;
  e.evs.clear();
}

GraphEntry& graph_entry(const GraphKey& k) {
  for (size_t i = 0; i < g_graphs.size(); ++i)
    if (g_graphs[i].key.same(k)) return g_graphs[i];
  if (g_graphs.size() >= kMaxGraphs) {
    RUTV_CK(cudaDeviceSynchronize());  // the evicted graph may still run
    drop_graph(g_graphs.front());
    g_graphs.erase(g_graphs.begin());
  }
  g_graphs.emplace_back();
  g_graphs.back().key = k;
  return g_graphs.back();
}

// The factorization proper (device pointers only).
constexpr int kRetry = 1000;  // factor_device: an optimistic CholeskyQR decision failed, redo synchronously

// on_final(c, st): work enqueued on the factorization's (internal) stream st has made columns
// 0..c-1 of T final (used to overlap the D2H of host-staged calls).
int factor_device(const randutv_opts& o, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int q,
                  uint64_t seed, int64_t k_stop, double* U, double* T, double* V, randutv_info* info,
                  void* ws, size_t ws_bytes, bool optimistic,
                  const std::function<void(int64_t, cudaStream_t)>& on_final =
                      std::function<void(int64_t, cudaStream_t)>()) {
  cudaStream_t ust = o.stream ? (cudaStream_t)o.stream : cudaStreamPerThread;  // the caller's stream
  cudaStream_t st = crit_stream();
  {
    cudaEvent_t e = overlap_event(8);
    RUTV_CK(cudaEventRecord(e, ust));
    RUTV_CK(cudaStreamWaitEvent(st, e, 0));
  }
  struct Join {  // every exit: the caller's stream waits for the internal one
    cudaStream_t ust, st;
    ~Join() {
      cudaEvent_t e = overlap_event(9);
      if (cudaEventRecord(e, st) != cudaSuccess || cudaStreamWaitEvent(ust, e, 0) != cudaSuccess) cudaGetLastError();
    }
  } join_guard{ust, st};
  const bool uv = (U != nullptr);
  const bool reortho = (o.no_reortho == 0);
  Plan p = make_plan(m, n, b, q, uv, o.oversample);
  Arena ar;
  ar.base = (char*)ws;
  ar.size = ws_bytes;
  Work w = carve(ar, p);
  int fallbacks = 0;
  w.qw.mode = o.qr_mode;
  w.qw.fallbacks = &fallbacks;
  int nflags = 0;
  if (optimistic && o.qr_mode == 0) {
    w.qw.dev_flags = w.qflags;
    w.qw.flag_count = &nflags;
    w.qw.flag_cap = w.qflags_cap;
  }
  // The re-orthonormalisations and QR(Y) of a step touch no part of T, so
  // their CholeskyQR decisions are checked per step: the step's device flags
  // are copied to the host right after QR(Y), ahead of the P = T W_v GEMM, and
  // read while that GEMM runs; if one failed (rank-deficient sketches: c5 step
  // 4), only this step's sketch and QR(Y) are redone with synchronous decisions
  // (Householder fallback in place) -- no whole-factorization retry.  The
  // column panel QR stays optimistic (flags checked once after the loop).
  QrWork qw_sync = w.qw;
  qw_sync.dev_flags = nullptr;
  qw_sync.flag_count = nullptr;
  const bool opt_y = optimistic && o.qr_mode == 0;
  static int* h_yflags = nullptr;  // pinned host copy of one step's flags
  if (opt_y && !h_yflags) RUTV_CK(cudaMallocHost(&h_yflags, sizeof(int) * kYFlags));
  cudaEvent_t ev_yflags = overlap_event(4);

  // ---- T <- A, ||A||_F, non-finite scan (one host sync)
  RUTV_CK(cudaMemsetAsync(w.flag, 0, sizeof(int), st));
  copy_norm_check(st, m, n, A, lda, T, m, w.nrm, w.scal, w.flag);
  double a2 = 0.0;
  int bad = 0;
  RUTV_CK(cudaMemcpyAsync(&a2, w.scal, sizeof(double), cudaMemcpyDeviceToHost, st));
  RUTV_CK(cudaMemcpyAsync(&bad, w.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RUTV_CK(cudaStreamSynchronize(st));
  if (bad) return RANDUTV_ERR_NONFINITE;
  const double a_fro = std::sqrt(a2);

  int64_t steps = 0, k_done = 0;
  bool final_block = false;
  const bool svd_side = jacobi_single_launch((int)b);
  cudaStream_t side = svd_side ? side_stream() : nullptr;
  std::vector<cudaEvent_t> evs;
  // graph mode (see GraphKey): every host decision of the enqueue is a function
  // of the arguments; the sketch side's CholeskyQR decisions are then deferred
  // to the once-per-call check like the column panels'
  const bool graph_ok = opt_y && o.tol == 0.0 && !on_final && !prof_active() && svd_side &&
                        jacobi_single_launch((int)(b + o.oversample)) && !getenv("RANDUTV_NO_GRAPH") &&
                        !getenv("RANDUTV_POISON_WORKSPACE");
  const bool defer_y = graph_ok;
  static const bool defer_reortho_env = [] {  // RANDUTV_NO_DEFER_REORTHO=1: A/B switch
    const char* e = getenv("RANDUTV_NO_DEFER_REORTHO");
    return !(e && atoi(e) != 0);
  }();
  const bool defer_reortho = defer_reortho_env && opt_y;
  static const bool sweep_at_defer = [] {  // RANDUTV_SWEEP_AT_DEFER=0/1: A/B switch
    const char* e = getenv("RANDUTV_SWEEP_AT_DEFER");
    return e ? atoi(e) != 0 : true;
  }();

  auto enqueue_all = [&]() {
  bool final_tall = false, final_fat = false;
  // The b x b SVDs of R11 are independent of later steps (R13): with
  // the single-cluster Jacobi kernel they run in chunks on the side stream.
  // steps per SVD chunk, measured at c3 with the incremental sweeps:
  // 4 / 6 / 8 / 10 / 12 = 269.0 / 268.0 / 265.3 / 266.6 / 268.0 ms
  // Factorizations with few steps (c1: 9, c2: 23) get shorter chunks so that
  // their SVDs start early and sweep beside the latency-bound chains instead
  // of all landing in the tail (RANDUTV_SVD_CHUNK=n forces n: A/B switch).
  static const int env_chunk = [] {
    const char* e = getenv("RANDUTV_SVD_CHUNK");
    return e ? atoi(e) : 0;
  }();
  const int64_t kSvdChunk = env_chunk > 0 ? env_chunk : std::max<int64_t>(2, std::min<int64_t>(8, p.nrand / 4));
  int64_t svd_done = 0;
  struct SvdChunk {
    int64_t s0, s1;
    cudaEvent_t done;
  };
  std::vector<SvdChunk> chunks;
  // With the incremental Jacobi (k <= 256) a chunk's SVDs advance one sweep
  // at the start of each latency-bound QR chain of the following steps (the
  // re-orthonormalisations and QR(Y), when most SMs are idle), and are
  // finished when the next chunk starts; otherwise a chunk runs in one go.
  const bool svd_incr = svd_side && jacobi_incremental((int)b);
  // after the loop: 0 = finish the active chunk, then the last steps' chunk
  // (sequential), 1 = one merged launch, 2 = both concurrently on two streams
  // (RANDUTV_SVD_TAIL: A/B switch)
  static const int tail_mode = [] {
    const char* e = getenv("RANDUTV_SVD_TAIL");
    return e ? atoi(e) : 2;
  }();
  struct ActiveChunk {
    int64_t s0 = 0, s1 = 0;
    bool on = false;
  } active;
  auto chunk_work = [&](int64_t s0) { return w.jwork + jacobi_work_elems((int)s0, (int)b); };
  auto finish_active = [&]() {
    if (!active.on) return;
    const int64_t s0 = active.s0, cnt = active.s1 - active.s0;
    jacobi_end(side, (int)cnt, (int)b, chunk_work(s0), w.Dall + s0 * b, w.Usall + size_t(s0) * b * b,
               w.Vsall + size_t(s0) * b * b, w.sweeps + s0);
    cudaEvent_t done;
    RUTV_CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    evs.push_back(done);
    RUTV_CK(cudaEventRecord(done, side));
    chunks.push_back({s0, active.s1, done});
    active.on = false;
  };
  // (Measured alternative, kept out: beginning every step's SVD right after its
  // R11 and sweeping a rolling range of the last 12 -- the tail is bounded by
  // the LAST step's SVD either way (~16 sweeps of one matrix after the loop),
  // and with a single fold chunk at the end the folds were exposed: c3 251.9 ->
  // 254.6 ms.)
  auto svd_sweep_here = [&]() {  // one sweep of the active chunk, starting at this point of st
    if (!active.on) return;
    cudaEvent_t e = overlap_event(4 + 1);
    RUTV_CK(cudaEventRecord(e, st));
    RUTV_CK(cudaStreamWaitEvent(side, e, 0));
    jacobi_sweeps(side, (int)(active.s1 - active.s0), (int)b, chunk_work(active.s0), 1);  // 1 / 2 / 3 per window: 265.3 / 267.5 / 269.5 ms
  };
  // merge (after the loop): the last steps' SVDs join the still active chunk
  // -- one launch finishes both (each matrix resumes from its own sweep), so
  // the tail holds one SVD latency instead of the active chunk's remaining
  // sweeps followed by a fresh chunk (c1: all 9 SVDs were in the tail, c2 ~14
  // + the rest of the previous chunk)
  auto launch_svd_chunk = [&](bool merge) {
    if (steps <= svd_done) return;
    cudaEvent_t e;
    RUTV_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    evs.push_back(e);
    RUTV_CK(cudaEventRecord(e, st));
    RUTV_CK(cudaStreamWaitEvent(side, e, 0));
    const int64_t s0 = svd_done, cnt = steps - svd_done;
    if (svd_incr && merge && tail_mode == 1 && active.on && active.s1 == s0) {
      jacobi_begin(side, (int)cnt, (int)b, w.Rall + size_t(s0) * b * b, b, b * b, chunk_work(s0));
      active.s1 = steps;
    } else if (svd_incr && merge && tail_mode == 2) {
      // the active chunk's remaining sweeps on the SVD stream, the last steps'
      // SVDs on a second one, concurrently: the tail holds one SVD latency and
      // the earlier chunk's folds run behind the last chunk's sweeps
      finish_active();
      cudaStream_t side3 = side_stream(3);
      RUTV_CK(cudaStreamWaitEvent(side3, e, 0));
      jacobi_begin(side3, (int)cnt, (int)b, w.Rall + size_t(s0) * b * b, b, b * b, chunk_work(s0));
      jacobi_end(side3, (int)cnt, (int)b, chunk_work(s0), w.Dall + s0 * b, w.Usall + size_t(s0) * b * b,
                 w.Vsall + size_t(s0) * b * b, w.sweeps + s0);
      cudaEvent_t done;
      RUTV_CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      evs.push_back(done);
      RUTV_CK(cudaEventRecord(done, side3));
      // the caller's stream joins side3 through the fold chain (main waits on done)
      chunks.push_back({s0, steps, done});
    } else if (svd_incr) {
      finish_active();
      jacobi_begin(side, (int)cnt, (int)b, w.Rall + size_t(s0) * b * b, b, b * b, chunk_work(s0));
      active.s0 = s0;
      active.s1 = steps;
      active.on = true;
    } else {
      jacobi_svd_batched(side, (int)cnt, (int)b, w.Rall + size_t(s0) * b * b, b, b * b, w.Dall + s0 * b,
                         w.Usall + size_t(s0) * b * b, w.Vsall + size_t(s0) * b * b, chunk_work(s0),
                         w.sweeps + s0);
      cudaEvent_t done;
      RUTV_CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      evs.push_back(done);
      RUTV_CK(cudaEventRecord(done, side));
      chunks.push_back({s0, steps, done});
    }
    svd_done = steps;
  };  // ---- folds into T, one SVD chunk at a time on the main stream
  // once that chunk's SVDs are done: T(I2,J2) = D, T(I2,J3) = Us^T T(I2,J3),
  // T(I1,J2) = T(I1,J2) Vs.  They act on rows above / columns left of the
  // trailing matrix and commute with the later steps' one-sided transforms
  // (left vs right products), so a chunk may be folded inside the loop one
  // chunk after its SVDs were launched; afterwards the column blocks of its
  // steps are final.
  size_t folded = 0;
  auto fold_chunk = [&](const SvdChunk& ch) {
    if (ch.done) RUTV_CK(cudaStreamWaitEvent(st, ch.done, 0));
    set_gemm_role(C_GEMM_OTHER);
    for (int64_t si = ch.s0; si < ch.s1; ++si) {
      const int64_t r0 = b * si;
      const double* Us = w.Usall + size_t(si) * b * b;
      const double* Vs = w.Vsall + size_t(si) * b * b;
      write_diag_block(st, b, b, w.Dall + si * b, T + r0 + r0 * m, m);            // T(I2,J2) = D
      const int64_t nc = n - r0 - b;
      if (nc > 0) {                                                                // T(I2,J3) = Us^T T(I2,J3)
        dg(w, st, true, false, b, nc, b, 1.0, Us, b, T + r0 + (r0 + b) * m, m, 0.0, w.fold, b);
        copy_matrix(st, b, nc, w.fold, b, T + r0 + (r0 + b) * m, m);
      }
      if (r0 > 0) {                                                                // T(I1,J2) = T(I1,J2) Vs
        dg(w, st, false, false, r0, b, b, 1.0, T + r0 * m, m, Vs, b, 0.0, w.fold, r0);
        copy_matrix(st, r0, b, w.fold, r0, T + r0 * m, m);
      }
    }
  };
  int64_t r0f = 0, nif = 0, mif = 0;
  double trailing = 0.0;
  bool stopped = false;
  // Look-ahead sketch.  With C = T(r0:m, J3) after the right apply, the next
  // step's trailing matrix is X' = rows b: of C - W_u Z', Z' = T_u^T W_u^T C
  // (the left apply), so its first sketch product is
  //   X'^T G_{i+1} = (U^T C)^T G' = C^T G'',  G' = [0_b; G_{i+1}],
  //   G'' = U G' = G' - W_u T_u (W_u^T G')
  // (the same product in exact arithmetic; G'' is formed beside the panel QR,
  // off the critical path): C^T W_u and X'^T G_{i+1} come out of ONE GEMM,
  // C^T [W_u | G''] (C read once), the left update is C -= (W_u T_u^T)(C^T W_u)^T, and the next
  // step's first re-orthonormalisation (or QR(Y) when q = 0) -- a latency-bound
  // chain -- runs on the critical stream while the left update C -= W_u Z'
  // runs on a side stream.  The next step waits for that update (ensure_lu)
  // before anything reads X.
  bool have_y0 = false;      // w.Y holds this step's X^T G from the look-ahead
  bool pending_lu = false;   // a look-ahead left update is in flight on side_stream(1)
  cudaEvent_t lu_join = overlap_event(7);
  auto ensure_lu = [&]() {
    if (!pending_lu) return;
    RUTV_CK(cudaStreamWaitEvent(st, lu_join, 0));
    pending_lu = false;
  };

  for (int64_t i = 1; i <= p.s; ++i) {
    const int64_t r0 = b * (i - 1);
    if (k_stop > 0 && r0 >= k_stop) { stopped = true; break; }
    const int64_t e2 = std::min(b * i, m), f2 = std::min(b * i, n);
    const int64_t mi = m - r0, ni = n - r0;
    double* X = T + r0 + r0 * m;
    if (b * i < m && b * i < n) {
      const int64_t si = i - 1;  // 0-based step slot
      double* Wv = nullptr;
      int64_t ldwv = n;
      double* Tv = w.Tv + size_t(si) * b * b;
      double* TJ = T + r0 * m;
      cudaStream_t upd = side_stream(1);  // side GEMMs: trailing right update, look-ahead left update, P_big
      // sketch, QR(Y) and P = T W_v, P2 = P T_v: reads T only
      auto sketch_qr_p = [&](const QrWork& qwy, bool copy_flags, bool use_y0) {
        // ---- sketch
        set_gemm_role(C_GEMM_SKETCH);
        const int64_t p_i = std::min<int64_t>(p.ovs, ni - b);  // over-sampling (R23); 0 = Fig. fig:randUTV
        const int64_t bw = b + p_i;                            // sketch width
        if (!use_y0) {
          ensure_lu();
          gaussian_fill(st, w.G, m, mi, bw, seed, uint32_t(i - 1), 0u);
          dg(w, st, true, false, ni, bw, mi, 1.0, X, m, w.G, m, 0.0, w.Y, n);
        }
        double* Ycur = w.Y;
        double* Yalt = w.Y2;
        for (int it = 0; it < q; ++it) {
          if (reortho) {
            // not beside the first chain of a look-ahead step: the left update
            // GEMM of the previous step fills the SMs there
            if (!(use_y0 && it == 0) && !(defer_reortho && !sweep_at_defer)) svd_sweep_here();
            // R26: Z = X (Y R^-1) = (X Y) R^-1 -- the Gram and the Cholesky run
            // on the priority stream while X Y runs here; only the TRMM stays
            // on the critical path.  The kappa decision is a device flag like
            // the others (a failure redoes the step's sketch synchronously).
            QrWork qd = qwy;
            qd.part = w.part2;  // the priority stream's own split-K scratch
            qd.part_elems = w.part2_elems;
            cudaEvent_t f = overlap_event(12), j = overlap_event(13);
            if (defer_reortho) {
              RUTV_CK(cudaEventRecord(f, st));
              RUTV_CK(cudaStreamWaitEvent(priority_stream(), f, 0));
            }
            if (defer_reortho && reortho_defer_begin(priority_stream(), ni, bw, Ycur, n, qd)) {
              RUTV_CK(cudaEventRecord(j, priority_stream()));
              ensure_lu();
              dg(w, st, false, false, mi, bw, ni, 1.0, X, m, Ycur, n, 0.0, w.Zp, m);     // Zp = X Y
              RUTV_CK(cudaStreamWaitEvent(st, j, 0));
              reortho_defer_apply(st, mi, bw, w.Zp, m, w.G, m, qwy);                   // Z = Zp R^-1
              dg(w, st, true, false, ni, bw, mi, 1.0, X, m, w.G, m, 0.0, Ycur, n);      // Y = X^T Z
              continue;
            }
            check_qr(rutv::reortho(st, ni, bw, Ycur, n, Yalt, n, w.Rtmp, w.Ttmp, w.tau, qwy));
            std::swap(Ycur, Yalt);
          }
          ensure_lu();
          dg(w, st, false, false, mi, bw, ni, 1.0, X, m, Ycur, n, 0.0, w.G, m);      // Z = X Y
          dg(w, st, true, false, ni, bw, mi, 1.0, X, m, w.G, m, 0.0, Ycur, n);       // Y = X^T Z
        }
        if (p_i > 0) {
          // Y <- the b dominant left singular vectors of the extended Y (P:1133-1135,
          // Fig. fig:stepUTVoversampling ``[Z,~,~] = svd(Y,'econ')``): Y = Q R,
          // R = Us D Vs^T, Z = Q Us(:, 1:b).  Column signs of Z are free (R9/A.3).
          GemmRole role(C_GEMM_QR);
          check_qr(panel_qr(st, ni, bw, Ycur, n, w.Ro, bw, w.tau, w.Ttmp, bw, qwy));
          thin_q(st, ni, bw, Ycur, n, w.Ttmp, bw, w.Qo, n, w.Rtmp, w.part, w.part_elems);
          jacobi_svd_batched(st, 1, (int)bw, w.Ro, bw, bw * bw, w.Do, w.Uso, w.Vso, w.jworko, nullptr);
          dg(w, st, false, false, ni, b, bw, 1.0, w.Qo, n, w.Uso, bw, 0.0, Yalt, n);
          std::swap(Ycur, Yalt);
        }
        // ---- V block: Householder QR of Y
        Wv = Ycur;
        ldwv = n;
        if (uv) {
          Wv = w.Wv_all + p.off_v[si];
          ldwv = ni;
          copy_matrix(st, ni, b, Ycur, n, Wv, ldwv);
        }
        svd_sweep_here();
        // ---- right apply to all m rows: P = T W_v, P2 = P T_v.
        // Optimistic CholeskyQR2 path: W_v = [L; -Q1(b:, :) M] (R20), so
        //   P = T(:, J2) L - (T(:, J3) Q1(b:, :)) M
        // and the big product P_big = T(:, J3) Q1(b:, :) needs only the first
        // CholeskyQR pass: it runs on the side stream (after the previous
        // step's look-ahead left update, stream order) while the second pass
        // and the reconstruction's latency-bound LU run here.
        const bool split = qwy.dev_flags && panel_qr_begin(st, ni, b, Wv, ldwv, qwy);
        if (split) {
          cudaEvent_t f = overlap_event(10), j = overlap_event(11);
          RUTV_CK(cudaEventRecord(f, st));
          RUTV_CK(cudaStreamWaitEvent(upd, f, 0));
          {
            GemmRole role(C_GEMM_RIGHT);
            dgemm(upd, false, false, m, b, ni - b, 1.0, TJ + b * m, m, qwy.q1 + b, ni, 0.0, w.Pbig, m, w.part2,
                  w.part2_elems);
          }
          RUTV_CK(cudaEventRecord(j, upd));
          panel_qr_finish(st, ni, b, Wv, ldwv, w.Rtmp, b, w.tau, Tv, b, qwy);
          if (copy_flags && *qwy.flag_count > 0) {
            RUTV_CK(cudaMemcpyAsync(h_yflags, qwy.dev_flags, sizeof(int) * *qwy.flag_count, cudaMemcpyDeviceToHost, st));
            RUTV_CK(cudaEventRecord(ev_yflags, st));
          }
          // P2 = P T_v = T(:, J2) (L T_v) - P_big (M T_v): two b x b products
          // replace one m x b x b pass.  Only the trailing rows r0:m are on the
          // critical path (the panel update and QR need them); the rows above
          // (I1, needed only by their own rank-b update) are formed on the side
          // stream, ahead of that update -- in the late steps r0 >> m_i.
          set_gemm_role(C_GEMM_RIGHT);
          int64_t ldm = 0;
          const double* M = panel_qr_M(qwy, b, &ldm);
          dg(w, st, false, false, b, b, b, 1.0, Wv, ldwv, Tv, b, 0.0, w.LT, b);          // L T_v
          dg(w, st, false, false, b, b, b, 1.0, M, ldm, Tv, b, 0.0, w.MT, b);            // M T_v
          if (r0 > 0) {  // rows I1 on the side stream (after P_big there, stream order)
            cudaEvent_t f1 = overlap_event(10);
            RUTV_CK(cudaEventRecord(f1, st));
            RUTV_CK(cudaStreamWaitEvent(upd, f1, 0));
            dgemm(upd, false, false, r0, b, b, 1.0, TJ, m, w.LT, b, 0.0, w.P2, m, nullptr, 0);
            dgemm(upd, false, false, r0, b, b, -1.0, w.Pbig, m, w.MT, b, 1.0, w.P2, m, nullptr, 0);
          }
          ensure_lu();
          dg(w, st, false, false, mi, b, b, 1.0, TJ + r0, m, w.LT, b, 0.0, w.P2 + r0, m);          // T(r0:, J2) L T_v
          RUTV_CK(cudaStreamWaitEvent(st, j, 0));
          dg(w, st, false, false, mi, b, b, -1.0, w.Pbig + r0, m, w.MT, b, 1.0, w.P2 + r0, m);   // - P_big M T_v
        } else {
          check_qr(panel_qr(st, ni, b, Wv, ldwv, w.Rtmp, b, w.tau, Tv, b, qwy));
          if (copy_flags && *qwy.flag_count > 0) {
            RUTV_CK(cudaMemcpyAsync(h_yflags, qwy.dev_flags, sizeof(int) * *qwy.flag_count, cudaMemcpyDeviceToHost, st));
            RUTV_CK(cudaEventRecord(ev_yflags, st));
          }
          set_gemm_role(C_GEMM_RIGHT);
          ensure_lu();
          dg(w, st, false, false, m, b, ni, 1.0, TJ, m, Wv, ldwv, 0.0, w.P, m);
          dg(w, st, false, false, m, b, b, 1.0, w.P, m, Tv, b, 0.0, w.P2, m);
        }
      };
      if (defer_y) {
        sketch_qr_p(w.qw, false, have_y0);  // decisions into the per-call flags
      } else if (opt_y) {
        int ny = 0;
        QrWork qwy = w.qw;
        qwy.dev_flags = w.qflags + w.qflags_cap;  // the kYFlags slots after the panel-QR ones
        qwy.flag_count = &ny;
        qwy.flag_cap = kYFlags;
        sketch_qr_p(qwy, true, have_y0);
        bool failed = false;
        if (ny > 0) {  // read while the P GEMM runs
          RUTV_CK(cudaEventSynchronize(ev_yflags));
          for (int f = 0; f < ny; ++f) failed |= h_yflags[f] != 0;
        }
        if (failed) sketch_qr_p(qw_sync, false, false);  // from scratch: Y = X^T G directly
      } else {
        sketch_qr_p(qw_sync, false, have_y0);
      }
      have_y0 = false;
      // the next step is randomized (and not cut by k_stop): look ahead
      const bool la_next = (b * (i + 1) < m && b * (i + 1) < n) && !(k_stop > 0 && b * i >= k_stop);
      const int64_t bw_next = la_next ? b + std::min<int64_t>(p.ovs, ni - 2 * b) : 0;
      // The panel QR below reads only the panel block T(r0:m, J2): update it
      // first on the main stream; the rest of the rank-b update (columns J3 and
      // the rows above the panel) runs on a low-priority side stream
      // concurrently with the latency-bound panel QR, and the left apply waits
      // for it.  Side GEMMs are unsplit (no shared split-K scratch).
      dg(w, st, false, true, mi, b, b, -1.0, w.P2 + r0, m, Wv, ldwv, 1.0, X, m);
      cudaEvent_t fork = overlap_event(0), join = overlap_event(1);
      RUTV_CK(cudaEventRecord(fork, st));
      RUTV_CK(cudaStreamWaitEvent(upd, fork, 0));
      if (r0 > 0) dgemm(upd, false, true, r0, b, b, -1.0, w.P2, m, Wv, ldwv, 1.0, TJ, m, nullptr, 0);
      dgemm(upd, false, true, m, ni - b, b, -1.0, w.P2, m, Wv + b, ldwv, 1.0, TJ + b * m, m, nullptr, 0);
      RUTV_CK(cudaEventRecord(join, upd));
      // ---- U block: Householder QR of the panel T(r0:m, J2)
      double* Wu = w.Vu;
      int64_t ldwu = m;
      if (uv) {
        Wu = w.Wu_all + p.off_u[si];
        ldwu = mi;
      }
      cudaStream_t hp = priority_stream();
      cudaEvent_t fork2 = overlap_event(2), join2 = overlap_event(3);
      RUTV_CK(cudaEventRecord(fork2, st));
      RUTV_CK(cudaStreamWaitEvent(hp, fork2, 0));
      // late steps: the trailing update (~2 m (n_i - b) b flops) is shorter than
      // the latency-bound panel QR, SMs idle there -- one more Jacobi sweep
      if (2.0 * double(m) * double(ni - b) * double(b) < 0.4e-3 * 30e12) svd_sweep_here();
      // G' = [0_b; G_{i+1}] next to W_u (Philox draw of step i+1), on a
      // helper stream beside the panel QR (only G'' below needs it)
      cudaEvent_t gdraw = overlap_event(14);
      if (la_next) {
        cudaStream_t gs = side_stream(3);
        RUTV_CK(cudaStreamWaitEvent(gs, fork2, 0));
        gaussian_fill(gs, w.WG + size_t(b) * m + b, m, mi - b, bw_next, seed, uint32_t(i), 0u);
        set_zero(gs, b, bw_next, w.WG + size_t(b) * m, m);
        RUTV_CK(cudaEventRecord(gdraw, gs));
      }
      double* Tu = w.Tu + size_t(si) * b * b;
      double* R11 = w.Rall + size_t(si) * b * b;
      QrWork qwu = w.qw;  // R11 enters T: CholeskyQR2 only while R is backward stable
      qwu.orth_tol = kRFactorOrthTol;
      qwu.in = X;         // the panel is read in place; W_u goes to Wu
      qwu.ldin = m;
      check_qr(panel_qr(hp, mi, b, Wu, ldwu, R11, b, w.tau, Tu, b, qwu));
      // T(I2,J2) = R11 (replaced by D after the batched SVD), T(I3,J2) = 0
      put_r_panel(hp, mi, b, R11, b, X, m);
      if (la_next) RUTV_CK(cudaStreamWaitEvent(hp, gdraw, 0));
      if (la_next) {
        // G'' = U G' = G' - W_u (T_u (W_u^T G')), so that C^T G'' = (U^T C)^T G'
        // = X'^T G_{i+1}; and WT = W_u T_u^T for the left update C -= WT (C^T W_u)^T.
        // G'' is formed here beside the trailing update, WT on the side stream.
        if (Wu != w.WG) copy_matrix(hp, mi, b, Wu, ldwu, w.WG, m);
        GemmRole role(C_GEMM_SKETCH);
        double* Gp = w.WG + size_t(b) * m;
        dg(w, hp, true, false, b, bw_next, mi, 1.0, w.WG, m, Gp, m, 0.0, w.H, b);        // H = W_u^T G'
        dg(w, hp, false, false, b, bw_next, b, 1.0, Tu, b, w.H, b, 0.0, w.Rtmp, b);     // T_u H
        dg(w, hp, false, false, mi, bw_next, b, -1.0, w.WG, m, w.Rtmp, b, 1.0, Gp, m);  // G'' = G' - W_u (T_u H)
      }
      RUTV_CK(cudaEventRecord(join2, hp));
      RUTV_CK(cudaStreamWaitEvent(st, join2, 0));
      if (la_next) {  // WT = W_u T_u^T for the left update, on the side stream (after its right update)
        RUTV_CK(cudaStreamWaitEvent(upd, join2, 0));
        GemmRole role(C_GEMM_LEFT);
        dgemm(upd, false, true, mi, b, b, 1.0, w.WG, m, Tu, b, 0.0, w.Pbig, m, nullptr, 0);
      }
      // ---- left apply to T(r0:m, J3), after the overlapped update
      RUTV_CK(cudaStreamWaitEvent(st, join, 0));
      set_gemm_role(C_GEMM_LEFT);
      const int64_t nc = n - f2;
      double* Cm = T + r0 + f2 * m;
      if (la_next) {
        // [C^T W_u | C^T G''] -> [Wt | Y]: Y = X'^T G_{i+1}, the next step's first sketch product
        dg(w, st, true, false, nc, b + bw_next, mi, 1.0, Cm, m, w.WG, m, 0.0, w.Wt, n);
        // C -= (W_u T_u^T)(C^T W_u)^T on the side stream, concurrent with the next step's first chain
        cudaEvent_t lf = overlap_event(6);
        RUTV_CK(cudaEventRecord(lf, st));
        RUTV_CK(cudaStreamWaitEvent(upd, lf, 0));
        {
          GemmRole role(C_GEMM_LEFT);
          dgemm(upd, false, true, mi, nc, b, -1.0, w.Pbig, m, w.Wt, n, 1.0, Cm, m, nullptr, 0);
        }
        RUTV_CK(cudaEventRecord(lu_join, upd));
        pending_lu = true;
        have_y0 = true;
      } else {
        dg(w, st, true, false, nc, b, mi, 1.0, Cm, m, Wu, ldwu, 0.0, w.Wt, n);       // C^T W_u
        dg(w, st, false, false, nc, b, b, 1.0, w.Wt, n, Tu, b, 0.0, w.Wt2, n);        // (C^T W_u) T_u
        dg(w, st, false, true, mi, nc, b, -1.0, Wu, ldwu, w.Wt2, n, 1.0, Cm, m);      // C -= W_u (.)^T
      }
      ++steps;
      k_done = f2;
      if (svd_side && steps - svd_done >= kSvdChunk) {
        // host-staged calls only: folding inside the loop puts the folds on the
        // critical path (+2 ms at c3) but lets T's final blocks stream back to
        // the host during the loop (-7 ms); device calls fold at the end, where
        // the folds hide behind the last SVD chunk
        if (on_final && folded < chunks.size()) {  // a chunk that ended at least one chunk ago
          ensure_lu();
          fold_chunk(chunks[folded]);
          if (on_final) on_final(b * chunks[folded].s1, st);
          ++folded;
        }
        launch_svd_chunk(false);
      }
      if (o.tol > 0.0) {
        double t2 = 0.0;
        ensure_lu();
        fro2(st, m - e2, n - f2, T + e2 + f2 * m, m, w.nrm, w.scal);
        RUTV_CK(cudaMemcpyAsync(&t2, w.scal, sizeof(double), cudaMemcpyDeviceToHost, st));
        RUTV_CK(cudaStreamSynchronize(st));
        trailing = std::sqrt(t2);
        if (trailing <= o.tol * a_fro) { stopped = true; break; }
      }
    } else {
      // ---- final block: economical SVD of T(r0:m, r0:n)
      ensure_lu();
      final_block = true;
      r0f = r0; mif = mi; nif = ni;
      if (mi > ni) {
        final_tall = true;
        double* Wf = uv ? (w.Wu_all + p.off_u[i - 1]) : w.Vu;
        int64_t ldwf = uv ? mi : m;
        copy_matrix(st, mi, ni, X, m, Wf, ldwf);
        QrWork qwf = w.qw;
        qwf.orth_tol = kRFactorOrthTol;
        check_qr(panel_qr(st, mi, ni, Wf, ldwf, w.Rfin, ni, w.tau, w.Tu + size_t(p.nrand) * b * b, ni, qwf));
      } else if (mi < ni) {
        // fat (Remark "The case m < n"): unpivoted QR of the ROWS,
        // X^T = Q [Rf; 0]; with Rf = Ur D Vr^T: X = Vr [D 0] (Q blockdiag(Ur, I))^T
        final_fat = true;
        double* Wf = uv ? (w.Wv_all + p.off_v[i - 1]) : w.Wt;
        int64_t ldwf = uv ? ni : n;
        transpose_matrix(st, mi, ni, X, m, Wf, ldwf);
        QrWork qwf = w.qw;
        qwf.orth_tol = kRFactorOrthTol;
        check_qr(panel_qr(st, ni, mi, Wf, ldwf, w.Rfin, mi, w.tau, w.Tu + size_t(p.nrand) * b * b, mi, qwf));
      } else {
        copy_matrix(st, ni, ni, X, m, w.Rfin, ni);
      }
      k_done = std::min(m, n);
      break;
    }
  }
  ensure_lu();
  if (!final_block && !stopped) k_done = std::min(k_done, std::min(m, n));
  const int64_t kf = std::min(mif, nif);  // order of the final block's SVD

  set_gemm_role(C_GEMM_OTHER);
  // ---- batched small SVDs
  if (svd_side) {
    launch_svd_chunk(true);
    finish_active();
  } else if (steps > 0) {
    jacobi_svd_batched(st, (int)steps, (int)b, w.Rall, b, b * b, w.Dall, w.Usall, w.Vsall, w.jwork, w.sweeps);
    chunks.push_back({0, steps, nullptr});
  }
  if (final_block)
    jacobi_svd_batched(st, 1, (int)kf, w.Rfin, kf, kf * kf, w.Dfin, w.Usfin, w.Vsfin, w.jworkf, w.sweeps + steps);

  // ---- the remaining folds (the last chunks)
  for (; folded < chunks.size(); ++folded) {
    fold_chunk(chunks[folded]);
    // host-staged calls: this chunk's column blocks are final -- their copy back overlaps the
    // wait for the last chunk's SVDs and its folds
    if (on_final) on_final(b * chunks[folded].s1, st);
  }
  if (final_block && final_fat) {
    // T(I2, J) = [diag(D) 0];  T(I1, J) <- T(I1, J) Q blockdiag(Ur, I)
    write_diag_block(st, mif, mif, w.Dfin, T + r0f + r0f * m, m);
    set_zero(st, mif, nif - mif, T + r0f + (r0f + mif) * m, m);
    if (r0f > 0) {
      const double* Wf = uv ? (w.Wv_all + p.off_v[p.s - 1]) : w.Wt;
      const int64_t ldwf = uv ? nif : n;
      const double* Tf = w.Tu + size_t(p.nrand) * b * b;
      double* TJ = T + r0f * m;
      dg(w, st, false, false, r0f, mif, nif, 1.0, TJ, m, Wf, ldwf, 0.0, w.P, r0f);
      dg(w, st, false, false, r0f, mif, mif, 1.0, w.P, r0f, Tf, mif, 0.0, w.P2, r0f);
      dg(w, st, false, true, r0f, nif, mif, -1.0, w.P2, r0f, Wf, ldwf, 1.0, TJ, m);
      dg(w, st, false, false, r0f, mif, mif, 1.0, TJ, m, w.Usfin, mif, 0.0, w.fold, r0f);
      copy_matrix(st, r0f, mif, w.fold, r0f, TJ, m);
    }
  } else if (final_block) {
    write_diag_block(st, mif, nif, w.Dfin, T + r0f + r0f * m, m);               // [diag(D); 0]
    if (r0f > 0) {
      dg(w, st, false, false, r0f, nif, nif, 1.0, T + r0f * m, m, w.Vsfin, nif, 0.0, w.fold, r0f);
      copy_matrix(st, r0f, nif, w.fold, r0f, T + r0f * m, m);
    }
  }

  // ---- U, V by backward accumulation
  if (uv) {
    set_identity(st, n, n, V, n);
    set_identity(st, m, m, U, m);
    if (final_block && final_tall) {
      const double* Wf = w.Wu_all + p.off_u[p.s - 1];
      const double* Tf = w.Tu + size_t(p.nrand) * b * b;
      double* Ub = U + r0f + r0f * m;
      dg(w, st, true, false, nif, mif, mif, 1.0, Wf, mif, Ub, m, 0.0, w.fold, nif);   // Wf^T U'
      dg(w, st, false, false, nif, mif, nif, 1.0, Tf, nif, w.fold, nif, 0.0, w.P, nif);  // Tf (.)
      dg(w, st, false, false, mif, mif, nif, -1.0, Wf, mif, w.P, nif, 1.0, Ub, m);      // U' -= Wf (.)
    }
    if (final_block && final_fat) {  // V' <- Q V' with Q = I - Wf Tf Wf^T (ni x ni, mi reflectors)
      const double* Wf = w.Wv_all + p.off_v[p.s - 1];
      const double* Tf = w.Tu + size_t(p.nrand) * b * b;
      double* Vb = V + r0f + r0f * n;
      dg(w, st, true, false, mif, nif, nif, 1.0, Wf, nif, Vb, n, 0.0, w.fold, mif);
      dg(w, st, false, false, mif, nif, mif, 1.0, Tf, mif, w.fold, mif, 0.0, w.Wt2, mif);
      dg(w, st, false, false, nif, nif, mif, -1.0, Wf, nif, w.Wt2, mif, 1.0, Vb, n);
    }
    for (int64_t si = steps - 1; si >= 0; --si) {
      const int64_t r0 = b * si, mi = m - r0, ni = n - r0;
      const double* Wv = w.Wv_all + p.off_v[si];
      const double* Wu = w.Wu_all + p.off_u[si];
      const double* Tv = w.Tv + size_t(si) * b * b;
      const double* Tu = w.Tu + size_t(si) * b * b;
      double* Vb = V + r0 + r0 * n;
      double* Ub = U + r0 + r0 * m;
      // V' <- (I - Wv Tv Wv^T) V'
      dg(w, st, true, false, b, ni, ni, 1.0, Wv, ni, Vb, n, 0.0, w.Wt, b);
      dg(w, st, false, false, b, ni, b, 1.0, Tv, b, w.Wt, b, 0.0, w.Wt2, b);
      dg(w, st, false, false, ni, ni, b, -1.0, Wv, ni, w.Wt2, b, 1.0, Vb, n);
      // U' <- (I - Wu Tu Wu^T) U'
      dg(w, st, true, false, b, mi, mi, 1.0, Wu, mi, Ub, m, 0.0, w.fold, b);
      dg(w, st, false, false, b, mi, b, 1.0, Tu, b, w.fold, b, 0.0, w.P, b);
      dg(w, st, false, false, mi, mi, b, -1.0, Wu, mi, w.P, b, 1.0, Ub, m);
    }
    // column folds with the small SVD factors
    for (int64_t si = 0; si < steps; ++si) {
      const int64_t r0 = b * si;
      dg(w, st, false, false, m, b, b, 1.0, U + r0 * m, m, w.Usall + size_t(si) * b * b, b, 0.0, w.fold, m);
      copy_matrix(st, m, b, w.fold, m, U + r0 * m, m);
      dg(w, st, false, false, n, b, b, 1.0, V + r0 * n, n, w.Vsall + size_t(si) * b * b, b, 0.0, w.fold, n);
      copy_matrix(st, n, b, w.fold, n, V + r0 * n, n);
    }
    if (final_block) {  // fat: U_small = Vr, V_small = Q blockdiag(Ur, I)
      const double* Uf = final_fat ? w.Vsfin : w.Usfin;
      const double* Vf = final_fat ? w.Usfin : w.Vsfin;
      dg(w, st, false, false, m, kf, kf, 1.0, U + r0f * m, m, Uf, kf, 0.0, w.fold, m);
      copy_matrix(st, m, kf, w.fold, m, U + r0f * m, m);
      dg(w, st, false, false, n, kf, kf, 1.0, V + r0f * n, n, Vf, kf, 0.0, w.fold, n);
      copy_matrix(st, n, kf, w.fold, n, V + r0f * n, n);
    }
  }
  (void)trailing;
  };  // enqueue_all

  if (!graph_ok) {
    enqueue_all();
  } else {
    GraphKey key{current_device(), m, n, lda, b, k_stop, q, seed, A, U, T, V, ws, ws_bytes,
                 o.no_reortho, o.qr_mode, o.oversample};
    GraphEntry& ge = graph_entry(key);
    if (ge.exec) {  // replay
      RUTV_CK(cudaGraphLaunch(ge.exec, st));
      for (int c = 0; c < K_NCLASS; ++c) count_launch(c, (int)ge.launches[c]);
      steps = ge.steps;
      k_done = ge.k_done;
      final_block = ge.final_block;
      nflags = ge.nflags;
    } else if (ge.seen < 1) {  // first occurrence: eager (also sets every kernel attribute)
      ++ge.seen;
      enqueue_all();
    } else {  // second occurrence: capture, instantiate, launch
      long long before[K_NCLASS], after[K_NCLASS];
      launches_by_class(before);
      RUTV_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
      cudaGraph_t graph = nullptr;
      try {
        enqueue_all();
      } catch (...) {
        cudaStreamEndCapture(st, &graph);
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        throw;
      }
      RUTV_CK(cudaStreamEndCapture(st, &graph));
      launches_by_class(after);
      // per-node priorities (copied from the capturing streams): the panel QR / critical / side
      // stream scheme survives the capture (without the flag: c3 260 -> 277 ms)
      cudaError_t e = cudaGraphInstantiateWithFlags(&ge.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(graph);
      RUTV_CK(e);
      for (int c = 0; c < K_NCLASS; ++c) ge.launches[c] = after[c] - before[c];
      ge.evs.swap(evs);  // the graph records them: they live as long as it does
      ge.steps = steps;
      ge.k_done = k_done;
      ge.final_block = final_block;
      ge.nflags = nflags;
      RUTV_CK(cudaGraphLaunch(ge.exec, st));
    }
  }
  if (nflags > 0) {  // optimistic CholeskyQR decisions: one read per call
    std::vector<int> hf(nflags);
    RUTV_CK(cudaMemcpyAsync(hf.data(), w.qflags, sizeof(int) * nflags, cudaMemcpyDeviceToHost, st));
    RUTV_CK(cudaStreamSynchronize(st));
    if (getenv("RANDUTV_DEBUG_FLAGS")) {  // diagnostics only
      for (int i = 0; i < nflags; ++i)
        if (hf[i]) fprintf(stderr, "randutv: CholeskyQR decision %d of %d failed\n", i, nflags);
    }
    for (int f : hf)
      if (f) {
        if (svd_side) RUTV_CK(cudaStreamSynchronize(side));
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
        return kRetry;
      }
  }
  for (cudaEvent_t e : evs) cudaEventDestroy(e);

  if (info) {
    info->k_done = k_done;
    info->steps = (int32_t)steps;
    info->final_block = final_block ? 1 : 0;
    info->a_fro = a_fro;
    int nsw = (int)steps + (final_block ? 1 : 0);
    std::vector<int> sw(std::max(nsw, 1), 0);
    if (nsw > 0) {
      RUTV_CK(cudaMemcpyAsync(sw.data(), w.sweeps, sizeof(int) * nsw, cudaMemcpyDeviceToHost, st));
    }
    if (k_done < n) {
      double t2 = 0.0;
      fro2(st, m - k_done, n - k_done, T + k_done + k_done * m, m, w.nrm, w.scal);
      RUTV_CK(cudaMemcpyAsync(&t2, w.scal, sizeof(double), cudaMemcpyDeviceToHost, st));
      RUTV_CK(cudaStreamSynchronize(st));
      info->trailing_fro = std::sqrt(t2);
    } else {
      RUTV_CK(cudaStreamSynchronize(st));
      info->trailing_fro = 0.0;
    }
    info->qr_fallbacks = fallbacks;
    info->max_sweeps = 0;
    for (int v : sw) info->max_sweeps = std::max(info->max_sweeps, v);
    if (getenv("RANDUTV_DEBUG_SWEEPS")) {  // diagnostics only
      for (int v : sw) fprintf(stderr, "%d ", v);
      fprintf(stderr, "\n");
    }
  }
  return RANDUTV_OK;
}

// grow-only cached device buffer of the current device (a regrow waits for
// the device: earlier calls may still use the old block)
void* cached_buffer(void*& p, size_t& have, size_t bytes) {
  if (bytes > have) {
    if (p) {
      RUTV_CK(cudaDeviceSynchronize());
      cudaFree(p);
      p = nullptr;
      have = 0;
    }
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return nullptr;
    }
    have = bytes;
  }
  return p;
}

void* cached_ws(size_t bytes) {
  DevState& d = dev_state();
  void* ws = cached_buffer(d.ws, d.ws_bytes, bytes);
  if (ws && getenv("RANDUTV_POISON_WORKSPACE")) {  // test hook, see poison_workspace (misc.cu)
    RUTV_CK(cudaDeviceSynchronize());
    RUTV_CK(cudaMemset(ws, 0xFF, d.ws_bytes));
    RUTV_CK(cudaDeviceSynchronize());
  }
  return ws;
}

void* cached_stage(size_t bytes) {
  DevState& d = dev_state();
  return cached_buffer(d.stage, d.stage_bytes, bytes);
}

int validate(int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int32_t q, int64_t k_stop, double* U,
             double* T, double* V) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (!A) return -3;
  if (lda < m) return -4;
  if (b < 1 || b > RANDUTV_MAX_B) return -5;
  if (q < 0) return -6;
  if (k_stop < 0) return -8;
  if ((U == nullptr) != (V == nullptr)) return -9;
  if (!T) return -10;
  return 0;
}

}  // namespace

extern "C" {

const char* randutv_version(void) { return "randutv-b200 0.1 (sm_100a, DMMA fp64)"; }

const char* randutv_strerror(int code) {
  switch (code) {
    case RANDUTV_OK: return "success";
    case RANDUTV_ERR_NONFINITE: return "input holds NaN or Inf";
    case RANDUTV_ERR_CUDA: return "CUDA runtime error";
    case RANDUTV_ERR_NOMEM: return "device allocation failed";
    case RANDUTV_ERR_NCCL: return "NCCL error";
    case RANDUTV_ERR_UNSUPPORTED: return "unsupported shape for this build";
    default: break;
  }
  if (code < 0) return "invalid argument (-code = 1-based position in randutv_factor)";
  return "unknown error";
}

size_t randutv_workspace_size(int64_t m, int64_t n, int64_t b, int32_t q, int32_t with_uv) {
  return randutv_workspace_size_ex(m, n, b, q, with_uv, 0);
}

size_t randutv_workspace_size_ex(int64_t m, int64_t n, int64_t b, int32_t q, int32_t with_uv, int32_t oversample) {
  if (m < 1 || n < 1 || b < 1 || oversample < 0) return 0;
  b = std::min<int64_t>(b, std::max(m, n));
  return workspace_bytes(make_plan(m, n, b, q, with_uv != 0, oversample));
}

int randutv_factor_ex(const randutv_opts* opts, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b,
                      int32_t q, uint64_t seed, int64_t k_stop, double* U, double* T, double* V,
                      randutv_info* info) {
  int rc = validate(m, n, A, lda, b, q, k_stop, U, T, V);
  if (rc) return rc;
  randutv_opts o{};
  if (opts) o = *opts;
  if (o.tol < 0 || std::isnan(o.tol)) return -12;
  if (o.qr_mode < 0 || o.qr_mode > 1) return -12;
  if (o.oversample < 0 || b + o.oversample > RANDUTV_MAX_B) return -12;
  if (b > std::min(m, n)) b = std::min(m, n);  // a single final-SVD step, same result as any larger b
  std::lock_guard<std::mutex> lock(g_mu);
  try {
    const bool host = mem_kind(A) == MEM_HOST || mem_kind(T) == MEM_HOST || (U && mem_kind(U) == MEM_HOST) ||
                      (V && mem_kind(V) == MEM_HOST);
    cudaStream_t st = o.stream ? (cudaStream_t)o.stream : cudaStreamPerThread;
    CallOrder order(st);
    const size_t need = workspace_bytes(make_plan(m, n, b, q, U != nullptr, o.oversample));
    void* ws = o.workspace;
    size_t wsb = o.workspace_bytes;
    if (!ws) {
      ws = cached_ws(need);
      wsb = need;
      if (!ws) return RANDUTV_ERR_NOMEM;
    } else if (wsb < need) {
      return -12;
    }
    poison_workspace(ws, wsb, st);
    // Optimistic first (no host synchronisation per panel QR); the synchronous
    // per-panel fallback run only if a CholeskyQR decision failed.  Not when T
    // aliases A (the first run would have destroyed the input).
    auto overlaps = [&](const double* X, size_t xbytes) {
      const char* a0 = (const char*)A;
      const char* a1 = a0 + sizeof(double) * (size_t(lda) * (n - 1) + m);
      const char* x0 = (const char*)X;
      return x0 < a1 && a0 < x0 + xbytes;
    };
    const bool opt = !overlaps(T, sizeof(double) * size_t(m) * n);
    if (!host) {
      int rc2 = factor_device(o, m, n, A, lda, b, q, seed, k_stop, U, T, V, info, ws, wsb, opt);
      if (rc2 == kRetry) rc2 = factor_device(o, m, n, A, lda, b, q, seed, k_stop, U, T, V, info, ws, wsb, false);
      return rc2;
    }
    // host buffers: stage through device memory inside the call
    const size_t elems = size_t(m) * n + (U ? size_t(m) * m + size_t(n) * n : 0);
    double* stage = (double*)cached_stage(elems * sizeof(double));
    if (!stage) return RANDUTV_ERR_NOMEM;
    double* dT = stage;
    double* dU = U ? stage + size_t(m) * n : nullptr;
    double* dV = U ? dU + size_t(m) * m : nullptr;
    auto stage_in = [&]() {  // contiguous input: one linear copy
      if (lda == m)
        RUTV_CK(cudaMemcpyAsync(dT, A, sizeof(double) * size_t(m) * n, cudaMemcpyDefault, st));
      else
        RUTV_CK(cudaMemcpy2DAsync(dT, sizeof(double) * m, A, sizeof(double) * lda, sizeof(double) * m, n,
                                  cudaMemcpyDefault, st));
    };
    stage_in();
    // T host buffer pinned: copy T's column blocks back as they become final
    // (after each in-loop fold) on a copy stream, overlapping the rest of the
    // factorization; the remainder is copied at the end.  Not when T aliases
    // A (in place): a retry after a failed optimistic CholeskyQR decision
    // re-stages A, which must then still be the input.
    int64_t copied = 0;
    cudaStream_t cps = nullptr;
    cudaEvent_t cev = nullptr;
    std::function<void(int64_t, cudaStream_t)> on_final;
    cudaPointerAttributes tat;
    if (!U && opt && cudaPointerGetAttributes(&tat, T) == cudaSuccess && tat.type == cudaMemoryTypeHost) {
      cps = side_stream(2);
      RUTV_CK(cudaEventCreateWithFlags(&cev, cudaEventDisableTiming));
      on_final = [&](int64_t cols, cudaStream_t fst) {  // fst: the stream the factorization enqueues on
        cols = std::min(cols, n);
        if (cols <= copied) return;
        RUTV_CK(cudaEventRecord(cev, fst));
        RUTV_CK(cudaStreamWaitEvent(cps, cev, 0));
        RUTV_CK(cudaMemcpyAsync(T + size_t(copied) * m, dT + size_t(copied) * m, sizeof(double) * m * (cols - copied),
                                cudaMemcpyDeviceToHost, cps));
        copied = cols;
      };
    } else {
      cudaGetLastError();
    }
    rc = factor_device(o, m, n, dT, m, b, q, seed, k_stop, dU, dT, dV, info, ws, wsb, true, on_final);
    if (rc == kRetry) {  // the input was factored in place: stage it again
      if (cps) RUTV_CK(cudaStreamSynchronize(cps));  // in-flight copies of the discarded run
      copied = 0;
      stage_in();
      rc = factor_device(o, m, n, dT, m, b, q, seed, k_stop, dU, dT, dV, info, ws, wsb, false, on_final);
    }
    if (rc == RANDUTV_OK) {
      if (copied < n)
        RUTV_CK(cudaMemcpyAsync(T + size_t(copied) * m, dT + size_t(copied) * m, sizeof(double) * m * (n - copied),
                                cudaMemcpyDefault, st));
      if (U) {
        RUTV_CK(cudaMemcpyAsync(U, dU, sizeof(double) * m * m, cudaMemcpyDefault, st));
        RUTV_CK(cudaMemcpyAsync(V, dV, sizeof(double) * n * n, cudaMemcpyDefault, st));
      }
    }
    RUTV_CK(cudaStreamSynchronize(st));
    if (cps) RUTV_CK(cudaStreamSynchronize(cps));
    if (cev) cudaEventDestroy(cev);
    return rc;
  } catch (const CudaError& e) {
    fprintf(stderr, "randutv: CUDA error %s at %s\n", cudaGetErrorString(e.e), e.where);
    return e.e == cudaErrorMemoryAllocation ? RANDUTV_ERR_NOMEM : RANDUTV_ERR_CUDA;
  } catch (int code) {
    return code;
  }
}

int randutv_factor(int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int32_t q, uint64_t seed,
                   int64_t k_stop, double* U, double* T, double* V) {
  randutv_opts o{};
  int rc = randutv_factor_ex(&o, m, n, A, lda, b, q, seed, k_stop, U, T, V, nullptr);
  if (rc == 0 && cudaStreamSynchronize(cudaStreamPerThread) != cudaSuccess) return RANDUTV_ERR_CUDA;
  return rc;
}

long long randutv_launch_count(void) { return launches_total(); }

int randutv_profile_begin(void) {
  std::lock_guard<std::mutex> lock(g_mu);
  prof_begin();
  return 0;
}

int randutv_profile_end(double* ms, double* flops, long long* launches) {
  std::lock_guard<std::mutex> lock(g_mu);
  double m4[K_NCLASS], f4[K_NCLASS];
  long long c4[K_NCLASS];
  static_assert(K_NCLASS <= 16, "profile arrays hold 16 classes");
  try {
    prof_end(m4, f4, c4);
  } catch (const CudaError&) {
    return RANDUTV_ERR_CUDA;
  }
  for (int i = 0; i < 16; ++i) {
    if (ms) ms[i] = i < K_NCLASS ? m4[i] : 0.0;
    if (flops) flops[i] = i < K_NCLASS ? f4[i] : 0.0;
    if (launches) launches[i] = i < K_NCLASS ? c4[i] : 0;
  }
  return 0;
}

long long randutv_profile_timeline(double* out, long long max_launches) {
  std::lock_guard<std::mutex> lock(g_mu);
  const std::vector<double>& tl = prof_timeline();
  const long long n = (long long)(tl.size() / 4);
  if (out)
    for (long long i = 0; i < std::min(n, max_launches) * 4; ++i) out[i] = tl[size_t(i)];
  return n;
}

const char* randutv_profile_class_name(int cls) {
  static const char* names[K_NCLASS] = {"gemm_sketch", "gemm_right_apply", "gemm_left_apply", "gemm_panel_qr",
                                        "gemm_other",  "qr_leaf",          "qr_small",        "jacobi_svd",
                                        "memory_helpers"};
  return (cls >= 0 && cls < K_NCLASS) ? names[cls] : nullptr;
}

int randutv_gaussian(double* G, int64_t ldg, int64_t rows, int64_t cols, uint64_t seed, uint32_t step,
                     uint32_t purpose, void* stream) {
  if (!G) return -1;
  if (ldg < rows) return -2;
  if (rows < 0) return -3;
  if (cols < 0) return -4;
  try {
    gaussian_fill(stream ? (cudaStream_t)stream : cudaStreamPerThread, G, ldg, rows, cols, seed, step, purpose);
  } catch (const CudaError&) {
    return RANDUTV_ERR_CUDA;
  }
  return 0;
}

int randutv_dgemm(int32_t transa, int32_t transb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  if (M < 0) return -3;
  if (N < 0) return -4;
  if (K < 0) return -5;
  if (lda < std::max<int64_t>(1, transa ? K : M)) return -8;
  if (ldb < std::max<int64_t>(1, transb ? N : K)) return -10;
  if (ldc < std::max<int64_t>(1, M)) return -13;
  std::lock_guard<std::mutex> lock(g_mu);
  try {
    size_t part = size_t(12) * std::max<int64_t>(M, 1) * std::max<int64_t>(N, 1) + size_t(148) * 32 * 1024;
    part = std::min(part, size_t(1) << 30);
    cudaStream_t st = stream ? (cudaStream_t)stream : cudaStreamPerThread;
    CallOrder order(st);
    double* ws = (double*)cached_ws(part * sizeof(double));
    if (!ws) return RANDUTV_ERR_NOMEM;
    dgemm(st, transa != 0, transb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, part);
  } catch (const CudaError&) {
    return RANDUTV_ERR_CUDA;
  }
  return 0;
}

int randutv_panel_qr_ex(int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
                        double* Tw, int64_t ldt, int32_t mode, int32_t* fallback, void* stream) {
  if (b < 1 || b > RANDUTV_MAX_B) return -2;
  if (m < b) return -1;
  if (!V || ldv < m) return -4;
  if (!R || ldr < b) return -6;
  if (!tau) return -7;
  if (!Tw || ldt < b) return -9;
  if (mode < 0 || mode > 1) return -10;
  std::lock_guard<std::mutex> lock(g_mu);
  try {
    size_t part = size_t(12) * m * b + size_t(148) * 32 * 1024;
    size_t extra = size_t(3) * 32 * b + 1024;
    size_t q1 = size_t(m) * b, sm = small_work_elems(b) + 64;
    cudaStream_t st = stream ? (cudaStream_t)stream : cudaStreamPerThread;
    CallOrder order(st);
    double* ws = (double*)cached_ws((part + extra + q1 + sm) * sizeof(double));
    if (!ws) return RANDUTV_ERR_NOMEM;
    QrWork w{ws, part, ws + part, ws + part + 32 * b, ws + part + 64 * b};
    w.q1 = ws + part + extra;
    w.q1_elems = q1;
    w.small = (double*)(((uintptr_t)(w.q1 + q1) + 255) & ~uintptr_t(255));
    w.mode = mode;
    w.orth_tol = kRFactorOrthTol;  // the caller keeps R
    int fb = 0;
    w.fallbacks = &fb;
    int rc = panel_qr(st, m, b, V, ldv, R, ldr, tau, Tw, ldt, w);
    if (fallback) *fallback = fb;
    return rc;
  } catch (const CudaError&) {
    return RANDUTV_ERR_CUDA;
  }
}

int randutv_panel_qr(int64_t m, int64_t b, double* V, int64_t ldv, double* R, int64_t ldr, double* tau,
                     double* Tw, int64_t ldt, void* stream) {
  return randutv_panel_qr_ex(m, b, V, ldv, R, ldr, tau, Tw, ldt, 0, nullptr, stream);
}

// Randomized SVD (Remark remark:RSVD): the first stage is the
// sketch of one randUTV step (Philox G of step 0, power loop with
// re-orthonormalization, Householder-equivalent QR for Q), the second stage
// B = A Q, B = Q_B R_B, R_B = Us D Vs^T, U = Q_B Us, V = Q Vs.
int randutv_rsvd(const randutv_opts* opts, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int32_t q,
                 uint64_t seed, double* U, int64_t ldu, double* D, double* V, int64_t ldv) {
  randutv_opts o{};
  if (opts) o = *opts;
  if (o.oversample < 0 || o.qr_mode < 0 || o.qr_mode > 1) return -1;
  if (m < 1) return -2;
  if (n < 1) return -3;
  if (!A) return -4;
  if (lda < m) return -5;
  const int64_t bs = b + o.oversample;
  if (b < 1 || bs > std::min(m, n) || bs > RANDUTV_MAX_B) return -6;
  if (q < 0) return -7;
  if (!U || ldu < m) return -9;
  if (!D) return -11;
  if (!V || ldv < n) return -12;
  std::lock_guard<std::mutex> lock(g_mu);
  try {
    cudaStream_t st = o.stream ? (cudaStream_t)o.stream : cudaStreamPerThread;
    CallOrder order(st);
    const int64_t mx = std::max(m, n);
    Arena ar;
    ar.dry = true;
    auto carve_rsvd = [&](Arena& a, double** bufs, QrWork& qw) {
      bufs[0] = a.take<double>(size_t(m) * bs);   // G, then B = A Q
      bufs[1] = a.take<double>(size_t(n) * bs);   // Y
      bufs[2] = a.take<double>(size_t(n) * bs);   // Y2 / Q
      bufs[3] = a.take<double>(size_t(m) * bs);   // Z, then Q_B
      bufs[4] = a.take<double>(size_t(bs) * bs);  // R (of Y, then of B)
      bufs[5] = a.take<double>(size_t(bs) * bs);  // T_w
      bufs[6] = a.take<double>(size_t(bs) * bs);  // tmp
      bufs[7] = a.take<double>(size_t(bs));       // tau
      bufs[8] = a.take<double>(size_t(bs));       // D (all bs)
      bufs[9] = a.take<double>(size_t(bs) * bs);  // Us
      bufs[10] = a.take<double>(size_t(bs) * bs); // Vs
      bufs[11] = a.take<double>(jacobi_work_elems(1, (int)bs));
      qw.part_elems = size_t(12) * mx * bs + size_t(148) * 32 * 1024;
      qw.part = a.take<double>(qw.part_elems);
      qw.sfull = a.take<double>(size_t(32) * bs);
      qw.s2 = a.take<double>(size_t(32) * bs);
      qw.z = a.take<double>(size_t(32) * bs);
      qw.q1_elems = size_t(mx) * bs;
      qw.q1 = a.take<double>(qw.q1_elems);
      qw.small = a.take<double>(small_work_elems(bs));
    };
    double* bf[12];
    QrWork qw{};
    carve_rsvd(ar, bf, qw);
    void* ws = cached_ws(ar.off + 4096);
    if (!ws) return RANDUTV_ERR_NOMEM;
    Arena ar2;
    ar2.base = (char*)ws;
    ar2.size = ar.off + 4096;
    carve_rsvd(ar2, bf, qw);
    qw.mode = o.qr_mode;
    double *G = bf[0], *Y = bf[1], *Y2 = bf[2], *Z = bf[3], *R = bf[4], *Tw = bf[5], *tmp = bf[6], *tau = bf[7],
           *Dall = bf[8], *Us = bf[9], *Vs = bf[10], *jw = bf[11];
    auto dgq = [&](bool ta, bool tb, int64_t M, int64_t N, int64_t K, const double* X, int64_t ldx, const double* Bm,
                   int64_t ldb, double* C, int64_t ldc) {
      dgemm(st, ta, tb, M, N, K, 1.0, X, ldx, Bm, ldb, 0.0, C, ldc, qw.part, qw.part_elems);
    };
    set_gemm_role(C_GEMM_SKETCH);
    gaussian_fill(st, G, m, m, bs, seed, 0u, 0u);                       // step 1
    dgq(true, false, n, bs, m, A, lda, G, m, Y, n);                     // Y = A^T G
    for (int it = 0; it < q; ++it) {                                    // step 2
      if (o.no_reortho == 0) {
        int rc = rutv::reortho(st, n, bs, Y, n, Y2, n, tmp, Tw, tau, qw);
        if (rc != OK) return rc;
        std::swap(Y, Y2);
      }
      dgq(false, false, m, bs, n, A, lda, Y, n, Z, m);                  // Z = A Y
      dgq(true, false, n, bs, m, A, lda, Z, m, Y, n);                   // Y = A^T Z
    }
    set_gemm_role(C_GEMM_QR);
    int rc = panel_qr(st, n, bs, Y, n, R, bs, tau, Tw, bs, qw);         // step 3: Q = orth(Y)
    if (rc != OK) return rc;
    thin_q(st, n, bs, Y, n, Tw, bs, Y2, n, tmp, qw.part, qw.part_elems);
    set_gemm_role(C_GEMM_OTHER);
    dgq(false, false, m, bs, n, A, lda, Y2, n, G, m);                   // B = A Q
    set_gemm_role(C_GEMM_QR);
    QrWork qwb = qw;  // R_B feeds the SVD: CholeskyQR2 only while R is backward stable (R20)
    qwb.orth_tol = kRFactorOrthTol;
    rc = panel_qr(st, m, bs, G, m, R, bs, tau, Tw, bs, qwb);            // B = Q_B R_B
    if (rc != OK) return rc;
    thin_q(st, m, bs, G, m, Tw, bs, Z, m, tmp, qw.part, qw.part_elems);
    jacobi_svd_batched(st, 1, (int)bs, R, bs, bs * bs, Dall, Us, Vs, jw, nullptr);  // R_B = Us D Vs^T
    set_gemm_role(C_GEMM_OTHER);
    dgq(false, false, m, b, bs, Z, m, Us, bs, U, ldu);                  // U = Q_B Us(:, 1:b)
    dgq(false, false, n, b, bs, Y2, n, Vs, bs, V, ldv);                 // V = Q Vs(:, 1:b)
    RUTV_CK(cudaMemcpyAsync(D, Dall, sizeof(double) * b, cudaMemcpyDeviceToDevice, st));
    return RANDUTV_OK;
  } catch (const CudaError& e) {
    fprintf(stderr, "randutv_rsvd: CUDA error %s at %s\n", cudaGetErrorString(e.e), e.where);
    return e.e == cudaErrorMemoryAllocation ? RANDUTV_ERR_NOMEM : RANDUTV_ERR_CUDA;
  } catch (int code) {
    return code;
  }
}

int randutv_small_svd_batched(int32_t batch, int32_t k, const double* R, int64_t ldr, int64_t strideR, double* D,
                              double* Us, double* Vs, int32_t* sweeps, void* stream) {
  if (batch < 0) return -1;
  if (k < 1 || k > RANDUTV_MAX_B) return -2;
  if (!R || ldr < k) return -4;
  std::lock_guard<std::mutex> lock(g_mu);
  try {
    size_t need = jacobi_work_elems(batch, k);
    cudaStream_t st = stream ? (cudaStream_t)stream : cudaStreamPerThread;
    CallOrder order(st);
    double* ws = (double*)cached_ws(need * sizeof(double));
    if (!ws) return RANDUTV_ERR_NOMEM;
    jacobi_svd_batched(st, batch, k, R, ldr, strideR, D, Us, Vs, ws, sweeps);
  } catch (const CudaError&) {
    return RANDUTV_ERR_CUDA;
  }
  return 0;
}

}  // extern "C"
