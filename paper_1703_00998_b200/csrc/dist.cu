// Multi-GPU randUTV: A, T in 1-D block-cyclic
// column blocks of width b (block j on rank j mod P), T-only mode.
//
// Every step of Fig. fig:randUTV maps onto rank-local DMMA
// GEMMs plus a fixed set of collectives per step:
//   sketch      G_i on every rank (Philox, no communication);  Y_loc = X_loc^T G
//   power loop  C1  allreduce of the b x b Gram (CholeskyQR re-orthonormalization)
//               C1' allreduce of Z = X Y = sum_r X_loc Y_loc  (m_i x b)
//   QR(Y)       C2  allreduce of the two Grams + broadcast of the top b x b block
//               of Q1 from the owner of block i; the reconstruction runs
//               redundantly (deterministically) on every rank, so W_v stays
//               distributed by rows exactly like the columns of X
//   right apply C3  allreduce of P = T(:,J) W_v = sum_r T_loc W_v,loc  (m x b)
//   panel QR    C4  broadcast of (W_u, T_u, R11) from the owner of block i
//   left apply  local;   early stop: allreduce of the trailing ||.||_F^2
// The b x b SVDs (R11 is on every rank) and their folds run after the loop:
// the row folds T(I2,J3) <- Us^T T(I2,J3) on every rank's local columns, the
// column folds T(I1,J2) <- T(I1,J2) Vs on the owner.
//
// Collectives go through a small interface with two implementations: NCCL (one
// process per GPU; the symbols are resolved with dlopen from the libnccl the
// process already loaded, e.g. torch's) and a loopback that drives P virtual
// ranks on ONE device with host-ordered collectives (bulk-synchronous phases:
// no kernel ever waits on another rank) -- the latter exists to check the
// distributed arithmetic against the oracle on a single GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/randutv.h"
#include "common.cuh"
#include "kernels.h"

using namespace rutv;

// ----------------------------------------------------------------------------- block-cyclic layout
namespace {
inline int64_t nblocks(int64_t n, int64_t b) { return cdiv(n, b); }
// local column count of rank r
inline int64_t local_cols(int64_t n, int64_t b, int r, int P) {
  const int64_t nb = nblocks(n, b);
  int64_t c = 0;
  for (int64_t j = r; j < nb; j += P) c += std::min(b, n - j * b);
  return c;
}
// number of blocks of rank r with global index < p
inline int64_t blocks_before(int64_t p, int r, int P) { return (p > r) ? (p - r + P - 1) / P : 0; }
}  // namespace

// ----------------------------------------------------------------------------- communicators
namespace rutv {

struct Comm {
  virtual ~Comm() {}
  int P = 1;                // world size
  std::vector<int> ranks;   // global ranks this process drives (1 for NCCL, P for loopback)
  int dev = 0;
  bool aborted = false;     // NCCL: aborted after an asynchronous error or a timeout; unusable
  // collectives issued (one per call, whatever the number of local ranks) and
  // their payload per rank in bytes: [0] allreduce, [1] broadcast, [2] allgather
  long long ncoll[3] = {0, 0, 0}, nbytes[3] = {0, 0, 0};
  void note(int kind, size_t count) {
    ++ncoll[kind];
    nbytes[kind] += (long long)(count * sizeof(double));
  }
  // host waits (the only ones of the distributed factorization): NCCL
  // overrides them to poll for asynchronous communicator errors and a timeout
  virtual void sync(cudaStream_t st) { RUTV_CK(cudaStreamSynchronize(st)); }
  virtual void sync_event(cudaEvent_t e) { RUTV_CK(cudaEventSynchronize(e)); }
  // in-place sum over all ranks of bufs[l] (count doubles each)
  virtual void allreduce(const std::vector<double*>& bufs, size_t count, cudaStream_t st) = 0;
  // bufs[l] <- bufs[root]
  virtual void bcast(const std::vector<double*>& bufs, size_t count, int root, cudaStream_t st) = 0;
  // recv[l] = concat over ranks of send[.] (count each)
  virtual void allgather(const std::vector<double*>& send, const std::vector<double*>& recv, size_t count,
                         cudaStream_t st) = 0;
};

namespace {
__global__ void add_k(size_t n, const double* __restrict__ s, double* __restrict__ d) {
  pdl_begin();
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    d[i] += s[i];
}
void add_into(cudaStream_t st, size_t n, const double* s, double* d) {
  if (n == 0) return;
  const int blocks = (int)std::min<size_t>((n + 255) / 256, 2048);
  { ProfScope _p(st, K_MISC, 0.0); count_launch(K_MISC); launch_k(add_k, dim3(blocks), dim3(256), 0, st, n, s, d); }
  RUTV_LAUNCH_CK();
}

struct LoopComm : Comm {
  explicit LoopComm(int p) {
    P = p;
    for (int r = 0; r < p; ++r) ranks.push_back(r);
    RUTV_CK(cudaGetDevice(&dev));
  }
  void allreduce(const std::vector<double*>& bufs, size_t count, cudaStream_t st) override {
    note(0, count);
    // fixed order: ((b0 + b1) + b2) + ...  accumulated in b0, then copied out
    for (int r = 1; r < P; ++r) add_into(st, count, bufs[r], bufs[0]);
    for (int r = 1; r < P; ++r)
      if (count) RUTV_CK(cudaMemcpyAsync(bufs[r], bufs[0], count * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  void bcast(const std::vector<double*>& bufs, size_t count, int root, cudaStream_t st) override {
    note(1, count);
    for (int r = 0; r < P; ++r)
      if (r != root && count)
        RUTV_CK(cudaMemcpyAsync(bufs[r], bufs[root], count * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  void allgather(const std::vector<double*>& send, const std::vector<double*>& recv, size_t count,
                 cudaStream_t st) override {
    note(2, count);
    for (int l = 0; l < P; ++l)
      for (int r = 0; r < P; ++r)
        if (count)
          RUTV_CK(cudaMemcpyAsync(recv[l] + size_t(r) * count, send[r], count * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
  }
};

// NCCL entry points, resolved at run time (no link-time dependency on libnccl)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;  // optional
  ncclResult_t (*Abort)(ncclComm_t) = nullptr;                         // optional
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GetAsyncError = (decltype(api.GetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.Abort = (decltype(api.Abort))dlsym(h, "ncclCommAbort");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Broadcast &&
             api.AllGather;
  });
  return api;
}

struct NcclError {
  ncclResult_t r;
};
#define RUTV_NCCL(x)                            \
  do {                                          \
    ncclResult_t _r = (x);                      \
    if (_r != ncclSuccess) throw NcclError{_r}; \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  double timeout_s = 600.0;  // RANDUTV_NCCL_TIMEOUT_S at creation: a host wait longer than this aborts
  NcclComm(int p, int rank, const ncclUniqueId& id) {
    P = p;
    ranks.push_back(rank);
    RUTV_CK(cudaGetDevice(&dev));
    if (const char* e = getenv("RANDUTV_NCCL_TIMEOUT_S")) timeout_s = atof(e);
    RUTV_NCCL(nccl().CommInitRank(&c, p, id, rank));
  }
  ~NcclComm() override {
    if (c) nccl().CommDestroy(c);
  }
  ncclComm_t live() {
    if (aborted || !c) throw NcclError{ncclInvalidUsage};
    return c;
  }
  void abort_comm() {
    aborted = true;
    if (c && nccl().Abort) nccl().Abort(c);  // unblocks kernels waiting on dead peers
    c = nullptr;
  }
  // Wait until query() reports completion, polling ncclCommGetAsyncError (a
  // failed peer or network error) and the timeout (a peer that never arrives);
  // either aborts the communicator and throws -> RANDUTV_ERR_NCCL.
  template <class Q>
  void wait_for(Q query) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0;; ++it) {
      const cudaError_t e = query();
      if (e == cudaSuccess) return;
      if (e != cudaErrorNotReady) RUTV_CK(e);
      ncclResult_t ae = ncclSuccess;
      if (c && nccl().GetAsyncError && nccl().GetAsyncError(c, &ae) == ncclSuccess && ae != ncclSuccess &&
          ae != ncclInProgress) {
        abort_comm();
        throw NcclError{ae};
      }
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > timeout_s) {
        fprintf(stderr, "randutv: NCCL collective not complete after %.3g s: aborting the communicator\n", el);
        abort_comm();
        throw NcclError{ncclSystemError};
      }
      if (it > 2000) std::this_thread::sleep_for(std::chrono::microseconds(20));  // spin first, then back off
    }
  }
  void sync(cudaStream_t st) override {
    wait_for([&] { return cudaStreamQuery(st); });
  }
  void sync_event(cudaEvent_t ev) override {
    wait_for([&] { return cudaEventQuery(ev); });
  }
  void allreduce(const std::vector<double*>& bufs, size_t count, cudaStream_t st) override {
    note(0, count);
    if (count) RUTV_NCCL(nccl().AllReduce(bufs[0], bufs[0], count, ncclFloat64, ncclSum, live(), st));
  }
  void bcast(const std::vector<double*>& bufs, size_t count, int root, cudaStream_t st) override {
    note(1, count);
    if (count) RUTV_NCCL(nccl().Broadcast(bufs[0], bufs[0], count, ncclFloat64, root, live(), st));
  }
  void allgather(const std::vector<double*>& send, const std::vector<double*>& recv, size_t count,
                 cudaStream_t st) override {
    note(2, count);
    if (count) RUTV_NCCL(nccl().AllGather(send[0], recv[0], count, ncclFloat64, live(), st));
  }
};

// ----------------------------------------------------------------------------- helper kernels
// full (global trailing order) <-> per-rank pieces of the block-cyclic rows of Y:
// global trailing row t*b + i (block j = p + t, owner r = j mod P, local block
// k = (j - first_r)/P) <-> piece r, local row k*b + i.
__global__ void gather_rows_k(int64_t nrows, int64_t cols, int64_t b, int64_t p, int P, const double* __restrict__ pieces,
                              int64_t piece_rows, double* __restrict__ full, int64_t ldf) {
  pdl_begin();
  const int64_t tot = nrows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gr = e % nrows, c = e / nrows;
    const int64_t t = gr / b, i = gr % b, j = p + t;
    const int r = int(j % P);
    const int64_t first = p + ((r - p) % P + P) % P;
    const int64_t k = (j - first) / P;
    full[gr + c * ldf] = pieces[int64_t(r) * piece_rows * cols + (k * b + i) + c * piece_rows];
  }
}
__global__ void scatter_rows_k(int64_t nrows, int64_t cols, int64_t b, int64_t p, int P, int r,
                               const double* __restrict__ full, int64_t ldf, double* __restrict__ loc, int64_t ldl) {
  pdl_begin();
  // local rows of rank r: its blocks j >= p in order
  const int64_t first = p + ((r - p) % P + P) % P;
  const int64_t tot = nrows * cols;  // nrows = global trailing rows; only rank-r rows are written
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gr = e % nrows, c = e / nrows;
    const int64_t t = gr / b, i = gr % b, j = p + t;
    if (j % P != r) continue;
    const int64_t k = (j - first) / P;
    loc[(k * b + i) + c * ldl] = full[gr + c * ldf];
  }
}
// X_loc = the rank-r columns of the rows x rows identity (block-cyclic, width b)
__global__ void cyclic_identity_k(int64_t rows, int64_t nl, int64_t b, int r, int P, double* __restrict__ X,
                                  int64_t ldx) {
  pdl_begin();
  const int64_t tot = rows * nl;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, jl = e / rows;
    const int64_t g = ((jl / b) * P + r) * b + jl % b;
    X[i + jl * ldx] = (i == g) ? 1.0 : 0.0;
  }
}
inline int grid_for_n(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 2048)); }
}  // namespace

// ----------------------------------------------------------------------------- the distributed driver
namespace {

constexpr int kDistYFlags = 16;  // per-step sketch-side CholeskyQR decision slots (reorthos, QR(Y))

struct RankWork {
  // shapes: m rows; nl = local columns
  double *G, *Y, *Y2, *Z, *P, *P2, *S, *S2, *pack, *q1, *small, *part, *fold;
  double *Rall, *Dall, *Usall, *Vsall, *jwork;
  double *Rfin, *Dfin, *Usfin, *Vsfin, *jworkf, *Tfin, *tau, *Ttmp, *Rtmp;
  double *piece, *gath, *Yfull, *scal, *nrm;
  double *Ro, *Do, *Uso, *Vso, *jworko;  // over-sampling (R23): R of the gathered Y', its SVD
  // U, V formation (DistPlan::uv): replicated W_u / T_u / T_v of every step,
  // this rank's rows of every W_v
  double *Wu_all, *Tu_all, *Wvl_all, *Tv_all;
  int* flag;
  int* sweeps;
  int* qflags;  // optimistic CholeskyQR decision flags (device)
  int qflags_cap;
  size_t part_elems;
  QrWork qw;
};

struct DistPlan {
  int64_t m, n, b, s, nrand, nl_max, maxpiece;
  int64_t bs;  // sketch width b + p (over-sampling p, R23)
  int P;
  bool uv = false;
  std::vector<size_t> off_u, off_vl;  // per step: offsets into Wu_all (m_i x b) / Wvl_all (piece_i x b)
  size_t elems_u = 0, elems_vl = 0;
};

// rows of W_v of step p held by the rank with the most (padding of the allgather)
inline int64_t max_piece(int64_t n, int64_t b, int64_t p, int P) {
  int64_t mp = 1;
  for (int r = 0; r < P; ++r) mp = std::max(mp, local_cols(n, b, r, P) - b * blocks_before(p, r, P));
  return mp;
}

RankWork carve_rank(Arena& ar, const DistPlan& d) {
  RankWork w{};
  const int64_t m = d.m, b = d.b, nl = std::max<int64_t>(d.nl_max, 1), mx = std::max(m, d.n);
  const int64_t sb = std::max<int64_t>(d.nrand, 1), bs = d.bs;
  w.G = ar.take<double>(size_t(m) * bs);
  w.Y = ar.take<double>(size_t(nl) * bs);
  w.Y2 = ar.take<double>(size_t(nl) * bs);
  w.Z = ar.take<double>(size_t(m) * bs);
  w.P = ar.take<double>(size_t(mx) * b);  // mx: also k x n_loc scratch of the V formation (fat inputs)
  w.P2 = ar.take<double>(size_t(mx) * b);
  w.S = ar.take<double>(size_t(nl) * b);
  w.S2 = ar.take<double>(size_t(nl) * b);
  w.pack = ar.take<double>(std::max(size_t(m) * b + 2 * size_t(b) * b, size_t(bs) * bs) + 64);
  w.q1 = ar.take<double>(size_t(mx) * bs);
  w.small = ar.take<double>(small_work_elems(bs));
  w.part_elems = size_t(12) * mx * bs + size_t(148) * 32 * 1024;
  w.part = ar.take<double>(w.part_elems);
  w.fold = ar.take<double>(size_t(mx) * b);
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
  w.Tfin = ar.take<double>(size_t(b) * b);
  w.tau = ar.take<double>(size_t(bs));
  w.Ttmp = ar.take<double>(size_t(bs) * bs);
  w.Rtmp = ar.take<double>(size_t(bs) * bs);
  w.piece = ar.take<double>(size_t(d.maxpiece) * bs + 1);
  w.gath = ar.take<double>(size_t(d.P) * d.maxpiece * bs + 1);
  w.Yfull = ar.take<double>(size_t(d.n) * bs);
  if (bs > b) {
    w.Ro = ar.take<double>(size_t(bs) * bs);
    w.Do = ar.take<double>(size_t(bs));
    w.Uso = ar.take<double>(size_t(bs) * bs);
    w.Vso = ar.take<double>(size_t(bs) * bs);
    w.jworko = ar.take<double>(jacobi_work_elems(1, (int)bs));
  }
  w.scal = ar.take<double>(16);
  w.nrm = ar.take<double>(8192);
  if (d.uv) {
    w.Wu_all = ar.take<double>(d.elems_u);
    w.Tu_all = ar.take<double>(size_t(sb + 1) * b * b);
    w.Wvl_all = ar.take<double>(d.elems_vl);
    w.Tv_all = ar.take<double>(size_t(sb) * b * b);
  }
  w.flag = ar.take<int>(16);
  w.sweeps = ar.take<int>(size_t(sb) + 16);
  w.qflags_cap = int(16 * sb + 16);  // panel-QR decisions
  w.qflags = ar.take<int>(size_t(w.qflags_cap) + kDistYFlags);  // + one step's sketch-side decisions
  w.qw.part = w.part;
  w.qw.part_elems = w.part_elems;
  w.qw.sfull = ar.take<double>(size_t(32) * bs);
  w.qw.s2 = ar.take<double>(size_t(32) * bs);
  w.qw.z = ar.take<double>(size_t(32) * bs);
  w.qw.q1 = w.q1;
  w.qw.q1_elems = size_t(mx) * bs;
  w.qw.small = w.small;
  return w;
}

DistPlan make_dist_plan(int64_t m, int64_t n, int64_t b, int P, bool uv, int64_t ovs = 0) {
  DistPlan d;
  d.uv = uv;
  d.m = m;
  d.n = n;
  d.b = b;
  d.bs = b + ovs;
  d.P = P;
  d.s = std::min(cdiv(m, b), cdiv(n, b));
  d.nrand = 0;
  for (int64_t i = 1; i <= d.s; ++i)
    if (b * i < m && b * i < n) d.nrand = i;
  d.nl_max = 0;
  for (int r = 0; r < P; ++r) d.nl_max = std::max(d.nl_max, local_cols(n, b, r, P));
  d.maxpiece = std::max<int64_t>(d.nl_max, 1);
  if (uv) {  // randomized steps, then the final (tall) block's reflectors in slot nrand
    for (int64_t si = 0; si <= d.nrand; ++si) {
      d.off_u.push_back(d.elems_u);
      d.elems_u += size_t(m - b * si) * b;
    }
    for (int64_t si = 0; si < d.nrand; ++si) {
      d.off_vl.push_back(d.elems_vl);
      d.elems_vl += size_t(max_piece(n, b, si, P)) * b;
    }
    d.elems_vl = std::max<size_t>(d.elems_vl, 1);
  }
  return d;
}

size_t dist_rank_bytes(const DistPlan& d) {
  Arena ar;
  ar.dry = true;
  carve_rank(ar, d);
  return ar.off + 4096;
}

struct LocalRank {
  int r;                 // global rank
  const double* A;
  int64_t lda;
  double* T;
  int64_t ldt;
  double *U, *V;         // shards of U (m x mloc) and V (n x nl), or NULL (T-only)
  int64_t ldu, ldv;
  int64_t nl;            // local columns
  RankWork w;
  SmallWork sw;
};

void dg(const RankWork& w, cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
        const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
        bool b_upper = false) {
  dgemm(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, w.part, w.part_elems, 0, b_upper);
}

int read_int_sync(Comm& comm, cudaStream_t st, const int* d) {
  int h = 0;
  RUTV_CK(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  comm.sync(st);
  return h;
}

class DistFactor {
 public:
  DistFactor(Comm& c, const randutv_opts& o, int64_t m, int64_t n, int64_t b, int q, uint64_t seed,
             int64_t k_stop, std::vector<LocalRank>& L, const DistPlan& plan)
      : comm(c), o(o), m(m), n(n), b(b), q(q), seed(seed), k_stop(k_stop), L(L), P(c.P), plan_(plan) {
    st = o.stream ? (cudaStream_t)o.stream : cudaStreamPerThread;
  }

  // optimistic: CholeskyQR decisions go to device flags instead of host
  // synchronisations; returns kDistRetry if any rank raised one (all ranks see
  // the allreduced verdict and retry together in the synchronous mode).
  int run(randutv_info* info, bool optimistic);
  ~DistFactor() {
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_fork2_) cudaEventDestroy(ev_fork2_);
    if (ev_join2_) cudaEventDestroy(ev_join2_);
    if (ev_yflags_) cudaEventDestroy(ev_yflags_);
    if (ev_sweep_) cudaEventDestroy(ev_sweep_);
    if (h_yflags_) cudaFreeHost(h_yflags_);
  }

 private:
  Comm& comm;
  const randutv_opts& o;
  int64_t m, n, b;
  int q;
  uint64_t seed;
  int64_t k_stop;
  std::vector<LocalRank>& L;
  int P;
  const DistPlan& plan_;
  cudaStream_t st;
  int fallbacks = 0;
  double a_fro_ = 0.0;
  bool opt_ = false;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;  // owner's right-apply overlap
  cudaEvent_t ev_fork2_ = nullptr, ev_join2_ = nullptr;  // owner's panel QR on the priority stream
  cudaEvent_t ev_yflags_ = nullptr;  // the step's sketch-side decision flags are on the host
  cudaEvent_t ev_sweep_ = nullptr;   // start of a QR chain: an SVD sweep may run beside it
  int* h_yflags_ = nullptr;          // pinned
  std::vector<int> nflags_;  // per local rank: optimistic flag slots used
  // number of steps si < s with si = r (mod P), i.e. the slot of the next owned step
  int64_t own_slot(int64_t s, int r) const { return blocks_before(s, r, P); }
  std::vector<double*> bufs(double* RankWork::*member) {
    std::vector<double*> v;
    for (auto& lr : L) v.push_back(lr.w.*member);
    return v;
  }

  // Gram of the distributed n_i x wd matrix held in `src` (local rows nt) -> W1 of
  // every rank's small workspace (allreduced), then chol_inv (redundant).
  // wd = b, or the over-sampled sketch width b + p_i (R23) with the small
  // workspace carved for that width (small_of).
  void dist_gram_chol(double* RankWork::*src, const std::vector<int64_t>& nt, int which /*1: W1, 2: W2*/,
                      int64_t wd) {
    for (size_t l = 0; l < L.size(); ++l) {  // packed wd x wd (ld wd) Gram, allreduced, then into the padded slot
      auto& lr = L[l];
      dg(lr.w, st, true, false, wd, wd, nt[l], 1.0, lr.w.*src, std::max<int64_t>(nt[l], 1), lr.w.*src,
         std::max<int64_t>(nt[l], 1), 0.0, lr.w.pack, wd);
    }
    comm.allreduce(bufs(&RankWork::pack), size_t(wd) * wd, st);
    for (auto& lr : L) {
      const SmallWork sw = small_of(lr, wd);
      copy_matrix(st, wd, wd, lr.w.pack, wd, (which == 1) ? sw.W1 : sw.W2, sw.bp);
    }
    if (which == 1)
      for (auto& lr : L) small_chol_inv(st, wd, small_of(lr, wd));
  }
  static SmallWork small_of(const LocalRank& lr, int64_t wd) { return carve_small(lr.w.small, wd); }

  // the distributed n_i x wd matrix in `src` (local rows nt) -> Yfull (n_i x wd,
  // ld n_i) on every rank: padded allgather of the row pieces
  void gather_full(int64_t p, int64_t ni, int64_t wd, double* RankWork::*src, const std::vector<int64_t>& nt) {
    const int64_t maxpiece = max_piece(n, b, p, P);
    for (size_t l = 0; l < L.size(); ++l) {
      auto& lr = L[l];
      set_zero(st, maxpiece, wd, lr.w.piece, maxpiece);
      copy_matrix(st, nt[l], wd, lr.w.*src, std::max<int64_t>(nt[l], 1), lr.w.piece, maxpiece);
    }
    comm.allgather(bufs(&RankWork::piece), bufs(&RankWork::gath), size_t(maxpiece) * wd, st);
    for (auto& lr : L) {
      ProfScope _p(st, K_MISC, 0.0);
      count_launch(K_MISC);
      launch_k(gather_rows_k, dim3(grid_for_n(ni * wd)), dim3(256), 0, st, ni, wd, b, p, P, lr.w.gath, maxpiece, lr.w.Yfull, ni);
      RUTV_LAUNCH_CK();
    }
  }

  // Over-sampling (R23; Fig. fig:stepUTVoversampling ``[Z,~,~] = svd(Y,'econ')``):
  // the distributed n_i x (b + p_i) sketch Y' in Y -> Y (local rows) = the rows
  // of Z = Q U_R(:, 1:b), with Y' = Q R and R = U_R D V_R^T computed redundantly
  // on every rank from the gathered Y' (the same kernels on the same data, so
  // every rank holds the same Z).  Householder panels: Y' after the power
  // iteration can be far too ill-conditioned for CholeskyQR.
  int dist_oversample(int64_t p, int64_t ni, int64_t wd, const std::vector<int64_t>& nt) {
    gather_full(p, ni, wd, &RankWork::Y, nt);
    for (size_t l = 0; l < L.size(); ++l) {
      auto& lr = L[l];
      QrWork qw = lr.w.qw;
      qw.mode = 1;
      int rc = panel_qr(st, ni, wd, lr.w.Yfull, ni, lr.w.Ro, wd, lr.w.tau, lr.w.Ttmp, wd, qw);
      if (rc != OK) return rc;
      thin_q(st, ni, wd, lr.w.Yfull, ni, lr.w.Ttmp, wd, lr.w.q1, ni, lr.w.Rtmp, lr.w.part, lr.w.part_elems);
      jacobi_svd_batched(st, 1, (int)wd, lr.w.Ro, wd, wd * wd, lr.w.Do, lr.w.Uso, lr.w.Vso, lr.w.jworko, nullptr);
      dg(lr.w, st, false, false, ni, b, wd, 1.0, lr.w.q1, ni, lr.w.Uso, wd, 0.0, lr.w.Yfull, ni);
      ProfScope _p(st, K_MISC, 0.0);
      count_launch(K_MISC);
      launch_k(scatter_rows_k, dim3(grid_for_n(ni * b)), dim3(256), 0, st, ni, b, b, p, P, lr.r, lr.w.Yfull, ni, lr.w.Y,
                                                          std::max<int64_t>(nt[l], 1));
      RUTV_LAUNCH_CK();
    }
    return OK;
  }

  // U = U_1 ... U_s blockdiag(Us_i), V likewise by
  // backward accumulation on each rank's column shards: a block reflector
  // acts on rows, so with W_u replicated (broadcast by the panel owner) the U
  // update is rank-local; W_v is row-distributed and is allgathered per step.
  void form_uv(int64_t steps, bool final_block, bool final_fat, int64_t r0f, int64_t mif, int64_t nif, int64_t pf);

  // Householder fallback for a distributed Y: allgather -> full Y on every rank,
  // panel QR there (redundant), then every rank takes its rows of the result.
  // mode 0: thin Q -> dst (re-orthonormalisation); mode 1: reflectors -> dst, Tv.
  // wd: column count (b; b + p_i for an over-sampled re-orthonormalization, mode 0)
  int dist_householder(int64_t p, int64_t ni, double* RankWork::*src, double* RankWork::*dst,
                       const std::vector<int64_t>& nt, int mode, double* const* Tv, int64_t wd) {
    gather_full(p, ni, wd, src, nt);
    for (size_t l = 0; l < L.size(); ++l) {
      auto& lr = L[l];
      QrWork qw = lr.w.qw;
      qw.mode = 1;
      int rc = panel_qr(st, ni, wd, lr.w.Yfull, ni, lr.w.Rtmp, wd, lr.w.tau, mode == 1 ? Tv[l] : lr.w.Ttmp, wd, qw);
      if (rc != OK) return rc;
      double* out = lr.w.Yfull;
      if (mode == 0) {  // thin Q into q1 (ni x wd), then scatter
        thin_q(st, ni, wd, lr.w.Yfull, ni, lr.w.Ttmp, wd, lr.w.q1, ni, lr.w.Rtmp, lr.w.part, lr.w.part_elems);
        out = lr.w.q1;
      }
      {
        ProfScope _p(st, K_MISC, 0.0);
        count_launch(K_MISC);
        launch_k(scatter_rows_k, dim3(grid_for_n(ni * wd)), dim3(256), 0, st, ni, wd, b, p, P, lr.r, out, ni, lr.w.*dst,
                                                             std::max<int64_t>(nt[l], 1));
        RUTV_LAUNCH_CK();
      }
    }
    ++fallbacks;
    return OK;
  }
};

constexpr int kDistRetry = 1000;

// low-priority side stream of this device for the deferred SVD chunks
cudaStream_t dist_side_stream() {
  static cudaStream_t streams[64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) {
    int least = 0, greatest = 0;
    RUTV_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    RUTV_CK(cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, least));
  }
  return streams[dev];
}

// highest-priority stream for the owner's panel QR (see driver.cu priority_stream)
cudaStream_t dist_priority_stream() {
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

// low-priority side stream for the owner's trailing right-apply update
cudaStream_t dist_update_stream() {
  static cudaStream_t streams[64] = {};
  int dev = 0;
  RUTV_CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) {
    int least = 0, greatest = 0;
    RUTV_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    RUTV_CK(cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, least));
  }
  return streams[dev];
}

int DistFactor::run(randutv_info* info, bool optimistic) {
  const bool reortho = (o.no_reortho == 0);
  const int64_t s = std::min(cdiv(m, b), cdiv(n, b));
  const int bp = small_pad(b);
  opt_ = optimistic && o.qr_mode == 0;
  nflags_.assign(L.size(), 0);
  fallbacks = 0;
  if (!ev_fork_) RUTV_CK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  if (!ev_join_) RUTV_CK(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  if (!ev_fork2_) RUTV_CK(cudaEventCreateWithFlags(&ev_fork2_, cudaEventDisableTiming));
  if (!ev_join2_) RUTV_CK(cudaEventCreateWithFlags(&ev_join2_, cudaEventDisableTiming));
  if (!ev_yflags_) RUTV_CK(cudaEventCreateWithFlags(&ev_yflags_, cudaEventDisableTiming));
  if (!ev_sweep_) RUTV_CK(cudaEventCreateWithFlags(&ev_sweep_, cudaEventDisableTiming));
  if (!h_yflags_) RUTV_CK(cudaMallocHost(&h_yflags_, sizeof(int) * kDistYFlags));

  // ---- T <- A, ||A||_F^2 and the non-finite flag (allreduced)
  for (auto& lr : L) {
    RUTV_CK(cudaMemsetAsync(lr.w.flag, 0, sizeof(int), st));
    if (lr.nl > 0) {
      copy_norm_check(st, m, lr.nl, lr.A, lr.lda, lr.T, lr.ldt, lr.w.nrm, lr.w.scal, lr.w.flag);
    } else {
      RUTV_CK(cudaMemsetAsync(lr.w.scal, 0, sizeof(double), st));
    }
  }
  {
    // pack [sum of squares, non-finite flag, T aliases A] and allreduce
    for (auto& lr : L) {
      RUTV_CK(cudaMemcpyAsync(lr.w.pack, lr.w.scal, sizeof(double), cudaMemcpyDeviceToDevice, st));
      int hf = read_int_sync(comm, st, lr.w.flag);
      double fv[2] = {hf ? 1.0 : 0.0, 0.0};
      if (lr.nl > 0) {  // an in-place factorization cannot be redone from A
        const char* a0 = (const char*)lr.A;
        const char* a1 = a0 + sizeof(double) * (size_t(lr.lda) * (lr.nl - 1) + m);
        const char* t0 = (const char*)lr.T;
        const char* t1 = t0 + sizeof(double) * (size_t(lr.ldt) * (lr.nl - 1) + m);
        fv[1] = (t0 < a1 && a0 < t1) ? 1.0 : 0.0;
      }
      RUTV_CK(cudaMemcpyAsync(lr.w.pack + 1, fv, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
      comm.sync(st);
    }
    comm.allreduce(bufs(&RankWork::pack), 3, st);
    double h[3];
    RUTV_CK(cudaMemcpyAsync(h, L[0].w.pack, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    comm.sync(st);
    if (h[1] != 0.0) return RANDUTV_ERR_NONFINITE;
    a_fro_ = std::sqrt(h[0]);
    if (h[2] != 0.0) opt_ = false;
  }

  int64_t steps = 0, k_done = 0;
  bool final_block = false, final_fat = false;
  int64_t r0f = 0, mif = 0, nif = 0, pf = 0;
  std::vector<int64_t> nt(L.size()), c0(L.size());

  // Deferred b x b SVDs (R11 is on every rank) in chunks of 8 steps on a
  // low-priority side stream, as in the single-GPU driver (R13).
  constexpr int64_t kSvdChunk = 8;
  const bool svd_side = jacobi_single_launch((int)b);
  cudaStream_t side = svd_side ? dist_side_stream() : nullptr;
  struct SvdChunk {
    int64_t s0, s1;
    cudaEvent_t done;
  };
  std::vector<SvdChunk> chunks;
  std::vector<cudaEvent_t> evs;
  int64_t svd_done = 0;
  // incremental SVDs (k <= 256): as in the single-GPU driver, a chunk
  // advances one sweep at the start of each QR chain of the following steps
  const bool svd_incr = svd_side && jacobi_incremental((int)b);
  struct ActiveChunk {
    int64_t s0 = 0, s1 = 0;
    bool on = false;
  } active;
  auto own_range = [&](const LocalRank& lr, int64_t s0, int64_t s1, int64_t& j0, int64_t& j1) {
    j0 = own_slot(s0, lr.r);  // this rank's own blocks: steps si = r (mod P), slot j = si / P
    j1 = own_slot(s1, lr.r);
  };
  auto finish_active = [&]() {
    if (!active.on) return;
    for (auto& lr : L) {
      int64_t j0, j1;
      own_range(lr, active.s0, active.s1, j0, j1);
      if (j1 > j0)
        jacobi_end(side, (int)(j1 - j0), (int)b, lr.w.jwork + jacobi_work_elems((int)j0, (int)b),
                   lr.w.Dall + j0 * b, lr.w.Usall + size_t(j0) * b * b, lr.w.Vsall + size_t(j0) * b * b,
                   lr.w.sweeps + j0);
    }
    cudaEvent_t done;
    RUTV_CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    evs.push_back(done);
    RUTV_CK(cudaEventRecord(done, side));
    chunks.push_back({active.s0, active.s1, done});
    active.on = false;
  };
  auto svd_sweep_here = [&]() {
    if (!active.on) return;
    RUTV_CK(cudaEventRecord(ev_sweep_, st));
    RUTV_CK(cudaStreamWaitEvent(side, ev_sweep_, 0));
    for (auto& lr : L) {
      int64_t j0, j1;
      own_range(lr, active.s0, active.s1, j0, j1);
      if (j1 > j0) jacobi_sweeps(side, (int)(j1 - j0), (int)b, lr.w.jwork + jacobi_work_elems((int)j0, (int)b), 1);
    }
  };
  auto launch_svd_chunk = [&]() {
    if (steps <= svd_done) return;
    cudaEvent_t fork;
    RUTV_CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    evs.push_back(fork);
    RUTV_CK(cudaEventRecord(fork, st));
    RUTV_CK(cudaStreamWaitEvent(side, fork, 0));
    const int64_t s0 = svd_done, s1 = steps;
    if (svd_incr) {
      finish_active();
      for (auto& lr : L) {
        int64_t j0, j1;
        own_range(lr, s0, s1, j0, j1);
        if (j1 > j0)
          jacobi_begin(side, (int)(j1 - j0), (int)b, lr.w.Rall + size_t(j0 * P + lr.r) * b * b, b,
                       int64_t(P) * b * b, lr.w.jwork + jacobi_work_elems((int)j0, (int)b));
      }
      active.s0 = s0;
      active.s1 = s1;
      active.on = true;
    } else {
      for (auto& lr : L) {
        int64_t j0, j1;
        own_range(lr, s0, s1, j0, j1);
        if (j1 > j0)
          jacobi_svd_batched(side, (int)(j1 - j0), (int)b, lr.w.Rall + size_t(j0 * P + lr.r) * b * b, b,
                             int64_t(P) * b * b, lr.w.Dall + j0 * b, lr.w.Usall + size_t(j0) * b * b,
                             lr.w.Vsall + size_t(j0) * b * b, lr.w.jwork + jacobi_work_elems((int)j0, (int)b),
                             lr.w.sweeps + j0);
      }
      cudaEvent_t done;
      RUTV_CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      evs.push_back(done);
      RUTV_CK(cudaEventRecord(done, side));
      chunks.push_back({s0, s1, done});
    }
    svd_done = steps;
  };
  auto drop_events = [&]() {
    if (side) RUTV_CK(cudaStreamSynchronize(side));
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    evs.clear();
  };

  for (int64_t i = 1; i <= s; ++i) {
    const int64_t p = i - 1, r0 = b * p;
    if (k_stop > 0 && r0 >= k_stop) break;
    const int64_t mi = m - r0, ni = n - r0;
    const int owner = int(p % P);
    for (size_t l = 0; l < L.size(); ++l) {
      c0[l] = b * blocks_before(p, L[l].r, P);
      nt[l] = L[l].nl - c0[l];
    }
    if (b * i < m && b * i < n) {
      const int64_t si = p;
      // Sketch, QR(Y) and the partial P = T W_v touch no part of T: the sketch
      // side's CholeskyQR decisions are read per step while the P GEMM runs,
      // and a failure redoes only this step's part with synchronous decisions
      // (Householder fallback) on every rank alike.
      std::vector<double*> Tv(L.size());
      int lam_err = OK;
      auto sketch_qr_p = [&](bool opt_y) -> int {
        int ny = 0;
        // ---- sketch; over-sampled to b + p_i columns (R23)
        const int64_t p_i = std::min<int64_t>(o.oversample, ni - b);
        const int64_t bw = b + p_i;
        set_gemm_role(C_GEMM_SKETCH);
        for (size_t l = 0; l < L.size(); ++l) {
          auto& lr = L[l];
          gaussian_fill(st, lr.w.G, m, mi, bw, seed, uint32_t(p), 0u);
          dg(lr.w, st, true, false, nt[l], bw, mi, 1.0, lr.T + r0 + c0[l] * lr.ldt, lr.ldt, lr.w.G, m, 0.0, lr.w.Y,
             std::max<int64_t>(nt[l], 1));
        }
        for (int it = 0; it < q; ++it) {
          if (reortho) {
            set_gemm_role(C_GEMM_QR);
            svd_sweep_here();
            dist_gram_chol(&RankWork::Y, nt, 1, bw);
            bool ok;
            if (opt_y && ny < kDistYFlags) {  // decision flags on the device, read after QR(Y)
              for (size_t l = 0; l < L.size(); ++l)
                reortho_flag(st, small_of(L[l], bw).stats, 1e4, L[l].w.qflags + L[l].w.qflags_cap + ny);
              ++ny;
              ok = true;
            } else {
              double h[3];
              RUTV_CK(cudaMemcpyAsync(h, small_of(L[0], bw).stats, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
              comm.sync(st);
              ok = o.qr_mode == 0 && h[0] == 0.0 && h[2] <= 1e4 * h[1];
            }
            if (ok) {
              for (size_t l = 0; l < L.size(); ++l) {
                auto& lr = L[l];
                const SmallWork sw = small_of(lr, bw);
                dg(lr.w, st, false, false, nt[l], bw, bw, 1.0, lr.w.Y, std::max<int64_t>(nt[l], 1), sw.R1i, sw.bp,
                   0.0, lr.w.Y2, std::max<int64_t>(nt[l], 1), true);
              }
            } else {
              int rc = dist_householder(p, ni, &RankWork::Y, &RankWork::Y2, nt, 0, nullptr, bw);
              if (rc != OK) { lam_err = rc; return -1; }
            }
            for (auto& lr : L) std::swap(lr.w.Y, lr.w.Y2);
            set_gemm_role(C_GEMM_SKETCH);
          }
          for (size_t l = 0; l < L.size(); ++l) {  // Z = X Y  (partial)
            auto& lr = L[l];
            dg(lr.w, st, false, false, mi, bw, nt[l], 1.0, lr.T + r0 + c0[l] * lr.ldt, lr.ldt, lr.w.Y,
               std::max<int64_t>(nt[l], 1), 0.0, lr.w.Z, mi);
          }
          comm.allreduce(bufs(&RankWork::Z), size_t(mi) * bw, st);
          for (size_t l = 0; l < L.size(); ++l) {  // Y = X^T Z
            auto& lr = L[l];
            dg(lr.w, st, true, false, nt[l], bw, mi, 1.0, lr.T + r0 + c0[l] * lr.ldt, lr.ldt, lr.w.Z, mi, 0.0,
               lr.w.Y, std::max<int64_t>(nt[l], 1));
          }
        }
        if (p_i > 0) {  // Y <- the rows of Z = Q U_R(:, 1:b) (R23)
          set_gemm_role(C_GEMM_QR);
          int rc = dist_oversample(p, ni, bw, nt);
          if (rc != OK) { lam_err = rc; return -1; }
        }
        // ---- QR(Y) -> W_v (rows distributed), T_v
        set_gemm_role(C_GEMM_QR);
        for (size_t l = 0; l < L.size(); ++l) Tv[l] = L[l].w.Tfin;  // T_v of this step
        bool qr_ok = false;
        svd_sweep_here();
        if (o.qr_mode == 0) {
          dist_gram_chol(&RankWork::Y, nt, 1, b);
          for (size_t l = 0; l < L.size(); ++l) {
            auto& lr = L[l];
            dg(lr.w, st, false, false, nt[l], b, b, 1.0, lr.w.Y, std::max<int64_t>(nt[l], 1), lr.sw.R1i, bp, 0.0,
               lr.w.q1, std::max<int64_t>(nt[l], 1), true);
          }
          // G2 = Q1^T Q1 (partial Grams) and the top b x b block of Q1 (global rows
          // 0..b-1 = the owner's first local block; the other ranks contribute
          // exact zeros, so the sum is that block bit for bit) in ONE allreduce
          for (size_t l = 0; l < L.size(); ++l) {
            auto& lr = L[l];
            const int64_t ldq = std::max<int64_t>(nt[l], 1);
            dg(lr.w, st, true, false, b, b, nt[l], 1.0, lr.w.q1, ldq, lr.w.q1, ldq, 0.0, lr.w.pack, b);
            if (lr.r == owner) copy_matrix(st, b, b, lr.w.q1, ldq, lr.w.pack + size_t(b) * b, b);
            else set_zero(st, b, b, lr.w.pack + size_t(b) * b, b);
          }
          comm.allreduce(bufs(&RankWork::pack), 2 * size_t(b) * b, st);
          for (size_t l = 0; l < L.size(); ++l) {
            auto& lr = L[l];
            copy_matrix(st, b, b, lr.w.pack, b, lr.sw.W2, lr.sw.bp);
            SmallWork sw = lr.sw;
            if (opt_y && ny < kDistYFlags) sw.flag = lr.w.qflags + lr.w.qflags_cap + ny;
            small_recon(st, b, sw, lr.w.pack + size_t(b) * b, b, lr.w.Rtmp, b, lr.w.tau, lr.w.Tfin, b, lr.w.part,
                        lr.w.part_elems);
          }
          const bool qr_flagged = opt_y && ny < kDistYFlags;
          if (qr_flagged) ++ny;
          qr_ok = qr_flagged ? true : (read_int_sync(comm, st, L[0].sw.flag) == 0);
          if (qr_ok) {
            for (size_t l = 0; l < L.size(); ++l) {
              auto& lr = L[l];
              if (nt[l] > 0)
                dg(lr.w, st, false, false, nt[l], b, b, -1.0, lr.w.q1, nt[l], lr.sw.M, bp, 0.0, lr.w.Y, nt[l], true);
              if (lr.r == owner) small_put_unit_lower(st, b, lr.sw, lr.w.Y, std::max<int64_t>(nt[l], 1));
            }
          }
        }
        if (!qr_ok) {
          int rc = dist_householder(p, ni, &RankWork::Y, &RankWork::Y2, nt, 1, Tv.data(), b);
          if (rc != OK) { lam_err = rc; return -1; }
          for (auto& lr : L) std::swap(lr.w.Y, lr.w.Y2);
        }
        if (plan_.uv)  // keep this rank's rows of W_v and T_v for the V formation
          for (size_t l = 0; l < L.size(); ++l) {
            auto& lr = L[l];
            const int64_t ldy = std::max<int64_t>(nt[l], 1);
            if (nt[l] > 0) copy_matrix(st, nt[l], b, lr.w.Y, ldy, lr.w.Wvl_all + plan_.off_vl[si], ldy);
            copy_matrix(st, b, b, Tv[l], b, lr.w.Tv_all + size_t(si) * b * b, b);
          }
        // the step's sketch-side flags (identical on every rank: computed from
        // allreduced Grams and the broadcast Q1 block) to the host, read while
        // the P GEMM below runs
        if (opt_y && ny > 0) {
          RUTV_CK(cudaMemcpyAsync(h_yflags_, L[0].w.qflags + L[0].w.qflags_cap, sizeof(int) * ny,
                                  cudaMemcpyDeviceToHost, st));
          RUTV_CK(cudaEventRecord(ev_yflags_, st));
        }
        // ---- right apply to all m rows
        set_gemm_role(C_GEMM_RIGHT);
        for (size_t l = 0; l < L.size(); ++l) {
          auto& lr = L[l];
          dg(lr.w, st, false, false, m, b, nt[l], 1.0, lr.T + c0[l] * lr.ldt, lr.ldt, lr.w.Y,
             std::max<int64_t>(nt[l], 1), 0.0, lr.w.P, m);
        }
        return opt_y ? ny : 0;
      };
      int ny = sketch_qr_p(opt_);
      if (ny < 0) return lam_err;
      if (ny > 0) {
        comm.sync_event(ev_yflags_);
        bool failed = false;
        for (int f = 0; f < ny; ++f) failed |= h_yflags_[f] != 0;
        if (failed && sketch_qr_p(false) < 0) return lam_err;
      }
      comm.allreduce(bufs(&RankWork::P), size_t(m) * b, st);
      bool joined = false;
      for (size_t l = 0; l < L.size(); ++l) {
        auto& lr = L[l];
        const int64_t ldy = std::max<int64_t>(nt[l], 1);
        dg(lr.w, st, false, false, m, b, b, 1.0, lr.w.P, m, Tv[l], b, 0.0, lr.w.P2, m);
        if (lr.r != owner) {
          dg(lr.w, st, false, true, m, nt[l], b, -1.0, lr.w.P2, m, lr.w.Y, ldy, 1.0, lr.T + c0[l] * lr.ldt, lr.ldt);
          continue;
        }
        // owner: the panel QR below reads only T(r0:m, block p) -- update it
        // first; the rest of its rank-b update runs on a low-priority side
        // stream concurrently with the panel QR (the other ranks wait for the
        // owner's broadcast), joined before the left apply.  Unsplit GEMMs.
        double* TJ = lr.T + c0[l] * lr.ldt;
        dg(lr.w, st, false, true, mi, b, b, -1.0, lr.w.P2 + r0, m, lr.w.Y, ldy, 1.0, TJ + r0, lr.ldt);
        cudaStream_t upd = dist_update_stream();
        RUTV_CK(cudaEventRecord(ev_fork_, st));
        RUTV_CK(cudaStreamWaitEvent(upd, ev_fork_, 0));
        if (r0 > 0) dgemm(upd, false, true, r0, b, b, -1.0, lr.w.P2, m, lr.w.Y, ldy, 1.0, TJ, lr.ldt, nullptr, 0);
        if (nt[l] > b)
          dgemm(upd, false, true, m, nt[l] - b, b, -1.0, lr.w.P2, m, lr.w.Y + b, ldy, 1.0, TJ + b * lr.ldt, lr.ldt,
                nullptr, 0);
        RUTV_CK(cudaEventRecord(ev_join_, upd));
        joined = true;
      }
      // ---- panel QR on the owner of block p, broadcast (W_u, T_u, R11)
      const size_t wun = size_t(mi) * b;
      for (size_t l = 0; l < L.size(); ++l) {
        auto& lr = L[l];
        if (lr.r != owner) continue;
        // the owner's panel QR runs on the highest-priority stream so that its
        // GEMMs are not queued behind the side-stream update's CTAs
        cudaStream_t hp = dist_priority_stream();
        RUTV_CK(cudaEventRecord(ev_fork2_, st));
        RUTV_CK(cudaStreamWaitEvent(hp, ev_fork2_, 0));
        double* X = lr.T + r0 + c0[l] * lr.ldt;
        double* Wu = lr.w.pack;
        copy_matrix(hp, mi, b, X, lr.ldt, Wu, mi);
        QrWork qw = lr.w.qw;
        qw.mode = o.qr_mode;
        qw.fallbacks = &fallbacks;
        if (opt_) {
          qw.dev_flags = lr.w.qflags;
          qw.flag_count = &nflags_[l];
          qw.flag_cap = lr.w.qflags_cap;
        }
        qw.orth_tol = kRFactorOrthTol;  // R11 enters T
        int rc = panel_qr(hp, mi, b, Wu, mi, Wu + wun + size_t(b) * b, b, lr.w.tau, Wu + wun, b, qw);
        if (rc != OK) return rc;
        // T(I2,J2) = R11 (replaced by D after the SVD), T(I3,J2) = 0
        copy_matrix(hp, b, b, Wu + wun + size_t(b) * b, b, X, lr.ldt);
        set_zero(hp, mi - b, b, X + b, lr.ldt);
        RUTV_CK(cudaEventRecord(ev_join2_, hp));
        RUTV_CK(cudaStreamWaitEvent(st, ev_join2_, 0));
      }
      comm.bcast(bufs(&RankWork::pack), wun + 2 * size_t(b) * b, owner, st);
      for (auto& lr : L) {  // keep R11 for the deferred SVD (and W_u, T_u for U)
        copy_matrix(st, b, b, lr.w.pack + wun + size_t(b) * b, b, lr.w.Rall + size_t(si) * b * b, b);
        if (plan_.uv) {
          copy_matrix(st, mi, b, lr.w.pack, mi, lr.w.Wu_all + plan_.off_u[si], mi);
          copy_matrix(st, b, b, lr.w.pack + wun, b, lr.w.Tu_all + size_t(si) * b * b, b);
        }
      }
      // ---- left apply to the local columns right of block p
      if (joined) RUTV_CK(cudaStreamWaitEvent(st, ev_join_, 0));
      set_gemm_role(C_GEMM_LEFT);
      for (size_t l = 0; l < L.size(); ++l) {
        auto& lr = L[l];
        const int64_t cs = c0[l] + ((lr.r == owner) ? b : 0), nc = lr.nl - cs;
        if (nc <= 0) continue;
        double* Cm = lr.T + r0 + cs * lr.ldt;
        const double* Wu = lr.w.pack;
        dg(lr.w, st, true, false, nc, b, mi, 1.0, Cm, lr.ldt, Wu, mi, 0.0, lr.w.S, nc);
        dg(lr.w, st, false, false, nc, b, b, 1.0, lr.w.S, nc, Wu + wun, b, 0.0, lr.w.S2, nc);
        dg(lr.w, st, false, true, mi, nc, b, -1.0, Wu, mi, lr.w.S2, nc, 1.0, Cm, lr.ldt);
      }
      ++steps;
      k_done = std::min(b * i, n);
      if (svd_side && steps - svd_done >= kSvdChunk) launch_svd_chunk();
      if (o.tol > 0.0) {  // ||T(I3, J3)||_F over all ranks
        const int64_t e2 = std::min(b * i, m);
        for (size_t l = 0; l < L.size(); ++l) {
          auto& lr = L[l];
          const int64_t cs = c0[l] + ((lr.r == owner) ? b : 0), nc = lr.nl - cs;
          fro2(st, m - e2, std::max<int64_t>(nc, 0), lr.T + e2 + cs * lr.ldt, lr.ldt, lr.w.nrm, lr.w.pack);
        }
        comm.allreduce(bufs(&RankWork::pack), 1, st);
        double t2 = 0.0;
        RUTV_CK(cudaMemcpyAsync(&t2, L[0].w.pack, sizeof(double), cudaMemcpyDeviceToHost, st));
        comm.sync(st);
        if (std::sqrt(t2) <= o.tol * a_fro_) break;
      }
    } else {
      // ---- final block on its owner: economical SVD of T(r0:m, r0:n)
      final_block = true;
      r0f = r0;
      mif = mi;
      nif = ni;
      pf = p;
      if (mi < ni) {
        // fat (Remark "The case m < n"): unpivoted QR of the ROWS of
        // X, X^T = Q [Rf; 0].  X^T's rows are X's columns, distributed like Y:
        // allgather them and factor redundantly on every rank (the same kernels
        // on the same data: identical reflectors W_f (in Yfull), T_f, R_f).
        final_fat = true;
        for (size_t l = 0; l < L.size(); ++l) {
          auto& lr = L[l];
          if (nt[l] > 0) transpose_matrix(st, mi, nt[l], lr.T + r0 + c0[l] * lr.ldt, lr.ldt, lr.w.Y, nt[l]);
        }
        gather_full(p, ni, mi, &RankWork::Y, nt);
        for (auto& lr : L) {
          QrWork qw = lr.w.qw;
          qw.mode = 1;
          int rc = panel_qr(st, ni, mi, lr.w.Yfull, ni, lr.w.Rfin, mi, lr.w.tau, lr.w.Tfin, mi, qw);
          if (rc != OK) return rc;
        }
        k_done = m;
        break;
      }
      for (size_t l = 0; l < L.size(); ++l) {
        auto& lr = L[l];
        if (lr.r != owner) continue;
        double* X = lr.T + r0 + c0[l] * lr.ldt;
        if (mi > ni) {
          double* Wf = lr.w.pack;
          copy_matrix(st, mi, ni, X, lr.ldt, Wf, mi);
          QrWork qw = lr.w.qw;
          qw.mode = o.qr_mode;
          qw.fallbacks = &fallbacks;
          qw.orth_tol = kRFactorOrthTol;
          int rc = panel_qr(st, mi, ni, Wf, mi, lr.w.Rfin, ni, lr.w.tau, lr.w.Tfin, ni, qw);
          if (rc != OK) return rc;
        } else {
          copy_matrix(st, ni, ni, X, lr.ldt, lr.w.Rfin, ni);
        }
      }
      if (plan_.uv && mi > ni) {  // the tall block's reflectors to every rank (U formation)
        for (auto& lr : L)
          if (lr.r == owner) copy_matrix(st, ni, ni, lr.w.Tfin, ni, lr.w.pack + size_t(mi) * ni, ni);
        comm.bcast(bufs(&RankWork::pack), size_t(mi) * ni + size_t(ni) * ni, owner, st);
        for (auto& lr : L) {
          copy_matrix(st, mi, ni, lr.w.pack, mi, lr.w.Wu_all + plan_.off_u[p], mi);
          copy_matrix(st, ni, ni, lr.w.pack + size_t(mi) * ni, ni, lr.w.Tu_all + size_t(p) * b * b, ni);
        }
      }
      k_done = n;
      break;
    }
  }

  // ---- optimistic CholeskyQR decisions: one check for the whole loop, the
  // verdict allreduced so that every rank retries (or not) together
  if (opt_) {
    for (size_t l = 0; l < L.size(); ++l) {
      double any = 0.0;
      if (nflags_[l] > 0) {
        std::vector<int> hf(nflags_[l]);
        RUTV_CK(cudaMemcpyAsync(hf.data(), L[l].w.qflags, sizeof(int) * hf.size(), cudaMemcpyDeviceToHost, st));
        comm.sync(st);
        for (int f : hf) any += f ? 1.0 : 0.0;
      }
      RUTV_CK(cudaMemcpyAsync(L[l].w.pack, &any, sizeof(double), cudaMemcpyHostToDevice, st));
      comm.sync(st);
    }
    comm.allreduce(bufs(&RankWork::pack), 1, st);
    double tot = 0.0;
    RUTV_CK(cudaMemcpyAsync(&tot, L[0].w.pack, sizeof(double), cudaMemcpyDeviceToHost, st));
    comm.sync(st);
    if (tot != 0.0) {
      drop_events();
      return kDistRetry;
    }
  }

  // ---- b x b SVDs (R11 on every rank: run redundantly) and folds
  // (P:965-968), chunk by chunk as the side-stream SVDs complete
  set_gemm_role(C_GEMM_OTHER);
  if (svd_side) {
    launch_svd_chunk();
    finish_active();
  } else if (steps > 0) {
    for (auto& lr : L) {
      const int64_t j1 = own_slot(steps, lr.r);
      if (j1 > 0)
        jacobi_svd_batched(st, (int)j1, (int)b, lr.w.Rall + size_t(lr.r) * b * b, b, int64_t(P) * b * b, lr.w.Dall,
                           lr.w.Usall, lr.w.Vsall, lr.w.jwork, lr.w.sweeps);
    }
    chunks.push_back({0, steps, nullptr});
  }
  for (const SvdChunk& ch : chunks) {
  if (ch.done) RUTV_CK(cudaStreamWaitEvent(st, ch.done, 0));
  // the chunk's Us (each computed by its step's owner) -> every rank, for the
  // row folds: ONE allreduce of the chunk's slots, every slot but the owner's
  // zero on each rank (the sum is the owner's block bit for bit)
  const int64_t cnt = ch.s1 - ch.s0;
  for (auto& lr : L) {
    set_zero(st, b, cnt * b, lr.w.pack, b);
    for (int64_t si = ch.s0; si < ch.s1; ++si)
      if (lr.r == int(si % P))
        copy_matrix(st, b, b, lr.w.Usall + size_t(si / P) * b * b, b, lr.w.pack + size_t(si - ch.s0) * b * b, b);
  }
  comm.allreduce(bufs(&RankWork::pack), size_t(cnt) * b * b, st);
  for (int64_t si = ch.s0; si < ch.s1; ++si) {
    const int64_t r0 = b * si;
    const int owner = int(si % P);
    const int64_t js = si / P;  // the owner's slot of step si
    for (size_t l = 0; l < L.size(); ++l) {
      auto& lr = L[l];
      const double* Us = lr.w.pack + size_t(si - ch.s0) * b * b;
      const double* Vs = lr.w.Vsall + size_t(js) * b * b;  // used on the owner only
      const int64_t cb = b * blocks_before(si, lr.r, P);  // local offset of block si (if owned) / of J3
      const int64_t cs = cb + ((lr.r == owner) ? b : 0), nc = lr.nl - cs;
      if (nc > 0) {  // T(I2, J3) = Us^T T(I2, J3) on the local columns
        dg(lr.w, st, true, false, b, nc, b, 1.0, Us, b, lr.T + r0 + cs * lr.ldt, lr.ldt, 0.0, lr.w.fold, b);
        copy_matrix(st, b, nc, lr.w.fold, b, lr.T + r0 + cs * lr.ldt, lr.ldt);
      }
      if (lr.r == owner) {
        write_diag_block(st, b, b, lr.w.Dall + js * b, lr.T + r0 + cb * lr.ldt, lr.ldt);
        if (r0 > 0) {  // T(I1, J2) = T(I1, J2) Vs
          dg(lr.w, st, false, false, r0, b, b, 1.0, lr.T + cb * lr.ldt, lr.ldt, Vs, b, 0.0, lr.w.fold, r0);
          copy_matrix(st, r0, b, lr.w.fold, r0, lr.T + cb * lr.ldt, lr.ldt);
        }
      }
    }
  }
  }
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  evs.clear();
  if (final_block && final_fat) {
    // T(I2, J) = [diag(D) 0];  T(I1, J) <- T(I1, J) Q blockdiag(Us, I) with
    // Q = I - W_f T_f W_f^T acting on the columns J (distributed): P = T(I1, J) W_f
    // from the local columns, allreduced (r0 x m_i), then the local rank-m_i update
    const int owner = int(pf % P);
    for (auto& lr : L) {
      const int64_t cs = b * blocks_before(pf, lr.r, P), nc = lr.nl - cs;
      if (lr.r == owner)
        jacobi_svd_batched(st, 1, (int)mif, lr.w.Rfin, mif, mif * mif, lr.w.Dfin, lr.w.Usfin, lr.w.Vsfin,
                           lr.w.jworkf, lr.w.sweeps + steps);
      if (nc > 0) set_zero(st, mif, nc, lr.T + r0f + cs * lr.ldt, lr.ldt);
      if (lr.r == owner) write_diag_block(st, mif, mif, lr.w.Dfin, lr.T + r0f + cs * lr.ldt, lr.ldt);
    }
    if (r0f > 0) {
      for (auto& lr : L) {
        const int64_t cs = b * blocks_before(pf, lr.r, P), nc = lr.nl - cs;
        if (nc > 0) {
          ProfScope _p(st, K_MISC, 0.0);
          count_launch(K_MISC);
          launch_k(scatter_rows_k, dim3(grid_for_n(nif * mif)), dim3(256), 0, st, nif, mif, b, pf, P, lr.r, lr.w.Yfull, nif, lr.w.Y, nc);
          RUTV_LAUNCH_CK();
          dg(lr.w, st, false, false, r0f, mif, nc, 1.0, lr.T + cs * lr.ldt, lr.ldt, lr.w.Y, nc, 0.0, lr.w.P, r0f);
        } else {
          set_zero(st, r0f, mif, lr.w.P, r0f);
        }
      }
      comm.allreduce(bufs(&RankWork::P), size_t(r0f) * mif, st);
      for (auto& lr : L) {
        const int64_t cs = b * blocks_before(pf, lr.r, P), nc = lr.nl - cs;
        if (nc <= 0) continue;
        dg(lr.w, st, false, false, r0f, mif, mif, 1.0, lr.w.P, r0f, lr.w.Tfin, mif, 0.0, lr.w.P2, r0f);
        dg(lr.w, st, false, true, r0f, nc, mif, -1.0, lr.w.P2, r0f, lr.w.Y, nc, 1.0, lr.T + cs * lr.ldt, lr.ldt);
        if (lr.r == owner) {  // the first m_i columns of J (block pf, on its owner): . Us
          dg(lr.w, st, false, false, r0f, mif, mif, 1.0, lr.T + cs * lr.ldt, lr.ldt, lr.w.Usfin, mif, 0.0,
             lr.w.fold, r0f);
          copy_matrix(st, r0f, mif, lr.w.fold, r0f, lr.T + cs * lr.ldt, lr.ldt);
        }
      }
    }
  } else if (final_block) {
    const int owner = int(pf % P);
    for (auto& lr : L) {
      if (lr.r != owner) continue;
      const int64_t cb = b * blocks_before(pf, lr.r, P);
      jacobi_svd_batched(st, 1, (int)nif, lr.w.Rfin, nif, nif * nif, lr.w.Dfin, lr.w.Usfin, lr.w.Vsfin, lr.w.jworkf,
                         lr.w.sweeps + steps);
      write_diag_block(st, mif, nif, lr.w.Dfin, lr.T + r0f + cb * lr.ldt, lr.ldt);
      if (r0f > 0) {
        dg(lr.w, st, false, false, r0f, nif, nif, 1.0, lr.T + cb * lr.ldt, lr.ldt, lr.w.Vsfin, nif, 0.0, lr.w.fold,
           r0f);
        copy_matrix(st, r0f, nif, lr.w.fold, r0f, lr.T + cb * lr.ldt, lr.ldt);
      }
    }
  }

  if (plan_.uv) form_uv(steps, final_block, final_fat, r0f, mif, nif, pf);

  if (info) {
    info->k_done = k_done;
    info->steps = (int32_t)steps;
    info->final_block = final_block ? 1 : 0;
    info->a_fro = a_fro_;
    info->qr_fallbacks = fallbacks;
    info->max_sweeps = 0;
    info->trailing_fro = 0.0;
    if (k_done < n) {
      for (size_t l = 0; l < L.size(); ++l) {
        auto& lr = L[l];
        const int64_t cs = b * blocks_before(cdiv(k_done, b), lr.r, P), nc = lr.nl - cs;
        fro2(st, m - k_done, std::max<int64_t>(nc, 0), lr.T + k_done + cs * lr.ldt, lr.ldt, lr.w.nrm, lr.w.pack);
      }
      comm.allreduce(bufs(&RankWork::pack), 1, st);
      double t2 = 0.0;
      RUTV_CK(cudaMemcpyAsync(&t2, L[0].w.pack, sizeof(double), cudaMemcpyDeviceToHost, st));
      info->trailing_fro = std::sqrt(t2);
    }
    comm.sync(st);
  }
  return RANDUTV_OK;
}

void DistFactor::form_uv(int64_t steps, bool final_block, bool final_fat, int64_t r0f, int64_t mif, int64_t nif,
                         int64_t pf) {
  set_gemm_role(C_GEMM_OTHER);
  for (auto& lr : L) {
    const int64_t mloc = local_cols(m, b, lr.r, P);
    if (mloc > 0) {
      ProfScope _p(st, K_MISC, 0.0);
      count_launch(K_MISC);
      launch_k(cyclic_identity_k, dim3(grid_for_n(m * mloc)), dim3(256), 0, st, m, mloc, b, lr.r, P, lr.U, lr.ldu);
      RUTV_LAUNCH_CK();
    }
    if (lr.nl > 0) {
      ProfScope _p(st, K_MISC, 0.0);
      count_launch(K_MISC);
      launch_k(cyclic_identity_k, dim3(grid_for_n(n * lr.nl)), dim3(256), 0, st, n, lr.nl, b, lr.r, P, lr.V, lr.ldv);
      RUTV_LAUNCH_CK();
    }
  }
  // X(r0:, local columns of blocks >= p) <- (I - W Tw W^T) X(r0:, ...)   (W rows x k)
  auto apply_left = [&](LocalRank& lr, double* X, int64_t ldx, int64_t ncols_loc, int64_t p, int64_t rows,
                        int64_t k, const double* W, int64_t ldw, const double* Tw, int64_t ldtw) {
    const int64_t cs = b * blocks_before(p, lr.r, P), nc = ncols_loc - cs;
    if (nc <= 0 || rows <= 0 || k <= 0) return;
    double* Xb = X + b * p + cs * ldx;
    dg(lr.w, st, true, false, k, nc, rows, 1.0, W, ldw, Xb, ldx, 0.0, lr.w.fold, k);
    dg(lr.w, st, false, false, k, nc, k, 1.0, Tw, ldtw, lr.w.fold, k, 0.0, lr.w.P, k);
    dg(lr.w, st, false, false, rows, nc, k, -1.0, W, ldw, lr.w.P, k, 1.0, Xb, ldx);
  };
  if (final_block && final_fat)  // V' <- Q_f V' (W_f, T_f replicated: the redundant QR of X^T)
    for (auto& lr : L) apply_left(lr, lr.V, lr.ldv, lr.nl, pf, nif, mif, lr.w.Yfull, nif, lr.w.Tfin, mif);
  if (final_block && mif > nif)
    for (auto& lr : L)
      apply_left(lr, lr.U, lr.ldu, local_cols(m, b, lr.r, P), pf, mif, nif, lr.w.Wu_all + plan_.off_u[pf], mif,
                 lr.w.Tu_all + size_t(pf) * b * b, nif);
  for (int64_t si = steps - 1; si >= 0; --si) {
    const int64_t r0 = b * si, mi = m - r0, ni = n - r0;
    // full W_v of step si on every rank: padded allgather of the row pieces
    const int64_t mp = max_piece(n, b, si, P);
    for (auto& lr : L) {
      const int64_t nt = lr.nl - b * blocks_before(si, lr.r, P), ldy = std::max<int64_t>(nt, 1);
      set_zero(st, mp, b, lr.w.piece, mp);
      if (nt > 0) copy_matrix(st, nt, b, lr.w.Wvl_all + plan_.off_vl[si], ldy, lr.w.piece, mp);
    }
    comm.allgather(bufs(&RankWork::piece), bufs(&RankWork::gath), size_t(mp) * b, st);
    for (auto& lr : L) {
      {
        ProfScope _p(st, K_MISC, 0.0);
        count_launch(K_MISC);
        launch_k(gather_rows_k, dim3(grid_for_n(ni * b)), dim3(256), 0, st, ni, b, b, si, P, lr.w.gath, mp, lr.w.Yfull, ni);
        RUTV_LAUNCH_CK();
      }
      apply_left(lr, lr.V, lr.ldv, lr.nl, si, ni, b, lr.w.Yfull, ni, lr.w.Tv_all + size_t(si) * b * b, b);
      apply_left(lr, lr.U, lr.ldu, local_cols(m, b, lr.r, P), si, mi, b, lr.w.Wu_all + plan_.off_u[si], mi,
                 lr.w.Tu_all + size_t(si) * b * b, b);
    }
  }
  // column folds with the small SVD factors, on the owner of each block
  auto fold_cols = [&](LocalRank& lr, double* X, int64_t rows, int64_t ldx, int64_t p, int64_t k, const double* F) {
    double* Xb = X + b * blocks_before(p, lr.r, P) * ldx;
    dg(lr.w, st, false, false, rows, k, k, 1.0, Xb, ldx, F, k, 0.0, lr.w.fold, rows);
    copy_matrix(st, rows, k, lr.w.fold, rows, Xb, ldx);
  };
  for (int64_t si = 0; si < steps; ++si)
    for (auto& lr : L) {
      if (int(si % P) != lr.r) continue;
      const int64_t js = si / P;
      fold_cols(lr, lr.U, m, lr.ldu, si, b, lr.w.Usall + size_t(js) * b * b);
      fold_cols(lr, lr.V, n, lr.ldv, si, b, lr.w.Vsall + size_t(js) * b * b);
    }
  if (final_block)
    for (auto& lr : L) {
      if (int(pf % P) != lr.r) continue;
      const int64_t kf = std::min(mif, nif);
      // fat: X = Vs [D 0] (Q blockdiag(Us, I))^T -- U takes Vs, V takes Us
      fold_cols(lr, lr.U, m, lr.ldu, pf, kf, final_fat ? lr.w.Vsfin : lr.w.Usfin);
      fold_cols(lr, lr.V, n, lr.ldv, pf, kf, final_fat ? lr.w.Usfin : lr.w.Vsfin);
    }
  (void)r0f;
}

std::mutex g_dmu;
void* g_dws[kMaxDevices] = {};        // cached workspace, per device
size_t g_dws_bytes[kMaxDevices] = {};

void* dist_ws(size_t bytes) {
  const int d = current_device();
  if (bytes > g_dws_bytes[d]) {
    if (g_dws[d]) {
      RUTV_CK(cudaDeviceSynchronize());
      cudaFree(g_dws[d]);
      g_dws[d] = nullptr;
      g_dws_bytes[d] = 0;
    }
    if (cudaMalloc(&g_dws[d], bytes) != cudaSuccess) {
      cudaGetLastError();
      g_dws[d] = nullptr;
      return nullptr;
    }
    g_dws_bytes[d] = bytes;
  }
  return g_dws[d];
}

}  // namespace
}  // namespace rutv

// ----------------------------------------------------------------------------- C ABI
struct randutv_comm {
  std::unique_ptr<rutv::Comm> c;
};

extern "C" {

int randutv_nccl_unique_id(void* id_out) {
  if (!id_out) return -1;
  auto& api = rutv::nccl();
  if (!api.ok) return RANDUTV_ERR_NCCL;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return RANDUTV_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == RANDUTV_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

int randutv_comm_init_nccl(int32_t nranks, int32_t rank, const void* id, randutv_comm** out) {
  if (nranks < 1) return -1;
  if (rank < 0 || rank >= nranks) return -2;
  if (!id) return -3;
  if (!out) return -4;
  if (!rutv::nccl().ok) return RANDUTV_ERR_NCCL;
  try {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto* h = new randutv_comm;
    h->c.reset(new rutv::NcclComm(nranks, rank, uid));
    *out = h;
    return 0;
  } catch (const rutv::NcclError&) {
    return RANDUTV_ERR_NCCL;
  } catch (const rutv::CudaError&) {
    return RANDUTV_ERR_CUDA;
  }
}

int randutv_comm_init_loopback(int32_t nranks, randutv_comm** out) {
  if (nranks < 1) return -1;
  if (!out) return -2;
  try {
    auto* h = new randutv_comm;
    h->c.reset(new rutv::LoopComm(nranks));
    *out = h;
    return 0;
  } catch (const rutv::CudaError&) {
    return RANDUTV_ERR_CUDA;
  }
}

int randutv_comm_destroy(randutv_comm* c) {
  delete c;
  return 0;
}

int randutv_comm_stats(const randutv_comm* c, long long* counts, long long* bytes) {
  if (!c) return -1;
  for (int k = 0; k < 3; ++k) {
    if (counts) counts[k] = c->c->ncoll[k];
    if (bytes) bytes[k] = c->c->nbytes[k];
  }
  return c->c->aborted ? RANDUTV_ERR_NCCL : 0;
}

int randutv_comm_local_ranks(const randutv_comm* c, int32_t* world, int32_t* ranks_out, int32_t max_ranks) {
  if (!c) return -1;
  if (world) *world = c->c->P;
  const int nl = (int)c->c->ranks.size();
  for (int i = 0; i < nl && i < max_ranks; ++i)
    if (ranks_out) ranks_out[i] = c->c->ranks[i];
  return nl;
}

int64_t randutv_dist_local_cols(int64_t n, int64_t b, int32_t rank, int32_t nranks) {
  if (n < 0 || b < 1 || nranks < 1 || rank < 0 || rank >= nranks) return -1;
  return local_cols(n, b, rank, nranks);
}

int64_t randutv_dist_global_col(int64_t local_col, int64_t b, int32_t rank, int32_t nranks) {
  if (local_col < 0 || b < 1 || nranks < 1 || rank < 0 || rank >= nranks) return -1;
  const int64_t k = local_col / b, i = local_col % b;
  return (k * nranks + rank) * b + i;
}

int randutv_factor_dist(const randutv_opts* opts, randutv_comm* comm, int64_t m, int64_t n, const double* const* A_loc,
                        const int64_t* lda_loc, int64_t b, int32_t q, uint64_t seed, int64_t k_stop,
                        double* const* U_loc, const int64_t* ldu_loc, double* const* T_loc, const int64_t* ldt_loc,
                        double* const* V_loc, const int64_t* ldv_loc, randutv_info* info) {
  if (!comm) return -2;
  if (m < 1) return -3;
  if (n < 1) return -4;
  if (!A_loc || !lda_loc) return -5;
  if (b < 1 || b > RANDUTV_MAX_B) return -7;
  if (q < 0) return -8;
  if (k_stop < 0) return -10;
  if (!T_loc || !ldt_loc) return -13;
  const bool uv = (U_loc != nullptr);
  if (uv && !ldu_loc) return -12;
  if (uv != (V_loc != nullptr) || (V_loc && !ldv_loc)) return -16;
  randutv_opts o{};
  if (opts) o = *opts;
  if (o.tol < 0 || std::isnan(o.tol) || o.qr_mode < 0 || o.qr_mode > 1 || o.oversample < 0) return -1;
  if (b + o.oversample > RANDUTV_MAX_B) return -1;
  if (b > n) b = n;
  rutv::Comm& c = *comm->c;
  if (c.aborted) return RANDUTV_ERR_NCCL;  // aborted after an error or a timeout: unusable
  const int nlr = (int)c.ranks.size();
  for (int l = 0; l < nlr; ++l) {
    const int64_t nl = local_cols(n, b, c.ranks[l], c.P);
    if (nl > 0 && (!A_loc[l] || lda_loc[l] < m)) return -5;
    if (nl > 0 && (!T_loc[l] || ldt_loc[l] < m)) return -13;
    if (uv && local_cols(m, b, c.ranks[l], c.P) > 0 && (!U_loc[l] || ldu_loc[l] < m)) return -12;
    if (uv && nl > 0 && (!V_loc[l] || ldv_loc[l] < n)) return -16;
  }
  std::lock_guard<std::mutex> lock(rutv::g_dmu);
  try {
    struct Order {  // device-side ordering after the previous library call (CallOrder, driver.cu)
      cudaStream_t st;
      explicit Order(cudaStream_t s) : st(s) { rutv::call_order_begin(st); }
      ~Order() { rutv::call_order_end(st); }
    } order(o.stream ? (cudaStream_t)o.stream : cudaStreamPerThread);
    rutv::DistPlan d = rutv::make_dist_plan(m, n, b, c.P, uv, o.oversample);
    const size_t per = rutv::dist_rank_bytes(d);
    char* ws = (char*)rutv::dist_ws(per * nlr);
    if (!ws) return RANDUTV_ERR_NOMEM;
    rutv::poison_workspace(ws, per * nlr, o.stream ? (cudaStream_t)o.stream : cudaStreamPerThread);
    std::vector<rutv::LocalRank> L(nlr);
    for (int l = 0; l < nlr; ++l) {
      auto& lr = L[l];
      lr.r = c.ranks[l];
      lr.A = A_loc[l];
      lr.lda = lda_loc[l];
      lr.T = T_loc[l];
      lr.ldt = ldt_loc[l];
      lr.U = uv ? U_loc[l] : nullptr;
      lr.V = uv ? V_loc[l] : nullptr;
      lr.ldu = uv ? ldu_loc[l] : 0;
      lr.ldv = uv ? ldv_loc[l] : 0;
      lr.nl = local_cols(n, b, lr.r, c.P);
      rutv::Arena ar;
      ar.base = ws + per * l;
      ar.size = per;
      lr.w = rutv::carve_rank(ar, d);
      lr.w.qw.mode = o.qr_mode;
      lr.sw = rutv::carve_small(lr.w.small, b);
    }
    // optimistic first (no per-panel host synchronisation; run() falls back to
    // the synchronous mode on every rank if any rank factors in place)
    rutv::DistFactor f(c, o, m, n, b, q, seed, k_stop, L, d);
    int rc = f.run(info, true);
    if (rc == rutv::kDistRetry) rc = f.run(info, false);
    return rc;
  } catch (const rutv::CudaError& e) {
    fprintf(stderr, "randutv_factor_dist: CUDA error %s at %s\n", cudaGetErrorString(e.e), e.where);
    return RANDUTV_ERR_CUDA;
  } catch (const rutv::NcclError& e) {
    fprintf(stderr, "randutv_factor_dist: NCCL error %d\n", (int)e.r);
    return RANDUTV_ERR_NCCL;
  } catch (int code) {
    return code;
  }
}

}  // extern "C"
