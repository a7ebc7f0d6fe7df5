// hgks.cu — C ABI (include/hgks.h, include/hgks_test.h) and host runtime of libhgks.so.
//
// Owns: device state buffers (double-buffered Q^n / R, Q*), the three face-flux arrays, the
// control block, the compute stream, the NCCL communicator (slab halos along z + the 8-byte
// max-allreduce of the CFL wave speed), and launch/timing instrumentation.
// Every compute step is a kernel from hgks_kernels.cuh; there is no host or CPU fallback.
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hgks.h"
#include "../../include/hgks_test.h"
#include "hgks_kernels.cuh"
#include "diag_kernels.cuh"

using namespace hgks;

#ifdef HGKS_PHASE_TIMING
extern "C" int hgks_debug_phase_cycles(unsigned long long out[4], int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
  }
  return 0;
}
#endif

namespace {

thread_local std::string g_thread_err;

struct Prof {
  bool on = false;
  bool created = false;
  cudaEvent_t ev[2 * 4096] = {};
  int nev = 0;
  int cls[4096];
  double ms[HGKS_K_COUNT] = {0};
  long long launches[HGKS_K_COUNT] = {0};
};

struct LoopGroup;

}  // namespace

struct hgks_ctx {
  hgks_params p{};
  int n[3] = {0, 0, 0};  // global
  int nzl = 0, z0 = 0;
  double h[3] = {0, 0, 0};
  bool fp32 = false;
  size_t esz = 8;
  size_t qelems = 0;     // elements of one ghosted state
  size_t nface[3] = {0, 0, 0};
  void* Q[2] = {nullptr, nullptr};
  void* Qs = nullptr;
  void* F[3] = {nullptr, nullptr, nullptr};
  void* metric = nullptr;   // per axis: jf[n+1], jg[2n], iw[n] (T), see Geo
  size_t metric_off[3][3] = {};
  double* dmetric = nullptr;  // fp64 per axis: J at the cell centres [n], cell widths [n] (diagnostics)
  double* diag_dev = nullptr; // DIAG_BLOCKS * NDIAG block partials, then NDIAG results
  double* diag_host = nullptr;  // pinned NDIAG
  double* stats_dev = nullptr;  // ny * NSTAT plane sums (hgks_plane_stats)
  double* bulk_dev = nullptr;   // 2 per update block: (sum rho dV, sum rho U dV) partials (O-27)
  // per-step diagnostic history (hgks_history_enable): NDIAG partials per update block, HIST_RB second
  // level partials, rows [cap][NDIAG] of rank-local sums and [cap][2] (t, dt)
  double *dpart = nullptr, *dpart2 = nullptr, *hist = nullptr, *hist_td = nullptr;
  int hist_cap = 0;
  long long hist_pending = 0;  // upper bound of rows written since the last read (host)
  double hist_rho0 = 1.0;
  size_t red_tmp_count = 0;
  void* FF[2] = {nullptr, nullptr};  // face fields (recon_kernel output), alternating per direction
  size_t ff_elems = 0;
  cudaStream_t s2 = nullptr;          // reconstruction stream when HGKS_RECON_OVERLAP (recon d+1 beside flux d)
  cudaStream_t sc = nullptr;          // communication stream (high priority): the z halo of each stage
  cudaEvent_t ev_in = nullptr, ev_rec[3] = {}, ev_flux[3] = {};
  cudaEvent_t ev_recA = nullptr;      // first x-sweep reconstruction: the lines of z < zA landed
  cudaEvent_t ev_xy = nullptr;        // x/y ghosts of the stage input written (halo may start)
  cudaEvent_t ev_halo = nullptr;      // z ghosts of the stage input landed
  // loopback group (params.group_key): ordering events of the halo copies and the reductions
  cudaEvent_t lb_post = nullptr, lb_done = nullptr, lb_rpost = nullptr, lb_rdone = nullptr;
  LoopGroup* grp = nullptr;
  bool flux_attr_set[2] = {false, false};  // max dynamic shared memory set for the stage-1/2 flux kernels
  bool graphs = true;                       // replay pairs of steps as CUDA graphs (run_steps_graphed)
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};  // per parity of c->cur
  long long graph_launches = 0;             // kernels in one replay (launch accounting)
  void* red_tmp = nullptr;            // loopback reduction result before the in-place write-back
  double* stage64 = nullptr;  // fp64 [5][nzl][ny][nx] staging for set/get
  // asynchronous host I/O (hgks_upload_state / commit / download / io_wait), allocated on first use:
  // an I/O stream whose copies run on the copy engines beside the step, an upload and a download buffer
  cudaStream_t sio = nullptr, sio_up = nullptr;  // downloads (device -> host) / uploads (host -> device):
                                                 // one stream per direction, so PCIe runs both at once
  double *up64 = nullptr, *down64 = nullptr;
  cudaEvent_t ev_up = nullptr, ev_upfree = nullptr, ev_packed = nullptr, ev_downdone = nullptr;
  bool up_pending = false;
  Ctl* ctl = nullptr;
  Ctl* ctl_host = nullptr;    // pinned, mapped
  Ctl* ctl_host_dev = nullptr;  // device alias of ctl_host
  int cur = 0;
  bool have_state = false;
  cudaStream_t s = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;       // reductions (compute stream s)
  ncclComm_t comm_halo = nullptr;  // z-halo send/recv (communication stream sc): a communicator of
                                   // its own (ncclCommSplit), so the two streams never share one
  hgks_halo_plan plan{};
  int dev = 0;
  int num_sms = 148;
  long long total_launches = 0;
  Prof prof;
  std::string err;
};

static int fail(hgks_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_thread_err = buf;
  return code;
}

#define CUDA_TRY(c, call)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail((c), HGKS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define NCCL_TRY(c, call)                                                                   \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess) return fail((c), HGKS_ENCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

// Wait for the compute stream.  With NCCL, poll instead of blocking so that a failed or hung peer
// surfaces as HGKS_ENCCL (ncclCommGetAsyncError, or no progress for HGKS_NCCL_TIMEOUT_S seconds,
// default 300) and the communicators are aborted, rather than blocking the caller forever.
static void abort_comms(hgks_ctx* c) {
  if (c->comm_halo) ncclCommAbort(c->comm_halo);
  if (c->comm) ncclCommAbort(c->comm);
  c->comm_halo = c->comm = nullptr;
}
static int sync_s(hgks_ctx* c) {
  if (!c->comm) {
    CUDA_TRY(c, cudaStreamSynchronize(c->s));
    return HGKS_OK;
  }
  static const double timeout_s = [] {
    const char* e = getenv("HGKS_NCCL_TIMEOUT_S");
    return e ? atof(e) : 300.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(c->s);
    if (e == cudaSuccess) return HGKS_OK;
    if (e != cudaErrorNotReady) return fail(c, HGKS_ECUDA, "stream: %s", cudaGetErrorString(e));
    for (ncclComm_t cm : {c->comm, c->comm_halo}) {
      ncclResult_t ar = ncclSuccess;
      if (cm && ncclCommGetAsyncError(cm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
        abort_comms(c);
        return fail(c, HGKS_ENCCL, "NCCL asynchronous error: %s (communicators aborted)", ncclGetErrorString(ar));
      }
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      abort_comms(c);
      return fail(c, HGKS_ENCCL, "no progress for %.0f s (a peer rank is gone?); communicators aborted", timeout_s);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}
#define SYNC_TRY(c)              \
  do {                           \
    const int rc_ = sync_s(c);   \
    if (rc_) return rc_;         \
  } while (0)

// control block -> its mapped host copy (one block, 8-byte words, made visible to the host before the
// kernel completes); the caller synchronises the stream before reading c->ctl_host
__global__ void ctl_readback_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src) {
  for (int i = threadIdx.x; i < (int)(sizeof(Ctl) / 8); i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}
static_assert(sizeof(Ctl) % 8 == 0, "Ctl copied as 8-byte words");
#define CTL_READBACK(c)                                                                                   \
  do {                                                                                                    \
    ctl_readback_kernel<<<1, 32, 0, (c)->s>>>((unsigned long long*)(c)->ctl_host_dev,                      \
                                              (const unsigned long long*)(c)->ctl);                      \
    (c)->total_launches += 1;                                                                             \
    CUDA_TRY(c, cudaGetLastError());                                                                      \
  } while (0)

// ---- instrumentation ------------------------------------------------------------------------
static void prof_begin(hgks_ctx* c, int cls, cudaStream_t st = nullptr) {
  c->prof.launches[cls] += 1;
  if (!c->prof.on || c->prof.nev >= 4096) return;
  int k = c->prof.nev;
  c->prof.cls[k] = cls;
  cudaEventRecord(c->prof.ev[2 * k], st ? st : c->s);
}
static void prof_end(hgks_ctx* c, int cls, cudaStream_t st = nullptr) {
  (void)cls;
  if (!c->prof.on || c->prof.nev >= 4096) return;
  cudaEventRecord(c->prof.ev[2 * c->prof.nev + 1], st ? st : c->s);
  c->prof.nev += 1;
}
static void prof_flush(hgks_ctx* c) {  // fold recorded events into ms[] (caller synchronised)
  for (int k = 0; k < c->prof.nev; ++k) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->prof.ev[2 * k], c->prof.ev[2 * k + 1]) == cudaSuccess) c->prof.ms[c->prof.cls[k]] += ms;
  }
  c->prof.nev = 0;
}

template <typename T>
static Geo<T> make_geo(const hgks_ctx* c) {
  Geo<T> g;
  g.n[0] = c->n[0];
  g.n[1] = c->n[1];
  g.n[2] = c->nzl;
  g.px = c->n[0] + 6;
  g.py = c->n[1] + 6;
  g.vs = (long long)g.py * g.px;
  g.plane = 5 * g.vs;
  for (int d = 0; d < 3; ++d) {
    g.h[d] = T(c->h[d]);
    g.ih[d] = T(1.0 / c->h[d]);
  }
  g.z0 = c->z0;
  g.nx_g = c->n[0];
  g.ny_g = c->n[1];
  for (int d = 0; d < 3; ++d) {
    const T* base = (const T*)c->metric;
    g.jf[d] = base + c->metric_off[d][0];
    g.jg[d] = base + c->metric_off[d][1];
    g.iw[d] = base + c->metric_off[d][2];
    g.wall[d] = c->p.bc[d] == HGKS_WALL_ISOTHERMAL;
  }
  g.T_wall = T(c->p.T_wall);
  return g;
}

// Metric tables of one axis (reading O-18), computed here in fp64: the reconstruction works in the
// uniform cell-index coordinate zeta (face j at zeta = j); J = d zeta / dx.  For HGKS_TANH,
// x(zeta) = (lo+hi)/2 + (hi-lo)/2 tanh(b (2 zeta/N - 1)) / tanh(b).
static void axis_tables(const hgks_params& p, int d, int N, int j0, int n, double* jf, double* jg, double* iw,
                        double* jc, double* wc) {
  const double lo = p.lo[d], hi = p.hi[d];
  if (p.stretch[d] != HGKS_TANH) {
    const double ih = N / (hi - lo), h = (hi - lo) / N;
    for (int j = 0; j <= n; ++j) jf[j] = ih;
    for (int j = 0; j < 2 * n; ++j) jg[j] = ih;
    for (int j = 0; j < n; ++j) iw[j] = jc[j] = ih;
    for (int j = 0; j < n; ++j) wc[j] = h;
    return;
  }
  const double b = p.stretch_b[d], tb = tanh(b), hh = 0.5 * (hi - lo), cc = 0.5 * (lo + hi);
  auto x = [&](double z) { return cc + hh * tanh(b * (2.0 * z / N - 1.0)) / tb; };
  auto J = [&](double z) {
    const double ch = cosh(b * (2.0 * z / N - 1.0));
    return 1.0 / (hh / tb * b * (2.0 / N) / (ch * ch));
  };
  const double s3 = sqrt(3.0) / 6.0;
  for (int j = 0; j <= n; ++j) jf[j] = J(j0 + j);
  for (int j = 0; j < n; ++j) {
    jg[j] = J(j0 + j + 0.5 - s3);
    jg[n + j] = J(j0 + j + 0.5 + s3);
    iw[j] = 1.0 / (x(j0 + j + 1) - x(j0 + j));
    jc[j] = J(j0 + j + 0.5);
    wc[j] = x(j0 + j + 1) - x(j0 + j);
  }
}

template <typename T>
static GasK<T> make_gas(const hgks_params& p) {
  GasK<T> g;
  g.K = T((5.0 - 3.0 * p.gamma) / (p.gamma - 1.0));  // P:202, evaluated in fp64 (O-20)
  g.gamma = T(p.gamma);
  g.mu_ref = T(p.mu_ref);
  g.T_ref = T(p.T_ref > 0 ? p.T_ref : 1.0);
  g.omega = T(p.omega);
  g.mu_law = (int)p.mu_law;
  g.prf = T(1.0 / p.prandtl - 1.0);
  g.ik3 = T(1.0 / ((5.0 - 3.0 * p.gamma) / (p.gamma - 1.0) + 3.0));
  return g;
}

static int blocks_for(long long n, int tpb) { return (int)std::min<long long>((n + tpb - 1) / tpb, 148LL * 64); }

// ---- collectives: NCCL (one process per GPU) or the in-process loopback group --------------------
// The loopback group (params.group_key) runs nranks contexts of one process, one host thread each,
// possibly on one device.  A collective = publish (pointer + event recorded on the caller's
// stream) -> host barrier -> every rank's stream waits on the peers' events and reads their
// buffers -> completion event -> host barrier -> every rank's stream waits on the peers'
// completion events, so no rank overwrites a buffer a peer is still reading.
namespace {

constexpr int LB_MAX = 16;
constexpr double LB_TIMEOUT_S = 120.0;

struct LoopGroup {
  int n = 0, joined = 0, refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  hgks_ctx* m[LB_MAX] = {};
  const void* ptr[LB_MAX] = {};
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::duration<double>(LB_TIMEOUT_S), [&] { return gen != g; });
  }
};

std::mutex g_groups_mu;
std::map<long long, LoopGroup*> g_groups;

struct LbPtrs {
  const void* p[LB_MAX];
};

// out[k] = op over ranks r = 0..n-1 (fixed order) of src_r[k]; op 0: max of u64, 1: sum of f64
__global__ void lb_reduce_kernel(LbPtrs src, int n, long long count, int op, void* out) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count; k += (long long)gridDim.x * blockDim.x) {
    if (op == 0) {
      unsigned long long v = 0;
      for (int r = 0; r < n; ++r) v = max(v, ((const unsigned long long*)src.p[r])[k]);
      ((unsigned long long*)out)[k] = v;
    } else {
      double v = 0.0;
      for (int r = 0; r < n; ++r) v += ((const double*)src.p[r])[k];
      ((double*)out)[k] = v;
    }
  }
}

}  // namespace

static int lb_barrier(hgks_ctx* c) {
  if (!c->grp->barrier()) return fail(c, HGKS_ENCCL, "loopback group: barrier timed out after %.0f s", LB_TIMEOUT_S);
  return HGKS_OK;
}

// in-place allreduce of count elements of buf (device) on stream c->s; op 0: max u64, 1: sum f64
static int coll_allreduce(hgks_ctx* c, void* buf, size_t count, int op) {
  if (c->comm) {  // NCCL (also a one-rank communicator, see hgks_create)
    NCCL_TRY(c, ncclAllReduce(buf, buf, count, op == 0 ? ncclUint64 : ncclFloat64, op == 0 ? ncclMax : ncclSum, c->comm, c->s));
    return HGKS_OK;
  }
  if (c->p.nranks == 1) return HGKS_OK;
  LoopGroup* G = c->grp;
  const int r = c->p.rank, n = c->p.nranks;
  int rc;
  CUDA_TRY(c, cudaEventRecord(c->lb_rpost, c->s));
  G->ptr[r] = buf;
  if ((rc = lb_barrier(c))) return rc;
  LbPtrs src{};
  for (int q = 0; q < n; ++q) {
    src.p[q] = G->ptr[q];
    if (q != r) CUDA_TRY(c, cudaStreamWaitEvent(c->s, G->m[q]->lb_rpost, 0));
  }
  if (count > c->red_tmp_count) return fail(c, HGKS_EINVAL, "loopback allreduce of %zu > %zu elements", count, c->red_tmp_count);
  lb_reduce_kernel<<<(int)std::min<size_t>((count + 255) / 256, 64), 256, 0, c->s>>>(src, n, (long long)count, op, c->red_tmp);
  c->total_launches += 1;
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaEventRecord(c->lb_rdone, c->s));
  if ((rc = lb_barrier(c))) return rc;
  for (int q = 0; q < n; ++q)
    if (q != r) CUDA_TRY(c, cudaStreamWaitEvent(c->s, G->m[q]->lb_rdone, 0));
  CUDA_TRY(c, cudaMemcpyAsync(buf, c->red_tmp, count * 8, cudaMemcpyDeviceToDevice, c->s));
  return HGKS_OK;
}

// z halo of the ghosted state q (elements of esz bytes) on the communication stream c->sc, which
// has already waited for the x/y ghosts (ev_xy).  Records ev_halo when the ghost planes landed.
static int coll_halo(hgks_ctx* c, void* q, size_t esz) {
  const hgks_halo_plan& pl = c->plan;
  char* b = (char*)q;
  const size_t bytes = (size_t)pl.count * esz;
  if (c->p.nranks == 1 && !c->comm) {  // periodic wrap within the slab
    CUDA_TRY(c, cudaMemcpyAsync(b + pl.recv_down * esz, b + pl.send_up * esz, bytes, cudaMemcpyDeviceToDevice, c->sc));
    CUDA_TRY(c, cudaMemcpyAsync(b + pl.recv_up * esz, b + pl.send_down * esz, bytes, cudaMemcpyDeviceToDevice, c->sc));
  } else if (c->comm) {  // (one rank: up == down == self, NCCL's self send/recv does the periodic wrap)  // one grouped send/recv per neighbour (Alg. 2; O-22: no ordering needed)
    ncclDataType_t ty = esz == 8 ? ncclFloat64 : ncclFloat32;
    NCCL_TRY(c, ncclGroupStart());
    NCCL_TRY(c, ncclSend(b + pl.send_up * esz, pl.count, ty, pl.up, c->comm_halo, c->sc));
    NCCL_TRY(c, ncclRecv(b + pl.recv_down * esz, pl.count, ty, pl.down, c->comm_halo, c->sc));
    NCCL_TRY(c, ncclSend(b + pl.send_down * esz, pl.count, ty, pl.down, c->comm_halo, c->sc));
    NCCL_TRY(c, ncclRecv(b + pl.recv_up * esz, pl.count, ty, pl.up, c->comm_halo, c->sc));
    NCCL_TRY(c, ncclGroupEnd());
  } else {  // loopback: pull both ghost chunks from the neighbours' buffers
    LoopGroup* G = c->grp;
    const int r = c->p.rank;
    int rc;
    CUDA_TRY(c, cudaEventRecord(c->lb_post, c->sc));
    G->ptr[r] = q;
    if ((rc = lb_barrier(c))) return rc;
    hgks_ctx* dn = G->m[pl.down];
    hgks_ctx* up = G->m[pl.up];
    CUDA_TRY(c, cudaStreamWaitEvent(c->sc, dn->lb_post, 0));
    CUDA_TRY(c, cudaStreamWaitEvent(c->sc, up->lb_post, 0));
    const char* bd = (const char*)G->ptr[pl.down];
    const char* bu = (const char*)G->ptr[pl.up];
    CUDA_TRY(c, cudaMemcpyAsync(b + pl.recv_down * esz, bd + dn->plan.send_up * esz, bytes, cudaMemcpyDeviceToDevice, c->sc));
    CUDA_TRY(c, cudaMemcpyAsync(b + pl.recv_up * esz, bu + up->plan.send_down * esz, bytes, cudaMemcpyDeviceToDevice, c->sc));
    CUDA_TRY(c, cudaEventRecord(c->lb_done, c->sc));
    if ((rc = lb_barrier(c))) return rc;
    CUDA_TRY(c, cudaStreamWaitEvent(c->sc, dn->lb_done, 0));
    CUDA_TRY(c, cudaStreamWaitEvent(c->sc, up->lb_done, 0));
  }
  CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->sc));
  return HGKS_OK;
}

// join (or create) the loopback group of the context's key; returns once all ranks have joined
static int lb_join(hgks_ctx* c) {
  const long long key = (long long)c->p.group_key;
  LoopGroup* G;
  {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto it = g_groups.find(key);
    if (it == g_groups.end()) {
      G = new LoopGroup();
      G->n = c->p.nranks;
      g_groups[key] = G;
    } else {
      G = it->second;
    }
    if (G->n != c->p.nranks) return fail(c, HGKS_ENCCL, "loopback group %lld: nranks %d != %d", key, c->p.nranks, G->n);
    if (G->m[c->p.rank]) return fail(c, HGKS_ENCCL, "loopback group %lld: rank %d joined twice", key, c->p.rank);
    G->m[c->p.rank] = c;
    G->refs += 1;
    c->grp = G;
  }
  int rc = lb_barrier(c);
  if (rc) return rc;
  // ranks on different devices read each other's buffers (halo copies, reduction kernel): peer access
  for (int q = 0; q < c->p.nranks; ++q) {
    const int d = G->m[q]->dev;
    if (d == c->dev) continue;
    int can = 0;
    CUDA_TRY(c, cudaDeviceCanAccessPeer(&can, c->dev, d));
    if (!can) return fail(c, HGKS_ECUDA, "loopback group: device %d cannot access peer device %d", c->dev, d);
    const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(c, HGKS_ECUDA, "peer access: %s", cudaGetErrorString(e));
    cudaGetLastError();  // clear a sticky "already enabled"
  }
  return lb_barrier(c);
}

static void lb_leave(hgks_ctx* c) {
  LoopGroup* G = c->grp;
  if (!G) return;
  std::lock_guard<std::mutex> lk(g_groups_mu);
  G->m[c->p.rank] = nullptr;
  if (--G->refs == 0) {
    for (auto it = g_groups.begin(); it != g_groups.end(); ++it)
      if (it->second == G) {
        g_groups.erase(it);
        break;
      }
    delete G;
  }
  c->grp = nullptr;
}

// ---- ghost layers: x/y periodic / wall kernels on the compute stream, then the z halo (local
// periodic copy, NCCL, or loopback) on the communication stream c->sc -> ev_halo.  With
// wait_halo the compute stream waits for the halo; flux_sweeps instead lets the interior lines
// of the first reconstruction sweep run while the halo is in flight.
template <typename T>
static int fill_ghosts(hgks_ctx* c, T* q, bool wait_halo) {
  Geo<T> g = make_geo<T>(c);
  prof_begin(c, HGKS_K_GHOST);
  if (g.wall[0] || g.wall[1]) {
    ghost_wall_kernel<T><<<blocks_for((long long)g.n[2] * 6 * std::max(g.n[0], g.n[1]), 256), 256, 0, c->s>>>(
        q, g, c->p.gamma, c->ctl);
    c->total_launches += 1;
  }
  ghost_xy_kernel<T><<<blocks_for((long long)g.n[2] * 5 * (6LL * g.px + 6LL * g.n[1]), 256), 256, 0, c->s>>>(q, g, c->ctl);
  prof_end(c, HGKS_K_GHOST);
  c->total_launches += 1;
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaEventRecord(c->ev_xy, c->s));
  CUDA_TRY(c, cudaStreamWaitEvent(c->sc, c->ev_xy, 0));
  prof_begin(c, HGKS_K_HALO, c->sc);
  int rc = coll_halo(c, q, sizeof(T));
  prof_end(c, HGKS_K_HALO, c->sc);
  if (rc) return rc;
  if (wait_halo) CUDA_TRY(c, cudaStreamWaitEvent(c->s, c->ev_halo, 0));
  return HGKS_OK;
}

// function attributes belong to the device: kept per context (one device each), not process-wide;
// also set before a graph capture (no attribute calls while capturing)
template <typename T, int STAGE>
static int set_flux_attrs(hgks_ctx* c) {
  if (c->flux_attr_set[STAGE - 1]) return HGKS_OK;
  const int sm = (int)flux_smem_bytes<T>();
  auto set = [&](auto kern) -> cudaError_t { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); };
  CUDA_TRY(c, set(flux_kernel<T, 0, STAGE, 0>));
  CUDA_TRY(c, set(flux_kernel<T, 1, STAGE, 0>));
  CUDA_TRY(c, set(flux_kernel<T, 2, STAGE, 0>));
  CUDA_TRY(c, set(flux_kernel<T, 0, STAGE, 1>));
  CUDA_TRY(c, set(flux_kernel<T, 1, STAGE, 1>));
  CUDA_TRY(c, set(flux_kernel<T, 2, STAGE, 1>));
  CUDA_TRY(c, set(flux_kernel<T, 0, STAGE, 2>));
  CUDA_TRY(c, set(flux_kernel<T, 1, STAGE, 2>));
  CUDA_TRY(c, set(flux_kernel<T, 2, STAGE, 2>));
  CUDA_TRY(c, set(flux_kernel<T, 0, STAGE, 3>));
  CUDA_TRY(c, set(flux_kernel<T, 1, STAGE, 3>));
  CUDA_TRY(c, set(flux_kernel<T, 2, STAGE, 3>));
  c->flux_attr_set[STAGE - 1] = true;
  return HGKS_OK;
}

template <typename T, int STAGE>
static int flux_sweeps(hgks_ctx* c, const T* q) {
  Geo<T> g = make_geo<T>(c);
  GasK<T> gas = make_gas<T>(c->p);
  const size_t smem = flux_smem_bytes<T>();
  int rc0;
  if ((rc0 = set_flux_attrs<T, STAGE>(c))) return rc0;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
#ifndef HGKS_RECON_OVERLAP
#define HGKS_RECON_OVERLAP 0
#endif
  // The reconstruction stream.  HGKS_RECON_OVERLAP = 1: the reconstruction sweep of the next direction
  // (memory-bound) runs on s2 while the flux sweep of the current one (FP64-bound) runs on s.
  // Measured (round 2, TGV 256^3): the flux kernel that runs beside a reconstruction slows down by that
  // reconstruction's own serial time -- three blocks per SM fill the register file, so a concurrent
  // reconstruction block always displaces flux work -- and the step rate is the same either way
  // (314.8M serial vs 314M overlapped; thin slabs 256 x 256 x 32: -1 %).  Default: the reconstruction
  // runs on the compute stream between the flux sweeps, so every flux launch runs alone and its event
  // time is its own (roofline.frac 0.571 instead of 0.546 with the reconstruction's time inside the
  // x-flux events).  The halo overlap below is unaffected: the halo runs on its own stream.
  cudaStream_t rs = HGKS_RECON_OVERLAP ? c->s2 : c->s;
  // Face-field buffer FF[pos & 1] by position in the sweep order; recon(pos 2) waits for flux(pos 0)
  // before reusing its buffer.
  // Stage input: x/y ghosts written (ev_xy, recorded by fill_ghosts on c->s); z ghosts land on
  // c->sc (ev_halo).  The first sweep's face lines of the interior z planes need no z ghost, so
  // they run while the halo is in flight; its ghost-plane lines (z = -2, -1, nz, nz+1) and every
  // later sweep wait for ev_halo.
#ifndef HGKS_SWEEP_ORDER
#define HGKS_SWEEP_ORDER 0  // 0: x, y, z ; 1: y, x, z
#endif
  const int order[3] = {HGKS_SWEEP_ORDER ? 1 : 0, HGKS_SWEEP_ORDER ? 0 : 1, 2};
  int pos_of[3];
  for (int k = 0; k < 3; ++k) pos_of[order[k]] = k;
  CUDA_TRY(c, cudaStreamWaitEvent(rs, c->ev_xy, 0));
  const int n3[3] = {nx, ny, nz};
  auto ffbuf = [&](int d) { return (T*)c->FF[pos_of[d] & 1]; };
  // Each reconstruction thread marches along the normal; on thin slabs (few lines) the march is
  // split into segments (>= 16 faces each) so a launch still has ~HGKS_RECON_THREADS threads.
#ifndef HGKS_RECON_THREADS
#define HGKS_RECON_THREADS 1500000  // measured: 1 (no split) < 6e5 < 1.5e6 ~ 3e6 ~ 8e6
#endif
  auto segments = [&](int d, long long nthreads) {
    const int nf = n3[d] + 1;
    const long long want = (HGKS_RECON_THREADS + nthreads - 1) / nthreads;
    return (int)std::max<long long>(1, std::min<long long>(want, nf / 16));
  };
  auto recon_launch = [&](int d, long long lbeg, long long lcnt, long long gap_at, long long gap) {
    T* ff = ffbuf(d);
    const LineRange lr{lbeg, lcnt, gap_at, gap};
    if (d == 1) {  // y sweep: z-fastest face-field lines, lr ranges over z
      const long long lines = lcnt * (nx + 4);
      const int nseg = segments(1, 5 * lines);
      dim3 grid((unsigned)((lcnt + RZ_Z - 1) / RZ_Z), (nx + 4 + RZ_X - 1) / RZ_X, 5 * nseg);
      recon_yz_kernel<T><<<grid, RZ_Z * RZ_X, 0, rs>>>(q, ff, g, c->ctl, lr, nseg);
    } else {
      const int nseg = segments(d, 5 * lcnt);
      const int blocks = (int)((5 * lcnt * nseg + 127) / 128);
      if (d == 0) recon_kernel<T, 0><<<blocks, 128, 0, rs>>>(q, ff, g, c->ctl, lr, nseg);
      if (d == 2) recon_kernel<T, 2><<<blocks, 128, 0, rs>>>(q, ff, g, c->ctl, lr, nseg);
    }
    c->total_launches += 1;
  };
  // The first sweep is x (t2 = z): its flux tiles whose face-field lines (z in [8j - 2, 8j + 10)) lie in
  // the lower half of the interior planes run as soon as those lines are reconstructed (ev_recA), while
  // the rest of the reconstruction (and, on several ranks, the halo) proceeds: only the first half of
  // the reconstruction is exposed before the flux starts.
#ifndef HGKS_XSPLIT
#define HGKS_XSPLIT 0  // measured: 312.3M vs 314.7M (the early x tiles run beside the rest of the reconstruction and slow down more than the hidden half saves)
#endif
  constexpr int TT2X = FluxCfg<T>::TT2;
  const int JX = (nz + TT2X - 1) / TT2X;      // t2 tiles of the x sweep
  const int zA = nz / 2;                      // interior planes reconstructed in part A
  const int J1 = (zA - 2) / TT2X;             // tiles 1 .. J1-1 need lines z <= TT2X J1 + 1 < zA
  const bool xsplit = HGKS_XSPLIT && order[0] == 0 && J1 >= 3 && J1 < JX;
  auto recon = [&](int d) -> int {
    const int n1 = n3[(d + 1) % 3], n2 = n3[(d + 2) % 3];
    const long long nl = (long long)ff_pitch(n1, (int)sizeof(T)) * (n2 + 4);
    prof_begin(c, HGKS_K_RECON, rs);
    if (pos_of[d] == 0) {  // first sweep: interior z lines, then (after the halo) the ghost-plane ones
      if (d == 1) {
        recon_launch(1, 0, nz, nz, 0);
      } else {  // x sweep lines (t1 = y, t2 = z): interior z planes are one contiguous range
        const long long w0 = ff_pitch(ny, (int)sizeof(T));
        if (xsplit) {
          recon_launch(0, 2 * w0, (long long)zA * w0, nl, 0);
          CUDA_TRY(c, cudaEventRecord(c->ev_recA, rs));
          recon_launch(0, (2LL + zA) * w0, (long long)(nz - zA) * w0, nl, 0);
        } else {
          recon_launch(0, 2 * w0, (long long)nz * w0, nl, 0);
        }
      }
      prof_end(c, HGKS_K_RECON, rs);
      CUDA_TRY(c, cudaStreamWaitEvent(rs, c->ev_halo, 0));
      prof_begin(c, HGKS_K_RECON, rs);
      if (d == 1) {
        recon_launch(1, -2, 4, 2, nz);
      } else {
        const long long w0 = ff_pitch(ny, (int)sizeof(T));
        recon_launch(0, 0, 4 * w0, 2 * w0, (long long)nz * w0);
      }
    } else if (d == 1) {
      recon_launch(1, -2, nz + 4, nz + 4, 0);
    } else {
      recon_launch(d, 0, nl, nl, 0);
    }
    prof_end(c, HGKS_K_RECON, rs);
    CUDA_TRY(c, cudaEventRecord(c->ev_rec[d], rs));
    return HGKS_OK;
  };
  auto flux = [&](int d) -> int {
    T* ff = ffbuf(d);
    const int n1 = n3[(d + 1) % 3], n2 = n3[(d + 2) % 3];
    // faces per block along the normal: at most HGKS_FLUX_TPB (measured at 256^3: 16 > 8 > 4 > 2 by
    // 0.4 % / 1 % / 2 %), chosen to balance that against the last partial wave of blocks (thin
    // slabs: 256 x 256 x 32 gives 7.35 waves at 16 faces per block, 14.7 at 8)
    constexpr int TT1 = FluxCfg<T>::TT1, TT2 = FluxCfg<T>::TT2;
    const long long tiles = (long long)((n1 + TT1 - 1) / TT1) * ((n2 + TT2 - 1) / TT2);
    const double slots = (double)c->num_sms * FluxCfg<T>::MINB;
    int fpb = HGKS_FLUX_TPB;
    double best = -1.0;
    for (int f = HGKS_FLUX_TPB; f >= 2; f /= 2) {
      const double waves = (double)(tiles * ((n3[d] + 1 + f - 1) / f)) / slots;
      const double face_eff = f >= 16 ? 1.0 : (f >= 8 ? 0.996 : (f >= 4 ? 0.99 : 0.98));
      const double eff = face_eff * waves / std::ceil(waves);
      if (eff > best + 1e-9) {
        best = eff;
        fpb = f;
      }
    }
    const dim3 grid((n1 + TT1 - 1) / TT1, (n2 + TT2 - 1) / TT2, (n3[d] + 1 + fpb - 1) / fpb);
    // flux_kernel VAR: bit 0 = Pr != 1 (heat-flux fix), bit 1 = power-law viscosity
    const int var = (c->p.prandtl != 1.0 ? 1 : 0) | (c->p.mu_law == HGKS_MU_POWER ? 2 : 0);
    const dim3 blk(FluxCfg<T>::NT);
    T* fo = (T*)c->F[d];
    auto launch = [&](unsigned ntiles2, int jofs) {
      const dim3 gr(grid.x, ntiles2, grid.z);
      switch (d * 4 + var) {
        case 0: flux_kernel<T, 0, STAGE, 0><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 1: flux_kernel<T, 0, STAGE, 1><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 2: flux_kernel<T, 0, STAGE, 2><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 3: flux_kernel<T, 0, STAGE, 3><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 4: flux_kernel<T, 1, STAGE, 0><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 5: flux_kernel<T, 1, STAGE, 1><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 6: flux_kernel<T, 1, STAGE, 2><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 7: flux_kernel<T, 1, STAGE, 3><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 8: flux_kernel<T, 2, STAGE, 0><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 9: flux_kernel<T, 2, STAGE, 1><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        case 10: flux_kernel<T, 2, STAGE, 2><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
        default: flux_kernel<T, 2, STAGE, 3><<<gr, blk, smem, c->s>>>(ff, fo, g, gas, c->ctl, jofs); break;
      }
    };
    if (d == 0 && xsplit) {
      CUDA_TRY(c, cudaStreamWaitEvent(c->s, c->ev_recA, 0));
      prof_begin(c, HGKS_K_FLUX_X + d);
      launch((unsigned)(J1 - 1), 1);  // tiles 1 .. J1-1: lines of the planes reconstructed first
      CUDA_TRY(c, cudaStreamWaitEvent(c->s, c->ev_rec[d], 0));
      launch(1u, 0);                            // tile 0 (z ghost lines)
      launch((unsigned)(JX - J1), J1);          // tiles J1 .. JX-1
      c->total_launches += 2;
    } else {
      CUDA_TRY(c, cudaStreamWaitEvent(c->s, c->ev_rec[d], 0));
      prof_begin(c, HGKS_K_FLUX_X + d);
      launch(grid.y, 0);
    }
    prof_end(c, HGKS_K_FLUX_X + d);
    CUDA_TRY(c, cudaEventRecord(c->ev_flux[d], c->s));
    return HGKS_OK;
  };
  // enqueue order matters: an event must be recorded before a wait on it is enqueued
  int rc;
  if ((rc = recon(order[0])) || (rc = recon(order[1])) || (rc = flux(order[0]))) return rc;
  CUDA_TRY(c, cudaStreamWaitEvent(rs, c->ev_flux[order[0]], 0));  // its face-field buffer is free again
  if ((rc = recon(order[2])) || (rc = flux(order[1])) || (rc = flux(order[2]))) return rc;
  c->total_launches += 3;
  CUDA_TRY(c, cudaGetLastError());
  return HGKS_OK;
}

static DiagGeo diag_geo(const hgks_ctx* c) {
  DiagGeo dg;
  const int nloc[3] = {c->n[0], c->n[1], c->nzl};
  for (int d = 0, off = 0; d < 3; off += 2 * nloc[d], ++d) {
    dg.jc[d] = c->dmetric + off;
    dg.w[d] = c->dmetric + off + nloc[d];
  }
  return dg;
}

template <typename T>
static int diagnostics_t(hgks_ctx* c) {
  Geo<T> g = make_geo<T>(c);
  T* Q = (T*)c->Q[c->cur];
  // ghosts of the current state (a halted hgks_step leaves ctl->halt set, which gates the ghost
  // kernels; hgks_step resets it on entry anyway)
  CUDA_TRY(c, cudaMemsetAsync(&c->ctl->halt, 0, sizeof(int), c->s));
  int rc;
  if ((rc = fill_ghosts<T>(c, Q, true))) return rc;
  const DiagGeo dg = diag_geo(c);
  double* out = c->diag_dev + DIAG_BLOCKS * NDIAG;
  diag_kernel<T><<<DIAG_BLOCKS, DIAG_TPB, 0, c->s>>>(Q, g, dg, c->p.gamma, c->diag_dev);
  diag_final_kernel<NDIAG><<<1, DIAG_TPB, 0, c->s>>>(c->diag_dev, DIAG_BLOCKS, out);
  c->total_launches += 2;
  CUDA_TRY(c, cudaGetLastError());
  if ((rc = coll_allreduce(c, out, NDIAG, 1))) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(c->diag_host, out, NDIAG * sizeof(double), cudaMemcpyDeviceToHost, c->s));
  SYNC_TRY(c);
  return HGKS_OK;
}

template <typename T>
static int run_steps(hgks_ctx* c, int nsteps) {
  Geo<T> g = make_geo<T>(c);
  const long long ncell = (long long)g.n[0] * g.n[1] * g.n[2];
  const int tpb = 256;
  const dim3 ugrid((g.n[0] + UPD_X - 1) / UPD_X, (g.n[1] + UPD_Y - 1) / UPD_Y, g.n[2]);
  const int ublocks = (int)(ugrid.x * ugrid.y * ugrid.z);
  const DiagGeo dg = diag_geo(c);
  const bool bulk = c->p.force_mode == HGKS_FORCE_BULK;
  int rc;
  for (int s = 0; s < nsteps; ++s) {
    T* Qn = (T*)c->Q[c->cur];
    T* R = (T*)c->Q[c->cur ^ 1];
    T* Qs = (T*)c->Qs;
    prof_begin(c, HGKS_K_DT);
    dt_kernel<<<1, 32, 0, c->s>>>(c->ctl);
    prof_end(c, HGKS_K_DT);
    c->total_launches += 1;
    // stage 1 at Q^n
    if ((rc = fill_ghosts<T>(c, Qn, false))) return rc;
    if ((rc = flux_sweeps<T, 1>(c, Qn))) return rc;
    prof_begin(c, HGKS_K_UPDATE);
    if (c->hist_cap > 0) {  // + volume diagnostics of Q^n (per-step history, NEXT-2)
      const dim3 dgrid((g.n[0] + UPDD_X - 1) / UPDD_X, (g.n[1] + UPDD_Y - 1) / UPDD_Y, g.n[2]);
      update_kernel<T, 1, true><<<dgrid, tpb, 0, c->s>>>(Qn, Qs, R, (T*)c->F[0], (T*)c->F[1], (T*)c->F[2], g, dg,
                                                           c->p.gamma, c->ctl, c->bulk_dev, c->dpart);
      hist_reduce_kernel<<<HIST_RB, DIAG_TPB, 0, c->s>>>(c->dpart, (long long)dgrid.x * dgrid.y * dgrid.z, c->dpart2,
                                                         c->ctl);
      hist_final_kernel<<<1, DIAG_TPB, 0, c->s>>>(c->dpart2, c->hist, c->hist_td, c->ctl);
      c->total_launches += 2;
    } else {
      update_kernel<T, 1><<<ugrid, tpb, 0, c->s>>>(Qn, Qs, R, (T*)c->F[0], (T*)c->F[1], (T*)c->F[2], g, dg, c->p.gamma,
                                                     c->ctl, c->bulk_dev);
    }
    prof_end(c, HGKS_K_UPDATE);
    // stage 2 at Q* (same dt and windows, O-11)
    if ((rc = fill_ghosts<T>(c, Qs, false))) return rc;
    if ((rc = flux_sweeps<T, 2>(c, Qs))) return rc;
    prof_begin(c, HGKS_K_UPDATE);
    update_kernel<T, 2><<<ugrid, tpb, 0, c->s>>>(Qn, Qs, R, (T*)c->F[0], (T*)c->F[1], (T*)c->F[2], g, dg, c->p.gamma,
                                                   c->ctl, c->bulk_dev);
    prof_end(c, HGKS_K_UPDATE);
    c->total_launches += 2;
    if (bulk) {  // bulk momentum / density of Q^{n+1} for the force controller (O-27)
      diag_final_kernel<2><<<1, DIAG_TPB, 0, c->s>>>(c->bulk_dev, ublocks, &c->ctl->bulk_new[0]);
      c->total_launches += 1;
    }
    CUDA_TRY(c, cudaGetLastError());
    // global max wave speed + global error flag; bulk sums of the force controller
    if ((rc = coll_allreduce(c, &c->ctl->red[0], 2, 0))) return rc;
    if (bulk && (rc = coll_allreduce(c, &c->ctl->bulk_new[0], 2, 1))) return rc;
    c->cur ^= 1;
  }
  commit_kernel<<<1, 32, 0, c->s>>>(c->ctl);
  c->total_launches += 1;
  CUDA_TRY(c, cudaGetLastError());
  return HGKS_OK;
}

// CUDA graph of two S2O4 steps (dt/commit, ghosts, halo, 3 reconstruction + 3 flux sweeps and the
// update of both stages, across the three streams), one per parity of the Q^n / R buffers, replayed
// for each pair of steps.  Every kernel argument is fixed for the context's lifetime (dt, force and
// halt live in the device control block), so a graph is captured once.  Single-rank contexts with
// profiling off only (NCCL and loopback collectives stay on the plain path); HGKS_GRAPHS=0 disables.
template <typename T>
static int run_steps_graphed(hgks_ctx* c, int nsteps) {
  if (!c->graphs || c->prof.on || c->p.nranks != 1 || c->comm || nsteps < 2) return run_steps<T>(c, nsteps);
  const int par = c->cur;
  int rc;
  if (!c->gexec[par]) {
    if ((rc = set_flux_attrs<T, 1>(c)) || (rc = set_flux_attrs<T, 2>(c))) return rc;
    const long long tl = c->total_launches;
    cudaGraph_t graph = nullptr;
    CUDA_TRY(c, cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
    rc = run_steps<T>(c, 2);  // enqueues (records) two steps; toggles cur twice
    const cudaError_t e = cudaStreamEndCapture(c->s, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return fail(c, HGKS_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    c->graph_launches = c->total_launches - tl;
    c->total_launches = tl;
    const cudaError_t ei = cudaGraphInstantiate(&c->gexec[par], graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return fail(c, HGKS_ECUDA, "graph instantiate: %s", cudaGetErrorString(ei));
  }
  for (int i = 0; i + 1 < nsteps; i += 2) {
    CUDA_TRY(c, cudaGraphLaunch(c->gexec[par], c->s));
    c->total_launches += c->graph_launches;
  }
  return (nsteps & 1) ? run_steps<T>(c, 1) : HGKS_OK;
}

// ---------------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------------
extern "C" {

const char* hgks_last_error(const hgks_ctx* c) { return c ? c->err.c_str() : g_thread_err.c_str(); }

size_t hgks_nccl_id_bytes(void) { return sizeof(ncclUniqueId); }

int hgks_get_nccl_id(void* out) {
  if (!out) return fail(nullptr, HGKS_EINVAL, "hgks_get_nccl_id: out is NULL");
  ncclUniqueId id;
  NCCL_TRY(nullptr, ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return HGKS_OK;
}

int hgks_slab_of(int32_t nz, int32_t rank, int32_t nranks, int32_t* z_begin, int32_t* nz_local) {
  if (nranks < 1 || rank < 0 || rank >= nranks || nz < nranks || !z_begin || !nz_local)
    return fail(nullptr, HGKS_EINVAL, "hgks_slab_of: bad arguments (nz=%d rank=%d nranks=%d)", nz, rank, nranks);
  int base = nz / nranks, rem = nz % nranks;
  *nz_local = base + (rank < rem ? 1 : 0);
  *z_begin = rank * base + (rank < rem ? rank : rem);
  return HGKS_OK;
}

int hgks_make_halo_plan(int32_t nx, int32_t ny, int32_t nz_local, int32_t rank, int32_t nranks, hgks_halo_plan* out) {
  if (!out || nx < 1 || ny < 1 || nz_local < 3 || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(nullptr, HGKS_EINVAL, "hgks_make_halo_plan: bad arguments");
  const int64_t plane = 5LL * (ny + 6) * (nx + 6);  // one ghosted z plane (all 5 variables)
  out->up = (rank + 1) % nranks;
  out->down = (rank + nranks - 1) % nranks;
  out->count = 3 * plane;
  out->send_up = (int64_t)nz_local * plane;         // interior planes nz_l-3..nz_l-1 (ghosted z = nz_l..nz_l+2)
  out->recv_down = 0;                               // ghost planes -3..-1
  out->send_down = 3 * plane;                       // interior planes 0..2
  out->recv_up = (int64_t)(nz_local + 3) * plane;   // ghost planes nz_l..nz_l+2
  return HGKS_OK;
}

int hgks_create(const hgks_params* p, hgks_ctx** out) {
  if (!out) return fail(nullptr, HGKS_EINVAL, "hgks_create: out is NULL");
  *out = nullptr;
  if (!p) return fail(nullptr, HGKS_EINVAL, "hgks_create: params is NULL");
  for (int d = 0; d < 3; ++d) {
    if (p->n[d] < 5) return fail(nullptr, HGKS_EINVAL, "n[%d]=%d < 5", d, p->n[d]);
    if (!(p->hi[d] > p->lo[d])) return fail(nullptr, HGKS_EINVAL, "hi[%d] <= lo[%d]", d, d);
    if (p->bc[d] != HGKS_PERIODIC && p->bc[d] != HGKS_WALL_ISOTHERMAL) return fail(nullptr, HGKS_EINVAL, "bc[%d] invalid", d);
    if (p->stretch[d] != HGKS_UNIFORM && p->stretch[d] != HGKS_TANH) return fail(nullptr, HGKS_EINVAL, "stretch[%d] invalid", d);
    if (d == 2 && (p->bc[d] != HGKS_PERIODIC || p->stretch[d] != HGKS_UNIFORM))
      return fail(nullptr, HGKS_EINVAL, "z is the slab axis: it must be periodic and uniform");
    if (p->stretch[d] == HGKS_TANH && !(p->stretch_b[d] > 0.0)) return fail(nullptr, HGKS_EINVAL, "stretch_b[%d] must be > 0", d);
    if (p->bc[d] == HGKS_WALL_ISOTHERMAL && !(p->T_wall > 0.0)) return fail(nullptr, HGKS_EINVAL, "T_wall must be > 0 with walls");
  }
  // walls on both in-plane axes (a duct) would need the corner ghosts mirrored along both axes;
  // the paper's wall-bounded case is the channel (walls in y only)
  if (p->bc[0] == HGKS_WALL_ISOTHERMAL && p->bc[1] == HGKS_WALL_ISOTHERMAL)
    return fail(nullptr, HGKS_EINVAL, "walls on both x and y are not supported (corner ghosts); use one wall axis");
  if (!(p->gamma > 1.0 && p->gamma <= 5.0 / 3.0 + 1e-12)) return fail(nullptr, HGKS_EINVAL, "gamma=%g outside (1, 5/3]", p->gamma);
  if (!(p->prandtl > 0.0)) return fail(nullptr, HGKS_EINVAL, "prandtl=%g must be > 0", p->prandtl);
  if (!(p->mu_ref >= 0.0)) return fail(nullptr, HGKS_EINVAL, "mu_ref < 0");
  if (p->mu_law == HGKS_MU_POWER && !(p->T_ref > 0.0)) return fail(nullptr, HGKS_EINVAL, "T_ref must be > 0 for the power law");
  if (!(p->dt_fixed > 0.0) && !(p->cfl > 0.0)) return fail(nullptr, HGKS_EINVAL, "need cfl > 0 or dt_fixed > 0");
  if (p->precision != HGKS_FP64 && p->precision != HGKS_FP32) return fail(nullptr, HGKS_EINVAL, "bad precision");
  if (p->nranks < 1 || p->rank < 0 || p->rank >= p->nranks) return fail(nullptr, HGKS_EINVAL, "bad rank/nranks");
  if (p->force_mode != HGKS_FORCE_NONE && p->force_mode != HGKS_FORCE_CONST && p->force_mode != HGKS_FORCE_BULK)
    return fail(nullptr, HGKS_EINVAL, "bad force_mode");
  if (p->force_mode != HGKS_FORCE_NONE && !std::isfinite(p->force)) return fail(nullptr, HGKS_EINVAL, "force not finite");
  if (p->nranks > 1 && !p->nccl_id && p->group_key == 0)
    return fail(nullptr, HGKS_EINVAL, "nranks > 1 needs nccl_id or a loopback group_key");
  if (p->nccl_id && p->group_key != 0) return fail(nullptr, HGKS_EINVAL, "nccl_id and group_key are exclusive");
  if (p->group_key != 0 && p->nranks > LB_MAX) return fail(nullptr, HGKS_EINVAL, "loopback group: nranks > %d", LB_MAX);
  if (p->n[2] / p->nranks < 3) return fail(nullptr, HGKS_EINVAL, "nz/nranks < 3");

  hgks_ctx* c = new hgks_ctx();
  c->p = *p;
  {
    const char* ge = getenv("HGKS_GRAPHS");
    c->graphs = !(ge && ge[0] == '0');
  }
  c->p.nccl_id = nullptr;
  for (int d = 0; d < 3; ++d) {
    c->n[d] = p->n[d];
    c->h[d] = (p->hi[d] - p->lo[d]) / p->n[d];
  }
  hgks_slab_of(p->n[2], p->rank, p->nranks, &c->z0, &c->nzl);
  c->fp32 = p->precision == HGKS_FP32;
  c->esz = c->fp32 ? 4 : 8;
  c->dev = p->device;
  auto bail = [&](int code) {
    std::string e = c->err;
    hgks_destroy(c);
    g_thread_err = e;
    return code;
  };
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    delete c;
    return fail(nullptr, HGKS_ECUDA, "no CUDA device available (libhgks has no CPU fallback)");
  }
  if (cudaSetDevice(c->dev) != cudaSuccess) {
    fail(c, HGKS_ECUDA, "cudaSetDevice(%d) failed", c->dev);
    return bail(HGKS_ECUDA);
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->dev);
  if (p->stream) {
    c->s = (cudaStream_t)p->stream;
  } else {
    // a BLOCKING stream: it orders with the legacy default stream, so a device buffer written by
    // pending legacy-stream work (torch's default stream) is complete before set_state reads it
    if (cudaStreamCreateWithFlags(&c->s, cudaStreamDefault) != cudaSuccess) {
      fail(c, HGKS_ECUDA, "stream creation failed");
      return bail(HGKS_ECUDA);
    }
    c->own_stream = true;
  }
  hgks_make_halo_plan(c->n[0], c->n[1], c->nzl, p->rank, p->nranks, &c->plan);
  c->qelems = (size_t)(c->nzl + 6) * 5 * (c->n[1] + 6) * (c->n[0] + 6);
  c->nface[0] = (size_t)(c->n[0] + 1) * c->n[1] * c->nzl;
  c->nface[1] = (size_t)c->n[0] * (c->n[1] + 1) * c->nzl;
  c->nface[2] = (size_t)c->n[0] * c->n[1] * (c->nzl + 1);
  bool ok = true;
  for (int b = 0; b < 2; ++b) ok = ok && cudaMalloc(&c->Q[b], c->qelems * c->esz) == cudaSuccess;
  ok = ok && cudaMalloc(&c->Qs, c->qelems * c->esz) == cudaSuccess;
  for (int d = 0; d < 3; ++d) ok = ok && cudaMalloc(&c->F[d], 10 * c->nface[d] * c->esz) == cudaSuccess;
  // face-field buffer: 30 values per face-line, lines include the +-2 tangential halo
  c->ff_elems = 0;
  for (int d = 0; d < 3; ++d) {
    const int n3[3] = {c->n[0], c->n[1], c->nzl};
    const int n1 = n3[(d + 1) % 3], n2 = n3[(d + 2) % 3];
    const size_t p1 = (size_t)ff_pitch(n1, (int)c->esz);
    const size_t e = 30ull * (n3[d] + 1) * p1 * (n2 + 4) + 16;  // +16: slack for 16-byte copies
    if (e > c->ff_elems) c->ff_elems = e;
  }
  for (int b = 0; b < 2; ++b) {
    ok = ok && cudaMalloc(&c->FF[b], c->ff_elems * c->esz) == cudaSuccess;
    ok = ok && cudaMemset(c->FF[b], 0, c->ff_elems * c->esz) == cudaSuccess;  // pad lines stay 0
  }
  ok = ok && cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking) == cudaSuccess;
  {
    int lo_pri = 0, hi_pri = 0;
    cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
    ok = ok && cudaStreamCreateWithPriority(&c->sc, cudaStreamNonBlocking, hi_pri) == cudaSuccess;
  }
  ok = ok && cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) == cudaSuccess;
  for (cudaEvent_t* e : {&c->ev_xy, &c->ev_halo, &c->lb_post, &c->lb_done, &c->lb_rpost, &c->lb_rdone})
    ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  c->red_tmp_count = (size_t)c->n[1] * NSTAT + NDIAG + 16;  // largest allreduce (history rows: resized)
  ok = ok && cudaMalloc(&c->red_tmp, c->red_tmp_count * 8) == cudaSuccess;
  for (int d = 0; d < 3; ++d) {
    ok = ok && cudaEventCreateWithFlags(&c->ev_rec[d], cudaEventDisableTiming) == cudaSuccess;
    if (d == 0) ok = ok && cudaEventCreateWithFlags(&c->ev_recA, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_flux[d], cudaEventDisableTiming) == cudaSuccess;
  }
  ok = ok && cudaMalloc(&c->stage64, 5 * (size_t)c->n[0] * c->n[1] * c->nzl * sizeof(double)) == cudaSuccess;
  {  // metric tables of the three axes (local extents; z uses the global plane index)
    const int nloc[3] = {c->n[0], c->n[1], c->nzl}, j0[3] = {0, 0, c->z0};
    size_t tot = 0;
    for (int d = 0; d < 3; ++d) {
      c->metric_off[d][0] = tot;
      c->metric_off[d][1] = tot + nloc[d] + 1;
      c->metric_off[d][2] = tot + nloc[d] + 1 + 2 * nloc[d];
      tot += (nloc[d] + 1) + 2 * nloc[d] + nloc[d];
    }
    double* h = (double*)malloc(tot * sizeof(double));
    const size_t dtot = 2 * ((size_t)nloc[0] + nloc[1] + nloc[2]);
    double* hd = (double*)malloc(dtot * sizeof(double));
    for (int d = 0, off = 0; d < 3; off += 2 * nloc[d], ++d)
      axis_tables(*p, d, p->n[d], j0[d], nloc[d], h + c->metric_off[d][0], h + c->metric_off[d][1], h + c->metric_off[d][2],
                  hd + off, hd + off + nloc[d]);
    ok = ok && cudaMalloc(&c->dmetric, dtot * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMemcpy(c->dmetric, hd, dtot * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
    free(hd);
    ok = ok && cudaMalloc(&c->diag_dev, (DIAG_BLOCKS + 1) * NDIAG * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMallocHost(&c->diag_host, NDIAG * sizeof(double)) == cudaSuccess;
    const size_t ublocks = (size_t)((nloc[0] + UPD_X - 1) / UPD_X) * ((nloc[1] + UPD_Y - 1) / UPD_Y) * nloc[2];
    ok = ok && cudaMalloc(&c->bulk_dev, 2 * ublocks * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMalloc(&c->stats_dev, (size_t)nloc[1] * NSTAT * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMalloc(&c->metric, tot * c->esz) == cudaSuccess;
    if (ok) {
      if (c->fp32) {
        float* f = (float*)malloc(tot * sizeof(float));
        for (size_t k = 0; k < tot; ++k) f[k] = (float)h[k];
        ok = cudaMemcpy(c->metric, f, tot * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess;
        free(f);
      } else {
        ok = cudaMemcpy(c->metric, h, tot * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
      }
    }
    free(h);
  }
  ok = ok && cudaMalloc(&c->ctl, sizeof(Ctl)) == cudaSuccess;
  // the host copy of the control block is MAPPED pinned memory: readbacks are a one-block kernel writing
  // over PCIe, not a copy-engine transfer that would queue behind an in-flight multi-100-MB state download
  ok = ok && cudaHostAlloc((void**)&c->ctl_host, sizeof(Ctl), cudaHostAllocMapped) == cudaSuccess &&
       cudaHostGetDevicePointer((void**)&c->ctl_host_dev, c->ctl_host, 0) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    fail(c, HGKS_ENOMEM, "device allocation failed");
    return bail(HGKS_ENOMEM);
  }
  // zero ghosts once (they are always overwritten before use) and the face arrays
  for (int b = 0; b < 2; ++b) cudaMemsetAsync(c->Q[b], 0, c->qelems * c->esz, c->s);
  cudaMemsetAsync(c->Qs, 0, c->qelems * c->esz, c->s);
  Ctl h{};
  h.t = 0;
  h.dt_fixed = p->dt_fixed;
  h.cfl = p->cfl;
  h.force_mode = (int)p->force_mode;
  h.f_init = h.f_prev = h.force = p->force_mode == HGKS_FORCE_NONE ? 0.0 : p->force;
  h.force_target = p->force_target;
  h.bad_cell = ~0ull;
  *c->ctl_host = h;
  if (cudaMemcpyAsync(c->ctl, c->ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice, c->s) != cudaSuccess ||
      cudaStreamSynchronize(c->s) != cudaSuccess) {
    fail(c, HGKS_ECUDA, "initialisation copy failed");
    return bail(HGKS_ECUDA);
  }
  if (p->nranks > 1 && p->group_key != 0) {
    int rc = lb_join(c);
    if (rc) return bail(rc);
  } else if (p->nccl_id) {  // nranks >= 1: with one rank a one-member communicator (self send/recv)
    ncclUniqueId id;
    memcpy(&id, p->nccl_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&c->comm, p->nranks, id, p->rank);
    if (r != ncclSuccess) {
      fail(c, HGKS_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
      c->comm = nullptr;
      return bail(HGKS_ENCCL);
    }
    r = ncclCommSplit(c->comm, 0, p->rank, &c->comm_halo, nullptr);
    if (r != ncclSuccess) {
      fail(c, HGKS_ENCCL, "ncclCommSplit (halo communicator): %s", ncclGetErrorString(r));
      c->comm_halo = nullptr;
      return bail(HGKS_ENCCL);
    }
  }
  *out = c;
  return HGKS_OK;
}

int hgks_local_extent(const hgks_ctx* c, int32_t* z_begin, int32_t* nz_local) {
  if (!c || !z_begin || !nz_local) return fail(nullptr, HGKS_EINVAL, "hgks_local_extent: NULL argument");
  *z_begin = c->z0;
  *nz_local = c->nzl;
  return HGKS_OK;
}

}  // extern "C"

template <typename T>
static int set_state_t(hgks_ctx* c, const double* src) {
  Geo<T> g = make_geo<T>(c);
  const long long ncell = (long long)g.n[0] * g.n[1] * g.n[2];
  T* Q = (T*)c->Q[c->cur];
  pack_kernel<T><<<blocks_for(5 * ncell, 256), 256, 0, c->s>>>(src, Q, g);
  int rc;
  if (c->p.force_mode != HGKS_FORCE_NONE && (rc = diagnostics_t<T>(c))) return rc;  // bulk of Q^0 (O-27)
  Ctl* h = c->ctl_host;
  CTL_READBACK(c);
  SYNC_TRY(c);
  if (c->p.force_mode != HGKS_FORCE_NONE) {  // restart the controller from this state
    const double* a = c->diag_host;
    h->volume = a[HGKS_DIAG_VOLUME];
    h->m_cur = a[HGKS_DIAG_MOM_X] / h->volume;
    h->rho_cur = a[HGKS_DIAG_MASS] / h->volume;
    h->hist = 0;
    h->f_prev = h->force = c->p.force;
  }
  h->red[0] = 0;
  h->red[1] = 0;
  h->bad_cell = ~0ull;
  h->halt = 0;
  h->pending = 0;
  CUDA_TRY(c, cudaMemcpyAsync(c->ctl, h, sizeof(Ctl), cudaMemcpyHostToDevice, c->s));
  cfl_kernel<T><<<blocks_for(ncell, 256), 256, 0, c->s>>>(Q, g, c->p.gamma, c->ctl);
  c->total_launches += 2;
  CUDA_TRY(c, cudaGetLastError());
  if ((rc = coll_allreduce(c, &c->ctl->red[0], 2, 0))) return rc;
  CTL_READBACK(c);
  SYNC_TRY(c);
  if (h->red[1]) {
    if (h->bad_cell != ~0ull) {
      unsigned long long b = h->bad_cell;
      long long i = b % c->n[0], j = (b / c->n[0]) % c->n[1], k = b / ((unsigned long long)c->n[0] * c->n[1]);
      return fail(c, HGKS_ESTATE, "invalid state (rho<=0, p<=0 or non-finite) at global cell (i,j,k)=(%lld,%lld,%lld)", i, j, k);
    }
    return fail(c, HGKS_ESTATE, "invalid state on another rank");
  }
  h->smax_cur = h->red[0];
  h->red[0] = 0;
  CUDA_TRY(c, cudaMemcpyAsync(c->ctl, h, sizeof(Ctl), cudaMemcpyHostToDevice, c->s));
  SYNC_TRY(c);
  c->have_state = true;
  return HGKS_OK;
}

extern "C" {

int hgks_set_state(hgks_ctx* c, const double* q, int on_device) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_set_state: ctx is NULL");
  if (!q) return fail(c, HGKS_EINVAL, "hgks_set_state: q is NULL");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  size_t bytes = 5 * (size_t)c->n[0] * c->n[1] * c->nzl * sizeof(double);
  CUDA_TRY(c, cudaMemcpyAsync(c->stage64, q, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->s));
  return c->fp32 ? set_state_t<float>(c, c->stage64) : set_state_t<double>(c, c->stage64);
}

// ---- asynchronous host I/O (hgks.h: hgks_upload_state .. hgks_io_wait) --------------------------
static int io_init(hgks_ctx* c) {
  if (c->sio) return HGKS_OK;
  const size_t bytes = 5 * (size_t)c->n[0] * c->n[1] * c->nzl * sizeof(double);
  bool ok = cudaStreamCreateWithFlags(&c->sio, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->sio_up, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaMalloc(&c->up64, bytes) == cudaSuccess && cudaMalloc(&c->down64, bytes) == cudaSuccess;
  for (cudaEvent_t* e : {&c->ev_up, &c->ev_upfree, &c->ev_packed, &c->ev_downdone})
    ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) return fail(c, HGKS_ENOMEM, "asynchronous I/O: stream / buffers / events could not be created");
  // nothing in flight yet: the 'buffer free' events start recorded
  CUDA_TRY(c, cudaEventRecord(c->ev_upfree, c->s));
  CUDA_TRY(c, cudaEventRecord(c->ev_downdone, c->sio));
  return HGKS_OK;
}

int hgks_upload_state(hgks_ctx* c, const double* q) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_upload_state: ctx is NULL");
  if (!q) return fail(c, HGKS_EINVAL, "hgks_upload_state: q is NULL");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  int rc;
  if ((rc = io_init(c))) return rc;
  const size_t bytes = 5 * (size_t)c->n[0] * c->n[1] * c->nzl * sizeof(double);
  CUDA_TRY(c, cudaStreamWaitEvent(c->sio_up, c->ev_upfree, 0));  // the previous commit has read up64
  CUDA_TRY(c, cudaMemcpyAsync(c->up64, q, bytes, cudaMemcpyHostToDevice, c->sio_up));
  CUDA_TRY(c, cudaEventRecord(c->ev_up, c->sio_up));
  c->up_pending = true;
  return HGKS_OK;
}

int hgks_commit_state(hgks_ctx* c) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_commit_state: ctx is NULL");
  if (!c->up_pending) return fail(c, HGKS_EINVAL, "hgks_commit_state: no hgks_upload_state pending");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  CUDA_TRY(c, cudaStreamWaitEvent(c->s, c->ev_up, 0));
  c->up_pending = false;
  const int rc = c->fp32 ? set_state_t<float>(c, c->up64) : set_state_t<double>(c, c->up64);
  CUDA_TRY(c, cudaEventRecord(c->ev_upfree, c->s));
  return rc;
}

int hgks_download_state(hgks_ctx* c, double* q) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_download_state: ctx is NULL");
  if (!q) return fail(c, HGKS_EINVAL, "hgks_download_state: q is NULL");
  if (!c->have_state) return fail(c, HGKS_EINVAL, "hgks_download_state: no state set");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  int rc;
  if ((rc = io_init(c))) return rc;
  const long long ncell = (long long)c->n[0] * c->n[1] * c->nzl;
  CUDA_TRY(c, cudaStreamWaitEvent(c->s, c->ev_downdone, 0));  // the previous D2H has read down64
  if (c->fp32) unpack_kernel<float><<<blocks_for(5 * ncell, 256), 256, 0, c->s>>>((const float*)c->Q[c->cur], c->down64, make_geo<float>(c));
  else unpack_kernel<double><<<blocks_for(5 * ncell, 256), 256, 0, c->s>>>((const double*)c->Q[c->cur], c->down64, make_geo<double>(c));
  c->total_launches += 1;
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaEventRecord(c->ev_packed, c->s));
  CUDA_TRY(c, cudaStreamWaitEvent(c->sio, c->ev_packed, 0));
  CUDA_TRY(c, cudaMemcpyAsync(q, c->down64, 5 * ncell * sizeof(double), cudaMemcpyDeviceToHost, c->sio));
  CUDA_TRY(c, cudaEventRecord(c->ev_downdone, c->sio));
  return HGKS_OK;
}

int hgks_io_wait(hgks_ctx* c) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_io_wait: ctx is NULL");
  if (!c->sio) return HGKS_OK;
  CUDA_TRY(c, cudaSetDevice(c->dev));
  CUDA_TRY(c, cudaStreamSynchronize(c->sio_up));
  CUDA_TRY(c, cudaStreamSynchronize(c->sio));
  return HGKS_OK;
}

int hgks_get_state(hgks_ctx* c, double* q, int on_device) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_get_state: ctx is NULL");
  if (!q) return fail(c, HGKS_EINVAL, "hgks_get_state: q is NULL");
  if (!c->have_state) return fail(c, HGKS_EINVAL, "hgks_get_state: no state set");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  const long long ncell = (long long)c->n[0] * c->n[1] * c->nzl;
  if (c->fp32) unpack_kernel<float><<<blocks_for(5 * ncell, 256), 256, 0, c->s>>>((const float*)c->Q[c->cur], c->stage64, make_geo<float>(c));
  else unpack_kernel<double><<<blocks_for(5 * ncell, 256), 256, 0, c->s>>>((const double*)c->Q[c->cur], c->stage64, make_geo<double>(c));
  c->total_launches += 1;
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaMemcpyAsync(q, c->stage64, 5 * ncell * sizeof(double), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->s));
  SYNC_TRY(c);
  return HGKS_OK;
}

int hgks_step(hgks_ctx* c, int32_t nsteps, double t_end, double* t_inout, double* dt_last) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_step: ctx is NULL");
  if (!t_inout) return fail(c, HGKS_EINVAL, "hgks_step: t_inout is NULL");
  if (nsteps < 0) return fail(c, HGKS_EINVAL, "hgks_step: nsteps < 0");
  if (!c->have_state) return fail(c, HGKS_EINVAL, "hgks_step: call hgks_set_state first");
  if (c->hist_cap > 0 && c->hist_pending + nsteps > c->hist_cap)
    return fail(c, HGKS_EINVAL, "hgks_step: %d steps would overflow the diagnostic history (%lld of %d rows pending; "
                "call hgks_history_read)", nsteps, c->hist_pending, c->hist_cap);
  CUDA_TRY(c, cudaSetDevice(c->dev));
  if (c->hist_cap > 0) c->hist_pending += nsteps;
  // reset per-call control: t, t_end, counters (one small H2D copy)
  Ctl* h = c->ctl_host;
  CTL_READBACK(c);
  SYNC_TRY(c);
  h->t = *t_inout;
  h->t_end = t_end;
  h->halt = 0;
  h->pending = 0;
  h->steps_done = 0;
  h->bad_cell = ~0ull;
  CUDA_TRY(c, cudaMemcpyAsync(c->ctl, h, sizeof(Ctl), cudaMemcpyHostToDevice, c->s));
  const int cur0 = c->cur;
  // With a t_end the run may halt early (every later kernel then returns at once): enqueue in
  // chunks and read the halt word between them, so a generous nsteps costs no idle launches.
  // Without t_end everything is enqueued at once (a halt then only follows an invalid state).
  const int chunk = t_end > 0.0 ? 16 : (nsteps > 0 ? nsteps : 1);
  for (int done = 0; done < nsteps || done == 0; done += chunk) {
    const int n = std::min(chunk, nsteps - done);
    int rc = c->fp32 ? run_steps_graphed<float>(c, n) : run_steps_graphed<double>(c, n);
    if (rc) return rc;
    CTL_READBACK(c);
    SYNC_TRY(c);
    if (h->halt || n <= 0) break;
  }
  c->cur = cur0 ^ (int)(h->steps_done & 1);  // buffer holding the last committed state
  *t_inout = h->t;
  if (dt_last) *dt_last = h->dt_last;
  if (h->halt == 1) {
    if (h->bad_cell != ~0ull) {
      unsigned long long b = h->bad_cell;
      long long i = b % c->n[0], j = (b / c->n[0]) % c->n[1], k = b / ((unsigned long long)c->n[0] * c->n[1]);
      return fail(c, HGKS_ESTATE, "invalid state after step %lld at global cell (i,j,k)=(%lld,%lld,%lld); rolled back",
                  h->steps_done, i, j, k);
    }
    return fail(c, HGKS_ESTATE, "invalid state after step %lld on another rank; rolled back", h->steps_done);
  }
  return HGKS_OK;
}

}  // extern "C"

extern "C" {

}  // extern "C"

// raw volume sums a[NDIAG] -> the hgks_diagnostics normalisation (O-24, O-25)
static void normalise_diag(const hgks_ctx* c, double rho0, const double* a, double* out) {
  const double vol = a[HGKS_DIAG_VOLUME], mu = c->p.mu_ref;
  for (int k = 0; k < NDIAG; ++k) out[k] = a[k];
  out[HGKS_DIAG_EK] = a[HGKS_DIAG_EK] / (rho0 * vol);
  out[HGKS_DIAG_ENSTROPHY] = a[HGKS_DIAG_ENSTROPHY] / (rho0 * vol);
  out[HGKS_DIAG_EPS_S] = mu * a[HGKS_DIAG_EPS_S] / (rho0 * vol);
  out[HGKS_DIAG_EPS_D] = 4.0 / 3.0 * mu * a[HGKS_DIAG_EPS_D] / (rho0 * vol);
  out[HGKS_DIAG_PDIL] = a[HGKS_DIAG_PDIL] / (rho0 * vol);
}

static int set_ctl_hist(hgks_ctx* c, int n, int cap) {
  Ctl* h = c->ctl_host;
  CTL_READBACK(c);
  SYNC_TRY(c);
  h->hist_n = n;
  h->hist_cap = cap;
  CUDA_TRY(c, cudaMemcpyAsync(c->ctl, h, sizeof(Ctl), cudaMemcpyHostToDevice, c->s));
  SYNC_TRY(c);
  return HGKS_OK;
}

extern "C" {

int hgks_history_enable(hgks_ctx* c, int32_t capacity, double rho0) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_history_enable: ctx is NULL");
  if (capacity < 0 || !(rho0 > 0.0)) return fail(c, HGKS_EINVAL, "hgks_history_enable: capacity < 0 or rho0 <= 0");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  SYNC_TRY(c);
  for (double** b : {&c->dpart, &c->dpart2, &c->hist, &c->hist_td}) {
    cudaFree(*b);
    *b = nullptr;
  }
  for (int b = 0; b < 2; ++b)  // captured graphs hold the update variant: recapture
    if (c->gexec[b]) {
      cudaGraphExecDestroy(c->gexec[b]);
      c->gexec[b] = nullptr;
    }
  c->hist_cap = 0;
  c->hist_pending = 0;
  c->hist_rho0 = rho0;
  if (capacity > 0) {
    const size_t ublocks = (size_t)((c->n[0] + UPDD_X - 1) / UPDD_X) * ((c->n[1] + UPDD_Y - 1) / UPDD_Y) * c->nzl;
    bool ok = cudaMalloc(&c->dpart, ublocks * NDIAG * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMalloc(&c->dpart2, (size_t)HIST_RB * NDIAG * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMalloc(&c->hist, (size_t)capacity * NDIAG * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMalloc(&c->hist_td, (size_t)capacity * 2 * sizeof(double)) == cudaSuccess;
    if (ok && (size_t)capacity * NDIAG > c->red_tmp_count) {
      cudaFree(c->red_tmp);
      c->red_tmp_count = (size_t)capacity * NDIAG;
      ok = cudaMalloc(&c->red_tmp, c->red_tmp_count * 8) == cudaSuccess;
    }
    if (!ok) {
      cudaGetLastError();
      return fail(c, HGKS_ENOMEM, "hgks_history_enable: device allocation failed");
    }
    c->hist_cap = capacity;
  }
  return set_ctl_hist(c, 0, c->hist_cap);
}

int hgks_history_read(hgks_ctx* c, double* out, int32_t max_rows, int32_t* rows) {
  if (!c || !rows) return fail(c, HGKS_EINVAL, "hgks_history_read: NULL argument");
  if (c->hist_cap <= 0) return fail(c, HGKS_EINVAL, "hgks_history_read: history not enabled");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  Ctl* h = c->ctl_host;
  CTL_READBACK(c);
  SYNC_TRY(c);
  const int n = h->hist_n;
  if (n > max_rows || (n > 0 && !out))
    return fail(c, HGKS_EINVAL, "hgks_history_read: %d rows pending, buffer holds %d", n, max_rows);
  *rows = n;
  if (n > 0) {
    int rc;
    if ((rc = coll_allreduce(c, c->hist, (size_t)n * NDIAG, 1))) return rc;  // rank-local sums -> global
    std::vector<double> a((size_t)n * NDIAG), td((size_t)n * 2);
    CUDA_TRY(c, cudaMemcpyAsync(a.data(), c->hist, a.size() * sizeof(double), cudaMemcpyDeviceToHost, c->s));
    CUDA_TRY(c, cudaMemcpyAsync(td.data(), c->hist_td, td.size() * sizeof(double), cudaMemcpyDeviceToHost, c->s));
    SYNC_TRY(c);
    for (int r = 0; r < n; ++r) {
      double* o = out + (size_t)r * HGKS_HIST_COLS;
      o[0] = td[2 * r];
      o[1] = td[2 * r + 1];
      normalise_diag(c, c->hist_rho0, &a[(size_t)r * NDIAG], o + 2);
    }
  }
  c->hist_pending = 0;
  return set_ctl_hist(c, 0, c->hist_cap);
}

int hgks_diagnostics(hgks_ctx* c, double rho0, double out[HGKS_DIAG_COUNT]) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_diagnostics: ctx is NULL");
  if (!out) return fail(c, HGKS_EINVAL, "hgks_diagnostics: out is NULL");
  if (!(rho0 > 0.0)) return fail(c, HGKS_EINVAL, "hgks_diagnostics: rho0 must be > 0");
  if (!c->have_state) return fail(c, HGKS_EINVAL, "hgks_diagnostics: no state set");
  static_assert(HGKS_DIAG_COUNT == NDIAG, "diagnostic count");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  int rc = c->fp32 ? diagnostics_t<float>(c) : diagnostics_t<double>(c);
  if (rc) return rc;
  normalise_diag(c, rho0, c->diag_host, out);
  return HGKS_OK;
}

}  // extern "C"

template <typename T>
static int plane_stats_t(hgks_ctx* c, double* out) {
  Geo<T> g = make_geo<T>(c);
  plane_stats_kernel<T><<<c->n[1], DIAG_TPB, 0, c->s>>>((const T*)c->Q[c->cur], g, c->p.gamma, c->stats_dev);
  c->total_launches += 1;
  CUDA_TRY(c, cudaGetLastError());
  const size_t cnt = (size_t)c->n[1] * NSTAT;
  int rc;
  if ((rc = coll_allreduce(c, c->stats_dev, cnt, 1))) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(out, c->stats_dev, cnt * sizeof(double), cudaMemcpyDeviceToHost, c->s));
  SYNC_TRY(c);
  const double inv = 1.0 / ((double)c->n[0] * c->n[2]);
  for (size_t k = 0; k < cnt; ++k) out[k] *= inv;
  return HGKS_OK;
}

extern "C" {

int hgks_plane_stats(hgks_ctx* c, double* out) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_plane_stats: ctx is NULL");
  if (!out) return fail(c, HGKS_EINVAL, "hgks_plane_stats: out is NULL");
  if (!c->have_state) return fail(c, HGKS_EINVAL, "hgks_plane_stats: no state set");
  static_assert(HGKS_STAT_COUNT == NSTAT, "statistic count");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  return c->fp32 ? plane_stats_t<float>(c, out) : plane_stats_t<double>(c, out);
}

int hgks_get_forcing(hgks_ctx* c, double* force, double* bulk_momentum, double* bulk_density) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_get_forcing: ctx is NULL");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  Ctl* h = c->ctl_host;
  CTL_READBACK(c);
  SYNC_TRY(c);
  const bool b = c->p.force_mode == HGKS_FORCE_BULK;
  if (force) *force = h->f_prev;
  if (bulk_momentum) *bulk_momentum = b ? h->m_cur : 0.0;
  if (bulk_density) *bulk_density = b ? h->rho_cur : 0.0;
  return HGKS_OK;
}

int hgks_destroy(hgks_ctx* c) {
  if (!c) return HGKS_OK;
  cudaSetDevice(c->dev);
  // loopback group: destroy is collective -- a rank returning from its last collective may still
  // be followed by peers that read its context (event handles) on the host, so nobody frees
  // anything until every rank has entered destroy (a timeout only delays the teardown)
  if (c->grp) c->grp->barrier();
  if (c->s) cudaStreamSynchronize(c->s);
  if (c->sc) cudaStreamSynchronize(c->sc);
  for (int b = 0; b < 2; ++b)
    if (c->gexec[b]) cudaGraphExecDestroy(c->gexec[b]);
  if (c->comm_halo) ncclCommDestroy(c->comm_halo);
  if (c->comm) ncclCommDestroy(c->comm);
  lb_leave(c);
  cudaFree(c->red_tmp);
  if (c->sc) cudaStreamDestroy(c->sc);
  for (cudaEvent_t e : {c->ev_xy, c->ev_halo, c->lb_post, c->lb_done, c->lb_rpost, c->lb_rdone})
    if (e) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) cudaFree(c->Q[b]);
  cudaFree(c->Qs);
  for (int d = 0; d < 3; ++d) cudaFree(c->F[d]);
  for (int b = 0; b < 2; ++b) cudaFree(c->FF[b]);
  cudaFree(c->metric);
  cudaFree(c->dmetric);
  cudaFree(c->diag_dev);
  cudaFree(c->bulk_dev);
  cudaFree(c->stats_dev);
  for (double* b : {c->dpart, c->dpart2, c->hist, c->hist_td}) cudaFree(b);
  if (c->diag_host) cudaFreeHost(c->diag_host);
  if (c->s2) cudaStreamDestroy(c->s2);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  for (int d = 0; d < 3; ++d) {
    if (c->ev_rec[d]) cudaEventDestroy(c->ev_rec[d]);
    if (d == 0 && c->ev_recA) cudaEventDestroy(c->ev_recA);
    if (c->ev_flux[d]) cudaEventDestroy(c->ev_flux[d]);
  }
  cudaFree(c->stage64);
  for (cudaStream_t st : {c->sio, c->sio_up}) {
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
  cudaFree(c->up64);
  cudaFree(c->down64);
  for (cudaEvent_t e : {c->ev_up, c->ev_upfree, c->ev_packed, c->ev_downdone})
    if (e) cudaEventDestroy(e);
  cudaFree(c->ctl);
  if (c->ctl_host) cudaFreeHost(c->ctl_host);
  for (int k = 0; k < 2 * 4096; ++k)
    if (c->prof.ev[k]) cudaEventDestroy(c->prof.ev[k]);
  if (c->own_stream && c->s) cudaStreamDestroy(c->s);
  delete c;
  return HGKS_OK;
}

int hgks_profile_enable(hgks_ctx* c, int enable) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_profile_enable: ctx is NULL");
  SYNC_TRY(c);
  if (enable && !c->prof.created) {
    for (int k = 0; k < 2 * 4096; ++k) CUDA_TRY(c, cudaEventCreate(&c->prof.ev[k]));
    c->prof.created = true;
  }
  c->prof.on = enable != 0;
  c->prof.nev = 0;
  for (int k = 0; k < HGKS_K_COUNT; ++k) {
    c->prof.ms[k] = 0;
    c->prof.launches[k] = 0;
  }
  c->total_launches = 0;
  return HGKS_OK;
}

int hgks_profile_read(hgks_ctx* c, double ms[HGKS_K_COUNT], int64_t launches[HGKS_K_COUNT], int64_t* total_launches) {
  if (!c) return fail(nullptr, HGKS_EINVAL, "hgks_profile_read: ctx is NULL");
  SYNC_TRY(c);
  prof_flush(c);
  for (int k = 0; k < HGKS_K_COUNT; ++k) {
    if (ms) ms[k] = c->prof.ms[k];
    if (launches) launches[k] = c->prof.launches[k];
  }
  if (total_launches) *total_launches = c->total_launches;
  return HGKS_OK;
}

// ---- test entry points (include/hgks_test.h) --------------------------------------------------
int hgks_test_gp_flux(int precision, double gamma, int mu_law, double mu_ref, double T_ref, double omega,
                      double prandtl, double dt, const double* in, int64_t n, double* out) {
  if (!in || !out || n < 0 || !(prandtl > 0)) return fail(nullptr, HGKS_EINVAL, "hgks_test_gp_flux: bad arguments");
  if (n == 0) return HGKS_OK;
  hgks_params p{};
  p.gamma = gamma;
  p.mu_law = (hgks_mu_law)mu_law;
  p.mu_ref = mu_ref;
  p.T_ref = T_ref;
  p.omega = omega;
  double *din = nullptr, *dout = nullptr;
  CUDA_TRY(nullptr, cudaMalloc(&din, 55 * n * sizeof(double)));
  CUDA_TRY(nullptr, cudaMalloc(&dout, 11 * n * sizeof(double)));
  CUDA_TRY(nullptr, cudaMemcpy(din, in, 55 * n * sizeof(double), cudaMemcpyHostToDevice));
  int blocks = (int)((n + 127) / 128);
  p.prandtl = prandtl;
  const bool prf = prandtl != 1.0;
  if (precision == HGKS_FP32) {
    if (prf) gp_flux_test_kernel<float, true><<<blocks, 128>>>(din, dout, n, make_gas<float>(p), (float)dt);
    else gp_flux_test_kernel<float, false><<<blocks, 128>>>(din, dout, n, make_gas<float>(p), (float)dt);
  } else {
    if (prf) gp_flux_test_kernel<double, true><<<blocks, 128>>>(din, dout, n, make_gas<double>(p), dt);
    else gp_flux_test_kernel<double, false><<<blocks, 128>>>(din, dout, n, make_gas<double>(p), dt);
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, 11 * n * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(din);
  cudaFree(dout);
  if (e != cudaSuccess) return fail(nullptr, HGKS_ECUDA, "hgks_test_gp_flux: %s", cudaGetErrorString(e));
  return HGKS_OK;
}

}  // extern "C"

template <typename T>
static int test_operator_t(hgks_ctx* c, double dt, double* L, double* dL) {
  Geo<T> g = make_geo<T>(c);
  T* Q = (T*)c->Q[c->cur];
  Ctl* h = c->ctl_host;
  CTL_READBACK(c);
  SYNC_TRY(c);
  h->dt = dt;
  h->idt = 1.0 / dt;
  h->halt = 0;
  CUDA_TRY(c, cudaMemcpyAsync(c->ctl, h, sizeof(Ctl), cudaMemcpyHostToDevice, c->s));
  int rc;
  if ((rc = fill_ghosts<T>(c, Q, false))) return rc;
  if ((rc = flux_sweeps<T, 1>(c, Q))) return rc;
  const long long ncell = (long long)g.n[0] * g.n[1] * g.n[2];
  double *dL_ = nullptr, *dDL = nullptr;
  CUDA_TRY(c, cudaMalloc(&dL_, 5 * ncell * sizeof(double)));
  CUDA_TRY(c, cudaMalloc(&dDL, 5 * ncell * sizeof(double)));
  operator_out_kernel<T><<<(int)((ncell + 255) / 256), 256, 0, c->s>>>((T*)c->F[0], (T*)c->F[1], (T*)c->F[2], g, dL_, dDL);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(L, dL_, 5 * ncell * sizeof(double), cudaMemcpyDeviceToHost, c->s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dL, dDL, 5 * ncell * sizeof(double), cudaMemcpyDeviceToHost, c->s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->s);
  cudaFree(dL_);
  cudaFree(dDL);
  if (e != cudaSuccess) return fail(c, HGKS_ECUDA, "hgks_test_operator: %s", cudaGetErrorString(e));
  return HGKS_OK;
}

extern "C" {

int hgks_test_face_flux(hgks_ctx* c, int dir, double* out) {
  if (!c || !out || dir < 0 || dir > 2) return fail(c, HGKS_EINVAL, "hgks_test_face_flux: bad arguments");
  const size_t n = 10 * c->nface[dir];
  SYNC_TRY(c);
  if (c->fp32) {
    float* h = (float*)malloc(n * sizeof(float));
    cudaError_t e = cudaMemcpy(h, c->F[dir], n * sizeof(float), cudaMemcpyDeviceToHost);
    for (size_t k = 0; k < n; ++k) out[k] = h[k];
    free(h);
    if (e != cudaSuccess) return fail(c, HGKS_ECUDA, "hgks_test_face_flux: %s", cudaGetErrorString(e));
  } else {
    CUDA_TRY(c, cudaMemcpy(out, c->F[dir], n * sizeof(double), cudaMemcpyDeviceToHost));
  }
  return HGKS_OK;
}

int hgks_test_operator(hgks_ctx* c, double dt, double* L, double* dL) {
  if (!c || !L || !dL || !(dt > 0)) return fail(c, HGKS_EINVAL, "hgks_test_operator: bad arguments");
  if (!c->have_state) return fail(c, HGKS_EINVAL, "hgks_test_operator: no state");
  CUDA_TRY(c, cudaSetDevice(c->dev));
  return c->fp32 ? test_operator_t<float>(c, dt, L, dL) : test_operator_t<double>(c, dt, L, dL);
}

}  // extern "C"
