// npm_capi.cu -- the C ABI (include/npm.h) and the model runtime: config
// validation, level schedule, device state, host/device pointer staging,
// kernel orchestration for encode / decode / pdf / sample / train.
#include "../../include/npm.h"
#include "npm_kernels.cuh"

#include <cmath>
#include <dlfcn.h>
#include <nccl.h>   // types only: the functions are resolved at run time (dlopen), see Nccl below
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using namespace npm;

namespace {

thread_local std::string g_err;

npm_status fail(npm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      return fail(NPM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));           \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t b) {
    if (b <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

}  // namespace

struct npm_model {
  npm_config cfg;
  int device = 0;
  int num_sms = 148;
  NetShape shape{};
  GridDesc grid{};
  int res[kMaxLevels] = {};
  int64_t entries[kMaxLevels] = {};
  int64_t n_mlp = 0, n_grid = 0, n_alpha = 0, n_total = 0;
  float* buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // params, grads, m, v, ema
  int64_t t = 0;
  // device statistics: [0] loss, [1] grad norm^2 ; counters [0] used [1] zero [2] dropped [3] nonfinite
  double* dstats = nullptr;
  unsigned long long* dcount = nullptr;
  DevBuf dbg_clock;                // NPM_DEBUG=4 phase stamps (measurement only)
  DevBuf wimg;                     // split-bf16 weight image of the training kernel
  int train_ws = 1;                // training kernel: 1 warp-specialised (npm_train_ws.cuh), 0 the r01 two-group kernel (NPM_TRAIN_WS)
  DevBuf stage[24];                // host-pointer staging slots
  std::mutex stage_mu;
  int64_t launches = 0;
  // kernel timing (npm_profile_*): CUDA events around each launch, on its stream
  bool prof = false;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  int64_t prof_launches[16] = {};
  double prof_ms[16] = {};
  bool use_bin = true; // spatial binning of batches >= kBinMin samples (NPM_BIN=0 disables)
  bool bin_train = false;  // also bin training batches (NPM_BIN_TRAIN=1)
  DevBuf bin_keys, bin_perm, bin_hist;
  // The binning scratch is one set per model; calls on different streams are
  // ordered through it: a binning pass waits for bin_free, recorded after the
  // kernel that consumed the previous permutation (two device-
  // pointer queries on different streams raced on bin_perm).
  cudaEvent_t bin_free = nullptr;
  // privatised coarse-level gradients (TrainArgs::priv): one copy per SM
  DevBuf priv;
  uint32_t priv_mask = 0;
  int64_t priv_stride = 0, priv_off[16] = {};
  // host-batch pipelining (HostPipe): a copy stream, staging buffers, events
  cudaStream_t copy_stream = nullptr, d2h_stream = nullptr;
  // input staging: double-buffered per call kind (0 queries, 1 training), so a
  // call's input copies never wait for the kernels of the previous call of
  // the same kind (nor of the other kind)
  DevBuf pipe_in[4][16], pipe_out[8];
  int pipe_parity[2] = {0, 0};
  cudaEvent_t pipe_in_free[4] = {nullptr, nullptr, nullptr, nullptr};   // last kernel that read pipe_in[set]
  cudaEvent_t pipe_out_free = nullptr;                 // last device->host copy out of pipe_out
  std::vector<cudaEvent_t> sync_events;
  ncclComm_t comm = nullptr;   // npm_comm_init: GRADS exchanged inside npm_optimizer_step
  int comm_world = 1, comm_rank = 0;
  int exchange = NPM_EXCHANGE_ALLREDUCE;   // npm_set_exchange
  bool pipeline = true;    // NPM_PIPELINE=0 disables
  int pipe_chunks = 3;     // NPM_PIPE_CHUNKS (c2 e2e: 2 -> 1.31, 3 -> 1.32, 4 -> 1.28, 8 -> 1.13 G/s)
  int query_groups = 1;    // NPM_QUERY_GROUPS
  int query_ws = 1;        // NPM_QUERY_WS
  int qws_groups = 2;      // chain groups of query_ws_kernel's plain calls (NPM_QWS_GROUPS)
};

namespace {

struct Pending {
  void* host;
  const void* dev;
  size_t bytes;
  bool pageable;
};

// Host/device pointer resolution (npm.h "POINTERS MAY BE HOST OR DEVICE").
struct Stager {
  npm_model* m;
  cudaStream_t st;
  int next = 0;
  std::vector<Pending> outs;
  bool any_pageable = false;
  cudaError_t err = cudaSuccess;

  static int kind(const void* p) {  // 0 host-pageable, 1 host-pinned, 2 device/managed
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return 2;
    if (at.type == cudaMemoryTypeHost) return 1;
    return 0;
  }
  // Errors are sticky: once a staging allocation or copy failed, every later
  // in()/out() returns NULL without touching err, so the caller's err check
  // sees the first failure (and no kernel runs on a NULL or stale input).
  template <class T>
  const T* in(const T* p, size_t count) {
    if (err != cudaSuccess) return nullptr;
    if (!p || count == 0) return p;
    const int k = kind(p);
    if (k == 2) return p;
    if (next >= 24) { err = cudaErrorMemoryAllocation; return nullptr; }
    DevBuf& b = m->stage[next++];
    err = b.ensure(count * sizeof(T));
    if (err != cudaSuccess) return nullptr;
    err = cudaMemcpyAsync(b.p, p, count * sizeof(T), cudaMemcpyHostToDevice, st);
    return static_cast<const T*>(b.p);
  }
  template <class T>
  T* out(T* p, size_t count) {
    if (err != cudaSuccess) return nullptr;
    if (!p || count == 0) return p;
    const int k = kind(p);
    if (k == 2) return p;
    if (next >= 24) { err = cudaErrorMemoryAllocation; return nullptr; }
    DevBuf& b = m->stage[next++];
    err = b.ensure(count * sizeof(T));
    if (err != cudaSuccess) return nullptr;
    outs.push_back({p, b.p, count * sizeof(T), k == 0});
    any_pageable |= (k == 0);
    return static_cast<T*>(b.p);
  }
  cudaError_t finish() {
    for (auto& o : outs) {
      cudaError_t e = cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return e;
    }
    if (any_pageable) return cudaStreamSynchronize(st);
    return cudaSuccess;
  }
};

bool query_ok(const npm_model* m, const npm_query* q) {
  if (!q || q->n < 0) return false;
  if (q->n == 0) return true;
  if (!q->px || !q->py || !q->pz) return false;
  if (m->cfg.mode == NPM_PRODUCT &&
      (!q->wox || !q->woy || !q->woz || !q->nx || !q->ny || !q->nz || !q->rough))
    return false;
  return true;
}

// Stage all query inputs (x, and product-mode conditioning).
void stage_query(Stager& s, const npm_model* m, const npm_query* q, npm_query& d) {
  d = *q;
  const size_t n = (size_t)q->n;
  d.px = s.in(q->px, n); d.py = s.in(q->py, n); d.pz = s.in(q->pz, n);
  if (m->cfg.mode == NPM_PRODUCT) {
    d.wox = s.in(q->wox, n); d.woy = s.in(q->woy, n); d.woz = s.in(q->woz, n);
    d.nx = s.in(q->nx, n); d.ny = s.in(q->ny, n); d.nz = s.in(q->nz, n);
    d.rough = s.in(q->rough, n);
  } else {
    d.wox = d.woy = d.woz = d.nx = d.ny = d.nz = d.rough = nullptr;
  }
  d.bsdf_pdf = m->n_alpha ? s.in(q->bsdf_pdf, n) : nullptr;
}

// ---------------------------------------------------------------------------
// HostPipe: a call whose arrays are ALL host pointers (and n >= 2 kPipeMin) is
// processed in kPipeChunks chunks so that the host->device copy of chunk j+1
// and the device->host copy of chunk j-1 (on the model's copy stream) overlap
// the kernels of chunk j (on the caller's stream).  Every array is [comps][n]
// on the host; chunk j of it is staged compactly as [comps][C_j] (one 2-D
// copy), so the kernels see an ordinary batch of C_j samples.  Ordering: the
// copy streams first wait for the caller's stream (earlier work may still
// read the staging buffers); the caller's stream finally waits for the last
// output copy.
constexpr int64_t kPipeMin = 65536;

struct PipeArr {
  const float* host_in;   // inputs
  float* host_out;        // outputs
  int comps;
};

struct HostPipe {
  npm_model* m;
  cudaStream_t st;
  int64_t n, C;
  int kind = 0;   // 0 query-type call, 1 training call (separate staging sets)
  int nch;
  std::vector<PipeArr> ins, outs;
  cudaError_t err = cudaSuccess;   // the FIRST failure (keep())
  bool pageable = false;
  int set = 0;

  bool keep(cudaError_t e) {
    if (e != cudaSuccess && err == cudaSuccess) err = e;
    return err == cudaSuccess;
  }

  static bool usable(const npm_model* m, int64_t n, std::initializer_list<const void*> ptrs) {
    if (!m->pipeline || n < 2 * kPipeMin || m->n_alpha) return false;   // (learn_alpha: staged path)
    for (const void* p : ptrs)
      if (p && Stager::kind(p) == 2) return false;   // a device array: the plain path
    return true;
  }
  cudaEvent_t ev(int i) {
    while ((int)m->sync_events.size() <= i) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      m->sync_events.push_back(e);
    }
    return m->sync_events[i];
  }
  // chunk j's device pointer of input / output array k
  const float* din(int k, int j) const {
    return static_cast<const float*>(m->pipe_in[set][k].p) + (size_t)j * C * ins[k].comps;
  }
  float* dout(int k, int j) const { return static_cast<float*>(m->pipe_out[k].p) + (size_t)j * C * outs[k].comps; }
  int64_t cn(int j) const { return j == nch - 1 ? n - (int64_t)j * C : C; }
  // Three component arrays (x/y/z): when they are the rows of one [3][n]
  // host array they move as one 2-D copy per chunk (fewer API calls).
  struct Tri { int k; bool packed; };
  Tri in3(const float* a, const float* b, const float* c) {
    Tri t{(int)ins.size(), a && b == a + n && c == a + 2 * n};
    if (t.packed) ins.push_back({a, nullptr, 3});
    else for (const float* p : {a, b, c}) ins.push_back({p, nullptr, 1});
    return t;
  }
  Tri out3(float* a, float* b, float* c) {
    Tri t{(int)outs.size(), a && b == a + n && c == a + 2 * n};
    if (t.packed) outs.push_back({nullptr, a, 3});
    else for (float* p : {a, b, c}) outs.push_back({nullptr, p, 1});
    return t;
  }
  const float* din3(Tri t, int comp, int j) const {
    return t.packed ? din(t.k, j) + (size_t)comp * cn(j) : din(t.k + comp, j);
  }
  float* dout3(Tri t, int comp, int j) const {
    return t.packed ? dout(t.k, j) + (size_t)comp * cn(j) : dout(t.k + comp, j);
  }

  // Runs launch(j, cn) for every chunk; launch enqueues chunk j's kernels on st.
  template <class F>
  npm_status run(F&& launch) {
    const int chunks = m->pipe_chunks;
    C = (n + chunks - 1) / chunks;
    if (C < kPipeMin) C = kPipeMin;
    nch = (int)((n + C - 1) / C);
    if (!m->copy_stream && cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      return NPM_ERR_CUDA;
    if (!m->d2h_stream && cudaStreamCreateWithFlags(&m->d2h_stream, cudaStreamNonBlocking) != cudaSuccess)
      return NPM_ERR_CUDA;
    // input staging alternates between two buffer sets, so this call's input
    // copies wait only for the kernels of the call before the previous one
    set = 2 * kind + m->pipe_parity[kind];
    m->pipe_parity[kind] ^= 1;
    for (size_t k = 0; k < ins.size(); ++k) {
      if ((err = m->pipe_in[set][k].ensure((size_t)n * ins[k].comps * sizeof(float))) != cudaSuccess)
        return NPM_ERR_OOM;
      pageable |= ins[k].host_in && Stager::kind(ins[k].host_in) == 0;
    }
    for (size_t k = 0; k < outs.size(); ++k) {
      if ((err = m->pipe_out[k].ensure((size_t)n * outs[k].comps * sizeof(float))) != cudaSuccess) return NPM_ERR_OOM;
      pageable |= outs[k].host_out && Stager::kind(outs[k].host_out) == 0;
    }
    // H2D on copy_stream, D2H on d2h_stream: a chunk's input copy never queues
    // behind the previous chunk's output copy
    cudaStream_t cs = m->copy_stream, ds = m->d2h_stream;
    // every copy / event call is checked (keep()): a failed input copy must
    // not be followed by kernels reading stale staging data
    if (m->pipe_in_free[set]) keep(cudaStreamWaitEvent(cs, m->pipe_in_free[set], 0));
    else if (keep(cudaEventCreateWithFlags(&m->pipe_in_free[set], cudaEventDisableTiming)) &&
             keep(cudaEventRecord(ev(0), st)))
      keep(cudaStreamWaitEvent(cs, ev(0), 0));
    for (int j = 0; j < nch && err == cudaSuccess; ++j) {
      const int64_t c = cn(j);
      for (size_t k = 0; k < ins.size(); ++k)
        if (ins[k].host_in)
          keep(cudaMemcpy2DAsync(const_cast<float*>(din((int)k, j)), (size_t)c * 4, ins[k].host_in + (size_t)j * C,
                                 (size_t)n * 4, (size_t)c * 4, ins[k].comps, cudaMemcpyHostToDevice, cs));
      keep(cudaEventRecord(ev(1 + 2 * j), cs));
    }
    if (err != cudaSuccess) return NPM_ERR_CUDA;
    // the kernels write pipe_out: the previous call's output copies (possibly
    // issued for another caller stream) must have drained
    if (!outs.empty() && m->pipe_out_free) keep(cudaStreamWaitEvent(st, m->pipe_out_free, 0));
    for (int j = 0; j < nch; ++j) {
      const int64_t c = cn(j);
      if (!keep(cudaStreamWaitEvent(st, ev(1 + 2 * j), 0))) return NPM_ERR_CUDA;
      npm_status r = launch(j, c);
      if (r != NPM_OK) return r;
      if (outs.empty()) continue;
      keep(cudaEventRecord(ev(2 + 2 * j), st));
      keep(cudaStreamWaitEvent(ds, ev(2 + 2 * j), 0));
      for (size_t k = 0; k < outs.size(); ++k)
        if (outs[k].host_out)
          keep(cudaMemcpy2DAsync(outs[k].host_out + (size_t)j * C, (size_t)n * 4, dout((int)k, j), (size_t)c * 4,
                                 (size_t)c * 4, outs[k].comps, cudaMemcpyDeviceToHost, ds));
      if (err != cudaSuccess) return NPM_ERR_CUDA;
    }
    keep(cudaEventRecord(m->pipe_in_free[set], st));   // after the last kernel reading pipe_in[set]
    if (!outs.empty()) {
      if (!m->pipe_out_free) keep(cudaEventCreateWithFlags(&m->pipe_out_free, cudaEventDisableTiming));
      if (keep(cudaEventRecord(m->pipe_out_free, ds))) keep(cudaStreamWaitEvent(st, m->pipe_out_free, 0));
    }
    if (err != cudaSuccess) return NPM_ERR_CUDA;
    if (pageable && !keep(cudaStreamSynchronize(ds))) return NPM_ERR_CUDA;
    return NPM_OK;
  }
};

void fill_query_args(const npm_model* m, const npm_query& d, int use_ema, QueryArgs& a) {
  memset(&a, 0, sizeof(a));
  a.n = d.n;
  a.px = d.px; a.py = d.py; a.pz = d.pz;
  a.wox = d.wox; a.woy = d.woy; a.woz = d.woz; a.nx = d.nx; a.ny = d.ny; a.nz = d.nz; a.rough = d.rough;
  a.params = use_ema ? m->buf[NPM_BUF_EMA] : m->buf[NPM_BUF_PARAMS];
  a.grid = m->grid;
  a.log_kmin = logf(m->cfg.kappa_min);
  a.log_kmax = logf(m->cfg.kappa_max);
  a.query_groups = m->query_groups;
  a.qws = m->query_ws;
  a.qws_groups = m->qws_groups;
  a.alpha_w = m->n_alpha ? a.params + m->n_mlp + m->n_grid : nullptr;
}

const char* kKindNames[] = {"query", "encode", "train_forward", "train_backward", "weight_grad", "adam",
                            "train_fused", "bin", "unwind", "fold"};
enum Kind { kKQuery = 0, kKEncode, kKTrainFwd, kKTrainBwd, kKWgrad, kKAdam, kKTrainFused, kKBin, kKUnwind, kKFold,
            kKinds };
constexpr int64_t kBinMin = 65536;  // batches at least this large are spatially binned
constexpr int64_t kBufPad = 8 + 4 * 64;   // floats past n_total in every parameter buffer
constexpr int kMaxShardWorld = 64;

// ZeRO-1 shard of rank in world: [begin, begin + count) of the flat parameter
// vector, chunk = ceil(n_total / world / 4) * 4 floats per rank (float4 Adam).
void shard_of(const npm_model* m, int rank, int world, int64_t& begin, int64_t& count, int64_t& chunk) {
  chunk = ((m->n_total + world - 1) / world + 3) / 4 * 4;
  begin = (int64_t)rank * chunk;
  count = m->n_total - begin;
  count = count < 0 ? 0 : (count > chunk ? chunk : count);
}

cudaEvent_t take_event(npm_model* m) {
  if (!m->pool.empty()) { cudaEvent_t e = m->pool.back(); m->pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Timed launch: records events around `f()` when profiling is on.
template <class F>
int timed(npm_model* m, int kind, cudaStream_t st, F&& f) {
  if (!m->prof) return f();
  cudaEvent_t a = take_event(m), b = take_event(m);
  cudaEventRecord(a, st);
  const int r = f();
  cudaEventRecord(b, st);
  m->pending.push_back({kind, a, b});
  return r;
}

npm_status check_launch(npm_model* m, int r) {
  if (r < 0) return fail(NPM_ERR_INVALID, "unsupported decoder shape");
  m->launches += r;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NPM_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return NPM_OK;
}

// Sort-chunk of the binning (npm_bin.cu): with L2-resident grid tables the
// scattered SoA I/O of a binned launch is the cost, so batches are sorted in
// chunks of kSortChunk (B200, c3: query 3.47 -> 2.38 ms); with HBM-resident
// tables (> 64 MB) the gathers dominate and one global sort keeps the most
// coherence (c5: chunking cost +0.2 ms).
static int64_t sort_chunk(const npm_model* m, int64_t n) {
  return m->n_grid * 4 > ((int64_t)64 << 20) ? n : (n < kSortChunk ? n : kSortChunk);
}

// Spatial binning of a device-resident position batch (npm_bin.cu); returns
// the processing order, or NULL (identity) for small batches / when disabled.
npm_status maybe_bin(npm_model* m, const float* px, const float* py, const float* pz, int64_t n, cudaStream_t st,
                     const uint32_t** perm) {
  *perm = nullptr;
  if (!m->use_bin || n < kBinMin) return NPM_OK;
  if (m->bin_free) CUDA_TRY(cudaStreamWaitEvent(st, m->bin_free, 0));
  cudaError_t e;
  if ((e = m->bin_keys.ensure(n * sizeof(uint32_t))) != cudaSuccess ||
      (e = m->bin_perm.ensure(n * sizeof(uint32_t))) != cudaSuccess ||
      (e = m->bin_hist.ensure((size_t)bin_hist_entries(n, sort_chunk(m, n)) * sizeof(uint32_t))) != cudaSuccess)
    return fail(NPM_ERR_OOM, "binning scratch");
  uint32_t* p = static_cast<uint32_t*>(m->bin_perm.p);
  npm_status r = check_launch(m, timed(m, kKBin, st, [&] {
    return launch_bin(px, py, pz, n, sort_chunk(m, n), m->n_grid * 4 > ((int64_t)64 << 20), m->grid,
                      static_cast<uint32_t*>(m->bin_keys.p),
                      static_cast<uint32_t*>(m->bin_hist.p), p, m->num_sms, st);
  }));
  if (r == NPM_OK) *perm = p;
  return r;
}

// After the launch that read a permutation from maybe_bin: later binning
// passes (on any stream) wait for it.
npm_status bin_release(npm_model* m, cudaStream_t st, const uint32_t* perm) {
  if (!perm) return NPM_OK;
  if (!m->bin_free) CUDA_TRY(cudaEventCreateWithFlags(&m->bin_free, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(m->bin_free, st));
  return NPM_OK;
}

// The fused query kernel (+ releasing the binning scratch it read).
npm_status query_launch(npm_model* m, const QueryArgs& a, cudaStream_t st) {
  npm_status r = check_launch(m, timed(m, kKQuery, st, [&] { return launch_query_tc(m->shape, a, m->num_sms, st); }));
  if (r != NPM_OK) return r;
  return bin_release(m, st, a.perm);
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

// NCCL, resolved at run time: the process may already hold the library (e.g.
// through torch); dlopen("libnccl.so.2") then returns that same copy, and a
// process without NCCL still loads libnpm (the calls return NPM_ERR_NCCL).
namespace {
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};
const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
    r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(dlsym(h, "ncclAllReduce"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    r.reduce_scatter = reinterpret_cast<decltype(r.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
    r.all_gather = reinterpret_cast<decltype(r.all_gather)>(dlsym(h, "ncclAllGather"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    r.ok = r.get_unique_id && r.comm_init_rank && r.all_reduce && r.comm_destroy && r.reduce_scatter && r.all_gather;
    return r;
  }();
  return n;
}
npm_status nccl_fail(ncclResult_t e, const char* what) {
  const Nccl& n = nccl();
  return fail(NPM_ERR_NCCL, std::string(what) + ": " + (n.error_string ? n.error_string(e) : "NCCL error"));
}

void nccl_destroy(ncclComm_t c) {
  if (nccl().ok && c) nccl().comm_destroy(c);
}
}  // namespace

// ===========================================================================
extern "C" {

int npm_version(void) { return NPM_VERSION; }
const char* npm_last_error(void) { return g_err.c_str(); }


npm_status npm_get_unique_id(uint8_t out[128]) {
  if (!out) return fail(NPM_ERR_INVALID, "null argument");
  const Nccl& n = nccl();
  if (!n.ok) return fail(NPM_ERR_NCCL, "libnccl.so.2 not available");
  ncclUniqueId id;
  const ncclResult_t e = n.get_unique_id(&id);
  if (e != ncclSuccess) return nccl_fail(e, "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return NPM_OK;
}

npm_status npm_comm_init(npm_model* m, int rank, int world, const uint8_t uid[128]) {
  if (!m || !uid || world < 1 || rank < 0 || rank >= world) return fail(NPM_ERR_INVALID, "bad argument");
  if (m->comm) return fail(NPM_ERR_STATE, "communicator already attached");
  const Nccl& n = nccl();
  if (!n.ok) return fail(NPM_ERR_NCCL, "libnccl.so.2 not available");
  DeviceGuard g(m->device);
  ncclUniqueId id;
  memcpy(&id, uid, 128);
  const ncclResult_t e = n.comm_init_rank(&m->comm, world, id, rank);
  if (e != ncclSuccess) { m->comm = nullptr; return nccl_fail(e, "ncclCommInitRank"); }
  m->comm_world = world;
  m->comm_rank = rank;
  return NPM_OK;
}

npm_status npm_set_exchange(npm_model* m, int mode) {
  if (!m || (mode != NPM_EXCHANGE_ALLREDUCE && mode != NPM_EXCHANGE_ZERO1)) return fail(NPM_ERR_INVALID, "bad argument");
  m->exchange = mode;
  return NPM_OK;
}

npm_status npm_shard_range(const npm_model* m, int rank, int world, int64_t* begin, int64_t* count, int64_t* chunk) {
  if (!m || world < 1 || world > kMaxShardWorld || rank < 0 || rank >= world) return fail(NPM_ERR_INVALID, "bad argument");
  int64_t b, c, ch;
  shard_of(m, rank, world, b, c, ch);
  if (begin) *begin = b;
  if (count) *count = c;
  if (chunk) *chunk = ch;
  return NPM_OK;
}

void npm_abi_sizes(int32_t* config, int32_t* query, int32_t* stats) {
  if (config) *config = (int32_t)sizeof(npm_config);
  if (query) *query = (int32_t)sizeof(npm_query);
  if (stats) *stats = (int32_t)sizeof(npm_step_stats);
}

void npm_default_config(npm_config* c) {
  memset(c, 0, sizeof(*c));
  c->mode = NPM_RADIANCE;
  c->n_lobes = 8;
  c->n_levels = 8;
  c->n_features = 4;
  c->base_res = 8;
  c->max_res = 86;
  c->log2_hashmap = 18;      // C-A4
  c->mlp_linear_layers = 3;
  c->mlp_width = 64;
  c->sh_bands = 4;           // C-A20
  for (int a = 0; a < 3; ++a) { c->aabb_lo[a] = -1.0f; c->aabb_hi[a] = 1.0f; }
  c->lr = 5e-3f;
  c->beta1 = 0.9f; c->beta2 = 0.999f; c->adam_eps = 1e-8f;  // C-A14
  c->ema_decay = 0.99f;      // C-A15
  c->kappa_min = 1e-5f; c->kappa_max = 1e5f;                 // C-A8
  c->init_seed = 0x4E504DULL;
}

npm_status npm_create(const npm_config* cfg, int dev, npm_model** out) {
  if (!cfg || !out) return fail(NPM_ERR_INVALID, "null argument");
  const npm_config& c = *cfg;
  if (c.mode != NPM_RADIANCE && c.mode != NPM_PRODUCT) return fail(NPM_ERR_INVALID, "bad mode");
  if (c.n_features != 4) return fail(NPM_ERR_INVALID, "n_features must be 4");
  if (c.n_levels < 1 || c.n_levels > kMaxLevels) return fail(NPM_ERR_INVALID, "n_levels out of range [1,16]");
  if (c.n_lobes < 1 || c.n_lobes > kMaxLobes) return fail(NPM_ERR_INVALID, "n_lobes out of range [1,16]");
  if (c.base_res < 2 || c.max_res < c.base_res || (c.n_levels > 1 && c.max_res <= c.base_res))
    return fail(NPM_ERR_INVALID, "need 2 <= D_1 < D_L");
  if (c.log2_hashmap < 0 || c.log2_hashmap > 30) return fail(NPM_ERR_INVALID, "log2_hashmap out of range");
  if (c.divergence < 0 || c.divergence > 2)
    return fail(NPM_ERR_INVALID, "divergence must be 0 (KL), 1 (chi^2) or 2 (variance-aware target)");
  if (c.divergence == 2 && (c.mode != NPM_RADIANCE || c.n_lobes != 8))
    return fail(NPM_ERR_INVALID, "variance-aware target: radiance-mode shapes with K = 8 only");
  if (c.divergence == 2 && c.learn_alpha)
    return fail(NPM_ERR_INVALID, "variance-aware target and learn_alpha are exclusive");
  if (c.learn_alpha != 0 && c.learn_alpha != 1) return fail(NPM_ERR_INVALID, "learn_alpha must be 0 or 1");
  if (c.learn_alpha && (c.mode != NPM_RADIANCE || c.n_lobes != 8))
    return fail(NPM_ERR_INVALID, "learn_alpha: radiance-mode shapes with K = 8 only");
  for (int a = 0; a < 3; ++a)
    if (!(c.aabb_hi[a] > c.aabb_lo[a]) || !std::isfinite(c.aabb_lo[a]) || !std::isfinite(c.aabb_hi[a]))
      return fail(NPM_ERR_INVALID, "degenerate AABB");
  if (c.mode == NPM_PRODUCT && c.sh_bands != 4) return fail(NPM_ERR_INVALID, "product mode needs sh_bands = 4");
  if (!(c.kappa_min > 0) || !(c.kappa_max > c.kappa_min)) return fail(NPM_ERR_INVALID, "bad kappa range");
  if (!(c.ema_decay >= 0 && c.ema_decay < 1)) return fail(NPM_ERR_INVALID, "ema_decay must be in [0,1)");

  NetShape s;
  s.n_in = c.n_levels * c.n_features + (c.mode == NPM_PRODUCT ? 2 * c.sh_bands * c.sh_bands + 1 : 0);
  s.width = c.mlp_width;
  s.n_layers = c.mlp_linear_layers;
  s.n_out = 4 * c.n_lobes;
  s.product = c.mode == NPM_PRODUCT;
  if (!shape_supported(s)) return fail(NPM_ERR_INVALID, "unsupported decoder shape (see npm.h)");

  DeviceGuard g(dev);
  auto* m = new npm_model();
  m->cfg = c;
  m->device = dev;
  m->shape = s;
  if (const char* e = getenv("NPM_BIN")) m->use_bin = !(e[0] == '0');
  if (const char* e = getenv("NPM_PIPELINE")) m->pipeline = !(e[0] == '0');
  if (const char* e = getenv("NPM_PIPE_CHUNKS")) m->pipe_chunks = atoi(e) > 0 ? atoi(e) : 3;
  // Query kernel layout: two 256-thread CTAs per SM, or one CTA running two
  // tile groups over a single copy of the weights (frees one weight copy of
  // smem for L1).  Measured on B200: the product shape (53 KB of split-bf16
  // weights) gains (c4 query 2.38 -> 2.05 ms); c2 / c5 lose 5 % / 3 %.
  m->query_groups = c.mode == NPM_PRODUCT ? 2 : 1;
  if (const char* e = getenv("NPM_QUERY_GROUPS")) m->query_groups = atoi(e) == 2 ? 2 : 1;
  if (const char* e = getenv("NPM_QUERY_WS")) m->query_ws = atoi(e);
  if (cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    delete m;
    return fail(NPM_ERR_CUDA, "no CUDA device");
  }
  // Level schedule (C-O2 / C-A3) and table sizes (C-A4).
  const int L = c.n_levels;
  if (L == 1) {
    m->res[0] = c.max_res;
  } else {
    const double b = std::pow((double)c.max_res / (double)c.base_res, 1.0 / (L - 1));
    for (int l = 0; l < L; ++l) m->res[l] = (int)std::ceil((double)c.base_res * std::pow(b, (double)l) - 1e-9);
    m->res[L - 1] = c.max_res;
  }
  GridDesc& gd = m->grid;
  gd.L = L;
  gd.hashed_mask = 0;
  int64_t off = 0;
  const int64_t T = c.log2_hashmap ? (int64_t(1) << c.log2_hashmap) : 0;
  for (int l = 0; l < L; ++l) {
    const int64_t d3 = (int64_t)m->res[l] * m->res[l] * m->res[l];
    int64_t e = d3;
    if (T && d3 > T) { e = T; gd.hashed_mask |= 1u << l; }
    if (e > 0xFFFFFFFFLL) { delete m; return fail(NPM_ERR_INVALID, "level too large for 32-bit indices"); }
    m->entries[l] = e;
    gd.res[l] = m->res[l];
    gd.resm1f[l] = (float)(m->res[l] - 1);
    gd.cellmax[l] = m->res[l] > 2 ? m->res[l] - 2 : 0;
    gd.cellmaxf[l] = (float)gd.cellmax[l];
    gd.tsize[l] = (uint32_t)e;
    gd.off[l] = off;
    off += e;
  }
  for (int a = 0; a < 3; ++a) {
    gd.lo[a] = c.aabb_lo[a];
    gd.inv[a] = (float)(1.0 / ((double)c.aabb_hi[a] - (double)c.aabb_lo[a]));  // C-O1
  }
  m->n_grid = off * c.n_features;
  // Bin training batches when the grid tables are not L2-resident: measured
  // on B200, c5 (632 MB tables) train 9.05 -> 6.92 ms; c2/c3 (10 MB) neutral
  // or slower (the binned scatter-adds collide on L2 lines).
  m->bin_train = m->n_grid * 4 > ((int64_t)64 << 20);
  if (const char* e = getenv("NPM_BIN_TRAIN")) m->bin_train = e[0] == '1';
  // query_ws_kernel chain groups (B200, same box): two for L2-resident
  // radiance tables (c2 205 vs 232 us with one), one for HBM-resident tables
  // (c5 3.04 -> 2.34 ms) and the product shape (c4 1.84 -> 1.59 ms)
  m->qws_groups = (c.mode == NPM_PRODUCT || m->n_grid * 4 > ((int64_t)64 << 20)) ? 1 : 2;
  if (const char* e = getenv("NPM_QWS_GROUPS")) m->qws_groups = atoi(e) == 1 ? 1 : 2;
  // Training kernel per shape (B200 measurements): the warp-
  // specialised kernel for L2-resident tables (c2 612 vs 632 us; c3 equal);
  // the r01 two-group kernel for HBM-resident tables, whose binned,
  // privatised scatter it does not have (c5 4.8 vs 6.3 ms).
  m->train_ws = m->bin_train ? 0 : 1;
  if (const char* e = getenv("NPM_TRAIN_WS")) m->train_ws = atoi(e);
  if (c.learn_alpha || c.divergence == 2) m->train_ws = 1;   // (C-A34 / C-A35 live in the warp-specialised kernel)
  // Privatise the scatter of small (coarse) levels when training batches are
  // binned: coherent records then add to the same few coarse entries from
  // every SM and the reductions queue on the same L2 lines.  Each SM
  // accumulates them in its own copy; fold_priv adds the copies after the
  // launch.  Measured on B200 (c5, levels up to 65,536 entries: the three
  // coarsest, 109 MB of copies): train 6.37 -> 5.29 ms, fold 89 us; unbinned
  // c2 gains nothing (its random-order reductions do not collide): off there.
  if (m->bin_train) {
    int64_t per = 0;
    int64_t priv_max = 65536;
    if (const char* e = getenv("NPM_PRIV_MAX")) priv_max = atoll(e);   // measurement knob
    for (int l = 0; l < L; ++l) {
      if (m->entries[l] > priv_max) continue;
      if ((per + m->entries[l]) * 16 * m->num_sms > ((int64_t)256 << 20)) break;
      m->priv_mask |= 1u << l;
      m->priv_off[l] = per;
      per += m->entries[l];
    }
    m->priv_stride = per;
    if (const char* e = getenv("NPM_PRIV")) if (e[0] == '0') m->priv_mask = 0;
  }
  int64_t nm = 0;
  {
    int dims[4] = {s.n_in, s.width, s.width, s.n_out};
    if (s.n_layers == 2) dims[2] = s.n_out;
    for (int k = 0; k < s.n_layers; ++k) nm += (int64_t)dims[k] * dims[k + 1] + dims[k + 1];
  }
  m->n_mlp = nm;
  if (nm % 4) { delete m; return fail(NPM_ERR_INVALID, "internal: MLP size not 16B aligned"); }
  m->n_alpha = c.learn_alpha ? ((int64_t)c.mlp_width + 1 + 3) / 4 * 4 : 0;   // C-A34 head after the grid
  m->n_total = m->n_mlp + m->n_grid + m->n_alpha;
  for (int b = 0; b < 5; ++b) {
    // + kBufPad floats: the paired grid gathers (gather_level) read the 32-B
    // entry pair containing the last table entry, and the ZeRO-1 exchange
    // views world * chunk >= n_total floats (npm_shard_range, world <= 64)
    if (cudaMalloc(&m->buf[b], (m->n_total + kBufPad) * sizeof(float)) != cudaSuccess) {
      npm_destroy(m);
      return fail(NPM_ERR_OOM, "parameter buffers");
    }
    cudaMemsetAsync(m->buf[b] + m->n_total, 0, kBufPad * sizeof(float), 0);
  }
  if (cudaMalloc(&m->dstats, 2 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&m->dcount, 4 * sizeof(unsigned long long)) != cudaSuccess) {
    npm_destroy(m);
    return fail(NPM_ERR_OOM, "stats");
  }
  cudaStream_t st = 0;
  launch_init_params(m->buf[NPM_BUF_PARAMS], m->n_mlp, m->n_mlp + m->n_grid, s, c.init_seed, st);
  m->launches += 1;
  if (m->n_alpha)   // the selection head starts at a = 0, c = 0: alpha = 1/2 (the paper's fixed choice)
    cudaMemsetAsync(m->buf[NPM_BUF_PARAMS] + m->n_mlp + m->n_grid, 0, m->n_alpha * sizeof(float), st);
  cudaMemsetAsync(m->buf[NPM_BUF_GRADS], 0, m->n_total * sizeof(float), st);
  if (m->priv_mask) {
    const size_t pb = (size_t)m->priv_stride * m->num_sms * 16;
    if (m->priv.ensure(pb) != cudaSuccess) { npm_destroy(m); return fail(NPM_ERR_OOM, "private gradient copies"); }
    cudaMemsetAsync(m->priv.p, 0, pb, st);
  }
  cudaMemsetAsync(m->buf[NPM_BUF_ADAM_M], 0, m->n_total * sizeof(float), st);
  cudaMemsetAsync(m->buf[NPM_BUF_ADAM_V], 0, m->n_total * sizeof(float), st);
  cudaMemcpyAsync(m->buf[NPM_BUF_EMA], m->buf[NPM_BUF_PARAMS], m->n_total * sizeof(float),
                  cudaMemcpyDeviceToDevice, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    npm_destroy(m);
    return fail(NPM_ERR_CUDA, std::string("init: ") + cudaGetErrorString(e));
  }
  *out = m;
  return NPM_OK;
}

npm_status npm_destroy(npm_model* m) {
  if (!m) return NPM_OK;
  DeviceGuard g(m->device);
  for (auto& b : m->buf) if (b) cudaFree(b);
  if (m->dstats) cudaFree(m->dstats);
  if (m->dcount) cudaFree(m->dcount);
  m->dbg_clock.release();
  m->wimg.release();
  m->bin_keys.release();
  m->bin_perm.release();
  m->bin_hist.release();
  if (m->bin_free) cudaEventDestroy(m->bin_free);
  m->priv.release();
  for (auto& s : m->stage) s.release();
  for (auto& set : m->pipe_in) for (auto& b : set) b.release();
  for (auto e : m->pipe_in_free) if (e) cudaEventDestroy(e);
  if (m->pipe_out_free) cudaEventDestroy(m->pipe_out_free);
  for (auto& b : m->pipe_out) b.release();
  for (auto e : m->sync_events) cudaEventDestroy(e);
  if (m->comm) nccl_destroy(m->comm);
  if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
  if (m->d2h_stream) cudaStreamDestroy(m->d2h_stream);
  for (auto& r : m->pending) { m->pool.push_back(r.a); m->pool.push_back(r.b); }
  for (auto e : m->pool) cudaEventDestroy(e);
  delete m;
  return NPM_OK;
}

npm_status npm_param_count(const npm_model* m, int64_t* n_grid, int64_t* n_mlp) {
  if (!m) return fail(NPM_ERR_INVALID, "null model");
  if (n_grid) *n_grid = m->n_grid;
  if (n_mlp) *n_mlp = m->n_mlp;
  return NPM_OK;
}

npm_status npm_level_info(const npm_model* m, int32_t* res, int64_t* entries) {
  if (!m) return fail(NPM_ERR_INVALID, "null model");
  for (int l = 0; l < m->cfg.n_levels; ++l) {
    if (res) res[l] = m->res[l];
    if (entries) entries[l] = m->entries[l];
  }
  return NPM_OK;
}

npm_status npm_get_step(const npm_model* m, int64_t* t) {
  if (!m || !t) return fail(NPM_ERR_INVALID, "null argument");
  *t = m->t;
  return NPM_OK;
}
npm_status npm_set_step(npm_model* m, int64_t t) {
  if (!m || t < 0) return fail(NPM_ERR_INVALID, "bad argument");
  m->t = t;
  return NPM_OK;
}

npm_status npm_buffer_device_ptr(npm_model* m, npm_buffer which, float** ptr, int64_t* count) {
  if (!m || (int)which < 0 || (int)which > 4 || !ptr) return fail(NPM_ERR_INVALID, "bad argument");
  *ptr = m->buf[which];
  if (count) *count = m->n_total;
  return NPM_OK;
}

int64_t npm_launch_count(const npm_model* m) { return m ? m->launches : 0; }

static void prof_drain(npm_model* m) {
  for (auto& r : m->pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    m->prof_ms[r.kind] += ms;
    m->prof_launches[r.kind] += 1;
    m->pool.push_back(r.a);
    m->pool.push_back(r.b);
  }
  m->pending.clear();
}

int npm_profile_kinds(void) { return kKinds; }

npm_status npm_profile_enable(npm_model* m, int enable) {
  if (!m) return fail(NPM_ERR_INVALID, "null model");
  DeviceGuard g(m->device);
  prof_drain(m);
  m->prof = enable != 0;
  return NPM_OK;
}

npm_status npm_profile_reset(npm_model* m) {
  if (!m) return fail(NPM_ERR_INVALID, "null model");
  DeviceGuard g(m->device);
  prof_drain(m);
  for (int k = 0; k < 16; ++k) { m->prof_ms[k] = 0; m->prof_launches[k] = 0; }
  return NPM_OK;
}

npm_status npm_profile_read(npm_model* m, int kind, const char** name, int64_t* launches, double* total_ms) {
  if (!m || kind < 0 || kind >= kKinds) return fail(NPM_ERR_INVALID, "bad argument");
  DeviceGuard g(m->device);
  prof_drain(m);
  if (name) *name = kKindNames[kind];
  if (launches) *launches = m->prof_launches[kind];
  if (total_ms) *total_ms = m->prof_ms[kind];
  return NPM_OK;
}

npm_status npm_get_buffer(npm_model* m, npm_buffer which, float* dst, int64_t count, void* stream) {
  if (!m || (int)which < 0 || (int)which > 4 || !dst) return fail(NPM_ERR_INVALID, "bad argument");
  if (count != m->n_total) return fail(NPM_ERR_INVALID, "count must equal n_mlp + n_grid");
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(dst, m->buf[which], count * sizeof(float), cudaMemcpyDefault, st));
  if (Stager::kind(dst) != 2) CUDA_TRY(cudaStreamSynchronize(st));
  return NPM_OK;
}

npm_status npm_set_buffer(npm_model* m, npm_buffer which, const float* src, int64_t count, void* stream) {
  if (!m || (int)which < 0 || (int)which > 4 || !src) return fail(NPM_ERR_INVALID, "bad argument");
  if (count != m->n_total) return fail(NPM_ERR_INVALID, "count must equal n_mlp + n_grid");
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(m->buf[which], src, count * sizeof(float), cudaMemcpyDefault, st));
  if (Stager::kind(src) != 2) CUDA_TRY(cudaStreamSynchronize(st));
  return NPM_OK;
}

// ---------------------------------------------------------------------------
npm_status npm_encode(npm_model* m, const npm_query* q, int use_ema, float* feat, void* stream) {
  if (!m || !query_ok(m, q) || (q->n > 0 && !feat)) return fail(NPM_ERR_INVALID, "bad argument");
  if (q->n == 0) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const int LF = m->cfg.n_levels * m->cfg.n_features;
  float* f = s.out(feat, (size_t)LF * q->n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  QueryArgs a;
  fill_query_args(m, d, use_ema, a);
  a.params += m->n_mlp;  // grid section
  a.feat = f;
  npm_status r = check_launch(m, timed(m, kKEncode, st, [&] { return launch_encode(m->cfg.n_levels, a, m->num_sms, st); }));
  if (r != NPM_OK) return r;
  CUDA_TRY(s.finish());
  return NPM_OK;
}

npm_status npm_encode_debug(npm_model* m, const npm_query* q, uint32_t* idx, float* w, void* stream) {
  if (!m || !query_ok(m, q)) return fail(NPM_ERR_INVALID, "bad argument");
  if (q->n == 0 || (!idx && !w)) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const size_t cnt = (size_t)m->cfg.n_levels * 8 * q->n;
  uint32_t* di = s.out(idx, cnt);
  float* dw = s.out(w, cnt);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  QueryArgs a;
  fill_query_args(m, d, 0, a);
  a.params += m->n_mlp;
  a.dbg_idx = di;
  a.dbg_w = dw;
  npm_status r = check_launch(m, timed(m, kKEncode, st, [&] { return launch_encode(m->cfg.n_levels, a, m->num_sms, st); }));
  if (r != NPM_OK) return r;
  CUDA_TRY(s.finish());
  return NPM_OK;
}

npm_status npm_decode(npm_model* m, const npm_query* q, const float* feat, int use_ema, float* raw,
                      float* lambda, float* kappa, float* mu, void* stream) {
  if (!m || !query_ok(m, q)) return fail(NPM_ERR_INVALID, "bad argument");
  if (feat && m->cfg.mode == NPM_PRODUCT) return fail(NPM_ERR_INVALID, "feat input is radiance-mode only");
  if (q->n == 0 || (!raw && !lambda && !kappa && !mu)) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const size_t n = (size_t)q->n, K = (size_t)m->cfg.n_lobes;
  const float* fi = s.in(feat, (size_t)m->cfg.n_levels * m->cfg.n_features * n);
  QueryArgs a;
  fill_query_args(m, d, use_ema, a);
  a.feat_in = fi;
  a.raw = s.out(raw, 4 * K * n);
  a.lambda = s.out(lambda, K * n);
  a.kappa = s.out(kappa, K * n);
  a.mu = s.out(mu, 3 * K * n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  npm_status r = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
  if (r != NPM_OK) return r;
  r = query_launch(m, a, st);
  if (r != NPM_OK) return r;
  CUDA_TRY(s.finish());
  return NPM_OK;
}

npm_status npm_pdf(npm_model* m, const npm_query* q, const float* wix, const float* wiy, const float* wiz,
                   int use_ema, float* pdf, void* stream) {
  if (!m || !query_ok(m, q) || (q->n > 0 && (!wix || !wiy || !wiz || !pdf)))
    return fail(NPM_ERR_INVALID, "bad argument");
  if (q->n == 0) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const size_t n = (size_t)q->n;
  QueryArgs a;
  fill_query_args(m, d, use_ema, a);
  a.wx = s.in(wix, n); a.wy = s.in(wiy, n); a.wz = s.in(wiz, n);
  a.pdf = s.out(pdf, n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  npm_status r = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
  if (r != NPM_OK) return r;
  r = query_launch(m, a, st);
  if (r != NPM_OK) return r;
  CUDA_TRY(s.finish());
  return NPM_OK;
}

npm_status npm_sample(npm_model* m, const npm_query* q, const float* u, uint64_t seed, uint64_t offset,
                      int use_ema, float* wix, float* wiy, float* wiz, float* pdf, const float* qx,
                      const float* qy, const float* qz, float* pdf_q, void* stream) {
  if (!m || !query_ok(m, q) || (q->n > 0 && (!wix || !wiy || !wiz || !pdf)))
    return fail(NPM_ERR_INVALID, "bad argument");
  const bool fused = qx && qy && qz && pdf_q;
  if ((qx || qy || qz || pdf_q) && !fused) return fail(NPM_ERR_INVALID, "fused query needs qx, qy, qz, pdf_q");
  if (q->n == 0) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  const bool prod = m->cfg.mode == NPM_PRODUCT;
  if (HostPipe::usable(m, q->n, {q->px, q->py, q->pz, prod ? q->wox : nullptr, prod ? q->nx : nullptr,
                                 prod ? q->rough : nullptr, u, qx, wix, pdf, pdf_q})) {
    HostPipe hp{m, st, q->n};
    const HostPipe::Tri tx = hp.in3(q->px, q->py, q->pz);
    HostPipe::Tri two{}, tn{};
    int kr = -1;
    if (prod) {
      two = hp.in3(q->wox, q->woy, q->woz);
      tn = hp.in3(q->nx, q->ny, q->nz);
      kr = (int)hp.ins.size();
      hp.ins.push_back({q->rough, nullptr, 1});
    }
    const int ku = u ? (int)hp.ins.size() : -1;
    if (u) hp.ins.push_back({u, nullptr, 3});
    HostPipe::Tri tq{};
    if (fused) tq = hp.in3(qx, qy, qz);
    const HostPipe::Tri tw = hp.out3(wix, wiy, wiz);
    const int kp = (int)hp.outs.size();
    hp.outs.push_back({nullptr, pdf, 1});
    const int kpq = (int)hp.outs.size();
    if (fused) hp.outs.push_back({nullptr, pdf_q, 1});
    const npm_status r = hp.run([&](int j, int64_t c) -> npm_status {
      npm_query d{};
      d.n = c;
      d.px = hp.din3(tx, 0, j); d.py = hp.din3(tx, 1, j); d.pz = hp.din3(tx, 2, j);
      if (prod) {
        d.wox = hp.din3(two, 0, j); d.woy = hp.din3(two, 1, j); d.woz = hp.din3(two, 2, j);
        d.nx = hp.din3(tn, 0, j); d.ny = hp.din3(tn, 1, j); d.nz = hp.din3(tn, 2, j); d.rough = hp.din(kr, j);
      }
      QueryArgs a;
      fill_query_args(m, d, use_ema, a);
      a.do_sample = 1;
      a.u = ku >= 0 ? hp.din(ku, j) : nullptr;
      a.seed = seed;
      a.offset = offset + (uint64_t)j * (uint64_t)hp.C;   // Philox counter = global sample index
      if (fused) {
        a.wx = hp.din3(tq, 0, j); a.wy = hp.din3(tq, 1, j); a.wz = hp.din3(tq, 2, j);
        a.pdf = hp.dout(kpq, j);
      }
      a.sx = hp.dout3(tw, 0, j); a.sy = hp.dout3(tw, 1, j); a.sz = hp.dout3(tw, 2, j); a.spdf = hp.dout(kp, j);
      npm_status rr = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
      if (rr != NPM_OK) return rr;
      return query_launch(m, a, st);
    });
    if (r != NPM_OK) return fail(r, hp.err != cudaSuccess ? cudaGetErrorString(hp.err) : "pipelined sample");
    return NPM_OK;
  }
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const size_t n = (size_t)q->n;
  QueryArgs a;
  fill_query_args(m, d, use_ema, a);
  a.do_sample = 1;
  a.u = s.in(u, 3 * n);
  a.seed = seed;
  a.offset = offset;
  if (fused) {
    a.wx = s.in(qx, n); a.wy = s.in(qy, n); a.wz = s.in(qz, n);
    a.pdf = s.out(pdf_q, n);
  }
  a.sx = s.out(wix, n); a.sy = s.out(wiy, n); a.sz = s.out(wiz, n); a.spdf = s.out(pdf, n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  npm_status r = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
  if (r != NPM_OK) return r;
  const char* dbg = getenv("NPM_DEBUG");
  if (dbg && (atoi(dbg) & 4)) {   // measurement only: per-phase stamps of CTA 0 (NPM_QUERY_STAMPS builds)
    CUDA_TRY(m->dbg_clock.ensure(2 * 64 * 16 * sizeof(long long)));
    a.dbg_clock = static_cast<long long*>(m->dbg_clock.p);
    CUDA_TRY(cudaMemsetAsync(a.dbg_clock, 0, 2 * 64 * 16 * sizeof(long long), st));
  }
  r = query_launch(m, a, st);
  if (r != NPM_OK) return r;
  if (a.dbg_clock) {
    long long h[2 * 64 * 16];
    CUDA_TRY(cudaMemcpyAsync(h, a.dbg_clock, sizeof(h), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int ser = 0; ser < 2; ++ser) {   // series 0: chain / r01 kernel; 1: query_ws memory warps
      const long long* hs = h + ser * 64 * 16;
      double since[16] = {};
      int cs = 0;
      for (int t = 1; t < 63; ++t) {
        if (hs[(t + 1) * 16] == 0) break;
        for (int j = 1; j < 15; ++j) if (hs[t * 16 + j]) since[j] += (double)(hs[t * 16 + j] - hs[t * 16]);
        since[15] += (double)(hs[(t + 1) * 16] - hs[t * 16]);
        ++cs;
      }
      if (!cs) continue;
      fprintf(stderr, "NPM_QSTAMPS%s tiles=%d", ser ? "_MEM" : "", cs);
      for (int j = 1; j < 16; ++j) fprintf(stderr, " s%d=%.0f", j, since[j] / cs);
      fprintf(stderr, "\n");
    }
  }
  CUDA_TRY(s.finish());
  return NPM_OK;
}

npm_status npm_sample_cosine_product(npm_model* m, const npm_query* q, const float* nx, const float* ny,
                                     const float* nz, float kappa_c, const float* u, uint64_t seed, uint64_t offset,
                                     int use_ema, float* wix, float* wiy, float* wiz, float* pdf, const float* qx,
                                     const float* qy, const float* qz, float* pdf_q, float* lambda, float* kappa,
                                     float* mu, void* stream) {
  if (!m || !query_ok(m, q) || !(kappa_c >= 0.0f && kappa_c <= 1e5f) ||
      (q->n > 0 && (!nx || !ny || !nz || !wix || !wiy || !wiz || !pdf)))
    return fail(NPM_ERR_INVALID, "bad argument");
  const bool fused = qx && qy && qz && pdf_q;
  if ((qx || qy || qz || pdf_q) && !fused) return fail(NPM_ERR_INVALID, "fused query needs qx, qy, qz, pdf_q");
  if (q->n == 0) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const size_t n = (size_t)q->n;
  const size_t K = (size_t)m->cfg.n_lobes;
  QueryArgs a;
  fill_query_args(m, d, use_ema, a);
  a.do_sample = 1;
  a.cos_product = 1;
  a.kappa_c = kappa_c;
  {
    const double kc = kappa_c;
    const double r = kc > 0.0 ? kc / -std::expm1(-2.0 * kc) : 0.5;
    a.log_c_kc = (float)(std::log(r) - std::log(2.0 * 3.14159265358979323846));
  }
  a.u = s.in(u, 3 * n);
  a.seed = seed;
  a.offset = offset;
  a.bnx = s.in(nx, n); a.bny = s.in(ny, n); a.bnz = s.in(nz, n);
  if (fused) {
    a.wx = s.in(qx, n); a.wy = s.in(qy, n); a.wz = s.in(qz, n);
    a.pdf = s.out(pdf_q, n);
  }
  a.sx = s.out(wix, n); a.sy = s.out(wiy, n); a.sz = s.out(wiz, n); a.spdf = s.out(pdf, n);
  a.lambda = s.out(lambda, K * n);
  a.kappa = s.out(kappa, K * n);
  a.mu = s.out(mu, 3 * K * n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  npm_status r = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
  if (r != NPM_OK) return r;
  r = query_launch(m, a, st);
  if (r != NPM_OK) return r;
  CUDA_TRY(s.finish());
  return NPM_OK;
}

npm_status npm_combined_sample(npm_model* m, const npm_query* q, const float* nx, const float* ny,
                               const float* nz, float alpha, const float* u, uint64_t seed, uint64_t offset,
                               int use_ema, float* wix, float* wiy, float* wiz, float* pdf, float* guide_pdf,
                               int32_t* technique, void* stream) {
  if (!m || !query_ok(m, q) || !(alpha >= 0.0f && alpha <= 1.0f) ||
      (q->n > 0 && (!nx || !ny || !nz || !wix || !wiy || !wiz || !pdf)))
    return fail(NPM_ERR_INVALID, "bad argument");
  if (q->n == 0) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const size_t n = (size_t)q->n;
  QueryArgs a;
  fill_query_args(m, d, use_ema, a);
  a.do_sample = 1;
  a.combined = 1;
  a.alpha = alpha;
  a.u = s.in(u, 4 * n);
  a.seed = seed;
  a.offset = offset;
  a.bnx = s.in(nx, n); a.bny = s.in(ny, n); a.bnz = s.in(nz, n);
  a.sx = s.out(wix, n); a.sy = s.out(wiy, n); a.sz = s.out(wiz, n); a.spdf = s.out(pdf, n);
  a.gpdf = s.out(guide_pdf, n);
  a.tech = s.out(technique, n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  npm_status r = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
  if (r != NPM_OK) return r;
  r = query_launch(m, a, st);
  if (r != NPM_OK) return r;
  CUDA_TRY(s.finish());
  return NPM_OK;
}

npm_status npm_unwind_records(npm_model* m, const float* le, const float* fs, const float* cos_theta,
                              const float* pdf, const int32_t* depth, int channels, int max_depth, int64_t n_paths,
                              int product, float* target, void* stream) {
  if (!m || n_paths < 0 || max_depth < 0 || (channels != 1 && channels != 3) ||
      (n_paths > 0 && max_depth > 0 && (!le || !fs || !cos_theta || !pdf || !depth || !target)))
    return fail(NPM_ERR_INVALID, "bad argument");
  if (n_paths == 0 || max_depth == 0) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Stager s{m, st};
  const size_t nv = (size_t)max_depth * (size_t)n_paths, nc = (size_t)channels * nv;
  UnwindArgs a;
  a.le = s.in(le, nc); a.fs = s.in(fs, nc); a.cosv = s.in(cos_theta, nv); a.pdf = s.in(pdf, nv);
  a.depth = s.in(depth, (size_t)n_paths);
  a.target = s.out(target, nc);
  a.channels = channels; a.max_depth = max_depth; a.n = n_paths; a.product = product ? 1 : 0;
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  npm_status r = check_launch(m, timed(m, kKUnwind, st, [&] { return launch_unwind(a, m->num_sms, st); }));
  if (r != NPM_OK) return r;
  CUDA_TRY(s.finish());
  return NPM_OK;
}

// ---------------------------------------------------------------------------
static npm_status read_stats(npm_model* m, cudaStream_t st, npm_step_stats* out, bool train_part, bool opt_part) {
  double ds[2];
  unsigned long long dc[4];
  CUDA_TRY(cudaMemcpyAsync(ds, m->dstats, sizeof(ds), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(dc, m->dcount, sizeof(dc), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (train_part) {
    out->loss_proxy = ds[0];
    out->n_used = (int64_t)dc[0];
    out->n_zero_target = (int64_t)dc[1];
    out->n_dropped = (int64_t)dc[2];
  }
  if (opt_part) {
    out->grad_norm_sq = ds[1];
    out->n_nonfinite_grad = (int64_t)dc[3];
  }
  return NPM_OK;
}

// Add the per-SM private copies of the privatised levels into GRADS (and zero them).
static npm_status fold_priv(npm_model* m, cudaStream_t st) {
  FoldArgs f;
  memset(&f, 0, sizeof(f));
  f.priv = static_cast<float4*>(m->priv.p);
  f.priv_stride = m->priv_stride;
  f.ctas = m->num_sms;
  f.grads = m->buf[NPM_BUF_GRADS] + m->n_mlp;
  for (int l = 0; l < m->cfg.n_levels; ++l) {
    if (!((m->priv_mask >> l) & 1u)) continue;
    f.lev_priv_off[f.nlev] = m->priv_off[l];
    f.lev_grid_off[f.nlev] = m->grid.off[l];
    f.lev_entries[f.nlev] = m->grid.tsize[l];
    ++f.nlev;
  }
  return check_launch(m, timed(m, kKFold, st, [&] { return launch_fold_priv(f, m->num_sms, st); }));
}

static npm_status accumulate(npm_model* m, const npm_query* q, const float* wix, const float* wiy,
                             const float* wiz, const float* target, int channels, const float* spdf,
                             int64_t n_global, cudaStream_t st, Stager& s, int64_t target_stride = -1,
                             bool reset_stats = true) {
  const size_t n = (size_t)q->n;
  npm_query d;
  stage_query(s, m, q, d);
  TrainArgs a;
  memset(&a, 0, sizeof(a));
  a.n = q->n;
  a.px = d.px; a.py = d.py; a.pz = d.pz;
  a.wox = d.wox; a.woy = d.woy; a.woz = d.woz; a.nx = d.nx; a.ny = d.ny; a.nz = d.nz; a.rough = d.rough;
  a.wx = s.in(wix, n); a.wy = s.in(wiy, n); a.wz = s.in(wiz, n);
  a.target = s.in(target, (size_t)channels * n);
  a.target_stride = target_stride < 0 ? (int64_t)n : target_stride;   // strided only for device slices
  a.channels = channels;
  a.spdf = s.in(spdf, n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  a.inv_n_global = 1.0 / (double)n_global;
  a.params = m->buf[NPM_BUF_PARAMS];
  a.grads = m->buf[NPM_BUF_GRADS];
  a.grid = m->grid;
  a.log_kmin = logf(m->cfg.kappa_min);
  a.log_kmax = logf(m->cfg.kappa_max);
  a.stats = m->dstats;
  a.counters = m->dcount;
  if (const char* e = getenv("NPM_DEBUG")) a.debug = atoi(e);   // measurement only
  a.divergence = m->cfg.divergence;
  a.ws = m->train_ws;
  if (m->n_alpha) {
    if (!d.bsdf_pdf) return fail(NPM_ERR_INVALID, "learn_alpha: training records need bsdf_pdf");
    a.alpha_w = m->buf[NPM_BUF_PARAMS] + m->n_mlp + m->n_grid;
    a.alpha_g = m->buf[NPM_BUF_GRADS] + m->n_mlp + m->n_grid;
    a.bsdf_pdf = d.bsdf_pdf;
  }
  CUDA_TRY(m->wimg.ensure(64 * 1024));
  a.wimg = static_cast<uint8_t*>(m->wimg.p);
  a.wimg_bytes = 64 * 1024;
  if (m->priv_mask) {
    a.priv = static_cast<float4*>(m->priv.p);
    a.priv_mask = m->priv_mask;
    a.priv_stride = m->priv_stride;
    for (int l = 0; l < 16; ++l) a.priv_off[l] = m->priv_off[l];
  }
  const NetShape& sh = m->shape;
  {
    if (reset_stats) {
      CUDA_TRY(cudaMemsetAsync(m->dstats, 0, sizeof(double), st));
      CUDA_TRY(cudaMemsetAsync(m->dcount, 0, 3 * sizeof(unsigned long long), st));
    }
    // Training batches are not binned by default: measured on B200 (c2) the
    // coherent gathers gain ~50 us but the scatter-adds then collide on the
    // same L2 lines (+54 us) and the binning pass costs ~85 us (NPM_BIN_TRAIN=1).
    if (m->bin_train) {
      npm_status r = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
      if (r != NPM_OK) return r;
    }
    if (a.debug & 4) {   // measurement only: per-phase clock stamps of CTA 0
      CUDA_TRY(m->dbg_clock.ensure(2 * 64 * 16 * sizeof(long long)));
      long long* dclk = static_cast<long long*>(m->dbg_clock.p);
      cudaMemsetAsync(dclk, 0, 2 * 64 * 16 * sizeof(long long), st);
      a.dbg_clock = dclk;
      npm_status r = check_launch(m, timed(m, kKTrainFused, st, [&] { return launch_train_tc(sh, a, m->num_sms, st); }));
      if (r == NPM_OK) r = bin_release(m, st, a.perm);
      long long h[2 * 64 * 16];
      cudaMemcpyAsync(h, dclk, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      double acc[16] = {};
      int cnt = 0;
      for (int t = 1; t < 64; ++t) {   // skip tile 0 (weight staging)
        if (h[t * 16 + 15] == 0) break;
        for (int j = 1; j < 16; ++j) {
          long long prev = 0;   // the last stamp before j (13, 14 unused below NL = 4)
          for (int i = j - 1; i >= 0 && !prev; --i) prev = h[t * 16 + i];
          if (h[t * 16 + j]) acc[j] += (double)(h[t * 16 + j] - prev);
        }
        acc[0] += (double)(h[t * 16 + 15] - h[t * 16 + 0]);
        ++cnt;
      }
      fprintf(stderr, "NPM_PHASES tiles=%d total=%.0f", cnt, cnt ? acc[0] / cnt : 0.0);
      for (int j = 1; j < 16; ++j) fprintf(stderr, " p%d=%.0f", j, cnt ? acc[j] / cnt : 0.0);
      fprintf(stderr, "\n");
      // the same stamps as cycles since the tile's stamp 0 (stamp indices need
      // not be in time order)
      double since[16] = {};
      int cs = 0;
      for (int t = 1; t < 64; ++t) {
        if (h[t * 16 + 15] == 0) break;
        for (int j = 1; j < 16; ++j) if (h[t * 16 + j]) since[j] += (double)(h[t * 16 + j] - h[t * 16]);
        ++cs;
      }
      fprintf(stderr, "NPM_STAMPS");
      for (int j = 1; j < 16; ++j) fprintf(stderr, " s%d=%.0f", j, cs ? since[j] / cs : 0.0);
      fprintf(stderr, "\n");
      // warp-specialised kernel: the memory role's stamps of the same tiles
      // (gather of tile t: m0..m3; scatter of tile t-1: m4..m6), cycles since
      // the chain's stamp 0 of tile t
      double ms[16] = {};
      int cm = 0;
      for (int t = 2; t < 63; ++t) {
        if (h[t * 16 + 15] == 0 || h[1024 + t * 16] == 0) break;
        for (int j = 0; j < 7; ++j) if (h[1024 + t * 16 + j]) ms[j] += (double)(h[1024 + t * 16 + j] - h[t * 16]);
        ++cm;
      }
      if (cm) {
        fprintf(stderr, "NPM_MEMSTAMPS");
        for (int j = 0; j < 7; ++j) fprintf(stderr, " m%d=%.0f", j, ms[j] / cm);
        fprintf(stderr, "\n");
      }
      if (r != NPM_OK || !a.priv_mask) return r;
      return fold_priv(m, st);
    }
    npm_status r = check_launch(m, timed(m, kKTrainFused, st, [&] { return launch_train_tc(sh, a, m->num_sms, st); }));
    if (r == NPM_OK) r = bin_release(m, st, a.perm);
    if (r != NPM_OK || !a.priv_mask) return r;
    return fold_priv(m, st);
  }
}

static bool train_args_ok(const npm_model* m, const npm_query* q, const float* wix, const float* wiy,
                          const float* wiz, const float* target, int channels, const float* spdf, int64_t n_global) {
  if (!m || !query_ok(m, q)) return false;
  if (channels != 1 && channels != 3) return false;
  if (q->n > 0 && (!wix || !wiy || !wiz || !target || !spdf)) return false;
  if (n_global < q->n || n_global <= 0) return false;
  return true;
}

// accumulate() over host arrays through HostPipe (all-host batches); returns
// NPM_ERR_STATE when the batch does not qualify (caller takes the plain path).
static npm_status accumulate_pipelined(npm_model* m, const npm_query* q, const float* wix, const float* wiy,
                                       const float* wiz, const float* target, int channels, const float* spdf,
                                       int64_t n_global, cudaStream_t st) {
  const bool prod = m->cfg.mode == NPM_PRODUCT;
  if (!HostPipe::usable(m, q->n, {q->px, q->py, q->pz, prod ? q->wox : nullptr, prod ? q->nx : nullptr,
                                                prod ? q->rough : nullptr, wix, wiy, wiz, target, spdf}))
    return NPM_ERR_STATE;
  HostPipe hp{m, st, q->n};
  hp.kind = 1;
  const HostPipe::Tri tx = hp.in3(q->px, q->py, q->pz);
  HostPipe::Tri two{}, tn{};
  int kr = -1;
  if (prod) {
    two = hp.in3(q->wox, q->woy, q->woz);
    tn = hp.in3(q->nx, q->ny, q->nz);
    kr = (int)hp.ins.size();
    hp.ins.push_back({q->rough, nullptr, 1});
  }
  const HostPipe::Tri tw = hp.in3(wix, wiy, wiz);
  const int kt = (int)hp.ins.size();
  hp.ins.push_back({target, nullptr, channels});
  hp.ins.push_back({spdf, nullptr, 1});
  const npm_status r = hp.run([&](int j, int64_t c) -> npm_status {
    npm_query d{};
    d.n = c;
    d.px = hp.din3(tx, 0, j); d.py = hp.din3(tx, 1, j); d.pz = hp.din3(tx, 2, j);
    if (prod) {
      d.wox = hp.din3(two, 0, j); d.woy = hp.din3(two, 1, j); d.woz = hp.din3(two, 2, j);
      d.nx = hp.din3(tn, 0, j); d.ny = hp.din3(tn, 1, j); d.nz = hp.din3(tn, 2, j); d.rough = hp.din(kr, j);
    }
    Stager s2{m, st};   // device chunk pointers: pass-through
    return accumulate(m, &d, hp.din3(tw, 0, j), hp.din3(tw, 1, j), hp.din3(tw, 2, j), hp.din(kt, j), channels,
                      hp.din(kt + 1, j), n_global, st, s2, -1, j == 0);
  });
  if (r != NPM_OK) return fail(r, hp.err != cudaSuccess ? cudaGetErrorString(hp.err) : "pipelined accumulate");
  return NPM_OK;
}

npm_status npm_accumulate_grads(npm_model* m, const npm_query* q, const float* wix, const float* wiy,
                                const float* wiz, const float* target, int channels, const float* spdf,
                                int64_t n_global, npm_step_stats* stats, void* stream) {
  if (!train_args_ok(m, q, wix, wiy, wiz, target, channels, spdf, n_global))
    return fail(NPM_ERR_INVALID, "bad argument");
  if (stats) memset(stats, 0, sizeof(*stats));
  if (q->n == 0) return NPM_OK;
  DeviceGuard g(m->device);
  std::lock_guard<std::mutex> lk(m->stage_mu);
  cudaStream_t st = (cudaStream_t)stream;
  npm_status r = accumulate_pipelined(m, q, wix, wiy, wiz, target, channels, spdf, n_global, st);
  if (r == NPM_ERR_STATE) {
    Stager s{m, st};
    r = accumulate(m, q, wix, wiy, wiz, target, channels, spdf, n_global, st, s);
  }
  if (r != NPM_OK) return r;
  if (stats) return read_stats(m, st, stats, true, false);
  return NPM_OK;
}

// Adam (+ EMA) over [begin, begin + count) of the flat vector (the whole
// vector, or a ZeRO-1 shard); statistics over that range.
static npm_status adam_range(npm_model* m, int64_t begin, int64_t count, bool ema, cudaStream_t st) {
  const npm_config& c = m->cfg;
  AdamArgs a;
  a.n_total = count;
  a.n_mlp = m->n_mlp - begin < 0 ? 0 : (m->n_mlp - begin > count ? count : m->n_mlp - begin);
  const int64_t ge = m->n_mlp + m->n_grid - begin;
  a.grid_end = ge < 0 ? 0 : (ge > count ? count : ge);
  a.p = m->buf[NPM_BUF_PARAMS] + begin; a.g = m->buf[NPM_BUF_GRADS] + begin; a.m = m->buf[NPM_BUF_ADAM_M] + begin;
  a.v = m->buf[NPM_BUF_ADAM_V] + begin; a.e = m->buf[NPM_BUF_EMA] + begin;
  a.lr = c.lr; a.beta1 = c.beta1; a.beta2 = c.beta2; a.eps = c.adam_eps; a.decay = c.ema_decay;
  a.c1 = (float)(1.0 / (1.0 - std::pow((double)c.beta1, (double)m->t)));
  a.c2 = (float)(1.0 / (1.0 - std::pow((double)c.beta2, (double)m->t)));
  a.ema = ema ? 1 : 0;
  a.gnorm = m->dstats + 1;
  a.nonfinite = m->dcount + 3;
  CUDA_TRY(cudaMemsetAsync(m->dstats + 1, 0, sizeof(double), st));
  CUDA_TRY(cudaMemsetAsync(m->dcount + 3, 0, sizeof(unsigned long long), st));
  return check_launch(m, timed(m, kKAdam, st, [&] { return launch_adam(a, m->num_sms, st); }));
}

// ZeRO-1 after the shard's Adam: GRADS outside the shard back to zero (the
// shard's part was zeroed by Adam) -- the next accumulation starts from zero.
static npm_status zero_grads_outside(npm_model* m, int64_t begin, int64_t count, cudaStream_t st) {
  float* g = m->buf[NPM_BUF_GRADS];
  if (begin > 0) CUDA_TRY(cudaMemsetAsync(g, 0, (size_t)begin * sizeof(float), st));
  const int64_t end = begin + count, cap = m->n_total + kBufPad;
  if (end < cap) CUDA_TRY(cudaMemsetAsync(g + end, 0, (size_t)(cap - end) * sizeof(float), st));
  return NPM_OK;
}

static npm_status optimizer(npm_model* m, cudaStream_t st) {
  if (m->comm && m->exchange == NPM_EXCHANGE_ZERO1 && m->comm_world > 1) {
    // ZeRO-1: reduce-scatter GRADS, Adam on this rank's 1/P,
    // all-gather PARAMS, EMA locally over the whole (replicated) vector --
    // the same result as allreduce + replicated Adam + EMA, with 1/P of the
    // optimiser's m / v traffic per rank and no EMA exchange
    int64_t b, c, ch;
    shard_of(m, m->comm_rank, m->comm_world, b, c, ch);
    float* g = m->buf[NPM_BUF_GRADS];
    ncclResult_t e = nccl().reduce_scatter(g, g + b, (size_t)ch, ncclFloat32, ncclSum, m->comm, st);
    if (e != ncclSuccess) return nccl_fail(e, "ncclReduceScatter(GRADS)");
    m->t += 1;
    npm_status r = adam_range(m, b, c, false, st);
    if (r != NPM_OK) return r;
    if ((r = zero_grads_outside(m, b, c, st)) != NPM_OK) return r;
    float* p = m->buf[NPM_BUF_PARAMS];
    e = nccl().all_gather(p + b, p, (size_t)ch, ncclFloat32, m->comm, st);
    if (e != ncclSuccess) return nccl_fail(e, "ncclAllGather(PARAMS)");
    // the statistics of the step are sums over the shards
    e = nccl().all_reduce(m->dstats + 1, m->dstats + 1, 1, ncclFloat64, ncclSum, m->comm, st);
    if (e == ncclSuccess) e = nccl().all_reduce(m->dcount + 3, m->dcount + 3, 1, ncclUint64, ncclSum, m->comm, st);
    if (e != ncclSuccess) return nccl_fail(e, "ncclAllReduce(stats)");
    return check_launch(m, timed(m, kKAdam, st, [&] {
      return launch_ema(m->buf[NPM_BUF_EMA], p, m->n_total, m->cfg.ema_decay, m->num_sms, st);
    }));
  }
  if (m->comm) {   // A11: the one exchange step -- sum of the ranks' GRADS (each already / N_global)
    const ncclResult_t e = nccl().all_reduce(m->buf[NPM_BUF_GRADS], m->buf[NPM_BUF_GRADS], (size_t)m->n_total,
                                             ncclFloat32, ncclSum, m->comm, st);
    if (e != ncclSuccess) return nccl_fail(e, "ncclAllReduce(GRADS)");
  }
  m->t += 1;
  return adam_range(m, 0, m->n_total, true, st);
}

npm_status npm_train_stream(npm_model* m, const npm_query* q, const float* wix, const float* wiy,
                            const float* wiz, const float* target, int channels, const float* spdf,
                            int64_t micro_batch, npm_step_stats* per_step, void* stream) {
  if (!train_args_ok(m, q, wix, wiy, wiz, target, channels, spdf, q ? (q->n > 0 ? q->n : 1) : 1) ||
      micro_batch <= 0)
    return fail(NPM_ERR_INVALID, "bad argument");
  if (q->n == 0) return NPM_OK;
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(m->stage_mu);
  // stage the whole frame batch once; micro-steps then address device slices
  Stager s{m, st};
  npm_query d;
  stage_query(s, m, q, d);
  const int64_t n = q->n;
  const float* dwx = s.in(wix, (size_t)n);
  const float* dwy = s.in(wiy, (size_t)n);
  const float* dwz = s.in(wiz, (size_t)n);
  const float* dtg = s.in(target, (size_t)channels * n);
  const float* dpd = s.in(spdf, (size_t)n);
  if (s.err != cudaSuccess) return fail(NPM_ERR_CUDA, cudaGetErrorString(s.err));
  int64_t j = 0;
  for (int64_t a0 = 0; a0 < n; a0 += micro_batch, ++j) {
    const int64_t b = a0 + micro_batch < n ? micro_batch : n - a0;
    npm_query sub = d;
    sub.n = b;
    auto sl = [&](const float* p) { return p ? p + a0 : p; };
    sub.px = sl(d.px); sub.py = sl(d.py); sub.pz = sl(d.pz);
    sub.wox = sl(d.wox); sub.woy = sl(d.woy); sub.woz = sl(d.woz);
    sub.nx = sl(d.nx); sub.ny = sl(d.ny); sub.nz = sl(d.nz); sub.rough = sl(d.rough);
    sub.bsdf_pdf = sl(d.bsdf_pdf);
    Stager s2{m, st};   // device slices: pass-through
    // one optimisation step per micro-batch: Eq. 9's 1/N over the micro-batch
    npm_status r = accumulate(m, &sub, dwx + a0, dwy + a0, dwz + a0, dtg + a0, channels, dpd + a0, b, st, s2, n);
    if (r != NPM_OK) return r;
    if ((r = optimizer(m, st)) != NPM_OK) return r;
    if (per_step) {
      memset(per_step + j, 0, sizeof(npm_step_stats));
      if ((r = read_stats(m, st, per_step + j, true, true)) != NPM_OK) return r;
    }
  }
  return NPM_OK;
}

npm_status npm_step_stats_async(npm_model* m, npm_step_stats* out, void* stream) {
  if (!m || !out) return fail(NPM_ERR_INVALID, "bad argument");
  static_assert(sizeof(npm_step_stats) == 2 * sizeof(double) + 4 * sizeof(int64_t), "stats layout");
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  // device: dstats = {loss, grad_norm_sq}, dcount = {used, zero, dropped, nonfinite}: the struct's order
  CUDA_TRY(cudaMemcpyAsync(&out->loss_proxy, m->dstats, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&out->n_used, m->dcount, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  return NPM_OK;
}

npm_status npm_optimizer_step(npm_model* m, npm_step_stats* stats, void* stream) {
  if (!m) return fail(NPM_ERR_INVALID, "null model");
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  npm_status r = optimizer(m, st);
  if (r != NPM_OK) return r;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    return read_stats(m, st, stats, false, true);
  }
  return NPM_OK;
}

npm_status npm_optimizer_step_shard(npm_model* m, int rank, int world, npm_step_stats* stats, void* stream) {
  if (!m || world < 1 || world > kMaxShardWorld || rank < 0 || rank >= world) return fail(NPM_ERR_INVALID, "bad argument");
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  int64_t b, c, ch;
  shard_of(m, rank, world, b, c, ch);
  m->t += 1;
  npm_status r = adam_range(m, b, c, false, st);
  if (r != NPM_OK) return r;
  if ((r = zero_grads_outside(m, b, c, st)) != NPM_OK) return r;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    return read_stats(m, st, stats, false, true);
  }
  return NPM_OK;
}

npm_status npm_ema_update(npm_model* m, void* stream) {
  if (!m) return fail(NPM_ERR_INVALID, "null model");
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  return check_launch(m, timed(m, kKAdam, st, [&] {
    return launch_ema(m->buf[NPM_BUF_EMA], m->buf[NPM_BUF_PARAMS], m->n_total, m->cfg.ema_decay, m->num_sms, st);
  }));
}

npm_status npm_frame_step(npm_model* m, const npm_query* q, const float* u, uint64_t seed, uint64_t offset,
                          int use_ema, float* wix, float* wiy, float* wiz, float* pdf, const float* qx,
                          const float* qy, const float* qz, float* pdf_q, const npm_query* tq, const float* twx,
                          const float* twy, const float* twz, const float* target, int channels,
                          const float* spdf, int64_t n_global, npm_step_stats* stats, void* stream) {
  if (!m || !query_ok(m, q) || (q->n > 0 && (!wix || !wiy || !wiz || !pdf)))
    return fail(NPM_ERR_INVALID, "bad argument");
  if (!train_args_ok(m, tq, twx, twy, twz, target, channels, spdf, n_global)) return fail(NPM_ERR_INVALID, "bad argument");
  const bool fused = qx && qy && qz && pdf_q;
  if ((qx || qy || qz || pdf_q) && !fused) return fail(NPM_ERR_INVALID, "fused query needs qx, qy, qz, pdf_q");
  if (stats) memset(stats, 0, sizeof(*stats));
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  const bool prod = m->cfg.mode == NPM_PRODUCT;
  // one chunked pipeline over both phases when every array is a host pointer
  // and the two batches have the same size (a record per queried vertex)
  if (q->n == tq->n && q->n > 0 &&
      HostPipe::usable(m, q->n, {q->px, q->py, q->pz, prod ? q->wox : nullptr, prod ? q->nx : nullptr,
                                 prod ? q->rough : nullptr, u, qx, wix, pdf, pdf_q, tq->px, tq->py, tq->pz,
                                 prod ? tq->wox : nullptr, prod ? tq->nx : nullptr, prod ? tq->rough : nullptr, twx,
                                 twy, twz, target, spdf})) {
    std::lock_guard<std::mutex> lk(m->stage_mu);
    HostPipe hp{m, st, q->n};
    auto cond = [&](const npm_query* qq, HostPipe::Tri& two, HostPipe::Tri& tn, int& kr) {
      if (!prod) return;
      two = hp.in3(qq->wox, qq->woy, qq->woz);
      tn = hp.in3(qq->nx, qq->ny, qq->nz);
      kr = (int)hp.ins.size();
      hp.ins.push_back({qq->rough, nullptr, 1});
    };
    const HostPipe::Tri tx = hp.in3(q->px, q->py, q->pz);
    HostPipe::Tri two{}, tn{}, ttwo{}, ttn{};
    int kr = -1, tkr = -1;
    cond(q, two, tn, kr);
    const int ku = u ? (int)hp.ins.size() : -1;
    if (u) hp.ins.push_back({u, nullptr, 3});
    HostPipe::Tri tqd{};
    if (fused) tqd = hp.in3(qx, qy, qz);
    const HostPipe::Tri ttx = hp.in3(tq->px, tq->py, tq->pz);
    cond(tq, ttwo, ttn, tkr);
    const HostPipe::Tri tw = hp.in3(twx, twy, twz);
    const int kt = (int)hp.ins.size();
    hp.ins.push_back({target, nullptr, channels});
    hp.ins.push_back({spdf, nullptr, 1});
    const HostPipe::Tri to = hp.out3(wix, wiy, wiz);
    const int kp = (int)hp.outs.size();
    hp.outs.push_back({nullptr, pdf, 1});
    const int kpq = (int)hp.outs.size();
    if (fused) hp.outs.push_back({nullptr, pdf_q, 1});
    const npm_status r = hp.run([&](int j, int64_t c) -> npm_status {
      // queries of chunk j (EMA or live weights; GRADS untouched) ...
      npm_query d{};
      d.n = c;
      d.px = hp.din3(tx, 0, j); d.py = hp.din3(tx, 1, j); d.pz = hp.din3(tx, 2, j);
      if (prod) {
        d.wox = hp.din3(two, 0, j); d.woy = hp.din3(two, 1, j); d.woz = hp.din3(two, 2, j);
        d.nx = hp.din3(tn, 0, j); d.ny = hp.din3(tn, 1, j); d.nz = hp.din3(tn, 2, j); d.rough = hp.din(kr, j);
      }
      QueryArgs a;
      fill_query_args(m, d, use_ema, a);
      a.do_sample = 1;
      a.u = ku >= 0 ? hp.din(ku, j) : nullptr;
      a.seed = seed;
      a.offset = offset + (uint64_t)j * (uint64_t)hp.C;   // Philox counter = global sample index
      if (fused) {
        a.wx = hp.din3(tqd, 0, j); a.wy = hp.din3(tqd, 1, j); a.wz = hp.din3(tqd, 2, j);
        a.pdf = hp.dout(kpq, j);
      }
      a.sx = hp.dout3(to, 0, j); a.sy = hp.dout3(to, 1, j); a.sz = hp.dout3(to, 2, j); a.spdf = hp.dout(kp, j);
      npm_status rr = maybe_bin(m, a.px, a.py, a.pz, a.n, st, &a.perm);
      if (rr == NPM_OK) rr = query_launch(m, a, st);
      if (rr != NPM_OK) return rr;
      // ... then the records of chunk j into GRADS
      npm_query dt{};
      dt.n = c;
      dt.px = hp.din3(ttx, 0, j); dt.py = hp.din3(ttx, 1, j); dt.pz = hp.din3(ttx, 2, j);
      if (prod) {
        dt.wox = hp.din3(ttwo, 0, j); dt.woy = hp.din3(ttwo, 1, j); dt.woz = hp.din3(ttwo, 2, j);
        dt.nx = hp.din3(ttn, 0, j); dt.ny = hp.din3(ttn, 1, j); dt.nz = hp.din3(ttn, 2, j); dt.rough = hp.din(tkr, j);
      }
      Stager s2{m, st};   // device chunk pointers: pass-through
      return accumulate(m, &dt, hp.din3(tw, 0, j), hp.din3(tw, 1, j), hp.din3(tw, 2, j), hp.din(kt, j), channels,
                        hp.din(kt + 1, j), n_global, st, s2, -1, j == 0);
    });
    if (r != NPM_OK) return fail(r, hp.err != cudaSuccess ? cudaGetErrorString(hp.err) : "pipelined frame step");
  } else {
    npm_status r = npm_sample(m, q, u, seed, offset, use_ema, wix, wiy, wiz, pdf, qx, qy, qz, pdf_q, stream);
    if (r != NPM_OK) return r;
    if (tq->n > 0) {
      std::lock_guard<std::mutex> lk(m->stage_mu);
      Stager s{m, st};
      if ((r = accumulate(m, tq, twx, twy, twz, target, channels, spdf, n_global, st, s)) != NPM_OK) return r;
    } else {
      CUDA_TRY(cudaMemsetAsync(m->dstats, 0, sizeof(double), st));
      CUDA_TRY(cudaMemsetAsync(m->dcount, 0, 3 * sizeof(unsigned long long), st));
    }
  }
  npm_status r = optimizer(m, st);
  if (r != NPM_OK) return r;
  if (stats) return read_stats(m, st, stats, true, true);
  return NPM_OK;
}

npm_status npm_train_step(npm_model* m, const npm_query* q, const float* wix, const float* wiy,
                          const float* wiz, const float* target, int channels, const float* spdf,
                          int64_t n_global, npm_step_stats* stats, void* stream) {
  if (!train_args_ok(m, q, wix, wiy, wiz, target, channels, spdf, n_global))
    return fail(NPM_ERR_INVALID, "bad argument");
  if (stats) memset(stats, 0, sizeof(*stats));
  DeviceGuard g(m->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (q->n > 0) {
    std::lock_guard<std::mutex> lk(m->stage_mu);
    npm_status r = accumulate_pipelined(m, q, wix, wiy, wiz, target, channels, spdf, n_global, st);
    if (r == NPM_ERR_STATE) {
      Stager s{m, st};
      r = accumulate(m, q, wix, wiy, wiz, target, channels, spdf, n_global, st, s);
    }
    if (r != NPM_OK) return r;
  } else {
    CUDA_TRY(cudaMemsetAsync(m->dstats, 0, sizeof(double), st));
    CUDA_TRY(cudaMemsetAsync(m->dcount, 0, 3 * sizeof(unsigned long long), st));
  }
  npm_status r = optimizer(m, st);
  if (r != NPM_OK) return r;
  if (stats) return read_stats(m, st, stats, true, true);
  return NPM_OK;
}

}  // extern "C"
