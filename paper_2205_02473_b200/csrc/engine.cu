// libdpro_cuda.so: engine context, batch arenas, launches and the C ABI of
// include/dpro_cuda.h. Host code is plain C++ over the CUDA runtime; the
// kernels live in replay_kernel.cuh (K1) and critical_path_kernel.cuh (K3).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/cub.cuh>

#include "critical_path_kernel.cuh"
#include "memory_kernel.cuh"
#include "delta_kernel.cuh"
#include "dpro_cuda.h"
#include "overlay.h"
#include "pack_kernel.cuh"
#include "replay_fast.cuh"

static_assert(dpro_ov::kSparseMax == dpro_k::kOvListMax, "sparse overlay list capacity");
#include "replay_kernel.cuh"
#include "tsync_kernel.cuh"

struct dpro_graph;
dpro_graph* dpro_internal_tsync_graph(const dpro_cluster_desc* cluster,
                                      int64_t bytes, int32_t k,
                                      std::string* err);

namespace {

// DPRO_TRACE=1: per-phase wall times of batch registration on stderr.
struct Tracer {
  bool on = std::getenv("DPRO_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t s = nullptr, bool sync = false) {
    if (!on) return;
    if (sync) cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dpro] %-28s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

using dpro_k::Cand;
using dpro_k::CpScratch;
using dpro_k::DevSt;
using dpro_k::FastCfg;
using dpro_k::Outs;
using dpro_k::PackOut;
using dpro_k::Scratch;

constexpr int kWarpsPerBlock = 4;
constexpr size_t kSmemHeader = 16 * 8;

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    // grow by >= 1.25x so batches that keep growing (a search whose accepted
    // states add ops) do not reallocate every round
    const size_t want = std::max<size_t>(std::max(bytes, cap + cap / 4), 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {  // fall back to the exact size
      cudaGetLastError();
      e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
      if (e == cudaSuccess) cap = std::max<size_t>(bytes, 256);
      else cap = 0;
      return e;
    }
    cap = want;
    return e;
  }
  template <typename T>
  T* as(size_t byte_off = 0) const {
    return reinterpret_cast<T*>(static_cast<char*>(p) + byte_off);
  }
};

struct HostPinned {
  void* p = nullptr;
  size_t cap = 0;
  ~HostPinned() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMallocHost(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
};

// Persistent host worker threads (one pool per context): jobs are index
// ranges handed out through an atomic counter; the caller may keep working
// (e.g. issuing H2D copies) until wait().
class Pool {
 public:
  explicit Pool(int threads) {
    const int n = threads > 0 ? threads : std::max(1, (int)std::thread::hardware_concurrency());
    for (int t = 0; t < n; ++t) th_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return static_cast<int>(th_.size()); }
  void start(int32_t n, std::function<void(int32_t)> fn) {
    auto j = std::make_shared<Job>();
    j->fn = std::move(fn);
    j->n = n;
    j->left = n;
    std::lock_guard<std::mutex> g(m_);
    job_ = std::move(j);
    ++gen_;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return !job_ || job_->left == 0; });
  }
  void run(int32_t n, std::function<void(int32_t)> fn) {
    start(n, std::move(fn));
    wait();
  }

 private:
  // Every claim is tied to its job: a worker that wakes late for a finished
  // job finds that job's counter exhausted and never runs its fn, and its
  // completions are credited to that job only (not to the next one).
  struct Job {
    std::function<void(int32_t)> fn;
    int32_t n = 0;
    int32_t left = 0;  // guarded by m_
    std::atomic<int32_t> next{0};
  };
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Job> j;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        j = job_;
      }
      int32_t did = 0;
      for (int32_t i; (i = j->next.fetch_add(1)) < j->n;) {
        j->fn(i);
        ++did;
      }
      if (did) {
        std::lock_guard<std::mutex> g(m_);
        j->left -= did;
        if (j->left == 0) done_.notify_all();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace

struct dpro_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  size_t smem_optin = 0;
  int smem_per_sm = 228 * 1024;
  std::string err;
  HostPinned staging;
  std::unique_ptr<Pool> pool;  // created on first use
  int pack_clusters = 0;       // co-resident pack clusters (queried once)
  cudaStream_t copy_stream = nullptr;  // H2D of delta chunks (overlaps the merges)
  cudaStream_t side_stream = nullptr;  // overlay batches: known deep-queue candidates
  cudaEvent_t side_ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> chunk_ev;   // one per in-flight chunk copy
  int host_threads = 0;  // option "host_threads": pool size (0 = all hardware threads)
  Pool& workers() {
    if (!pool) pool = std::make_unique<Pool>(host_threads);
    return *pool;
  }
  int fast = 1;       // option "fast"
  uint32_t ring = 4;  // option "ring"
  int warps = 0;      // option "warps": warps (1, 2, 4, 8) per candidate; 0 = by device count
  int gcnt = 0;       // option "gcnt": 1 = fast-path counters always in global scratch
  int deep_first = -1;  // option "deep_first": -1 auto (mean V > 1M), 0 never, 1 always
  int overlay = 0;      // option "overlay": 1 = delta batches replay on the base + overlays
  int tsync_host = 0;   // option "tsync_host": 1 = t_sync graphs built on host threads (A/B)
  int gring0 = -1;      // option "gring0": overlay residency pass with device rings in global
                        // memory (-1 auto: multi-million-op graphs, 1 on, 0 off)
  DevBuf gring0_buf;
  DevBuf gring;         // pass 3 of the fast kernels: device rings in global memory
  dpro_batch* spare = nullptr;  // recycled arenas for repeated small calls
};

struct dpro_resident {
  DevBuf buf;
  dpro_k::ResDev dev{};
  uint32_t n = 0, e = 0, d = 0;
  bool dur32 = true;
  std::vector<uint32_t> succ_off, succ, indeg;  // host copy (edge counts)
  std::vector<int64_t> dur_h;                   // host copies for the overlay builder
  std::vector<uint16_t> dev_h;
  std::vector<uint8_t> flags_h;
  // overlay batches (overlay.h): the base packed once (a 1-candidate batch
  // over the resident CSR) and its host view
  dpro_batch* packed = nullptr;
  dpro_ov::BaseHost bh;
  dpro_k::OvBase ob{};
  ~dpro_resident();
};

// A deep host copy of a dpro_delta (overlay batches re-run rare candidates
// through the materialized path after the replay).
struct DeltaCopy {
  dpro_delta d{};
  std::vector<uint32_t> removed, new_pos, new_succ_off, new_succ, extra_src, extra_dst, cut;
  std::vector<int64_t> new_dur;
  std::vector<uint16_t> new_dev;
  std::vector<uint8_t> new_flags;
  void set(const dpro_delta& x) {
    removed.assign(x.removed, x.removed + x.n_removed);
    new_pos.assign(x.new_pos, x.new_pos + x.n_new);
    new_dur.assign(x.new_dur, x.new_dur + x.n_new);
    new_dev.assign(x.new_dev, x.new_dev + x.n_new);
    new_flags.assign(x.new_flags, x.new_flags + x.n_new);
    new_succ_off.assign(x.new_succ_off, x.new_succ_off + x.n_new + 1);
    new_succ.assign(x.new_succ, x.new_succ + x.new_succ_off[x.n_new]);
    extra_src.assign(x.extra_src, x.extra_src + x.n_extra);
    extra_dst.assign(x.extra_dst, x.extra_dst + x.n_extra);
    cut.assign(x.cut, x.cut + x.n_cut);
    d = x;
    d.removed = removed.data();
    d.new_pos = new_pos.data();
    d.new_dur = new_dur.data();
    d.new_dev = new_dev.data();
    d.new_flags = new_flags.data();
    d.new_succ_off = new_succ_off.data();
    d.new_succ = new_succ.data();
    d.extra_src = extra_src.data();
    d.extra_dst = extra_dst.data();
    d.cut = cut.data();
  }
};

struct dpro_batch {
  int32_t n = 0;
  int32_t memspace = DPRO_HOST;
  std::vector<Cand> hc;              // host copy of descriptors
  std::vector<uint32_t> n_ops, n_dev, n_edges;
  unsigned long long sum_n = 0, sum_d = 0, sum_dof = 0, sum_e = 0;
  uint32_t max_d = 0;
  DevBuf arena;   // uploaded CSR (host memspace)
  DevBuf desc;    // Cand[n]
  DevBuf scratch; // op / device scratch
  DevBuf outs;    // results
  DevBuf work;    // work counter
  DevBuf cp;      // critical-path scratch
  DevBuf pack;    // packed replay layout (rec, erec, cnt0, offsets, info)
  DevBuf dblob;   // uploaded deltas (delta batches)
  DevBuf ddesc;   // DeltaDev[n]
  DevBuf rank;    // merge rank scratch
  DevBuf pred1;   // delta batches: a predecessor per op (written by the merge)
  const dpro_resident* res = nullptr;  // delta batches: the base
  uint32_t smem_ind = 0;               // merge kernel in-degree smem words
  size_t s_cnt0 = 0;
  Scratch S{};
  Outs O{};
  PackOut P{};
  FastCfg F{};
  int blocks_per_sm_fast = 0;
  std::vector<dpro_k::PackInfo> info;  // host copy (read once after pack)
  bool replayed = false;
  bool with_schedule = false;
  bool qpos_ready = false;  // qpos derived from qbuf since the last replay
  // overlay batches: candidates replayed on the resident base + overlays
  bool overlay = false;
  std::vector<dpro_ov::OverlayHost> ovh;
  std::vector<DeltaCopy> dcopy;
  std::vector<size_t> ov_off;   // per candidate byte offset in ovstage / ovarena
  size_t ov_bytes = 0;
  DevBuf ovarena;               // overlay arrays
  DevBuf ovdesc;                // OvCand[n]
  DevBuf ovgcnt;                // global counters (when they do not fit smem)
  std::vector<dpro_k::OvCand> ovc;
  HostPinned ovstage;           // host image of ovarena (pinned: fast H2D)
  uint32_t max_cnt_ov = 0;      // max base + overlay counters of a candidate
  int32_t n_mat = 0;            // candidates re-run through the materialized path
  uint32_t ring_hint = 0;       // residency-pass ring capacity learned from the last replay
  std::vector<int32_t> g3;      // candidates that needed global rings (run first next time)
  DevBuf hint;                  // device list of this replay's global-ring candidates
  DevBuf order;                 // candidate order of the residency pass: long ones first,
                                // then [n] side-stream flags (pass 4 candidates)
  std::vector<uint32_t> side_h;
  bool side_any = false;
  // pass timing of the last fast / overlay replay (dpro_cuda_batch_diag):
  // events before pass 0, after pass 0, 1, 3 and the general hand-off
  cudaEvent_t pev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool pev_valid = false;
  void mark(int k, cudaStream_t st) {
    if (!pev[k] && cudaEventCreate(&pev[k]) != cudaSuccess) return;
    cudaEventRecord(pev[k], st);
  }
  ~dpro_batch() {
    for (auto& e : pev)
      if (e) cudaEventDestroy(e);
  }
};

dpro_resident::~dpro_resident() { delete packed; }

namespace {

int set_err(dpro_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

#define CU(call)                                                          \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess)                                                \
      return set_err(ctx, e_ == cudaErrorMemoryAllocation ? DPRO_ENOMEM   \
                                                          : DPRO_ECUDA,   \
                     std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

bool fits_i32(const int64_t* d, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i)
    if (d[i] > INT32_MAX || d[i] < INT32_MIN) return false;
  return true;
}

// Uploads host CSR arrays into one device arena through pinned staging.
// Host threads (1) check which candidates' durations fit int32, (2) pack
// candidates in order into staging; the calling thread issues one H2D copy
// per finished chunk of candidates, so packing overlaps the DMA.
int upload_host(dpro_ctx* ctx, dpro_batch* b, const dpro_csr* cands) {
  Tracer tr;
  const int32_t n = b->n;
  const int nt = std::max(1, std::min<int>(n, (int)std::thread::hardware_concurrency()));
  auto parallel = [&](auto&& fn) {
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(fn, t);
    fn(0);
    for (auto& th : pool) th.join();
  };
  std::vector<uint8_t> d32(n, 0);
  {
    std::atomic<int32_t> next{0};
    parallel([&](int) {
      for (int32_t i; (i = next.fetch_add(1)) < n;) {
        const dpro_csr& c = cands[i];
        d32[i] = c.dur_bits == 32 || c.n_ops == 0 ||
                 fits_i32(static_cast<const int64_t*>(c.dur), c.n_ops);
      }
    });
  }
  std::vector<size_t> off(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    const dpro_csr& c = cands[i];
    size_t sz = align16(size_t(c.n_ops) * (d32[i] ? 4 : 8));
    sz += align16(size_t(c.n_ops) * 2);
    sz += align16(size_t(c.n_ops));
    sz += align16(size_t(c.n_ops + 1) * 4);
    sz += align16(size_t(c.n_edges) * 4);
    sz += align16(size_t(c.n_ops) * 4);
    off[i + 1] = off[i] + sz;
  }
  const size_t total = off[n];
  tr.mark("host: sizes + dur range");
  // the staging buffer may still feed an earlier in-flight upload
  CU(cudaStreamSynchronize(ctx->stream));
  CU(b->arena.ensure(total));
  CU(ctx->staging.ensure(total));
  char* stage = static_cast<char*>(ctx->staging.p);
  auto pack_one = [&](int32_t i) {
    const dpro_csr& c = cands[i];
    char* p = stage + off[i];
    size_t o = 0;
    Cand& hc = b->hc[i];
    const size_t base = off[i];
    if (d32[i]) {
      int32_t* dd = reinterpret_cast<int32_t*>(p + o);
      if (c.n_ops == 0) {
      } else if (c.dur_bits == 32) {
        std::memcpy(dd, c.dur, size_t(c.n_ops) * 4);
      } else {
        const int64_t* src = static_cast<const int64_t*>(c.dur);
        for (uint32_t k = 0; k < c.n_ops; ++k) dd[k] = static_cast<int32_t>(src[k]);
      }
      hc.dur64 = 0;
    } else {
      std::memcpy(p + o, c.dur, size_t(c.n_ops) * 8);
      hc.dur64 = 1;
    }
    hc.dur = b->arena.as<void>(base + o);
    o += align16(size_t(c.n_ops) * (d32[i] ? 4 : 8));
    if (c.n_ops) std::memcpy(p + o, c.dev, size_t(c.n_ops) * 2);
    hc.dev = b->arena.as<uint16_t>(base + o);
    o += align16(size_t(c.n_ops) * 2);
    if (c.n_ops) std::memcpy(p + o, c.flags, c.n_ops);
    hc.flags = b->arena.as<uint8_t>(base + o);
    o += align16(c.n_ops);
    if (c.succ_off)
      std::memcpy(p + o, c.succ_off, size_t(c.n_ops + 1) * 4);
    else
      std::memset(p + o, 0, 4);
    hc.succ_off = b->arena.as<uint32_t>(base + o);
    o += align16(size_t(c.n_ops + 1) * 4);
    if (c.n_edges) std::memcpy(p + o, c.succ, size_t(c.n_edges) * 4);
    hc.succ = b->arena.as<uint32_t>(base + o);
    o += align16(size_t(c.n_edges) * 4);
    uint32_t* ind = reinterpret_cast<uint32_t*>(p + o);
    if (c.indeg) {
      if (c.n_ops) std::memcpy(ind, c.indeg, size_t(c.n_ops) * 4);
    } else {
      std::memset(ind, 0, size_t(c.n_ops) * 4);
      for (uint32_t e = 0; e < c.n_edges; ++e) ind[c.succ[e]]++;
    }
    hc.indeg = b->arena.as<uint32_t>(base + o);
  };
  // chunks of ~16 MB; workers pack candidates in order, the caller copies
  std::vector<int32_t> chunk_end;
  for (int32_t i = 0; i < n;) {
    int32_t j = i + 1;
    while (j < n && off[j] - off[i] < (size_t(16) << 20)) ++j;
    chunk_end.push_back(j);
    i = j;
  }
  const int nchunks = static_cast<int>(chunk_end.size());
  std::vector<std::atomic<int32_t>> left(nchunks);
  std::vector<int> chunk_of(n);
  for (int k = 0, i = 0; k < nchunks; ++k) {
    left[k] = chunk_end[k] - i;
    for (; i < chunk_end[k]; ++i) chunk_of[i] = k;
  }
  std::atomic<int32_t> next{0};
  auto worker = [&](int) {
    for (int32_t i; (i = next.fetch_add(1)) < n;) {
      pack_one(i);
      left[chunk_of[i]].fetch_sub(1, std::memory_order_release);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(worker, t);
  int err = DPRO_OK;
  for (int k = 0, i = 0; k < nchunks; ++k) {
    while (left[k].load(std::memory_order_acquire) > 0) std::this_thread::yield();
    const size_t a = off[i], z = off[chunk_end[k]];
    if (err == DPRO_OK && z > a) {
      const cudaError_t e = cudaMemcpyAsync(b->arena.as<char>(a), stage + a, z - a,
                                            cudaMemcpyHostToDevice, ctx->stream);
      if (e != cudaSuccess) err = set_err(ctx, DPRO_ECUDA, cudaGetErrorString(e));
    }
    i = chunk_end[k];
  }
  for (auto& th : pool) th.join();
  tr.mark("host pack || H2D (issued)");
  if (err != DPRO_OK) return err;
  tr.mark("H2D", ctx->stream, true);
  return DPRO_OK;
}

int finish_batch(dpro_ctx* ctx, dpro_batch* b);
int alloc_batch(dpro_ctx* ctx, dpro_batch* b, const std::vector<uint32_t>& e_cap,
                bool upload_desc);
int run_pack(dpro_ctx* ctx, dpro_batch* b);
int launch_pack(dpro_ctx* ctx, dpro_batch* b, int32_t c0, int32_t c1);
int read_pack_info(dpro_ctx* ctx, dpro_batch* b);
int run_merge(dpro_ctx* ctx, dpro_batch* b, int32_t c0, int32_t c1);

int build_batch(dpro_ctx* ctx, dpro_batch* b, const dpro_csr* cands) {
  const int32_t n = b->n;
  b->hc.resize(n);
  b->n_ops.resize(n);
  b->n_dev.resize(n);
  b->n_edges.resize(n);
  unsigned long long so = 0, sd = 0, sdo = 0, se = 0;
  for (int32_t i = 0; i < n; ++i) {
    const dpro_csr& c = cands[i];
    if (c.n_ops > 0 && (!c.dur || !c.dev || !c.flags || !c.succ_off))
      return set_err(ctx, DPRO_EINVAL, "candidate " + std::to_string(i) + ": null CSR array");
    if (c.n_edges > 0 && !c.succ)
      return set_err(ctx, DPRO_EINVAL, "candidate " + std::to_string(i) + ": null succ");
    if (c.dur_bits != 32 && c.dur_bits != 64)
      return set_err(ctx, DPRO_EINVAL, "dur_bits must be 32 or 64");
    Cand& h = b->hc[i];
    std::memset(&h, 0, sizeof h);
    h.n = c.n_ops;
    h.e = c.n_edges;
    h.d = c.n_devices;
    h.op_off = so;
    h.dev_off = sd;
    h.dof_off = sdo;
    b->n_ops[i] = c.n_ops;
    b->n_dev[i] = c.n_devices;
    b->n_edges[i] = c.n_edges;
    b->max_d = std::max(b->max_d, c.n_devices);
    so += c.n_ops;
    sd += c.n_devices;
    sdo += c.n_devices + 1;
    se += c.n_edges;
    if (b->memspace == DPRO_DEVICE) {
      h.dur = c.dur;
      h.dur64 = c.dur_bits == 64;
      h.dev = c.dev;
      h.flags = c.flags;
      h.succ_off = c.succ_off;
      h.succ = c.succ;
      h.indeg = c.indeg;
    }
  }
  b->sum_n = so;
  b->sum_d = sd;
  b->sum_dof = sdo;
  b->sum_e = se;
  if (b->memspace == DPRO_HOST) {
    int st = upload_host(ctx, b, cands);
    if (st != DPRO_OK) return st;
  }
  return finish_batch(ctx, b);
}

// Scratch, outputs, descriptors and the pack kernel for a batch whose
// b->hc descriptors point at device CSR arrays.
int finish_batch(dpro_ctx* ctx, dpro_batch* b) {
  const int st = alloc_batch(ctx, b, b->n_edges, true);
  if (st != DPRO_OK) return st;
  return run_pack(ctx, b);
}

// Scratch, outputs and the packed layout of a batch. e_cap: per-candidate
// edge capacity of the expanded lists (exact counts, or bounds when the
// counts are not known yet); upload_desc: copy b->hc to the device.
int alloc_batch(dpro_ctx* ctx, dpro_batch* b, const std::vector<uint32_t>& e_cap,
                bool upload_desc) {
  const int32_t n = b->n;
  const unsigned long long so = b->sum_n, sd = b->sum_d, sdo = b->sum_dof;
  // scratch: indeg, qbuf, qpos, vstack (u32), sched (u8), devoff, dstate, busy
  const size_t s_u32 = align16(so * 4 + 4);
  const size_t s_u8 = align16(so + 1);
  const size_t s_dof = align16(sdo * 4 + 4);
  const size_t s_dst = align16(sd * sizeof(DevSt) + 16);
  const size_t s_busy = align16(sd * 8 + 8);
  const size_t s_dh = align16(sd * 4 + 4);
  CU(b->scratch.ensure(4 * s_u32 + s_u8 + s_dof + s_dst + s_busy + s_dh));
  size_t o = 0;
  b->S.indeg = b->scratch.as<uint32_t>(o); o += s_u32;
  b->S.qbuf = b->scratch.as<uint32_t>(o); o += s_u32;
  b->S.qpos = b->scratch.as<uint32_t>(o); o += s_u32;
  b->S.vstack = b->scratch.as<uint32_t>(o); o += s_u32;
  b->S.sched = b->scratch.as<uint8_t>(o); o += s_u8;
  b->S.devoff = b->scratch.as<uint32_t>(o); o += s_dof;
  b->S.dstate = b->scratch.as<DevSt>(o); o += s_dst;
  b->S.busy = b->scratch.as<long long>(o); o += s_busy;
  b->S.dhead = b->scratch.as<uint32_t>(o); o += s_dh;
  // outputs: makespan, err (i64), status (i32), start, end (i64 [sum n])
  const size_t o_b64 = align16(size_t(n) * 8 + 8);
  const size_t o_b32 = align16(size_t(n) * 4 + 4);
  const size_t o_op = align16(so * 8 + 8);
  CU(b->outs.ensure(2 * o_b64 + o_b32 + 2 * o_op));
  o = 0;
  b->O.makespan = b->outs.as<long long>(o); o += o_b64;
  b->O.err = b->outs.as<long long>(o); o += o_b64;
  b->O.status = b->outs.as<int>(o); o += o_b32;
  b->O.start = b->outs.as<long long>(o); o += o_op;
  b->O.end = b->outs.as<long long>(o); o += o_op;
  CU(b->desc.ensure(sizeof(Cand) * std::max(n, 1)));
  if (upload_desc)
    CU(cudaMemcpyAsync(b->desc.p, b->hc.data(), sizeof(Cand) * n, cudaMemcpyHostToDevice,
                       ctx->stream));
  CU(b->work.ensure(48));
  // packed replay layout (pack_kernel.cuh)
  {
    std::vector<unsigned long long> r_off(n), e_off(n), c_off(n);
    unsigned long long ro = 0, eo = 0, co = 0;
    for (int32_t i = 0; i < n; ++i) {
      r_off[i] = ro;
      e_off[i] = eo;
      c_off[i] = co;
      ro += b->n_ops[i] + 1;
      eo += e_cap[i];
      co += 2ull * ((b->n_ops[i] + 15) & ~15u);  // room for u16 counters
    }
    const size_t s_rec = align16(ro * 16 + 16), s_erec = align16(eo * 16 + 16),
                 s_cnt = align16(co + 16), s_u32 = align16(so * 4 + 4),
                 s_off = align16(size_t(n) * 8 + 8),
                 s_info = align16(size_t(n) * sizeof(dpro_k::PackInfo) + 16);
    const size_t s_xoff = align16(ro * 4 + 16), s_spl = align16(so + 16);
    CU(b->pack.ensure(s_rec + s_erec + 2 * s_cnt + 2 * s_u32 + s_xoff + s_spl + 3 * s_off +
                      s_info));
    size_t po = 0;
    b->P.rec = b->pack.as<uint4>(po); po += s_rec;
    b->P.erec = b->pack.as<uint4>(po); po += s_erec;
    b->P.cnt0 = b->pack.as<uint8_t>(po); po += s_cnt;
    b->P.gcnt = b->pack.as<uint8_t>(po); po += s_cnt;
    b->P.srcs = b->pack.as<uint32_t>(po); po += s_u32;
    b->P.cidx = b->pack.as<uint32_t>(po); po += s_u32;
    b->P.xoff = b->pack.as<uint32_t>(po); po += s_xoff;
    b->P.spl = b->pack.as<uint8_t>(po); po += s_spl;
    b->P.pred1 = b->res ? b->pred1.as<uint32_t>() : nullptr;
    b->P.r_off = b->pack.as<unsigned long long>(po); po += s_off;
    b->P.e_off = b->pack.as<unsigned long long>(po); po += s_off;
    b->P.c_off = b->pack.as<unsigned long long>(po); po += s_off;
    b->P.info = b->pack.as<dpro_k::PackInfo>(po); po += s_info;
    CU(cudaMemcpyAsync(b->P.r_off, r_off.data(), size_t(n) * 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(b->P.e_off, e_off.data(), size_t(n) * 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(b->P.c_off, c_off.data(), size_t(n) * 8, cudaMemcpyHostToDevice, ctx->stream));
    b->s_cnt0 = s_cnt;
  }
  return DPRO_OK;
}

// The pack kernel (and count_indeg when a candidate came without in-degrees)
// for candidates [c0, c1) on the batch's device CSR.
int launch_pack(dpro_ctx* ctx, dpro_batch* b, int32_t c0, int32_t c1) {
  if (c1 <= c0) return DPRO_OK;
  bool need_indeg = false;
  for (int32_t i = c0; i < c1; ++i) need_indeg |= (b->hc[i].indeg == nullptr);
  if (need_indeg)
    dpro_k::count_indeg_kernel<<<std::min<int>(c1 - c0, ctx->sm_count * 8), 256, 0,
                                 ctx->stream>>>(b->desc.as<Cand>() + c0, c1 - c0, b->S);
  if (ctx->pack_clusters == 0) {  // co-resident clusters of the pack kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(dpro_k::kPackCluster * (ctx->sm_count / dpro_k::kPackCluster));
    cfg.blockDim = dim3(dpro_k::kPackThreads);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = dpro_k::kPackCluster;
    attr.val.clusterDim.y = attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int m = 0;
    if (cudaOccupancyMaxActiveClusters(&m, dpro_k::pack_kernel, &cfg) != cudaSuccess || m < 1)
      m = ctx->sm_count / dpro_k::kPackCluster;
    ctx->pack_clusters = m;
  }
  const int clusters = std::max(1, std::min<int>(c1 - c0, ctx->pack_clusters));
  dpro_k::pack_kernel<<<clusters * dpro_k::kPackCluster, dpro_k::kPackThreads, 0,
                        ctx->stream>>>(b->desc.as<Cand>(), c0, c1, b->S, b->P);
  CU(cudaGetLastError());
  return DPRO_OK;
}

// PackInfo of every candidate to the host (the replay launch sizes its
// shared memory from it).
int read_pack_info(dpro_ctx* ctx, dpro_batch* b) {
  const int32_t n = b->n;
  b->info.assign(n, dpro_k::PackInfo{});
  if (n > 0) {
    CU(cudaMemcpyAsync(b->info.data(), b->P.info, size_t(n) * sizeof(dpro_k::PackInfo),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  b->replayed = b->with_schedule = false;
  return DPRO_OK;
}

int run_pack(dpro_ctx* ctx, dpro_batch* b) {
  CU(cudaMemsetAsync(b->P.cnt0, 0, b->s_cnt0, ctx->stream));
  Tracer tr;
  const int st = launch_pack(ctx, b, 0, b->n);
  if (st != DPRO_OK) return st;
  tr.mark("pack kernel", ctx->stream, true);
  return read_pack_info(ctx, b);
}

}  // namespace

extern "C" {

int dpro_cuda_abi_version(void) { return DPRO_ABI_VERSION; }

dpro_ctx* dpro_cuda_create(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count)
    return nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  auto* ctx = new dpro_ctx;
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  ctx->smem_optin = static_cast<size_t>(optin);
  cudaDeviceGetAttribute(&ctx->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaFuncSetAttribute(dpro_k::replay_batch_kernel,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  return ctx;
}

void dpro_cuda_destroy(dpro_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->side_stream) {
    cudaStreamSynchronize(ctx->side_stream);
    cudaStreamDestroy(ctx->side_stream);
    for (auto e : ctx->side_ev) cudaEventDestroy(e);
  }
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  for (cudaEvent_t ev : ctx->chunk_ev) cudaEventDestroy(ev);
  delete ctx->spare;
  delete ctx;
}

int dpro_cuda_set_stream(dpro_ctx* ctx, void* stream) {
  if (!ctx) return DPRO_EINVAL;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return DPRO_OK;
}

const char* dpro_cuda_last_error(dpro_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

}  // extern "C"

namespace {

dpro_batch* acquire_batch(dpro_ctx* ctx, int32_t n, int32_t memspace) {
  dpro_batch* b = ctx->spare;
  ctx->spare = nullptr;
  if (b) {  // keep the device buffers (they only grow), reset the rest
    b->hc.clear();
    b->n_ops.clear();
    b->n_dev.clear();
    b->n_edges.clear();
    b->sum_n = b->sum_d = b->sum_dof = b->sum_e = 0;
    b->max_d = 0;
    b->replayed = b->with_schedule = false;
    b->overlay = false;
    b->n_mat = 0;
  } else {
    b = new dpro_batch;
  }
  b->n = n;
  b->memspace = memspace;
  b->res = nullptr;
  return b;
}

template <typename F>
void parallel_for(int32_t n, F&& fn) {
  const int nt = std::max(1, std::min<int>(n, (int)std::thread::hardware_concurrency()));
  std::atomic<int32_t> next{0};
  auto work = [&]() {
    for (int32_t i; (i = next.fetch_add(1)) < n;) fn(i);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

bool ascending(const uint32_t* a, uint32_t n, bool strict) {
  for (uint32_t i = 1; i < n; ++i)
    if (strict ? a[i] <= a[i - 1] : a[i] < a[i - 1]) return false;
  return true;
}

// Host checks of one delta and its merged sizes (include/dpro_cuda.h).
std::string check_delta(const dpro_resident& r, const dpro_delta& D, uint32_t& n_ops,
                        uint32_t& n_edges, bool& dur32) {
  const uint32_t nb = r.n;
  if ((D.n_removed && !D.removed) || (D.n_new && (!D.new_pos || !D.new_dur || !D.new_dev ||
                                                  !D.new_flags)) ||
      !D.new_succ_off || (D.n_extra && (!D.extra_src || !D.extra_dst)) || (D.n_cut && !D.cut))
    return "null delta array";
  if (!ascending(D.removed, D.n_removed, true) || (D.n_removed && D.removed[D.n_removed - 1] >= nb))
    return "removed must be ascending base indices";
  if (!ascending(D.new_pos, D.n_new, false) || (D.n_new && D.new_pos[D.n_new - 1] > nb))
    return "new_pos must be non-decreasing and <= base n_ops";
  if (D.n_devices < r.d) return "n_devices below the base's";
  n_ops = nb - D.n_removed + D.n_new;
  const uint32_t ne = D.new_succ_off[D.n_new];
  if (D.new_succ_off[0] != 0 || !ascending(D.new_succ_off, D.n_new + 1, false) || (ne && !D.new_succ))
    return "bad new_succ_off";
  // removed-op bitmap (thread-local, reused across candidates)
  thread_local std::vector<uint64_t> bits;
  bits.assign((nb >> 6) + 1, 0);
  for (uint32_t k = 0; k < D.n_removed; ++k) bits[D.removed[k] >> 6] |= 1ull << (D.removed[k] & 63);
  auto removed = [&](uint32_t b) { return (bits[b >> 6] >> (b & 63)) & 1ull; };
  dur32 = r.dur32;
  for (uint32_t j = 0; j < D.n_new; ++j) {
    if (D.new_dev[j] >= D.n_devices) return "new_dev out of range";
    if (D.new_dur[j] > INT32_MAX || D.new_dur[j] < INT32_MIN) dur32 = false;
    for (uint32_t k = D.new_succ_off[j]; k < D.new_succ_off[j + 1]; ++k)
      if (D.new_succ[k] >= n_ops || (k > D.new_succ_off[j] && D.new_succ[k] <= D.new_succ[k - 1]))
        return "new_succ must be ascending final indices";
  }
  for (uint32_t k = 0; k < D.n_extra; ++k) {
    if (D.extra_src[k] >= nb || removed(D.extra_src[k]) || D.extra_dst[k] >= n_ops)
      return "extra edge out of range";
    if (k && (D.extra_src[k] < D.extra_src[k - 1] ||
              (D.extra_src[k] == D.extra_src[k - 1] && D.extra_dst[k] <= D.extra_dst[k - 1])))
      return "extra edges must be sorted by (src, dst)";
  }
  // kept base edges: all minus those touching removed ops minus cut ones
  uint64_t lost = 0;
  for (uint32_t k = 0; k < D.n_removed; ++k) {
    const uint32_t u = D.removed[k];
    lost += r.succ_off[u + 1] - r.succ_off[u];  // out-edges of u
    lost += r.indeg[u];                          // in-edges of u ...
    for (uint32_t e = r.succ_off[u]; e < r.succ_off[u + 1]; ++e)
      lost -= static_cast<uint64_t>(removed(r.succ[e]));  // ... counted once
  }
  if (!ascending(D.cut, D.n_cut, true)) return "cut must be ascending";
  for (uint32_t k = 0; k < D.n_cut; ++k) {
    const uint32_t e = D.cut[k];
    if (e >= r.e) return "cut edge out of range";
    const uint32_t u = static_cast<uint32_t>(
        std::upper_bound(r.succ_off.begin(), r.succ_off.end(), e) - r.succ_off.begin() - 1);
    if (removed(u) || removed(r.succ[e])) return "cut edges must join kept ops";
    ++lost;
  }
  // an extra edge must not repeat a kept, uncut base edge (the merge would
  // emit it twice: successor lists must stay strictly ascending and the
  // in-degrees must match what GraphBuilder's edge set gives)
  auto final_of = [&](uint32_t b) {
    return b - static_cast<uint32_t>(std::lower_bound(D.removed, D.removed + D.n_removed, b) -
                                     D.removed) +
           static_cast<uint32_t>(std::upper_bound(D.new_pos, D.new_pos + D.n_new, b) -
                                 D.new_pos);
  };
  for (uint32_t k = 0; k < D.n_extra; ++k) {
    const uint32_t u = D.extra_src[k];
    for (uint32_t e = r.succ_off[u]; e < r.succ_off[u + 1]; ++e) {
      const uint32_t s = r.succ[e];
      if (removed(s) || std::binary_search(D.cut, D.cut + D.n_cut, e)) continue;
      if (final_of(s) == D.extra_dst[k]) return "extra edge repeats a kept base edge";
    }
  }
  n_edges = static_cast<uint32_t>(uint64_t(r.e) - lost + D.n_extra + ne);
  return "";
}

int build_delta_batch(dpro_ctx* ctx, dpro_batch* b, const dpro_resident* r,
                      const dpro_delta* deltas) {
  Tracer tr;
  const int32_t n = b->n;
  // Sizes known without the checks: op counts exactly, edges as a bound
  // (base edges + added ones), devices. They fix the arena and descriptor
  // layouts up front, so every chunk of candidates can be copied and merged
  // as soon as the pool has checked and staged it (host work || H2D || K0).
  std::vector<size_t> boff(n + 1, 0), aoff(n + 1, 0);
  std::vector<uint32_t> nops(n), nedges(n);
  b->hc.assign(n, Cand{});
  b->n_ops.resize(n);
  b->n_dev.resize(n);
  b->n_edges.resize(n);
  unsigned long long so = 0, sd = 0, sdo = 0;
  uint32_t max_n = 0;
  for (int32_t i = 0; i < n; ++i) {
    const dpro_delta& D = deltas[i];
    if (!D.new_succ_off || D.n_removed > r->n)
      return set_err(ctx, DPRO_EINVAL, "delta " + std::to_string(i) + ": bad sizes");
    const size_t nn = D.n_new;
    const size_t ne = D.new_succ_off[nn];
    boff[i + 1] = boff[i] + align16(size_t(D.n_removed) * 4) + align16(nn * 4) +
                  align16(nn * 8) + align16(nn * 2) + align16(nn) + align16((nn + 1) * 4) +
                  align16(ne * 4) + 2 * align16(size_t(D.n_extra) * 4) +
                  align16(size_t(D.n_cut) * 4);
    nops[i] = r->n - D.n_removed + D.n_new;
    const size_t v = nops[i], e_bound = size_t(r->e) + D.n_extra + ne;
    // dur slot sized for int64: the int32 decision needs the checks
    aoff[i + 1] = aoff[i] + align16(v * 8) + align16(v * 2) + align16(v) +
                  align16((v + 1) * 4) + align16(e_bound * 4) + align16(v * 4);
    Cand& h = b->hc[i];
    h.n = nops[i];
    h.d = D.n_devices;
    h.op_off = so;
    h.dev_off = sd;
    h.dof_off = sdo;
    so += h.n;
    sd += h.d;
    sdo += h.d + 1;
    max_n = std::max(max_n, h.n);
  }
  CU(cudaStreamSynchronize(ctx->stream));  // staging may feed an earlier copy
  if (!ctx->copy_stream)
    CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  CU(cudaStreamSynchronize(ctx->copy_stream));
  CU(b->dblob.ensure(boff[n] + 16));
  CU(ctx->staging.ensure(boff[n] + 16));
  CU(b->arena.ensure(aoff[n] + 16));
  tr.mark("sizes + buffers");
  const uint32_t W = (r->n >> 5) + 1;
  const size_t rank_words = (3 * size_t(W) + 1 + r->n + 3) & ~size_t(3);
  CU(b->rank.ensure(rank_words * 4 * size_t(std::max(n, 1))));
  CU(b->ddesc.ensure(sizeof(dpro_k::DeltaDev) * std::max(n, 1)));
  CU(b->desc.ensure(sizeof(Cand) * std::max(n, 1)));
  CU(b->pred1.ensure(so * 4 + 16));
  b->res = r;
  b->smem_ind = std::min(max_n, dpro_k::kMergeIndegSmem);
  // scratch, outputs and the packed layout (edge capacities = the bounds), so
  // each wave can be packed right after its merge
  std::vector<uint32_t> e_cap(n);
  for (int32_t i = 0; i < n; ++i) {
    b->n_ops[i] = b->hc[i].n;
    b->n_dev[i] = b->hc[i].d;
    b->max_d = std::max(b->max_d, b->hc[i].d);
    e_cap[i] = static_cast<uint32_t>(size_t(r->e) + deltas[i].n_extra +
                                     deltas[i].new_succ_off[deltas[i].n_new]);
  }
  b->sum_n = so;
  b->sum_d = sd;
  b->sum_dof = sdo;
  {
    const int st = alloc_batch(ctx, b, e_cap, false);
    if (st != DPRO_OK) return st;
  }
  CU(cudaMemsetAsync(b->P.cnt0, 0, b->s_cnt0, ctx->stream));
  char* stage = static_cast<char*>(ctx->staging.p);
  std::vector<dpro_k::DeltaDev> dd(n);
  std::vector<std::string> errs(n);
  std::vector<int32_t> chunk_end;  // one merge wave (a candidate per SM) per chunk
  for (int32_t i = 0; i < n;) {
    const int32_t j = std::min<int32_t>(n, i + ctx->sm_count);
    chunk_end.push_back(j);
    i = j;
  }
  const int nchunks = static_cast<int>(chunk_end.size());
  std::vector<std::atomic<int32_t>> left(nchunks);
  std::vector<int> chunk_of(n);
  for (int k = 0, i = 0; k < nchunks; ++k) {
    left[k] = chunk_end[k] - i;
    for (; i < chunk_end[k]; ++i) chunk_of[i] = k;
  }
  ctx->workers().start(n, [&](int32_t i) {
    const dpro_delta& D = deltas[i];
    bool d32 = true;
    uint32_t v = 0;
    errs[i] = check_delta(*r, D, v, nedges[i], d32);
    if (errs[i].empty()) {
      dpro_k::DeltaDev& x = dd[i];
      size_t o = boff[i];
      auto put = [&](const void* src, size_t bytes) {
        if (bytes) std::memcpy(stage + o, src, bytes);
        const void* dptr = b->dblob.as<char>(o);
        o += align16(bytes);
        return dptr;
      };
      const size_t nn = D.n_new;
      x.removed = static_cast<const uint32_t*>(put(D.removed, size_t(D.n_removed) * 4));
      x.new_pos = static_cast<const uint32_t*>(put(D.new_pos, nn * 4));
      x.new_dur = static_cast<const long long*>(put(D.new_dur, nn * 8));
      x.new_dev = static_cast<const uint16_t*>(put(D.new_dev, nn * 2));
      x.new_flags = static_cast<const uint8_t*>(put(D.new_flags, nn));
      x.new_succ_off = static_cast<const uint32_t*>(put(D.new_succ_off, (nn + 1) * 4));
      x.new_succ = static_cast<const uint32_t*>(put(D.new_succ, size_t(D.new_succ_off[nn]) * 4));
      x.extra_src = static_cast<const uint32_t*>(put(D.extra_src, size_t(D.n_extra) * 4));
      x.extra_dst = static_cast<const uint32_t*>(put(D.extra_dst, size_t(D.n_extra) * 4));
      x.cut = static_cast<const uint32_t*>(put(D.cut, size_t(D.n_cut) * 4));
      x.n_removed = D.n_removed;
      x.n_new = D.n_new;
      x.n_extra = D.n_extra;
      x.n_cut = D.n_cut;
      x.rank_off = rank_words * size_t(i);
      Cand& h = b->hc[i];
      h.e = nedges[i];
      h.dur64 = d32 ? 0 : 1;
      size_t o2 = aoff[i];
      h.dur = b->arena.as<void>(o2); o2 += align16(size_t(h.n) * 8);
      h.dev = b->arena.as<uint16_t>(o2); o2 += align16(size_t(h.n) * 2);
      h.flags = b->arena.as<uint8_t>(o2); o2 += align16(h.n);
      h.succ_off = b->arena.as<uint32_t>(o2); o2 += align16((size_t(h.n) + 1) * 4);
      h.succ = b->arena.as<uint32_t>(o2);
      o2 += align16((size_t(r->e) + D.n_extra + D.new_succ_off[nn]) * 4);
      h.indeg = b->arena.as<uint32_t>(o2);  // written by the merge
    }
    left[chunk_of[i]].fetch_sub(1, std::memory_order_release);
  });
  int err = DPRO_OK;
  for (int k = 0, i = 0; k < nchunks; ++k) {
    while (left[k].load(std::memory_order_acquire) > 0) std::this_thread::yield();
    const int32_t c0 = i, c1 = chunk_end[k];
    bool ok = err == DPRO_OK;
    for (int32_t j = c0; j < c1 && ok; ++j) ok = errs[j].empty();
    if (ok) {  // this chunk: copies on the copy stream, merge on the compute
               // stream after them -- while the pool stages the next chunk and
               // the copy stream uploads it
      const size_t a0 = boff[c0], z0 = boff[c1];
      cudaStream_t cs = ctx->copy_stream;
      cudaError_t e = cudaSuccess;
      while (ctx->chunk_ev.size() <= size_t(k) && e == cudaSuccess) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) ctx->chunk_ev.push_back(ev);
      }
      if (e == cudaSuccess && z0 > a0)
        e = cudaMemcpyAsync(b->dblob.as<char>(a0), stage + a0, z0 - a0, cudaMemcpyHostToDevice,
                            cs);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(b->ddesc.as<dpro_k::DeltaDev>() + c0, dd.data() + c0,
                            sizeof(dpro_k::DeltaDev) * (c1 - c0), cudaMemcpyHostToDevice, cs);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(b->desc.as<Cand>() + c0, b->hc.data() + c0,
                            sizeof(Cand) * (c1 - c0), cudaMemcpyHostToDevice, cs);
      if (e == cudaSuccess) e = cudaEventRecord(ctx->chunk_ev[k], cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->stream, ctx->chunk_ev[k], 0);
      if (e != cudaSuccess) err = set_err(ctx, DPRO_ECUDA, cudaGetErrorString(e));
      if (err == DPRO_OK) err = run_merge(ctx, b, c0, c1);
      if (err == DPRO_OK) err = launch_pack(ctx, b, c0, c1);
    }
    i = c1;
  }
  ctx->workers().wait();
  tr.mark("host check + stage (merges queued)");
  if (err != DPRO_OK) return err;
  for (int32_t i = 0; i < n; ++i)
    if (!errs[i].empty())
      return set_err(ctx, DPRO_EINVAL, "delta " + std::to_string(i) + ": " + errs[i]);
  unsigned long long se = 0;
  for (int32_t i = 0; i < n; ++i) {
    b->n_edges[i] = b->hc[i].e;
    se += b->hc[i].e;
  }
  b->sum_e = se;
  // exact descriptors (edge counts) for the replay; same stream order
  CU(cudaMemcpyAsync(b->desc.p, b->hc.data(), sizeof(Cand) * n, cudaMemcpyHostToDevice,
                     ctx->stream));
  tr.mark("remaining H2D + merge + pack", ctx->stream, true);
  return read_pack_info(ctx, b);
}

// K0 for candidates [c0, c1) (descriptors already on the device).
int run_merge(dpro_ctx* ctx, dpro_batch* b, int32_t c0, int32_t c1) {
  if (c1 <= c0) return DPRO_OK;
  // rank structures (3W+1 words) in shared memory next to the in-degree
  // counters when both fit
  const uint32_t W = (b->res->n >> 5) + 1;
  const size_t rank_bytes = (3 * size_t(W) + 1) * 4;
  const size_t limit = ctx->smem_optin - 8192;  // static smem + slack
  const uint32_t rank_smem = size_t(b->smem_ind) * 4 + rank_bytes <= limit ? 1u : 0u;
  const size_t smem = size_t(b->smem_ind) * 4 + (rank_smem ? rank_bytes : 0);
  CU(cudaFuncSetAttribute(dpro_k::delta_merge_kernel,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dpro_k::delta_merge_kernel<<<std::min<int>(c1 - c0, ctx->sm_count), dpro_k::kMergeThreads,
                               smem, ctx->stream>>>(
      b->res->dev, b->ddesc.as<dpro_k::DeltaDev>() + c0, b->desc.as<Cand>() + c0, c1 - c0,
      b->rank.as<uint32_t>(), b->smem_ind, b->pred1.as<uint32_t>(), rank_smem);
  CU(cudaGetLastError());
  return DPRO_OK;
}

// ---------------------------------------------------------------------------
// Overlay batches (overlay.h): delta candidates replayed on the resident
// base's packed layout plus per-candidate overlays -- no per-candidate copy
// of the graph, so far more candidates are resident at once.
// ---------------------------------------------------------------------------

// Packs the resident base once (a 1-candidate batch over its device CSR)
// and builds the host view the overlay builder reads.
int ensure_base_packed(dpro_ctx* ctx, dpro_resident* r) {
  if (r->packed) return DPRO_OK;
  Tracer tr;
  dpro_csr c{r->n, r->e, r->d, r->dur32 ? 32 : 64, r->dev.dur, r->dev.dev, r->dev.flags,
             r->dev.succ_off, r->dev.succ, nullptr};
  auto* pb = new dpro_batch;
  pb->n = 1;
  pb->memspace = DPRO_DEVICE;
  const int st = build_batch(ctx, pb, &c);
  if (st != DPRO_OK) {
    delete pb;
    return st;
  }
  r->packed = pb;
  dpro_ov::BaseHost& B = r->bh;
  const dpro_k::PackInfo& inf = pb->info[0];
  B.n = r->n;
  B.e = r->e;
  B.d = r->d;
  B.dur = r->dur_h;
  B.dev = r->dev_h;
  B.flags = r->flags_h;
  B.succ_off = r->succ_off;
  B.succ = r->succ;
  B.indeg = r->indeg;
  B.ok = (inf.not_fast & ~dpro_k::kWideCnt) == 0;
  B.wide = inf.wide != 0;
  B.n_cnt = inf.n_cnt;
  B.rec.resize(4 * (size_t(r->n) + 1));
  CU(cudaMemcpyAsync(B.rec.data(), pb->P.rec, 16 * (size_t(r->n) + 1), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  B.pred_off.assign(r->n + 1, 0);
  for (uint32_t x : r->succ) B.pred_off[x + 1]++;
  for (uint32_t i = 0; i < r->n; ++i) B.pred_off[i + 1] += B.pred_off[i];
  B.pred.resize(r->e);
  {
    std::vector<uint32_t> fill(B.pred_off.begin(), B.pred_off.end() - 1);
    for (uint32_t u = 0; u < r->n; ++u)
      for (uint32_t e = r->succ_off[u]; e < r->succ_off[u + 1]; ++e) B.pred[fill[r->succ[e]]++] = u;
  }
  B.devcnt.assign(r->d, 0);
  B.srcs.clear();
  B.missing.clear();
  for (uint32_t i = 0; i < r->n; ++i) {
    const bool v = B.flags[i] & DPRO_FLAG_VIRTUAL;
    if (!v && B.dev[i] < r->d) B.devcnt[B.dev[i]]++;
    if (B.indeg[i] == 0) B.srcs.push_back(i);
    if (!v && B.dur[i] < 0) B.missing.push_back(i);
  }
  r->ob = {pb->P.rec, pb->P.erec, pb->P.cnt0, B.n_cnt, B.wide ? 1u : 0u};
  tr.mark("base packed for overlays");
  return DPRO_OK;
}

// Host image of every candidate's overlay arrays (b->ovstage, offsets in
// b->ov_off) and the OvCand descriptors pointing into b->ovarena.
int stage_overlays(dpro_ctx* ctx, dpro_batch* b) {
  const int32_t n = b->n;
  const dpro_resident* r = b->res;
  b->ov_off.assign(n + 1, 0);
  size_t o = 0;
  auto sz = [](size_t bytes) { return align16(bytes); };
  for (int32_t i = 0; i < n; ++i) {
    const auto& O = b->ovh[i];
    b->ov_off[i] = o;
    if (!O.fast) continue;
    o += sz(O.rec.size() * 4) + sz(O.erec.size() * 4) + sz(O.fin.size() * 4) +
         sz(O.cnt.size() * 2) + sz(O.src.size() * 4) + sz(O.blk.size() * 4) + sz(O.ovf.size() * 4) +
         sz(O.sx.size() * 4) + sz(O.sbp.size() * 4);
  }
  b->ov_off[n] = o;
  b->ov_bytes = o;
  CU(b->ovstage.ensure(std::max<size_t>(o, 16)));
  CU(b->ovarena.ensure(std::max<size_t>(o, 16)));
  b->ovc.assign(n, dpro_k::OvCand{});
  // global counter slices (u16, base + overlay counters)
  std::vector<unsigned long long> goff(n + 1, 0);
  b->max_cnt_ov = 0;
  for (int32_t i = 0; i < n; ++i) {
    const uint32_t nc = r->bh.n_cnt + static_cast<uint32_t>(b->ovh[i].cnt.size());
    b->max_cnt_ov = std::max(b->max_cnt_ov, nc);
    goff[i + 1] = goff[i] + align16(size_t(nc) * 2);
  }
  CU(b->ovgcnt.ensure(std::max<size_t>(goff[n], 16)));
  ctx->workers().run(n, [&](int32_t i) {
    const auto& O = b->ovh[i];
    dpro_k::OvCand& c = b->ovc[i];
    c.gcnt_off = goff[i];
    c.first_missing = O.first_missing;
    if (!O.fast) {
      c.pad = 1;  // materialized path
      return;
    }
    size_t q = b->ov_off[i];
    auto put = [&](const void* src, size_t bytes) {
      if (bytes) std::memcpy(static_cast<char*>(b->ovstage.p) + q, src, bytes);
      const char* dptr = b->ovarena.as<char>(q);
      q += align16(bytes);
      return dptr;
    };
    c.v.rec = reinterpret_cast<const uint4*>(put(O.rec.data(), O.rec.size() * 4));
    c.v.erec = reinterpret_cast<const uint4*>(put(O.erec.data(), O.erec.size() * 4));
    c.v.fin = reinterpret_cast<const uint32_t*>(put(O.fin.data(), O.fin.size() * 4));
    c.cnt = reinterpret_cast<const uint16_t*>(put(O.cnt.data(), O.cnt.size() * 2));
    c.src = reinterpret_cast<const uint4*>(put(O.src.data(), O.src.size() * 4));
    c.v.blk = reinterpret_cast<const uint32_t*>(put(O.blk.data(), O.blk.size() * 4));
    c.v.ovf = reinterpret_cast<const uint32_t*>(put(O.ovf.data(), O.ovf.size() * 4));
    c.sx = reinterpret_cast<const uint2*>(put(O.sx.data(), O.sx.size() * 4));
    c.sbp = reinterpret_cast<const uint2*>(put(O.sbp.data(), O.sbp.size() * 4));
    c.n_sx = static_cast<uint32_t>(O.sx.size() / 2);
    c.n_sbp = static_cast<uint32_t>(O.sbp.size() / 2);
    c.ovmin = O.ovmin;
    c.sparse = O.sparse ? 1u : 0u;
    c.n_cnt = static_cast<uint32_t>(O.cnt.size());
    c.n_src = static_cast<uint32_t>(O.src.size() / 4);
    c.pad = 0;
  });
  return DPRO_OK;
}

// H2D of the staged overlays, descriptors and timeline regions: the
// device-side preparation of an overlay batch (dpro_cuda_batch_prepare).
int upload_overlays(dpro_ctx* ctx, dpro_batch* b) {
  const int32_t n = b->n;
  if (b->ov_bytes)
    CU(cudaMemcpyAsync(b->ovarena.p, b->ovstage.p, b->ov_bytes, cudaMemcpyHostToDevice,
                       ctx->stream));
  CU(b->ovdesc.ensure(sizeof(dpro_k::OvCand) * std::max(n, 1)));
  if (n)
    CU(cudaMemcpyAsync(b->ovdesc.p, b->ovc.data(), sizeof(dpro_k::OvCand) * n,
                       cudaMemcpyHostToDevice, ctx->stream));
  return DPRO_OK;
}

int build_overlay_batch(dpro_ctx* ctx, dpro_batch* b, dpro_resident* r,
                        const dpro_delta* deltas) {
  Tracer tr;
  const int32_t n = b->n;
  int st = ensure_base_packed(ctx, r);
  if (st != DPRO_OK) return st;
  b->res = r;
  b->overlay = true;
  b->ovh.resize(n);
  b->dcopy.resize(n);
  b->hc.assign(n, Cand{});
  b->n_ops.resize(n);
  b->n_dev.resize(n);
  b->n_edges.resize(n);
  std::vector<std::string> errs(n);
  ctx->workers().run(n, [&](int32_t i) {
    uint32_t v = 0, e = 0;
    bool d32 = true;
    errs[i] = check_delta(*r, deltas[i], v, e, d32);
    if (!errs[i].empty()) return;
    b->n_ops[i] = v;
    b->n_edges[i] = e;
    b->n_dev[i] = deltas[i].n_devices;
    b->dcopy[i].set(deltas[i]);
    dpro_ov::build_overlay(r->bh, b->dcopy[i].d, b->ovh[i]);
  });
  for (int32_t i = 0; i < n; ++i)
    if (!errs[i].empty())
      return set_err(ctx, DPRO_EINVAL, "delta " + std::to_string(i) + ": " + errs[i]);
  tr.mark("overlays built");
  unsigned long long so = 0, sd = 0, sdo = 0, se = 0;
  b->n_mat = 0;
  b->max_d = 0;
  for (int32_t i = 0; i < n; ++i) {
    Cand& h = b->hc[i];
    h.n = b->n_ops[i];
    h.e = b->n_edges[i];
    h.d = b->n_dev[i];
    h.op_off = so;
    h.dev_off = sd;
    h.dof_off = sdo;
    so += h.n;
    sd += h.d;
    sdo += h.d + 1;
    se += h.e;
    b->max_d = std::max(b->max_d, h.d);
    b->n_mat += b->ovh[i].fast ? 0 : 1;
  }
  b->sum_n = so;
  b->sum_d = sd;
  b->sum_dof = sdo;
  b->sum_e = se;
  // scratch (timelines, regions, per-device busy / dispatched prefix) and outputs
  const size_t s_u32 = align16(so * 4 + 4), s_dof = align16(sdo * 4 + 4),
               s_busy = align16(sd * 8 + 8), s_dh = align16(sd * 4 + 4),
               s_u8 = align16(so + 1);
  CU(b->scratch.ensure(s_u32 + s_dof + s_busy + s_dh + s_u8));
  size_t o = 0;
  b->S = Scratch{};  // no qpos: K3 does not run on overlay batches
  b->S.qbuf = b->scratch.as<uint32_t>(o); o += s_u32;
  b->S.devoff = b->scratch.as<uint32_t>(o); o += s_dof;
  b->S.busy = b->scratch.as<long long>(o); o += s_busy;
  b->S.dhead = b->scratch.as<uint32_t>(o); o += s_dh;
  b->S.sched = b->scratch.as<uint8_t>(o); o += s_u8;
  const size_t o_b64 = align16(size_t(n) * 8 + 8), o_b32 = align16(size_t(n) * 4 + 4),
               o_op = align16(so * 8 + 8);
  CU(b->outs.ensure(2 * o_b64 + o_b32 + 2 * o_op));
  o = 0;
  b->O.makespan = b->outs.as<long long>(o); o += o_b64;
  b->O.err = b->outs.as<long long>(o); o += o_b64;
  b->O.status = b->outs.as<int>(o); o += o_b32;
  b->O.start = b->outs.as<long long>(o); o += o_op;
  b->O.end = b->outs.as<long long>(o); o += o_op;
  CU(b->desc.ensure(sizeof(Cand) * std::max(n, 1)));
  if (n) CU(cudaMemcpyAsync(b->desc.p, b->hc.data(), sizeof(Cand) * n, cudaMemcpyHostToDevice,
                            ctx->stream));
  CU(b->work.ensure(48));
  {  // timeline regions from the overlays (materialized candidates: their pack)
    std::vector<uint32_t> dof(std::max<unsigned long long>(sdo, 1), 0);
    for (int32_t i = 0; i < n; ++i)
      if (b->ovh[i].fast)
        std::copy(b->ovh[i].devoff.begin(), b->ovh[i].devoff.end(), dof.begin() + b->hc[i].dof_off);
    if (sdo) CU(cudaMemcpyAsync(b->S.devoff, dof.data(), sdo * 4, cudaMemcpyHostToDevice,
                                ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));  // dof is a local
  }
  st = stage_overlays(ctx, b);
  if (st != DPRO_OK) return st;
  st = upload_overlays(ctx, b);
  if (st != DPRO_OK) return st;
  b->info.assign(n, dpro_k::PackInfo{});
  for (int32_t i = 0; i < n; ++i) {
    b->info[i].first_missing = b->ovh[i].first_missing;
    b->info[i].not_fast = b->ovh[i].fast ? 0u : 1u;
  }
  // whole-graph rewrites (recompute / grad-accum variants: 100x the median
  // overlay) are the long candidates of a batch (the grad-accum variant's
  // link queues are 230 deep): they start first, on the side stream with
  // global rings, so they overlap everything else instead of trailing it
  b->g3.clear();
  {
    std::vector<size_t> sz;
    for (int32_t i = 0; i < n; ++i)
      if (b->ovh[i].fast) sz.push_back(b->ovh[i].fin.size());
    size_t cut = SIZE_MAX;
    if (!sz.empty()) {
      std::nth_element(sz.begin(), sz.begin() + sz.size() / 2, sz.end());
      cut = std::max<size_t>(100 * sz[sz.size() / 2], r->n / 100);
    }
    std::vector<uint32_t> ord;
    for (int32_t i = 0; i < n; ++i)
      if (b->ovh[i].fast && b->ovh[i].fin.size() > cut) {
        ord.push_back(i);
        b->g3.push_back(i);  // and straight to the side stream (global rings)
      }
    for (int32_t i = 0; i < n; ++i)
      if (!(b->ovh[i].fast && b->ovh[i].fin.size() > cut)) ord.push_back(i);
    CU(b->order.ensure(4 * (2 * size_t(n) + 1)));  // order, then side flags
    if (n) CU(cudaMemsetAsync(b->order.as<unsigned>() + n, 0, 4 * size_t(n), ctx->stream));
    b->side_any = false;
    if (n) CU(cudaMemcpyAsync(b->order.p, ord.data(), 4 * size_t(n), cudaMemcpyHostToDevice,
                              ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));  // ord is a local
  }
  b->replayed = b->with_schedule = false;
  tr.mark("overlay batch staged + uploaded", ctx->stream, true);
  return DPRO_OK;
}

}  // namespace

extern "C" {

dpro_resident* dpro_cuda_resident_create(dpro_ctx* ctx, const dpro_csr* c) {
  if (!ctx || !c) return nullptr;
  if (c->n_ops > 0 && (!c->dur || !c->dev || !c->flags || !c->succ_off) ||
      (c->n_edges > 0 && !c->succ) || (c->dur_bits != 32 && c->dur_bits != 64)) {
    ctx->err = "bad base CSR";
    return nullptr;
  }
  if (cudaSetDevice(ctx->device) != cudaSuccess) return nullptr;
  auto r = std::make_unique<dpro_resident>();
  r->n = c->n_ops;
  r->e = c->n_edges;
  r->d = c->n_devices;
  r->succ_off.assign(c->succ_off, c->succ_off + c->n_ops + 1);
  r->succ.assign(c->succ, c->succ + c->n_edges);
  r->indeg.assign(c->n_ops, 0);
  for (uint32_t x : r->succ) r->indeg.at(x)++;
  r->dev_h.assign(c->dev, c->dev + c->n_ops);
  r->flags_h.assign(c->flags, c->flags + c->n_ops);
  r->dur_h.resize(c->n_ops);
  for (uint32_t i = 0; i < c->n_ops; ++i)
    r->dur_h[i] = c->dur_bits == 32 ? static_cast<const int32_t*>(c->dur)[i]
                                    : static_cast<const int64_t*>(c->dur)[i];
  r->dur32 = c->dur_bits == 32 || fits_i32(static_cast<const int64_t*>(c->dur), c->n_ops);
  const size_t v = c->n_ops, sd = align16(v * (r->dur32 ? 4 : 8)), s2 = align16(v * 2),
               s1 = align16(v), so = align16((v + 1) * 4), se = align16(size_t(c->n_edges) * 4);
  if (r->buf.ensure(sd + s2 + s1 + so + se + 16) != cudaSuccess) {
    ctx->err = "resident base: out of device memory";
    return nullptr;
  }
  std::vector<int32_t> d32;
  const void* dsrc = c->dur;
  if (r->dur32 && c->dur_bits == 64) {
    d32.resize(v);
    for (size_t i = 0; i < v; ++i) d32[i] = static_cast<int32_t>(static_cast<const int64_t*>(c->dur)[i]);
    dsrc = d32.data();
  }
  char* p = r->buf.as<char>();
  bool ok = cudaMemcpy(p, dsrc, v * (r->dur32 ? 4 : 8), cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemcpy(p + sd, c->dev, v * 2, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemcpy(p + sd + s2, c->flags, v, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemcpy(p + sd + s2 + s1, c->succ_off, (v + 1) * 4, cudaMemcpyHostToDevice) ==
                cudaSuccess &&
            (c->n_edges == 0 || cudaMemcpy(p + sd + s2 + s1 + so, c->succ,
                                           size_t(c->n_edges) * 4,
                                           cudaMemcpyHostToDevice) == cudaSuccess);
  if (!ok) {
    ctx->err = "resident base: upload failed";
    return nullptr;
  }
  r->dev = {p, reinterpret_cast<const uint16_t*>(p + sd),
            reinterpret_cast<const uint8_t*>(p + sd + s2),
            reinterpret_cast<const uint32_t*>(p + sd + s2 + s1),
            reinterpret_cast<const uint32_t*>(p + sd + s2 + s1 + so), r->n,
            r->dur32 ? 0u : 1u};
  return r.release();
}

void dpro_cuda_resident_destroy(dpro_ctx* ctx, dpro_resident* r) {
  if (!r) return;
  if (ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
  }
  delete r;
}

dpro_batch* dpro_cuda_batch_create_delta(dpro_ctx* ctx, const dpro_resident* r,
                                         const dpro_delta* deltas, int32_t n) {
  if (!ctx || !r || n < 0 || (n > 0 && !deltas)) {
    if (ctx) ctx->err = "bad delta batch arguments";
    return nullptr;
  }
  cudaSetDevice(ctx->device);
  if (ctx->overlay) {
    auto* b = new dpro_batch;
    b->n = n;
    b->memspace = DPRO_DEVICE;
    if (build_overlay_batch(ctx, b, const_cast<dpro_resident*>(r), deltas) != DPRO_OK) {
      delete b;
      return nullptr;
    }
    return b;
  }
  dpro_batch* b = acquire_batch(ctx, n, DPRO_DEVICE);
  if (build_delta_batch(ctx, b, r, deltas) != DPRO_OK) {
    delete b;
    return nullptr;
  }
  return b;
}

int dpro_cuda_batch_sizes(dpro_batch* b, uint32_t* n_ops, uint32_t* n_edges,
                          uint32_t* n_devices) {
  if (!b) return DPRO_EINVAL;
  for (int32_t i = 0; i < b->n; ++i) {
    if (n_ops) n_ops[i] = b->n_ops[i];
    if (n_edges) n_edges[i] = b->n_edges[i];
    if (n_devices) n_devices[i] = b->n_dev[i];
  }
  return DPRO_OK;
}

int dpro_cuda_batch_pack_info(dpro_batch* b, uint32_t* out) {
  if (!b || !out) return DPRO_EINVAL;
  for (int32_t i = 0; i < b->n; ++i) {
    const auto& f = b->info[i];
    out[4 * i] = f.first_missing;
    out[4 * i + 1] = f.not_fast;
    out[4 * i + 2] = f.n_cnt;
    out[4 * i + 3] = f.n_src;
  }
  return DPRO_OK;
}

int dpro_cuda_batch_prepare(dpro_ctx* ctx, dpro_batch* b) {
  if (!ctx || !b) return DPRO_EINVAL;
  CU(cudaSetDevice(ctx->device));
  if (b->overlay) return upload_overlays(ctx, b);
  if (b->res) {
    const int st = run_merge(ctx, b, 0, b->n);
    if (st != DPRO_OK) return st;
  }
  return run_pack(ctx, b);
}

int dpro_cuda_replay_delta_batch(dpro_ctx* ctx, const dpro_resident* r,
                                 const dpro_delta* deltas, int32_t n, int64_t* makespan,
                                 int32_t* status, int64_t* err) {
  if (!ctx) return DPRO_EINVAL;
  dpro_batch* b = dpro_cuda_batch_create_delta(ctx, r, deltas, n);
  if (!b) return DPRO_EINVAL;
  int st = dpro_cuda_batch_replay(ctx, b, 0);
  if (st == DPRO_OK) st = dpro_cuda_batch_results(ctx, b, makespan, status, err, nullptr, nullptr);
  dpro_cuda_batch_destroy(ctx, b);
  return st;
}

dpro_batch* dpro_cuda_batch_create(dpro_ctx* ctx, const dpro_csr* cands,
                                   int32_t n_cands, int32_t memspace) {
  if (!ctx || (n_cands > 0 && !cands) || n_cands < 0 ||
      (memspace != DPRO_HOST && memspace != DPRO_DEVICE)) {
    if (ctx) ctx->err = "bad batch arguments";
    return nullptr;
  }
  cudaSetDevice(ctx->device);
  dpro_batch* b = acquire_batch(ctx, n_cands, memspace);
  if (build_batch(ctx, b, cands) != DPRO_OK) {
    delete b;
    return nullptr;
  }
  return b;
}

void dpro_cuda_batch_destroy(dpro_ctx* ctx, dpro_batch* b) {
  if (!b) return;
  if (ctx) {
    cudaStreamSynchronize(ctx->stream);
    if (!ctx->spare && !b->overlay) {  // overlay batches are big: never kept
      ctx->spare = b;
      return;
    }
  }
  delete b;
}

int dpro_cuda_set_option(dpro_ctx* ctx, const char* key, int64_t value) {
  if (!ctx || !key) return DPRO_EINVAL;
  const std::string k(key);
  if (k == "fast" && (value == 0 || value == 1)) {
    ctx->fast = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "warps" && (value == 0 || value == 1 || value == 2 || value == 4 || value == 8)) {
    ctx->warps = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "host_threads" && value >= 0 && value <= 4096) {
    if (ctx->pool && ctx->host_threads != static_cast<int>(value)) ctx->pool.reset();
    ctx->host_threads = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "gring0" && value >= -1 && value <= 1) {
    ctx->gring0 = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "tsync_host" && (value == 0 || value == 1)) {
    ctx->tsync_host = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "overlay" && (value == 0 || value == 1)) {
    ctx->overlay = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "gcnt" && (value == 0 || value == 1)) {
    ctx->gcnt = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "deep_first" && value >= -1 && value <= 1) {
    ctx->deep_first = static_cast<int>(value);
    return DPRO_OK;
  }
  if (k == "ring" && value >= 2 && value <= 64 && (value & (value - 1)) == 0) {
    ctx->ring = static_cast<uint32_t>(value);
    return DPRO_OK;
  }
  return set_err(ctx, DPRO_EINVAL, "unknown option or value: " + k);
}

}  // extern "C"

namespace {

// filter != 0: only the candidates the fast kernel handed off (status ==
// filter), after its passes on the same stream.
int launch_general(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule, int filter = 0) {
  size_t budget = std::min<size_t>(ctx->smem_optin, 200 * 1024);
  uint32_t dcap = static_cast<uint32_t>((budget - kSmemHeader) / (kWarpsPerBlock * sizeof(DevSt)));
  dcap = std::min<uint32_t>(dcap, std::max<uint32_t>(b->max_d, 1));
  const size_t smem = kSmemHeader + size_t(kWarpsPerBlock) * dcap * sizeof(DevSt);
  int blocks_per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &blocks_per_sm, dpro_k::replay_batch_kernel, 32 * kWarpsPerBlock, smem));
  blocks_per_sm = std::max(blocks_per_sm, 1);
  const int need = (b->n + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int grid = std::max(1, std::min(need, ctx->sm_count * blocks_per_sm));
  CU(cudaMemsetAsync(b->work.as<unsigned>() + (filter ? 9 : 0), 0, 4, ctx->stream));
  const int g = filter ? std::max(1, std::min(ctx->sm_count * blocks_per_sm,
                                              (b->n + kWarpsPerBlock - 1) / kWarpsPerBlock))
                       : grid;
  dpro_k::replay_batch_kernel<<<g, 32 * kWarpsPerBlock, smem, ctx->stream>>>(
      b->desc.as<Cand>(), b->n, b->S, b->O, want_schedule ? 1 : 0,
      b->work.as<unsigned>(), dcap, filter);
  CU(cudaGetLastError());
  return DPRO_OK;
}

// Fast-path shared memory per candidate (one warp per block):
// devices x (DevF + ring) + virtual worklist + misc words + u8 counters.
size_t fast_bytes(uint32_t dcap, uint32_t qc, uint32_t rl, uint32_t ccap, int nw);

size_t fast_bytes(uint32_t dcap, uint32_t qc, uint32_t rl, uint32_t ccap, int nw) {
  return size_t(dcap) * (sizeof(dpro_k::DevF) + 16 * qc + dpro_k::kTailBytesPerDev) +
         8 * size_t(rl) + 4 * dpro_k::fast_misc_words(nw) + ccap;
}

// Pass 3 (after the deep-ring pass): candidates whose device queues
// outgrew even the deepest shared-memory rings (e.g. the grad-accum variant
// of config 4: a 230-deep link queue), rings in global memory (one slice
// per CTA, one CTA per SM). Returns false when there is nothing to gain.
bool pass3_cfg(dpro_ctx* ctx, const FastCfg& deep, int nw, FastCfg& G, uint32_t extra = 0) {
  constexpr size_t kBudget = size_t(512) << 20;
  G = deep;
  G.qc = 4096;
  while (G.qc > deep.qc && size_t(ctx->sm_count) * G.dcap * G.qc * 16 > kBudget) G.qc /= 2;
  if (G.qc <= deep.qc) return false;
  G.rl = 8192;
  if (ctx->gring.ensure(size_t(ctx->sm_count) * G.dcap * G.qc * 16) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  G.gq = ctx->gring.as<uint4>();
  G.warp_bytes = static_cast<uint32_t>(fast_bytes(G.dcap, 0, G.rl, G.ccap, nw)) + extra;
  return G.warp_bytes + 1024 <= ctx->smem_optin;
}

template <int NW, int KD>
int launch_fast_kd(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule, FastCfg F) {
  auto kern = dpro_k::replay_fast_kernel<NW, KD>;
  const size_t smem = F.warp_bytes;
  cudaFuncAttributes fa{};
  CU(cudaFuncGetAttributes(&fa, kern));
  const size_t dyn_max = ctx->smem_optin - fa.sharedSizeBytes;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max));
  int blocks_per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, 32 * NW, smem));
  blocks_per_sm = std::max(blocks_per_sm, 1);
  b->blocks_per_sm_fast = blocks_per_sm;
  const int grid = std::max(1, std::min(b->n, ctx->sm_count * blocks_per_sm));
  CU(cudaMemsetAsync(b->work.p, 0, 48, ctx->stream));
  b->F = F;
  // graphs of millions of ops (configs 4/5) overflow the residency-sized
  // rings every time: send them straight to the deep-ring pass
  const bool deep_first = ctx->deep_first >= 0
                              ? ctx->deep_first == 1
                              : (b->n > 0 && b->sum_n / b->n > 1000000ull);
  b->mark(0, ctx->stream);
  kern<<<grid, 32 * NW, smem, ctx->stream>>>(b->desc.as<Cand>(), b->n, b->S, b->O, b->P, F,
                                             want_schedule ? 1 : 0, b->work.as<unsigned>(),
                                             deep_first ? 2 : 0);
  CU(cudaGetLastError());
  b->mark(1, ctx->stream);
  // pass 1: candidates whose device queues outgrew the ring, one CTA per SM
  // with the deepest rings the shared memory holds
  FastCfg D = F;
  D.rl = std::max<uint32_t>(F.rl, 2048);
  const size_t limit = dyn_max;
  while (D.qc < 4096 && fast_bytes(D.dcap, D.qc * 2, D.rl, D.ccap, NW) <= limit) D.qc *= 2;
  D.warp_bytes = static_cast<uint32_t>(fast_bytes(D.dcap, D.qc, D.rl, D.ccap, NW));
  kern<<<ctx->sm_count, 32 * NW, D.warp_bytes, ctx->stream>>>(
      b->desc.as<Cand>(), b->n, b->S, b->O, b->P, D, want_schedule ? 1 : 0,
      b->work.as<unsigned>(), 1);
  CU(cudaGetLastError());
  b->mark(2, ctx->stream);
  FastCfg G;
  if (pass3_cfg(ctx, D, NW, G)) {
    kern<<<ctx->sm_count, 32 * NW, G.warp_bytes, ctx->stream>>>(
        b->desc.as<Cand>(), b->n, b->S, b->O, b->P, G, want_schedule ? 1 : 0,
        b->work.as<unsigned>(), 3);
    CU(cudaGetLastError());
  }
  b->mark(3, ctx->stream);
  // whatever the fast passes could not represent: the general kernel
  const int st = launch_general(ctx, b, want_schedule, dpro_k::kRetryGen);
  b->mark(4, ctx->stream);
  b->pev_valid = true;
  return st;
}

template <int NW>
int launch_fast_nw(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule) {
  FastCfg F;
  F.qc = ctx->ring;
  F.rl = 128;
  uint32_t max_cnt = 16;  // counter bytes
  for (const auto& inf : b->info) max_cnt = std::max(max_cnt, (inf.wide ? 2u : 1u) * inf.n_cnt);
  const uint32_t nt = 32 * NW;
  uint32_t kd = std::max<uint32_t>(1, (b->max_d + nt - 1) / nt);
  if (kd > 8) kd = kd <= 12 ? 12 : 16;
  if (b->max_d > dpro_k::kMaxDev) kd = 16;
  F.kd = kd;
  F.dcap = std::max<uint32_t>(1, std::min<uint32_t>(b->max_d, nt * kd));
  F.ccap = (max_cnt + 15) & ~15u;
  const size_t limit = ctx->smem_optin - 64;
  // counters that would leave fewer than 4 candidates per SM stay in global
  // scratch instead (large graphs: configs 4/5 have 10^5+ multi-pred ops)
  if (ctx->gcnt || fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW) > size_t(ctx->smem_per_sm) / 4)
    F.ccap = 16;
  while (fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW) > limit && F.ccap > 16)
    F.ccap = std::max<uint32_t>(16, (F.ccap / 2 + 15) & ~15u);
  while (fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW) > limit && F.dcap > 1) F.dcap /= 2;
  // Deeper rings while the candidate still fits the residency target (the
  // whole batch resident: ~8 candidates per SM) -- deep device queues
  // (e.g. ring all-reduce links) otherwise fall back to the general kernel.
  const size_t target = std::max<size_t>(fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW),
                                         size_t(ctx->smem_per_sm) / 8 - 1024);
  while (F.qc < 64 && fast_bytes(F.dcap, F.qc * 2, F.rl, F.ccap, NW) <= std::min(target, limit))
    F.qc *= 2;
  F.warp_bytes = static_cast<uint32_t>(fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW));
  switch (kd) {
    case 1: return launch_fast_kd<NW, 1>(ctx, b, want_schedule, F);
    case 2: return launch_fast_kd<NW, 2>(ctx, b, want_schedule, F);
    case 3: return launch_fast_kd<NW, 3>(ctx, b, want_schedule, F);
    case 4: return launch_fast_kd<NW, 4>(ctx, b, want_schedule, F);
    case 5: return launch_fast_kd<NW, 5>(ctx, b, want_schedule, F);
    case 6: return launch_fast_kd<NW, 6>(ctx, b, want_schedule, F);
    case 7: return launch_fast_kd<NW, 7>(ctx, b, want_schedule, F);
    case 8: return launch_fast_kd<NW, 8>(ctx, b, want_schedule, F);
    case 12: return launch_fast_kd<NW, 12>(ctx, b, want_schedule, F);
    default: return launch_fast_kd<NW, 16>(ctx, b, want_schedule, F);
  }
}

int launch_fast(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule) {
  // auto (option warps = 0): the CTA's lanes own the devices, so graphs with
  // few devices waste most of a 4-warp CTA in every round's barriers
  // (config 1, 16 devices: 1 warp 8.5 ms vs 4 warps 11.2 ms; config 2, 144
  // devices: 4 warps 2.95 ms vs 1 warp 8.5 ms -- tools/warps_sweep.py)
  int nw = ctx->warps;
  if (nw == 0) nw = b->max_d <= 32 ? 1 : b->max_d <= 64 ? 2 : 4;
  switch (nw) {
    case 1: return launch_fast_nw<1>(ctx, b, want_schedule);
    case 2: return launch_fast_nw<2>(ctx, b, want_schedule);
    case 8: return launch_fast_nw<8>(ctx, b, want_schedule);
    default: return launch_fast_nw<4>(ctx, b, want_schedule);
  }
}

// Overlay batches: replay_ov_kernel, the same two passes as the fast path.
template <int NW, int KD>
int launch_ov_kd(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule, FastCfg F) {
  auto kern = dpro_k::replay_ov_kernel<NW, KD>;
  cudaFuncAttributes fa{};
  CU(cudaFuncGetAttributes(&fa, kern));
  const size_t dyn_max = ctx->smem_optin - fa.sharedSizeBytes;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max));
  // residency pass: for multi-million-op graphs the 16-entry device rings
  // (32 KB of 44 KB per CTA) cap residency at 5 CTAs per SM; in global
  // memory (L2) they cost latency per access but 8 CTAs per SM fit
  // (register bound): +31 % replays/s on config 4 (profiles/r02_*)
  const bool gring0 = ctx->gring0 == 1 ||
                      (ctx->gring0 < 0 && b->n > 0 && b->sum_n / b->n > 1000000ull);
  FastCfg F0 = F;
  if (gring0) {
    F0.warp_bytes = F.warp_bytes - 16 * F.dcap * F.qc;
    F0.gq = nullptr;  // set below, once the grid is known
  }
  int blocks_per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, 32 * NW, F0.warp_bytes));
  blocks_per_sm = std::max(blocks_per_sm, 1);
  b->blocks_per_sm_fast = blocks_per_sm;
  const int grid = std::max(1, std::min(b->n, ctx->sm_count * blocks_per_sm));
  if (gring0) {
    CU(ctx->gring0_buf.ensure(size_t(grid) * F.dcap * F.qc * 16));
    F0.gq = ctx->gring0_buf.as<uint4>();
  }
  CU(cudaMemsetAsync(b->work.p, 0, 48, ctx->stream));
  b->F = F0;
  const dpro_resident* r = b->res;
  CU(b->hint.ensure(4 * (size_t(b->n) + 1)));
  unsigned* hint = b->hint.as<unsigned>();
  b->mark(0, ctx->stream);
  // candidates known (from an earlier replay) to need global rings start
  // first, on the side stream, so they overlap the residency pass
  FastCfg D = F;  // pass 1: ring overflows, one CTA per SM, deepest rings
  D.rl = std::max<uint32_t>(F.rl, 2048);
  const size_t lim = dyn_max - dpro_k::kOvListBytes - 16 * D.dcap;
  while (D.qc < 4096 && fast_bytes(D.dcap, D.qc * 2, D.rl, D.ccap, NW) <= lim) D.qc *= 2;
  D.warp_bytes = static_cast<uint32_t>(fast_bytes(D.dcap, D.qc, D.rl, D.ccap, NW)) +
                 dpro_k::kOvListBytes + 16 * D.dcap;
  FastCfg G;
  const bool g3ok = pass3_cfg(ctx, D, NW, G, dpro_k::kOvListBytes + 16 * D.dcap);
  const bool side = g3ok && !b->g3.empty();
  if (!side && b->side_any) {
    CU(cudaMemsetAsync(b->order.as<unsigned>() + b->n, 0, 4 * size_t(b->n), ctx->stream));
  }
  b->side_any = side;
  if (side) {
    if (!ctx->side_stream) {
      CU(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&ctx->side_ev[0], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ctx->side_ev[1], cudaEventDisableTiming));
    }
    // side flags after the order permutation: pass 0 skips these whatever
    // their status (pass 4 may already have finished one)
    b->side_h.assign(b->n, 0u);
    for (int32_t c : b->g3) b->side_h[c] = 1u;
    CU(cudaMemcpyAsync(b->order.as<unsigned>() + b->n, b->side_h.data(), 4 * size_t(b->n),
                       cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaEventRecord(ctx->side_ev[0], ctx->stream));
    CU(cudaStreamWaitEvent(ctx->side_stream, ctx->side_ev[0], 0));
    const int g4 = std::max(1, std::min<int>(ctx->sm_count, static_cast<int>(b->g3.size())));
    kern<<<g4, 32 * NW, G.warp_bytes, ctx->side_stream>>>(
        b->desc.as<Cand>(), b->ovdesc.as<dpro_k::OvCand>(), b->n, r->ob, b->S, b->O,
        b->ovgcnt.as<uint8_t>(), G, want_schedule ? 1 : 0, b->work.as<unsigned>(), 4, hint,
        b->order.as<unsigned>());
    CU(cudaGetLastError());
    CU(cudaEventRecord(ctx->side_ev[1], ctx->side_stream));
  }
  kern<<<grid, 32 * NW, F0.warp_bytes, ctx->stream>>>(
      b->desc.as<Cand>(), b->ovdesc.as<dpro_k::OvCand>(), b->n, r->ob, b->S, b->O,
      b->ovgcnt.as<uint8_t>(), F0, want_schedule ? 1 : 0, b->work.as<unsigned>(), 0, hint,
      b->order.as<unsigned>());
  CU(cudaGetLastError());
  b->mark(1, ctx->stream);
  kern<<<ctx->sm_count, 32 * NW, D.warp_bytes, ctx->stream>>>(
      b->desc.as<Cand>(), b->ovdesc.as<dpro_k::OvCand>(), b->n, r->ob, b->S, b->O,
      b->ovgcnt.as<uint8_t>(), D, want_schedule ? 1 : 0, b->work.as<unsigned>(), 1, hint,
      b->order.as<unsigned>());
  CU(cudaGetLastError());
  b->mark(2, ctx->stream);
  if (g3ok) {
    kern<<<ctx->sm_count, 32 * NW, G.warp_bytes, ctx->stream>>>(
        b->desc.as<Cand>(), b->ovdesc.as<dpro_k::OvCand>(), b->n, r->ob, b->S, b->O,
        b->ovgcnt.as<uint8_t>(), G, want_schedule ? 1 : 0, b->work.as<unsigned>(), 3, hint,
        b->order.as<unsigned>());
    CU(cudaGetLastError());
  }
  if (side) CU(cudaStreamWaitEvent(ctx->stream, ctx->side_ev[1], 0));
  b->mark(3, ctx->stream);
  b->mark(4, ctx->stream);
  b->pev_valid = true;
  return DPRO_OK;
}

template <int NW>
int launch_ov_nw(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule) {
  FastCfg F;
  // multi-million-op graphs (configs 4/5) need 16-entry device rings in the
  // residency pass; a replay that overflowed raises the hint for the next
  F.qc = std::max<uint32_t>(ctx->ring, b->ring_hint);
  if (b->n > 0 && b->sum_n / b->n > 1000000ull) F.qc = std::max<uint32_t>(F.qc, 16);
  // range list: every op completing in one round pushes one; identical
  // workers complete together (config 4: 64 BW + 64 IN cascades per round)
  F.rl = std::max<uint32_t>(128, std::min<uint32_t>(1024, 4 * b->max_d));
  const uint32_t nt = 32 * NW;
  uint32_t kd = std::max<uint32_t>(1, (b->max_d + nt - 1) / nt);
  if (kd > 8) kd = kd <= 12 ? 12 : 16;
  F.kd = kd;
  F.dcap = std::max<uint32_t>(1, std::min<uint32_t>(b->max_d, nt * kd));
  F.ccap = (2 * b->max_cnt_ov + 15) & ~15u;  // u16 counters
  const size_t limit = ctx->smem_optin - 64;
  if (ctx->gcnt || fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW) > size_t(ctx->smem_per_sm) / 4)
    F.ccap = 16;
  while (fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW) > limit && F.dcap > 1) F.dcap /= 2;
  const size_t target = std::max<size_t>(fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW),
                                         size_t(ctx->smem_per_sm) / 8 - 1024);
  while (F.qc < 64 && fast_bytes(F.dcap, F.qc * 2, F.rl, F.ccap, NW) <= std::min(target, limit))
    F.qc *= 2;
  F.warp_bytes = static_cast<uint32_t>(fast_bytes(F.dcap, F.qc, F.rl, F.ccap, NW)) +
                 dpro_k::kOvListBytes + 16 * F.dcap;
  switch (kd) {
    case 1: return launch_ov_kd<NW, 1>(ctx, b, want_schedule, F);
    case 2: return launch_ov_kd<NW, 2>(ctx, b, want_schedule, F);
    case 3: return launch_ov_kd<NW, 3>(ctx, b, want_schedule, F);
    case 4: return launch_ov_kd<NW, 4>(ctx, b, want_schedule, F);
    case 5: return launch_ov_kd<NW, 5>(ctx, b, want_schedule, F);
    case 6: return launch_ov_kd<NW, 6>(ctx, b, want_schedule, F);
    case 7: return launch_ov_kd<NW, 7>(ctx, b, want_schedule, F);
    case 8: return launch_ov_kd<NW, 8>(ctx, b, want_schedule, F);
    default: return set_err(ctx, DPRO_EUNSUPPORTED, "overlay replay: too many devices");
  }
}

// Candidates the overlay replay could not finish (materialized: !fast
// overlays, kRetryMat after the kernel) re-run as an ordinary delta batch;
// their results are copied into this batch's layout.
int finish_overlay_mat(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule) {
  unsigned w[12] = {0};
  CU(cudaMemcpyAsync(w, b->work.p, 48, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (w[5] > static_cast<unsigned>(b->n) / 8 && b->F.qc < 64) b->ring_hint = 2 * b->F.qc;
  if (w[11]) {  // global-ring candidates: run them first next time
    std::vector<uint32_t> h(std::min<unsigned>(w[11], static_cast<unsigned>(b->n)));
    CU(cudaMemcpy(h.data(), b->hint.p, 4 * h.size(), cudaMemcpyDeviceToHost));
    for (uint32_t c : h)
      if (std::find(b->g3.begin(), b->g3.end(), static_cast<int32_t>(c)) == b->g3.end())
        b->g3.push_back(static_cast<int32_t>(c));
  }
  if (b->n_mat == 0 && w[1] == 0) return DPRO_OK;
  std::vector<int32_t> stv(b->n);
  CU(cudaMemcpy(stv.data(), b->O.status, 4 * size_t(b->n), cudaMemcpyDeviceToHost));
  std::vector<int32_t> idx;
  std::vector<dpro_delta> ds;
  for (int32_t i = 0; i < b->n; ++i)
    if (!b->ovh[i].fast || stv[i] == dpro_k::kRetryMat) {
      idx.push_back(i);
      ds.push_back(b->dcopy[i].d);
    }
  if (idx.empty()) return DPRO_OK;
  dpro_batch sub;
  sub.n = static_cast<int32_t>(idx.size());
  sub.memspace = DPRO_DEVICE;
  int st = build_delta_batch(ctx, &sub, b->res, ds.data());
  if (st != DPRO_OK) return st;
  st = ctx->fast ? launch_fast(ctx, &sub, want_schedule) : launch_general(ctx, &sub, want_schedule);
  if (st != DPRO_OK) return st;
  for (size_t k = 0; k < idx.size(); ++k) {
    const Cand& p = b->hc[idx[k]];
    const Cand& q = sub.hc[k];
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream)
                   : cudaSuccess;
    };
    const int32_t i = idx[k];
    CU(cp(b->O.makespan + i, sub.O.makespan + k, 8));
    CU(cp(b->O.err + i, sub.O.err + k, 8));
    CU(cp(b->O.status + i, sub.O.status + k, 4));
    if (want_schedule) {
      CU(cp(b->O.start + p.op_off, sub.O.start + q.op_off, 8 * size_t(p.n)));
      CU(cp(b->O.end + p.op_off, sub.O.end + q.op_off, 8 * size_t(p.n)));
    }
    CU(cp(b->S.qbuf + p.op_off, sub.S.qbuf + q.op_off, 4 * size_t(p.n)));
    CU(cp(b->S.sched + p.op_off, sub.S.sched + q.op_off, size_t(p.n)));
    CU(cp(b->S.devoff + p.dof_off, sub.S.devoff + q.dof_off, 4 * (size_t(p.d) + 1)));
    CU(cp(b->S.busy + p.dev_off, sub.S.busy + q.dev_off, 8 * size_t(p.d)));
    CU(cp(b->S.dhead + p.dev_off, sub.S.dhead + q.dev_off, 4 * size_t(p.d)));
  }
  CU(cudaStreamSynchronize(ctx->stream));  // sub's buffers die here
  return DPRO_OK;
}

int launch_overlay(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule) {
  int nw = ctx->warps;
  if (nw == 0) nw = b->max_d <= 32 ? 1 : b->max_d <= 64 ? 2 : 4;
  // global-ring residency pass (multi-million-op graphs): registers, not
  // shared memory, bound the CTAs per SM, so 2-warp CTAs (16 per SM) keep
  // twice the candidates in flight of 4-warp ones (config 4: +16 %)
  if (ctx->warps == 0 && ctx->gring0 != 0 && b->max_d <= 128 && b->n > 0 &&
      b->sum_n / b->n > 1000000ull)
    nw = 2;
  int st;
  switch (nw) {
    case 1: st = launch_ov_nw<1>(ctx, b, want_schedule); break;
    case 2: st = launch_ov_nw<2>(ctx, b, want_schedule); break;
    case 8: st = launch_ov_nw<8>(ctx, b, want_schedule); break;
    default: st = launch_ov_nw<4>(ctx, b, want_schedule); break;
  }
  if (st != DPRO_OK) return st;
  return finish_overlay_mat(ctx, b, want_schedule);
}

}  // namespace

extern "C" {

int dpro_cuda_batch_replay(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule) {
  if (!ctx || !b) return DPRO_EINVAL;
  if (b->n == 0) {  // nothing to launch; results are empty
    b->replayed = true;
    b->with_schedule = want_schedule != 0;
    return DPRO_OK;
  }
  CU(cudaSetDevice(ctx->device));
  const int st = b->overlay ? launch_overlay(ctx, b, want_schedule)
                 : ctx->fast ? launch_fast(ctx, b, want_schedule)
                             : launch_general(ctx, b, want_schedule);
  if (st != DPRO_OK) return st;
  b->replayed = true;
  b->with_schedule = want_schedule != 0;
  b->qpos_ready = false;
  return DPRO_OK;
}

#ifdef DPRO_PROFILE
extern "C" int dpro_debug_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, dpro_k::g_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(dpro_k::g_prof, z, sizeof z);
  return 0;
}
#endif

int dpro_cuda_batch_stats(dpro_ctx* ctx, dpro_batch* b, int64_t* stats) {
  if (!ctx || !b || !stats) return DPRO_EINVAL;
  CU(cudaSetDevice(ctx->device));
  unsigned w[4] = {0, 0, 0, 0};
  CU(cudaMemcpyAsync(w, b->work.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  stats[0] = ctx->fast ? w[1] : b->n;
  stats[1] = b->F.warp_bytes;
  stats[2] = b->blocks_per_sm_fast;
  stats[3] = b->F.qc;
  stats[4] = ctx->fast ? w[3] : 0;
  return DPRO_OK;
}

int dpro_cuda_batch_diag(dpro_ctx* ctx, dpro_batch* b, int64_t* out, int32_t n) {
  if (!ctx || !b || !out || n < 0) return DPRO_EINVAL;
  CU(cudaSetDevice(ctx->device));
  unsigned w[12] = {0};
  CU(cudaMemcpyAsync(w, b->work.p, 48, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  int64_t v[10] = {w[5], w[6], w[7], w[8], b->overlay ? 1 : 0, b->n_mat, -1, -1, -1, -1};
  if (b->pev_valid)
    for (int k = 0; k < 4; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, b->pev[k], b->pev[k + 1]) == cudaSuccess)
        v[6 + k] = static_cast<int64_t>(ms * 1000.0f);
      else
        cudaGetLastError();
    }
  for (int32_t i = 0; i < n && i < 10; ++i) out[i] = v[i];
  return DPRO_OK;
}

int dpro_cuda_batch_device_results(dpro_batch* b, int64_t** makespan,
                                   int32_t** status, int64_t** err,
                                   int64_t** start, int64_t** end) {
  if (!b) return DPRO_EINVAL;
  if (makespan) *makespan = reinterpret_cast<int64_t*>(b->O.makespan);
  if (status) *status = b->O.status;
  if (err) *err = reinterpret_cast<int64_t*>(b->O.err);
  if (start) *start = reinterpret_cast<int64_t*>(b->O.start);
  if (end) *end = reinterpret_cast<int64_t*>(b->O.end);
  return DPRO_OK;
}

int dpro_cuda_batch_results(dpro_ctx* ctx, dpro_batch* b, int64_t* makespan,
                            int32_t* status, int64_t* err, int64_t* start,
                            int64_t* end) {
  if (!ctx || !b) return DPRO_EINVAL;
  if (!b->replayed) return set_err(ctx, DPRO_EINVAL, "batch not replayed");
  CU(cudaSetDevice(ctx->device));
  const size_t n = b->n;
  if (makespan) CU(cudaMemcpyAsync(makespan, b->O.makespan, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (status) CU(cudaMemcpyAsync(status, b->O.status, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (err) CU(cudaMemcpyAsync(err, b->O.err, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if ((start || end) && !b->with_schedule)
    return set_err(ctx, DPRO_EINVAL, "replay ran without want_schedule");
  if (start) CU(cudaMemcpyAsync(start, b->O.start, b->sum_n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (end) CU(cudaMemcpyAsync(end, b->O.end, b->sum_n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DPRO_OK;
}

int dpro_cuda_batch_timelines(dpro_ctx* ctx, dpro_batch* b, int32_t cand,
                              uint32_t* order, uint32_t* dev_off,
                              int64_t* busy) {
  if (!ctx || !b || cand < 0 || cand >= b->n) return DPRO_EINVAL;
  if (!b->replayed) return set_err(ctx, DPRO_EINVAL, "batch not replayed");
  CU(cudaSetDevice(ctx->device));
  const Cand& h = b->hc[cand];
  // queue regions hold only the dispatched prefix [devoff[d], dhead[d]);
  // ops never scheduled (cycles / init quirk) leave holes: compact them out
  std::vector<uint32_t> q(h.n), doff(h.d + 1), dh(h.d);
  if (h.n) CU(cudaMemcpyAsync(q.data(), b->S.qbuf + h.op_off, size_t(h.n) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(doff.data(), b->S.devoff + h.dof_off, size_t(h.d + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (h.d) CU(cudaMemcpyAsync(dh.data(), b->S.dhead + h.dev_off, size_t(h.d) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (busy && h.d) CU(cudaMemcpyAsync(busy, b->S.busy + h.dev_off, size_t(h.d) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  // a candidate that stopped before replaying (missing duration) has no
  // timelines; regions are clamped so stale scratch can never overrun
  int32_t stc = 0;
  CU(cudaMemcpy(&stc, b->O.status + cand, 4, cudaMemcpyDeviceToHost));
  uint32_t k = 0;
  for (uint32_t d = 0; d < h.d; ++d) {
    if (dev_off) dev_off[d] = k;
    if (stc == DPRO_MISSING_PROFILE) continue;
    const uint32_t lo = std::min(doff[d], h.n), hi = std::min(std::min(dh[d], doff[d + 1]), h.n);
    for (uint32_t p = lo; p < hi; ++p, ++k)
      if (order) order[k] = q[p];
  }
  if (dev_off) dev_off[h.d] = k;
  return DPRO_OK;
}

int dpro_cuda_batch_scheduled(dpro_ctx* ctx, dpro_batch* b, int32_t cand,
                              uint8_t* scheduled) {
  if (!ctx || !b || cand < 0 || cand >= b->n || !scheduled) return DPRO_EINVAL;
  if (!b->replayed) return set_err(ctx, DPRO_EINVAL, "batch not replayed");
  CU(cudaSetDevice(ctx->device));
  const Cand& h = b->hc[cand];
  CU(cudaMemcpyAsync(scheduled, b->S.sched + h.op_off, h.n, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DPRO_OK;
}

int dpro_cuda_batch_critical_paths(dpro_ctx* ctx, dpro_batch* b,
                                   uint32_t* paths, int64_t* path_len) {
  if (!ctx || !b) return DPRO_EINVAL;
  if (!b->replayed || !b->with_schedule)
    return set_err(ctx, DPRO_EINVAL, "critical path needs a replay with want_schedule");
  if (b->overlay)
    return set_err(ctx, DPRO_EUNSUPPORTED,
                   "critical paths need materialized candidates (option overlay=0)");
  CU(cudaSetDevice(ctx->device));
  const size_t n = b->n;
  std::vector<unsigned long long> e_off(n), po_off(n);
  unsigned long long eo = 0, po = 0;
  for (size_t i = 0; i < n; ++i) {
    e_off[i] = eo;
    po_off[i] = po;
    eo += b->n_edges[i];
    po += b->n_ops[i] + 1;
  }
  const size_t s_po = align16(po * 4 + 4), s_e = align16(eo * 4 + 4),
               s_n = align16(b->sum_n * 4 + 4), s_off = align16(n * 8 + 8);
  const size_t s_paths = align16(b->sum_n * 4 + 4), s_len = align16(n * 8 + 8);
  CU(b->cp.ensure(s_po + s_e + 2 * s_n + 2 * s_off + s_paths + s_len));
  CpScratch P;
  size_t o = 0;
  P.pred_off = b->cp.as<uint32_t>(o); o += s_po;
  P.pred = b->cp.as<uint32_t>(o); o += s_e;
  P.good = b->cp.as<uint32_t>(o); o += s_n;
  P.stack = b->cp.as<uint32_t>(o); o += s_n;
  P.e_off = b->cp.as<unsigned long long>(o); o += s_off;
  P.po_off = b->cp.as<unsigned long long>(o); o += s_off;
  uint32_t* d_paths = b->cp.as<uint32_t>(o); o += s_paths;
  long long* d_len = b->cp.as<long long>(o); o += s_len;
  CU(cudaMemcpyAsync(P.e_off, e_off.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(P.po_off, po_off.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (!b->qpos_ready)
    dpro_k::qpos_scatter_kernel<<<std::max<int>(1, std::min<int>(n, ctx->sm_count * 8)), 256, 0,
                                  ctx->stream>>>(b->desc.as<Cand>(), b->n, b->S, b->O);
  b->qpos_ready = true;
  const int threads = 128;
  const int grid = std::max<int>(1, std::min<int>((n * 32 + threads - 1) / threads, ctx->sm_count * 8));
  dpro_k::critical_path_kernel<<<grid, threads, 0, ctx->stream>>>(
      b->desc.as<Cand>(), b->n, b->S, b->O, P, d_paths, d_len);
  CU(cudaGetLastError());
  if (paths) CU(cudaMemcpyAsync(paths, d_paths, b->sum_n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (path_len) CU(cudaMemcpyAsync(path_len, d_len, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DPRO_OK;
}

int dpro_cuda_batch_peak_memory(dpro_ctx* ctx, dpro_batch* b, const int64_t* op_bytes,
                                const int32_t* op_node, const int32_t* n_nodes,
                                const int64_t* persistent, int64_t* peak) {
  if (!ctx || !b || !op_bytes || !op_node || !n_nodes || !persistent || !peak)
    return DPRO_EINVAL;
  if (!b->replayed || !b->with_schedule)
    return set_err(ctx, DPRO_EINVAL, "peak memory needs a replay with want_schedule");
  if (b->overlay)
    return set_err(ctx, DPRO_EUNSUPPORTED,
                   "peak memory needs materialized candidates (option overlay=0)");
  CU(cudaSetDevice(ctx->device));
  const size_t n = b->n, N = b->sum_n;
  std::vector<unsigned long long> seg0(n);
  unsigned long long S = 0;
  for (size_t i = 0; i < n; ++i) {
    seg0[i] = S;
    S += static_cast<unsigned long long>(std::max(0, n_nodes[i]));
  }
  // event count bound: 2 per op (exact counts come from mem_count_kernel)
  const size_t s_b = align16(N * 8 + 8), s_n = align16(N * 4 + 4), s_s0 = align16(n * 8 + 8),
               s_cnt = align16(S * 4 + 4), s_off = align16((S + 1) * 8 + 8),
               s_ev = align16(2 * N * 8 + 8), s_seg8 = align16(S * 8 + 8);
  DevBuf buf;
  size_t cub_tmp = 0, sort_tmp = 0;
  CU(cub::DeviceScan::ExclusiveSum(nullptr, cub_tmp, (unsigned int*)nullptr,
                                   (unsigned long long*)nullptr, (int)std::max<unsigned long long>(S + 1, 1)));
  CU(cub::DeviceSegmentedRadixSort::SortPairs(
      nullptr, sort_tmp, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
      (const long long*)nullptr, (long long*)nullptr, (int64_t)(2 * N), (int64_t)S,
      (const unsigned long long*)nullptr, (const unsigned long long*)nullptr));
  const size_t s_tmp = align16(std::max(cub_tmp, sort_tmp) + 16);
  CU(buf.ensure(s_b + s_n + s_s0 + s_cnt + 2 * s_off + 4 * s_ev + 2 * s_seg8 + s_tmp));
  size_t o = 0;
  auto take = [&](size_t bytes) { void* q = buf.as<char>(o); o += bytes; return q; };
  dpro_k::MemIn M;
  long long* d_bytes = static_cast<long long*>(take(s_b));
  int* d_node = static_cast<int*>(take(s_n));
  unsigned long long* d_seg0 = static_cast<unsigned long long*>(take(s_s0));
  M.seg_cnt = static_cast<unsigned int*>(take(s_cnt));
  M.seg_off = static_cast<unsigned long long*>(take(s_off));
  M.cursor = static_cast<unsigned long long*>(take(s_off));
  M.keys = static_cast<unsigned long long*>(take(s_ev));
  unsigned long long* keys_out = static_cast<unsigned long long*>(take(s_ev));
  M.vals = static_cast<long long*>(take(s_ev));
  long long* vals_sorted = static_cast<long long*>(take(s_ev));
  long long* d_pers = static_cast<long long*>(take(s_seg8));
  long long* d_peak = static_cast<long long*>(take(s_seg8));
  void* tmp = take(s_tmp);
  M.bytes = d_bytes;
  M.node = d_node;
  M.seg0 = d_seg0;
  CU(cudaMemcpyAsync(d_bytes, op_bytes, N * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(d_node, op_node, N * 4, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(d_seg0, seg0.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (S) CU(cudaMemcpyAsync(d_pers, persistent, S * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(M.seg_cnt, 0, s_cnt, ctx->stream));
  const int grid = std::max<int>(1, std::min<int>((int)n, ctx->sm_count * 8));
  dpro_k::mem_count_kernel<<<grid, 256, 0, ctx->stream>>>(b->desc.as<Cand>(), b->n, M);
  CU(cudaGetLastError());
  size_t t1 = cub_tmp;
  CU(cub::DeviceScan::ExclusiveSum(tmp, t1, M.seg_cnt, M.seg_off, (int)(S + 1), ctx->stream));
  CU(cudaMemcpyAsync(M.cursor, M.seg_off, S * 8 + 8, cudaMemcpyDeviceToDevice, ctx->stream));
  dpro_k::mem_fill_kernel<<<grid, 256, 0, ctx->stream>>>(b->desc.as<Cand>(), b->n, b->O, M);
  CU(cudaGetLastError());
  unsigned long long total = 0;
  CU(cudaMemcpyAsync(&total, M.seg_off + S, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (total > 0) {
    size_t t2 = sort_tmp;
    CU(cub::DeviceSegmentedRadixSort::SortPairs(tmp, t2, M.keys, keys_out, M.vals, vals_sorted,
                                                (int64_t)total, (int64_t)S, M.seg_off,
                                                M.seg_off + 1, 0, 64, ctx->stream));
  }
  if (S) {
    const int sg = std::max<int>(1, std::min<int>((int)((S * 32 + 255) / 256), ctx->sm_count * 16));
    dpro_k::mem_scan_kernel<<<sg, 256, 0, ctx->stream>>>(S, M.seg_off, vals_sorted, d_pers,
                                                         d_peak);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(peak, d_peak, S * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return DPRO_OK;
}

int dpro_cuda_critical_path(dpro_ctx* ctx, const dpro_csr* graph,
                            const int64_t* start, const int64_t* end,
                            int64_t makespan, uint32_t* path,
                            int64_t* path_len) {
  if (!ctx || !graph || !path_len) return DPRO_EINVAL;
  if (graph->n_ops > 0 && (!start || !end || !path)) return DPRO_EINVAL;
  dpro_batch* b = dpro_cuda_batch_create(ctx, graph, 1, DPRO_HOST);
  if (!b) return DPRO_EINVAL;
  int st = DPRO_OK;
  const size_t n = graph->n_ops;
  auto run = [&]() -> int {
    // the execution graph already carries the timeline edges: no qpos links
    CU(cudaMemsetAsync(b->S.qpos, 0xFF, n * 4 + 4, ctx->stream));
    if (n) {
      CU(cudaMemcpyAsync(b->O.start, start, n * 8, cudaMemcpyHostToDevice, ctx->stream));
      CU(cudaMemcpyAsync(b->O.end, end, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    const long long T = makespan;
    const int ok = 0;
    CU(cudaMemcpyAsync(b->O.makespan, &T, 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(b->O.status, &ok, 4, cudaMemcpyHostToDevice, ctx->stream));
    b->replayed = true;
    b->with_schedule = true;
    b->qpos_ready = true;  // no timelines: the exec graph's edges stand for them
    return dpro_cuda_batch_critical_paths(ctx, b, path, path_len);
  };
  st = run();
  dpro_cuda_batch_destroy(ctx, b);
  return st;
}

int dpro_cuda_replay_batch(dpro_ctx* ctx, const dpro_csr* cands,
                           int32_t n_cands, int32_t memspace,
                           int64_t* makespan, int64_t* start, int64_t* end,
                           int32_t* status, int64_t* err) {
  if (!ctx) return DPRO_EINVAL;
  dpro_batch* b = dpro_cuda_batch_create(ctx, cands, n_cands, memspace);
  if (!b) return DPRO_EINVAL;
  int st = dpro_cuda_batch_replay(ctx, b, (start || end) ? 1 : 0);
  if (st == DPRO_OK)
    st = dpro_cuda_batch_results(ctx, b, makespan, status, err, start, end);
  dpro_cuda_batch_destroy(ctx, b);
  return st;
}

}  // extern "C"

namespace {

// K2 host side: tables of the index order / devices / link parameters of
// the comm-only graphs, then tsync_*_kernel writes every graph's CSR into
// the batch arena and the batch is packed like any device-memspace batch.
uint64_t tsync_fnv1a(const std::string& x) {  // graph.cpp:57-64
  uint64_t h = 1469598103934665603ULL;
  for (unsigned char c : x) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}

// rank of each decimal string of 0..X-1 in byte order, and its inverse
void decimal_ranks(int X, std::vector<int>& rank, std::vector<int>& inv) {
  inv.resize(X);
  for (int x = 0; x < X; ++x) inv[x] = x;
  std::sort(inv.begin(), inv.end(),
            [](int a, int b) { return std::to_string(a) < std::to_string(b); });
  rank.resize(X);
  for (int r = 0; r < X; ++r) rank[inv[r]] = r;
}

// Appends v to the host staging image (device offset off, image offset
// off - base) and sets dptr to where it lands in buf.
template <typename T>
void upload_table(DevBuf& buf, size_t base, size_t& off, const std::vector<T>& v, const T*& dptr,
                  std::vector<char>& stage) {
  const size_t bytes = v.size() * sizeof(T);
  if (stage.size() < off - base + align16(bytes)) stage.resize(off - base + align16(bytes));
  if (bytes) std::memcpy(stage.data() + (off - base), v.data(), bytes);
  dptr = reinterpret_cast<const T*>(static_cast<char*>(buf.p) + off);
  off += align16(bytes);
}

int build_tsync_batch(dpro_ctx* ctx, dpro_batch* b, const dpro_cluster_desc& cd,
                      const std::vector<int64_t>& bytes, const std::vector<int32_t>& ks) {
  Tracer tr;
  const int32_t n = static_cast<int32_t>(bytes.size());
  std::vector<std::string> names(cd.n_nodes);
  for (int i = 0; i < cd.n_nodes; ++i) names[i] = cd.node_ids[i];
  std::map<std::pair<int, int>, std::pair<double, double>> link;  // first wins
  for (int l = 0; l < cd.n_links; ++l)
    link.emplace(std::make_pair(cd.link_src[l], cd.link_dst[l]),
                 std::make_pair(cd.link_bw[l], cd.link_lat[l]));
  auto bwlat = [&](int a, int z) {
    auto it = link.find({a, z});
    return it == link.end() ? std::make_pair(1.0, 0.0) : it->second;
  };
  std::vector<int> workers, ps;
  for (int i = 0; i < cd.n_nodes; ++i) {
    if (cd.node_role[i] == 0) workers.push_back(i);
    if (cd.node_role[i] == 1) ps.push_back(i);
  }
  auto by_name = [&](int a, int z) { return names[a] < names[z]; };
  std::sort(workers.begin(), workers.end(), by_name);
  std::sort(ps.begin(), ps.end(), by_name);
  int kmax = 1;
  for (int32_t x : ks) kmax = std::max(kmax, x);
  std::vector<int> inv_p, inv_p_off(kmax + 2, 0);
  for (int kk = 1; kk <= kmax; ++kk) {
    std::vector<int> r, inv;
    decimal_ranks(kk, r, inv);
    inv_p_off[kk] = static_cast<int>(inv_p.size());
    inv_p.insert(inv_p.end(), inv.begin(), inv.end());
  }
  std::vector<dpro_k::TsyncDesc> desc(n);
  std::vector<uint32_t> n_dev(n);
  std::vector<char> stage;
  size_t toff = 0;
  dpro_k::TsyncRing R{};
  dpro_k::TsyncPs P{};
  // host vectors kept alive until the upload
  std::vector<int> rank_c, inv_c, rank_s, inv_s, server_of, srv_off, pull_w, push_w, dev_off;
  std::vector<uint16_t> link_dev, dev_push, dev_pull;
  std::vector<double> lbw, llat, bw_push, lat_push, bw_pull, lat_pull;
  if (cd.scheme == 0) {
    std::vector<int> ring;
    if (cd.n_ring > 0) ring.assign(cd.ring_order, cd.ring_order + cd.n_ring);
    else ring = workers;
    const int N = static_cast<int>(ring.size());
    if (N < 2) return set_err(ctx, DPRO_EINVAL, "degenerate ring: allreduce needs at least 2 workers");
    const int C = cd.chunks_per_tensor > 0 ? cd.chunks_per_tensor : N, S = 2 * (N - 1);
    decimal_ranks(C, rank_c, inv_c);
    decimal_ranks(S, rank_s, inv_s);
    std::vector<std::pair<std::string, std::string>> lk(N);
    for (int i = 0; i < N; ++i) lk[i] = {names[ring[i]], names[ring[(i + 1) % N]]};
    std::vector<std::pair<std::string, std::string>> sorted_lk(lk);
    std::sort(sorted_lk.begin(), sorted_lk.end());
    sorted_lk.erase(std::unique(sorted_lk.begin(), sorted_lk.end()), sorted_lk.end());
    link_dev.resize(N);
    lbw.resize(N);
    llat.resize(N);
    for (int i = 0; i < N; ++i) {
      link_dev[i] = static_cast<uint16_t>(
          std::lower_bound(sorted_lk.begin(), sorted_lk.end(), lk[i]) - sorted_lk.begin());
      const auto bl = bwlat(ring[i], ring[(i + 1) % N]);
      lbw[i] = bl.first;
      llat[i] = bl.second;
    }
    R.n_workers = N;
    R.chunks = C;
    R.steps = S;
    unsigned long long oo = 0, eo = 0;
    for (int32_t i = 0; i < n; ++i) {
      const uint64_t kcs = uint64_t(ks[i]) * C * S;
      if (2 * kcs >= (1ull << 31)) return set_err(ctx, DPRO_EINVAL, "t_sync graph too large");
      desc[i] = {bytes[i], ks[i], static_cast<uint32_t>(2 * kcs),
                 static_cast<uint32_t>(2 * kcs - uint64_t(ks[i]) * C), oo, eo};
      n_dev[i] = static_cast<uint32_t>(sorted_lk.size());
      oo += desc[i].n;
      eo += desc[i].e;
    }
  } else {
    if (ps.empty()) return set_err(ctx, DPRO_EINVAL, "parameter-server scheme requires at least one ps node");
    if (workers.empty()) return set_err(ctx, DPRO_EINVAL, "parameter-server scheme requires at least one worker");
    const int W = static_cast<int>(workers.size()), NS = static_cast<int>(ps.size());
    // worker order of the pull ids ("...#pull#<server>#<w>") and the push
    // ids ("...#push#<w>#<server>") per server
    pull_w.resize(size_t(NS) * W);
    push_w.resize(size_t(NS) * W);
    for (int sv = 0; sv < NS; ++sv) {
      std::vector<int> o(W);
      for (int w = 0; w < W; ++w) o[w] = w;
      std::sort(o.begin(), o.end(), [&](int a, int z) { return names[workers[a]] < names[workers[z]]; });
      std::copy(o.begin(), o.end(), pull_w.begin() + size_t(sv) * W);
      const std::string& sn = names[ps[sv]];
      std::sort(o.begin(), o.end(), [&](int a, int z) {
        return names[workers[a]] + "#" + sn < names[workers[z]] + "#" + sn;
      });
      std::copy(o.begin(), o.end(), push_w.begin() + size_t(sv) * W);
    }
    bw_push.resize(size_t(NS) * W);
    lat_push.resize(size_t(NS) * W);
    bw_pull.resize(size_t(NS) * W);
    lat_pull.resize(size_t(NS) * W);
    for (int sv = 0; sv < NS; ++sv)
      for (int w = 0; w < W; ++w) {
        const auto a = bwlat(workers[w], ps[sv]), z = bwlat(ps[sv], workers[w]);
        bw_push[size_t(sv) * W + w] = a.first;
        lat_push[size_t(sv) * W + w] = a.second;
        bw_pull[size_t(sv) * W + w] = z.first;
        lat_pull[size_t(sv) * W + w] = z.second;
      }
    // per k: the server of each partition (by rank) and the dense device ids
    // over the links those servers use
    srv_off.assign(kmax + 2, 0);
    dev_off.assign(kmax + 2, 0);
    std::vector<uint32_t> ndev_k(kmax + 1, 0);
    for (int kk = 1; kk <= kmax; ++kk) {
      srv_off[kk] = static_cast<int>(server_of.size());
      std::vector<char> used(NS, 0);
      for (int pr = 0; pr < kk; ++pr) {
        const int p = inv_p[inv_p_off[kk] + pr];
        const std::string unit = kk == 1 ? "tsync" : "tsync#p" + std::to_string(p);
        const int sv = static_cast<int>(tsync_fnv1a(unit) % static_cast<uint64_t>(NS));
        server_of.push_back(sv);
        used[sv] = 1;
      }
      std::vector<std::pair<std::string, std::string>> lk;
      for (int sv = 0; sv < NS; ++sv)
        if (used[sv])
          for (int w = 0; w < W; ++w) {
            lk.push_back({names[workers[w]], names[ps[sv]]});
            lk.push_back({names[ps[sv]], names[workers[w]]});
          }
      std::sort(lk.begin(), lk.end());
      lk.erase(std::unique(lk.begin(), lk.end()), lk.end());
      dev_off[kk] = static_cast<int>(dev_push.size());
      dev_push.resize(dev_push.size() + size_t(NS) * W, 0);
      dev_pull.resize(dev_pull.size() + size_t(NS) * W, 0);
      for (int sv = 0; sv < NS; ++sv)
        if (used[sv])
          for (int w = 0; w < W; ++w) {
            const std::pair<std::string, std::string> a{names[workers[w]], names[ps[sv]]},
                z{names[ps[sv]], names[workers[w]]};
            dev_push[dev_off[kk] + size_t(sv) * W + w] =
                static_cast<uint16_t>(std::lower_bound(lk.begin(), lk.end(), a) - lk.begin());
            dev_pull[dev_off[kk] + size_t(sv) * W + w] =
                static_cast<uint16_t>(std::lower_bound(lk.begin(), lk.end(), z) - lk.begin());
          }
      ndev_k[kk] = static_cast<uint32_t>(lk.size());
    }
    P.n_workers = W;
    unsigned long long oo = 0, eo = 0;
    for (int32_t i = 0; i < n; ++i) {
      const uint64_t kk = ks[i];
      if (4 * kk * W + kk * W * W >= (1ull << 31))
        return set_err(ctx, DPRO_EINVAL, "t_sync graph too large");
      desc[i] = {bytes[i], ks[i], static_cast<uint32_t>(4 * kk * W),
                 static_cast<uint32_t>(kk * W * W + 2 * kk * W), oo, eo};
      n_dev[i] = ndev_k[ks[i]];
      oo += desc[i].n;
      eo += desc[i].e;
    }
  }
  // device arena: CSR arrays + tables
  unsigned long long so = 0, se = 0;
  for (int32_t i = 0; i < n; ++i) {
    so += desc[i].n;
    se += desc[i].e;
  }
  const size_t a_dur = align16(so * 8 + 8), a_dev = align16(so * 2 + 2), a_fl = align16(so + 1),
               a_so = align16((so + n) * 4 + 4), a_su = align16(se * 4 + 4), a_in = align16(so * 4 + 4);
  const size_t csr_bytes = a_dur + a_dev + a_fl + a_so + a_su + a_in;
  // tables after the CSR arrays
  CU(b->arena.ensure(csr_bytes + (1u << 20) + 64 * (dev_push.size() + pull_w.size() + inv_p.size() +
                                                      rank_c.size() + rank_s.size() + 16 * link_dev.size() + 64)));
  size_t off = csr_bytes;
  const size_t t0 = off;
  if (cd.scheme == 0) {
    upload_table(b->arena, t0, off, rank_c, R.rank_c, stage);
    upload_table(b->arena, t0, off, inv_c, R.inv_c, stage);
    upload_table(b->arena, t0, off, rank_s, R.rank_s, stage);
    upload_table(b->arena, t0, off, inv_s, R.inv_s, stage);
    upload_table(b->arena, t0, off, inv_p, R.inv_p, stage);
    upload_table(b->arena, t0, off, inv_p_off, R.inv_p_off, stage);
    upload_table(b->arena, t0, off, link_dev, R.link_dev, stage);
    upload_table(b->arena, t0, off, lbw, R.link_bw, stage);
    upload_table(b->arena, t0, off, llat, R.link_lat, stage);
  } else {
    upload_table(b->arena, t0, off, inv_p, P.inv_p, stage);
    upload_table(b->arena, t0, off, inv_p_off, P.inv_p_off, stage);
    upload_table(b->arena, t0, off, server_of, P.server_of, stage);
    upload_table(b->arena, t0, off, srv_off, P.srv_off, stage);
    upload_table(b->arena, t0, off, pull_w, P.pull_w, stage);
    upload_table(b->arena, t0, off, push_w, P.push_w, stage);
    upload_table(b->arena, t0, off, dev_off, P.dev_off, stage);
    upload_table(b->arena, t0, off, dev_push, P.dev_push, stage);
    upload_table(b->arena, t0, off, dev_pull, P.dev_pull, stage);
    upload_table(b->arena, t0, off, bw_push, P.bw_push, stage);
    upload_table(b->arena, t0, off, lat_push, P.lat_push, stage);
    upload_table(b->arena, t0, off, bw_pull, P.bw_pull, stage);
    upload_table(b->arena, t0, off, lat_pull, P.lat_pull, stage);
  }
  {
    std::vector<dpro_k::TsyncDesc> dd(desc);
    const dpro_k::TsyncDesc* dptr = nullptr;
    upload_table(b->arena, t0, off, dd, dptr, stage);
    if (off > b->arena.cap) return set_err(ctx, DPRO_ENOMEM, "t_sync tables");
    CU(cudaMemcpyAsync(b->arena.as<char>(t0), stage.data(), off - t0, cudaMemcpyHostToDevice,
                       ctx->stream));
    dpro_k::TsyncOut O;
    size_t o = 0;
    O.dur = b->arena.as<long long>(o); o += a_dur;
    O.dev = b->arena.as<uint16_t>(o); o += a_dev;
    O.flags = b->arena.as<uint8_t>(o); o += a_fl;
    O.succ_off = b->arena.as<uint32_t>(o); o += a_so;
    O.succ = b->arena.as<uint32_t>(o); o += a_su;
    O.indeg = b->arena.as<uint32_t>(o); o += a_in;
    const int grid = std::max(1, std::min<int>(n, ctx->sm_count * 8));
    if (n > 0) {
      if (cd.scheme == 0)
        dpro_k::tsync_ring_kernel<<<grid, 256, 0, ctx->stream>>>(dptr, n, R, O);
      else
        dpro_k::tsync_ps_kernel<<<grid, 256, 0, ctx->stream>>>(dptr, n, P, O);
      CU(cudaGetLastError());
    }
    CU(cudaStreamSynchronize(ctx->stream));  // stage is a local
    // the batch: device CSRs in the arena, packed like any device batch
    std::vector<dpro_csr> csrs(n);
    for (int32_t i = 0; i < n; ++i) {
      const auto& c = desc[i];
      csrs[i] = {c.n, c.e, n_dev[i], 64, O.dur + c.op_off, O.dev + c.op_off, O.flags + c.op_off,
                 O.succ_off + c.op_off + i, O.succ + c.e_off, O.indeg + c.op_off};
    }
    b->memspace = DPRO_DEVICE;
    tr.mark("t_sync graphs generated (K2)");
    return build_batch(ctx, b, csrs.data());
  }
}

}  // namespace

extern "C" {

dpro_batch* dpro_cuda_batch_create_tsync(dpro_ctx* ctx, const dpro_cluster_desc* cluster,
                                         const int64_t* bytes, const int32_t* k, int32_t n) {
  if (!ctx || !cluster || n < 0 || (n > 0 && (!bytes || !k))) return nullptr;
  for (int32_t i = 0; i < n; ++i)
    if (k[i] < 1) {
      ctx->err = "sync_makespan: partition count must be >= 1, got " + std::to_string(k[i]);
      return nullptr;
    }
  cudaSetDevice(ctx->device);
  dpro_batch* b = acquire_batch(ctx, n, DPRO_DEVICE);
  if (build_tsync_batch(ctx, b, *cluster, std::vector<int64_t>(bytes, bytes + n),
                        std::vector<int32_t>(k, k + n)) != DPRO_OK) {
    delete b;
    return nullptr;
  }
  return b;
}

int dpro_cuda_tsync_grid(dpro_ctx* ctx, const dpro_cluster_desc* cluster,
                         const int64_t* bytes, const int32_t* k, int32_t n,
                         int64_t* out, int32_t* status) {
  if (!ctx || !cluster || n < 0) return DPRO_EINVAL;
  if (!ctx->tsync_host) {  // K2: graphs generated on the device
    std::vector<int64_t> bb;
    std::vector<int32_t> kk;
    std::vector<int> idx;
    int st = DPRO_OK;
    for (int32_t i = 0; i < n; ++i) {
      if (k[i] >= 1) {
        bb.push_back(bytes[i]);
        kk.push_back(k[i]);
        idx.push_back(i);
      } else {
        if (status) status[i] = DPRO_EINVAL;
        out[i] = 0;
        ctx->err = "sync_makespan: partition count must be >= 1, got " + std::to_string(k[i]);
      }
    }
    if (idx.empty()) return DPRO_OK;
    cudaSetDevice(ctx->device);
    // a recycled batch (ctx->spare): repeated small grids (the greedy
    // search's opt_part_num) reuse its device buffers instead of allocating
    dpro_batch* b = acquire_batch(ctx, static_cast<int32_t>(idx.size()), DPRO_DEVICE);
    st = build_tsync_batch(ctx, b, *cluster, bb, kk);
    if (st == DPRO_OK) st = dpro_cuda_batch_replay(ctx, b, 0);
    std::vector<int64_t> ms(idx.size()), er(idx.size());
    std::vector<int32_t> ss(idx.size());
    if (st == DPRO_OK)
      st = dpro_cuda_batch_results(ctx, b, ms.data(), ss.data(), er.data(), nullptr, nullptr);
    for (size_t j = 0; j < idx.size(); ++j) {
      out[idx[j]] = st == DPRO_OK ? ms[j] : 0;
      if (status) status[idx[j]] = st == DPRO_OK ? ss[j] : st;
    }
    dpro_cuda_batch_destroy(ctx, b);  // synchronizes; keeps it as the spare
    return st;
  }
  std::vector<dpro_graph*> graphs(n, nullptr);
  std::vector<std::string> errs(n);
  std::vector<int> idx;
  const int nt = std::max(1, std::min<int>(n, (int)std::thread::hardware_concurrency()));
  auto work = [&](int tid) {
    for (int i = tid; i < n; i += nt)
      if (k[i] >= 1) graphs[i] = dpro_internal_tsync_graph(cluster, bytes[i], k[i], &errs[i]);
      else errs[i] = "sync_makespan: partition count must be >= 1, got " + std::to_string(k[i]);
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  std::vector<dpro_csr> csrs;
  for (int i = 0; i < n; ++i) {
    if (!graphs[i]) {
      if (status) status[i] = DPRO_EINVAL;
      out[i] = 0;
      ctx->err = errs[i];
      continue;
    }
    dpro_csr c;
    dpro_graph_csr(graphs[i], &c);
    csrs.push_back(c);
    idx.push_back(i);
  }
  int st = DPRO_OK;
  if (!csrs.empty()) {
    std::vector<int64_t> ms(csrs.size()), er(csrs.size());
    std::vector<int32_t> ss(csrs.size());
    st = dpro_cuda_replay_batch(ctx, csrs.data(), (int32_t)csrs.size(), DPRO_HOST,
                                ms.data(), nullptr, nullptr, ss.data(), er.data());
    for (size_t j = 0; j < idx.size(); ++j) {
      out[idx[j]] = ms[j];
      if (status) status[idx[j]] = st == DPRO_OK ? ss[j] : st;
    }
  }
  for (auto* g : graphs)
    if (g) dpro_graph_free(g);
  return st;
}

}  // extern "C"
