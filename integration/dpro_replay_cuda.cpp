// Reference-side adapter: the five functions of proj/include/dpro/replay.hpp
// implemented over the B200 C ABI (include/dpro_cuda.h). A maintainer adds
// this file to the reference build in place of proj/src/replay.cpp; every
// caller (search, synth, CLI, tests) then replays on the GPU unchanged.
//
// Marshalling follows the C ABI contract: op index order = GlobalDFG index
// order (graph.cpp:278-297), dense device ids in DeviceId order, int64
// durations. Errors come back as status codes and are rethrown as the
// reference's exception types with the reference's messages
// (replay.cpp:39-44, 108-117, 229-232; partial_replay 248-258).
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "dpro/errors.hpp"
#include "dpro/replay.hpp"
#include "dpro_cuda.h"

namespace dpro {

namespace {

struct Engine {
  dpro_ctx* ctx = nullptr;
  std::mutex mu;  // a context is used by one host thread at a time
  Engine() { ctx = dpro_cuda_create(0); }
  ~Engine() {
    if (ctx) dpro_cuda_destroy(ctx);
  }
};

Engine& engine() {
  static Engine e;
  if (!e.ctx) throw Error("dpro_cuda: no usable CUDA device");
  return e;
}

struct Csr {
  std::vector<int64_t> dur;
  std::vector<uint16_t> dev;
  std::vector<uint8_t> flags;
  std::vector<uint32_t> off, succ, indeg;
  std::vector<DeviceId> devices;
  dpro_csr view{};

  explicit Csr(const GlobalDFG& g) {
    const size_t n = g.size();
    std::map<DeviceId, uint16_t> index;
    for (const auto& op : g.ops()) index.emplace(op.device, 0);
    uint16_t k = 0;
    for (auto& [d, v] : index) {
      v = k++;
      devices.push_back(d);
    }
    dur.resize(n);
    dev.resize(n);
    flags.resize(n);
    off.assign(n + 1, 0);
    indeg.resize(n);
    for (size_t i = 0; i < n; ++i) {
      const Op& op = g.op_at(i);
      dur[i] = op.dur;
      dev[i] = index.at(op.device);
      flags[i] = static_cast<uint8_t>((is_virtual(op.kind) ? DPRO_FLAG_VIRTUAL : 0u) |
                                      (is_communication(op.kind) ? DPRO_FLAG_COMM : 0u));
      indeg[i] = static_cast<uint32_t>(g.pred_indices(i).size());
      off[i + 1] = off[i] + static_cast<uint32_t>(g.succ_indices(i).size());
      for (auto s : g.succ_indices(i)) succ.push_back(s);
    }
    view = dpro_csr{static_cast<uint32_t>(n), static_cast<uint32_t>(succ.size()),
                    static_cast<uint32_t>(devices.size()), 64, dur.data(), dev.data(),
                    flags.data(), off.data(), succ.data(), indeg.data()};
  }
};

void check(int rc, dpro_ctx* ctx, const char* what) {
  if (rc != DPRO_OK)
    throw Error(std::string("dpro_cuda ") + what + ": " + dpro_cuda_last_error(ctx));
}

}  // namespace

ReplayResult replay(const GlobalDFG& g) {
  Engine& e = engine();
  std::lock_guard<std::mutex> lock(e.mu);
  Csr m(g);
  const size_t n = g.size();
  dpro_batch* b = dpro_cuda_batch_create(e.ctx, &m.view, 1, DPRO_HOST);
  if (!b) check(DPRO_EINVAL, e.ctx, "batch_create");
  struct Guard {
    dpro_ctx* c;
    dpro_batch* b;
    ~Guard() { dpro_cuda_batch_destroy(c, b); }
  } guard{e.ctx, b};
  check(dpro_cuda_batch_replay(e.ctx, b, 1), e.ctx, "replay");
  int64_t T = 0, err = 0;
  int32_t status = 0;
  std::vector<int64_t> start(n + 1), end(n + 1);
  check(dpro_cuda_batch_results(e.ctx, b, &T, &status, &err, start.data(), end.data()),
        e.ctx, "results");
  if (status == DPRO_MISSING_PROFILE)
    throw MissingProfileError("op " + g.op_at(static_cast<size_t>(err)).id + " has no duration");
  if (status == DPRO_CYCLE) {
    std::vector<uint8_t> sched(n + 1);
    check(dpro_cuda_batch_scheduled(e.ctx, b, 0, sched.data()), e.ctx, "scheduled");
    std::vector<std::string> stuck;
    for (size_t i = 0; i < n; ++i)
      if (!sched[i]) stuck.push_back(g.op_at(i).id);
    throw CycleError("replay requires an acyclic graph; " + std::to_string(stuck.size()) +
                         " ops never became ready",
                     stuck);
  }
  check(status, e.ctx, "status");
  ReplayResult r;
  r.iteration_time_us = T;
  for (size_t i = 0; i < n; ++i) {
    const Op& op = g.op_at(i);
    r.schedule[op.id] = {start[i], end[i], op.device};
  }
  const size_t D = m.devices.size();
  std::vector<uint32_t> order(n + 1), dev_off(D + 1);
  std::vector<int64_t> busy(D + 1);
  check(dpro_cuda_batch_timelines(e.ctx, b, 0, order.data(), dev_off.data(), busy.data()),
        e.ctx, "timelines");
  for (size_t d = 0; d < D; ++d) {
    if (dev_off[d + 1] == dev_off[d]) continue;  // created on dispatch only
    auto& tl = r.device_timelines[m.devices[d]];
    for (uint32_t p = dev_off[d]; p < dev_off[d + 1]; ++p) tl.push_back(g.op_at(order[p]).id);
    r.utilization[m.devices[d]] =
        T > 0 ? static_cast<double>(busy[d]) / static_cast<double>(T) : 0.0;
  }
  return r;
}

GlobalDFG execution_graph(const GlobalDFG& g, const ReplayResult& result) {
  GraphBuilder b(g);
  for (const auto& kv : result.device_timelines) {
    const auto& tl = kv.second;
    for (size_t i = 0; i + 1 < tl.size(); ++i) b.add_edge(tl[i], tl[i + 1]);
  }
  return b.build();
}

CriticalPath critical_path(const GlobalDFG& exec_graph, const ReplayResult& result) {
  CriticalPath path;
  path.total_us = result.iteration_time_us;
  const size_t n = exec_graph.size();
  if (n == 0) {
    path.conforming = true;
    return path;
  }
  Engine& e = engine();
  std::lock_guard<std::mutex> lock(e.mu);
  Csr m(exec_graph);
  std::vector<int64_t> start(n), end(n);
  for (size_t i = 0; i < n; ++i) {
    const auto& s = result.schedule.at(exec_graph.op_at(i).id);
    start[i] = s.start;
    end[i] = s.end;
  }
  std::vector<uint32_t> idx(n);
  int64_t len = 0;
  check(dpro_cuda_critical_path(e.ctx, &m.view, start.data(), end.data(),
                                result.iteration_time_us, idx.data(), &len),
        e.ctx, "critical_path");
  for (int64_t k = 0; k < len; ++k) {
    const Op& op = exec_graph.op_at(idx[k]);
    path.ops.push_back({op.id, op.dur, is_communication(op.kind)});
  }
  for (const auto& entry : path.ops) {
    const Op& op = exec_graph.op(entry.op);
    if (is_virtual(op.kind)) continue;
    const bool comm = is_communication(op.kind);
    if (path.runs.empty() || path.runs.back().communication != comm)
      path.runs.push_back({comm, {}, 0});
    path.runs.back().ops.push_back(entry.op);
    path.runs.back().dur_us += entry.dur;
  }
  path.conforming = path.runs.size() <= 2 &&
                    (path.runs.size() < 2 ||
                     (!path.runs[0].communication && path.runs[1].communication));
  return path;
}

Us sync_makespan(const ClusterSpec& cluster, std::int64_t bytes, int k) {
  if (k < 1)
    throw Error("sync_makespan: partition count must be >= 1, got " + std::to_string(k));
  std::map<std::string, int32_t> index;
  std::vector<const char*> ids;
  std::vector<int32_t> role, src, dst, ring;
  std::vector<double> bw, lat;
  for (const auto& nd : cluster.nodes) {
    index[nd.id] = static_cast<int32_t>(ids.size());
    ids.push_back(nd.id.c_str());
    role.push_back(nd.role == "worker" ? 0 : (nd.role == "ps" ? 1 : 2));
  }
  for (const auto& l : cluster.links) {
    src.push_back(index.at(l.src));
    dst.push_back(index.at(l.dst));
    bw.push_back(l.bandwidth_bytes_per_us);
    lat.push_back(l.latency_us);
  }
  for (const auto& w : cluster.ring_order) ring.push_back(index.at(w));
  const dpro_cluster_desc desc{
      cluster.scheme == CommScheme::kPs ? 1 : 0, static_cast<int32_t>(ids.size()),
      ids.data(), role.data(), static_cast<int32_t>(src.size()), src.data(), dst.data(),
      bw.data(), lat.data(), static_cast<int32_t>(ring.size()), ring.data(),
      cluster.chunks_per_tensor};
  Engine& e = engine();
  std::lock_guard<std::mutex> lock(e.mu);
  int64_t out = 0;
  int32_t status = 0;
  const int32_t kk = k;
  const int rc = dpro_cuda_tsync_grid(e.ctx, &desc, &bytes, &kk, 1, &out, &status);
  if (rc != DPRO_OK || status != DPRO_OK)
    throw TopologyError(std::string("sync_makespan: ") + dpro_cuda_last_error(e.ctx));
  return out;
}

Us partial_replay(const GlobalDFG& g, const std::string& tensor, int k) {
  std::int64_t bytes = 0;
  if (g.has_base(tensor))
    bytes = g.base_bytes(tensor);
  else if (g.has_tensor_unit(tensor))
    bytes = g.tensor_unit(tensor).bytes;
  else
    throw LookupError("unknown tensor: " + tensor);
  return sync_makespan(g.cluster(), bytes, k);
}

}  // namespace dpro
