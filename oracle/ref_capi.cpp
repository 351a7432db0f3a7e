// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (proj/src/*.cpp,
// compiled in place by oracle/Makefile). Python tests, golden-vector
// generators and bench.py's CPU arm call the reference through this file
// (ctypes). Every entry point forwards to a public reference function:
//
//   replay / execution_graph / critical_path  proj/include/dpro/replay.hpp:48-82
//   sync_makespan / partial_replay             proj/include/dpro/replay.hpp:84-91
//   gen_synthetic + ingest_bundle              proj/include/dpro/synth.hpp:82,
//                                              proj/include/dpro/ingest.hpp:108
//   apply_tensor_partition / _fusion / op fusion proj/include/dpro/optimize.hpp:91-111
//
// Graphs cross the boundary as opaque handles (heap GlobalDFG) and are
// exported as index-ordered CSR (index = reference op index = byte-lex id
// order, proj/src/graph.cpp:278-297) with dense device ids assigned in
// DeviceId order (proj/include/dpro/graph.hpp:57-72).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "dpro/errors.hpp"
#include "dpro/ingest.hpp"
#include "dpro/memory.hpp"
#include "dpro/optimize.hpp"
#include "dpro/replay.hpp"
#include "dpro/synth.hpp"

using namespace dpro;

namespace {

struct Handle {
  GlobalDFG g;
  std::vector<DeviceId> devices;             // dense id -> DeviceId
  std::map<DeviceId, int> dev_index;         // DeviceId -> dense id
  std::vector<std::string> device_strs;
  void index_devices() {
    std::map<DeviceId, int> seen;
    for (const auto& op : g.ops()) seen.emplace(op.device, 0);
    int k = 0;
    for (auto& [d, v] : seen) {
      v = k++;
      devices.push_back(d);
      device_strs.push_back(d.str());
    }
    dev_index = std::move(seen);
  }
};

thread_local std::string g_err;
thread_local std::vector<std::string> g_cycle;

int fail(const std::exception& e) {
  g_err = e.what();
  return 3;
}

Handle* wrap(GlobalDFG g) {
  auto* h = new Handle{std::move(g), {}, {}, {}};
  h->index_devices();
  return h;
}

// Runs fn, mapping the reference's exception types onto status codes:
// 1 MissingProfileError, 2 CycleError (cycle list kept), 4 LookupError,
// 5 TransformError, 3 any other dpro::Error / std::exception.
template <typename F>
int guarded(F&& fn) {
  g_err.clear();
  g_cycle.clear();
  try {
    fn();
    return 0;
  } catch (const MissingProfileError& e) {
    g_err = e.what();
    return 1;
  } catch (const CycleError& e) {
    g_err = e.what();
    g_cycle = e.cycle;
    return 2;
  } catch (const LookupError& e) {
    g_err = e.what();
    return 4;
  } catch (const TransformError& e) {
    g_err = e.what();
    return 5;
  } catch (const MissingMetaError& e) {
    g_err = e.what();
    return 6;
  } catch (const BudgetError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int64_t ref_last_cycle_len() { return static_cast<int64_t>(g_cycle.size()); }
const char* ref_last_cycle_id(int64_t i) { return g_cycle.at(i).c_str(); }

// Ops are given as parallel arrays; device = (dev_kind 0 compute / 1 link,
// dev_node, dev_peer). kinds follow dpro::OpKind's enumerator order.
void* ref_graph_from_arrays(int64_t n, const char** ids, const int32_t* kinds,
                            const int32_t* dev_kind, const char** dev_node,
                            const char** dev_peer, const int64_t* dur,
                            int64_t m, const char** ea, const char** eb,
                            int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    GraphBuilder b;
    for (int64_t i = 0; i < n; ++i) {
      Op op;
      op.id = ids[i];
      op.kind = static_cast<OpKind>(kinds[i]);
      op.node = dev_node[i];
      op.device = dev_kind[i] == 0 ? DeviceId::compute(dev_node[i])
                                   : DeviceId::link(dev_node[i], dev_peer[i]);
      op.dur = dur[i];
      b.add_op(std::move(op));
    }
    for (int64_t e = 0; e < m; ++e) b.add_edge(ea[e], eb[e]);
    out = wrap(b.build());
  });
  return out;
}

// Nominal graph of the reference synthetic generator: gen_synthetic, then
// ingest of its own traces (what `dpro gen` + `dpro replay` would see).
void* ref_synth_graph(const char* spec_json, int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    SynthSpec spec = SynthSpec::from_json(nlohmann::json::parse(spec_json));
    SynthResult r = gen_synthetic(spec);
    out = wrap(ingest_bundle(r.traces, r.deps, r.cluster));
  });
  return out;
}

void* ref_apply_partition(void* h, const char* tensor, int32_t k,
                          int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    out = wrap(apply_tensor_partition(static_cast<Handle*>(h)->g, tensor, k));
  });
  return out;
}

void* ref_apply_tensor_fusion(void* h, const char* t1, const char* t2,
                              int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    out = wrap(apply_tensor_fusion(static_cast<Handle*>(h)->g, t1, t2));
  });
  return out;
}

void* ref_apply_op_fusion(void* h, const char* a, const char* b,
                          int64_t dur_override, int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    CostModel cost;
    out = wrap(apply_op_fusion(static_cast<Handle*>(h)->g, a, b, cost,
                               dur_override));
  });
  return out;
}

// The CLI's timeline.json for replay(g) (checker for report.py): a
// restatement of proj/tools/dpro_main.cpp:90-116 (timeline_json) and 64-70
// (write_json: dump(2) + newline) on the reference's own GlobalDFG and
// replay -- the CLI itself needs CLI11, absent here. Returns the byte size;
// the text is copied into buf when cap is large enough.
thread_local std::string g_timeline;
int64_t ref_timeline_json(void* hv, char* buf, int64_t cap, int32_t* status) {
  auto* h = static_cast<Handle*>(hv);
  *status = guarded([&] {
    const ReplayResult r = replay(h->g);
    nlohmann::json events = nlohmann::json::array();
    for (const auto& [id, entry] : r.schedule) {
      const Op& op = h->g.op(id);
      if (is_virtual(op.kind)) continue;
      nlohmann::json e;
      e["name"] = id;
      e["ph"] = "X";
      e["pid"] = entry.device.str();
      e["tid"] = op.node;
      e["ts"] = entry.start;
      e["dur"] = entry.end - entry.start;
      e["cat"] = to_string(op.kind);
      e["args"]["kind"] = to_string(op.kind);
      e["args"]["iteration"] = 0;
      if (is_communication(op.kind)) {
        e["args"]["tensor"] = op.tensor;
        e["args"]["bytes"] = op.bytes;
        e["args"]["transaction"] = op.transaction;
      }
      events.push_back(std::move(e));
    }
    nlohmann::json j;
    j["traceEvents"] = std::move(events);
    j["displayTimeUnit"] = "ms";
    g_timeline = j.dump(2) + "\n";
  });
  if (*status) return 0;
  if (buf && cap >= static_cast<int64_t>(g_timeline.size()))
    std::memcpy(buf, g_timeline.data(), g_timeline.size());
  return static_cast<int64_t>(g_timeline.size());
}

// search(g, options) (optimize.cpp:1327-1650) -> {"before_us", "after_us",
// "strategies": [Strategy::to_json()...]} as JSON text (checker for
// search.reference_search).
thread_local std::string g_search;
int64_t ref_search(void* hv, const char* opts_json, char* buf, int64_t cap, int32_t* status) {
  auto* h = static_cast<Handle*>(hv);
  *status = guarded([&] {
    const auto j = nlohmann::json::parse(opts_json);
    SearchOptions o;
    o.time_budget_s = j.value("time_budget_s", 30.0);
    o.kmax = j.value("kmax", 16);
    o.use_coarsen = j.value("use_coarsen", true);
    o.use_symmetry = j.value("use_symmetry", true);
    o.use_partial_replay = j.value("use_partial_replay", true);
    o.use_theorems = j.value("use_theorems", true);
    o.convergence_pct = j.value("convergence_pct", 0.5);
    o.convergence_rounds = j.value("convergence_rounds", 5);
    if (j.contains("passes"))
      for (const auto& p : j["passes"]) o.passes.push_back(p.get<std::string>());
    const SearchOutcome out = search(h->g, o);
    nlohmann::json r;
    r["before_us"] = out.strategies.before_us;
    r["after_us"] = out.strategies.after_us;
    r["strategies"] = nlohmann::json::array();
    for (const auto& st : out.strategies.strategies) r["strategies"].push_back(st.to_json());
    g_search = r.dump();
  });
  if (*status) return 0;
  if (buf && cap >= static_cast<int64_t>(g_search.size()))
    std::memcpy(buf, g_search.data(), g_search.size());
  return static_cast<int64_t>(g_search.size());
}

// The synthetic generator's trace bundle + dependency spec (gen_synthetic,
// synth.cpp) as JSON, for checking ingest.ingest_bundle against the
// reference's ingest_bundle (which ref_synth_graph runs on the same bundle).
thread_local std::string g_bundle;
int64_t ref_synth_bundle(const char* spec_json, char* buf, int64_t cap, int32_t* status) {
  *status = guarded([&] {
    const SynthSpec spec = SynthSpec::from_json(nlohmann::json::parse(spec_json));
    const SynthResult r = gen_synthetic(spec);
    nlohmann::json j;
    j["events"] = nlohmann::json::array();
    for (const auto& e : r.traces.events) {
      j["events"].push_back({{"name", e.name}, {"node", e.node}, {"start", e.start},
                             {"dur", e.dur}, {"kind", static_cast<int>(e.kind)},
                             {"iteration", e.iteration}, {"tensor", e.tensor},
                             {"bytes", e.bytes}, {"transaction", e.transaction}});
    }
    j["deps"] = r.deps.to_json();
    g_bundle = j.dump();
  });
  if (*status) return 0;
  if (buf && cap >= static_cast<int64_t>(g_bundle.size()))
    std::memcpy(buf, g_bundle.data(), g_bundle.size());
  return static_cast<int64_t>(g_bundle.size());
}

// ingest_bundle (ingest.cpp:452-493) on a bundle given as JSON: events as
// ref_synth_bundle writes them, a DependencySpec, a ClusterSpec.
void* ref_ingest(const char* bundle_json, const char* cluster_json, int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    const auto j = nlohmann::json::parse(bundle_json);
    TraceBundle tb;
    for (const auto& e : j["events"]) {
      TraceEvent ev;
      ev.name = e["name"].get<std::string>();
      ev.node = e["node"].get<std::string>();
      ev.start = e.value("start", Us{0});
      ev.dur = e.value("dur", Us{0});
      ev.kind = static_cast<OpKind>(e.value("kind", 0));
      ev.iteration = e.value("iteration", 0);
      ev.tensor = e.value("tensor", std::string());
      ev.bytes = e.value("bytes", std::int64_t{0});
      ev.transaction = e.value("transaction", std::string());
      tb.events.push_back(std::move(ev));
    }
    const DependencySpec deps = DependencySpec::from_json(j["deps"]);
    const ClusterSpec cluster = ClusterSpec::from_json(nlohmann::json::parse(cluster_json));
    out = wrap(ingest_bundle(tb, deps, cluster));
  });
  return out;
}

// apply_strategy for the parameterless memory rewrites (kind 3 recompute,
// 4 grad-accum), optimize.cpp:506-531.
void* ref_apply_memory_strategy(void* h, int32_t kind, const char* meta_json,
                                int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    const ModelMeta meta = ModelMeta::from_json(nlohmann::json::parse(meta_json));
    Strategy st;
    st.kind = static_cast<StrategyKind>(kind);
    out = wrap(apply_strategy(static_cast<Handle*>(h)->g, st, CostModel{}, meta));
  });
  return out;
}

// memory_pass (optimize.cpp:972-1021): the returned graph, the applied
// strategy kind (-1 none) and k, or status 7 with best_peak (BudgetError).
void* ref_memory_pass(void* h, int64_t budget, const char* meta_json, int32_t* status,
                      int32_t* applied_kind, int32_t* applied_k, int64_t* best_peak) {
  Handle* out = nullptr;
  *applied_kind = -1;
  *status = guarded([&] {
    const ModelMeta meta = ModelMeta::from_json(nlohmann::json::parse(meta_json));
    std::vector<Strategy> applied;
    try {
      out = wrap(memory_pass(static_cast<Handle*>(h)->g, budget, meta, &applied));
    } catch (const BudgetError& e) {
      *best_peak = e.best_peak_bytes;
      throw;
    }
    if (!applied.empty()) {
      *applied_kind = static_cast<int32_t>(applied[0].kind);
      *applied_k = applied[0].k;
    }
  });
  return out;
}

// Copy with per-op duration overrides (candidate perturbation).
void* ref_with_durations(void* h, const int64_t* dur, int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    const GlobalDFG& g = static_cast<Handle*>(h)->g;
    GraphBuilder b(g);
    for (std::size_t i = 0; i < g.size(); ++i) b.op(g.op_at(i).id).dur = dur[i];
    out = wrap(b.build());
  });
  return out;
}

void ref_graph_free(void* h) { delete static_cast<Handle*>(h); }
int64_t ref_graph_num_ops(void* h) {
  return static_cast<int64_t>(static_cast<Handle*>(h)->g.size());
}
int64_t ref_graph_num_edges(void* h) {
  return static_cast<int64_t>(static_cast<Handle*>(h)->g.edge_count());
}
int32_t ref_graph_num_devices(void* h) {
  return static_cast<int32_t>(static_cast<Handle*>(h)->devices.size());
}
const char* ref_graph_op_id(void* h, int64_t i) {
  return static_cast<Handle*>(h)->g.op_at(i).id.c_str();
}
const char* ref_graph_device_str(void* h, int32_t d) {
  return static_cast<Handle*>(h)->device_strs.at(d).c_str();
}
int32_t ref_graph_device_kind(void* h, int32_t d) {
  return static_cast<Handle*>(h)->devices.at(d).kind == DeviceKind::kCompute
             ? 0
             : 1;
}
uint64_t ref_graph_hash(void* h) {
  return static_cast<Handle*>(h)->g.content_hash();
}

// Index-ordered CSR export. succ lists are ascending (graph.cpp:290-295).
void ref_graph_export(void* hv, int64_t* dur, int32_t* kind, int32_t* dev,
                      uint32_t* succ_off, uint32_t* succ, int64_t* bytes) {
  auto* h = static_cast<Handle*>(hv);
  const GlobalDFG& g = h->g;
  uint32_t e = 0;
  for (std::size_t i = 0; i < g.size(); ++i) {
    const Op& op = g.op_at(i);
    if (dur) dur[i] = op.dur;
    if (kind) kind[i] = static_cast<int32_t>(op.kind);
    if (dev) dev[i] = h->dev_index.at(op.device);
    if (bytes) bytes[i] = op.bytes;
    if (succ_off) succ_off[i] = e;
    for (auto s : g.succ_indices(i)) {
      if (succ) succ[e] = s;
      ++e;
    }
  }
  if (succ_off) succ_off[g.size()] = e;
}

// dpro::replay. start/end per op index; tl_pos = position of the op in its
// device timeline (-1: virtual); busy/util per dense device.
int32_t ref_replay(void* hv, int64_t* start, int64_t* end, int64_t* T,
                   int32_t* tl_pos, double* util) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&] {
    const ReplayResult r = replay(h->g);
    *T = r.iteration_time_us;
    const GlobalDFG& g = h->g;
    for (std::size_t i = 0; i < g.size(); ++i) {
      const auto& s = r.schedule.at(g.op_at(i).id);
      if (start) start[i] = s.start;
      if (end) end[i] = s.end;
      if (tl_pos) tl_pos[i] = -1;
    }
    if (tl_pos) {
      for (const auto& [d, tl] : r.device_timelines)
        for (std::size_t p = 0; p < tl.size(); ++p)
          tl_pos[g.index_of(tl[p])] = static_cast<int32_t>(p);
    }
    if (util) {
      for (std::size_t d = 0; d < h->devices.size(); ++d) util[d] = -1.0;
      for (const auto& [d, u] : r.utilization) util[h->dev_index.at(d)] = u;
    }
  });
}

// critical_path(execution_graph(g, replay(g)), replay(g)).
// path: op indices; run_comm/run_dur: one entry per run.
int32_t ref_critical_path(void* hv, uint32_t* path, int64_t* path_len,
                          int64_t* total, int32_t* conforming,
                          int32_t* run_comm, int64_t* run_dur,
                          int64_t* run_len, int64_t* n_runs) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&] {
    const ReplayResult r = replay(h->g);
    const GlobalDFG exec = execution_graph(h->g, r);
    const CriticalPath cp = critical_path(exec, r);
    *path_len = static_cast<int64_t>(cp.ops.size());
    for (std::size_t i = 0; i < cp.ops.size(); ++i)
      path[i] = static_cast<uint32_t>(h->g.index_of(cp.ops[i].op));
    *total = cp.total_us;
    *conforming = cp.conforming ? 1 : 0;
    *n_runs = static_cast<int64_t>(cp.runs.size());
    for (std::size_t i = 0; i < cp.runs.size(); ++i) {
      run_comm[i] = cp.runs[i].communication ? 1 : 0;
      run_dur[i] = cp.runs[i].dur_us;
      run_len[i] = static_cast<int64_t>(cp.runs[i].ops.size());
    }
  });
}

int64_t ref_execution_graph_edges(void* hv) {
  auto* h = static_cast<Handle*>(hv);
  const ReplayResult r = replay(h->g);
  return static_cast<int64_t>(execution_graph(h->g, r).edge_count());
}

// estimate_peak_memory(g, replay(g), meta) (memory.cpp:122-167): peaks per
// compute node in node-name order (the result map's order); names via
// ref_peak_node(i).
thread_local std::vector<std::string> g_peak_nodes;
int32_t ref_peak_memory(void* hv, const char* meta_json, int64_t* peaks, int32_t* n_nodes) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&] {
    const ModelMeta meta = ModelMeta::from_json(nlohmann::json::parse(meta_json));
    const auto peak = estimate_peak_memory(h->g, replay(h->g), meta);
    g_peak_nodes.clear();
    int32_t k = 0;
    for (const auto& [node, v] : peak) {
      if (peaks) peaks[k] = v;
      g_peak_nodes.push_back(node);
      ++k;
    }
    *n_nodes = k;
  });
}
const char* ref_peak_node(int32_t i) { return g_peak_nodes.at(i).c_str(); }

int32_t ref_sync_makespan(const char* cluster_json, int64_t bytes, int32_t k,
                          int64_t* out) {
  return guarded([&] {
    const ClusterSpec c = ClusterSpec::from_json(nlohmann::json::parse(cluster_json));
    *out = sync_makespan(c, bytes, k);
  });
}

int32_t ref_partial_replay(void* hv, const char* tensor, int32_t k,
                           int64_t* out) {
  return guarded([&] {
    *out = partial_replay(static_cast<Handle*>(hv)->g, tensor, k);
  });
}

// Comm-only graph of sync_makespan (replay.cpp:228-246), built with the
// reference's own expand_tensor, as a handle (for exporting to the engine).
void* ref_tsync_graph(const char* cluster_json, int64_t bytes, int32_t k,
                      int32_t* status) {
  Handle* out = nullptr;
  *status = guarded([&] {
    const ClusterSpec c = ClusterSpec::from_json(nlohmann::json::parse(cluster_json));
    GraphBuilder builder;
    builder.set_cluster(c);
    const std::int64_t base = bytes / k, rem = bytes % k;
    for (int i = 0; i < k; ++i) {
      const std::string unit = (k == 1) ? "tsync" : "tsync#p" + std::to_string(i);
      const CommTopology topo = expand_tensor(unit, base + (i < rem ? 1 : 0), c);
      for (const auto& op : topo.ops) builder.add_op(op);
      for (const auto& [a, b] : topo.edges) builder.add_edge(a, b);
    }
    out = wrap(builder.build());
  });
  return out;
}

// CPU baseline: dpro::replay over `n` graphs (graph i % n_graphs) with a pool
// of `threads` std::threads; only replay() is inside the timed region.
int32_t ref_replay_bench(void** hs, int64_t n_graphs, int64_t n_replays,
                         int32_t threads, int64_t* makespans, double* seconds) {
  return guarded([&] {
    std::atomic<int64_t> next{0};
    auto worker = [&] {
      for (;;) {
        const int64_t i = next.fetch_add(1);
        if (i >= n_replays) break;
        const auto* h = static_cast<Handle*>(hs[i % n_graphs]);
        const ReplayResult r = replay(h->g);
        if (makespans) makespans[i] = r.iteration_time_us;
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"
