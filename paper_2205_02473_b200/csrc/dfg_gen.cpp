// Host-side candidate-graph construction straight into index-ordered CSR.
//
// Builds the graphs the reference builds through string-keyed GraphBuilder
// copies (proj/src/graph.cpp:199-297), without the per-rewrite map copies:
//   * the layered data-parallel model of proj/src/synth.cpp:200-245 as
//     ingested by proj/src/ingest.cpp:187-266,386-454 (local DFGs + splice);
//   * ring all-reduce / PS expansion, proj/src/ingest.cpp:37-67,268-384;
//   * tensor partition re-expansion, proj/src/optimize.cpp:459-492;
//   * the comm-only t_sync graph of proj/src/replay.cpp:228-246.
// Op ids are generated with the reference naming so the byte-lexicographic
// sort reproduces the reference op index (the replay tie-break order).
#include <algorithm>
#include <cstdio>
#include <array>
#include <atomic>
#include <charconv>
#include <cmath>
#include <unordered_map>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "dpro_cuda.h"

namespace {

thread_local std::string g_gen_err;

// Reference OpKind enumerator order (graph.hpp:30-38).
enum Kind : int32_t { kFw = 0, kBw, kUpdate, kSend, kRecv, kVin, kVout };

// round half to even, proj/include/dpro/time_util.hpp:28-35.
int64_t round_half_even(double value) {
  const double f = std::floor(value);
  const double frac = value - f;
  const int64_t lo = static_cast<int64_t>(f);
  if (frac > 0.5) return lo + 1;
  if (frac < 0.5) return lo;
  return (lo % 2 == 0) ? lo : lo + 1;
}

// FNV-1a, proj/src/graph.cpp:57-64 (PS placement hash).
uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}

struct Cluster {
  int scheme = 0;
  std::vector<std::string> nodes;
  std::vector<int> role;
  std::map<std::pair<int, int>, std::pair<double, double>> link;  // first wins
  std::vector<int> ring;  // node indices
  std::vector<int> sorted_workers;
  std::vector<int> sorted_ps;
  int chunks = 0;

  explicit Cluster(const dpro_cluster_desc& d) {
    scheme = d.scheme;
    for (int i = 0; i < d.n_nodes; ++i) {
      nodes.emplace_back(d.node_ids[i]);
      role.push_back(d.node_role[i]);
    }
    for (int l = 0; l < d.n_links; ++l)
      link.emplace(std::make_pair(d.link_src[l], d.link_dst[l]),
                   std::make_pair(d.link_bw[l], d.link_lat[l]));
    for (int i = 0; i < d.n_nodes; ++i) {
      if (role[i] == 0) sorted_workers.push_back(i);
      if (role[i] == 1) sorted_ps.push_back(i);
    }
    auto by_name = [&](int a, int b) { return nodes[a] < nodes[b]; };
    std::sort(sorted_workers.begin(), sorted_workers.end(), by_name);
    std::sort(sorted_ps.begin(), sorted_ps.end(), by_name);
    if (d.n_ring > 0)
      ring.assign(d.ring_order, d.ring_order + d.n_ring);
    else
      ring = sorted_workers;  // ingest.cpp:63-67,271-272
    chunks = d.chunks_per_tensor;
  }

  // hop_dur, ingest.cpp:37-48
  int64_t hop(int64_t bytes, int src, int dst) const {
    double bw = 1.0, lat = 0.0;
    auto it = link.find({src, dst});
    if (it != link.end()) {
      bw = it->second.first;
      lat = it->second.second;
    }
    return round_half_even(static_cast<double>(bytes) / bw + lat);
  }
};

struct Gen {
  struct Op {
    std::string id;
    int32_t kind;
    uint32_t devkey;
    int64_t dur;
    int32_t unit = -1;   // comm ops: tensor unit (index into units)
    int64_t bytes = 0;   // comm ops: bytes moved
  };
  std::vector<Op> ops;
  std::vector<std::pair<uint32_t, uint32_t>> edges;  // creation indices
  std::vector<std::string> units;  // tensor units named by comm ops
  // devices keyed by (kind, node index, peer index); resolved to DeviceId
  // order (kind, node name, peer name -- graph.hpp:57-72) in finalize()
  std::unordered_map<uint64_t, uint32_t> devkeys;
  std::vector<std::array<int, 3>> devs;  // key id -> (kind, node, peer)
  const std::vector<std::string>* names = nullptr;

  uint32_t device(int dkind, int node, int peer) {
    const uint64_t key = (uint64_t(dkind) << 62) | (uint64_t(uint32_t(node)) << 31) |
                         uint64_t(uint32_t(peer + 1));  // == dev_key()
    auto it = devkeys.emplace(key, static_cast<uint32_t>(devs.size()));
    if (it.second) devs.push_back({dkind, node, peer});
    return it.first->second;
  }
  uint32_t add(std::string id, int32_t kind, uint32_t dev, int64_t dur) {
    ops.push_back({std::move(id), kind, dev, dur});
    return static_cast<uint32_t>(ops.size() - 1);
  }
  void edge(uint32_t a, uint32_t b) { edges.emplace_back(a, b); }
};

// Appends decimal v to s (no temporaries).
inline void append_num(std::string& s, int64_t v) {
  char buf[24];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  s.append(buf, r.ptr);
}

// One tensor unit's comm topology spliced onto per-node IN/OUT ops
// (ingest.cpp:268-384 expansion + assemble_global_dfg 404-441 splice).
// in_op/out_op: node index -> creation index (UINT32_MAX when absent).
void expand_unit(Gen& g, const Cluster& c, const std::string& unit,
                 int64_t bytes, const std::vector<uint32_t>* in_op,
                 const std::vector<uint32_t>* out_op) {
  auto link_dev = [&](int s, int d) { return g.device(1, s, d); };
  const int32_t uidx = static_cast<int32_t>(g.units.size());
  g.units.push_back(unit);
  auto tag = [&](uint32_t op, int64_t b) {  // Op::tensor / Op::bytes of a comm op
    g.ops[op].unit = uidx;
    g.ops[op].bytes = b;
  };
  auto need = [&](const std::vector<uint32_t>* v, int node) -> uint32_t {
    if (!v) return UINT32_MAX;
    uint32_t x = (*v)[node];
    if (x == UINT32_MAX)
      throw std::runtime_error("tensor " + unit + " attaches to node " +
                               c.nodes[node] + " which has no IN/OUT op");
    return x;
  };
  if (c.scheme == 0) {
    const int n = static_cast<int>(c.ring.size());
    if (n < 2)
      throw std::runtime_error("degenerate ring: allreduce needs at least 2 workers");
    const int chunks = c.chunks > 0 ? c.chunks : n;
    const int steps = 2 * (n - 1);
    const int64_t base = bytes / chunks, rem = bytes % chunks;
    for (int ch = 0; ch < chunks; ++ch) {
      const int64_t cb = base + (ch < rem ? 1 : 0);
      uint32_t prev_recv = UINT32_MAX;
      for (int s = 0; s < steps; ++s) {
        const int src = c.ring[(ch + s) % n];
        const int dst = c.ring[(ch + s + 1) % n];
        std::string txn;
        txn.reserve(unit.size() + 32);
        txn += unit;
        txn += "#c";
        append_num(txn, ch);
        txn += "#s";
        append_num(txn, s);
        txn += '#';
        txn += c.nodes[src];
        txn += '#';
        txn += c.nodes[dst];
        const uint32_t dv = link_dev(src, dst);
        std::string sid = "SEND.", rid = "RECV.";
        sid += txn;
        rid += txn;
        const uint32_t snd = g.add(std::move(sid), kSend, dv, 0);
        const uint32_t rcv = g.add(std::move(rid), kRecv, dv, c.hop(cb, src, dst));
        tag(snd, cb);
        tag(rcv, cb);
        g.edge(snd, rcv);
        if (s == 0) {
          const uint32_t in = need(in_op, src);
          if (in != UINT32_MAX) g.edge(in, snd);
        } else {
          g.edge(prev_recv, snd);
        }
        if (s >= n - 2) {
          const uint32_t out = need(out_op, dst);
          if (out != UINT32_MAX) g.edge(rcv, out);
        }
        prev_recv = rcv;
      }
    }
  } else {
    if (c.sorted_ps.empty())
      throw std::runtime_error("parameter-server scheme requires at least one ps node");
    if (c.sorted_workers.empty())
      throw std::runtime_error("parameter-server scheme requires at least one worker");
    const int server = c.sorted_ps[fnv1a(unit) % c.sorted_ps.size()];
    std::vector<uint32_t> push_recvs, pull_sends;
    for (int w : c.sorted_workers) {
      const std::string push = unit + "#push#" + c.nodes[w] + "#" + c.nodes[server];
      const uint32_t dpush = link_dev(w, server);
      const uint32_t ps = g.add("SEND." + push, kSend, dpush, 0);
      const uint32_t pr = g.add("RECV." + push, kRecv, dpush, c.hop(bytes, w, server));
      tag(ps, bytes);
      tag(pr, bytes);
      g.edge(ps, pr);
      const uint32_t in = need(in_op, w);
      if (in != UINT32_MAX) g.edge(in, ps);
      push_recvs.push_back(pr);
      const std::string pull = unit + "#pull#" + c.nodes[server] + "#" + c.nodes[w];
      const uint32_t dpull = link_dev(server, w);
      const uint32_t ls = g.add("SEND." + pull, kSend, dpull, 0);
      const uint32_t lr = g.add("RECV." + pull, kRecv, dpull, c.hop(bytes, server, w));
      tag(ls, bytes);
      tag(lr, bytes);
      g.edge(ls, lr);
      const uint32_t out = need(out_op, w);
      if (out != UINT32_MAX) g.edge(lr, out);
      pull_sends.push_back(ls);
    }
    for (uint32_t pull : pull_sends)
      for (uint32_t push : push_recvs) g.edge(push, pull);
  }
}

}  // namespace

struct dpro_graph {
  // ids of a full build; delta builds (dpro_graph_from_base_batch) leave it
  // empty and resolve ids through the shared base graph instead
  std::vector<std::string> ids;
  std::shared_ptr<const void> base_keep;
  const std::vector<std::string>* base_ids = nullptr;
  std::vector<uint32_t> id_ref;  // high bit: new_ids index, else base index
  std::vector<std::string> new_ids;
  std::vector<int32_t> kind;
  std::vector<int64_t> dur;
  std::vector<uint16_t> dev;
  std::vector<uint8_t> flags;
  std::vector<uint32_t> succ_off, succ, indeg;
  std::vector<std::string> device_strs;
  std::vector<std::string> mem_nodes;  // dpro_graph_memory_inputs: compute nodes, name order
  // comm-op metadata (Op::tensor / bytes; the transaction is the id after
  // "SEND." / "RECV."): unit index into units (-1 otherwise), bytes
  std::vector<int32_t> cunit;
  std::vector<int64_t> cbytes;
  std::vector<std::string> units;
};

namespace {

// Sort ops by id (std::map order in GraphBuilder::build), dense device ids in
// DeviceId order, ascending deduplicated succ lists (std::set of edges).
dpro_graph* finalize(Gen& g, std::vector<uint32_t>* rank_out = nullptr,
                     std::vector<std::array<int, 3>>* devs_out = nullptr) {
  const uint32_t n = static_cast<uint32_t>(g.ops.size());
  // byte-lexicographic order of ids (std::map<std::string> order): compare
  // 16-byte big-endian prefixes first, full strings only on prefix ties
  struct Key {
    uint64_t a, b;
    uint32_t i;
  };
  std::vector<Key> keys(n);
  for (uint32_t i = 0; i < n; ++i) {
    unsigned char buf[16] = {0};
    const std::string& id = g.ops[i].id;
    std::memcpy(buf, id.data(), std::min<size_t>(16, id.size()));
    uint64_t a = 0, b = 0;
    for (int k = 0; k < 8; ++k) a = (a << 8) | buf[k];
    for (int k = 8; k < 16; ++k) b = (b << 8) | buf[k];
    keys[i] = {a, b, i};
  }
  std::sort(keys.begin(), keys.end(), [&](const Key& x, const Key& y) {
    if (x.a != y.a) return x.a < y.a;
    if (x.b != y.b) return x.b < y.b;
    return g.ops[x.i].id < g.ops[y.i].id;  // shared 16-byte prefix (or short ids)
  });
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; ++i) order[i] = keys[i].i;
  for (uint32_t i = 1; i < n; ++i)
    if (g.ops[order[i]].id == g.ops[order[i - 1]].id)
      throw std::runtime_error("duplicate op id '" + g.ops[order[i]].id + "'");
  std::vector<uint32_t> rank(n);
  for (uint32_t i = 0; i < n; ++i) rank[order[i]] = i;

  // dense device ids in DeviceId order: (kind, node name, peer name)
  const std::vector<std::string>& nm = *g.names;
  std::vector<uint32_t> dorder(g.devs.size());
  std::iota(dorder.begin(), dorder.end(), 0u);
  auto dname = [&](int idx) -> const std::string& {
    static const std::string empty;
    return idx < 0 ? empty : nm[idx];
  };
  std::sort(dorder.begin(), dorder.end(), [&](uint32_t x, uint32_t y) {
    const auto& a = g.devs[x];
    const auto& b = g.devs[y];
    if (a[0] != b[0]) return a[0] < b[0];
    const int cn = dname(a[1]).compare(dname(b[1]));
    if (cn != 0) return cn < 0;
    return dname(a[2]) < dname(b[2]);
  });
  std::vector<uint32_t> dev_rank(g.devs.size());
  auto* out = new dpro_graph;
  for (uint32_t k = 0; k < dorder.size(); ++k) {
    dev_rank[dorder[k]] = k;
    const auto& d = g.devs[dorder[k]];
    out->device_strs.push_back(d[0] == 0 ? dname(d[1]) : dname(d[1]) + ">" + dname(d[2]));
  }
  if (g.devs.size() > 65535) {
    delete out;
    throw std::runtime_error("more than 65535 devices");
  }
  out->ids.resize(n);
  out->kind.resize(n);
  out->dur.resize(n);
  out->dev.resize(n);
  out->flags.resize(n);
  out->cunit.resize(n);
  out->cbytes.resize(n);
  out->units = std::move(g.units);
  for (uint32_t i = 0; i < n; ++i) {
    auto& op = g.ops[order[i]];
    out->cunit[i] = op.unit;
    out->cbytes[i] = op.bytes;
    out->ids[i] = std::move(op.id);
    out->kind[i] = op.kind;
    out->dur[i] = op.dur;
    out->dev[i] = static_cast<uint16_t>(dev_rank[op.devkey]);
    out->flags[i] = static_cast<uint8_t>(
        (op.kind == kVin || op.kind == kVout ? DPRO_FLAG_VIRTUAL : 0u) |
        (op.kind == kSend || op.kind == kRecv ? DPRO_FLAG_COMM : 0u));
  }
  for (auto& e : g.edges) e = {rank[e.first], rank[e.second]};
  std::sort(g.edges.begin(), g.edges.end());
  g.edges.erase(std::unique(g.edges.begin(), g.edges.end()), g.edges.end());
  out->succ_off.assign(n + 1, 0);
  out->indeg.assign(n, 0);
  out->succ.resize(g.edges.size());
  for (size_t e = 0; e < g.edges.size(); ++e) {
    out->succ_off[g.edges[e].first + 1]++;
    out->indeg[g.edges[e].second]++;
    out->succ[e] = g.edges[e].second;
  }
  for (uint32_t i = 0; i < n; ++i) out->succ_off[i + 1] += out->succ_off[i];
  if (rank_out) *rank_out = std::move(rank);
  if (devs_out)
    for (uint32_t k = 0; k < dorder.size(); ++k) devs_out->push_back(g.devs[dorder[k]]);
  return out;
}

// Synchronization units of a layered candidate: groups of layer tensors
// fused in the given member order (apply_tensor_fusion, optimize.cpp:366-455
// -- fusing t1 then t2 names the unit "t1+t2", its IN is fed by every
// member's producer and its OUT feeds every member's consumer), each
// partitioned k ways (apply_tensor_partition, optimize.cpp:459-492).
struct Groups {
  std::vector<std::vector<int>> members;
  std::vector<int> k;
  // op fusion on every worker (optimize.cpp:245-317, applied left to right
  // with the default cost model): fw_join[i] fuses FW.l<i> with FW.l<i+1>,
  // bw_join[i] fuses BW.l<i+1> with BW.l<i>; empty = none
  std::vector<uint8_t> fw_join, bw_join;
  // the joins apply to this worker only (node index); -1 = every worker
  int join_worker = -1;
};

// Creation indices of the structural ops of a layered build (for delta
// construction against it).
struct Record {
  std::vector<std::vector<uint32_t>> fw, bw, up;  // [node][layer]
  std::vector<std::vector<uint32_t>> in, out;     // [group][node]
  std::vector<std::pair<uint32_t, uint32_t>> comm;  // [group] creation range
};

// Memory rewrites applied while generating (optimize.cpp:819-959 on the
// synth/ingest graph): 1 = recompute (sqrt(L) checkpoint segments per worker,
// RFW.l<i> re-runs feeding the backward ops), 2 = grad-accum (two
// micro-batches FW/BW.l<i>@mb0/@mb1 with round_us(dur * scale)).
struct MemVariant {
  int kind = 0;
  double scale = 0.5;
};

dpro_graph* build_layered(const dpro_layered_model& m, const Cluster& c, const Groups& G,
                          Record* rec = nullptr, std::vector<uint32_t>* rank_out = nullptr,
                          std::vector<std::array<int, 3>>* devs_out = nullptr,
                          MemVariant var = {}) {
  Gen g;
  g.names = &c.nodes;
  const int L = m.layers;
  if (L < 1) throw std::runtime_error("synthetic model needs at least one layer");
  const int N = static_cast<int>(c.nodes.size());
  const int NG = static_cast<int>(G.members.size());
  std::vector<int> group_of(L, -1);
  std::vector<std::string> gname(NG);
  for (int q = 0; q < NG; ++q) {
    if (G.members[q].empty()) throw std::runtime_error("empty tensor group");
    for (size_t x = 0; x < G.members[q].size(); ++x) {
      const int i = G.members[q][x];
      if (i < 0 || i >= L || group_of[i] >= 0)
        throw std::runtime_error("tensor groups must partition the layers");
      group_of[i] = q;
      gname[q] += (x ? "+g" : "g") + std::to_string(i);
    }
  }
  for (int i = 0; i < L; ++i)
    if (group_of[i] < 0) throw std::runtime_error("tensor groups must cover every layer");
  std::vector<int> workers;
  for (int i = 0; i < N; ++i)
    if (c.role[i] == 0) workers.push_back(i);
  if (rec) {
    rec->fw.assign(N, std::vector<uint32_t>(L, UINT32_MAX));
    rec->bw = rec->fw;
    rec->up = rec->fw;
    rec->comm.assign(NG, {0, 0});
  }
  // per group: IN/OUT creation index per node
  std::vector<std::vector<uint32_t>> in_op(NG, std::vector<uint32_t>(N, UINT32_MAX));
  std::vector<std::vector<uint32_t>> out_op(NG, std::vector<uint32_t>(N, UINT32_MAX));
  if (var.kind == 1 && L < 2)
    throw std::runtime_error("re-computation does not apply to this graph");
  for (int w : workers) {
    const std::string& node = c.nodes[w];
    const uint32_t dv = g.device(0, w, -1);
    std::vector<uint32_t> fw(L), bw(L), up(L);
    if (var.kind == 2) {  // grad-accum: micro-batch copies of every FW/BW op
      std::vector<uint32_t> fw0(L), fw1(L), bw0(L), bw1(L);
      auto mb = [&](int64_t d) { return round_half_even(static_cast<double>(d) * var.scale); };
      for (int i = 0; i < L; ++i) {
        const std::string li = std::to_string(i);
        fw0[i] = g.add(node + "->FW.l" + li + "@mb0", kFw, dv, mb(m.fw_dur[i]));
        fw1[i] = g.add(node + "->FW.l" + li + "@mb1", kFw, dv, mb(m.fw_dur[i]));
        bw0[i] = g.add(node + "->BW.l" + li + "@mb0", kBw, dv, mb(m.bw_dur[i]));
        bw1[i] = g.add(node + "->BW.l" + li + "@mb1", kBw, dv, mb(m.bw_dur[i]));
        up[i] = g.add(node + "->UPDATE.l" + li, kUpdate, dv, m.update_dur);
      }
      for (int q = 0; q < NG; ++q) {
        in_op[q][w] = g.add(node + "->IN." + gname[q], kVin, dv, 0);
        out_op[q][w] = g.add(node + "->OUT." + gname[q], kVout, dv, 0);
      }
      for (int i = 0; i < L; ++i) {  // optimize.cpp:913-928 edge rules
        if (i > 0) {
          g.edge(fw0[i - 1], fw0[i]);
          g.edge(fw1[i - 1], fw1[i]);
        }
        if (i + 1 < L) {
          g.edge(bw0[i + 1], bw0[i]);
          g.edge(bw1[i + 1], bw1[i]);
        }
        g.edge(fw0[i], bw0[i]);
        g.edge(fw1[i], bw1[i]);
        g.edge(bw1[i], in_op[group_of[i]][w]);   // duplicated -> plain: from @mb1
        g.edge(out_op[group_of[i]][w], up[i]);
      }
      g.edge(bw0[0], fw1[0]);  // second micro-batch after the first's backward
      continue;
    }
    for (int i = 0; i < L; ++i) {
      const std::string li = std::to_string(i);
      fw[i] = g.add(node + "->FW.l" + li, kFw, dv, m.fw_dur[i]);
      bw[i] = g.add(node + "->BW.l" + li, kBw, dv, m.bw_dur[i]);
      up[i] = g.add(node + "->UPDATE.l" + li, kUpdate, dv, m.update_dur);
      if (rec) {
        rec->fw[w][i] = fw[i];
        rec->bw[w][i] = bw[i];
        rec->up[w][i] = up[i];
      }
    }
    for (int q = 0; q < NG; ++q) {
      in_op[q][w] = g.add(node + "->IN." + gname[q], kVin, dv, 0);
      out_op[q][w] = g.add(node + "->OUT." + gname[q], kVout, dv, 0);
    }
    // synth.cpp:200-212 deps, resolved by build_local_dfg (ingest.cpp:243-265)
    std::vector<uint8_t> fw_to_bw(L, 1);
    if (var.kind == 1) {  // recompute, optimize.cpp:831-870
      const int cseg = static_cast<int>(std::ceil(std::sqrt(static_cast<double>(L))));
      const int seg_base = L / cseg, seg_rem = L % cseg;
      int lo = 0, prev_cp = -1;
      for (int sgi = 0; sgi < cseg; ++sgi) {
        const int len = seg_base + (sgi < seg_rem ? 1 : 0);
        const int cp = lo + len - 1;
        uint32_t prev_rfw = UINT32_MAX;
        for (int i = lo; i < cp; ++i) {
          const uint32_t rfw = g.add(node + "->RFW.l" + std::to_string(i), kFw, dv, m.fw_dur[i]);
          fw_to_bw[i] = 0;  // FW.l_i -> BW.l_i becomes RFW.l_i -> BW.l_i
          g.edge(rfw, bw[i]);
          if (prev_rfw == UINT32_MAX) {
            if (prev_cp >= 0) g.edge(fw[prev_cp], rfw);
            g.edge(bw[cp], rfw);  // gate: the checkpoint's backward
          } else {
            g.edge(prev_rfw, rfw);
          }
          prev_rfw = rfw;
        }
        prev_cp = cp;
        lo += len;
      }
    }
    for (int i = 0; i < L; ++i) {
      if (i > 0) g.edge(fw[i - 1], fw[i]);
      if (i + 1 < L) g.edge(bw[i + 1], bw[i]);
      if (fw_to_bw[i]) g.edge(fw[i], bw[i]);
      g.edge(bw[i], in_op[group_of[i]][w]);   // producer feeds IN (ingest.cpp:242)
      g.edge(out_op[group_of[i]][w], up[i]);  // OUT(g_i) -> UPDATE.l_i
    }
  }
  for (int q = 0; q < NG; ++q) {
    int64_t bytes = 0;
    for (int i : G.members[q]) bytes += m.tensor_bytes[i];
    const int k = G.k[q];
    if (k < 1)
      throw std::runtime_error("partition count must be >= 1, got " + std::to_string(k));
    if (k > bytes)
      throw std::runtime_error("cannot split " + std::to_string(bytes) + " bytes of " +
                               gname[q] + " into " + std::to_string(k) + " partitions");
    const int64_t base = bytes / k, rem = bytes % k;
    const uint32_t c0 = static_cast<uint32_t>(g.ops.size());
    for (int p = 0; p < k; ++p) {
      const std::string unit = k == 1 ? gname[q] : gname[q] + "#p" + std::to_string(p);
      expand_unit(g, c, unit, base + (p < rem ? 1 : 0), &in_op[q], &out_op[q]);
    }
    if (rec) rec->comm[q] = {c0, static_cast<uint32_t>(g.ops.size())};
  }
  if (rec) {
    rec->in = in_op;
    rec->out = out_op;
  }
  return finalize(g, rank_out, devs_out);
}

dpro_graph* build_layered(const dpro_layered_model& m, const Cluster& c,
                          const int32_t* part_k) {
  Groups G;
  for (int i = 0; i < m.layers; ++i) {
    G.members.push_back({i});
    G.k.push_back(part_k ? part_k[i] : 1);
  }
  return build_layered(m, c, G);
}

Groups make_groups(int32_t n_groups, const int32_t* group_off, const int32_t* members,
                   const int32_t* group_k) {
  Groups G;
  for (int q = 0; q < n_groups; ++q) {
    G.members.emplace_back(members + group_off[q], members + group_off[q + 1]);
    G.k.push_back(group_k ? group_k[q] : 1);
  }
  return G;
}

dpro_graph* build_tsync(const Cluster& c, int64_t bytes, int k) {
  if (k < 1)
    throw std::invalid_argument("sync_makespan: partition count must be >= 1, got " +
                                std::to_string(k));
  Gen g;
  g.names = &c.nodes;
  const int64_t base = bytes / k, rem = bytes % k;
  for (int i = 0; i < k; ++i) {
    const std::string unit = k == 1 ? "tsync" : "tsync#p" + std::to_string(i);
    expand_unit(g, c, unit, base + (i < rem ? 1 : 0), nullptr, nullptr);
  }
  return finalize(g);
}

template <typename F>
dpro_graph* guarded(F&& f, int32_t* status) {
  try {
    dpro_graph* g = f();
    if (status) *status = DPRO_OK;
    return g;
  } catch (const std::bad_alloc&) {
    g_gen_err = "out of host memory";
    if (status) *status = DPRO_ENOMEM;
  } catch (const std::exception& e) {
    g_gen_err = e.what();
    if (status) *status = DPRO_EINVAL;
  }
  return nullptr;
}


// ---------------------------------------------------------------------------
// Delta construction: a fusion/partition candidate is the
// base layered graph minus the comm ops (and, for fused units, the IN/OUT
// ops) of its changed units plus the newly expanded ones. Only the new ops
// are named and sorted; they are merged into the base's index order by
// binary search, and every kept base op keeps its relative order, so the
// result is the same index-ordered CSR a full rebuild produces (tested
// against it and against the reference's rewrite chain).
// ---------------------------------------------------------------------------
struct BaseData {
  Cluster c;
  std::vector<int64_t> fw_dur, bw_dur, tensor_bytes;
  int64_t update_dur = 0;
  int L = 0, N = 0;
  std::vector<int> workers;
  std::unique_ptr<dpro_graph> g;
  std::vector<std::array<int, 3>> devs;  // dense id -> (kind, node, peer)
  std::vector<std::vector<uint32_t>> fw, bw, up;  // [node][layer] final index
  std::vector<std::vector<uint32_t>> in, out;     // [layer][node]
  std::vector<std::vector<uint32_t>> comm;        // [layer] comm op final indices
  std::unordered_map<uint64_t, uint16_t> devindex;  // Gen device key -> dense id
  explicit BaseData(const dpro_cluster_desc& d) : c(d) {}
};

inline uint64_t dev_key(int dkind, int node, int peer) {
  return (uint64_t(dkind) << 62) | (uint64_t(uint32_t(node)) << 31) | uint64_t(uint32_t(peer + 1));
}

constexpr uint32_t kBaseRef = 0x80000000u;

bool dev_less(const std::vector<std::string>& nm, const std::array<int, 3>& a,
              const std::array<int, 3>& b) {
  static const std::string empty;
  auto nmf = [&](int i) -> const std::string& { return i < 0 ? empty : nm[i]; };
  if (a[0] != b[0]) return a[0] < b[0];
  const int cn = nmf(a[1]).compare(nmf(b[1]));
  if (cn != 0) return cn < 0;
  return nmf(a[2]) < nmf(b[2]);
}

std::shared_ptr<BaseData> build_base(const dpro_layered_model& m, const dpro_cluster_desc& cd) {
  auto B = std::make_shared<BaseData>(cd);
  B->L = m.layers;
  B->N = static_cast<int>(B->c.nodes.size());
  B->fw_dur.assign(m.fw_dur, m.fw_dur + m.layers);
  B->bw_dur.assign(m.bw_dur, m.bw_dur + m.layers);
  B->tensor_bytes.assign(m.tensor_bytes, m.tensor_bytes + m.layers);
  B->update_dur = m.update_dur;
  for (int i = 0; i < B->N; ++i)
    if (B->c.role[i] == 0) B->workers.push_back(i);
  Groups G;
  for (int i = 0; i < m.layers; ++i) {
    G.members.push_back({i});
    G.k.push_back(1);
  }
  Record rec;
  std::vector<uint32_t> rank;
  B->g.reset(build_layered(m, B->c, G, &rec, &rank, &B->devs));
  auto R = [&](uint32_t ci) { return ci == UINT32_MAX ? UINT32_MAX : rank[ci]; };
  auto map2 = [&](const std::vector<std::vector<uint32_t>>& v) {
    std::vector<std::vector<uint32_t>> o(v.size());
    for (size_t a = 0; a < v.size(); ++a)
      for (uint32_t x : v[a]) o[a].push_back(R(x));
    return o;
  };
  B->fw = map2(rec.fw);
  B->bw = map2(rec.bw);
  B->up = map2(rec.up);
  B->in = map2(rec.in);
  B->out = map2(rec.out);
  B->comm.resize(m.layers);
  for (int i = 0; i < m.layers; ++i)
    for (uint32_t ci = rec.comm[i].first; ci < rec.comm[i].second; ++ci)
      B->comm[i].push_back(rank[ci]);
  for (size_t d = 0; d < B->devs.size(); ++d)
    B->devindex[dev_key(B->devs[d][0], B->devs[d][1], B->devs[d][2])] = static_cast<uint16_t>(d);
  return B;
}

// The changed part of a candidate: new ops (Gen, creation order; edges hold
// kBaseRef | base index or creation index), the removed base ops, the new
// ops in id order (snew) and their insertion points among the base ids.
struct DeltaParts {
  Gen g;
  std::vector<uint8_t> removed;  // [nb]
  std::vector<uint32_t> snew, pos;
};

void prepare_delta(const BaseData& B, const Groups& G, DeltaParts& P) {
  const dpro_graph& bg = *B.g;
  const int L = B.L, NG = static_cast<int>(G.members.size());
  const uint32_t nb = static_cast<uint32_t>(bg.kind.size());
  // validate: groups partition the layers
  std::vector<int> group_of(L, -1);
  std::vector<std::string> gname(NG);
  for (int q = 0; q < NG; ++q) {
    if (G.members[q].empty()) throw std::runtime_error("empty tensor group");
    for (size_t x = 0; x < G.members[q].size(); ++x) {
      const int i = G.members[q][x];
      if (i < 0 || i >= L || group_of[i] >= 0)
        throw std::runtime_error("tensor groups must partition the layers");
      group_of[i] = q;
      gname[q] += (x ? "+g" : "g") + std::to_string(i);
    }
  }
  for (int i = 0; i < L; ++i)
    if (group_of[i] < 0) throw std::runtime_error("tensor groups must cover every layer");

  Gen& g = P.g;
  g.names = &B.c.nodes;
  std::vector<uint8_t>& removed = P.removed;
  removed.assign(nb, 0);
  // op fusion: refs of every worker's FW / BW op of each layer (a fused run
  // is one new op; kBaseRef | base index otherwise)
  const bool opf = !G.fw_join.empty() || !G.bw_join.empty();
  if (opf && ((!G.fw_join.empty() && G.fw_join.size() != size_t(L - 1)) ||
              (!G.bw_join.empty() && G.bw_join.size() != size_t(L - 1))))
    throw std::runtime_error("op fusion joins need layers - 1 entries");
  auto fwj = [&](int i) { return !G.fw_join.empty() && G.fw_join[i]; };
  auto bwj = [&](int i) { return !G.bw_join.empty() && G.bw_join[i]; };
  auto fused_dur = [](int64_t a, int64_t b) {  // CostModel{} fallback 0.8 (optimize.cpp:84-103)
    return round_half_even(0.8 * (static_cast<double>(a) + static_cast<double>(b)));
  };
  std::vector<std::vector<uint32_t>> xr(B.N), yr(B.N);
  for (int w : B.workers) {
    xr[w].resize(L);
    yr[w].resize(L);
    for (int i = 0; i < L; ++i) {
      xr[w][i] = kBaseRef | B.fw[w][i];
      yr[w][i] = kBaseRef | B.bw[w][i];
    }
    if (!opf || (G.join_worker >= 0 && w != G.join_worker)) continue;
    const std::string& node = B.c.nodes[w];
    const uint32_t dv = g.device(0, w, -1);
    for (int a = 0; a < L;) {  // FW runs, fused left to right
      int b = a;
      while (b + 1 < L && fwj(b)) ++b;
      if (b > a) {
        std::string id = node + "->FW.l" + std::to_string(a);
        int64_t d = B.fw_dur[a];
        for (int j = a + 1; j <= b; ++j) {
          id += "+FW.l" + std::to_string(j);
          d = fused_dur(d, B.fw_dur[j]);
        }
        const uint32_t x = g.add(std::move(id), kFw, dv, d);
        for (int j = a; j <= b; ++j) {
          removed[B.fw[w][j]] = 1;
          xr[w][j] = x;
        }
      }
      a = b + 1;
    }
    for (int top = L - 1; top >= 0;) {  // BW runs, fused from the top layer down
      int lo = top;
      while (lo - 1 >= 0 && bwj(lo - 1)) --lo;
      if (lo < top) {
        std::string id = node + "->BW.l" + std::to_string(top);
        int64_t d = B.bw_dur[top];
        for (int j = top - 1; j >= lo; --j) {
          id += "+BW.l" + std::to_string(j);
          d = fused_dur(d, B.bw_dur[j]);
        }
        const uint32_t y = g.add(std::move(id), kBw, dv, d);
        for (int j = lo; j <= top; ++j) {
          removed[B.bw[w][j]] = 1;
          yr[w][j] = y;
        }
      }
      top = lo - 1;
    }
  }
  // IN op of every (group, worker): the base one or the tensor-fused one
  std::vector<std::vector<uint32_t>> in_of(NG, std::vector<uint32_t>(B.N, UINT32_MAX));
  for (int q = 0; q < NG; ++q) {
    const auto& mem = G.members[q];
    const int k = G.k[q];
    const bool fused = mem.size() > 1;
    if (!fused && k == 1) continue;
    int64_t bytes = 0;
    for (int i : mem) bytes += B.tensor_bytes[i];
    if (k < 1)
      throw std::runtime_error("partition count must be >= 1, got " + std::to_string(k));
    if (k > bytes)
      throw std::runtime_error("cannot split " + std::to_string(bytes) + " bytes of " +
                               gname[q] + " into " + std::to_string(k) + " partitions");
    for (int i : mem)
      for (uint32_t b : B.comm[i]) removed[b] = 1;
    std::vector<uint32_t> in_ref(B.N, UINT32_MAX), out_ref(B.N, UINT32_MAX);
    if (fused) {
      for (int i : mem)
        for (int w : B.workers) {
          removed[B.in[i][w]] = 1;
          removed[B.out[i][w]] = 1;
        }
      for (int w : B.workers) {
        const uint32_t dv = g.device(0, w, -1);
        in_ref[w] = g.add(B.c.nodes[w] + "->IN." + gname[q], kVin, dv, 0);
        out_ref[w] = g.add(B.c.nodes[w] + "->OUT." + gname[q], kVout, dv, 0);
        for (int i : mem) {
          g.edge(yr[w][i], in_ref[w]);                // every producer feeds IN
          g.edge(out_ref[w], kBaseRef | B.up[w][i]);  // OUT feeds every consumer
        }
      }
    } else {
      for (int w : B.workers) {
        in_ref[w] = kBaseRef | B.in[mem[0]][w];
        out_ref[w] = kBaseRef | B.out[mem[0]][w];
      }
    }
    const int64_t base = bytes / k, rem = bytes % k;
    for (int p = 0; p < k; ++p) {
      const std::string unit = k == 1 ? gname[q] : gname[q] + "#p" + std::to_string(p);
      expand_unit(g, B.c, unit, base + (p < rem ? 1 : 0), &in_ref, &out_ref);
    }
    if (fused)
      for (int w : B.workers) in_of[q][w] = in_ref[w];
  }
  // op-fusion edges with a new endpoint (edges between kept base ops exist;
  // those into removed ops vanish); duplicates are dropped when emitting
  if (opf) {
    auto is_new = [](uint32_t r) { return !(r & kBaseRef); };
    auto add = [&](uint32_t a, uint32_t b) {
      if (a != b && (is_new(a) || is_new(b))) g.edge(a, b);
    };
    for (int w : B.workers)
      for (int i = 0; i < L; ++i) {
        if (i > 0) add(xr[w][i - 1], xr[w][i]);
        if (i + 1 < L) add(yr[w][i + 1], yr[w][i]);
        add(xr[w][i], yr[w][i]);
        const int q = group_of[i];
        const uint32_t in = in_of[q][w] != UINT32_MAX ? in_of[q][w] : (kBaseRef | B.in[i][w]);
        add(yr[w][i], in);
      }
  }
  const uint32_t nn = static_cast<uint32_t>(g.ops.size());
  // sort the new ops, then place each among the base ids (binary search)
  P.snew.resize(nn);
  std::iota(P.snew.begin(), P.snew.end(), 0u);
  std::sort(P.snew.begin(), P.snew.end(),
            [&](uint32_t a, uint32_t b) { return g.ops[a].id < g.ops[b].id; });
  P.pos.resize(nn);
  for (uint32_t j = 0; j < nn; ++j) {
    const std::string& id = g.ops[P.snew[j]].id;
    const auto it = std::lower_bound(bg.ids.begin(), bg.ids.end(), id);
    if (it != bg.ids.end() && *it == id && !removed[it - bg.ids.begin()])
      throw std::runtime_error("duplicate op id '" + id + "'");
    P.pos[j] = static_cast<uint32_t>(it - bg.ids.begin());
  }
}

dpro_graph* build_delta(const std::shared_ptr<BaseData>& Bp, const Groups& G) {
  const BaseData& B = *Bp;
  const dpro_graph& bg = *B.g;
  const uint32_t nb = static_cast<uint32_t>(bg.kind.size());
  DeltaParts P;
  prepare_delta(B, G, P);
  Gen& g = P.g;
  const std::vector<uint8_t>& removed = P.removed;
  const std::vector<uint32_t>& snew = P.snew;
  const std::vector<uint32_t>& pos = P.pos;
  const uint32_t nn = static_cast<uint32_t>(g.ops.size());
  // final order: merge kept base ops with the new ops at their positions
  std::vector<uint32_t> fb(nb, UINT32_MAX), fnew(nn, UINT32_MAX);
  auto* out = new dpro_graph;
  out->base_keep = Bp;
  out->base_ids = &bg.ids;
  uint32_t f = 0;
  {
    uint32_t j = 0;
    out->id_ref.reserve(nb + nn);
    for (uint32_t b = 0; b <= nb; ++b) {
      for (; j < nn && pos[j] == b; ++j) {
        fnew[snew[j]] = f++;
        out->id_ref.push_back(kBaseRef | snew[j]);
      }
      if (b < nb && !removed[b]) {
        fb[b] = f++;
        out->id_ref.push_back(b);
      }
    }
  }
  const uint32_t n = f;
  for (auto& op : g.ops) out->new_ids.push_back(std::move(op.id));
  // devices: union of the base's and the new ops' devices, DeviceId order
  std::vector<std::array<int, 3>> udev = B.devs;
  for (const auto& d : g.devs)
    if (std::find(udev.begin(), udev.end(), d) == udev.end()) udev.push_back(d);
  std::sort(udev.begin(), udev.end(),
            [&](const auto& a, const auto& b) { return dev_less(B.c.nodes, a, b); });
  if (udev.size() > 65535) {
    delete out;
    throw std::runtime_error("more than 65535 devices");
  }
  auto dense = [&](const std::array<int, 3>& d) {
    return static_cast<uint16_t>(std::lower_bound(udev.begin(), udev.end(), d,
                                                  [&](const auto& a, const auto& b) {
                                                    return dev_less(B.c.nodes, a, b);
                                                  }) - udev.begin());
  };
  std::vector<uint16_t> bdev(B.devs.size()), ndev(g.devs.size());
  for (size_t d = 0; d < B.devs.size(); ++d) bdev[d] = dense(B.devs[d]);
  for (size_t d = 0; d < g.devs.size(); ++d) ndev[d] = dense(g.devs[d]);
  for (const auto& d : udev) {
    static const std::string empty;
    const std::string& a = d[1] < 0 ? empty : B.c.nodes[d[1]];
    out->device_strs.push_back(d[0] == 0 ? a : a + ">" + B.c.nodes[d[2]]);
  }
  out->kind.resize(n);
  out->dur.resize(n);
  out->dev.resize(n);
  out->flags.resize(n);
  out->cunit.resize(n);
  out->cbytes.resize(n);
  out->units = bg.units;  // base units, then the candidate's new ones
  const int32_t uoff = static_cast<int32_t>(bg.units.size());
  out->units.insert(out->units.end(), g.units.begin(), g.units.end());
  for (uint32_t b = 0; b < nb; ++b) {
    const uint32_t x = fb[b];
    if (x == UINT32_MAX) continue;
    out->kind[x] = bg.kind[b];
    out->dur[x] = bg.dur[b];
    out->dev[x] = bdev[bg.dev[b]];
    out->flags[x] = bg.flags[b];
    out->cunit[x] = bg.cunit[b];
    out->cbytes[x] = bg.cbytes[b];
  }
  for (uint32_t j = 0; j < nn; ++j) {
    const uint32_t x = fnew[j];
    const auto& op = g.ops[j];
    out->cunit[x] = op.unit >= 0 ? op.unit + uoff : -1;
    out->cbytes[x] = op.bytes;
    out->kind[x] = op.kind;
    out->dur[x] = op.dur;
    out->dev[x] = ndev[op.devkey];
    out->flags[x] = static_cast<uint8_t>(
        (op.kind == kVin || op.kind == kVout ? DPRO_FLAG_VIRTUAL : 0u) |
        (op.kind == kSend || op.kind == kRecv ? DPRO_FLAG_COMM : 0u));
  }
  // devices whose every op was removed disappear (DeviceId order over the
  // ops actually present, like a full build)
  {
    std::vector<uint16_t> remap(udev.size(), 0xFFFF);
    for (uint32_t i = 0; i < n; ++i) remap[out->dev[i]] = 0;
    std::vector<std::string> strs;
    uint16_t k = 0;
    for (size_t d = 0; d < udev.size(); ++d)
      if (remap[d] == 0) {
        remap[d] = k++;
        strs.push_back(out->device_strs[d]);
      }
    if (k != udev.size()) {
      for (uint32_t i = 0; i < n; ++i) out->dev[i] = remap[out->dev[i]];
      out->device_strs = std::move(strs);
    }
  }
  // edges: kept base edges (remapped) + new edges, ascending per source
  auto fin = [&](uint32_t r) { return (r & kBaseRef) ? fb[r & ~kBaseRef] : fnew[r]; };
  std::vector<std::pair<uint32_t, uint32_t>> extra;
  extra.reserve(g.edges.size());
  for (const auto& e : g.edges) extra.emplace_back(fin(e.first), fin(e.second));
  std::sort(extra.begin(), extra.end());
  extra.erase(std::unique(extra.begin(), extra.end()), extra.end());
  out->succ_off.assign(n + 1, 0);
  std::vector<uint32_t> bcnt(n, 0);  // kept base successors per op
  for (uint32_t b = 0; b < nb; ++b) {
    if (fb[b] == UINT32_MAX) continue;
    uint32_t cnt = 0;
    for (uint32_t e = bg.succ_off[b]; e < bg.succ_off[b + 1]; ++e)
      cnt += fb[bg.succ[e]] != UINT32_MAX;
    bcnt[fb[b]] = cnt;
    out->succ_off[fb[b] + 1] = cnt;
  }
  for (const auto& e : extra) out->succ_off[e.first + 1]++;
  for (uint32_t i = 0; i < n; ++i) out->succ_off[i + 1] += out->succ_off[i];
  out->succ.resize(out->succ_off[n]);
  std::vector<uint32_t> fill(out->succ_off.begin(), out->succ_off.end() - 1);
  for (uint32_t b = 0; b < nb; ++b) {
    const uint32_t x = fb[b];
    if (x == UINT32_MAX) continue;
    for (uint32_t e = bg.succ_off[b]; e < bg.succ_off[b + 1]; ++e) {
      const uint32_t t = fb[bg.succ[e]];
      if (t != UINT32_MAX) out->succ[fill[x]++] = t;  // ascending: fb is monotone
    }
  }
  for (const auto& e : extra) out->succ[fill[e.first]++] = e.second;  // ascending
  out->indeg.assign(n, 0);
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t* a = out->succ.data() + out->succ_off[i];
    uint32_t* z = out->succ.data() + out->succ_off[i + 1];
    if (bcnt[i] && a + bcnt[i] < z) std::inplace_merge(a, a + bcnt[i], z);
    for (uint32_t* p = a; p < z; ++p) out->indeg[*p]++;
  }
  return out;
}

// A candidate as a dpro_delta against the base (include/dpro_cuda.h): the
// same candidate build_delta() merges on the host, left unmerged for the
// engine to merge next to the resident base graph in HBM.
struct DeltaHost {
  std::vector<uint32_t> removed, new_pos, new_succ_off, new_succ, extra_src, extra_dst, cut;
  std::vector<int64_t> new_dur;
  std::vector<uint16_t> new_dev;
  std::vector<uint8_t> new_flags;
  std::vector<std::string> extra_dev_strs;  // devices beyond the base's
  uint32_t n_devices = 0;
};

void emit_delta(const BaseData& B, const Groups& G, DeltaHost& D) {
  const dpro_graph& bg = *B.g;
  DeltaParts P;
  prepare_delta(B, G, P);
  const Gen& g = P.g;
  const uint32_t nb = static_cast<uint32_t>(bg.kind.size());
  const uint32_t nn = static_cast<uint32_t>(g.ops.size());
  D.removed.clear();
  for (uint32_t b = 0; b < nb; ++b)
    if (P.removed[b]) D.removed.push_back(b);
  const auto& R = D.removed;
  auto r_of = [&](uint32_t x) {
    return static_cast<uint32_t>(std::lower_bound(R.begin(), R.end(), x) - R.begin());
  };
  auto q_of = [&](uint32_t b) {
    return static_cast<uint32_t>(std::upper_bound(P.pos.begin(), P.pos.end(), b) - P.pos.begin());
  };
  std::vector<uint32_t> sorted_of(nn), fnew(nn);
  for (uint32_t j = 0; j < nn; ++j) {
    sorted_of[P.snew[j]] = j;
    fnew[P.snew[j]] = P.pos[j] - r_of(P.pos[j]) + j;
  }
  auto fin = [&](uint32_t ref) {  // kBaseRef marks base indices
    if (!(ref & kBaseRef)) return fnew[ref];
    const uint32_t b = ref & ~kBaseRef;
    return b - r_of(b) + q_of(b);
  };
  // devices: the base's dense ids, unseen ones appended
  std::vector<uint16_t> ndev(g.devs.size());
  D.extra_dev_strs.clear();
  uint32_t nd = static_cast<uint32_t>(bg.device_strs.size());
  for (size_t d = 0; d < g.devs.size(); ++d) {
    const auto& k = g.devs[d];
    const auto it = B.devindex.find(dev_key(k[0], k[1], k[2]));
    if (it != B.devindex.end()) {
      ndev[d] = it->second;
    } else {
      if (nd >= 65535) throw std::runtime_error("more than 65535 devices");
      ndev[d] = static_cast<uint16_t>(nd++);
      const std::string& a = B.c.nodes[k[1]];
      D.extra_dev_strs.push_back(k[0] == 0 ? a : a + ">" + B.c.nodes[k[2]]);
    }
  }
  D.n_devices = nd;
  D.new_pos = P.pos;
  D.new_dur.resize(nn);
  D.new_dev.resize(nn);
  D.new_flags.resize(nn);
  for (uint32_t j = 0; j < nn; ++j) {
    const auto& op = g.ops[P.snew[j]];
    D.new_dur[j] = op.dur;
    D.new_dev[j] = ndev[op.devkey];
    D.new_flags[j] = static_cast<uint8_t>(
        (op.kind == kVin || op.kind == kVout ? DPRO_FLAG_VIRTUAL : 0u) |
        (op.kind == kSend || op.kind == kRecv ? DPRO_FLAG_COMM : 0u));
  }
  // edges out of new ops -> new_succ (by sorted position); out of base ops -> extra
  std::vector<std::pair<uint32_t, uint32_t>> ne, xe;
  ne.reserve(g.edges.size());
  for (const auto& e : g.edges) {
    const uint32_t dst = fin(e.second);
    if (e.first & kBaseRef)
      xe.emplace_back(e.first & ~kBaseRef, dst);
    else
      ne.emplace_back(sorted_of[e.first], dst);
  }
  std::sort(ne.begin(), ne.end());
  ne.erase(std::unique(ne.begin(), ne.end()), ne.end());
  std::sort(xe.begin(), xe.end());
  xe.erase(std::unique(xe.begin(), xe.end()), xe.end());
  D.new_succ_off.assign(nn + 1, 0);
  D.new_succ.resize(ne.size());
  for (size_t k = 0; k < ne.size(); ++k) {
    D.new_succ_off[ne[k].first + 1]++;
    D.new_succ[k] = ne[k].second;
  }
  for (uint32_t j = 0; j < nn; ++j) D.new_succ_off[j + 1] += D.new_succ_off[j];
  D.extra_src.resize(xe.size());
  D.extra_dst.resize(xe.size());
  for (size_t k = 0; k < xe.size(); ++k) {
    D.extra_src[k] = xe[k].first;
    D.extra_dst[k] = xe[k].second;
  }
}

}  // namespace

extern "C" {

const char* dpro_graph_last_error(void) { return g_gen_err.c_str(); }

dpro_graph* dpro_graph_layered(const dpro_layered_model* model,
                               const dpro_cluster_desc* cluster,
                               const int32_t* part_k, int32_t* status) {
  return guarded([&] { return build_layered(*model, Cluster(*cluster), part_k); },
                 status);
}

dpro_graph* dpro_graph_layered_variant(const dpro_layered_model* model,
                                       const dpro_cluster_desc* cluster,
                                       const int32_t* part_k, int32_t variant,
                                       double microbatch_scale, int32_t* status) {
  return guarded(
      [&] {
        if (variant < 0 || variant > 2) throw std::invalid_argument("unknown variant");
        Groups G;
        for (int i = 0; i < model->layers; ++i) {
          G.members.push_back({i});
          G.k.push_back(part_k ? part_k[i] : 1);
        }
        return build_layered(*model, Cluster(*cluster), G, nullptr, nullptr, nullptr,
                             MemVariant{variant, microbatch_scale});
      },
      status);
}

int dpro_graph_layered_batch(const dpro_layered_model* model,
                             const dpro_cluster_desc* cluster,
                             const int32_t* part_k, int32_t n, int32_t threads,
                             dpro_graph** out) {
  const Cluster c(*cluster);
  if (threads < 1) threads = 1;
  std::vector<int32_t> st(n, DPRO_OK);
  std::vector<std::string> errs(threads);
  auto work = [&](int tid) {
    for (int i = tid; i < n; i += threads) {
      try {
        out[i] = build_layered(*model, c, part_k ? part_k + (size_t)i * model->layers : nullptr);
      } catch (const std::exception& e) {
        out[i] = nullptr;
        st[i] = DPRO_EINVAL;
        errs[tid] = e.what();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int i = 0; i < n; ++i)
    if (st[i] != DPRO_OK) {
      for (auto& e : errs)
        if (!e.empty()) g_gen_err = e;
      return st[i];
    }
  return DPRO_OK;
}

dpro_graph* dpro_graph_layered_groups(const dpro_layered_model* model,
                                      const dpro_cluster_desc* cluster, int32_t n_groups,
                                      const int32_t* group_off, const int32_t* members,
                                      const int32_t* group_k, int32_t* status) {
  return guarded(
      [&] {
        return build_layered(*model, Cluster(*cluster),
                             make_groups(n_groups, group_off, members, group_k));
      },
      status);
}

int dpro_graph_layered_groups_batch(const dpro_layered_model* model,
                                    const dpro_cluster_desc* cluster, int32_t n,
                                    const int32_t* n_groups, const int64_t* spec_off,
                                    const int32_t* group_off, const int32_t* members,
                                    const int32_t* group_k, int32_t threads,
                                    dpro_graph** out) {
  const Cluster c(*cluster);
  if (threads < 1) threads = 1;
  std::vector<int32_t> st(n, DPRO_OK);
  std::vector<std::string> errs(threads);
  std::atomic<int32_t> next{0};
  auto work = [&](int tid) {
    for (int32_t i; (i = next.fetch_add(1)) < n;) {
      try {
        // candidate i: groups [spec_off[i], spec_off[i] + n_groups[i]) of
        // the flattened group_off / group_k arrays (group_off is global)
        const int64_t g0 = spec_off[i];
        Groups G;
        for (int32_t q = 0; q < n_groups[i]; ++q) {
          G.members.emplace_back(members + group_off[g0 + q], members + group_off[g0 + q + 1]);
          G.k.push_back(group_k ? group_k[g0 + q] : 1);
        }
        out[i] = build_layered(*model, c, G);
      } catch (const std::exception& e) {
        out[i] = nullptr;
        st[i] = DPRO_EINVAL;
        errs[tid] = e.what();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int32_t i = 0; i < n; ++i)
    if (st[i] != DPRO_OK) {
      for (auto& e : errs)
        if (!e.empty()) g_gen_err = e;
      return st[i];
    }
  return DPRO_OK;
}

dpro_graph* dpro_graph_tsync(const dpro_cluster_desc* cluster, int64_t bytes,
                             int32_t k, int32_t* status) {
  return guarded([&] { return build_tsync(Cluster(*cluster), bytes, k); }, status);
}

int dpro_graph_csr(const dpro_graph* g, dpro_csr* out) {
  if (!g || !out) return DPRO_EINVAL;
  out->n_ops = static_cast<uint32_t>(g->kind.size());
  out->n_edges = static_cast<uint32_t>(g->succ.size());
  out->n_devices = static_cast<uint32_t>(g->device_strs.size());
  out->dur_bits = 64;
  out->dur = g->dur.data();
  out->dev = g->dev.data();
  out->flags = g->flags.data();
  out->succ_off = g->succ_off.data();
  out->succ = g->succ.data();
  out->indeg = g->indeg.data();
  return DPRO_OK;
}

const char* dpro_graph_op_id(const dpro_graph* g, uint32_t i) {
  if (!g->ids.empty() || !g->base_ids) return g->ids.at(i).c_str();
  const uint32_t r = g->id_ref.at(i);
  return (r & kBaseRef) ? g->new_ids.at(r & ~kBaseRef).c_str() : g->base_ids->at(r).c_str();
}

struct dpro_base {
  std::shared_ptr<BaseData> b;
};

dpro_base* dpro_base_layered(const dpro_layered_model* model,
                             const dpro_cluster_desc* cluster, int32_t* status) {
  try {
    auto* out = new dpro_base{build_base(*model, *cluster)};
    if (status) *status = DPRO_OK;
    return out;
  } catch (const std::exception& e) {
    g_gen_err = e.what();
    if (status) *status = DPRO_EINVAL;
    return nullptr;
  }
}

void dpro_base_free(dpro_base* b) { delete b; }

int dpro_graph_from_base_batch_ops(const dpro_base* base, int32_t n, const int32_t* n_groups,
                                   const int64_t* spec_off, const int32_t* group_off,
                                   const int32_t* members, const int32_t* group_k,
                                   const uint8_t* fw_join, const uint8_t* bw_join,
                                   int32_t threads, dpro_graph** out) {
  if (!base) return DPRO_EINVAL;
  if (threads < 1) threads = 1;
  const int L = base->b->L;
  std::vector<int32_t> st(n, DPRO_OK);
  std::vector<std::string> errs(threads);
  std::atomic<int32_t> next{0};
  auto work = [&](int tid) {
    for (int32_t i; (i = next.fetch_add(1)) < n;) {
      try {
        const int64_t g0 = spec_off[i];
        Groups G;
        for (int32_t q = 0; q < n_groups[i]; ++q) {
          G.members.emplace_back(members + group_off[g0 + q], members + group_off[g0 + q + 1]);
          G.k.push_back(group_k ? group_k[g0 + q] : 1);
        }
        if (fw_join && L > 1) G.fw_join.assign(fw_join + size_t(i) * (L - 1), fw_join + size_t(i + 1) * (L - 1));
        if (bw_join && L > 1) G.bw_join.assign(bw_join + size_t(i) * (L - 1), bw_join + size_t(i + 1) * (L - 1));
        out[i] = build_delta(base->b, G);
      } catch (const std::exception& e) {
        out[i] = nullptr;
        st[i] = DPRO_EINVAL;
        errs[tid] = e.what();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int32_t i = 0; i < n; ++i)
    if (st[i] != DPRO_OK) {
      for (auto& e : errs)
        if (!e.empty()) g_gen_err = e;
      return st[i];
    }
  return DPRO_OK;
}

int dpro_graph_from_base_batch(const dpro_base* base, int32_t n, const int32_t* n_groups,
                               const int64_t* spec_off, const int32_t* group_off,
                               const int32_t* members, const int32_t* group_k,
                               int32_t threads, dpro_graph** out) {
  return dpro_graph_from_base_batch_ops(base, n, n_groups, spec_off, group_off, members, group_k,
                                        nullptr, nullptr, threads, out);
}
struct dpro_delta_set {
  std::shared_ptr<BaseData> base;
  std::vector<DeltaHost> d;
  std::vector<dpro_delta> views;
  void fill_views();
};

int dpro_base_delta_batch_ex(const dpro_base* base, int32_t n, const int32_t* n_groups,
                             const int64_t* spec_off, const int32_t* group_off,
                             const int32_t* members, const int32_t* group_k,
                             const uint8_t* fw_join, const uint8_t* bw_join,
                             const int32_t* join_worker, int32_t threads,
                             dpro_delta_set** out) {
  const int L = base ? base->b->L : 0;
  if (!base || !out || n < 0) return DPRO_EINVAL;
  *out = nullptr;
  if (threads < 1) threads = 1;
  auto set = std::make_unique<dpro_delta_set>();
  set->base = base->b;
  set->d.resize(n);
  std::vector<int32_t> st(n, DPRO_OK);
  std::vector<std::string> errs(threads);
  std::atomic<int32_t> next{0};
  auto work = [&](int tid) {
    for (int32_t i; (i = next.fetch_add(1)) < n;) {
      try {
        const int64_t g0 = spec_off[i];
        Groups G;
        for (int32_t q = 0; q < n_groups[i]; ++q) {
          G.members.emplace_back(members + group_off[g0 + q], members + group_off[g0 + q + 1]);
          G.k.push_back(group_k ? group_k[g0 + q] : 1);
        }
        if (fw_join && L > 1) G.fw_join.assign(fw_join + size_t(i) * (L - 1), fw_join + size_t(i + 1) * (L - 1));
        if (bw_join && L > 1) G.bw_join.assign(bw_join + size_t(i) * (L - 1), bw_join + size_t(i + 1) * (L - 1));
        if (join_worker && join_worker[i] >= 0) {
          if (join_worker[i] >= static_cast<int32_t>(base->b->workers.size()))
            throw std::runtime_error("join_worker out of range");
          G.join_worker = base->b->workers[join_worker[i]];
        }
        emit_delta(*base->b, G, set->d[i]);
      } catch (const std::exception& e) {
        st[i] = DPRO_EINVAL;
        errs[tid] = e.what();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int32_t i = 0; i < n; ++i)
    if (st[i] != DPRO_OK) {
      for (auto& e : errs)
        if (!e.empty()) g_gen_err = e;
      return st[i];
    }
  set->fill_views();
  *out = set.release();
  return DPRO_OK;
}

int dpro_base_delta_batch_ops(const dpro_base* base, int32_t n, const int32_t* n_groups,
                              const int64_t* spec_off, const int32_t* group_off,
                              const int32_t* members, const int32_t* group_k,
                              const uint8_t* fw_join, const uint8_t* bw_join, int32_t threads,
                              dpro_delta_set** out) {
  return dpro_base_delta_batch_ex(base, n, n_groups, spec_off, group_off, members, group_k,
                                  fw_join, bw_join, nullptr, threads, out);
}

void dpro_delta_set::fill_views() {
  views.resize(d.size());
  for (size_t i = 0; i < d.size(); ++i) {
    const DeltaHost& D = d[i];
    dpro_delta& v = views[i];
    std::memset(&v, 0, sizeof v);
    v.n_devices = D.n_devices;
    v.n_removed = static_cast<uint32_t>(D.removed.size());
    v.removed = D.removed.data();
    v.n_new = static_cast<uint32_t>(D.new_pos.size());
    v.new_pos = D.new_pos.data();
    v.new_dur = D.new_dur.data();
    v.new_dev = D.new_dev.data();
    v.new_flags = D.new_flags.data();
    v.new_succ_off = D.new_succ_off.data();
    v.new_succ = D.new_succ.data();
    v.n_extra = static_cast<uint32_t>(D.extra_src.size());
    v.extra_src = D.extra_src.data();
    v.extra_dst = D.extra_dst.data();
    v.n_cut = static_cast<uint32_t>(D.cut.size());
    v.cut = D.cut.data();
  }
}

// A generated graph (any rewrite: recompute, grad-accum, fusion, partition,
// ...) as a delta against the base: both graphs are index-ordered by op id,
// so one merge walk over the ids splits the ops into kept (same id, kind,
// duration and device), removed and new; kept ops' successor lists are
// diffed into extra and cut edges. Final indices equal the candidate's own
// indices (tested: the engine's merge reproduces the candidate CSR).
namespace {
void delta_from_graph(const BaseData& B, const dpro_graph& g, DeltaHost& D) {
  const dpro_graph& bg = *B.g;
  const uint32_t nb = static_cast<uint32_t>(bg.kind.size());
  const uint32_t nc = static_cast<uint32_t>(g.kind.size());
  std::unordered_map<std::string, uint16_t> bdev;
  for (size_t d = 0; d < bg.device_strs.size(); ++d)
    bdev.emplace(bg.device_strs[d], static_cast<uint16_t>(d));
  std::vector<uint16_t> cdev(g.device_strs.size());
  D.extra_dev_strs.clear();
  uint32_t nd = static_cast<uint32_t>(bg.device_strs.size());
  for (size_t d = 0; d < g.device_strs.size(); ++d) {
    const auto it = bdev.find(g.device_strs[d]);
    if (it != bdev.end()) {
      cdev[d] = it->second;
    } else {
      if (nd >= 65535) throw std::runtime_error("more than 65535 devices");
      cdev[d] = static_cast<uint16_t>(nd++);
      D.extra_dev_strs.push_back(g.device_strs[d]);
    }
  }
  D.n_devices = nd;
  auto bid = [&](uint32_t b) -> const std::string& { return bg.ids[b]; };
  auto cid = [&](uint32_t x) -> const char* { return dpro_graph_op_id(&g, x); };
  std::vector<uint32_t> fb(nb, UINT32_MAX);  // kept base op -> candidate index
  std::vector<uint32_t> newj(nc, UINT32_MAX);
  D.removed.clear();
  D.new_pos.clear();
  D.new_dur.clear();
  D.new_dev.clear();
  D.new_flags.clear();
  uint32_t b = 0, x = 0;
  while (b < nb || x < nc) {
    int c;
    if (b == nb) c = 1;
    else if (x == nc) c = -1;
    else c = bid(b).compare(cid(x));
    if (c == 0) {
      if (bg.kind[b] == g.kind[x] && bg.dur[b] == g.dur[x] &&
          bg.dev[b] == cdev[g.dev[x]] && bg.flags[b] == g.flags[x]) {
        fb[b] = x;
      } else {  // same id, different op: removed + re-added at its place
        D.removed.push_back(b);
        newj[x] = static_cast<uint32_t>(D.new_pos.size());
        D.new_pos.push_back(b);
        D.new_dur.push_back(g.dur[x]);
        D.new_dev.push_back(cdev[g.dev[x]]);
        D.new_flags.push_back(g.flags[x]);
      }
      ++b;
      ++x;
    } else if (c < 0) {
      D.removed.push_back(b++);
    } else {
      newj[x] = static_cast<uint32_t>(D.new_pos.size());
      D.new_pos.push_back(b);  // lower_bound among the base ids
      D.new_dur.push_back(g.dur[x]);
      D.new_dev.push_back(cdev[g.dev[x]]);
      D.new_flags.push_back(g.flags[x]);
      ++x;
    }
  }
  // removed came out ascending except for re-added ids (pushed in order too)
  const uint32_t nn = static_cast<uint32_t>(D.new_pos.size());
  D.new_succ_off.assign(nn + 1, 0);
  D.new_succ.clear();
  for (uint32_t y = 0; y < nc; ++y) {
    if (newj[y] == UINT32_MAX) continue;
    D.new_succ.insert(D.new_succ.end(), g.succ.begin() + g.succ_off[y],
                      g.succ.begin() + g.succ_off[y + 1]);
    D.new_succ_off[newj[y] + 1] = g.succ_off[y + 1] - g.succ_off[y];
  }
  for (uint32_t j = 0; j < nn; ++j) D.new_succ_off[j + 1] += D.new_succ_off[j];
  D.extra_src.clear();
  D.extra_dst.clear();
  D.cut.clear();
  for (uint32_t u = 0; u < nb; ++u) {
    const uint32_t xu = fb[u];
    if (xu == UINT32_MAX) continue;
    uint32_t e = bg.succ_off[u];
    const uint32_t ee = bg.succ_off[u + 1];
    uint32_t k = g.succ_off[xu];
    const uint32_t kk = g.succ_off[xu + 1];
    while (e < ee || k < kk) {
      if (e < ee && fb[bg.succ[e]] == UINT32_MAX) {  // edge to a removed op: gone anyway
        ++e;
        continue;
      }
      const uint32_t mb = e < ee ? fb[bg.succ[e]] : UINT32_MAX;
      const uint32_t mc = k < kk ? g.succ[k] : UINT32_MAX;
      if (mb == mc) {
        ++e;
        ++k;
      } else if (mb < mc) {
        D.cut.push_back(e++);
      } else {
        D.extra_src.push_back(u);
        D.extra_dst.push_back(mc);
        ++k;
      }
    }
  }
}
}  // namespace

int dpro_base_delta_from_graphs(const dpro_base* base, const dpro_graph* const* graphs,
                                int32_t n, int32_t threads, dpro_delta_set** out) {
  if (!base || !out || n < 0 || (n && !graphs)) return DPRO_EINVAL;
  *out = nullptr;
  if (threads < 1) threads = 1;
  auto set = std::make_unique<dpro_delta_set>();
  set->base = base->b;
  set->d.resize(n);
  std::vector<int32_t> st(n, DPRO_OK);
  std::vector<std::string> errs(threads);
  std::atomic<int32_t> next{0};
  auto work = [&](int tid) {
    for (int32_t i; (i = next.fetch_add(1)) < n;) {
      try {
        if (!graphs[i]) throw std::runtime_error("null graph");
        delta_from_graph(*base->b, *graphs[i], set->d[i]);
      } catch (const std::exception& e) {
        st[i] = DPRO_EINVAL;
        errs[tid] = e.what();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int32_t i = 0; i < n; ++i)
    if (st[i] != DPRO_OK) {
      for (auto& e : errs)
        if (!e.empty()) g_gen_err = e;
      return st[i];
    }
  set->fill_views();
  *out = set.release();
  return DPRO_OK;
}

const char* dpro_base_worker(const dpro_base* base, int32_t k) {
  if (!base || k < 0 || k >= static_cast<int32_t>(base->b->workers.size())) return nullptr;
  return base->b->c.nodes[base->b->workers[k]].c_str();
}

int dpro_base_delta_batch(const dpro_base* base, int32_t n, const int32_t* n_groups,
                          const int64_t* spec_off, const int32_t* group_off,
                          const int32_t* members, const int32_t* group_k, int32_t threads,
                          dpro_delta_set** out) {
  return dpro_base_delta_batch_ops(base, n, n_groups, spec_off, group_off, members, group_k,
                                   nullptr, nullptr, threads, out);
}

const dpro_delta* dpro_delta_set_deltas(const dpro_delta_set* s) { return s->views.data(); }
int32_t dpro_delta_set_size(const dpro_delta_set* s) { return static_cast<int32_t>(s->views.size()); }
const char* dpro_delta_set_device_str(const dpro_delta_set* s, int32_t cand, uint32_t d) {
  const dpro_graph& bg = *s->base->g;
  if (d < bg.device_strs.size()) return bg.device_strs[d].c_str();
  return s->d.at(cand).extra_dev_strs.at(d - bg.device_strs.size()).c_str();
}
void dpro_delta_set_free(dpro_delta_set* s) { delete s; }
const dpro_graph* dpro_base_graph(const dpro_base* base) { return base->b->g.get(); }

// memory.cpp:71-119 output_bytes_for over a (key -> bytes) table.
namespace {
int64_t local_output_bytes(const std::unordered_map<std::string, int64_t>& t, std::string local) {
  auto lookup = [&](const std::string& k) -> int64_t {
    const auto it = t.find(k);
    return it == t.end() ? -1 : it->second;
  };
  int64_t v = lookup(local);
  if (v >= 0) return v;
  const auto at = local.rfind("@mb");
  if (at != std::string::npos) {
    local = local.substr(0, at);
    v = lookup(local);
    if (v >= 0) return (v + 1) / 2;
  }
  if (local.rfind("RFW.", 0) == 0) return lookup("FW." + local.substr(4));
  return -1;
}

int64_t output_bytes_for(const std::unordered_map<std::string, int64_t>& t, const std::string& id) {
  const auto d = t.find(id);
  if (d != t.end()) return d->second;
  std::string local = id;
  const auto arrow = local.find("->");
  if (arrow != std::string::npos) local = local.substr(arrow + 2);
  const int64_t v = local_output_bytes(t, local);
  if (v >= 0) return v;
  if (local.find('+') == std::string::npos) return -1;
  int64_t total = 0;
  size_t pos = 0;
  for (;;) {
    const auto next = local.find('+', pos);
    const int64_t pb = local_output_bytes(
        t, next == std::string::npos ? local.substr(pos) : local.substr(pos, next - pos));
    if (pb < 0) return -1;
    total += pb;
    if (next == std::string::npos) return total;
    pos = next + 1;
  }
}
}  // namespace

int dpro_graph_memory_inputs(dpro_graph* g, int32_t n_entries, const char* const* keys,
                             const int64_t* bytes, int64_t* op_bytes, int32_t* op_node,
                             int32_t* n_nodes, uint32_t* missing_op) {
  if (!g || (n_entries > 0 && (!keys || !bytes)) || !op_bytes || !op_node || !n_nodes)
    return DPRO_EINVAL;
  std::unordered_map<std::string, int64_t> table;
  table.reserve(size_t(n_entries) * 2);
  for (int32_t k = 0; k < n_entries; ++k) table[keys[k]] = bytes[k];
  const uint32_t n = static_cast<uint32_t>(g->kind.size());
  // compute nodes (the device of a computation op is its node), name order
  std::vector<int32_t> node_of_dev(g->device_strs.size(), -1);
  std::vector<uint8_t> used(g->device_strs.size(), 0);
  for (uint32_t i = 0; i < n; ++i)
    if (g->kind[i] == kFw || g->kind[i] == kBw || g->kind[i] == kUpdate) used[g->dev[i]] = 1;
  std::vector<std::pair<std::string, uint32_t>> nodes;
  for (size_t d = 0; d < used.size(); ++d)
    if (used[d]) nodes.emplace_back(g->device_strs[d], static_cast<uint32_t>(d));
  std::sort(nodes.begin(), nodes.end());
  g->mem_nodes.clear();
  for (size_t k = 0; k < nodes.size(); ++k) {
    node_of_dev[nodes[k].second] = static_cast<int32_t>(k);
    g->mem_nodes.push_back(nodes[k].first);
  }
  *n_nodes = static_cast<int32_t>(nodes.size());
  if (missing_op) *missing_op = UINT32_MAX;
  for (uint32_t i = 0; i < n; ++i) {
    const int32_t k = g->kind[i];
    if (k != kFw && k != kBw && k != kUpdate) {
      op_bytes[i] = 0;
      op_node[i] = -1;
      continue;
    }
    op_node[i] = node_of_dev[g->dev[i]];
    int64_t b = output_bytes_for(table, dpro_graph_op_id(g, i));
    if (b < 0) {
      if (k != kUpdate) {  // MissingMetaError("no output bytes for op <id>")
        if (missing_op) *missing_op = i;
        return DPRO_EINVAL;
      }
      b = 0;
    }
    op_bytes[i] = b;
  }
  return DPRO_OK;
}

const char* dpro_graph_memory_node(const dpro_graph* g, int32_t i) {
  return g->mem_nodes.at(i).c_str();
}

const char* dpro_graph_comm_info(const dpro_graph* g, uint32_t i, int64_t* bytes) {
  if (!g || i >= g->kind.size() || g->cunit.empty() || g->cunit[i] < 0) return nullptr;
  if (bytes) *bytes = g->cbytes[i];
  return g->units.at(g->cunit[i]).c_str();
}

namespace {
const char* kind_name(int32_t k) {  // graph.cpp:25-43
  static const char* names[] = {"FW", "BW", "UPDATE", "SEND", "RECV", "VIRTUAL_IN",
                                "VIRTUAL_OUT"};
  return (k >= 0 && k < 7) ? names[k] : "UNKNOWN";
}
// A JSON string as nlohmann::json::dump writes it (UTF-8 kept, control
// characters escaped).
void json_str(std::string& o, const std::string& v) {
  o += '"';
  for (const unsigned char ch : v) {
    switch (ch) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (ch < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", ch);
          o += buf;
        } else {
          o += static_cast<char>(ch);
        }
    }
  }
  o += '"';
}
}  // namespace

int dpro_graph_write_timeline(const dpro_graph* g, const int64_t* start, const int64_t* end,
                              const char* path) {
  if (!g || !start || !end || !path) return DPRO_EINVAL;
  std::FILE* f = std::fopen(path, "wb");
  if (!f) {
    g_gen_err = std::string("cannot open ") + path;
    return DPRO_EINVAL;
  }
  // proj/tools/dpro_main.cpp:90-116 as written by write_json (64-70):
  // nlohmann dump(2), keys in byte order, trailing newline
  std::string o;
  o.reserve(1 << 20);
  o += "{\n  \"displayTimeUnit\": \"ms\",\n  \"traceEvents\": [";
  bool any = false;
  const uint32_t n = static_cast<uint32_t>(g->kind.size());
  for (uint32_t i = 0; i < n; ++i) {
    const int32_t k = g->kind[i];
    if (k == kVin || k == kVout) continue;
    const std::string id = dpro_graph_op_id(g, i);
    const std::string& dev = g->device_strs[g->dev[i]];
    std::string node = dev;
    const bool comm = k == kSend || k == kRecv;
    if (comm) {  // Op::node: the sender for SEND, the receiver for RECV
      const auto gt = dev.find('>');
      node = k == kSend ? dev.substr(0, gt) : dev.substr(gt + 1);
    }
    o += any ? ",\n    {\n" : "\n    {\n";
    any = true;
    o += "      \"args\": {\n";
    if (comm) {
      o += "        \"bytes\": " + std::to_string(g->cbytes.empty() ? 0 : g->cbytes[i]) + ",\n";
    }
    o += "        \"iteration\": 0,\n        \"kind\": ";
    json_str(o, kind_name(k));
    if (comm) {
      o += ",\n        \"tensor\": ";
      json_str(o, (g->cunit.empty() || g->cunit[i] < 0) ? std::string() : g->units[g->cunit[i]]);
      o += ",\n        \"transaction\": ";
      json_str(o, id.substr(5));  // "SEND." / "RECV." + transaction
    }
    o += "\n      },\n      \"cat\": ";
    json_str(o, kind_name(k));
    o += ",\n      \"dur\": " + std::to_string(end[i] - start[i]) + ",\n      \"name\": ";
    json_str(o, id);
    o += ",\n      \"ph\": \"X\",\n      \"pid\": ";
    json_str(o, dev);
    o += ",\n      \"tid\": ";
    json_str(o, node);
    o += ",\n      \"ts\": " + std::to_string(start[i]) + "\n    }";
    if (o.size() > (1u << 20)) {
      std::fwrite(o.data(), 1, o.size(), f);
      o.clear();
    }
  }
  o += any ? "\n  ]\n}\n" : "]\n}\n";
  std::fwrite(o.data(), 1, o.size(), f);
  const bool ok = std::fclose(f) == 0;
  return ok ? DPRO_OK : DPRO_EINVAL;
}

int32_t dpro_graph_op_kind(const dpro_graph* g, uint32_t i) { return g->kind.at(i); }
const char* dpro_graph_device_str(const dpro_graph* g, uint32_t d) {
  return g->device_strs.at(d).c_str();
}
void dpro_graph_free(dpro_graph* g) { delete g; }

}  // extern "C"

// Internal entry for the engine's t_sync grid (engine.cu).
dpro_graph* dpro_internal_tsync_graph(const dpro_cluster_desc* cluster,
                                      int64_t bytes, int32_t k,
                                      std::string* err) {
  try {
    return build_tsync(Cluster(*cluster), bytes, k);
  } catch (const std::exception& e) {
    if (err) *err = e.what();
    return nullptr;
  }
}
