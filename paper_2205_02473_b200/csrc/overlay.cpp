// Host builder of candidate overlays (overlay.h). O(changed ops + their
// lists + the base blocks they touch) per candidate; the base is never
// copied. The index order, in-degrees, splices and expanded lists follow
// exactly what the merge (delta_kernel.cuh) + pack (pack_kernel.cuh) would
// produce for the same delta, so the replay sees the same candidate.
#include "overlay.h"

#include <algorithm>
#include <array>
#include <functional>
#include <cstring>
#include <stdexcept>
#include <unordered_map>

namespace dpro_ov {
namespace {

constexpr uint32_t kOpMask = 0xFFFFFFu;
constexpr uint32_t kFVirt = 1u << 10;
constexpr uint32_t kFMulti = 1u << 11;
constexpr uint32_t kCntShift = 12;
constexpr uint32_t kCntMax = 63u;
constexpr uint32_t kMaxOps = 1u << 24;
constexpr uint32_t kMaxDev = 1u << 10;
constexpr uint32_t kMaxCnt = 1u << 22;
constexpr int kMaxSplice = 8;

// An op of the candidate: kept base op (b) or new op (j).
struct Ref {
  uint32_t id;
  bool is_new;
};

struct Work {
  const BaseHost& B;
  const dpro_delta& D;
  OverlayHost& O;
  std::vector<uint32_t> fin_new;          // final index of new op j
  std::vector<uint32_t> kept_rank_key;    // removed[i] - i
  std::unordered_map<uint32_t, int32_t> ddeg;   // in-degree change of kept base ops
  std::vector<uint32_t> new_indeg;        // candidate in-degree of new ops
  std::vector<uint32_t> dirty;            // sorted kept dirty base ops
  std::unordered_map<uint32_t, uint32_t> dslot;  // dirty base op -> slot
  std::vector<uint32_t> cnt_slot;         // per overlay slot: counter slot or UINT32_MAX

  Work(const BaseHost& b, const dpro_delta& d, OverlayHost& o) : B(b), D(d), O(o) {}

  bool removed(uint32_t b) const {
    return std::binary_search(D.removed, D.removed + D.n_removed, b);
  }
  uint32_t rem_lt(uint32_t b) const {
    return static_cast<uint32_t>(std::lower_bound(D.removed, D.removed + D.n_removed, b) -
                                 D.removed);
  }
  uint32_t new_le(uint32_t b) const {
    return static_cast<uint32_t>(std::upper_bound(D.new_pos, D.new_pos + D.n_new, b) -
                                 D.new_pos);
  }
  uint32_t fin_base(uint32_t b) const { return b - rem_lt(b) + new_le(b); }
  // candidate final index -> op
  Ref of_final(uint32_t f) const {
    const auto it = std::lower_bound(fin_new.begin(), fin_new.end(), f);
    if (it != fin_new.end() && *it == f)
      return {static_cast<uint32_t>(it - fin_new.begin()), true};
    const uint32_t k = f - static_cast<uint32_t>(it - fin_new.begin());  // k-th kept base op
    const uint32_t b = k + static_cast<uint32_t>(
                               std::upper_bound(kept_rank_key.begin(), kept_rank_key.end(), k) -
                               kept_rank_key.begin());
    return {b, false};
  }
  bool is_dirty(uint32_t b) const { return dslot.count(b) != 0; }
  uint32_t slot_of(const Ref& r) const {
    return r.is_new ? static_cast<uint32_t>(dirty.size()) + r.id : dslot.at(r.id);
  }
  uint32_t cand_indeg(const Ref& r) const {
    if (r.is_new) return new_indeg[r.id];
    const auto it = ddeg.find(r.id);
    return static_cast<uint32_t>(static_cast<int64_t>(B.indeg[r.id]) +
                                 (it == ddeg.end() ? 0 : it->second));
  }
  bool virt(const Ref& r) const {
    return ((r.is_new ? D.new_flags[r.id] : B.flags[r.id]) & DPRO_FLAG_VIRTUAL) != 0;
  }
  int64_t dur(const Ref& r) const { return r.is_new ? D.new_dur[r.id] : B.dur[r.id]; }
  uint32_t dev(const Ref& r) const { return r.is_new ? D.new_dev[r.id] : B.dev[r.id]; }
  bool pure(const Ref& r) const { return !r.is_new && !is_dirty(r.id); }
  bool spliced(const Ref& r) const { return virt(r) && cand_indeg(r) == 1; }

  // candidate successor list (final indices, ascending) of an overlay op
  void cand_succ(const Ref& r, std::vector<uint32_t>& out) const {
    out.clear();
    if (r.is_new) {
      out.assign(D.new_succ + D.new_succ_off[r.id], D.new_succ + D.new_succ_off[r.id + 1]);
      return;
    }
    const uint32_t u = r.id;
    for (uint32_t e = B.succ_off[u]; e < B.succ_off[u + 1]; ++e) {
      const uint32_t s = B.succ[e];
      if (removed(s) || std::binary_search(D.cut, D.cut + D.n_cut, e)) continue;
      out.push_back(fin_base(s));
    }
    const auto lo = std::lower_bound(D.extra_src, D.extra_src + D.n_extra, u);
    const auto hi = std::upper_bound(D.extra_src, D.extra_src + D.n_extra, u);
    const size_t mid = out.size();
    for (auto p = lo; p < hi; ++p) out.push_back(D.extra_dst[p - D.extra_src]);
    std::inplace_merge(out.begin(), out.begin() + mid, out.end());
  }
};

inline void put4(std::vector<uint32_t>& v, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  v.push_back(x);
  v.push_back(y);
  v.push_back(z);
  v.push_back(w);
}

}  // namespace

void build_overlay(const BaseHost& B, const dpro_delta& D, OverlayHost& O) {
  O.rec.clear();
  O.erec.clear();
  O.fin.clear();
  O.cnt.clear();
  O.src.clear();
  O.blk.clear();
  O.ovf.clear();
  O.devoff.clear();
  O.sx.clear();
  O.sbp.clear();
  O.sparse = false;
  O.ovmin = 0;
  O.fast = true;
  O.why.clear();
  O.first_missing = UINT32_MAX;
  const uint32_t nb = B.n, nn = D.n_new;
  O.n_ops = nb - D.n_removed + nn;
  O.n_devices = D.n_devices;
  auto slow = [&](const char* why) {
    O.fast = false;
    O.why = why;
  };
  if (!B.ok) return slow("base not packed for the fast path");
  if (O.n_ops >= kMaxOps) return slow(">= 2^24 ops");
  if (D.n_devices > kMaxDev) return slow("> 1024 devices");
  Work W(B, D, O);
  // final indices of the new ops (ascending in j)
  W.fin_new.resize(nn);
  for (uint32_t j = 0; j < nn; ++j) W.fin_new[j] = D.new_pos[j] - W.rem_lt(D.new_pos[j]) + j;
  W.kept_rank_key.resize(D.n_removed);
  for (uint32_t i = 0; i < D.n_removed; ++i) W.kept_rank_key[i] = D.removed[i] - i;
  // in-degree changes
  W.new_indeg.assign(nn, 0);
  auto add_in = [&](uint32_t f, int32_t v) {
    const Ref r = W.of_final(f);
    if (r.is_new) W.new_indeg[r.id] += v;
    else W.ddeg[r.id] += v;
  };
  for (uint32_t k = 0; k < D.n_removed; ++k) {
    const uint32_t u = D.removed[k];
    for (uint32_t e = B.succ_off[u]; e < B.succ_off[u + 1]; ++e)
      if (!W.removed(B.succ[e])) W.ddeg[B.succ[e]] -= 1;
  }
  for (uint32_t k = 0; k < D.n_cut; ++k) W.ddeg[B.succ[D.cut[k]]] -= 1;
  for (uint32_t k = 0; k < D.n_extra; ++k) add_in(D.extra_dst[k], 1);
  for (uint32_t k = 0; k < D.new_succ_off[nn]; ++k) add_in(D.new_succ[k], 1);
  // dirty kept base ops
  std::vector<uint32_t> dl;
  for (const auto& kv : W.ddeg)
    if (kv.second != 0) dl.push_back(kv.first);
  for (uint32_t k = 0; k < D.n_removed; ++k) {  // preds of removed ops lose an edge
    const uint32_t r = D.removed[k];
    for (uint32_t p = B.pred_off[r]; p < B.pred_off[r + 1]; ++p)
      if (!W.removed(B.pred[p])) dl.push_back(B.pred[p]);
  }
  for (uint32_t k = 0; k < D.n_cut; ++k) {
    const uint32_t e = D.cut[k];
    dl.push_back(static_cast<uint32_t>(
        std::upper_bound(B.succ_off.begin(), B.succ_off.end(), e) - B.succ_off.begin() - 1));
  }
  for (uint32_t k = 0; k < D.n_extra; ++k) dl.push_back(D.extra_src[k]);
  std::sort(dl.begin(), dl.end());
  dl.erase(std::unique(dl.begin(), dl.end()), dl.end());
  // a base list inlines its spliced virtual successors: when such a v is
  // dirty or removed, its (single) base predecessor's list changes too
  {
    std::vector<uint32_t> todo(dl.begin(), dl.end());
    for (uint32_t k = 0; k < D.n_removed; ++k) todo.push_back(D.removed[k]);
    std::vector<uint32_t> add;
    while (!todo.empty()) {
      const uint32_t v = todo.back();
      todo.pop_back();
      if (!((B.flags[v] & DPRO_FLAG_VIRTUAL) && B.indeg[v] == 1)) continue;
      const uint32_t p = B.pred[B.pred_off[v]];
      if (W.removed(p) || std::binary_search(dl.begin(), dl.end(), p)) continue;
      dl.insert(std::upper_bound(dl.begin(), dl.end(), p), p);
      todo.push_back(p);
    }
  }
  W.dirty = dl;
  const uint32_t nd = static_cast<uint32_t>(dl.size());
  for (uint32_t s = 0; s < nd; ++s) W.dslot[dl[s]] = s;
  const uint32_t no = nd + nn;
  if (no >= kMaxOps) return slow("overlay too large");
  auto ref_of_slot = [&](uint32_t s) -> Ref { return s < nd ? Ref{dl[s], false} : Ref{s - nd, true}; };
  auto fin_of = [&](const Ref& r) { return r.is_new ? W.fin_new[r.id] : W.fin_base(r.id); };
  // first op without a duration (replay.cpp:39-44), in final order
  for (uint32_t j = 0; j < nn; ++j)
    if (!(D.new_flags[j] & DPRO_FLAG_VIRTUAL) && D.new_dur[j] < 0)
      O.first_missing = std::min(O.first_missing, W.fin_new[j]);
  for (uint32_t b : B.missing)
    if (!W.removed(b)) {
      O.first_missing = std::min(O.first_missing, W.fin_base(b));
      break;
    }
  // counters, fast-path checks, final indices of the overlay ops
  O.fin.resize(no);
  W.cnt_slot.assign(no, UINT32_MAX);
  for (uint32_t s = 0; s < no; ++s) {
    const Ref r = ref_of_slot(s);
    O.fin[s] = fin_of(r);
    const uint32_t ind = W.cand_indeg(r);
    const bool v = W.virt(r);
    if (ind >= 65535u) return slow("in-degree >= 65535");
    if (v && ind == 0) return slow("virtual op without predecessors (init quirk)");
    if (!v && (W.dur(r) > 0x7FFFFFFFLL || W.dur(r) < -0x80000000LL))
      return slow("duration needs more than 32 bits");
    if (!v && W.dev(r) >= D.n_devices) return slow("device id out of range");
    bool multi = ind >= 2;
    if (v && ind == 1) {  // not inlined anywhere when its predecessor is a pure base op
      std::vector<uint32_t> tmp;
      bool pure_pred = false;
      if (!r.is_new) {
        // its single candidate predecessor: a kept base pred not removed
        // whose edge is not cut, or the source of an extra edge
        for (uint32_t p = B.pred_off[r.id]; p < B.pred_off[r.id + 1]; ++p) {
          const uint32_t q = B.pred[p];
          if (W.removed(q)) continue;
          uint32_t e = B.succ_off[q];
          while (B.succ[e] != r.id) ++e;
          if (std::binary_search(D.cut, D.cut + D.n_cut, e)) continue;
          pure_pred = !W.is_dirty(q);
        }
      }
      multi = pure_pred;
    }
    if (multi) {
      W.cnt_slot[s] = B.n_cnt + static_cast<uint32_t>(O.cnt.size());
      O.cnt.push_back(static_cast<uint16_t>(ind));
    }
  }
  if (B.n_cnt + O.cnt.size() >= kMaxCnt) return slow(">= 2^22 counters");
  // expanded list sizes (pass 1) and contents (pass 2)
  std::vector<uint32_t> xoff(no + 1, 0);
  std::vector<uint32_t> lst, lst2;
  auto rec_of = [&](const Ref& r, uint32_t xo, uint32_t cntv) -> std::array<uint32_t, 4> {
    if (W.pure(r)) {
      const uint32_t* q = &B.rec[4 * size_t(r.id)];
      return {q[0], q[1], q[2], q[3]};
    }
    const uint32_t s = W.slot_of(r);
    const bool v = W.virt(r);
    const uint32_t ci = W.cnt_slot[s] == UINT32_MAX ? 0u : W.cnt_slot[s];
    const uint32_t z = (W.dev(r) & 0x3FFu) | (v ? kFVirt : 0u) |
                       (W.cnt_slot[s] != UINT32_MAX ? kFMulti : 0u) |
                       (std::min(cntv, kCntMax) << kCntShift) | ((ci >> 8) << 18);
    const int64_t du = v ? 0 : W.dur(r);
    return {(s & kOpMask) | ((ci & 0xFFu) << 24),
            static_cast<uint32_t>(static_cast<int32_t>(du)), z, xo | kOv};
  };
  // emit(r, depth): the expanded candidate list of overlay op / spliced op r
  bool deep = false;
  std::function<uint32_t(const Ref&, int, bool)> walk = [&](const Ref& r, int depth,
                                                            bool write) -> uint32_t {
    std::vector<uint32_t> succ;
    if (W.pure(r)) {  // a pure spliced op inlined into an overlay list
      for (uint32_t e = B.succ_off[r.id]; e < B.succ_off[r.id + 1]; ++e)
        succ.push_back(W.fin_base(B.succ[e]));
    } else {
      W.cand_succ(r, succ);
    }
    uint32_t len = 0;
    for (uint32_t f : succ) {
      const Ref t = W.of_final(f);
      if (W.spliced(t)) {
        if (depth + 1 >= kMaxSplice) {
          deep = true;
          return len;
        }
        if (write) {
          if (W.pure(t)) put4(O.erec, t.id & kOpMask, 0u, kFVirt, 0u);
          else put4(O.erec, W.slot_of(t) & kOpMask, 0u, kFVirt, kOv);
        }
        len += 1 + walk(t, depth + 1, write);
      } else {
        if (write) {
          std::array<uint32_t, 4> q;
          if (W.pure(t)) {
            q = rec_of(t, 0, 0);
          } else {
            const uint32_t st = W.slot_of(t);
            q = rec_of(t, xoff[st], xoff[st + 1] - xoff[st]);
          }
          put4(O.erec, q[0], q[1], q[2], q[3]);
        }
        ++len;
      }
    }
    return len;
  };
  for (uint32_t s = 0; s < no; ++s) {
    const Ref r = ref_of_slot(s);
    xoff[s + 1] = xoff[s] + walk(r, 0, false);
    if (deep) return slow("virtual chain deeper than the splice limit");
  }
  if (xoff[no] >= kOv) return slow("overlay lists too large");
  O.erec.reserve(4 * size_t(xoff[no]));
  for (uint32_t s = 0; s < no; ++s) {
    const Ref r = ref_of_slot(s);
    const auto q = rec_of(r, xoff[s], xoff[s + 1] - xoff[s]);
    put4(O.rec, q[0], q[1], q[2], q[3]);
    walk(r, 0, true);
  }
  put4(O.rec, 0u, 0u, 0u, xoff[no] | kOv);
  // sources: pure base sources + overlay ops without predecessors
  for (uint32_t b : B.srcs)
    if (!W.removed(b) && !W.is_dirty(b)) {
      const uint32_t* q = &B.rec[4 * size_t(b)];
      put4(O.src, q[0], q[1], q[2], q[3]);
    }
  for (uint32_t s = 0; s < no; ++s)
    if (W.cand_indeg(ref_of_slot(s)) == 0) {
      const uint32_t* q = &O.rec[4 * size_t(s)];
      put4(O.src, q[0], q[1], q[2], q[3]);
    }
  // timeline regions: non-virtual ops per device
  O.devoff.assign(D.n_devices + 1, 0);
  for (uint32_t d = 0; d < B.d && d < D.n_devices; ++d) O.devoff[d + 1] = B.devcnt[d];
  for (uint32_t k = 0; k < D.n_removed; ++k)
    if (!(B.flags[D.removed[k]] & DPRO_FLAG_VIRTUAL)) O.devoff[B.dev[D.removed[k]] + 1] -= 1;
  for (uint32_t j = 0; j < nn; ++j)
    if (!(D.new_flags[j] & DPRO_FLAG_VIRTUAL)) O.devoff[D.new_dev[j] + 1] += 1;
  for (uint32_t d = 0; d < D.n_devices; ++d) O.devoff[d + 1] += O.devoff[d];
  // sparse form: the shift of final(b) = b - #removed<b + #new_pos<=b
  // changes at r + 1 for every removed r (-1) and at every new_pos (+1)
  {
    std::vector<std::pair<uint32_t, int32_t>> ch;
    for (uint32_t k = 0; k < D.n_removed && ch.size() <= 2 * kSparseMax; ++k)
      ch.emplace_back(D.removed[k] + 1, -1);
    for (uint32_t j = 0; j < nn && ch.size() <= 2 * kSparseMax; ++j) ch.emplace_back(D.new_pos[j], 1);
    if (nd <= kSparseMax && ch.size() <= 2 * kSparseMax) {
      std::sort(ch.begin(), ch.end());
      int32_t sh = 0;
      for (size_t k = 0; k < ch.size();) {
        const uint32_t pos = ch[k].first;
        int32_t dsh = 0;
        for (; k < ch.size() && ch[k].first == pos; ++k) dsh += ch[k].second;
        if (dsh == 0) continue;
        sh += dsh;
        O.sbp.push_back(pos);
        O.sbp.push_back(static_cast<uint32_t>(sh));
      }
      if (O.sbp.size() / 2 <= kSparseMax) {
        O.sparse = true;
        for (uint32_t s = 0; s < nd; ++s) {
          O.sx.push_back(dl[s]);
          O.sx.push_back(s);
        }
        O.ovmin = UINT32_MAX;
        if (!O.sbp.empty()) O.ovmin = O.sbp[0];
        if (nd) O.ovmin = std::min(O.ovmin, dl[0]);
      } else {
        O.sbp.clear();
      }
    }
  }
  // block table: uniform shift, or per-op entries where removed ops, dirty
  // ops or insertion points fall inside the block
  const uint32_t nblk = (nb + kBlk - 1) / kBlk + 1;
  std::vector<uint8_t> flag(nblk, 0);
  for (uint32_t k = 0; k < D.n_removed; ++k) flag[D.removed[k] >> kBlkShift] = 1;
  for (uint32_t b : dl) flag[b >> kBlkShift] = 1;
  for (uint32_t j = 0; j < nn; ++j) {
    const uint32_t p = D.new_pos[j];
    if ((p & (kBlk - 1)) != 0) flag[p >> kBlkShift] = 1;
  }
  O.blk.resize(nblk);
  uint32_t rp = 0, np_ = 0;  // sweep: removed < b0, new_pos <= b0
  for (uint32_t k = 0; k < nblk; ++k) {
    const uint32_t b0 = k << kBlkShift;
    while (rp < D.n_removed && D.removed[rp] < b0) ++rp;
    while (np_ < nn && D.new_pos[np_] <= b0) ++np_;
    if (!flag[k]) {
      const int64_t sh = int64_t(np_) - int64_t(rp);
      O.blk[k] = static_cast<uint32_t>(sh + kBlkBias);
      continue;
    }
    const uint32_t m = static_cast<uint32_t>(O.ovf.size() / kBlk);
    O.blk[k] = kBlkOvf | m;
    for (uint32_t i = 0; i < kBlk; ++i) {
      const uint32_t b = b0 + i;
      uint32_t v = kOvfNone;
      if (b < nb && !W.removed(b)) {
        const auto it = W.dslot.find(b);
        v = it != W.dslot.end() ? (kOvfDirty | it->second) : W.fin_base(b);
      }
      O.ovf.push_back(v);
    }
  }
}

}  // namespace dpro_ov
