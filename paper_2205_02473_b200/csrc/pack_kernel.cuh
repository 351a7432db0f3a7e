// Pack: caller CSR (SoA, index order) -> the engine's replay layout.
//
// Runs once when a batch is registered (engine.cu). Per candidate:
//   rec[i]  = 16-byte record of op i (format below), plus a sentinel rec[n]
//   erec[k] = the record of s for edge k: i -> s (same format)
//   cnt0[c] = indeg of the c-th multi-predecessor op (compact u8 counters)
//   srcs    = ops with no predecessor (unordered; the replay sorts them)
//   devoff  = exclusive scan of non-virtual ops per device (timeline regions)
//   info    = first op without duration, fast-path eligibility, sizes.
// Virtual ops with exactly one predecessor are SPLICED: in the predecessor's
// list the edge to v becomes a stamp record for v (virtual, not multi)
// followed by v's own (expanded) successors. replay.cpp:60-72 completes such
// a v in the same round as its predecessor and readies its successors at the
// same t, so processing them from the predecessor's list is exact; the
// expanded lists have exactly E entries in total.
// The per-edge record carries everything the replay needs at the moment the
// edge's completion makes s ready (device, virtual flag, duration, successor
// range, counter slot) -- exactly what proj/src/replay.cpp:60-72,80-87 reads
// about s then -- so an event round touches one record per edge.
#pragma once

#include <cub/block/block_scan.cuh>

#include "replay_kernel.cuh"

namespace dpro_k {

// 16-byte op record (rec[i] for op i; erec[k] = record of s for edge i->s):
//   x = s (24 bits) | cidx bits 0..7 << 24
//   y = dur (int32; 0 for virtual ops, which never run)
//   z = dev (10 bits) | virtual << 10 | multi << 11 | succ count (6 bits,
//       63 = "read succ_end from rec[s+1].w") << 12 | cidx bits 8..21 << 18
//   w = succ_beg
// rec has n+1 entries; rec[n].w = n_edges, so succ_end(s) = rec[s+1].w.
constexpr uint32_t kOpMask = 0xFFFFFFu;
constexpr uint32_t kDevMask = 0x3FFu;
constexpr uint32_t kFVirt = 1u << 10;
constexpr uint32_t kFMulti = 1u << 11;  // >= 2 predecessors: has a counter
constexpr uint32_t kCntShift = 12;
constexpr uint32_t kCntMax = 63u;
constexpr uint32_t kMaxOps = 1u << 24;
constexpr uint32_t kMaxDev = 1u << 10;
constexpr uint32_t kMaxCnt = 1u << 22;

// not_fast bits
constexpr uint32_t kNfDur = 1u;       // |dur| >= 2^31 or sum of dur >= 2^31
constexpr uint32_t kNfIndeg = 2u;     // some indeg >= 255
constexpr uint32_t kNfVsrc = 4u;      // virtual op without predecessors
constexpr uint32_t kNfDev = 8u;       // device id out of range / > 1024 devices
constexpr uint32_t kNfSize = 16u;     // >= 2^24 ops or >= 2^22 counters
constexpr uint32_t kNfChain = 32u;    // virtual chain deeper than kMaxSplice
constexpr int kMaxSplice = 8;

struct PackInfo {
  uint32_t first_missing;  // kNone: every non-virtual op has dur >= 0
  uint32_t not_fast;
  uint32_t n_cnt;          // multi-predecessor ops (compact counters)
  uint32_t n_src;          // ops without predecessors
  unsigned long long dur_sum;
};

struct PackOut {
  uint4* rec;                  // [sum (n+1)]
  uint4* erec;                 // [sum e]
  uint8_t* cnt0;               // [sum n16]
  uint32_t* srcs;              // [sum n]
  uint32_t* cidx;              // [sum n] scratch: counter slot per op
  uint32_t* xoff;              // [sum (n+1)] scratch: expanded list offsets
  uint8_t* spl;                // [sum n] scratch: spliced virtual op marks
  unsigned long long* r_off;   // per candidate offset into rec (in records)
  unsigned long long* e_off;   // per candidate offset into erec (in edges)
  unsigned long long* c_off;   // per candidate byte offset into cnt0
  PackInfo* info;              // [B]
};

__device__ __forceinline__ bool spliced(const Cand& c, const uint32_t* indeg, uint32_t s) {
  return (c.flags[s] & 1u) && indeg[s] == 1u;
}

// Record of s; its successor range is its EXPANDED list [xoff[s], xoff[s+1]).
__device__ __forceinline__ uint4 make_rec(uint32_t s, const Cand& c, const uint32_t* indeg,
                                          const uint32_t* cidx, const uint32_t* xoff) {
  const uint32_t f = c.flags[s];
  const uint32_t ind = indeg[s];
  const bool virt = f & 1u;
  const uint32_t ci = ind >= 2 ? cidx[s] : 0u;
  const uint32_t cnt = min(xoff[s + 1] - xoff[s], kCntMax);
  const uint32_t z = (uint32_t(c.dev[s]) & kDevMask) | (virt ? kFVirt : 0u) |
                     (ind >= 2 ? kFMulti : 0u) | (cnt << kCntShift) | ((ci >> 8) << 18);
  const long long du = virt ? 0 : ld_dur(c, s);
  return make_uint4((s & kOpMask) | ((ci & 0xFFu) << 24),
                    static_cast<uint32_t>(static_cast<int>(du)), z, xoff[s]);
}

// Walks the expanded successor list of op i (DFS through spliced virtual
// successors, in order): emit(s, spliced) per entry. spl[s] = 1 for a
// virtual op with exactly one predecessor. Returns false when a spliced
// chain is deeper than kMaxSplice. Lists with splices at most one level
// deep (all generated graphs) stay in registers; deeper ones use a stack.
template <typename Emit>
__device__ bool walk_deep(uint32_t i, const Cand& c, const uint8_t* spl, Emit&& emit) {
  uint32_t stk_op[kMaxSplice], stk_k[kMaxSplice];
  int sp = 0;
  stk_op[0] = i;
  stk_k[0] = c.succ_off[i];
  for (;;) {
    const uint32_t v = stk_op[sp];
    if (stk_k[sp] == c.succ_off[v + 1]) {
      if (sp == 0) return true;
      --sp;
      continue;
    }
    const uint32_t s = c.succ[stk_k[sp]++];
    const bool sv = spl[s];
    emit(s, sv);
    if (sv) {
      if (sp + 1 >= kMaxSplice) return false;
      ++sp;
      stk_op[sp] = s;
      stk_k[sp] = c.succ_off[s];
    }
  }
}

template <typename Emit>
__device__ bool walk_list(uint32_t i, const Cand& c, const uint8_t* spl, Emit&& emit) {
  // first pass over the top-level list: any splice with a spliced child?
  const uint32_t a = c.succ_off[i], z = c.succ_off[i + 1];
  bool nested = false;
  for (uint32_t k = a; k < z && !nested; ++k) {
    const uint32_t s = c.succ[k];
    if (spl[s])
      for (uint32_t t = c.succ_off[s]; t < c.succ_off[s + 1]; ++t) nested |= spl[c.succ[t]] != 0;
  }
  if (nested) return walk_deep(i, c, spl, emit);
  for (uint32_t k = a; k < z; ++k) {
    const uint32_t s = c.succ[k];
    const bool sv = spl[s];
    emit(s, sv);
    if (sv)
      for (uint32_t t = c.succ_off[s]; t < c.succ_off[s + 1]; ++t) emit(c.succ[t], false);
  }
  return true;
}

constexpr int kPackThreads = 1024;
constexpr uint32_t kPackHist = 4096;  // devices counted in shared memory

// In-place exclusive scan of a[0..n) by one block; returns the total.
template <int NT, typename Scan>
__device__ uint32_t block_exclusive_scan(uint32_t* a, uint32_t n,
                                         typename Scan::TempStorage& tmp, uint32_t& s_carry) {
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n; base += NT) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < n ? a[i] : 0u;
    uint32_t excl, total;
    Scan(tmp).ExclusiveSum(v, excl, total);
    const uint32_t carry = s_carry;
    if (i < n) a[i] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + total;
    __syncthreads();
  }
  return s_carry;
}

// One 1024-thread block per candidate, one block per SM (grid = SM count):
// the ~150 candidates in flight keep their CSR and scratch in L2, so the
// per-edge gathers of pass 2/3b are L2 hits. indeg must be present (host
// upload or delta merge) or computed by count_indeg_kernel.
__global__ void __launch_bounds__(kPackThreads, 1) pack_kernel(const Cand* __restrict__ cands,
                                                               int n_cands, Scratch S,
                                                               PackOut P) {
  using Scan = cub::BlockScan<uint32_t, kPackThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t s_first, s_flags, s_ncnt, s_nsrc, s_carry;
  __shared__ unsigned long long s_sum;
  __shared__ uint32_t s_hist[kPackHist];
  const uint32_t lane = threadIdx.x & 31;
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const Cand c = cands[cid];
    const uint32_t n = c.n;
    const uint32_t* indeg = c.indeg ? c.indeg : S.indeg + c.op_off;
    uint4* rec = P.rec + P.r_off[cid];
    uint4* erec = P.erec + P.e_off[cid];
    uint8_t* cnt0 = P.cnt0 + P.c_off[cid];
    uint32_t* srcs = P.srcs + c.op_off;
    uint32_t* cidx = P.cidx + c.op_off;
    uint8_t* spl = P.spl + c.op_off;
    uint32_t* xoff = P.xoff + P.r_off[cid];
    if (threadIdx.x == 0) {
      s_first = kNone;
      s_flags = (n >= kMaxOps ? kNfSize : 0u) | (c.d > kMaxDev ? kNfDev : 0u);
      s_ncnt = 0;
      s_nsrc = 0;
      s_sum = 0;
    }
    const bool hist_smem = c.d <= kPackHist;
    for (uint32_t d = threadIdx.x; d < kPackHist; d += kPackThreads) s_hist[d] = 0;
    uint32_t* devoff = S.devoff + c.dof_off;
    if (!hist_smem)
      for (uint32_t d = threadIdx.x; d <= c.d; d += kPackThreads) devoff[d] = 0;
    __syncthreads();
    // pass 1 (coalesced): checks, counter slots and sources (warp-aggregated),
    // splice marks, per-device op counts
    uint32_t flags = 0, first = kNone;
    unsigned long long sum = 0;
    const uint32_t n_up = (n + 31) & ~31u;
    for (uint32_t i = threadIdx.x; i < n_up; i += kPackThreads) {
      const bool ok = i < n;
      uint32_t ind = 0;
      bool virt = false;
      if (ok) {
        const long long du = ld_dur(c, i);
        virt = c.flags[i] & 1u;
        ind = indeg[i];
        const uint32_t dv = c.dev[i];
        if (!virt && du < 0) first = min(first, i);
        if (!virt && (du > 0x7FFFFFFFLL || du < -0x80000000LL)) flags |= kNfDur;
        if (!virt && du > 0) sum += static_cast<unsigned long long>(du);
        if (ind >= 255u) flags |= kNfIndeg;
        if (virt && ind == 0u) flags |= kNfVsrc;
        if (!virt && dv >= c.d) flags |= kNfDev;
        spl[i] = virt && ind == 1u;
        if (!virt && dv < c.d) atomicAdd(hist_smem ? &s_hist[dv] : &devoff[dv], 1u);
      }
      const bool multi = ok && ind >= 2u, src = ok && ind == 0u;
      const unsigned mm = __ballot_sync(kFull, multi), ms = __ballot_sync(kFull, src);
      uint32_t bm = 0, bs = 0;
      if (lane == 0) {
        if (mm) bm = atomicAdd(&s_ncnt, __popc(mm));
        if (ms) bs = atomicAdd(&s_nsrc, __popc(ms));
      }
      bm = __shfl_sync(kFull, bm, 0);
      bs = __shfl_sync(kFull, bs, 0);
      const unsigned lt = (1u << lane) - 1u;
      if (multi) {
        const uint32_t slot = bm + __popc(mm & lt);
        cidx[i] = slot;
        if (slot < kMaxCnt) cnt0[slot] = static_cast<uint8_t>(min(ind, 255u));
      } else if (src) {
        srcs[bs + __popc(ms & lt)] = i;
      }
    }
    if (first != kNone) atomicMin(&s_first, first);
    if (flags) atomicOr(&s_flags, flags);
    if (sum) atomicAdd(&s_sum, sum);
    __syncthreads();
    // pass 2: expanded list sizes (spliced virtual ops own no list)
    bool deep = false;
    for (uint32_t i = threadIdx.x; i < n; i += kPackThreads) {
      uint32_t len = 0;
      if (!spl[i]) deep |= !walk_list(i, c, spl, [&](uint32_t, bool) { ++len; });
      xoff[i] = len;
    }
    if (deep) atomicOr(&s_flags, kNfChain);
    __syncthreads();
    const uint32_t total = block_exclusive_scan<kPackThreads, Scan>(xoff, n, scan_tmp, s_carry);
    if (threadIdx.x == 0) xoff[n] = total;
    __syncthreads();
    // pass 3a (coalesced): every op's record
    for (uint32_t i = threadIdx.x; i < n; i += kPackThreads) rec[i] = make_rec(i, c, indeg, cidx, xoff);
    if (threadIdx.x == 0) rec[n] = make_uint4(0u, 0u, 0u, total);
    __syncthreads();  // rec[] visible to the block
    // pass 3b: expanded lists = gathered records (stamps for spliced ops)
    for (uint32_t i = threadIdx.x; i < n; i += kPackThreads) {
      if (spl[i]) continue;
      uint4* dst = erec + xoff[i];
      walk_list(i, c, spl, [&](uint32_t s, bool sv) {  // erec is write-once: stream it
        __stcs(dst++, sv ? make_uint4(s & kOpMask, 0u, kFVirt, 0u) : rec[s]);
      });
    }
    if (threadIdx.x == 0) {
      PackInfo inf;
      inf.first_missing = s_first;
      inf.not_fast = s_flags | (s_sum >= 0x7FFFFFFFull ? kNfDur : 0u) |
                     (s_ncnt >= kMaxCnt ? kNfSize : 0u);
      inf.n_cnt = s_ncnt;
      inf.n_src = s_nsrc;
      inf.dur_sum = s_sum;
      P.info[cid] = inf;
    }
    // timeline regions: exclusive scan of the per-device counts
    if (hist_smem)
      for (uint32_t d = threadIdx.x; d < c.d; d += kPackThreads) devoff[d] = s_hist[d];
    __syncthreads();
    const uint32_t dtot = block_exclusive_scan<kPackThreads, Scan>(devoff, c.d, scan_tmp, s_carry);
    if (threadIdx.x == 0) devoff[c.d] = dtot;
    __syncthreads();
  }
}

// indeg for device batches registered without it.
__global__ void count_indeg_kernel(const Cand* __restrict__ cands, int n_cands,
                                   Scratch S) {
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const Cand c = cands[cid];
    if (c.indeg) continue;
    uint32_t* ind = S.indeg + c.op_off;
    for (uint32_t i = threadIdx.x; i < c.n; i += blockDim.x) ind[i] = 0;
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < c.e; k += blockDim.x) atomicAdd(&ind[c.succ[k]], 1u);
    __syncthreads();
  }
}

}  // namespace dpro_k
