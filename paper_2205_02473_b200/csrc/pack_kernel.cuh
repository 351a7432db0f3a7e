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

#include <cooperative_groups.h>
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
constexpr uint32_t kNfDur = 1u;       // some |dur| >= 2^31 (the record holds int32)
constexpr uint32_t kNfIndeg = 2u;     // some indeg >= 65535
constexpr uint32_t kWideCnt = 1u << 8;  // (PackInfo::wide) some indeg >= 255: u16 counters
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
  uint32_t wide;           // kWideCnt: u16 counters (cnt0 as uint16_t)
  uint32_t pad;
};

struct PackOut {
  uint4* rec;                  // [sum (n+1)]
  uint4* erec;                 // [sum e]
  uint8_t* cnt0;               // [sum 2*n16] u8 counters, or u16 for wide candidates
  uint8_t* gcnt;               // [sum 2*n16] replay's counters when they exceed smem
  uint32_t* srcs;              // [sum n]
  uint32_t* cidx;              // [sum n] scratch: counter slot per op
  uint32_t* xoff;              // [sum (n+1)] scratch: expanded list offsets
  uint8_t* spl;                // [sum n] scratch: spliced virtual op marks
  const uint32_t* pred1;       // [sum n] a predecessor of each op (delta batches), or null
  unsigned long long* r_off;   // per candidate offset into rec (in records)
  unsigned long long* e_off;   // per candidate offset into erec (in edges)
  unsigned long long* c_off;   // per candidate byte offset into cnt0
  PackInfo* info;              // [B]
};

constexpr int kPackClusterSize = 1;  // == kPackCluster (below); chooses the gather loads

// Loads of data another CTA of the cluster may have written: through L2
// when the cluster spans SMs, else the normal (L1-cached) path.
template <typename T>
__device__ __forceinline__ T ld_shared_pass(const T* p) {
  if constexpr (kPackClusterSize > 1) return __ldcg(p);
  else return *p;
}

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

// Warp-cooperative list passes for candidates without nested splices: a
// warp takes 32 consecutive ops; their successor lists are one contiguous
// range of succ[], which the lanes stride over (coalesced reads, 32 gathers
// in flight, coalesced erec writes). src(k) comes from a shuffle binary
// search over the 33 list offsets held one per lane.
__device__ __forceinline__ uint32_t warp_src(uint32_t off_lane, uint32_t k) {
  uint32_t j = 0;
#pragma unroll
  for (uint32_t step = 16; step; step >>= 1) {
    const uint32_t v = __shfl_sync(kFull, off_lane, j + step);
    if (j + step < 32 && v <= k) j += step;
  }
  return j;
}

// Expanded list sizes of ops [i0, i1) into xoff (0 for spliced ops).
// Unrolled by 4 so four coalesced succ loads and four gathers are in
// flight per lane (the loop is latency-bound otherwise).
__device__ void coop_sizes(const Cand& c, const uint8_t* spl, uint32_t i0, uint32_t i1,
                           uint32_t* xoff, uint32_t* wlen) {
  constexpr int U = 4;
  const uint32_t lane = threadIdx.x & 31;
  wlen[lane] = 0;
  const uint32_t me = min(i0 + lane, i1);
  const uint32_t off = c.succ_off[me];
  const bool mysp = i0 + lane < i1 && spl[i0 + lane];
  const uint32_t spmask = __ballot_sync(kFull, mysp);
  const uint32_t E0 = __shfl_sync(kFull, off, 0), E1 = c.succ_off[i1];
  __syncwarp();
  for (uint32_t kb = E0; kb < E1; kb += 32 * U) {
    uint32_t sv[U], src[U];
    bool live[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = kb + 32 * u + lane;
      src[u] = warp_src(off, k);
      live[u] = k < E1 && !((spmask >> src[u]) & 1u);
      sv[u] = live[u] ? c.succ[k] : 0u;
    }
    uint32_t sp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) sp[u] = live[u] ? ld_shared_pass(spl + sv[u]) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (live[u])
        atomicAdd(&wlen[src[u]], sp[u] ? 1u + c.succ_off[sv[u] + 1] - c.succ_off[sv[u]] : 1u);
  }
  __syncwarp();
  if (i0 + lane < i1) xoff[i0 + lane] = mysp ? 0u : wlen[lane];
  __syncwarp();
}

// Expanded lists of ops [i0, i1) into erec (records gathered from rec);
// unrolled by 2 with all loads of both halves issued first.
__device__ void coop_lists(const Cand& c, const uint8_t* spl, uint32_t i0, uint32_t i1,
                           const uint32_t* xoff, const uint4* rec, uint4* erec, uint32_t* segp) {
#ifndef DPRO_LIST_U
#define DPRO_LIST_U 2
#endif
  constexpr int U = DPRO_LIST_U;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t me = min(i0 + lane, i1);
  const uint32_t off = c.succ_off[me];
  const uint32_t xo = i0 + lane < i1 ? xoff[i0 + lane] : 0u;
  const bool mysp = i0 + lane < i1 && spl[i0 + lane];
  const uint32_t spmask = __ballot_sync(kFull, mysp);
  const uint32_t E0 = __shfl_sync(kFull, off, 0), E1 = c.succ_off[i1];
  uint32_t carry = 0;  // splice extras of earlier edges of this chunk
  for (uint32_t kb = E0; kb < E1; kb += 32 * U) {
    uint32_t s[U], src[U];
    bool live[U], sv[U];
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = kb + 32 * u + lane;
      src[u] = warp_src(off, k);
      live[u] = k < E1 && !((spmask >> src[u]) & 1u);
      s[u] = live[u] ? c.succ[k] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) sv[u] = live[u] && ld_shared_pass(spl + s[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      r[u] = (live[u] && !sv[u]) ? ld_shared_pass(rec + s[u]) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = kb + 32 * u + lane;
      const uint32_t o_src = __shfl_sync(kFull, off, src[u]);
      const uint32_t x_src = __shfl_sync(kFull, xo, src[u]);
      uint32_t sa = 0, sz = 0;
      if (sv[u]) {
        sa = c.succ_off[s[u]];
        sz = c.succ_off[s[u] + 1];
      }
      const uint32_t ex = sz - sa;
      uint32_t incl = ex;  // inclusive warp scan of the extras
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, d);
        if ((int)lane >= d) incl += y;
      }
      const uint32_t P = carry + incl - ex;
      if (live[u] && k == o_src) segp[src[u]] = P;
      __syncwarp();
      if (live[u]) {
        uint32_t pos = x_src + (k - o_src) + (P - segp[src[u]]);
        if (sv[u]) {
          __stcs(erec + pos, make_uint4(s[u] & kOpMask, 0u, kFVirt, 0u));
          for (uint32_t t = sa; t < sz; ++t) __stcs(erec + (++pos), ld_shared_pass(rec + c.succ[t]));
        } else {
          __stcs(erec + pos, r[u]);
        }
      }
      carry += __shfl_sync(kFull, incl, 31);
      __syncwarp();
    }
  }
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

// One candidate per thread-block CLUSTER of kPackCluster CTAs (1024 threads
// each, one per SM). Larger clusters keep fewer candidates in flight so their
// CSR, scratch and records stay in L2 across the passes, but on config 2
// (1,024 candidates, B200) the lost memory-level parallelism costs more:
// cluster 1: 2.49 ms, 2: 3.09 ms, 4: 4.38 ms (33 co-resident clusters), so
// kPackCluster = 1 (one candidate per SM). Rank r owns op chunks
// [C*r/R, C*(r+1)/R) (chunks of 32 ops); per-candidate counters live in rank
// 0's shared memory (DSMEM atomics); cluster barriers separate the passes,
// and records written by other SMs are read through L2 (__ldcg). indeg must
// be present (host upload / delta merge) or computed by count_indeg_kernel.
constexpr int kPackCluster = kPackClusterSize;

__global__ void __cluster_dims__(kPackCluster, 1, 1) __launch_bounds__(kPackThreads, 1)
    pack_kernel(const Cand* __restrict__ cands, int c0, int n_cands, Scratch S, PackOut P) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  using Scan = cub::BlockScan<uint32_t, kPackThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  struct Ctr {  // per-candidate counters, used in rank 0's copy
    unsigned long long sum;
    uint32_t first, flags, ncnt, nsrc, nested;
    uint32_t tot[kPackCluster];
    uint32_t hist[kPackHist];
  };
  __shared__ Ctr s_ctr;
  __shared__ uint32_t s_carry, s_len;
  __shared__ uint32_t s_warp[kPackThreads];  // per-warp 32-word scratch
  __shared__ uint32_t s_lhist[kPackHist];    // this CTA's device counts
  const uint32_t rank = cluster.block_rank();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* wbuf = s_warp + 32 * warp;
  Ctr* R0 = cluster.map_shared_rank(&s_ctr, 0);
  const int n_clusters = gridDim.x / kPackCluster;
  for (int cid = c0 + blockIdx.x / kPackCluster; cid < n_cands; cid += n_clusters) {
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
    uint32_t* devoff = S.devoff + c.dof_off;
    const uint32_t n_chunks = (n + 31) / 32;
    const uint32_t ch_lo = n_chunks * rank / kPackCluster;
    const uint32_t ch_hi = n_chunks * (rank + 1) / kPackCluster;
    const uint32_t lo = min(n, ch_lo * 32), hi = min(n, ch_hi * 32);
    const bool hist_smem = c.d <= kPackHist;
    if (rank == 0) {
      if (threadIdx.x == 0) {
        s_ctr.first = kNone;
        s_ctr.flags = (n >= kMaxOps ? kNfSize : 0u) | (c.d > kMaxDev ? kNfDev : 0u);
        s_ctr.ncnt = 0;
        s_ctr.nsrc = 0;
        s_ctr.sum = 0;
        s_ctr.nested = 0;
      }
      for (uint32_t d = threadIdx.x; d < kPackHist; d += kPackThreads) s_ctr.hist[d] = 0;
      if (!hist_smem)
        for (uint32_t d = threadIdx.x; d <= c.d; d += kPackThreads) devoff[d] = 0;
    }
    if (threadIdx.x == 0) s_len = 0;
    if (hist_smem)
      for (uint32_t d = threadIdx.x; d < c.d; d += kPackThreads) s_lhist[d] = 0;
    cluster.sync();
    // pass 1 (coalesced): checks, counter slots and sources (warp-aggregated),
    // splice marks, per-device op counts
    uint32_t flags = 0, first = kNone;
    unsigned long long sum = 0;
    for (uint32_t i = lo + threadIdx.x; i < ((hi + 31) & ~31u) && lo < hi;
         i += kPackThreads) {
      const bool ok = i < hi;
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
        if (ind >= 255u) flags |= kWideCnt;
        if (ind >= 65535u) flags |= kNfIndeg;
        if (virt && ind == 0u) flags |= kNfVsrc;
        if (!virt && dv >= c.d) flags |= kNfDev;
        spl[i] = virt && ind == 1u;
        if (!virt && dv < c.d) atomicAdd(hist_smem ? &s_lhist[dv] : &devoff[dv], 1u);
      }
      const bool multi = ok && ind >= 2u, src = ok && ind == 0u;
      const unsigned mm = __ballot_sync(kFull, multi), ms = __ballot_sync(kFull, src);
      uint32_t bm = 0, bs = 0;
      if (lane == 0) {
        if (mm) bm = atomicAdd(&R0->ncnt, __popc(mm));
        if (ms) bs = atomicAdd(&R0->nsrc, __popc(ms));
      }
      bm = __shfl_sync(kFull, bm, 0);
      bs = __shfl_sync(kFull, bs, 0);
      const unsigned lt = (1u << lane) - 1u;
      if (multi) {
        const uint32_t slot = bm + __popc(mm & lt);
        cidx[i] = slot;  // cnt0[slot] is written in pass 3a (u8 or u16)
      } else if (src) {
        srcs[bs + __popc(ms & lt)] = i;
      }
    }
    if (first != kNone) atomicMin(&R0->first, first);
    if (flags) atomicOr(&R0->flags, flags);
    if (sum) atomicAdd(&R0->sum, sum);
    __syncthreads();
    if (hist_smem)
      for (uint32_t d = threadIdx.x; d < c.d; d += kPackThreads)
        if (s_lhist[d]) atomicAdd(&R0->hist[d], s_lhist[d]);
    cluster.sync();  // spl complete
    // nested splices (a spliced op with a spliced successor) take the
    // per-thread DFS walk; otherwise the warp-cooperative passes
    for (uint32_t i = lo + threadIdx.x; i < hi; i += kPackThreads)
      if (spl[i])
        for (uint32_t t = c.succ_off[i]; t < c.succ_off[i + 1]; ++t)
          if (__ldcg(spl + c.succ[t])) atomicOr(&R0->nested, 1u);
    cluster.sync();
    const bool nested = R0->nested != 0;
    // pass 2: expanded list sizes (spliced virtual ops own no list)
    if (nested) {
      bool deep = false;
      uint32_t part = 0;
      for (uint32_t i = lo + threadIdx.x; i < hi; i += kPackThreads) {
        uint32_t len = 0;
        if (!spl[i]) deep |= !walk_list(i, c, spl, [&](uint32_t, bool) { ++len; });
        xoff[i] = len;
        part += len;
      }
      if (deep) atomicOr(&R0->flags, kNfChain);
      if (part) atomicAdd(&s_len, part);
    } else if (P.pred1) {
      // out-degrees, then each spliced op adds its list to its single
      // predecessor's (O(V) + O(spliced) instead of a pass over the edges)
      const uint32_t* p1 = P.pred1 + c.op_off;
      for (uint32_t i = lo + threadIdx.x; i < hi; i += kPackThreads)
        xoff[i] = spl[i] ? 0u : c.succ_off[i + 1] - c.succ_off[i];
      cluster.sync();
      for (uint32_t i = lo + threadIdx.x; i < hi; i += kPackThreads)
        if (spl[i]) atomicAdd(&xoff[p1[i]], c.succ_off[i + 1] - c.succ_off[i]);
      cluster.sync();
      uint32_t part = 0;
      for (uint32_t i = lo + threadIdx.x; i < hi; i += kPackThreads) part += __ldcg(xoff + i);
      if (part) atomicAdd(&s_len, part);
    } else {
      uint32_t part = 0;
      for (uint32_t ch = ch_lo + warp; ch < ch_hi; ch += kPackThreads / 32) {
        coop_sizes(c, spl, ch * 32, min(n, ch * 32 + 32), xoff, wbuf);
        if (ch * 32 + lane < n) part += xoff[ch * 32 + lane];
      }
      if (part) atomicAdd(&s_len, part);
    }
    __syncthreads();
    if (threadIdx.x == 0) R0->tot[rank] = s_len;
    cluster.sync();
    // exclusive scan of xoff over the cluster: local scan + lower ranks' totals
    uint32_t base = 0, total = 0;
    for (uint32_t r = 0; r < kPackCluster; ++r) {
      const uint32_t t = R0->tot[r];
      if (r < rank) base += t;
      total += t;
    }
    if (threadIdx.x == 0) s_carry = base;
    __syncthreads();
    for (uint32_t b0 = lo; b0 < hi; b0 += kPackThreads) {
      const uint32_t i = b0 + threadIdx.x;
      const uint32_t v = i < hi ? xoff[i] : 0u;
      uint32_t excl, tsum;
      Scan(scan_tmp).ExclusiveSum(v, excl, tsum);
      const uint32_t carry = s_carry;
      if (i < hi) xoff[i] = carry + excl;
      __syncthreads();
      if (threadIdx.x == 0) s_carry = carry + tsum;
      __syncthreads();
    }
    if (rank == kPackCluster - 1 && threadIdx.x == 0) xoff[n] = total;
    cluster.sync();  // xoff complete (rec[i] reads xoff[i + 1] across ranks)
    // pass 3a (coalesced): every op's record, and the counter of every
    // multi-predecessor op (u16 when some in-degree exceeds a byte)
    const bool wide = (R0->flags & kWideCnt) != 0;
    for (uint32_t i = lo + threadIdx.x; i < hi; i += kPackThreads) {
      const uint32_t f = c.flags[i];
      const uint32_t ind = indeg[i];
      const bool virt = f & 1u;
      const uint32_t ci = ind >= 2 ? cidx[i] : 0u;
      if (ind >= 2 && ci < kMaxCnt) {
        if (wide) reinterpret_cast<uint16_t*>(cnt0)[ci] = static_cast<uint16_t>(min(ind, 65535u));
        else cnt0[ci] = static_cast<uint8_t>(ind);
      }
      const uint32_t x0 = xoff[i], x1 = __ldcg(xoff + i + 1);
      const uint32_t cnt = min(x1 - x0, kCntMax);
      const uint32_t z = (uint32_t(c.dev[i]) & kDevMask) | (virt ? kFVirt : 0u) |
                         (ind >= 2 ? kFMulti : 0u) | (cnt << kCntShift) | ((ci >> 8) << 18);
      const long long du = virt ? 0 : ld_dur(c, i);
      rec[i] = make_uint4((i & kOpMask) | ((ci & 0xFFu) << 24),
                          static_cast<uint32_t>(static_cast<int>(du)), z, x0);
    }
    if (rank == kPackCluster - 1 && threadIdx.x == 0) rec[n] = make_uint4(0u, 0u, 0u, total);
    cluster.sync();  // rec visible to the cluster
    // pass 3b: expanded lists = gathered records (stamps for spliced ops)
    if (nested) {
      for (uint32_t i = lo + threadIdx.x; i < hi; i += kPackThreads) {
        if (spl[i]) continue;
        uint4* dst = erec + xoff[i];
        walk_list(i, c, spl, [&](uint32_t s, bool sv) {
          __stcs(dst++, sv ? make_uint4(s & kOpMask, 0u, kFVirt, 0u) : __ldcg(rec + s));
        });
      }
    } else {
      for (uint32_t ch = ch_lo + warp; ch < ch_hi; ch += kPackThreads / 32)
        coop_lists(c, spl, ch * 32, min(n, ch * 32 + 32), xoff, rec, erec, wbuf);
    }
    // rank 0: info and timeline regions (exclusive scan of per-device counts)
    if (rank == 0) {
      if (threadIdx.x == 0) {
        PackInfo inf;
        inf.first_missing = s_ctr.first;
        // times are 64-bit in every kernel: only a single duration that
        // does not fit the record's int32 field leaves the fast path
        inf.not_fast = (s_ctr.flags & ~kWideCnt) | (s_ctr.ncnt >= kMaxCnt ? kNfSize : 0u);
        inf.wide = s_ctr.flags & kWideCnt;
        inf.pad = 0;
        inf.n_cnt = s_ctr.ncnt;
        inf.n_src = s_ctr.nsrc;
        inf.dur_sum = s_ctr.sum;
        P.info[cid] = inf;
      }
      if (hist_smem)
        for (uint32_t d = threadIdx.x; d < c.d; d += kPackThreads) devoff[d] = s_ctr.hist[d];
      __syncthreads();
      const uint32_t dtot = block_exclusive_scan<kPackThreads, Scan>(devoff, c.d, scan_tmp, s_carry);
      if (threadIdx.x == 0) devoff[c.d] = dtot;
    }
    cluster.sync();  // rank 0's counters are reset for the next candidate
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
