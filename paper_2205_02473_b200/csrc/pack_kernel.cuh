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
// successors, in order). emit(rec) per entry; returns false when a spliced
// chain is deeper than kMaxSplice.
template <bool kBuild, typename Emit>
__device__ bool expand_list(uint32_t i, const Cand& c, const uint32_t* indeg,
                            const uint32_t* cidx, const uint32_t* xoff, Emit&& emit) {
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
    if (spliced(c, indeg, s)) {
      emit(make_uint4(s & kOpMask, 0u, kFVirt, 0u));  // stamp: virtual, not multi
      if (sp + 1 >= kMaxSplice) return false;
      ++sp;
      stk_op[sp] = s;
      stk_k[sp] = c.succ_off[s];
    } else {
      emit(kBuild ? make_rec(s, c, indeg, cidx, xoff) : make_uint4(0, 0, 0, 0));
    }
  }
}

// One block per candidate (grid-stride). indeg must be present (host upload
// computes it; device batches without it go through count_indeg_kernel).
__global__ void __launch_bounds__(256) pack_kernel(const Cand* __restrict__ cands,
                                                   int n_cands, Scratch S,
                                                   PackOut P) {
  __shared__ uint32_t s_first, s_flags, s_ncnt, s_nsrc;
  __shared__ unsigned long long s_sum;
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const Cand c = cands[cid];
    const uint32_t n = c.n;
    const uint32_t* indeg = c.indeg ? c.indeg : S.indeg + c.op_off;
    uint4* rec = P.rec + P.r_off[cid];
    uint4* erec = P.erec + P.e_off[cid];
    uint8_t* cnt0 = P.cnt0 + P.c_off[cid];
    uint32_t* srcs = P.srcs + c.op_off;
    uint32_t* cidx = P.cidx + c.op_off;
    if (threadIdx.x == 0) {
      s_first = kNone;
      s_flags = (n >= kMaxOps ? kNfSize : 0u) | (c.d > kMaxDev ? kNfDev : 0u);
      s_ncnt = 0;
      s_nsrc = 0;
      s_sum = 0;
    }
    __syncthreads();
    uint32_t flags = 0, first = kNone;
    unsigned long long sum = 0;
    // pass 1: counter slots, sources, checks
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const long long du = ld_dur(c, i);
      const bool virt = c.flags[i] & 1u;
      const uint32_t ind = indeg[i];
      if (!virt && du < 0) first = min(first, i);
      if (!virt && (du > 0x7FFFFFFFLL || du < -0x80000000LL)) flags |= kNfDur;
      if (!virt && du > 0) sum += static_cast<unsigned long long>(du);
      if (ind >= 255u) flags |= kNfIndeg;
      if (virt && ind == 0u) flags |= kNfVsrc;
      if (!virt && c.dev[i] >= c.d) flags |= kNfDev;
      if (ind >= 2u) {
        const uint32_t slot = atomicAdd(&s_ncnt, 1u);
        cidx[i] = slot;
        if (slot < kMaxCnt) cnt0[slot] = static_cast<uint8_t>(min(ind, 255u));
      } else if (ind == 0u) {
        srcs[atomicAdd(&s_nsrc, 1u)] = i;
      }
    }
    if (first != kNone) atomicMin(&s_first, first);
    if (flags) atomicOr(&s_flags, flags);
    if (sum) atomicAdd(&s_sum, sum);
    __syncthreads();
    // pass 2: expanded list sizes (spliced virtual ops own no list)
    uint32_t* xoff = P.xoff + P.r_off[cid];
    bool deep = false;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      uint32_t len = 0;
      if (!spliced(c, indeg, i))
        deep |= !expand_list<false>(i, c, indeg, cidx, xoff, [&](const uint4&) { ++len; });
      xoff[i] = len;
    }
    if (deep) atomicOr(&s_flags, kNfChain);
    __syncthreads();
    // exclusive scan of xoff[0..n) (chunked block scan), xoff[n] = total
    {
      __shared__ uint32_t s_part[256];
      const uint32_t chunk = (n + blockDim.x - 1) / blockDim.x;
      const uint32_t lo = min(n, threadIdx.x * chunk), hi = min(n, lo + chunk);
      uint32_t sum = 0;
      for (uint32_t i = lo; i < hi; ++i) sum += xoff[i];
      s_part[threadIdx.x] = sum;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t t = 0; t < blockDim.x; ++t) {
          const uint32_t v = s_part[t];
          s_part[t] = run;
          run += v;
        }
        xoff[n] = run;
      }
      __syncthreads();
      uint32_t run = s_part[threadIdx.x];
      for (uint32_t i = lo; i < hi; ++i) {
        const uint32_t v = xoff[i];
        xoff[i] = run;
        run += v;
      }
    }
    __syncthreads();
    // pass 3: records and expanded lists
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      rec[i] = make_rec(i, c, indeg, cidx, xoff);
      if (!spliced(c, indeg, i)) {
        uint4* dst = erec + xoff[i];
        expand_list<true>(i, c, indeg, cidx, xoff, [&](const uint4& r) { *dst++ = r; });
      }
    }
    if (threadIdx.x == 0) {
      rec[n] = make_uint4(0u, 0u, 0u, xoff[n]);
      PackInfo inf;
      inf.first_missing = s_first;
      inf.not_fast = s_flags | (s_sum >= 0x7FFFFFFFull ? kNfDur : 0u) |
                     (s_ncnt >= kMaxCnt ? kNfSize : 0u);
      inf.n_cnt = s_ncnt;
      inf.n_src = s_nsrc;
      inf.dur_sum = s_sum;
      P.info[cid] = inf;
    }
    // timeline regions: per-device non-virtual op counts, exclusive scan
    uint32_t* devoff = S.devoff + c.dof_off;
    for (uint32_t d = threadIdx.x; d <= c.d; d += blockDim.x) devoff[d] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
      if (!(c.flags[i] & 1u) && c.dev[i] < c.d) atomicAdd(&devoff[c.dev[i]], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      for (uint32_t d = 0; d < c.d; ++d) {
        const uint32_t v = devoff[d];
        devoff[d] = run;
        run += v;
      }
      devoff[c.d] = run;
    }
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
