// K3: critical path on the execution graph, one warp per candidate.
//
// critical_path(execution_graph(g, r), r) of proj/src/replay.cpp:136-226
// without materializing the execution graph: its edges are the DFG edges
// plus, per device, timeline[k-1] -> timeline[k] (replay.cpp:136-144); the
// timelines are K1's queue regions (qbuf), so an op's timeline neighbours
// are qbuf[qpos-1] / qbuf[qpos+1] inside its device region.
//   1. tight-edge backward closure from every op with end == T (166-185),
//      over a predecessor CSR built here by transposing succ;
//   2. start: smallest-index good op with start == 0 (187-193);
//   3. walk: smallest-index good tight successor until end == T (194-209).
#pragma once

#include "replay_kernel.cuh"

namespace dpro_k {

struct CpScratch {
  uint32_t* pred_off;  // [sum (n+1)]
  uint32_t* pred;      // [sum e]
  uint32_t* good;      // [sum n]
  uint32_t* stack;     // [sum n]
  unsigned long long* e_off;    // per candidate offset into pred (host-built)
  unsigned long long* po_off;   // per candidate offset into pred_off
};

__device__ __forceinline__ uint32_t tl_prev(uint32_t v, const Cand& c,
                                            const uint32_t* qbuf,
                                            const uint32_t* qpos,
                                            const uint32_t* devoff) {
  if (c.flags[v] & 1u) return kNone;
  const uint32_t q = qpos[v];
  if (q == kNone) return kNone;
  return q > devoff[c.dev[v]] ? qbuf[q - 1] : kNone;
}
__device__ __forceinline__ uint32_t tl_next(uint32_t v, const Cand& c,
                                            const uint32_t* qbuf,
                                            const uint32_t* qpos,
                                            const uint32_t* dhead) {
  if (c.flags[v] & 1u) return kNone;
  const uint32_t q = qpos[v];
  if (q == kNone) return kNone;
  return q + 1 < dhead[c.dev[v]] ? qbuf[q + 1] : kNone;
}

// qpos (an op's position in its device timeline) from the timelines in qbuf,
// for the candidates K3 walks: the fast replay kernels write only qbuf.
__global__ void __launch_bounds__(256) qpos_scatter_kernel(const Cand* __restrict__ cands,
                                                           int n_cands, Scratch S, Outs O) {
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    if (O.status[cid] != kOk) continue;
    const Cand c = cands[cid];
    const uint32_t* qbuf = S.qbuf + c.op_off;
    uint32_t* qpos = S.qpos + c.op_off;
    const uint32_t total = S.devoff[c.dof_off + c.d];  // every non-virtual op ran
    for (uint32_t p = threadIdx.x; p < total; p += blockDim.x) qpos[qbuf[p]] = p;
  }
}

__global__ void __launch_bounds__(128) critical_path_kernel(
    const Cand* __restrict__ cands, int n_cands, Scratch S, Outs O,
    CpScratch P, uint32_t* paths, long long* path_len) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int cid = gw; cid < n_cands; cid += nw) {
    const Cand c = cands[cid];
    const uint32_t n = c.n;
    const unsigned long long oo = c.op_off;
    if (O.status[cid] != kOk || n == 0) {
      if (lane == 0) path_len[cid] = 0;
      continue;
    }
    const long long T = O.makespan[cid];
    const long long* st = O.start + oo;
    const long long* en = O.end + oo;
    const uint32_t* qbuf = S.qbuf + oo;
    const uint32_t* qpos = S.qpos + oo;
    const uint32_t* devoff = S.devoff + c.dof_off;
    const uint32_t* dhead = S.dhead + c.dev_off;
    uint32_t* poff = P.pred_off + P.po_off[cid];
    uint32_t* pred = P.pred + P.e_off[cid];
    uint32_t* good = P.good + oo;
    uint32_t* stack = P.stack + oo;
    uint32_t* cursor = S.indeg + oo;  // indeg scratch is free after replay

    // predecessor CSR: counts, exclusive scan, fill
    for (uint32_t i = lane; i < n; i += 32) cursor[i] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32)
      for (uint32_t k = c.succ_off[i]; k < c.succ_off[i + 1]; ++k)
        atomicAdd(&cursor[c.succ[k]], 1u);
    __syncwarp();
    uint32_t running = 0;
    for (uint32_t b = 0; b < n; b += 32) {
      const uint32_t i = b + lane;
      const uint32_t v = i < n ? __ldcg(&cursor[i]) : 0;
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (i < n) {
        poff[i] = running + x - v;
        cursor[i] = running + x - v;
      }
      running += __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) poff[n] = running;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32)
      for (uint32_t k = c.succ_off[i]; k < c.succ_off[i + 1]; ++k)
        pred[atomicAdd(&cursor[c.succ[k]], 1u)] = i;

    // 1. backward closure (worklist; order-free)
    __shared__ uint32_t tops[4];
    volatile uint32_t* top = tops + ((threadIdx.x >> 5) & 3);
    if (lane == 0) *top = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) {
      const bool g = en[i] == T;
      good[i] = g ? 1u : 0u;
      if (g) stack[atomicAdd(const_cast<uint32_t*>(top), 1u)] = i;
    }
    __syncwarp();
    for (;;) {
      const uint32_t cnt = *top;
      if (cnt == 0) break;
      const uint32_t k = cnt < 32 ? cnt : 32;
      const uint32_t v = (uint32_t)lane < k ? stack[cnt - 1 - lane] : kNone;
      __syncwarp();
      if (lane == 0) *top = cnt - k;
      __syncwarp();
      if (v != kNone) {
        const long long sv = st[v];
        const uint32_t pb = poff[v], pe = poff[v + 1];
        for (uint32_t e = pb; e <= pe; ++e) {
          const uint32_t p = e < pe ? pred[e] : tl_prev(v, c, qbuf, qpos, devoff);
          if (p == kNone) continue;
          if (en[p] == sv && atomicExch(&good[p], 1u) == 0u)
            stack[atomicAdd(const_cast<uint32_t*>(top), 1u)] = p;
        }
      }
      __syncwarp();
    }
    // 2. start op
    uint32_t cur = kNone;
    for (uint32_t b = 0; b < n && cur == kNone; b += 32) {
      const uint32_t i = b + lane;
      const bool ok = i < n && __ldcg(&good[i]) && st[i] == 0;
      const unsigned m = __ballot_sync(kFull, ok);
      if (m) cur = b + __ffs(m) - 1;
    }
    // 3. forward walk
    long long len = 0;
    uint32_t* path = paths + oo;
    while (cur != kNone) {
      if (lane == 0) path[len] = cur;
      ++len;
      const long long ec = en[cur];
      if (ec == T) break;
      const uint32_t sb = c.succ_off[cur], se = c.succ_off[cur + 1];
      uint32_t best = kNone;
      for (uint32_t e = sb + lane; e < se + 32; e += 32) {
        uint32_t s = kNone;
        if (e < se)
          s = c.succ[e];
        else if (e == se)
          s = tl_next(cur, c, qbuf, qpos, dhead);
        if (s != kNone && __ldcg(&good[s]) && st[s] == ec) best = min(best, s);
        if (e >= se) break;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
      cur = best;
    }
    if (lane == 0) path_len[cid] = len;
  }
}

}  // namespace dpro_k
