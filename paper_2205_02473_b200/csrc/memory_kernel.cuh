// K5: batched peak-memory estimate on the replayed schedule (no transfer).
//
// estimate_peak_memory (proj/src/memory.cpp:122-167) for every candidate of
// a replayed batch: per compute node, every computation op with an output
// buffer allocates at its start and frees when its last computation
// consumer ends (at its own end without one); peak = persistent bytes + the
// maximum running sum of the node's (time, delta) events, frees before
// allocations at equal times. Here: events are written to per-(candidate,
// node) segments (key = time << 1 | is_alloc, value = delta), the segments
// are sorted with CUB's segmented radix sort, and one warp per segment
// scans them. Ordering within one key is irrelevant: at a given time all
// frees precede all allocations, and the running maximum over a run of
// allocations is reached at its end.
#pragma once

#include "replay_kernel.cuh"

namespace dpro_k {

struct MemIn {
  const long long* bytes;            // [sum n] output buffer bytes (0: none)
  const int* node;                   // [sum n] dense compute node, -1 otherwise
  const unsigned long long* seg0;    // [B] first segment of each candidate
  unsigned int* seg_cnt;             // [S] events per segment
  unsigned long long* seg_off;       // [S+1] exclusive offsets
  unsigned long long* cursor;        // [S]
  unsigned long long* keys;          // [events]
  long long* vals;                   // [events]
};

__global__ void mem_count_kernel(const Cand* __restrict__ cands, int n_cands, MemIn M) {
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const Cand c = cands[cid];
    const unsigned long long oo = c.op_off;
    for (uint32_t i = threadIdx.x; i < c.n; i += blockDim.x) {
      const int nd = M.node[oo + i];
      if (nd >= 0 && M.bytes[oo + i] > 0) atomicAdd(&M.seg_cnt[M.seg0[cid] + nd], 2u);
    }
  }
}

__global__ void mem_fill_kernel(const Cand* __restrict__ cands, int n_cands, Outs O, MemIn M) {
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const Cand c = cands[cid];
    const unsigned long long oo = c.op_off;
    for (uint32_t i = threadIdx.x; i < c.n; i += blockDim.x) {
      const int nd = M.node[oo + i];
      const long long b = M.bytes[oo + i];
      if (nd < 0 || b <= 0) continue;
      long long freed = O.end[oo + i];
      for (uint32_t k = c.succ_off[i]; k < c.succ_off[i + 1]; ++k) {
        const uint32_t s = c.succ[k];
        if (M.node[oo + s] >= 0) freed = max(freed, O.end[oo + s]);  // computation consumer
      }
      const unsigned long long seg = M.seg0[cid] + nd;
      const unsigned long long p = atomicAdd(&M.cursor[seg], 2ull);
      M.keys[p] = (static_cast<unsigned long long>(O.start[oo + i]) << 1) | 1ull;
      M.vals[p] = b;
      M.keys[p + 1] = static_cast<unsigned long long>(freed) << 1;
      M.vals[p + 1] = -b;
    }
  }
}

// One warp per segment: running sum in sorted order, maximum.
__global__ void mem_scan_kernel(unsigned long long n_segs, const unsigned long long* seg_off,
                                const long long* vals, const long long* persistent,
                                long long* peak) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned long long w = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nw = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  for (unsigned long long s = w; s < n_segs; s += nw) {
    const unsigned long long a = seg_off[s], z = seg_off[s + 1];
    long long run = 0, best = 0;
    for (unsigned long long base = a; base < z; base += 32) {
      const unsigned long long i = base + lane;
      const long long v = i < z ? vals[i] : 0;
      long long x = v;  // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(kFull, x, o);
        if ((int)lane >= o) x += y;
      }
      long long m = i < z ? run + x : run;
#pragma unroll
      for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
      best = max(best, m);
      run += __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) peak[s] = persistent[s] + best;
  }
}

}  // namespace dpro_k
