// Pack: caller CSR (SoA, index order) -> the engine's replay layout.
//
// Runs once when a batch is registered (engine.cu). Per candidate:
//   rec[i]  = {dur_i, devflags_i, succ_beg_i, succ_end_i}         (uint4)
//   erec[k] = {s, dur_s, devflags_s, succ_beg_s} for edge k: i->s  (uint4)
//   cnt0[i] = min(indeg_i, 255)                                    (u8)
//   devoff  = exclusive scan of non-virtual ops per device (timeline regions)
//   info    = first op without duration, eligibility for the fast path.
// The per-edge record carries everything the replay needs when the edge's
// completion makes s ready (its device, virtual flag, duration and successor
// range), so an event round touches one 16-byte record per edge instead of
// five dependent SoA loads (proj/src/replay.cpp:60-72,80-87 read kind,
// device, dur and succ of s at exactly that moment).
#pragma once

#include "replay_kernel.cuh"

namespace dpro_k {

constexpr uint32_t kDevMask = 0xFFFFu;
constexpr uint32_t kFVirt = 1u << 16;
constexpr uint32_t kFComm = 1u << 17;
constexpr uint32_t kFMulti = 1u << 18;   // indeg >= 2: counted in smem
constexpr uint32_t kCntShift = 20;       // successor count; kCntMax: see rec
constexpr uint32_t kCntMax = 4095u;

struct PackInfo {
  uint32_t first_missing;  // kNone: every non-virtual op has dur >= 0
  uint32_t not_fast;       // bit0 dur>int32, bit1 indeg>=255, bit2 virtual
                           // source, bit3 bad device id
  uint32_t max_indeg;
  uint32_t pad;
};

struct PackOut {
  uint4* rec;                  // [sum n]
  uint4* erec;                 // [sum e]
  uint8_t* cnt0;               // [sum n16] (each candidate 16-byte aligned)
  unsigned long long* e_off;   // per candidate offset into erec
  unsigned long long* c_off;   // per candidate offset into cnt0
  PackInfo* info;              // [B]
};

__device__ __forceinline__ uint32_t devflags_of(const Cand& c, uint32_t i,
                                                uint32_t indeg) {
  const uint32_t f = c.flags[i];
  const uint32_t cnt = c.succ_off[i + 1] - c.succ_off[i];
  return (uint32_t(c.dev[i]) & kDevMask) | ((f & 1u) ? kFVirt : 0u) |
         ((f & 2u) ? kFComm : 0u) | (indeg >= 2 ? kFMulti : 0u) |
         (min(cnt, kCntMax) << kCntShift);
}

// One block per candidate (grid-stride). indeg must be present (the host
// upload computes it when the caller passes NULL; device batches without
// indeg are counted into S.indeg first by count_indeg_kernel).
__global__ void __launch_bounds__(256) pack_kernel(const Cand* __restrict__ cands,
                                                   int n_cands, Scratch S,
                                                   PackOut P) {
  __shared__ uint32_t s_first, s_flags, s_max;
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const Cand c = cands[cid];
    const uint32_t n = c.n;
    const uint32_t* indeg = c.indeg ? c.indeg : S.indeg + c.op_off;
    uint4* rec = P.rec + c.op_off;
    uint4* erec = P.erec + P.e_off[cid];
    uint8_t* cnt0 = P.cnt0 + P.c_off[cid];
    if (threadIdx.x == 0) {
      s_first = kNone;
      s_flags = 0;
      s_max = 0;
    }
    __syncthreads();
    uint32_t flags = 0, mx = 0, first = kNone;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const long long du = ld_dur(c, i);
      const uint32_t f = c.flags[i];
      const uint32_t ind = indeg[i];
      const bool virt = f & 1u;
      if (!virt && du < 0) first = min(first, i);
      if (du > 0x7FFFFFFFLL || du < -0x80000000LL) flags |= 1u;
      if (ind >= 255u) flags |= 2u;
      if (virt && ind == 0u) flags |= 4u;
      if (!virt && c.dev[i] >= c.d) flags |= 8u;
      mx = max(mx, ind);
      const uint32_t df = devflags_of(c, i, ind);
      rec[i] = make_uint4(static_cast<uint32_t>(static_cast<int>(du)), df,
                          c.succ_off[i], c.succ_off[i + 1]);
      cnt0[i] = static_cast<uint8_t>(min(ind, 255u));
      for (uint32_t k = c.succ_off[i]; k < c.succ_off[i + 1]; ++k) {
        const uint32_t s = c.succ[k];
        erec[k] = make_uint4(s, static_cast<uint32_t>(static_cast<int>(ld_dur(c, s))),
                             devflags_of(c, s, indeg[s]), c.succ_off[s]);
      }
    }
    if (first != kNone) atomicMin(&s_first, first);
    if (flags) atomicOr(&s_flags, flags);
    if (mx) atomicMax(&s_max, mx);
    __syncthreads();
    if (threadIdx.x == 0) {
      P.info[cid].first_missing = s_first;
      P.info[cid].not_fast = s_flags;
      P.info[cid].max_indeg = s_max;
      P.info[cid].pad = 0;
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
