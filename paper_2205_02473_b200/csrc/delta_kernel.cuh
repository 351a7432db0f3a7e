// K0: merge of per-candidate deltas with the resident base graph into the
// index-ordered CSR the pack/replay kernels read (dpro_delta,
// include/dpro_cuda.h). One CTA per candidate; the base arrays are shared by
// every candidate, so after the first CTAs touch them they are served from
// L2. Rank queries are O(1): a removed-op bitmap with per-word prefix
// counts (r) and per-word counts of insertion points (q), built by the CTA
// in its own scratch slice.
//
//   kept base op b  -> f = b - r(b) + q(b),  r(b) = #removed < b,
//                                            q(b) = #new_pos <= b
//   new op j        -> f = new_pos[j] - r(new_pos[j]) + j
// Successors of a kept base op: its base successors that are kept and not
// cut (mapped, ascending because the map is monotone) merged with its
// ascending extra edges; of a new op: its given list.
#pragma once

#include <cub/block/block_scan.cuh>

#include "replay_kernel.cuh"

namespace dpro_k {

struct ResDev {
  const void* dur;  // int32 or int64 (dur64)
  const uint16_t* dev;
  const uint8_t* flags;
  const uint32_t* succ_off;
  const uint32_t* succ;
  uint32_t n, dur64;
};

struct DeltaDev {
  const uint32_t* removed;
  const uint32_t* new_pos;
  const long long* new_dur;
  const uint16_t* new_dev;
  const uint8_t* new_flags;
  const uint32_t* new_succ_off;
  const uint32_t* new_succ;
  const uint32_t* extra_src;
  const uint32_t* extra_dst;
  const uint32_t* cut;
  uint32_t n_removed, n_new, n_extra, n_cut;
  unsigned long long rank_off;  // words into the rank scratch (3W+1 rank words, nb map)
};

constexpr int kMergeThreads = 1024;
constexpr uint32_t kMergeIndegSmem = 49152;  // ops whose in-degrees fit in smem

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct Ranks {
  const uint32_t* bits;  // [W] removed bitmap
  const uint32_t* rpre;  // [W] #removed in earlier words
  const uint32_t* qpre;  // [W+1] #new_pos < 32*w
  const uint32_t* new_pos;
  uint32_t n_removed, n_new, nb;
  __device__ __forceinline__ bool removed(uint32_t b) const {
    return (bits[b >> 5] >> (b & 31)) & 1u;
  }
  __device__ __forceinline__ uint32_t r(uint32_t b) const {  // #removed < b
    if (b >= nb) return n_removed;
    return rpre[b >> 5] + __popc(bits[b >> 5] & ((1u << (b & 31)) - 1u));
  }
  __device__ __forceinline__ uint32_t q(uint32_t b) const {  // #new_pos <= b
    const uint32_t w = b >> 5;
    uint32_t k = qpre[w];
    const uint32_t z = qpre[w + 1];
    while (k < z && __ldg(new_pos + k) <= b) ++k;
    return k;
  }
  __device__ __forceinline__ uint32_t f(uint32_t b) const { return b - r(b) + q(b); }
};

__device__ __forceinline__ bool is_cut(const DeltaDev& D, uint32_t e) {
  if (D.n_cut == 0) return false;
  const uint32_t k = lower_bound_u32(D.cut, D.n_cut, e);
  return k < D.n_cut && __ldg(D.cut + k) == e;
}

// Also writes each candidate's in-degrees (C.indeg), counted in shared
// memory (dynamic smem of smem_ind words; larger candidates count in HBM).
__global__ void __launch_bounds__(kMergeThreads, 1)
    delta_merge_kernel(ResDev B, const DeltaDev* __restrict__ deltas, const Cand* __restrict__ cands,
                       int n_cands, uint32_t* __restrict__ rank_scratch, uint32_t smem_ind,
                       uint32_t* __restrict__ pred1, uint32_t rank_smem) {
  using Scan = cub::BlockScan<uint32_t, kMergeThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t s_carry;
  extern __shared__ uint32_t s_ind[];
  const uint32_t nb = B.n, W = (nb >> 5) + 1;
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const DeltaDev D = deltas[cid];
    const Cand C = cands[cid];
    // rank structures in shared memory after the in-degree counters when
    // they fit (rank_smem), else in this candidate's global scratch
    uint32_t* bits = rank_smem ? s_ind + smem_ind : rank_scratch + D.rank_off;
    uint32_t* rpre = bits + W;
    uint32_t* qpre = rpre + W;
    // ---- rank structures
    for (uint32_t w = threadIdx.x; w < W; w += blockDim.x) bits[w] = 0;
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < D.n_removed; k += blockDim.x) {
      const uint32_t b = __ldg(D.removed + k);
      atomicOr(&bits[b >> 5], 1u << (b & 31));
    }
    for (uint32_t w = threadIdx.x; w <= W; w += blockDim.x) {
      qpre[w] = lower_bound_u32(D.new_pos, D.n_new, w << 5);
      if (w < W) rpre[w] = lower_bound_u32(D.removed, D.n_removed, w << 5);
    }
    __syncthreads();
    const Ranks R{bits, rpre, qpre, D.new_pos, D.n_removed, D.n_new, nb};
    // final index of every base op (removed ones: UINT32_MAX)
    // final index of base op b (UINT32_MAX: removed): from the shared-memory
    // ranks directly, or through a map in global scratch when they are global
    uint32_t* fmap = rank_scratch + D.rank_off + 3 * W + 1;
    if (!rank_smem) {
      for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
        fmap[b] = R.removed(b) ? UINT32_MAX : R.f(b);
      __syncthreads();
    }
    auto fm = [&](uint32_t b) -> uint32_t {
      if (!rank_smem) return fmap[b];
      return R.removed(b) ? UINT32_MAX : R.f(b);
    };
    uint32_t* ind_g = const_cast<uint32_t*>(C.indeg);
    const bool ind_smem = C.n <= smem_ind;
    uint32_t* ind = ind_smem ? s_ind : ind_g;
    for (uint32_t i = threadIdx.x; i < C.n; i += blockDim.x) ind[i] = 0;
    uint32_t* off = const_cast<uint32_t*>(C.succ_off);
    uint32_t* p1 = pred1 + C.op_off;  // a predecessor of every op (exact when indeg is 1)
    uint32_t* succ = const_cast<uint32_t*>(C.succ);
    uint16_t* dev = const_cast<uint16_t*>(C.dev);
    uint8_t* flags = const_cast<uint8_t*>(C.flags);
    // ---- per-op fields and out-degrees (written at off[f + 1])
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
      const uint32_t f = fm(b);
      if (f == UINT32_MAX) continue;
      const long long d = B.dur64 ? __ldg(static_cast<const long long*>(B.dur) + b)
                                  : (long long)__ldg(static_cast<const int*>(B.dur) + b);
      if (C.dur64) static_cast<long long*>(const_cast<void*>(C.dur))[f] = d;
      else static_cast<int*>(const_cast<void*>(C.dur))[f] = (int)d;
      dev[f] = __ldg(B.dev + b);
      flags[f] = __ldg(B.flags + b);
      uint32_t deg = 0;
      const uint32_t e1 = __ldg(B.succ_off + b + 1);
      for (uint32_t e = __ldg(B.succ_off + b); e < e1; ++e)
        deg += !R.removed(__ldg(B.succ + e)) && !is_cut(D, e);
      if (D.n_extra) {
        const uint32_t x0 = lower_bound_u32(D.extra_src, D.n_extra, b);
        uint32_t x1 = x0;
        while (x1 < D.n_extra && __ldg(D.extra_src + x1) == b) ++x1;
        deg += x1 - x0;
      }
      off[f + 1] = deg;
    }
    for (uint32_t j = threadIdx.x; j < D.n_new; j += blockDim.x) {
      const uint32_t p = __ldg(D.new_pos + j);
      const uint32_t f = p - R.r(p) + j;
      const long long d = __ldg(D.new_dur + j);
      if (C.dur64) static_cast<long long*>(const_cast<void*>(C.dur))[f] = d;
      else static_cast<int*>(const_cast<void*>(C.dur))[f] = (int)d;
      dev[f] = __ldg(D.new_dev + j);
      flags[f] = __ldg(D.new_flags + j);
      off[f + 1] = __ldg(D.new_succ_off + j + 1) - __ldg(D.new_succ_off + j);
    }
    if (threadIdx.x == 0) {
      off[0] = 0;
      s_carry = 0;
    }
    __syncthreads();
    // ---- in-place inclusive scan of off[1..n]
    for (uint32_t base = 0; base < C.n; base += blockDim.x) {
      const uint32_t i = base + threadIdx.x;
      const uint32_t v = i < C.n ? off[i + 1] : 0u;
      uint32_t incl, total;
      Scan(scan_tmp).InclusiveSum(v, incl, total);
      const uint32_t carry = s_carry;
      if (i < C.n) off[i + 1] = carry + incl;
      __syncthreads();
      if (threadIdx.x == 0) s_carry = carry + total;
      __syncthreads();
    }
    // ---- successor lists
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
      const uint32_t fb = fm(b);
      if (fb == UINT32_MAX) continue;
      uint32_t o = off[fb];
      uint32_t e = __ldg(B.succ_off + b);
      const uint32_t e1 = __ldg(B.succ_off + b + 1);
      uint32_t x = 0, x1 = 0;
      if (D.n_extra) {
        x = lower_bound_u32(D.extra_src, D.n_extra, b);
        x1 = x;
        while (x1 < D.n_extra && __ldg(D.extra_src + x1) == b) ++x1;
      }
      uint32_t nxt = UINT32_MAX;  // next mapped kept base successor
      auto advance = [&]() {
        nxt = UINT32_MAX;
        for (; e < e1; ++e) {
          const uint32_t m = fm(__ldg(B.succ + e));
          if (m != UINT32_MAX && !is_cut(D, e)) {
            nxt = m;
            ++e;
            break;
          }
        }
      };
      advance();
      while (nxt != UINT32_MAX || x < x1) {
        const uint32_t xv = x < x1 ? __ldg(D.extra_dst + x) : UINT32_MAX;
        if (nxt <= xv) {  // extras never repeat a kept base edge (dpro_delta)
          succ[o++] = nxt;
          atomicAdd(&ind[nxt], 1u);
          p1[nxt] = fb;
          advance();
        } else {
          succ[o++] = xv;
          atomicAdd(&ind[xv], 1u);
          p1[xv] = fb;
          ++x;
        }
      }
    }
    for (uint32_t j = threadIdx.x; j < D.n_new; j += blockDim.x) {
      const uint32_t p = __ldg(D.new_pos + j);
      const uint32_t fj = p - R.r(p) + j;
      uint32_t o = off[fj];
      for (uint32_t k = __ldg(D.new_succ_off + j); k < __ldg(D.new_succ_off + j + 1); ++k) {
        const uint32_t t = __ldg(D.new_succ + k);
        succ[o++] = t;
        atomicAdd(&ind[t], 1u);
        p1[t] = fj;
      }
    }
    __syncthreads();
    if (ind_smem)
      for (uint32_t i = threadIdx.x; i < C.n; i += blockDim.x) ind_g[i] = s_ind[i];
    __syncthreads();
  }
}

}  // namespace dpro_k
