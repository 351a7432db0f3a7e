// K1 fast path: exact batched replay with all mutable state on chip.
//
// Same round semantics as replay_kernel.cuh (proj/src/replay.cpp:37-134);
// what changes is where the state lives and what an event round touches.
//   * one warp per candidate; lane l owns devices d = l + 32 j (j < KD); the
//     in-flight end time of each owned device lives in a lane register, so
//     the next event time is one REDUX.MIN over the warp (32-bit times: the
//     pack pass proves sum(dur) < 2^31, hence every time fits);
//   * a round only visits devices that completed or received arrivals
//     (per-lane dirty bitmask in shared memory, set by producers);
//   * per-device FIFOs are shared-memory rings of 16-byte entries
//     {op, dur, succ_beg, succ_end}, sorted by (ready, index) on arrival;
//   * in-degree countdowns exist only for ops with >= 2 predecessors, as
//     compact u8 counters in shared memory (4 per word, word atomics);
//   * the completing op's 16-byte edge records (pack_kernel.cuh) are loaded
//     when the op is dispatched -- into registers for the in-flight
//     positive-duration op of each owned device, into a per-lane cp.async
//     stage for zero-duration ops (which complete next round) -- so the
//     completion itself rarely waits on memory.
// Whatever the fast path cannot represent (ring or worklist overflow, a
// virtual source -> init quirk, indeg >= 255, durations that need 64-bit
// times, too many devices / counters, a cycle) falls back inside the same
// launch to the general kernel (replay_candidate, global state): every
// candidate's result is exact either way.
#pragma once

#include "pack_kernel.cuh"
#include "replay_kernel.cuh"

namespace dpro_k {

constexpr uint32_t kT32Inf = 0xFFFFFFFFu;

struct __align__(16) DevF {
  uint32_t head, tail, tsort, segbeg;
  uint32_t zlo, zhi, segt, busy;
  uint4 ient;  // in-flight positive-duration op {op, dur, sb, se}
};
static_assert(sizeof(DevF) == 48, "DevF layout");

struct FastCfg {
  uint32_t dcap;   // devices per warp
  uint32_t ccap;   // compact counters per warp (bytes, multiple of 16)
  uint32_t qc;     // ring capacity per device (power of two)
  uint32_t vs;     // virtual worklist capacity
  uint32_t warp_bytes;
  uint32_t kd;     // devices per lane (template parameter)
};

#ifndef DPRO_KSTAGE
#define DPRO_KSTAGE 1
#endif
constexpr int kStage = DPRO_KSTAGE;  // edge records staged in registers per in-flight op
constexpr int kZStage = 4;  // zero-duration ops staged per lane per round

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__host__ __device__ constexpr size_t fast_misc_words() { return 4 + 32; }

template <int KD>
struct FastWarp {
  const uint4* __restrict__ rec;
  const uint4* __restrict__ erec;
  DevF* dv;
  uint4* q;                 // [dcap][qc]
  uint4* vstk;              // [vs]
  uint4* zst;               // [32][kZStage] zero-op staging (cp.async)
  volatile uint32_t* misc;  // [0] vtop [1] overflow [4..35] dirty masks
  uint32_t* cw;             // compact counters (u8 in words)
  uint32_t qc, vs;
  uint32_t* qbuf;
  uint32_t* qpos;
  const uint32_t* devoff;
  long long* start;
  long long* end;
  bool want;
  int lane;
  uint32_t vcount = 0, dcount = 0, tmax = 0, zn = 0;

  __device__ __forceinline__ uint4* ring(uint32_t d) { return q + (size_t)d * qc; }

  // ready(s, t) of replay.cpp:60-72 for s reached through a packed record.
  __device__ __forceinline__ void ready(const uint4& a, uint32_t t) {
    const uint32_t s = a.x & kOpMask;
    const uint32_t cnt = (a.z >> kCntShift) & kCntMax;
    const uint32_t se = cnt == kCntMax ? __ldg(&rec[s + 1].w) : a.w + cnt;
    const uint4 e = make_uint4(s, a.y, a.w, se);  // {op, dur, sb, se}
    if (a.z & kFVirt) {
      if (want) {
        start[s] = t;
        end[s] = t;
      }
      ++vcount;
      tmax = max(tmax, t);
      const uint32_t p = atomicAdd(const_cast<uint32_t*>(&misc[0]), 1u);
      if (p < vs)
        vstk[p] = e;
      else
        misc[1] = 1u;
    } else {
      const uint32_t d = a.z & kDevMask;
      DevF& sd = dv[d];
      const uint32_t pos = atomicAdd(&sd.tail, 1u);
      const uint32_t zl = *reinterpret_cast<volatile uint32_t*>(&sd.zlo);
      const uint32_t zh = *reinterpret_cast<volatile uint32_t*>(&sd.zhi);
      const uint32_t low = zl < zh ? zl : *reinterpret_cast<volatile uint32_t*>(&sd.head);
      if (pos - low >= qc) {
        misc[1] = 1u;
      } else {
        ring(d)[pos & (qc - 1)] = e;
        atomicOr(const_cast<uint32_t*>(&misc[4 + (d & 31)]), 1u << (d >> 5));
      }
    }
    if (se > a.w) prefetch_l2(erec + a.w);
  }

  __device__ __forceinline__ void edge(const uint4& a, uint32_t t) {
    if ((a.z & (kFVirt | kFMulti)) == kFVirt) {  // spliced single-pred virtual
      const uint32_t s = a.x & kOpMask;
      if (want) {
        start[s] = t;
        end[s] = t;
      }
      ++vcount;
      tmax = max(tmax, t);
      return;  // its successors follow in this same list
    }
    if (a.z & kFMulti) {
      const uint32_t ci = (a.x >> 24) | ((a.z >> 18) << 8);
      const uint32_t sh = 8u * (ci & 3u);
      const uint32_t old = atomicSub(&cw[ci >> 2], 1u << sh);
      if (((old >> sh) & 0xFFu) != 1u) return;
    }
    ready(a, t);
  }

  // Completion of e at t (replay.cpp:100-103); the first kStage records were
  // loaded into `st` when e was dispatched.
  __device__ __forceinline__ void complete_staged(const uint4& e, const uint4 (&st)[kStage],
                                                  uint32_t t) {
    const uint32_t n = e.w - e.z;
#pragma unroll
    for (int f = 0; f < kStage; ++f)
      if (f < n) edge(st[f], t);
    for (uint32_t k = e.z + kStage; k < e.w; ++k) edge(__ldg(erec + k), t);
  }

  __device__ __forceinline__ void complete(const uint4& e, uint32_t t) {
    for (uint32_t k = e.z; k < e.w; ++k) edge(__ldg(erec + k), t);
  }

  __device__ void drain_virtual(uint32_t t) {
    __syncwarp();
    for (;;) {
      const uint32_t n = misc[0];
      if (n == 0 || misc[1]) break;
      const uint32_t k = n < 32 ? n : 32;
      uint4 item = make_uint4(kNone, 0, 0, 0);
      if ((uint32_t)lane < k) item = vstk[n - 1 - lane];
      __syncwarp();
      if (lane == 0) misc[0] = n - k;
      __syncwarp();
      if (item.x != kNone) complete(item, t);
      __syncwarp();
    }
  }

  // Owner-lane dispatch(t) for device d (replay.cpp:74-90) after merging
  // this round's arrivals into the (ready, index)-ordered tail segment.
  // Returns the in-flight end (kT32Inf: idle); loads the in-flight op's first
  // edge records into `st`; stages the first record of zero-duration ops
  // (they complete next round) with cp.async; sets *zero when any ran.
  __device__ __forceinline__ uint32_t dispatch_dev(uint32_t d, uint32_t t, uint32_t iend,
                                                   uint4 (&st)[kStage], bool* zero) {
    DevF& s = dv[d];
    uint4* r = ring(d);
    const uint32_t tail = *reinterpret_cast<volatile uint32_t*>(&s.tail);
    const uint32_t m = qc - 1;
    uint32_t head = s.head;
    if (tail != s.tsort) {
      if (s.segt != t) {
        s.segbeg = s.tsort;
        s.segt = t;
      }
      const uint32_t lo = max(s.segbeg, head);
      for (uint32_t p = s.tsort; p < tail; ++p) {
        const uint4 x = r[p & m];
        uint32_t qq = p;
        while (qq > lo) {
          const uint4 y = r[(qq - 1) & m];
          if (y.x < x.x) break;
          r[qq & m] = y;
          --qq;
        }
        r[qq & m] = x;
      }
      s.tsort = tail;
    }
    if (iend == kT32Inf && head < tail) {
      const uint32_t zlo = head;
      uint32_t busy = 0;
      const uint32_t base = devoff[d];
      bool infl = false;
      while (head < tail) {
        const uint4 x = r[head & m];
        const uint32_t en = t + x.y;
        if (want) {
          start[x.x] = t;
          end[x.x] = en;
          qpos[x.x] = base + head;
        }
        qbuf[base + head] = x.x;
        ++head;
        ++dcount;
        busy += x.y;
        tmax = max(tmax, en);
        if (x.y > 0) {
          s.ient = x;
          iend = en;
          infl = true;
#pragma unroll
          for (int f = 0; f < kStage; ++f)
            if (x.z + f < x.w) st[f] = __ldg(erec + x.z + f);
          if (x.w > x.z + kStage) prefetch_l2(erec + x.z + kStage);
          break;
        }
        if (x.w > x.z && zn < kZStage) cp_async16(zst + lane * kZStage + zn++, erec + x.z);
      }
      s.busy += busy;
      s.head = head;
      s.zlo = zlo;
      const uint32_t zhi = infl ? head - 1 : head;
      s.zhi = zhi;
      if (zlo < zhi) *zero = true;
    }
    return iend;
  }
};

// Returns false when the candidate must take the general path.
template <int KD>
__device__ bool replay_fast(const Cand& c, int cid, const uint4* rec, const uint4* erec,
                            const uint8_t* cnt0, const uint32_t* srcs, const PackInfo& info,
                            unsigned char* wsm, const FastCfg& F, const Scratch& S,
                            const Outs& O, bool want_schedule) {
  const int lane = threadIdx.x & 31;
  const uint32_t n = c.n, D = c.d;
  DevF* dv = reinterpret_cast<DevF*>(wsm);
  uint4* q = reinterpret_cast<uint4*>(wsm + sizeof(DevF) * F.dcap);
  uint4* vstk = q + (size_t)F.dcap * F.qc;
  uint4* zst = vstk + F.vs;
  volatile uint32_t* misc = reinterpret_cast<volatile uint32_t*>(zst + 32 * kZStage);
  uint32_t* cw = const_cast<uint32_t*>(misc) + fast_misc_words();
  const unsigned long long oo = c.op_off;

  FastWarp<KD> W{rec, erec, dv, q, vstk, zst, misc, cw, F.qc, F.vs, S.qbuf + oo, S.qpos + oo,
                 S.devoff + c.dof_off,
                 want_schedule ? O.start + oo : nullptr,
                 want_schedule ? O.end + oo : nullptr, want_schedule, lane};

  // ---- state init ----
  {
    const uint32_t nv = (info.n_cnt + 15) / 16;
    const uint4* src = reinterpret_cast<const uint4*>(cnt0);
    uint4* dst = reinterpret_cast<uint4*>(cw);
    for (uint32_t i = lane; i < nv; i += 32) dst[i] = __ldg(src + i);
  }
  for (uint32_t d = lane; d < D; d += 32) {
    DevF z;
    z.head = z.tail = z.tsort = z.segbeg = 0;
    z.zlo = z.zhi = z.segt = z.busy = 0;
    z.ient = make_uint4(0, 0, 0, 0);
    dv[d] = z;
  }
  if (lane < 4) misc[lane] = 0;
  misc[4 + lane] = 0;
  __syncwarp();
  // ---- sources (replay.cpp:92-94). No virtual sources reach the fast path
  // (pack flags them), so there are no cascades and no init quirk. ----
  for (uint32_t k = lane; k < info.n_src; k += 32) W.ready(__ldg(rec + __ldg(srcs + k)), 0u);
  __syncwarp();
  if (__any_sync(kFull, misc[1] != 0)) return false;
  for (uint32_t d = lane; d < D; d += 32) {  // t = 0 arrivals in index order
    DevF& s = dv[d];
    uint4* r = W.ring(d);
    const uint32_t m = F.qc - 1;
    for (uint32_t p = 1; p < s.tail; ++p) {
      const uint4 x = r[p & m];
      uint32_t qq = p;
      while (qq > 0 && r[(qq - 1) & m].x > x.x) {
        r[qq & m] = r[(qq - 1) & m];
        --qq;
      }
      r[qq & m] = x;
    }
    s.tsort = s.tail;
  }
  __syncwarp();

  // ---- dispatch(0) + event loop (replay.cpp:95-106) ----
  uint32_t iend[KD];
  uint4 stg[KD][kStage];
  uint32_t zmask = 0;
#pragma unroll
  for (int j = 0; j < KD; ++j) {
    iend[j] = kT32Inf;
#pragma unroll
    for (int f = 0; f < kStage; ++f) stg[j][f] = make_uint4(0, 0, 0, 0);
    const uint32_t d = lane + 32 * j;
    if (d < D) {
      bool z = false;
      iend[j] = W.dispatch_dev(d, 0u, kT32Inf, stg[j], &z);
      if (z) zmask |= 1u << j;
    }
  }
  cp_async_commit();
  misc[4 + lane] = 0;  // all devices were just visited
  uint32_t t = 0;
  for (;;) {
    const bool zero_round = __any_sync(kFull, zmask != 0);
    uint32_t freed = 0;
    if (zero_round) {
      // zero-duration ops dispatched last round complete now (same t); their
      // first edge records were staged by cp.async in that dispatch
      cp_async_wait_all();
      uint32_t zi = 0;
      uint32_t zm = zmask;
      while (zm) {
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        const uint32_t d = lane + 32 * j;
        DevF& s = dv[d];
        const uint4* r = W.ring(d);
        const uint32_t zh = s.zhi;
        for (uint32_t p = s.zlo; p < zh; ++p) {
          const uint4 e = r[p & (F.qc - 1)];
          if (e.w > e.z) {
            uint32_t k = e.z;
            if (zi < kZStage) {
              W.edge(zst[lane * kZStage + zi++], t);
              ++k;
            }
            for (; k < e.w; ++k) W.edge(__ldg(erec + k), t);
          }
        }
        *reinterpret_cast<volatile uint32_t*>(&s.zlo) = zh;
      }
      zmask = 0;
    } else {
      uint32_t lmin = kT32Inf;
#pragma unroll
      for (int j = 0; j < KD; ++j) lmin = min(lmin, iend[j]);
      const uint32_t tn = __reduce_min_sync(kFull, lmin);
      if (tn == kT32Inf) break;
      t = tn;
#pragma unroll
      for (int j = 0; j < KD; ++j) {
        if (iend[j] == t) {
          iend[j] = kT32Inf;
          freed |= 1u << j;
          W.complete_staged(dv[lane + 32 * j].ient, stg[j], t);
        }
      }
    }
    W.drain_virtual(t);
    __syncwarp();
    if (__any_sync(kFull, misc[1] != 0)) return false;
    const uint32_t todo = freed | misc[4 + lane];
    misc[4 + lane] = 0;
    W.zn = 0;
#pragma unroll
    for (int j = 0; j < KD; ++j) {
      if (todo & (1u << j)) {
        bool z = false;
        iend[j] = W.dispatch_dev(lane + 32 * j, t, iend[j], stg[j], &z);
        if (z) zmask |= 1u << j;
      }
    }
    cp_async_commit();
  }
  cp_async_wait_all();

  const uint32_t vc = __reduce_add_sync(kFull, W.vcount);
  const uint32_t dc = __reduce_add_sync(kFull, W.dcount);
  if (vc + dc != n) return false;  // cycle: the general path reports it exactly
  const uint32_t T = __reduce_max_sync(kFull, W.tmax);
  for (uint32_t d = lane; d < D; d += 32) {
    S.busy[c.dev_off + d] = dv[d].busy;
    S.dhead[c.dev_off + d] = W.devoff[d] + dv[d].head;
  }
  if (lane == 0) {
    O.status[cid] = kOk;
    O.err[cid] = 0;
    O.makespan[cid] = T;
  }
  return true;
}

template <int KD>
#ifndef DPRO_MINB
#define DPRO_MINB 8
#endif
__global__ void __launch_bounds__(32, DPRO_MINB) replay_fast_kernel(
    const Cand* __restrict__ cands, int n_cands, Scratch S, Outs O, PackOut P,
    FastCfg F, int want_schedule, unsigned* work, unsigned* fallbacks) {
  extern __shared__ __align__(16) unsigned char fsm[];
  for (;;) {
    int cid = 0;
    if (threadIdx.x == 0) cid = static_cast<int>(atomicAdd(work, 1u));
    cid = __shfl_sync(kFull, cid, 0);
    if (cid >= n_cands) break;
    const Cand c = cands[cid];
    const PackInfo info = P.info[cid];
    if (info.first_missing != kNone) {  // replay.cpp:39-44
      if (threadIdx.x == 0) {
        O.status[cid] = kMissing;
        O.err[cid] = info.first_missing;
        O.makespan[cid] = 0;
      }
      continue;
    }
    bool done = false;
    if (info.not_fast == 0 && c.d <= F.dcap && c.d <= 32u * KD && info.n_cnt <= F.ccap)
      done = replay_fast<KD>(c, cid, P.rec + P.r_off[cid], P.erec + P.e_off[cid],
                             P.cnt0 + P.c_off[cid], P.srcs + c.op_off, info, fsm, F, S, O,
                             want_schedule != 0);
    __syncwarp();
    if (!done) {
      if (threadIdx.x == 0) atomicAdd(fallbacks, 1u);
      volatile uint32_t* vtop = reinterpret_cast<volatile uint32_t*>(fsm);
      replay_candidate(c, cid, S.dstate + c.dev_off, vtop, S, O, want_schedule != 0);
    }
    __syncwarp();
  }
}

}  // namespace dpro_k
