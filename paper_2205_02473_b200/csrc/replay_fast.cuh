// K1 fast path: exact batched replay with all mutable state on chip.
//
// Same round semantics as replay_kernel.cuh (and proj/src/replay.cpp:37-134);
// what changes is where the state lives and what an event round touches:
//   * per-candidate in-degree countdowns: u8 in shared memory (4 per 32-bit
//     word, decremented with word atomics); ops with a single predecessor
//     skip the counter entirely (devflags kFMulti);
//   * per-device queues: shared-memory rings of QC 16-byte records (the
//     packed successor record of pack_kernel.cuh), so dispatch reads the
//     duration and the successor range from the queue entry itself;
//   * device state: shared memory, lane-owned (device d -> lane d % 32);
//   * the one global read left in a round is the completing op's edge
//     records, prefetched to L2 when the op is enqueued and dispatched.
// Anything the fast path cannot represent (a ring overflow, a virtual source
// -> init quirk, indeg >= 255, int64 durations, more devices or ops than the
// shared-memory budget, a cycle) falls back, inside the same launch, to the
// general kernel (replay_candidate, global-memory state), so every
// candidate's result is exact.
#pragma once

#include "pack_kernel.cuh"
#include "replay_kernel.cuh"

namespace dpro_k {

struct __align__(16) DevF {
  uint32_t head, tail, tsort, segbeg;
  uint32_t zlo, zhi, iop, pad;
  long long iend, segt, busy, pad2;
  uint4 ient;
};
static_assert(sizeof(DevF) == 80, "DevF layout");

struct FastCfg {
  uint32_t dcap;     // devices per warp
  uint32_t vcap;     // ops per warp (u8 counters), multiple of 16
  uint32_t qc;       // ring capacity per device (power of two)
  uint32_t vs;       // virtual worklist capacity
  uint32_t warp_bytes;
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

struct FastWarp {
  const Cand& c;
  const uint4* __restrict__ rec;
  const uint4* __restrict__ erec;
  DevF* dv;
  uint4* q;            // [dcap][qc]
  uint4* vstk;         // [vs]
  uint32_t* cnt32;     // u8 counters packed in words
  volatile uint32_t* misc;  // [0] vtop, [1] overflow
  uint32_t qc, vs;
  uint32_t* qbuf;
  uint32_t* qpos;
  const uint32_t* devoff;
  long long* start;
  long long* end;
  bool want;
  unsigned long long vcount = 0, dcount = 0;
  long long tmax = 0;

  __device__ __forceinline__ uint4* ring(uint32_t d) { return q + (size_t)d * qc; }

  __device__ __forceinline__ void ready(const uint4& x, long long t) {
    prefetch_l2(erec + x.w);  // its completion reads these edge records
    if (x.z & kFVirt) {
      if (want) {
        start[x.x] = t;
        end[x.x] = t;
      }
      ++vcount;
      tmax = max(tmax, t);
      const uint32_t p = atomicAdd(const_cast<uint32_t*>(&misc[0]), 1u);
      if (p < vs)
        vstk[p] = x;
      else
        misc[1] = 1u;
    } else {
      const uint32_t d = x.z & kDevMask;
      DevF& s = dv[d];
      const uint32_t pos = atomicAdd(&s.tail, 1u);
      const uint32_t zl = *reinterpret_cast<volatile uint32_t*>(&s.zlo);
      const uint32_t zh = *reinterpret_cast<volatile uint32_t*>(&s.zhi);
      const uint32_t low = zl < zh ? zl : s.head;
      if (pos - low >= qc)
        misc[1] = 1u;
      else
        ring(d)[pos & (qc - 1)] = x;
    }
  }

  __device__ __forceinline__ void complete(const uint4& e, long long t) {
    const uint32_t sb = e.w;
    const uint32_t cnt = e.z >> kCntShift;
    const uint32_t se = cnt == kCntMax ? __ldg(&rec[e.x].w) : sb + cnt;
    for (uint32_t k = sb; k < se; ++k) {
      const uint4 x = __ldg(erec + k);
      if (x.z & kFMulti) {
        const uint32_t sh = 8u * (x.x & 3u);
        const uint32_t old = atomicSub(&cnt32[x.x >> 2], 1u << sh);
        if (((old >> sh) & 0xFFu) != 1u) continue;
      }
      ready(x, t);
    }
  }

  __device__ void drain_virtual(long long t, int lane) {
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

  __device__ __forceinline__ void dispatch_dev(uint32_t d, long long t,
                                               long long& lane_min, bool& lane_zero) {
    DevF& s = dv[d];
    uint4* r = ring(d);
    const uint32_t tail = *reinterpret_cast<volatile uint32_t*>(&s.tail);
    const uint32_t m = qc - 1;
    if (tail != s.tsort) {
      if (s.segt != t) {
        s.segbeg = s.tsort;
        s.segt = t;
      }
      const uint32_t lo = max(s.segbeg, s.head);
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
    if (s.iop == kNone && s.head < tail) {
      const uint32_t zlo = s.head;
      uint32_t h = s.head;
      long long busy = 0;
      const uint32_t base = devoff[d];
      bool infl = false;
      while (h < tail) {
        const uint4 x = r[h & m];
        const long long du = static_cast<int>(x.y);
        const long long en = t + du;
        if (want) {
          start[x.x] = t;
          end[x.x] = en;
          qpos[x.x] = base + h;
        }
        qbuf[base + h] = x.x;
        ++h;
        ++dcount;
        busy += du;
        tmax = max(tmax, en);
        prefetch_l2(erec + x.w);
        if (du > 0) {
          s.iop = x.x;
          s.iend = en;
          s.ient = x;
          infl = true;
          break;
        }
      }
      s.busy += busy;
      s.head = h;
      s.zlo = zlo;
      s.zhi = infl ? h - 1 : h;
    }
    if (s.iop != kNone) lane_min = min(lane_min, s.iend);
    if (s.zlo < s.zhi) lane_zero = true;
  }
};

// Returns false when the candidate must take the general path.
__device__ bool replay_fast(const Cand& c, int cid, const uint4* rec, const uint4* erec,
                            const uint8_t* cnt0, unsigned char* wsm, const FastCfg& F,
                            const Scratch& S, const Outs& O, bool want_schedule) {
  const int lane = threadIdx.x & 31;
  const uint32_t n = c.n, D = c.d;
  DevF* dv = reinterpret_cast<DevF*>(wsm);
  uint4* q = reinterpret_cast<uint4*>(wsm + sizeof(DevF) * F.dcap);
  uint4* vstk = q + (size_t)F.dcap * F.qc;
  volatile uint32_t* misc = reinterpret_cast<volatile uint32_t*>(vstk + F.vs);
  uint32_t* cnt32 = const_cast<uint32_t*>(misc) + 4;
  const unsigned long long oo = c.op_off;

  FastWarp W{c, rec, erec, dv, q, vstk, cnt32, misc, F.qc, F.vs,
             S.qbuf + oo, S.qpos + oo, S.devoff + c.dof_off,
             want_schedule ? O.start + oo : nullptr, want_schedule ? O.end + oo : nullptr,
             want_schedule};

  // ---- state init: counters (16 B vector copies), devices ----
  {
    const uint32_t nv = (n + 15) / 16;
    const uint4* src = reinterpret_cast<const uint4*>(cnt0);
    uint4* dst = reinterpret_cast<uint4*>(cnt32);
    for (uint32_t i = lane; i < nv; i += 32) dst[i] = __ldg(src + i);
  }
  for (uint32_t d = lane; d < D; d += 32) {
    DevF z;
    z.head = z.tail = z.tsort = z.segbeg = 0;
    z.zlo = z.zhi = 0;
    z.iop = kNone;
    z.pad = 0;
    z.iend = 0;
    z.segt = 0;
    z.busy = 0;
    z.pad2 = 0;
    z.ient = make_uint4(0, 0, 0, 0);
    dv[d] = z;
  }
  if (lane == 0) {
    misc[0] = 0;
    misc[1] = 0;
  }
  __syncwarp();
  // ---- sources (replay.cpp:92-94): indeg-0 ops in index order. Virtual
  // sources never reach here (pack flags them), so there are no cascades and
  // no init quirk; arrivals at t=0 are sorted per device below. ----
  {
    const uint32_t nw = (n + 3) / 4;
    for (uint32_t w = lane; w < nw; w += 32) {
      const uint32_t v = cnt32[w];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t i = w * 4 + b;
        if (i < n && ((v >> (8 * b)) & 0xFFu) == 0u) {
          const uint4 r = __ldg(rec + i);
          W.ready(make_uint4(i, r.x, r.y, r.z), 0);
        }
      }
    }
  }
  __syncwarp();
  if (__any_sync(kFull, misc[1] != 0)) return false;
  for (uint32_t d = lane; d < D; d += 32) {  // sort the t=0 arrivals by index
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

  // ---- dispatch(0) + event loop ----
  long long lane_min = kTInf, t = 0;
  bool lane_zero = false;
  for (uint32_t d = lane; d < D; d += 32) W.dispatch_dev(d, 0, lane_min, lane_zero);
  for (;;) {
    const bool zero_round = __any_sync(kFull, lane_zero);
    if (!zero_round) {
      const long long tn = warp_min64(lane_min);
      if (tn == kTInf) break;
      t = tn;
    }
    for (uint32_t d = lane; d < D; d += 32) {
      DevF& s = dv[d];
      if (zero_round) {
        const uint4* r = W.ring(d);
        for (uint32_t p = s.zlo; p < s.zhi; ++p) W.complete(r[p & (F.qc - 1)], t);
        *reinterpret_cast<volatile uint32_t*>(&s.zlo) = s.zhi;
      } else if (s.iop != kNone && s.iend == t) {
        s.iop = kNone;
        W.complete(s.ient, t);
      }
    }
    W.drain_virtual(t, lane);
    __syncwarp();
    if (__any_sync(kFull, misc[1] != 0)) return false;
    lane_min = kTInf;
    lane_zero = false;
    for (uint32_t d = lane; d < D; d += 32) W.dispatch_dev(d, t, lane_min, lane_zero);
  }

  const unsigned long long vc = warp_sum64(W.vcount);
  const unsigned long long dc = warp_sum64(W.dcount);
  if (vc + dc != n) return false;  // cycle: the general path reports it exactly
  const long long T = warp_max64(W.tmax);
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

__global__ void __launch_bounds__(32) replay_fast_kernel(
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
    if (info.not_fast == 0 && c.d <= F.dcap && c.n <= F.vcap)
      done = replay_fast(c, cid, P.rec + c.op_off, P.erec + P.e_off[cid],
                         P.cnt0 + P.c_off[cid], fsm, F, S, O, want_schedule != 0);
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
