// K1: batched exact replay, one warp per candidate DFG (sm_100a).
//
// Semantics are those of dpro::replay (proj/src/replay.cpp:37-134), in the
// round-based form validated in SURVEY.md Appendix A ("twin"):
//   * per device a FIFO ordered by (ready time, op index); all entries made
//     ready in one round share the round's time t, so only the tail segment
//     with ready == t ever needs re-ordering (replay.cpp:28-33,76-79);
//   * a device runs at most one positive-duration op at a time; the next
//     event time is the min over in-flight ends (replay.cpp:96-98);
//   * zero-duration ops dispatched at t complete in the NEXT round at the same
//     t, after everything dispatched at t (replay.hpp:41-44);
//   * virtual ops complete the instant they are ready and cascade
//     (replay.cpp:60-72); the serial init scan re-tests indeg after earlier
//     cascades (replay.cpp:92-94, the init quirk of SURVEY Appendix A).
//
// Mapping: lane l owns devices d == l (mod 32); their state (queue
// head/tail, in-flight op, zero-range) lives in shared memory (global
// fallback for very wide graphs). The next event time is a warp min-reduce
// of per-lane minima. Successor decrements are global atomics on the
// candidate's indeg scratch; newly ready ops are appended to the owning
// device's queue region (sized by the device's op count, so it never
// overflows) and merged into the tail segment by the owner lane. The queue
// regions double as the device timelines (ReplayResult::device_timelines).
#pragma once

#include <cstdint>

namespace dpro_k {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr long long kTInf = 0x7FFFFFFFFFFFFFFFLL;
constexpr unsigned kFull = 0xFFFFFFFFu;

struct DevSt {
  uint32_t head, tail, tsort, segbeg;
  uint32_t infl, zlo, zhi, pad;
  long long infl_end, segt, busy;
};
static_assert(sizeof(DevSt) == 56, "DevSt layout");

// Per-candidate device descriptor (built by the host, engine.cu).
struct Cand {
  const void* dur;
  const uint16_t* dev;
  const uint8_t* flags;
  const uint32_t* succ_off;
  const uint32_t* succ;
  const uint32_t* indeg;  // may be null
  uint32_t n, e, d, dur64;
  unsigned long long op_off;   // into per-op arrays (outputs + scratch)
  unsigned long long dev_off;  // into per-device scratch (sum of d)
  unsigned long long dof_off;  // into device-offset scratch (sum of d+1)
};

struct Scratch {
  uint32_t* indeg;   // [sum n]
  uint32_t* qbuf;    // [sum n]  per-device dispatch queues == timelines
  uint32_t* qpos;    // [sum n]  position of an op in qbuf
  uint8_t* sched;    // [sum n]
  uint32_t* vstack;  // [sum n]  virtual-op worklist
  uint32_t* devoff;  // [sum (d+1)]
  DevSt* dstate;     // [sum d]  global fallback for device state
  long long* busy;   // [sum d]
  uint32_t* dhead;   // [sum d]  end of the dispatched prefix of each region
};

struct Outs {
  long long* makespan;  // [B]
  int* status;          // [B]
  long long* err;       // [B]
  long long* start;     // [sum n] (null: makespan only)
  long long* end;
};

enum { kOk = 0, kMissing = 1, kCycle = 2, kInval = 3 };

__device__ __forceinline__ long long ld_dur(const Cand& c, uint32_t i) {
  return c.dur64 ? reinterpret_cast<const long long*>(c.dur)[i]
                 : static_cast<long long>(reinterpret_cast<const int*>(c.dur)[i]);
}

__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ long long warp_max64(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

struct Replayer {
  const Cand& c;
  DevSt* ds;
  uint32_t* indeg;
  uint32_t* qbuf;
  uint32_t* qpos;
  uint8_t* sched;
  uint32_t* vstack;
  volatile uint32_t* vtop;  // per-warp shared counter
  long long* start;
  long long* end;
  int lane;
  bool want;
  // lane-local accumulators
  unsigned long long vcount = 0, dcount = 0;
  long long tmax = 0;

  __device__ __forceinline__ uint32_t tail_of(DevSt& s) {
    return *reinterpret_cast<volatile uint32_t*>(&s.tail);
  }

  // ready(s, t) of replay.cpp:60-72 for ops reached through a completion.
  __device__ __forceinline__ void ready(uint32_t s, long long t) {
    if (c.flags[s] & 1u) {
      if (want) {
        start[s] = t;
        end[s] = t;
      }
      sched[s] = 1;
      ++vcount;
      tmax = max(tmax, t);
      const uint32_t p = atomicAdd(const_cast<uint32_t*>(vtop), 1u);
      vstack[p] = s;
    } else {
      const uint32_t p = atomicAdd(&ds[c.dev[s]].tail, 1u);
      qbuf[p] = s;
    }
  }

  // Completion of op i at t: decrement successors (replay.cpp:100-103).
  __device__ __forceinline__ void complete(uint32_t i, long long t) {
    const uint32_t b = c.succ_off[i], e = c.succ_off[i + 1];
    for (uint32_t k = b; k < e; ++k) {
      const uint32_t s = c.succ[k];
      if (atomicSub(&indeg[s], 1u) == 1u) ready(s, t);
    }
  }

  // Drain the virtual worklist (cascades at the same t, same round).
  __device__ void drain_virtual(long long t) {
    __syncwarp();
    for (;;) {
      const uint32_t cnt = *vtop;
      if (cnt == 0) break;
      const uint32_t k = cnt < 32 ? cnt : 32;
      const uint32_t item = (uint32_t)lane < k ? vstack[cnt - 1 - lane] : kNone;
      __syncwarp();
      if (lane == 0) *vtop = cnt - k;
      __syncwarp();
      if (item != kNone) complete(item, t);
      __syncwarp();
    }
  }

  // Owner-lane dispatch(t) for device d (replay.cpp:74-90), after merging
  // this round's arrivals into the (ready, index)-ordered tail segment.
  __device__ __forceinline__ void dispatch_dev(uint32_t d, long long t,
                                               long long& lane_min,
                                               bool& lane_zero) {
    DevSt& s = ds[d];
    const uint32_t tail = tail_of(s);
    if (tail != s.tsort) {
      if (s.segt != t) {
        s.segbeg = s.tsort;
        s.segt = t;
      }
      const uint32_t lo = max(s.segbeg, s.head);
      for (uint32_t p = s.tsort; p < tail; ++p) {
        const uint32_t x = qbuf[p];
        uint32_t q = p;
        while (q > lo) {
          const uint32_t y = qbuf[q - 1];
          if (y < x) break;
          qbuf[q] = y;
          --q;
        }
        qbuf[q] = x;
      }
      s.tsort = tail;
    }
    if (s.infl == kNone && s.head < tail) {
      const uint32_t zlo = s.head;
      uint32_t h = s.head;
      long long busy = 0;
      while (h < tail) {
        const uint32_t i = qbuf[h];
        const long long du = ld_dur(c, i);
        if (want) {
          qpos[i] = h;
          start[i] = t;
          end[i] = t + du;
        }
        sched[i] = 1;
        ++h;
        ++dcount;
        busy += du;
        tmax = max(tmax, t + du);
        if (du > 0) {
          s.infl = i;
          s.infl_end = t + du;
          break;
        }
      }
      s.busy += busy;
      s.head = h;
      s.zlo = zlo;
      s.zhi = (s.infl != kNone) ? h - 1 : h;
    }
    if (s.infl != kNone) lane_min = min(lane_min, s.infl_end);
    if (s.zlo < s.zhi) lane_zero = true;
  }
};

// One candidate, whole warp. Returns nothing; writes outs[cid].
__device__ void replay_candidate(const Cand& c, int cid, DevSt* ds,
                                 volatile uint32_t* vtop, const Scratch& S,
                                 const Outs& O, bool want_schedule) {
  const int lane = threadIdx.x & 31;
  const uint32_t n = c.n, D = c.d;
  const unsigned long long oo = c.op_off;
  uint32_t* indeg = S.indeg + oo;
  uint32_t* qbuf = S.qbuf + oo;
  uint32_t* qpos = S.qpos + oo;
  uint8_t* sched = S.sched + oo;
  uint32_t* devoff = S.devoff + c.dof_off;
  long long* start = want_schedule ? O.start + oo : nullptr;
  long long* end = want_schedule ? O.end + oo : nullptr;

  // ---- device state + per-device op counts + missing-profile check ----
  for (uint32_t d = lane; d < D; d += 32) {
    DevSt z;
    z.head = z.tail = z.tsort = z.segbeg = 0;
    z.infl = kNone;
    z.zlo = z.zhi = 0;
    z.pad = 0;
    z.infl_end = 0;
    z.segt = -1;
    z.busy = 0;
    ds[d] = z;
  }
  if (lane == 0) *vtop = 0;
  __syncwarp();
  uint32_t first_bad = kNone;
  int bad_kind = kOk;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t i = base + lane;
    bool missing = false, inval = false;
    if (i < n && !(c.flags[i] & 1u)) {
      const uint32_t dv = c.dev[i];
      if (ld_dur(c, i) < 0)
        missing = true;  // replay.cpp:39-44
      else if (dv >= D)
        inval = true;
      else
        atomicAdd(&ds[dv].tail, 1u);
    }
    const unsigned mm = __ballot_sync(kFull, missing);
    const unsigned mi = __ballot_sync(kFull, inval);
    if (mm | mi) {
      const unsigned m = mm | mi;
      first_bad = base + __ffs(m) - 1;
      bad_kind = (mm & (1u << (__ffs(m) - 1))) ? kMissing : kInval;
      break;
    }
  }
  if (first_bad != kNone) {
    // The missing-profile scan must report the FIRST missing op even when an
    // invalid device id precedes it: rescan for missing only.
    if (bad_kind == kInval) {
      for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        const bool missing = i < n && !(c.flags[i] & 1u) && ld_dur(c, i) < 0;
        const unsigned mm = __ballot_sync(kFull, missing);
        if (mm) {
          first_bad = base + __ffs(mm) - 1;
          bad_kind = kMissing;
          break;
        }
      }
    }
    if (lane == 0) {
      O.status[cid] = bad_kind;
      O.err[cid] = first_bad;
      O.makespan[cid] = 0;
    }
    return;
  }
  __syncwarp();
  // exclusive scan of per-device counts -> queue regions
  {
    uint32_t running = 0;
    for (uint32_t b = 0; b < D; b += 32) {
      const uint32_t d = b + lane;
      const uint32_t v = d < D ? ds[d].tail : 0;
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t off = running + x - v;
      if (d < D) {
        ds[d].head = ds[d].tail = ds[d].tsort = ds[d].segbeg = off;
        devoff[d] = off;
      }
      running += __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) devoff[D] = running;
  }
  // ---- working indeg, flags ----
  for (uint32_t i = lane; i < n; i += 32) {
    indeg[i] = c.indeg ? c.indeg[i] : 0u;
    sched[i] = 0;
    qpos[i] = kNone;
  }
  __syncwarp();
  if (!c.indeg) {
    for (uint32_t i = lane; i < n; i += 32)
      for (uint32_t k = c.succ_off[i]; k < c.succ_off[i + 1]; ++k)
        atomicAdd(&indeg[c.succ[k]], 1u);
  }
  __syncwarp();

  Replayer R{c, ds, indeg, qbuf, qpos, sched, S.vstack + oo, vtop, start, end,
             lane, want_schedule};

  bool quirk = false;  // lane 0 only
  // ---- init scan (replay.cpp:92-94), quirk-exact ----
  // Candidates: indeg == 0 now and (virtual, or not yet queued). A virtual op
  // zeroed by an earlier cascade is readied again (double cascade), a
  // non-virtual one is a std::set no-op. qpos doubles as the "queued" mark.
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t i = base + lane;
    uint32_t from = base;
    for (;;) {
      bool cand = false, virt = false;
      if (i < n && i >= from) {
        virt = c.flags[i] & 1u;
        cand = __ldcg(&indeg[i]) == 0u &&
               (virt || __ldcg(&qpos[i]) == kNone);
      }
      const unsigned m = __ballot_sync(kFull, cand);
      if (!m) break;
      const unsigned vm = __ballot_sync(kFull, cand && virt);
      // non-virtual candidates below the first virtual one: enqueue in parallel
      const unsigned lim = vm ? ((1u << (__ffs(vm) - 1)) - 1u) : kFull;
      if (cand && !virt && ((1u << lane) & lim)) {
        const uint32_t p = atomicAdd(&ds[c.dev[i]].tail, 1u);
        qbuf[p] = i;
        atomicExch(&qpos[i], 0u);  // queued mark
      }
      __syncwarp();
      if (!vm) break;
      const uint32_t v = base + __ffs(vm) - 1;
      if (lane == 0) {
        // serial cascade from v at t = 0 (order-free: a worklist)
        if (want_schedule) {
          start[v] = 0;
          end[v] = 0;
        }
        if (sched[v]) quirk = true;  // double cascade
        sched[v] = 1;
        ++R.vcount;
        uint32_t top = 0;
        R.vstack[top++] = v;
        while (top > 0) {
          const uint32_t x = R.vstack[--top];
          for (uint32_t k = c.succ_off[x]; k < c.succ_off[x + 1]; ++k) {
            const uint32_t s = c.succ[k];
            if (atomicSub(&indeg[s], 1u) != 1u) continue;
            if (c.flags[s] & 1u) {
              if (want_schedule) {
                start[s] = 0;
                end[s] = 0;
              }
              sched[s] = 1;
              ++R.vcount;
              R.vstack[top++] = s;
            } else if (__ldcg(&qpos[s]) == kNone) {
              const uint32_t p = atomicAdd(&ds[c.dev[s]].tail, 1u);
              qbuf[p] = s;
              atomicExch(&qpos[s], 0u);
            }
          }
        }
      }
      __syncwarp();
      from = v + 1;
    }
  }
  __syncwarp();
  // init arrivals all have ready time 0: sort each queue by index
  for (uint32_t d = lane; d < D; d += 32) {
    DevSt& s = ds[d];
    const uint32_t tail = R.tail_of(s);
    for (uint32_t p = s.head + 1; p < tail; ++p) {
      const uint32_t x = qbuf[p];
      uint32_t q = p;
      while (q > s.head && qbuf[q - 1] > x) {
        qbuf[q] = qbuf[q - 1];
        --q;
      }
      qbuf[q] = x;
    }
    s.tsort = tail;
    s.segbeg = s.head;
    s.segt = 0;
  }
  __syncwarp();

  // ---- dispatch(0) and the event loop (replay.cpp:95-106) ----
  long long lane_min = kTInf;
  bool lane_zero = false;
  long long t = 0;
  for (uint32_t d = lane; d < D; d += 32) R.dispatch_dev(d, t, lane_min, lane_zero);
  for (;;) {
    const bool zero_round = __any_sync(kFull, lane_zero);
    if (!zero_round) {
      const long long tn = warp_min64(lane_min);
      if (tn == kTInf) break;
      t = tn;
    }
    // completions of this round
    for (uint32_t d = lane; d < D; d += 32) {
      DevSt& s = ds[d];
      if (zero_round) {
        for (uint32_t p = s.zlo; p < s.zhi; ++p) R.complete(qbuf[p], t);
        s.zlo = s.zhi;
      } else if (s.infl != kNone && s.infl_end == t) {
        const uint32_t i = s.infl;
        s.infl = kNone;
        R.complete(i, t);
      }
    }
    R.drain_virtual(t);
    __syncwarp();
    lane_min = kTInf;
    lane_zero = false;
    for (uint32_t d = lane; d < D; d += 32) R.dispatch_dev(d, t, lane_min, lane_zero);
  }

  // ---- termination (replay.cpp:108-123) ----
  const unsigned long long vc = warp_sum64(R.vcount);
  const unsigned long long dc = warp_sum64(R.dcount);
  const long long T = warp_max64(R.tmax);
  for (uint32_t d = lane; d < D; d += 32) {
    S.busy[c.dev_off + d] = ds[d].busy;
    S.dhead[c.dev_off + d] = ds[d].head;
  }
  const uint32_t remaining = n - static_cast<uint32_t>(vc + dc);  // uint32 wrap
  if (remaining != 0u) {
    unsigned long long stuck = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) stuck += sched[i] ? 0 : 1;
    stuck = warp_sum64(stuck);
    if (lane == 0) {
      O.status[cid] = kCycle;
      O.err[cid] = static_cast<long long>(stuck);
      O.makespan[cid] = 0;
    }
    return;
  }
  // Init-quirk graphs can end "successfully" with ops never scheduled; the
  // reference reports them at start = end = 0 (replay.cpp:57,119-123).
  if (__any_sync(kFull, quirk) && want_schedule) {
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32)
      if (!sched[i]) start[i] = end[i] = 0;
  }
  if (lane == 0) {
    O.status[cid] = kOk;
    O.err[cid] = 0;
    O.makespan[cid] = T;
  }
}

// Persistent warps pull candidates from a global counter (sizes vary).
// filter != 0: only candidates whose status is `filter` (the fast kernels'
// hand-offs), pulled from work[9].
__global__ void __launch_bounds__(128) replay_batch_kernel(
    const Cand* __restrict__ cands, int n_cands, Scratch S, Outs O,
    int want_schedule, unsigned* work, uint32_t dcap, int filter = 0) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  volatile uint32_t* vtops = reinterpret_cast<volatile uint32_t*>(smem_raw);
  DevSt* sdev = reinterpret_cast<DevSt*>(smem_raw + 16 * 8) + (size_t)warp * dcap;
  for (;;) {
    int cid = 0;
    if ((threadIdx.x & 31) == 0) cid = static_cast<int>(atomicAdd(work + (filter ? 9 : 0), 1u));
    cid = __shfl_sync(kFull, cid, 0);
    if (cid >= n_cands) break;
    if (filter && O.status[cid] != filter) continue;
    const Cand c = cands[cid];
    DevSt* ds = (c.d <= dcap) ? sdev : S.dstate + c.dev_off;
    replay_candidate(c, cid, ds, vtops + warp * 4, S, O, want_schedule != 0);
    __syncwarp();
  }
  (void)wpb;
}

}  // namespace dpro_k
