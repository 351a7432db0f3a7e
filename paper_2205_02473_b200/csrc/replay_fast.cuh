// K1 fast path: exact batched replay with all mutable state on chip.
//
// Same round semantics as replay_kernel.cuh (proj/src/replay.cpp:37-134);
// what changes is where the state lives and what an event round touches.
//   * one CTA of NW warps per candidate (NW = 1, 2 or 4, chosen by device
//     count); thread l owns devices d = l + 32 NW j (j < KD); the in-flight
//     end of each owned device lives in a register as a 32-bit offset from
//     the current time t (every in-flight end lies in (t, t + 2^31): op
//     durations fit int32), so the next event time is one REDUX.MIN and t
//     itself is 64-bit (integer us or ns: a config-4 makespan in ns is
//     ~10^12);
//   * a round only visits devices that completed or received arrivals
//     (per-lane dirty bitmask in shared memory, set by producers);
//   * per-device FIFOs are shared-memory rings of 16-byte entries
//     {op, dur, succ_beg, succ_end}, sorted by (ready, index) on arrival;
//   * in-degree countdowns exist only for ops with >= 2 predecessors, as
//     compact u8 counters in shared memory (4 per word, word atomics);
//   * the out-edge records of every op completing in a round (16-byte
//     records, pack_kernel.cuh) are expanded by all 32 lanes at once: the
//     completing lanes publish {succ_beg, count} ranges, a warp scan assigns
//     records to lanes, so a round costs one record-load latency however
//     many successors complete (a PS push RECV has 16);
// Whatever the fast path cannot represent (ring or worklist overflow, a
// virtual source -> init quirk, indeg >= 65535, an op duration >= 2^31,
// too many devices / counters, a cycle) falls back inside the same launch
// to the general kernel (replay_candidate, global state): every
// candidate's result is exact either way.
#pragma once

#include "pack_kernel.cuh"
#include "replay_kernel.cuh"

namespace dpro_k {

constexpr uint32_t kT32Inf = 0xFFFFFFFFu;
// Register budget of the fast kernels. ptxas picks 56 registers (a few
// spills to L1-resident local memory); capping at 64 via a minimum CTA count
// removes the spills but measured 10 % slower on config 4 (1,475 vs 1,645
// replays/s, profiles/r02_c4_regbudget_ab.log): it stays behind DPRO_MINB.
#ifdef DPRO_MINB
#define DPRO_FAST_BOUNDS(NW, KD) __launch_bounds__(32 * NW, (KD <= 5 ? 32 : 16) / NW)
#else
#define DPRO_FAST_BOUNDS(NW, KD) __launch_bounds__(32 * NW)
#endif
// The overlay kernel holds the in-flight ops' records in registers
// (kRegPrefetch): a bound of 12 CTAs of 2 warps per SM (85 registers) keeps
// them out of local memory -- 1,780-1,798 vs 1,647-1,676 replays/s unbounded
// (72 registers + spills) and 1,704-1,742 without the prefetch
// (profiles/r02_c4_regprefetch_ab.log).
#define DPRO_OV_BOUNDS(NW, KD) __launch_bounds__(32 * NW, (KD <= 5 ? 24 : 16) / NW)
// replay_fast outcomes / bail-out causes
constexpr uint32_t kDone = 0, kBailRing = 1, kBailOther = 2, kBailRl = 3;
constexpr uint32_t kMiscRl = 4;  // misc[1] bit: a round's range list overflowed
__device__ __forceinline__ uint32_t bail_code(uint32_t m) {
  return (m & kBailOther) ? kBailOther : (m & kBailRing) ? kBailRing : kBailRl;
}
constexpr int kRetry = 9;   // status of a candidate queued for the deep-ring pass
constexpr int kRetry2 = 11;  // queued for the global-ring pass (pass 3)
constexpr int kRetryGen = 12;  // handed to the general kernel (replay_batch_kernel)

// segt: the event-time EPOCH (count of distinct event times so far) of the
// device's last arrival segment -- a time-independent stand-in for "the
// arrivals at the current t", exact for any time unit.
struct __align__(16) DevF {
  uint32_t head, tail, tsort, segbeg;
  uint32_t zlo, zhi, segt, qoff;  // qoff: the device's offset in qbuf (devoff)
  uint32_t busy_lo, busy_hi;  // summed dur of the dispatched ops (64-bit)
  uint32_t isb, ise;          // successor range of the in-flight op
};
static_assert(sizeof(DevF) == 48, "DevF layout");

struct FastCfg {
  uint32_t dcap;   // devices per warp
  uint32_t ccap;   // compact counters per warp (bytes, multiple of 16)
  uint32_t qc;     // ring capacity per device (power of two)
  uint32_t rl;     // successor-range list capacity per round
  uint32_t warp_bytes;
  uint32_t kd;     // devices per lane (template parameter)
  uint4* gq = nullptr;  // pass 3: device rings in global memory, dcap * qc per CTA
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// shared-memory bytes per device after the counters: the successor range of
// a lone zero-duration op (its completion round reads it instead of the ring).
// (Copying the in-flight op's records into a 32-byte slot per device with
// cp.async at dispatch measured 12 % slower on config 4: the larger CTA
// leaves too few slots per SM -- profiles/r02_c4_prefetch_ab.log.)
// 1-D bulk copies global -> shared memory on the TMA engine (no tensor map:
// cp.async.bulk), completing on an mbarrier: the candidate's contiguous
// counter image and sparse overlay lists at candidate start. One thread arms
// the barrier with the byte count and issues the copies; every thread waits
// on the barrier's phase. Addresses and sizes are multiples of 16 bytes.
struct BulkBar {
  uint64_t* bar;   // shared-memory mbarrier (arrival count 1)
  uint32_t phase;  // parity of the next completion
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_bar_init(uint64_t* bar) {
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}
// thread 0 only: arm with the total bytes of the copies that follow
__device__ __forceinline__ void bulk_arm(BulkBar& b, uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after generic smem use
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b.bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, BulkBar& b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b.bar)) : "memory");
}
__device__ __forceinline__ void bulk_wait(BulkBar& b) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(b.bar)), "r"(b.phase) : "memory");
  b.phase ^= 1u;
}

// Per-op outputs (start, end, device-queue order) are written once and not
// read again by the replay: streaming stores (evict-first in L2), so they do
// not push the rings, counters and shared base records out of L2.
#ifdef DPRO_PLAIN_STORES
template <typename T, typename V>
__device__ __forceinline__ void st_out(T* p, V v) { *p = static_cast<T>(v); }
#else
__device__ __forceinline__ void st_out(long long* p, unsigned long long v) {
  __stcs(p, static_cast<long long>(v));
}
__device__ __forceinline__ void st_out(long long* p, long long v) { __stcs(p, v); }
__device__ __forceinline__ void st_out(uint32_t* p, uint32_t v) { __stcs(p, v); }
#endif

#ifdef DPRO_NO_ZR
constexpr uint32_t kTailBytesPerDev = 0;  // A/B builds: zero rounds read the ring
#else
constexpr uint32_t kTailBytesPerDev = 8;
#endif

#ifndef DPRO_MLP
#define DPRO_MLP 1
#endif
constexpr int kMlp = DPRO_MLP;  // record loads in flight per lane in expand()
#ifdef DPRO_NO_REG_PREFETCH
constexpr bool kRegPrefetch = false;  // A/B builds: completions push ranges
#else
constexpr bool kRegPrefetch = true;
#endif
constexpr uint32_t kNoPre = 0xFFu;

#ifdef DPRO_NO_LANE_EXPAND
constexpr bool kLaneExpand = false;  // A/B builds: always the scan expansion
#else
constexpr bool kLaneExpand = true;
#endif

// misc words: [0],[2] range counts (double-buffered by round parity),
// [1] overflow, [4, 4+NT) per-thread dirty masks, then 4*NW words of
// double-buffered reduction scratch.
// (rounded up to 4 words: the u8 counters after it are copied as uint4)
__host__ __device__ constexpr size_t fast_misc_words(int nw) {
  return (4 + 32 * nw + 4 * nw + 3) & ~size_t(3);
}

// threadIdx.x read once per candidate through an opaque move: ptxas otherwise
// re-reads the special register (S2R) and rebuilds every tid-derived
// address in the round loop when registers are tight (profiles/r02_c4_*).
__device__ __forceinline__ uint32_t tid_once() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(r));
  return r;
}

// Group-wide collectives for one candidate replayed by NW warps (one CTA).
template <int NW>
__device__ __forceinline__ void gsync() {
  if (NW == 1)
    __syncwarp();
  else
    __syncthreads();
}
template <int NW>
__device__ __forceinline__ bool gany(bool p) {
  if (NW == 1) return __any_sync(kFull, p);
  return __syncthreads_or(p) != 0;
}
template <int NW>
__device__ __forceinline__ uint32_t gmin(uint32_t v, volatile uint32_t* red, uint32_t& par,
                                         uint32_t tid) {
  v = __reduce_min_sync(kFull, v);
  if (NW == 1) return v;
  volatile uint32_t* r = red + (par & 1u) * 2 * NW;  // same buffers as round_head
  ++par;
  if ((tid & 31) == 0) r[tid >> 5] = v;
  __syncthreads();
  uint32_t m = r[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) m = min(m, r[w]);
  return m;
}
// Round head: (any thread has zero-duration completions pending, min next
// event time) in ONE barrier. red holds 2 x NW words per parity buffer.
template <int NW>
__device__ __forceinline__ void round_head(bool zero, uint32_t lmin, volatile uint32_t* red,
                                           uint32_t& par, bool& any_zero, uint32_t& tmin,
                                           uint32_t tid) {
  const bool wz = __any_sync(kFull, zero);
  const uint32_t wm = __reduce_min_sync(kFull, lmin);
  if (NW == 1) {
    any_zero = wz;
    tmin = wm;
    return;
  }
  volatile uint32_t* r = red + (par & 1u) * 2 * NW;
  ++par;
  if ((tid & 31) == 0) {
    r[tid >> 5] = wz ? 1u : 0u;
    r[NW + (tid >> 5)] = wm;
  }
  __syncthreads();
  bool z = false;
  uint32_t m = kT32Inf;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    z |= r[w] != 0u;
    m = min(m, r[NW + w]);
  }
  any_zero = z;
  tmin = m;
}

template <int NW>
__device__ __forceinline__ uint32_t gsum(uint32_t v, volatile uint32_t* red, uint32_t& par,
                                         uint32_t tid) {
  v = __reduce_add_sync(kFull, v);
  if (NW == 1) return v;
  volatile uint32_t* r = red + (par & 1u) * 2 * NW;  // same buffers as round_head
  ++par;
  if ((tid & 31) == 0) r[tid >> 5] = v;
  __syncthreads();
  uint32_t m = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) m += r[w];
  return m;
}
template <int NW>
__device__ __forceinline__ uint32_t gmax(uint32_t v, volatile uint32_t* red, uint32_t& par,
                                         uint32_t tid) {
  v = __reduce_max_sync(kFull, v);
  if (NW == 1) return v;
  volatile uint32_t* r = red + (par & 1u) * 2 * NW;  // same buffers as round_head
  ++par;
  if ((tid & 31) == 0) r[tid >> 5] = v;
  __syncthreads();
  uint32_t m = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) m = max(m, r[w]);
  return m;
}

template <int NW>
__device__ __forceinline__ unsigned long long gmax64(unsigned long long v, volatile uint32_t* red,
                                                     uint32_t& par, uint32_t tid) {
  const uint32_t hi = gmax<NW>(static_cast<uint32_t>(v >> 32), red, par, tid);
  const uint32_t lo = gmax<NW>((v >> 32) == hi ? static_cast<uint32_t>(v) : 0u, red, par, tid);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// Overlay mode (OV, overlay.h): candidates replayed on the resident base's
// packed layout plus a per-candidate overlay. rec/erec are the BASE arrays;
// records in overlay form carry kOv in w (slot in x, final index in fin[]);
// ranges and ring entries carry kOv in their start word when they index
// the overlay's lists.
constexpr uint32_t kOvF = 0x80000000u;
constexpr uint32_t kBlkShiftF = 10;
constexpr uint32_t kBlkOvfF = 0x80000000u;
constexpr uint32_t kBlkBiasF = 0x40000000u;
constexpr uint32_t kOvfDirtyF = 0x80000000u;

struct OvView {
  const uint4* rec;      // [no + 1] overlay records
  const uint4* erec;     // overlay expanded lists
  const uint32_t* fin;   // [no] final index per overlay op
  const uint32_t* blk;   // per 1024 base ids: shift + kBlkBias, or kBlkOvf | block
  const uint32_t* ovf;   // 1024 entries per flagged block
};

// One overlay candidate (device copy; arrays in the batch's overlay arena).
struct OvCand {
  OvView v;
  const uint16_t* cnt;         // initial counts of the overlay counters
  const uint4* src;            // source records (base or overlay form)
  const uint2* sx;             // sparse form: (base id, slot) of the dirty ops
  const uint2* sbp;            // sparse form: (first base id, shift) runs
  unsigned long long gcnt_off; // byte offset of the candidate's global counters
  uint32_t n_cnt, n_src, first_missing, pad;
  uint32_t n_sx, n_sbp, ovmin, sparse;
};
// shared memory for the sparse lists (48 + 48 pairs: config 4's residency
// pass fits 15 CTAs per SM)
constexpr uint32_t kOvListMax = 48;
constexpr uint32_t kOvListBytes = 2 * 8 * kOvListMax;

// The resident base's packed layout (overlay batches).
struct OvBase {
  const uint4* rec;
  const uint4* erec;
  const uint8_t* cnt0;  // u8, or u16 when wide
  uint32_t n_cnt, wide;
};

template <int NW, int KD, bool OV = false>
struct FastWarp {
  static constexpr uint32_t NT = 32u * NW;
  const uint4* __restrict__ rec;
  const uint4* __restrict__ erec;
  OvView ov{};
  DevF* dv;
  uint4* q;                 // [dcap][qc] per-device rings
  uint2* rl;                // [rlcap] {succ_beg, count} ranges to expand
  volatile uint32_t* misc;
  uint32_t* cw;             // compact counters (u8 or u16 in words)
  uint32_t qc, rlcap;
  uint32_t* qbuf;
  uint32_t* qpos;
  const uint32_t* devoff;
  long long* start;
  long long* end;
  bool want;
  int lane;
  int tid;
  uint32_t vcount = 0, dcount = 0;
  unsigned long long tmax = 0;
  bool wide = false;  // u16 counters (some in-degree >= 255)
  uint4* last = nullptr;        // OV: [dcap] each device's latest arrival (shared memory)
  uint2* zr = nullptr;          // [dcap] successor range of a lone zero-duration op
  const uint2* sxs = nullptr;   // OV sparse lists in shared memory
  const uint2* sbps = nullptr;
  uint32_t n_sx = 0, n_sbp = 0, ovmin = 0;
  bool sparse = false;

  __device__ __forceinline__ uint4* ring(uint32_t d) { return q + (size_t)d * qc; }

  volatile uint32_t* rlc = nullptr;  // this round's range counter

  // The range counter's high bits count the ranges of more than 2 records:
  // while there are none, expand() gives every thread its own ranges.
  static constexpr uint32_t kRlLong = 1u << 20;
  __device__ __forceinline__ void push_range(uint32_t sb, uint32_t n) {
    const uint32_t p =
        atomicAdd(const_cast<uint32_t*>(rlc), n > 2u ? 1u + kRlLong : 1u) & (kRlLong - 1u);
    if (p < rlcap)
      rl[p] = make_uint2(sb, n);
    else
      atomicOr(const_cast<uint32_t*>(&misc[1]), kMiscRl);  // capacity: retry deeper
  }

  // OV: final index of the op a record stands for; a base-form record of a
  // dirty op is replaced by the op's overlay record (block table lookup).
  __device__ __forceinline__ uint32_t resolve(uint4& a) const {
    if constexpr (!OV) {
      return a.x & kOpMask;
    } else {
      if (a.w & kOvF) return __ldg(ov.fin + (a.x & kOpMask));
      const uint32_t b = a.x & kOpMask;
      if (sparse) {  // shared-memory lists; most ops lie below every change
        if (b < ovmin) return b;
        uint32_t lo = 0, hi = n_sx;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (sxs[mid].x < b) lo = mid + 1;
          else hi = mid;
        }
        if (lo < n_sx && sxs[lo].x == b) {
          const uint32_t slot = sxs[lo].y;
          a = __ldg(ov.rec + slot);
          return __ldg(ov.fin + slot);
        }
        lo = 0;
        hi = n_sbp;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (sbps[mid].x <= b) lo = mid + 1;
          else hi = mid;
        }
        return lo ? b + sbps[lo - 1].y : b;
      }
      const uint32_t e = __ldg(ov.blk + (b >> kBlkShiftF));
      if (!(e & kBlkOvfF)) return b + e - kBlkBiasF;
      const uint32_t v = __ldg(ov.ovf + (size_t(e & ~kBlkOvfF) << kBlkShiftF) + (b & 1023u));
      if (!(v & kOvfDirtyF)) return v;
      const uint32_t slot = v & ~kOvfDirtyF;
      a = __ldg(ov.rec + slot);
      return __ldg(ov.fin + slot);
    }
  }

  // ready(s, t) of replay.cpp:60-72 for s reached through a packed record
  // (s = final index; OV: a may be in overlay form).
  __device__ __forceinline__ void ready(const uint4& a, unsigned long long t, uint32_t s) {
    const uint32_t cnt = (a.z >> kCntShift) & kCntMax;
    const uint32_t fl = OV ? (a.w & kOvF) : 0u;  // list lives in the overlay
    const uint32_t sb = a.w & ~fl;
    uint32_t se;
    if (cnt != kCntMax) se = sb + cnt;
    else if (OV && fl) se = __ldg(&ov.rec[(a.x & kOpMask) + 1].w) & ~kOvF;
    else se = __ldg(&rec[(a.x & kOpMask) + 1].w);
    if (a.z & kFVirt) {  // multi-predecessor virtual: completes now, cascade
      if (want) {
        st_out(start + s, t);
        st_out(end + s, t);
      }
      ++vcount;
      tmax = max(tmax, t);
      if (se > sb) push_range(sb | fl, se - sb);
      return;
    }
    const uint32_t d = a.z & kDevMask;
    DevF& sd = dv[d];
    const uint32_t pos = atomicAdd(&sd.tail, 1u);
    const uint32_t zl = *reinterpret_cast<volatile uint32_t*>(&sd.zlo);
    const uint32_t zh = *reinterpret_cast<volatile uint32_t*>(&sd.zhi);
    const uint32_t low = zl < zh ? zl : *reinterpret_cast<volatile uint32_t*>(&sd.head);
    if (pos - low >= qc) {
      atomicOr(const_cast<uint32_t*>(&misc[1]), kBailRing);
    } else {
      const uint4 e = make_uint4(s, a.y, sb | fl, se);  // {op, dur, sb, se}
      ring(d)[pos & (qc - 1)] = e;
      if (OV) last[d] = e;  // a lone arrival is dispatched from here (no ring read)
      atomicOr(const_cast<uint32_t*>(&misc[4 + (d % NT)]), 1u << (d / NT));
    }
    if (se > sb) prefetch_l2((OV && fl ? ov.erec : erec) + sb);  // read when s completes
  }

  // One out-edge record of a completing op (replay.cpp:100-103).
  __device__ __forceinline__ void edge(uint4 a, unsigned long long t) {
    const uint32_t s = resolve(a);
    if ((a.z & (kFVirt | kFMulti)) == kFVirt) {  // spliced single-pred virtual
      if (want) {
        st_out(start + s, t);
        st_out(end + s, t);
      }
      ++vcount;
      tmax = max(tmax, t);
      return;  // its successors follow in this same list
    }
    if (a.z & kFMulti) {
      const uint32_t ci = (a.x >> 24) | ((a.z >> 18) << 8);
      if (wide) {  // u16 counters, 2 per word
        const uint32_t sh = 16u * (ci & 1u);
        const uint32_t old = atomicSub(&cw[ci >> 1], 1u << sh);
        if (((old >> sh) & 0xFFFFu) != 1u) return;
      } else {     // u8 counters, 4 per word
        const uint32_t sh = 8u * (ci & 3u);
        const uint32_t old = atomicSub(&cw[ci >> 2], 1u << sh);
        if (((old >> sh) & 0xFFu) != 1u) return;
      }
    }
    ready(a, t, s);
  }

  __device__ __forceinline__ uint4 record(uint32_t sb, uint32_t k) const {
    if (OV && (sb & kOvF)) return __ldg(ov.erec + (sb & ~kOvF) + k);
    return __ldg(erec + sb + k);
  }

  // Expands every range pushed this round (and the virtual cascades they
  // trigger) with all 32 lanes: the round's out-edge records are loaded and
  // applied in parallel instead of one lane walking each list.
  // The caller has made this round's ranges visible (barrier). Each pass
  // expands ranges [lo, hi) and ends with a barrier; virtual cascades
  // pushed during a pass are expanded by the next one.
  // Returns kDone, or the bail-out cause.
  __device__ __forceinline__ uint32_t expand(unsigned long long t) {
    uint32_t lo = 0;
    for (;;) {
      const uint32_t rc = *rlc;
      const uint32_t hi = rc & (kRlLong - 1u);
      if (misc[1]) return bail_code(misc[1]);
      if (hi > rlcap) return kBailRl;
      if (lo == hi) return kDone;
      if (kLaneExpand && rc < kRlLong) {
        // every range has <= 2 records (config 4: no op has more than 2
        // successors): each thread loads and applies its own ranges, no scan
        for (uint32_t r = lo + tid; r < hi; r += NT) {
          const uint2 mine = rl[r];
          uint4 a0 = make_uint4(0, 0, 0, 0), a1 = a0;
          if (mine.y) a0 = record(mine.x, 0);
          if (mine.y > 1u) a1 = record(mine.x, 1);
          if (mine.y) edge(a0, t);
          if (mine.y > 1u) edge(a1, t);
          // (only if the long-range count wrapped: still exact)
          for (uint32_t k = 2; k < mine.y; ++k) edge(record(mine.x, k), t);
        }
        gsync<NW>();
        lo = hi;
        continue;
      }
      for (uint32_t g = lo; g < hi; g += 32) {
        const uint32_t r = g + lane;
        uint2 mine = make_uint2(0u, 0u);
        if (r < hi) mine = rl[r];
        uint32_t incl = mine.y;
#ifndef DPRO_SCAN_SKIP
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
#else
        if (hi - g > 1) {
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
        }
#endif
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        const uint32_t nr = min(32u, hi - g);
        // lane r holds range r's first item index; items map to ranges by a
        // 5-step shuffle binary search (no shared-memory walk)
        const uint32_t excl = (uint32_t)lane < nr ? incl - mine.y : 0xFFFFFFFFu;
        // memory-level parallelism: each thread issues up to kMlp record
        // loads back to back, then applies them (edge() has atomics, so the
        // compiler would otherwise serialize load -> apply -> next load)
        for (uint32_t base = 0; base < total; base += NT * kMlp) {
          uint4 a[kMlp];
#pragma unroll
          for (int b = 0; b < kMlp; ++b) {
            const uint32_t qi = base + tid + NT * b;
            int k = 0;
#ifdef DPRO_SEARCH_STEPS
#pragma unroll
            for (int step = DPRO_SEARCH_STEPS; step; step >>= 1) {
#else
#pragma unroll
            for (int step = 16; step; step >>= 1) {
#endif
              const int cand = k + step;
              const uint32_t v = __shfl_sync(kFull, excl, cand & 31);
              if (cand < 32 && v <= qi) k = cand;
            }
            const uint32_t sb = __shfl_sync(kFull, mine.x, k);
            const uint32_t ex = __shfl_sync(kFull, excl, k);
            if (qi < total) {
              if (OV && (sb & kOvF)) a[b] = __ldg(ov.erec + (sb & ~kOvF) + (qi - ex));
              else a[b] = __ldg(erec + sb + (qi - ex));
            }
          }
#pragma unroll
          for (int b = 0; b < kMlp; ++b)
            if (base + tid + NT * b < total) edge(a[b], t);
        }
      }
      gsync<NW>();
      lo = hi;
    }
  }

  // Owner-lane dispatch(t) for device d (replay.cpp:74-90) after merging
  // this round's arrivals into the (ready, index)-ordered tail segment.
  // Returns the in-flight op's end - t (kT32Inf: idle); sets *zero when
  // zero-duration ops ran (they complete next round). epoch: number of
  // distinct event times so far.
  __device__ __forceinline__ uint32_t dispatch_dev(uint32_t d, unsigned long long t,
                                                   uint32_t epoch, uint32_t iend, bool* zero,
                                                   uint4& p0, uint4& p1, uint32_t& pn) {
    DevF& s = dv[d];
    uint4* r = ring(d);
    const uint32_t tail = *reinterpret_cast<volatile uint32_t*>(&s.tail);
    const uint32_t m = qc - 1;
    uint32_t head = s.head;
    // OV: with one arrival this round its entry is in last[d] (shared
    // memory) -- the rings may live in global memory
    const bool lone = OV && tail == s.tsort + 1;
    uint4 lone_e = make_uint4(0, 0, 0, 0);
    uint32_t lone_pos = 0;
    if (lone) lone_e = last[d];
    if (tail != s.tsort) {
      if (s.segt != epoch) {
        s.segbeg = s.tsort;
        s.segt = epoch;
      }
      const uint32_t lo = max(s.segbeg, head);
      for (uint32_t p = s.tsort; p < tail; ++p) {
        const uint4 x = lone ? lone_e : r[p & m];
        uint32_t qq = p;
        while (qq > lo) {
          const uint4 y = r[(qq - 1) & m];
          if (y.x < x.x) break;
          r[qq & m] = y;
          --qq;
        }
        if (!lone || qq != p) r[qq & m] = x;  // (a lone entry in place is already there)
        lone_pos = qq;
      }
      s.tsort = tail;
    }
    if (iend == kT32Inf && head < tail) {
      const uint32_t zlo = head;
      unsigned long long busy = 0;
      const uint32_t base = s.qoff;
      bool infl = false;
      uint2 z0 = make_uint2(0u, 0u);  // range of the first dispatched op
      while (head < tail) {
        const uint4 x = (lone && head == lone_pos) ? lone_e : r[head & m];
        if (head == zlo) z0 = make_uint2(x.z, x.w);
        const unsigned long long en = t + x.y;
        if (want) {  // (qpos is derived from qbuf only when K3 needs it)
          st_out(start + x.x, t);
          st_out(end + x.x, en);
        }
        st_out(qbuf + base + head, x.x);
        ++head;
        ++dcount;
        busy += x.y;
        tmax = max(tmax, en);
        if (x.y > 0) {
          s.isb = x.z;
          s.ise = x.w;
          iend = x.y;
          infl = true;
          if (kRegPrefetch && OV) {
            // the in-flight op's out-edge records (<= 2) are loaded into the
            // owner's registers now and applied by the owner when it
            // completes (a later round): no record load on that round's path
            const uint32_t ne = x.w - (x.z & ~kOvF);
            if (ne <= 2u) {
              if (ne) p0 = record(x.z, 0);
              if (ne == 2u) p1 = record(x.z, 1);
              pn = ne;
            } else {
              pn = kNoPre;
            }
          }
          break;
        }
      }
      const unsigned long long bz =
          ((static_cast<unsigned long long>(s.busy_hi) << 32) | s.busy_lo) + busy;
      s.busy_lo = static_cast<uint32_t>(bz);
      s.busy_hi = static_cast<uint32_t>(bz >> 32);
      s.head = head;
      s.zlo = zlo;
      const uint32_t zhi = infl ? head - 1 : head;
      s.zhi = zhi;
      if (zlo < zhi) *zero = true;
      if (kTailBytesPerDev && zhi - zlo == 1u) zr[d] = z0;  // a lone zero op: its range without a ring read
    }
    return iend;
  }
};

#ifdef DPRO_PROFILE
// per-candidate phase counters (experiment builds only): written to
// Scratch::busy of device 0 region? no -- to a global debug array.
__device__ unsigned long long g_prof[16];
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(i_, v_) if (threadIdx.x == 0) atomicAdd(&g_prof[i_], (unsigned long long)(v_))
#else
#define PROF_T(v)
#define PROF_ADD(i, x)
#endif

// Returns kDone, kBailRing (a device queue outgrew its ring or a round its
// range list: retry with deeper ones) or kBailOther (take the general path).
template <int NW, int KD, bool OV = false>
__device__ __forceinline__ uint32_t replay_fast(const Cand& c, int cid, const uint4* rec, const uint4* erec,
                            const uint8_t* cnt0, const uint32_t* srcs, const PackInfo& info,
                            unsigned char* wsm, const FastCfg& F, const Scratch& S,
                            const Outs& O, bool want_schedule, uint32_t* gcw,
                            const OvCand* ovc = nullptr, const OvBase* ob = nullptr,
                            BulkBar* bb = nullptr) {
  constexpr uint32_t NT = 32u * NW;
  const int tid = static_cast<int>(tid_once());
  const int lane = tid & 31;
  const uint32_t n = c.n, D = c.d;
  DevF* dv = reinterpret_cast<DevF*>(wsm);
  uint4* q = F.gq ? F.gq + size_t(blockIdx.x) * F.dcap * F.qc
                  : reinterpret_cast<uint4*>(wsm + sizeof(DevF) * F.dcap);
  uint2* rl = reinterpret_cast<uint2*>(wsm + sizeof(DevF) * F.dcap +
                                       (F.gq ? 0 : 16 * size_t(F.dcap) * F.qc));
  volatile uint32_t* misc = reinterpret_cast<volatile uint32_t*>(rl + F.rl);
  // compact counters: shared memory, or (graphs with more multi-predecessor
  // ops than fit) this candidate's slice of global scratch, same word atomics
  uint32_t* cw = gcw ? gcw : const_cast<uint32_t*>(misc) + fast_misc_words(NW);
  volatile uint32_t* red = misc + 4 + NT;  // 4 * NW words
  uint32_t par = 0;
  const unsigned long long oo = c.op_off;

  FastWarp<NW, KD, OV> W{rec, erec, {}, dv, q, rl, misc, cw, F.qc, F.rl, S.qbuf + oo,
                     S.qpos + oo, S.devoff + c.dof_off,
                     want_schedule ? O.start + oo : nullptr,
                     want_schedule ? O.end + oo : nullptr, want_schedule, lane, tid};
  W.wide = info.wide != 0;
  W.zr = reinterpret_cast<uint2*>(reinterpret_cast<unsigned char*>(
                                      const_cast<uint32_t*>(misc) + fast_misc_words(NW)) +
                                  F.ccap + (OV ? kOvListBytes + 16 * F.dcap : 0u));

  // ---- state init ----
  if constexpr (OV) {
    // u16 counters: the base's (u8 or u16), then the overlay's
    W.ov = ovc->v;
    W.wide = true;
    W.last = reinterpret_cast<uint4*>(reinterpret_cast<char*>(
                 const_cast<uint32_t*>(misc) + fast_misc_words(NW)) + F.ccap + kOvListBytes);
    if (ovc->sparse) {  // sparse lists after the counter region (bulk copies)
      uint2* sl = reinterpret_cast<uint2*>(reinterpret_cast<char*>(
                      const_cast<uint32_t*>(misc) + fast_misc_words(NW)) + F.ccap);
      const uint32_t bx = (8u * ovc->n_sx + 15u) & ~15u, bp = (8u * ovc->n_sbp + 15u) & ~15u;
      if (!bb) {
        for (uint32_t i = tid; i < ovc->n_sx; i += NT) sl[i] = __ldg(ovc->sx + i);
        for (uint32_t i = tid; i < ovc->n_sbp; i += NT) sl[kOvListMax + i] = __ldg(ovc->sbp + i);
      } else if (bx + bp) {
        if (tid == 0) {
          bulk_arm(*bb, bx + bp);
          if (bx) bulk_g2s(sl, ovc->sx, bx, *bb);
          if (bp) bulk_g2s(sl + kOvListMax, ovc->sbp, bp, *bb);
        }
        bulk_wait(*bb);
      }
      W.sxs = sl;
      W.sbps = sl + kOvListMax;
      W.n_sx = ovc->n_sx;
      W.n_sbp = ovc->n_sbp;
      W.ovmin = ovc->ovmin;
      W.sparse = true;
    }
    uint16_t* c16 = reinterpret_cast<uint16_t*>(cw);
    const uint32_t nb = ob->n_cnt, nc = nb + ovc->n_cnt;
    for (uint32_t i = tid; i < nc; i += NT)
      c16[i] = i < nb ? (ob->wide ? __ldg(reinterpret_cast<const uint16_t*>(ob->cnt0) + i)
                                  : static_cast<uint16_t>(__ldg(ob->cnt0 + i)))
                      : __ldg(ovc->cnt + (i - nb));
  } else {
    const uint32_t nv = ((info.wide ? 2u : 1u) * info.n_cnt + 15) / 16;
    const uint4* src = reinterpret_cast<const uint4*>(cnt0);
    uint4* dst = reinterpret_cast<uint4*>(cw);
    if (gcw || !bb) {  // global counter slice: a plain copy
      for (uint32_t i = tid; i < nv; i += NT) dst[i] = __ldg(src + i);
    } else if (nv) {  // the counter image into shared memory: one bulk copy
      if (tid == 0) {
        bulk_arm(*bb, 16u * nv);
        bulk_g2s(dst, src, 16u * nv, *bb);
      }
      bulk_wait(*bb);
    }
  }
  for (uint32_t d = tid; d < D; d += NT) {
    DevF z;
    z.head = z.tail = z.tsort = z.segbeg = 0;
    z.zlo = z.zhi = z.segt = 0;
    z.qoff = __ldg(W.devoff + d);
    z.busy_lo = z.busy_hi = z.isb = z.ise = 0;
    dv[d] = z;
  }
  if (tid < 4) misc[tid] = 0;
  misc[4 + tid] = 0;
  W.rlc = misc;  // sources never push ranges (no virtual sources)
  gsync<NW>();
  // ---- sources (replay.cpp:92-94). No virtual sources reach the fast path
  // (pack flags them), so there are no cascades and no init quirk. ----
  if constexpr (OV) {
    for (uint32_t k = tid; k < ovc->n_src; k += NT) {
      uint4 a = __ldg(ovc->src + k);
      const uint32_t s = W.resolve(a);
      W.ready(a, 0ull, s);
    }
  } else {
    for (uint32_t k = tid; k < info.n_src; k += NT) {
      const uint32_t s = __ldg(srcs + k);
      W.ready(__ldg(rec + s), 0ull, s);
    }
  }
  gsync<NW>();
  if (gany<NW>(misc[1] != 0)) return bail_code(misc[1]);
  for (uint32_t d = tid; d < D; d += NT) {  // t = 0 arrivals in index order
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
  gsync<NW>();

  // ---- dispatch(0) + event loop (replay.cpp:95-106) ----
  uint32_t iend[KD];  // in-flight end - t per owned device (kT32Inf: idle)
  uint4 pr0[KD], pr1[KD];  // the in-flight op's out-edge records (kRegPrefetch)
  uint32_t prn[KD];        // their count, kNoPre: push the range instead
  uint32_t zmask = 0, epoch = 0;
#pragma unroll
  for (int j = 0; j < KD; ++j) {
    iend[j] = kT32Inf;
    prn[j] = kNoPre;
    pr0[j] = pr1[j] = make_uint4(0, 0, 0, 0);
    const uint32_t d = tid + NT * j;
    if (d < D) {
      bool z = false;
      iend[j] = W.dispatch_dev(d, 0ull, 0u, kT32Inf, &z, pr0[j], pr1[j], prn[j]);
      if (z) zmask |= 1u << j;
    }
  }
  misc[4 + tid] = 0;  // all devices were just visited
  unsigned long long t = 0;
  uint32_t rpar = 0;
  for (;;) {
    PROF_T(p0);
    uint32_t lmin = kT32Inf;
#pragma unroll
    for (int j = 0; j < KD; ++j) lmin = min(lmin, iend[j]);
    bool zero_round;
    uint32_t dt;
    round_head<NW>(zmask != 0, lmin, red, par, zero_round, dt, tid);
    uint32_t freed = 0;
    if (!zero_round) {
      if (dt == kT32Inf) break;
      t += dt;
      ++epoch;
#pragma unroll
      for (int j = 0; j < KD; ++j)
        if (iend[j] != kT32Inf) iend[j] -= dt;  // offsets from the new t
    }
    PROF_T(p1);
    // range counters alternate by round: this round's was zeroed last round
    W.rlc = misc + 2 * (rpar & 1u);
    if (tid == 0) misc[2 * ((rpar + 1) & 1u)] = 0;
    ++rpar;
    if (zero_round) {
      // zero-duration ops dispatched last round complete now (same t)
      uint32_t zm = zmask;
      while (zm) {
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        DevF& s = dv[tid + NT * j];
        const uint4* r = W.ring(tid + NT * j);
        const uint32_t zh = s.zhi;
        if (kTailBytesPerDev && zh - s.zlo == 1u) {
          const uint2 e = W.zr[tid + NT * j];
          const uint32_t eb = e.x & ~kOvF;
          if (e.y > eb) W.push_range(e.x, e.y - eb);
        } else {
          for (uint32_t p = s.zlo; p < zh; ++p) {
            const uint4 e = r[p & (F.qc - 1)];
            const uint32_t eb = e.z & ~kOvF;
            if (e.w > eb) W.push_range(e.z, e.w - eb);
          }
        }
        *reinterpret_cast<volatile uint32_t*>(&s.zlo) = zh;
      }
      zmask = 0;
    } else {
#pragma unroll
      for (int j = 0; j < KD; ++j) {
        if (iend[j] == 0u) {
          iend[j] = kT32Inf;
          freed |= 1u << j;
          if (kRegPrefetch && OV && prn[j] != kNoPre) {  // records already in registers
            if (prn[j]) W.edge(pr0[j], t);
            if (prn[j] == 2u) W.edge(pr1[j], t);
          } else {
            const DevF& sd = dv[tid + NT * j];
            const uint32_t ez = sd.isb, ew = sd.ise;
            const uint32_t eb = ez & ~kOvF;
            if (ew > eb) W.push_range(ez, ew - eb);
          }
        }
      }
    }
    gsync<NW>();
    PROF_T(p2);
#ifdef DPRO_PROFILE
    const uint32_t nranges = *W.rlc & (W.kRlLong - 1u);
#endif
    if (const uint32_t bail = W.expand(t)) return bail;
    PROF_T(p3);
    const uint32_t todo = freed | misc[4 + tid];
    misc[4 + tid] = 0;
#pragma unroll
    for (int j = 0; j < KD; ++j) {
      if (todo & (1u << j)) {
        bool z = false;
        iend[j] = W.dispatch_dev(tid + NT * j, t, epoch, iend[j], &z, pr0[j], pr1[j], prn[j]);
        if (z) zmask |= 1u << j;
      }
    }
#ifdef DPRO_PROFILE
    gsync<NW>();
    PROF_T(p4);
    PROF_ADD(0, 1);
    PROF_ADD(1, zero_round ? 1 : 0);
    PROF_ADD(2, p1 - p0);
    PROF_ADD(3, p2 - p1);
    PROF_ADD(4, p3 - p2);
    PROF_ADD(5, p4 - p3);
    PROF_ADD(6, nranges);
    const uint32_t ndisp = gsum<NW>(todo != 0 ? 1u : 0u, red, par, tid);
    PROF_ADD(7, ndisp);
#endif
  }

  const uint32_t vc = gsum<NW>(W.vcount, red, par, tid);
  const uint32_t dc = gsum<NW>(W.dcount, red, par, tid);
  if (vc + dc != n) return kBailOther;  // cycle: the general path reports it exactly
  const unsigned long long T = gmax64<NW>(W.tmax, red, par, tid);
  for (uint32_t d = tid; d < D; d += NT) {
    S.busy[c.dev_off + d] =
        static_cast<long long>((static_cast<unsigned long long>(dv[d].busy_hi) << 32) |
                               dv[d].busy_lo);
    S.dhead[c.dev_off + d] = W.devoff[d] + dv[d].head;
  }
  if (tid == 0) {
    O.status[cid] = kOk;
    O.err[cid] = 0;
    O.makespan[cid] = static_cast<long long>(T);
  }
  return kDone;
}

// One CTA of NW warps per candidate, persistent over the batch.
// pass 0: every candidate; ring overflows are marked kRetry.
// pass 1: only kRetry candidates, with rings as deep as shared memory allows
// (one CTA per SM); anything still failing takes the general path.
// pass 2 (instead of 0, for batches of multi-million-op graphs whose device
// queues never fit the residency-sized rings): mark every candidate kRetry.
// work: [0] pass-0 counter, [1] general fallbacks, [2] pass-1 counter,
// [3] deep-ring retries.
template <int NW, int KD>
__global__ void DPRO_FAST_BOUNDS(NW, KD) replay_fast_kernel(
    const Cand* __restrict__ cands, int n_cands, Scratch S, Outs O, PackOut P,
    FastCfg F, int want_schedule, unsigned* work, int pass) {
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ int s_cid;
  __shared__ uint64_t s_bar;
  bulk_bar_init(&s_bar);
  BulkBar bb{&s_bar, 0u};
  // counters: [0] passes 0 and 2, [2] pass 1, [4] pass 3
  unsigned* counter = work + (pass == 1 ? 2 : pass == 3 ? 4 : 0);
  for (;;) {
    if (threadIdx.x == 0) s_cid = static_cast<int>(atomicAdd(counter, 1u));
    __syncthreads();
    const int cid = s_cid;
    __syncthreads();
    if (cid >= n_cands) break;
    if (pass == 1 && O.status[cid] != kRetry) continue;
    if (pass == 3 && O.status[cid] != kRetry2) continue;
    if (pass == 2) {  // large graphs: straight to the deep-ring pass
      if (threadIdx.x == 0) {
        O.status[cid] = kRetry;
        atomicAdd(work + 3, 1u);
      }
      continue;
    }
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
    uint32_t rc = kBailOther;
    if (info.not_fast == 0 && c.d <= F.dcap && c.d <= 32u * NW * KD)
      rc = replay_fast<NW, KD>(
          c, cid, P.rec + P.r_off[cid], P.erec + P.e_off[cid], P.cnt0 + P.c_off[cid],
          P.srcs + c.op_off, info, fsm, F, S, O, want_schedule != 0,
          (info.wide ? 2u : 1u) * info.n_cnt <= F.ccap
              ? nullptr
              : reinterpret_cast<uint32_t*>(P.gcnt + P.c_off[cid]),
          nullptr, nullptr, &bb);
    __syncthreads();
    if ((rc == kBailRing || rc == kBailRl) && (pass == 0 || pass == 1)) {
      if (threadIdx.x == 0) {
        O.status[cid] = pass == 0 ? kRetry : kRetry2;
        atomicAdd(work + 3, 1u);
        atomicAdd(work + (rc == kBailRing ? 5 : 6) + (pass == 1 ? 2 : 0), 1u);
      }
    } else if (rc != kDone) {  // the general kernel runs it after the passes
      if (threadIdx.x == 0) {
        O.status[cid] = kRetryGen;
        atomicAdd(work + 1, 1u);
      }
    }
    __syncthreads();
  }
}

// Overlay batches: one CTA of NW warps per candidate, persistent; the same
// passes as replay_fast_kernel (0: residency rings, 1: deep rings for the
// kRetry ones). Candidates the fast path cannot finish (kBailOther) are
// marked kRetryMat: the host re-runs them through the materialized path.
constexpr int kRetryMat = 10;

// pass 4: candidates flagged in order[n_cands + cid] (whole-graph rewrites,
// or sent to the global-ring pass by a previous replay), run first on a side
// stream with global rings so they
// overlap the residency pass instead of trailing it; hint[] records the
// candidates that reach the global-ring pass (count in work[11]).
template <int NW, int KD>
__global__ void DPRO_OV_BOUNDS(NW, KD) replay_ov_kernel(
    const Cand* __restrict__ cands, const OvCand* __restrict__ ovc, int n_cands, OvBase base,
    Scratch S, Outs O, uint8_t* gcnt, FastCfg F, int want_schedule, unsigned* work, int pass,
    unsigned* hint, const unsigned* order) {
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ int s_cid;
  __shared__ uint64_t s_bar;
  bulk_bar_init(&s_bar);
  BulkBar bb{&s_bar, 0u};
  unsigned* counter = work + (pass == 1 ? 2 : pass == 3 ? 4 : pass == 4 ? 10 : 0);
  for (;;) {
    if (threadIdx.x == 0) {
      // order: the batch's long candidates first, so they overlap the rest
      const unsigned k = atomicAdd(counter, 1u);
      s_cid = k < static_cast<unsigned>(n_cands) ? static_cast<int>(order[k]) : n_cands;
    }
    __syncthreads();
    const int cid = s_cid;
    __syncthreads();
    if (cid >= n_cands) break;
    const bool side = order[n_cands + cid] != 0u;
    if (pass == 0 && side) continue;
    if (pass == 1 && O.status[cid] != kRetry) continue;
    if (pass == 3 && O.status[cid] != kRetry2) continue;
    if (pass == 4 && !side) continue;
    const Cand c = cands[cid];
    const OvCand oc = ovc[cid];
    if (oc.pad) continue;  // materialized path (host)
    if (oc.first_missing != kNone) {  // replay.cpp:39-44
      if (threadIdx.x == 0) {
        O.status[cid] = kMissing;
        O.err[cid] = oc.first_missing;
        O.makespan[cid] = 0;
      }
      continue;
    }
    PackInfo info{};
    info.first_missing = kNone;
    const uint32_t nc2 = 2u * (base.n_cnt + oc.n_cnt);
    uint32_t rc = kBailOther;
    if (c.d <= F.dcap && c.d <= 32u * NW * KD)
      rc = replay_fast<NW, KD, true>(
          c, cid, base.rec, base.erec, nullptr, nullptr, info, fsm, F, S, O,
          want_schedule != 0,
          nc2 <= F.ccap ? nullptr : reinterpret_cast<uint32_t*>(gcnt + oc.gcnt_off), &oc, &base,
          &bb);
    __syncthreads();
    if (threadIdx.x == 0) {
      if ((rc == kBailRing || rc == kBailRl) && (pass == 0 || pass == 1)) {
        O.status[cid] = pass == 0 ? kRetry : kRetry2;
        atomicAdd(work + 3, 1u);
        atomicAdd(work + (rc == kBailRing ? 5 : 6) + (pass == 1 ? 2 : 0), 1u);
        if (pass == 1) hint[atomicAdd(work + 11, 1u)] = static_cast<unsigned>(cid);
      } else if (rc != kDone) {
        O.status[cid] = kRetryMat;
        atomicAdd(work + 1, 1u);
      }
    }
    __syncthreads();
  }
}

}  // namespace dpro_k
