// Candidate overlays on the resident base layout (engine-internal).
//
// A delta candidate (include/dpro_cuda.h dpro_delta) is replayed directly on
// the resident base graph's packed records (pack_kernel.cuh layout, built
// once per base) plus a small per-candidate overlay, instead of merging and
// packing a private copy of the whole graph: for config 4 (4.8M ops) a
// private copy is ~290 MB per candidate, the overlay of an op-fusion
// candidate a few KB, so ~8x more candidates fit in HBM at once -- and the
// replay is latency-bound per candidate, so concurrency is throughput.
//
// Ops are addressed by base index b (kept base ops) or by overlay slot.
// A kept base op is PURE when its record and its expanded successor list
// are unchanged (same in-degree, no removed / cut / extra out-edge, no
// changed spliced virtual successor); its base record is used as is.
// Every other kept op ("dirty") and every new op gets an overlay record
// and an overlay list. The replay resolves a base-form record of op b via
// the block table: blk[b >> 10] is either a uniform index shift for the
// block (final(b) = b + shift) or a pointer to 1024 per-op entries (final
// index, or kOvfDirty | slot for a dirty op). Overlay-form records carry
// their slot in x and kOv in w; their final index is fin[slot].
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "dpro_cuda.h"

namespace dpro_ov {

constexpr uint32_t kOv = 0x80000000u;        // record w / range flag: overlay list
constexpr uint32_t kBlkShift = 10;
constexpr uint32_t kBlk = 1u << kBlkShift;
constexpr uint32_t kBlkOvf = 0x80000000u;    // blk entry: ovf block index follows
constexpr uint32_t kBlkBias = 0x40000000u;   // clean blk entry: shift + kBlkBias
constexpr uint32_t kOvfDirty = 0x80000000u;  // ovf entry: dirty, overlay slot follows
constexpr uint32_t kOvfNone = 0xFFFFFFFFu;   // ovf entry of a removed op
// sparse form: at most this many dirty ops and shift runs (the kernel keeps
// both lists in shared memory: replay_fast.cuh kOvListMax)
constexpr uint32_t kSparseMax = 48;

// The base as the overlay builder needs it (host copies, built once).
struct BaseHost {
  uint32_t n = 0, e = 0, d = 0;
  std::vector<int64_t> dur;
  std::vector<uint16_t> dev;
  std::vector<uint8_t> flags;
  std::vector<uint32_t> succ_off, succ, indeg;
  std::vector<uint32_t> pred_off, pred;  // transposed CSR
  std::vector<uint32_t> rec;             // packed records, 4 words per op (n + 1)
  std::vector<uint32_t> devcnt;          // non-virtual ops per device
  std::vector<uint32_t> srcs;            // ops without predecessors, ascending
  std::vector<uint32_t> missing;         // non-virtual ops with dur < 0, ascending
  uint32_t n_cnt = 0;                    // base counters (multi-predecessor ops)
  bool wide = false;                     // base counters are u16
  bool ok = false;                       // base packed for the fast path
};

// One candidate's overlay (host side, uploaded as is).
struct OverlayHost {
  std::vector<uint32_t> rec;   // 4 words per overlay op (+ sentinel)
  std::vector<uint32_t> erec;  // 4 words per expanded list entry
  std::vector<uint32_t> fin;   // final index per overlay op
  std::vector<uint16_t> cnt;   // initial counts of the overlay counters
  std::vector<uint32_t> src;   // 4 words per source record
  std::vector<uint32_t> blk;   // per 1024-id base block
  std::vector<uint32_t> ovf;   // 1024 entries per flagged block
  std::vector<uint32_t> devoff;  // timeline regions [n_devices + 1]
  // sparse form (few dirty ops and index shifts: op-fusion / partition
  // candidates), read from shared memory: (base id, slot) of the dirty ops
  // and (first base id, shift) runs of the final-index shift, both sorted;
  // base ids below ovmin are pure with final index == base index
  std::vector<uint32_t> sx, sbp;
  uint32_t ovmin = 0;
  bool sparse = false;
  uint32_t n_ops = 0, n_devices = 0;
  uint32_t first_missing = UINT32_MAX;  // final index, UINT32_MAX: none
  bool fast = true;            // false: needs the materialized path
  std::string why;             // reason when !fast
};

// Builds the overlay of delta D; scratch vectors are reused per thread.
void build_overlay(const BaseHost& B, const dpro_delta& D, OverlayHost& O);

}  // namespace dpro_ov
