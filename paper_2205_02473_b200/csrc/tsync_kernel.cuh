// K2: the comm-only graphs of sync_makespan(cluster, bytes, k)
// (proj/src/replay.cpp:228-246: k balanced partitions "tsync" / "tsync#p<i>"
// of `bytes`, each expanded by expand_tensor, ingest.cpp:268-373) generated
// directly in the reference's index order on the GPU, one CTA per (bytes, k)
// pair, straight into the CSR arrays the replay kernels read.
//
// The index order is the byte order of the op ids. For a ring the ids are
// "<RECV|SEND>.tsync[#p<i>]#c<c>#s<s>#<src>#<dst>": (p, c, s) fixes the op
// of each kind, and the decimal fields compare as strings with '#' after
// them ("#s1#" < "#s10" < "#s2#"), so index = kind * kCS + rank(p) * CS +
// rank(c) * S + rank(s) with rank() = position of the decimal string among
// the field's values in byte order (host tables). For a parameter server the
// ids are "<kind>.tsync[#p<i>]#pull#<server>#<w>" (< "#push#") and
// "...#push#<w>#<server>": per partition the pull ops of every worker, then
// the push ops, each in the host-computed byte order of the worker names.
#pragma once

#include <cstdint>

namespace dpro_k {

struct TsyncDesc {        // one (bytes, k) pair
  long long bytes;
  int k;
  uint32_t n, e;          // ops, edges
  unsigned long long op_off, e_off;
};

struct TsyncRing {
  int n_workers, chunks, steps;      // ring size, C, S = 2 (n - 1)
  const int* rank_c;                 // [C] rank of c among 0..C-1 (decimal order)
  const int* inv_c;                  // [C] c of a rank
  const int* rank_s;                 // [S]
  const int* inv_s;
  const int* inv_p;                  // [kmax] p of a rank (per k: ranks of 0..k-1)
  const int* inv_p_off;              // [kmax + 1] offset of k's table in inv_p
  const uint16_t* link_dev;          // [n] dense device of ring link i (ring[i] -> ring[i+1])
  const double* link_bw;             // [n]
  const double* link_lat;            // [n]
};

struct TsyncPs {
  int n_workers;
  const int* inv_p;                  // as in TsyncRing
  const int* inv_p_off;
  const int* server_of;              // [k_off + p]: server index of partition p
  const int* srv_off;                // [kmax + 1] offset of k's server table
  const int* pull_w;                 // [n_servers * W] worker (sorted index) at pull rank, per server
  const int* push_w;                 // [n_servers * W] worker at push rank, per server
  const int* dev_off;                // [kmax + 1] offset of k's device tables (dense ids
                                     // depend on the servers k's partitions use)
  const uint16_t* dev_push;          // [dev_off[k] + server * W + w] dense device of w -> server
  const uint16_t* dev_pull;          // [dev_off[k] + server * W + w] dense device of server -> w
  const double* bw_push;             // [n_servers * W]
  const double* lat_push;
  const double* bw_pull;
  const double* lat_pull;
};

struct TsyncOut {
  long long* dur;        // [sum n]
  uint16_t* dev;
  uint8_t* flags;
  uint32_t* succ_off;    // [sum (n + 1)]: per candidate n + 1 entries at op_off + index
  uint32_t* succ;        // [sum e]
  uint32_t* indeg;       // [sum n]
};

// hop_dur (ingest.cpp:37-48) + round_us (time_util.hpp:28-35): IEEE double
// division and add (no fast math), then round half to even.
__device__ __forceinline__ long long tsync_hop(long long bytes, double bw, double lat) {
  const double v = __dadd_rn(__ddiv_rn(static_cast<double>(bytes), bw), lat);
  const double f = floor(v);
  const double frac = v - f;
  const long long lo = static_cast<long long>(f);
  if (frac > 0.5) return lo + 1;
  if (frac < 0.5) return lo;
  return (lo % 2 == 0) ? lo : lo + 1;
}

constexpr uint8_t kTsyncComm = 2;  // DPRO_FLAG_COMM

__global__ void __launch_bounds__(256) tsync_ring_kernel(const TsyncDesc* __restrict__ cands,
                                                         int n_cands, TsyncRing R, TsyncOut O) {
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const TsyncDesc c = cands[cid];
    const int k = c.k, C = R.chunks, S = R.steps, N = R.n_workers;
    const uint32_t CS = static_cast<uint32_t>(C) * S, kCS = static_cast<uint32_t>(k) * CS;
    const int* invp = R.inv_p + R.inv_p_off[k];
    long long* dur = O.dur + c.op_off;
    uint16_t* dev = O.dev + c.op_off;
    uint8_t* flags = O.flags + c.op_off;
    uint32_t* soff = O.succ_off + c.op_off + cid;  // n + 1 entries per candidate
    uint32_t* succ = O.succ + c.e_off;
    uint32_t* indeg = O.indeg + c.op_off;
    const long long pbase = c.bytes / k, prem = c.bytes % k;
    const int last_rank = R.rank_s[S - 1];  // the RECV without a successor in each (p, c)
    for (uint32_t i = threadIdx.x; i < 2 * kCS; i += blockDim.x) {
      const bool send = i >= kCS;
      const uint32_t j = send ? i - kCS : i;
      const uint32_t pr = j / CS, cr = (j / S) % C, sr = j % S;
      const int p = invp[pr], ch = R.inv_c[cr], s = R.inv_s[sr];
      const long long pb = pbase + (p < prem ? 1 : 0);
      const long long cb = pb / C + (ch < pb % C ? 1 : 0);
      const int link = (ch + s) % N;  // ring[link] -> ring[link + 1]
      dev[i] = R.link_dev[link];
      flags[i] = kTsyncComm;
      dur[i] = send ? 0 : tsync_hop(cb, R.link_bw[link], R.link_lat[link]);
      // successor lists: SEND(p,c,s) -> RECV(p,c,s); RECV(p,c,s) -> SEND(p,c,s+1)
      const uint32_t grp = pr * C + cr;  // (p, c) group index
      if (send) {
        soff[i] = (kCS - static_cast<uint32_t>(k) * C) + j;
        succ[soff[i]] = j;  // its RECV
        indeg[i] = s > 0 ? 1u : 0u;
      } else {
        soff[i] = j - grp - (sr > static_cast<uint32_t>(last_rank) ? 1u : 0u);
        if (s + 1 < S) succ[soff[i]] = kCS + grp * S + R.rank_s[s + 1];
        indeg[i] = 1u;
      }
    }
    if (threadIdx.x == 0) soff[2 * kCS] = c.e;
  }
}

__global__ void __launch_bounds__(256) tsync_ps_kernel(const TsyncDesc* __restrict__ cands,
                                                       int n_cands, TsyncPs P, TsyncOut O) {
  for (int cid = blockIdx.x; cid < n_cands; cid += gridDim.x) {
    const TsyncDesc c = cands[cid];
    const int k = c.k, W = P.n_workers;
    const uint32_t per = 2u * W;  // ops of one kind in one partition (pull W + push W)
    const uint32_t half = static_cast<uint32_t>(k) * per;  // RECV ops, then SEND ops
    const int* invp = P.inv_p + P.inv_p_off[k];
    const int* srv = P.server_of + P.srv_off[k];
    long long* dur = O.dur + c.op_off;
    uint16_t* dev = O.dev + c.op_off;
    uint8_t* flags = O.flags + c.op_off;
    uint32_t* soff = O.succ_off + c.op_off + cid;
    uint32_t* succ = O.succ + c.e_off;
    uint32_t* indeg = O.indeg + c.op_off;
    const long long pbase = c.bytes / k, prem = c.bytes % k;
    // successor counts: push RECV -> every pull SEND of its partition (W);
    // pull SEND -> pull RECV (1); push SEND -> push RECV (1); pull RECV -> none
    for (uint32_t i = threadIdx.x; i < 2 * half; i += blockDim.x) {
      const bool send = i >= half;
      const uint32_t j = send ? i - half : i;
      const uint32_t pr = j / per, q = j % per;
      const bool push = q >= static_cast<uint32_t>(W);
      const uint32_t wr = push ? q - W : q;
      const int p = invp[pr], sv = srv[pr];
      const long long pb = pbase + (p < prem ? 1 : 0);
      const int w = push ? P.push_w[sv * W + wr] : P.pull_w[sv * W + wr];
      const uint32_t slot = static_cast<uint32_t>(sv) * W + w;
      dev[i] = push ? P.dev_push[P.dev_off[k] + slot] : P.dev_pull[P.dev_off[k] + slot];
      flags[i] = kTsyncComm;
      dur[i] = send ? 0 : (push ? tsync_hop(pb, P.bw_push[slot], P.lat_push[slot])
                                : tsync_hop(pb, P.bw_pull[slot], P.lat_pull[slot]));
      // list offsets: RECVs first (push RECVs carry W successors each)
      const uint32_t recv_edges_before_p = pr * static_cast<uint32_t>(W) * W;
      uint32_t off;
      if (!send) {
        off = recv_edges_before_p + (push ? wr * W : 0u);
      } else {
        off = static_cast<uint32_t>(k) * W * W + j;
      }
      soff[i] = off;
      if (!send && push) {  // -> every pull SEND of partition pr (ascending)
        for (int x = 0; x < W; ++x) succ[off + x] = half + pr * per + x;
      } else if (send) {
        succ[off] = j;  // its RECV
      }
      indeg[i] = send ? (push ? 0u : static_cast<uint32_t>(W)) : 1u;
    }
    if (threadIdx.x == 0) soff[2 * half] = c.e;
  }
}

}  // namespace dpro_k
