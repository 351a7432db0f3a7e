/* dpro_cuda.h -- C ABI of the B200 Replayer (libdpro_cuda.so).
 *
 * Drop-in boundary for the reference's replay operator API,
 * proj/include/dpro/replay.hpp:48-91. The reference keeps its C++ signatures
 * (replay / execution_graph / critical_path / sync_makespan / partial_replay);
 * a thin adapter marshals GlobalDFG into the index-ordered
 * CSR below and calls these entry points. Plain C: no exceptions, no torch or
 * STL types, caller-owned buffers, status codes instead of throws.
 *
 * Index order is the reference op index (byte-lexicographic op id order,
 * proj/src/graph.cpp:278-297); succ lists ascending (graph.cpp:290-295);
 * dense device ids in DeviceId order (graph.hpp:57-72). Times are integers in
 * the caller's unit (the reference's microseconds, or ns): replay only adds
 * and compares durations, so any integer unit is exact.
 *
 * Status codes map onto the reference exceptions:
 *   DPRO_MISSING_PROFILE  MissingProfileError  (replay.cpp:39-44)
 *                         err = index of the first non-virtual op with dur<0
 *   DPRO_CYCLE            CycleError           (replay.cpp:108-117)
 *                         err = number of ops never scheduled
 *   DPRO_EINVAL           dpro::Error          (e.g. sync_makespan k<1,
 *                         replay.cpp:229-232) or a malformed CSR
 */
#ifndef DPRO_CUDA_H_
#define DPRO_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPRO_ABI_VERSION 1

enum dpro_status {
  DPRO_OK = 0,
  DPRO_MISSING_PROFILE = 1,
  DPRO_CYCLE = 2,
  DPRO_EINVAL = 3,
  DPRO_ECUDA = 4,
  DPRO_ENOMEM = 5,
  DPRO_EUNSUPPORTED = 6
};

enum dpro_memspace { DPRO_HOST = 0, DPRO_DEVICE = 1 };

/* op flag bits (dpro::OpKind, proj/include/dpro/graph.hpp:30-50) */
#define DPRO_FLAG_VIRTUAL 0x1u /* kVirtualIn / kVirtualOut          */
#define DPRO_FLAG_COMM 0x2u    /* kSend / kRecv (is_communication) */

/* One candidate data flow graph (GlobalDFG, graph.hpp:110-160) as CSR. */
typedef struct dpro_csr {
  uint32_t n_ops;
  uint32_t n_edges;
  uint32_t n_devices;         /* dense device ids are < n_devices         */
  int32_t dur_bits;           /* 64: int64_t dur (dpro::Us), 32: int32_t  */
  const void* dur;            /* [n_ops] op duration (virtual: ignored)   */
  const uint16_t* dev;        /* [n_ops] dense device id                  */
  const uint8_t* flags;       /* [n_ops] DPRO_FLAG_*                      */
  const uint32_t* succ_off;   /* [n_ops+1]                                */
  const uint32_t* succ;       /* [n_edges] ascending within each op       */
  const uint32_t* indeg;      /* [n_ops] |preds|, or NULL (computed)      */
} dpro_csr;

/* ClusterSpec (proj/include/dpro/cluster.hpp:43-65). */
typedef struct dpro_cluster_desc {
  int32_t scheme;                /* 0 ring all-reduce, 1 parameter server */
  int32_t n_nodes;
  const char* const* node_ids;   /* [n_nodes]                             */
  const int32_t* node_role;      /* [n_nodes] 0 worker, 1 ps              */
  int32_t n_links;
  const int32_t* link_src;       /* [n_links] node index                  */
  const int32_t* link_dst;
  const double* link_bw;         /* bytes per time unit                   */
  const double* link_lat;        /* time units                            */
  int32_t n_ring;                /* 0: workers in byte-lexicographic order */
  const int32_t* ring_order;     /* [n_ring] node indices                 */
  int32_t chunks_per_tensor;     /* 0: ring size                          */
} dpro_cluster_desc;

/* ------------------------------------------------------------------------
 * Engine context: one per GPU; used by one host thread at a time.
 * --------------------------------------------------------------------- */
typedef struct dpro_ctx dpro_ctx;
typedef struct dpro_batch dpro_batch;

int dpro_cuda_abi_version(void);
dpro_ctx* dpro_cuda_create(int device);
void dpro_cuda_destroy(dpro_ctx* ctx);
/* cudaStream_t the engine launches on (NULL: the legacy default stream). */
int dpro_cuda_set_stream(dpro_ctx* ctx, void* stream);
/* Engine options: "fast" (1: on-chip fast path with exact fallback, 0: the
 * general kernel only), "ring" (fast-path queue capacity per device, power
 * of two), "warps" (1, 2, 4 or 8 warps = one CTA cooperating on a candidate in
 * the fast path; 0 = by device count, the default), "gcnt" (1: fast-path
 * counters always in global scratch), "deep_first" (-1 auto, 0 never, 1
 * always start in the deep-ring pass), "host_threads" (host pool size for
 * delta batches; 0 = all hardware threads), "overlay" (1: delta batches
 * replay on the resident base + per-candidate overlays), "tsync_host" (1:
 * t_sync graphs built on host threads instead of on the GPU). Returns
 * DPRO_EINVAL for unknown keys or values. */
int dpro_cuda_set_option(dpro_ctx* ctx, const char* key, int64_t value);
const char* dpro_cuda_last_error(dpro_ctx* ctx);

/* ------------------------------------------------------------------------
 * Batched replay (replaces dpro::replay, replay.cpp:37-134, for B graphs).
 * --------------------------------------------------------------------- */

/* Registers a batch. memspace DPRO_HOST: the CSR arrays are uploaded into
 * one engine-owned device arena (dur packed to int32 when it fits).
 * DPRO_DEVICE: the arrays are used in place (must stay alive). */
dpro_batch* dpro_cuda_batch_create(dpro_ctx* ctx, const dpro_csr* cands,
                                   int32_t n_cands, int32_t memspace);
void dpro_cuda_batch_destroy(dpro_ctx* ctx, dpro_batch* b);
/* Replays every candidate on the GPU (stream-ordered, asynchronous).
 * want_schedule=0 skips the per-op start/end writes (makespan only). */
int dpro_cuda_batch_replay(dpro_ctx* ctx, dpro_batch* b, int32_t want_schedule);
/* Device pointers of the batch results (valid until the next replay):
 * makespan/err [n_cands] int64, status [n_cands] int32, start/end
 * concatenated per candidate in batch order ([sum n_ops] int64). */
int dpro_cuda_batch_device_results(dpro_batch* b, int64_t** makespan,
                                   int32_t** status, int64_t** err,
                                   int64_t** start, int64_t** end);
/* Copies results to host buffers (any may be NULL); synchronizes. */
int dpro_cuda_batch_results(dpro_ctx* ctx, dpro_batch* b, int64_t* makespan,
                            int32_t* status, int64_t* err, int64_t* start,
                            int64_t* end);
/* Per-device dispatch order of candidate `cand` after a replay
 * (ReplayResult::device_timelines): order[dev_off[d]..dev_off[d+1]) are the
 * op indices device d ran, in order; busy[d] = summed dur (utilization
 * numerator, replay.cpp:124-132). Host buffers: order [n_ops],
 * dev_off [n_devices+1], busy [n_devices]; any may be NULL. */
int dpro_cuda_batch_timelines(dpro_ctx* ctx, dpro_batch* b, int32_t cand,
                              uint32_t* order, uint32_t* dev_off,
                              int64_t* busy);
/* Counters of the last replay: stats[0] = candidates that took the general
 * (fallback) path, stats[1] = fast-path shared memory bytes per candidate,
 * stats[2] = fast-path candidates resident per SM, stats[3] = ring capacity
 * per device, stats[4] = candidates re-run with deep rings (second pass).
 * stats must hold 5 entries. */
int dpro_cuda_batch_stats(dpro_ctx* ctx, dpro_batch* b, int64_t* stats);
/* Diagnostics of the last replay, up to n of: [0] pass-0 ring overflows,
 * [1] pass-0 range-list overflows, [2] / [3] the same in the deep-ring pass,
 * [4] 1 for an overlay batch, [5] overlay candidates on the materialized
 * path, [6..9] microseconds of pass 0, the deep-ring pass, the global-ring
 * pass and the general-kernel hand-off (-1: not timed). */
int dpro_cuda_batch_diag(dpro_ctx* ctx, dpro_batch* b, int64_t* out, int32_t n);
/* scheduled[i] = 1 for ops the replay scheduled (host buffer [n_ops]); the
 * ids with 0 form CycleError::cycle (replay.cpp:108-117). */
int dpro_cuda_batch_scheduled(dpro_ctx* ctx, dpro_batch* b, int32_t cand,
                              uint8_t* scheduled);
/* critical_path(execution_graph(g, r), r) (replay.cpp:136-226) for every
 * candidate of the last replay. paths: concatenated per candidate with
 * capacity n_ops each (same offsets as start/end); path_len [n_cands].
 * Host buffers. */
int dpro_cuda_batch_critical_paths(dpro_ctx* ctx, dpro_batch* b,
                                   uint32_t* paths, int64_t* path_len);

/* estimate_peak_memory (proj/src/memory.cpp:122-167) for every candidate of
 * the last replay (want_schedule=1), on the schedule already in HBM. Host
 * inputs, flat in batch order: op_bytes [sum n_ops] output buffer bytes of
 * each computation op (0: none; the caller resolves output_bytes_for and
 * raises MissingMetaError), op_node [sum n_ops] dense compute node of each
 * computation op (-1 for other ops), n_nodes [n_cands], persistent
 * [sum n_nodes]. Output peak [sum n_nodes]: persistent + max live bytes. */
int dpro_cuda_batch_peak_memory(dpro_ctx* ctx, dpro_batch* b,
                                const int64_t* op_bytes, const int32_t* op_node,
                                const int32_t* n_nodes, const int64_t* persistent,
                                int64_t* peak);

/* critical_path(exec_graph, result) (replay.cpp:146-226) for ONE graph and
 * a caller-supplied schedule (start/end per op, makespan): the exact
 * reference signature, where the execution graph already contains the
 * timeline edges. Host buffers; path capacity n_ops. */
int dpro_cuda_critical_path(dpro_ctx* ctx, const dpro_csr* graph,
                            const int64_t* start, const int64_t* end,
                            int64_t makespan, uint32_t* path,
                            int64_t* path_len);

/* One-shot convenience with the reference-style signature: create, replay,
 * copy back (host outputs), destroy. start/end may be NULL. */
int dpro_cuda_replay_batch(dpro_ctx* ctx, const dpro_csr* cands,
                           int32_t n_cands, int32_t memspace,
                           int64_t* makespan, int64_t* start, int64_t* end,
                           int32_t* status, int64_t* err);

/* ------------------------------------------------------------------------
 * Resident base graph + per-candidate deltas (SURVEY 7 "Scale", 8(f) row
 * 1). The search's candidates differ from one base graph in a few units, so
 * the base CSR is uploaded once and stays in HBM (and L2); a batch uploads
 * only each candidate's delta and the engine merges it on the GPU into the
 * index-ordered CSR the replay kernels read. No counterpart in the
 * reference, whose search builds every candidate with a GraphBuilder copy
 * (optimize.cpp:1211-1227, 1382-1392).
 *
 * A candidate = base minus `removed` base ops (and their edges) minus the
 * `cut` base edges plus `n_new` ops, in the base's index order: new op j
 * sits before base op new_pos[j] (its lower_bound among the base ids); new
 * ops sharing a position keep their order. Final indices: kept base op b ->
 * b - #removed<b + #new_pos<=b; new op j -> new_pos[j] - #removed<new_pos[j]
 * + j. Added edges: out of new ops in new_succ, out of kept base ops in
 * extra_src/extra_dst; destinations are final indices.
 * --------------------------------------------------------------------- */
typedef struct dpro_delta {
  uint32_t n_devices;            /* base dense ids, new devices appended    */
  uint32_t n_removed;
  const uint32_t* removed;       /* [n_removed] ascending base indices      */
  uint32_t n_new;
  const uint32_t* new_pos;       /* [n_new] non-decreasing, <= base n_ops   */
  const int64_t* new_dur;        /* [n_new]                                 */
  const uint16_t* new_dev;       /* [n_new]                                 */
  const uint8_t* new_flags;      /* [n_new] DPRO_FLAG_*                     */
  const uint32_t* new_succ_off;  /* [n_new+1]                               */
  const uint32_t* new_succ;      /* final indices, ascending per op         */
  uint32_t n_extra;
  const uint32_t* extra_src;     /* [n_extra] kept base index, ascending    */
  const uint32_t* extra_dst;     /* [n_extra] final index, ascending per src;
                                    never a kept, uncut base successor of src */
  uint32_t n_cut;
  const uint32_t* cut;           /* [n_cut] ascending positions in the base
                                    succ[] of dropped edges between kept ops */
} dpro_delta;

typedef struct dpro_resident dpro_resident;
/* Uploads a base graph (host CSR) to HBM; it stays resident until destroyed. */
dpro_resident* dpro_cuda_resident_create(dpro_ctx* ctx, const dpro_csr* base);
void dpro_cuda_resident_destroy(dpro_ctx* ctx, dpro_resident* r);
/* A batch of n candidates given as host deltas against r: H2D copies of
 * the deltas, the merge on the GPU, then the same packing as
 * dpro_cuda_batch_create. The batch holds merged copies; r must stay alive
 * only while dpro_cuda_batch_prepare may be called on the batch. */
dpro_batch* dpro_cuda_batch_create_delta(dpro_ctx* ctx, const dpro_resident* r,
                                         const dpro_delta* deltas, int32_t n);
/* Per-candidate op / edge / device counts of a registered batch (any
 * argument may be NULL). */
int dpro_cuda_batch_sizes(dpro_batch* b, uint32_t* n_ops, uint32_t* n_edges,
                          uint32_t* n_devices);
/* Pack diagnostics, 4 words per candidate: first op without a duration
 * (UINT32_MAX: none), fast-path ineligibility bits (pack_kernel.cuh kNf*),
 * multi-predecessor ops, source ops. */
int dpro_cuda_batch_pack_info(dpro_batch* b, uint32_t* out);
/* Re-runs a batch's device-side preparation on the inputs already in HBM
 * (delta merge for delta batches, then the pack kernel): with a replay, one
 * full pass of the path without host work -- what bench.py times. */
int dpro_cuda_batch_prepare(dpro_ctx* ctx, dpro_batch* b);
/* One-shot: create from deltas, replay (makespan only), copy back, destroy. */
int dpro_cuda_replay_delta_batch(dpro_ctx* ctx, const dpro_resident* r,
                                 const dpro_delta* deltas, int32_t n,
                                 int64_t* makespan, int32_t* status, int64_t* err);

/* ------------------------------------------------------------------------
 * t_sync grid (replaces sync_makespan, replay.cpp:228-246, and the memoized
 * SearchCtx::sync grid of optimize.cpp:562-576,1170-1194): out[i] =
 * makespan of syncing bytes[i] as k[i] balanced partitions under the
 * cluster's scheme. status[i] = DPRO_EINVAL when k[i] < 1.
 * --------------------------------------------------------------------- */
int dpro_cuda_tsync_grid(dpro_ctx* ctx, const dpro_cluster_desc* cluster,
                         const int64_t* bytes, const int32_t* k, int32_t n,
                         int64_t* out, int32_t* status);
/* The comm-only graphs of the same grid as a batch (K2: generated on the GPU
 * straight into CSR, in the reference's index order -- no host graph, no
 * upload): replay / results / timelines / critical paths as for any batch.
 * NULL with dpro_cuda_last_error set for k < 1 or a degenerate cluster. */
dpro_batch* dpro_cuda_batch_create_tsync(dpro_ctx* ctx, const dpro_cluster_desc* cluster,
                                         const int64_t* bytes, const int32_t* k, int32_t n);

/* ------------------------------------------------------------------------
 * Host-side CSR graph construction (candidate generation; no GPU needed).
 * Builds the same graph the reference ingest/rewrite path builds
 * (ingest.cpp:187-454, optimize.cpp:459-492) directly in index order.
 * --------------------------------------------------------------------- */
typedef struct dpro_graph dpro_graph;

/* Layered data-parallel model of proj/src/synth.cpp:200-217: FW chain,
 * mirrored BW chain producing tensor g<i> per layer, UPDATE.l<i> gated on
 * OUT(g<i>). */
typedef struct dpro_layered_model {
  int32_t layers;
  const int64_t* fw_dur;        /* [layers] */
  const int64_t* bw_dur;        /* [layers] */
  const int64_t* tensor_bytes;  /* [layers] */
  int64_t update_dur;
} dpro_layered_model;

/* part_k: [layers] partition count per tensor (NULL: all 1), as applied by
 * apply_tensor_partition (optimize.cpp:459-492). */
dpro_graph* dpro_graph_layered(const dpro_layered_model* model,
                               const dpro_cluster_desc* cluster,
                               const int32_t* part_k, int32_t* status);
/* Tensor-fusion + partition candidate: n_groups synchronization units; unit
 * q fuses layers members[group_off[q] .. group_off[q+1]) in that order
 * (apply_tensor_fusion, optimize.cpp:366-455: unit "g3+g4" feeds every
 * member's UPDATE and waits for every member's BW) and is partitioned
 * group_k[q] ways (NULL: 1). The groups must partition the layers. */
dpro_graph* dpro_graph_layered_groups(const dpro_layered_model* model,
                                      const dpro_cluster_desc* cluster,
                                      int32_t n_groups, const int32_t* group_off,
                                      const int32_t* members,
                                      const int32_t* group_k, int32_t* status);
/* n fusion/partition candidates on `threads` host threads. Candidate i owns
 * groups [spec_off[i], spec_off[i] + n_groups[i]) of the flattened arrays:
 * group g spans members[group_off[g] .. group_off[g+1]) with partition
 * count group_k[g]. */
int dpro_graph_layered_groups_batch(const dpro_layered_model* model,
                                    const dpro_cluster_desc* cluster, int32_t n,
                                    const int32_t* n_groups, const int64_t* spec_off,
                                    const int32_t* group_off, const int32_t* members,
                                    const int32_t* group_k, int32_t threads,
                                    dpro_graph** out);
/* Delta construction: a base layered graph (every
 * tensor its own unit, k = 1) built once; candidates are then produced as
 * base minus their changed units' ops plus the re-expanded ones, merged into
 * the base index order -- the same CSR a full rebuild gives, without
 * re-naming and re-sorting the unchanged ops. Spec arrays as in
 * dpro_graph_layered_groups_batch. */
typedef struct dpro_base dpro_base;
dpro_base* dpro_base_layered(const dpro_layered_model* model,
                             const dpro_cluster_desc* cluster, int32_t* status);
void dpro_base_free(dpro_base* base);
int dpro_graph_from_base_batch(const dpro_base* base, int32_t n,
                               const int32_t* n_groups, const int64_t* spec_off,
                               const int32_t* group_off, const int32_t* members,
                               const int32_t* group_k, int32_t threads,
                               dpro_graph** out);
/* The same candidates as dpro_graph_from_base_batch, left as deltas against
 * the base graph (dpro_delta, above) for dpro_cuda_batch_create_delta: only
 * the changed units' ops are named, sorted and placed; the O(V) merge runs
 * on the GPU. Device ids are the base graph's (new devices appended). */
typedef struct dpro_delta_set dpro_delta_set;
int dpro_base_delta_batch(const dpro_base* base, int32_t n,
                          const int32_t* n_groups, const int64_t* spec_off,
                          const int32_t* group_off, const int32_t* members,
                          const int32_t* group_k, int32_t threads,
                          dpro_delta_set** out);
/* The same with op fusion on every worker (optimize.cpp:245-317, applied
 * left to right with the default cost model, ratio 0.8): fw_join[c*(L-1)+i]
 * fuses FW.l<i> with FW.l<i+1>, bw_join[c*(L-1)+i] fuses BW.l<i+1> with
 * BW.l<i> in candidate c (NULL: none). Fused ids are the reference's
 * ("w0->FW.l3+FW.l4", "w0->BW.l4+BW.l3"). */
int dpro_base_delta_batch_ops(const dpro_base* base, int32_t n,
                              const int32_t* n_groups, const int64_t* spec_off,
                              const int32_t* group_off, const int32_t* members,
                              const int32_t* group_k, const uint8_t* fw_join,
                              const uint8_t* bw_join, int32_t threads,
                              dpro_delta_set** out);
/* As dpro_base_delta_batch_ops, with the op-fusion joins of candidate c
 * applied on ONE worker, join_worker[c] (ordinal among the workers, see
 * dpro_base_worker; -1 = every worker). A single-worker join is the
 * reference's own op-fusion candidate: apply_op_fusion(g, a, b) on two
 * adjacent ops of one node (optimize.cpp:245-318, 1424-1432). NULL
 * join_worker = every worker. */
int dpro_base_delta_batch_ex(const dpro_base* base, int32_t n,
                             const int32_t* n_groups, const int64_t* spec_off,
                             const int32_t* group_off, const int32_t* members,
                             const int32_t* group_k, const uint8_t* fw_join,
                             const uint8_t* bw_join, const int32_t* join_worker,
                             int32_t threads, dpro_delta_set** out);
/* Name of the k-th worker of the base's cluster (NULL when out of range). */
const char* dpro_base_worker(const dpro_base* base, int32_t k);
/* Any n graphs (e.g. recompute / grad-accum variants from
 * dpro_graph_layered_variant) as deltas against the base: ops are matched
 * by id (kept when id, kind, duration and device agree), kept ops'
 * successor lists are diffed into extra and cut edges. Merging a delta
 * reproduces the graph's own CSR exactly. */
int dpro_base_delta_from_graphs(const dpro_base* base, const dpro_graph* const* graphs,
                                int32_t n, int32_t threads, dpro_delta_set** out);
int dpro_graph_from_base_batch_ops(const dpro_base* base, int32_t n,
                                   const int32_t* n_groups, const int64_t* spec_off,
                                   const int32_t* group_off, const int32_t* members,
                                   const int32_t* group_k, const uint8_t* fw_join,
                                   const uint8_t* bw_join, int32_t threads,
                                   dpro_graph** out);
const dpro_delta* dpro_delta_set_deltas(const dpro_delta_set* s);  /* [size] */
int32_t dpro_delta_set_size(const dpro_delta_set* s);
const char* dpro_delta_set_device_str(const dpro_delta_set* s, int32_t cand,
                                      uint32_t d);
void dpro_delta_set_free(dpro_delta_set* s);
/* The base graph itself (owned by the base; CSR via dpro_graph_csr). */
const dpro_graph* dpro_base_graph(const dpro_base* base);

/* The layered graph with a memory rewrite applied while generating it:
 * variant 1 = recompute_candidate, 2 = grad_accum_candidate with
 * microbatch_scale (optimize.cpp:819-959), 0 = none. Same graph as the
 * rewrite applied to dpro_graph_layered's output, at generator speed. */
dpro_graph* dpro_graph_layered_variant(const dpro_layered_model* model,
                                       const dpro_cluster_desc* cluster,
                                       const int32_t* part_k, int32_t variant,
                                       double microbatch_scale, int32_t* status);
/* Inputs of dpro_cuda_batch_peak_memory for one generated graph, resolved
 * natively (memory.cpp:71-157): op_bytes[i] = output_bytes_for(meta, op)
 * over the (keys, bytes) table for computation ops (UPDATE without an entry
 * -> 0; other ops 0), op_node[i] = dense compute node (-1 for other ops).
 * *n_nodes = compute nodes, named by dpro_graph_memory_node in name order.
 * DPRO_EINVAL with *missing_op = the first computation op without bytes
 * (MissingMetaError). */
int dpro_graph_memory_inputs(dpro_graph* g, int32_t n_entries, const char* const* keys,
                             const int64_t* bytes, int64_t* op_bytes, int32_t* op_node,
                             int32_t* n_nodes, uint32_t* missing_op);
const char* dpro_graph_memory_node(const dpro_graph* g, int32_t i);
/* Comm-op metadata (Op::tensor unit name, *bytes) of op i; NULL for other
 * ops. The transaction is the op id after "SEND." / "RECV.". */
const char* dpro_graph_comm_info(const dpro_graph* g, uint32_t i, int64_t* bytes);
/* The CLI's timeline.json for a replayed schedule (start/end in the graph's
 * index order), streamed natively: proj/tools/dpro_main.cpp:90-116 written
 * as write_json does (64-70, nlohmann dump(2) + newline), byte for byte. */
int dpro_graph_write_timeline(const dpro_graph* g, const int64_t* start,
                              const int64_t* end, const char* path);
/* n graphs with part_k[n*layers], built on `threads` host threads. */
int dpro_graph_layered_batch(const dpro_layered_model* model,
                             const dpro_cluster_desc* cluster,
                             const int32_t* part_k, int32_t n,
                             int32_t threads, dpro_graph** out);
/* Comm-only graph of sync_makespan(cluster, bytes, k). */
dpro_graph* dpro_graph_tsync(const dpro_cluster_desc* cluster, int64_t bytes,
                             int32_t k, int32_t* status);
/* Host CSR view (pointers owned by the graph; dur_bits = 64). */
int dpro_graph_csr(const dpro_graph* g, dpro_csr* out);
const char* dpro_graph_op_id(const dpro_graph* g, uint32_t i);
int32_t dpro_graph_op_kind(const dpro_graph* g, uint32_t i);
const char* dpro_graph_device_str(const dpro_graph* g, uint32_t d);
void dpro_graph_free(dpro_graph* g);
const char* dpro_graph_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* DPRO_CUDA_H_ */
