/* TEST INFRASTRUCTURE ONLY (checker, never the product path).
 *
 * Plain-C restatement of the reference Replayer, proj/src/replay.cpp:26-226,
 * over an index-ordered CSR (index = byte-lexicographic op id order,
 * proj/src/graph.cpp:278-297). Parity status: pinned -- tests/test_oracle.py
 * checks it against the compiled reference (oracle/_ref) on the reference's
 * own fixtures (proj/tests/test_replay.cpp), the random-DAG families of
 * proj/tests/test_replay.cpp:214-238 and acceptance_main.cpp:293-342, the
 * SURVEY Appendix A vectors and ingest-built ring/PS graphs.
 */
#ifndef DPRO_REPLAY_ORACLE_H_
#define DPRO_REPLAY_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_MISSING_PROFILE = 1, ORC_CYCLE = 2, ORC_EINVAL = 3 };

/* flags bit0: virtual op (VIRTUAL_IN / VIRTUAL_OUT), bit1: communication op.
 * dev: dense device id in DeviceId order (0 <= dev < n_dev).
 * Outputs (caller-allocated, n entries unless noted):
 *   start/end     schedule (replay.cpp:119-123)
 *   tl_pos        position in the device timeline, -1 for virtual ops
 *   busy          per device: summed dur over its timeline (n_dev entries)
 *   scheduled     1 if the op was scheduled (for the CycleError id list)
 * Returns a status; *err = first op without duration (MISSING_PROFILE) or
 * number of ops never scheduled (CYCLE), mirroring replay.cpp:39-44,108-117. */
int32_t orc_replay(uint32_t n, const int64_t* dur, const uint32_t* dev,
                   const uint8_t* flags, uint32_t n_dev,
                   const uint32_t* succ_off, const uint32_t* succ,
                   int64_t* start, int64_t* end, int64_t* makespan,
                   int32_t* tl_pos, int64_t* busy, uint8_t* scheduled,
                   int64_t* err);

/* critical_path(execution_graph(g, r), r), replay.cpp:136-226, given the
 * schedule and timeline positions from orc_replay. Writes op indices to
 * path (capacity n) and returns the path length. */
int64_t orc_critical_path(uint32_t n, const uint32_t* dev, uint32_t n_dev,
                          const uint32_t* succ_off, const uint32_t* succ,
                          const int64_t* start, const int64_t* end,
                          int64_t makespan, const int32_t* tl_pos,
                          uint32_t* path);

#ifdef __cplusplus
}
#endif

#endif /* DPRO_REPLAY_ORACLE_H_ */
