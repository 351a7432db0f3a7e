/* TEST INFRASTRUCTURE ONLY -- the CPU checker for the CUDA Replayer.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this; the product path never does.
 *
 * A line-by-line restatement of the reference replay semantics
 * (proj/src/replay.cpp) in C over index-ordered CSR. It deliberately keeps
 * the reference's data structures -- a (end, index) min-heap of dispatched
 * ops (replay.cpp:54), a (ready, index)-ordered pending set per device
 * (replay.cpp:28-33) and the full device scan per event time
 * (replay.cpp:74-90) -- so that it is an independent check of the CUDA
 * kernel, which uses a different (round-based, per-device FIFO) formulation.
 */
#include "replay_oracle.h"

#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t key;
  uint32_t idx;
} Item;

typedef struct {
  Item* a;
  uint32_t n;
} Heap;

static int item_lt(Item x, Item y) {
  return x.key < y.key || (x.key == y.key && x.idx < y.idx);
}

static void heap_push(Heap* h, Item it) {
  uint32_t i = h->n++;
  h->a[i] = it;
  while (i > 0) {
    uint32_t p = (i - 1) / 2;
    if (!item_lt(h->a[i], h->a[p])) break;
    Item t = h->a[p];
    h->a[p] = h->a[i];
    h->a[i] = t;
    i = p;
  }
}

static Item heap_pop(Heap* h) {
  Item top = h->a[0];
  h->a[0] = h->a[--h->n];
  uint32_t i = 0;
  for (;;) {
    uint32_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && item_lt(h->a[l], h->a[m])) m = l;
    if (r < h->n && item_lt(h->a[r], h->a[m])) m = r;
    if (m == i) break;
    Item t = h->a[m];
    h->a[m] = h->a[i];
    h->a[i] = t;
    i = m;
  }
  return top;
}

typedef struct {
  uint32_t n;
  const int64_t* dur;
  const uint32_t* dev;
  const uint8_t* flags;
  const uint32_t* succ_off;
  const uint32_t* succ;
  uint32_t* indeg;
  int64_t* start;
  int64_t* end;
  uint8_t* sched;
  uint8_t* queued;
  Heap* pending; /* per device */
  uint32_t remaining; /* uint32 like replay.cpp:56 (wraps on the init quirk) */
  uint32_t* stk_op;   /* explicit recursion stack for ready() */
  uint32_t* stk_pos;
} Ctx;

/* replay.cpp:60-72: virtual ops finish at t and cascade depth-first through
 * successors in ascending index order; others join their device queue. */
static void ready(Ctx* c, uint32_t root, int64_t t) {
  if (!(c->flags[root] & 1u)) {
    if (!c->queued[root]) { /* std::set insert of an existing (t,i): no-op */
      Item it = {t, root};
      heap_push(&c->pending[c->dev[root]], it);
      c->queued[root] = 1;
    }
    return;
  }
  uint32_t sp = 0;
  c->start[root] = c->end[root] = t;
  c->sched[root] = 1;
  --c->remaining;
  c->stk_op[sp] = root;
  c->stk_pos[sp] = c->succ_off[root];
  ++sp;
  while (sp > 0) {
    uint32_t v = c->stk_op[sp - 1];
    uint32_t p = c->stk_pos[sp - 1];
    if (p == c->succ_off[v + 1]) {
      --sp;
      continue;
    }
    c->stk_pos[sp - 1] = p + 1;
    uint32_t s = c->succ[p];
    if (--c->indeg[s] != 0) continue;
    if (c->flags[s] & 1u) {
      c->start[s] = c->end[s] = t;
      c->sched[s] = 1;
      --c->remaining;
      c->stk_op[sp] = s;
      c->stk_pos[sp] = c->succ_off[s];
      ++sp;
    } else if (!c->queued[s]) {
      Item it = {t, s};
      heap_push(&c->pending[c->dev[s]], it);
      c->queued[s] = 1;
    }
  }
}

int32_t orc_replay(uint32_t n, const int64_t* dur, const uint32_t* dev,
                   const uint8_t* flags, uint32_t n_dev,
                   const uint32_t* succ_off, const uint32_t* succ,
                   int64_t* start, int64_t* end, int64_t* makespan,
                   int32_t* tl_pos, int64_t* busy, uint8_t* scheduled,
                   int64_t* err) {
  *err = 0;
  *makespan = 0;
  /* replay.cpp:39-44 */
  for (uint32_t i = 0; i < n; ++i) {
    if (dur[i] < 0 && !(flags[i] & 1u)) {
      *err = i;
      return ORC_MISSING_PROFILE;
    }
  }
  for (uint32_t i = 0; i < n; ++i)
    if (!(flags[i] & 1u) && dev[i] >= n_dev) return ORC_EINVAL;

  Ctx c;
  memset(&c, 0, sizeof c);
  c.n = n;
  c.dur = dur;
  c.dev = dev;
  c.flags = flags;
  c.succ_off = succ_off;
  c.succ = succ;
  c.start = start;
  c.end = end;
  c.indeg = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
  c.sched = scheduled;
  c.queued = (uint8_t*)calloc(n + 1, 1);
  c.stk_op = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  c.stk_pos = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  c.pending = (Heap*)calloc(n_dev + 1, sizeof(Heap));
  uint32_t* per_dev = (uint32_t*)calloc(n_dev + 1, sizeof(uint32_t));
  int64_t* dfree = (int64_t*)calloc(n_dev + 1, sizeof(int64_t));
  int32_t* tl_len = (int32_t*)calloc(n_dev + 1, sizeof(int32_t));
  Heap pq;
  pq.a = (Item*)malloc((n + 1) * sizeof(Item));
  pq.n = 0;

  memset(scheduled, 0, n);
  for (uint32_t i = 0; i < n; ++i) {
    start[i] = end[i] = 0;
    if (tl_pos) tl_pos[i] = -1;
    if (!(flags[i] & 1u)) per_dev[dev[i]]++;
  }
  for (uint32_t d = 0; d < n_dev; ++d) {
    c.pending[d].a = (Item*)malloc((per_dev[d] + 1) * sizeof(Item));
    c.pending[d].n = 0;
    if (busy) busy[d] = 0;
  }
  /* replay.cpp:46-49 */
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t e = succ_off[i]; e < succ_off[i + 1]; ++e) c.indeg[succ[e]]++;
  c.remaining = n;

  /* replay.cpp:74-90 */
#define DISPATCH(T)                                                        \
  do {                                                                     \
    int64_t t_ = (T);                                                      \
    for (uint32_t d = 0; d < n_dev; ++d) {                                 \
      Heap* q = &c.pending[d];                                             \
      while (dfree[d] <= t_ && q->n > 0) {                                 \
        if (q->a[0].key > t_) break;                                       \
        Item it = heap_pop(q);                                             \
        uint32_t i = it.idx;                                               \
        start[i] = dfree[d] > it.key ? dfree[d] : it.key;                  \
        end[i] = start[i] + dur[i];                                        \
        scheduled[i] = 1;                                                  \
        --c.remaining;                                                     \
        dfree[d] = end[i];                                                 \
        if (tl_pos) tl_pos[i] = tl_len[d];                                 \
        tl_len[d]++;                                                       \
        if (busy) busy[d] += dur[i];                                       \
        Item ev = {end[i], i};                                             \
        heap_push(&pq, ev);                                                \
      }                                                                    \
    }                                                                      \
  } while (0)

  /* replay.cpp:92-95 -- indeg re-tested after earlier cascades (the init
   * quirk of SURVEY Appendix A is reproduced, not avoided). */
  for (uint32_t i = 0; i < n; ++i)
    if (c.indeg[i] == 0) ready(&c, i, 0);
  DISPATCH(0);
  /* replay.cpp:96-106 */
  while (pq.n > 0) {
    int64_t t = pq.a[0].key;
    while (pq.n > 0 && pq.a[0].key == t) {
      Item it = heap_pop(&pq);
      uint32_t i = it.idx;
      for (uint32_t e = succ_off[i]; e < succ_off[i + 1]; ++e) {
        uint32_t s = succ[e];
        if (--c.indeg[s] == 0) ready(&c, s, t);
      }
    }
    DISPATCH(t);
  }
#undef DISPATCH

  int32_t status = ORC_OK;
  if (c.remaining > 0) {
    int64_t stuck = 0;
    for (uint32_t i = 0; i < n; ++i) stuck += scheduled[i] ? 0 : 1;
    *err = stuck;
    status = ORC_CYCLE;
  } else {
    int64_t T = 0;
    for (uint32_t i = 0; i < n; ++i) T = end[i] > T ? end[i] : T;
    *makespan = T;
  }

  for (uint32_t d = 0; d < n_dev; ++d) free(c.pending[d].a);
  free(c.pending);
  free(per_dev);
  free(dfree);
  free(tl_len);
  free(pq.a);
  free(c.indeg);
  free(c.queued);
  free(c.stk_op);
  free(c.stk_pos);
  return status;
}

/* replay.cpp:146-226 over the execution graph = DFG edges plus consecutive
 * timeline pairs (replay.cpp:136-144). */
int64_t orc_critical_path(uint32_t n, const uint32_t* dev, uint32_t n_dev,
                          const uint32_t* succ_off, const uint32_t* succ,
                          const int64_t* start, const int64_t* end,
                          int64_t makespan, const int32_t* tl_pos,
                          uint32_t* path) {
  if (n == 0) return 0;
  /* timeline neighbours */
  uint32_t* tl_prev = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* tl_next = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* dev_cnt = (uint32_t*)calloc(n_dev + 1, sizeof(uint32_t));
  uint32_t* dev_base = (uint32_t*)calloc(n_dev + 1, sizeof(uint32_t));
  for (uint32_t i = 0; i < n; ++i)
    if (tl_pos[i] >= 0) dev_cnt[dev[i]]++;
  uint32_t acc = 0;
  for (uint32_t d = 0; d < n_dev; ++d) {
    dev_base[d] = acc;
    acc += dev_cnt[d];
  }
  uint32_t* order = (uint32_t*)malloc((acc + 1) * sizeof(uint32_t));
  for (uint32_t i = 0; i < n; ++i) {
    tl_prev[i] = tl_next[i] = UINT32_MAX;
    if (tl_pos[i] >= 0) order[dev_base[dev[i]] + (uint32_t)tl_pos[i]] = i;
  }
  for (uint32_t d = 0; d < n_dev; ++d) {
    for (uint32_t p = 1; p < dev_cnt[d]; ++p) {
      uint32_t a = order[dev_base[d] + p - 1], b = order[dev_base[d] + p];
      tl_next[a] = b;
      tl_prev[b] = a;
    }
  }
  /* predecessor CSR */
  uint32_t* pred_off = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
  uint32_t E = succ_off[n];
  uint32_t* pred = (uint32_t*)malloc((E + 1) * sizeof(uint32_t));
  for (uint32_t e = 0; e < E; ++e) pred_off[succ[e] + 1]++;
  for (uint32_t i = 0; i < n; ++i) pred_off[i + 1] += pred_off[i];
  uint32_t* fill = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  memcpy(fill, pred_off, (n + 1) * sizeof(uint32_t));
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t e = succ_off[i]; e < succ_off[i + 1]; ++e)
      pred[fill[succ[e]]++] = i;

  /* replay.cpp:166-185: tight-edge backward closure from end == T */
  uint8_t* good = (uint8_t*)calloc(n, 1);
  uint32_t* stack = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t sp = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (end[i] == makespan) {
      good[i] = 1;
      stack[sp++] = i;
    }
  while (sp > 0) {
    uint32_t v = stack[--sp];
    for (uint32_t e = pred_off[v]; e <= pred_off[v + 1]; ++e) {
      uint32_t p = (e < pred_off[v + 1]) ? pred[e] : tl_prev[v];
      if (p == UINT32_MAX) continue;
      if (!good[p] && end[p] == start[v]) {
        good[p] = 1;
        stack[sp++] = p;
      }
    }
  }
  /* replay.cpp:187-209: smallest-index good op starting at 0, then the
   * smallest-index good tight successor until an op ends at T. */
  int64_t cur = -1, len = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (good[i] && start[i] == 0) {
      cur = i;
      break;
    }
  while (cur >= 0) {
    path[len++] = (uint32_t)cur;
    if (end[cur] == makespan) break;
    int64_t next = -1;
    for (uint32_t e = succ_off[cur]; e <= succ_off[cur + 1]; ++e) {
      uint32_t s = (e < succ_off[cur + 1]) ? succ[e] : tl_next[cur];
      if (s == UINT32_MAX) continue;
      if (good[s] && end[cur] == start[s])
        if (next < 0 || s < (uint32_t)next) next = s;
    }
    cur = next;
  }
  free(tl_prev);
  free(tl_next);
  free(dev_cnt);
  free(dev_base);
  free(order);
  free(pred_off);
  free(pred);
  free(fill);
  free(good);
  free(stack);
  return len;
}
