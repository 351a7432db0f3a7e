"""Batched candidate evaluator and search driver over the GPU Replayer.

The reference evaluates one candidate graph per `replay()` call inside its
greedy Alg. 1 (proj/src/optimize.cpp:1327-1650; gate 1382-1392), building
each through string-keyed GraphBuilder copies. Here a whole round of
candidates is built as deltas of one base graph on host threads
(csrc/dfg_gen.cpp, dpro_base_delta_batch), uploaded as deltas, merged into
the resident base graph on the GPU and replayed in ONE batched launch;
across GPUs every
rank evaluates its own shard and the round's best candidate is agreed on
with two int64 MIN all-reduces (the K4 exchange of DESIGN.md, exchange.py).

* `opt_part_num`        optimize.cpp:562-576 (k* over a batched t_sync grid)
* `should_fuse_ops`     optimize.cpp:545-551 (Theorem 1)
* `should_fuse_tensors` optimize.cpp:553-560 (Theorem 2)
* `SyncSearch`          tensor-fusion + partition search over a layered
                        model; MCMC with the acceptance rule of the paper's
                        (excised) MCMC algorithm, P = min(1, exp(beta (T - T'))),
                        PAPER.md:928. The reference ships no MCMC (SURVEY
                        section 0.1), so trajectories are "parity unpinned";
                        every evaluated candidate's makespan is exact (equal
                        to the reference replay of the same rewritten graph).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from .engine import Engine, default_engine
from .graph import ClusterSpec
from .ingest import LayeredBase, LayeredModel
from .exchange import broadcast_from, exchange_best, metropolis_accept
from .replay import sync_makespan_grid


def _layers_of_op(op_id: str) -> list[int]:
    """Layers an op of a layered-model graph belongs to: "w0->BW.l5" -> [5],
    "SEND.g3+g4#p1#c0#s2#w0#w1" / "w1->IN.g3+g4" -> [3, 4]."""
    local = op_id.split("->", 1)[1] if "->" in op_id else op_id
    kind, _, rest = local.partition(".")
    if kind in ("FW", "BW", "UPDATE", "RFW"):
        return [int(rest[1:])] if rest.startswith("l") and rest[1:].isdigit() else []
    unit = rest.split("#", 1)[0]
    return [int(t[1:]) for t in unit.split("+") if t.startswith("g") and t[1:].isdigit()]


def opt_part_num(bytes_: int, kmax: int, t_sync: Callable[[int, int], int]) -> int:
    """optimize.cpp:562-576: argmin_k t_sync(bytes, k), k in [1, min(kmax, bytes)],
    ties -> smallest k."""
    if bytes_ < 1:
        return 1
    cap = min(max(kmax, 1), bytes_)
    best_k, best = 1, t_sync(bytes_, 1)
    for k in range(2, cap + 1):
        v = t_sync(bytes_, k)
        if v < best:
            best, best_k = v, k
    return best_k


class SyncTable:
    """Memoized t_sync(bytes, k) (SearchCtx::sync, optimize.cpp:1170-1194)
    filled by batched GPU grids instead of one replay per (bytes, k)."""

    def __init__(self, cluster: ClusterSpec, engine: Engine | None = None):
        self.cluster = cluster
        self.engine = engine
        self.memo: dict[tuple[int, int], int] = {}

    def fill(self, pairs: Sequence[tuple[int, int]]) -> None:
        todo = sorted({p for p in pairs if p not in self.memo})
        if todo:
            vals = sync_makespan_grid(self.cluster, [b for b, _ in todo], [k for _, k in todo],
                                      engine=self.engine)
            self.memo.update(zip(todo, vals))

    def __call__(self, bytes_: int, k: int) -> int:
        if (bytes_, k) not in self.memo:
            self.fill([(bytes_, k)])
        return self.memo[(bytes_, k)]

    def opt_part_num_many(self, sizes: Sequence[int], kmax: int) -> list[int]:
        """k* for many tensor sizes with ONE grid launch."""
        self.fill([(b, k) for b in sizes for k in range(1, min(max(kmax, 1), b) + 1)])
        return [opt_part_num(b, kmax, self) for b in sizes]


def should_fuse_ops(p_prev_dur: int, p_cur_dur: int, fused_dur: float, q_prev_dur: int) -> bool:
    """Theorem 1, optimize.cpp:545-551."""
    gain = float(p_prev_dur) + float(p_cur_dur) - fused_dur
    return float(q_prev_dur) <= gain + 1e-9


def should_fuse_tensors(q_prev_end: int, p_cur_end: int, s_prev: int, s_cur: int, kmax: int,
                        t_sync: Callable[[int, int], int]) -> bool:
    """Theorem 2, optimize.cpp:553-560."""
    fused = s_prev + s_cur
    fused_sync = t_sync(fused, opt_part_num(fused, kmax, t_sync))
    cur_sync = t_sync(s_cur, opt_part_num(s_cur, kmax, t_sync))
    return q_prev_end > p_cur_end + fused_sync - cur_sync


@dataclass
class SyncState:
    """Synchronization units of a layered model: groups of consecutive layers
    fused in layer order (apply_tensor_fusion chain), each with a partition
    count (apply_tensor_partition); optionally op fusion of adjacent FW / BW
    ops on every worker (fw_join / bw_join, apply_op_fusion chains)."""
    groups: list[list[int]]
    ks: list[int]
    makespan: int = -1
    fw_join: list[int] = field(default_factory=list)
    bw_join: list[int] = field(default_factory=list)

    def key(self) -> tuple:
        return (tuple(tuple(g) for g in self.groups), tuple(self.ks), tuple(self.fw_join),
                tuple(self.bw_join))

    def copy(self) -> "SyncState":
        return SyncState([list(g) for g in self.groups], list(self.ks), self.makespan,
                         list(self.fw_join), list(self.bw_join))


@dataclass
class SearchLog:
    rounds: int = 0
    evaluated: int = 0
    accepted: int = 0
    history: list[int] = field(default_factory=list)


class SyncSearch:
    """Batched MCMC over tensor fusion + partition (BASELINE config 3).

    Each round proposes `batch` neighbours of the current state (fuse two
    adjacent units, split a unit, re-partition a unit), replays them all in
    one GPU batch (makespan only), takes the best as the proposal and
    accepts it with P = min(1, exp(beta * (T - T'))).
    With `dist` (torch.distributed) every rank proposes its own batch. In
    the default "shared" mode the round's proposal is the global best (two
    MIN all-reduces, exchange.exchange_best, then a broadcast from its
    owner); with chains="independent" every rank runs its own chain and only
    the best-cost strategy found so far is exchanged each round."""

    def __init__(self, model: LayeredModel, cluster: ClusterSpec, engine: Engine | None = None,
                 kmax: int = 16, beta: float = 0.01, seed: int = 0, threads: int = 8,
                 dist=None, rank: int = 0, guided: float = 0.0, op_fusion: bool = False,
                 chains: str = "shared"):
        if chains not in ("shared", "independent"):
            raise ValueError(f"chains must be 'shared' or 'independent', got {chains!r}")
        self.model, self.cluster = model, cluster
        # "shared": one chain, each round's proposal is the best over all
        # ranks' batches; "independent": one chain per rank (north_star),
        # only the best-cost strategy is exchanged per round
        self.chains, self.seed = chains, seed
        self.engine = engine or default_engine()
        self.kmax, self.beta, self.threads = kmax, beta, threads
        # fraction of proposals that modify a unit on the current critical
        # path (CandidateSelection, Alg. 1; critical path = K3)
        self.guided = guided
        self._critical: np.ndarray | None = None
        # op-fusion moves (toggle FW.l<i>+FW.l<i+1> / BW.l<i+1>+BW.l<i> on
        # every worker): BASELINE config 4's strategy mix
        self.op_fusion = op_fusion
        self.rng = np.random.default_rng([seed, rank])
        self.dist, self.rank = dist, rank
        L = model.layers
        self.base = LayeredBase(model, cluster)  # delta construction of candidates
        # the base graph stays in HBM; each round uploads only the deltas
        self.resident = self.engine.resident(self.base.graph().csr)
        self.state = SyncState([[i] for i in range(L)], [1] * L)
        self.best = None
        self.log = SearchLog()

    # ---- candidates ---------------------------------------------------
    def _bytes(self, g: list[int]) -> int:
        return int(sum(self.model.tensor_bytes[i] for i in g))

    def propose(self, s: SyncState) -> SyncState:
        c = s.copy()
        n = len(c.groups)
        move = self.rng.integers(0, 3)
        if move == 0 and n > 1:  # tensor fusion of two adjacent units
            i = int(self.rng.integers(0, n - 1))
            c.groups[i:i + 2] = [c.groups[i] + c.groups[i + 1]]
            c.ks[i:i + 2] = [1]
        elif move == 1 and any(len(g) > 1 for g in c.groups):  # un-fuse
            cand = [i for i, g in enumerate(c.groups) if len(g) > 1]
            i = cand[int(self.rng.integers(0, len(cand)))]
            cut = int(self.rng.integers(1, len(c.groups[i])))
            g = c.groups[i]
            c.groups[i:i + 1] = [g[:cut], g[cut:]]
            c.ks[i:i + 1] = [1, 1]
        else:  # re-partition a unit
            i = int(self.rng.integers(0, n))
            cap = min(self.kmax, self._bytes(c.groups[i]))
            c.ks[i] = int(self.rng.integers(1, cap + 1))
        return c

    # ---- vectorized proposals --------------------------------------------
    # A state of a layered model is its fusion boundaries (cuts[i]: layers i
    # and i+1 sync as different units) plus the partition count of each unit
    # (kl[start of unit]); units are always contiguous layer ranges.
    def _cuts_kl(self, s: SyncState):
        L = self.model.layers
        cuts = np.zeros(max(L - 1, 0), bool)
        kl = np.ones(L, np.int32)
        for g, k in zip(s.groups, s.ks):
            kl[g[0]] = k
            if g[-1] < L - 1:
                cuts[g[-1]] = True
        return cuts, kl

    @staticmethod
    def _state(cuts: np.ndarray, kl: np.ndarray, fj=None, bj=None) -> SyncState:
        starts = [0] + (np.flatnonzero(cuts) + 1).tolist()
        ends = starts[1:] + [len(kl)]
        return SyncState([list(range(a, b)) for a, b in zip(starts, ends)],
                         [int(kl[a]) for a in starts], -1,
                         [] if fj is None or not fj.any() else fj.astype(int).tolist(),
                         [] if bj is None or not bj.any() else bj.astype(int).tolist())

    def _joins0(self, s: SyncState):
        L = self.model.layers
        fj = np.zeros(max(L - 1, 0), np.uint8)
        bj = np.zeros(max(L - 1, 0), np.uint8)
        if s.fw_join:
            fj[:] = s.fw_join
        if s.bw_join:
            bj[:] = s.bw_join
        return fj, bj

    def critical_layers(self, s: SyncState) -> np.ndarray:
        """Layers whose compute or synchronization ops lie on the critical
        path of s (replay with schedule + K3 on the GPU): bool[L]."""
        spec = [(s.groups, s.ks)]
        b = self.engine.delta_batch(self.resident, self.base.deltas(spec, 1))
        b.replay(want_schedule=True)
        path = b.critical_paths()[0]
        g = self.base.candidates(spec, 1)[0]
        crit = np.zeros(self.model.layers, bool)
        for i in path.tolist():
            for layer in _layers_of_op(g.op_id(int(i))):
                if 0 <= layer < len(crit):
                    crit[layer] = True
        return crit

    def _pick_units(self, n: int, G: int, starts, sizes, allowed: np.ndarray | None):
        """A unit index per row: uniform over all units, or (guided rows)
        over units that contain a critical layer."""
        gi = self.rng.integers(0, G, n)
        if allowed is not None and self.guided > 0 and self._critical is not None:
            crit_units = np.flatnonzero(allowed & np.array(
                [self._critical[a:a + z].any() for a, z in zip(starts, sizes)]))
            if len(crit_units):
                g_rows = self.rng.random(n) < self.guided
                gi[g_rows] = crit_units[self.rng.integers(0, len(crit_units), int(g_rows.sum()))]
        return gi

    def propose_many(self, s: SyncState, n: int):
        """n neighbours of s at once (same moves and probabilities as
        propose()): (cuts[n, L-1], kl[n, L])."""
        L = self.model.layers
        cuts0, kl0 = self._cuts_kl(s)
        starts = np.array([g[0] for g in s.groups])
        sizes = np.array([len(g) for g in s.groups])
        G = len(starts)
        ctb = np.concatenate([[0], np.cumsum(np.asarray(self.model.tensor_bytes, np.int64))])
        gbytes = ctb[starts + sizes] - ctb[starts]
        multi = np.flatnonzero(sizes > 1)
        cuts = np.repeat(cuts0[None], n, 0)
        kl = np.repeat(kl0[None], n, 0)
        fj0, bj0 = self._joins0(s)
        fj = np.repeat(fj0[None], n, 0)
        bj = np.repeat(bj0[None], n, 0)
        move = self.rng.integers(0, 5 if self.op_fusion and L > 1 else 3, n)
        for mv, arr in ((3, fj), (4, bj)):  # toggle one op-fusion join
            rows = np.flatnonzero(move == mv)
            if len(rows):
                i = self.rng.integers(0, L - 1, len(rows))
                arr[rows, i] ^= 1
        move = np.where(move >= 3, -1, move)
        m0 = (move == 0) & (G > 1)
        m1 = (move == 1) & (len(multi) > 0)
        m2 = ~(m0 | m1) & (move >= 0)
        r0 = np.flatnonzero(m0)
        if len(r0):  # fuse units j, j+1
            ok = np.ones(G, bool)
            ok[-1] = False
            j = self._pick_units(len(r0), G, starts, sizes, ok)
            j = np.minimum(j, G - 2)
            cuts[r0, starts[j + 1] - 1] = False
            kl[r0, starts[j]] = 1
        r1 = np.flatnonzero(m1)
        if len(r1):  # split a multi-layer unit at a random inner point
            gi = multi[self.rng.integers(0, len(multi), len(r1))]
            if self.guided > 0 and self._critical is not None:
                ok = np.zeros(G, bool)
                ok[multi] = True
                pick = self._pick_units(len(r1), G, starts, sizes, ok)
                gi = np.where(ok[pick], pick, gi)
            cut = (self.rng.random(len(r1)) * (sizes[gi] - 1)).astype(np.int64) + 1
            cuts[r1, starts[gi] + cut - 1] = True
            kl[r1, starts[gi]] = 1
            kl[r1, starts[gi] + cut] = 1
        r2 = np.flatnonzero(m2)
        if len(r2):  # re-partition a unit, k uniform in [1, min(kmax, bytes)]
            gi = self._pick_units(len(r2), G, starts, sizes, np.ones(G, bool))
            cap = np.minimum(self.kmax, gbytes[gi])
            kl[r2, starts[gi]] = (self.rng.random(len(r2)) * cap).astype(np.int64) + 1
        self._last_joins = (fj, bj)
        return cuts, kl

    def _spec_arrays(self, cuts: np.ndarray, kl: np.ndarray):
        """Flattened dpro_base_delta_batch specs of a proposal matrix."""
        n, L = kl.shape
        smask = np.concatenate([np.ones((n, 1), bool), cuts], axis=1)
        r, p = np.nonzero(smask)  # row-major: units of each row in layer order
        nxt = np.append(np.where(r[1:] == r[:-1], p[1:], L), L)
        n_groups = np.bincount(r, minlength=n).astype(np.int32)
        spec_off = np.concatenate([[0], np.cumsum(n_groups)[:-1]]).astype(np.int64)
        group_off = np.concatenate([[0], np.cumsum(nxt - p)]).astype(np.int32)
        members = np.tile(np.arange(L, dtype=np.int32), n)
        return n_groups, spec_off, group_off, members, kl[r, p].astype(np.int32)

    def evaluate_arrays(self, cuts: np.ndarray, kl: np.ndarray, fj=None, bj=None) -> np.ndarray:
        """Exact makespans of a proposal matrix: one GPU batch."""
        deltas = self.base.deltas_from_arrays(*self._spec_arrays(cuts, kl), threads=self.threads,
                                              fw_join=fj, bw_join=bj)
        b = self.engine.delta_batch(self.resident, deltas)
        b.replay(want_schedule=False)
        ms, st, *_ = b.results()
        if np.any(st != 0):
            raise RuntimeError(f"replay failed for {int((st != 0).sum())} candidates")
        self.log.evaluated += len(ms)
        return ms

    def evaluate(self, states: Sequence[SyncState]) -> np.ndarray:
        """Exact makespans of candidate states: deltas against the resident
        base graph, merged, packed and replayed in one GPU batch."""
        joins = [self._joins0(st) for st in states]
        deltas = self.base.deltas([(st.groups, st.ks) for st in states], self.threads,
                                  fw_join=[j[0] for j in joins], bw_join=[j[1] for j in joins])
        b = self.engine.delta_batch(self.resident, deltas)
        b.replay(want_schedule=False)
        ms, st, *_ = b.results()
        if np.any(st != 0):
            raise RuntimeError(f"replay failed for {int((st != 0).sum())} candidates")
        self.log.evaluated += len(states)
        return ms

    # ---- one round ----------------------------------------------------
    def _dev(self) -> str:
        return f"cuda:{self.engine.device}" if self.dist.get_backend() == "nccl" else "cpu"

    def _exchange(self, best_ms: int, best_i: int, cand: SyncState) -> SyncState:
        """The global best proposal of this round (exchange.exchange_best:
        MIN makespan, then lowest (rank, index) among the ties), broadcast
        from its owner."""
        if self.dist is None:
            return cand
        ms, owner, _ = exchange_best(self.dist, best_ms, best_i, self.rank, self._dev())
        out = broadcast_from(self.dist, cand, owner, self.rank)
        out.makespan = ms
        return out

    def step(self, batch: int) -> SearchLog:
        s = self.state
        if s.makespan < 0:
            s.makespan = int(self.evaluate([s])[0])
            self.best = s.copy()
            if self.dist is not None and self.chains == "independent":
                self.best = self._exchange(self.best.makespan, 0, self.best.copy())
        if self.guided > 0 and self._critical is None:
            self._critical = self.critical_layers(s)
        cuts, kl = self.propose_many(s, batch)
        fj, bj = self._last_joins if self.op_fusion else (None, None)
        ms = self.evaluate_arrays(cuts, kl, fj, bj) if self.op_fusion else \
            self.evaluate_arrays(cuts, kl)
        i = int(np.argmin(ms))
        cand = self._state(cuts[i], kl[i], None if fj is None else fj[i],
                           None if bj is None else bj[i])
        cand.makespan = int(ms[i])
        if self.chains == "independent":
            # every rank walks its own chain (own proposals, own uniform
            # draw); only the best-cost strategy crosses ranks
            prop = cand
            u = float(np.random.default_rng([self.seed, self.rank, self.log.rounds, 7]).random())
        else:
            # one chain shared by all ranks: the global best proposal and a
            # shared uniform draw, so every rank takes the same decision
            prop = self._exchange(int(ms[i]), i, cand)
            u = float(np.random.default_rng([self.log.rounds, 7]).random())
        if metropolis_accept(self.beta, s.makespan, prop.makespan, u):
            self.state = prop
            self.log.accepted += 1
            self._critical = None  # recomputed for the new state
        if self.chains == "independent" and self.dist is not None:
            mine = self.state if self.state.makespan < self.best.makespan else self.best
            self.best = self._exchange(mine.makespan, 0, mine.copy())
        elif self.state.makespan < self.best.makespan:
            self.best = self.state.copy()
        self.log.rounds += 1
        self.log.history.append(self.state.makespan)
        return self.log

    def run(self, rounds: int, batch: int) -> SyncState:
        for _ in range(rounds):
            self.step(batch)
        return self.best


class StrategySearch:
    """Batched MCMC over the reference's full strategy space on a GlobalDFG
    (BASELINE config 4's op fusion + recomputation + gradient accumulation,
    plus tensor fusion and partition): every round applies `batch` random
    strategies to the current graph with the reference-exact rewrites
    (rewrite.py), turns each result into a delta of the current graph
    (delta.make_delta) and evaluates them all in ONE GPU batch against the
    current graph resident in HBM; acceptance as SyncSearch. Host rewrites
    cost O(V + E) Python per candidate, so this path suits graphs of up to
    ~10^4 ops; layered models at scale use SyncSearch's native deltas."""

    def __init__(self, g, engine: Engine | None = None, meta=None, cost=None, kmax: int = 8,
                 beta: float = 0.01, seed: int = 0, kinds=(0, 1, 2, 3, 4)):
        from .rewrite import CostModel
        from .memory import ModelMeta
        self.engine = engine or default_engine()
        self.meta = meta or ModelMeta()
        self.cost = cost or CostModel()
        self.kmax, self.beta, self.kinds = kmax, beta, tuple(kinds)
        self.rng = np.random.default_rng(seed)
        self.g = g
        self.makespan = -1
        self.applied: list = []
        self.best = (g, -1, [])
        self.log = SearchLog()
        self._resident = None

    def _random_strategy(self, g):
        from .rewrite import Strategy, StrategyKind
        kind = StrategyKind(int(self.rng.choice(self.kinds)))
        if kind == StrategyKind.OP_FUSION:
            comp = [o.id for o in g.ops() if int(o.kind) in (0, 1)]
            if not comp:
                return None
            a = comp[int(self.rng.integers(0, len(comp)))]
            succ = [s for s in g.succs(a) if int(g.op(s).kind) in (0, 1)]
            if not succ:
                return None
            return Strategy(kind, a, succ[int(self.rng.integers(0, len(succ)))])
        bases = sorted({u.base for u in g.tensor_units().values()})
        if kind == StrategyKind.TENSOR_FUSION:
            if len(bases) < 2:
                return None
            i = int(self.rng.integers(0, len(bases) - 1))
            return Strategy(kind, bases[i], bases[i + 1])
        if kind == StrategyKind.PARTITION:
            if not bases:
                return None
            return Strategy(kind, bases[int(self.rng.integers(0, len(bases)))], "",
                            int(self.rng.integers(1, self.kmax + 1)))
        return Strategy(kind)  # recompute / grad-accum

    def propose(self, n: int):
        """Up to n (strategy, graph) candidates (rewrites that raise the
        reference's errors are dropped)."""
        from .errors import Error
        from .rewrite import apply_strategy
        out = []
        for _ in range(n * 3):
            if len(out) == n:
                break
            st = self._random_strategy(self.g)
            if st is None:
                continue
            try:
                out.append((st, apply_strategy(self.g, st, self.cost, self.meta)))
            except Error:
                continue
        return out

    def evaluate(self, graphs) -> np.ndarray:
        from .delta import DeltaList, make_delta
        from .engine import Csr
        if self._resident is None:
            self._resident = self.engine.resident(Csr.from_dict(self.g.to_csr()))
        b = self.engine.delta_batch(self._resident,
                                    DeltaList([make_delta(self.g, c) for c in graphs]))
        b.replay(want_schedule=False)
        ms, st, *_ = b.results()
        if np.any(st != 0):
            raise RuntimeError(f"replay failed for {int((st != 0).sum())} candidates")
        self.log.evaluated += len(graphs)
        return ms

    def step(self, batch: int) -> SearchLog:
        from .replay import replay
        if self.makespan < 0:
            self.makespan = replay(self.g).iteration_time_us
            self.best = (self.g, self.makespan, [])
        cands = self.propose(batch)
        if cands:
            ms = self.evaluate([c[1] for c in cands])
            i = int(np.argmin(ms))
            u = float(np.random.default_rng([self.log.rounds, 11]).random())
            if metropolis_accept(self.beta, self.makespan, int(ms[i]), u):
                self.g, self.makespan = cands[i][1], int(ms[i])
                self.applied = self.applied + [cands[i][0]]
                self._resident = None  # the next round's base is the new graph
                self.log.accepted += 1
                if self.makespan < self.best[1]:
                    self.best = (self.g, self.makespan, list(self.applied))
        self.log.rounds += 1
        self.log.history.append(self.makespan)
        return self.log

    def run(self, rounds: int, batch: int):
        for _ in range(rounds):
            self.step(batch)
        return self.best
