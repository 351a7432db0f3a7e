"""B200-native dPRO Replayer (arxiv 2205.02473): batched exact replay of
candidate data-flow graphs on sm_100a, behind the reference's replay API.

Product path: libdpro_cuda.so (csrc/, C ABI include/dpro_cuda.h). There is
no CPU fallback -- importing this package fails if the library is missing.
"""
from . import _native  # noqa: F401  (fails loudly without libdpro_cuda.so)
from .engine import Batch, Csr, Engine, default_engine
from .errors import (CycleError, EngineError, Error, IoError, LookupError_, MissingMetaError,
                     MissingProfileError, ParseError, TopologyError, TransformError)
from .graph import (ClusterSpec, DeviceId, DeviceKind, GlobalDFG, GraphBuilder, LinkSpec,
                    NodeSpec, Op, OpKind, TensorUnit, comp, round_us, synth_cluster)
from .replay import (CriticalPath, PathEntry, PathRun, ReplayResult, ScheduleEntry,
                     critical_path, execution_graph, partial_replay, replay, replay_many,
                     sync_makespan, sync_makespan_grid)
from .rewrite import (BudgetError, Strategy, StrategyKind, apply_grad_accum, apply_recompute,
                      memory_pass)
from .report import timeline_json, timeline_text, write_timeline
from .greedy import SearchOptions, SearchOutcome, reference_search
from .memory import (ModelMeta, estimate_peak_memory, estimate_peak_memory_many,
                     output_bytes_for)

__all__ = [
    "Batch", "Csr", "Engine", "default_engine", "CycleError", "EngineError", "Error",
    "LookupError_", "MissingProfileError", "ClusterSpec", "DeviceId", "DeviceKind",
    "GlobalDFG", "GraphBuilder", "LinkSpec", "NodeSpec", "Op", "OpKind", "TensorUnit",
    "comp", "round_us", "synth_cluster", "CriticalPath", "PathEntry", "PathRun",
    "ReplayResult", "ScheduleEntry", "critical_path", "execution_graph", "partial_replay",
    "replay", "replay_many", "sync_makespan", "sync_makespan_grid", "IoError",
    "MissingMetaError", "ParseError", "ModelMeta", "estimate_peak_memory",
    "estimate_peak_memory_many", "output_bytes_for", "TopologyError", "TransformError",
    "BudgetError", "Strategy", "StrategyKind", "apply_grad_accum", "apply_recompute",
    "memory_pass", "timeline_json", "timeline_text", "write_timeline", "SearchOptions",
    "SearchOutcome", "reference_search",
]
