"""Trace bundle + dependency spec -> GlobalDFG, the
reference's ingest restated (proj/src/ingest.cpp:71-493):

    DependencySpec.from_json       ingest.cpp:71-117
    op_duration_profile(events)    ingest.cpp:145-181 (mean durations; RECV
                                   service time from its SEND's start)
    build_local_dfg(events, deps)  ingest.cpp:183-266
    assemble_global_dfg(...)       ingest.cpp:386-450
    ingest_bundle(events, deps, cluster)   ingest.cpp:452-493

Pure host construction (string work; same op ids, hence the same index
order and tie-breaks as the reference). Tested against the reference's own
ingest_bundle on its synthetic bundles (tests/test_trace_ingest.py). The
generated-graph fast path for layered models is dfg_gen.cpp.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .errors import SchemaError, SpliceError, TransformError, UnknownSymbolError
from .graph import ClusterSpec, DeviceId, GlobalDFG, GraphBuilder, Op, OpKind, TensorUnit, \
    base_of_unit_name, is_computation, round_us
from .ingest import CommTopology, expand_tensor


@dataclass
class TraceEvent:
    """trace_io.hpp:32-43."""
    name: str
    node: str
    start: int = 0
    dur: int = 0
    kind: OpKind = OpKind.FW
    iteration: int = 0
    tensor: str = ""
    bytes: int = 0
    transaction: str = ""

    @staticmethod
    def from_dict(d: dict) -> "TraceEvent":
        return TraceEvent(d["name"], d["node"], int(d.get("start", 0)), int(d.get("dur", 0)),
                          OpKind(int(d.get("kind", 0))), int(d.get("iteration", 0)),
                          d.get("tensor", ""), int(d.get("bytes", 0)), d.get("transaction", ""))


@dataclass
class DependencySpec:
    """ingest.hpp DependencySpec: [pred, succ] name pairs, producer -> tensors,
    tensor -> bytes."""
    deps: list[tuple[str, str]] = field(default_factory=list)
    produces: dict[str, list[str]] = field(default_factory=dict)
    tensor_bytes: dict[str, int] = field(default_factory=dict)

    @staticmethod
    def from_json(j) -> "DependencySpec":
        if not isinstance(j, dict):
            raise SchemaError("dependency spec must be a JSON object", "deps")
        d = DependencySpec()
        if "deps" in j:
            if not isinstance(j["deps"], list):
                raise SchemaError("'deps' must be an array of [pred, succ] pairs", "deps")
            for pair in j["deps"]:
                if not (isinstance(pair, list) and len(pair) == 2 and
                        all(isinstance(x, str) for x in pair)):
                    raise SchemaError("'deps' entries must be [pred, succ] string pairs", "deps")
                d.deps.append((pair[0], pair[1]))
        if "produces" in j:
            if not isinstance(j["produces"], dict):
                raise SchemaError("'produces' must map op name to tensor list", "produces")
            for op, tensors in sorted(j["produces"].items()):
                if not isinstance(tensors, list):
                    raise SchemaError("'produces' values must be arrays", "produces")
                d.produces[op] = [str(t) for t in tensors]
        if "tensor_bytes" in j:
            if not isinstance(j["tensor_bytes"], dict):
                raise SchemaError("'tensor_bytes' must map tensor name to bytes", "tensor_bytes")
            for t, b in sorted(j["tensor_bytes"].items()):
                if not isinstance(b, int) or isinstance(b, bool):
                    raise SchemaError("'tensor_bytes' values must be integers", "tensor_bytes")
                d.tensor_bytes[t] = b
        return d


@dataclass
class OpProfile:
    comp_mean: dict[str, float] = field(default_factory=dict)
    recv_mean: dict[str, float] = field(default_factory=dict)


def op_duration_profile(events: list[TraceEvent]) -> OpProfile:
    """ingest.cpp:145-181."""
    send_start: dict[tuple[str, int], int] = {}
    for e in events:
        if e.kind == OpKind.SEND:
            send_start.setdefault((e.transaction, e.iteration), e.start)
    comp: dict[str, list] = {}
    recv: dict[str, list] = {}
    for e in events:
        if is_computation(e.kind):
            acc = comp.setdefault(f"{e.node}->{e.name}", [0.0, 0])
            acc[0] += float(e.dur)
            acc[1] += 1
        elif e.kind == OpKind.RECV:
            end = e.start + e.dur
            begin = max(e.start, send_start.get((e.transaction, e.iteration), e.start))
            acc = recv.setdefault(e.transaction, [0.0, 0])
            acc[0] += float(max(0, end - begin))
            acc[1] += 1
    return OpProfile({k: v[0] / v[1] for k, v in sorted(comp.items())},
                     {k: v[0] / v[1] for k, v in sorted(recv.items())})


@dataclass
class LocalDFG:
    node: str = ""
    ops: list[Op] = field(default_factory=list)
    edges: list[tuple[str, str]] = field(default_factory=list)
    tensor_inout: dict[str, tuple[str, str]] = field(default_factory=dict)


def build_local_dfg(events: list[TraceEvent], deps: DependencySpec) -> LocalDFG:
    """ingest.cpp:183-266: one node's computation ops (mean durations), an
    IN/OUT virtual pair per produced tensor, the dependency edges."""
    local = LocalDFG()
    durs: dict[str, list] = {}
    kinds: dict[str, OpKind] = {}
    for e in events:
        if not is_computation(e.kind):
            continue
        if not local.node:
            local.node = e.node
        elif local.node != e.node:
            raise SchemaError(f"local graph events span nodes {local.node} and {e.node}", "pid")
        acc = durs.setdefault(e.name, [0.0, 0])
        acc[0] += float(e.dur)
        acc[1] += 1
        kinds.setdefault(e.name, e.kind)
    dev = DeviceId.compute(local.node)
    for name in sorted(durs):
        acc = durs[name]
        local.ops.append(Op(f"{local.node}->{name}", kinds[name], local.node, dev,
                            round_us(acc[0] / acc[1]), produces=list(deps.produces.get(name, []))))
    for producer in sorted(deps.produces):
        if producer not in durs:
            continue
        for tensor in deps.produces[producer]:
            if tensor in local.tensor_inout:
                raise TransformError(f"tensor {tensor} has more than one producer on node "
                                     f"{local.node}")
            ins, outs = f"{local.node}->IN.{tensor}", f"{local.node}->OUT.{tensor}"
            local.ops.append(Op(ins, OpKind.VIRTUAL_IN, local.node, dev, 0))
            local.ops.append(Op(outs, OpKind.VIRTUAL_OUT, local.node, dev, 0))
            local.tensor_inout[tensor] = (ins, outs)
            local.edges.append((f"{local.node}->{producer}", ins))

    def resolve(name: str) -> str:
        if name in durs:
            return f"{local.node}->{name}"
        for prefix in ("IN(", "OUT("):
            if name.startswith(prefix) and name.endswith(")"):
                tensor = name[len(prefix):-1]
                if tensor not in local.tensor_inout:
                    raise UnknownSymbolError(name)
                return local.tensor_inout[tensor][0 if prefix == "IN(" else 1]
        raise UnknownSymbolError(name)

    for pred, succ in deps.deps:
        local.edges.append((resolve(pred), resolve(succ)))
    return local


def assemble_global_dfg(locals_: list[LocalDFG], topologies: list[CommTopology],
                        cluster: ClusterSpec) -> GlobalDFG:
    """ingest.cpp:386-450."""
    from .rewrite import validate
    b = GraphBuilder()
    b.set_cluster(cluster)
    for lo in locals_:
        for op in lo.ops:
            b.add_op(op)
    for lo in locals_:
        for x, y in lo.edges:
            b.add_edge(x, y)
    spliced = set()
    for topo in topologies:
        base = base_of_unit_name(topo.unit)
        for op in topo.ops:
            b.add_op(op)
        for x, y in topo.edges:
            b.add_edge(x, y)
        unit = TensorUnit(topo.unit, base, topo.bytes, topo.part_index, topo.part_count,
                          topo.ps_node, sorted(op.id for op in topo.ops))
        for node, ids in topo.entry.items():
            ins = f"{node}->IN.{base}"
            if not b.has_op(ins):
                raise SpliceError(f"tensor {topo.unit} enters at node {node} which has no {ins}")
            for i in ids:
                b.add_edge(ins, i)
            unit.vin[node] = ins
            spliced.add((node, base))
        for node, ids in topo.exit.items():
            outs = f"{node}->OUT.{base}"
            if not b.has_op(outs):
                raise SpliceError(f"tensor {topo.unit} exits at node {node} which has no {outs}")
            for i in ids:
                b.add_edge(i, outs)
            unit.vout[node] = outs
            spliced.add((node, base))
        b.add_tensor_unit(unit)
    for lo in locals_:
        for tensor in lo.tensor_inout:
            if (lo.node, tensor) not in spliced:
                raise SpliceError(f"tensor {tensor} has In/Out ops on node {lo.node} but no "
                                  "communication topology")
    g = b.build()
    if not validate(g):
        raise TransformError("assembled graph fails validation")
    return g


def ingest_bundle(events: list[TraceEvent], deps: DependencySpec,
                  cluster: ClusterSpec) -> GlobalDFG:
    """ingest.cpp:452-493."""
    profile = op_duration_profile(events)
    per_node: dict[str, list[TraceEvent]] = {}
    for e in events:
        if is_computation(e.kind):
            per_node.setdefault(e.node, []).append(e)
    locals_, tensors = [], set()
    for node in sorted(per_node):
        locals_.append(build_local_dfg(per_node[node], deps))
        tensors.update(locals_[-1].tensor_inout)
    topologies = []
    for tensor in sorted(tensors):
        if tensor not in deps.tensor_bytes:
            raise SchemaError(f"tensor_bytes has no entry for tensor {tensor}", "tensor_bytes")
        topo = expand_tensor(tensor, deps.tensor_bytes[tensor], cluster)
        for op in topo.ops:
            if op.kind == OpKind.RECV and op.transaction in profile.recv_mean:
                op.dur = round_us(profile.recv_mean[op.transaction])
        topologies.append(topo)
    return assemble_global_dfg(locals_, topologies, cluster)
