"""Report writers for replayed schedules.

    timeline_json(g, result)        proj/tools/dpro_main.cpp:90-116: one Chrome
                                    Trace "X" slice per non-virtual op, one
                                    process lane per device
    timeline_text(g, result)        ... serialized like the CLI's write_json
                                    (dpro_main.cpp:64-70: nlohmann dump(2) +
                                    newline: sorted keys, 2-space indent), so
                                    the bytes equal the CLI's timeline.json
    write_timeline(path, g, result)

Tested byte for byte against the reference's timeline on its own graphs
(tests/test_report.py).
"""
from __future__ import annotations

import json

from .graph import GlobalDFG, is_communication, is_virtual


def timeline_json(g: GlobalDFG, result) -> dict:
    events = []
    for op in g.ops():  # the schedule map's order: ids ascending
        if is_virtual(op.kind):
            continue
        e = result.schedule[op.id]
        kind = op.kind.name
        args = {"kind": kind, "iteration": 0}
        if is_communication(op.kind):
            args.update(tensor=op.tensor, bytes=int(op.bytes), transaction=op.transaction)
        events.append({"name": op.id, "ph": "X", "pid": e.device.str(), "tid": op.node,
                       "ts": int(e.start), "dur": int(e.end - e.start), "cat": kind,
                       "args": args})
    return {"traceEvents": events, "displayTimeUnit": "ms"}


def timeline_text(g: GlobalDFG, result) -> str:
    # nlohmann::json dump(2): object keys in byte order, ", " never used
    # (one item per line), ": " between key and value, UTF-8 kept as is
    return json.dumps(timeline_json(g, result), indent=2, sort_keys=True,
                      ensure_ascii=False) + "\n"


def write_timeline(path: str, g: GlobalDFG, result) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write(timeline_text(g, result))
