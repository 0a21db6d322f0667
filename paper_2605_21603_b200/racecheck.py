"""Static race detector for compiled schedules.

Two dispatches may run concurrently unless one happens-before the other
(same lane earlier, or reachable through the cross-lane event waits the
engine records).  For every unordered pair this checks the arena byte ranges
each dispatch reads and writes: a write/write or read/write overlap is a data
race the device would exhibit nondeterministically.  Works on
Session.schedule() / dry_run() dumps, so it runs on CPU.
"""
from __future__ import annotations

from typing import Dict, List, Tuple


def _ranges(launch: dict, which: str) -> List[Tuple[int, int]]:
    out = []
    for v in launch[which]:
        if v["src"] != "arena":
            continue
        n = 1
        for s in v["shape"]:
            n *= s
        lo = v["block_off"] + v["elem_offset"] * v["elem_bytes"]
        out.append((lo, lo + n * v["elem_bytes"]))
    if which == "out" and launch.get("ws_bytes", 0) > 0:
        out.append((launch["ws_off"], launch["ws_off"] + launch["ws_bytes"]))
    return out


def happens_before(sched: dict) -> List[int]:
    """Bitmask per dispatch of all dispatches that happen before it."""
    ds = sched["dispatches"]
    before = [0] * len(ds)
    last_on_lane: Dict[int, int] = {}
    for d in ds:
        i = d["id"]
        preds = list(d["wait_on"])
        if d["lane"] in last_on_lane:
            preds.append(last_on_lane[d["lane"]])
        m = 0
        for p in preds:
            m |= before[p] | (1 << p)
        before[i] = m
        last_on_lane[d["lane"]] = i
    return before


def find_races(sched: dict) -> List[tuple]:
    ds = sched["dispatches"]
    before = happens_before(sched)
    reads, writes = [], []
    for d in ds:
        r, w = [], []
        for l in d["launches"]:
            r += _ranges(l, "in")
            w += _ranges(l, "out")
        reads.append(r)
        writes.append(w)

    def overlap(a, b):
        return any(x0 < y1 and y0 < x1 for x0, x1 in a for y0, y1 in b)

    races = []
    for i in range(len(ds)):
        for j in range(i + 1, len(ds)):
            if (before[j] >> i) & 1:
                continue  # i happens before j (j cannot precede i in issue order)
            if overlap(writes[i], writes[j]) or overlap(writes[i], reads[j]) or overlap(reads[i], writes[j]):
                races.append((i, j, ds[i]["labels"], ds[j]["labels"]))
    return races
