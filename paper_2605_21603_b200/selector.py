"""Context-aware strategy selection from measured B200 timings.

DynaFlow's claim is that the best schedule depends on the batch (PAPER.md
78-83, 606-608): splitting into nano-batches adds a fixed cost per extra
micro-batch ("an additional read of the model weights", SPEC.md CostParams,
SPEC.md:47-50) and only pays once enough per-token work can overlap.  The SPEC
models every duration as `alpha + beta * rows` and guards the
split strategies with a token threshold.  This module fits
that model from the engine's own device timings instead of assuming it:

* `StrategySelector` — per candidate schedule, the forward time
  t_c(rows) = alpha_c + beta_c * rows, least squares over calibration row
  counts (alpha, beta >= 0, the SPEC invariant).  `choose(rows)` is the argmin;
  the crossovers of the fitted lines are the split thresholds, emitted as a
  decision table `{"name": "auto", "table": [...]}` that the engine resolves per
  batch without timing (`Session::choose`), one cached CUDA graph per decision.
  `margin` keeps the first candidate (normally `sequential`) unless another is
  predicted faster by that fraction — the threshold guard.
* `fit_op_costs` / `apply_op_costs` — per operator alpha/beta from the engine's
  per-launch trace at several row counts, written back into a graph
  description's op `cost` (what `partition`'s dominant class weighs,
  `proj/src/partition.cpp:55-70`).

Host logic only (numpy); the timings come from `calibrate()` on a device
session or from any callable.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import Any, Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np


def fit_line(rows: Sequence[float], ms: Sequence[float]) -> Tuple[float, float]:
    """Least-squares alpha + beta * rows with alpha, beta >= 0 (SPEC CostParams
    invariant).  One point: a pure per-row slope (alpha 0)."""
    r = np.asarray(rows, dtype=np.float64)
    t = np.asarray(ms, dtype=np.float64)
    if r.size == 0:
        raise ValueError("fit_line needs at least one point")
    if r.size == 1 or np.ptp(r) == 0:
        return 0.0, float(max(t.mean(), 0.0) / max(r.mean(), 1.0))
    beta, alpha = np.polyfit(r, t, 1)
    if alpha < 0:  # refit through the origin
        alpha, beta = 0.0, float((r * t).sum() / (r * r).sum())
    if beta < 0:  # rows-independent
        alpha, beta = float(t.mean()), 0.0
    return float(max(alpha, 0.0)), float(max(beta, 0.0))


def _key(spec: Any) -> str:
    return json.dumps(spec, sort_keys=True)


@dataclass
class StrategySelector:
    """Fitted per-candidate cost lines and the rows -> strategy decision."""

    candidates: List[dict]
    margin: float = 0.0
    samples: Dict[str, List[Tuple[int, float]]] = field(default_factory=dict)
    lines: Dict[str, Tuple[float, float]] = field(default_factory=dict)

    def __post_init__(self):
        if not self.candidates:
            raise ValueError("StrategySelector needs at least one candidate")
        if not 0.0 <= self.margin < 1.0:
            raise ValueError("margin must be in [0, 1)")
        for c in self.candidates:
            self.samples.setdefault(_key(c), [])

    # ---- calibration data
    def add(self, spec: dict, rows: int, ms: float) -> None:
        k = _key(spec)
        if k not in self.samples:
            raise KeyError(f"not a candidate: {spec}")
        self.samples[k].append((int(rows), float(ms)))

    def fit(self) -> "StrategySelector":
        for c in self.candidates:
            pts = self.samples[_key(c)]
            if not pts:
                raise ValueError(f"no timings for candidate {c}")
            self.lines[_key(c)] = fit_line([p[0] for p in pts], [p[1] for p in pts])
        return self

    # ---- prediction
    def predict(self, spec: dict, rows: int) -> float:
        a, b = self.lines[_key(spec)]
        return a + b * rows

    def _score(self, i: int) -> Tuple[float, float]:
        """Comparison line of candidate i: the baseline (index 0) is credited
        with the margin, so a challenger must beat it by that fraction."""
        a, b = self.lines[_key(self.candidates[i])]
        return (a * (1.0 - self.margin), b * (1.0 - self.margin)) if i == 0 else (a, b)

    def _argmin(self, rows: int) -> int:
        best, best_v = 0, math.inf
        for i in range(len(self.candidates)):
            a, b = self._score(i)
            v = a + b * rows
            if v < best_v - 1e-12:  # ties keep the earlier candidate
                best, best_v = i, v
        return best

    def choose(self, rows: int) -> dict:
        if not self.lines:
            self.fit()
        return self.candidates[self._argmin(int(rows))]

    def table(self) -> List[dict]:
        """Exact lower envelope of the fitted lines over rows >= 0, as
        [{"min_rows": R, "strategy": spec}, ...] (R ascending, first R = 0).
        The argmin of lines only changes at pairwise crossovers, so evaluating
        at 0 and on both sides of every crossover is exhaustive."""
        if not self.lines:
            self.fit()
        pts = {0}
        n = len(self.candidates)
        for i in range(n):
            ai, bi = self._score(i)
            for j in range(i + 1, n):
                aj, bj = self._score(j)
                if bi != bj:
                    x = (aj - ai) / (bi - bj)
                    if x > 0 and math.isfinite(x):
                        f = int(math.floor(x))  # +-1 around it: near-ties in floating point
                        pts.update(r for r in (f - 1, f, f + 1, f + 2) if r >= 0)
        out: List[dict] = []
        for r in sorted(pts):
            w = self._argmin(r)
            if not out or _key(out[-1]["strategy"]) != _key(self.candidates[w]):
                out.append({"min_rows": r, "strategy": self.candidates[w]})
        return out

    def thresholds(self) -> List[int]:
        """Row counts where the chosen strategy changes (the split thresholds)."""
        return [e["min_rows"] for e in self.table()[1:]]

    def spec(self) -> dict:
        """The engine-side decision table (`Session::choose`, no run-time timing)."""
        return {"name": "auto", "table": self.table()}

    def report(self) -> dict:
        return {"margin": self.margin,
                "lines_ms": [{"strategy": c, "alpha_ms": self.lines[_key(c)][0],
                              "beta_ms_per_row": self.lines[_key(c)][1],
                              "samples": sorted(self.samples[_key(c)])} for c in self.candidates],
                "table": self.table()}


# ------------------------------------------------------------------ device calibration
def time_forward(session, spec: dict, reps: int = 5, warmup: int = 1) -> float:
    """Device ms per forward of `spec` on a bound session (CUDA events on the
    launching stream; the first run builds and captures the plan)."""
    import torch
    st = torch.cuda.current_stream()
    for _ in range(max(1, warmup)):
        session.run(spec, stream=st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        session.run(spec, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def calibrate(bind_rows: Callable[[int], Any], candidates: Sequence[dict], rows_points: Sequence[int],
              reps: int = 5, rounds: int = 3, margin: float = 0.0) -> StrategySelector:
    """Time every candidate at every calibration row count and fit.  `bind_rows(r)`
    returns a session whose batched inputs / outputs are bound with r rows (e.g.
    row-prefix views of max-size buffers).  Candidates are timed in `rounds`
    interleaved passes and the median kept, so GPU clock drift (B200 power
    capping) does not favour whichever runs first."""
    sel = StrategySelector(list(candidates), margin=margin)
    for r in rows_points:
        s = bind_rows(int(r))
        per: Dict[str, List[float]] = {_key(c): [] for c in candidates}
        for _ in range(max(1, rounds)):
            for c in candidates:
                per[_key(c)].append(time_forward(s, c, reps=reps))
        for c in candidates:
            sel.add(c, r, float(np.median(per[_key(c)])))
    return sel.fit()


# ------------------------------------------------------------------ per-operator costs
def op_times_from_trace(trace: Sequence[dict]) -> Dict[str, float]:
    """Per-op device ms from a per-launch engine trace (`Session.trace()` with
    OPF_TRACE_LAUNCHES=1; event names are "<op> u<k>", dur in microseconds).
    Nano-batch launches of one op are summed."""
    out: Dict[str, float] = {}
    for e in trace:
        name = e.get("name", "")
        op = name.rsplit(" u", 1)[0] if " u" in name else name
        out[op] = out.get(op, 0.0) + float(e.get("dur", 0.0)) * 1e-3
    return out


def trace_op_times(session, spec: Optional[dict] = None) -> Dict[str, float]:
    """Run `spec` (default sequential) once, then a per-launch profiled replay."""
    session.run(spec or {"name": "sequential"})
    prev = os.environ.get("OPF_TRACE_LAUNCHES")
    os.environ["OPF_TRACE_LAUNCHES"] = "1"
    try:
        tr = session.trace()
    finally:
        if prev is None:
            os.environ.pop("OPF_TRACE_LAUNCHES", None)
        else:
            os.environ["OPF_TRACE_LAUNCHES"] = prev
    return op_times_from_trace(tr)


def fit_op_costs(points: Dict[int, Dict[str, float]]) -> Dict[str, Tuple[float, float]]:
    """{rows: {op: ms}} -> {op: (alpha, beta)} in microseconds (alpha per
    invocation, beta per row), the units of the builders' CostParams."""
    ops = sorted({o for m in points.values() for o in m})
    out = {}
    for o in ops:
        rs = [r for r in sorted(points) if o in points[r]]
        a, b = fit_line(rs, [points[r][o] * 1e3 for r in rs])
        out[o] = (a, b)
    return out


def apply_op_costs(desc: Any, costs: Dict[str, Tuple[float, float]]) -> Any:
    """Copy of a graph description (GraphDescription, dict or JSON text) with
    each measured op's `cost` replaced by its fitted (alpha, beta).  Ops with
    no launch of their own (fused into a producer's epilogue) get (0, 0)."""
    from . import opflow as of
    if isinstance(desc, of.GraphDescription):
        g = of.GraphDescription.from_json(desc.to_json())
        for op in g.operators:
            if op.name in costs:
                op.cost = of.CostParams(*costs[op.name])
            elif op.cost is not None and costs:
                op.cost = of.CostParams(0.0, 0.0)
        return g
    d = json.loads(desc) if isinstance(desc, str) else json.loads(json.dumps(desc))
    for op in d["operators"]:
        if op["name"] in costs:
            op["cost"] = list(costs[op["name"]])
        elif "cost" in op and costs:
            op["cost"] = [0.0, 0.0]
    return d if not isinstance(desc, str) else json.dumps(d)
