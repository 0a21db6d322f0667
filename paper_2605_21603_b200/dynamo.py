"""TorchDynamo frontend: DynaFlow as a ``torch.compile`` backend.

The paper's user surface ("We built DynaFlow as a
torch.compile backend ... The frontend acquires the model's computational graph
by using TorchDynamo") over this repo's engine:

    import torch
    from paper_2605_21603_b200 import dynamo as dyn

    backend = dyn.backend(rules=[dyn.SplitModule(Attention), dyn.SplitFunc("attn_prefill")],
                          strategy={"name": "split_overlap", "n_microbatches": 2, "lane_mode": "ubatch"})
    fast = torch.compile(model, backend=backend, fullgraph=True, dynamic=False)
    y = fast(x, positions)

Graph-partition annotations: ``SplitFunc(pattern)`` splits
around a function call (``PartitionRule.by_func``), ``SplitModule(cls)`` at the
boundaries of every instance of an ``nn.Module`` class (``by_module`` on the
instance path from Dynamo's ``nn_module_stack``), and ``mark(tag)`` wraps any
code block (``by_region``; carried through ``torch.fx.traceback.annotate``).
Strategies are the same specs / ``opflow.Scheduler`` subclasses
``Session.run`` takes.

Lowering (FX graph -> the reference's ``GraphDescription``,
proj/include/opflow/graph.hpp:79-106): Dynamo's torch-level nodes map onto the
engine's operators —

    F.linear(x, W) / x @ W             -> MatMul (the weight bound as [K, N])
    torch.rms_norm(x, (H,), g, eps)    -> Custom rmsnorm
    a + b                              -> ElemAdd, or add_rmsnorm when the sum
                                          feeds an rms_norm (x1 and h outputs)
    torch.ops.opflow.rope / attn_prefill / silu_mul / all_reduce
                                       -> Custom rope / attn_prefill / silu_mul,
                                          AllReduce

Anything else raises ``opflow.Error`` (ConfigError) naming the op: the backend
never falls back to eager execution.  The ``torch.ops.opflow.*`` operators
carry eager PyTorch semantics so that the uncompiled model runs (that is the
user's reference model, not a path of this backend).

Runtime: one engine ``Session`` per compiled graph; weights are bound once
(frozen for inference: a weight whose version counter changes is re-copied and
re-packed); batched inputs are copied into static buffers so the captured CUDA
graph replays every call; outputs are cloned out of the static buffers unless
``static_outputs=True``.
"""
from __future__ import annotations

import contextlib
import operator
import re
from dataclasses import dataclass
from typing import Any, Dict, List, Optional, Sequence

import torch
import torch.nn.functional as F

from . import opflow as of

# ------------------------------------------------------------------ operator library
# Eager semantics (the uncompiled reference model); the compiled graph runs the
# engine's sm_100a kernels for these.


@torch.library.custom_op("opflow::rope", mutates_args=())
def rope(qkv: torch.Tensor, positions: torch.Tensor, heads: int, kv_heads: int, head_dim: int,
         theta: float) -> torch.Tensor:
    """Rotate-half RoPE on the q and k heads of fused qkv rows (v unrotated)."""
    y = qkv.float().clone()
    half = head_dim // 2
    inv = theta ** (-2.0 * torch.arange(half, dtype=torch.float64, device=qkv.device) / head_dim)
    ang = positions.double()[:, None] * inv[None, :]
    c, s = ang.cos().float(), ang.sin().float()
    for h in range(heads + kv_heads):
        a = y[:, h * head_dim:h * head_dim + half].clone()
        b = y[:, h * head_dim + half:(h + 1) * head_dim].clone()
        y[:, h * head_dim:h * head_dim + half] = a * c - b * s
        y[:, h * head_dim + half:(h + 1) * head_dim] = b * c + a * s
    return y.to(qkv.dtype)


@rope.register_fake
def _rope_fake(qkv, positions, heads, kv_heads, head_dim, theta):
    return torch.empty_like(qkv)


@torch.library.custom_op("opflow::attn_prefill", mutates_args=())
def attn_prefill(qkv: torch.Tensor, heads: int, kv_heads: int, head_dim: int, seq_len: int) -> torch.Tensor:
    """Causal GQA attention over fused qkv rows, sequences of seq_len rows."""
    T = qkv.shape[0]
    n = T // seq_len
    x = qkv.float().view(n, seq_len, heads + 2 * kv_heads, head_dim).transpose(1, 2)
    q, k, v = x[:, :heads], x[:, heads:heads + kv_heads], x[:, heads + kv_heads:]
    grp = heads // kv_heads
    k = k.repeat_interleave(grp, dim=1)
    v = v.repeat_interleave(grp, dim=1)
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    return o.transpose(1, 2).reshape(T, heads * head_dim).to(qkv.dtype)


@attn_prefill.register_fake
def _attn_prefill_fake(qkv, heads, kv_heads, head_dim, seq_len):
    return qkv.new_empty(qkv.shape[0], heads * head_dim)


@torch.library.custom_op("opflow::silu_mul", mutates_args=())
def silu_mul(gu: torch.Tensor) -> torch.Tensor:
    """silu(gate) * up over [gate | up] halves."""
    g, u = gu.float().chunk(2, dim=-1)
    return (F.silu(g) * u).to(gu.dtype)


@silu_mul.register_fake
def _silu_mul_fake(gu):
    return gu.new_empty(gu.shape[0], gu.shape[1] // 2)


@torch.library.custom_op("opflow::all_reduce", mutates_args=())
def all_reduce(x: torch.Tensor, world_size: int) -> torch.Tensor:
    """Sum over the tensor-parallel group.  Without an initialised process group
    this is the reference's single-process stand-in, x * world_size
    (proj/src/eval.cpp:63-70)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() == world_size and world_size > 1:
        y = x.clone()
        dist.all_reduce(y)
        return y
    return x * world_size


@all_reduce.register_fake
def _all_reduce_fake(x, world_size):
    return torch.empty_like(x)


# ------------------------------------------------------------------ annotations
@dataclass(frozen=True)
class SplitFunc:
    """Split around calls of a function: its ops become their
    own subgraphs (``PartitionRule.by_func``; the pattern globs the op's
    function name, e.g. "attn_prefill", "AllReduce", "rmsnorm")."""
    pattern: str


@dataclass(frozen=True)
class SplitModule:
    """Split on the boundaries of every instance of a module class
    (``PartitionRule.by_module`` on each instance path)."""
    target_cls: type


@contextlib.contextmanager
def mark(tag: str):
    """Split on a code block: ops traced inside carry the
    region tag (``PartitionRule.by_region``)."""
    import torch.fx.traceback as fxt
    with fxt.annotate({"opflow_region": tag}):
        yield


# ------------------------------------------------------------------ lowering
_DT = {torch.bfloat16: "bf16", torch.float32: "f32", torch.int64: "i64"}


def _module_path(stack_path: str) -> str:
    """Dynamo's "L['self'].layers[0].attn" / "L['s'].layers.0.attn" -> "layers.0.attn"."""
    p = re.sub(r"^L\['[^']*'\]\.?", "", stack_path)
    p = re.sub(r"\[(\w+)\]", r".\1", p)
    p = re.sub(r"\['([^']*)'\]", r".\1", p)
    return p.strip(".")


def _param_name(node_name: str) -> str:
    """Dynamo placeholder "l_self_modules_layers_modules_0_modules_norm_parameters_weight_"
    -> "layers.0.norm.weight"; user inputs "l_x_" -> "x"."""
    s = node_name
    if s.startswith("l_"):
        s = s[2:]
    s = s.rstrip("_")
    m = re.match(r"^[^_]+_((?:modules|parameters|buffers)_.*)$", s)
    if m:
        s = m.group(1)
        s = re.sub(r"(^|_)(modules|parameters|buffers)_", ".", s).strip(".")
    return s


@dataclass
class Lowered:
    """A Dynamo graph restated as a GraphDescription plus how to bind it."""
    description: dict
    inputs: List[tuple]           # (tensor name, placeholder index, "batched" | "weight" | "weight_t")
    outputs: List[tuple]          # (tensor name, shape, torch dtype)
    rows: int
    rules: List[of.PartitionRule]

    def json(self) -> str:
        import json
        return json.dumps(self.description)


def _tgt(node) -> Any:
    t = node.target
    return getattr(t, "_overloadpacket", t)


def lower(gm: torch.fx.GraphModule, example_inputs: Sequence[Any], annotations: Sequence[Any] = ()) -> Lowered:
    """FX graph from TorchDynamo -> GraphDescription (see the module docstring)."""
    nodes = list(gm.graph.nodes)
    placeholders = [n for n in nodes if n.op == "placeholder"]
    if len(placeholders) != len(example_inputs):
        raise of.Error(int(of.Errc.ConfigError), "DynaFlow backend: placeholder / example input mismatch")
    ex_of = {n: e for n, e in zip(placeholders, example_inputs)}
    users: Dict[Any, list] = {n: list(n.users) for n in nodes}
    # which placeholders are weights, and which are used transposed (F.linear)
    linear_w = {n.args[1] for n in nodes if n.op == "call_function" and n.target is F.linear}

    def meta(n):
        v = n.meta.get("example_value")
        if v is None and n in ex_of:
            v = ex_of[n]
        return v

    tensors, ops, names = [], [], {}
    inputs, outputs = [], []
    rows = 0
    used_names: Dict[str, int] = {}

    def uniq(base: str) -> str:
        k = used_names.get(base, 0)
        used_names[base] = k + 1
        return base if k == 0 else f"{base}#{k}"

    def err(msg: str):
        raise of.Error(int(of.Errc.ConfigError), "DynaFlow backend: " + msg)

    for i, n in enumerate(placeholders):
        e = ex_of[n]
        if not isinstance(e, torch.Tensor):
            err(f"non-tensor graph input {n.name} ({type(e).__name__}); compile with dynamic=False")
        if e.dtype not in _DT:
            err(f"unsupported dtype {e.dtype} for {n.name}")
        is_w = isinstance(e, torch.nn.Parameter) or n in linear_w
        name = uniq(_param_name(n.name))
        names[n] = name
        if is_w:
            if n in linear_w:
                if e.dim() != 2:
                    err(f"linear weight {name} must be 2-D")
                shape = [int(e.shape[1]), int(e.shape[0])]  # bound transposed: [K, N]
                kind = "weight_t"
            else:
                shape = [int(s) for s in e.shape]
                kind = "weight"
            tensors.append({"name": name, "shape": shape, "batch": "replicated", "dtype": _DT[e.dtype],
                            "role": "weight"})
        else:
            if e.dim() < 1:
                err(f"scalar graph input {name}")
            rows = rows or int(e.shape[0])
            if int(e.shape[0]) != rows:
                err("batched inputs disagree on rows (dim 0)")
            tensors.append({"name": name, "shape": [int(s) for s in e.shape], "batch": "batched",
                            "dtype": _DT[e.dtype], "role": "input"})
            kind = "batched"
        inputs.append((name, i, kind))

    def op_common(n) -> dict:
        stack = n.meta.get("nn_module_stack") or {}
        path = _module_path(list(stack.values())[-1][0]) if stack else ""
        custom = n.meta.get("custom") or {}
        tags = [custom["opflow_region"]] if "opflow_region" in custom else []
        return {"module_path": path, "region_tags": tags}

    def out_tensor(n, suffix: str = "") -> str:
        v = meta(n)
        if not isinstance(v, torch.Tensor):
            err(f"{n.name}: non-tensor value")
        if v.dtype not in _DT:
            err(f"{n.name}: unsupported dtype {v.dtype}")
        common = op_common(n)
        name = uniq((common["module_path"] + "." if common["module_path"] else "") + n.name + suffix)
        tensors.append({"name": name, "shape": [int(s) for s in v.shape], "batch": "batched",
                        "dtype": _DT[v.dtype], "role": "intermediate"})
        return name

    def ref(a) -> str:
        if a not in names:
            err(f"operand {a} is not a tensor produced in the graph")
        return names[a]

    fused_norm = set()  # rms_norm nodes folded into a preceding add (add_rmsnorm)
    for n in nodes:
        if n.op in ("placeholder", "output"):
            continue
        if n.op != "call_function":
            err(f"unsupported node {n.op} {n.target}")
        if n in fused_norm:
            continue
        t = _tgt(n)
        common = op_common(n)
        opname = uniq((common["module_path"] + "." if common["module_path"] else "") + n.name)
        if t is F.linear:
            x, w = n.args[0], n.args[1]
            bias = n.args[2] if len(n.args) > 2 else n.kwargs.get("bias")
            if bias is not None:
                err(f"{n.name}: F.linear with a bias is not lowered")
            names[n] = out_tensor(n)
            ops.append({"name": opname, "kind": "MatMul", "inputs": [ref(x), ref(w)], "outputs": [names[n]],
                        **common})
        elif t in (torch.matmul, operator.matmul):
            x, w = n.args
            if tensors[[tt["name"] for tt in tensors].index(ref(w))]["role"] != "weight":
                err(f"{n.name}: matmul's right operand must be a weight")
            names[n] = out_tensor(n)
            ops.append({"name": opname, "kind": "MatMul", "inputs": [ref(x), ref(w)], "outputs": [names[n]],
                        **common})
        elif t is torch.rms_norm or t is F.rms_norm:
            x, _shape, g = n.args[0], n.args[1], n.args[2] if len(n.args) > 2 else n.kwargs.get("weight")
            eps = n.args[3] if len(n.args) > 3 else n.kwargs.get("eps")
            if g is None or eps is None:
                err(f"{n.name}: rms_norm needs a weight and an explicit eps")
            names[n] = out_tensor(n)
            ops.append({"name": opname, "kind": "Custom", "inputs": [ref(x), ref(g)], "outputs": [names[n]],
                        "resource_class": "memory", **common,
                        "attrs": {"custom_name": "rmsnorm", "params": {"eps": float(eps)}}})
        elif t in (operator.add, torch.add):
            a, b = n.args[0], n.args[1]
            if n.kwargs.get("alpha", 1) != 1:
                err(f"{n.name}: add with alpha")
            norms = [u for u in users[n] if u.op == "call_function" and _tgt(u) in (torch.rms_norm, F.rms_norm)]
            if norms:  # residual add feeding a norm: one add_rmsnorm (x1, h)
                nn_ = norms[0]
                g = nn_.args[2] if len(nn_.args) > 2 else nn_.kwargs.get("weight")
                eps = nn_.args[3] if len(nn_.args) > 3 else nn_.kwargs.get("eps")
                if g is None or eps is None:
                    err(f"{nn_.name}: rms_norm needs a weight and an explicit eps")
                names[n] = out_tensor(n)
                names[nn_] = out_tensor(nn_)
                fused_norm.add(nn_)
                tags = op_common(nn_)["region_tags"]  # a mark() around the norm tags the fused op
                common = dict(common, region_tags=sorted(set(common["region_tags"]) | set(tags)))
                ops.append({"name": opname, "kind": "Custom", "inputs": [ref(a), ref(b), ref(g)],
                            "outputs": [names[n], names[nn_]], "resource_class": "memory", **common,
                            "attrs": {"custom_name": "add_rmsnorm", "params": {"eps": float(eps)}}})
            else:
                names[n] = out_tensor(n)
                ops.append({"name": opname, "kind": "ElemAdd", "inputs": [ref(a), ref(b)], "outputs": [names[n]],
                            **common})
        elif t is torch.ops.opflow.rope:
            qkv, pos, heads, kvh, hd, theta = n.args
            names[n] = out_tensor(n)
            ops.append({"name": opname, "kind": "Custom", "inputs": [ref(qkv), ref(pos)], "outputs": [names[n]],
                        "resource_class": "memory", **common,
                        "attrs": {"custom_name": "rope", "params": {"heads": heads, "kv_heads": kvh,
                                                                    "head_dim": hd, "theta": float(theta)}}})
        elif t is torch.ops.opflow.attn_prefill:
            qkv, heads, kvh, hd, S = n.args
            names[n] = out_tensor(n)
            ops.append({"name": opname, "kind": "Custom", "inputs": [ref(qkv)], "outputs": [names[n]],
                        "resource_class": "compute", **common,
                        "attrs": {"custom_name": "attn_prefill", "params": {"heads": heads, "kv_heads": kvh,
                                                                            "head_dim": hd, "seq_len": S}}})
        elif t is torch.ops.opflow.silu_mul:
            names[n] = out_tensor(n)
            ops.append({"name": opname, "kind": "Custom", "inputs": [ref(n.args[0])], "outputs": [names[n]],
                        "resource_class": "memory", **common, "attrs": {"custom_name": "silu_mul", "params": {}}})
        elif t is torch.ops.opflow.all_reduce:
            names[n] = out_tensor(n)
            ops.append({"name": opname, "kind": "AllReduce", "inputs": [ref(n.args[0])], "outputs": [names[n]],
                        **common, "attrs": {"world_size": int(n.args[1])}})
        else:
            err(f"unsupported op {getattr(t, '__name__', t)} (node {n.name}); supported: F.linear, matmul, "
                "torch.rms_norm, add, torch.ops.opflow.{rope, attn_prefill, silu_mul, all_reduce}")

    out_node = [n for n in nodes if n.op == "output"][0]
    outs = out_node.args[0]
    outs = list(outs) if isinstance(outs, (tuple, list)) else [outs]
    tix = {t["name"]: t for t in tensors}
    for o in outs:
        nm = ref(o)
        if tix[nm]["role"] != "intermediate":
            err(f"graph output {nm} is an input or weight")
        tix[nm]["role"] = "output"
        v = meta(o)
        outputs.append((nm, tuple(int(s) for s in v.shape), v.dtype))
    desc = {"tensors": tensors, "operators": ops}

    # annotations -> the reference's partition rules
    rules: List[of.PartitionRule] = []
    for a in annotations:
        if isinstance(a, SplitFunc):
            rules.append(of.PartitionRule.by_func(a.pattern))
        elif isinstance(a, SplitModule):
            paths = []
            for n in nodes:
                for path, cls in (n.meta.get("nn_module_stack") or {}).values():
                    if isinstance(cls, type) and issubclass(cls, a.target_cls):
                        p = _module_path(path)
                        if p and p not in paths:
                            paths.append(p)
            rules += [of.PartitionRule.by_module(p) for p in paths]
        elif isinstance(a, str):  # a mark() tag
            rules.append(of.PartitionRule.by_region(a))
        elif isinstance(a, of.PartitionRule):
            rules.append(a)
        else:
            err(f"unknown annotation {a!r}")
    return Lowered(desc, inputs, outputs, rows, rules)


# ------------------------------------------------------------------ runtime
class CompiledGraph:
    """One compiled Dynamo graph: engine Session + static input / output buffers."""

    def __init__(self, lowered: Lowered, strategy: Any, config: Optional[dict], comm, static_outputs: bool):
        self.lowered = lowered
        self.graph = of.build_graph(lowered.json())
        self.plan = of.partition(self.graph, lowered.rules)
        self.strategy = strategy
        self.config = dict(config or {})
        self.comm = comm
        self.static_outputs = static_outputs
        self.sess: Optional[of.Session] = None
        self.static: Dict[str, torch.Tensor] = {}
        self.wkey: Dict[str, tuple] = {}
        self.outs: List[torch.Tensor] = []

    def __call__(self, *args):
        low = self.lowered
        dev = None
        for name, i, kind in low.inputs:
            if kind == "batched":
                dev = args[i].device
                break
        if dev is None:
            dev = args[low.inputs[0][1]].device
        if dev.type != "cuda":
            raise of.Error(int(of.Errc.ConfigError),
                           "DynaFlow backend: inputs must be CUDA tensors (the engine has no CPU path)")
        if self.sess is None:
            cfg = {"lanes": 3, "device": dev.index or 0}
            cfg.update(self.config)
            self.sess = of.Session(self.graph, self.plan, cfg, self.comm)
            for nm, shape, dt in low.outputs:
                t = torch.empty(shape, dtype=dt, device=dev)
                self.outs.append(t)
                self.sess.bind(nm, t)
        for name, i, kind in low.inputs:
            x = args[i]
            if kind == "batched":
                buf = self.static.get(name)
                if buf is None:
                    buf = torch.empty_like(x, memory_format=torch.contiguous_format)
                    self.static[name] = buf
                    self.sess.bind(name, buf)
                buf.copy_(x, non_blocking=True)
                continue
            key = (x.data_ptr(), x._version)
            if self.wkey.get(name) == key:
                continue
            w = x.detach()
            w = w.t().contiguous() if kind == "weight_t" else w.contiguous().clone()
            self.static[name] = w
            self.wkey[name] = key
            self.sess.bind(name, w)
        self.sess.run(self.strategy, torch.cuda.current_stream(dev))
        if self.static_outputs:
            return list(self.outs)
        return [o.clone() for o in self.outs]


class DynaFlowBackend:
    """``torch.compile(model, backend=DynaFlowBackend(...))``.

    rules: SplitFunc / SplitModule / mark tags (str) / opflow.PartitionRule.
    strategy: a strategy spec (dict) or an ``opflow.Scheduler`` instance.
    config: Session config overrides ({"lanes": 3} by default).
    dry: lower and plan only (``self.lowered`` / ``self.plans``), then run the
         captured graph eagerly — for inspecting the lowering on a host without
         a GPU; the engine is not involved.
    """

    def __init__(self, rules: Sequence[Any] = (), strategy: Any = None, config: Optional[dict] = None,
                 comm=None, static_outputs: bool = False, dry: bool = False):
        self.rules = list(rules)
        self.strategy = strategy if strategy is not None else {"name": "sequential"}
        self.config = config
        self.comm = comm
        self.static_outputs = static_outputs
        self.dry = dry
        self.lowered: List[Lowered] = []
        self.compiled: List[CompiledGraph] = []

    def __call__(self, gm: torch.fx.GraphModule, example_inputs):
        low = lower(gm, example_inputs, self.rules)
        self.lowered.append(low)
        if self.dry:
            g = of.build_graph(low.json())
            of.validate_plan(of.partition(g, low.rules), g)
            return gm.forward
        cg = CompiledGraph(low, self.strategy, self.config, self.comm, self.static_outputs)
        self.compiled.append(cg)
        return cg


def backend(rules: Sequence[Any] = (), strategy: Any = None, config: Optional[dict] = None, comm=None,
            static_outputs: bool = False, dry: bool = False) -> DynaFlowBackend:
    return DynaFlowBackend(rules, strategy, config, comm, static_outputs, dry)


__all__ = ["SplitFunc", "SplitModule", "mark", "backend", "DynaFlowBackend", "lower", "Lowered",
           "rope", "attn_prefill", "silu_mul", "all_reduce"]
