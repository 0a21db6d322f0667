"""Python host API over the C-ABI, mirroring the reference's opflow interface.

Same names and meaning as /root/reference/proj/include/opflow/*.hpp
(GraphDescription / TensorDecl / OpDecl / build_graph / PartitionRule /
partition / validate_plan / builders / alltoall_permutation, the Errc error
taxonomy raised as `Error`), plus the SPEC's scheduling API
(split / get_ready_ops / execute) and the B200 `Session`.

Everything runs in libopflow_b200.so; this module only marshals JSON and
pointers.  Device memory and streams come from PyTorch (plumbing only).
"""
from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass, field
from typing import Any, Callable, Dict, Iterable, List, Optional, Sequence

from . import _lib
from ._lib import ERRC, lib, opf_handle, opf_view, take_string

Errc = enum.IntEnum("Errc", {name: i for i, name in enumerate(ERRC)})


class Error(RuntimeError):
    """opflow::Error: carries the Errc code (reference common.hpp:50-58)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRC[code] if 0 <= code < len(ERRC) else code}: {msg}")
        self.code = Errc(code) if 0 <= code < len(ERRC) else code


def check(status: int) -> None:
    if status != 0:
        raise Error(status - 1, lib().opf_last_error().decode(errors="replace"))


class Dtype(enum.IntEnum):
    kI64 = 0
    kF32 = 1
    kBF16 = 2


DTYPE_NAME = {Dtype.kI64: "i64", Dtype.kF32: "f32", Dtype.kBF16: "bf16"}


class BatchSemantics(enum.IntEnum):
    kBatched = 0
    kReplicated = 1


class TensorRole(enum.IntEnum):
    kGraphInput = 0
    kWeight = 1
    kIntermediate = 2
    kGraphOutput = 3


ROLE_NAME = {TensorRole.kGraphInput: "input", TensorRole.kWeight: "weight",
             TensorRole.kIntermediate: "intermediate", TensorRole.kGraphOutput: "output"}


class OperatorKind(enum.IntEnum):
    kMatMul = 0
    kElemAdd = 1
    kRowScale = 2
    kAllReduce = 3
    kAllToAll = 4
    kAttention = 5
    kCustom = 6


KIND_NAME = ["MatMul", "ElemAdd", "RowScale", "AllReduce", "AllToAll", "Attention", "Custom"]


class ResourceClass(enum.IntEnum):
    kCompute = 0
    kMemory = 1
    kNetwork = 2


RC_NAME = ["compute", "memory", "network"]


@dataclass
class CostParams:
    alpha: float = 0.0
    beta: float = 0.0


@dataclass
class OpAttrs:
    world_size: int = 1
    seed: int = 0
    custom_name: str = ""
    params: Dict[str, float] = field(default_factory=dict)


@dataclass
class TensorDecl:
    name: str
    shape: List[int]
    batch: BatchSemantics = BatchSemantics.kBatched
    dtype: Dtype = Dtype.kI64
    role: TensorRole = TensorRole.kIntermediate


@dataclass
class OpDecl:
    name: str = ""
    kind: OperatorKind = OperatorKind.kElemAdd
    inputs: List[str] = field(default_factory=list)
    outputs: List[str] = field(default_factory=list)
    resource_class: Optional[ResourceClass] = None
    module_path: str = ""
    region_tags: List[str] = field(default_factory=list)
    cost: Optional[CostParams] = None
    attrs: OpAttrs = field(default_factory=OpAttrs)

    def to_json(self) -> dict:
        d = {"name": self.name, "kind": KIND_NAME[int(self.kind)], "inputs": list(self.inputs),
             "outputs": list(self.outputs), "module_path": self.module_path,
             "region_tags": list(self.region_tags),
             "attrs": {"world_size": int(self.attrs.world_size), "seed": int(self.attrs.seed),
                       "custom_name": self.attrs.custom_name,
                       "params": {k: float(v) for k, v in self.attrs.params.items()}}}
        if self.resource_class is not None:
            d["resource_class"] = RC_NAME[int(self.resource_class)]
        if self.cost is not None:
            d["cost"] = [float(self.cost.alpha), float(self.cost.beta)]
        return d


@dataclass
class GraphDescription:
    tensors: List[TensorDecl] = field(default_factory=list)
    operators: List[OpDecl] = field(default_factory=list)

    def to_json(self) -> str:
        return json.dumps({
            "tensors": [{"name": t.name, "shape": [int(x) for x in t.shape],
                         "batch": "batched" if t.batch == BatchSemantics.kBatched else "replicated",
                         "dtype": DTYPE_NAME[Dtype(t.dtype)], "role": ROLE_NAME[TensorRole(t.role)]}
                        for t in self.tensors],
            "operators": [o.to_json() for o in self.operators]})

    @staticmethod
    def from_json(text: str) -> "GraphDescription":
        d = json.loads(text)
        inv_role = {v: k for k, v in ROLE_NAME.items()}
        inv_dt = {v: k for k, v in DTYPE_NAME.items()}
        g = GraphDescription()
        for t in d["tensors"]:
            g.tensors.append(TensorDecl(t["name"], list(t["shape"]),
                                        BatchSemantics.kBatched if t.get("batch", "batched") == "batched"
                                        else BatchSemantics.kReplicated,
                                        inv_dt[t.get("dtype", "i64")], inv_role[t.get("role", "intermediate")]))
        for o in d["operators"]:
            a = o.get("attrs", {})
            g.operators.append(OpDecl(
                o["name"], OperatorKind(KIND_NAME.index(o["kind"])), list(o.get("inputs", [])),
                list(o.get("outputs", [])),
                ResourceClass(RC_NAME.index(o["resource_class"])) if o.get("resource_class") else None,
                o.get("module_path", ""), list(o.get("region_tags", [])),
                CostParams(*o["cost"]) if o.get("cost") is not None else None,
                OpAttrs(a.get("world_size", 1), a.get("seed", 0), a.get("custom_name", ""),
                        dict(a.get("params", {})))))
        return g


def _desc_json(desc: Any) -> str:
    if isinstance(desc, GraphDescription):
        return desc.to_json()
    if isinstance(desc, dict):
        return json.dumps(desc)
    return str(desc)


@dataclass
class OperatorNode:
    name: str
    kind: OperatorKind
    inputs: List[int]
    outputs: List[int]
    resource_class: ResourceClass


@dataclass
class TensorMeta:
    name: str
    shape: List[int]
    producer: int
    consumers: List[int]


class Graph:
    """Built, topologically ordered graph (handle to the C++ opflow::Graph)."""

    def __init__(self, handle: int, desc_json: str):
        self._h = C.c_void_p(handle)
        self.desc_json = desc_json
        p = C.c_void_p()
        check(lib().opf_graph_dump(self._h, C.byref(p)))
        self.dump_json = take_string(p)
        d = json.loads(self.dump_json)
        self.ops = [OperatorNode(o["name"], OperatorKind(KIND_NAME.index(o["kind"])), o["inputs"],
                                 o["outputs"], ResourceClass(RC_NAME.index(o["resource_class"])))
                    for o in d["ops"]]
        self.tensors = [TensorMeta(t["name"], t["shape"], t["producer"], t["consumers"])
                        for t in d["tensors"]]
        self.graph_inputs: List[int] = d["graph_inputs"]
        self.weights: List[int] = d["weights"]
        self.graph_outputs: List[int] = d["graph_outputs"]
        self.tensor_index = {t.name: i for i, t in enumerate(self.tensors)}
        self.op_index = {o.name: i for i, o in enumerate(self.ops)}
        self.description = json.loads(desc_json)

    def tensor_id(self, name: str) -> int:
        if name not in self.tensor_index:
            raise Error(int(Errc.UnknownTensor), f"no tensor named '{name}'")
        return self.tensor_index[name]

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and lib is not None:  # None at interpreter exit
            lib().opf_graph_free(self._h)
            self._h = C.c_void_p()


def build_graph(desc: Any) -> Graph:
    text = _desc_json(desc)
    h = C.c_void_p()
    check(lib().opf_graph_build(text.encode(), C.byref(h)))
    return Graph(h.value, text)


@dataclass
class PartitionRule:
    kind: str  # "module" | "func" | "region"
    pattern: str

    @staticmethod
    def by_module(p: str) -> "PartitionRule":
        return PartitionRule("module", p)

    @staticmethod
    def by_func(p: str) -> "PartitionRule":
        return PartitionRule("func", p)

    @staticmethod
    def by_region(p: str) -> "PartitionRule":
        return PartitionRule("region", p)


def rules_json(rules: Sequence[PartitionRule]) -> str:
    return json.dumps([{"kind": r.kind, "pattern": r.pattern} for r in rules])


@dataclass
class Subgraph:
    id: int
    ops: List[int]
    boundary_inputs: List[int]
    boundary_outputs: List[int]
    label: str
    dominant_class: ResourceClass


class PartitionPlan:
    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        p = C.c_void_p()
        check(lib().opf_plan_dump(self._h, C.byref(p)))
        self.dump_json = take_string(p)
        d = json.loads(self.dump_json)
        self.subgraphs = [Subgraph(s["id"], s["ops"], s["boundary_inputs"], s["boundary_outputs"],
                                   s["label"], ResourceClass(RC_NAME.index(s["dominant_class"])))
                          for s in d["subgraphs"]]
        self.sg_edges = [tuple(e) for e in d["sg_edges"]]
        self.rule_trace: List[str] = d["rule_trace"]
        self.op_to_subgraph: List[int] = d["op_to_subgraph"]
        n = len(self.subgraphs)
        self.sg_succ = [[b for a, b in self.sg_edges if a == i] for i in range(n)]
        self.sg_pred = [[a for a, b in self.sg_edges if b == i] for i in range(n)]

    def size(self) -> int:
        return len(self.subgraphs)

    def __len__(self) -> int:
        return len(self.subgraphs)

    def find_label(self, label: str) -> Optional[Subgraph]:
        for s in self.subgraphs:
            if s.label == label:
                return s
        return None

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and lib is not None:  # None at interpreter exit
            lib().opf_plan_free(self._h)
            self._h = C.c_void_p()


def partition(g: Graph, rules: Sequence[PartitionRule] = ()) -> PartitionPlan:
    h = C.c_void_p()
    check(lib().opf_partition(g._h, rules_json(rules).encode(), C.byref(h)))
    return PartitionPlan(h.value)


def hand_plan(g: Graph, subgraph_ops: Sequence[Sequence[int]], labels: Sequence[str] = ()) -> PartitionPlan:
    """Hand-assembled plan + finalize_plan (reference partition.hpp:69-70)."""
    sgs = [{"ops": list(map(int, ops)), "label": (labels[i] if i < len(labels) else f"hand{i}")}
           for i, ops in enumerate(subgraph_ops)]
    h = C.c_void_p()
    check(lib().opf_plan_from_json(g._h, json.dumps({"subgraphs": sgs}).encode(), C.byref(h)))
    return PartitionPlan(h.value)


def validate_plan(plan: PartitionPlan, g: Graph) -> None:
    check(lib().opf_validate_plan(plan._h, g._h))


# ------------------------------------------------------------------ builders
def builder_json(name: str, **params: Any) -> str:
    p = C.c_void_p()
    check(lib().opf_builder_json(name.encode(), json.dumps(params).encode(), C.byref(p)))
    return take_string(p)


def dense_tp_graph(layers: int, batch: int, hidden: int, dtype: str = "i64", costs=None) -> str:
    kw = dict(layers=layers, batch=batch, hidden=hidden, dtype=dtype)
    if costs:
        kw["costs"] = costs
    return builder_json("dense_tp", **kw)


def moe_ep_graph(layers: int, batch: int, hidden: int, dtype: str = "i64", costs=None) -> str:
    kw = dict(layers=layers, batch=batch, hidden=hidden, dtype=dtype)
    if costs:
        kw["costs"] = costs
    return builder_json("moe_ep", **kw)


def fuse_chain_graph(layers: int, batch: int, hidden: int, dtype: str = "i64", costs=None) -> str:
    kw = dict(layers=layers, batch=batch, hidden=hidden, dtype=dtype)
    if costs:
        kw["costs"] = costs
    return builder_json("fuse_chain", **kw)


def llama_graph(**params: Any) -> str:
    return builder_json("llama", **params)


def llama_decode_graph(**params: Any) -> str:
    return builder_json("llama_decode", **params)


def toy_decoder_graph(**params: Any) -> str:
    return builder_json("toy_decoder", **params)


def qwen3_moe_graph(**params: Any) -> str:
    """Qwen3-30B-A3B-shaped layer(s): q/k-norm attention + routed MoE FFN
    (router GEMM, top-k, dispatch, grouped expert GEMMs, combine); BASELINE configs[4]."""
    return builder_json("qwen3_moe", **params)


def alltoall_permutation(seed: int, cols: int) -> List[int]:
    buf = (C.c_uint32 * cols)()
    check(lib().opf_alltoall_permutation(C.c_uint64(seed & (2**64 - 1)), cols, buf))
    return list(buf)


# ------------------------------------------------------------------ scheduling API
@dataclass(frozen=True)
class OpHandle:
    subgraph: int
    ubatch: int
    topo_index: int


class SchedContext:
    """The strategy's view: split / get_ready_ops / execute."""

    def __init__(self, ptr: int):
        self._p = C.c_void_p(ptr)

    def split(self, sizes: Sequence[int]) -> List[int]:
        arr = (C.c_int64 * len(sizes))(*sizes)
        check(lib().opf_sched_split(self._p, arr, len(sizes)))
        return list(range(len(sizes)))

    def get_ready_ops(self, ubatch: int) -> List[OpHandle]:
        cap = 4096
        buf = (opf_handle * cap)()
        n = C.c_int32()
        check(lib().opf_sched_ready(self._p, ubatch, buf, cap, C.byref(n)))
        return [OpHandle(buf[i].subgraph, buf[i].ubatch, buf[i].topo_index) for i in range(n.value)]

    def handle(self, subgraph: int, ubatch: int) -> OpHandle:
        h = opf_handle()
        check(lib().opf_sched_handle(self._p, subgraph, ubatch, C.byref(h)))
        return OpHandle(h.subgraph, h.ubatch, h.topo_index)

    def execute(self, ops: Sequence[OpHandle] | OpHandle, lane: int = 0,
                replace_fn: Optional[str] = None) -> None:
        if isinstance(ops, OpHandle):
            ops = [ops]
        arr = (opf_handle * len(ops))(*[opf_handle(h.subgraph, h.ubatch, h.topo_index) for h in ops])
        check(lib().opf_sched_execute(self._p, arr, len(ops), lane,
                                      replace_fn.encode() if replace_fn else None))

    @property
    def rows(self) -> int:
        r = C.c_int64()
        check(lib().opf_sched_rows(self._p, C.byref(r)))
        return r.value

    def num_subgraphs(self) -> int:
        n = C.c_int32()
        check(lib().opf_sched_num_subgraphs(self._p, C.byref(n)))
        return n.value

    def label(self, subgraph: int) -> str:
        buf = C.create_string_buffer(512)
        check(lib().opf_sched_label(self._p, subgraph, buf, 512))
        return buf.value.decode()

    def unfinished(self) -> int:
        n = C.c_int32()
        check(lib().opf_sched_unfinished(self._p, C.byref(n)))
        return n.value


class Scheduler:
    """User strategy base class (the paper's OpSchedulerBase)."""

    cache_key: str = "custom"

    def schedule(self, ctx: SchedContext) -> None:  # pragma: no cover - abstract
        raise NotImplementedError


def _callback(strategy: Scheduler):
    err: List[BaseException] = []

    def fn(ctx_ptr, _user):
        try:
            strategy.schedule(SchedContext(ctx_ptr))
            return 0
        except Error as e:
            err.append(e)
            return int(e.code) + 1
        except BaseException as e:  # noqa: BLE001 - propagate after the C frame unwinds
            err.append(e)
            return int(Errc.SchedulerError) + 1

    return _lib.SCHEDULE_FN(fn), err


def dry_run(g: Graph, plan: PartitionPlan, strategy: Any = None, rows: Optional[int] = None,
            config: Optional[dict] = None, repeats: int = 1) -> tuple[dict, dict]:
    """Plan a schedule without a GPU: returns (schedule dump, stats)."""
    if rows is None:
        rows = max([g.tensors[t].shape[0] for t in g.graph_inputs] or [1])
    sched, stats = C.c_void_p(), C.c_void_p()
    cfg = json.dumps(config or {}).encode()
    if isinstance(strategy, Scheduler):
        cb, err = _callback(strategy)
        st = lib().opf_dry_run_custom(g._h, plan._h, cfg, strategy.cache_key.encode(), cb, None,
                                      rows, C.byref(sched), C.byref(stats))
        if st != 0 and err and not isinstance(err[0], Error):
            raise err[0]
        check(st)
    else:
        spec = json.dumps(strategy if strategy is not None else {"name": "sequential"})
        check(lib().opf_dry_run(g._h, plan._h, cfg, spec.encode(), rows, repeats, C.byref(sched),
                                C.byref(stats)))
    return json.loads(take_string(sched)), json.loads(take_string(stats))


# ------------------------------------------------------------------ device session
_TORCH_DT = {"i64": Dtype.kI64, "f32": Dtype.kF32, "bf16": Dtype.kBF16}


def view_of(t, batched: bool = True) -> opf_view:
    """opf_view of a contiguous torch tensor (device memory stays torch-owned)."""
    import torch
    dt = {torch.int64: Dtype.kI64, torch.float32: Dtype.kF32, torch.bfloat16: Dtype.kBF16}[t.dtype]
    assert t.is_contiguous()
    v = opf_view()
    v.base = t.data_ptr()
    v.elem_offset = 0
    v.dtype = int(dt)
    v.rank = t.dim()
    for i, s in enumerate(t.shape):
        v.shape[i] = int(s)
    v.batched = 1 if batched else 0
    return v


class Comm:
    """NCCL communicator for one rank (one process per GPU)."""

    def __init__(self, world: int, rank: int, device: int, uid: Optional[bytes] = None):
        self.world, self.rank = world, rank
        if uid is None:
            uid = Comm.unique_id()
        arr = (C.c_uint8 * 128)(*uid)
        h = C.c_void_p()
        check(lib().opf_comm_init(arr, world, rank, device, C.byref(h)))
        self._h = h

    @staticmethod
    def peer(world: int, rank: int, device: int) -> "Comm":
        """Peer-window-only communicator (no NCCL): every collective runs over
        the CUDA-IPC window at any message size.  Call enable_window() next.
        Works for ranks that cannot form an NCCL communicator, e.g. two
        processes sharing one GPU."""
        c = Comm.__new__(Comm)
        c.world, c.rank = world, rank
        h = C.c_void_p()
        check(lib().opf_comm_init_peer(world, rank, device, C.byref(h)))
        c._h = h
        return c

    @staticmethod
    def unique_id() -> bytes:
        arr = (C.c_uint8 * 128)()
        check(lib().opf_comm_unique_id(arr))
        return bytes(arr)

    def enable_window(self, stage_bytes: int) -> None:
        """Symmetric peer window (CUDA IPC) for the one-shot all-reduce and the
        fused all-reduce+RMSNorm kernels; handles travel over torch.distributed."""
        import torch.distributed as dist
        h = (C.c_uint8 * 64)()
        check(lib().opf_comm_window_alloc(self._h, stage_bytes, h))
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(h))
        flat = (C.c_uint8 * (64 * self.world))(*b"".join(allh))
        check(lib().opf_comm_window_open(self._h, flat))

    @staticmethod
    def virtual(world: int, device: int, stage_bytes: int) -> List["Comm"]:
        """`world` ranks sharing ONE device (tests of the peer-memory protocol)."""
        arr = (C.c_void_p * world)()
        check(lib().opf_comm_create_virtual(world, device, stage_bytes, arr))
        out = []
        for r in range(world):
            c = Comm.__new__(Comm)
            c.world, c.rank, c._h = world, r, C.c_void_p(arr[r])
            out.append(c)
        return out

    def window_error(self) -> int:
        e = C.c_uint32()
        check(lib().opf_comm_window_error(self._h, C.byref(e)))
        return e.value

    def set_epochs(self, value: int) -> None:
        """Test hook: seed every barrier epoch / flag of this rank's window."""
        check(lib().opf_comm_window_set_epochs(self._h, value & 0xFFFFFFFF))

    def push_calls(self) -> int:
        """Fused GEMM -> all-reduce calls that used the peer-memory push path."""
        e = C.c_uint32()
        check(lib().opf_comm_push_calls(self._h, C.byref(e)))
        return e.value

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and lib is not None:  # None at interpreter exit
            lib().opf_comm_free(self._h)
            self._h = C.c_void_p()


class Session:
    """A graph + plan bound to one GPU: CUDA-graph-replayed schedules."""

    def __init__(self, g: Graph, plan: PartitionPlan, config: Optional[dict] = None,
                 comm: Optional[Comm] = None):
        self.graph, self.plan = g, plan
        self._keep: Dict[str, Any] = {}
        h = C.c_void_p()
        check(lib().opf_session_create(g._h, plan._h, json.dumps(config or {}).encode(),
                                       comm._h if comm else None, C.byref(h)))
        self._h = h
        self._comm = comm

    def bind(self, name: str, tensor) -> None:
        tid = self.graph.tensor_id(name)
        batched = self.graph.description["tensors"][tid].get("batch", "batched") == "batched"
        v = view_of(tensor, batched)
        check(lib().opf_session_bind(self._h, name.encode(), C.byref(v)))
        self._keep[name] = tensor

    def run(self, strategy: Any = None, stream=None) -> None:
        s = stream.cuda_stream if stream is not None and hasattr(stream, "cuda_stream") else stream
        if isinstance(strategy, Scheduler):
            cb, err = _callback(strategy)
            self._keep["_cb"] = cb
            st = lib().opf_session_run_custom(self._h, strategy.cache_key.encode(), cb, None, s)
            if st != 0 and err and not isinstance(err[0], Error):
                raise err[0]
            check(st)
            return
        spec = json.dumps(strategy if strategy is not None else {"name": "sequential"})
        check(lib().opf_session_run(self._h, spec.encode(), s))

    def check(self) -> None:
        """Wait for the last run; raise SchedulerError if a peer-window barrier
        of any run so far timed out (its outputs are invalid)."""
        check(lib().opf_session_check(self._h))

    def prepare(self, strategy: Any = None, stream=None) -> None:
        """Plan + prepack + capture without launching (virtual peer ranks on one
        device prepare every rank before any rank launches)."""
        s = stream.cuda_stream if stream is not None and hasattr(stream, "cuda_stream") else stream
        spec = json.dumps(strategy if strategy is not None else {"name": "sequential"})
        check(lib().opf_session_prepare(self._h, spec.encode(), s))

    def enable_peer_arena(self, min_bytes: int = 0) -> None:
        """Symmetric arena for expert-parallel ops (one process per GPU): export
        my arena's CUDA IPC handle, all-gather over torch.distributed, map peers."""
        import torch.distributed as dist
        h = (C.c_uint8 * 64)()
        check(lib().opf_session_arena_export(self._h, min_bytes, h))
        allh = [None] * self._comm.world
        dist.all_gather_object(allh, bytes(h))
        flat = (C.c_uint8 * (64 * self._comm.world))(*b"".join(allh))
        check(lib().opf_session_arena_open(self._h, flat))

    @staticmethod
    def link_virtual(sessions: Sequence["Session"], min_bytes: int) -> None:
        """Wire the arenas of `world` virtual-rank sessions sharing one device."""
        arr = (C.c_void_p * len(sessions))(*[s_._h for s_ in sessions])
        check(lib().opf_session_arena_link_local(arr, len(sessions), min_bytes))

    def stats(self) -> dict:
        p = C.c_void_p()
        check(lib().opf_session_stats(self._h, C.byref(p)))
        return json.loads(take_string(p))

    def schedule(self) -> dict:
        p = C.c_void_p()
        check(lib().opf_session_schedule_dump(self._h, C.byref(p)))
        return json.loads(take_string(p))

    def trace(self) -> list:
        p = C.c_void_p()
        check(lib().opf_session_trace(self._h, C.byref(p)))
        return json.loads(take_string(p))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and lib is not None:  # None at interpreter exit
            lib().opf_session_free(self._h)
            self._h = C.c_void_p()


class KvCache:
    """Paged KV-cache manager (per-layer bf16 K / V page pools + a free-list page
    allocator).  append() reserves cache slots for new tokens of sequences (the
    kv_write op stores K / V there), block_table() gives attn_decode its rows.
    dry=True runs the allocator without device pools (CPU)."""

    def __init__(self, layers: int, pages: int, kv_heads: int, head_dim: int = 128, page_size: int = 16,
                 kv_layout: int = 0, device: int = 0, dry: bool = False):
        self._h = C.c_void_p()
        check(lib().opf_kv_create(layers, pages, page_size, kv_heads, head_dim, kv_layout, device, int(dry),
                                  C.byref(self._h)))
        self.layers, self.pages, self.page_size = layers, pages, page_size
        self.kv_heads, self.head_dim, self.kv_layout = kv_heads, head_dim, kv_layout

    def cache(self, layer: int, which: str):
        """The layer's K ('k') or V ('v') pool as a torch bf16 tensor (a view of
        the manager's device memory, shaped for attn_decode / kv_write)."""
        import torch
        p = C.c_void_p()
        check(lib().opf_kv_cache_ptr(self._h, layer, 0 if which == "k" else 1, C.byref(p)))
        shape = ((self.pages, self.kv_heads, self.page_size, self.head_dim) if self.kv_layout == 1
                 else (self.pages, self.page_size, self.kv_heads, self.head_dim))
        n = self.pages * self.page_size * self.kv_heads * self.head_dim
        return _device_tensor(p.value, n, torch.bfloat16).view(*shape)

    def append(self, seq_ids: Sequence[int], n_new: Sequence[int]):
        """Reserve n_new[i] tokens for seq_ids[i]; returns (slots, positions) int64 numpy arrays."""
        import numpy as np
        n = len(seq_ids)
        ids = (C.c_int64 * max(n, 1))(*seq_ids)
        cnt = (C.c_int32 * max(n, 1))(*n_new)
        total = int(sum(n_new))
        slots = (C.c_int64 * max(total, 1))()
        pos = (C.c_int64 * max(total, 1))()
        check(lib().opf_kv_append(self._h, ids, cnt, n, slots, pos))
        return np.ctypeslib.as_array(slots)[:total].copy(), np.ctypeslib.as_array(pos)[:total].copy()

    def release(self, seq_id: int) -> None:
        check(lib().opf_kv_release(self._h, seq_id))

    def block_table(self, seq_ids: Sequence[int], max_pages: int):
        """(table [n, max_pages] int64 with -1 past each sequence's pages, lens [n]) as numpy."""
        import numpy as np
        n = len(seq_ids)
        ids = (C.c_int64 * max(n, 1))(*seq_ids)
        tab = (C.c_int64 * max(n * max_pages, 1))()
        lens = (C.c_int64 * max(n, 1))()
        check(lib().opf_kv_block_table(self._h, ids, n, max_pages, tab, lens))
        return (np.ctypeslib.as_array(tab)[:n * max_pages].reshape(n, max_pages).copy(),
                np.ctypeslib.as_array(lens)[:n].copy())

    def stats(self) -> dict:
        f, q = C.c_int64(), C.c_int64()
        check(lib().opf_kv_stats(self._h, C.byref(f), C.byref(q)))
        return {"free_pages": f.value, "sequences": q.value}

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and lib is not None:
            lib().opf_kv_free(self._h)
            self._h = C.c_void_p()


def _device_tensor(ptr: int, numel: int, dtype):
    """A torch tensor aliasing device memory owned by the library (no copy)."""
    import torch

    class _Holder:
        def __init__(self, p, nbytes):
            self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (p, False),
                                             "version": 3}

    nbytes = numel * torch.tensor([], dtype=dtype).element_size()
    return torch.as_tensor(_Holder(ptr, nbytes), device="cuda").view(dtype)


# ------------------------------------------------------------------ operator registry
@dataclass
class OpCtx:
    """What a registered op sees of its launch (opf_op_ctx, include/opflow_b200.h)."""
    op_name: str
    custom_name: str
    world_size: int
    seed: int
    params: Dict[str, float]
    max_ctas: int
    workspace: int
    workspace_bytes: int


_TORCH_OF_DT = {0: "int64", 1: "float32", 2: "bfloat16"}
_REGISTERED: Dict[str, Any] = {}  # keeps the ctypes trampolines alive


def view_tensor(v: opf_view):
    """A torch tensor aliasing an opf_view's device memory (no copy)."""
    import torch
    dt = getattr(torch, _TORCH_OF_DT[v.dtype])
    shape = [int(v.shape[i]) for i in range(v.rank)]
    numel = 1
    for x in shape:
        numel *= x
    esz = torch.tensor([], dtype=dt).element_size()
    return _device_tensor(int(v.base or 0) + int(v.elem_offset) * esz, numel, dt).view(*shape)


def register_op(name: str, fn: Callable, resource_class: ResourceClass = ResourceClass.kCompute,
                n_in: int = -1, n_out: int = -1) -> None:
    """CustomRegistry::fns[name] = fn (reference eval.hpp:19-28) for device ops.

    `fn(ctx: OpCtx, ins: list[Tensor], outs: list[Tensor], rows: int, stream)`
    launches its kernels on `stream` (a torch.cuda.ExternalStream of the
    engine's lane) and writes into `outs` in place — they are caller-owned
    views, possibly nano-batch row slices of the engine's arena; it must not
    allocate device memory (the call may be under CUDA-graph capture: the
    engine calls it once per nano-batch when it captures, replays re-run the
    captured kernels).  A Custom op with attrs.custom_name == name runs it,
    and PartitionRule.by_func(name) isolates it."""
    import sys
    import traceback

    def tramp(ctx_p, in_p, n_in_, out_p, n_out_, rows, stream):
        try:
            import torch
            c = ctx_p.contents
            params = {c.param_names[i].decode(): float(c.param_values[i]) for i in range(c.n_params)}
            ctx = OpCtx((c.op_name or b"").decode(), (c.custom_name or b"").decode(), int(c.world_size),
                        int(c.seed), params, int(c.max_ctas), int(c.workspace or 0), int(c.workspace_bytes))
            ins = [view_tensor(in_p[i]) for i in range(n_in_)]
            outs = [view_tensor(out_p[i]) for i in range(n_out_)]
            st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            fn(ctx, ins, outs, int(rows), st)
            return 0
        except Error as e:
            print(f"[opflow] registered op '{name}': {e}", file=sys.stderr)
            return int(e.code) + 1
        except BaseException:  # noqa: BLE001 - reported through the status code
            traceback.print_exc()
            return int(Errc.SchedulerError) + 1

    cb = _lib.KERNEL_FN(tramp)
    check(lib().opf_register_op(name.encode(), cb, int(resource_class), n_in, n_out))
    _REGISTERED[name] = (cb, fn)


def has_op(name: str) -> bool:
    p = C.c_int32()
    check(lib().opf_has_op(name.encode(), C.byref(p)))
    return bool(p.value)


def launch(op: OpDecl | dict, inputs: Sequence, outputs: Sequence, rows: int, stream=None,
           comm: Optional[Comm] = None, max_ctas: int = 0) -> None:
    """Device eval_op_into: run one operator into caller-provided tensors."""
    opj = json.dumps(op.to_json() if isinstance(op, OpDecl) else op)
    iv = (opf_view * max(1, len(inputs)))(*[view_of(t) for t in inputs])
    ov = (opf_view * max(1, len(outputs)))(*[view_of(t) for t in outputs])
    s = stream.cuda_stream if stream is not None and hasattr(stream, "cuda_stream") else stream
    if comm is not None or max_ctas:
        check(lib().opf_launch_comm(opj.encode(), iv, len(inputs), ov, len(outputs), rows,
                                    comm._h if comm else None, max_ctas, s))
        return
    check(lib().opf_launch(opj.encode(), iv, len(inputs), ov, len(outputs), rows, s))
