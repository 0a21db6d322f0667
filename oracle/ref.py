"""TEST INFRASTRUCTURE ONLY — ctypes driver for oracle/_ref/libopflow_ref.so.

The library is the reference's own C++ (/root/reference/proj/src, unmodified)
compiled by oracle/Makefile plus oracle/ref_shim.cpp.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference legs may use
it, and only as the checker or the timed reference arm — never as the product.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libopflow_ref.so"
_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # Errc ordinal


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise FileNotFoundError(f"{LIB} not built (run `make -C oracle`)")
        _lib = C.CDLL(str(LIB))
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_free.argtypes = [C.c_void_p]
        _lib.ref_graph_plan.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_void_p)]
        _lib.ref_validate_hand_plan.argtypes = [C.c_char_p, C.POINTER(C.c_int32),
                                                C.POINTER(C.c_int32), C.c_int32,
                                                C.POINTER(C.c_void_p)]
        _lib.ref_builder.argtypes = [C.c_char_p, C.c_int, C.c_int64, C.c_int64, C.c_int,
                                     C.POINTER(C.c_void_p), C.c_char_p, C.POINTER(C.c_void_p)]
        _lib.ref_alltoall_permutation.argtypes = [C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32)]
        _lib.ref_eval.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.POINTER(C.c_char_p),
                                  C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_double)]
        _lib.ref_backend.restype = C.c_char_p
    return _lib


def _take(p: C.c_void_p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().ref_free(p)
    return s


def _check(st: int) -> None:
    if st != 0:
        raise RefError(st - 1, lib().ref_last_error().decode())


def graph_and_plan(desc_json: str, rules: Optional[Sequence[dict]] = None) -> Tuple[str, Optional[str]]:
    """Reference build_graph (+ partition + validate_plan when rules is not None)."""
    g, p = C.c_void_p(), C.c_void_p()
    rj = json.dumps(list(rules)).encode() if rules is not None else None
    _check(lib().ref_graph_plan(desc_json.encode(), rj, C.byref(g), C.byref(p) if rules is not None else None))
    return _take(g), (_take(p) if rules is not None else None)


def hand_plan(desc_json: str, subgraph_ops: Sequence[Sequence[int]]) -> str:
    flat = [int(o) for ops in subgraph_ops for o in ops]
    ops = (C.c_int32 * max(1, len(flat)))(*flat)
    counts = (C.c_int32 * max(1, len(subgraph_ops)))(*[len(o) for o in subgraph_ops])
    p = C.c_void_p()
    st = lib().ref_validate_hand_plan(desc_json.encode(), ops, counts, len(subgraph_ops), C.byref(p))
    out = _take(p) if p.value else ""
    _check(st)
    return out


def alltoall_permutation(seed: int, cols: int) -> List[int]:
    buf = (C.c_uint32 * cols)()
    lib().ref_alltoall_permutation(C.c_uint64(seed & (2**64 - 1)), cols, buf)
    return list(buf)


def backend() -> str:
    return lib().ref_backend().decode()


def evaluate(desc_json: str, rows: int, bindings: Dict[str, np.ndarray],
             timed: bool = False):
    """Reference eval_reference on host arrays (bf16 graphs evaluate in fp32).

    Returns {output_name: array} (and seconds spent inside eval_reference when
    timed=True)."""
    d = json.loads(desc_json)
    names, keep = [], []
    for t in d["tensors"]:
        if t["role"] in ("input", "weight"):
            a = bindings[t["name"]]
            dt = np.int64 if t.get("dtype") == "i64" else np.float32
            a = np.ascontiguousarray(a, dtype=dt)
            names.append(t["name"])
            keep.append(a)
    outs, out_names = [], []
    for t in d["tensors"]:
        if t["role"] == "output":
            shape = list(t["shape"])
            if t.get("batch", "batched") == "batched":
                shape[0] = rows
            outs.append(np.zeros(shape, dtype=np.int64 if t.get("dtype") == "i64" else np.float32))
            out_names.append(t["name"])
    cnames = (C.c_char_p * len(names))(*[n.encode() for n in names])
    cdata = (C.c_void_p * len(keep))(*[a.ctypes.data for a in keep])
    codata = (C.c_void_p * len(outs))(*[a.ctypes.data for a in outs])
    secs = C.c_double(0.0)
    _check(lib().ref_eval(desc_json.encode(), rows, len(names), cnames, cdata, len(outs), codata,
                          C.byref(secs)))
    res = dict(zip(out_names, outs))
    return (res, secs.value) if timed else res
