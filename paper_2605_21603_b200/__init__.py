"""B200-native DynaFlow execution backend (arXiv 2605.21603), sm_100a.

C++ host runtime + hand-written CUDA kernels in libopflow_b200.so behind the
C-ABI of include/opflow_b200.h; `opflow` is the Python mirror of the
reference's opflow API used by tests, bench and users.
"""
from . import opflow  # noqa: F401
from .opflow import (  # noqa: F401
    Error, Errc, GraphDescription, OpDecl, TensorDecl, PartitionRule, Scheduler, SchedContext,
    Session, build_graph, partition, validate_plan,
)
