"""B200-native PAT (Parallel Aggregated Trees) all-gather / reduce-scatter.

The product is ``libpatb200.so`` (sm_100a kernels + C++ host runtime behind the C ABI in
``include/pat_b200.h``). This package is its thin Python face:

* ``schedule``  — the reference's schedule/algorithms API (pat_allgather, mirror_schedule,
                  validate, trees_from_buffer, ...), computed by the C++ host code;
* ``comm``      — communicators (one process for all GPUs, or one process per rank) and the
                  NCCL-shaped collectives;
* ``simulate``  — the reference executor's API (run_allgather / run_reduce_scatter over a
                  Payload) running on the GPU.
"""
from . import _lib
from ._lib import BFLOAT16, FLOAT16, FLOAT32, FLOAT64, INT8, INT32, INT64, MAX, MIN, PROD, SUM, UINT8, UINT32, UINT64
from ._lib import PROTO_AUTO, PROTO_LL, PROTO_LL32, PROTO_PULL, PROTO_SIMPLE, PatError
from .comm import PatComm, group

__all__ = ["PatComm", "PatError", "group", "schedule", "simulate", "comm", "SUM", "PROD", "MAX", "MIN",
           "INT8", "UINT8", "INT32", "UINT32", "INT64", "UINT64", "FLOAT16", "FLOAT32", "FLOAT64", "BFLOAT16",
           "PROTO_AUTO", "PROTO_LL", "PROTO_LL32", "PROTO_SIMPLE", "PROTO_PULL", "library_path"]


def library_path() -> str:
    return _lib.LIB_PATH
