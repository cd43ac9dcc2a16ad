"""ctypes binding of libpatb200.so (the C ABI in include/pat_b200.h).

The shared library is built in-tree by ``paper_2506_20252_b200/csrc/Makefile``
(``python -c "import __graft_entry__ as g; g.build()"``). There is no fallback: if the
library is missing every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PAT_LIB_VARIANT=x loads libpatb200_x.so (an in-tree A/B build of the same sources, tools/)
LIB_PATH = os.path.join(HERE, "libpatb200" + (f"_{os.environ['PAT_LIB_VARIANT']}" if os.environ.get("PAT_LIB_VARIANT") else "") + ".so")
HANDLE_BYTES = 128
MAX_RANKS = 8

# patResult_t -> name; the reference's exception class names for the typed ones
RESULTS = {
    0: "Success", 1: "UnhandledCudaError", 2: "SystemError", 3: "InternalError",
    4: "InvalidArgument", 5: "InvalidUsage", 6: "RemoteError",
    20: "ScheduleError", 21: "NonPowerOfTwoError", 22: "InvalidTreeCountError",
    23: "BufferTooSmallError", 24: "RankOutOfRangeError", 30: "SimulationError",
    31: "PayloadShapeError", 32: "UnsupportedOpError", 33: "InvalidScheduleError",
    40: "Timeout", 41: "Capacity",
}

# datatypes (ncclDataType_t numbering) and ops (ncclRedOp_t numbering)
INT8, UINT8, INT32, UINT32, INT64, UINT64, FLOAT16, FLOAT32, FLOAT64, BFLOAT16 = range(10)
SUM, PROD, MAX, MIN = range(4)
PROTO_AUTO, PROTO_LL, PROTO_SIMPLE, PROTO_PULL, PROTO_LL32, PROTO_FUSED = 0, 1, 2, 3, 5, 6
PROTO_NAMES = {PROTO_LL: "LL", PROTO_SIMPLE: "SIMPLE", PROTO_PULL: "PULL", PROTO_LL32: "LL32", PROTO_FUSED: "FUSED"}
DTYPE_SIZE = {INT8: 1, UINT8: 1, INT32: 4, UINT32: 4, INT64: 8, UINT64: 8, FLOAT16: 2,
              FLOAT32: 4, FLOAT64: 8, BFLOAT16: 2}


class PatError(RuntimeError):
    """A non-success patResult_t. ``kind`` names the reference exception it stands for."""

    def __init__(self, code: int, where: str = ""):
        self.code = code
        self.kind = RESULTS.get(code, f"error{code}")
        msg = lib().patGetErrorString(code).decode() if _lib is not None else self.kind
        super().__init__(f"{where}: {self.kind} ({msg})" if where else f"{self.kind} ({msg})")


class Config(ctypes.Structure):
    _fields_ = [
        ("size", ctypes.c_size_t),
        ("staging_bytes", ctypes.c_size_t),
        ("slice_bytes", ctypes.c_size_t),
        ("ll_threshold", ctypes.c_size_t),
        ("trees", ctypes.c_int),
        ("max_channels", ctypes.c_int),
        ("protocol", ctypes.c_int),
        ("timeout_ms", ctypes.c_int),
        ("threads", ctypes.c_int),
        ("depth", ctypes.c_int),
        ("direct", ctypes.c_int),
        ("send_warps", ctypes.c_int),
        ("fused", ctypes.c_int),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("protocol", ctypes.c_int),
        ("trees", ctypes.c_int),
        ("rounds", ctypes.c_int),
        ("channels", ctypes.c_int),
        ("iterations", ctypes.c_int),
        ("threads", ctypes.c_int),
        ("launches", ctypes.c_int),
        ("slots_per_step", ctypes.c_int),
        ("slice_bytes", ctypes.c_size_t),
        ("pool_bytes", ctypes.c_size_t),
        ("bytes_sent_per_rank", ctypes.c_int64),
        ("peak_intermediate_slots", ctypes.c_int),
        ("predicted_us", ctypes.c_double),
        ("staged_slots_per_step", ctypes.c_int),
        ("depth", ctypes.c_int),
        ("staging_bytes_used", ctypes.c_size_t),
    ]

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["protocol_name"] = PROTO_NAMES.get(self.protocol, str(self.protocol))
        return d


class MemInfo(ctypes.Structure):
    _fields_ = [
        ("pool_bytes_per_rank", ctypes.c_size_t),
        ("allocated_bytes", ctypes.c_size_t),
        ("pools_allocated", ctypes.c_int),
        ("depth", ctypes.c_int),
        ("depth_poll", ctypes.c_int),
        ("region_channels", ctypes.c_int * 4),
        ("region_bytes", ctypes.c_size_t * 4),
        ("slot_bytes", ctypes.c_size_t * 4),
    ]

    def as_dict(self) -> dict:
        names = ("simple_pull", "ll", "ll32")
        return {"pool_bytes_per_rank": self.pool_bytes_per_rank, "allocated_bytes": self.allocated_bytes,
                "pools_allocated": bool(self.pools_allocated), "depth": self.depth, "depth_poll": self.depth_poll,
                "regions": {names[i]: {"channels": self.region_channels[i], "bytes": self.region_bytes[i],
                                       "slot_bytes": self.slot_bytes[i]} for i in range(3)}}


class ExecStats(ctypes.Structure):
    _fields_ = [
        ("rounds", ctypes.c_int32),
        ("max_chunks_per_message", ctypes.c_int32),
        ("messages", ctypes.c_int64),
        ("bytes_sent_per_rank", ctypes.c_int64),
        ("peak_intermediate_slots", ctypes.c_int32),
        ("n_occupancy", ctypes.c_int32),
        ("occupancy_per_round", ctypes.c_int32 * 512),
    ]


# every symbol include/pat_b200.h declares (tests check the library exports all of them)
SYMBOLS = [
    "patGetErrorString", "patGetVersion", "patConfigInit", "patCommInitAll",
    "patCommInitRankPrepare", "patCommInitRankFinish", "patCommDestroy", "patCommCount",
    "patCommLocalRanks", "patCommGetAsyncError", "patCommPlan", "patAllGather",
    "patReduceScatter", "patAllGatherSchedule", "patReduceScatterSchedule", "patScheduleBuild",
    "patScheduleMirror", "patScheduleValidate", "patScheduleStats", "patScheduleTraceCsv",
    "patMaxTrees", "patTreesFromBuffer", "patPatBufferSlots", "patRoundCountFormula", "patCommTraceRead",
    "patCommMemInfo", "patCommRegisterPrepare", "patCommRegisterFinish", "patCommDeregister", "patCommBarrier", "patCommStatsRead", "patGroupStart", "patGroupEnd",
]

_lib = None
VP = ctypes.c_void_p
PP = ctypes.POINTER(ctypes.c_void_p)
I32P = ctypes.POINTER(ctypes.c_int32)
IP = ctypes.POINTER(ctypes.c_int)
SZP = ctypes.POINTER(ctypes.c_size_t)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.patGetErrorString.restype = ctypes.c_char_p
        L.patGetErrorString.argtypes = [ctypes.c_int]
        L.patGetVersion.argtypes = [IP]
        L.patConfigInit.argtypes = [ctypes.POINTER(Config)]
        L.patCommInitAll.argtypes = [PP, ctypes.c_int, IP, ctypes.POINTER(Config)]
        L.patCommInitRankPrepare.argtypes = [PP, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Config), VP]
        L.patCommInitRankFinish.argtypes = [VP, VP]
        L.patCommDestroy.argtypes = [VP]
        L.patCommCount.argtypes = [VP, IP]
        L.patCommLocalRanks.argtypes = [VP, IP, IP, IP]
        L.patCommGetAsyncError.argtypes = [VP, IP]
        L.patCommPlan.argtypes = [VP, ctypes.c_int, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(PlanInfo)]
        L.patAllGather.argtypes = [VP, PP, PP, ctypes.c_size_t, ctypes.c_int, PP]
        L.patReduceScatter.argtypes = [VP, PP, PP, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, PP]
        L.patAllGatherSchedule.argtypes = [VP, I32P, ctypes.c_size_t, PP, PP, ctypes.c_size_t, ctypes.c_int, PP]
        L.patReduceScatterSchedule.argtypes = [VP, I32P, ctypes.c_size_t, PP, PP, ctypes.c_size_t, ctypes.c_int,
                                               ctypes.c_int, PP]
        L.patScheduleBuild.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, I32P,
                                       ctypes.c_size_t, SZP]
        L.patScheduleMirror.argtypes = [I32P, ctypes.c_size_t, I32P, ctypes.c_size_t, SZP]
        L.patScheduleValidate.argtypes = [I32P, ctypes.c_size_t, IP, ctypes.c_char_p, ctypes.c_size_t]
        L.patScheduleStats.argtypes = [I32P, ctypes.c_size_t, ctypes.c_int64, ctypes.POINTER(ExecStats)]
        L.patScheduleTraceCsv.argtypes = [I32P, ctypes.c_size_t, ctypes.c_int64, ctypes.c_char_p,
                                          ctypes.c_size_t, SZP]
        L.patMaxTrees.argtypes = [ctypes.c_int, IP]
        L.patTreesFromBuffer.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, IP]
        L.patPatBufferSlots.argtypes = [ctypes.c_int, ctypes.c_int, IP]
        L.patRoundCountFormula.argtypes = [ctypes.c_int, ctypes.c_int, IP]
        L.patCommTraceRead.argtypes = [VP, ctypes.c_int, VP, ctypes.c_size_t, SZP, IP, IP]
        L.patCommMemInfo.argtypes = [VP, ctypes.POINTER(MemInfo)]
        L.patCommRegisterPrepare.argtypes = [VP, VP, ctypes.c_size_t, VP]
        L.patCommRegisterFinish.argtypes = [VP, VP, VP]
        L.patCommDeregister.argtypes = [VP, VP]
        L.patCommBarrier.argtypes = [VP, PP]
        L.patCommStatsRead.argtypes = [VP, I32P, IP, IP]
        L.patGroupStart.argtypes = []
        L.patGroupEnd.argtypes = []
        _lib = L
    return _lib


_fast = None


def fast():
    """The CPython fast-call module (csrc/pyfast.c, built in-tree next to libpatb200.so), bound
    to this library's patAllGather / patReduceScatter. None if it was not built."""
    global _fast
    if _fast is None:
        L = lib()
        try:
            from . import _patfast as F
        except ImportError:
            _fast = False
            return None
        F.bind(ctypes.cast(L.patAllGather, ctypes.c_void_p).value,
               ctypes.cast(L.patReduceScatter, ctypes.c_void_p).value)
        _fast = F
    return _fast or None


def check(rc: int, where: str = "") -> None:
    if rc != 0:
        raise PatError(rc, where)


def ptr_array(values) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = int(v) if v is not None else None
    return arr
