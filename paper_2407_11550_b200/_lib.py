"""ctypes binding of the C ABI (include/adakv_b200.h) -> lib/libadakv_b200.so.

There is no fallback: if the CUDA library is missing this raises at import of
any op.  Build it with ``python -c "import __graft_entry__ as g; g.build()"``
(or ``make -C paper_2407_11550_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libadakv_b200.so")

F32, F64, BF16 = 0, 1, 2
KINDS = {"snapkv": 0, "pyramid": 1, "ada_snapkv": 2, "ada_pyramid": 3, "streaming_llm": 4}
ALLOC_ADAPTIVE, ALLOC_UNIFORM, ALLOC_GIVEN = 0, 1, 2
DECODE_CHAINED = 1  # adakv_decode flag: the previous kernel on the stream is a decode of other segments

STATUS = {0: "ok", 1: "invalid_argument", 2: "out_of_range", 3: "format_error", 4: "io_error",
          5: "cuda_error", 6: "unsupported", 7: "workspace_too_small"}


class AdaKVError(RuntimeError):
    """Raised for a non-OK adakv_status; ``kind`` names the reference exception type."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS.get(status, "error")


class InvalidArgument(AdaKVError, ValueError):
    pass


class OutOfRange(AdaKVError, IndexError):
    pass


class FormatError(AdaKVError):
    """Malformed or unsupported on-disk content (serde.hpp:18-21)."""


class IoError(AdaKVError, OSError):
    """Underlying I/O failure (serde.hpp:24-27)."""


class PolicyConfig(C.Structure):
    _fields_ = [("kind", C.c_int32), ("scale", C.c_int32), ("window_size", C.c_int64),
                ("pool_kernel", C.c_int64), ("alpha", C.c_double), ("sink_tokens", C.c_int64),
                ("gqa_group_size", C.c_int64)]


class LayerShape(C.Structure):
    _fields_ = [("problems", C.c_int64), ("q_heads", C.c_int64), ("kv_groups", C.c_int64),
                ("window", C.c_int64), ("outside", C.c_int64), ("head_dim", C.c_int64)]


class SelectConfig(C.Structure):
    _fields_ = [("alloc_mode", C.c_int32), ("blend", C.c_int32), ("repair", C.c_int32),
                ("streaming", C.c_int32), ("alpha", C.c_double), ("sink_tokens", C.c_int64)]


_lib = None

VP = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
SZ = C.c_size_t
PI64 = C.POINTER(C.c_int64)
PSZ = C.POINTER(C.c_size_t)


def _sig(L):
    S = C.c_int
    L.adakv_last_error.restype = C.c_char_p
    L.adakv_abi_version.restype = C.c_int
    L.adakv_set_tensor_core_scoring.argtypes = [C.c_int]
    L.adakv_set_tensor_core_scoring.restype = C.c_int
    L.adakv_workspace_status.argtypes = [VP, VP]
    L.adakv_clear_workspace_status.argtypes = [VP, VP]
    L.adakv_validate_finite.argtypes = [S, VP, I64, VP, VP]
    L.adakv_host_device_pointer.argtypes = [VP, C.POINTER(VP)]
    L.adakv_set_decode_overlap.argtypes = [C.c_int]
    L.adakv_set_decode_overlap.restype = C.c_int
    L.adakv_compress.argtypes = [S, C.POINTER(LayerShape), C.POINTER(PolicyConfig), I64, VP, VP, VP, VP, I64,
                                 VP, VP, VP, VP, VP, VP, VP, VP, VP, SZ, VP]
    L.adakv_compress_split.argtypes = L.adakv_compress.argtypes + [VP]
    L.adakv_shard_pack_candidates.argtypes = [VP, VP, VP, I64, I64, I64, VP, VP]
    L.adakv_shard_build_union.argtypes = [VP, I64, I64, I64, I64, VP, VP]
    L.adakv_compress_workspace.argtypes = [S, C.POINTER(LayerShape), C.POINTER(PolicyConfig), PSZ]
    L.adakv_cache_rows.argtypes = [C.POINTER(LayerShape), I64, VP, I64]
    L.adakv_cache_rows.restype = I64
    L.adakv_window_scores.argtypes = [S, C.POINTER(LayerShape), I64, I32, VP, VP, VP, VP, VP, SZ, VP]
    L.adakv_window_scores_workspace.argtypes = [S, C.POINTER(LayerShape), PSZ]
    L.adakv_segmented_select.argtypes = [S, I64, I64, PI64, VP, I64, VP, C.POINTER(SelectConfig), VP, VP, VP,
                                         VP, I64, VP, SZ, VP]
    L.adakv_segmented_select_workspace.argtypes = [I64, I64, PSZ]
    L.adakv_gather.argtypes = [S, C.POINTER(LayerShape), I64, VP, VP, VP, VP, VP, I64, I64, VP, VP, VP, VP, VP, VP,
                               VP]
    L.adakv_decode.argtypes = [S, I64, I64, I64, I64, I32, VP, VP, VP, I64, VP, VP, VP, I64, VP, VP, VP, VP, SZ,
                               C.c_uint32, VP]
    L.adakv_decode_workspace.argtypes = [I64, I64, I64, I64, I64, PSZ]
    L.adakv_append_kv.argtypes = [S, I64, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP]
    L.adakv_append_rows.argtypes = [S, I64, I64, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP]
    L.adakv_apportion.argtypes = [VP, I64, I64, VP, VP]
    L.adakv_uniform_allocation.argtypes = [I64, I64, VP, VP]
    L.adakv_safeguard_blend.argtypes = [VP, I64, I64, I64, C.c_double, VP, VP]
    L.adakv_repair_zero_budgets.argtypes = [VP, VP, I64]
    L.adakv_pyramid_layer_budgets.argtypes = [I64, I64, C.c_double, C.c_double, VP]
    return L


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA library must be built (no CPU fallback exists). "
                "Run `make -C paper_2407_11550_b200/csrc -j` or __graft_entry__.build().")
        _lib = _sig(C.CDLL(LIB_PATH))
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().adakv_last_error().decode()
        if status == 1:
            raise InvalidArgument(status, msg)
        if status == 2:
            raise OutOfRange(status, msg)
        if status == 3:
            raise FormatError(status, msg)
        if status == 4:
            raise IoError(status, msg)
        raise AdaKVError(status, msg)
