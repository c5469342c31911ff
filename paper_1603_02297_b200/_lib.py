"""ctypes binding of libttb.so (include/ttb.h).

The product path is native: every call here goes straight into the CUDA
engine.  There is no Python or CPU fallback -- if the library is missing the
import of this module fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("TTB_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libttb.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libttb.so not built ({LIB_PATH}); run `python -m paper_1603_02297_b200._build` "
        "(or __graft_entry__.build()) -- there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

i32p = C.POINTER(C.c_int)
i64p = C.POINTER(C.c_int64)
vp = C.c_void_p

_SIGS = {
    "ttb_last_error": ([], C.c_char_p),
    "ttb_version": ([], C.c_char_p),
    "ttb_validate": ([C.c_int, i32p, C.c_int, i64p, C.c_int, i64p, C.c_int, i64p, C.c_int, C.c_int],
                     C.c_int),
    "ttb_required_elements_a": ([C.c_int, i64p, i64p], C.c_int64),
    "ttb_required_elements_b": ([C.c_int, i32p, i64p, i64p], C.c_int64),
    "ttb_merge_indices": ([C.c_int, i32p, i64p, i64p, i64p, i32p, i32p, i64p, i64p, i64p, i32p,
                           i32p], C.c_int),
    "ttb_canonical_key": ([C.c_int, C.c_int, C.c_int, i32p, i64p, i64p, i64p, C.c_double,
                           C.c_double, C.c_char_p, C.c_size_t], C.c_int),
    "ttb_bandwidth_gbs": ([C.c_int, C.c_int, C.c_int64, C.c_double, C.c_double], C.c_double),
    "ttb_transpose": ([C.c_int, C.c_int, C.c_int, i32p, i64p, i64p, i64p, C.c_double, vp,
                       C.c_int64, C.c_double, vp, C.c_int64, vp], C.c_int),
    "ttb_plan_create": ([C.POINTER(vp), C.c_int, C.c_int, C.c_int, i32p, i64p, i64p, i64p,
                         C.c_double, C.c_double, C.c_int], C.c_int),
    "ttb_plan_destroy": ([vp], C.c_int),
    "ttb_plan_execute": ([vp, vp, vp, vp], C.c_int),
    "ttb_plan_execute_host": ([vp, vp, vp], C.c_int),
    "ttb_plan_execute_host_async": ([vp, vp, vp], C.c_int),
    "ttb_plan_host_sync": ([vp], C.c_int),
    "ttb_plan_autotune": ([vp, vp, vp, C.c_int, C.c_int, vp], C.c_int),
    "ttb_plan_describe": ([vp, C.c_char_p, C.c_size_t], C.c_int),
    "ttb_plan_candidates": ([vp, C.c_char_p, C.c_size_t], C.c_int),
    "ttb_plan_select": ([vp, C.c_char_p], C.c_int),
    "ttb_plan_launches": ([vp, i32p], C.c_int),
    "ttb_emit_source": ([C.c_int, C.c_int, C.c_int, i32p, i64p, i64p, i64p, C.c_double, C.c_double,
                         C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t,
                         C.c_char_p, C.c_size_t], C.c_int),
    "ttb_shard_boxes": ([C.c_int, i32p, i64p, C.c_int, C.c_int, i64p, i64p, i32p], C.c_int),
    "ttb_fill_uniform": ([C.c_int, C.c_int, i64p, i64p, i64p, i64p, C.c_uint64, vp, vp], C.c_int),
    "ttb_fill_sentinel": ([C.c_int, C.c_int64, vp, vp], C.c_int),
    "ttb_checksum": ([C.c_int, C.c_int, i64p, i64p, i64p, i64p, vp, C.POINTER(C.c_uint64), vp],
                     C.c_int),
    "ttb_launch_count": ([], C.c_uint64),
    "ttb_cache_store": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_double], C.c_int),
    "ttb_cache_lookup": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t,
                          C.POINTER(C.c_double), C.c_char_p, C.c_size_t, i32p], C.c_int),
    "ttb_hardware_key": ([C.c_char_p, C.c_size_t], C.c_int),
    "ttb_plan_tune_cached": ([vp, C.c_char_p, vp, vp, C.c_int, C.c_int, vp, i32p], C.c_int),
    "ttb_benchmark_manifest": ([C.c_int64, C.c_int, C.c_uint64, C.c_char_p, C.c_size_t], C.c_int),
    "ttb_debug_candidates": ([C.c_int, C.c_int, C.c_int, i32p, i64p, i64p, i64p, C.c_double,
                              C.c_double, C.c_char_p, C.c_size_t], C.c_int),
}

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)  # AttributeError here = header/library mismatch
    _f.argtypes = _args
    _f.restype = _res

EXPORTS = tuple(_SIGS)

TTB_OK, TTB_EINVAL, TTB_ECUDA, TTB_ENOMEM, TTB_EINTERNAL = 0, 1, 2, 3, 4


class TTBError(RuntimeError):
    """Non-argument failure of the engine (CUDA error, allocation, internal)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def last_error() -> str:
    return lib.ttb_last_error().decode()


def check(rc: int) -> None:
    """Map a status code to the reference's exception kinds: std::invalid_argument
    becomes ValueError (same message text), everything else TTBError."""
    if rc == TTB_OK:
        return
    msg = last_error()
    if rc == TTB_EINVAL:
        raise ValueError(msg)
    if rc == TTB_ENOMEM:
        raise MemoryError(msg)
    raise TTBError(rc, msg)


def ints(v):
    return None if v is None else (C.c_int * max(len(v), 1))(*[int(x) for x in v])


def longs(v):
    return None if v is None else (C.c_int64 * max(len(v), 1))(*[int(x) for x in v])
