"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU oracles.

* ``COracle``  : our plain-C restatement (oracle/ttb_oracle.c -> build/libttb_oracle.so)
* ``RefOracle``: the unmodified reference compiled in place (oracle/_ref/libttune_ref.so)

Only tests/, bench.py's CPU legs and __graft_entry__.smoke() import this module,
and only as the checker.  The product (paper_1603_02297_b200) never imports it.

Buffers are flat numpy arrays of SCALARS (float32 for kinds s/c, float64 for
d/z); complex kinds hold interleaved (re, im) pairs, exactly the reference's
TensorBuffer storage (executor.hpp:45-70).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libttb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libttune_ref.so")

KINDS = {"s": 0, "d": 1, "c": 2, "z": 3}
SCALAR = {0: np.float32, 1: np.float64, 2: np.float32, 3: np.float64}
COMPONENTS = {0: 1, 1: 1, 2: 2, 3: 2}
EBYTES = {0: 4, 1: 8, 2: 8, 3: 16}

_i32p = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)


def kind_id(k) -> int:
    return KINDS[k] if isinstance(k, str) else int(k)


def _ia(v: Optional[Sequence[int]]):
    if v is None:
        return None
    return (C.c_int * max(len(v), 1))(*v)


def _la(v: Optional[Sequence[int]]):
    if v is None:
        return None
    return (C.c_int64 * max(len(v), 1))(*v)


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def scalar_buffer(kind, elements: int, fill=0.0) -> np.ndarray:
    k = kind_id(kind)
    return np.full(elements * COMPONENTS[k], fill, dtype=SCALAR[k])


def b_sizes(perm: Sequence[int], sizes: Sequence[int]):
    sb = [0] * len(perm)
    for a, p in enumerate(perm):
        sb[p - 1] = sizes[a]
    return sb


class COracle:
    """Plain-C restatement of the reference hot path (see ttb_oracle.h)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        L = self.lib = C.CDLL(path)
        L.orc_validate.argtypes = [C.c_int, _i32p, C.c_int, _i64p, C.c_int, _i64p, C.c_int, _i64p,
                                   C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.orc_required_elements_a.argtypes = [C.c_int, _i64p, _i64p]
        L.orc_required_elements_a.restype = C.c_int64
        L.orc_required_elements_b.argtypes = [C.c_int, _i32p, _i64p, _i64p]
        L.orc_required_elements_b.restype = C.c_int64
        L.orc_merge.argtypes = [C.c_int, _i32p, _i64p, _i64p, _i64p, _i32p, _i64p, _i64p, _i64p,
                                _i32p, _i32p]
        L.orc_transpose.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i64p, _i64p, _i64p,
                                    C.c_double, C.c_void_p, C.c_double, C.c_void_p]
        L.orc_reference_nest.argtypes = L.orc_transpose.argtypes + [C.c_int]
        L.orc_fill_uniform.argtypes = [C.c_int, C.c_int, _i64p, _i64p, _i64p, _i64p, C.c_uint64,
                                       C.c_void_p]
        L.orc_fill_sentinel.argtypes = [C.c_int, C.c_int64, C.c_void_p]
        L.orc_checksum.argtypes = [C.c_int, C.c_int, _i64p, _i64p, _i64p, _i64p, C.c_void_p]
        L.orc_checksum.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_bandwidth_gbs.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double]
        L.orc_bandwidth_gbs.restype = C.c_double

    # problem.cpp:107-159
    def validate(self, perm, sizes, lda=None, ldb=None, kind_a="s", kind_b="s") -> Optional[str]:
        msg = C.create_string_buffer(512)
        rc = self.lib.orc_validate(len(perm), _ia(perm), len(sizes), _la(sizes),
                                   -1 if lda is None else len(lda), _la(lda),
                                   -1 if ldb is None else len(ldb), _la(ldb),
                                   kind_id(kind_a), kind_id(kind_b), msg, 512)
        return msg.value.decode() if rc else None

    def required_elements_a(self, sizes, lda=None) -> int:
        return self.lib.orc_required_elements_a(len(sizes), _la(sizes), _la(lda))

    def required_elements_b(self, perm, sizes, ldb=None) -> int:
        return self.lib.orc_required_elements_b(len(perm), _ia(perm), _la(sizes), _la(ldb))

    # problem.cpp:270-340
    def merge(self, perm, sizes, lda=None, ldb=None):
        n = len(perm)
        op, os_, ola, olb = (C.c_int * n)(), (C.c_int64 * n)(), (C.c_int64 * n)(), (C.c_int64 * n)()
        lo, hi = (C.c_int * n)(), (C.c_int * n)()
        r = self.lib.orc_merge(n, _ia(perm), _la(sizes), _la(lda), _la(ldb), op, os_, ola, olb, lo, hi)
        if r < 0:
            raise ValueError(self.validate(perm, sizes, lda, ldb))
        return (list(op[:r]), list(os_[:r]), list(ola[:r]), list(olb[:r]),
                list(zip(lo[:r], hi[:r])))

    def transpose(self, kind_a, kind_b, perm, sizes, lda, ldb, alpha, A: np.ndarray, beta,
                  B: np.ndarray) -> None:
        self.lib.orc_transpose(kind_id(kind_a), kind_id(kind_b), len(perm), _ia(perm), _la(sizes),
                               _la(lda), _la(ldb), alpha, _ptr(A), beta, _ptr(B))

    def reference_nest(self, kind_a, kind_b, perm, sizes, lda, ldb, alpha, A, beta, B,
                       threads=1) -> None:
        self.lib.orc_reference_nest(kind_id(kind_a), kind_id(kind_b), len(perm), _ia(perm),
                                    _la(sizes), _la(lda), _la(ldb), alpha, _ptr(A), beta,
                                    _ptr(B), threads)

    def fill_uniform(self, kind, sizes, ld, seed, buf: np.ndarray, origin=None,
                     global_sizes=None) -> None:
        self.lib.orc_fill_uniform(kind_id(kind), len(sizes), _la(sizes), _la(ld), _la(origin),
                                  _la(global_sizes), seed, _ptr(buf))

    def fill_sentinel(self, kind, buf: np.ndarray) -> None:
        k = kind_id(kind)
        self.lib.orc_fill_sentinel(k, buf.size // COMPONENTS[k], _ptr(buf))

    def checksum(self, kind, sizes, ld, buf: np.ndarray, origin=None, global_sizes=None) -> int:
        return self.lib.orc_checksum(kind_id(kind), len(sizes), _la(sizes), _la(ld), _la(origin),
                                     _la(global_sizes), _ptr(buf))

    def splitmix64(self, x: int) -> int:
        return self.lib.orc_splitmix64(x)

    def bandwidth_gbs(self, elements, kind_a, kind_b, beta, seconds) -> float:
        return self.lib.orc_bandwidth_gbs(elements, kind_id(kind_a), kind_id(kind_b), beta, seconds)


class RefOracle:
    """The reference itself (ttune sources compiled by oracle/Makefile)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference build missing: {path}")
        L = self.lib = C.CDLL(path)
        L.ref_validate.argtypes = [C.c_int, _i32p, C.c_int, _i64p, C.c_int, _i64p, C.c_int, _i64p,
                                   C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.ref_merge.argtypes = [C.c_int, _i32p, _i64p, _i64p, _i64p, _i32p, _i32p, _i64p, _i64p,
                                _i64p, _i32p, _i32p, C.c_char_p, C.c_size_t]
        L.ref_canonical_key.argtypes = [C.c_int, _i32p, _i64p, _i64p, _i64p, C.c_int, C.c_int,
                                        C.c_double, C.c_double, C.c_char_p, C.c_size_t]
        L.ref_bandwidth_gibs.argtypes = [C.c_int, _i32p, _i64p, C.c_int, C.c_int, C.c_double,
                                         C.c_double]
        L.ref_bandwidth_gibs.restype = C.c_double
        L.ref_run.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i64p, _i64p, _i64p, C.c_double,
                              C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64, C.c_int,
                              C.c_int, C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_session_create.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i64p, _i64p, _i64p,
                                         C.c_double, C.c_double, C.c_int, C.c_char_p, C.c_size_t]
        L.ref_session_create.restype = C.c_void_p
        L.ref_session_destroy.argtypes = [C.c_void_p]
        for f in ("ref_session_a", "ref_session_b"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_void_p
        for f in ("ref_session_a_elems", "ref_session_b_elems"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_int64
        L.ref_session_run.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.ref_session_run.restype = C.c_double
        L.ref_session_tune.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                       C.c_size_t, C.POINTER(C.c_double)]
        L.ref_benchmark_manifest.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_char_p,
                                             C.c_size_t]
        L.ref_cache_store.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_double,
                                      C.c_char_p]
        L.ref_cache_lookup.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t,
                                       C.POINTER(C.c_double), _i32p]

    def benchmark_manifest(self, volume_bytes: int, kind, seed: int):
        """build_benchmark + write_benchmark_manifest of the reference."""
        out = C.create_string_buffer(1 << 16)
        if self.lib.ref_benchmark_manifest(volume_bytes, kind_id(kind), seed, out, 1 << 16):
            raise ValueError("reference build_benchmark failed")
        return [l for l in out.value.decode().split("\n") if l]

    def cache_store(self, file, pkey, hkey, plan, gibs, ts="2026-01-01T00:00:00Z"):
        if self.lib.ref_cache_store(str(file).encode(), pkey.encode(), hkey.encode(),
                                    plan.encode(), gibs, ts.encode()):
            raise ValueError("reference SolutionCache::store failed")

    def cache_lookup(self, file, pkey, hkey):
        out = C.create_string_buffer(1024)
        gibs = C.c_double(0)
        found = C.c_int(0)
        if self.lib.ref_cache_lookup(str(file).encode(), pkey.encode(), hkey.encode(), out, 1024,
                                     C.byref(gibs), C.byref(found)):
            raise ValueError("reference SolutionCache::lookup failed")
        return (out.value.decode(), gibs.value) if found.value else None

    def validate(self, perm, sizes, lda=None, ldb=None, kind_a="s", kind_b="s") -> Optional[str]:
        msg = C.create_string_buffer(512)
        rc = self.lib.ref_validate(len(perm), _ia(perm), len(sizes), _la(sizes),
                                   -1 if lda is None else len(lda), _la(lda),
                                   -1 if ldb is None else len(ldb), _la(ldb),
                                   kind_id(kind_a), kind_id(kind_b), msg, 512)
        return msg.value.decode() if rc else None

    def merge(self, perm, sizes, lda=None, ldb=None):
        n = len(perm)
        rank = C.c_int(0)
        op, os_, ola, olb = (C.c_int * n)(), (C.c_int64 * n)(), (C.c_int64 * n)(), (C.c_int64 * n)()
        lo, hi = (C.c_int * n)(), (C.c_int * n)()
        msg = C.create_string_buffer(512)
        rc = self.lib.ref_merge(n, _ia(perm), _la(sizes), _la(lda), _la(ldb), C.byref(rank), op,
                                os_, ola, olb, lo, hi, msg, 512)
        if rc:
            raise ValueError(msg.value.decode())
        r = rank.value
        return (list(op[:r]), list(os_[:r]), list(ola[:r]), list(olb[:r]),
                list(zip(lo[:r], hi[:r])))

    def canonical_key(self, perm, sizes, lda=None, ldb=None, kind_a="s", kind_b="s", alpha=1.0,
                      beta=0.0) -> str:
        out = C.create_string_buffer(1024)
        self.lib.ref_canonical_key(len(perm), _ia(perm), _la(sizes), _la(lda), _la(ldb),
                                   kind_id(kind_a), kind_id(kind_b), alpha, beta, out, 1024)
        return out.value.decode()

    def run(self, kind_a, kind_b, perm, sizes, lda, ldb, alpha, A: np.ndarray, beta,
            B: np.ndarray, threads=1, which=0, plan=None) -> None:
        """which: 0 reference_transpose, 1 tsup::oracle_transpose, 2 execute_plan(plan)."""
        ka, kb = kind_id(kind_a), kind_id(kind_b)
        msg = C.create_string_buffer(512)
        rc = self.lib.ref_run(ka, kb, len(perm), _ia(perm), _la(sizes), _la(lda), _la(ldb),
                              alpha, _ptr(A), A.size // COMPONENTS[ka], beta, _ptr(B),
                              B.size // COMPONENTS[kb], threads, which,
                              plan.encode() if plan else None, msg, 512)
        if rc:
            raise ValueError(msg.value.decode())


class RefSession:
    """Reference-owned buffers for timing the reference's CPU path."""

    def __init__(self, ref: RefOracle, kind_a, kind_b, perm, sizes, lda=None, ldb=None,
                 alpha=1.0, beta=0.0, merge=True):
        self.ref = ref
        self.ka, self.kb = kind_id(kind_a), kind_id(kind_b)
        msg = C.create_string_buffer(512)
        self.h = ref.lib.ref_session_create(self.ka, self.kb, len(perm), _ia(perm), _la(sizes),
                                            _la(lda), _la(ldb), alpha, beta, int(merge), msg, 512)
        if not self.h:
            raise ValueError(msg.value.decode())

    def a(self) -> np.ndarray:
        n = self.ref.lib.ref_session_a_elems(self.h) * COMPONENTS[self.ka]
        p = self.ref.lib.ref_session_a(self.h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float if SCALAR[self.ka] == np.float32
                                                          else C.c_double)), shape=(n,))

    def b(self) -> np.ndarray:
        n = self.ref.lib.ref_session_b_elems(self.h) * COMPONENTS[self.kb]
        p = self.ref.lib.ref_session_b(self.h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float if SCALAR[self.kb] == np.float32
                                                          else C.c_double)), shape=(n,))

    def run(self, threads: int, plan: Optional[str] = None) -> float:
        return self.ref.lib.ref_session_run(self.h, plan.encode() if plan else None, threads)

    def tune(self, threads: int, max_impl=8, warmups=1, reps=3):
        out = C.create_string_buffer(256)
        g = C.c_double(0)
        rc = self.ref.lib.ref_session_tune(self.h, threads, max_impl, warmups, reps, out, 256,
                                           C.byref(g))
        if rc:
            raise RuntimeError("reference tune failed")
        return out.value.decode(), g.value

    def close(self):
        if self.h:
            self.ref.lib.ref_session_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def have_ref() -> bool:
    return os.path.exists(REF_SO)
