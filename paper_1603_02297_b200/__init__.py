"""B200-native tensor transposition engine (arXiv:1603.02297, Eq. 1).

    B_perm(i1..iN) <- alpha * A(i1..iN) + beta * B_perm(i1..iN)

Python mirror of the reference's interface (ttune, /root/reference/proj):
``make_problem``/``validate``/``merge_indices``/``canonical_key`` of
problem.hpp, ``TensorBuffer``/``make_buffer_a``/``make_buffer_b``/
``reference_transpose``/``execute_plan`` of executor.hpp and ``bandwidth`` of
tuner.hpp -- same names, argument meaning and error behaviour
(``std::invalid_argument`` -> ``ValueError`` with the same text).  Every call
goes through the C ABI of libttb.so (include/ttb.h); buffers live in device
memory (torch CUDA tensors are used only as HBM allocations) and the work is
done by the sm_100a kernels.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from . import _lib
from ._lib import TTBError, check, ints, last_error, lib, longs

__all__ = [
    "ElementKind", "Permutation", "TransposeProblem", "NormalizedProblem", "MergeRecord",
    "make_problem", "validate", "sizes_b", "element_strides_a", "element_strides_b",
    "element_strides_b_for_a", "b_stride1_axis", "required_elements_a", "required_elements_b",
    "canonical_key", "merge_indices", "TensorBuffer", "make_buffer_a", "make_buffer_b",
    "reference_transpose", "execute_plan", "GpuPlan", "bandwidth_gbs", "shard_boxes",
    "fill_uniform", "fill_sentinel", "checksum", "launch_count", "TTBError", "version",
    "SolutionEntry", "SolutionCache", "hardware_key", "BenchmarkCase", "build_benchmark",
    "benchmark_case_line", "EmittedKernel", "emit_source", "write_kernel_files",
]


class ElementKind(enum.IntEnum):
    """problem.hpp:11 -- codes s/d/c/z."""
    real32 = 0
    real64 = 1
    complex64 = 2
    complex128 = 3

    @property
    def code(self) -> str:
        return "sdcz"[self]

    @property
    def bytes(self) -> int:
        return (4, 8, 8, 16)[self]

    @property
    def components(self) -> int:
        return 2 if self >= 2 else 1

    @classmethod
    def from_code(cls, c: str) -> "ElementKind":
        return cls("sdcz".index(c))


def _kind(k) -> ElementKind:
    if isinstance(k, str):
        return ElementKind.from_code(k)
    return ElementKind(int(k))


@dataclass
class Permutation:
    """1-based scatter map: map[a] is B's position of A index a+1 (problem.hpp:22-35)."""
    map: List[int]

    def rank(self) -> int:
        return len(self.map)

    def is_valid(self) -> bool:
        n = len(self.map)
        return n > 0 and sorted(self.map) == list(range(1, n + 1))

    def is_identity(self) -> bool:
        return self.rank() > 0 and all(v == a + 1 for a, v in enumerate(self.map))

    def preserves_stride1(self) -> bool:
        return bool(self.map) and self.map[0] == 1

    def inverse(self) -> "Permutation":
        inv = [0] * len(self.map)
        for a, v in enumerate(self.map):
            inv[v - 1] = a + 1
        return Permutation(inv)

    @classmethod
    def from_gather(cls, gather: Sequence[int]) -> "Permutation":
        """Paper/BASELINE tuple (B index k is A index gather[k], 0-based)."""
        m = [0] * len(gather)
        for k, a in enumerate(gather):
            m[a] = k + 1
        return cls(m)


@dataclass
class TransposeProblem:
    """problem.hpp:37-49."""
    perm: Permutation
    sizes: List[int]
    lda: List[int]
    ldb: List[int]
    alpha: float = 1.0
    beta: float = 0.0
    kind_a: ElementKind = ElementKind.real32
    kind_b: ElementKind = ElementKind.real32

    def rank(self) -> int:
        return self.perm.rank()

    def total_elements(self) -> int:
        n = 1
        for s in self.sizes:
            n *= s
        return n

    def _args(self):
        n = self.rank()
        return (int(self.kind_a), int(self.kind_b), n, ints(self.perm.map), longs(self.sizes),
                longs(self.lda), longs(self.ldb))


def make_problem(perm_map: Sequence[int], sizes: Sequence[int], kind_a=ElementKind.real32,
                 kind_b=ElementKind.real32, alpha: float = 1.0, beta: float = 0.0,
                 lda: Optional[Sequence[int]] = None,
                 ldb: Optional[Sequence[int]] = None) -> TransposeProblem:
    """problem.hpp:51-58: lda defaults to sizes, ldb to sizes_b (dense)."""
    p = TransposeProblem(Permutation(list(perm_map)), list(sizes), [], [], float(alpha),
                         float(beta), _kind(kind_a), _kind(kind_b))
    p.lda = list(lda) if lda else list(p.sizes)
    if ldb:
        p.ldb = list(ldb)
    elif p.perm.is_valid() and len(p.sizes) == p.rank():
        p.ldb = sizes_b(p)
    return p


def validate(p: TransposeProblem) -> TransposeProblem:
    """problem.cpp:107-159, checked natively; raises ValueError with the reference's text."""
    check(lib.ttb_validate(len(p.perm.map), ints(p.perm.map), len(p.sizes), longs(p.sizes),
                           len(p.lda), longs(p.lda), len(p.ldb), longs(p.ldb), int(p.kind_a),
                           int(p.kind_b)))
    return p


def sizes_b(p: TransposeProblem) -> List[int]:
    sb = [0] * p.rank()
    for a, k in enumerate(p.perm.map):
        sb[k - 1] = p.sizes[a]
    return sb


def _prefix(ld):
    out, acc = [], 1
    for v in ld:
        out.append(acc)
        acc *= v
    return out


def element_strides_a(p: TransposeProblem) -> List[int]:
    return _prefix(p.lda)


def element_strides_b(p: TransposeProblem) -> List[int]:
    return _prefix(p.ldb)


def element_strides_b_for_a(p: TransposeProblem) -> List[int]:
    sb = element_strides_b(p)
    return [sb[k - 1] for k in p.perm.map]


def b_stride1_axis(p: TransposeProblem) -> int:
    return p.perm.map.index(1) if 1 in p.perm.map else -1


def required_elements_a(p: TransposeProblem) -> int:
    return lib.ttb_required_elements_a(p.rank(), longs(p.sizes), longs(p.lda))


def required_elements_b(p: TransposeProblem) -> int:
    return lib.ttb_required_elements_b(p.rank(), ints(p.perm.map), longs(p.sizes), longs(p.ldb))


def canonical_key(p: TransposeProblem) -> str:
    buf = C.create_string_buffer(4096)
    check(lib.ttb_canonical_key(*p._args(), p.alpha, p.beta, buf, 4096))
    return buf.value.decode()


@dataclass
class MergeRecord:
    from_first: int
    from_last: int
    to: int


@dataclass
class NormalizedProblem:
    problem: TransposeProblem
    merge_trace: List[MergeRecord] = field(default_factory=list)


def merge_indices(p: TransposeProblem) -> NormalizedProblem:
    """problem.cpp:270-340 (native)."""
    validate(p)
    n = p.rank()
    r = C.c_int(0)
    op, os_ = (C.c_int * n)(), (C.c_int64 * n)()
    ola, olb = (C.c_int64 * n)(), (C.c_int64 * n)()
    lo, hi = (C.c_int * n)(), (C.c_int * n)()
    check(lib.ttb_merge_indices(n, ints(p.perm.map), longs(p.sizes), longs(p.lda), longs(p.ldb),
                                C.byref(r), op, os_, ola, olb, lo, hi))
    k = r.value
    q = TransposeProblem(Permutation(list(op[:k])), list(os_[:k]), list(ola[:k]), list(olb[:k]),
                         p.alpha, p.beta, p.kind_a, p.kind_b)
    return NormalizedProblem(q, [MergeRecord(lo[i], hi[i], i + 1) for i in range(k)])


def bandwidth_gbs(p: TransposeProblem, seconds: float) -> float:
    """tuner.cpp:18-25 byte count, decimal GB/s."""
    v = lib.ttb_bandwidth_gbs(int(p.kind_a), int(p.kind_b), p.total_elements(), p.beta, seconds)
    if v < 0:
        raise ValueError("bandwidth: time must be positive")
    return v


def debug_candidates(p: TransposeProblem) -> List[str]:
    """The planner's ranked candidates for p (host only, no device needed)."""
    buf = C.create_string_buffer(1 << 14)
    check(lib.ttb_debug_candidates(*p._args(), p.alpha, p.beta, buf, 1 << 14))
    return [s for s in buf.value.decode().split("\n") if s]


def version() -> str:
    return lib.ttb_version().decode()


def launch_count() -> int:
    return int(lib.ttb_launch_count())


# ------------------------------------------------- persistent solutions --

@dataclass
class SolutionEntry:
    """tuner.hpp:45-51: one line of the solution file (bandwidth in GiB/s)."""
    problem_key: str
    hardware_key: str
    plan: str
    bandwidth_gibs: float
    timestamp: str = ""


class SolutionCache:
    """The reference's SolutionCache (tuner.cpp:81-205) backed by the native
    store: tab-separated lines under flock, last matching entry wins."""

    def __init__(self, file):
        self.file = str(file)

    def lookup(self, problem_key: str, hardware_key: str) -> Optional[SolutionEntry]:
        plan = C.create_string_buffer(1024)
        ts = C.create_string_buffer(64)
        bw = C.c_double(0.0)
        found = C.c_int(0)
        check(lib.ttb_cache_lookup(self.file.encode(), problem_key.encode(),
                                   hardware_key.encode(), plan, 1024, C.byref(bw), ts, 64,
                                   C.byref(found)))
        if not found.value:
            return None
        return SolutionEntry(problem_key, hardware_key, plan.value.decode(), bw.value,
                             ts.value.decode())

    def store(self, entry: SolutionEntry) -> None:
        check(lib.ttb_cache_store(self.file.encode(), entry.problem_key.encode(),
                                  entry.hardware_key.encode(), entry.plan.encode(),
                                  float(entry.bandwidth_gibs)))


def hardware_key() -> str:
    """"<device>:sm<cc>:<SMs>sms:ttb<version>" of the current CUDA device."""
    buf = C.create_string_buffer(512)
    check(lib.ttb_hardware_key(buf, 512))
    return buf.value.decode()


# ------------------------------------------------------- benchmark suite --

@dataclass
class BenchmarkCase:
    """benchmark.hpp:17-22."""
    id: str
    problem: "TransposeProblem"
    category: str
    config: str


def _manifest(volume_bytes: int, kind, seed: int) -> List[str]:
    k = ElementKind.from_code(kind) if isinstance(kind, str) else ElementKind(kind)
    n = 1 << 16
    buf = C.create_string_buffer(n)
    check(lib.ttb_benchmark_manifest(int(volume_bytes), int(k.value), int(seed), buf, n))
    return [l for l in buf.value.decode().split("\n") if l]


def build_benchmark(volume_bytes: int, kind="s", seed: int = 42) -> List[BenchmarkCase]:
    """benchmark.cpp:166-220: the paper's 57 cases (alpha = beta = 1)."""
    cases = []
    for line in _manifest(volume_bytes, kind, seed):
        f = dict(kv.split("=", 1) for kv in line.split(";"))
        perm = [int(x) for x in f["perm"].split(",")]
        sizes = [int(x) for x in f["size"].split(",")]
        p = make_problem(perm, sizes, f["kinds"][0], f["kinds"][1], float(f["alpha"]),
                         float(f["beta"]))
        cases.append(BenchmarkCase(f["case"], p, f["category"], f["config"]))
    return cases


def benchmark_case_line(case: BenchmarkCase) -> str:
    """benchmark.cpp:258-266 -- the manifest line of a case."""
    p = case.problem
    kinds = p.kind_a.code + p.kind_b.code
    return (f"case={case.id};perm={','.join(map(str, p.perm.map))};"
            f"size={','.join(map(str, p.sizes))};kinds={kinds};alpha={p.alpha:.6g};"
            f"beta={p.beta:.6g};category={case.category};config={case.config}")


# ----------------------------------------------------------------- buffers --

def _torch():
    import torch  # noqa: PLC0415  (device memory only)
    return torch


class TensorBuffer:
    """Element-kind tagged DEVICE storage (executor.hpp:45-70).  Backed by a
    torch CUDA tensor of scalars (complex kinds: interleaved re/im)."""

    def __init__(self, kind, elements: int, device=None, tensor=None):
        torch = _torch()
        self._kind = _kind(kind)
        if elements < 0:
            raise ValueError("buffer: negative element count")
        self._elements = int(elements)
        dt = torch.float64 if self._kind in (ElementKind.real64, ElementKind.complex128) \
            else torch.float32
        n = self._elements * self._kind.components
        if tensor is None:
            tensor = torch.zeros(n, dtype=dt, device=device or "cuda")
        elif tensor.numel() < n or tensor.dtype != dt or not tensor.is_cuda:
            raise ValueError("buffer: tensor does not match kind/elements on a CUDA device")
        self.tensor = tensor

    def kind(self) -> ElementKind:
        return self._kind

    def elements(self) -> int:
        return self._elements

    def scalars(self) -> int:
        return self._elements * self._kind.components

    def bytes(self) -> int:
        return self._elements * self._kind.bytes

    def data_ptr(self) -> int:
        return self.tensor.data_ptr()


def make_buffer_a(p: TransposeProblem, device=None) -> TensorBuffer:
    return TensorBuffer(p.kind_a, required_elements_a(validate(p)), device)


def make_buffer_b(p: TransposeProblem, device=None) -> TensorBuffer:
    return TensorBuffer(p.kind_b, required_elements_b(validate(p)), device)


def _stream(stream):
    if stream is None:
        return C.c_void_p(_torch().cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _check_kinds(p: TransposeProblem, a: TensorBuffer, b: TensorBuffer):
    if a.kind() != p.kind_a:
        raise ValueError("A buffer: element kind mismatch")
    if b.kind() != p.kind_b:
        raise ValueError("B buffer: element kind mismatch")


def reference_transpose(p: TransposeProblem, a: TensorBuffer, b: TensorBuffer,
                        stream=None) -> None:
    """executor.hpp:80-83 on the GPU: plan from the cache (heuristic on a miss),
    asynchronous on `stream` (default: torch's current stream)."""
    validate(p)
    _check_kinds(p, a, b)
    check(lib.ttb_transpose(*p._args(), p.alpha, C.c_void_p(a.data_ptr()), a.elements(), p.beta,
                            C.c_void_p(b.data_ptr()), b.elements(), _stream(stream)))


class GpuPlan:
    """The sm_100a counterpart of ttune::CandidatePlan (plan.hpp) plus its
    executor: variant, tile, vector widths, launch shape for one problem."""

    def __init__(self, p: TransposeProblem, cache: bool = True):
        validate(p)
        self.problem = p
        h = C.c_void_p()
        check(lib.ttb_plan_create(C.byref(h), *p._args(), p.alpha, p.beta, 0 if cache else 1))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.ttb_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass

    def _pointers(self, a, b):
        """Device addresses of A and B.  TensorBuffers are checked like
        execute_plan's check_buffers (executor.cpp:315-322): kind, then
        capacity; torch tensors by byte capacity; raw integers are taken as
        they are (the C ABI cannot size a bare pointer)."""
        p = self.problem
        for name, buf, kind, need in (("A", a, p.kind_a, required_elements_a(p)),
                                      ("B", b, p.kind_b, required_elements_b(p))):
            if isinstance(buf, TensorBuffer):
                if buf.kind() != kind:
                    raise ValueError(f"{name} buffer: element kind mismatch")
                if buf.elements() < need:
                    raise ValueError(f"{name} buffer: too small for problem")
            elif hasattr(buf, "numel") and hasattr(buf, "element_size"):
                if buf.numel() * buf.element_size() < need * kind.bytes:
                    raise ValueError(f"{name} buffer: too small for problem")
        pa = a.data_ptr() if hasattr(a, "data_ptr") else int(a)
        pb = b.data_ptr() if hasattr(b, "data_ptr") else int(b)
        return pa, pb

    def execute(self, a, b, stream=None) -> None:
        pa, pb = self._pointers(a, b)
        check(lib.ttb_plan_execute(self._h, C.c_void_p(pa), C.c_void_p(pb), _stream(stream)))

    def execute_host(self, a_host, b_host, wait: bool = True) -> None:
        """End-to-end on host (numpy/pinned torch) buffers: H2D, kernel, D2H.
        Both buffers are sized like execute's (the C ABI cannot size them).
        wait=False queues the call and returns (ttb_plan_execute_host_async):
        b_host is valid, and both buffers reusable, after host_sync(); calls on
        different plans overlap."""
        p = self.problem
        for name, buf, kind, need in (("A", a_host, p.kind_a, required_elements_a(p)),
                                      ("B", b_host, p.kind_b, required_elements_b(p))):
            nbytes = buf.nbytes if hasattr(buf, "nbytes") else buf.numel() * buf.element_size()
            if nbytes < need * kind.bytes:
                raise ValueError(f"{name} buffer: too small for problem")
        pa = a_host.ctypes.data if hasattr(a_host, "ctypes") else a_host.data_ptr()
        pb = b_host.ctypes.data if hasattr(b_host, "ctypes") else b_host.data_ptr()
        fn = lib.ttb_plan_execute_host if wait else lib.ttb_plan_execute_host_async
        check(fn(self._h, C.c_void_p(pa), C.c_void_p(pb)))

    def host_sync(self) -> None:
        """Wait for the host call queued by execute_host(..., wait=False)."""
        check(lib.ttb_plan_host_sync(self._h))

    def autotune(self, a, b, warmups: int = 2, reps: int = 3, stream=None) -> str:
        pa, pb = self._pointers(a, b)
        check(lib.ttb_plan_autotune(self._h, C.c_void_p(pa), C.c_void_p(pb), warmups, reps,
                                    _stream(stream)))
        return self.describe()

    def tune_cached(self, a, b, cache_file: str, warmups: int = 2, reps: int = 3,
                    stream=None) -> bool:
        """pipeline.cpp:102-185 for this plan: select the cached plan of (canonical
        key, hardware key) from `cache_file`, or autotune and append the winner.
        Returns True on a cache hit.  B holds one application afterwards."""
        pa, pb = self._pointers(a, b)
        hit = C.c_int(0)
        check(lib.ttb_plan_tune_cached(self._h, str(cache_file).encode(), C.c_void_p(pa),
                                       C.c_void_p(pb), warmups, reps, _stream(stream),
                                       C.byref(hit)))
        return bool(hit.value)

    def describe(self) -> str:
        buf = C.create_string_buffer(512)
        check(lib.ttb_plan_describe(self._h, buf, 512))
        return buf.value.decode()

    def candidates(self) -> List[str]:
        buf = C.create_string_buffer(1 << 14)
        check(lib.ttb_plan_candidates(self._h, buf, 1 << 14))
        return [s for s in buf.value.decode().split("\n") if s]

    def select(self, text: str) -> None:
        check(lib.ttb_plan_select(self._h, text.encode()))

    def launches(self) -> int:
        """Kernel launches per execute (one per box for oversized problems)."""
        n = C.c_int(0)
        check(lib.ttb_plan_launches(self._h, C.byref(n)))
        return n.value


class EmittedKernel:
    """emit.hpp:27-34: entry symbol, header / source text and file names."""

    def __init__(self, entry_symbol: str, include_name: str, header_text: str, source_text: str):
        self.entry_symbol = entry_symbol
        self.include_name = include_name
        self.header_text = header_text
        self.source_text = source_text
        self.source_extension = "cu"
        self.header_extension = "h"


def emit_source(p: TransposeProblem, plan=None, basename: str = "") -> EmittedKernel:
    """Standalone sm_100a CUDA source for `plan` (a GpuPlan, a plan text or None)
    on `p` (emit.cpp:622-715 analogue; no device needed)."""
    validate(p)
    text = plan.describe() if isinstance(plan, GpuPlan) else plan
    ent = C.create_string_buffer(1024)
    hdr = C.create_string_buffer(1 << 14)
    src = C.create_string_buffer(1 << 17)
    check(lib.ttb_emit_source(*p._args(), p.alpha, p.beta, text.encode() if text else None,
                              basename.encode() if basename else None, ent, 1024, hdr, 1 << 14,
                              src, 1 << 17))
    entry = ent.value.decode()
    return EmittedKernel(entry, f"{basename or entry}.h", hdr.value.decode(), src.value.decode())


def write_kernel_files(kernel: EmittedKernel, base) -> Tuple[str, str]:
    """emit.cpp write_kernel_files: <base>.cu and the header next to it."""
    import os  # noqa: PLC0415
    base = str(base)
    d = os.path.dirname(base)
    if d:
        os.makedirs(d, exist_ok=True)
    src = base + "." + kernel.source_extension
    hdr = os.path.join(d, kernel.include_name)
    with open(src, "w") as f:
        f.write(kernel.source_text)
    with open(hdr, "w") as f:
        f.write(kernel.header_text)
    return src, hdr


def execute_plan(p: TransposeProblem, plan: Optional[GpuPlan], a: TensorBuffer, b: TensorBuffer,
                 stream=None) -> None:
    """executor.hpp:85-88: run a given plan (None = cached heuristic plan)."""
    if plan is None:
        return reference_transpose(p, a, b, stream)
    validate(p)
    _check_kinds(p, a, b)
    if a.elements() < required_elements_a(p):
        raise ValueError("A buffer: too small for problem")
    if b.elements() < required_elements_b(p):
        raise ValueError("B buffer: too small for problem")
    plan.execute(a, b, stream)


# --------------------------------------------------------- partition/data --

def shard_boxes(p: TransposeProblem, world: int, rank: int) -> List[Tuple[List[int], List[int]]]:
    """Boxes (origin, extent in A order) of `rank`'s slab of B."""
    n = p.rank()
    cnt = C.c_int(0)
    check(lib.ttb_shard_boxes(n, ints(p.perm.map), longs(p.sizes), world, rank, None, None,
                              C.byref(cnt)))
    o, e = (C.c_int64 * (cnt.value * n))(), (C.c_int64 * (cnt.value * n))()
    check(lib.ttb_shard_boxes(n, ints(p.perm.map), longs(p.sizes), world, rank, o, e,
                              C.byref(cnt)))
    return [(list(o[i * n:(i + 1) * n]), list(e[i * n:(i + 1) * n])) for i in range(cnt.value)]


def fill_uniform(kind, sizes, ld, seed: int, ptr: int, origin=None, global_sizes=None,
                 stream=None) -> None:
    check(lib.ttb_fill_uniform(int(_kind(kind)), len(sizes), longs(sizes), longs(ld),
                               longs(origin), longs(global_sizes), seed, C.c_void_p(ptr),
                               _stream(stream)))


def fill_sentinel(kind, elements: int, ptr: int, stream=None) -> None:
    check(lib.ttb_fill_sentinel(int(_kind(kind)), elements, C.c_void_p(ptr), _stream(stream)))


def checksum(kind, sizes, ld, ptr: int, origin=None, global_sizes=None, stream=None) -> int:
    out = C.c_uint64(0)
    check(lib.ttb_checksum(int(_kind(kind)), len(sizes), longs(sizes), longs(ld), longs(origin),
                           longs(global_sizes), C.c_void_p(ptr), C.byref(out), _stream(stream)))
    return out.value
