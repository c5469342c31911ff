"""Build libttb.so (the CUDA engine + C ABI) in-tree with nvcc for sm_100a.

    python -m paper_1603_02297_b200._build [--verbose]

Objects go to paper_1603_02297_b200/_lib/obj, the library to
paper_1603_02297_b200/_lib/libttb.so (git-ignored; it travels to the GPU box
with the snapshot).  Sources compile in parallel; unchanged objects are reused.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "libttb.so")
ROOT = os.path.dirname(PKG)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _host_cxx() -> str:
    # the system g++: its shared libstdc++ keeps C++ exceptions sane when the
    # library is dlopen'ed from Python (see oracle/Makefile)
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")


def _flags() -> list:
    return [
        "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O3", "-ccbin", _host_cxx(),
        "-I", CSRC, "-I", os.path.join(ROOT, "include"),
        # bit-exact epilogue: no FMA contraction anywhere, IEEE fp32 (no FTZ)
        "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    ]


def _deps() -> list:
    return sorted(glob.glob(os.path.join(CSRC, "*.h*")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "ttb.h")])


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, os.path.basename(src) + ".o")
    newest_dep = max(os.path.getmtime(d) for d in _deps() + [src, __file__])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [_nvcc(), *_flags(), "-c", src, "-o", obj]
    if verbose and src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or max(os.path.getmtime(o) for o in objs) > os.path.getmtime(LIB):
        cmd = [_nvcc(), *ARCH, "-shared", "-ccbin", _host_cxx(), "-o", LIB + ".tmp", *objs,
               "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    _build_cli()
    return LIB


CLI_SRC = os.path.join(PKG, "tools", "ttb_cli.cpp")
CLI = os.path.join(LIBDIR, "ttb")


def _build_cli() -> None:
    """tools/ttb_cli.cpp -> _lib/ttb, a C-ABI client of libttb.so (rpath $ORIGIN)."""
    if os.path.exists(CLI) and os.path.getmtime(CLI) >= max(
            os.path.getmtime(CLI_SRC), os.path.getmtime(LIB),
            os.path.getmtime(os.path.join(ROOT, "include", "ttb.h"))):
        return
    cmd = [_nvcc(), "-std=c++17", "-O2", "-ccbin", _host_cxx(), "-I", os.path.join(ROOT, "include"),
           CLI_SRC, "-o", CLI + ".tmp", "-L", LIBDIR, "-lttb", "-Xlinker", "-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cli build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(CLI + ".tmp", CLI)


def build_variant(name: str, defines: list, only=None) -> str:
    """Experiment build: sources with extra -D flags into _lib/libttb_<name>.so
    (load it with TTB_LIB_PATH; the product always uses libttb.so).  `only`:
    recompile just these source basenames, the rest from the product objects."""
    build()
    objdir = os.path.join(LIBDIR, f"obj_{name}")
    os.makedirs(objdir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))

    def one(src):
        if only and os.path.basename(src) not in only:
            return os.path.join(OBJDIR, os.path.basename(src) + ".o")
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [_nvcc(), *_flags(), *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        subprocess.run(cmd, check=True, capture_output=True)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, srcs))
    out = os.path.join(LIBDIR, f"libttb_{name}.so")
    subprocess.run([_nvcc(), *ARCH, "-shared", "-ccbin", _host_cxx(), "-o", out, *objs], check=True)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        args = sys.argv[3:]
        only = [a[len("--only="):] for a in args if a.startswith("--only=")]
        print(build_variant(sys.argv[2], [a for a in args if not a.startswith("--only=")],
                            only=only or None))
    else:
        print(build(verbose="--verbose" in sys.argv))
