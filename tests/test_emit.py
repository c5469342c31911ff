"""Source emission: the standalone sm_100a kernel of one
plan on one problem, the counterpart of ttune's emit_source (emit.cpp:622-715,
tests test_emit.cpp:97-205).  CPU part: entry symbols name the problem as the
reference's do (test_emit.cpp:97-122), the header declares the reference's
prototype, banners carry problem key and plan, the files land next to each
other, and the source compiles with nvcc for sm_100a.  The device run is in
test_gpu_emit.py.
"""
import os
import shutil
import subprocess

import pytest

import paper_1603_02297_b200 as ttb

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


def test_entry_symbols_name_the_problem():
    k = ttb.emit_source(ttb.make_problem([2, 1], [200, 200]))
    assert k.entry_symbol == "transpose_21_200x200_ss"
    assert k.include_name == "transpose_21_200x200_ss.h"
    m = ttb.make_problem([3, 2, 1], [5, 6, 7], "d", "d")
    assert ttb.emit_source(m).entry_symbol == "transpose_321_5x6x7_dd"
    rev = list(range(10, 0, -1))
    w = ttb.emit_source(ttb.make_problem(rev, [2] * 10))
    assert w.entry_symbol == "transpose_10_9_8_7_6_5_4_3_2_1_2x2x2x2x2x2x2x2x2x2_ss"
    named = ttb.emit_source(ttb.make_problem([2, 1], [8, 8]), None, "mykernel")
    assert named.include_name == "mykernel.h"
    assert '#include "mykernel.h"' in named.source_text
    assert "#ifndef TTB_MYKERNEL_H" in named.header_text


def test_emitted_text_structure():
    p = ttb.make_problem([2, 1], [50, 42], "s", "d")
    plan = "kern=smem;kx=1;ky=1;tx=16;ty=8;order=0;occ=0;st=2;bp=1;vec=1"
    k = ttb.emit_source(p, plan, "k")
    # the reference's prototype (emit.cpp header slot), device pointers
    assert "void transpose_21_50x42_sd(const float* A, double* B, double alpha, double beta);" \
        in k.header_text
    assert 'extern "C"' in k.header_text
    assert "cudaStream_t stream" in k.header_text
    assert "plan: " + plan in k.source_text
    assert "problem: " + ttb.canonical_key(p) in k.source_text
    assert "#define TX 16LL" in k.source_text and "#define TY 8LL" in k.source_text
    assert "__dmul_rn" in k.source_text and "__dadd_rn" in k.source_text  # W = double (s -> d)
    # case 1 and rank 1 are copies along the shared stride-1 run
    c1 = ttb.emit_source(ttb.make_problem([1, 3, 2], [13, 6, 10]), None, "c1")
    assert "TX" not in c1.source_text and "% 13LL" in c1.source_text


def test_emit_rejects_invalid_requests():
    p = ttb.make_problem([2, 1], [16, 16])
    with pytest.raises(ValueError, match="emit: cannot parse plan text"):
        ttb.emit_source(p, "kern=warp;x=1")
    with pytest.raises(ValueError, match="emit: basename must be a plain file name"):
        ttb.emit_source(p, None, "../evil")
    with pytest.raises(ValueError, match="perm: not a permutation"):
        ttb.emit_source(ttb.make_problem([1, 1], [4, 4]))


def test_kernel_files_land_next_to_each_other(tmp_path):
    k = ttb.emit_source(ttb.make_problem([2, 1], [8, 8]), None, "pair")
    src, hdr = ttb.write_kernel_files(k, tmp_path / "nested" / "pair")
    assert src == str(tmp_path / "nested" / "pair.cu")
    assert hdr == str(tmp_path / "nested" / "pair.h")
    assert open(src).read() == k.source_text and open(hdr).read() == k.header_text


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not available")
@pytest.mark.parametrize("kind_a,kind_b,perm,sizes,lda,ldb,alpha,beta,plan", [
    ("s", "s", [3, 2, 1], [48, 7, 32], None, None, 2.0, 1.0,
     "kern=smem;kx=1;ky=1;tx=16;ty=8;order=0;occ=0;st=2;bp=1;vec=1"),
    ("z", "z", [2, 1], [21, 10], None, None, 2.0, 1.5, None),
    ("s", "d", [3, 1, 2], [19, 5, 7], [19, 6, 7], None, 2.0, 3.0, None),
    ("c", "c", [1], [2311], None, None, 2.0, 3.0, None),
])
def test_emitted_source_compiles_for_sm100a(tmp_path, kind_a, kind_b, perm, sizes, lda, ldb, alpha,
                                            beta, plan):
    p = ttb.make_problem(perm, sizes, kind_a, kind_b, alpha, beta, lda, ldb)
    k = ttb.emit_source(p, plan, "k")
    src, _ = ttb.write_kernel_files(k, tmp_path / "k")
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-c",
                        "-o", str(tmp_path / "k.o"), src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
