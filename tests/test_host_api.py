"""Host-side logic of the engine through its C ABI (CPU only, no device).

Covers: the library loads and exports every symbol include/ttb.h declares;
validate / merge_indices / canonical_key / required_elements / bandwidth match
the reference (golden fixtures + live reference where built); the planner's
candidate lists; the multi-GPU partition; the in-kernel 32-bit divider.
"""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1603_02297_b200 as ttb
from paper_1603_02297_b200 import _lib
from paper_1603_02297_b200.workloads import ALL, CONFIGS, C5
from golden_util import load_merge_validate
from problems import random_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "ttb.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(ttb_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 24
    missing = [s for s in declared if not hasattr(_lib.lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) >= declared
    assert ttb.version() == "0.1.0"


def test_validate_messages_match_golden():
    g = load_merge_validate()
    for v in g["invalid"]:
        p = ttb.make_problem(v["perm"], v["sizes"], v["kind_a"], v["kind_b"], 1.0, 0.0,
                             v["lda"], v["ldb"])
        if v["message"] is None:
            ttb.validate(p)
            continue
        with pytest.raises(ValueError) as ei:
            ttb.validate(p)
        assert str(ei.value) == v["message"]


def test_validate_random_matches_reference(refo):
    rng = np.random.default_rng(99)
    for _ in range(300):
        perm, sizes, lda, ldb = random_problem(rng, 5)
        r = rng.integers(0, 5)
        if r == 0:
            lda = [max(0, v - 2) for v in lda]
        elif r == 1:
            ldb = [max(0, v - 2) for v in ldb]
        elif r == 2:
            perm = [p if rng.integers(0, 4) else 1 for p in perm]
        p = ttb.make_problem(perm, sizes, "s", "s", 1.0, 0.0, lda, ldb)
        want = refo.validate(perm, sizes, lda, ldb)
        try:
            ttb.validate(p)
            got = None
        except ValueError as e:
            got = str(e)
        assert got == want


def test_merge_matches_golden():
    g = load_merge_validate()
    for m in g["merges"]:
        p = ttb.make_problem(m["perm"], m["sizes"], "s", "s", 1.0, 0.0, m["lda"], m["ldb"])
        n = ttb.merge_indices(p)
        w = m["out"]
        assert n.problem.perm.map == w["perm"]
        assert n.problem.sizes == w["sizes"]
        assert n.problem.lda == w["lda"]
        assert n.problem.ldb == w["ldb"]
        assert [[t.from_first, t.from_last] for t in n.merge_trace] == w["trace"]


def test_merge_matches_reference_live(refo):
    rng = np.random.default_rng(5150)
    for t in range(400):
        perm, sizes, lda, ldb = random_problem(rng, 6, allow_padding=(t % 2 == 0))
        n = ttb.merge_indices(ttb.make_problem(perm, sizes, "s", "s", 1.0, 0.0, lda, ldb))
        mp, ms, mla, mlb, trace = refo.merge(perm, sizes, lda, ldb)
        assert (n.problem.perm.map, n.problem.sizes, n.problem.lda, n.problem.ldb) == \
            (mp, ms, mla, mlb)
        assert [(t.from_first, t.from_last) for t in n.merge_trace] == trace


def test_canonical_key_matches_golden():
    for k in load_merge_validate()["keys"]:
        p = ttb.make_problem(k["perm"], k["sizes"], k["kind_a"], k["kind_b"], k["alpha"],
                             k["beta"], k["lda"], k["ldb"])
        assert ttb.canonical_key(p) == k["key"]
    # test_problem.cpp:85-91
    assert ttb.canonical_key(ttb.make_problem([2, 1], [4, 4])) == \
        "perm=2,1;size=4,4;lda=4,4;ldb=4,4;kinds=ss;beta=z"


def test_geometry_known_answers():
    # test_problem.cpp:42-64
    p = ttb.make_problem([3, 1, 2], [4, 5, 6])
    assert p.lda == [4, 5, 6] and p.ldb == [5, 6, 4]
    assert ttb.sizes_b(p) == [5, 6, 4]
    assert ttb.element_strides_a(p) == [1, 4, 20]
    assert ttb.element_strides_b(p) == [1, 5, 30]
    assert ttb.element_strides_b_for_a(p) == [30, 1, 5]
    assert ttb.b_stride1_axis(p) == 1
    assert ttb.required_elements_a(p) == 120 and ttb.required_elements_b(p) == 120
    q = ttb.make_problem([2, 1], [4, 6], "s", "s", 1.0, 0.0, [5, 6], [8, 4])
    assert ttb.required_elements_a(q) == 1 + 3 * 1 + 5 * 5
    assert ttb.required_elements_b(q) == 1 + 5 * 1 + 3 * 8
    assert ttb.Permutation([3, 1, 2]).inverse().map == [2, 3, 1]
    assert ttb.Permutation.from_gather((2, 0, 3, 1)).map == [2, 4, 1, 3]


def test_bandwidth_formula():
    # test_tuner.cpp:36-51 in decimal GB/s
    z = ttb.make_problem([2, 1], [1 << 10, 1 << 10], "s", "d")
    assert ttb.bandwidth_gbs(z, 0.5) == pytest.approx((1 << 20) * 12 / 1e9 / 0.5, rel=1e-12)
    nz = ttb.make_problem([2, 1], [1 << 10, 1 << 10], "s", "d", 1.0, 2.0)
    assert ttb.bandwidth_gbs(nz, 2.0) == pytest.approx((1 << 20) * 20 / 1e9 / 2.0, rel=1e-12)
    c = ttb.make_problem([2, 1], [64, 64], "z", "z", 1.0, 1.0)
    assert ttb.bandwidth_gbs(c, 1.0) == pytest.approx(64 * 64 * 48 / 1e9, rel=1e-12)
    with pytest.raises(ValueError, match="bandwidth: time must be positive"):
        ttb.bandwidth_gbs(z, 0.0)
    for w in CONFIGS:  # workloads.py byte counts agree with the engine's
        p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                             w.lda and list(w.lda), w.ldb and list(w.ldb))
        assert ttb.bandwidth_gbs(p, 1.0) == pytest.approx(w.algorithmic_bytes / 1e9)


def _problem(w):
    return ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                            w.lda and list(w.lda), w.ldb and list(w.ldb))


def test_planner_candidates_for_baseline_configs():
    plans = {w.name: ttb.debug_candidates(_problem(w)) for w in ALL}
    for name, c in plans.items():
        assert c, name
        # the list always ends with an alignment-free plan
        assert c[-1].startswith("kern=smem") or c[-1].startswith("kern=copy;v=1")
    # c1: fp32 2-D, both leads 7264: in-register 4x4 micro-tiles are available
    assert any(s.startswith("kern=rt;mx=4;my=4") for s in plans["c1"])
    # c2b keeps the stride-1 index: the vectorised copy kernel is offered, and
    # the bulk tile with the shared lead ranks first (384-byte rows: measured
    # 1.25x the row kernel, profiles/r02_cands)
    assert any(s.startswith("kern=copy;v=4") for s in plans["c2b"])
    assert plans["c2b"][0].startswith("kern=smem") and "vec=3" in plans["c2b"][0]
    # beta != 0 with every stride a 16-byte multiple: the tensor-map tile leads
    assert plans["c3"][0].startswith("kern=tma")
    # long shared rows keep a row kernel first
    assert plans["c5_t01"][0].startswith("kern=copy")
    # c3 fp64: 16-byte vectors on both sides
    assert any(s.startswith("kern=rt;mx=2;my=2") for s in plans["c3"])
    # c4s: padded A lead still allows 16-byte (2 x complex64) loads
    assert any(s.startswith("kern=rt;mx=2;my=2") for s in plans["c4s"])


def test_planner_offers_bulk_tiles_and_row_alignment():
    """The bulk-copy staged tile (btile.cuh, plan text vec=3 column walk / vec=4
    linear walk) and the long-row segment alignment (copy, order bits 1-2)."""
    c = {w.name: ttb.debug_candidates(_problem(w)) for w in ALL}
    # fp32 2-D: 128 x 128 tiles (512-byte runs on both sides, big warp roles)
    assert any("tx=128;ty=128" in s and "vec=3" in s for s in c["c1"])
    # shared stride-1 lead of 49 floats (run_case1 shape): bulk tiles of rows
    assert any(s.startswith("kern=smem") and "vec=3" in s for s in c["c5_t10"])
    # B lead of 2 doubles: the linear walk, and B read directly (bp=0) with beta != 0
    assert any("vec=4" in s and "bp=0" in s for s in c["c5_t15"])
    # long shared rows: the two segment alignments next to the plain order
    assert any(s.startswith("kern=copy") and "order=2" in s for s in c["c5_t01"])
    assert any(s.startswith("kern=copy") and "order=4" in s for s in c["c5_t01"])
    # column walks with 8 / 16 lanes per column (8 x 4 rows x columns per warp)
    assert any("vec=3" in s and s.endswith("ly=8") for s in c["c5_t22"])
    # B continuing from Y into X's second axis: the column-permuted linear walk
    assert any("vec=4" in s and s.endswith("xp=1") for s in c["c5_t18"])
    # mixed kind pairs get bulk tiles too (A rows and B columns fetched with
    # their own element sizes, converting epilogue)
    p = ttb.make_problem([2, 1], [512, 640], "s", "d", 1.0, 0.0)
    assert any("vec=3" in s or "vec=4" in s for s in ttb.debug_candidates(p))


def test_planner_candidates_random_problems_are_well_formed():
    rng = np.random.default_rng(7)
    for t in range(200):
        perm, sizes, lda, ldb = random_problem(rng, 6)
        kind = "sdcz"[t % 4]
        p = ttb.make_problem(perm, sizes, kind, kind, 1.0, 0.0 if t % 2 else 0.5, lda, ldb)
        c = ttb.debug_candidates(p)
        assert c and all(s.startswith("kern=") for s in c)


def _b_linear_indices(w, boxes):
    """B-linear logical indices covered by boxes (A-order origin/extent)."""
    sizes = list(w.sizes)
    perm = w.perm
    sb = [0] * len(perm)
    for a, k in enumerate(perm):
        sb[k - 1] = sizes[a]
    stride_b = [1] * len(perm)
    for k in range(1, len(perm)):
        stride_b[k] = stride_b[k - 1] * sb[k - 1]
    out = []
    for origin, ext in boxes:
        grids = np.meshgrid(*[np.arange(o, o + e) for o, e in zip(origin, ext)], indexing="ij")
        lin = np.zeros(grids[0].shape, np.int64)
        for a in range(len(perm)):
            lin += grids[a] * stride_b[perm[a] - 1]
        out.append(lin.ravel())
    return np.concatenate(out) if out else np.zeros(0, np.int64)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_boxes_partition_b(world):
    """Every rank's boxes are disjoint, together they cover B exactly, and
    ranks own contiguous B-linear ranges (a slab) whenever the split axes are
    B's outermost positions in order (shard.cpp moves A's stride-1 axis last)."""
    from paper_1603_02297_b200.workloads import Workload
    rng = np.random.default_rng(world)
    shapes = [Workload("x", "s", tuple(rng.permutation(d)), tuple(int(v) for v in
              rng.integers(1, 7, d)), 1.0, 0.0, 0) for d in (2, 3, 4, 5) for _ in range(6)]
    shapes.append(Workload("t15", "d", (4, 0, 2, 1, 5, 3), (6, 4, 3, 9, 2, 5), 1.0, 0.0, 0))
    for w in shapes:
        p = _problem(w)
        total = p.total_elements()
        seen = []
        n = p.rank()
        for r in range(world):
            boxes = ttb.shard_boxes(p, world, r)
            assert len(boxes) <= 2 * p.rank() - 1
            idx = _b_linear_indices(w, boxes)
            # a slab per rank whenever the axes its boxes restrict are B's
            # outermost positions (shard.cpp: stride-1 axes last, a single
            # evenly splitting axis preferred)
            cut = {p.perm.map[a] - 1 for _, e in boxes for a in range(n) if e[a] < p.sizes[a]}
            slab = (n <= 2 or p.perm.map[0] <= 2) and cut == set(range(n - len(cut), n))
            if idx.size and slab:
                s = np.sort(idx)
                assert s[-1] - s[0] + 1 == s.size  # contiguous slab of B
            seen.append(idx)
        allidx = np.sort(np.concatenate(seen))
        assert np.array_equal(allidx, np.arange(total)), w


def test_shard_balance_on_sweep():
    """the flattened outer-k split keeps max/mean <= 1.05 at 8 ranks; a
    single axis that splits within 1.07 is taken alone (one box per rank)."""
    for w in C5:
        p = _problem(w)
        sizes = [sum(int(np.prod(e)) for _, e in ttb.shard_boxes(p, 8, r)) for r in range(8)]
        assert sum(sizes) == p.total_elements()
        assert max(sizes) / (sum(sizes) / 8) <= 1.07, (w.name, sizes)


def test_div32_formula(tmp_path):
    """The in-kernel 32-bit divider (params.hpp Div32) is exact."""
    src = tmp_path / "d.cpp"
    src.write_text(r"""
#include "params.hpp"
#include <cstdio>
#include <random>
using namespace ttb;
static uint32_t udiv_h(uint32_t n, const Div32& f) {
  uint64_t hi = (static_cast<uint64_t>(n) * f.m) >> 32;
  return static_cast<uint32_t>((hi + n) >> f.s);
}
int main() {
  std::mt19937_64 r(1);
  const uint32_t ds[] = {1u, 2u, 3u, 7u, 24u, 96u, 227u, 7264u, 65535u, 65537u, 1u << 20,
                         2147483647u, 2147483648u, 4294967295u};
  for (uint32_t d : ds) {
    Div32 f = Div32::make(d);
    for (int i = 0; i < 200000; ++i) {
      uint32_t n = (i < 1000) ? i : static_cast<uint32_t>(r());
      if (i == 1001) n = 4294967295u;
      if (udiv_h(n, f) != n / d) { std::printf("FAIL %u %u\n", n, d); return 1; }
    }
  }
  for (int i = 0; i < 200000; ++i) {
    uint32_t d = static_cast<uint32_t>(r() % 100000) + 1, n = static_cast<uint32_t>(r());
    if (udiv_h(n, Div32::make(d)) != n / d) { std::printf("FAIL %u %u\n", n, d); return 1; }
  }
  std::puts("ok");
}
""")
    exe = tmp_path / "d"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I",
                    os.path.join(ROOT, "paper_1603_02297_b200", "csrc"), str(src), "-o", str(exe)],
                   check=True)
    assert subprocess.run([str(exe)], capture_output=True, text=True).stdout.strip() == "ok"


def test_plan_create_without_device_fails_loudly():
    """No CPU fallback: planning/execution needs the CUDA device."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    p = ttb.make_problem([2, 1], [8, 8])
    with pytest.raises((ttb.TTBError, MemoryError)):
        ttb.GpuPlan(p)
