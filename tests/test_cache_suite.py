"""Persistent solution cache and the paper's benchmark suite (host-only parts
of SURVEY s8(f) rows 2 and 3), CPU only.

The cache file format and semantics follow the reference's SolutionCache
(tuner.cpp:81-205): tab-separated lines appended under flock, malformed lines
skipped, the last matching entry wins, single-line non-empty fields enforced
with the reference's message.  Files written by either side are read by the
other.  The suite generator follows build_benchmark (benchmark.cpp:166-220)
and must reproduce the reference's manifest line for line.
"""
import json
import multiprocessing as mp
import os

import pytest

import paper_1603_02297_b200 as ttb

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PLAN = "order=1,2;bA=16;bB=16;d=5;ss=0;w=8"  # a plan text the reference can parse


def test_cache_store_lookup_last_entry_wins(tmp_path):
    f = tmp_path / "solutions.tsv"
    c = ttb.SolutionCache(f)
    assert c.lookup("k1", "hw") is None  # no file yet
    c.store(ttb.SolutionEntry("k1", "hw", "kern=rt;mx=4;my=4", 12.5))
    c.store(ttb.SolutionEntry("k2", "hw", "kern=copy;v=4", 7.0))
    c.store(ttb.SolutionEntry("k1", "hw", "kern=smem;tx=32;ty=32", 13.25))
    c.store(ttb.SolutionEntry("k1", "other-hw", "kern=copy;v=1", 1.0))
    e = c.lookup("k1", "hw")
    assert e.plan == "kern=smem;tx=32;ty=32" and e.bandwidth_gibs == 13.25
    assert len(e.timestamp) == 20 and e.timestamp.endswith("Z")
    assert c.lookup("k1", "nope") is None
    lines = f.read_text().splitlines()
    assert len(lines) == 4 and all(len(l.split("\t")) == 5 for l in lines)


def test_cache_skips_malformed_lines(tmp_path, capfd):
    f = tmp_path / "solutions.tsv"
    f.write_text("garbage\nk1\thw\tkern=x\tnot-a-number\tts\n\nk1\thw\tkern=good\t2.5\tts\n"
                 "k1\t\tkern=x\t1\tts\n")
    e = ttb.SolutionCache(f).lookup("k1", "hw")
    assert e.plan == "kern=good" and e.bandwidth_gibs == 2.5
    assert "skipped 3 malformed line(s)" in capfd.readouterr().err


@pytest.mark.parametrize("bad", [("", "hw", "p"), ("k\t1", "hw", "p"), ("k", "h\nw", "p"),
                                 ("k", "hw", "")])
def test_cache_rejects_multiline_or_empty_fields(tmp_path, bad):
    with pytest.raises(ValueError, match="cache: entry fields must be non-empty single-line text"):
        ttb.SolutionCache(tmp_path / "s.tsv").store(ttb.SolutionEntry(*bad, 1.0))


def _appender(args):
    path, who, n = args
    c = ttb.SolutionCache(path)
    for i in range(n):
        c.store(ttb.SolutionEntry(f"key{i % 7}", f"hw{who}", f"kern=p{who}_{i}", float(i)))


def test_cache_concurrent_appends_stay_whole_lines(tmp_path):
    f = str(tmp_path / "shared.tsv")
    with mp.get_context("spawn").Pool(4) as pool:
        pool.map(_appender, [(f, w, 60) for w in range(4)])
    lines = open(f).read().splitlines()
    assert len(lines) == 240
    assert all(len(l.split("\t")) == 5 for l in lines)
    for w in range(4):
        assert ttb.SolutionCache(f).lookup("key0", f"hw{w}").plan == f"kern=p{w}_56"


def test_cache_file_interoperates_with_reference(refo, tmp_path):
    f = tmp_path / "both.tsv"
    key = refo.canonical_key([2, 1], [64, 32])
    assert key == ttb.canonical_key(ttb.make_problem([2, 1], [64, 32]))
    refo.cache_store(f, key, "host:t8:w8", REF_PLAN, 5.95)
    e = ttb.SolutionCache(f).lookup(key, "host:t8:w8")
    assert e.plan == REF_PLAN and e.bandwidth_gibs == 5.95
    ttb.SolutionCache(f).store(ttb.SolutionEntry(key, "host:t8:w8", REF_PLAN, 6.5))
    assert refo.cache_lookup(f, key, "host:t8:w8") == (REF_PLAN, 6.5)


def test_benchmark_manifest_matches_golden():
    with open(os.path.join(HERE, "golden", "benchmark_manifest.json")) as fh:
        golden = json.load(fh)
    assert len(golden) == 3
    for name, lines in golden.items():
        mib, kind, seed = name.split("_")
        got = [ttb.benchmark_case_line(c)
               for c in ttb.build_benchmark(int(mib[:-3]) << 20, kind, int(seed))]
        assert got == lines, name


@pytest.mark.parametrize("vol,kind,seed", [(1 << 20, "s", 42), (16 << 20, "z", 3),
                                           (300 << 20, "d", 1234), (50 << 20, "c", 0)])
def test_benchmark_manifest_matches_reference_live(refo, vol, kind, seed):
    ours = [ttb.benchmark_case_line(c) for c in ttb.build_benchmark(vol, kind, seed)]
    assert ours == refo.benchmark_manifest(vol, kind, seed)


def test_benchmark_suite_shape():
    cases = ttb.build_benchmark(200 << 20, "s", 42)
    assert len(cases) == 57
    dims = [c.problem.rank() for c in cases]
    assert [dims.count(d) for d in range(2, 7)] == [3, 9, 15, 15, 15]
    for c in cases:
        n = 1
        for s in c.problem.sizes:
            n *= s
        assert abs(n * 4 / (200 << 20) - 1) <= 0.10
        m = c.problem.perm.map
        assert all(m[a + 1] != m[a] + 1 for a in range(len(m) - 1))  # nothing merges
        assert c.problem.alpha == 1.0 and c.problem.beta == 1.0
    with pytest.raises(ValueError, match="volume must be at least 1 MiB"):
        ttb.build_benchmark(1000, "s", 1)
