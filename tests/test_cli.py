"""The `ttb` command-line front end (tools/ttb_cli.cpp): the reference CLI's
flags (cli.cpp:14-71) and exit codes (pipeline.cpp:189-200: 0 ok, 1 invalid
argument, 2 other error), its text / JSON report and CSV benchmark mode
(pipeline.cpp:102-185, benchmark.cpp:272-285).  Argument handling runs here;
the device runs are marked gpu."""
import csv
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1603_02297_b200", "_lib", "ttb")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="ttb CLI not built")


def run(*args, env=None):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, **(env or {})))
    return r.returncode, r.stdout, r.stderr


def test_help_and_usage_errors():
    rc, out, _ = run("--help")
    assert rc == 0 and out.startswith("usage: ttb --perm=")
    rc, _, err = run("--perm=2,1")
    assert rc == 1 and "--perm and --size are required" in err
    rc, _, err = run("--perm=2,1", "--size=3,4", "--dataType=q")
    assert rc == 1 and "dataType" in err
    rc, _, err = run("--perm=2,1", "--size=3,x")
    assert rc == 1 and "--size" in err
    rc, _, err = run("--perm", "2,1", "--size", "3,4", "--bogus=1")
    assert rc == 1 and "unknown option --bogus" in err


@pytest.mark.parametrize("args", [
    ("--perm=2,2", "--size=3,4"),
    ("--perm=2,1", "--size=3,0"),
    ("--perm=2,1", "--size=3,4", "--lda=2,4"),
    ("--perm=3,1,2", "--size=3,4,5", "--ldb=5,3,3"),
    ("--perm=2,1", "--size=3,4,5"),
])
def test_invalid_problems_exit_1_with_reference_message(refo, args):
    rc, _, err = run(*args)
    assert rc == 1
    kv = dict(a[2:].split("=", 1) for a in args)
    perm = [int(x) for x in kv["perm"].split(",")]
    sizes = [int(x) for x in kv["size"].split(",")]
    lda = [int(x) for x in kv["lda"].split(",")] if "lda" in kv else None
    ldb = [int(x) for x in kv["ldb"].split(",")] if "ldb" in kv else None
    assert err.strip() == "ttb: " + refo.validate(perm, sizes, lda, ldb)


def test_ignores_cpu_search_flags_until_the_device():
    rc, _, err = run("--perm=2,1", "--size=64,64", "--prefetchDistances=0,5", "--threads=4",
                     "--no-streaming-stores", "--blockings=16x16")
    assert "unknown option" not in err
    assert rc in (0, 2)  # 2 = no CUDA device in this container


@pytest.mark.gpu
def test_single_mode_miss_then_hit(tmp_path):
    cache = str(tmp_path / "c.tsv")
    args = ("--perm=3,1,2", "--size=96,80,70", "--dataType=d", "--alpha=0.5", "--beta=2",
            f"--cacheFile={cache}")
    rc, out, err = run(*args, "--json")
    assert rc == 0, err
    j = json.loads(out)
    assert j["cacheHit"] is False and j["measuredCandidates"] > 1
    assert j["problemKey"].startswith("perm=3,1,2;size=96,80,70;") and "sm100" in j["hardwareKey"]
    assert j["bandwidthGiBs"] > 0 and len(j["trialSeconds"]) == 3
    rc, out, err = run(*args)
    assert rc == 0, err
    lines = dict(l.split(": ", 1) for l in out.strip().splitlines())
    assert lines["cache"].startswith("hit") and lines["candidates measured"] == "0"
    assert lines["solution"].startswith(j["plan"]["serialized"].split(";fn=")[0])
    rc, out, _ = run(*args, env={"TTUNE_CACHE": cache})  # env default as the reference
    assert "cache: hit" in out
    # --emit: the solution's standalone kernel next to its header (pipeline.cpp:142-146)
    base = str(tmp_path / "out" / "k1")
    os.makedirs(os.path.dirname(base))
    rc, out, err = run(*args, f"--emit={base}", "--json")
    assert rc == 0, err
    j = json.loads(out)
    assert j["emitted"] == {"source": base + ".cu", "header": base + ".h"}
    src = open(base + ".cu").read()
    assert '#include "k1.h"' in src and "plan: " in src
    assert "void transpose_21_96x5600_dd(const double* A, double* B, double alpha, double beta);" \
        in open(base + ".h").read()


@pytest.mark.gpu
def test_benchmark_mode_csv_and_manifest(tmp_path):
    man = str(tmp_path / "m.txt")
    rc, out, err = run("--benchmark", "--volume=2", "--seed=3", f"--manifest={man}",
                       "--warmups=1", "--reps=1")
    assert rc == 0, err
    rows = list(csv.DictReader(io.StringIO(out)))
    assert len(rows) == 57
    assert list(rows[0]) == ["caseId", "dim", "perm", "sizes", "category", "config", "refGiBs",
                             "tunedGiBs", "speedup", "plan"]
    assert all(float(r["tunedGiBs"]) > 0 for r in rows)
    import paper_1603_02297_b200 as ttb
    want = [ttb.benchmark_case_line(c) for c in ttb.build_benchmark(2 << 20, "s", 3)]
    assert open(man).read().splitlines() == want
