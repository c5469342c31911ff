"""Generate the golden fixtures from the REFERENCE itself (run in the build
container, where /root/reference exists and oracle/_ref is built).

    python tests/golden/make_golden.py [--skip-configs]

Writes:
  small_cases.json / small_cases.npz  -- 96 small problems: inputs, reference
                                         reference_transpose outputs (bytes)
  merge_validate.json                 -- reference merge_indices results and
                                         validate messages
  benchmark_manifest.json             -- the reference's 57-case suite manifests
                                         (build_benchmark, benchmark.cpp:166-220)
  config_checksums.json               -- u64 checksums (oracle/ttb_oracle.c
                                         orc_checksum) of the reference's output
                                         for every BASELINE config at full size

Inputs come from the counter-based generator (orc_fill_uniform) so the GPU
tests can regenerate full-size inputs on the device and compare checksums
without the reference present.  Padding of A and B holds a NaN sentinel.
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

from oracle import COMPONENTS, SCALAR, COracle, RefOracle, RefSession, kind_id  # noqa: E402
from problems import b_sizes, random_problem  # noqa: E402
from paper_1603_02297_b200.workloads import ALL  # noqa: E402

PAIRS = [("s", "s"), ("d", "d"), ("c", "c"), ("z", "z"), ("s", "d"), ("d", "s"), ("c", "z"),
         ("z", "c")]
AB = [(1.0, 0.0), (2.0, 0.0), (1.3, 0.0), (0.7, 1.1), (2.0, 3.0), (0.5, 1.0), (0.0, 1.0),
      (1.0, 0.5)]


def make_inputs(co, ka, kb, perm, sizes, lda, ldb, seed_a, seed_b, beta):
    na = co.required_elements_a(sizes, lda)
    nb = co.required_elements_b(perm, sizes, ldb)
    A = np.zeros(na * COMPONENTS[kind_id(ka)], SCALAR[kind_id(ka)])
    B = np.zeros(nb * COMPONENTS[kind_id(kb)], SCALAR[kind_id(kb)])
    co.fill_sentinel(ka, A)
    co.fill_sentinel(kb, B)
    co.fill_uniform(ka, sizes, lda, seed_a, A)
    if beta != 0.0:
        co.fill_uniform(kb, b_sizes(perm, sizes), ldb, seed_b, B)
    return A, B


def small_cases(co, ref):
    rng = np.random.default_rng(1603)
    meta, arrays = [], {}
    shapes = []
    for t in range(72):
        shapes.append(random_problem(rng, 6, allow_padding=(t % 3 != 0), allow_ones=True))
    for t in range(24):  # larger extents, exercise tiles and remainders
        perm, sizes, lda, ldb = random_problem(rng, 3, allow_padding=(t % 2 == 0),
                                               allow_ones=False, lo=3, hi=33)
        shapes.append((perm, sizes, lda, ldb))
    for i, (perm, sizes, lda, ldb) in enumerate(shapes):
        ka, kb = PAIRS[i % len(PAIRS)]
        alpha, beta = AB[(i // len(PAIRS)) % len(AB)]
        A, B = make_inputs(co, ka, kb, perm, sizes, lda, ldb, 100 + i, 200 + i, beta)
        out = B.copy()
        ref.run(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, out, threads=1)
        meta.append(dict(id=i, kind_a=ka, kind_b=kb, perm=perm, sizes=sizes, lda=lda, ldb=ldb,
                         alpha=alpha, beta=beta, seed_a=100 + i, seed_b=200 + i,
                         sha_a=hashlib.sha256(A.tobytes()).hexdigest(),
                         sha_b=hashlib.sha256(B.tobytes()).hexdigest()))
        # inputs are regenerated from the seeds (make_inputs); only the
        # reference's output is stored, with input hashes to pin the generator
        arrays[f"out{i}"] = out
    # SPEC.md:242 known answer
    meta.append(dict(id=len(meta), kind_a="s", kind_b="s", perm=[2, 1], sizes=[2, 2], lda=None,
                     ldb=None, alpha=1.0, beta=0.0, seed_a=None, seed_b=None))
    j = len(meta) - 1
    arrays[f"a{j}"] = np.array([1, 2, 3, 4], np.float32)
    arrays[f"b{j}"] = np.zeros(4, np.float32)
    out = arrays[f"b{j}"].copy()
    ref.run("s", "s", [2, 1], [2, 2], None, None, 1.0, arrays[f"a{j}"], 0.0, out)
    arrays[f"out{j}"] = out
    assert out.tolist() == [1, 3, 2, 4]
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump(meta, f, indent=0)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    print(f"small cases: {len(meta)}")


def merge_validate(ref):
    rng = np.random.default_rng(4242)
    merges = []
    for t in range(200):
        perm, sizes, lda, ldb = random_problem(rng, 6, allow_padding=(t % 2 == 0))
        mp, ms, mla, mlb, trace = ref.merge(perm, sizes, lda, ldb)
        merges.append(dict(perm=perm, sizes=sizes, lda=lda, ldb=ldb,
                           out=dict(perm=mp, sizes=ms, lda=mla, ldb=mlb, trace=trace)))
    for w in ALL:  # the BASELINE configs themselves (none of c1-c4 merge)
        mp, ms, mla, mlb, trace = ref.merge(w.perm, list(w.sizes), w.lda and list(w.lda),
                                            w.ldb and list(w.ldb))
        merges.append(dict(name=w.name, perm=w.perm, sizes=list(w.sizes),
                           lda=w.lda and list(w.lda), ldb=w.ldb and list(w.ldb),
                           out=dict(perm=mp, sizes=ms, lda=mla, ldb=mlb, trace=trace)))
    invalid = [
        ([], [], None, None, "s", "s"), ([1, 1], [2, 2], None, None, "s", "s"),
        ([0, 1, 2], [2, 2, 2], None, None, "s", "s"), ([2, 1], [2], None, None, "s", "s"),
        ([2, 1], [2, 0], None, None, "s", "s"), ([2, 1], [4, 4], [3, 4], None, "s", "s"),
        ([2, 1], [4, 4], [4, 4], [4, 3], "s", "s"), ([2, 1], [4, 4], [4], None, "s", "s"),
        ([2, 1], [4, 4], None, [4, 4, 4], "s", "s"), ([2, 1], [4, 4], None, None, "d", "z"),
        ([2, 1], [4, 4], None, None, "s", "c"), ([2, 1], [1 << 40, 1 << 40], None, None, "s", "s"),
        ([3, 2, 1], [4, 4096, 3072], [8, 4096, 3072], [8, 4096, 3072], "c", "c"),
        ([2, 1], [8, 8], None, None, "s", "d"),
    ]
    msgs = [dict(perm=p, sizes=s, lda=la, ldb=lb, kind_a=ka, kind_b=kb,
                 message=ref.validate(p, s, la, lb, ka, kb)) for (p, s, la, lb, ka, kb) in invalid]
    keys = []
    for (p, s, la, lb, ka, kb, al, be) in [([2, 1], [4, 4], None, None, "s", "s", 1.0, 0.0),
                                           ([2, 1], [4, 4], None, None, "s", "d", 1.0, 0.5),
                                           ([3, 2, 1], [4, 4096, 3072], [8, 4096, 3072],
                                            [3072, 4096, 8], "c", "c", 1.0, 0.0)]:
        keys.append(dict(perm=p, sizes=s, lda=la, ldb=lb, kind_a=ka, kind_b=kb, alpha=al,
                         beta=be, key=ref.canonical_key(p, s, la, lb, ka, kb, al, be)))
    with open(os.path.join(HERE, "merge_validate.json"), "w") as f:
        json.dump(dict(merges=merges, invalid=msgs, keys=keys), f, indent=0)
    print(f"merges: {len(merges)}, invalid: {len(msgs)}")


def config_checksums(co, ref, threads):
    res = {}
    for w in ALL:
        t0 = time.time()
        sizes = list(w.sizes)
        lda = list(w.lda) if w.lda else None
        ldb = list(w.ldb) if w.ldb else None
        s = RefSession(ref, w.kind, w.kind, w.perm, sizes, lda, ldb, w.alpha, w.beta, merge=False)
        A, B = s.a(), s.b()
        co.fill_sentinel(w.kind, A)
        co.fill_sentinel(w.kind, B)
        co.fill_uniform(w.kind, sizes, lda, w.seed_a, A)
        if w.beta != 0.0:
            co.fill_uniform(w.kind, w.sizes_b, ldb, w.seed_b, B)
        sec = s.run(threads)
        ck = co.checksum(w.kind, w.sizes_b, ldb, B)
        res[w.name] = dict(checksum=str(ck), ref_seconds=sec, threads=threads)
        s.close()
        print(f"{w.name}: checksum {ck} reference_transpose {sec:.3f}s ({time.time()-t0:.1f}s)",
              flush=True)
    with open(os.path.join(HERE, "config_checksums.json"), "w") as f:
        json.dump(res, f, indent=1)


# the paper's suite at its default volume (200 MiB) and two
# more (kind, seed) points, as the reference's build_benchmark writes them
MANIFESTS = [(200 << 20, "s", 42), (200 << 20, "d", 42), (64 << 20, "c", 7)]


def benchmark_manifests(ref):
    out = {f"{v >> 20}MiB_{k}_{s}": ref.benchmark_manifest(v, k, s) for v, k, s in MANIFESTS}
    with open(os.path.join(HERE, "benchmark_manifest.json"), "w") as f:
        json.dump(out, f, indent=0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-configs", action="store_true")
    ap.add_argument("--only", choices=["manifest"], default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    co, ref = COracle(), RefOracle()
    benchmark_manifests(ref)
    if args.only == "manifest":
        return
    small_cases(co, ref)
    merge_validate(ref)
    if not args.skip_configs:
        config_checksums(co, ref, args.threads)


if __name__ == "__main__":
    main()
