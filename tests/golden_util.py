"""Load the reference-generated golden fixtures (tests/golden/)."""
import hashlib
import json
import os

import numpy as np

from oracle import COMPONENTS, SCALAR, kind_id
from problems import b_sizes

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_small_cases():
    with open(os.path.join(GOLDEN, "small_cases.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    return meta, arrays


def load_merge_validate():
    with open(os.path.join(GOLDEN, "merge_validate.json")) as f:
        return json.load(f)


def load_config_checksums():
    with open(os.path.join(GOLDEN, "config_checksums.json")) as f:
        return {k: int(v["checksum"]) for k, v in json.load(f).items()}


def case_inputs(coracle, case, arrays):
    """Regenerate a case's A and initial B exactly as make_golden.py did."""
    i = case["id"]
    if case["seed_a"] is None:
        return arrays[f"a{i}"].copy(), arrays[f"b{i}"].copy()
    ka, kb = case["kind_a"], case["kind_b"]
    perm, sizes, lda, ldb = case["perm"], case["sizes"], case["lda"], case["ldb"]
    na = coracle.required_elements_a(sizes, lda)
    nb = coracle.required_elements_b(perm, sizes, ldb)
    A = np.zeros(na * COMPONENTS[kind_id(ka)], SCALAR[kind_id(ka)])
    B = np.zeros(nb * COMPONENTS[kind_id(kb)], SCALAR[kind_id(kb)])
    coracle.fill_sentinel(ka, A)
    coracle.fill_sentinel(kb, B)
    coracle.fill_uniform(ka, sizes, lda, case["seed_a"], A)
    if case["beta"] != 0.0:
        coracle.fill_uniform(kb, b_sizes(perm, sizes), ldb, case["seed_b"], B)
    assert hashlib.sha256(A.tobytes()).hexdigest() == case["sha_a"]
    assert hashlib.sha256(B.tobytes()).hexdigest() == case["sha_b"]
    return A, B
