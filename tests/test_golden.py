"""The C oracle reproduces the reference's golden outputs (CPU only).

Fixtures were produced by the reference itself (tests/golden/make_golden.py);
this is what pins the oracle on machines where the reference is absent.
"""
import pytest

from golden_util import case_inputs, load_merge_validate, load_small_cases


def test_oracle_reproduces_reference_outputs(coracle):
    meta, arrays = load_small_cases()
    assert len(meta) >= 90
    for case in meta:
        A, B = case_inputs(coracle, case, arrays)
        coracle.transpose(case["kind_a"], case["kind_b"], case["perm"], case["sizes"],
                          case["lda"], case["ldb"], case["alpha"], A, case["beta"], B)
        assert B.tobytes() == arrays[f"out{case['id']}"].tobytes(), case


def test_oracle_nest_reproduces_reference_outputs(coracle):
    meta, arrays = load_small_cases()
    for case in meta[::3]:
        A, B = case_inputs(coracle, case, arrays)
        coracle.reference_nest(case["kind_a"], case["kind_b"], case["perm"], case["sizes"],
                               case["lda"], case["ldb"], case["alpha"], A, case["beta"], B,
                               threads=3)
        assert B.tobytes() == arrays[f"out{case['id']}"].tobytes(), case


def test_oracle_merge_matches_golden(coracle):
    g = load_merge_validate()
    for m in g["merges"]:
        out = coracle.merge(m["perm"], m["sizes"], m["lda"], m["ldb"])
        want = m["out"]
        assert out[:4] == (want["perm"], want["sizes"], want["lda"], want["ldb"])
        assert [list(t) for t in out[4]] == want["trace"]


def test_oracle_validate_matches_golden(coracle):
    g = load_merge_validate()
    for v in g["invalid"]:
        assert coracle.validate(v["perm"], v["sizes"], v["lda"], v["ldb"], v["kind_a"],
                                v["kind_b"]) == v["message"]
