"""GPU parity: the sm_100a engine against the CPU oracle and the reference's
golden outputs (needs a B200; run with -m gpu).

Bar: bit-exact bytes of the WHOLE B buffer (padding included, as the
reference's own tests compare, support.hpp:93-96) for every kind pair, every
alpha/beta, every kernel variant the planner offers.  Full-size BASELINE
configs are checked by u64 checksum against the reference's output
(tests/golden/config_checksums.json, produced by the reference itself).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_02297_b200 as ttb  # noqa: E402
from paper_1603_02297_b200.workloads import ALL, CONFIGS  # noqa: E402
from golden_util import case_inputs, load_config_checksums, load_small_cases  # noqa: E402
from oracle import COMPONENTS, SCALAR, kind_id  # noqa: E402
from problems import b_sizes, random_problem  # noqa: E402

PAIRS = [("s", "s"), ("d", "d"), ("c", "c"), ("z", "z"), ("s", "d"), ("d", "s"), ("c", "z"),
         ("z", "c")]


def _dev(x: np.ndarray):
    return torch.from_numpy(x.copy()).cuda()


def run_gpu(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, B, plan_text=None):
    p = ttb.make_problem(perm, sizes, ka, kb, alpha, beta, lda, ldb)
    dA, dB = _dev(A), _dev(B)
    if plan_text is None:
        ttb.reference_transpose(
            p, ttb.TensorBuffer(ka, A.size // COMPONENTS[kind_id(ka)], tensor=dA),
            ttb.TensorBuffer(kb, B.size // COMPONENTS[kind_id(kb)], tensor=dB))
    else:
        plan = ttb.GpuPlan(p, cache=False)
        plan.select(plan_text)
        plan.execute(dA, dB)
    torch.cuda.synchronize()
    return dB.cpu().numpy()


def all_plans(ka, kb, perm, sizes, lda, ldb, alpha, beta):
    p = ttb.make_problem(perm, sizes, ka, kb, alpha, beta, lda, ldb)
    return ttb.GpuPlan(p, cache=False).candidates()


def test_golden_small_cases_every_variant(coracle):
    """Reference outputs (tests/golden) reproduced bit for bit by every plan."""
    meta, arrays = load_small_cases()
    n_plans = 0
    for case in meta:
        A, B = case_inputs(coracle, case, arrays)
        want = arrays[f"out{case['id']}"]
        args = (case["kind_a"], case["kind_b"], case["perm"], case["sizes"], case["lda"],
                case["ldb"])
        got = run_gpu(*args, case["alpha"], A, case["beta"], B)
        assert got.tobytes() == want.tobytes(), case
        for text in all_plans(*args, case["alpha"], case["beta"]):
            got = run_gpu(*args, case["alpha"], A, case["beta"], B, plan_text=text)
            assert got.tobytes() == want.tobytes(), (case, text)
            n_plans += 1
    assert n_plans > len(meta)


def _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, beta):
    na = coracle.required_elements_a(sizes, lda)
    nb = coracle.required_elements_b(perm, sizes, ldb)
    A = np.zeros(na * COMPONENTS[kind_id(ka)], SCALAR[kind_id(ka)])
    B = np.zeros(nb * COMPONENTS[kind_id(kb)], SCALAR[kind_id(kb)])
    coracle.fill_sentinel(ka, A)
    coracle.fill_sentinel(kb, B)
    coracle.fill_uniform(ka, sizes, lda, int(rng.integers(1 << 30)), A)
    if beta != 0.0:
        coracle.fill_uniform(kb, b_sizes(perm, sizes), ldb, int(rng.integers(1 << 30)), B)
    return A, B


@pytest.mark.parametrize("ka,kb", PAIRS)
def test_random_problems_every_variant(coracle, ka, kb):
    rng = np.random.default_rng(kind_id(ka) * 10 + kind_id(kb))
    for t in range(24):
        big = t % 3 == 0
        perm, sizes, lda, ldb = random_problem(rng, 4 if big else 6, allow_padding=(t % 2 == 0),
                                               allow_ones=not big, lo=(9 if big else None),
                                               hi=(70 if big else None))
        alpha, beta = [(1.0, 0.0), (1.3, 0.0), (0.7, 1.1), (2.0, 3.0)][t % 4]
        A, B = _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, beta)
        want = B.copy()
        coracle.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want)
        for text in [None] + all_plans(ka, kb, perm, sizes, lda, ldb, alpha, beta):
            got = run_gpu(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, B, plan_text=text)
            assert got.tobytes() == want.tobytes(), (perm, sizes, lda, ldb, alpha, beta, text)


def test_device_generator_and_checksum_match_oracle(coracle):
    for kind in "sdcz":
        sizes, ld = [7, 5, 3], [9, 5, 4]
        n = 9 * 5 * 4
        h = np.zeros(n * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
        coracle.fill_sentinel(kind, h)
        coracle.fill_uniform(kind, sizes, ld, 77, h, origin=[1, 2, 3], global_sizes=[10, 9, 8])
        d = torch.from_numpy(np.zeros_like(h)).cuda()
        ttb.fill_sentinel(kind, n, d.data_ptr())
        ttb.fill_uniform(kind, sizes, ld, 77, d.data_ptr(), origin=[1, 2, 3],
                         global_sizes=[10, 9, 8])
        torch.cuda.synchronize()
        assert d.cpu().numpy().tobytes() == h.tobytes()
        assert ttb.checksum(kind, sizes, ld, d.data_ptr(), origin=[1, 2, 3],
                            global_sizes=[10, 9, 8]) == \
            coracle.checksum(kind, sizes, ld, h, origin=[1, 2, 3], global_sizes=[10, 9, 8])


def _full_size(w, plan_text=None, autotune=False):
    p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                         w.lda and list(w.lda), w.ldb and list(w.ldb))
    na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
    a = ttb.TensorBuffer(w.kind, na)
    b = ttb.TensorBuffer(w.kind, nb)
    ttb.fill_sentinel(w.kind, na, a.data_ptr())
    ttb.fill_sentinel(w.kind, nb, b.data_ptr())
    ttb.fill_uniform(w.kind, list(w.sizes), w.lda and list(w.lda), w.seed_a, a.data_ptr())
    if w.beta != 0.0:
        ttb.fill_uniform(w.kind, w.sizes_b, w.ldb and list(w.ldb), w.seed_b, b.data_ptr())
    plan = ttb.GpuPlan(p, cache=False)
    if plan_text:
        plan.select(plan_text)
    if autotune:
        plan.autotune(a, b)   # beta != 0 tunes on scratch; beta == 0 leaves one application
    else:
        plan.execute(a, b)
    ck = ttb.checksum(w.kind, w.sizes_b, w.ldb and list(w.ldb), b.data_ptr())
    return ck, plan


@pytest.mark.parametrize("w", CONFIGS, ids=[w.name for w in CONFIGS])
def test_baseline_configs_match_reference_checksums(w):
    golden = load_config_checksums()
    ck, plan = _full_size(w)
    assert ck == golden[w.name], plan.describe()
    for text in plan.candidates()[:6]:
        ck, _ = _full_size(w, plan_text=text)
        assert ck == golden[w.name], text
    ck, plan = _full_size(w, autotune=True)
    assert ck == golden[w.name], plan.describe()


@pytest.mark.slow
def test_sweep_rows_match_reference_checksums():
    golden = load_config_checksums()
    for w in ALL[len(CONFIGS):]:
        ck, plan = _full_size(w)
        assert ck == golden[w.name], (w.name, plan.describe())
        torch.cuda.empty_cache()


@pytest.mark.parametrize("kind", ["s", "d", "c"])
def test_vector_tile_shapes(coracle, kind):
    """vtile_kernel (vector cp.async rows / vector column stores): shapes whose
    strides admit vectors on one or both sides, ragged tile edges (partial
    zero-filled chunks, element-wise column tails), padding, every mode; every
    candidate plan is run and at least one of them must be a vector tile."""
    rng = np.random.default_rng(40 + kind_id(kind))
    cases = [
        ([2, 1], [64, 48], None, None),
        ([2, 1], [84, 36], None, None),
        ([2, 1], [130, 70], None, None),            # partial chunks and column tails
        ([2, 1], [37, 44], [40, 44], [44, 40]),     # padded, odd extent
        ([3, 1, 2], [20, 12, 9], None, None),
        ([2, 3, 1], [36, 5, 10], None, None),
        ([5, 2, 4, 1, 3], [10, 8, 3, 36, 2], None, None),
        ([4, 3, 1, 2], [12, 9, 4, 14], [12, 10, 4, 14], [4, 15, 9, 12]),
        # odd extents: rows / columns at arbitrary offsets (shifted tiles, vec=2)
        ([2, 1], [37, 45], None, None),
        ([3, 1, 2], [19, 21, 7], None, None),
        ([2, 3, 1], [35, 3, 33], None, None),
        ([2, 1], [41, 29], [43, 29], [30, 41]),
        ([3, 2, 1], [7, 9, 11], None, None),
    ]
    seen = 0
    for perm, sizes, lda, ldb in cases:
        for alpha, beta in [(1.0, 0.0), (1.5, 0.0), (0.5, -2.0)]:
            A, B = _inputs(coracle, rng, kind, kind, perm, sizes, lda, ldb, beta)
            want = B.copy()
            coracle.transpose(kind, kind, perm, sizes, lda, ldb, alpha, A, beta, want)
            p = ttb.make_problem(perm, sizes, kind, kind, alpha, beta, lda, ldb)
            for text in all_plans(kind, kind, perm, sizes, lda, ldb, alpha, beta):
                plan = ttb.GpuPlan(p, cache=False)
                plan.select(text)
                seen += plan.describe().endswith("fn=vtile")
                got = run_gpu(kind, kind, perm, sizes, lda, ldb, alpha, A, beta, B, plan_text=text)
                assert got.tobytes() == want.tobytes(), (perm, sizes, alpha, beta, text)
            # explicit vector tiles (tile sides that are multiples of the vector width)
            for tx, ty, vec in [(16, 12, 1), (20, 8, 1), (32, 32, 1), (12, 36, 1), (16, 12, 2),
                                (32, 8, 2), (8, 32, 2), (64, 64, 2)]:
                bp = int(beta != 0) if (tx + ty) % 3 else 0
                text = f"kern=smem;kx=1;ky=1;tx={tx};ty={ty};order=0;occ=0;st=2;bp={bp};vec={vec}"
                plan = ttb.GpuPlan(p, cache=False)
                try:
                    plan.select(text)
                except ValueError:
                    continue
                seen += plan.describe().endswith("fn=vtile")
                got = run_gpu(kind, kind, perm, sizes, lda, ldb, alpha, A, beta, B, plan_text=text)
                assert got.tobytes() == want.tobytes(), (perm, sizes, alpha, beta, text)
    assert seen > 0


def test_edge_cases(coracle):
    rng = np.random.default_rng(3)
    cases = [
        ([1], [1009], None, None),                # rank 1 (executor.cpp:354-355)
        ([1], [1], None, None),                   # single element
        ([2, 1, 3], [1, 1, 1], None, None),       # all ones
        ([1, 2, 3], [3, 4, 5], None, None),       # identity -> rank-1 copy
        ([2, 1], [1, 7], None, None),             # size-1 dims
        ([3, 1, 2], [37, 5, 6], [40, 5, 7], [5, 8, 37]),  # padded (test_executor.cpp:129-149)
        ([1, 3, 2], [8, 6, 5], [9, 6, 5], [8, 5, 7]),     # padded case 1
        ([2, 1], [1009, 7], None, None),          # primes
        ([2, 1], [7, 1009], None, None),
        ([6, 5, 4, 3, 2, 1], [3, 2, 5, 2, 3, 4], None, None),
    ]
    for (perm, sizes, lda, ldb) in cases:
        for ka, kb in PAIRS:
            for alpha, beta in [(1.0, 0.0), (2.5, 0.0), (2.0, 3.0), (0.0, 1.0)]:
                A, B = _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, beta)
                want = B.copy()
                coracle.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want)
                got = run_gpu(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, B)
                assert got.tobytes() == want.tobytes(), (perm, sizes, ka, kb, alpha, beta)
                if alpha == 0.0 and beta == 1.0:
                    assert got.tobytes() == B.tobytes()


def test_beta_zero_never_reads_b(coracle):
    """B full of NaN must not leak into a beta == 0 result (executor.hpp:33-40)."""
    rng = np.random.default_rng(4)
    for perm, sizes in [([2, 1], [300, 200]), ([1, 3, 2], [64, 9, 70]), ([3, 2, 1], [4, 96, 40])]:
        for text in all_plans("s", "s", perm, sizes, None, None, 1.3, 0.0):
            A, B = _inputs(coracle, rng, "s", "s", perm, sizes, None, None, 0.0)
            B[:] = np.nan
            want = np.zeros_like(B)
            coracle.transpose("s", "s", perm, sizes, None, None, 1.3, A, 0.0, want)
            got = run_gpu("s", "s", perm, sizes, None, None, 1.3, A, 0.0, B, plan_text=text)
            assert got.tobytes() == want.tobytes(), text


def test_misaligned_buffers_take_the_fallback(coracle):
    rng = np.random.default_rng(5)
    perm, sizes = [2, 1], [64, 48]
    p = ttb.make_problem(perm, sizes, "s", "s", 1.0, 0.0)
    A, B = _inputs(coracle, rng, "s", "s", perm, sizes, None, None, 0.0)
    want = B.copy()
    coracle.transpose("s", "s", perm, sizes, None, None, 1.0, A, 0.0, want)
    dA = torch.zeros(A.size + 1, dtype=torch.float32, device="cuda")
    dB = torch.zeros(B.size + 1, dtype=torch.float32, device="cuda")
    dA[1:] = torch.from_numpy(A).cuda()
    dB[1:] = torch.from_numpy(B).cuda()
    plan = ttb.GpuPlan(p, cache=False)
    plan.execute(dA.data_ptr() + 4, dB.data_ptr() + 4)  # 4-byte aligned, not 16
    torch.cuda.synchronize()
    assert dB[1:].cpu().numpy().tobytes() == want.tobytes()


def test_buffer_errors_match_reference_messages():
    p = ttb.make_problem([2, 1], [8, 8])
    a, b = ttb.make_buffer_a(p), ttb.make_buffer_b(p)
    with pytest.raises(ValueError, match="A buffer: element kind mismatch"):
        ttb.reference_transpose(p, ttb.TensorBuffer("d", 64), b)
    with pytest.raises(ValueError, match="A buffer: too small for problem"):
        ttb.reference_transpose(p, ttb.TensorBuffer("s", 63), b)
    with pytest.raises(ValueError, match="B buffer: too small for problem"):
        ttb.reference_transpose(p, a, ttb.TensorBuffer("s", 63))
    with pytest.raises(ValueError, match="perm: not a permutation of 1..2"):
        ttb.reference_transpose(ttb.make_problem([1, 1], [8, 8]), a, b)


def test_sharded_execution_equals_single_call(coracle):
    """1 rank vs P ranks: executing every rank's boxes gives the same bytes."""
    rng = np.random.default_rng(6)
    for perm, sizes, kind, beta in [([3, 1, 2], [30, 7, 9], "s", 0.0),
                                    ([2, 4, 3, 6, 1, 5], [6, 4, 3, 9, 2, 5], "d", 0.5),
                                    ([2, 1], [101, 37], "c", 0.0)]:
        p = ttb.make_problem(perm, sizes, kind, kind, 1.0, beta)
        A, B = _inputs(coracle, rng, kind, kind, perm, sizes, None, None, beta)
        want = B.copy()
        coracle.transpose(kind, kind, perm, sizes, None, None, 1.0, A, beta, want)
        sa = ttb.element_strides_a(p)
        sbA = ttb.element_strides_b_for_a(p)
        esz = ttb.ElementKind.from_code(kind).bytes
        for world in (2, 3, 8):
            dA, dB = _dev(A), _dev(B)
            for r in range(world):
                for origin, ext in ttb.shard_boxes(p, world, r):
                    q = ttb.make_problem(perm, ext, kind, kind, 1.0, beta, p.lda, p.ldb)
                    offa = sum(o * s for o, s in zip(origin, sa)) * esz
                    offb = sum(o * s for o, s in zip(origin, sbA)) * esz
                    ttb.GpuPlan(q).execute(dA.data_ptr() + offa, dB.data_ptr() + offb)
            torch.cuda.synchronize()
            assert dB.cpu().numpy().tobytes() == want.tobytes(), (perm, world)


def test_host_end_to_end_path(coracle):
    rng = np.random.default_rng(8)
    for perm, sizes, lda, ldb, beta in [([2, 1], [300, 200], None, None, 0.0),
                                        ([3, 1, 2], [37, 5, 6], [40, 5, 7], [5, 8, 37], 0.0),
                                        ([2, 3, 1], [33, 20, 7], None, None, 1.5)]:
        A, B = _inputs(coracle, rng, "d", "d", perm, sizes, lda, ldb, beta)
        want = B.copy()
        coracle.transpose("d", "d", perm, sizes, lda, ldb, 0.5, A, beta, want)
        plan = ttb.GpuPlan(ttb.make_problem(perm, sizes, "d", "d", 0.5, beta, lda, ldb))
        got = B.copy()
        plan.execute_host(A, got)
        assert got.tobytes() == want.tobytes()


def test_host_pinned_overlapped_path(coracle, monkeypatch):
    """Pinned host buffers take the slab pipeline (H2D of slab i+1 overlapping
    the kernel and the D2H of slab i); the thresholds are lowered so these
    small problems cut into several slabs, padded rows and clipped tails
    included.  The second pass per problem reuses the slab plans."""
    monkeypatch.setenv("TTB_HOST_MIN_SLAB_KB", "1")
    monkeypatch.setenv("TTB_HOST_MIN_ROW", "4")
    rng = np.random.default_rng(9)
    for kind, perm, sizes, lda, ldb, beta in [
            ("d", [2, 1], [300, 200], None, None, 0.0),
            ("s", [3, 1, 2], [37, 50, 61], [40, 50, 70], [50, 80, 37], 0.0),
            ("c", [2, 3, 1], [33, 20, 70], None, None, 1.5),
            ("s", [1, 2], [1000, 77], [1003, 77], None, 0.0),
            ("z", [4, 3, 2, 1], [9, 10, 11, 120], None, None, -1.0),
            ("d", [2, 1, 3], [31, 17, 9], [33, 17, 9], [19, 31, 10], 0.0),
            ("s", [1, 3, 2], [8, 60, 50], [9, 60, 50], [8, 55, 61], 2.0)]:
        A, B = _inputs(coracle, rng, kind, kind, perm, sizes, lda, ldb, beta)
        want = B.copy()
        coracle.transpose(kind, kind, perm, sizes, lda, ldb, 0.5, A, beta, want)
        plan = ttb.GpuPlan(ttb.make_problem(perm, sizes, kind, kind, 0.5, beta, lda, ldb))
        ha = torch.from_numpy(A.view(np.uint8).copy()).pin_memory()
        hb = torch.from_numpy(B.view(np.uint8).copy()).pin_memory()
        for _ in range(2):  # the second pass reuses the chunk plans
            hb.copy_(torch.from_numpy(B.view(np.uint8).copy()))
            plan.execute_host(ha, hb)
            assert hb.numpy().tobytes() == want.tobytes(), (kind, perm, sizes)


def test_host_async_calls_overlap_across_plans(coracle, monkeypatch):
    """execute_host(wait=False) / host_sync (ttb_plan_execute_host_async): several
    plans in flight at once on pinned buffers, each output bit-exact after its
    own sync; a second call on a plan whose first is still in flight waits for
    it (one set of staging buffers per plan)."""
    monkeypatch.setenv("TTB_HOST_MIN_SLAB_KB", "1")
    monkeypatch.setenv("TTB_HOST_MIN_ROW", "4")
    rng = np.random.default_rng(19)
    jobs = []
    for kind, perm, sizes, lda, ldb, beta in [
            ("d", [2, 1], [300, 200], None, None, 0.0),
            ("s", [3, 1, 2], [37, 50, 61], [40, 50, 70], [50, 80, 37], 0.0),
            ("c", [2, 3, 1], [33, 20, 70], None, None, 1.5),
            ("s", [1, 3, 2], [8, 60, 50], [9, 60, 50], [8, 55, 61], 2.0)]:
        A, B = _inputs(coracle, rng, kind, kind, perm, sizes, lda, ldb, beta)
        want = B.copy()
        coracle.transpose(kind, kind, perm, sizes, lda, ldb, 0.5, A, beta, want)
        plan = ttb.GpuPlan(ttb.make_problem(perm, sizes, kind, kind, 0.5, beta, lda, ldb))
        ha = torch.from_numpy(A.view(np.uint8).copy()).pin_memory()
        hb = torch.from_numpy(B.view(np.uint8).copy()).pin_memory()
        jobs.append((plan, ha, hb, B, want))
    for rep in range(2):
        for plan, ha, hb, B, _ in jobs:
            hb.copy_(torch.from_numpy(B.view(np.uint8).copy()))
        for plan, ha, hb, _, _ in jobs:
            plan.execute_host(ha, hb, wait=False)
        for plan, ha, hb, _, want in jobs:
            plan.host_sync()
            assert hb.numpy().tobytes() == want.tobytes(), rep
    # back-to-back calls on ONE plan: the second waits for the first
    plan, ha, hb, B, want = jobs[2]  # beta != 0: a second application on the first result would differ
    hb2 = torch.from_numpy(B.view(np.uint8).copy()).pin_memory()
    hb.copy_(torch.from_numpy(B.view(np.uint8).copy()))
    plan.execute_host(ha, hb, wait=False)
    plan.execute_host(ha, hb2, wait=False)
    plan.host_sync()
    assert hb.numpy().tobytes() == want.tobytes()
    assert hb2.numpy().tobytes() == want.tobytes()


def test_kernels_actually_launch():
    before = ttb.launch_count()
    p = ttb.make_problem([2, 1], [64, 64])
    a, b = ttb.make_buffer_a(p), ttb.make_buffer_b(p)
    ttb.reference_transpose(p, a, b)
    torch.cuda.synchronize()
    assert ttb.launch_count() == before + 1


def test_tune_cached_miss_then_hit(tmp_path, coracle):
    """pipeline.cpp:102-185: first call autotunes and appends the winner under
    (canonical key, hardware key); the second call is a hit that selects it;
    a stale entry (plan that no longer applies) is re-tuned.  Output exact."""
    rng = np.random.default_rng(77)
    perm, sizes = [3, 1, 2], [40, 33, 20]
    A, B = _inputs(coracle, rng, "s", "s", perm, sizes, None, None, 0.5)
    want = B.copy()
    coracle.transpose("s", "s", perm, sizes, None, None, 1.0, A, 0.5, want)
    p = ttb.make_problem(perm, sizes, "s", "s", 1.0, 0.5)
    f = tmp_path / "solutions.tsv"
    hw = ttb.hardware_key()
    assert "sm100" in hw and "sms:ttb" in hw
    for expect_hit in (False, True):
        dA, dB = _dev(A), _dev(B)
        plan = ttb.GpuPlan(p, cache=False)
        assert plan.tune_cached(dA, dB, f) is expect_hit
        torch.cuda.synchronize()
        assert dB.cpu().numpy().tobytes() == want.tobytes()
        e = ttb.SolutionCache(f).lookup(ttb.canonical_key(p), hw)
        assert e is not None and e.plan.startswith("kern=") and e.bandwidth_gibs > 0
        assert plan.describe().startswith(e.plan)
    assert len(f.read_text().splitlines()) == 1
    # a later line whose plan is not a GPU plan is malformed for this reader:
    # it does not shadow the valid entry (still a hit, nothing appended)
    ttb.SolutionCache(f).store(ttb.SolutionEntry(ttb.canonical_key(p), hw, "kern=bogus", 1.0))
    dA, dB = _dev(A), _dev(B)
    assert ttb.GpuPlan(p, cache=False).tune_cached(dA, dB, f) is True
    torch.cuda.synchronize()
    assert dB.cpu().numpy().tobytes() == want.tobytes()
    assert len(f.read_text().splitlines()) == 2
    # a GPU plan that parses but does not apply to the problem is stale: re-tune, append
    ttb.SolutionCache(f).store(ttb.SolutionEntry(ttb.canonical_key(p), hw,
                                                 "kern=copy;v=4;kx=0;ky=0;tx=1;ty=1;order=0;occ=0", 1.0))
    dA, dB = _dev(A), _dev(B)
    assert ttb.GpuPlan(p, cache=False).tune_cached(dA, dB, f) is False
    torch.cuda.synchronize()
    assert dB.cpu().numpy().tobytes() == want.tobytes()
    assert len(f.read_text().splitlines()) == 4


def test_large_rank1_copy_every_copy_variant():
    """An identity permutation merges to rank 1 (executor.cpp:354-355, run_copy_1d):
    a 1.15 GB fp32 copy whose vector count exceeds the short-row kernel's 32-bit
    group index runs on the long-row kernel, every segment alignment bit-exact."""
    import torch
    sizes = [1 << 14, 17500]
    p = ttb.make_problem([1, 2], sizes, "s", "s", 1.0, 0.0)
    n = sizes[0] * sizes[1]
    a = ttb.TensorBuffer("s", n)
    b = ttb.TensorBuffer("s", n)
    ttb.fill_uniform("s", sizes, None, 77, a.data_ptr())
    plan = ttb.GpuPlan(p, cache=False)
    texts = plan.candidates()
    assert any("order=2" in t for t in texts) and any("order=4" in t for t in texts)
    for t in texts:
        b.tensor.zero_()
        plan.select(t)
        plan.execute(a, b)
        torch.cuda.synchronize()
        assert torch.equal(a.tensor, b.tensor), t


@pytest.mark.parametrize("ka,perm,sizes,alpha,beta", [
    ("s", [2, 1], [1000, 1200], 1.3, 0.0),          # fp32 128x128 bulk tiles (big warp roles)
    ("d", [2, 1], [520, 700], 0.7, 1.1),            # fp64 64x64 bulk tiles with the B ring
    ("c", [3, 2, 1], [4, 300, 260], 1.0, 0.0),      # c4-like, complex64
    ("s", [1, 3, 2], [49, 300, 70], 1.0, 0.5),      # c5_t10-like: shared lead S = 49
    ("s", [5, 2, 4, 1, 3], [10, 64, 6, 36, 5], 1.0, 0.5),  # c5_t18-like: column-permuted walk (xp)
    ("sd", [2, 1], [1000, 700], 1.3, 0.0),          # mixed kinds on the bulk tiles (s -> d)
    ("ds", [3, 1, 2], [75, 40, 130], 0.7, 1.1),     # d -> s with the B ring
    ("cz", [3, 2, 1], [5, 300, 130], 1.0, 0.5),     # c -> z, X group of two axes
    ("zc", [2, 1], [300, 170], 2.0, 0.0),
])
def test_medium_problems_every_variant(coracle, ka, perm, sizes, alpha, beta):
    """Tiles of 32-64 KB only exist on problems of a few hundred per side: every
    candidate of these (incl. the big bulk tiles, and the mixed kind pairs on
    them) bit-exact against the oracle."""
    ka, kb = (ka[0], ka[1]) if len(ka) == 2 else (ka, ka)
    rng = np.random.default_rng(sum(sizes))
    A, B = _inputs(coracle, rng, ka, kb, perm, sizes, None, None, beta)
    want = B.copy()
    coracle.transpose(ka, kb, perm, sizes, None, None, alpha, A, beta, want)
    texts = all_plans(ka, kb, perm, sizes, None, None, alpha, beta)
    assert any("vec=3" in t or "vec=4" in t for t in texts)
    for text in texts:
        got = run_gpu(ka, kb, perm, sizes, None, None, alpha, A, beta, B, plan_text=text)
        assert got.tobytes() == want.tobytes(), text
