"""Product paths beyond the parity grid (needs a B200):

* problems whose footprint reaches 2^31 elements run as boxes below that
  size (api.cpp split_boxes), every box on the 32-bit kernels -- checked
  bit for bit against a torch fp32 reference of the same op (separate
  roundings, as executor.hpp:18-40) on an 8.6 GB tensor;
* the one-shot plan cache is re-entrant: host threads transposing while
  another thread autotunes (which drops the one-shot plans);
* btile's work-stealing counters: the same plan launched on several streams
  at once.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_02297_b200 as ttb  # noqa: E402


def _free_gb():
    free, _ = torch.cuda.mem_get_info()
    return free / 1e9


@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (0.7, 1.1)])
def test_oversized_2d_runs_as_boxes_bit_exact(alpha, beta):
    n = 46344                      # n*n = 2.148e9 elements > 2^31 (8.6 GB of fp32)
    if _free_gb() < 40:
        pytest.skip("needs ~35 GB of free device memory")
    p = ttb.make_problem([2, 1], [n, n], "s", "s", alpha, beta)
    plan = ttb.GpuPlan(p, cache=False)
    assert plan.launches() > 1 and "boxes=" in plan.describe()
    a = torch.empty(n * n, dtype=torch.float32, device="cuda")
    ttb.fill_uniform("s", [n, n], None, 11, a.data_ptr())
    b = torch.empty_like(a)
    if beta != 0.0:
        ttb.fill_uniform("s", [n, n], None, 12, b.data_ptr())
        want = a.view(n, n).t().mul(alpha).add_(b.view(n, n).mul(beta)).reshape(-1)
    else:
        b.fill_(float("nan"))      # beta == 0 never reads B
        want = a.view(n, n).t().contiguous().reshape(-1)
    plan.execute(a, b)
    torch.cuda.synchronize()
    assert torch.equal(b.view(torch.int32), want.view(torch.int32))
    del a, b, want
    torch.cuda.empty_cache()


def test_oversized_3d_every_first_box_candidate():
    """A 3D fp32 problem of 2.15e9 elements (case 2, X group of two axes):
    the box plans of each candidate the first box accepts, bit-exact."""
    s0, s1, s2 = 4, 1024, 524544      # 2.1487e9 elements
    if _free_gb() < 40:
        pytest.skip("needs ~35 GB of free device memory")
    p = ttb.make_problem([3, 2, 1], [s0, s1, s2], "s", "s", 1.0, 0.0)
    plan = ttb.GpuPlan(p, cache=False)
    assert plan.launches() > 1
    n = s0 * s1 * s2
    a = torch.empty(n, dtype=torch.float32, device="cuda")
    ttb.fill_uniform("s", [s0, s1, s2], None, 13, a.data_ptr())
    want = a.view(s2, s1, s0).permute(2, 1, 0).contiguous().reshape(-1)
    b = torch.empty_like(a)
    for text in plan.candidates()[:6]:
        try:
            plan.select(text)
        except ValueError:
            continue
        b.fill_(float("nan"))
        plan.execute(a, b)
        torch.cuda.synchronize()
        assert torch.equal(b.view(torch.int32), want.view(torch.int32)), text
    del a, b, want
    torch.cuda.empty_cache()


def test_plan_cache_reentrant_while_autotuning():
    """Two threads run the one-shot API (plans shared through the cache) while a
    third autotunes a cached plan of the same problem, which invalidates the
    one-shot plans; every output stays exact."""
    perm, sizes = [3, 1, 2], [96, 70, 130]
    p = ttb.make_problem(perm, sizes, "s", "s", 1.0, 0.0)
    n = int(np.prod(sizes))
    a = torch.rand(n, device="cuda")
    want = a.view(sizes[2], sizes[1], sizes[0]).permute(2, 0, 1).contiguous().reshape(-1)
    errors = []

    def worker():
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(60):
                    b = ttb.TensorBuffer("s", n)
                    ttb.reference_transpose(p, ttb.TensorBuffer("s", n, tensor=a), b, stream=s)
                    s.synchronize()
                    if not torch.equal(b.tensor, want):
                        errors.append("wrong output")
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    def tuner():
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(4):
                    plan = ttb.GpuPlan(p)          # cached: autotune drops the one-shot plans
                    b = ttb.TensorBuffer("s", n)
                    plan.autotune(ttb.TensorBuffer("s", n, tensor=a), b, warmups=0, reps=1, stream=s)
                    s.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=worker), threading.Thread(target=worker), threading.Thread(target=tuner)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:3]


def test_btile_plan_on_concurrent_streams():
    """The same work-stealing bulk tile plan launched on four streams at once
    (each launch takes its own counter slot): every output exact."""
    perm, sizes = [2, 1], [2000, 1800]
    p = ttb.make_problem(perm, sizes, "s", "s", 1.0, 0.0)
    plan = ttb.GpuPlan(p, cache=False)
    texts = [t for t in plan.candidates() if "vec=3" in t or "vec=4" in t]
    assert texts
    plan.select(texts[0])
    assert "btile" in plan.describe()
    n = sizes[0] * sizes[1]
    srcs = [torch.rand(n, device="cuda") for _ in range(4)]
    wants = [x.view(sizes[1], sizes[0]).t().contiguous().reshape(-1) for x in srcs]
    outs = [torch.empty(n, device="cuda") for _ in range(4)]
    streams = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize()
    for rep in range(20):
        for i in range(4):
            with torch.cuda.stream(streams[i]):
                plan.execute(srcs[i], outs[i], stream=streams[i])
    torch.cuda.synchronize()
    for o, w in zip(outs, wants):
        assert torch.equal(o, w)


def test_dynamic_smem_just_under_48k_plus_static_barriers():
    """A bulk tile whose ring takes 49,056 bytes of dynamic shared memory: with
    the kernel's static mbarriers that exceeds 48 KB, so the launcher must opt
    in (found by the sharded-execution test: 'invalid argument' at launch)."""
    q = ttb.make_problem([2, 1], [50, 37], "c", "c", 1.0, 0.0, [101, 37], [37, 101])
    plan = ttb.GpuPlan(q, cache=False)
    plan.select("kern=smem;kx=1;ky=1;tx=50;ty=37;order=0;occ=0;st=3;bp=1;vec=3")
    a = torch.rand(37 * 101 * 2, device="cuda")     # A[i1][i0][re/im], lda (101, 37)
    b = torch.zeros(50 * 37 * 2, device="cuda")       # B[i0][i1][re/im], ldb (37, 101)
    plan.execute(a, b)
    torch.cuda.synchronize()
    want = a.view(37, 101, 2)[:, :50].permute(1, 0, 2)
    assert torch.equal(b.view(50, 37, 2), want)


def test_every_plan_takes_the_fallback_on_misaligned_buffers():
    """Buffers at a 4-byte offset (element-aligned, not 16): every candidate --
    tensor-map tiles and bulk tiles with tensor-map sides included, whose maps
    need 16-byte aligned bases -- must fall back and stay exact (found when
    the sharded bench rows offset their sub-box pointers)."""
    for perm, sizes, beta in [([2, 1], [516, 130], 0.5), ([2, 1], [130, 516], 0.5),
                              ([3, 1, 2], [60, 20, 36], 0.0)]:
        n = int(np.prod(sizes))
        p = ttb.make_problem(perm, sizes, "s", "s", 1.0, beta)
        a = torch.rand(n + 1, device="cuda")
        b0 = torch.rand(n + 1, device="cuda")
        sb = [sizes[perm.index(k + 1)] for k in range(len(sizes))]
        at = a[1:].view(*reversed(sizes))
        want = at.permute(*[len(sizes) - 1 - perm.index(len(sizes) - k) for k in range(len(sizes))])
        want = want.contiguous().reshape(-1)
        if beta:
            want = want + beta * b0[1:]
        plan = ttb.GpuPlan(p, cache=False)
        texts = plan.candidates()
        assert any("kern=tma" in t or "ts=" in t for t in texts)
        for text in texts:
            plan.select(text)
            b = b0.clone()
            plan.execute(a.data_ptr() + 4, b.data_ptr() + 4)
            torch.cuda.synchronize()
            assert torch.equal(b[1:], want), (perm, sizes, text)
            assert b[0] == b0[0]
