"""Multi-rank path on the CPU (torch.distributed, gloo, world size 2).

The GPU path shards B's outer index space across ranks (ttb_shard_boxes) with
no collective on the data path; ranks only exchange verification checksums
and timings.  Here each rank computes its boxes with the CPU oracle on the
global-index data, checksums its slab with its global origin, and the
checksums are all-gathered: their sum must equal the checksum of the whole
single-rank result -- the same composition bench.py uses with NCCL.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

PROBLEMS = [
    ("s", (1, 0), (37, 29)),
    ("d", (2, 0, 1), (6, 9, 5)),
    ("s", (4, 0, 2, 1, 5, 3), (6, 4, 3, 9, 2, 5)),   # c5 t=15 shape class: B outer extent 9
    ("c", (2, 1, 0), (4, 16, 12)),
    ("d", (0, 3, 2, 1), (7, 5, 3, 6)),               # shared stride-1 index
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scatter(gather):
    m = [0] * len(gather)
    for k, a in enumerate(gather):
        m[a] = k + 1
    return m


def _worker(rank, world, port, results):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import paper_1603_02297_b200 as ttb
    from oracle import COMPONENTS, SCALAR, COracle, kind_id

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    co = COracle()
    ok = True
    for kind, gather, sizes in PROBLEMS:
        perm = _scatter(gather)
        p = ttb.make_problem(perm, list(sizes), kind, kind, 0.5, 0.0)
        k = kind_id(kind)
        n = int(np.prod(sizes))
        sb = ttb.sizes_b(p)
        A = np.zeros(n * COMPONENTS[k], SCALAR[k])
        co.fill_uniform(kind, list(sizes), None, 42, A)
        B = np.zeros(n * COMPONENTS[k], SCALAR[k])
        sa, sbA = ttb.element_strides_a(p), ttb.element_strides_b_for_a(p)
        C = COMPONENTS[k]
        local = 0
        for origin, ext in ttb.shard_boxes(p, world, rank):
            offa = sum(o * s for o, s in zip(origin, sa)) * C
            offb = sum(o * s for o, s in zip(origin, sbA)) * C
            Ab, Bb = A[offa:].copy(), B[offb:].copy()
            co.transpose(kind, kind, perm, ext, list(sizes), sb, 0.5, Ab, 0.0, Bb)
            ext_b = [ext[a] for a in sorted(range(len(ext)), key=lambda a: perm[a])]
            org_b = [origin[a] for a in sorted(range(len(ext)), key=lambda a: perm[a])]
            local += co.checksum(kind, ext_b, sb, Bb, origin=org_b, global_sizes=sb)
        gathered = [None] * world
        dist.all_gather_object(gathered, local % (1 << 64))
        whole = np.zeros_like(B)
        co.transpose(kind, kind, perm, list(sizes), None, None, 0.5, A, 0.0, whole)
        want = co.checksum(kind, sb, None, whole)
        ok = ok and (sum(gathered) % (1 << 64) == want)
        # the timing reduction the bench uses (max over ranks)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = ok and t.item() == float(world)
    results[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_checksums_compose_over_gloo(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert dict(results) == {r: True for r in range(world)}
