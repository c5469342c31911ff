"""The multi-GPU data path of bench.py, rank by rank on one GPU: every c5 row
split over 2, 4 and 8 ranks (ttb_shard_boxes); each rank
allocates the bounding boxes of its A region and B slab, fills them from the
global-index generator, runs its boxes, and checksums its slab.  The sum of
the per-rank checksums must equal the reference's checksum of the whole row
(tests/golden/config_checksums.json) -- the same check bench.py makes after
gathering the checksums over NCCL.
"""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1603_02297_b200 as ttb  # noqa: E402
from paper_1603_02297_b200.workloads import C5  # noqa: E402


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bench_rows_per_rank_sum_to_reference_checksum(world):
    golden = bench.golden_checksums()
    for w in C5:
        total = 0
        elements = 0
        for rank in range(world):
            r = bench.Row(w, world, rank, torch, ttb)
            r.allocate()
            r.run()
            total = (total + r.checksum()) % (1 << 64)
            elements += r.elements
            r.free()
            torch.cuda.empty_cache()
        assert elements == w.elements, (w.name, world)
        assert total == golden[w.name], (w.name, world)
