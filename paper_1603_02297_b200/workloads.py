"""BASELINE.json workloads (configs c1-c4s and the 24-row c5 scaling sweep).

Permutations are written in the paper's GATHER form as BASELINE.json does
(B index k is A index gather[k]); ``Workload.perm`` converts to the
reference's 1-based scatter map (SURVEY.md s8 "Conventions").  Data seeds
follow BASELINE.json; the c5 manifest is the frozen table of SURVEY.md s8(d)
(generated once from seed 5 and hard-coded, as the survey instructs).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

KIND_BYTES = {"s": 4, "d": 8, "c": 8, "z": 16}


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str                      # element kind code s/d/c/z (same on A and B)
    gather: Tuple[int, ...]        # paper/BASELINE gather tuple, 0-based
    sizes: Tuple[int, ...]         # A index order
    alpha: float
    beta: float
    seed_a: int
    seed_b: int = 0
    lda: Optional[Tuple[int, ...]] = None   # A order
    ldb: Optional[Tuple[int, ...]] = None   # B order

    @property
    def perm(self) -> List[int]:
        m = [0] * len(self.gather)
        for k, a in enumerate(self.gather):
            m[a] = k + 1
        return m

    @property
    def sizes_b(self) -> List[int]:
        return [self.sizes[a] for a in self.gather]

    @property
    def elements(self) -> int:
        n = 1
        for s in self.sizes:
            n *= s
        return n

    @property
    def algorithmic_bytes(self) -> int:
        """bytes = N*bytes(A) + N*bytes(B) + [beta!=0]*N*bytes(B) (tuner.cpp:18-25)."""
        eb = KIND_BYTES[self.kind]
        return self.elements * eb * (3 if self.beta != 0.0 else 2)


CONFIGS: List[Workload] = [
    Workload("c1", "s", (1, 0), (7264, 7264), 1.0, 0.0, 0),
    Workload("c2a", "s", (2, 0, 3, 1), (96, 128, 72, 64), 1.3, 0.0, 1),
    Workload("c2b", "s", (0, 3, 2, 1), (96, 128, 72, 64), 1.3, 0.0, 1),
    Workload("c3", "d", (5, 2, 0, 4, 1, 3), (24, 20, 22, 18, 24, 16), 0.7, 1.1, 2, 3),
    Workload("c4", "c", (2, 1, 0), (4, 4096, 3072), 1.0, 0.0, 4),
    Workload("c4s", "c", (2, 1, 0), (4, 4096, 3072), 1.0, 0.0, 4,
             lda=(8, 4096, 3072), ldb=(3072, 4096, 8)),
]

# SURVEY.md s8(d) frozen c5 manifest: (t, dtype, beta, gather perm, sizes)
_C5 = [
    (0, "s", 0.0, (3, 2, 0, 4, 1), (79, 42, 11, 245, 45)),
    (1, "d", 0.0, (0, 2, 1), (902, 251, 883)),
    (2, "s", 0.5, (2, 1, 0, 3, 4, 5), (188, 6, 26, 128, 12, 9)),
    (3, "d", 0.5, (1, 0), (24414, 8192)),
    (4, "s", 0.0, (0, 1, 3, 2), (63, 289, 458, 48)),
    (5, "d", 0.0, (0, 2, 1), (1186, 208, 811)),
    (6, "s", 0.5, (3, 0, 4, 1, 2), (216, 18, 211, 21, 23)),
    (7, "d", 0.5, (1, 0), (26547, 7534)),
    (8, "s", 0.0, (4, 2, 1, 3, 0, 5), (14, 87, 9, 16, 22, 104)),
    (9, "d", 0.0, (3, 1, 2, 0), (26, 1016, 34, 223)),
    (10, "s", 0.5, (0, 3, 2, 1), (49, 307, 47, 566)),
    (11, "d", 0.5, (0, 4, 5, 3, 1, 2), (12, 60, 8, 45, 13, 59)),
    (12, "s", 0.0, (0, 4, 1, 5, 2, 3), (7, 36, 9, 106, 118, 14)),
    (13, "d", 0.0, (1, 2, 0), (443, 4965, 91)),
    (14, "s", 0.5, (2, 0, 1, 3), (508, 15, 197, 266)),
    (15, "d", 0.5, (4, 0, 2, 1, 5, 3), (54, 132, 89, 9, 2, 18)),
    (16, "s", 0.0, (3, 1, 0, 2), (167, 99, 39, 620)),
    (17, "d", 0.0, (1, 2, 0, 3), (111, 258, 81, 86)),
    (18, "s", 0.5, (4, 1, 2, 5, 3, 0), (10, 16, 31, 38, 36, 59)),
    (19, "d", 0.5, (0, 1, 2, 4, 3), (34, 90, 106, 60, 10)),
    (20, "s", 0.0, (2, 0, 5, 1, 4, 3), (11, 40, 76, 88, 20, 7)),
    (21, "d", 0.0, (2, 3, 1, 0, 4), (114, 41, 74, 5, 116)),
    (22, "s", 0.5, (1, 2, 3, 0), (283, 49, 542, 53)),
    (23, "d", 0.5, (3, 2, 1, 0), (124, 106, 417, 36)),
]

C5: List[Workload] = [
    Workload(f"c5_t{t:02d}", k, g, s, 1.0, b, 5000 + t, 6000 + t) for (t, k, b, g, s) in _C5
]

ALL: List[Workload] = CONFIGS + C5

# kernel-tuning probes (not BASELINE configs): the c5 t=0 permutation with
# sector-aligned and unaligned leading extents
PROBES: List[Workload] = [
    Workload("p_t00_a80", "s", (3, 2, 0, 4, 1), (80, 42, 11, 248, 44), 1.0, 0.0, 7000),
    Workload("p_t00_a79", "s", (3, 2, 0, 4, 1), (79, 42, 11, 245, 45), 1.0, 0.0, 7001),
    Workload("p_copy_a", "s", (0, 1), (1 << 15, 12288), 1.0, 0.0, 7002),
    # pure streaming copy (identity, merges to rank 1) and long-row transposes
    Workload("p_copy_1d", "d", (0, 1), (1 << 15, 6400), 1.0, 0.0, 7003),
    Workload("p_rows_d", "d", (0, 2, 1), (1024, 400, 500), 1.0, 0.0, 7004),
    Workload("p_rows_s", "s", (0, 2, 1), (2048, 400, 500), 1.0, 0.0, 7005),
    Workload("p_rows_s_b", "s", (0, 2, 1), (2048, 400, 500), 1.0, 0.5, 7006, 7007),
    Workload("p_2d_s_b", "s", (1, 0), (20480, 20480), 1.0, 0.5, 7008, 7009),
    # long-row copies: row length vs row count (c5_t19 is 600 rows of 2.6 MB)
    Workload("p_lrow_b", "d", (0, 2, 1), (324360, 60, 10), 1.0, 0.5, 7010, 7011),
    Workload("p_lrow_0", "d", (0, 2, 1), (324360, 60, 10), 1.0, 0.0, 7012),
    Workload("p_mrow_b", "d", (0, 2, 1), (8192, 160, 150), 1.0, 0.5, 7013, 7014),
    Workload("p_srow_b", "d", (0, 2, 1), (1024, 400, 475), 1.0, 0.5, 7015, 7016),
    # the suite's slowest case (d3_132_balanced, 200 MiB fp32, alpha = beta = 1):
    # case-1 rows of 375 floats (1500 bytes) at alternating 16-byte phases
    Workload("p_suite_d3_132", "s", (0, 2, 1), (375, 375, 373), 1.0, 1.0, 7017, 7018),
]

BY_NAME = {w.name: w for w in ALL + PROBES}
