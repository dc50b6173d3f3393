"""The BASELINE.json workloads (configs[0..4]) as concrete synthetic inputs.

Shapes, sizes and distributions follow SURVEY.md §8(d); the values that the
paper leaves open (mass/velocity ranges, Plummer bounds) are proposals
listed in DESIGN.md "Input recipe".
"""
from __future__ import annotations

from dataclasses import dataclass, field

ALL_OPS = ("sum", "min", "max", "avg")


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    dist: int              # 0 uniform (+ central body), 1 Plummer
    seed: int
    axes: tuple            # column names used as coordinate axes
    res: tuple
    lo: tuple
    hi: tuple
    attrs: tuple           # binned column names
    ops: tuple = ALL_OPS   # reductions applied to every attribute
    central: int = 1
    note: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "c1": Workload("c1_uniform_1k_32x32", 1000, 0, 1, ("x", "y"), (32, 32), (-1.0, -1.0), (1.0, 1.0),
                   ("mass",), note="configs[0]: 1,000 uniform, 32x32, count + sum/min/max/avg of mass"),
    "c2": Workload("c2_uniform_10M_256x256_4attr", 10_000_000, 0, 2, ("x", "y"), (256, 256),
                   (-1.0, -1.0), (1.0, 1.0), ("mass", "vx", "vy", "vz"),
                   note="configs[1]: 10M uniform, 256x256, mass/vx/vy/vz"),
    "c3": Workload("c3_plummer_100M_512x512", 100_000_000, 1, 3, ("x", "y"), (512, 512),
                   (-16.0, -16.0), (16.0, 16.0), ("mass",), central=0,
                   note="configs[2]: 100M Plummer, 512x512, count + sum/min/max/avg of mass, sharded 1/2/4/8"),
    "c4": Workload("c4_uniform_1B_256cube", 1_000_000_000, 0, 4, ("x", "y", "z"), (256, 256, 256),
                   (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), ("mass",),
                   note="configs[3]: 1B uniform, 256^3 (global-atomic path)"),
    "c5": Workload("c5_placement_50M_512x512", 50_000_000, 0, 5, ("x", "y"), (512, 512),
                   (-1.0, -1.0), (1.0, 1.0), ("mass",),
                   note="configs[4]: placement study, 50M uniform, 100 steps"),
}
