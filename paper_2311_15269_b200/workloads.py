"""Named search workloads C1..C5 (BASELINE.json `configs`).

Each entry is a deterministic placement plus the ``search`` arguments it is
quoted with.  C4b and C5 are spelled out explicitly so no RNG is involved.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

from .placement import BlockSpec, CostModel, COST_PRESETS, PlacementSpec, make_shape

# C5: kshape D=16 time costs by stage id (a0..a7, c0..c7, X, Xb, ab7..ab0,
# cb7..cb0); backward = 2 x mirrored forward.  SURVEY.md §8(d).
C5_TIMES = [2, 2, 1, 2, 3, 2, 2, 2, 2, 2, 3, 1, 3, 1, 2, 1,
            1, 2, 4, 4, 4, 6, 4, 2, 4, 4, 2, 4, 2, 6, 2, 6, 4, 4]


def c4b_placement() -> PlacementSpec:
    """Forward-only nnshape D=8: E, e0..e7 (devices 7..0), g0..g7 (devices
    7..0), time 1, mem +1, chain deps."""
    d = 8
    blocks = [BlockSpec(0, "E", "forward", frozenset(range(d)), 1, 1)]
    for i in range(d):
        blocks.append(BlockSpec(1 + i, f"e{i}", "forward", frozenset([d - 1 - i]), 1, 1))
    for i in range(d):
        blocks.append(BlockSpec(1 + d + i, f"g{i}", "forward", frozenset([d - 1 - i]), 1, 1))
    base = make_shape("nnshape", d)
    deps = frozenset((i, i + 1) for i in range(len(blocks) - 1))
    return PlacementSpec(d, base.mem_capacity, tuple(blocks), deps)


def c5_placement() -> PlacementSpec:
    base = make_shape("kshape", 16, COST_PRESETS["recompute"])
    blocks = tuple(replace(b, time_cost=C5_TIMES[b.stage_id]) for b in base.blocks)
    return PlacementSpec(base.num_devices, base.mem_capacity, blocks, base.deps)


@dataclass(frozen=True)
class Workload:
    name: str
    mem_capacity: Optional[int]
    max_nr: Optional[int]
    note: str

    def placement(self) -> PlacementSpec:
        return _PLACEMENTS[self.name.split("@")[0]]()


_PLACEMENTS = {
    "C1": lambda: make_shape("vshape", 4, CostModel(1, 1, 1, -1), mem_capacity=4),
    "C2": lambda: make_shape("xshape", 8, CostModel(1, 2, 1, -1)),
    "C3": lambda: make_shape("mshape", 8, COST_PRESETS["recompute"]),
    "C4a": lambda: make_shape("nnshape", 8, COST_PRESETS["recompute"]),
    "C4b": c4b_placement,
    "C5": c5_placement,
}

WORKLOADS = {
    "C1": Workload("C1", 4, 4, "vshape D=4 unit fwd/bwd, cap 4"),
    "C2@3": Workload("C2@3", None, 3, "xshape D=8 1:2, max_nr=3"),
    "C2@4": Workload("C2@4", None, 4, "xshape D=8 1:2, max_nr=4 (parity; CPU 156 s)"),
    "C2@5": Workload("C2@5", None, 5, "xshape D=8 1:2, max_nr=5 (GPU throughput)"),
    "C2@6": Workload("C2@6", None, 6, "xshape D=8 1:2, max_nr=6 (GPU throughput)"),
    "C2@8": Workload("C2@8", None, 8, "xshape D=8 1:2, 8 micro-batches (BASELINE configs[1])"),
    "C3@9": Workload("C3@9", 9, None, "mshape D=8 recompute, cap 9 (inflight limit 3)"),
    "C3@12": Workload("C3@12", 12, None, "mshape D=8 recompute, cap 12 (inflight limit 4)"),
    "C4a@3": Workload("C4a@3", None, 3, "nnshape D=8 recompute training, max_nr=3"),
    "C4a@4": Workload("C4a@4", None, 4, "nnshape D=8 recompute training, max_nr=4"),
    "C4b": Workload("C4b", None, 8, "nnshape D=8 forward-only inference, max_nr=8"),
    "C5@2": Workload("C5@2", None, 2, "kshape D=16 heterogeneous, max_nr=2"),
    "C5@3": Workload("C5@3", None, 3, "kshape D=16 heterogeneous, max_nr=3"),
    "C5@4": Workload("C5@4", None, 4, "kshape D=16 heterogeneous, max_nr=4 (GPU only)"),
    "C5@5": Workload("C5@5", None, 5, "kshape D=16 heterogeneous, max_nr=5 (GPU only)"),
}
