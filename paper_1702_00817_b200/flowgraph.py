"""The 14-addition flow graph as a host-side API (reference fast.py:30-282).

On the GPU the same stages run inside every kernel (csrc/adct_device.cuh
fwd8/inv8).  This module keeps the reference's single-vector entry points and
its instrumented operation count for users of the reference API; they are
not on the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .transforms import stage_matrices

#: Largest |line value| in the flow graph for 8-bit input: 4 * 2 * 255 (fast.py:24-27).
EIGHT_BIT_PEAK = 2040


@dataclass(frozen=True)
class OpCount:
    additions: int = 0
    multiplications: int = 0
    shifts: int = 0

    @property
    def total(self) -> int:
        return self.additions + self.multiplications + self.shifts

    def __add__(self, other: "OpCount") -> "OpCount":
        return OpCount(self.additions + other.additions, self.multiplications + other.multiplications,
                       self.shifts + other.shifts)


def stage_costs() -> tuple[tuple[str, int], ...]:
    """(stage, additions) counted from the stage matrices themselves, the way
    the reference tallies its FactorStage steps (fast.py:50-126, 236-241): an
    output line that combines k > 1 inputs costs k - 1 additions; a copy, a
    negation (sign folded into a later add) or a permutation costs nothing.
    Entries are only 0/+-1, so there are no multiplications or shifts."""
    out = []
    for name, m in zip(("A1", "A2", "A3", "P"), stage_matrices()):
        assert set(np.unique(m).tolist()) <= {-1, 0, 1}
        out.append((name, int(sum(max(0, int(np.count_nonzero(row)) - 1) for row in m))))
    return tuple(out)


def count_operations() -> OpCount:
    """14 additions, 0 multiplications, 0 shifts (paper Table 1), tallied
    from the flow graph's stages (A1 8, A2 4, A3 2, P 0)."""
    return OpCount(additions=sum(c for _, c in stage_costs()))


def flow_intermediates(x: Sequence) -> list[list]:
    """Per-stage output vectors (fast.py:275-282)."""
    v = np.asarray(list(x))
    outs = []
    for m in stage_matrices():
        v = m @ v
        outs.append(v.tolist())
    return outs


def fast_forward(x: Sequence) -> tuple[np.ndarray, OpCount]:
    """T x through the four stages with the operation tally (fast.py:255-272)."""
    values = [v.item() if isinstance(v, np.generic) else v for v in x]
    if len(values) != 8:
        raise ValueError("expected an 8-vector")
    if not all(math.isfinite(v) for v in values):
        raise ValueError("input must be finite")
    eight_bit = all(0 <= v <= 255 for v in values)
    stages = flow_intermediates(values)
    if eight_bit:
        peak = max(abs(v) for st in stages for v in st)
        assert peak <= EIGHT_BIT_PEAK, f"flow-graph overflow: |{peak}| > {EIGHT_BIT_PEAK}"
    return np.asarray(stages[-1]), count_operations()
