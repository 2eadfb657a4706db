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


# (name, additions) per stage in application order: A1 8, A2 4 (+3 free
# negations), A3 2 (+1), P 0 (fast.py:130-168)
STAGE_COSTS = (("A1", 8), ("A2", 4), ("A3", 2), ("P", 0))


def count_operations() -> OpCount:
    """14 additions, 0 multiplications, 0 shifts (paper Table 1)."""
    return OpCount(additions=sum(c for _, c in STAGE_COSTS))


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
