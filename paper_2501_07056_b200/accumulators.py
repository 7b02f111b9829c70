"""Accumulator selection knobs -- API mirror of the reference's `accumulators.py`.

Only the policy lives here (`AccumThresholds` :34-41, `select_accumulator`
:132-134, `merge_chunks_for_sort` :137-157); the accumulators themselves are
CUDA kernels in `csrc/`.  On the device the crossover decides, per fine chunk,
which summation association an output value gets:

* DENSE (chunk holds >= crossover elements): sequential in ascending k from
  +0.0, the association of the reference's dense accumulator
  (np.bincount / np.add.at, accumulators.py:88-95);
* SORT (fewer): x0 + pairwise(x1..x_{d-1}), the association of the
  reference's sort accumulator (np.add.reduceat, accumulators.py:129).

`merge_chunks_for_sort` regroups consecutive sort chunks; it never changes a
value (all contributions to a column live in one chunk), so the device does
not need it -- it is kept for API parity.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .errors import InputError


class Accum(enum.Enum):
    SORT = "sort"
    DENSE = "dense"


@dataclass(frozen=True)
class AccumThresholds:
    sort_dense_crossover: int = 256
    sort_sweet_spot: int = 32

    def __post_init__(self):
        if self.sort_sweet_spot > self.sort_dense_crossover:
            raise InputError("sort_sweet_spot must not exceed sort_dense_crossover")
        if self.sort_dense_crossover < 1:
            raise InputError("sort_dense_crossover must be >= 1")


def select_accumulator(n_elems: int, thresholds: AccumThresholds) -> Accum:
    return Accum.SORT if n_elems < thresholds.sort_dense_crossover else Accum.DENSE


def merge_chunks_for_sort(chunk_sizes, target: int) -> np.ndarray:
    """Greedy grouping of consecutive sort chunks toward ``target`` (ties close the group)."""
    sizes = [int(s) for s in chunk_sizes]
    bounds = [0]
    if not sizes:
        return np.asarray(bounds, dtype=np.int64)
    total = sizes[0]
    for i in range(1, len(sizes)):
        grown = total + sizes[i]
        if abs(grown - target) < abs(total - target):
            total = grown
        else:
            bounds.append(i)
            total = sizes[i]
    bounds.append(len(sizes))
    return np.asarray(bounds, dtype=np.int64)
