"""Logical counters (mirrors counters.py:15-58 of the reference).

The reference increments its counters per batch (operator.py:227-245); the
B200 plan computes the same algorithmic totals once at plan creation
(``tmf_plan_info.flops_alg`` = the reference counter formula) and
adds them per apply.
"""

from __future__ import annotations

from collections import defaultdict


class FlopCounters:
    def __init__(self):
        self.values = defaultdict(int)

    def reset(self) -> None:
        self.values.clear()

    def add(self, name: str, amount: int) -> None:
        self.values[name] += int(amount)

    def __getitem__(self, name: str) -> int:
        return int(self.values.get(name, 0))

    @property
    def total_flops(self) -> int:
        return self["total_flops_alg"]

    def as_dict(self) -> dict:
        return dict(self.values)
