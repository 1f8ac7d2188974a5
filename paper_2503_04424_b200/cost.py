"""Closed-form cost model of the blocked symmetric factorisation (oocdet cost.py:1-137).

FMA counts are exact rationals and need n_b | m; transfer counts and scratch slots are the
reference schedule's (whole blocks).  The engine reports these as reference-equivalent
counters and uses `total_flops` (m^3/6 FMA = m^3/3 flops) as its algorithmic work."""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .errors import CostDomainError

CASES = ("generic", "symmetric")


def predicted_reads(n_b: int, case: str = "symmetric") -> int:
    n = n_b
    if case == "generic":
        return (2 * n ** 3 - 3 * n ** 2 + 4 * n) // 3
    return (2 * n ** 3 - 3 * n ** 2 + 7 * n) // 6


def predicted_writes(n_b: int, case: str = "symmetric") -> int:
    n = n_b
    if n <= 2:
        return 0
    if case == "generic":
        return (n ** 3 - 4 * n - 3) // 3
    return (n ** 3 + 3 * n ** 2 - 22 * n + 24) // 6


def scratch_slots(n_b: int, case: str = "symmetric") -> int:
    n = n_b
    if n <= 2:
        return 0
    if case == "generic":
        return n * n - n - 1
    return (n * n + n - 8) // 2


@dataclass(frozen=True)
class OpCost:
    count: Fraction
    flops_per_op: Fraction

    @property
    def total(self) -> Fraction:
        return self.count * self.flops_per_op


@dataclass(frozen=True)
class CostBreakdown:
    m: int
    n_b: int
    case: str
    decomposition: OpCost
    lower_solve: OpCost
    upper_solve: OpCost
    full_multiply: OpCost
    gramian_multiply: OpCost
    blocks_read: int
    blocks_written: int
    scratch_slots: int

    @property
    def total_flops(self) -> Fraction:
        return sum((o.total for o in (self.decomposition, self.lower_solve, self.upper_solve,
                                       self.full_multiply, self.gramian_multiply)), Fraction(0))


def predicted_cost(m: int, n_b: int, case: str = "symmetric") -> CostBreakdown:
    if case not in CASES:
        raise ValueError(f"case must be one of {CASES}, got {case!r}")
    if m < 1 or n_b < 1:
        raise ValueError(f"m and n_b must be >= 1, got m={m}, n_b={n_b}")
    if m % n_b:
        raise CostDomainError(f"cost model requires n_b | m; {n_b} does not divide {m}")
    n, b = Fraction(n_b), Fraction(m, n_b)
    tri = (n * n - n) / 2
    zero = OpCost(Fraction(0), Fraction(0))
    lower = OpCost(tri, (b ** 3 - b ** 2) / 2)
    if case == "generic":
        dec = OpCost(n, b ** 3 / 3 - b ** 2 / 2 + b / 6)
        upper, full, gram = lower, OpCost(n ** 3 / 3 - n ** 2 / 2 + n / 6, b ** 3), zero
    else:
        dec = OpCost(n, b ** 3 / 6 - b ** 2 / 4 + b / 12)
        upper, full, gram = zero, OpCost(n ** 3 / 6 - n ** 2 / 2 + n / 3, b ** 3), OpCost(tri, b ** 3 / 2)
    return CostBreakdown(m, n_b, case, dec, lower, upper, full, gram, predicted_reads(n_b, case),
                         predicted_writes(n_b, case), scratch_slots(n_b, case))


def logdet_flops(m: int) -> float:
    """The metric's algorithmic work: m^3/3 flops (2 x the m^3/6 FMA of a symmetric
    factorisation, BASELINE.json)."""
    return m ** 3 / 3.0
