"""Objective and fitness scalings (mirror of hm/evaluation.py).

collection   = chi   * sum_i O_i * C[i][a_i]
distribution = delta * sum_j D_j * C[j][a_j]       (node -> hub leg)
transfer     = alpha * sum_ij W_ij * C[a_i][a_j]

The three sums are computed on the GPU (K2 + K3 of libhubgpu); this module
keeps the reference's API, exceptions and scaling arithmetic.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .model import Instance, Solution, validate


class InfeasibleSolutionError(ValueError):
    """hm/evaluation.py:30-35"""

    def __init__(self, violations):
        super().__init__("infeasible solution: " + "; ".join(violations))
        self.violations = tuple(violations)


class ZeroTotalFlowError(ValueError):
    """hm/evaluation.py:38"""


class StatisticUndefinedError(ValueError):
    """hm/evaluation.py:42"""


class FitnessMode(enum.Enum):
    """hm/evaluation.py:46-63"""

    CAB_NORMALIZED = "cab"
    STANDARD_MILLI = "milli"
    RAW = "raw"

    @classmethod
    def from_string(cls, s: str) -> "FitnessMode":
        try:
            return cls(s.lower())
        except ValueError:
            raise ValueError(f"unknown fitness mode {s!r}; expected cab, milli or raw") from None


@dataclass(frozen=True)
class CostBreakdown:
    collection_cost: float
    transfer_cost: float
    distribution_cost: float
    raw_total: float
    scaled_fitness: float


def scale(raw_total: float, mode: FitnessMode, total_flow: float) -> float:
    """hm/evaluation.py:75-83 -- milli is raw * 1e-3 (exactly that product)."""
    if mode is FitnessMode.CAB_NORMALIZED:
        if total_flow == 0.0:
            raise ZeroTotalFlowError("flow-normalized fitness undefined: total flow is zero")
        return raw_total / total_flow
    if mode is FitnessMode.STANDARD_MILLI:
        return raw_total * 1e-3
    return raw_total


def objective(inst: Instance, sol: Solution, mode: FitnessMode = FitnessMode.RAW) -> CostBreakdown:
    """hm/evaluation.py:86-100: validate on the host, score on the GPU."""
    report = validate(sol, inst)
    if not report.ok:
        raise InfeasibleSolutionError(report.violations)
    coll, tran, dist, raw = (float(v) for v in
                             inst.device().evaluate(sol.hubs[None, :], sol.alloc[None, :])[0])
    return CostBreakdown(coll, tran, dist, raw, scale(raw, mode, inst.total_flow))


def fitness(inst: Instance, sol: Solution, mode: FitnessMode) -> float:
    return objective(inst, sol, mode).scaled_fitness


def evaluate_population(inst: Instance, hubs: np.ndarray, alloc: np.ndarray | None = None,
                        unique: bool = False) -> np.ndarray:
    """Batched objective: B sorted hub sets (B x p) -> B x 4 array of
    (collection, transfer, distribution, raw).  ``alloc=None`` scores the
    nearest allocation of each hub set (what the GA and _Evaluator.evaluate,
    hm/engine.py:116-129, score); otherwise ``alloc`` (B x n) must be a
    feasible allocation onto the given hubs (not re-validated here).
    ``unique=True`` (nearest allocation only) scores each distinct hub set
    once on the device and copies its row to every repeat -- the reference's
    memo (_Evaluator) for batches with many repeated sets."""
    hubs = np.asarray(hubs, dtype=np.int64)
    if hubs.ndim != 2 or hubs.shape[1] != inst.p:
        raise ValueError(f"hubs must be B x p={inst.p}, got {hubs.shape}")
    # range / order of every hub set (and alloc range) is validated on the
    # device by the C-ABI; a bad batch raises ValueError naming the first row
    return inst.device().evaluate(hubs, alloc, unique=unique)


def avg_interhub_distance(inst: Instance, sol: Solution) -> float:
    """Mean dist[k][l] over ordered hub pairs k != l (hm/evaluation.py:128-143);
    an analysis statistic, host side (p^2 values)."""
    report = validate(sol, inst)
    if not report.ok:
        raise InfeasibleSolutionError(report.violations)
    hubs = sol.hubs
    p = hubs.size
    if p < 2:
        raise StatisticUndefinedError("average inter-hub distance undefined for p = 1")
    return float(np.sum(inst.dist[np.ix_(hubs, hubs)])) / (p * (p - 1))
