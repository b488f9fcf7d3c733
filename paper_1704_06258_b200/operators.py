"""GA operators, single-solution API (mirror of hm/operators.py).

The island GA never calls these: it runs the same operators batched on the
device (csrc/k_ga.cu).  These wrappers keep the reference's per-solution
API: draws come from the caller's stream on the host, in the reference's
order, and the mask work (splice, swap, correction) runs on the GPU.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .model import Instance, Solution, nearest_allocation
from .rng import RngStream, derive_stream  # noqa: F401  (re-exported like the reference)

__all__ = ["RngStream", "derive_stream", "crossover", "crossover_hub_arrays", "correction",
           "correct_hub_set", "mutation", "swap_random_hub_spoke", "perturb",
           "StructureMismatch"]


class StructureMismatch(ValueError):
    """Operator arguments do not structurally agree (hm/operators.py:37)."""


def crossover_hub_arrays(ha: np.ndarray, hb: np.ndarray, rng) -> tuple[np.ndarray, np.ndarray]:
    """Single cut at 1 + randint(n-1), tails exchanged; n == 1 copies with no
    draw (hm/operators.py:41-57).  The splice runs on the GPU."""
    ha = np.asarray(ha, dtype=bool)
    hb = np.asarray(hb, dtype=bool)
    n = ha.shape[0]
    if hb.shape[0] != n:
        raise StructureMismatch(f"parent lengths differ: {n} vs {hb.shape[0]}")
    if n == 1:
        return ha.copy(), hb.copy()
    cut = 1 + rng.randint(n - 1)
    c1, c2 = _lib.crossover_masks(ha[None, :], hb[None, :], np.array([cut]))
    return c1[0].astype(bool), c2[0].astype(bool)


def crossover(a: Solution, b: Solution, rng) -> tuple[np.ndarray, np.ndarray]:
    return crossover_hub_arrays(a.hub, b.hub, rng)


def correct_hub_set(raw_hub: np.ndarray, inst: Instance) -> np.ndarray:
    """Repair to exactly p hubs (hm/operators.py:69-101), on the GPU (K4c)."""
    raw_hub = np.asarray(raw_hub, dtype=bool)
    if raw_hub.shape != (inst.n,):
        raise StructureMismatch(f"hub array has length {raw_hub.shape[0]}, instance n={inst.n}")
    return inst.device().correct(raw_hub[None, :])[0]


def correct_hub_sets(masks: np.ndarray, inst: Instance) -> np.ndarray:
    """Batched correction: B x n masks -> B x p sorted hub sets."""
    masks = np.asarray(masks, dtype=bool)
    if masks.ndim != 2 or masks.shape[1] != inst.n:
        raise StructureMismatch(f"masks must be B x n={inst.n}, got {masks.shape}")
    return inst.device().correct(masks)


def correction(raw_hub: np.ndarray, inst: Instance, rng=None) -> Solution:
    """Deterministic repair + nearest allocation; `rng` is never consumed
    (hm/operators.py:104-110)."""
    return nearest_allocation(correct_hub_set(raw_hub, inst), inst)


def swap_random_hub_spoke(raw_hub: np.ndarray, rng) -> np.ndarray:
    """Close the randint(#open)-th open node, open the randint(#closed)-th
    closed node (list taken before closing); identity without draws on an
    all-open / all-closed mask (hm/operators.py:113-124)."""
    raw_hub = np.asarray(raw_hub, dtype=bool)
    n = raw_hub.shape[0]
    on = int(raw_hub.sum())
    if on == 0 or on == n:
        return raw_hub.copy()
    r_close = rng.randint(on)
    r_open = rng.randint(n - on)
    out = _lib.swap_masks(raw_hub[None, :], np.array([r_close]), np.array([r_open]))
    return out[0].astype(bool)


def mutation(sol: Solution, inst: Instance, rng) -> Solution:
    new_hub = swap_random_hub_spoke(np.asarray(sol.hub, dtype=bool), rng)
    return nearest_allocation(np.flatnonzero(new_hub), inst)


def perturb(ancestor: Solution, inst: Instance, rng, strength: int) -> Solution:
    """`strength` swaps then one allocation (hm/operators.py:134-146)."""
    if not 1 <= strength <= inst.p:
        raise ValueError(f"perturbation strength {strength} outside [1, p={inst.p}]")
    hub = np.asarray(ancestor.hub, dtype=bool)
    for _ in range(strength):
        hub = swap_random_hub_spoke(hub, rng)
    return nearest_allocation(np.flatnonzero(hub), inst)
