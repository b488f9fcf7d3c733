"""Exhaustive search over hub sets (mirror of hm/oracle.py:42-54).

restricted_optimum sweeps every p-subset of nodes under nearest allocation --
the search space the GA walks -- on the GPU: hub sets are unranked on the
device in itertools.combinations order, scored by K2+K3 in batches of 65,536
and reduced to the first strict minimum of raw (ties keep the
lexicographically smallest set, as the reference's strict '<' over its
ordered loop).  Nothing crosses the PCIe bus but the winner.
"""

from __future__ import annotations

from math import comb

from . import _lib
from .model import Instance, Solution, nearest_allocation

DEFAULT_LIMIT = 10_000_000


class EnumerationLimitError(ValueError):
    """hm/oracle.py:32-40 (same attributes and message)."""

    def __init__(self, required: int, limit: int):
        self.required = required
        self.limit = limit
        super().__init__(
            f"enumeration needs {required} candidates, over the limit of {limit}; "
            f"raise `limit` explicitly to allow it"
        )


def restricted_optimum(inst: Instance, limit: int = DEFAULT_LIMIT) -> tuple[Solution, float]:
    """Best solution whose allocation is nearest-hub, by full hub-set sweep."""
    count = comb(inst.n, inst.p)
    if count > limit:
        raise EnumerationLimitError(count, limit)
    hubs, raw, _ = _lib.restricted_optimum(inst.device(), limit)
    return nearest_allocation(hubs, inst), raw
