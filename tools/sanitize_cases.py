"""Small launches of every kernel family for compute-sanitizer (one tool per
run, see tools/sanitize.sh): K1 scan/planes, K2 (fast and exact legs), K3-TC/P
(fixed-order on the triangular fold, full W, exact; one and several K chunks;
two byte planes), the fp64 K3, K4a-c and K5 through one GA generation, the
device generator, the restricted optimum and the unique-set path."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1704_06258_b200 as hg  # noqa: E402
from paper_1704_06258_b200 import _lib  # noqa: E402


def run() -> None:
    hg.set_device(0)
    cases = [
        hg.generate_urand(300, 10, 1704, (3.0, 0.75, 2.0), device=True),   # one chunk, tri
        hg.generate_urand(1100, 7, 5, (1.0, 0.75, 1.0), device=True),     # two K chunks
    ]
    # two byte planes (flows up to 300) and an asymmetric cost matrix (no fold)
    rng = np.random.default_rng(3)
    n = 200
    xy = rng.random((n, 2)) * 100
    dist = np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1))
    dist[0, 1] += 1.0  # asymmetric
    flow = rng.integers(0, 300, (n, n)).astype(np.float64)
    np.fill_diagonal(flow, 0.0)
    cases.append(hg.Instance(n, 6, dist, flow, 1.0, 0.75, 1.0))
    for inst in cases:
        pop = hg.random_population(inst.n, inst.p, 40, key=9)
        hg.evaluate_population(inst, pop)
        for exact in (True, False):
            hg.set_exact_sums(exact)
            hg.evaluate_population(inst, pop)
        hg.set_exact_sums(False)
        d = inst.device()
        d.set_fitness(_lib.FIT_FP64)
        hg.evaluate_population(inst, pop[:8])
        d.set_fitness(_lib.FIT_AUTO)
        hg.evaluate_population(inst, np.concatenate([pop[:8], pop[:8]]), unique=True)
        hg.solve(inst, hg.GaParams(islands=2, pop_size=8, inner_iters=2, outer_iters=1, seed=1))
    small = hg.generate_urand(12, 3, 1, (1.0, 0.75, 1.0))
    hg.restricted_optimum(small)
    print("sanitize cases done")


if __name__ == "__main__":
    run()
