"""The N>1 host path on CPU: world_size 2 over gloo.

The GPU island runner is replaced by a test double built from the oracle's
island loop (same streams keyed by global island id), so this checks the
sharding, the champion all_gather and the incumbent/trace logic of
``engine._solve`` -- and that 2 ranks reproduce the reference's result
(golden fixture) exactly, as 1 rank does.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden, orc, params_of, problem_from


class OracleShard:
    def __init__(self, pr, params, strength, lo, hi):
        self.pr = pr
        self.params = params
        self.strength = strength
        self.lo, self.hi = lo, hi
        self.streams = [orc.island_streams(params.seed, g) for g in range(lo, hi)]

    def run_round(self, ancestor_hubs, audit=None):
        anc = orc.indicator(ancestor_hubs, self.pr.n)
        raws, hubs = [], []
        for st in self.streams:
            (r, h), _ = orc.run_island(self.pr, st, anc, self.params.pop_size,
                                       self.params.inner_iters, self.strength,
                                       self.params.strict_paper,
                                       lambda hh: orc.raw_cost(self.pr, hh))
            raws.append(r)
            hubs.append(h)
        return np.array(raws), np.array(hubs)


def _run(label, group):
    import paper_1704_06258_b200 as hg
    from paper_1704_06258_b200 import engine

    g = golden("ga")
    pr = problem_from(g, label)
    inst = hg.Instance(pr.n, pr.p, pr.C, pr.W, pr.chi, pr.alpha, pr.delta)
    params = hg.GaParams(**params_of(g, label))
    mode = hg.FitnessMode.from_string(str(g[f"{label}_mode"]))

    def seed_eval(_inst):
        hubs = np.sort(pr.rank[:pr.p])
        sol = hg.Solution(hub=orc.indicator(hubs, pr.n), alloc=orc.nearest(pr.C, hubs))
        return sol, orc.raw_cost(pr, hubs)

    def finish(hubs, _inst):
        return hg.Solution(hub=orc.indicator(hubs, pr.n), alloc=orc.nearest(pr.C, hubs))

    rep = engine._solve(inst, params, mode, None,
                        lambda i, p_, s, lo, hi: OracleShard(pr, p_, s, lo, hi), group,
                        seed_eval=seed_eval, finish=finish)
    return rep, g


def _check(rep, g, label):
    assert np.array_equal(rep.best_solution.hubs, g[f"{label}_hubs"])
    assert [rep.raw_objective, rep.scaled_fitness] == g[f"{label}_raw"].tolist()
    assert list(rep.trace) == g[f"{label}_trace"].tolist()
    assert rep.evaluations == int(g[f"{label}_evals"][0])


def _worker(rank, world, port, labels, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for label in labels:
            rep, g = _run(label, dist.group.WORLD)
            _check(rep, g, label)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


LABELS = ["small", "strict", "asym", "mid", "midstrict"]


@pytest.mark.parametrize("label", LABELS)
def test_single_rank_host_loop_matches_reference(label):
    rep, g = _run(label, None)
    _check(rep, g, label)


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_reproduce_reference(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, LABELS, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(results) == [(r, "ok") for r in range(world)], results
