"""Island-model GA on B200 (mirror of hm/engine.py).

Control flow of the reference ``solve`` (hm/engine.py:170-243), with the
islands' inner loop (_run_island, hm/engine.py:138-167) running on the GPU:
one CUDA-graph launch per generation evolves and scores every island of a
device at once (libhubgpu ``hg_ga_*``).  Python keeps the outer loop so
Ctrl-C is honoured between rounds, exactly where the reference honours it.

Multi-GPU: pass ``group`` (a torch.distributed process group, one process
per GPU).  Islands are sharded contiguously by GLOBAL island index, the
streams are keyed by that index, and at each round barrier the per-rank
champion records {raw, island, hubs} are exchanged with one all_gather
(NCCL over NVLink on GPUs, gloo on CPU tests); every rank then picks the
minimum (raw, island), i.e. the reference's "first strict minimum in island
order" (hm/engine.py:216-220).  Results are identical for any GPU count.
"""

from __future__ import annotations

import enum
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .evaluation import FitnessMode, scale
from .model import Instance, Solution, initial_solution, nearest_allocation, nearest_allocations
from .rng import RngStream, derive_stream


class Role(enum.IntEnum):
    """Stream roles (hm/engine.py:40-45)."""

    POPULATION = 0
    CROSSOVER = 1
    MUTATION = 2


def resolve_rng(seed: int, island: int, role) -> RngStream:
    """derive_stream(seed, island, role) (hm/engine.py:48-54)."""
    return derive_stream(seed, island, int(role))


@dataclass(frozen=True)
class GaParams:
    """Search budget and seeding knobs (hm/engine.py:57-88)."""

    islands: int = 64
    pop_size: int = 64
    inner_iters: int = 50
    outer_iters: int = 10
    seed: int = 0
    perturb_strength: int | None = None
    strict_paper: bool = False
    # draw generator: "replay" = the reference's SplitMix64 streams (identical
    # trajectories); "philox" = Philox4x32-10 on the same stream keys and draw
    # accounting (an independent stream; not part of the reference API)
    rng: str = "replay"

    def __post_init__(self):
        for label in ("islands", "pop_size", "inner_iters", "outer_iters"):
            v = getattr(self, label)
            if v < 1:
                raise ValueError(f"{label} must be >= 1, got {v}")
        if self.pop_size % 2:
            raise ValueError(f"pop_size must be even for pairwise crossover, got {self.pop_size}")
        if self.rng not in ("replay", "philox"):
            raise ValueError(f"rng must be 'replay' or 'philox', got {self.rng!r}")
        if self.perturb_strength is not None and self.perturb_strength < 1:
            raise ValueError(f"perturb_strength must be >= 1, got {self.perturb_strength}")

    def resolved_strength(self, p: int) -> int:
        s = min(p, 3) if self.perturb_strength is None else self.perturb_strength
        if s > p:
            raise ValueError(f"perturb_strength {s} exceeds p={p}")
        return s


@dataclass(frozen=True)
class SolveReport:
    best_solution: Solution
    raw_objective: float
    scaled_fitness: float
    trace: tuple
    evaluations: int
    wall_time: float
    interrupted: bool = False


def island_shard(islands: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of global island ids owned by `rank`."""
    return islands * rank // world, islands * (rank + 1) // world


_ga_lock = threading.Lock()


class DeviceIslands:
    """Islands [lo, hi) of one run on this process's GPU."""

    def __init__(self, inst: Instance, params: GaParams, strength: int, lo: int, hi: int):
        self.inst = inst
        self.params = params
        self.lo, self.hi = lo, hi
        # one hg_ga per (instance, islands, shard, shape): a later solve() with
        # the same shape reseeds it instead of allocating and capturing anew.
        # A GA is checked out of the cache for the solve (close() returns it),
        # so concurrent solves on one shared Instance never share one
        dinst = inst.device()
        self._cache = dinst.__dict__.setdefault("_ga_cache", {})
        self._key = (params.islands, lo, hi, params.pop_size, strength, params.strict_paper,
                     params.rng, _lib.exact_default())
        with _ga_lock:
            free = self._cache.get(self._key)
            ga = free.pop() if free else None
        if ga is None:
            ga = _lib.DeviceGa(dinst, params.islands, lo, hi, params.pop_size, strength,
                               params.strict_paper, params.seed, params.rng)
        else:
            ga.reseed(params.seed)
        self.ga = ga

    def close(self) -> None:
        """Return the GA object to the instance's cache."""
        ga, self.ga = self.ga, None
        if ga is not None:
            with _ga_lock:
                self._cache.setdefault(self._key, []).append(ga)

    def run_round(self, ancestor_hubs: np.ndarray, audit=None):
        """One outer round: N1 generations from the ancestor.  Returns the
        per-island results (raw[n_local], hubs[n_local, p])."""
        ga = self.ga
        ga.begin_round(ancestor_hubs)
        if audit is None:
            ga.generations(self.params.inner_iters)
        else:
            kids = []
            for _ in range(self.params.inner_iters):
                ga.generations(1)
                kids.append(ga.last_children()[0])
            self._replay_audit(kids, audit)
        return ga.round_results()

    def _replay_audit(self, kids, audit):
        # the reference evaluates island by island (workers=1): island-major,
        # then generation, then child order
        pop = self.params.pop_size
        gens = np.stack(kids)  # [N1, n_local*pop, p]
        nloc = self.hi - self.lo
        order = gens.reshape(len(kids), nloc, pop, -1).transpose(1, 0, 2, 3).reshape(-1, gens.shape[-1])
        allocs = nearest_allocations(self.inst, order)
        for hubs, alloc in zip(order, allocs):
            hub = np.zeros(self.inst.n, dtype=bool)
            hub[hubs] = True
            audit(Solution(hub=hub, alloc=alloc))


def _first_min(raw: np.ndarray) -> int:
    # np.argmin returns the first minimum: the reference's strict '<' scan
    return int(np.argmin(raw))


def exchange_champion(raw: float, island: int, hubs: np.ndarray, group):
    """All-gather one champion record per rank and return the global winner
    (min raw, ties to the lowest island)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rec = np.concatenate([[raw, float(island)], np.asarray(hubs, dtype=np.float64)])
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cpu")
    mine = torch.from_numpy(rec).to(dev)
    every = torch.empty(world * rec.size, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(every, mine, group=group)
    recs = every.cpu().numpy().reshape(world, rec.size)
    k = np.lexsort((recs[:, 1], recs[:, 0]))[0]
    return float(recs[k, 0]), int(recs[k, 1]), recs[k, 2:].astype(np.int64)


def _device_seed(inst: Instance):
    sol = initial_solution(inst)
    return sol, float(inst.device().evaluate(sol.hubs[None, :])[0, 3])


def _solve(inst: Instance, params: GaParams, mode: FitnessMode, audit, make_shard, group,
           seed_eval=_device_seed, finish=nearest_allocation):
    """The outer loop.  ``make_shard(inst, params, strength, lo, hi)`` builds the
    island runner for this rank's islands; ``seed_eval`` / ``finish`` score the
    seed ancestor and build the returned Solution (device versions by default;
    the multi-rank CPU tests substitute host test doubles)."""
    t0 = time.perf_counter()
    strength = params.resolved_strength(inst.p)

    seed_sol, seed_raw = seed_eval(inst)
    seed_hubs = seed_sol.hubs
    seed_scaled = scale(seed_raw, mode, inst.total_flow)
    if audit is not None:
        audit(seed_sol)
    inc = (seed_raw, seed_scaled, seed_hubs)
    best = inc

    if group is None:
        rank, world = 0, 1
    else:
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = island_shard(params.islands, rank, world)
    shard = make_shard(inst, params, strength, lo, hi) if hi > lo else None

    trace: list[float] = []
    evaluations = 0
    interrupted = False
    try:
        for _ in range(params.outer_iters):
            if shard is not None:
                raw, hubs = shard.run_round(inc[2], audit)
                k = _first_min(raw)
                c_raw, c_island, c_hubs = float(raw[k]), lo + k, hubs[k]
            else:
                c_raw, c_island, c_hubs = float("inf"), params.islands, np.zeros(inst.p, np.int64)
            if world > 1:
                c_raw, c_island, c_hubs = exchange_champion(c_raw, c_island, c_hubs, group)
            champion = (c_raw, scale(c_raw, mode, inst.total_flow), np.asarray(c_hubs))
            evaluations += params.islands * params.inner_iters * params.pop_size
            if params.strict_paper:
                inc = champion
                if champion[0] < best[0]:
                    best = champion
                trace.append(champion[1])
            else:
                if champion[0] < inc[0]:
                    inc = champion
                best = inc
                trace.append(inc[1])
    except KeyboardInterrupt:
        interrupted = True
    finally:
        if shard is not None and hasattr(shard, "close"):
            shard.close()

    return SolveReport(
        best_solution=finish(best[2], inst),
        raw_objective=best[0],
        scaled_fitness=best[1],
        trace=tuple(trace),
        evaluations=evaluations,
        wall_time=time.perf_counter() - t0,
        interrupted=interrupted,
    )


def solve(inst: Instance, params: GaParams, mode: FitnessMode = FitnessMode.RAW,
          workers: int | None = None, audit=None, *, group=None) -> SolveReport:
    """Run the island GA (hm/engine.py:170-243) on the GPU.

    ``workers`` is accepted for API compatibility and never changes the
    result (the reference's own guarantee).  ``audit`` receives every
    evaluated Solution, seed first, in the reference's serial order.
    ``group``: torch.distributed group to shard islands over (one rank per
    GPU); None runs every island on this process's device."""
    del workers
    return _solve(inst, params, mode, audit, DeviceIslands, group)
