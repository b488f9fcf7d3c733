"""CPU oracle for the p-hub-median GA hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  The shipped package
(``paper_1704_06258_b200``) must not import anything from here.

It restates, in numpy, the algorithm of the reference package ``hubmedian``
0.1.0 (``/root/reference/pkg/src/hubmedian``, abbreviated ``hm/`` below) for
the path BASELINE.json's north star names: score a population (nearest-hub
allocation + closed-form objective) and evolve it (island GA with
crossover / swap mutation / correction / perturbation), plus the
SplitMix64 streams and the synthetic instance generator that feed it.

Bit-level choices follow the reference wherever they decide bits:
* sums use ``np.sum`` over the same arrays (numpy pairwise summation) and
  the flow aggregation uses an index-ordered weighted ``np.bincount``
  (hm/evaluation.py:109-119);
* argmin ties resolve to the first (lowest) hub (hm/model.py:205);
* every draw is computed *by index* on the counter-based SplitMix64
  stream, ``mix64(state + k*gamma)`` (hm/rng.py:84-89), which is how the
  CUDA kernels replay it.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this module
against ``tests/golden/*.npz``, produced by running the real reference in
the build container (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# SplitMix64 (hm/rng.py:43-48, 58-99, 102-107)
# ---------------------------------------------------------------------------

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB
TWO_M53 = 2.0 ** -53


def mix64(z: int) -> int:
    """SplitMix64 finaliser (hm/rng.py:43-48)."""
    z &= M64
    z ^= z >> 30
    z = (z * _C1) & M64
    z ^= z >> 27
    z = (z * _C2) & M64
    return z ^ (z >> 31)


def mix64_vec(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, *keys: int) -> int:
    """Starting state of ``derive_stream(seed, *keys)`` (hm/rng.py:102-107)."""
    s = mix64(seed)
    for k in keys:
        s = mix64(s ^ mix64(k + GOLDEN))
    return s


def draw_u64(state: int, k: int) -> int:
    """k-th output (1-based) of a stream whose state is ``state``."""
    return mix64((state + k * GOLDEN) & M64)


def u64_to_unit(x: int) -> float:
    return float(x >> 11) * TWO_M53


def unit_to_below(u: float, bound: int) -> int:
    # hm/rng.py:76 -- int(random() * bound)
    return int(u * bound)


class Stream:
    """Counter view of a SplitMix64 stream: ``taken`` draws consumed so far."""

    __slots__ = ("state", "taken")

    def __init__(self, state: int, taken: int = 0):
        self.state = state & M64
        self.taken = taken

    def u64(self) -> int:
        self.taken += 1
        return draw_u64(self.state, self.taken)

    def unit(self) -> float:
        return u64_to_unit(self.u64())

    def below(self, bound: int) -> int:
        if bound <= 0:
            raise ValueError("bound must be positive")
        return unit_to_below(self.unit(), bound)

    def u64_block(self, count: int) -> np.ndarray:
        ks = np.arange(self.taken + 1, self.taken + count + 1, dtype=np.uint64)
        self.taken += count
        return mix64_vec(np.uint64(self.state) + np.uint64(GOLDEN) * ks)

    def unit_block(self, count: int) -> np.ndarray:
        return (self.u64_block(count) >> np.uint64(11)).astype(np.float64) * TWO_M53

    def below_block(self, count: int, bound: int) -> np.ndarray:
        return (self.unit_block(count) * bound).astype(np.int64)

    # The reference's method names, so reference-style test helpers
    # (ScriptedRng-like callers) can drive the oracle operators.
    randint = below
    random = unit


# ---------------------------------------------------------------------------
# Problem data (hm/model.py:33-105) and the generator (hm/io.py:143-210)
# ---------------------------------------------------------------------------


@dataclass
class Problem:
    n: int
    p: int
    C: np.ndarray          # dist, fp64 n x n, C[i][k] = unit cost i -> k
    W: np.ndarray          # flow, fp64 n x n
    chi: float
    alpha: float
    delta: float
    O: np.ndarray = field(init=False)
    D: np.ndarray = field(init=False)
    total: float = field(init=False)
    rank: np.ndarray = field(init=False)

    def __post_init__(self):
        self.C = np.ascontiguousarray(self.C, dtype=np.float64)
        self.W = np.ascontiguousarray(self.W, dtype=np.float64)
        self.O = self.W.sum(axis=1)             # hm/model.py:79
        self.D = self.W.sum(axis=0)             # hm/model.py:80
        self.total = float(self.W.sum())        # hm/model.py:81
        # hm/model.py:103 -- stable sort of distance-row sums
        self.rank = np.argsort(self.C.sum(axis=1), kind="stable")


def euclid(xy: np.ndarray) -> np.ndarray:
    """hm/io.py:143-147 (separate subtract / multiply / add / sqrt)."""
    x = xy[:, 0]
    y = xy[:, 1]
    ddx = x[:, None] - x[None, :]
    ddy = y[:, None] - y[None, :]
    return np.sqrt(ddx * ddx + ddy * ddy)


def urand_problem(n: int, p: int, seed: int, factors) -> Problem:
    """hm/io.py:188-210: 2n uniforms for coordinates (x0 y0 x1 y1 ...) scaled
    by 1e5, then n*n bounded draws in [0, 100] row-major, diagonal zeroed."""
    st = Stream(stream_key(seed, n, p))
    xy = st.unit_block(2 * n).reshape(n, 2) * 100000.0
    W = st.below_block(n * n, 101).astype(np.float64).reshape(n, n)
    W[np.arange(n), np.arange(n)] = 0.0
    chi, alpha, delta = factors
    return Problem(n, p, euclid(xy), W, chi, alpha, delta)


def stream_problem(seed: int, n: int, p: int, *, chi=1.0, alpha=0.75, delta=1.0,
                   symmetric=True, self_flow=False) -> Problem:
    """Instance built straight from a stream, the recipe of the reference's
    test helper (hm tests conftest.py:18-32): n*n uniforms*100 for dist
    (symmetrised by D + D^T when asked, zero diagonal), then n*n bounded
    draws in [0, 100] for flow (diagonal zeroed unless self_flow)."""
    st = Stream(stream_key(seed, 0xBEEF))
    C = np.array([[st.unit() * 100 for _ in range(n)] for _ in range(n)])
    if symmetric:
        C = C + C.T
    C[np.arange(n), np.arange(n)] = 0.0
    W = np.array([[float(st.below(101)) for _ in range(n)] for _ in range(n)])
    if not self_flow:
        W[np.arange(n), np.arange(n)] = 0.0
    return Problem(n, p, C, W, chi, alpha, delta)


# ---------------------------------------------------------------------------
# Allocation and objective (hm/model.py:202-207, hm/evaluation.py:103-120)
# ---------------------------------------------------------------------------


def nearest(C: np.ndarray, hubs: np.ndarray) -> np.ndarray:
    """Nearest-hub allocation over sorted ``hubs``: first minimum wins, then
    every hub serves itself (hm/model.py:205-206)."""
    hubs = np.asarray(hubs, dtype=np.int64)
    pick = np.argmin(C[:, hubs], axis=1)
    a = hubs[pick]
    a[hubs] = hubs
    return a


def cost_terms(pr: Problem, hubs: np.ndarray, alloc: np.ndarray):
    """(collection, transfer, distribution) -- hm/evaluation.py:103-120.

    legs are node->hub for both spoke legs (C[i][a(i)]); the inter-cluster
    flow F is an index-ordered weighted bincount of keys c_i*p + c_j."""
    hubs = np.asarray(hubs, dtype=np.int64)
    alloc = np.asarray(alloc, dtype=np.int64)
    n, p = pr.n, hubs.size
    legs = pr.C[np.arange(n), alloc]
    coll = pr.chi * float(np.sum(pr.O * legs))
    dist = pr.delta * float(np.sum(pr.D * legs))
    pos = np.zeros(n, dtype=np.int64)
    pos[hubs] = np.arange(p)
    c = pos[alloc]
    F = np.bincount((c[:, None] * p + c[None, :]).ravel(), weights=pr.W.ravel(),
                    minlength=p * p)
    T = pr.C[np.ix_(hubs, hubs)].ravel()
    tran = pr.alpha * float(np.sum(F * T))
    return coll, tran, dist


def raw_cost(pr: Problem, hubs, alloc=None) -> float:
    hubs = np.sort(np.asarray(hubs, dtype=np.int64))
    if alloc is None:
        alloc = nearest(pr.C, hubs)
    coll, tran, dist = cost_terms(pr, hubs, alloc)
    return coll + tran + dist               # hm/evaluation.py:93


def scaled(raw: float, mode: str, total: float) -> float:
    """hm/evaluation.py:75-83 (milli is raw*1e-3, not raw/1000)."""
    if mode == "cab":
        if total == 0.0:
            raise ZeroDivisionError("total flow is zero")
        return raw / total
    if mode == "milli":
        return raw * 1e-3
    return raw


def path_sum(pr: Problem, alloc) -> float:
    """Literal per-pair path sum with fsum (reference tests conftest.py:52-68)."""
    C = pr.C.tolist()
    W = pr.W.tolist()
    a = [int(v) for v in alloc]
    terms = []
    for i in range(pr.n):
        for j in range(pr.n):
            w = W[i][j]
            if w:
                terms.append(w * (pr.chi * C[i][a[i]] + pr.alpha * C[a[i]][a[j]]
                                  + pr.delta * C[j][a[j]]))
    return math.fsum(terms)


def transfer_gather(pr: Problem, hubs, alloc) -> float:
    """S_T = sum_ij W_ij * C[a_i][a_j] -- the gather form the CUDA kernel
    computes (hm/oracle.py:126-127 is the reference's own batched use)."""
    alloc = np.asarray(alloc, dtype=np.int64)
    return float((pr.W * pr.C[alloc][:, alloc]).sum())


# ---------------------------------------------------------------------------
# Operators (hm/operators.py:41-146)
# ---------------------------------------------------------------------------


def splice(a: np.ndarray, b: np.ndarray, cut: int):
    """Children of a single cut at ``cut`` (hm/operators.py:55-56)."""
    return (np.concatenate([a[:cut], b[cut:]]), np.concatenate([b[:cut], a[cut:]]))


def cross(a: np.ndarray, b: np.ndarray, st) -> tuple:
    """hm/operators.py:41-57: cut = 1 + randint(n-1); n == 1 draws nothing."""
    n = a.shape[0]
    if n == 1:
        return a.copy(), b.copy()
    return splice(a, b, 1 + st.randint(n - 1))


def swap(mask: np.ndarray, st) -> np.ndarray:
    """hm/operators.py:113-124: close the r1-th open node, then open the r2-th
    node of the closed list taken BEFORE closing; identity with no draws on an
    all-open or all-closed mask."""
    on = np.flatnonzero(mask)
    off = np.flatnonzero(~mask)
    out = mask.copy()
    if on.size == 0 or off.size == 0:
        return out
    out[on[st.randint(on.size)]] = False
    out[off[st.randint(off.size)]] = True
    return out


def repair(mask: np.ndarray, pr: Problem) -> np.ndarray:
    """hm/operators.py:69-101 -> sorted hub indices, exactly p of them.

    deficit: open closed nodes in middle-rank order; excess: repeatedly
    drop the hub whose nearest-allocated nodes carry the least O+D
    (index-ordered bincount; first minimum)."""
    mask = np.asarray(mask, dtype=bool)
    hubs = np.flatnonzero(mask)
    if hubs.size < pr.p:
        m = mask.copy()
        missing = pr.p - hubs.size
        for v in pr.rank:
            if missing == 0:
                break
            if not m[v]:
                m[v] = True
                missing -= 1
        hubs = np.flatnonzero(m)
    w = pr.O + pr.D
    while hubs.size > pr.p:
        a = nearest(pr.C, hubs)
        pos = np.zeros(pr.n, dtype=np.int64)
        pos[hubs] = np.arange(hubs.size)
        load = np.bincount(pos[a], weights=w, minlength=hubs.size)
        hubs = np.delete(hubs, int(np.argmin(load)))
    return hubs


def indicator(hubs, n: int) -> np.ndarray:
    m = np.zeros(n, dtype=bool)
    m[np.asarray(hubs, dtype=np.int64)] = True
    return m


# ---------------------------------------------------------------------------
# Island GA (hm/engine.py:138-243)
# ---------------------------------------------------------------------------


@dataclass
class GaResult:
    hubs: np.ndarray
    raw: float
    scaled: float
    trace: tuple
    evaluations: int


def strength_for(p: int, strength) -> int:
    s = min(p, 3) if strength is None else strength         # hm/engine.py:84-88
    if s > p:
        raise ValueError(f"perturb_strength {s} exceeds p={p}")
    return s


def island_streams(seed: int, island: int):
    """(population, crossover, mutation) streams of one island (hm/engine.py:189-194)."""
    return tuple(Stream(stream_key(seed, island, role)) for role in (0, 1, 2))


def run_island(pr: Problem, streams, anc: np.ndarray, pop: int, inner: int, s: int,
               strict: bool, score):
    """One island for one outer round (hm/engine.py:138-167).
    Returns ((raw, hubs), evaluations)."""
    sp, sc, sm = streams
    local = anc
    best = None
    champ = None
    evals = 0
    for _gen in range(inner):
        members = [] if strict else [local]
        while len(members) < pop:
            h = local
            for _k in range(s):
                h = swap(h, sp)
            members.append(h)
        champ = None
        for j in range(0, pop, 2):
            for child in cross(members[j], members[j + 1], sc):
                hubs = repair(swap(child, sm), pr)
                r = score(hubs)
                evals += 1
                if champ is None or r < champ[0]:
                    champ = (r, hubs)
        local = indicator(champ[1], pr.n)
        if best is None or champ[0] < best[0]:
            best = champ
    return (champ if strict else best), evals


def island_ga(pr: Problem, islands: int, pop: int, inner: int, outer: int, seed: int = 0,
              strength=None, strict: bool = False, mode: str = "raw",
              island_range=None, on_round=None) -> GaResult:
    """The reference GA, restated.  Streams are per (seed, island, role) with
    roles population=0, crossover=1, mutation=2 (hm/engine.py:40-54), created
    once and consumed across rounds.

    ``island_range`` restricts the islands simulated (a shard); the caller
    then combines shards -- used by the multi-rank host tests."""
    s = strength_for(pr.p, strength)
    memo: dict = {}

    def score(h):
        key = h.tobytes()
        v = memo.get(key)
        if v is None:
            v = raw_cost(pr, h)
            memo[key] = v
        return v

    seed_hubs = np.sort(pr.rank[:pr.p])
    inc_raw = score(seed_hubs)
    inc_hubs = seed_hubs
    best_raw, best_hubs = inc_raw, inc_hubs
    lo, hi = (0, islands) if island_range is None else island_range
    streams = {g: island_streams(seed, g) for g in range(lo, hi)}
    trace = []
    evals = 0
    for _ in range(outer):
        anc = indicator(inc_hubs, pr.n)
        results = []
        for g in range(lo, hi):
            res, k = run_island(pr, streams[g], anc, pop, inner, s, strict, score)
            results.append(res)
            evals += k
        win = None
        for cand in results:
            if win is None or cand[0] < win[0]:
                win = cand
        if on_round is not None:
            win = on_round(win)
        if strict:
            inc_raw, inc_hubs = win
            if win[0] < best_raw:
                best_raw, best_hubs = win
            trace.append(scaled(win[0], mode, pr.total))
        else:
            if win[0] < inc_raw:
                inc_raw, inc_hubs = win
            best_raw, best_hubs = inc_raw, inc_hubs
            trace.append(scaled(inc_raw, mode, pr.total))
    return GaResult(np.asarray(best_hubs, dtype=np.int64), best_raw,
                    scaled(best_raw, mode, pr.total), tuple(trace), evals)


# ---------------------------------------------------------------------------
# Exhaustive oracle over hub sets (hm/oracle.py:42-54)
# ---------------------------------------------------------------------------


def restricted_best(pr: Problem):
    """Lexicographically-first hub set minimising the nearest-allocation raw."""
    best = None
    for combo in itertools.combinations(range(pr.n), pr.p):
        r = raw_cost(pr, np.array(combo, dtype=np.int64))
        if best is None or r < best[0]:
            best = (r, combo)
    return np.array(best[1], dtype=np.int64), best[0]


# ---------------------------------------------------------------------------
# Benchmark population: individual b's hub set is the p
# smallest of derive_stream(1, b).random_block(n) (stable argsort), sorted.
# ---------------------------------------------------------------------------


def bench_population(n: int, p: int, count: int, key: int = 1, start: int = 0) -> np.ndarray:
    out = np.empty((count, p), dtype=np.int64)
    for b in range(count):
        u = Stream(stream_key(key, start + b)).unit_block(n)
        out[b] = np.sort(np.argsort(u, kind="stable")[:p])
    return out
