"""Round-2 parity and robustness on the GPU (marked gpu).

* BIG (n=6000, p=50): the reference's own cost breakdowns (tests/golden/big.npz,
  made by running hubmedian) -- within 1e-12 by default, bit-identical in
  exact mode -- and 256 more individuals against a restatement of
  hm/evaluation.py:103-120 within 1e-12;
* complete solve() runs at the BASELINE GA shapes: AP 16 x 64 x 3 x 2 and
  UR 128 x 64 x 1 x 1 (best hubs, raw, trace, evaluation count);
* an Instance shared by 8 threads (the reference's Instance is "safe to share
  across worker threads", hm/model.py:35);
* instances of different p used alternately (per-kernel launch attributes);
* the island GA across 2 and 3 processes (real DeviceIslands on the GPU,
  champion exchange over gloo) reproducing the reference's SolveReport.
"""

from __future__ import annotations

import hashlib
import json
import os
import socket
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

from conftest import golden, orc

import paper_1704_06258_b200 as hg

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu

REL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if hg.device_count() < 1:
        pytest.fail("no CUDA device: the gpu tests must run on a B200")


def _rel_ok(a, b, rel=REL):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.all(np.abs(a - b) <= rel * np.abs(b))


def _instance(g, label, device=True):
    n, p, seed, c, a, d = g[f"{label}_args"]
    inst = hg.generate_urand(int(n), int(p), int(seed), (c, a, d), device=device)
    sha = g[f"{label}_sha"]
    assert hashlib.sha256(inst.dist.tobytes()).hexdigest() == sha[0]
    assert hashlib.sha256(inst.flow.tobytes()).hexdigest() == sha[1]
    return inst


@pytest.fixture(scope="module")
def big():
    return _instance(golden("big"), "big")


def _costs_matrix_form(inst, hubs, alloc):
    """(coll, tran, dist, raw) of hm/evaluation.py:103-120 in matrix form:
    F = OneHot^T W OneHot (p x p) instead of the index-ordered bincount (the
    same sum in another order, so the bar is 1e-12, not bits)."""
    n, p = inst.n, inst.p
    legs = inst.dist[np.arange(n), alloc]
    coll = inst.chi * float(np.sum(inst.out_flow * legs))
    dist = inst.delta * float(np.sum(inst.in_flow * legs))
    pos = np.zeros(n, dtype=np.int64)
    pos[hubs] = np.arange(p)
    oh = np.zeros((n, p))
    oh[np.arange(n), pos[alloc]] = 1.0
    F = oh.T @ (inst.flow @ oh)
    tran = inst.alpha * float(np.sum(F * inst.dist[np.ix_(hubs, hubs)]))
    return np.array([coll, tran, dist, coll + tran + dist])


class TestBig:
    def test_reference_breakdowns(self, big):
        g = golden("big")
        out = hg.evaluate_population(big, g["big_hubs"])
        assert _rel_ok(out, g["big_comp"])
        allocs = hg.nearest_allocations(big, g["big_hubs"])
        shas = [hashlib.sha256(a.astype(np.int64).tobytes()).hexdigest() for a in allocs]
        assert shas == g["big_alloc_sha"].tolist()

    def test_reference_breakdowns_exact(self, big):
        # total flow 1.8e9 < 2^32: the integer bins span every K chunk, so
        # every term is the reference's np.sum bit for bit
        assert big.total_flow < 2**32
        g = golden("big")
        hg.set_exact_sums(True)
        try:
            out = hg.evaluate_population(big, g["big_hubs"])
        finally:
            hg.set_exact_sums(False)
        assert np.array_equal(out, g["big_comp"]), np.abs(out - g["big_comp"]).max(axis=0)

    def test_256_individuals(self, big):
        pop = hg.random_population(big.n, big.p, 256, key=77)
        out = hg.evaluate_population(big, pop)
        allocs = hg.nearest_allocations(big, pop)
        for b in range(256):
            assert np.array_equal(allocs[b], orc.nearest(big.dist, pop[b])), b
            assert _rel_ok(out[b], _costs_matrix_form(big, pop[b], allocs[b])), b

    def test_fp64_kernel_agrees(self, big):
        from paper_1704_06258_b200 import _lib

        g = golden("big")
        d = big.device()
        tens = hg.evaluate_population(big, g["big_hubs"])
        d.set_fitness(_lib.FIT_FP64)
        try:
            f64 = hg.evaluate_population(big, g["big_hubs"])
        finally:
            d.set_fitness(_lib.FIT_AUTO)
        assert _rel_ok(f64, g["big_comp"])
        assert _rel_ok(tens, f64, 1e-13)


class TestGaFullShapes:
    @pytest.mark.parametrize("label", ["ap", "ur"])
    def test_solve_matches_reference(self, label):
        g = golden("big")
        inst = _instance(g, label)
        params = hg.GaParams(**json.loads(str(g[f"{label}_params"])))
        rep = hg.solve(inst, params, hg.FitnessMode.STANDARD_MILLI)
        assert np.array_equal(rep.best_solution.hubs, g[f"{label}_hubs"])
        assert _rel_ok([rep.raw_objective, rep.scaled_fitness], g[f"{label}_raw"])
        assert _rel_ok(rep.trace, g[f"{label}_trace"])
        assert rep.evaluations == int(g[f"{label}_evals"][0])


class TestSharedInstance:
    def test_eight_threads(self):
        inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
        pops = [hg.random_population(1000, 20, 64 + 8 * k, key=200 + k) for k in range(16)]
        serial = [hg.evaluate_population(inst, pop) for pop in pops]
        sols = [hg.nearest_allocation(pop[0], inst) for pop in pops]
        serial_obj = [hg.objective(inst, s).raw_total for s in sols]

        def work(k):
            got = []
            for _ in range(4):
                got.append((hg.evaluate_population(inst, pops[k]),
                            hg.objective(inst, sols[k]).raw_total))
            return got

        with ThreadPoolExecutor(8) as ex:
            results = list(ex.map(work, range(16)))
        for k, got in enumerate(results):
            for out, raw in got:
                assert np.array_equal(out, serial[k])
                assert raw == serial_obj[k]

    def test_concurrent_solves(self):
        inst = hg.generate_urand(200, 10, 1704, (3.0, 0.75, 2.0))
        params = hg.GaParams(islands=4, pop_size=16, inner_iters=3, outer_iters=2, seed=3)
        ref = hg.solve(inst, params, hg.FitnessMode.STANDARD_MILLI)
        with ThreadPoolExecutor(4) as ex:
            reps = list(ex.map(lambda _: hg.solve(inst, params, hg.FitnessMode.STANDARD_MILLI),
                               range(8)))
        for r in reps:
            assert np.array_equal(r.best_solution.hubs, ref.best_solution.hubs)
            assert r.raw_objective == ref.raw_objective
            assert r.trace == ref.trace


class TestInstancesOfDifferentShape:
    def test_alternating_p(self):
        # a p=50 instance first, then p=20: each kernel's launch attribute
        # must still admit the larger p=50 launches (and its captured graph)
        a = hg.generate_urand(1000, 50, 5, (1.0, 0.75, 1.0))
        pa = hg.random_population(1000, 50, 40, key=3)
        ref_a = hg.evaluate_population(a, pa)
        pa_ga = hg.GaParams(islands=2, pop_size=8, inner_iters=2, outer_iters=1, seed=1)
        ga_a = hg.solve(a, pa_ga)
        b = hg.generate_urand(1000, 20, 6, (1.0, 0.75, 1.0))
        pb = hg.random_population(1000, 20, 40, key=4)
        ref_b = hg.evaluate_population(b, pb)
        for _ in range(3):
            assert np.array_equal(hg.evaluate_population(a, pa), ref_a)
            assert np.array_equal(hg.evaluate_population(b, pb), ref_b)
            assert hg.solve(a, pa_ga).raw_objective == ga_a.raw_objective


# ---------------------------------------------------------------------------
# the island GA across processes: real device islands, gloo exchange
# ---------------------------------------------------------------------------

def _mp_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1704_06258_b200 as hg2

        hg2.set_device(0)
        g = golden("big")
        n, p, seed, c, a, d = g["ap_args"]
        inst = hg2.generate_urand(int(n), int(p), int(seed), (c, a, d))
        params = hg2.GaParams(**json.loads(str(g["ap_params"])))
        rep = hg2.solve(inst, params, hg2.FitnessMode.STANDARD_MILLI, group=dist.group.WORLD)
        q.put((rank, rep.best_solution.hubs.tolist(), rep.raw_objective, list(rep.trace),
               rep.evaluations))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_islands_across_processes(world):
    """Islands sharded over `world` processes on one GPU (each its own CUDA
    context; the kernels never wait on another process -- the exchange is a
    host all_gather at the round barrier) give the reference's report."""
    import torch.multiprocessing as mp

    g = golden("big")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    for rank, hubs, raw, trace, evals in res:
        assert raw is not None, hubs
        assert hubs == g["ap_hubs"].tolist()
        assert _rel_ok(raw, g["ap_raw"][0])
        assert _rel_ok(trace, g["ap_trace"])
        assert evals == int(g["ap_evals"][0])


class TestFractionalFlows:
    """Non-integer flows on the tensor cores: Q = rint(W / q) on up to 8 byte
    planes, q a power of two keeping every nonzero flow to 2^-41 relative, so
    every cost term (and the non-negative transfer sum) is within 2^-41 of the
    reference's -- the test bar stays 1e-12 relative."""

    @staticmethod
    def _instance(n, p, flows, symmetric=True, seed=3):
        base = hg.generate_urand(n, p, seed, (3.0, 0.75, 2.0))
        dist = base.dist
        if not symmetric:
            dist = dist.copy()
            dist[np.triu_indices(n, 1)] *= 1.0 + 1e-3
        return hg.Instance(n, p, dist, flows, 3.0, 0.75, 2.0)

    @pytest.mark.parametrize("case", ["decimals", "wide", "asymmetric", "bigger"])
    def test_tensor_path_matches_oracle(self, case):
        rng = np.random.default_rng(11)
        n, p = (1100, 12) if case == "bigger" else (300, 10)
        if case == "wide":  # flows over four decades: 7 planes, folded one at a time
            flows = 10.0 ** rng.uniform(-2.0, 2.0, (n, n))
        else:  # decimals in [0.1, 37.6): 6 planes (the fold of W + W^T: 7)
            flows = rng.integers(0, 100, (n, n)) * 0.37 + 0.1 + 0.9 * rng.random((n, n))
        np.fill_diagonal(flows, 0.0)
        inst = self._instance(n, p, flows, symmetric=case != "asymmetric")
        d = inst.device()
        assert d.flags & 4
        assert d.fitness_kernel == ("tensor-pair-full" if case == "asymmetric" else "tensor-pair")
        pop = hg.random_population(n, p, 200, key=5)
        tc = hg.evaluate_population(inst, pop)
        from paper_1704_06258_b200 import _lib

        d.set_fitness(_lib.FIT_FP64)
        try:
            fp = hg.evaluate_population(inst, pop)
        finally:
            d.set_fitness(_lib.FIT_AUTO)
        assert np.array_equal(tc[:, [0, 2]], fp[:, [0, 2]])
        assert _rel_ok(tc, fp)
        pr = orc.Problem(n, p, inst.dist, inst.flow, 3.0, 0.75, 2.0)
        for b in range(0, 200, 23):
            a = orc.nearest(pr.C, pop[b])
            c, t, dd = orc.cost_terms(pr, pop[b], a)
            assert _rel_ok(tc[b], [c, t, dd, c + t + dd]), b

    def test_range_beyond_eight_planes_uses_fp64(self):
        rng = np.random.default_rng(2)
        flows = 10.0 ** rng.uniform(-9.0, 9.0, (200, 200))
        np.fill_diagonal(flows, 0.0)
        inst = self._instance(200, 8, flows)
        assert inst.device().fitness_kernel == "fp64"
        assert not inst.device().flags & 4

    def test_ga_replays_on_fractional_flows(self):
        rng = np.random.default_rng(4)
        flows = rng.integers(0, 100, (200, 200)) * 0.5 + 0.1 + 0.9 * rng.random((200, 200))
        np.fill_diagonal(flows, 0.0)
        inst = self._instance(200, 10, flows)
        assert inst.device().fitness_kernel == "tensor-pair"
        pr = orc.Problem(200, 10, inst.dist, inst.flow, 3.0, 0.75, 2.0)
        rep = hg.solve(inst, hg.GaParams(islands=4, pop_size=16, inner_iters=3, outer_iters=2),
                       hg.FitnessMode.STANDARD_MILLI)
        ref = orc.island_ga(pr, 4, 16, 3, 2, 0, None, False, "milli")
        assert np.array_equal(rep.best_solution.hubs, ref.hubs)
        assert _rel_ok(rep.raw_objective, ref.raw)

    def test_power_of_two_multiples_are_exact(self):
        # flows in quarter units: exact integers Q = 4 W on the byte planes,
        # so even the exact mode is bit-identical to the reference's sums
        base = hg.generate_urand(300, 10, 7, (3.0, 0.75, 2.0))
        inst = hg.Instance(300, 10, base.dist, base.flow * 0.25, 3.0, 0.75, 2.0)
        assert inst.device().fitness_kernel == "tensor-pair"
        pop = hg.random_population(300, 10, 64, key=9)
        pr = orc.Problem(300, 10, inst.dist, inst.flow, 3.0, 0.75, 2.0)
        hg.set_exact_sums(True)
        try:
            ex = hg.evaluate_population(inst, pop)
        finally:
            hg.set_exact_sums(False)
        for b in range(0, 64, 7):
            a = orc.nearest(pr.C, pop[b])
            c, t, d = orc.cost_terms(pr, pop[b], a)
            assert np.array_equal(ex[b], [c, t, d, c + t + d]), b


@pytest.mark.gpu
def test_ga_replays_with_duplicate_grouping_forced():
    """The GA's per-generation duplicate grouping must leave the
    trajectory unchanged: rerun the GA replay tests with it forced on for every
    tensor-kernel GA (the switch is read once per process, hence the child)."""
    env = dict(os.environ, HUBGPU_GA_DEDUPE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p",
                        "no:cacheprovider", "tests/test_gpu_parity.py::TestGa",
                        "tests/test_gpu_round2.py::TestGaFullShapes",
                        "tests/test_gpu_round2.py::TestFractionalFlows"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


class TestEvaluateGraph:
    """hg_evaluate replays its pipelined copies + kernels as one CUDA graph
    when the hub sets and the results are page-locked, patching each call's
    host pointers into the graph's copy nodes: results must equal the stream
    path's (pageable hub sets) bit for bit, for alternating buffers and batch
    sizes, and a bad row must still be reported."""

    def test_replays_match_stream_path(self):
        from paper_1704_06258_b200 import _lib

        inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
        pops = [hg.random_population(1000, 20, B, key=40 + k)
                for k, B in enumerate((8192, 8192, 4096, 8192))]
        ref = [hg.evaluate_population(inst, pop) for pop in pops]  # pageable: stream path
        pinned = []
        for pop in pops:
            buf = _lib.pinned_array(pop.shape, np.int64)
            buf[...] = pop
            pinned.append(buf)
        for rnd in range(3):
            for k, buf in enumerate(pinned):
                assert np.array_equal(hg.evaluate_population(inst, buf), ref[k]), (rnd, k)
        bad = _lib.pinned_array(pops[0].shape, np.int64)
        bad[...] = pops[0]
        bad[77, 3] = bad[77, 2]
        with pytest.raises(ValueError, match="hub set 77:"):
            hg.evaluate_population(inst, bad)
        assert np.array_equal(hg.evaluate_population(inst, pinned[0]), ref[0])


@pytest.mark.gpu
def test_zero_copy_evaluate_matches():
    """HUBGPU_EVAL_ZEROCOPY=1 (opt-in): K2 reads the page-locked int64 hub sets
    over PCIe and validates them itself (the fused k_hubs_in), K3 writes the
    costs into the page-locked result buffer.  Same results as the default
    path, same bad-row report (child process: the switch is read once)."""
    code = r'''
import numpy as np, pytest, sys
sys.path.insert(0, ".")
import paper_1704_06258_b200 as hg
from paper_1704_06258_b200 import _lib
inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
inst2 = hg.generate_urand(300, 40, 9, (1.0, 0.5, 2.0))
for ins, B in ((inst, 8192), (inst, 300), (inst2, 777)):
    pop = hg.random_population(ins.n, ins.p, B, key=B)
    buf = _lib.pinned_array(pop.shape, np.int64)
    buf[...] = pop
    np.save(sys.stdout.buffer, hg.evaluate_population(ins, buf))
bad = _lib.pinned_array((64, 20), np.int64)
bad[...] = hg.random_population(1000, 20, 64, key=3)
bad[41, 5] = 5000
try:
    hg.evaluate_population(inst, bad)
    print("NOERROR")
except ValueError as e:
    assert "hub set 41:" in str(e), e
'''
    outs = []
    for zc in ("0", "1"):
        env = dict(os.environ, HUBGPU_EVAL_ZEROCOPY=zc)
        r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr.decode()[-3000:]
        assert b"NOERROR" not in r.stdout
        import io
        f = io.BytesIO(r.stdout)
        outs.append([np.load(f) for _ in range(3)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


class TestDeferredFoldShapes:
    """K3-TC/P's deferred fold (one K chunk, >= 4 output tiles) at the shapes
    around its edges -- 4..8 tiles, ragged last tiles, odd unit counts (a
    dummy slot in one CTA of a pair), p from 5 to 37 -- against the fp64
    kernel, within the 1e-12 bar; and the pair path (HUBGPU_TCP_DEFER=0 is
    covered by the shapes below 4 tiles)."""

    @pytest.mark.parametrize("n,p,B", [(385, 5, 1001), (500, 13, 777), (640, 20, 2049),
                                       (700, 37, 333), (1024, 20, 4097), (900, 8, 65),
                                       (600, 64, 301), (900, 40, 1000), (1000, 90, 128)])
    def test_vs_fp64_kernel(self, n, p, B):
        from paper_1704_06258_b200 import _lib

        inst = hg.generate_urand(n, p, 11 + n, (1.0, 0.75, 1.0))
        pop = hg.random_population(n, p, B, key=n + p)
        d = inst.device()
        tens = hg.evaluate_population(inst, pop)
        d.set_fitness(_lib.FIT_FP64)
        try:
            f64 = hg.evaluate_population(inst, pop)
        finally:
            d.set_fitness(_lib.FIT_AUTO)
        assert _rel_ok(tens, f64, 1e-12)
        # and batch invariance across the slot partition
        part = hg.evaluate_population(inst, pop[B // 3:B // 3 + 17])
        assert np.array_equal(part, tens[B // 3:B // 3 + 17])
