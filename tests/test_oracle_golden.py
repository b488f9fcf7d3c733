"""Pin the CPU oracle to the reference's own outputs (CPU only).

The fixtures were produced by running hubmedian 0.1.0 itself
(tests/golden/make_golden.py); the oracle must reproduce them bit-for-bit
(integer/index work, and fp64 values since the oracle uses the same numpy
reductions), before it is trusted as the checker for the CUDA path.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import EVAL_LABELS, GA_LABELS, golden, orc, params_of, problem_from


class TestRng:
    def test_known_answer(self):
        g = golden("rng")
        assert orc.mix64(orc.GOLDEN) == int(g["kat"][0]) == 0xE220A8397B1DCDAF

    def test_streams_match_reference(self):
        g = golden("rng")
        keys = json.loads(str(g["keys_json"]))
        seeds = [0, 1, 9, 42, 1704, 2**63 + 5, -1]
        row = 0
        for s in seeds:
            for k in keys:
                state = orc.stream_key(s, *k)
                assert state == int(g["states"][row])
                st = orc.Stream(state)
                assert [st.u64() for _ in range(8)] == [int(v) for v in g["outs"][row]]
                assert st.unit_block(4).tolist() == g["rnd"][row].tolist()
                got = [st.below(b) for b in (1, 2, 3, 7, 100, 1001, 2**20, 999_983)]
                assert got == g["rint"][row].tolist()
                row += 1

    def test_block_equals_scalar(self):
        a, b = orc.Stream(9), orc.Stream(9)
        assert a.u64_block(257).tolist() == [b.u64() for _ in range(257)]
        assert a.u64() == b.u64()


class TestGenerator:
    @pytest.mark.parametrize("idx", range(4))
    def test_small_urand_bitwise(self, idx):
        g = golden("instances")
        n, p, seed, *f = g[f"urand{idx}_args"]
        pr = orc.urand_problem(int(n), int(p), int(seed), tuple(f))
        assert np.array_equal(pr.C, g[f"urand{idx}_dist"])
        assert np.array_equal(pr.W, g[f"urand{idx}_flow"])
        assert np.array_equal(pr.rank, g[f"urand{idx}_rank"])

    @pytest.mark.parametrize("idx", range(2))
    def test_big_urand_digest(self, idx):
        g = golden("instances")
        n, p, seed, *f = g[f"big{idx}_args"]
        pr = orc.urand_problem(int(n), int(p), int(seed), tuple(f))
        sha = [hashlib.sha256(pr.C.tobytes()).hexdigest(),
               hashlib.sha256(pr.W.tobytes()).hexdigest()]
        assert sha == g[f"big{idx}_sha"].tolist()
        assert np.array_equal(pr.rank, g[f"big{idx}_rank"])
        assert pr.total == float(g[f"big{idx}_total"][0])

    @pytest.mark.parametrize("idx", range(3))
    def test_stream_instances(self, idx):
        g = golden("instances")
        seed, n, p, kw = json.loads(str(g[f"mk{idx}_args"]))
        pr = orc.stream_problem(seed, n, p, **kw)
        assert np.array_equal(pr.C, g[f"mk{idx}_dist"])
        assert np.array_equal(pr.W, g[f"mk{idx}_flow"])


class TestEvaluation:
    @pytest.mark.parametrize("label", EVAL_LABELS)
    def test_population_alloc_and_cost_bitwise(self, label):
        g = golden("evaluation")
        pr = problem_from(g, label)
        assert np.array_equal(orc.bench_population(pr.n, pr.p, len(g[f"{label}_hubs"])),
                              g[f"{label}_hubs"])
        for hubs, alloc, comp in zip(g[f"{label}_hubs"], g[f"{label}_alloc"],
                                     g[f"{label}_comp"]):
            a = orc.nearest(pr.C, hubs)
            assert np.array_equal(a, alloc)
            c, t, d = orc.cost_terms(pr, hubs, a)
            assert [c, t, d, c + t + d] == comp.tolist()

    @pytest.mark.parametrize("label", EVAL_LABELS)
    def test_random_feasible_allocations(self, label):
        g = golden("evaluation")
        pr = problem_from(g, label)
        for hubs, alloc, comp in zip(g[f"{label}_rhubs"], g[f"{label}_ralloc"],
                                     g[f"{label}_rcomp"]):
            c, t, d = orc.cost_terms(pr, hubs, alloc)
            assert [c, t, d, c + t + d] == comp.tolist()
            if pr.n <= 70:
                assert c + t + d == pytest.approx(orc.path_sum(pr, alloc), rel=1e-9)
            # gather form (what the CUDA kernel sums) agrees to fp64 rounding
            gt = pr.alpha * orc.transfer_gather(pr, hubs, alloc)
            assert gt == pytest.approx(t, rel=1e-12, abs=1e-9)

    @pytest.mark.parametrize("label", ["tie", "ovr"])
    def test_tie_and_override(self, label):
        g = golden("evaluation")
        pr = problem_from(g, label)
        for hubs, alloc in zip(g[f"{label}_hubs"], g[f"{label}_alloc"]):
            assert np.array_equal(orc.nearest(pr.C, hubs), alloc)


class TestOperators:
    def test_correction_small(self):
        g = golden("operators")
        pr = problem_from(g, "op")
        for m, h in zip(g["corr_masks"], g["corr_hubs"]):
            assert np.array_equal(orc.repair(m, pr), h)

    def test_correction_ap(self):
        g = golden("operators")
        pr = problem_from(g, "opbig")
        for m, h in zip(g["corrbig_masks"], g["corrbig_hubs"]):
            assert np.array_equal(orc.repair(m, pr), h)

    def test_crossover_and_swap_replay(self):
        g = golden("operators")
        st = orc.Stream(orc.stream_key(15))
        for cr, sw in zip(g["xs_cross"], g["xs_swap"]):
            c1, c2 = orc.cross(g["xs_a"], g["xs_b"], st)
            assert np.array_equal(c1, cr[0]) and np.array_equal(c2, cr[1])
            assert np.array_equal(orc.swap(c1, st), sw)
        end = (orc.stream_key(15) + st.taken * orc.GOLDEN) & orc.M64
        assert end == int(g["xs_state_after"][0])


class TestGa:
    @pytest.mark.parametrize("label", GA_LABELS)
    def test_solve_matches_reference(self, label):
        g = golden("ga")
        pr = problem_from(g, label)
        kw = params_of(g, label)
        if label == "cab":
            kw = dict(kw)
        res = orc.island_ga(pr, kw["islands"], kw["pop_size"], kw["inner_iters"],
                            kw["outer_iters"], kw.get("seed", 0), kw.get("perturb_strength"),
                            kw.get("strict_paper", False), str(g[f"{label}_mode"]))
        assert np.array_equal(res.hubs, g[f"{label}_hubs"])
        assert [res.raw, res.scaled] == g[f"{label}_raw"].tolist()
        assert list(res.trace) == g[f"{label}_trace"].tolist()
        assert res.evaluations == int(g[f"{label}_evals"][0])


class TestRestricted:
    @pytest.mark.parametrize("idx", range(12))
    def test_restricted_optimum(self, idx):
        g = golden("restricted")
        pr = problem_from(g, f"r{idx}")
        hubs, raw = orc.restricted_best(pr)
        assert np.array_equal(hubs, g[f"r{idx}_hubs"])
        assert raw == float(g[f"r{idx}_raw"][0])
