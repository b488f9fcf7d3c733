"""Parity of the CUDA path against the reference's golden vectors and the
oracle (needs a B200: marked gpu).

Bars: allocations, corrected hub sets, crossover / swap masks and GA hub
sets are bit-exact; fp64 costs agree with the reference within 1e-12
relative (the north star asks 1e-9); GA raw values and traces within 1e-12.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import EVAL_LABELS, GA_LABELS, golden, orc, params_of

import paper_1704_06258_b200 as hg

pytestmark = pytest.mark.gpu

REL = 1e-12


def inst_from(g, prefix) -> hg.Instance:
    n, p, chi, alpha, delta = g[f"{prefix}_meta"]
    return hg.Instance(int(n), int(p), g[f"{prefix}_dist"], g[f"{prefix}_flow"], float(chi),
                       float(alpha), float(delta))


def close(a, b, rel=REL):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.all(np.abs(a - b) <= rel * np.maximum(np.abs(b), 1e-300) + 1e-300)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if hg.device_count() < 1:
        pytest.fail("no CUDA device: the gpu tests must run on a B200")


@pytest.fixture(params=["fp64", "tensor-pair", "tensor-pair-full"])
def kernel(request):
    """Run a test with the fp64 gather kernel (K3) and with the tensor-core
    kernel K3-TC/P, on the triangular fold of W (symmetric costs) and on the
    full W (used wherever the flows are integers below 2^32; elsewhere the
    instance stays on auto)."""
    from paper_1704_06258_b200 import _lib

    _lib.set_fitness_default(request.param)
    yield request.param
    _lib.set_fitness_default("auto")


class TestAllocation:
    @pytest.mark.parametrize("label", EVAL_LABELS + ["tie", "ovr"])
    def test_bit_exact_vs_reference(self, label):
        g = golden("evaluation")
        inst = inst_from(g, label)
        got = hg.nearest_allocations(inst, g[f"{label}_hubs"])
        assert np.array_equal(got, g[f"{label}_alloc"])

    def test_single_api(self):
        g = golden("evaluation")
        inst = inst_from(g, "ap")
        sol = hg.nearest_allocation(g["ap_hubs"][3], inst)
        assert np.array_equal(sol.alloc, g["ap_alloc"][3])
        assert hg.validate(sol, inst).ok
        with pytest.raises(ValueError, match="expected p=10"):
            hg.nearest_allocation([1, 2], inst)

    def test_ur_vs_oracle(self):
        inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
        pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
        pop = hg.random_population(1000, 20, 64)
        got = hg.nearest_allocations(inst, pop)
        for b in range(64):
            assert np.array_equal(got[b], orc.nearest(pr.C, pop[b]))


class TestObjective:
    @pytest.mark.parametrize("label", EVAL_LABELS)
    def test_population_components(self, label, kernel):
        g = golden("evaluation")
        inst = inst_from(g, label)
        out = hg.evaluate_population(inst, g[f"{label}_hubs"])
        assert close(out, g[f"{label}_comp"])

    @pytest.mark.parametrize("label", EVAL_LABELS)
    def test_arbitrary_feasible_allocations(self, label, kernel):
        g = golden("evaluation")
        inst = inst_from(g, label)
        for hubs, alloc, comp in zip(g[f"{label}_rhubs"], g[f"{label}_ralloc"],
                                     g[f"{label}_rcomp"]):
            hub = np.zeros(inst.n, dtype=bool)
            hub[hubs] = True
            bd = hg.objective(inst, hg.Solution(hub=hub, alloc=alloc))
            assert close([bd.collection_cost, bd.transfer_cost, bd.distribution_cost,
                          bd.raw_total], comp)

    def test_modes_exact(self):
        g = golden("evaluation")
        inst = inst_from(g, "cab")
        sol = hg.nearest_allocation(g["cab_hubs"][0], inst)
        raw = hg.objective(inst, sol).raw_total
        assert hg.fitness(inst, sol, hg.FitnessMode.STANDARD_MILLI) == raw * 1e-3
        assert hg.fitness(inst, sol, hg.FitnessMode.CAB_NORMALIZED) == raw / inst.total_flow

    def test_device_side_input_validation(self):
        inst = hg.generate_urand(300, 7, 9, (1.0, 0.75, 1.0))
        pop = hg.random_population(300, 7, 50)
        good = hg.evaluate_population(inst, pop)
        for bad_row, mutate in ((17, lambda h: h.__setitem__(2, h[1])),      # repeat
                                (3, lambda h: h.__setitem__(0, -1)),         # negative
                                (40, lambda h: h.__setitem__(6, 300)),       # >= n
                                (41, lambda h: h.__setitem__(6, 10**12)),    # far out
                                (49, lambda h: h.__setitem__(0, -10**12))):
            bad = pop.copy()
            mutate(bad[bad_row])
            with pytest.raises(ValueError, match=f"hub set {bad_row}:"):
                hg.evaluate_population(inst, bad)
            # the instance is usable afterwards and results are unchanged
            assert np.array_equal(hg.evaluate_population(inst, pop), good)
        with pytest.raises(ValueError, match="hub set 0:"):
            hg.nearest_allocations(inst, pop[:1, ::-1])

    def test_batch_invariance_bitwise(self, kernel):
        """A hub set's score does not depend on its batch or position."""
        inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
        pop = hg.random_population(1000, 20, 300)
        full = hg.evaluate_population(inst, pop)
        part = hg.evaluate_population(inst, pop[123:140])
        assert np.array_equal(full[123:140], part)
        rev = hg.evaluate_population(inst, pop[::-1])
        assert np.array_equal(full, rev[::-1])

    @pytest.mark.parametrize("n,p,f", [(1000, 20, (1.0, 0.75, 1.0)), (200, 10, (3.0, 0.75, 2.0)),
                                       (333, 7, (1.0, 0.5, 2.0)), (25, 3, (1.0, 0.2, 1.0)),
                                       (90, 50, (1.0, 0.75, 1.0))])
    def test_vs_oracle_random_configs(self, n, p, f, kernel):
        inst = hg.generate_urand(n, p, 77, f)
        pr = orc.Problem(n, p, inst.dist, inst.flow, *f)
        pop = hg.random_population(n, p, 40, key=5)
        out = hg.evaluate_population(inst, pop)
        ref = np.array([list(orc.cost_terms(pr, h, orc.nearest(pr.C, h))) for h in pop])
        ref = np.concatenate([ref, (ref[:, 0] + ref[:, 1] + ref[:, 2])[:, None]], axis=1)
        assert close(out, ref)

    def test_asymmetric_self_flow(self, kernel):
        pr = orc.stream_problem(24, 40, 6, symmetric=False, self_flow=True, chi=3.0, alpha=0.75,
                                delta=2.0)
        inst = hg.Instance(40, 6, pr.C, pr.W, 3.0, 0.75, 2.0)
        pop = hg.random_population(40, 6, 30, key=9)
        out = hg.evaluate_population(inst, pop)
        for b in range(30):
            a = orc.nearest(pr.C, pop[b])
            assert np.array_equal(hg.nearest_allocations(inst, pop[b:b + 1])[0], a)
            assert close(out[b, 3], orc.path_sum(pr, a), rel=1e-9)

    def test_big_instance_linearity(self, kernel):
        """n=6000, p=50 (BASELINE config 4): the transfer term is linear in
        alpha and in W; check against the oracle on a few individuals."""
        inst = hg.generate_urand(6000, 50, 1704, (1.0, 0.75, 1.0))
        pop = hg.random_population(6000, 50, 3)
        out = hg.evaluate_population(inst, pop)
        pr = orc.Problem(6000, 50, inst.dist, inst.flow, 1.0, 0.75, 1.0)
        for b in range(3):
            a = orc.nearest(pr.C, pop[b])
            st = 0.75 * orc.transfer_gather(pr, pop[b], a)
            assert close(out[b, 1], st, rel=1e-11)
        inst2 = inst.with_factors(alpha=1.5)
        out2 = hg.evaluate_population(inst2, pop)
        assert close(out2[:, 1], 2.0 * out[:, 1], rel=1e-14)
        assert np.array_equal(out2[:, 0], out[:, 0])


class TestKernels:
    def test_tensor_path_is_selected_for_u8_flows(self):
        inst = hg.generate_urand(300, 20, 3, (1.0, 0.75, 1.0))
        d = inst.device()
        assert d.flags & 4 and d.fitness_kernel == "tensor-pair"
        big = hg.generate_urand(1100, 20, 3, (1.0, 0.75, 1.0))
        assert big.device().fitness_kernel == "tensor-pair"  # K chunks of 1024 nodes
        with pytest.raises(ValueError, match="unknown fitness kernel"):
            big.device().set_fitness(4)  # the superseded TMEM one-CTA kernel is gone
        half = hg.Instance(inst.n, inst.p, inst.dist, inst.flow * 0.5, 1.0, 0.75, 1.0)
        assert half.device().fitness_kernel == "tensor-pair"  # quantum 2^-1: exact
        wide = np.where(inst.flow > 50, inst.flow * 1e12, inst.flow * 1e-9)  # 2^70 range
        frac = hg.Instance(inst.n, inst.p, inst.dist, wide, 1.0, 0.75, 1.0)
        assert frac.device().fitness_kernel == "fp64"
        with pytest.raises(ValueError, match="tensor-core"):
            frac.device().set_fitness(2)

    @pytest.mark.parametrize("n,p", [(1000, 20), (200, 10), (129, 50), (77, 3), (256, 1),
                                     (300, 17), (1024, 128), (640, 7), (1025, 20), (2100, 9),
                                     (3000, 60)])
    def test_tensor_equals_fp64(self, n, p):
        inst = hg.generate_urand(n, p, 21, (2.0, 0.6, 1.5))
        pop = hg.random_population(n, p, 301, key=4)  # odd: a pair's dummy unit
        d = inst.device()
        d.set_fitness(1)
        fp = hg.evaluate_population(inst, pop)
        for kind in (5, 6):  # CTA pair on the triangular fold / on the full W
            d.set_fitness(kind)
            tc = hg.evaluate_population(inst, pop)
            assert np.array_equal(tc[:, [0, 2]], fp[:, [0, 2]])
            assert close(tc, fp, rel=1e-13), kind


class TestOperators:
    def test_correction_vs_reference(self):
        g = golden("operators")
        inst = inst_from(g, "op")
        assert np.array_equal(hg.correct_hub_sets(inst=inst, masks=g["corr_masks"]),
                              g["corr_hubs"])
        inst = inst_from(g, "opbig")
        assert np.array_equal(hg.correct_hub_sets(inst=inst, masks=g["corrbig_masks"]),
                              g["corrbig_hubs"])
        assert np.array_equal(hg.correct_hub_set(g["corrbig_masks"][5], inst),
                              g["corrbig_hubs"][5])

    def test_correction_inexact_weights(self):
        """Non-integer flows: carried loads are summed in index order (np.bincount)."""
        pr = orc.stream_problem(31, 30, 4)
        W = pr.W * 0.1 + 1e-3
        pr2 = orc.Problem(30, 4, pr.C, W, 1.0, 0.75, 1.0)
        inst = hg.Instance(30, 4, pr.C, W, 1.0, 0.75, 1.0)
        rng = np.random.default_rng(3)
        masks = rng.random((200, 30)) < 0.4
        got = hg.correct_hub_sets(masks, inst)
        for m, h in zip(masks, got):
            assert np.array_equal(h, orc.repair(m, pr2))

    def test_crossover_and_swap_replay(self):
        g = golden("operators")
        st = hg.derive_stream(15)
        for cr, sw in zip(g["xs_cross"], g["xs_swap"]):
            c1, c2 = hg.crossover_hub_arrays(g["xs_a"], g["xs_b"], st)
            assert np.array_equal(c1, cr[0]) and np.array_equal(c2, cr[1])
            assert np.array_equal(hg.swap_random_hub_spoke(c1, st), sw)
        assert st.state == int(g["xs_state_after"][0])

    def test_perturb_matches_mutation_composition(self):
        pr = orc.stream_problem(57, 10, 4)
        inst = hg.Instance(10, 4, pr.C, pr.W, 1.0, 0.75, 1.0)
        sol = hg.nearest_allocation({0, 2, 5, 8}, inst)
        got = hg.perturb(sol, inst, hg.derive_stream(14), strength=3)
        exp = sol
        rng = hg.derive_stream(14)
        for _ in range(3):
            exp = hg.mutation(exp, inst, rng)
        assert got == exp

    def test_closure_pipelines(self):
        """crossover -> swap -> correction always yields a feasible solution
        (reference acceptance criterion 7, batched on the device)."""
        rng = np.random.default_rng(7)
        for n, p in ((9, 3), (64, 5), (300, 40)):
            inst = hg.generate_urand(n, p, 5, (1.0, 0.75, 1.0))
            masks = rng.random((2000, n)) < rng.random((2000, 1))
            hubs = hg.correct_hub_sets(masks, inst)
            assert (np.diff(hubs, axis=1) > 0).all() and hubs.min() >= 0 and hubs.max() < n
            pr = orc.Problem(n, p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
            for k in range(0, 2000, 97):
                assert np.array_equal(hubs[k], orc.repair(masks[k], pr))


class TestGa:
    @pytest.mark.parametrize("label", GA_LABELS)
    def test_solve_replays_reference(self, label, kernel):
        g = golden("ga")
        inst = inst_from(g, label)
        params = hg.GaParams(**params_of(g, label))
        mode = hg.FitnessMode.from_string(str(g[f"{label}_mode"]))
        rep = hg.solve(inst, params, mode)
        assert np.array_equal(rep.best_solution.hubs, g[f"{label}_hubs"])
        assert np.array_equal(rep.best_solution.alloc, g[f"{label}_alloc"])
        assert close([rep.raw_objective, rep.scaled_fitness], g[f"{label}_raw"])
        assert close(rep.trace, g[f"{label}_trace"])
        assert rep.evaluations == int(g[f"{label}_evals"][0])
        assert not rep.interrupted

    def test_audit_sees_every_evaluation_and_interrupt(self):
        pr = orc.stream_problem(86, 9, 3)
        inst = hg.Instance(9, 3, pr.C, pr.W, 1.0, 0.75, 1.0)
        seen = []
        params = hg.GaParams(islands=2, pop_size=4, inner_iters=3, outer_iters=2, seed=9)
        rep = hg.solve(inst, params, hg.FitnessMode.RAW, workers=1,
                       audit=lambda s: seen.append(hg.validate(s, inst).ok))
        assert all(seen) and len(seen) == rep.evaluations + 1

        calls = {"k": 0}

        def stop(_s):
            calls["k"] += 1
            if calls["k"] > 40:
                raise KeyboardInterrupt

        pr = orc.stream_problem(93, 9, 3)
        inst = hg.Instance(9, 3, pr.C, pr.W, 1.0, 0.75, 1.0)
        params = hg.GaParams(islands=2, pop_size=4, inner_iters=5, outer_iters=5, seed=6)
        rep = hg.solve(inst, params, hg.FitnessMode.RAW, workers=1, audit=stop)
        assert rep.interrupted and hg.validate(rep.best_solution, inst).ok
        assert len(rep.trace) < params.outer_iters

    def test_reaches_restricted_optimum(self):
        """Reference acceptance criterion 1 on a sample of its instance family."""
        hits = 0
        for k in range(20):
            meta = orc.Stream(orc.stream_key(777, k))
            n = 5 + meta.below(5)
            p = 2 + meta.below(2)
            inst = hg.generate_urand(n, p, 1000 + k, (1.0, 0.75, 1.0))
            pr = orc.Problem(n, p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
            _, rr = orc.restricted_best(pr)
            rep = hg.solve(inst, hg.GaParams(islands=8, pop_size=16, inner_iters=20,
                                             outer_iters=5, seed=k, perturb_strength=2),
                           hg.FitnessMode.STANDARD_MILLI)
            hits += abs(rep.raw_objective - rr) <= 1e-12 * rr
            assert all(b <= a for a, b in zip(rep.trace, rep.trace[1:]))
        assert hits >= 19

    def test_virtual_shards_identical(self, kernel):
        """Island sharding across devices reproduces the 1-device run: shards
        of [0, R) run one after another on this GPU with the same exchange."""
        from paper_1704_06258_b200 import engine

        inst = hg.generate_urand(200, 10, 1704, (3.0, 0.75, 2.0))
        params = hg.GaParams(islands=12, pop_size=16, inner_iters=4, outer_iters=3, seed=3)
        ref = hg.solve(inst, params, hg.FitnessMode.STANDARD_MILLI)
        for world in (2, 3, 4):
            shards = [engine.DeviceIslands(inst, params, params.resolved_strength(inst.p),
                                           *hg.island_shard(12, r, world)) for r in range(world)]

            class Joined:
                def run_round(self, anc, audit=None):
                    parts = [s.run_round(anc) for s in shards]
                    return (np.concatenate([q[0] for q in parts]),
                            np.concatenate([q[1] for q in parts]))

            rep = engine._solve(inst, params, hg.FitnessMode.STANDARD_MILLI, None,
                                lambda *a: Joined(), None)
            assert rep.raw_objective == ref.raw_objective
            assert rep.trace == ref.trace
            assert rep.best_solution == ref.best_solution


class TestNext:
    """device generator and GPU restricted optimum."""

    @pytest.mark.parametrize("idx", range(4))
    def test_device_generator_small_bit_exact(self, idx):
        g = golden("instances")
        n, p, seed, *f = g[f"urand{idx}_args"]
        inst = hg.generate_urand(int(n), int(p), int(seed), tuple(f), device=True)
        assert np.array_equal(inst.dist, g[f"urand{idx}_dist"])
        assert np.array_equal(inst.flow, g[f"urand{idx}_flow"])
        assert np.array_equal(inst.middle_rank, g[f"urand{idx}_rank"])

    @pytest.mark.parametrize("idx", range(2))
    def test_device_generator_big_digest(self, idx):
        import hashlib

        g = golden("instances")
        n, p, seed, *f = g[f"big{idx}_args"]
        inst = hg.generate_urand(int(n), int(p), int(seed), tuple(f), device=True)
        sha = [hashlib.sha256(inst.dist.tobytes()).hexdigest(),
               hashlib.sha256(inst.flow.tobytes()).hexdigest()]
        assert sha == g[f"big{idx}_sha"].tolist()
        assert inst.total_flow == float(g[f"big{idx}_total"][0])

    def test_device_generator_matches_host_at_bench_size(self):
        a = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0), device=True)
        b = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
        assert np.array_equal(a.dist, b.dist) and np.array_equal(a.flow, b.flow)

    @pytest.mark.parametrize("idx", range(12))
    def test_restricted_optimum_vs_reference(self, idx, kernel):
        g = golden("restricted")
        inst = inst_from(g, f"r{idx}")
        sol, raw = hg.restricted_optimum(inst)
        assert np.array_equal(sol.hubs, g[f"r{idx}_hubs"])
        assert close(raw, float(g[f"r{idx}_raw"][0]), rel=1e-12)

    def test_restricted_optimum_multi_batch(self):
        """C(40, 4) = 91,390 sets: two device batches; the winner and its raw
        equal a host sweep over the same scores (itertools order, first
        strict minimum)."""
        import itertools

        inst = hg.generate_urand(40, 4, 11, (1.0, 0.75, 1.0))
        combos = np.array(list(itertools.combinations(range(40), 4)), dtype=np.int64)
        raw = hg.evaluate_population(inst, combos)[:, 3]
        sol, best = hg.restricted_optimum(inst)
        k = int(np.argmin(raw))  # numpy argmin = first minimum
        assert np.array_equal(sol.hubs, combos[k]) and best == raw[k]

    def test_restricted_optimum_limit(self):
        inst = hg.generate_urand(30, 5, 2, (1.0, 0.75, 1.0))
        with pytest.raises(hg.EnumerationLimitError, match="142506 candidates"):
            hg.restricted_optimum(inst, limit=100_000)
        from paper_1704_06258_b200 import _lib

        with pytest.raises(ValueError, match="over the limit of 10"):
            _lib.restricted_optimum(inst.device(), 10)

    def test_unique_evaluation_matches(self, kernel):
        """Duplicate-aware scoring: every repeat gets its group's row, bit for
        bit, and each distinct set is scored once."""
        inst = hg.generate_urand(300, 12, 9, (1.0, 0.75, 1.0))
        base = hg.random_population(300, 12, 500, key=3)
        rng = np.random.default_rng(5)
        pop = base[rng.integers(0, 500, size=3000)]
        plain = hg.evaluate_population(inst, pop)
        uniq = hg.evaluate_population(inst, pop, unique=True)
        assert np.array_equal(plain, uniq)
        assert inst.device().last_groups == len(np.unique(pop, axis=0))
        allu = hg.evaluate_population(inst, base, unique=True)
        assert np.array_equal(allu, hg.evaluate_population(inst, base))
        assert inst.device().last_groups == 500

    def test_unique_evaluation_validates(self):
        inst = hg.generate_urand(50, 4, 9, (1.0, 0.75, 1.0))
        pop = hg.random_population(50, 4, 20, key=3)
        pop[7] = [3, 3, 4, 5]
        with pytest.raises(ValueError, match="hub set 7"):
            hg.evaluate_population(inst, pop, unique=True)
        assert hg.evaluate_population(inst, pop[:7], unique=True).shape == (7, 4)


class TestCli:
    """the command line runs the reference's manifests and
    emits its CSV schema v1 rows -- equal, field by field but the wall time,
    to the reference's own output (tests/golden/cli.npz); fp64 cost fields
    within the fp64 bar (the device sums in its own fixed order, not numpy's
    pairwise order, so the last digit of a repr can differ)."""

    @staticmethod
    def _run(args, capsys):
        from paper_1704_06258_b200 import cli

        rc = cli.main(args)
        return rc, capsys.readouterr().out

    @staticmethod
    def _write(tmp_path, idx):
        f = tmp_path / f"g{idx}.usaphmp"
        f.write_bytes(golden("cli")[f"gen{idx}_bytes"].tobytes())
        return f

    @pytest.mark.parametrize("idx", range(2))
    def test_solve_rows(self, idx, tmp_path, capsys):
        g = golden("cli")
        f = self._write(tmp_path, idx)
        rc, text = self._run(["solve", str(f), "--csv", "-"] + g[f"solve{idx}_args"].tolist(),
                             capsys)
        assert rc == 0
        rows = [[c for k, c in enumerate(ln.split(",")) if k != 9]
                for ln in text.strip().splitlines()]
        want = [ln.split(",") for ln in g[f"solve{idx}_rows"].tolist()]
        assert len(rows) == len(want)
        for got_row, want_row in zip(rows, want):
            assert len(got_row) == len(want_row)
            for a, b in zip(got_row, want_row):
                if "." in b and a != b:  # an fp64 cost: the fp64 bar, not repr identity
                    assert close(float(a), float(b)), (a, b)
                else:
                    assert a == b

    @pytest.mark.parametrize("idx", range(2))
    def test_oracle_text(self, idx, tmp_path, capsys):
        f = self._write(tmp_path, idx)
        rc, text = self._run(["oracle", str(f), "--which", "restricted"], capsys)
        assert rc == 0 and text == str(golden("cli")[f"oracle{idx}_text"])

    def test_eval_text(self, tmp_path, capsys):
        g = golden("cli")
        f = self._write(tmp_path, 0)
        sf = tmp_path / "s0.sol"
        sf.write_bytes(g["eval0_solution"].tobytes())
        rc, text = self._run(["eval", str(f), str(sf), "--fitness-mode", "cab"], capsys)
        assert rc == 0
        ref = str(g["eval0_text"]).splitlines()
        got = text.splitlines()
        assert [ln.split()[0] for ln in got] == [ln.split()[0] for ln in ref]
        assert close([float(ln.split()[-1]) for ln in got],
                     [float(ln.split()[-1]) for ln in ref], rel=1e-12)

    def test_bench_rows(self, tmp_path, capsys):
        g = golden("cli")
        self._write(tmp_path, 0)
        self._write(tmp_path, 1)
        (tmp_path / "m.csv").write_text("label,path,format,p,mode,known_best\n"
                                        "a,g0.usaphmp,,,milli,\n"
                                        "b,g1.usaphmp,canonical,2,raw,1e6\n")
        rc, text = self._run(["bench", str(tmp_path / "m.csv"), "--seeds", "0,1", "--islands",
                              "4", "--pop", "8", "--inner", "3", "--outer", "2", "--csv", "-"],
                             capsys)
        assert rc == int(g["bench_rc"][0])
        lines = [ln for ln in text.strip().splitlines() if "," in ln]
        rows = [",".join(c for k, c in enumerate(ln.split(",")) if k != 9) for ln in lines]
        assert rows == g["bench_rows"].tolist()

    def test_gen_on_device(self, tmp_path, capsys):
        g = golden("cli")
        n, p, seed, alpha = g["gen1_args"]
        out = tmp_path / "d.usaphmp"
        rc, _ = self._run(["gen", "-n", str(int(n)), "-p", str(int(p)), "--seed", str(int(seed)),
                           "--alpha", repr(float(alpha)), "-o", str(out), "--device"], capsys)
        assert rc == 0 and out.read_bytes() == g["gen1_bytes"].tobytes()


class TestPhilox:
    """rng='philox': the same operators and draw accounting on Philox4x32-10
    streams -- deterministic, shard-invariant, feasible, elitist-monotone."""

    def test_philox_ga(self):
        from paper_1704_06258_b200 import engine

        inst = hg.generate_urand(200, 10, 1704, (3.0, 0.75, 2.0))
        params = hg.GaParams(islands=12, pop_size=16, inner_iters=4, outer_iters=3, seed=3,
                             rng="philox")
        a = hg.solve(inst, params, hg.FitnessMode.STANDARD_MILLI)
        b = hg.solve(inst, params, hg.FitnessMode.STANDARD_MILLI)
        assert a.trace == b.trace and np.array_equal(a.best_solution.hubs, b.best_solution.hubs)
        assert hg.validate(a.best_solution, inst).ok
        assert all(y <= x for x, y in zip(a.trace, a.trace[1:]))
        rep = hg.solve(inst, hg.GaParams(islands=12, pop_size=16, inner_iters=4, outer_iters=3,
                                         seed=3), hg.FitnessMode.STANDARD_MILLI)
        assert rep.evaluations == a.evaluations
        # sharding the islands does not change the philox run either
        for world in (2, 3):
            shards = [engine.DeviceIslands(inst, params, params.resolved_strength(inst.p),
                                           *hg.island_shard(12, r, world)) for r in range(world)]
            anc = np.sort(inst.middle_rank[:inst.p])
            full = engine.DeviceIslands(inst, params, params.resolved_strength(inst.p), 0, 12)
            ref_raw, ref_hubs = full.run_round(anc)
            parts = [s.run_round(anc) for s in shards]
            assert np.array_equal(np.concatenate([r for r, _ in parts]), ref_raw)
            assert np.array_equal(np.concatenate([h for _, h in parts]), ref_hubs)


class TestPairChunks:
    """K3-TC/P with n > 1024: K chunks of 1024 nodes and a partial last chunk,
    whose one-hot quarters have different boundaries from a full chunk's.
    Large batches (many phases per CTA pair) against the fp64 kernel."""

    @pytest.mark.parametrize("n,p,B", [(1030, 5, 4096), (1100, 20, 2048), (2100, 9, 2048),
                                       (3000, 40, 512)])
    def test_partial_chunks_many_phases(self, n, p, B):
        inst = hg.generate_urand(n, p, 77, (1.0, 0.75, 1.0))
        pop = hg.random_population(n, p, B, key=6)
        d = inst.device()
        d.set_fitness(1)
        fp = hg.evaluate_population(inst, pop)
        d.set_fitness(5)
        for _ in range(3):  # repeated launches: a timing race would show up as a mismatch
            tc = hg.evaluate_population(inst, pop)
            assert np.array_equal(tc[:, [0, 2]], fp[:, [0, 2]])
            assert close(tc, fp, rel=1e-13)


class TestWidePlanes:
    """Integer flows above 255: K3-TC/P on 2..4 byte planes of W (exact), the
    one-plane kernels unavailable, results equal to the fp64 kernel."""

    @pytest.mark.parametrize("wmax,planes", [(300, 2), (70000, 3), (2**24 + 5, 4)])
    def test_planes_match_fp64(self, wmax, planes):
        base = hg.generate_urand(700, 12, 5, (1.0, 0.75, 1.0))
        rng = np.random.default_rng(planes)
        flow = rng.integers(0, wmax + 1, size=(700, 700)).astype(np.float64)
        np.fill_diagonal(flow, 0.0)
        flow[3, 4] = float(wmax)
        inst = hg.Instance(700, 12, base.dist, flow, 1.0, 0.75, 1.0)
        d = inst.device()
        assert d.flags & 4 and d.fitness_kernel == "tensor-pair"
        pop = hg.random_population(700, 12, 999, key=2)
        tc = hg.evaluate_population(inst, pop)  # triangular fold: W + W^T planes
        d.set_fitness(6)
        full = hg.evaluate_population(inst, pop)  # the full W's planes
        d.set_fitness(1)
        fp = hg.evaluate_population(inst, pop)
        for got in (tc, full):
            assert np.array_equal(got[:, [0, 2]], fp[:, [0, 2]])
            assert close(got, fp, rel=1e-13)

    def test_flows_from_2_32_use_fp64(self):
        base = hg.generate_urand(50, 4, 5, (1.0, 0.75, 1.0))
        flow = base.flow.copy()
        flow[1, 2] = 2.0**32
        inst = hg.Instance(50, 4, base.dist, flow, 1.0, 0.75, 1.0)
        assert inst.device().fitness_kernel == "fp64"


class TestAllocationVariants:
    """K2 has a register variant for p <= 32 (16x2 SIMD argmin, packed
    count/index) and the scalar kernel for every p: their outputs --
    cluster ids, allocations, hub-cost tables and the fp64 leg sums, hence
    the scored costs -- must agree bit for bit, quantised ties included
    (an integer-grid instance).  The choice is fixed per process
    (HUBGPU_K2_SCALAR), so each runs in a subprocess."""

    def test_register_and_scalar_k2_bit_identical(self):
        import os
        import subprocess
        import sys
        from pathlib import Path

        root = Path(__file__).resolve().parent.parent
        digests = []
        for scalar in ("0", "1"):
            env = dict(os.environ, HUBGPU_K2_SCALAR=scalar)
            r = subprocess.run([sys.executable, str(root / "tools" / "k2_ab.py")], env=env,
                               capture_output=True, text=True, timeout=600, check=True)
            digests.append([ln for ln in r.stdout.splitlines() if ln.startswith("ALL")][0])
        assert digests[0] == digests[1]


class TestExactSums:
    """set_exact_sums(True): the cost terms equal the reference's np.sum
    values bit for bit (hm/evaluation.py:110-118: legs products, bincount
    inter-cluster flows, hub distances) -- numpy's pairwise summation order
    replayed on the device for the collection / distribution sums (K2) and,
    with one K chunk on one byte plane, the transfer sum (K3-TC/P).  Both the
    nearest-allocation and the given-allocation paths; ragged n (n % 8 != 0,
    n < 8, a single leaf, several leaves)."""

    @pytest.fixture(autouse=True)
    def _exact(self):
        hg.set_exact_sums(True)
        yield
        hg.set_exact_sums(False)

    @pytest.mark.parametrize("n,p,B", [(25, 3, 200), (7, 2, 21), (8, 3, 56), (9, 4, 100),
                                       (129, 7, 200), (1000, 20, 120), (517, 32, 100),
                                       (300, 40, 60), (700, 12, 80)])
    def test_bit_identical_to_numpy(self, n, p, B):
        inst = hg.generate_urand(n, p, 1704 + n, (1.0, 0.75, 1.0))
        pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
        pop = hg.random_population(n, p, B, key=n + p)
        got = hg.evaluate_population(inst, pop)
        al = hg.nearest_allocations(inst, pop)
        got2 = hg.evaluate_population(inst, pop, alloc=al)
        want = np.empty((B, 4))
        for b in range(B):
            c, t, d = orc.cost_terms(pr, pop[b], al[b])
            want[b] = (c, t, d, c + t + d)
        assert np.array_equal(got, want)
        assert np.array_equal(got2, want)

    def test_full_batch_many_units(self):
        """8192 hub sets: every CTA pair runs ~9 units back to back, so the
        shared-memory terms, stacks and bins are reused across units; sampled
        rows bit-identical to numpy, the whole batch identical run to run."""
        inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
        pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
        pop = hg.random_population(1000, 20, 8192, key=11)
        got = hg.evaluate_population(inst, pop)
        again = hg.evaluate_population(inst, pop)
        assert np.array_equal(got, again)
        rows = np.arange(0, 8192, 129)
        al = hg.nearest_allocations(inst, pop[rows])
        for j, b in enumerate(rows):
            c, t, d = orc.cost_terms(pr, pop[b], al[j])
            assert np.array_equal(got[b], [c, t, d, c + t + d]), b

    @pytest.mark.parametrize("n,p,full", [(1024, 56, True), (1024, 8, True), (1000, 64, False),
                                          (1000, 100, False)])
    def test_large_p(self, n, p, full):
        """p up to ~56 keeps the [p][128] fp64 terms beside two W stages: all
        four terms bit-identical; beyond that the transfer sum is the
        fixed-order fold (within the fp64 bar), the leg sums stay exact."""
        inst = hg.generate_urand(n, p, 7 + p, (1.0, 0.75, 1.0))
        pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
        pop = hg.random_population(n, p, 60, key=p)
        got = hg.evaluate_population(inst, pop)
        al = hg.nearest_allocations(inst, pop)
        for b in range(60):
            c, t, d = orc.cost_terms(pr, pop[b], al[b])
            assert got[b, 0] == c and got[b, 2] == d
            if full:
                assert got[b, 1] == t and got[b, 3] == c + t + d
            else:
                assert close(got[b, 1], t) and close(got[b, 3], c + t + d)

    @pytest.mark.parametrize("n,p,wmax", [(1030, 9, None), (2100, 12, None), (3000, 20, None),
                                          (300, 7, 1000), (200, 12, 70000)])
    def test_multi_chunk_and_planes(self, n, p, wmax):
        """n > 1024 (K chunks) and flows >= 256 (byte planes): the integer
        bins accumulate over every chunk and plane (total flow < 2^32 here),
        so all four terms stay bit-identical."""
        inst = hg.generate_urand(n, p, 1704 + n, (1.0, 0.75, 1.0))
        if wmax is not None:
            rng = np.random.default_rng(n)
            flow = rng.integers(0, wmax + 1, size=(n, n)).astype(np.float64)
            np.fill_diagonal(flow, 0.0)
            inst = hg.Instance(n, p, inst.dist, flow, 1.0, 0.75, 1.0)
        pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
        pop = hg.random_population(n, p, 40, key=n + p)
        got = hg.evaluate_population(inst, pop)
        al = hg.nearest_allocations(inst, pop)
        for b in range(40):
            c, t, d = orc.cost_terms(pr, pop[b], al[b])
            assert np.array_equal(got[b], [c, t, d, c + t + d]), b

    def test_default_mode_within_an_ulp_or_so(self):
        hg.set_exact_sums(False)
        inst = hg.generate_urand(1000, 20, 2704, (1.0, 0.75, 1.0))
        pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, 1.0, 0.75, 1.0)
        pop = hg.random_population(1000, 20, 64, key=3)
        got = hg.evaluate_population(inst, pop)
        al = hg.nearest_allocations(inst, pop)
        for b in range(64):
            c, t, d = orc.cost_terms(pr, pop[b], al[b])
            assert close(got[b], (c, t, d, c + t + d), rel=1e-14)


class TestEdgeShapes:
    """Degenerate and extreme shapes (n = 1, p = n, p > 128 on the fp64 path,
    p = 255 on the scalar allocator, an empty batch, a 200k batch) in both
    summation modes, against the oracle."""

    @staticmethod
    def _check(inst, pop, exact):
        out = hg.evaluate_population(inst, pop)
        pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, inst.chi, inst.alpha, inst.delta)
        for b in range(0, len(pop), max(1, len(pop) // 5)):
            a = orc.nearest(pr.C, pop[b])
            c, t, d = orc.cost_terms(pr, pop[b], a)
            ref = np.array([c, t, d, c + t + d])
            if exact:
                assert out[b, 0] == c and out[b, 2] == d
            assert close(out[b], ref), (b, out[b], ref)

    @pytest.mark.parametrize("exact", [False, True])
    @pytest.mark.parametrize("n,p", [(1, 1), (2, 1), (2, 2), (3, 3), (16, 16), (300, 255),
                                     (1000, 129)])
    def test_shapes(self, n, p, exact):
        hg.set_exact_sums(exact)
        try:
            inst = hg.generate_urand(n, p, 3, (1.0, 0.75, 1.0))
            self._check(inst, hg.random_population(n, p, 7), exact)
        finally:
            hg.set_exact_sums(False)

    def test_empty_and_large_batches(self):
        inst = hg.generate_urand(1000, 20, 3, (1.0, 0.75, 1.0))
        assert hg.evaluate_population(inst, np.empty((0, 20), np.int64)).shape == (0, 4)
        self._check(inst, hg.random_population(1000, 20, 200000), False)
        assert hg.evaluate_population(inst, hg.random_population(1000, 20, 1),
                                      unique=True).shape == (1, 4)
