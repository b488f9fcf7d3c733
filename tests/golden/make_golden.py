"""Generate golden fixtures by running the REAL reference (``hubmedian`` 0.1.0).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  The fixtures pin the CPU oracle
(oracle/hm_oracle.py) and, on the GPU box (where /root/reference does not
exist), the CUDA path.  Every value here comes from a reference call; the
only non-reference code is the loop that picks the inputs.
"""

from __future__ import annotations

import itertools
import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

import hubmedian as hm  # noqa: E402
from hubmedian import evaluation as hm_eval  # noqa: E402
from hubmedian import model as hm_model  # noqa: E402
from hubmedian import operators as hm_ops  # noqa: E402
from hubmedian.rng import derive_stream, mix64  # noqa: E402
import conftest as ref_conftest  # noqa: E402  (reference test helpers)

OUT = Path(__file__).resolve().parent


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({sum(a.nbytes for a in map(np.asarray, arrays.values()))} B raw)")


def gen_rng():
    seeds = [0, 1, 9, 42, 1704, 2**63 + 5, -1]
    keys = [(), (0,), (1, 2), (7, 3, 1), (1000, 20)]
    states, outs, rnd, rint = [], [], [], []
    for s in seeds:
        for k in keys:
            st = derive_stream(s, *k)
            states.append(st._state)
            outs.append([st.next_u64() for _ in range(8)])
            rnd.append(st.random_block(4))
            rint.append([st.randint(b) for b in (1, 2, 3, 7, 100, 1001, 2**20, 999_983)])
    save("rng",
         kat=np.array([mix64(0x9E3779B97F4A7C15)], dtype=np.uint64),
         seeds=np.array([s & (2**64 - 1) for s in seeds], dtype=np.uint64),
         keys_json=np.array(json.dumps(keys)),
         states=np.array(states, dtype=np.uint64),
         outs=np.array(outs, dtype=np.uint64),
         rnd=np.array(rnd), rint=np.array(rint, dtype=np.int64))


def inst_arrays(prefix, inst):
    return {f"{prefix}_dist": inst.dist, f"{prefix}_flow": inst.flow,
            f"{prefix}_meta": np.array([inst.n, inst.p, inst.chi, inst.alpha, inst.delta]),
            f"{prefix}_rank": inst.middle_rank}


def gen_instances():
    """Generator outputs (small ones in full, big ones by digest)."""
    out = {}
    small = [(12, 3, 606, (1.0, 0.75, 1.0)), (25, 3, 1704, (1.0, 0.2, 1.0)),
             (4, 2, 31, (1.0, 1.0, 1.0)), (1, 1, 3, (1.0, 0.75, 1.0))]
    for idx, (n, p, seed, f) in enumerate(small):
        out.update(inst_arrays(f"urand{idx}", hm.generate_urand(n, p, seed, f)))
        out[f"urand{idx}_args"] = np.array([n, p, seed, *f])
    import hashlib
    big = [(200, 10, 1704, (3.0, 0.75, 2.0)), (1000, 20, 1704, (1.0, 0.75, 1.0))]
    for idx, (n, p, seed, f) in enumerate(big):
        inst = hm.generate_urand(n, p, seed, f)
        out[f"big{idx}_args"] = np.array([n, p, seed, *f])
        out[f"big{idx}_sha"] = np.array([hashlib.sha256(inst.dist.tobytes()).hexdigest(),
                                         hashlib.sha256(inst.flow.tobytes()).hexdigest()])
        out[f"big{idx}_rank"] = inst.middle_rank
        out[f"big{idx}_total"] = np.array([inst.total_flow])
    # conftest.make_instance (reference's independent test-instance builder)
    mk = [(11, 7, 2, {}), (24, 7, 3, dict(symmetric=False, self_flow=True, chi=3.0, alpha=0.75,
                                           delta=2.0)), (63, 9, 3, dict(chi=2.0, alpha=0.5,
                                                                        delta=3.0))]
    for idx, (seed, n, p, kw) in enumerate(mk):
        out.update(inst_arrays(f"mk{idx}", ref_conftest.make_instance(seed, n, p, **kw)))
        out[f"mk{idx}_args"] = np.array(json.dumps([seed, n, p, kw]))
    save("instances", **out)


def population(n, p, count, key):
    pop = np.empty((count, p), dtype=np.int64)
    for b in range(count):
        u = derive_stream(key, b).random_block(n)
        pop[b] = np.sort(np.argsort(u, kind="stable")[:p])
    return pop


def gen_eval():
    """Allocations and (coll, tran, dist, raw) for populations, from the
    reference's allocate_to_nearest / objective."""
    out = {}
    cases = [
        ("cab", hm.generate_urand(25, 3, 1704, (1.0, 0.2, 1.0)), 64),
        ("ap", hm.generate_urand(200, 10, 1704, (3.0, 0.75, 2.0)), 48),
        ("asym", ref_conftest.make_instance(24, 7, 3, symmetric=False, self_flow=True,
                                            chi=3.0, alpha=0.75, delta=2.0), 35),
        ("p1", ref_conftest.make_instance(22, 6, 1, chi=2.0, alpha=0.75, delta=3.0), 6),
        ("pn", ref_conftest.make_instance(21, 5, 5, alpha=0.6), 1),
        ("mid", hm.generate_urand(70, 40, 5, (1.0, 0.75, 1.0)), 16),
    ]
    for name, inst, count in cases:
        pop = population(inst.n, inst.p, count, 1)
        allocs, comps = [], []
        for hubs in pop:
            sol = hm.nearest_allocation(hubs, inst)
            bd = hm.objective(inst, sol)
            allocs.append(sol.alloc)
            comps.append([bd.collection_cost, bd.transfer_cost, bd.distribution_cost,
                          bd.raw_total])
        out.update(inst_arrays(name, inst))
        out[f"{name}_hubs"] = pop
        out[f"{name}_alloc"] = np.array(allocs)
        out[f"{name}_comp"] = np.array(comps)
        # random feasible (NOT nearest) allocations: objective must accept them
        rng = derive_stream(8)
        rhubs, ralloc, rcomp = [], [], []
        for _ in range(12):
            sol = ref_conftest.random_feasible_solution(inst, rng)
            bd = hm.objective(inst, sol)
            rhubs.append(sol.hubs)
            ralloc.append(sol.alloc)
            rcomp.append([bd.collection_cost, bd.transfer_cost, bd.distribution_cost,
                          bd.raw_total])
        out[f"{name}_rhubs"] = np.array(rhubs)
        out[f"{name}_ralloc"] = np.array(ralloc)
        out[f"{name}_rcomp"] = np.array(rcomp)
    # tie-break fixtures (reference tests test_model.py:145-151 style)
    d = np.zeros((5, 5))
    d[0, 1] = d[1, 0] = 2.0
    d[0, 2] = d[2, 0] = 2.0
    d[3, 4] = d[4, 3] = 1.0
    d[0, 3] = d[3, 0] = 5.0
    d[1, 3] = d[3, 1] = d[2, 3] = d[3, 2] = 4.0
    d[0, 4] = d[4, 0] = d[1, 4] = d[4, 1] = d[2, 4] = d[4, 2] = 3.0
    tie = hm.Instance(n=5, p=2, dist=d, flow=np.ones((5, 5)), chi=1, alpha=1, delta=1)
    tie_hubs = np.array(list(itertools.combinations(range(5), 2)))
    out.update(inst_arrays("tie", tie))
    out["tie_hubs"] = tie_hubs
    out["tie_alloc"] = np.array([hm.nearest_allocation(h, tie).alloc for h in tie_hubs])
    # hub-override case: two co-located nodes (C[h][h'] = 0 for a lower h')
    d2 = np.array([[0.0, 0.0, 3.0], [0.0, 0.0, 4.0], [3.0, 4.0, 0.0]])
    ov = hm.Instance(n=3, p=2, dist=d2, flow=np.ones((3, 3)), chi=1, alpha=1, delta=1)
    out.update(inst_arrays("ovr", ov))
    out["ovr_hubs"] = np.array([[0, 1], [1, 2], [0, 2]])
    out["ovr_alloc"] = np.array([hm.nearest_allocation(h, ov).alloc for h in out["ovr_hubs"]])
    save("evaluation", **out)


def gen_operators():
    out = {}
    inst = ref_conftest.make_instance(58, 9, 3)
    out.update(inst_arrays("op", inst))
    # correction on arbitrary raw masks
    rng = derive_stream(6)
    masks, hubs = [], []
    for _ in range(200):
        raw = np.array([rng.randint(2) == 1 for _ in range(inst.n)])
        masks.append(raw)
        hubs.append(hm_ops.correct_hub_set(raw, inst))
    out["corr_masks"] = np.array(masks)
    out["corr_hubs"] = np.array(hubs)
    big = hm.generate_urand(200, 10, 1704, (3.0, 0.75, 2.0))
    out.update(inst_arrays("opbig", big))
    rng = derive_stream(7)
    masks, hubs = [], []
    for t in range(120):
        k = [0, 3, 9, 10, 11, 14, 20, 37, 200][t % 9]
        raw = np.zeros(big.n, dtype=bool)
        if k:
            sel = np.argsort(derive_stream(70, t).random_block(big.n), kind="stable")[:k]
            raw[sel] = True
        masks.append(raw)
        hubs.append(hm_ops.correct_hub_set(raw, big))
    out["corrbig_masks"] = np.array(masks)
    out["corrbig_hubs"] = np.array(hubs)
    # swap and crossover driven by real streams
    st = derive_stream(15)
    a = np.zeros(inst.n, bool)
    a[[0, 1, 2]] = True
    b = np.zeros(inst.n, bool)
    b[[4, 6, 8]] = True
    cross_out, swap_out = [], []
    for _ in range(50):
        c1, c2 = hm_ops.crossover_hub_arrays(a, b, st)
        cross_out.append(np.stack([c1, c2]))
        swap_out.append(hm_ops.swap_random_hub_spoke(c1, st))
    out["xs_a"] = a
    out["xs_b"] = b
    out["xs_cross"] = np.array(cross_out)
    out["xs_swap"] = np.array(swap_out)
    out["xs_state_after"] = np.array([st._state], dtype=np.uint64)
    save("operators", **out)


GA_CASES = [
    # (label, instance builder, GaParams kwargs, mode)
    ("cab", lambda: hm.generate_urand(25, 3, 1704, (1.0, 0.2, 1.0)),
     dict(islands=1, pop_size=100, inner_iters=60, outer_iters=1, seed=0), "cab"),
    ("small", lambda: ref_conftest.make_instance(82, 6, 2),
     dict(islands=8, pop_size=16, inner_iters=20, outer_iters=5, seed=1, perturb_strength=2),
     "raw"),
    ("mk84", lambda: ref_conftest.make_instance(84, 9, 3),
     dict(islands=8, pop_size=16, inner_iters=20, outer_iters=5, seed=1, perturb_strength=2),
     "milli"),
    ("strict", lambda: ref_conftest.make_instance(91, 9, 3),
     dict(islands=4, pop_size=8, inner_iters=5, outer_iters=4, seed=2, strict_paper=True),
     "raw"),
    ("pn", lambda: ref_conftest.make_instance(81, 5, 5, alpha=0.4),
     dict(islands=2, pop_size=4, inner_iters=2, outer_iters=3, seed=0), "raw"),
    ("asym", lambda: ref_conftest.make_instance(24, 7, 3, symmetric=False, self_flow=True,
                                                chi=3.0, alpha=0.75, delta=2.0),
     dict(islands=3, pop_size=6, inner_iters=4, outer_iters=2, seed=5), "raw"),
    ("n1", lambda: hm.Instance(n=1, p=1, dist=np.zeros((1, 1)), flow=np.ones((1, 1)),
                                chi=1, alpha=1, delta=1),
     dict(islands=2, pop_size=2, inner_iters=2, outer_iters=2, seed=3), "raw"),
    ("ap", lambda: hm.generate_urand(200, 10, 1704, (3.0, 0.75, 2.0)),
     dict(islands=4, pop_size=16, inner_iters=3, outer_iters=2, seed=0), "milli"),
    ("mid", lambda: hm.generate_urand(60, 8, 11, (1.0, 0.75, 1.0)),
     dict(islands=6, pop_size=10, inner_iters=6, outer_iters=3, seed=9, perturb_strength=4),
     "milli"),
    ("midstrict", lambda: hm.generate_urand(40, 5, 12, (2.0, 0.5, 1.5)),
     dict(islands=5, pop_size=12, inner_iters=4, outer_iters=3, seed=4, strict_paper=True,
          perturb_strength=5), "cab"),
]


def gen_ga():
    out = {}
    for label, build, kw, mode in GA_CASES:
        inst = build()
        rep = hm.solve(inst, hm.GaParams(**kw), hm.FitnessMode.from_string(mode))
        out.update(inst_arrays(label, inst))
        out[f"{label}_params"] = np.array(json.dumps(kw))
        out[f"{label}_mode"] = np.array(mode)
        out[f"{label}_hubs"] = rep.best_solution.hubs
        out[f"{label}_alloc"] = rep.best_solution.alloc
        out[f"{label}_raw"] = np.array([rep.raw_objective, rep.scaled_fitness])
        out[f"{label}_trace"] = np.array(rep.trace)
        out[f"{label}_evals"] = np.array([rep.evaluations])
        print(f"  ga {label}: raw={rep.raw_objective!r} evals={rep.evaluations}")
    save("ga", **out)


def gen_restricted():
    out = {}
    for idx in range(12):
        meta = derive_stream(777, idx)
        n = 5 + meta.randint(5)
        p = 2 + meta.randint(2)
        inst = hm.generate_urand(n, p, 1000 + idx, (1.0, 0.75, 1.0))
        sol, raw = hm.restricted_optimum(inst)
        out.update(inst_arrays(f"r{idx}", inst))
        out[f"r{idx}_hubs"] = sol.hubs
        out[f"r{idx}_raw"] = np.array([raw])
    save("restricted", **out)


def gen_cli():
    """Reference command-line outputs (hm/cli.py, hm/bench.py): instance files
    written by `gen`, CSV schema v1 rows of `solve` and `bench` (wall time
    dropped), `oracle` text, `eval` text, and parameter fingerprints."""
    import contextlib
    import io as _io
    import tempfile

    from hubmedian import bench as hm_bench
    from hubmedian import cli as hm_cli

    def run(args):
        buf = _io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = hm_cli.main(args)
        return rc, buf.getvalue()

    out = {}
    fps = []
    for prm, mode in [((64, 64, 50, 10, 0, None, False), "raw"), ((8, 8, 5, 3, 42, None, False), "milli"),
                      ((2, 100, 20, 2, 1, 2, True), "cab")]:
        params = hm.GaParams(islands=prm[0], pop_size=prm[1], inner_iters=prm[2],
                             outer_iters=prm[3], seed=prm[4], perturb_strength=prm[5],
                             strict_paper=prm[6])
        fps.append([json.dumps(prm), mode,
                    hm_bench.params_fingerprint(params, hm.FitnessMode.from_string(mode))])
    out["fingerprints"] = np.array(fps)
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        texts = []
        for idx, (n, p, seed, alpha) in enumerate([(12, 3, 606, 0.75), (25, 3, 1704, 0.2)]):
            f = td / f"g{idx}.usaphmp"
            rc, text = run(["gen", "-n", str(n), "-p", str(p), "--seed", str(seed), "--alpha",
                            str(alpha), "-o", str(f)])
            out[f"gen{idx}_args"] = np.array([n, p, seed, alpha])
            out[f"gen{idx}_bytes"] = np.frombuffer(f.read_bytes(), dtype=np.uint8)
            solve_args = ["--fitness-mode", "milli", "--islands", "8", "--pop", "8", "--inner",
                          "5", "--outer", "3", "--seed", "42"]
            rc, text = run(["solve", str(f), "--csv", "-"] + solve_args)
            cells = text.strip().splitlines()
            rows = [",".join(c for k, c in enumerate(line.split(",")) if k != 9) for line in cells]
            out[f"solve{idx}_rows"] = np.array(rows)
            out[f"solve{idx}_args"] = np.array(solve_args)
            rc, text = run(["oracle", str(f), "--which", "restricted"])
            out[f"oracle{idx}_text"] = np.array(text)
        # eval of a solution file against instance 0
        from hubmedian import io as hm_io

        inst = hm_io.load_instance(td / "g0.usaphmp")
        sol = hm.nearest_allocation([1, 5, 9], inst)
        sf = td / "s0.sol"
        sf.write_bytes(hm_io.write_solution(sol))
        out["eval0_solution"] = np.frombuffer(sf.read_bytes(), dtype=np.uint8)
        rc, text = run(["eval", str(td / "g0.usaphmp"), str(sf), "--fitness-mode", "cab"])
        out["eval0_text"] = np.array(text)
        # a two-row manifest
        (td / "m.csv").write_text("label,path,format,p,mode,known_best\n"
                                  "a,g0.usaphmp,,,milli,\n"
                                  "b,g1.usaphmp,canonical,2,raw,1e6\n")
        rc, text = run(["bench", str(td / "m.csv"), "--seeds", "0,1", "--islands", "4",
                        "--pop", "8", "--inner", "3", "--outer", "2", "--csv", "-"])
        lines = [ln for ln in text.strip().splitlines() if "," in ln]
        out["bench_rows"] = np.array([",".join(c for k, c in enumerate(ln.split(",")) if k != 9)
                                      for ln in lines])
        out["bench_rc"] = np.array([rc])
    save("cli", **out)


def gen_big():
    """BASELINE shapes at full size (round 2): BIG (n=6000, p=50) cost
    breakdowns from the reference's objective for 24 uniform hub sets, and two
    complete solve() runs -- AP 16 x 64 x 3 x 2 and UR 128 x 64 x 1 x 1.  The
    instances are generate_urand(...) outputs (identified by arguments and
    SHA-256, rebuilt bit-exactly by the package's generator)."""
    import hashlib

    out = {}

    def ident(label, args, inst):
        out[f"{label}_args"] = np.array(args[:3] + list(args[3]), dtype=np.float64)
        out[f"{label}_sha"] = np.array([hashlib.sha256(inst.dist.tobytes()).hexdigest(),
                                        hashlib.sha256(inst.flow.tobytes()).hexdigest()])

    args = [6000, 50, 1704, (1.0, 0.75, 1.0)]
    big = hm.generate_urand(*args)
    ident("big", args, big)
    pop = population(big.n, big.p, 24, 1)
    comps, ahash = [], []
    for hubs in pop:
        sol = hm.nearest_allocation(hubs, big)
        bd = hm.objective(big, sol)
        comps.append([bd.collection_cost, bd.transfer_cost, bd.distribution_cost, bd.raw_total])
        ahash.append(hashlib.sha256(sol.alloc.astype(np.int64).tobytes()).hexdigest())
    out["big_hubs"] = pop
    out["big_comp"] = np.array(comps)
    out["big_alloc_sha"] = np.array(ahash)
    print(f"  big: {len(pop)} breakdowns")
    for label, args, kw in [
        ("ap", [200, 10, 1704, (3.0, 0.75, 2.0)],
         dict(islands=16, pop_size=64, inner_iters=3, outer_iters=2, seed=0)),
        ("ur", [1000, 20, 1704, (1.0, 0.75, 1.0)],
         dict(islands=128, pop_size=64, inner_iters=1, outer_iters=1, seed=0)),
    ]:
        inst = hm.generate_urand(*args)
        ident(label, args, inst)
        rep = hm.solve(inst, hm.GaParams(**kw), hm.FitnessMode.STANDARD_MILLI)
        out[f"{label}_params"] = np.array(json.dumps(kw))
        out[f"{label}_hubs"] = rep.best_solution.hubs
        out[f"{label}_raw"] = np.array([rep.raw_objective, rep.scaled_fitness])
        out[f"{label}_trace"] = np.array(rep.trace)
        out[f"{label}_evals"] = np.array([rep.evaluations])
        print(f"  ga {label}: raw={rep.raw_objective!r} evals={rep.evaluations}")
    save("big", **out)


if __name__ == "__main__":
    parts = sys.argv[1:] or ["cli", "rng", "instances", "eval", "operators", "ga", "restricted",
                             "big"]
    for part in parts:
        globals()[f"gen_{part}"]()
