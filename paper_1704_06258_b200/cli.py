"""Command line: ``python -m paper_1704_06258_b200 <command> ...`` (the
subcommands and machine output of hm/cli.py:62-120 and hm/bench.py:27-33, with
every solve / evaluation running on the GPU).

Commands: ``solve`` (island GA on an instance file), ``eval`` (score a
solution file), ``gen`` (random Euclidean instance; ``--device`` draws it on
the GPU), ``oracle`` (restricted optimum by full hub-set sweep on the GPU),
``bench`` (a manifest of instances x seeds against known bests) and ``sweep``
(solve over a grid of cost factors).  Machine-readable rows use CSV schema v1
(``BENCH_CSV_HEADER``); a row embeds the seed and a fingerprint of the other
parameters, so runs on either implementation compare row by row.

Exit codes: 0 ok, 1 usage error, 2 data error (parse, manifest, enumeration
limit, infeasible solution), 3 benchmark gap threshold exceeded, 4 internal
invariant violated (an infeasible best solution or a rising elitist trace).
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import hashlib
import itertools
import sys
from dataclasses import dataclass
from pathlib import Path

from . import fileio
from .engine import GaParams, SolveReport, solve
from .evaluation import (FitnessMode, InfeasibleSolutionError, StatisticUndefinedError,
                         avg_interhub_distance, objective)
from .exhaustive import restricted_optimum
from .io import generate_urand
from .model import Instance, validate

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_GAP, EXIT_INVARIANT = 0, 1, 2, 3, 4

BENCH_CSV_SCHEMA = "v1"
BENCH_CSV_HEADER = ("label,n,p,mode,seed,achieved,known_best,gap,"
                    "evaluations,wall_time_s,params_fingerprint")
SWEEP_CSV_HEADER = "chi,delta,alpha,fitness,avg_interhub_distance"
MANIFEST_HEADER = ["label", "path", "format", "p", "mode", "known_best"]
NEGATIVE_GAP_ALARM = -1e-6  # beating a proven optimum by more is a units/data error


class UsageError(Exception):
    pass


class InvariantError(Exception):
    pass


class ManifestError(ValueError):
    pass


# ---------------------------------------------------------------------------
# rows (schema v1)
# ---------------------------------------------------------------------------


def params_fingerprint(params: GaParams, mode: FitnessMode) -> str:
    """12 hex digits of sha256 over every search parameter but the seed; the
    same text as hm/bench.py:93-97, so fingerprints agree across the two
    implementations."""
    text = "|".join([BENCH_CSV_SCHEMA, f"islands={params.islands}", f"pop={params.pop_size}",
                     f"inner={params.inner_iters}", f"outer={params.outer_iters}",
                     f"perturb={params.perturb_strength}", f"strict={params.strict_paper}",
                     f"mode={mode.value}"])
    return hashlib.sha256(text.encode()).hexdigest()[:12]


@dataclass(frozen=True)
class Row:
    label: str
    n: int
    p: int
    mode: FitnessMode
    seed: int
    achieved: float
    known_best: float | None
    evaluations: int
    wall_time_s: float
    fingerprint: str

    @property
    def gap(self) -> float | None:
        if self.known_best is None:
            return None
        return (self.achieved - self.known_best) / self.known_best

    @property
    def anomalous(self) -> bool:
        return self.gap is not None and self.gap < NEGATIVE_GAP_ALARM

    def csv(self) -> str:
        opt = (lambda v: "" if v is None else repr(v))
        return ",".join([self.label, str(self.n), str(self.p), self.mode.value, str(self.seed),
                         repr(self.achieved), opt(self.known_best), opt(self.gap),
                         str(self.evaluations), repr(self.wall_time_s), self.fingerprint])


def make_row(label: str, inst: Instance, rep: SolveReport, mode: FitnessMode, params: GaParams,
             known_best: float | None = None) -> Row:
    return Row(label, inst.n, inst.p, mode, params.seed, rep.scaled_fitness, known_best,
               rep.evaluations, rep.wall_time, params_fingerprint(params, mode))


def rows_csv(rows) -> str:
    return "\n".join([BENCH_CSV_HEADER] + [r.csv() for r in rows]) + "\n"


# ---------------------------------------------------------------------------
# manifests
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class ManifestEntry:
    label: str
    path: Path
    format: str
    p: int | None
    mode: FitnessMode
    known_best: float | None


def read_manifest(path) -> list[ManifestEntry]:
    """CSV ``label,path,format,p,mode,known_best`` (paths relative to the
    manifest; format / p / known_best may be empty; ``#`` lines skipped)."""
    path = Path(path)
    lines = [ln for ln in path.read_text().splitlines()
             if ln.strip() and not ln.lstrip().startswith("#")]
    reader = csv.DictReader(lines)
    if reader.fieldnames != MANIFEST_HEADER:
        raise ManifestError(f"manifest header must be {','.join(MANIFEST_HEADER)}, "
                            f"got {reader.fieldnames}")
    out = []
    for lineno, rec in enumerate(reader, start=2):
        try:
            ipath = path.parent / rec["path"].strip()
            fmt = rec["format"].strip() or fileio.format_for_path(ipath)
            p = int(rec["p"]) if rec["p"].strip() else None
            mode = FitnessMode.from_string(rec["mode"].strip())
            kb = float(rec["known_best"]) if rec["known_best"].strip() else None
            if kb is not None and not kb > 0:
                raise ValueError(f"known_best must be positive, got {kb}")
        except (ValueError, KeyError, AttributeError, TypeError) as exc:
            raise ManifestError(f"manifest row {lineno}: {exc}") from None
        out.append(ManifestEntry(rec["label"].strip(), ipath, fmt, p, mode, kb))
    return out


# ---------------------------------------------------------------------------
# commands
# ---------------------------------------------------------------------------


def _params(ns) -> GaParams:
    try:
        return GaParams(islands=ns.islands, pop_size=ns.pop, inner_iters=ns.inner,
                        outer_iters=ns.outer, seed=ns.seed, perturb_strength=ns.perturb,
                        strict_paper=ns.strict_paper)
    except ValueError as exc:
        raise UsageError(str(exc)) from None


def _instance(path: Path, fmt, p=None) -> Instance:
    inst = fileio.load_instance(path, format=fmt)
    if p is not None:
        try:
            inst = inst.with_p(p)
        except ValueError as exc:
            raise UsageError(str(exc)) from None
    return inst


def _strength_ok(params: GaParams, inst: Instance) -> None:
    try:
        params.resolved_strength(inst.p)
    except ValueError as exc:
        raise UsageError(str(exc)) from None


def _check(rep: SolveReport, inst: Instance, strict: bool) -> None:
    if not validate(rep.best_solution, inst).ok:
        raise InvariantError("engine returned an infeasible solution")
    if not strict and any(b > a for a, b in zip(rep.trace, rep.trace[1:])):
        raise InvariantError("engine trace is not nonincreasing")


def _emit(text: str, target) -> None:
    if target == "-":
        sys.stdout.write(text)
    elif target is not None:
        Path(target).write_text(text)


def _one_based(idx) -> str:
    return " ".join(str(int(i) + 1) for i in idx)


def cmd_solve(ns) -> int:
    inst = _instance(ns.instance, ns.format, ns.p)
    params = _params(ns)
    _strength_ok(params, inst)
    mode = FitnessMode.from_string(ns.fitness_mode)
    rep = solve(inst, params, mode, workers=ns.workers)
    _check(rep, inst, params.strict_paper)
    label = inst.name or ns.instance.stem
    if ns.csv != "-":
        print(f"instance       {label}  (n={inst.n}, p={inst.p})")
        print(f"params         islands={params.islands} pop={params.pop_size} "
              f"inner={params.inner_iters} outer={params.outer_iters} "
              f"perturb={params.resolved_strength(inst.p)} "
              f"strict_paper={params.strict_paper} seed={params.seed}")
        print(f"fitness mode   {mode.value}")
        print(f"raw objective  {rep.raw_objective!r}")
        print(f"fitness        {rep.scaled_fitness!r}")
        print(f"hubs (1-based) {_one_based(rep.best_solution.hubs)}")
        print(f"evaluations    {rep.evaluations}")
        print(f"wall time      {rep.wall_time:.3f} s")
        print("trace          " + " ".join(f"{v:.6g}" for v in rep.trace))
        if rep.interrupted:
            print("NOTE: run interrupted; best-so-far reported")
    _emit(rows_csv([make_row(label, inst, rep, mode, params)]), ns.csv)
    return EXIT_OK


def cmd_eval(ns) -> int:
    inst = _instance(ns.instance, ns.format)
    n, p, sol = fileio.read_solution(ns.solution.read_bytes())
    if n != inst.n:
        raise fileio.ParseError(f"solution is for n={n}, instance has n={inst.n}")
    if p != inst.p:
        raise fileio.ParseError(f"solution is for p={p}, instance has p={inst.p}")
    mode = FitnessMode.from_string(ns.fitness_mode)
    try:
        bd = objective(inst, sol, mode)
    except InfeasibleSolutionError as exc:
        print("infeasible solution:", file=sys.stderr)
        for v in exc.violations:
            print(f"  - {v}", file=sys.stderr)
        return EXIT_DATA
    for label, v in (("collection", bd.collection_cost), ("transfer", bd.transfer_cost),
                     ("distribution", bd.distribution_cost), ("raw total", bd.raw_total)):
        print(f"{label:<15}{v!r}")
    print(f"fitness ({mode.value}) {bd.scaled_fitness!r}")
    return EXIT_OK


def cmd_gen(ns) -> int:
    try:
        inst = generate_urand(ns.nodes, ns.hubs, ns.seed, (ns.chi, ns.alpha, ns.delta),
                              device=ns.device)
    except ValueError as exc:
        raise UsageError(str(exc)) from None
    data = fileio.serialize_instance(inst)
    ns.out.write_bytes(data)
    print(f"wrote {ns.out}  n={inst.n} p={inst.p} sha256={fileio.sha256_hex(data)}")
    return EXIT_OK


def cmd_oracle(ns) -> int:
    if ns.which in ("exact", "both"):
        raise UsageError("exact_optimum (hub sets x spoke assignments) is not provided; "
                         "use --which restricted")
    inst = _instance(ns.instance, ns.format, ns.p)
    sol, raw = restricted_optimum(inst, limit=ns.limit)
    print(f"restricted optimum  {raw!r}")
    print(f"  hubs (1-based)    {_one_based(sol.hubs)}")
    return EXIT_OK


def cmd_bench(ns) -> int:
    entries = read_manifest(ns.manifest)
    params = _params(ns)
    try:
        seeds = [int(t) for t in ns.seeds.split(",") if t.strip()]
    except ValueError:
        raise UsageError(f"bad seed list {ns.seeds!r}") from None
    if not seeds:
        raise UsageError("at least one seed is required")
    rows, failures = [], []
    for e in entries:
        try:
            inst = fileio.load_instance(e.path, format=e.format)
            if e.p is not None:
                inst = inst.with_p(e.p)
        except (OSError, ValueError) as exc:
            failures.append((e.label, str(exc)))
            print(f"{e.label}: FAILED ({exc})")
            continue
        mine = []
        for seed in seeds:
            rp = dataclasses.replace(params, seed=seed)
            row = make_row(e.label, inst, solve(inst, rp, e.mode, workers=ns.workers), e.mode,
                           rp, known_best=e.known_best)
            rows.append(row)
            mine.append(row)
            gap = "" if row.gap is None else f"  gap={row.gap:+.3e}"
            print(f"{row.label}  seed={row.seed}  achieved={row.achieved:.6f}{gap}"
                  f"  t={row.wall_time_s:.2f}s")
        gaps = [r.gap for r in mine if r.gap is not None]
        extra = (f"  best_gap={min(gaps):+.3e}  mean_gap={sum(gaps) / len(gaps):+.3e}"
                 if gaps else "")
        print(f"summary {e.label}: best={min(r.achieved for r in mine):.6f}{extra}")
    _emit(rows_csv(rows), ns.csv)
    for label, msg in failures:
        print(f"FAILED {label}: {msg}", file=sys.stderr)
    for r in rows:
        if r.anomalous:
            print(f"ALARM {r.label} seed={r.seed}: achieved beats the recorded known best by "
                  f"{-r.gap:.3e} (relative); check units/data", file=sys.stderr)
    if failures or any(r.anomalous for r in rows):
        return EXIT_DATA
    if ns.gap_threshold is not None:
        gaps = [r.gap for r in rows if r.gap is not None]
        if gaps and max(gaps) > ns.gap_threshold:
            print(f"gap threshold exceeded: {max(gaps):.3e} > {ns.gap_threshold:.3e}",
                  file=sys.stderr)
            return EXIT_GAP
    return EXIT_OK


def _floats(text):
    if text is None:
        return None
    try:
        return [float(t) for t in text.split(",") if t.strip()]
    except ValueError:
        raise UsageError(f"bad float list {text!r}") from None


def cmd_sweep(ns) -> int:
    inst = _instance(ns.instance, ns.format)
    params = _params(ns)
    _strength_ok(params, inst)
    mode = FitnessMode.from_string(ns.fitness_mode)
    grid = itertools.product(_floats(ns.chis) or [inst.chi], _floats(ns.deltas) or [inst.delta],
                             _floats(ns.alphas) or [inst.alpha])
    out = [SWEEP_CSV_HEADER]
    for chi, delta, alpha in grid:
        point = inst.with_factors(chi=chi, alpha=alpha, delta=delta)
        rep = solve(point, params, mode, workers=ns.workers)
        try:
            avg = repr(avg_interhub_distance(point, rep.best_solution))
        except StatisticUndefinedError:
            avg = ""
        out.append(",".join([repr(chi), repr(delta), repr(alpha), repr(rep.scaled_fitness), avg]))
    text = "\n".join(out) + "\n"
    if ns.csv is None:
        sys.stdout.write(text)
    else:
        _emit(text, ns.csv)
    return EXIT_OK


# ---------------------------------------------------------------------------
# parser
# ---------------------------------------------------------------------------


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def _ga_args(sp) -> None:
    sp.add_argument("--seed", type=int, default=0)
    sp.add_argument("--islands", type=int, default=64)
    sp.add_argument("--pop", type=int, default=64)
    sp.add_argument("--inner", type=int, default=50)
    sp.add_argument("--outer", type=int, default=10)
    sp.add_argument("--perturb", type=int, default=None)
    sp.add_argument("--strict-paper", action="store_true")
    sp.add_argument("--workers", type=int, default=None,
                    help="accepted for compatibility; never affects results")


def build_parser() -> _Parser:
    ap = _Parser(prog="python -m paper_1704_06258_b200",
                 description="p-hub median on B200: GA, evaluation, oracle, benchmarks")
    sub = ap.add_subparsers(dest="command", required=True)
    fmt = dict(default=None, choices=[fileio.CANONICAL, fileio.COORDINATE])
    modes = dict(default="raw", choices=["cab", "milli", "raw"])

    s = sub.add_parser("solve")
    s.add_argument("instance", type=Path)
    s.add_argument("--p", type=int, default=None)
    s.add_argument("--csv", default=None)
    s.add_argument("--format", **fmt)
    s.add_argument("--fitness-mode", **modes)
    _ga_args(s)

    s = sub.add_parser("eval")
    s.add_argument("instance", type=Path)
    s.add_argument("solution", type=Path)
    s.add_argument("--format", **fmt)
    s.add_argument("--fitness-mode", **modes)

    s = sub.add_parser("gen")
    s.add_argument("-n", "--nodes", type=int, required=True)
    s.add_argument("-p", "--hubs", type=int, required=True)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--alpha", type=float, required=True)
    s.add_argument("--chi", type=float, default=1.0)
    s.add_argument("--delta", type=float, default=1.0)
    s.add_argument("-o", "--out", type=Path, required=True)
    s.add_argument("--device", action="store_true", help="draw the instance on the GPU")

    s = sub.add_parser("oracle")
    s.add_argument("instance", type=Path)
    s.add_argument("--p", type=int, default=None)
    s.add_argument("--which", default="restricted", choices=["exact", "restricted", "both"])
    s.add_argument("--limit", type=int, default=10_000_000)
    s.add_argument("--format", **fmt)

    s = sub.add_parser("bench")
    s.add_argument("manifest", type=Path)
    s.add_argument("--seeds", default="0")
    s.add_argument("--gap-threshold", type=float, default=None)
    s.add_argument("--csv", default=None)
    _ga_args(s)

    s = sub.add_parser("sweep")
    s.add_argument("instance", type=Path)
    s.add_argument("--chis", default=None)
    s.add_argument("--deltas", default=None)
    s.add_argument("--alphas", default=None)
    s.add_argument("--csv", default=None)
    s.add_argument("--format", **fmt)
    s.add_argument("--fitness-mode", **modes)
    _ga_args(s)
    return ap


COMMANDS = {"solve": cmd_solve, "eval": cmd_eval, "gen": cmd_gen, "oracle": cmd_oracle,
            "bench": cmd_bench, "sweep": cmd_sweep}


def main(argv=None) -> int:
    # the reference's own numbers, digit for digit: cost sums in numpy's
    # pairwise order while a command runs
    from . import _lib

    prev = _lib.exact_default()
    _lib.set_exact_default(True)
    try:
        ns = build_parser().parse_args(argv)
        return COMMANDS[ns.command](ns)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_DATA
    except InvariantError as exc:
        print(f"internal invariant violation: {exc}", file=sys.stderr)
        return EXIT_INVARIANT
    except RuntimeError as exc:  # no usable GPU / CUDA failure (HubGpuError)
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_DATA
    finally:
        _lib.set_exact_default(prev)


__all__ = ["main", "build_parser", "params_fingerprint", "read_manifest", "rows_csv",
           "BENCH_CSV_HEADER", "SWEEP_CSV_HEADER"]
