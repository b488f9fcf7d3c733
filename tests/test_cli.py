"""Command line and file formats against the reference's own outputs
(tests/golden/cli.npz, written by make_golden.gen_cli from hubmedian.cli).
CPU-side: formats, fingerprints, manifests, exit codes.  The GPU-side CLI runs
(solve / oracle / eval / bench rows) are in test_gpu_parity.py::TestCli."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import golden

import paper_1704_06258_b200 as hg
from paper_1704_06258_b200 import cli, fileio


def test_fingerprints_match_reference():
    for prm, mode, fp in golden("cli")["fingerprints"]:
        isl, pop, inner, outer, seed, strength, strict = json.loads(prm)
        params = hg.GaParams(islands=isl, pop_size=pop, inner_iters=inner, outer_iters=outer,
                             seed=seed, perturb_strength=strength, strict_paper=strict)
        assert cli.params_fingerprint(params, hg.FitnessMode.from_string(mode)) == fp


@pytest.mark.parametrize("idx", range(2))
def test_gen_bytes_match_reference(idx, tmp_path):
    g = golden("cli")
    n, p, seed, alpha = g[f"gen{idx}_args"]
    out = tmp_path / "x.usaphmp"
    assert cli.main(["gen", "-n", str(int(n)), "-p", str(int(p)), "--seed", str(int(seed)),
                     "--alpha", repr(float(alpha)), "-o", str(out)]) == 0
    assert out.read_bytes() == g[f"gen{idx}_bytes"].tobytes()


@pytest.mark.parametrize("idx", range(2))
def test_parse_serialize_round_trip(idx):
    g = golden("cli")
    data = g[f"gen{idx}_bytes"].tobytes()
    inst = fileio.parse_instance(data)
    n, p, seed, alpha = g[f"gen{idx}_args"]
    ref = hg.generate_urand(int(n), int(p), int(seed), (1.0, float(alpha), 1.0))
    assert np.array_equal(inst.dist, ref.dist) and np.array_equal(inst.flow, ref.flow)
    assert fileio.serialize_instance(inst) == data


def test_coordinate_format():
    text = "# three nodes\n3 1\n1 0.5 1\n0 0\n3 4\n\n0 8\n0 1 2\n1 0 1\n2 1 0\n"
    inst = fileio.parse_instance(text, format=fileio.COORDINATE)
    assert inst.dist[0, 1] == 5.0 and inst.dist[1, 2] == 5.0 and inst.dist[0, 2] == 8.0
    assert inst.alpha == 0.5


@pytest.mark.parametrize("text,msg", [
    ("", "unexpected end of file, expected header 'n p'"),
    ("2\n", "line 1: expected 'n p', got 1 tokens"),
    ("2 x\n", "line 1: n and p must be integers"),
    ("2 3\n", "line 1: hub count p=3 outside [1, 2]"),
    ("2 1\n1 0 1\n", "line 2: cost factors must be positive"),
    ("2 1\n1 1 1\n0 1\n1 1\n0 0\n0 0\n", "line 4: distance diagonal entry 2 must be zero"),
    ("2 1\n1 1 1\n0 1\n1 0\n0 -1\n0 0\n", "line 5: negative value in flow row 1"),
    ("2 1\n1 1 1\n0 nan\n1 0\n0 0\n0 0\n", "line 3: non-finite value in distance row 1"),
    ("2 1\n1 1 1\n0 a\n1 0\n0 0\n0 0\n", "line 3: non-numeric token in distance row 1"),
    ("2 1\n1 1 1\n0 1\n1 0\n0 0\n0 0\nextra\n", "line 7: unexpected trailing content: 'extra'"),
])
def test_strict_parse_errors(text, msg):
    with pytest.raises(fileio.ParseError) as e:
        fileio.parse_instance(text)
    assert str(e.value) == msg


def test_solution_files():
    g = golden("cli")
    n, p, sol = fileio.read_solution(g["eval0_solution"].tobytes())
    assert (n, p) == (12, 3) and sol.hubs.tolist() == [1, 5, 9]
    assert fileio.write_solution(sol) == g["eval0_solution"].tobytes()
    with pytest.raises(fileio.ParseError, match="hub index outside"):
        fileio.read_solution("3 1\n4\n1 1 1\n")


def test_manifest_errors(tmp_path):
    m = tmp_path / "m.csv"
    m.write_text("label,path,mode\na,x.usaphmp,raw\n")
    with pytest.raises(cli.ManifestError, match="manifest header must be"):
        cli.read_manifest(m)
    m.write_text("label,path,format,p,mode,known_best\na,x.usaphmp,,,raw,-3\n")
    with pytest.raises(cli.ManifestError, match="row 2: known_best must be positive"):
        cli.read_manifest(m)


def test_exit_codes(tmp_path, capsys):
    assert cli.main(["solve"]) == cli.EXIT_USAGE
    assert cli.main(["solve", str(tmp_path / "missing.usaphmp")]) == cli.EXIT_DATA
    bad = tmp_path / "bad.usaphmp"
    bad.write_text("2 1\n")
    assert cli.main(["eval", str(bad), str(bad)]) == cli.EXIT_DATA
    assert "line 1" not in capsys.readouterr().out
