"""Host-side logic of the package and the C-ABI boundary (CPU only)."""

from __future__ import annotations

import hashlib
import re

import numpy as np
import pytest

from conftest import ROOT, golden, orc

import paper_1704_06258_b200 as hg
from paper_1704_06258_b200 import _lib


class TestLibraryBoundary:
    def test_library_exports_every_header_symbol(self):
        header = (ROOT / "include" / "hubgpu.h").read_text()
        declared = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(hg_\w+)\(", header, re.M))
        assert len(declared) >= 25
        lib = _lib.load()
        for name in declared:
            assert hasattr(lib, name), name
        assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)

    def test_version(self):
        assert _lib.load().hg_version() == 100

    def test_fails_loudly_without_a_device(self):
        if _lib.device_count() > 0:
            pytest.skip("a GPU is visible")
        inst = hg.generate_urand(8, 2, 1, (1.0, 0.75, 1.0))
        with pytest.raises(_lib.HubGpuError, match="no CUDA device"):
            hg.nearest_allocation([0, 1], inst)
        with pytest.raises(_lib.HubGpuError):
            hg.objective(inst, hg.Solution(hub=np.eye(8, dtype=bool)[0] | np.eye(8, dtype=bool)[1],
                                           alloc=np.array([0, 1, 0, 0, 0, 0, 0, 0])))


class TestInstance:
    def test_derived_vectors(self):
        inst = hg.Instance(n=2, p=1, dist=np.array([[0.0, 1.0], [1.0, 0.0]]),
                           flow=np.array([[0.0, 5.0], [3.0, 2.0]]), chi=1.0, alpha=0.5, delta=1.0)
        assert inst.out_flow.tolist() == [5.0, 5.0]
        assert inst.in_flow.tolist() == [3.0, 7.0]
        assert inst.total_flow == 10.0

    @pytest.mark.parametrize("kw,match", [
        (dict(dist=np.array([[1.0, 1.0], [1.0, 0.0]])), "diagonal"),
        (dict(dist=np.array([[0.0, -1.0], [1.0, 0.0]])), "negative"),
        (dict(flow=np.array([[0.0, np.inf], [0.0, 0.0]])), "non-finite"),
        (dict(p=3), "hub count"),
        (dict(chi=0.0), "chi must be a positive"),
        (dict(dist=np.zeros((3, 3))), "dist must be 2x2"),
    ])
    def test_rejections(self, kw, match):
        args = dict(n=2, p=1, dist=np.zeros((2, 2)), flow=np.zeros((2, 2)), chi=1, alpha=1,
                    delta=1)
        args.update(kw)
        with pytest.raises(ValueError, match=match):
            hg.Instance(**args)

    def test_read_only_and_middle_rank(self):
        g = golden("instances")
        for idx in range(3):
            inst = hg.Instance(*[int(v) for v in g[f"mk{idx}_meta"][:2]], g[f"mk{idx}_dist"],
                               g[f"mk{idx}_flow"], *[float(v) for v in g[f"mk{idx}_meta"][2:]])
            assert np.array_equal(inst.middle_rank, g[f"mk{idx}_rank"])
            with pytest.raises(ValueError):
                inst.dist[0, 1] = 7.0
        assert np.array_equal(hg.middle_nodes(inst, 3), g["mk2_rank"][:3])
        with pytest.raises(ValueError):
            hg.middle_nodes(inst, 0)


class TestGenerator:
    @pytest.mark.parametrize("idx", range(4))
    def test_small_bitwise(self, idx):
        g = golden("instances")
        n, p, seed, *f = g[f"urand{idx}_args"]
        inst = hg.generate_urand(int(n), int(p), int(seed), tuple(f))
        assert np.array_equal(inst.dist, g[f"urand{idx}_dist"])
        assert np.array_equal(inst.flow, g[f"urand{idx}_flow"])

    def test_ur_digest(self):
        g = golden("instances")
        n, p, seed, *f = g["big1_args"]
        inst = hg.generate_urand(int(n), int(p), int(seed), tuple(f))
        assert hashlib.sha256(inst.dist.tobytes()).hexdigest() == str(g["big1_sha"][0])
        assert hashlib.sha256(inst.flow.tobytes()).hexdigest() == str(g["big1_sha"][1])
        assert inst.total_flow == float(g["big1_total"][0])

    def test_population_matches_oracle(self):
        for n, p in ((25, 3), (200, 10), (70, 40), (5, 5)):
            assert np.array_equal(hg.random_population(n, p, 40),
                                  orc.bench_population(n, p, 40))
        assert np.array_equal(hg.random_population(200, 10, 48),
                              golden("evaluation")["ap_hubs"])


class TestRng:
    def test_streams_match_reference(self):
        g = golden("rng")
        assert hg.mix64(0x9E3779B97F4A7C15) == int(g["kat"][0])
        st = hg.derive_stream(1704, 1000, 20)
        ref = orc.Stream(orc.stream_key(1704, 1000, 20))
        assert [st.next_u64() for _ in range(50)] == [ref.u64() for _ in range(50)]
        a, b = hg.RngStream(11), hg.RngStream(11)
        assert a.randint_block(64, 7).tolist() == [b.randint(7) for _ in range(64)]
        with pytest.raises(ValueError):
            hg.RngStream(1).randint(0)

    def test_resolve_rng_keys(self):
        a = hg.resolve_rng(42, 3, hg.Role.MUTATION)
        assert a.state == orc.stream_key(42, 3, 2)


class TestParamsAndScaling:
    def test_ga_params(self):
        with pytest.raises(ValueError, match="even"):
            hg.GaParams(pop_size=15)
        with pytest.raises(ValueError):
            hg.GaParams(islands=0)
        assert hg.GaParams().resolved_strength(2) == 2
        assert hg.GaParams().resolved_strength(10) == 3
        with pytest.raises(ValueError, match="exceeds p"):
            hg.GaParams(perturb_strength=5).resolved_strength(2)

    def test_scale_identities(self):
        raw = 167493060.0
        assert hg.scale(raw, hg.FitnessMode.STANDARD_MILLI, 1.0) == raw * 1e-3 == 167493.06
        assert hg.scale(raw, hg.FitnessMode.CAB_NORMALIZED, 7.0) == raw / 7.0
        with pytest.raises(hg.ZeroTotalFlowError):
            hg.scale(raw, hg.FitnessMode.CAB_NORMALIZED, 0.0)
        assert hg.FitnessMode.from_string("CAB") is hg.FitnessMode.CAB_NORMALIZED
        with pytest.raises(ValueError):
            hg.FitnessMode.from_string("bogus")

    def test_island_shards_cover_in_order(self):
        for R in (1, 7, 64, 128):
            for world in (1, 2, 3, 4, 8):
                spans = [hg.island_shard(R, r, world) for r in range(world)]
                assert spans[0][0] == 0 and spans[-1][1] == R
                assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


class TestValidate:
    def test_messages(self):
        inst = hg.Instance(n=3, p=2, dist=np.zeros((3, 3)), flow=np.ones((3, 3)), chi=1, alpha=1,
                           delta=1)
        sol = hg.Solution(hub=np.array([True, True, False]), alloc=np.array([0, 1, 2]))
        res = hg.validate(sol, inst)
        assert not res.ok and any("node 3" in v and "closed" in v for v in res.violations)
        sol = hg.Solution(hub=np.array([True, True, False]), alloc=np.array([1, 1, 1]))
        assert any("hub 1 not allocated to itself" in v for v in hg.validate(sol, inst).violations)
        with pytest.raises(hg.StructureError):
            hg.validate(hg.Solution(hub=np.array([True, False, False]),
                                    alloc=np.array([0, 0, 5])), inst)
        with pytest.raises(hg.InfeasibleSolutionError):
            hg.objective(inst, hg.Solution(hub=np.array([True, False, False]),
                                           alloc=np.array([0, 0, 0])))


def test_enumeration_limit_raised_on_host():
    """restricted_optimum checks C(n, p) against the limit before any device
    work, with the reference's exception and message (hm/oracle.py:32-40)."""
    inst = hg.generate_urand(30, 5, 2, (1.0, 0.75, 1.0))
    with pytest.raises(hg.EnumerationLimitError) as e:
        hg.restricted_optimum(inst, limit=1000)
    assert e.value.required == 142506 and e.value.limit == 1000
    assert str(e.value) == ("enumeration needs 142506 candidates, over the limit of 1000; "
                            "raise `limit` explicitly to allow it")
    assert isinstance(e.value, ValueError)


def test_bench_reference_arm_line():
    """bench.py --impl reference prints the contract's JSON line on the host
    cores (no GPU needed)."""
    import json
    import subprocess
    import sys

    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "3", "--ref-seconds", "0.05"],
                         capture_output=True, text=True, timeout=300, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["steps"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_philox_known_answers():
    """The GA's optional Philox4x32-10 generator (rng='philox') against the
    Random123 known-answer vectors (host entry of the same inline function the
    kernels use)."""
    kat = [([0, 0], [0, 0, 0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
           ([0xFFFFFFFF] * 2, [0xFFFFFFFF] * 4, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
           ([0xA4093822, 0x299F31D0], [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
            [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1])]
    for key, ctr, want in kat:
        assert _lib.philox4x32_10(key, ctr) == want


def test_rng_mode_validated():
    with pytest.raises(ValueError, match="rng must be"):
        hg.GaParams(rng="mt19937")
    assert hg.GaParams().rng == "replay"


def _replay_pairwise(a: np.ndarray) -> float:
    """The exact mode's device algorithm, step for step, in Python: per leaf
    the 8 strided accumulators (rows of 8 terms), their fixed combine, the
    last leaf's partial row term by term, then the tree sums on a stack."""
    m = a.size
    table = _lib.pairwise_leaves(m)
    rows, tail = m // 8, m % 8
    stack = []
    for k, e in enumerate(table):
        r0, nr, nsum = int(e & 0xFFFF), int((e >> 16) & 0xFF), int(e >> 24)
        last = k == len(table) - 1
        if nr == 0:
            acc = [0.0] * 8
        else:
            acc = [float(a[8 * r0 + j]) for j in range(8)]
            for q in range(1, nr):
                for j in range(8):
                    acc[j] = acc[j] + float(a[8 * (r0 + q) + j])
        c = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))
        if last:
            for u in range(tail):
                c = c + float(a[8 * rows + u])
        stack.append(c)
        for _ in range(len(stack) - 1 if last else nsum):
            right = stack.pop()
            stack[-1] = stack[-1] + right
    return stack[0]


@pytest.mark.parametrize("m", [0, 1, 5, 7, 8, 9, 15, 16, 100, 127, 128, 129, 136, 257, 400,
                               1000, 1024, 1030, 2100, 4096, 6000, 16384])
def test_pairwise_leaf_table_replays_numpy_sum(m):
    """hg_pairwise_leaves (the table exact mode replays on the device) gives
    np.sum's value bit for bit (hm/evaluation.py:110-118 sum products this
    way); leaves hold <= 16 rows and start on rows of 8."""
    rng = np.random.default_rng(m)
    a = rng.random(m) * rng.random(m) * 1e6
    table = _lib.pairwise_leaves(m)
    assert all(((e >> 16) & 0xFF) <= 16 for e in table)
    if m == 0:
        return
    assert _replay_pairwise(a) == float(np.sum(a))


class TestPinnedPool:
    """The pooled page-locked result buffers (_lib._PinnedPool) with a host
    stand-in for hg_host_alloc / hg_host_free (no GPU needed)."""

    class _StubLib:
        def __init__(self):
            import ctypes as C

            self.C = C
            self.blocks = {}
            self.freed = []

        def hg_host_alloc(self, nbytes, out):
            buf = (self.C.c_char * nbytes)()
            addr = self.C.addressof(buf)
            self.blocks[addr] = buf
            out._obj.value = addr
            return 0

        def hg_host_free(self, addr):
            self.freed.append(addr)

    def test_view_keeps_block(self, monkeypatch):
        import gc

        stub = self._StubLib()
        monkeypatch.setattr(_lib, "load", lambda: stub)
        pool = _lib._PinnedPool()
        a = pool.array((4, 4), np.float64)
        a[:] = 1.0
        col = a[:, 3]
        del a
        gc.collect()
        b = pool.array((4, 4), np.float64)  # must not reuse the block `col` views
        b[:] = 2.0
        assert col.tolist() == [1.0] * 4
        del b, col
        gc.collect()
        assert sum(len(v) for v in pool._free.values()) == 2

    def test_block_returns_after_last_view(self, monkeypatch):
        import gc

        stub = self._StubLib()
        monkeypatch.setattr(_lib, "load", lambda: stub)
        pool = _lib._PinnedPool()
        a = pool.array((8, 4), np.float64)
        v = a.reshape(-1)[5:]
        del a
        gc.collect()
        assert not pool._free.get(8 * 4 * 8)
        del v
        gc.collect()
        assert len(pool._free[8 * 4 * 8]) == 1
