"""K3-TC/P ablations: the kernel time under each tuning switch, one
subprocess per configuration (the switches are read from the environment).

    python tools/k3_ablate.py [n p B]            # table of configurations
    python tools/k3_ablate.py --one [n p B]      # one measurement (internal)

Switches (paper_1704_06258_b200/csrc/k_fitness_tcp.cu): HUBGPU_TCP_NOTRI=1
(full W instead of its triangular fold), HUBGPU_TCP_DBG bits (1 no bin atomics,
2 no MMA, 4 no fold/reduce, 8 no one-hot generation, 64 no epilogue warps),
HUBGPU_TC_TIMING=1 (phase counters of the MMA issuer and epilogue warp 4).
Results are wrong under DBG; only the times mean something."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def one(n: int, p: int, B: int) -> dict:
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    import paper_1704_06258_b200 as hg
    from paper_1704_06258_b200 import _lib

    inst = hg.generate_urand(n, p, 1704, (1.0, 0.75, 1.0), device=True)
    d = inst.device()
    pop = _lib.DevicePopulation(d, B)
    pop.load_hubs(hg.random_population(n, p, B).astype(np.int32))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.ExternalStream(d.stream)
    ms = []
    with torch.cuda.stream(st):
        for k in range(13):
            flush.zero_()
            pop.evaluate(B)
            if k >= 3:
                ms.append(pop.last_fitness_ms())
    k2 = []
    with torch.cuda.stream(st):
        for _ in range(5):
            flush.zero_()
            pop.evaluate(B)
            k2.append(pop.last_allocate_ms())
    out = {"k3_ms": float(np.median(ms)), "k2_ms": float(np.median(k2)),
           "kernel": d.fitness_kernel}
    if os.environ.get("HUBGPU_TC_TIMING") == "1":
        buf = np.zeros(32, dtype=np.uint64)
        _lib.check(_lib.load().hg_debug_tc_timing(buf.ctypes.data_as(_lib._u64p)))
        pop.evaluate(B)
        d.synchronize()
        _lib.check(_lib.load().hg_debug_tc_timing(buf.ctypes.data_as(_lib._u64p)))
        m = buf[0:4].astype(float)
        e = buf[16:26].astype(float)
        out["mma_warp_pct"] = dict(zip(["waitA", "waitAccEmpty", "waitW", "issue"],
                                       (100 * m / max(m.sum(), 1)).round(1).tolist()))
        out["epi_warp_pct"] = dict(zip(["stage", "gen", "waitAcc", "bins", "reduce", "tmemld",
                                        "sync", "tload", "fold", "kbfwait"],
                                       (100 * e / max(e.sum(), 1)).round(1).tolist()))
    return out


CONFIGS = [
    ("default (tri)", {}),
    ("no bin atomics", {"HUBGPU_TCP_DBG": "1"}),
    ("no fold/reduce", {"HUBGPU_TCP_DBG": "4"}),
    ("no one-hot generation", {"HUBGPU_TCP_DBG": "8"}),
    ("no MMA", {"HUBGPU_TCP_DBG": "2"}),
    ("no MMA, no atomics", {"HUBGPU_TCP_DBG": "3"}),
    ("no MMA: drain + W only", {"HUBGPU_TCP_DBG": "15"}),
    ("no epilogue warps", {"HUBGPU_TCP_DBG": "64"}),
    ("no epilogue, no MMA: W stream", {"HUBGPU_TCP_DBG": "66"}),
    ("MMA issue alone (no epilogue, no W stream)", {"HUBGPU_TCP_DBG": "112"}),
    ("full W", {"HUBGPU_TCP_NOTRI": "1"}),
]
# (phase counters, HUBGPU_TC_TIMING=1, need a timing build: make EXTRA=-DHG_TCP_TIMING)


def main() -> None:
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n, p, B = (int(a) for a in (args if len(args) == 3 else (1000, 20, 8192)))
    if "--one" in sys.argv:
        print(json.dumps(one(n, p, B)))
        return
    rows = []
    for name, env in CONFIGS:
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, __file__, "--one", str(n), str(p), str(B)], env=e,
                           capture_output=True, text=True, timeout=300)
        try:
            res = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            res = {"error": (r.stderr or r.stdout)[-300:]}
        res["config"] = name
        rows.append(res)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
