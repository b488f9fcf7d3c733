"""Per-generation duplicate grouping in the device GA: time one
generation with HUBGPU_GA_DEDUPE=0 and =1 on the BASELINE GA shapes and check
the two runs are identical (round results, last children and their costs).

    python tools/ga_dedupe_probe.py [--out profiles/ga_dedupe_r2.json]

Each setting runs in its own process (the switch is read once, at GA
creation). 128 islands x pop 64, strength from the reference's rule, 3 warm-up
generations, 50 timed generations with CUDA events on the instance stream.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
SHAPES = {  # name: (n, p, factors)
    "cab": (25, 3, (1.0, 0.2, 1.0)),
    "cab4": (25, 4, (1.0, 0.2, 1.0)),
    "ap": (200, 10, (3.0, 0.75, 2.0)),
    "ur": (1000, 20, (1.0, 0.75, 1.0)),
}


def child(name: str, dedupe: int, dump: str) -> dict:
    os.environ["HUBGPU_GA_DEDUPE"] = str(dedupe)
    sys.path.insert(0, str(ROOT))
    import torch

    import paper_1704_06258_b200 as hg

    n, p, f = SHAPES[name]
    inst = hg.generate_urand(n, p, 1704, f)
    dinst = hg._lib.device_instance(inst)
    strength = hg.GaParams(islands=128, pop_size=64).resolved_strength(p)
    ga = hg._lib.DeviceGa(dinst, 128, 0, 128, 64, strength, False, 7)
    ga.begin_round(np.sort(inst.middle_rank[:p]))
    stream = torch.cuda.ExternalStream(dinst.stream)  # the GA's graphs run there
    ga.generations(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ga.generations(50)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    raw, hubs = ga.round_results()
    khubs, kraw = ga.last_children()
    np.savez(dump, raw=raw, hubs=hubs, khubs=khubs, kraw=kraw)
    distinct = len({tuple(r) for r in khubs.tolist()})
    return {"ms_per_generation": ms, "launches_per_generation": ga.launches_per_generation,
            "children": int(khubs.shape[0]), "distinct_last_children": distinct}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "ga_dedupe_r2.json"))
    ap.add_argument("--child", nargs=3)
    a = ap.parse_args()
    if a.child:
        print(json.dumps(child(a.child[0], int(a.child[1]), a.child[2])))
        return
    res = {}
    for name in SHAPES:
        row = {}
        dumps = {}
        for d in (0, 1):
            dumps[d] = f"/tmp/ga_dedupe_{name}_{d}.npz"
            out = subprocess.run([sys.executable, __file__, "--child", name, str(d), dumps[d]],
                                 capture_output=True, text=True, check=True)
            row[f"dedupe={d}"] = json.loads(out.stdout.strip().splitlines()[-1])
        x, y = np.load(dumps[0]), np.load(dumps[1])
        row["identical"] = all(np.array_equal(x[k], y[k]) for k in ("raw", "hubs", "khubs", "kraw"))
        row["speedup"] = row["dedupe=0"]["ms_per_generation"] / row["dedupe=1"]["ms_per_generation"]
        row["shape"] = {"n": SHAPES[name][0], "p": SHAPES[name][1], "islands": 128, "pop": 64}
        res[name] = row
        print(name, json.dumps(row), flush=True)
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
