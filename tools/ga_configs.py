"""Island-GA generation throughput on the BASELINE configs (one GPU):
AP n=200 p=10 (pop 1024), UR n=1000 p=20 (128 x 64), BIG n=6000 p=50
(16 islands x 64 = one GPU's share of 128 islands over 8).  Prints JSON lines.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402

CONFIGS = [("AP", 200, 10, (3.0, 0.75, 2.0), 16, 64),
           ("UR", 1000, 20, (1.0, 0.75, 1.0), 128, 64),
           ("BIG", 6000, 50, (1.0, 0.75, 1.0), 16, 64)]
for name, n, p, f, R, pop in CONFIGS:
    inst = hg.generate_urand(n, p, 1704, f, device=True)
    d = inst.device()
    ga = hg._lib.DeviceGa(d, R, 0, R, pop, min(p, 3), False, 0)
    ga.begin_round(np.sort(inst.middle_rank[:p]))
    stream = torch.cuda.ExternalStream(d.stream)
    with torch.cuda.stream(stream):
        ga.generations(3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gens = 20 if n < 6000 else 5
        a.record(stream)
        ga.generations(gens)
        b.record(stream)
        b.synchronize()
    ms = a.elapsed_time(b) / gens
    print(json.dumps({"config": name, "n": n, "p": p, "islands": R, "pop": pop,
                      "ms_per_generation": ms, "child_evals_per_s": R * pop / (ms * 1e-3),
                      "kernel": d.fitness_kernel}), flush=True)
