"""Fitness-eval throughput sweep (BASELINE configs[4]):
population B x n x p on one GPU, device-resident hub sets, L2 flushed between
steps, CUDA-event timed (K2 + K3 + finalise).  Prints one JSON line per point.

    python tools/sweep.py [--quick]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402
from paper_1704_06258_b200 import _lib  # noqa: E402

quick = "--quick" in sys.argv
ns = [200, 1000, 6000]
ps = [5, 20, 50]
Bs = [4096, 16384, 65536] if quick else [4096, 8192, 16384, 32768, 65536]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in ns:
    insts = {}
    for p in ps:
        inst = hg.generate_urand(n, p, 1704, (1.0, 0.75, 1.0), device=True)
        d = inst.device()
        stream = torch.cuda.ExternalStream(d.stream)
        for B in Bs:
            pop = hg.random_population(n, p, B).astype(np.int32)
            popd = _lib.DevicePopulation(d, B)
            popd.load_hubs(pop)
            steps = 20 if n < 6000 else 5
            with torch.cuda.stream(stream):
                for _ in range(3):
                    popd.evaluate(B)
                ms = []
                for _ in range(steps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    popd.evaluate(B)
                    b.record(stream)
                    b.synchronize()
                    ms.append(a.elapsed_time(b))
                fit = []
                for _ in range(3):
                    flush.zero_()
                    popd.evaluate(B)
                    fit.append(popd.last_fitness_ms())
            t = float(np.median(ms))
            evals = B / (t * 1e-3)
            alg = 8.0 * n * n + 4.0 * n
            print(json.dumps({"n": n, "p": p, "B": B, "kernel": d.fitness_kernel,
                              "step_ms": t, "k3_ms": float(np.median(fit)),
                              "evals_per_s": evals,
                              "hbm_roofline_frac": evals * alg / 6450e9}), flush=True)
            del popd
        del d
