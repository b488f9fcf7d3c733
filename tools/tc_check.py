"""Quick K3-TC vs K3 (fp64) comparison: python tools/tc_check.py [n p B]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = int(sys.argv[2]) if len(sys.argv) > 2 else 20
B = int(sys.argv[3]) if len(sys.argv) > 3 else 24
inst = hg.generate_urand(n, p, 5, (1.0, 0.75, 1.0))
pop = hg.random_population(n, p, B)
d = inst.device()
print("flags", d.flags, "kernel", d.fitness_kernel, flush=True)
d.set_fitness(1)
fp = hg.evaluate_population(inst, pop)
d.set_fitness(2)
tc = hg.evaluate_population(inst, pop)
rel = np.abs(tc[:, 1] - fp[:, 1]) / np.abs(fp[:, 1])
print("max rel diff transfer:", rel.max(), "first:", tc[:3, 1], fp[:3, 1], flush=True)
