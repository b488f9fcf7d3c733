"""K3 time vs the number of W byte planes (integer flows up to 2^8P - 1),
UR shape n=1000 p=20, 8192 hub sets."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402
from paper_1704_06258_b200 import _lib  # noqa: E402

base = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
pop = hg.random_population(1000, 20, 8192).astype(np.int32)
for wmax in (100, 300, 70000, 2**24 + 5):
    rng = np.random.default_rng(1)
    flow = rng.integers(0, wmax + 1, size=(1000, 1000)).astype(np.float64)
    np.fill_diagonal(flow, 0.0)
    inst = hg.Instance(1000, 20, base.dist, flow, 1.0, 0.75, 1.0)
    d = inst.device()
    popd = _lib.DevicePopulation(d, 8192)
    popd.load_hubs(pop)
    for kind in ("tensor-pair", "fp64"):
        try:
            d.set_fitness(_lib.FIT_NAMES[kind])
        except ValueError:
            continue
        ms = []
        for _ in range(5):
            popd.evaluate(8192)
            ms.append(popd.last_fitness_ms())
        print(f"wmax={wmax:>9} kernel={kind:12s} K3 ms={np.median(ms[1:]):.3f}", flush=True)
