"""Hash of evaluate_population outputs over several shapes (run once with
HUBGPU_K2_SCALAR=1 and once without: the two K2 kernels must agree bit for bit)."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402

h = hashlib.sha256()
for n, p, B in ((1000, 20, 4096), (200, 3, 1000), (517, 32, 777), (1500, 17, 513), (64, 5, 300),
                (300, 29, 200), (400, 50, 300), (300, 64, 200), (1000, 40, 500), (200, 33, 100)):
    inst = hg.generate_urand(n, p, 1704 + n, (1.0, 0.75, 1.0))
    pop = hg.random_population(n, p, B, key=n + p)
    out = hg.evaluate_population(inst, pop)
    h.update(out.tobytes())
    h.update(hg.nearest_allocations(inst, pop[:256]).tobytes())  # the alloc output too
    print(n, p, B, hashlib.sha256(out.tobytes()).hexdigest()[:16])
# a tie-heavy instance: integer grid distances (many equal costs)
g = np.arange(12)
xy = np.stack(np.meshgrid(g, g), -1).reshape(-1, 2).astype(np.float64)
d = np.abs(xy[:, None, :] - xy[None, :, :]).sum(-1)
rng = np.random.default_rng(5)
f = rng.integers(0, 9, size=d.shape).astype(np.float64)
inst = hg.Instance(n=d.shape[0], p=12, dist=d, flow=f, chi=1.0, alpha=0.75, delta=1.0, name="grid")
pop = hg.random_population(inst.n, 12, 2000, key=3)
out = hg.evaluate_population(inst, pop)
h.update(out.tobytes())
h.update(hg.nearest_allocations(inst, pop).tobytes())
print("grid", hashlib.sha256(out.tobytes()).hexdigest()[:16])
print("ALL", h.hexdigest())
