"""Where the end-to-end evaluate_population time goes (UR, 8192 hub sets)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402
from paper_1704_06258_b200 import _lib  # noqa: E402

inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
B = 8192
pop = hg.random_population(1000, 20, B)
pin = torch.from_numpy(pop).pin_memory().numpy()
d = inst.device()
for _ in range(5):
    hg.evaluate_population(inst, pin)


def t(f, reps=50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t0) / reps * 1e6


print("evaluate_population pinned  us", t(lambda: hg.evaluate_population(inst, pin)))
print("evaluate_population pageable us", t(lambda: hg.evaluate_population(inst, pop)))
out = np.empty((B, 4))
print("hg_evaluate direct          us", t(lambda: _lib.check(_lib.load().hg_evaluate(
    d.handle, B, _lib.ptr(pin, _lib._i64p), None, _lib.ptr(out, _lib._f64p)))))
outp = torch.empty((B, 4), dtype=torch.float64).pin_memory().numpy()
print("hg_evaluate pinned out      us", t(lambda: _lib.check(_lib.load().hg_evaluate(
    d.handle, B, _lib.ptr(pin, _lib._i64p), None, _lib.ptr(outp, _lib._f64p)))))
popd = _lib.DevicePopulation(d, B)
popd.load_hubs(pop.astype(np.int32))
print("device evaluate+sync        us", t(lambda: (popd.evaluate(B), d.synchronize())))
