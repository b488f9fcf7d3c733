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


def t(f, reps=100):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t0) / reps * 1e6


out = np.empty((B, 4))
outp = torch.empty((B, 4), dtype=torch.float64).pin_memory().numpy()
popd = _lib.DevicePopulation(d, B)
popd.load_hubs(pop.astype(np.int32))
cases = {
    "evaluate_population (pinned hubs)": lambda: hg.evaluate_population(inst, pin),
    "evaluate_population (pageable hubs)": lambda: hg.evaluate_population(inst, pop),
    "hg_evaluate, pageable out": lambda: _lib.check(_lib.load().hg_evaluate(
        d.handle, B, _lib.ptr(pin, _lib._i64p), None, _lib.ptr(out, _lib._f64p))),
    "hg_evaluate, pinned out": lambda: _lib.check(_lib.load().hg_evaluate(
        d.handle, B, _lib.ptr(pin, _lib._i64p), None, _lib.ptr(outp, _lib._f64p))),
    "device evaluate + sync": lambda: (popd.evaluate(B), d.synchronize()),
}
for rep in range(2):
    for name, f in cases.items():
        print(f"{name:40s} {t(f):8.1f} us")
print("pool:", {k: len(v) for k, v in _lib._pinned._free.items()})
