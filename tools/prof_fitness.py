"""Small driver for ncu: score the URAND n=1000 p=20 population a few times.

    python tools/prof_fitness.py [n p pop reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 20
B = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
inst = hg.generate_urand(n, p, 1704, (1.0, 0.75, 1.0))
d = inst.device()
pop = hg._lib.DevicePopulation(d, B)
pop.load_hubs(hg.random_population(n, p, B).astype(np.int32))
for _ in range(reps):
    pop.evaluate(B)
d.synchronize()
print("fitness ms (last):", pop.last_fitness_ms())

if __import__("os").environ.get("HUBGPU_TC_TIMING") == "1":
    from paper_1704_06258_b200 import _lib

    buf = np.zeros(32, dtype=np.uint64)
    _lib.check(_lib.load().hg_debug_tc_timing(buf.ctypes.data_as(_lib._u64p)))
    names = ["Tstage", "waitB", "gen", "bar", "tmaW", "mmaIss", "waitMMA+A", "finalW", "prefetch",
             "epilog", "end", "unitTop"]
    for who, off in (("thread0", 0), ("thread32", 16)):
        tot = buf[off:off + 12].sum()
        print(who, " ".join(f"{nm}={100 * buf[off + k] / max(tot, 1):.1f}%" for k, nm in enumerate(names)))
