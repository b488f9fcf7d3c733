"""Phase counters of K3-TC/Y (run with HUBGPU_TC_TIMING=1)."""
import os
import sys
from pathlib import Path

os.environ["HUBGPU_TC_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402
from paper_1704_06258_b200 import _lib  # noqa: E402

n, p, B = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (1000, 20, 8192)))
inst = hg.generate_urand(n, p, 1704, (1.0, 0.75, 1.0))
d = inst.device()
pop = _lib.DevicePopulation(d, B)
pop.load_hubs(hg.random_population(n, p, B).astype(np.int32))
pop.evaluate(B)
d.synchronize()
buf = np.zeros(32, dtype=np.uint64)
_lib.check(_lib.load().hg_debug_tc_timing(buf.ctypes.data_as(_lib._u64p)))  # reset
pop.evaluate(B)
print("fitness ms", pop.last_fitness_ms())
_lib.check(_lib.load().hg_debug_tc_timing(buf.ctypes.data_as(_lib._u64p)))
m = buf[0:4].astype(float)
e = buf[16:22].astype(float)
print("MMA warp:", " ".join(f"{k}={100 * v / m.sum():.1f}%" for k, v in
                             zip(["waitA", "waitAccEmpty", "waitW", "issue"], m)))
print("epi warp:", " ".join(f"{k}={100 * v / e.sum():.1f}%" for k, v in
                             zip(["stage", "gen", "waitAcc", "math", "reduce", "tmemld"], e)))
print("cycles per CTA (MMA warp):", m.sum() / 148, " epi:", e.sum() / 148)
