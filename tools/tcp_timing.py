"""Phase counters of K3-TC/P (tuning only): where the MMA issuer and one
epilogue warp spend their cycles.  Needs a timing build:

    make -C paper_1704_06258_b200/csrc clean all EXTRA=-DHG_TCP_TIMING
    HUBGPU_TC_TIMING=1 python tools/tcp_timing.py [n p B]

(the counters are accumulated by the leader's MMA warp and the first
epilogue warp of every CTA; cycles per CTA = sum / CTAs)
"""
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
for _ in range(3):
    pop.evaluate(B)
d.synchronize()
buf = np.zeros(32, dtype=np.uint64)
_lib.check(_lib.load().hg_debug_tc_timing(buf.ctypes.data_as(_lib._u64p)))  # reset
pop.evaluate(B)
d.synchronize()
print("fitness ms", pop.last_fitness_ms())
_lib.check(_lib.load().hg_debug_tc_timing(buf.ctypes.data_as(_lib._u64p)))
m = buf[0:4].astype(float)
e = buf[16:27].astype(float)
mn = ["waitA", "waitAccEmpty", "waitW", "issue"]
en = ["stage", "gen", "waitAccFull", "binAtomics", "reduce", "tmemLd", "epiSync", "tload", "fold",
      "waitKbf", "smemDrain"]
ctas = 148
print("MMA warp (leaders, cycles per pair):",
      " ".join(f"{k}={v / (ctas / 2):.0f}" for k, v in zip(mn, m)), " total", m.sum() / (ctas / 2))
print("epi warp 4 (cycles per CTA):", " ".join(f"{k}={v / ctas:.0f}" for k, v in zip(en, e)),
      " total", e.sum() / ctas)
