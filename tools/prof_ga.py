"""Small driver for ncu: a few GA generations (128 islands x 64, UR).

    python tools/prof_ga.py [generations]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
d = inst.device()
ga = hg._lib.DeviceGa(d, 128, 0, 128, 64, 3, False, 0)
ga.begin_round(np.sort(inst.middle_rank[:20]))
ga.generations(gens)
d.synchronize()
print("ok")
