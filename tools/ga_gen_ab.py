"""A/B of the GA generation time (128 islands x 64 at UR): one subprocess per
library variant (HUBGPU_LIB_VARIANT, see tools/ab_k3.py), 50 generations
timed by CUDA events on the instance stream, median of 3.

    python tools/ga_gen_ab.py VARIANT [VARIANT ...]
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1704_06258_b200 as hg
inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
d = inst.device()
ga = hg._lib.DeviceGa(d, 128, 0, 128, 64, 3, False, 0)
ga.begin_round(np.sort(inst.middle_rank[:20]))
st = torch.cuda.ExternalStream(d.stream)
ga.generations(5)
ms = []
for _ in range(3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); ga.generations(50); b.record(st)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b) / 50)
print(sorted(ms)[1])
'''
for v in sys.argv[1:]:
    env = dict(os.environ)
    if v != "cur":
        env["HUBGPU_LIB_VARIANT"] = v
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True,
                       text=True)
    print(v, r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-300:],
          "ms/generation", flush=True)
