"""The bench's end-to-end step (L2 flush, then evaluate_population on pinned
hub sets): median of 40 calls, for A/B runs of the library's transfer
pipelining (HUBGPU_EVAL_CHUNKS=0: one chunk; HUBGPU_EVAL_WAVE=1: a first chunk
of one K3 wave; default: two equal chunks).  HUBGPU_E2E_TRACE=1 adds the
library's per-call device phase times on stderr."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402

inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
B = 8192
pop = hg.random_population(1000, 20, B)
pin = torch.from_numpy(pop).pin_memory().numpy()
d = inst.device()
st = torch.cuda.ExternalStream(d.stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tag = ("one chunk" if os.environ.get("HUBGPU_EVAL_CHUNKS") == "0" else
       "wave first" if os.environ.get("HUBGPU_EVAL_WAVE") == "1" else "two halves")
ts = []
with torch.cuda.stream(st):
    for k in range(45):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = hg.evaluate_population(inst, pin)
        ts.append(time.perf_counter() - t0)
ts = np.array(ts[5:]) * 1e6
print(f"{tag:12s}: median {np.median(ts):.1f} us, p10 {np.percentile(ts, 10):.1f}, "
      f"p90 {np.percentile(ts, 90):.1f}", flush=True)
