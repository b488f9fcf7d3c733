"""A/B timing of K3 / K2 builds on the same box (tuning only).

    python tools/ab_k3.py VARIANT [VARIANT ...] [--rounds 3] [--shape n,p,B]

VARIANT "cur" is paper_1704_06258_b200/libhubgpu.so; any other name X is
paper_1704_06258_b200/libhubgpu_X.so (built beforehand, e.g. from another
commit, and copied in).  A variant may carry environment settings:
"cur:HUBGPU_TCP_KBS=4,HUBGPU_TCP_STAGES=3".  Each (round, variant) is one subprocess of
`tools/k3_ablate.py --one`, variants interleaved so drift hits them alike;
prints the median K3 and K2 milliseconds per variant as JSON.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--shape", default="1000,20,8192")
    ap.add_argument("--env", action="append", default=[], help="KEY=VALUE for every run")
    a = ap.parse_args()
    n, p, B = a.shape.split(",")
    res = {v: {"k3": [], "k2": []} for v in a.variants}
    for _ in range(a.rounds):
        for v in a.variants:
            env = dict(os.environ)
            env.pop("HUBGPU_LIB_VARIANT", None)
            lib, _, extra = v.partition(":")
            if lib != "cur":
                env["HUBGPU_LIB_VARIANT"] = lib
            for kv in filter(None, extra.split(",")):
                k, _, val = kv.partition("=")
                env[k] = val
            for kv in a.env:
                k, _, val = kv.partition("=")
                env[k] = val
            out = subprocess.run([sys.executable, str(ROOT / "tools" / "k3_ablate.py"), "--one",
                                  n, p, B], env=env, capture_output=True, text=True)
            if out.returncode:
                print(v, "failed:", out.stderr[-500:], flush=True)
                continue
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[v]["k3"].append(d["k3_ms"])
            res[v]["k2"].append(d["k2_ms"])
    summary = {v: {"k3_ms": statistics.median(r["k3"]) if r["k3"] else None,
                   "k2_ms": statistics.median(r["k2"]) if r["k2"] else None,
                   "k3_all": r["k3"]} for v, r in res.items()}
    print(json.dumps({"shape": a.shape, "results": summary}))


if __name__ == "__main__":
    main()
