"""Event trace of K3-TC/P's CTA 0 (tuning only; needs the timing build):

    make -C paper_1704_06258_b200/csrc clean all EXTRA=-DHG_TCP_TIMING
    HUBGPU_TC_TIMING=1 python tools/tcp_trace.py [n p B] [--units 2,4]

Prints, for the chosen slots, the MMA issuer's and two epilogue warps' events
in clock64 cycles relative to the first event of the first chosen slot, and a
per-tile summary (MMA issue window, accumulator hand-off, epilogue drain).
Codes: MMA 1 wait acc-empty, 2 acc free, 3 W stage ready, 4/5 A-quarter wait
begin/end, 8 tile committed; epilogue 24 slot top, 26 T gather issued,
11/12 kbf wait begin/end, 19 cluster rows ready (deferred fold), 25 one-hot
stores issued, 13 one-hot generated, 14 acc-full wait, 15 acc full,
16 released, 17 bins done, 18 reduce done, 20 chunk end, 21 after sync 1,
22 fold done, 23 after sync 2.
"""

import os
import sys
from pathlib import Path

os.environ["HUBGPU_TC_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1704_06258_b200 as hg  # noqa: E402
from paper_1704_06258_b200 import _lib  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n, p, B = (int(a) for a in (args if len(args) == 3 else (1000, 20, 8192)))
u0, u1 = 2, 4
for a in sys.argv[1:]:
    if a.startswith("--units"):
        u0, u1 = (int(x) for x in a.split("=", 1)[1].split(","))
inst = hg.generate_urand(n, p, 1704, (1.0, 0.75, 1.0))
d = inst.device()
pop = _lib.DevicePopulation(d, B)
pop.load_hubs(hg.random_population(n, p, B).astype(np.int32))
for _ in range(3):
    pop.evaluate(B)
d.synchronize()
tr = np.zeros(3 * 8192, dtype=np.uint64)
_lib.check(_lib.load().hg_debug_tc_trace(tr.ctypes.data_as(_lib._u64p)))  # clear
pop.evaluate(B)
d.synchronize()
_lib.check(_lib.load().hg_debug_tc_trace(tr.ctypes.data_as(_lib._u64p)))
roles = []
for r in range(3):
    w = tr[r * 8192:(r + 1) * 8192]
    w = w[w != 0]
    roles.append([(int(x >> 56), int(x & ((1 << 56) - 1))) for x in w])

# slot boundaries: MMA = every 8 tiles (code 1 starts a tile); epilogue = code 24
mma = roles[0]
tile_starts = [i for i, (c, _) in enumerate(mma) if c == 1]
tiles_per_slot = None
epi_tops = [[i for i, (c, _) in enumerate(ev) if c == 24] for ev in roles[1:]]
nslots = len(epi_tops[0])
tiles_per_slot = len(tile_starts) // max(nslots, 1)
print(f"slots {nslots}, tiles per slot {tiles_per_slot}, MMA events {len(mma)}, "
      f"epi events {len(roles[1])}/{len(roles[2])}")
t0 = mma[tile_starts[u0 * tiles_per_slot]][1]
for name, ev, lo, hi in (
        ("MMA", mma, tile_starts[u0 * tiles_per_slot], tile_starts[min(u1 * tiles_per_slot, len(tile_starts) - 1)]),
        ("epi4", roles[1], epi_tops[0][u0], epi_tops[0][min(u1, nslots - 1)]),
        ("epi19", roles[2], epi_tops[1][u0], epi_tops[1][min(u1, nslots - 1)])):
    print(f"--- {name}")
    print(" ".join(f"{c}@{t - t0}" for c, t in ev[lo:hi]))

# per-slot aggregates over all slots (cycles)
def spans(ev, a, b):
    out, start = 0, None
    for c, t in ev:
        if c == a:
            start = t
        elif c == b and start is not None:
            out += t - start
            start = None
    return out

tot = mma[-1][1] - mma[0][1]
print("MMA: total", tot, "wait acc-empty", spans(mma, 1, 2), "wait A", spans(mma, 4, 5))
for name, ev in (("epi4", roles[1]), ("epi19", roles[2])):
    print(name, "wait acc-full", spans(ev, 14, 15), "drain", spans(ev, 15, 16),
          "bins", spans(ev, 16, 17), "kbf wait", spans(ev, 11, 12), "gen", spans(ev, 12, 13),
          "gen cready wait", spans(ev, 12, 19), "gen st wait", spans(ev, 25, 13),
          "sync1", spans(ev, 20, 21), "fold", spans(ev, 21, 22), "sync2", spans(ev, 22, 23),
          "reduce", spans(ev, 17, 18), "top", spans(ev, 24, 26))

# per-tile MMA waits of the first two traced slots: accumulator, W stage, A quarters
tiles, cur = [], None
for c, t in mma:
    if c == 1:
        if cur:
            tiles.append(cur)
        cur = {1: t, "A": 0}
    elif cur is not None:
        if c == 4:
            cur[4] = t
        elif c == 5:
            cur["A"] += t - cur[4]
        elif c not in cur:
            cur[c] = t
if cur:
    tiles.append(cur)
for i, x in enumerate(tiles[u0 * tiles_per_slot:(u0 + 2) * tiles_per_slot]):
    if 2 in x and 3 in x:
        print(f"tile {i % tiles_per_slot}: wait acc {x[2] - x[1]}, wait W {x[3] - x[2]}, "
              f"wait A {x['A']}, issue {x.get(8, x[3]) - x[3]}")
