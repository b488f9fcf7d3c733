import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, paper_1704_06258_b200 as hg
from paper_1704_06258_b200 import engine, _lib
inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
d = inst.device()
gp = hg.GaParams(islands=128, pop_size=64, inner_iters=10, outer_iters=5, seed=1)
for rep in range(2):
    t0 = time.perf_counter(); ga = engine.DeviceIslands(inst, gp, 3, 0, 128); t1 = time.perf_counter()
    anc = np.sort(inst.middle_rank[:20])
    for r in range(5):
        ga.run_round(anc)
    d.synchronize(); t2 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, 5 rounds x 10 gens {1e3*(t2-t1):.1f} ms")
for rep in range(2):
    t0 = time.perf_counter(); r = hg.solve(inst, gp, hg.FitnessMode.STANDARD_MILLI); t1 = time.perf_counter()
    print(f"solve {1e3*(t1-t0):.1f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
r = hg.solve(inst, gp, hg.FitnessMode.STANDARD_MILLI)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
