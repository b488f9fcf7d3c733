import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, paper_1704_06258_b200 as hg, time
from oracle import hm_oracle as orc
def check(inst, pop):
    out = hg.evaluate_population(inst, pop)
    pr = orc.Problem(inst.n, inst.p, inst.dist, inst.flow, inst.chi, inst.alpha, inst.delta)
    for b in range(0, len(pop), max(1, len(pop)//5)):
        a = orc.nearest(pr.C, pop[b]); c,t,d = orc.cost_terms(pr, pop[b], a)
        ref = np.array([c,t,d,c+t+d])
        assert np.all(np.abs(out[b]-ref) <= 1e-12*np.abs(ref)+1e-300), (b, out[b], ref)
    return out
for n,p in [(1,1),(2,1),(2,2),(3,3),(16,16),(300,255),(1000,129)]:
    inst = hg.generate_urand(n, p, 3, (1,0.75,1))
    pop = hg.random_population(n, p, 7)
    check(inst, pop); print("ok", n, p, inst.device().fitness_kernel)
inst = hg.generate_urand(1000, 20, 3, (1,0.75,1))
print(hg.evaluate_population(inst, np.empty((0,20), np.int64)).shape)
pop = hg.random_population(1000, 20, 200000)
t=time.time(); out = check(inst, pop); print("B=200k", time.time()-t)
u = hg.evaluate_population(inst, pop[:1], unique=True); print("unique B=1", u.shape)
