import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1704_06258_b200 as hg

inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))      # device=True draws it on the GPU
sol = hg.nearest_allocation([3, 17, 99], inst.with_p(3))         # reference API
bd = hg.objective(inst.with_p(3), sol, hg.FitnessMode.RAW)
pop = hg.random_population(1000, 20, 8192)
scores = hg.evaluate_population(inst, pop)                       # (collection, transfer, distribution, raw)
rep = hg.solve(inst, hg.GaParams(islands=128, pop_size=64, inner_iters=25, outer_iters=10),
               hg.FitnessMode.STANDARD_MILLI)
best, raw = hg.restricted_optimum(hg.generate_urand(30, 4, 1, (1.0, 0.75, 1.0)))
print(bd.raw_total, scores.shape, rep.raw_objective, best.hubs, raw)
