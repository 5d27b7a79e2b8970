"""Driver for ncu/launch lists: C2 problem, 2 GN steps (default config)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims, R = [400, 400, 400], 100
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, 1e-6)
p.set_factors(init)
ms, cg = p.time_gn_steps({}, 2)
print(f"2 GN steps: {ms:.2f} ms, {cg} CG iterations")
p.set_factors(init)
ms, cg = p.time_gn_steps({"cg_max_iters": 1000, "cg_tol": 1e-12}, 1)
print(f"1 GN step capped CG: {ms:.2f} ms, {cg} CG iterations")
