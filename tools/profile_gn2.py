"""ncu driver: C2, 2 steady-state GN steps (tree of the start cached first)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims, R = [400, 400, 400], 100
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, 1e-6)
p.set_factors(init)
print(p.time_gn_steps({}, 2))
