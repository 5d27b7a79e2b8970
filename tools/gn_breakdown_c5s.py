"""GN step breakdown on the C5s slice (order 4, s=200, R=200): device time in roots and CG."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims, R = [200, 200, 200, 200], 200
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, 1e-4)
p.set_factors(init)
p.time_gn_steps({}, 1)  # warm
for rep in range(2):
    p.set_factors(init)
    p.profile(True)
    ms, cg = p.time_gn_steps({}, 2)
    pm, pc = p.profile_read()
    p.profile(False)
    print(f"2 GN steps {ms:.3f} ms, cg iters {cg}; back {pm[0]:.3f} ms x{pc[0]}, front {pm[1]:.3f} ms x{pc[1]}, cg {pm[2]:.3f} ms x{pc[2]}")
