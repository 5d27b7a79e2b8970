"""GN step breakdown: device time in back/front roots and CG (profile events).
Usage: gn_breakdown.py [c2|c5s]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dims, R, noise = ([400] * 3, 100, 1e-6) if cfg == "c2" else ([200] * 4, 200, 1e-4)
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, noise)
p.set_factors(init)
p.time_gn_steps({}, 2)  # warm
for rep in range(3):
    p.set_factors(init)
    p.profile(True)
    ms, cg = p.time_gn_steps({}, 2)
    pm, pc = p.profile_read()
    p.profile(False)
    print(f"2 GN steps {ms:.3f} ms, cg iters {cg}; back {pm[0]:.3f} ms x{pc[0]}, front {pm[1]:.3f} ms x{pc[1]}, cg {pm[2]:.3f} ms x{pc[2]}")
