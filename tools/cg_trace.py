import os, sys
sys.path.insert(0, os.getcwd())
from paper_1910_12331_b200 import cpkit
dims=[400,400,400]; R=100
f = cpkit.random_factors(dims, R, 3); g = cpkit.random_factors(dims, R, 4, kind="gaussian")
p = cpkit.DeviceProblem(dims, R); p.set_factors(f); p.gamma_set()
for _ in range(2): print(p.cp_cg(g, 1e-3, {"cg_max_iters": 50, "cg_tol": 1e-14})[1:])
