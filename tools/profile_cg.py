import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "400,400,400").split(",")]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 100
p = cpkit.DeviceProblem(dims, R)
p.set_factors(cpkit.random_factors(dims, R, 3))
p.gamma_set()
g = cpkit.random_factors(dims, R, 4, kind="gaussian")
print(p.cp_cg(g, 1e-3, {"cg_max_iters": 50, "cg_tol": 1e-14})[1:])
