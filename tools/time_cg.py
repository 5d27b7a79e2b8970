"""Time the persistent CG kernel alone at several iteration caps (C2 shapes)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "400,400,400").split(",")]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 100
f = cpkit.random_factors(dims, R, 3)
g = cpkit.random_factors(dims, R, 4, kind="gaussian")
p = cpkit.DeviceProblem(dims, R)
p.set_factors(f)
p.gamma_set()
for cap in [1, 1, 10, 100] + [1000] * int(os.environ.get("REPEAT", "1")):
    t = time.perf_counter()
    v, it, hc, bd = p.cp_cg(g, 1e-3, {"cg_max_iters": cap, "cg_tol": 1e-14})
    dt = time.perf_counter() - t
    print(f"cap={cap:5d} iters={it:5d} wall={dt*1e3:8.2f} ms  per-iter={dt*1e3/max(1,it):.3f} ms")
