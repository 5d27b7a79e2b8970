"""Per-phase timestamps of the persistent CG kernel (CPKIT_CG_TRACE=1 prints them to stderr).
Usage: CPKIT_CG_TRACE=1 python tools/cg_trace.py [dims [R [cap]]]   (default C2: 400,400,400 100 50;
C5s shapes - the streaming kernel - are 200,200,200,200 200)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "400,400,400").split(",")]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 50
f = cpkit.random_factors(dims, R, 3)
g = cpkit.random_factors(dims, R, 4, kind="gaussian")
p = cpkit.DeviceProblem(dims, R)
p.set_factors(f)
p.gamma_set()
for _ in range(2):
    print(p.cp_cg(g, 1e-3, {"cg_max_iters": cap, "cg_tol": 1e-14})[1:])
