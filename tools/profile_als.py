"""ncu driver: C2 problem, warm ALS sweeps (graph replays) for a launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit

dims, R = [400, 400, 400], 100
if len(sys.argv) > 1:
    dims = [int(v) for v in sys.argv[1].split(",")]
    R = int(sys.argv[2])
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, 1e-6)
p.set_factors(init)
n = int(os.environ.get("SWEEPS", "6"))
for _ in range(n):
    p.als_sweep(0.0)
print("ok")
