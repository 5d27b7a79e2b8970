"""ALS sweep and GN iteration times for every BASELINE config that fits one GPU
(C1-C4, C5s), tensors generated on device from the reference's keyed RNG."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit

CONFIGS = [("C1", [50] * 3, 5, 0.0), ("C2", [400] * 3, 100, 1e-6), ("C3", [200] * 3, 20, 0.0),
           ("C4", [100] * 4, 50, 0.0), ("C5s", [200] * 4, 200, 1e-4)]
for name, dims, R, noise in CONFIGS:
    truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
    init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
    p = cpkit.DeviceProblem(dims, R)
    p.generate(truth, 1, noise)
    p.set_factors(init)
    p.time_als_sweeps(0.0, 4)
    n = 20 if name != "C5s" else 4
    als = p.time_als_sweeps(0.0, n) / n
    p.set_factors(init)
    p.time_gn_steps({}, 1)
    p.set_factors(init)
    gms, cg = p.time_gn_steps({}, 3)
    print(f"{name}: dims={dims} R={R}  ALS {als:.3f} ms/sweep ({1e3 / als:.0f} sweeps/s)  "
          f"GN {gms / 3:.3f} ms/iter ({3e3 / gms:.0f} it/s, {cg} CG iterations over 3 steps)", flush=True)
