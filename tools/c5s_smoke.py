"""C5s slice (order 4, s=200, R=200, 12.8 GB): generate on device, time ALS sweeps and GN steps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims, R = [200, 200, 200, 200], 200
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
t = time.perf_counter()
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, 1e-4)
print(f"generate {time.perf_counter() - t:.2f}s")
p.set_factors(init)
p.time_als_sweeps(0.0, 1)
ms = p.time_als_sweeps(0.0, 3)
flops = 4 * R * 200 ** 4
print(f"ALS sweep {ms/3:.1f} ms  ({flops / (ms / 3 * 1e-3) / 1e12:.1f} TFLOP/s in the two roots' flops)")
b, f = p.time_roots(2)
print(f"roots: back {b:.2f} ms front {f:.2f} ms")
p.set_factors(init)
gms, cg = p.time_gn_steps({}, 2)
print(f"GN: {gms/2:.1f} ms/iter, {cg} CG iterations over 2 steps")
