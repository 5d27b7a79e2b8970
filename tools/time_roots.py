"""Time the root contractions of a problem (kernel events), for tiling experiments."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
dims = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "400,400,400").split(",")]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 100
truth = cpkit.random_factors(dims, R, 1)
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, 0.0)
p.set_factors(cpkit.random_factors(dims, R, 2))
p.time_roots(2)
b, f = p.time_roots(10)
n = 1
for d in dims: n *= d
print(f"dims={dims} R={R} env={os.environ.get('CPKIT_TN_WN','-')} back {b*1e3:.1f}us {2*R*n/b/1e9:.2f}TF  front {f*1e3:.1f}us {2*R*n/f/1e9:.2f}TF")
