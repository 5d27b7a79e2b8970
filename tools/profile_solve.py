"""Small driver for ncu: one R x R SPD solve with `rows` right-hand sides (the
ALS row solve at C5s: R=200, 200 rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1910_12331_b200 import cpkit
R = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 200
a = cpkit.random_factors([R + 7], R, 3)[0]
s = a.T @ a
b = cpkit.random_factors([rows], R, 4)[0]
p = cpkit.DeviceProblem([3, 3], R)
for _ in range(3):
    y = p.spd_solve(s, b, 1e-3)
print(float(np.abs(y).sum()))
