"""Launch-list driver for the SPD kernels: spd_solve on s x R systems."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
for R, s in ((100, 400), (200, 400), (50, 100), (20, 200)):
    a = np.random.default_rng(R).standard_normal((R + 50, R))
    S = a.T @ a
    b = np.random.default_rng(1).standard_normal((s, R))
    p = cpkit.DeviceProblem([3, 3], R)
    for _ in range(3):
        y = p.spd_solve(S, b, 1e-3)
    print(R, s, np.linalg.norm(y @ (S + 1e-3 * np.eye(R)) - b) / np.linalg.norm(b))
