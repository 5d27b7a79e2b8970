"""Where the e2e (cpkit_decompose from host memory) time goes at C5s:
problem allocation, H2D upload (+ layout copy), sweeps, teardown."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1910_12331_b200 import cpkit
dims, R = [200, 200, 200, 200], 200
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, 1e-4)
n = p.slab()[2]
x = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
p.download_into(x)
p.close()
cfg = {"optimizer": "als", "als": {"max_sweeps": 20, "residual_tol": 0.0, "step_tol": 0.0}}
for rep in range(3):
    t0 = time.perf_counter()
    q = cpkit.DeviceProblem(dims, R)
    t1 = time.perf_counter()
    q.upload(x)
    q.norm2()  # forces completion of the upload + copies
    t2 = time.perf_counter()
    q.optimize(cfg, init)
    t3 = time.perf_counter()
    q.close()
    t4 = time.perf_counter()
    print(f"alloc {1e3*(t1-t0):7.1f} ms  upload {1e3*(t2-t1):7.1f} ms ({8*n/(t2-t1)/1e9:.1f} GB/s)  "
          f"optimize {1e3*(t3-t2):7.1f} ms  close {1e3*(t4-t3):7.1f} ms", flush=True)
t = cpkit.Tensor.create(x.reshape(dims))
c2 = dict(cfg, rank=R, seed=0, init={"distribution": "uniform", "a": 0.0, "b": 1.0})
for rep in range(3):
    t0 = time.perf_counter()
    m, r = cpkit.decompose(t, c2)
    print(f"decompose {1e3*(time.perf_counter()-t0):7.1f} ms", flush=True)
