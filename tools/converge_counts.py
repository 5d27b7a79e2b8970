"""Device-only: iterations to convergence for the BASELINE configs (sizing the
full-size to-convergence parity tests)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
for name, dims, R, noise in [("C2", [400] * 3, 100, 1e-6), ("C4", [100] * 4, 50, 0.0), ("C1", [50] * 3, 5, 0.0)]:
    truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
    init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
    p = cpkit.DeviceProblem(dims, R)
    p.generate(truth, noise_seed=1, noise_rel=noise)
    for opt, cfg in [("gn", {"gn": {"max_iters": 300}}), ("als", {"als": {"max_sweeps": 5000}})]:
        t = time.perf_counter()
        _, rep = p.optimize(dict(cfg, optimizer=opt), init)
        j = rep.to_json()
        r = j["records"]
        print(name, opt, j["status"], len(r), r[-1]["residual"] if r else None,
              sum(x["cg_iters"] for x in r), f"{time.perf_counter() - t:.2f}s", flush=True)
