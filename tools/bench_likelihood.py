"""Likelihood protocol (README example: uniform11, s=4, ranks 3,5,6,7,9, GN, 30 problems x 5 inits)
on the device (one CTA per instance) vs the oracle restatement on all host cores."""
import os, sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
from oracle import oracle as orc

opt = sys.argv[1] if len(sys.argv) > 1 else "gn"
ranks, problems, inits, seed, dims = [3, 5, 6, 7, 9], 30, 5, 42, [4, 4, 4]
cfg = {"problem": {"family": "uniform11", "dims": dims, "ranks": ranks}, "optimizer": opt,
       "problems": problems, "inits": inits, "seed": seed}
cpkit.run_likelihood({**cfg, "problems": 1, "inits": 1})  # warm
dev = 1e9
for _ in range(3):  # best of 3 (clock ramp after idle)
    t = time.perf_counter()
    rep = cpkit.run_likelihood(cfg).to_json()
    dev = min(dev, time.perf_counter() - t)
fr = {r["rank"]: r["fraction"] for r in rep["ranks"]}

jobs = []
for R in ranks:
    for p in range(problems):
        x = orc.reconstruct(orc.random_model(dims, R, orc.problem_seed(seed, R, p), kind="uniform", a=-1, b=1))
        for i in range(inits):
            jobs.append((x, orc.random_model(dims, R, orc.init_seed(seed, R, p, i), kind="gaussian")))
orc.set_threads(1) if hasattr(orc, "set_threads") else None


def one(j):
    x, init = j
    try:
        if opt == "gn":
            return orc.gn_optimize(x, init, orc.GnConfig())[2]
        return orc.als_optimize(x, init, orc.AlsConfig())[2]
    except orc.OracleError:
        return "numerical_failure"


cores = os.cpu_count()
t = time.perf_counter()
with ThreadPoolExecutor(cores) as ex:
    st = list(ex.map(one, jobs))
cpu = time.perf_counter() - t
print(f"{opt}: {len(jobs)} instances  device {dev*1e3:.1f} ms   oracle {cpu*1e3:.1f} ms on {cores} threads   "
      f"speedup {cpu/dev:.1f}x   fractions {fr}")
