import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from oracle import oracle as orc
from tests.helpers import swamp_factors
from paper_1910_12331_b200 import cpkit as ck
dims, R = [30, 30, 30], 5
truth = swamp_factors(orc, dims, R, 11)
x = orc.reconstruct(truth)
init = orc.random_model(dims, R, orc.init_seed(0, R, 0, 0))
p = ck.DeviceProblem(dims, R); p.upload(x)
_, rep = p.optimize({"optimizer":"gn","gn":{"max_iters":40,"residual_tol":1e-10}}, init)
j = rep.to_json()
_, recs, st = orc.gn_optimize(x, init, orc.GnConfig(max_iters=40, residual_tol=1e-10))
print(j["status"], st)
for a, b in zip(j["records"], recs):
    print(a["iter"], a["cg_iters"], b["cg_iters"], "%.12e %.12e %.2e" % (a["residual"], b["residual"], abs(a["residual"]-b["residual"])))
