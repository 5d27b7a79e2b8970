import os, sys, json
sys.path.insert(0, os.getcwd())
from tests.helpers import swamp_factors
from oracle import oracle as orc
from paper_1910_12331_b200 import cpkit as ck
orc.set_threads(16); ck.load()
dims, R = [200]*3, 20
truth = swamp_factors(orc, dims, R, 0)
p = ck.DeviceProblem(dims, R); p.generate(truth); x = p.download()
init = ck.random_factors(dims, R, ck.init_seed(0, R, 0, 0))
for opt, dc, oc in [("gn", {"gn": {"max_iters": 200, "residual_tol": 1e-10}}, orc.GnConfig(max_iters=200, residual_tol=1e-10)),
                    ("als", {"als": {"max_sweeps": 3000, "residual_tol": 1e-10}}, orc.AlsConfig(max_sweeps=3000, residual_tol=1e-10))]:
    f, rep = p.optimize(dict(dc, optimizer=opt), init); j = rep.to_json()
    fr, recs, st = (orc.gn_optimize if opt == "gn" else orc.als_optimize)(x, init, oc)
    print(opt, j["status"], st, len(j["records"]), len(recs))
    for k, (a, b) in enumerate(zip(j["records"], recs)):
        if opt == "gn" or k % 50 == 0 or k > len(recs) - 5:
            print(k, a["cg_iters"], b["cg_iters"], "%.15e %.15e %.2e" % (a["residual"], b["residual"], abs(a["residual"]-b["residual"])))
