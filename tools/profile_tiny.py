"""ncu driver: one likelihood batch (GN, s=4, rank 7, 30 problems x 5 inits) on the CTA-per-instance solver."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_12331_b200 import cpkit
opt = sys.argv[1] if len(sys.argv) > 1 else "gn"
cpkit.run_likelihood({"problem": {"family": "uniform11", "dims": [4, 4, 4], "ranks": [7]}, "optimizer": opt,
                      "problems": 30, "inits": 5, "seed": 42})
print("ok")
