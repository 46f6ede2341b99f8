"""Per-level apply timings (eager replay with events, HS_PROFILE) after one C2 factor."""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1811_11248_b200 import hsolve as H
from problems import gen_config
p = gen_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
os.environ["HS_PROFILE"] = "1"
for _ in range(3):
    H.hs_apply(f, np.asarray(p.b))
