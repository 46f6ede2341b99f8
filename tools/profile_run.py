"""HS_PROFILE run: per-level factor table and per-level apply times on a config."""
import os, sys, time
os.environ["HS_PROFILE"] = "1"
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1811_11248_b200 import hsolve as H
from problems import gen_config
from problems.generators import gen_config_scaled
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
base, _, k = name.partition("/")
p = gen_config_scaled(base, int(k)) if k else gen_config(base)
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
for rep in range(2):
    t = time.time()
    f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
    print("factor wall", time.time() - t, H.hs_factor_get_stats(f)["t_factor_s"], flush=True)
x = H.hs_apply(f, p.b)
x, r = H.hs_pcg(f, p.b, tol=p.tol)
print(r)
