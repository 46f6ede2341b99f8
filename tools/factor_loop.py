import sys, os
sys.path.insert(0, ".")
from paper_1811_11248_b200 import hsolve as H
from problems import gen_config
p = gen_config("C2")
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
for i in range(4):
    f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
    del f
