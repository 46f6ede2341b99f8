import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1811_11248_b200 import hsolve as H
from problems import gen_stokes_q1
p = gen_stokes_q1(12, 10, 5, leaf_columns=2)
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_columns=2)
v = np.random.default_rng(4).standard_normal(p.n)
f1 = H.hs_factor_create(h, a, p.vals, eps=1e-2)
x1 = H.hs_apply(f1, v)
f1b = H.hs_factor_create(h, a, p.vals, eps=1e-2)
print("repeat", np.abs(H.hs_apply(f1b, v) - x1).max())
for sc in (4.0, 2.0, 0.5, 1024.0):
    f4 = H.hs_factor_create(h, a, sc * p.vals, eps=1e-2)
    x4 = H.hs_apply(f4, v)
    L = H.hs_analysis_get_info(a)["L_top"]
    same = all(np.array_equal(H.hs_factor_export(f4, H.HS_FEXP_PIV, l), H.hs_factor_export(f1, H.HS_FEXP_PIV, l)) for l in range(L))
    print(sc, "pivots same", same, "rel diff", np.linalg.norm(sc * x4 - x1) / np.linalg.norm(x1), "top", H.hs_factor_export(f1, H.HS_FEXP_TOP))
