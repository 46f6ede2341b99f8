"""Debug aid: is the single-GPU factor bit-deterministic run to run?"""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1811_11248_b200 import hsolve as H
from problems import gen_laplace3d
p = gen_laplace3d(24, leaf_size=27)
h1 = H.hs_create(0)
a1 = H.hs_analyze(h1, p.n, p.rowptr, p.colind, p.coords, None, leaf_size=p.leaf_size)
ref = None
v = np.random.default_rng(1).standard_normal(p.n)
for it in range(8):
    f = H.hs_factor_create(h1, a1, p.vals, eps=1e-2)
    rk = np.concatenate([H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(6)])
    x = H.hs_apply(f, v)
    if ref is None:
        ref = (rk, x)
    else:
        print(it, "ranks equal", np.array_equal(rk, ref[0]), "apply max diff", np.abs(x - ref[1]).max(),
              "first diff", np.nonzero(rk != ref[0])[0][:5])
