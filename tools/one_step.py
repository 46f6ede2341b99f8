"""One hot-path step (factor + PCG) on a config, for profilers (ncu launch lists)."""
import sys
sys.path.insert(0, ".")
from paper_1811_11248_b200 import hsolve as H
from problems import gen_config
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
p = gen_config(name)
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
x, rep = H.hs_pcg(f, p.b, tol=p.tol)
print("iters", rep["iters"], "relres_true", rep["relres_true"], "launches", H.hs_launch_count())
