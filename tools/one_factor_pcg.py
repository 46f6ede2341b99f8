"""One C2 factor + one PCG (the bench step), for ncu launch lists (tools/profile_round.sh)."""
import sys
sys.path.insert(0, ".")
from paper_1811_11248_b200 import hsolve as H
from problems import gen_config
p = gen_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
x, rep = H.hs_pcg(f, p.b, tol=p.tol)
print(rep)
