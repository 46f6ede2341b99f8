"""One factor + one PCG (the bench step) of a config ("C2", "C4/2", ...), for ncu launch lists
(tools/profile_round.sh)."""
import sys
sys.path.insert(0, ".")
from paper_1811_11248_b200 import hsolve as H
from problems import gen_config
from problems.generators import gen_config_scaled
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
base, _, k = name.partition("/")
p = gen_config_scaled(base, int(k)) if k else gen_config(base)
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
x, rep = H.hs_pcg(f, p.b, tol=p.tol)
print(rep)
