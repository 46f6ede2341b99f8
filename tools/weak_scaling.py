"""NEXT f2: the weak-scaling families (6 and 11 element layers x 2 DOF/node, 4x DOFs per
level) on one GPU: analyze once per problem, factor twice (the second factor re-uses the
analysis and the cached pattern: P:763's sequence of systems with one pattern), PCG to the
config tolerance and GMRES(200) to 1e-12.  Prints one JSON line per problem.
usage: python tools/weak_scaling.py [max_level]"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1811_11248_b200 import hsolve as H
from problems import gen_family

max_level = int(sys.argv[1]) if len(sys.argv) > 1 else 3
h = H.hs_create(0)
for layers in (6, 11):
    for level in range(max_level + 1):
        p = gen_family(layers, level)
        t0 = time.perf_counter()
        a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                         leaf_columns=p.leaf_columns)
        t_an = time.perf_counter() - t0
        f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
        del f
        f = H.hs_factor_create(h, a, p.vals * 1.0, eps=p.eps)       # re-factor, same analysis
        st = H.hs_factor_get_stats(f)
        x, rp = H.hs_pcg(f, p.b, tol=p.tol, raise_not_converged=False)
        x2, rg = H.hs_gmres(f, p.b, tol=1e-12, restart=200, maxit=1000, raise_not_converged=False)
        print(json.dumps({"layers": layers, "level": level, "n": p.n, "t_analyze_s": round(t_an, 3),
                          "t_factor_s": st["t_factor_s"], "pcg_iters": rp["iters"], "t_pcg_s": rp["t_pcg_s"],
                          "pcg_relres_true": rp["relres_true"], "gmres_iters": rg["iters"],
                          "t_gmres_s": rg["t_pcg_s"], "gmres_relres_true": rg["relres_true"],
                          "dof_per_s": p.n / (st["t_factor_s"] + rp["t_pcg_s"]),
                          "factor_gb": st["factor_bytes"] / 1e9, "max_rank": st["max_rank"]}), flush=True)
        del f
