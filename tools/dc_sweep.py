"""NEXT f1 measurement: with vs without deferred compression (hs_factor_opts.dc = 1 / 0)
over eps in {1e-1, 1e-2, 1e-3, 1e-4} on C4-shaped (Q1 first-order-Stokes-type, 6 element
layers x 2 DOF) and C3-shaped (thin anisotropic slab, 10 layers) refinement families:
PCG (tol 1e-8) and GMRES(200) (tol 1e-12) iteration counts, factor time, memory.
The paper's contrast is Table `partition_steps` vs Table `ds` (iterations 83 -> 16 at 8 km,
eps = 1e-2) on Antarctica matrices that are not available; these are synthetic stand-ins.
usage: python tools/dc_sweep.py [max_level]   (one JSON line per run)"""
import json, sys
sys.path.insert(0, ".")
from paper_1811_11248_b200 import hsolve as H
from problems import gen_family, gen_slab

max_level = int(sys.argv[1]) if len(sys.argv) > 1 else 2
h = H.hs_create(0)
fams = [("q1-6layers", lambda lv: gen_family(6, lv)), ("slab-10layers", lambda lv: gen_slab(64 << lv, 10))]
for fname, gen in fams:
    for level in range(max_level + 1):
        p = gen(level)
        a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                         leaf_columns=p.leaf_columns)
        for eps in (1e-1, 1e-2, 1e-3, 1e-4):
            for dc in (1, 0):
                row = {"family": fname, "level": level, "n": p.n, "eps": eps, "dc": dc}
                try:
                    f = H.hs_factor_create(h, a, p.vals, eps=eps, dc=dc)
                    st = H.hs_factor_get_stats(f)
                    x, rp = H.hs_pcg(f, p.b, tol=1e-8, maxit=1000, raise_not_converged=False)
                    x2, rg = H.hs_gmres(f, p.b, tol=1e-12, restart=200, maxit=1000, raise_not_converged=False)
                    row.update({"t_factor_s": st["t_factor_s"], "factor_gb": st["factor_bytes"] / 1e9,
                                "pcg_iters": rp["iters"], "pcg_converged": rp["converged"],
                                "gmres_iters": rg["iters"], "gmres_converged": rg["converged"],
                                "gmres_relres_true": rg["relres_true"]})
                    del f
                except H.HSError as e:
                    row["error"] = str(e)[:160]
                print(json.dumps(row), flush=True)
