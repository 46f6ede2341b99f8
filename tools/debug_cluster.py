"""Debug aid: compare every cluster's elimination record (G, coarse rows, C) GPU vs oracle."""
import sys
import numpy as np
sys.path.insert(0, '.')
from problems import gen_stokes_q1, gen_laplace3d, gen_poisson2d
from oracle.analyze import analyze
from oracle.factor import factor
from paper_1811_11248_b200 import hsolve as H

cases = {"q1": (lambda: gen_stokes_q1(12, 10, 5, leaf_columns=2), {}, 1e-2),
         "3d8": (lambda: gen_laplace3d(8, leaf_size=8), dict(top_log2=2, nsub_log2=2), 0.0)}
for name, (gen, kw, eps) in cases.items():
    p = gen()
    an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                 leaf_columns=p.leaf_columns, top_log2=kw.get("top_log2", 3), nsub_log2=kw.get("nsub_log2", 3))
    h = H.hs_create(0)
    a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns, top_log2=kw.get("top_log2", 3), nsub_log2=kw.get("nsub_log2", 3))
    f = H.hs_factor_create(h, a, p.vals, eps=eps)
    fac = factor(an, p.rowptr, p.colind, p.vals, eps=eps, keep_debug=True)
    bad = 0
    for l, lv in enumerate(fac.elims):
        for bi, eb in enumerate(lv):
            for e in eb:
                g = H.cluster_record(f, l, e.s)
                if e.m == 0:
                    continue
                dG = np.abs(np.tril(g["G"]) - e.G).max() / np.abs(e.G).max()
                msg = f"{name} L{l} b{bi} s{e.s} m{e.m} r{e.r}/{g['r']} dG {dG:.1e}"
                if g["r"] == e.r and e.r > 0:
                    cw = np.abs(g["B"][:e.r, :g["kw"]] - e.coarse_w).max() / max(np.abs(e.coarse_w).max(), 1e-300)
                    msg += f" dcw {cw:.1e}"
                if dG > 1e-10 or g["r"] != e.r:
                    print(msg, "piv", e.piv[:6])
                    bad += 1
                    if bad > 5:
                        break
            if bad > 5:
                break
        if bad > 5:
            break
    print(name, "done, bad", bad)
