import sys, copy
import numpy as np
sys.path.insert(0, '.')
from problems import gen_stokes_q1
from oracle.analyze import analyze_problem
from oracle.factor import initial_blocks, eliminate
from oracle.dense import chol, tri_solve, apply_Q
from paper_1811_11248_b200 import hsolve as H
p = gen_stokes_q1(12, 10, 5, leaf_columns=2)
an = analyze_problem(p)
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
f = H.hs_factor_create(h, a, p.vals, eps=1e-2)
st = initial_blocks(an, p.rowptr, p.colind, p.vals)
lev = an.levels[0]
np.set_printoptions(precision=4, linewidth=220, suppress=True)
for B in lev.batches:
    for s in B:
        if s == 19:
            m = st.live[s]; ws = lev.wlist[s]; ns = lev.nlist[s]
            A_ss = st.get(s, s); A_sw = np.hstack([st.get(s, q) for q in ws]); A_sn = np.hstack([st.get(s, q) for q in ns])
            G = chol(A_ss); Bw = tri_solve(G, A_sw); Bn = tri_solve(G, A_sn)
            g = H.cluster_record(f, 0, s)
            print("shape", g["m"], g["r"], g["kw"], g["kn"], "oracle kw", Bw.shape, "kn", Bn.shape)
            Q = apply_Q(g["V"], g["tau"], np.eye(m))
            recon = Q @ g["B"]
            print("recon w err", np.abs(recon[:, :g["kw"]] - Bw).max(), "n err", np.abs(recon[:, g["kw"]:] - Bn).max())
            print("oracle nu", np.sqrt((Bw**2).sum(0)))
            print("gpu V cols", g["V"][:, :2].T)
            print("gpu tau", g["tau"])
            print("gpu B w-part rows 0..3\n", g["B"][:4, :g["kw"]])
            raise SystemExit
        eliminate(st, 0, s, lev.nlist[s], lev.wlist[s], 1e-2, True)
