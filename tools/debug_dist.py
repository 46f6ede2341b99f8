"""Debug aid: first cluster (elimination order) whose kept rank differs between the
single-GPU factor and the loopback-distributed factor."""
import sys, threading
sys.path.insert(0, ".")
import numpy as np
from paper_1811_11248_b200 import hsolve as H
from problems import gen_laplace3d, gen_poisson2d
from oracle.analyze import analyze
from oracle.dist import owner
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = gen_laplace3d(24, leaf_size=27)
an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
h1 = H.hs_create(0)
a1 = H.hs_analyze(h1, p.n, p.rowptr, p.colind, p.coords, None, leaf_size=p.leaf_size)
f1 = H.hs_factor_create(h1, a1, p.vals, eps=1e-2)
w = H.LoopbackWorld(world)
hs = [H.hs_create_loopback(0, w, r) for r in range(world)]
ans = [H.hs_analyze(hs[r], p.n, p.rowptr, p.colind, p.coords, None, leaf_size=p.leaf_size) for r in range(world)]
fs = [None] * world
def run(r):
    fs[r] = H.hs_factor_create(hs[r], ans[r], p.vals, eps=1e-2)
th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in th]; [t.join() for t in th]
for l, lev in enumerate(an.levels):
    r1 = H.hs_factor_export(f1, H.HS_FEXP_RANKS, l)
    rd = H.hs_factor_export(fs[0], H.HS_FEXP_RANKS, l)
    if np.array_equal(r1, rd):
        print("level", l, "ok"); continue
    for bi, B in enumerate(lev.batches):
        bad = [s for s in B if r1[s] != rd[s]]
        if bad:
            s = bad[0]
            print(f"level {l} batch {bi} (nphase1 {lev.nphase1}, {len(lev.batches)} batches) cluster {s}: r1 {r1[s]} rd {rd[s]}")
            print("  owner", owner(an, l, s, world), "interior", bool(lev.interior[s]))
            print("  n:", [(q, owner(an, l, q, world)) for q in lev.nlist[s]])
            print("  w:", [(q, owner(an, l, q, world)) for q in lev.wlist[s]])
            print("  other bad in batch:", bad[:10])
            break
    break
