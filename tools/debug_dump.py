"""Debug aid: compare the GPU block store after every batch (HS_DEBUG_DUMP) with the oracle's."""
import os, sys, copy, struct
import numpy as np
sys.path.insert(0, '.')
from problems import gen_stokes_q1, gen_laplace3d
from oracle.analyze import analyze
from oracle.factor import factor

def read_dump(path):
    data = open(path, 'rb').read()
    off = 0
    out = {}
    while off < len(data):
        p, q, rp, rq = struct.unpack_from('4i', data, off); off += 16
        M = np.frombuffer(data, dtype=np.float64, count=rp * rq, offset=off).reshape(rp, rq); off += 8 * rp * rq
        out[(p, q)] = M
    return out

name = sys.argv[1]
gen, kw, eps = {"q1": (lambda: gen_stokes_q1(12, 10, 5, leaf_columns=2), {}, 1e-2),
                "3d8": (lambda: gen_laplace3d(8, leaf_size=8), dict(top_log2=2, nsub_log2=2), 0.0)}[name]
p = gen()
kw = dict(top_log2=kw.get("top_log2", 3), nsub_log2=kw.get("nsub_log2", 3))
d = f"gpurun_out/dump_{name}"
if sys.argv[2] == "gpu":
    os.makedirs(d, exist_ok=True)
    os.environ["HS_DEBUG_DUMP"] = d
    from paper_1811_11248_b200 import hsolve as H
    h = H.hs_create(0)
    a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns, **kw)
    f = H.hs_factor_create(h, a, p.vals, eps=eps)
    print("dumped", len(os.listdir(d)))
else:
    an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns, **kw)
    snaps = {}
    factor(an, p.rowptr, p.colind, p.vals, eps=eps, snapshot=lambda l, b, st: snaps.__setitem__((l, b), copy.deepcopy(st)))
    for (l, b), st in sorted(snaps.items()):
        g = read_dump(f"{d}/l{l}_b{b}.bin")
        worst, where = 0.0, None
        scale = max(np.abs(st.get(a, b_)).max() if st.get(a, b_).size else 0.0 for (a, b_) in g)
        for (pp, qq), M in g.items():
            O = st.get(pp, qq)
            if pp == qq:          # diagonal blocks keep lower-triangle semantics on the GPU
                O, M = np.tril(O), np.tril(M)
            if O.shape != M.shape:
                print("shape", l, b, pp, qq, O.shape, M.shape); worst = np.inf; continue
            if M.size:
                e = np.abs(M - O).max() / scale
                if e > worst: worst, where = e, (pp, qq)
        print(f"l{l} b{b} worst {worst:.2e} at {where} batch {an.levels[l].batches[b][:8]}")
        if worst > 1e-8:
            pp, qq = where
            print(" gpu\n", g[where][:4, :6], "\n oracle\n", st.get(pp, qq)[:4, :6])
            break
if len(sys.argv) > 3:
    l, b, pp, qq = map(int, sys.argv[3:7])
    np.set_printoptions(precision=3, linewidth=200, suppress=True)
    print(read_dump(f"{d}/l{l}_b{b}.bin")[(pp, qq)])
    print(snaps[(l, b)].get(pp, qq))
