import sys, time
sys.path.insert(0, ".")
import torch
from paper_1811_11248_b200 import hsolve as H
from problems.generators import gen_config_scaled
name, scale = sys.argv[1], int(sys.argv[2])
p = gen_config_scaled(name, scale)
print(name, "scale", scale, "N", p.n, "nnz", p.nnz, flush=True)
h = H.hs_create(0)
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
print(H.hs_analysis_get_info(a), flush=True)
free0, tot = torch.cuda.mem_get_info()
for rep in range(2):
    t = time.time()
    f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
    st = H.hs_factor_get_stats(f)
    free1, _ = torch.cuda.mem_get_info()
    print(f"factor wall {time.time()-t:.2f}s dev {st['t_factor_s']:.3f}s batches {st['n_batches']} max_m {st['max_m']} "
          f"max_r {st['max_rank']} n_top {st['n_top']} GF {st['flops']/1e9:.1f} factorGB {st['factor_bytes']/1e9:.2f} "
          f"devmem used {(free0-free1)/1e9:.1f} GB", flush=True)
    x, r = H.hs_pcg(f, p.b, tol=p.tol, raise_not_converged=False)
    print("pcg", {k: r[k] for k in ("iters", "converged", "relres_true", "t_pcg_s")}, flush=True)
    del f
