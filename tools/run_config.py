"""Run factor + PCG on a config (or a horizontally scaled proxy "C4/4") on the GPU and print
shape/time statistics.  usage: python tools/run_config.py NAME [EPS]; env LEAF_COLUMNS,
COARSE_FILL (analyze reading), REPS."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_1811_11248_b200 import hsolve as H  # noqa: E402
from problems.generators import gen_config, gen_config_scaled  # noqa: E402

name = sys.argv[1]
eps = float(sys.argv[2]) if len(sys.argv) > 2 else None
kw = {}
if os.environ.get("LEAF_COLUMNS"):
    kw["leaf_columns"] = int(os.environ["LEAF_COLUMNS"])
t = time.time()
p = gen_config_scaled(*name.split("/")[:1], int(name.split("/")[1])) if "/" in name else gen_config(name, **kw)
tg = time.time() - t
if eps is not None:
    p.eps = eps
print(f"{name}: N={p.n} nnz={p.nnz} gen {tg:.1f}s", flush=True)
h = H.hs_create(0)
t = time.time()
a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                 leaf_columns=p.leaf_columns, coarse_fill=int(os.environ.get("COARSE_FILL", "0")))
print("analyze", round(time.time() - t, 2), H.hs_analysis_get_info(a), flush=True)
for rep in range(int(os.environ.get("REPS", "2"))):
    t = time.time()
    f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
    st = H.hs_factor_get_stats(f)
    print(f"factor wall {time.time()-t:.2f}s dev {st['t_factor_s']:.3f}s batches {st['n_batches']} levels {st['n_levels']} "
          f"max_m {st['max_m']} max_r {st['max_rank']} n_top {st['n_top']} GF {st['flops']/1e9:.1f} GB {st['factor_bytes']/1e9:.2f}",
          flush=True)
    print("  level device times (ms):", [round(1e3 * t, 2) for t in st["t_level_s"]], flush=True)
    x, rep_ = H.hs_pcg(f, p.b, tol=p.tol, raise_not_converged=False)
    print("pcg", {k: rep_[k] for k in ("iters", "converged", "relres_true", "t_pcg_s")}, flush=True)
    if rep == 0:
        ranks = [H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(st["n_levels"])]
        live = [H.hs_factor_export(f, H.HS_FEXP_LIVE0, l) for l in range(st["n_levels"])]
        for l, (r, m) in enumerate(zip(ranks, live)):
            print(f"  level {l}: sum m {m.sum()} sum r {r.sum()} mean m {m.mean():.1f} max m {m.max()} "
                  f"mean r {r.mean():.1f} max r {r.max()}", flush=True)
        del f
