"""C4 at full size on one GPU (-m gpu): BASELINE.json configs[3], the bench's default workload
(Q1 first-order-Stokes-type operator, 512 x 512 x 20 hexahedra, 2 DOF/node, 10,485,760 DOF,
eps 1e-2, PCG to 1e-8), in the launch configuration bench.py times.  At this size the factor
runs with the record space active (completed levels' T_s / C_s spilled to pinned host memory
while the 131 GB level-2 store is resident) and with oversized batches split into sub-batches
by the workspace budget -- the two paths only C4 takes.

The whole oracle factor of C4 is out of reach (hours of Python), and no cluster's input can be
reproduced on the host without replaying the elimination before it (the first batch of level 0,
whose blocks are A's own, has w(s) empty: no compression decision at all).  So this leg checks
what holds at any size (SURVEY §8(c) parity protocol, full-size leg):
  * the analysis (partition, cluster tree, every level's batches) bit-exact with oracle/analyze;
  * operator properties of the factor apply (symmetry, positivity, linearity);
  * PCG to the config's tolerance with the true residual recomputed against A on the host;
  * bitwise determinism across two factors (every level's kept ranks, the apply), i.e. the
    sub-batch split and the spill / restore of the records change nothing between runs.
The C4 operator itself is compared with the oracle on every cluster at 1/16 scale
(test_gpu_fullsize.py), and the spill / restore path bitwise against resident records there.
"""
import numpy as np
import pytest

from problems import gen_config
from oracle.analyze import analyze

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch
    from paper_1811_11248_b200 import hsolve
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    hsolve.lib()
    return hsolve


def test_c4_full_size(H):
    import gc
    p = gen_config("C4")
    assert p.n == 10_485_760
    h = H.hs_create(0)
    try:
        _c4_checks(H, h, p)
    finally:   # the handle's ~170 GB of cached device memory must not outlive the test
        h.close()
        gc.collect()


def _c4_checks(H, h, p):
    a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                 leaf_columns=p.leaf_columns)
    info = H.hs_analysis_get_info(a)
    assert info["L_top"] == an.L_top and info["depth"] == an.D
    assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_PERM), an.perm)
    for l, lev in enumerate(an.levels):
        flat = np.concatenate([np.asarray(b, dtype=np.int64) for b in lev.batches]) if lev.batches else np.zeros(0)
        assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_BATCH_IDX, l), flat), f"level {l} batches"

    L = H.hs_analysis_get_info(a)["L_top"]
    v = np.random.default_rng(5).standard_normal(p.n)
    runs = []
    for _ in range(2):
        f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
        runs.append(([H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(L)], H.hs_apply(f, v)))
        if len(runs) == 1:
            del f   # two C4 factors cannot coexist on one GPU
    assert all(np.array_equal(x, y) for x, y in zip(runs[0][0], runs[1][0]))
    assert np.array_equal(runs[0][1], runs[1][1])

    n = p.n
    for sd in (11, 12):
        rng = np.random.default_rng(sd)
        u, v = rng.standard_normal(n), rng.standard_normal(n)
        Mu, Mv = H.hs_apply(f, u), H.hs_apply(f, v)
        scale = np.linalg.norm(Mu) * np.linalg.norm(v)
        assert abs(Mu @ v - u @ Mv) <= 1e-12 * scale
        assert u @ Mu > 0 and v @ Mv > 0
        Mw = H.hs_apply(f, 0.75 * u - 1.5 * v)
        assert np.linalg.norm(Mw - (0.75 * Mu - 1.5 * Mv)) <= 1e-12 * np.linalg.norm(Mw)

    x, rep = H.hs_pcg(f, p.b, tol=p.tol)
    A = p.to_scipy()
    res = np.linalg.norm(p.b - A @ x) / np.linalg.norm(p.b)
    print(f"[C4] PCG {rep['iters']} iterations, true relative residual {res:.2e}")
    assert rep["converged"] and res <= 10 * p.tol
    assert abs(res - rep["relres_true"]) <= 1e-3 * res + 1e-15
