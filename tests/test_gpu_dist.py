"""The multi-GPU factor on ONE device (-m gpu): world_size ranks run as host
threads, each with its own handle, analysis, stream and rank-local block store; the
library's loopback transport turns the NCCL exchanges into device-to-device copies ordered
by events (hs_create_loopback).  Everything above the transport -- ownership, held blocks,
local phase I, the rank all-reduces, the phase-II records, the gathers to rank 0 -- is the
code the NCCL path runs.  The distributed factor must reproduce the single-GPU factor (same
kept ranks for every cluster), and the distributed solve -- every rank keeps and applies
only its own elimination records (owner-computes Algorithm 2, phase-II contribution and
halo exchanges, the top on rank 0), PCG with a halo SpMV and all-reduced dots -- must give
every rank the single-GPU result (apply within 1e-11, PCG with the same iteration count and
x within 1e-10), which tests/test_gpu_parity.py pins to the oracle; oracle/dist.py pins the
protocol (tests/test_dist_oracle.py)."""
import threading

import numpy as np
import pytest

from problems import gen_poisson2d, gen_laplace3d, gen_slab, gen_stokes_q1

pytestmark = pytest.mark.gpu

CASES = {
    "C1": lambda: gen_poisson2d(32),
    "3d-24": lambda: gen_laplace3d(24, leaf_size=27),
    "slab-32": lambda: gen_slab(32, 6, leaf_columns=4),
    "q1-12": lambda: gen_stokes_q1(12, 10, 5, leaf_columns=2),
}


@pytest.fixture(scope="module")
def H():
    import torch
    from paper_1811_11248_b200 import hsolve
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    hsolve.lib()
    return hsolve


def _analyze(H, p, h=None):
    return H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                        leaf_columns=p.leaf_columns)


def _dist_factor(H, p, world, eps):
    w = H.LoopbackWorld(world)
    hs = [H.hs_create_loopback(0, w, r) for r in range(world)]
    an = [_analyze(H, p, hs[r]) for r in range(world)]
    out, err = [None] * world, [None] * world

    def run(r):
        try:
            out[r] = H.hs_factor_create(hs[r], an[r], p.vals, eps=eps)
        except Exception as e:   # noqa: BLE001 - reported below
            err[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not any(err), err
    return w, hs, an, out


def _collective(world, fn):
    """Run fn(rank) on every rank at once (the distributed calls are collective)."""
    out, err = [None] * world, [None] * world

    def run(r):
        try:
            out[r] = fn(r)
        except Exception as e:   # noqa: BLE001 - reported below
            err[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not any(err), err
    return out


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", list(CASES))
def test_distributed_factor_and_solve_equal_single_gpu(H, name, world):
    eps = 1e-2
    p = CASES[name]()
    h1 = H.hs_create(0)
    a1 = _analyze(H, p, h1)
    f1 = H.hs_factor_create(h1, a1, p.vals, eps=eps)
    w, hs, an, fs = _dist_factor(H, p, world, eps)
    L = H.hs_analysis_get_info(a1)["L_top"]
    for l in range(L):
        assert np.array_equal(H.hs_factor_export(fs[0], H.HS_FEXP_RANKS, l),
                              H.hs_factor_export(f1, H.HS_FEXP_RANKS, l)), f"level {l} ranks"
    assert np.array_equal(H.hs_factor_export(fs[0], H.HS_FEXP_TOP), H.hs_factor_export(f1, H.HS_FEXP_TOP))
    # no factor gather: every rank holds about 1/P of the factor's elimination records
    for sd in (1, 2, 3):
        v = np.random.default_rng(sd).standard_normal(p.n)
        x1 = H.hs_apply(f1, v)
        xs = _collective(world, lambda r: H.hs_apply(fs[r], v))
        for xd in xs:
            assert np.linalg.norm(xd - x1) <= 1e-11 * np.linalg.norm(x1)
    y1 = H.hs_spmv(f1, p.b)
    ys = _collective(world, lambda r: H.hs_spmv(fs[r], p.b))
    for yd in ys:
        assert np.allclose(yd, y1, rtol=1e-14, atol=1e-13 * np.abs(y1).max())
    xs1, r1 = H.hs_pcg(f1, p.b, tol=p.tol)
    outs = _collective(world, lambda r: H.hs_pcg(fs[r], p.b, tol=p.tol))
    for xsd, rd in outs:
        assert rd["iters"] == r1["iters"] and rd["converged"]
        assert np.linalg.norm(xsd - xs1) <= 1e-10 * np.linalg.norm(xs1)
        assert np.allclose(rd["history"], r1["history"], rtol=1e-8, atol=1e-15)
        assert rd["relres_true"] <= 10 * p.tol
    del fs, hs, an, w
