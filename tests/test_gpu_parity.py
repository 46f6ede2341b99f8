"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle on the
same seeded inputs (SURVEY §8(c) parity protocol, north_star tolerances):
  * ranks identical for every cluster whose threshold margin mu_s >= 1e-10 and pivot
    margin pi_s >= 1e-11; flagged clusters are replayed in the oracle by decision
    injection with the GPU's pivots,
  * factor apply on 3 seeded N(0,1) vectors within 1e-9 relative,
  * PCG solution within 1e-8 relative and iterations within +-1,
  * eps = 0: exact Cholesky, relative residual <= 1e-12 and one PCG iteration.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from problems import gen_poisson2d, gen_laplace3d, gen_slab, gen_stokes_q1
from oracle.analyze import analyze
from oracle.factor import factor as ofactor
from oracle.solve import apply as oapply, pcg as opcg
from parity_helpers import oracle_with_injection, apply_parity as _apply_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch
    from paper_1811_11248_b200 import hsolve
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    hsolve.lib()
    return hsolve


@pytest.fixture(scope="module")
def handle(H):
    return H.hs_create(0)


def _both(H, handle, p, eps, kw=None, dc=1):
    kw = kw or {}
    top_log2 = kw.get("top_log2", 3)
    nsub_log2 = kw.get("nsub_log2", 3)
    an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                 leaf_columns=p.leaf_columns, top_log2=top_log2, nsub_log2=nsub_log2)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns, top_log2=top_log2, nsub_log2=nsub_log2)
    f = H.hs_factor_create(handle, a, p.vals, eps=eps, dc=dc)
    if eps == 0.0:
        # eps = 0 keeps every nonzero: decisions on rounding noise are not comparable,
        # and both sides are exact Cholesky factorizations (checked by the caller)
        return an, None, a, f, 0
    fac, flagged, injected, nelim = oracle_with_injection(H, f, an, p, eps, dc=dc)
    # decision injection is an exemption for fragile clusters, not a way to pass: report it
    # and bound it ("make the exemption visible")
    print(f"[parity] eliminations {nelim} flagged {flagged} injected {injected}")
    assert injected <= max(2, nelim // 200), f"{injected} of {nelim} clusters needed decision injection"
    assert np.array_equal(H.hs_factor_export(f, H.HS_FEXP_TOP), fac.top_sizes)
    return an, fac, a, f, injected


TINY = [
    ("C1", lambda: gen_poisson2d(32), {}),
    ("2d-8x8", lambda: gen_poisson2d(8, leaf_size=4), dict(top_log2=1, nsub_log2=1)),
    ("3d-8", lambda: gen_laplace3d(8, leaf_size=8), dict(top_log2=2, nsub_log2=2)),
    ("q1-4x4x3", lambda: gen_stokes_q1(4, 4, 3, leaf_columns=1), dict(top_log2=1, nsub_log2=1)),
]


@pytest.mark.parametrize("name,gen,kw", TINY, ids=[t[0] for t in TINY])
def test_eps0_exact_cholesky(H, handle, name, gen, kw):
    p = gen()
    an, fac, a, f, _ = _both(H, handle, p, 0.0, kw)
    A = p.to_scipy().toarray()
    x_ref = sla.cho_solve(sla.cho_factor(A), p.b)
    x = H.hs_apply(f, p.b)
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-12
    x2, rep = H.hs_pcg(f, p.b, tol=1e-10)
    assert rep["iters"] == 1 and rep["relres_true"] <= 1e-12


def _NoCoords(p):
    """The problem without coordinates: analyze uses graph bisection (NEXT f4)."""
    import copy
    q = copy.copy(p)
    q.coords, q.column_id, q.leaf_columns = None, None, 0
    return q


CASES = TINY + [
    ("graph-3d-16", lambda: _NoCoords(gen_laplace3d(16, leaf_size=16)), {}),
    ("graph-C1", lambda: _NoCoords(gen_poisson2d(32)), {}),
    ("aniso2d-ragged", lambda: gen_poisson2d(23, 17, aniso=1e-3, leaf_size=7), dict(top_log2=2, nsub_log2=1)),
    ("3d-24", lambda: gen_laplace3d(24, leaf_size=27), {}),
    ("slab-32", lambda: gen_slab(32, 6, leaf_columns=4), {}),
    ("q1-12", lambda: gen_stokes_q1(12, 10, 5, leaf_columns=2), {}),
    # clusters larger than the shared-memory POTRF/TRSM limit (m = 216 at level 0, up to 432 above)
    ("3d-12-bigleaf", lambda: gen_laplace3d(12, leaf_size=216), dict(top_log2=1, nsub_log2=1)),
]


def test_eps0_big_clusters(H, handle):
    p = gen_laplace3d(12, leaf_size=216)
    an, _, a, f, _ = _both(H, handle, p, 0.0, dict(top_log2=1, nsub_log2=1))
    A = p.to_scipy().toarray()
    x_ref = sla.cho_solve(sla.cho_factor(A), p.b)
    x = H.hs_apply(f, p.b)
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-12
    assert H.hs_factor_get_stats(f)["max_m"] > 128


@pytest.mark.parametrize("eps", [1e-2, 1e-1, 1e-4])
@pytest.mark.parametrize("name,gen,kw", CASES, ids=[t[0] for t in CASES])
def test_factor_apply_pcg_parity(H, handle, name, gen, kw, eps):
    p = gen()
    an, fac, a, f, flagged = _both(H, handle, p, eps, kw)
    _apply_parity(H, f, fac, p.n)
    xo, ro = opcg(p.to_scipy(), p.b, lambda r: oapply(fac, r), tol=p.tol)
    xg, rg = H.hs_pcg(f, p.b, tol=p.tol)
    assert abs(rg["iters"] - ro.iters) <= 1
    assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-8
    assert rg["relres_true"] <= 10 * p.tol


def test_device_pointers_and_spmv(H, handle):
    import torch
    p = gen_poisson2d(32)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, None, leaf_size=16)
    f = H.hs_factor_create(handle, a, p.vals, eps=1e-2)
    bt = torch.tensor(p.b, device="cuda", dtype=torch.float64)
    xt = H.hs_apply(f, bt)
    xh = H.hs_apply(f, p.b)
    assert np.array_equal(xt.cpu().numpy(), xh)
    y = H.hs_spmv(f, p.b)
    assert np.allclose(y, p.to_scipy() @ p.b, rtol=1e-14, atol=1e-13)
    xg, rep = H.hs_pcg(f, bt, tol=1e-10)
    assert rep["converged"] and rep["relres_true"] <= 1e-9


def test_not_spd_reports_breakdown(H, handle):
    p = gen_poisson2d(8, leaf_size=4)
    vals = p.vals.copy()
    # make row/col 0 strongly indefinite: diagonal -> -1
    d0 = p.rowptr[0] + np.searchsorted(p.colind[p.rowptr[0]:p.rowptr[1]], 0)
    vals[d0] = -1.0
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, None, leaf_size=4, top_log2=1, nsub_log2=1)
    with pytest.raises(H.HSError) as ei:
        H.hs_factor_create(handle, a, vals, eps=1e-2)
    assert ei.value.status == H.HS_E_NOT_SPD
    assert "level 0" in str(ei.value)


def test_empty_leaves_and_tiny(H, handle):
    # U = 10 DOFs, leaf 1 -> 16 leaves with 6 empty: degenerate clusters stay in the schedule
    p = gen_poisson2d(5, 2, leaf_size=1)
    an, fac, a, f, _ = _both(H, handle, p, 1e-2, dict(top_log2=1, nsub_log2=1))
    _apply_parity(H, f, fac, p.n)
    an, _, a, f, _ = _both(H, handle, p, 0.0, dict(top_log2=1, nsub_log2=1))
    A = p.to_scipy().toarray()
    assert np.linalg.norm(H.hs_apply(f, p.b) - np.linalg.solve(A, p.b)) <= 1e-12 * np.linalg.norm(np.linalg.solve(A, p.b))


@pytest.mark.parametrize("name,gen,kw", [CASES[0], CASES[7], CASES[9]], ids=[CASES[0][0], CASES[7][0], CASES[9][0]])
def test_gmres_parity(H, handle, name, gen, kw):
    """NEXT f3: the paper's Krylov protocol (right-preconditioned GMRES(200), tol 1e-12,
    P:810) on the GPU against the oracle's textbook GMRES with the oracle's factor."""
    from oracle.solve import gmres as ogmres
    p = gen()
    an, fac, a, f, flagged = _both(H, handle, p, 1e-2, kw)
    xo, ro = ogmres(p.to_scipy(), p.b, lambda r: oapply(fac, r), tol=1e-12, restart=200, maxit=1000)
    xg, rg = H.hs_gmres(f, p.b, tol=1e-12, restart=200, maxit=1000)
    assert ro.converged and rg["converged"]
    assert abs(rg["iters"] - ro.iters) <= 1
    assert np.linalg.norm(xg - xo) <= 1e-8 * np.linalg.norm(xo)
    assert rg["relres_true"] <= 1e-10
    # a short restart still converges (restarted path)
    xr, rr = H.hs_gmres(f, p.b, tol=1e-10, restart=2, maxit=1000)
    assert rr["converged"] and rr["relres_true"] <= 1e-8


def test_analyze_once_factor_many(H, handle):
    """NEXT f2 / P:763 (Newton and continuation produce a sequence of systems with one
    pattern) on the weak-scaling family (gen_family: the C4 operator at 6 element layers, the
    paper's Table `ilu` family shape): re-factoring new values on the same analysis (cached
    pattern and scatter map) matches the ORACLE on those values (ranks, pivots, apply, PCG),
    equals a fresh analysis bit for bit, and re-factoring the same values is deterministic.
    (Scaling A by alpha is NOT a symmetry of the method: the coarse DOFs live in the
    G-scaled space with diagonal I_r, so their couplings scale by sqrt(alpha) while
    unprocessed blocks scale by alpha; the oracle shows the same.)"""
    import copy
    from problems import gen_family
    p = gen_family(6, 0)
    an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size, leaf_columns=p.leaf_columns)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_columns=p.leaf_columns)
    f1 = H.hs_factor_create(handle, a, p.vals, eps=p.eps)
    # a symmetric perturbation: scale row i and column i by d_i (D A D stays SPD)
    d = 1.0 + 0.2 * np.sin(np.arange(p.n))
    rows = np.repeat(np.arange(p.n), np.diff(p.rowptr))
    p2 = copy.copy(p)
    p2.vals = p.vals * d[rows] * d[p.colind]
    f2 = H.hs_factor_create(handle, a, p2.vals, eps=p.eps)
    for q, f in ((p, f1), (p2, f2)):   # both factors of the sequence against the oracle
        fac, flagged, injected, nelim = oracle_with_injection(H, f, an, q, q.eps)
        assert injected <= max(2, nelim // 200)
        _apply_parity(H, f, fac, q.n)
        xo, ro = opcg(q.to_scipy(), q.b, lambda r: oapply(fac, r), tol=q.tol)
        xg, rg = H.hs_pcg(f, q.b, tol=q.tol)
        assert abs(rg["iters"] - ro.iters) <= 1
        assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-8
    a_new = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_columns=p.leaf_columns)
    f3 = H.hs_factor_create(handle, a_new, p2.vals, eps=p.eps)
    v = np.random.default_rng(4).standard_normal(p.n)
    assert np.array_equal(H.hs_apply(f2, v), H.hs_apply(f3, v))
    f4 = H.hs_factor_create(handle, a, p.vals, eps=p.eps)
    assert np.array_equal(H.hs_apply(f4, v), H.hs_apply(f1, v))


NODC = [CASES[0], CASES[3], CASES[7], CASES[8], CASES[9], CASES[10]]


@pytest.mark.parametrize("eps", [1e-2, 1e-1])
@pytest.mark.parametrize("name,gen,kw", NODC, ids=[t[0] for t in NODC])
def test_no_deferred_compression_parity(H, handle, name, gen, kw, eps):
    """NEXT f1: the original LoRaSp step (hs_factor_opts.dc = 0: CPQR of the unscaled A_sw,
    rotation of A_ss from both sides, fine Cholesky, coarse-block update) against
    oracle/factor.py eliminate_nodc: ranks and pivots (decision injection for flagged
    clusters), apply within 1e-9, PCG within 1e-8 and +-1 iteration."""
    p = gen()
    an, fac, a, f, flagged = _both(H, handle, p, eps, kw, dc=0)
    _apply_parity(H, f, fac, p.n)
    xo, ro = opcg(p.to_scipy(), p.b, lambda r: oapply(fac, r), tol=p.tol)
    xg, rg = H.hs_pcg(f, p.b, tol=p.tol)
    assert abs(rg["iters"] - ro.iters) <= 1
    assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-8


@pytest.mark.parametrize("name,gen,kw", TINY, ids=[t[0] for t in TINY])
def test_no_deferred_compression_eps0_exact(H, handle, name, gen, kw):
    p = gen()
    an, fac, a, f, _ = _both(H, handle, p, 0.0, kw, dc=0)
    A = p.to_scipy().toarray()
    x_ref = sla.cho_solve(sla.cho_factor(A), p.b)
    assert np.linalg.norm(H.hs_apply(f, p.b) - x_ref) / np.linalg.norm(x_ref) <= 1e-12


@pytest.mark.gpu
def test_repeated_factor_pipeline_is_deterministic(H, handle):
    """The factor pipelines batches (the host plans batch b+1 while batch b's second half
    is still queued, the apply plan is built on a host worker): repeated factors of the
    same system in one process must be bit-identical and never fault.  A larger 3-D case
    (hundreds of batches, many sequential ones) so that staging reuse is exercised."""
    p = gen_laplace3d(32, leaf_size=64)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=64)
    v = np.random.default_rng(7).standard_normal(p.n)
    ref = None
    for _ in range(6):
        f = H.hs_factor_create(handle, a, p.vals, eps=1e-2)
        x = H.hs_apply(f, v)
        if ref is None:
            ref = x
        else:
            assert np.array_equal(x, ref)
        del f


@pytest.mark.gpu
def test_pipeline_modes_agree(H, handle, monkeypatch):
    """The batch pipeline's modes compute the same factor: the device patch with the ranks
    read one batch late vs the synchronous host patch, and the direct write-back (CPQR /
    n-rotation write row s and C_s themselves) vs the write-back pass — bit for bit, since
    they only move the same values; the gather + POTRF + TRSM kernels vs the gather-free
    Cholesky + column-tile scaling to rounding.  (All with dense level-0 blocks: the modes
    without the direct write-back keep them dense; test_support_restricted_level0_* compares
    the support-restricted level 0 with it.)"""
    p = gen_laplace3d(24, leaf_size=27)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=27)
    v = np.random.default_rng(11).standard_normal(p.n)

    def run(**env):
        for k in ("HS_HOST_PATCH", "HS_NO_DIRECT_WB", "HS_NO_FUSED_POTRF_TRSM"):
            monkeypatch.delenv(k, raising=False)
        monkeypatch.setenv("HS_NO_KHAT", "1")
        for k, val in env.items():
            monkeypatch.setenv(k, val)
        f = H.hs_factor_create(handle, a, p.vals, eps=1e-2)
        x = H.hs_apply(f, v)
        r = [H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(H.hs_analysis_get_info(a)["L_top"])]
        del f
        return x, r

    x0, r0 = run()
    for env in ({"HS_HOST_PATCH": "1"}, {"HS_NO_DIRECT_WB": "1"}):
        x1, r1 = run(**env)
        assert all(np.array_equal(u, w) for u, w in zip(r0, r1)), env
        assert np.array_equal(x1, x0), env
    x2, r2 = run(HS_NO_FUSED_POTRF_TRSM="1")
    assert all(np.array_equal(u, w) for u, w in zip(r0, r2))
    assert np.linalg.norm(x2 - x0) <= 1e-11 * np.linalg.norm(x0)


def test_apply_nan_input_terminates(H, handle):
    """The apply polls contribution / x VALUES against an all-ones 'empty' pattern: a NaN
    carried in from the input (or produced inside) is stored canonically, so the sweeps
    terminate and the NaN propagates instead of hanging the GPU."""
    p = gen_laplace3d(16, leaf_size=16)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, None, leaf_size=16)
    f = H.hs_factor_create(handle, a, p.vals, eps=1e-2)
    b = p.b.copy()
    b[[3, p.n // 2]] = np.nan
    x = H.hs_apply(f, b)
    assert np.isnan(x).any()
    b[3] = -np.nan
    x = H.hs_apply(f, b)
    assert np.isnan(x).any()
    assert np.all(np.isfinite(H.hs_apply(f, p.b)))   # the factor is still usable


def test_device_inputs_from_torch_stream(H, handle):
    """Inputs produced by torch on its own stream (torch.randn on the GPU, no host round trip)
    are read only once they are written (the wrapper waits for torch's stream)."""
    import torch
    p = gen_laplace3d(24, leaf_size=27)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, None, leaf_size=27)
    f = H.hs_factor_create(handle, a, p.vals, eps=1e-2)
    g = torch.Generator(device="cuda").manual_seed(3)
    for _ in range(3):
        big = torch.randn(1 << 26, device="cuda", dtype=torch.float64, generator=g)   # keep torch's stream busy
        bt = torch.randn(p.n, device="cuda", dtype=torch.float64, generator=g) * 2.0 + big[:p.n] * 0.0
        xt = H.hs_apply(f, bt)
        xh = H.hs_apply(f, bt.cpu().numpy())
        assert np.array_equal(xt.cpu().numpy(), xh)
    with pytest.raises(H.HSError):
        H.hs_apply(f, torch.zeros(p.n - 1, device="cuda", dtype=torch.float64))
    with pytest.raises(H.HSError):
        H.hs_apply(f, torch.zeros(p.n, device="cuda", dtype=torch.float32))
    with pytest.raises(H.HSError):
        H.hs_apply(f, p.b, x=np.zeros(p.n, dtype=np.float32))
    # the report carries the residual history and the SpMV time
    x, rep = H.hs_pcg(f, p.b, tol=1e-8)
    h = rep["history"]
    assert len(h) == rep["iters"] + 1 and h[0] == 1.0 and h[-1] <= 1e-8 < h[-2]
    assert rep["t_spmv_s"] > 0
    st = H.hs_factor_get_stats(f)
    assert len(st["t_level_s"]) == st["n_levels"] and all(t > 0 for t in st["t_level_s"])
    assert abs(sum(st["flops_level"]) - st["flops"]) <= 1e-6 * st["flops"] + st["n_top"] ** 3
    kn0 = H.hs_factor_export(f, H.HS_FEXP_KN, 0)
    kw0 = H.hs_factor_export(f, H.HS_FEXP_KW, 0)
    nleaf = H.hs_analysis_export(a, H.HS_EXP_LEAF_OFF).size - 1
    assert kn0.size == kw0.size == nleaf and kn0.sum() > 0 and kw0.sum() > 0


@pytest.mark.gpu
def test_small_level_path_agrees_with_batch_pipeline(H, handle, monkeypatch):
    """Levels of small clusters run one device-planned kernel per wave (small.cu); the batch
    pipeline (HS_NO_SMALL_LEVELS=1) computes the same factor: identical kept ranks and pivots,
    the preconditioner to rounding.  (Both are compared with the oracle by the parity tests.)"""
    from problems import gen_slab
    p = gen_slab(64, 10, leaf_columns=8)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_columns=8)
    L = H.hs_analysis_get_info(a)["L_top"]
    v = np.random.default_rng(12).standard_normal(p.n)

    def run(**env):
        monkeypatch.delenv("HS_NO_SMALL_LEVELS", raising=False)
        for k, val in env.items():
            monkeypatch.setenv(k, val)
        f = H.hs_factor_create(handle, a, p.vals, eps=1e-2)
        out = ([H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(L)],
               [H.hs_factor_export(f, H.HS_FEXP_PIV, l) for l in range(L)], H.hs_apply(f, v))
        del f
        return out

    r0, p0, x0 = run()
    r1, p1, x1 = run(HS_NO_SMALL_LEVELS="1")
    assert all(np.array_equal(u, w) for u, w in zip(r0, r1))
    assert all(np.array_equal(u, w) for u, w in zip(p0, p1))
    assert np.linalg.norm(x1 - x0) <= 1e-11 * np.linalg.norm(x0)


@pytest.mark.parametrize("cfg", ["C3/4", "C2/2", "C4/16"])
def test_support_restricted_level0_is_the_dense_computation(H, handle, monkeypatch, cfg):
    """Level 0 runs on the structurally nonzero columns of each block only (support.cpp,
    SURVEY O2.10): a zero column stays zero through the scaling, the CPQR (never a pivot) and
    the rotation, and the Schur products only reach supported columns -- so the factor is the
    dense one (HS_NO_KHAT=1): identical kept ranks, canonical pivots and top block, the same
    preconditioner to rounding."""
    from problems.generators import gen_config_scaled
    name, k = cfg.split("/")
    p = gen_config_scaled(name, int(k))
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    L = H.hs_analysis_get_info(a)["L_top"]
    v = np.random.default_rng(21).standard_normal(p.n)

    def run(**env):
        monkeypatch.delenv("HS_NO_KHAT", raising=False)
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        f = H.hs_factor_create(handle, a, p.vals, eps=p.eps)
        st = H.hs_factor_get_stats(f)
        out = ([H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(L)],
               [H.hs_factor_export(f, H.HS_FEXP_PIV, l) for l in range(L)],
               H.hs_factor_export(f, H.HS_FEXP_TOP, 0), H.hs_apply(f, v), st["flops_level"][0])
        del f
        return out

    r0, p0, t0, x0, fl0 = run()
    r1, p1, t1, x1, fl1 = run(HS_NO_KHAT="1")
    assert all(np.array_equal(u, w) for u, w in zip(r0, r1))
    assert all(np.array_equal(u, w) for u, w in zip(p0, p1))
    assert np.array_equal(t0, t1)
    # the records hold the supported columns only: the apply sums fewer (zero) terms per
    # lane, so it agrees to rounding
    assert np.linalg.norm(x1 - x0) <= 1e-13 * np.linalg.norm(x1)
    assert fl0 < fl1   # the level-0 work shrinks with the supports


@pytest.mark.parametrize("cfg", ["C3/4", "C2/2"])
def test_batch_synchronous_apply_matches_dependency_sweep(H, handle, monkeypatch, cfg):
    """Levels of large batches apply the factor with one launch per batch (k_apply_fwd_b /
    k_apply_bwd_b); the dependency-driven level kernels (HS_APPLY_DEP=1) compute the same
    Algorithm 2 sweep with another summation order: the preconditioned vectors agree to
    rounding and PCG takes the same iterations."""
    from problems.generators import gen_config_scaled
    name, k = cfg.split("/")
    p = gen_config_scaled(name, int(k))
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    v = np.random.default_rng(22).standard_normal(p.n)

    def run(**env):
        monkeypatch.delenv("HS_APPLY_DEP", raising=False)
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        f = H.hs_factor_create(handle, a, p.vals, eps=p.eps)
        x = H.hs_apply(f, v)
        _, rep = H.hs_pcg(f, p.b, tol=p.tol)
        del f
        return x, rep["iters"]

    x0, i0 = run()
    x1, i1 = run(HS_APPLY_DEP="1")
    assert np.linalg.norm(x1 - x0) <= 1e-12 * np.linalg.norm(x0)
    assert i0 == i1
