"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (-m gpu):
the CUDA path against the oracle on EVERY cluster of EVERY level (ranks and pivot sequences,
decision injection only for clusters the margins flag, counted and bounded), the factor
apply on 3 seeded vectors (1e-9), PCG (1e-8, +-1 iteration) -- SURVEY §8(c) parity protocol.

  * C3 (the bench's default workload, 655,360 DOF) and C2 (262,144 DOF) at full size;
  * the C2 family at eps = 1e-4 (32^3; BASELINE configs[1] lists eps 1e-2 and 1e-4);
  * the C4 operator (Q1 first-order-Stokes-type, 2 DOF/node, 20 layers) on a 1/16 horizontal
    grid (40,960 DOF; its ranks make the oracle take ~2 min even so): C4 itself does not fit
    one B200 (bench.py docstring);
  * the C5 operator on a 1/64 grid (128-DOF leaves: the non-fused m > 112 path);
  * the CPQR kernel's global-memory mode (W streamed through L2, taken when a block does not
    fit a 16-CTA cluster's shared memory) forced on a case with wide blocks;
plus the analyze schedule bit-exact, operator properties (symmetry, positivity, linearity),
the SpMV on sampled rows, and bitwise determinism of repeated factors.
"""
import os
import time

import numpy as np
import pytest

from problems import gen_config, gen_laplace3d
from problems.generators import gen_config_scaled
from oracle.analyze import analyze
from oracle.solve import apply as oapply, pcg as opcg
from parity_helpers import oracle_with_injection, apply_parity

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


def _analysis_equal(H, a, an):
    info = H.hs_analysis_get_info(a)
    assert info["L_top"] == an.L_top and info["depth"] == an.D
    assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_PERM), an.perm)
    for l, lev in enumerate(an.levels):
        flat = np.concatenate([np.asarray(b, dtype=np.int64) for b in lev.batches]) if lev.batches else np.zeros(0)
        assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_BATCH_IDX, l), flat), f"level {l} batches"


def _operator_properties(H, f, n, seeds=(11, 12, 13)):
    for sd in seeds:
        rng = np.random.default_rng(sd)
        u, v = rng.standard_normal(n), rng.standard_normal(n)
        Mu, Mv = H.hs_apply(f, u), H.hs_apply(f, v)
        scale = np.linalg.norm(Mu) * np.linalg.norm(v)
        assert abs(Mu @ v - u @ Mv) <= 1e-12 * scale            # symmetry
        assert u @ Mu > 0 and v @ Mv > 0                        # positivity
        a, b = 0.75, -1.5
        Mw = H.hs_apply(f, a * u + b * v)
        assert np.linalg.norm(Mw - (a * Mu + b * Mv)) <= 1e-12 * np.linalg.norm(Mw)   # linearity


def _full_parity(H, handle, p, label):
    t0 = time.perf_counter()
    an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                 leaf_columns=p.leaf_columns)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    _analysis_equal(H, a, an)
    f = H.hs_factor_create(handle, a, p.vals, eps=p.eps)
    fac, flagged, injected, nelim = oracle_with_injection(H, f, an, p, p.eps)
    print(f"[fullsize {label}] N={p.n} eliminations {nelim} flagged {flagged} injected {injected} "
          f"(oracle {time.perf_counter() - t0:.0f} s)")
    assert injected <= max(2, nelim // 200)
    assert np.array_equal(H.hs_factor_export(f, H.HS_FEXP_TOP), fac.top_sizes)
    worst = apply_parity(H, f, fac, p.n)
    A = p.to_scipy()
    xo, ro = opcg(A, p.b, lambda r: oapply(fac, r), tol=p.tol)
    xg, rg = H.hs_pcg(f, p.b, tol=p.tol)
    print(f"[fullsize {label}] apply parity {worst:.2e}, PCG iters gpu {rg['iters']} oracle {ro.iters}, "
          f"x rel diff {np.linalg.norm(xg - xo) / np.linalg.norm(xo):.2e}")
    assert abs(rg["iters"] - ro.iters) <= 1
    assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-8
    res = np.linalg.norm(p.b - A @ xg) / np.linalg.norm(p.b)
    assert res <= 10 * p.tol and abs(res - rg["relres_true"]) <= 1e-3 * res + 1e-15
    return a, f


@pytest.mark.parametrize("name", ["C3", "C2"])
def test_full_size_config_parity(H, handle, name):
    p = gen_config(name)
    a, f = _full_parity(H, handle, p, name)
    _operator_properties(H, f, p.n)
    A = p.to_scipy()
    x = np.random.default_rng(5).standard_normal(p.n)
    y = H.hs_spmv(f, x)
    rows = np.random.default_rng(6).choice(p.n, 2000, replace=False)
    assert np.allclose(y[rows], A[rows] @ x, rtol=1e-13, atol=1e-12)


def test_c2_family_eps_1e4(H, handle):
    p = gen_laplace3d(32)
    p.eps = 1e-4
    _full_parity(H, handle, p, "C2 family 32^3 eps 1e-4")


def test_c4_operator_sixteenth_scale(H, handle):
    p = gen_config_scaled("C4", 16)
    _full_parity(H, handle, p, "C4/16")


def test_c5_operator_sixtyfourth_scale(H, handle):
    """The C5 operator (1024^2 x 16 node layers, aspect 1e4, 4-column leaves of 128 DOF: the
    clusters above the fused kernels' 112-DOF limit, i.e. the gather / k_potrf / k_trsm path,
    coarse clusters up to m = 318 and a 1,286-DOF top) on a 1/64 horizontal grid (8,192 DOF).
    At 1/32 a coarse cluster already exceeds the kernels' 512-DOF limit (HS_E_UNSUPPORTED,
    DESIGN.md §5); C5 itself needs several GPUs."""
    p = gen_config_scaled("C5", 64)
    _full_parity(H, handle, p, "C5/64")


def test_cpqr_global_memory_mode(H, handle, monkeypatch):
    """k_cpqr3's global-memory mode (the w-slices streamed through L2 instead of staged in
    distributed shared memory) on wide blocks: same decisions and factor as the oracle."""
    monkeypatch.setenv("HS_CPQR_GLOBAL", "1")
    p = gen_laplace3d(24, leaf_size=27)
    p.eps = 1e-4
    _full_parity(H, handle, p, "3d-24 eps 1e-4, CPQR global mode")


@pytest.mark.parametrize("name", ["C3", "C2"])
def test_refactor_is_bitwise_deterministic(H, handle, name):
    """At the bench's sizes, in the bench's launch configuration: two factors on the same
    analysis give bit-identical kept ranks and preconditioner applications (every sum in the
    pipeline has a fixed order: batched kernels, L2 reductions with one update per target
    element per launch, the apply's polled contributions summed in plan order)."""
    p = gen_config(name)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    L = H.hs_analysis_get_info(a)["L_top"]
    v = np.random.default_rng(5).standard_normal(p.n)
    out = []
    for _ in range(2):
        f = H.hs_factor_create(handle, a, p.vals, eps=p.eps)
        out.append(([H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(L)], H.hs_apply(f, v)))
        del f
    assert all(np.array_equal(x, y) for x, y in zip(out[0][0], out[1][0]))
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("name", ["C4/16", "C2"])
def test_record_space_spill_restore_bitwise(H, handle, monkeypatch, name):
    """Large factors keep their T_s / C_s records in a virtual range whose completed chunks
    spill to pinned host memory while a later level's block store needs the device memory,
    and come back at the same addresses before the apply (RecSpace; C4 on one B200).  Forced
    here on every level end: the kept ranks and the preconditioner application are bitwise
    those of the factor whose records never left the device."""
    base, _, k = name.partition("/")
    p = gen_config_scaled(base, int(k)) if k else gen_config(base)
    a = H.hs_analyze(handle, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    L = H.hs_analysis_get_info(a)["L_top"]
    v = np.random.default_rng(7).standard_normal(p.n)
    out = {}
    # "force" twice on the same handle: the second factor pre-copies its completed chunks on the
    # copy stream during later levels (budget = the first one's spill), so its spills are event
    # waits on those copies
    for mode in ("0", "1", "force", "force-precopied"):
        monkeypatch.setenv("HS_RECSPACE", mode.partition("-")[0])
        f = H.hs_factor_create(handle, a, p.vals, eps=p.eps)
        x, rep = H.hs_pcg(f, v, tol=p.tol)
        out[mode] = ([H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(L)], H.hs_apply(f, v), x,
                     rep["iters"])
        del f
    for mode in ("1", "force", "force-precopied"):
        assert all(np.array_equal(x, y) for x, y in zip(out["0"][0], out[mode][0])), mode
        assert np.array_equal(out["0"][1], out[mode][1]), mode
        assert np.array_equal(out["0"][2], out[mode][2]), mode
        assert out["0"][3] == out[mode][3]
