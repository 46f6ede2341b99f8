"""Boundary (CPU): libhsolve.so loads, exports every symbol include/hsolve.h declares,
and hs_analyze (host integer code) reproduces the oracle's analyze bit for bit
(SURVEY §8(c) parity protocol: "Analyze exports: bit-equal")."""
import os
import re

import numpy as np
import pytest

from problems import gen_poisson2d, gen_laplace3d, gen_slab, gen_stokes_q1
from oracle.analyze import analyze
from paper_1811_11248_b200 import hsolve as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "hsolve.h")).read()
    decl = set(re.findall(r"^\s*(?:hs_status|void|const char\*|int64_t)\s+(hs_\w+)\s*\(", hdr, re.M))
    assert decl == set(H.SYMBOLS)
    L = H.lib()
    for s in decl:
        assert hasattr(L, s), s


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HSError) as ei:
        H.hs_create(0)
    assert ei.value.status == H.HS_E_NO_DEVICE


def _csr(adj):
    ptr = [0]
    idx = []
    for r in adj:
        idx += list(r)
        ptr.append(len(idx))
    return np.array(ptr, dtype=np.int64), np.array(idx, dtype=np.int64)


CASES = [
    ("C1", lambda: gen_poisson2d(32), {}),
    ("C1-top1", lambda: gen_poisson2d(32), dict(top_log2=1, nsub_log2=1)),
    ("aniso2d-ragged", lambda: gen_poisson2d(23, 17, leaf_size=7), dict(top_log2=2, nsub_log2=1)),
    ("3d-16", lambda: gen_laplace3d(16, leaf_size=16), {}),
    ("C2", lambda: gen_laplace3d(64), {}),
    ("slab", lambda: gen_slab(40, 6, leaf_columns=5), {}),
    ("q1", lambda: gen_stokes_q1(13, 11, 4, leaf_columns=3), dict(top_log2=2, nsub_log2=2)),
]


def _NoCoords(p):
    """The problem with its coordinates removed: analyze falls back to graph bisection."""
    import copy
    q = copy.copy(p)
    q.coords, q.column_id, q.leaf_columns = None, None, 0
    if not q.leaf_size:
        q.leaf_size = 40
    return q


CASES += [
    ("graph-C1", lambda: _NoCoords(gen_poisson2d(32)), {}),
    ("graph-3d-16", lambda: _NoCoords(gen_laplace3d(16, leaf_size=16)), {}),
    ("graph-aniso-ragged", lambda: _NoCoords(gen_poisson2d(23, 17, leaf_size=7)), dict(top_log2=2, nsub_log2=1)),
    ("graph-q1", lambda: _NoCoords(gen_stokes_q1(9, 7, 3, leaf_columns=2)), {}),
]


@pytest.mark.parametrize("coarse_fill", [0, 1])
@pytest.mark.parametrize("name,gen,kw", CASES, ids=[c[0] for c in CASES])
def test_analyze_bit_exact(name, gen, kw, coarse_fill):
    p = gen()
    top_log2 = kw.get("top_log2", 3)
    nsub_log2 = kw.get("nsub_log2", 3)
    orc = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                  leaf_columns=p.leaf_columns, top_log2=top_log2, nsub_log2=nsub_log2, coarse_fill=coarse_fill)
    a = H.hs_analyze(None, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns, top_log2=top_log2, nsub_log2=nsub_log2, coarse_fill=coarse_fill)
    info = H.hs_analysis_get_info(a)
    assert (info["depth"], info["L_top"]) == (orc.D, orc.L_top)
    assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_PERM), orc.perm)
    assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_LEAF_OFF), orc.leaf_off)
    for l, lev in enumerate(orc.levels):
        for kp, ki, adj in [(H.HS_EXP_H_PTR, H.HS_EXP_H_IDX, lev.H), (H.HS_EXP_W_PTR, H.HS_EXP_W_IDX, lev.wlist),
                            (H.HS_EXP_BATCH_PTR, H.HS_EXP_BATCH_IDX, lev.batches),
                            (H.HS_EXP_F_PTR, H.HS_EXP_F_IDX, lev.Ffinal),
                            (H.HS_EXP_FS_PTR, H.HS_EXP_FS_IDX, lev.Fstart)]:
            ptr, idx = _csr(adj)
            assert np.array_equal(H.hs_analysis_export(a, kp, l), ptr), (l, kp)
            assert np.array_equal(H.hs_analysis_export(a, ki, l), idx), (l, ki)
        assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_INTERIOR, l), lev.interior.astype(np.int64))
        assert H.hs_analysis_export(a, H.HS_EXP_NPHASE1, l)[0] == lev.nphase1
    ptr, idx = _csr(orc.H_top)
    assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_HTOP_PTR), ptr)
    assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_HTOP_IDX), idx)


def test_analyze_errors():
    p = gen_poisson2d(8)
    with pytest.raises(H.HSError) as ei:   # graph bisection needs DOF units
        H.hs_analyze(None, p.n, p.rowptr, p.colind, None, np.zeros(p.n, dtype=np.int32), leaf_size=4,
                     leaf_columns=2)
    assert ei.value.status == H.HS_E_UNSUPPORTED
    with pytest.raises(H.HSError) as ei:
        H.hs_analyze(None, p.n, p.rowptr, p.colind, p.coords, None, leaf_size=0)
    assert ei.value.status == H.HS_E_INVALID_ARG
    # unsymmetric pattern: drop one stored entry
    colind = p.colind.copy()
    rowptr = p.rowptr.copy()
    keep = np.ones(p.nnz, dtype=bool)
    keep[1] = False
    counts = np.diff(rowptr)
    counts[0] -= 1
    rp = np.zeros_like(rowptr)
    rp[1:] = np.cumsum(counts)
    with pytest.raises(H.HSError) as ei:
        H.hs_analyze(None, p.n, rp, colind[keep], p.coords, None, leaf_size=4)
    assert ei.value.status == H.HS_E_NOT_SYMMETRIC
