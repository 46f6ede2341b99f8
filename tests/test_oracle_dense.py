"""Pins P5 and P9: the oracle's dense primitives against hand
examples (tests/golden/spec_examples.json), closed forms and the SVD."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle.dense import chol, tri_solve, cpqr, larfg, apply_Q, apply_Qt, NotSPD
from oracle.factor import BlockStore, eliminate

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_chol_hand_example():
    g = GOLD["chol_spd"]
    G = chol(np.array(g["A"]))
    assert np.allclose(G, np.array(g["G"]), rtol=0, atol=1e-15)


def test_chol_indefinite_reports_pivot():
    g = GOLD["chol_indefinite"]
    with pytest.raises(NotSPD) as ei:
        chol(np.array(g["A"]), level=3, cluster=7)
    assert ei.value.pivot == g["pivot"] and ei.value.level == 3 and ei.value.cluster == 7
    assert ei.value.value == pytest.approx(1.0 - 4.0)      # 1 - 2*2/1


def test_tri_solve_hand_example():
    g = GOLD["tri_solve"]
    X = tri_solve(np.array(g["G"]), np.array(g["B"]))
    assert np.allclose(X, np.array(g["X"]), rtol=0, atol=1e-15)


def test_exact_schur_hand_example():
    """Eliminating s={0} with w = {} (plain block Cholesky) leaves the
    exact Schur complement (Eq. exact_sc) on the neighbour block."""
    g = GOLD["exact_schur"]
    A = np.array(g["A"])
    st = BlockStore([1, 2])
    st.blocks[(0, 0)] = A[:1, :1]
    st.blocks[(1, 0)] = A[1:, :1]
    st.blocks[(1, 1)] = A[1:, 1:]
    e = eliminate(st, 0, 0, [1], [], 1e-2, True)
    assert e.r == 0
    assert np.allclose(st.get(1, 1), np.array(g["S"]), rtol=0, atol=1e-15)


def _synth(m, k, sigma, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, m)))
    V, _ = np.linalg.qr(rng.standard_normal((k, k)))
    S = np.zeros((m, k))
    for i, s in enumerate(sigma):
        S[i, i] = s
    return U @ S @ V.T


def test_truncation_rank_hand_example():
    g = GOLD["truncation_rank"]
    for seed in range(5):
        B = _synth(8, 12, g["sigma"], seed)
        res = cpqr(B, g["eps"], relative=False)
        assert res.r == g["rank"]


def test_larfg_convention():
    x = np.array([3.0, 4.0])
    v, tau, beta = larfg(x)
    assert beta == pytest.approx(-5.0)
    H = np.eye(2) - tau * np.outer(v, v)
    assert np.allclose(H @ x, [beta, 0.0], atol=1e-15)
    v, tau, beta = larfg(np.array([0.0, 2.0]))          # sign(0) = +1
    assert beta == pytest.approx(-2.0)
    v, tau, beta = larfg(np.array([-1.5, 0.0, 0.0]))    # zero sub-column -> H = I
    assert tau == 0.0 and beta == -1.5


@pytest.mark.parametrize("seed", range(6))
def test_cpqr_properties(seed):
    """P9: sigma_{r+1}(B) <= ||V2|| <= ||R22||_F <= sqrt(k-r) tau_s (so the SVD rank
    at threshold sqrt(k-r) tau_s never exceeds r); every kept |R_jj| > tau_s;
    U^T U = I; Q W = B; rank monotone in eps."""
    rng = np.random.default_rng(100 + seed)
    m, k = 24, 60
    sig = np.logspace(0, -8, m)
    B = _synth(m, k, sig, seed) * 3.7
    prev = -1
    for eps in [1e-1, 1e-2, 1e-3, 1e-4, 1e-6]:
        res = cpqr(B, eps)
        s = np.linalg.svd(B, compute_uv=False)
        tail = res.W[res.r:]
        nt = np.linalg.norm(tail, 2) if tail.size else 0.0
        if res.r < m:
            assert s[res.r] <= nt * (1 + 1e-10) + 1e-14
        assert int(np.sum(s > np.sqrt(k - res.r) * res.tau_s * (1 + 1e-12))) <= res.r
        assert all(abs(res.W[j, res.piv[j]]) > res.tau_s for j in range(res.r))
        assert nt <= np.linalg.norm(tail) + 1e-15
        assert np.linalg.norm(tail) <= np.sqrt(k - res.r) * res.tau_s * (1 + 1e-12)
        # orthogonality of U = Q and reconstruction B = Q W
        Q = apply_Q(res.V, res.tau, np.eye(m))
        assert np.abs(Q.T @ Q - np.eye(m)).max() < 1e-14
        assert np.abs(Q @ res.W - B).max() < 1e-13 * np.abs(B).max()
        assert np.allclose(apply_Qt(res.V, res.tau, B), res.W, atol=1e-13 * np.abs(B).max())
        assert res.r >= prev
        prev = res.r


def test_cpqr_matches_lapack_pivots_generic():
    """Independent implementation check: on a generic tie-free matrix the
    pivot order and |diag R| agree with LAPACK dgeqp3."""
    rng = np.random.default_rng(7)
    B = rng.standard_normal((10, 30)) * np.logspace(0, -3, 30)[None, :]
    res = cpqr(B, 0.0)
    Q, R, P = sla.qr(B, pivoting=True, mode="economic")
    assert list(res.piv) == list(P[:10])
    d = np.array([res.W[j, res.piv[j]] for j in range(10)])
    assert np.allclose(np.abs(d), np.abs(np.diag(R)), rtol=1e-12)


def test_cpqr_exact_rank_deficient():
    """Exactly rank-deficient inputs stop at the true rank for every eps >= 1e-12."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((16, 5))
    Y = rng.standard_normal((40, 5))
    B = X @ Y.T
    for eps in [1e-12, 1e-8, 1e-4]:
        assert cpqr(B, eps).r == 5
    Z = rng.standard_normal((16, 40))
    Z[9:] = 0.0                                   # zero rows: rank 9
    for eps in [1e-12, 1e-6]:
        assert cpqr(Z, eps).r == 9
    assert cpqr(np.zeros((4, 6)), 1e-2).r == 0


def test_cpqr_ties_pick_lowest_canonical_index():
    # columns 1 and 3 have exactly equal largest norms; column 1 must be chosen
    B = np.array([[0.0, 3.0, 1.0, 0.0],
                  [1.0, 4.0, 0.0, 5.0],
                  [0.0, 0.0, 1.0, 0.0]])
    res = cpqr(B, 0.0)
    assert res.piv[0] == 1
    B2 = B[:, [3, 0, 2, 1]]                        # now the tie sits at columns 0 and 3
    assert cpqr(B2, 0.0).piv[0] == 0


def test_cpqr_inject_replays_decisions():
    rng = np.random.default_rng(11)
    B = rng.standard_normal((8, 20))
    ref = cpqr(B, 1e-1)
    res = cpqr(B, 1e-1, inject=(ref.r, ref.piv))
    assert res.r == ref.r and list(res.piv) == list(ref.piv)
    assert np.array_equal(res.W, ref.W)
    forced = cpqr(B, 1e-1, inject=(3, [5, 1, 2]))
    assert forced.r == 3 and list(forced.piv) == [5, 1, 2]
