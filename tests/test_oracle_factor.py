"""Pins P1-P4 and P6 of the oracle's factor and apply.

P1  eps = 0 reduces the whole pipeline to an exact Cholesky: M^{-1} b equals
    the dense solve (scipy cho_solve) and PCG stops after one iteration.
P2  batch 0 of level 0 has w = {}: the block store after it equals the
    dense exact Schur complement of the batch's DOFs (Eq. exact_sc).
P3  per-cluster deferred-compression identities (Prop. 2, Eq. err_new):
    E_nn = 0, E_ww = V2 V2^T, ||E_nw|| <= ||A_ns|| ||V2|| / sigma_min(A_ss)^{1/2}.
P4  Corollary: the ww block of each step's Schur complement is SPD.
P6  the apply is linear, symmetric and positive definite (factored form).
"""
import copy

import numpy as np
import pytest
import scipy.linalg as sla

from problems import gen_poisson2d, gen_laplace3d, gen_stokes_q1
from oracle.analyze import analyze, analyze_problem
from oracle.factor import factor, initial_blocks, eliminate, next_level, ranks
from oracle.solve import apply, pcg


def tiny_problems():
    """(problem, analyze kwargs) on tiny grids with several hierarchical levels."""
    return [
        (gen_poisson2d(32), dict()),                                       # C1
        (gen_poisson2d(8, leaf_size=4), dict(top_log2=1, nsub_log2=1)),    # 8x8 2-D
        (gen_laplace3d(8, leaf_size=8), dict(top_log2=2, nsub_log2=2)),    # 8^3 3-D
        (gen_stokes_q1(4, 4, 3, leaf_columns=1), dict(top_log2=1, nsub_log2=1)),  # 4x4x3 Q1, 2 DOF
    ]


def _an(p, kw):
    return analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                   leaf_columns=p.leaf_columns, **kw)


@pytest.mark.parametrize("idx", range(4))
def test_P1_eps0_is_exact_cholesky(idx):
    p, kw = tiny_problems()[idx]
    an = _an(p, kw)
    assert an.L_top >= 1
    fac = factor(an, p.rowptr, p.colind, p.vals, eps=0.0)
    A = p.to_scipy().toarray()
    x_ref = sla.cho_solve(sla.cho_factor(A), p.b)
    x = apply(fac, p.b)
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-12
    x2, rep = pcg(p.to_scipy(), p.b, lambda r: apply(fac, r), tol=1e-10)
    assert rep.iters == 1 and rep.converged


def test_P2_batch0_is_exact_schur():
    p = gen_poisson2d(32)
    an = analyze_problem(p)
    A = p.to_scipy().toarray()[np.ix_(an.perm, an.perm)]
    snaps = {}

    def snap(l, b, st):
        if (l, b) == (0, 0):
            snaps["st"] = copy.deepcopy(st)

    factor(an, p.rowptr, p.colind, p.vals, eps=1e-2, snapshot=snap)
    st = snaps["st"]
    off = an.leaf_off
    B0 = an.levels[0].batches[0]
    assert all(not an.levels[0].wlist[s] for s in B0)
    bd = np.concatenate([np.arange(off[s], off[s + 1]) for s in B0])
    rest = [c for c in range(len(off) - 1) if c not in set(B0)]
    rd = np.concatenate([np.arange(off[c], off[c + 1]) for c in rest])
    S = A[np.ix_(rd, rd)] - A[np.ix_(rd, bd)] @ np.linalg.solve(A[np.ix_(bd, bd)], A[np.ix_(bd, rd)])
    ro = {c: i for i, c in enumerate(rest)}
    co = np.zeros(len(rest) + 1, dtype=int)
    co[1:] = np.cumsum([off[c + 1] - off[c] for c in rest])
    got = np.zeros_like(S)
    for p_ in rest:
        for q in rest:
            got[co[ro[p_]]:co[ro[p_] + 1], co[ro[q]]:co[ro[q] + 1]] = st.get(p_, q)
    for s in B0:
        assert st.live[s] == 0
    assert np.abs(got - S).max() <= 1e-13 * np.abs(S).max()


def _dense_local(st, idx_lists):
    """Dense matrix of the current state over the listed clusters."""
    sizes = [st.live[c] for c in idx_lists]
    o = np.zeros(len(sizes) + 1, dtype=int)
    o[1:] = np.cumsum(sizes)
    M = np.zeros((o[-1], o[-1]))
    for a, p in enumerate(idx_lists):
        for b, q in enumerate(idx_lists):
            M[o[a]:o[a + 1], o[b]:o[b + 1]] = st.get(p, q)
    return M, o


@pytest.mark.parametrize("idx,eps", [(0, 1e-2), (0, 1e-1), (1, 1e-2), (2, 1e-1), (3, 1e-2)])
def test_P3_P4_deferred_compression_identities(idx, eps):
    p, kw = tiny_problems()[idx]
    an = _an(p, kw)
    st = initial_blocks(an, p.rowptr, p.colind, p.vals)
    checked = 0
    for l, lev in enumerate(an.levels):
        for B in lev.batches:
            for s in B:
                ns, ws = lev.nlist[s], lev.wlist[s]
                before = copy.deepcopy(st)
                e = eliminate(st, l, s, ns, ws, eps, True, keep_debug=True)
                if sum(e.wsz) == 0 or e.m == 0:
                    continue
                # exact Schur complement of all of s (Eq. exact_sc) on (n, w)
                M0, o0 = _dense_local(before, [s] + ns + ws)
                m = e.m
                Ass, Asr, Arr = M0[:m, :m], M0[:m, m:], M0[m:, m:]
                SA = Arr - Asr.T @ np.linalg.solve(Ass, Asr)
                # algorithm: state after, then also eliminate s's coarse DOFs (diagonal I_r)
                M1, o1 = _dense_local(st, [s] + ns + ws)
                r = e.r
                assert np.allclose(M1[:r, :r], np.eye(r), atol=0)
                Salg = M1[r:, r:] - M1[r:, :r] @ M1[:r, r:]
                E = Salg - SA
                kn = sum(e.nsz)
                scale = max(1.0, np.abs(SA).max())
                amax = lambda X: float(np.abs(X).max()) if X.size else 0.0
                assert amax(E[:kn, :kn]) <= 1e-11 * scale                                # E_nn = 0
                V2t = e.tail_w                                                           # V2^T
                assert amax(E[kn:, kn:] - V2t.T @ V2t) <= 1e-11 * scale                  # E_ww = V2 V2^T
                assert amax(E[:kn, kn:] - e.C.T @ V2t) <= 1e-11 * scale                  # E_nw = A_ns G^-T U2 V2^T
                if kn:
                    Ans = M0[m:m + kn, :m]
                    smin = np.linalg.eigvalsh(Ass).min()
                    bound = np.linalg.norm(Ans, 2) * np.linalg.norm(V2t, 2) / np.sqrt(smin)
                    assert np.linalg.norm(E[:kn, kn:], 2) <= bound * (1 + 1e-9) + 1e-12 * scale
                assert np.linalg.eigvalsh(V2t.T @ V2t).min() >= -1e-12 * scale          # E_ww PSD
                np.linalg.cholesky(Salg[kn:, kn:])                                       # P4: ww block SPD
                checked += 1
        Hn = an.levels[l + 1].H if l + 1 < len(an.levels) else an.H_top
        st = next_level(st, Hn, lev.nclus // 2)
    assert checked > 0


def test_P6_apply_linear_symmetric_positive():
    p = gen_poisson2d(32)
    an = analyze_problem(p)
    fac = factor(an, p.rowptr, p.colind, p.vals, eps=1e-2)
    rng = np.random.default_rng(5)
    U = rng.standard_normal((p.n, 100))
    MU = np.stack([apply(fac, U[:, i]) for i in range(100)], axis=1)
    G = U.T @ MU
    assert np.abs(G - G.T).max() <= 1e-12 * np.abs(G).max()
    assert np.all(np.diag(G) > 0)
    a, b = 0.7, -2.5
    lin = apply(fac, a * U[:, 0] + b * U[:, 1])
    assert np.abs(lin - (a * MU[:, 0] + b * MU[:, 1])).max() <= 1e-12 * np.abs(lin).max()


def test_eps_error_decreases():
    """The preconditioned error ||I - M^{-1}A|| shrinks with eps (P:812 trade-off)."""
    p = gen_poisson2d(16, aniso=1e-2, leaf_size=8)
    an = analyze(p.n, p.rowptr, p.colind, p.coords, None, leaf_size=8, top_log2=2, nsub_log2=2)
    A = p.to_scipy().toarray()
    errs = []
    for eps in [1e-1, 1e-2, 1e-4]:
        fac = factor(an, p.rowptr, p.colind, p.vals, eps=eps)
        MA = np.stack([apply(fac, A[:, i]) for i in range(p.n)], axis=1)
        errs.append(np.linalg.norm(np.eye(p.n) - MA, 2))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-2


def test_gmres_minimal_residual_pin():
    """Pin of the oracle GMRES (NEXT f3): after k Arnoldi steps from x0 = 0 the iterate
    minimises ||b - A M^{-1} u|| over the Krylov space K_k(A M^{-1}, b) -- checked against
    a brute-force least-squares solve over an explicitly built, QR-orthonormalised Krylov
    basis (no Arnoldi, no Givens); with the exact inverse as preconditioner it stops after
    one step."""
    import scipy.sparse.linalg as spla
    from oracle.solve import gmres
    p = gen_poisson2d(8, leaf_size=4)
    A = p.to_scipy()
    b = p.b
    D = A.diagonal()
    M = lambda v: v / D                               # Jacobi
    AM = lambda v: A @ M(v)
    for k in range(1, 7):
        x, rep = gmres(A, b, M, tol=1e-300, restart=50, maxit=k)
        K = np.zeros((b.size, k))
        v = b.copy()
        for i in range(k):
            K[:, i] = v
            v = AM(v)
        Q, _ = np.linalg.qr(K)
        AQ = np.column_stack([AM(Q[:, i]) for i in range(k)])
        c, *_ = np.linalg.lstsq(AQ, b, rcond=None)
        best = np.linalg.norm(b - AQ @ c)
        assert rep.iters == k
        assert abs(np.linalg.norm(b - A @ x) - best) <= 1e-10 * np.linalg.norm(b)
    lu = spla.splu(A.tocsc())
    x, rep = gmres(A, b, lu.solve, tol=1e-12)
    assert rep.iters == 1 and rep.converged and rep.relres_true <= 1e-12


def test_gmres_restart_converges():
    from oracle.solve import gmres
    p = gen_poisson2d(12, leaf_size=4)
    A = p.to_scipy()
    x, rep = gmres(A, p.b, lambda v: v, tol=1e-10, restart=5, maxit=2000)
    assert rep.converged and rep.restarts > 1 and rep.relres_true <= 1e-9


@pytest.mark.parametrize("idx", [0, 1, 2])
@pytest.mark.parametrize("eps", [1e-1, 1e-2])
def test_prop1_no_deferred_compression(idx, eps):
    """NEXT f1 pin: the original LoRaSp step (eliminate_nodc) followed by the exact
    elimination of s's coarse DOFs is one Cholesky step on s in the compressed matrix A~
    (P:168-185), so its error against the exact Schur complement S_A (Eq. exact_sc) is
    Eq. err_old: E_nn = 0, E_nw = A_ns A_ss^{-1} U2 V2^T, E_ww = A_ws A_ss^{-1} A_sw -
    V1 U1^T A_ss^{-1} U1 V1^T, with Proposition 1's bound ||E_nw|| <= ||V2|| ||A_ns|| / s_min."""
    from oracle.factor import eliminate_nodc
    from oracle.dense import apply_Q
    p, kw = tiny_problems()[idx]
    an = _an(p, kw)
    st = initial_blocks(an, p.rowptr, p.colind, p.vals)
    checked = 0
    for l, lev in enumerate(an.levels):
        for B in lev.batches:
            for s in B:
                ns, ws = lev.nlist[s], lev.wlist[s]
                before = copy.deepcopy(st)
                e = eliminate_nodc(st, l, s, ns, ws, eps, True, keep_debug=True)
                if sum(e.wsz) == 0 or e.m == 0:
                    continue
                M0, o0 = _dense_local(before, [s] + ns + ws)
                m, r = e.m, e.r
                Ass, Asr, Arr = M0[:m, :m], M0[:m, m:], M0[m:, m:]
                SA = Arr - Asr.T @ np.linalg.solve(Ass, Asr)
                M1, o1 = _dense_local(st, [s] + ns + ws)
                Salg = M1[r:, r:] - M1[r:, :r] @ np.linalg.solve(M1[:r, :r], M1[:r, r:]) if r else M1[r:, r:]
                E = Salg - SA
                kn = sum(e.nsz)
                Ans, Asw = Asr[:, :kn].T, Asr[:, kn:]
                Q = apply_Q(e.V, e.tau, np.eye(m))
                U1V1t = Q[:, :r] @ e.coarse_w                                           # U1 V1^T
                U2V2t = Q[:, r:] @ e.tail_w                                             # U2 V2^T
                assert np.allclose(U1V1t + U2V2t, Asw, atol=1e-11 * max(1.0, np.abs(Asw).max()))
                scale = max(1.0, np.abs(SA).max())
                amax = lambda X: float(np.abs(X).max()) if X.size else 0.0
                assert amax(E[:kn, :kn]) <= 1e-10 * scale                              # E_nn = 0
                Enw = Ans @ np.linalg.solve(Ass, U2V2t)
                assert amax(E[:kn, kn:] - Enw) <= 1e-10 * scale                        # E_nw
                Eww = Asw.T @ np.linalg.solve(Ass, Asw) - U1V1t.T @ np.linalg.solve(Ass, U1V1t)
                assert amax(E[kn:, kn:] - Eww) <= 1e-10 * scale                        # E_ww
                if kn:
                    smin = np.linalg.eigvalsh(Ass).min()
                    bound = np.linalg.norm(e.tail_w, 2) * np.linalg.norm(Ans, 2) / smin
                    assert np.linalg.norm(E[:kn, kn:], 2) <= bound * (1 + 1e-9) + 1e-12 * scale
                checked += 1
        Hn = an.levels[l + 1].H if l + 1 < len(an.levels) else an.H_top
        st = next_level(st, Hn, lev.nclus // 2)
    assert checked > 0


@pytest.mark.parametrize("idx", [0, 1, 2, 3])
def test_P1_no_dc_eps0_exact(idx):
    """NEXT f1: with eps = 0 the original LoRaSp factorization is also an exact Cholesky."""
    p, kw = tiny_problems()[idx]
    an = _an(p, kw)
    fac = factor(an, p.rowptr, p.colind, p.vals, eps=0.0, dc=False)
    A = p.to_scipy().toarray()
    x = apply(fac, p.b)
    assert np.linalg.norm(x - np.linalg.solve(A, p.b)) <= 1e-12 * np.linalg.norm(np.linalg.solve(A, p.b))


def test_no_dc_apply_symmetric_positive():
    p = gen_poisson2d(32)
    an = analyze_problem(p)
    fac = factor(an, p.rowptr, p.colind, p.vals, eps=1e-2, dc=False)
    rng = np.random.default_rng(7)
    U = rng.standard_normal((p.n, 20))
    MU = np.stack([apply(fac, U[:, i]) for i in range(20)], axis=1)
    G = U.T @ MU
    assert np.abs(G - G.T).max() <= 1e-12 * np.abs(G).max()
    assert np.all(np.linalg.eigvalsh(0.5 * (G + G.T)) > 0)
