"""Shared GPU-parity helpers (SURVEY §8(c) parity protocol): decision injection for flagged
clusters and the factor-apply comparison."""
import numpy as np

from oracle.factor import factor as ofactor
from oracle.solve import apply as oapply


def oracle_with_injection(H, f, an, p, eps, max_rounds=200, dc=1):
    """Rank/pivot parity with the margin exemption: walk the clusters in elimination
    order; at the first disagreement, a flagged cluster gets the GPU's decisions
    injected into the oracle (which is re-run), an unflagged one fails the test.
    Returns (oracle factor, flagged clusters, injected clusters, eliminations)."""
    gpu = []
    for l in range(len(an.levels)):
        gpu.append((H.hs_factor_export(f, H.HS_FEXP_RANKS, l), H.hs_factor_export(f, H.HS_FEXP_PIV_PTR, l),
                    H.hs_factor_export(f, H.HS_FEXP_PIV, l)))
    inject = {}
    for _ in range(max_rounds):
        fac = ofactor(an, p.rowptr, p.colind, p.vals, eps=eps, inject=inject or None, dc=bool(dc))
        first = None
        nflag = nelim = 0
        for l, lv in enumerate(fac.elims):
            g_r, g_pp, g_pv = gpu[l]
            for eb in lv:
                for e in eb:
                    nflag += int(e.flagged)
                    nelim += 1
                    gpiv = g_pv[g_pp[e.s]:g_pp[e.s + 1]]
                    if (l, e.s) in inject or (g_r[e.s] == e.r and np.array_equal(gpiv, e.piv)):
                        continue
                    first = (l, e, gpiv)
                    break
                if first:
                    break
            if first:
                break
        if first is None:
            return fac, nflag, len(inject), nelim
        l, e, gpiv = first
        assert e.flagged, (f"decision mismatch at level {l} cluster {e.s} (unflagged, mu={e.mu:.2e}, "
                           f"pi={e.pi:.2e}): gpu r={gpu[l][0][e.s]} piv={list(gpiv)} oracle r={e.r} "
                           f"piv={list(e.piv)}")
        inject[(l, e.s)] = (int(gpu[l][0][e.s]), gpiv.tolist())
    raise AssertionError("decision injection did not converge")


def apply_parity(H, f, fac, n, seeds=(1, 2, 3), tol=1e-9):
    worst = 0.0
    for sd in seeds:
        v = np.random.default_rng(sd).standard_normal(n)
        xg = H.hs_apply(f, v)
        xo = oapply(fac, v)
        err = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
        worst = max(worst, err)
        assert err <= tol, f"apply parity {err:.3e}"
    return worst


