"""O4 Apply (Algorithm 2 `Hierarchical_Solve`) and O5 PCG (oracle; test infrastructure only).

Apply computes x = M^{-1} b with A^fac = W_0^{-1} ... W_{m-1}^{-1} diag(I, A_c^fac) W^{-T}...
(Alg. 1 line "return A^fac") and W_s = P_s G_s E_s S_s:
  forward  (y <- W_i y for i = 0..m-1):
      y_s <- U^T G_s^{-1} y_s ; y_f = y_s[r:] is final ; y_q -= C[:, q]^T y_f for q in n(s)
  top      y_top <- L^{-T} L^{-1} y_top (the base-case Cholesky)
  backward (x <- W_i^T x for i = m-1..0):
      x_f <- y_f - sum_q C[:, q] x_q ; x_s <- G_s^{-T} U [x_c; x_f]
PCG (O5) is the SPD Krylov driver named by north_star (the paper uses GMRES; reading Q16).
"""
from __future__ import annotations

import dataclasses
import numpy as np
import scipy.linalg as sla

from .dense import apply_Qt, apply_Q
from .factor import Factor


def apply(fac: Factor, b: np.ndarray) -> np.ndarray:
    an = fac.an
    b = np.asarray(b, dtype=np.float64)
    bp = b[an.perm]
    off = an.leaf_off
    y = [bp[off[c]:off[c + 1]].copy() for c in range(off.shape[0] - 1)]
    fine = {}
    # forward substitution
    for l, lv in enumerate(fac.elims):
        for eb in lv:
            for e in eb:
                t = sla.solve_triangular(e.G, y[e.s], lower=True) if e.m else y[e.s].copy()
                t = apply_Qt(e.V, e.tau, t)
                yf = t[e.r:]
                fine[(l, e.s)] = yf
                o = 0
                for q, k in zip(e.nlist, e.nsz):
                    assert y[q].shape[0] == k
                    y[q] = y[q] - e.C[:, o:o + k].T @ yf
                    o += k
                y[e.s] = t[:e.r]
        nclus = len(y) // 2
        y = [np.concatenate([y[2 * P], y[2 * P + 1]]) for P in range(nclus)]
    # top
    ytop = np.concatenate(y) if y else np.zeros(0)
    if ytop.shape[0]:
        z = sla.solve_triangular(fac.L, ytop, lower=True)
        xtop = sla.solve_triangular(fac.L, z, lower=True, trans="T")
    else:
        xtop = ytop
    x = []
    o = 0
    for c in range(len(y)):
        k = y[c].shape[0]
        x.append(xtop[o:o + k])
        o += k
    # backward substitution
    for l in reversed(range(len(fac.elims))):
        live_end = fac.live1[l]
        xs = []
        for P in range(len(x)):
            k0 = live_end[2 * P]
            xs.append(x[P][:k0])
            xs.append(x[P][k0:])
        x = xs
        for eb in reversed(fac.elims[l]):
            for e in reversed(eb):
                xf = fine[(l, e.s)].copy()
                o = 0
                for q, k in zip(e.nlist, e.nsz):
                    assert x[q].shape[0] == k
                    xf = xf - e.C[:, o:o + k] @ x[q]
                    o += k
                t = np.concatenate([x[e.s], xf])
                t = apply_Q(e.V, e.tau, t)
                x[e.s] = sla.solve_triangular(e.G, t, lower=True, trans="T") if e.m else t
    xp = np.concatenate(x)
    out = np.empty_like(xp)
    out[an.perm] = xp
    return out


@dataclasses.dataclass
class PCGReport:
    iters: int
    converged: bool
    relres: float           # recurrence ||r_k|| / ||b||
    relres_true: float      # ||b - A x|| / ||b||
    history: list


class PrecondNotPositive(Exception):
    pass


def pcg(A, b, precond, tol=1e-8, maxit=1000):
    """O5: x0 = 0; stop when ||r_k||/||b|| <= tol; the iteration count is the
    number of SpMVs.  <r, z> <= 0 raises PrecondNotPositive."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    nb = float(np.linalg.norm(b))
    hist = [1.0]
    if nb == 0.0:
        return x, PCGReport(0, True, 0.0, 0.0, hist)
    z = precond(r)
    p = z.copy()
    rho = float(r @ z)
    if rho <= 0:
        raise PrecondNotPositive(rho)
    k = 0
    conv = False
    while k < maxit:
        k += 1
        q = A @ p
        alpha = rho / float(p @ q)
        x += alpha * p
        r -= alpha * q
        rel = float(np.linalg.norm(r)) / nb
        hist.append(rel)
        if rel <= tol:
            conv = True
            break
        z = precond(r)
        rho2 = float(r @ z)
        if rho2 <= 0:
            raise PrecondNotPositive(rho2)
        p = z + (rho2 / rho) * p
        rho = rho2
    true = float(np.linalg.norm(b - A @ x)) / nb
    return x, PCGReport(k, conv, hist[-1], true, hist)
