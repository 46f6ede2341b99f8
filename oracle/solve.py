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
                if e.dc:
                    t = sla.solve_triangular(e.G, y[e.s], lower=True) if e.m else y[e.s].copy()
                    t = apply_Qt(e.V, e.tau, t)
                    yf = t[e.r:]
                else:   # original LoRaSp step: [y_c; y_f] = U^T y_s, y_f <- L_f^{-1} y_f, y_c -= C_c^T y_f
                    t = apply_Qt(e.V, e.tau, y[e.s])
                    yf = sla.solve_triangular(e.G, t[e.r:], lower=True) if e.m > e.r else t[e.r:]
                    t = np.concatenate([t[:e.r] - e.Cc.T @ yf, yf])
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
                if e.dc:
                    t = np.concatenate([x[e.s], xf])
                    t = apply_Q(e.V, e.tau, t)
                    x[e.s] = sla.solve_triangular(e.G, t, lower=True, trans="T") if e.m else t
                else:
                    xf = xf - e.Cc @ x[e.s]
                    xf = sla.solve_triangular(e.G, xf, lower=True, trans="T") if e.m > e.r else xf
                    x[e.s] = apply_Q(e.V, e.tau, np.concatenate([x[e.s], xf]))
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


@dataclasses.dataclass
class GMRESReport:
    iters: int              # Arnoldi steps (one A M^{-1} product each)
    converged: bool
    relres: float           # recurrence |g_{j+1}| / ||b||
    relres_true: float      # ||b - A x|| / ||b||
    restarts: int


def gmres(A, b, precond, tol=1e-12, restart=200, maxit=1000):
    """Right-preconditioned restarted GMRES — the paper's Krylov protocol: GMRES(200),
    tolerance 1e-12, at most 1000 iterations (NEXT f3).  Textbook form (Saad,
    "Iterative Methods for Sparse Linear Systems", Alg. 9.5 with the modified Gram-Schmidt
    Arnoldi of Alg. 6.2 and Givens rotations, Sec. 6.5.3): x0 = 0; solve A M^{-1} u = b,
    x = M^{-1} u; stop when |g_{j+1}| / ||b|| <= tol or after maxit Arnoldi steps."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    x = np.zeros(n)
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return x, GMRESReport(0, True, 0.0, 0.0, 0)
    its, restarts, rel = 0, 0, 1.0
    while True:
        r = b - A @ x
        beta = float(np.linalg.norm(r))
        rel = beta / nb
        if rel <= tol or its >= maxit:
            break
        V = [r / beta]
        H = np.zeros((restart + 1, restart))
        g = np.zeros(restart + 1)
        g[0] = beta
        cs, sn = np.zeros(restart), np.zeros(restart)
        k = 0
        for j in range(restart):
            its += 1
            w = A @ precond(V[j])
            for i in range(j + 1):                  # modified Gram-Schmidt
                H[i, j] = w @ V[i]
                w = w - H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            for i in range(j):                      # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            rel = abs(g[j + 1]) / nb
            if rel <= tol or its >= maxit or hn == 0.0:
                break
            V.append(w / hn)
        y = sla.solve_triangular(H[:k, :k], g[:k], lower=False)
        x = x + precond(np.column_stack(V[:k]) @ y)
        restarts += 1
        if rel <= tol or its >= maxit:
            break
    rt = float(np.linalg.norm(b - A @ x)) / nb
    return x, GMRESReport(its, rel <= tol, rel, rt, restarts)
