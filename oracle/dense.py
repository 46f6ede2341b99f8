"""Dense primitives of the oracle (test infrastructure only; see oracle/__init__.py).

chol       A_ss = G_s G_s^T                      P:141 (§2 "Cholesky factorization")
tri_solve  G_s^{-1} A_sw, G_s^{-1} A_sn          P:288-296 (deferred-compression scaling)
larfg      LAPACK dlarfg Householder convention
cpqr       column-pivoted QR of the scaled block G_s^{-1} A_sw to a relative eps
           ("computed using, e.g., a rank-revealing QR factorization (RRQR)", P:166,
           P:306-318, Eq. offdiag_new), with the readings Q1-Q5 of DESIGN.md:
             * exact column norms of the trailing rows recomputed every step,
             * tau_s = eps * (largest column norm of B_w) (relative, Q1),
             * keep step j iff nu_max > tau_s (strict, Q3),
             * pivot = lowest canonical column among nu_i >= (1-1e-10) nu_max (Q4).
"""
from __future__ import annotations

import dataclasses
import numpy as np
import scipy.linalg as sla

PIVOT_WINDOW = 1e-10      # Q4 tie window
# Decision-fragility flags (reading R-margin).  Two correct implementations
# differ in a computed trailing norm nu_i(j) by about m*u*kappa(G_s)*nu_max(0): the
# triangular solve G_s^{-1}A_sw has forward error <= m*u*kappa(G_s) (Higham, Thm 8.5) and the
# Householder rounding accumulates on the scale of the initial block.  A decision is
# robust only if its distance to the decision boundary, in units of nu_max(0), exceeds
# that.  With noise = FLAG_ABS * max(1, kappa(G_s)) (passed by the caller), flag when
#   threshold:  |nu_max(j) - tau_s| < max(1e-10 * tau_s, noise * nu_max(0))
#               (the first term is north_star's "within 1e-10 relative of the threshold")
#   pivot:      |nu_i(j) - (1 - 1e-10) nu_max(j)| < noise * nu_max(0) for some i != argmax
FLAG_ABS = 1e-13
# Noise floor (reading R-floor): for eps > 0 in relative mode,
#   tau_s = max(eps * nu_max(B_w), NOISE_FLOOR * max(nu_max(B_w), nu_max(B_n))).
# A w-block that is zero in exact arithmetic (cancelling fill) holds rounding noise of
# ~1e-15 of the row's scale; a purely relative eps would "compress" that noise and take
# decisions on it.  Columns below 1e-12 of the cluster's scaled row are numerically zero.
NOISE_FLOOR = 1e-12


class NotSPD(Exception):
    """A Cholesky pivot <= 0: the approximate Schur complement is indefinite
    ('the Cholesky factorization of diagonal blocks can break down')."""

    def __init__(self, level, cluster, pivot, value):
        super().__init__(f"NOT_SPD level={level} cluster={cluster} pivot={pivot} value={value!r}")
        self.level, self.cluster, self.pivot, self.value = level, cluster, pivot, value


def chol(A: np.ndarray, level=-1, cluster=-1) -> np.ndarray:
    """Lower Cholesky factor G with A = G G^T.  Raises NotSPD with the
    0-based pivot index on breakdown; no shift or jitter is ever applied."""
    m = A.shape[0]
    if m == 0:
        return np.zeros((0, 0))
    G, info = sla.lapack.dpotrf(np.array(A, dtype=np.float64, order="F"), lower=1, clean=1)
    if info > 0:
        j = info - 1
        L = np.linalg.cholesky(A[:j, :j]) if j > 0 else np.zeros((0, 0))
        l = sla.solve_triangular(L, A[:j, j], lower=True) if j > 0 else np.zeros(0)
        raise NotSPD(level, cluster, j, float(A[j, j] - l @ l))
    if info < 0:
        raise ValueError("dpotrf argument error")
    return np.tril(G)


def tri_solve(G: np.ndarray, B: np.ndarray) -> np.ndarray:
    """G^{-1} B for lower-triangular G (the scaling S_s of Eq. CC:eqn:scaling)."""
    if B.shape[1] == 0 or G.shape[0] == 0:
        return np.array(B, dtype=np.float64, copy=True)
    return sla.solve_triangular(G, B, lower=True)


def larfg(x: np.ndarray):
    """LAPACK dlarfg: H = I - tau v v^T, v[0] = 1, H x = beta e_1.
    beta = -sign(alpha) ||x|| with sign(0) = +1; tau = 0 (H = I, beta = alpha)
    when x[1:] is exactly zero."""
    alpha = float(x[0])
    xnorm = float(np.sqrt(np.dot(x[1:], x[1:]))) if x.shape[0] > 1 else 0.0
    v = np.zeros_like(x)
    v[0] = 1.0
    if xnorm == 0.0:
        return v, 0.0, alpha
    h = float(np.sqrt(alpha * alpha + xnorm * xnorm))
    beta = -h if alpha >= 0.0 else h
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


@dataclasses.dataclass
class CPQRResult:
    r: int                    # kept rank
    V: np.ndarray             # m x r Householder vectors (unit diagonal, zeros above)
    tau: np.ndarray           # r Householder scalars
    piv: np.ndarray           # r canonical pivot columns, in pivot order
    W: np.ndarray             # m x k transformed block Q^T B_w (pivot columns zeroed below the diagonal)
    tau_s: float              # threshold eps * nu_max(0)
    nu_max: list              # nu_max(j) for every decision j
    mu: float                 # threshold margin: min_j |nu_max(j) - tau_s| / nu_max(0)
    pi: float                 # pivot margin: min_j min_{i != argmax} |nu_i - (1-1e-10) nu_max(j)| / nu_max(0)
    flagged: bool = False     # a decision lies within rounding distance of its boundary


def cpqr(B: np.ndarray, eps: float, relative: bool = True, inject=None, noise: float = FLAG_ABS,
         row_scale: float = 0.0) -> CPQRResult:
    """Businger-Golub column-pivoted Householder QR directly on B (m x k),
    truncated at the first step whose largest trailing column norm is <= tau_s.

    Columns are never physically swapped, so W keeps the canonical column order
    and W[:r, :] is V_hat_1^T (the coarse-w rows); W[r:, :] is the dropped tail
    V_hat_2^T (Eq. offdiag_new).

    inject = (r, piv) replays a given rank and pivot sequence (decision
    injection for clusters flagged by the margins; SURVEY §8(c) parity protocol)."""
    m, k = B.shape
    W = np.array(B, dtype=np.float64, copy=True)
    V = np.zeros((m, 0))
    taus, pivs, numaxes = [], [], []
    active = np.ones(k, dtype=bool)
    tau_s = None
    mu = np.inf
    pi = np.inf
    r = min(m, k)
    stopped = False
    flagged = False
    nu0 = 0.0
    for j in range(min(m, k)):
        cols = np.nonzero(active)[0]
        nu = np.sqrt(np.sum(W[j:, cols] ** 2, axis=0))      # exact, no downdating
        numax = float(nu.max())
        if j == 0:
            tau_s = eps * numax if relative else eps
            if relative and eps > 0:
                tau_s = max(tau_s, NOISE_FLOOR * max(numax, row_scale))
            nu0 = numax
        numaxes.append(numax)
        if nu0 > 0 and not (tau_s == 0.0 and numax == 0.0):   # exact zeros are not fragile
            dist = abs(numax - tau_s)
            mu = min(mu, dist / nu0)
            if dist < max(1e-10 * tau_s, noise * nu0):
                flagged = True
        if inject is not None:
            keep = j < inject[0]
        else:
            keep = numax > tau_s                           # strict (Q3)
        if not keep:
            r = j
            stopped = True
            break
        if inject is not None:
            p = int(inject[1][j])
        else:
            cand = cols[nu >= (1.0 - PIVOT_WINDOW) * numax]   # Q4 window
            p = int(cand.min())                               # lowest canonical index
        if numax > 0:
            imax = int(np.argmax(nu))
            others = np.delete(nu, imax)
            if others.size:
                d = float(np.min(np.abs(others - (1.0 - PIVOT_WINDOW) * numax))) / nu0
                pi = min(pi, d)
                if d < noise:
                    flagged = True
        v, tau, beta = larfg(W[j:, p])
        act = cols[cols != p]
        if tau != 0.0:
            d = v @ W[j:, act]
            W[j:, act] -= tau * np.outer(v, d)
        W[j, p] = beta
        W[j + 1:, p] = 0.0
        active[p] = False
        vfull = np.zeros((m, 1))
        vfull[j:, 0] = v
        V = np.hstack([V, vfull])
        taus.append(tau)
        pivs.append(p)
    if tau_s is None:
        tau_s = 0.0
    if not stopped and inject is not None:
        r = min(r, inject[0])
    return CPQRResult(r=r, V=V, tau=np.array(taus), piv=np.array(pivs, dtype=np.int64), W=W,
                      tau_s=float(tau_s), nu_max=numaxes, mu=float(mu), pi=float(pi), flagged=flagged)


def apply_Qt(V: np.ndarray, tau: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Q^T X with Q = H_0 H_1 ... H_{r-1}: applies H_0 first (E_s of Eq. CC:eqn:sparse)."""
    Y = np.array(X, dtype=np.float64, copy=True)
    vec = Y.ndim == 1
    if vec:
        Y = Y[:, None]
    for j in range(V.shape[1]):
        v = V[j:, j]
        if tau[j] != 0.0:
            Y[j:] -= tau[j] * np.outer(v, v @ Y[j:])
    return Y[:, 0] if vec else Y


def apply_Q(V: np.ndarray, tau: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Q X: applies H_{r-1} first (E_s^T in the backward substitution)."""
    Y = np.array(X, dtype=np.float64, copy=True)
    vec = Y.ndim == 1
    if vec:
        Y = Y[:, None]
    for j in reversed(range(V.shape[1])):
        v = V[j:, j]
        if tau[j] != 0.0:
            Y[j:] -= tau[j] * np.outer(v, v @ Y[j:])
    return Y[:, 0] if vec else Y
