"""O3 Factor — Algorithm 1 `Hierarchical_Factor` with the
"scaled low-rank elimination" of §3.1 (oracle; test infrastructure only).

For every level l = 0 .. L_top-1, batches in order, s ascending in a batch
(reading Q8), the elimination of cluster s is, in the paper's order:

  1. extract A_ss, A_sn, A_sw from A_i                    (Alg. 1 "Extract A-bar")
  2. A_ss = G_s G_s^T                                     (Eq. CC:eqn:scaling)
  3. B_n = G_s^{-1} A_sn, B_w = G_s^{-1} A_sw            (deferred-compression scaling)
  4. G_s^{-1} A_sw = U1 V1^T + U2 V2^T by column-pivoted QR to eps
                                                          (Eq. offdiag_new; readings Q1-Q5)
  5. E_s = diag(U^T, I, I): coarse-n = U1^T B_n, C = U2^T B_n, coarse-w = V1^T
                                                          (Eq. CC:eqn:sparse)
  6. eliminate the fine DOFs: X_nn = A_nn - C^T C        (Eq. CC:eqn:elim)
  7. P_s moves the coarse DOFs on; row s becomes [I_r | coarse-n | coarse-w]
                                                          (Eq. CC:eqn:perm)
then A_c is extracted — parent = [coarse(child0); coarse(child1)]
(reading Q9) — and the recursion ends with a dense Cholesky at the first level
with <= top_clusters clusters (reading Q10).

State: dense blocks keyed (max id, min id), symmetric by construction
(reading Q20); the diagonal block of a processed cluster is stored explicitly
(I_r at write-back, then further Schur updates accumulate on it).
"""
from __future__ import annotations

import dataclasses
import numpy as np
import scipy.sparse as sp

from .analyze import Analysis
from .dense import chol, tri_solve, cpqr, apply_Qt, NotSPD, FLAG_ABS  # noqa: F401


@dataclasses.dataclass
class Elim:
    level: int
    s: int
    m: int
    r: int
    G: np.ndarray          # m x m lower
    V: np.ndarray          # m x r Householder vectors
    tau: np.ndarray        # r
    piv: np.ndarray        # r canonical pivots
    C: np.ndarray          # (m - r) x k_n  multiplier U2^T G^{-1} A_sn
    nlist: list
    nsz: list              # live sizes of n(s) at elimination time
    wlist: list
    wsz: list
    mu: float
    pi: float
    tau_s: float
    coarse_n: np.ndarray = None   # r x k_n (debug / parity)
    coarse_w: np.ndarray = None   # r x k_w
    tail_w: np.ndarray = None     # (m - r) x k_w dropped V2^T (debug, P3)
    flagged: bool = False         # a CPQR decision within rounding distance of its boundary
    dc: bool = True               # False: original LoRaSp step (eliminate_nodc); G = L_f
    Cc: np.ndarray = None         # dc = False: (m - r) x r, L_f^{-1} U2^T A_ss U1


@dataclasses.dataclass
class Factor:
    an: Analysis
    eps: float
    relative: bool
    elims: list            # elims[l][b] = list of Elim in batch order
    live0: list            # live sizes per level at the start of the level
    live1: list            # live sizes per level at the end of the level
    top_sizes: np.ndarray  # live sizes at L_top
    L: np.ndarray          # Cholesky factor of A_top
    snapshots: list = None  # optional block-store snapshots (debug)


class BlockStore:
    """Dense blocks A(p, q) keyed (max, min); get() transposes on read."""

    def __init__(self, live):
        self.live = list(live)
        self.blocks = {}

    def get(self, p, q):
        if p >= q:
            M = self.blocks.get((p, q))
            if M is None:
                return np.zeros((self.live[p], self.live[q]))
            return M
        M = self.blocks.get((q, p))
        if M is None:
            return np.zeros((self.live[p], self.live[q]))
        return M.T

    def set(self, p, q, M):
        if p >= q:
            self.blocks[(p, q)] = np.array(M, dtype=np.float64)
        else:
            self.blocks[(q, p)] = np.array(M.T, dtype=np.float64)


def initial_blocks(an: Analysis, rowptr, colind, vals) -> BlockStore:
    """Level-0 blocks of the permuted A (clusters and their neighbours)."""
    n = an.n
    A = sp.csr_matrix((vals, colind, rowptr), shape=(n, n))
    Ap = A[an.perm][:, an.perm].tocsr()
    off = an.leaf_off
    nleaf = off.shape[0] - 1
    st = BlockStore(np.diff(off).tolist())
    H0 = an.levels[0].H if an.levels else an.H_top
    for p in range(nleaf):
        r0, r1 = off[p], off[p + 1]
        slab = Ap[r0:r1].tocoo()
        cl = np.searchsorted(off, slab.col, side="right") - 1
        for q in [x for x in H0[p] if x < p] + [p]:
            sel = cl == q
            M = np.zeros((r1 - r0, off[q + 1] - off[q]))
            np.add.at(M, (slab.row[sel], slab.col[sel] - off[q]), slab.data[sel])
            st.blocks[(p, q)] = M
    return st


def _cols(sizes):
    o = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=o[1:])
    return o


def eliminate(st: BlockStore, l: int, s: int, nlist, wlist, eps, relative, inject=None,
              keep_debug=False) -> Elim:
    """One scaled low-rank elimination of cluster s."""
    m = st.live[s]
    nsz = [st.live[q] for q in nlist]
    wsz = [st.live[q] for q in wlist]
    no, wo = _cols(nsz), _cols(wsz)
    A_ss = st.get(s, s)
    A_sn = np.hstack([st.get(s, q) for q in nlist]) if nlist else np.zeros((m, 0))
    A_sw = np.hstack([st.get(s, q) for q in wlist]) if wlist else np.zeros((m, 0))
    G = chol(A_ss, l, s)                                   # step 2
    Bn = tri_solve(G, A_sn)                                # step 3 (deferred compression)
    Bw = tri_solve(G, A_sw)
    if Bw.shape[1] == 0 or m == 0:                         # w = {} : plain block Cholesky
        r, V, tau, piv, W = 0, np.zeros((m, 0)), np.zeros(0), np.zeros(0, dtype=np.int64), Bw
        mu = pi = np.inf
        tau_s = 0.0
        flagged = False
    else:
        kappa = float(np.linalg.cond(G)) if m > 0 else 1.0
        row_scale = float(np.sqrt(np.sum(Bn ** 2, axis=0)).max()) if Bn.shape[1] else 0.0
        res = cpqr(Bw, eps, relative, inject, noise=FLAG_ABS * max(1.0, kappa), row_scale=row_scale)   # step 4
        r, V, tau, piv, W = res.r, res.V[:, :res.r], res.tau[:res.r], res.piv[:res.r], res.W
        mu, pi, tau_s, flagged = res.mu, res.pi, res.tau_s, res.flagged
    Bt = apply_Qt(V, tau, Bn)                              # step 5: U^T G^{-1} A_sn
    coarse_n, C = Bt[:r], Bt[r:]
    coarse_w = W[:r]
    for a, p in enumerate(nlist):                          # step 6: X_nn = A_nn - C^T C
        Cp = C[:, no[a]:no[a + 1]]
        for b in range(a + 1):
            q = nlist[b]
            Cq = C[:, no[b]:no[b + 1]]
            st.set(p, q, st.get(p, q) - Cp.T @ Cq)
    st.live[s] = r                                         # step 7: write back row s
    st.set(s, s, np.eye(r))
    for a, q in enumerate(nlist):
        st.set(s, q, coarse_n[:, no[a]:no[a + 1]])
    for a, q in enumerate(wlist):
        st.set(s, q, coarse_w[:, wo[a]:wo[a + 1]])
    e = Elim(l, s, m, r, G, V, tau, piv, C, list(nlist), nsz, list(wlist), wsz, mu, pi, tau_s, flagged=flagged)
    if keep_debug:
        e.coarse_n, e.coarse_w, e.tail_w = coarse_n, coarse_w, W[r:]
    return e


def eliminate_nodc(st: BlockStore, l: int, s: int, nlist, wlist, eps, relative, inject=None,
                   keep_debug=False) -> Elim:
    """NEXT f1: one step of the ORIGINAL LoRaSp sparsified elimination, WITHOUT deferred
    compression (Eq. offdiag):
      1. compress the UNSCALED block A_sw = U V^T = U1 V1^T + U2 V2^T with the same CPQR as
         the DC path (readings Q1-Q5: tau_s relative to A_sw's largest column norm, R-floor
         with the largest column norm of A_sn);
      2. rotate row s by U^T and drop U2^T A_sw = V2^T: the fine DOFs f (the U2 part) no
         longer couple to w;
      3. eliminate f: A_ff = U2^T A_ss U2 = L_f L_f^T (not I: Table 1),
         C_c = L_f^{-1} U2^T A_ss U1, C_n = L_f^{-1} U2^T A_sn;
      4. Schur updates A_pq -= C_p^T C_q on n x n and on the coarse block of s:
         diag(s) = U1^T A_ss U1 - C_c^T C_c, coarse-n = U1^T A_sn - C_c^T C_n,
         coarse-w = V1^T (the kept CPQR rows).
    Eliminating f and then the coarse DOFs equals one Cholesky step on s in the compressed
    matrix A~ (Eq. sc_old), whose error against the exact Schur complement is Eq. err_old."""
    m = st.live[s]
    nsz = [st.live[q] for q in nlist]
    wsz = [st.live[q] for q in wlist]
    no, wo = _cols(nsz), _cols(wsz)
    A_ss = st.get(s, s)
    A_ss = np.tril(A_ss) + np.tril(A_ss, -1).T            # the store keeps the lower triangle
    A_sn = np.hstack([st.get(s, q) for q in nlist]) if nlist else np.zeros((m, 0))
    A_sw = np.hstack([st.get(s, q) for q in wlist]) if wlist else np.zeros((m, 0))
    if A_sw.shape[1] == 0 or m == 0:
        r, V, tau, piv, W = 0, np.zeros((m, 0)), np.zeros(0), np.zeros(0, dtype=np.int64), A_sw
        mu = pi = np.inf
        tau_s = 0.0
        flagged = False
    else:
        kappa = float(np.linalg.cond(A_ss)) if m > 0 else 1.0
        row_scale = float(np.sqrt(np.sum(A_sn ** 2, axis=0)).max()) if A_sn.shape[1] else 0.0
        res = cpqr(A_sw, eps, relative, inject, noise=FLAG_ABS * max(1.0, kappa), row_scale=row_scale)   # step 1
        r, V, tau, piv, W = res.r, res.V[:, :res.r], res.tau[:res.r], res.piv[:res.r], res.W
        mu, pi, tau_s, flagged = res.mu, res.pi, res.tau_s, res.flagged
    Ah = apply_Qt(V, tau, apply_Qt(V, tau, A_ss).T).T      # step 2: U^T A_ss U
    Bn = apply_Qt(V, tau, A_sn)                            #          U^T A_sn
    Lf = chol(Ah[r:, r:], l, s)                            # step 3
    Cc = tri_solve(Lf, Ah[r:, :r])
    C = tri_solve(Lf, Bn[r:])
    for a, p in enumerate(nlist):                          # step 4: n x n
        Cp = C[:, no[a]:no[a + 1]]
        for b in range(a + 1):
            q = nlist[b]
            Cq = C[:, no[b]:no[b + 1]]
            st.set(p, q, st.get(p, q) - Cp.T @ Cq)
    st.live[s] = r                                         # coarse block of s
    st.set(s, s, Ah[:r, :r] - Cc.T @ Cc)
    coarse_n = Bn[:r] - Cc.T @ C
    for a, q in enumerate(nlist):
        st.set(s, q, coarse_n[:, no[a]:no[a + 1]])
    coarse_w = W[:r]
    for a, q in enumerate(wlist):
        st.set(s, q, coarse_w[:, wo[a]:wo[a + 1]])
    e = Elim(l, s, m, r, Lf, V, tau, piv, C, list(nlist), nsz, list(wlist), wsz, mu, pi, tau_s, flagged=flagged,
             dc=False, Cc=Cc)
    if keep_debug:
        e.coarse_n, e.coarse_w, e.tail_w = coarse_n, coarse_w, W[r:]
    return e


def next_level(st: BlockStore, pattern_next, nclus_next) -> BlockStore:
    """Extract A_c: parent P = [coarse(2P); coarse(2P+1)], blocks are the
    2x2 assemblies of the child blocks (missing child blocks are zero)."""
    live = [st.live[2 * P] + st.live[2 * P + 1] for P in range(nclus_next)]
    nst = BlockStore(live)
    for P in range(nclus_next):
        for Q in [x for x in pattern_next[P] if x < P] + [P]:
            M = np.zeros((live[P], live[Q]))
            ro = [0, st.live[2 * P]]
            co = [0, st.live[2 * Q]]
            for a in (0, 1):
                for b in (0, 1):
                    blk = st.get(2 * P + a, 2 * Q + b)
                    M[ro[a]:ro[a] + blk.shape[0], co[b]:co[b] + blk.shape[1]] = blk
            nst.blocks[(P, Q)] = M
    return nst


def assemble_top(st: BlockStore, nclus):
    o = _cols([st.live[c] for c in range(nclus)])
    A = np.zeros((o[-1], o[-1]))
    for p in range(nclus):
        for q in range(p + 1):
            blk = st.get(p, q)
            A[o[p]:o[p + 1], o[q]:o[q + 1]] = blk
            A[o[q]:o[q + 1], o[p]:o[p + 1]] = blk.T
    return A, o


def factor(an: Analysis, rowptr, colind, vals, eps=1e-2, relative=True, inject=None,
           keep_debug=False, snapshot=None, max_levels=None, dc=True) -> Factor:
    """Algorithm 1.  inject: {(l, s): (r, piv)} decision injection.
    snapshot(l, b, store) is called after every batch when given (debug).
    max_levels: stop after that many levels (partial record for sampled parity at full
    size: elims only, no top factor)."""
    st = initial_blocks(an, rowptr, colind, vals)
    elims, live0, live1 = [], [], []
    for l, lev in enumerate(an.levels):
        live0.append(list(st.live))
        lv = []
        for bi, B in enumerate(lev.batches):
            eb = []
            for s in B:
                inj = None if inject is None else inject.get((l, s))
                elim = eliminate if dc else eliminate_nodc
                eb.append(elim(st, l, s, lev.nlist[s], lev.wlist[s], eps, relative, inj, keep_debug))
            lv.append(eb)
            if snapshot is not None:
                snapshot(l, bi, st)
        elims.append(lv)
        live1.append(list(st.live))
        if max_levels is not None and l + 1 >= max_levels:
            return Factor(an, eps, relative, elims, live0, live1, None, None)
        Hn = an.levels[l + 1].Fstart if l + 1 < len(an.levels) else an.H_top   # block pattern of A_c
        st = next_level(st, Hn, lev.nclus // 2)
    ntop = 1 << (an.D - an.L_top)
    A_top, _ = assemble_top(st, ntop)
    L = chol(A_top, an.L_top, -1)
    return Factor(an, eps, relative, elims, live0, live1, np.array(st.live[:ntop]), L)


def ranks(fac: Factor):
    """Per-level arrays of kept ranks r_s (indexed by cluster id)."""
    out = []
    for l, lv in enumerate(fac.elims):
        r = np.zeros(fac.an.levels[l].nclus, dtype=np.int64)
        for eb in lv:
            for e in eb:
                r[e.s] = e.r
        out.append(r)
    return out
