"""Distributed O3 — Algorithm 1 partitioned by subdomains over P ranks (oracle; test
infrastructure only).

The paper's parallel section is an empty stub that defers to parallel
LoRaSp: "data dependency is exactly the same as in the original LoRaSp method, the same
parallel algorithm works here (with minor changes on what data is communicated)"
(Thm 2).  This module follows the reconstruction of SURVEY §8(e):

  * the 8 fixed subdomains of analyze (O2.5) are owned by ranks: subdomain k -> rank
    k * P // 8; a cluster of level l < L_top lies in one subdomain, parents inherit the
    owner (O2.5, O2.6);
  * rank g holds every block (p, q) of the level with p or q owned by g ("ghost" copies
    of cross-owner blocks are identical on both owners);
  * phase-I batches (interior clusters) touch only their own subdomain (O2.8 "why phase I
    stays local"): each rank eliminates its own interior clusters, no communication;
  * a phase-II batch: the owner of s eliminates s from its own blocks (row s is held by
    the owner), then sends (r, C_s, coarse rows) to every rank holding a block the
    elimination writes: the Schur updates A_pq -= C_p^T C_q on blocks (p, q),
    p, q in n(s), and the write-back of row s; every receiver applies them to
    the blocks it holds, in source order (the sequential loop's order);
  * after phase I and at the level end the kept ranks are all-gathered (a phase-II fill
    block can join a remote cluster eliminated in phase I); parents are assembled from child blocks
    (P:636), each rank for the parent blocks it holds;
  * top: the blocks of the top level are gathered to rank 0, which factors A_top
    (P:626-628).

The exchange goes through `comm`, an object with all_gather(obj) -> list (rank order):
torch.distributed (gloo) in tests/test_dist_oracle.py.  The arithmetic per cluster is
oracle.factor.eliminate's; this module only decides who computes what and what is sent.
"""
from __future__ import annotations

import numpy as np

from .analyze import Analysis
from .factor import BlockStore, Factor, _cols, eliminate, initial_blocks
from .dense import chol


def owner(an: Analysis, level: int, c: int, world: int) -> int:
    """Rank owning cluster c of level l (subdomain k -> rank k * P / 2^nsub)."""
    nsub = 1 << min(an.nsub_log2, an.D)
    return an.subdomain(level, c) * world // nsub


class _Local(BlockStore):
    """Rank-local block store: keeps only blocks with an owned endpoint."""

    def __init__(self, live, own):
        super().__init__(live)
        self.own = own            # bool per cluster

    def holds(self, p, q):
        return bool(self.own[p] or self.own[q])

    def set(self, p, q, M):
        if self.holds(p, q):
            super().set(p, q, M)


def _restrict(st: BlockStore, own) -> _Local:
    loc = _Local(st.live, own)
    for (p, q), M in st.blocks.items():
        if loc.holds(p, q):
            loc.blocks[(p, q)] = M
    return loc


def _apply_message(st: _Local, msg):
    """Steps 6-7 of eliminate() for the blocks this rank holds (Eq. CC:eqn:elim P:569-588,
    Eq. CC:eqn:perm P:591-611), from the owner's record of s."""
    s, r, C, nlist, nsz, wlist, wsz, coarse_n, coarse_w = msg
    no, wo = _cols(nsz), _cols(wsz)
    for a, p in enumerate(nlist):
        Cp = C[:, no[a]:no[a + 1]]
        for b in range(a + 1):
            q = nlist[b]
            if not st.holds(p, q):
                continue
            Cq = C[:, no[b]:no[b + 1]]
            st.set(p, q, st.get(p, q) - Cp.T @ Cq)
    st.live[s] = r
    if st.own[s]:
        st.set(s, s, np.eye(r))
    for a, q in enumerate(nlist):
        st.set(s, q, coarse_n[:, no[a]:no[a + 1]])
    for a, q in enumerate(wlist):
        st.set(s, q, coarse_w[:, wo[a]:wo[a + 1]])


def _sync_live(st, own, nclus, comm):
    """All-gather the live sizes of the owned clusters (each cluster has one owner)."""
    live = np.zeros(nclus, dtype=np.int64)
    for c in range(nclus):
        if own[c]:
            live[c] = st.live[c]
    live = np.sum(comm.all_gather(live), axis=0)
    st.live = [int(x) for x in live]


def factor_dist(an: Analysis, rowptr, colind, vals, comm, rank: int, world: int, eps=1e-2, relative=True):
    """Rank `rank`'s part of the distributed factor.  Returns (elims, top) where elims is
    {level: {cluster: Elim}} of the clusters this rank eliminated and top = (top_sizes, L)
    on rank 0 (None elsewhere)."""
    full = initial_blocks(an, rowptr, colind, vals)
    nclus0 = len(full.live)
    own = np.array([owner(an, 0, c, world) == rank for c in range(nclus0)], dtype=bool)
    st = _restrict(full, own)
    del full
    mine = {}
    for l, lev in enumerate(an.levels):
        own = np.array([owner(an, l, c, world) == rank for c in range(lev.nclus)], dtype=bool)
        st.own = own
        mine[l] = {}
        for bi, B in enumerate(lev.batches):
            if bi == lev.nphase1:
                # phase II starts: fill blocks may now join a remote cluster q that was
                # eliminated in phase I, so every holder needs q's kept rank
                _sync_live(st, own, lev.nclus, comm)
            if bi < lev.nphase1:
                # phase I: interior clusters, everything they touch is local
                for s in B:
                    if own[s]:
                        mine[l][s] = eliminate(st, l, s, lev.nlist[s], lev.wlist[s], eps, relative)
                continue
            # phase II: the owner eliminates on a scratch copy of row s (its writes to
            # blocks it does not hold must not land anywhere), the record travels
            out = []
            for s in B:
                if not own[s]:
                    continue
                tmp = BlockStore(st.live)
                for q in [s] + list(lev.nlist[s]) + list(lev.wlist[s]):
                    tmp.set(s, q, st.get(s, q))
                e = eliminate(tmp, l, s, lev.nlist[s], lev.wlist[s], eps, relative, keep_debug=True)
                mine[l][s] = e
                out.append((s, e.r, e.C, e.nlist, e.nsz, e.wlist, e.wsz, e.coarse_n, e.coarse_w))
            msgs = [m for part in comm.all_gather(out) for m in part]
            for msg in sorted(msgs, key=lambda m: m[0]):     # source order (sequential loop)
                _apply_message(st, msg)
        # end of level: every rank needs every kept rank (ghost parents' sizes)
        _sync_live(st, own, lev.nclus, comm)
        nP = lev.nclus // 2
        Hn = an.levels[l + 1].Fstart if l + 1 < len(an.levels) else an.H_top   # block pattern of A_c
        lv_next = [st.live[2 * P] + st.live[2 * P + 1] for P in range(nP)]
        if l + 1 < len(an.levels):
            own_n = np.array([owner(an, l + 1, c, world) == rank for c in range(nP)], dtype=bool)
        else:
            own_n = np.array([owner(an, l + 1, c, world) == rank for c in range(nP)], dtype=bool)
        nst = _Local(lv_next, own_n)
        for P in range(nP):
            for Q in [x for x in Hn[P] if x < P] + [P]:
                if not nst.holds(P, Q):
                    continue
                M = np.zeros((lv_next[P], lv_next[Q]))
                ro = [0, st.live[2 * P]]
                co = [0, st.live[2 * Q]]
                for a in (0, 1):
                    for b in (0, 1):
                        blk = st.get(2 * P + a, 2 * Q + b)
                        M[ro[a]:ro[a] + blk.shape[0], co[b]:co[b] + blk.shape[1]] = blk
                nst.blocks[(P, Q)] = M
        st = nst
    # top: gather the blocks whose row cluster is owned here to rank 0
    ntop = 1 << (an.D - an.L_top)
    part = {(p, q): M for (p, q), M in st.blocks.items() if st.own[p]}
    parts = comm.all_gather(part)
    if rank != 0:
        return mine, None
    blocks = {}
    for pt in parts:
        blocks.update(pt)
    o = _cols([st.live[c] for c in range(ntop)])
    A = np.zeros((o[-1], o[-1]))
    for p in range(ntop):
        for q in range(p + 1):
            blk = blocks.get((p, q))
            if blk is None:
                continue
            A[o[p]:o[p + 1], o[q]:o[q + 1]] = blk
            A[o[q]:o[q + 1], o[p]:o[p + 1]] = blk.T
    L = chol(A, an.L_top, -1)
    return mine, (np.array(st.live[:ntop]), L)


def assemble_factor(an: Analysis, parts, top, eps=1e-2, relative=True) -> Factor:
    """Rank 0: the sequential Factor record from every rank's eliminations (batch order)."""
    elims, live0, live1 = [], [], []
    for l, lev in enumerate(an.levels):
        allm = {}
        for mine in parts:
            allm.update(mine[l])
        elims.append([[allm[s] for s in B] for B in lev.batches])
        live0.append([allm[s].m for s in range(lev.nclus)])
        live1.append([allm[s].r for s in range(lev.nclus)])
    top_sizes, L = top
    return Factor(an, eps, relative, elims, live0, live1, top_sizes, L)


# ---- distributed Algorithm 2 and PCG (SURVEY §8(e) "Apply", "PCG") ---------------------------
# Owner computes: every rank applies the elimination records of the clusters it eliminated
# (no gather of the factor); the vector lives in per-cluster segments at their owners.
#   forward, per batch: owners form y_s <- U^T G^{-1} y_s and the contributions C_s[:, q]^T y_f;
#     interior (phase-I) contributions stay local (O2.8); after each phase-II batch the
#     contributions are exchanged and every owner subtracts the ones for its clusters in
#     source order (no batch member is another's target, so this IS the sequential order);
#   top: rank 0 gathers the top segments, solves with L L^T and scatters the result;
#   backward, per batch in reverse: owners of a phase-II batch first receive the current x
#     segments of their remote neighbours, then x_f = y_f - sum_q C[:, q] x_q and
#     x_s = G^{-T} U [x_c; x_f] (Alg. 2).
# PCG: the iterate, residual and search direction are distributed the same way (the DOFs
# of owned leaves); the SpMV of an owned row needs the x entries of its ghost columns (halo
# exchange), each dot product is a sum of per-rank partial sums (all-reduce).

def owned_leaves(an: Analysis, rank: int, world: int):
    nleaf = an.leaf_off.shape[0] - 1
    lvl = 0 if an.levels else an.L_top
    return [c for c in range(nleaf) if owner(an, lvl, c, world) == rank]


def _own_rows(an, rank, world):
    return np.concatenate([np.arange(an.leaf_off[c], an.leaf_off[c + 1]) for c in owned_leaves(an, rank, world)]
                          or [np.zeros(0, dtype=np.int64)]).astype(np.int64)


def apply_dist(an: Analysis, mine, top, y0, comm, rank: int, world: int):
    """x = M^{-1} b for the distributed factor.  y0: {leaf: b segment (permuted order)} for
    the leaves this rank owns; returns {leaf: x segment} for the same leaves."""
    import scipy.linalg as sla
    from .dense import apply_Qt, apply_Q
    y = {c: np.array(v, dtype=np.float64) for c, v in y0.items()}
    fine = {}
    for l, lev in enumerate(an.levels):
        for bi, B in enumerate(lev.batches):
            out = []
            for s in B:
                e = mine[l].get(s)
                if e is None:
                    continue
                t = sla.solve_triangular(e.G, y[s], lower=True) if e.m else y[s].copy()
                t = apply_Qt(e.V, e.tau, t)
                yf = t[e.r:]
                fine[(l, s)] = yf
                y[s] = t[:e.r]
                o = 0
                for q, k in zip(e.nlist, e.nsz):
                    out.append((s, q, e.C[:, o:o + k].T @ yf))
                    o += k
            if bi >= lev.nphase1:   # phase II: contributions travel to their targets' owners
                out = [m for part in comm.all_gather(out) for m in part]
            for s, q, v in sorted(out, key=lambda m: m[0]):
                if owner(an, l, q, world) == rank:
                    y[q] = y[q] - v
        nP = lev.nclus // 2
        y = {P: np.concatenate([y[2 * P], y[2 * P + 1]]) for P in range(nP) if owner(an, l + 1, P, world) == rank}
    # top (rank 0)
    parts = comm.all_gather(y)
    ntop = 1 << (an.D - an.L_top)
    xtop = None
    if rank == 0:
        segs = {}
        for pt in parts:
            segs.update(pt)
        yt = np.concatenate([segs[c] for c in range(ntop)]) if ntop else np.zeros(0)
        top_sizes, L = top
        if yt.shape[0]:
            z = sla.solve_triangular(L, yt, lower=True)
            xt = sla.solve_triangular(L, z, lower=True, trans="T")
        else:
            xt = yt
        o = np.concatenate([[0], np.cumsum([segs[c].shape[0] for c in range(ntop)])]).astype(int)
        xtop = {c: xt[o[c]:o[c + 1]] for c in range(ntop)}
    xtop = comm.all_gather(xtop)[0]
    x = {c: v for c, v in xtop.items() if owner(an, an.L_top, c, world) == rank}
    for l in reversed(range(len(an.levels))):
        lev = an.levels[l]
        xs = {}
        for P, v in x.items():   # children of an owned parent are owned (same subdomain)
            r0 = mine[l][2 * P].r if 2 * P in mine[l] else 0
            xs[2 * P] = v[:r0]
            xs[2 * P + 1] = v[r0:]
        x = xs
        for bi in reversed(range(len(lev.batches))):
            B = lev.batches[bi]
            view = x
            if bi >= lev.nphase1:   # the remote neighbours' current segments (halo of the sweep)
                view = {}
                for pt in comm.all_gather(x):
                    view.update(pt)
            for s in reversed(B):
                e = mine[l].get(s)
                if e is None:
                    continue
                xf = fine[(l, s)].copy()
                o = 0
                for q, k in zip(e.nlist, e.nsz):
                    assert view[q].shape[0] == k
                    xf = xf - e.C[:, o:o + k] @ view[q]
                    o += k
                t = apply_Q(e.V, e.tau, np.concatenate([x[s], xf]))
                x[s] = sla.solve_triangular(e.G, t, lower=True, trans="T") if e.m else t
    return x


def pcg_dist(an: Analysis, mine, top, rowptr, colind, vals, b, comm, rank: int, world: int, tol=1e-8, maxit=1000):
    """O5 PCG on the distributed factor.  b: the full right-hand side (original order; each
    rank reads its own rows).  Returns (x full vector assembled on every rank, iterations,
    relative residual history)."""
    import scipy.sparse as sp
    n = an.n
    A = sp.csr_matrix((vals, colind, rowptr), shape=(n, n))
    Ap = A[an.perm][:, an.perm].tocsr()                  # permuted: owned leaves are row ranges
    rows = _own_rows(an, rank, world)
    A_loc = Ap[rows]
    ghost = np.setdiff1d(np.unique(A_loc.indices), rows)  # halo: columns owned elsewhere
    leaves = owned_leaves(an, rank, world)

    def spmv(v_loc):   # halo exchange: every rank publishes its owned entries, keeps only its ghosts
        pub = np.zeros(n)
        for rr, vv in comm.all_gather((rows, v_loc)):
            pub[rr] = vv
        full = np.zeros(n)          # owned + ghost entries only: the halo suffices for the owned rows
        full[rows] = v_loc
        full[ghost] = pub[ghost]
        return A_loc @ full

    def dot(u, v):     # all-reduce of per-rank partial sums, summed in rank order
        return float(sum(comm.all_gather(float(u @ v))))

    def prec(r_loc):
        segs, o = {}, 0
        for c in leaves:
            k = an.leaf_off[c + 1] - an.leaf_off[c]
            segs[c] = r_loc[o:o + k]
            o += k
        xs = apply_dist(an, mine, top, segs, comm, rank, world)
        return np.concatenate([xs[c] for c in leaves]) if leaves else np.zeros(0)

    bp = np.asarray(b, dtype=np.float64)[an.perm][rows]
    x = np.zeros_like(bp)
    r = bp.copy()
    nb = np.sqrt(dot(bp, bp))
    hist = [1.0]
    z = prec(r)
    p = z.copy()
    rho = dot(r, z)
    k = 0
    while k < maxit:
        k += 1
        q = spmv(p)
        alpha = rho / dot(p, q)
        x += alpha * p
        r -= alpha * q
        rel = np.sqrt(dot(r, r)) / nb
        hist.append(rel)
        if rel <= tol:
            break
        z = prec(r)
        rho2 = dot(r, z)
        p = z + (rho2 / rho) * p
        rho = rho2
    full = np.zeros(n)
    for rr, vv in comm.all_gather((rows, x)):
        full[rr] = vv
    out = np.empty(n)
    out[an.perm] = full
    return out, k, hist
