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
