"""O2 Analyze — partition, cluster tree and symbolic per-level schedule (oracle; test infrastructure only).

Integer-only; the library's `hs_analyze` must reproduce every output bit-exactly.

Paper passages:
  * clustering = a partition of the graph G_A, computed "algebraically ... with
    existing software packages" (§3 "Matrix Partitioning"); Zoltan
    geometric partition with clusters of about 100.  Reading Q11: RCB.
  * extruded partitioning: partition one layer, extrude so that every vertical
    line lies in one cluster (§4.2).  Reading Q19: a column's
    coordinate is the (x, y) of its lowest-index DOF.
  * neighbours: "pi_p and pi_q are neighbors if the matrix block A(pi_p,pi_q) != 0"
    (P:494), re-applied to A_c at every level (Alg. 1).  Reading
    Q6: n(s) is the structural block pattern of the level's input, fixed for
    the level; Q7: w(s) = current fill adjacency minus n(s).
  * Alg. 1 loops "for i <- 0 to m-1" over the clusters; reading Q8:
    greedy independent-set batches, interior clusters of 8 fixed subdomains
    first, then boundary clusters, ascending id.  Q9: binary cluster tree fixed
    here, parent = union of the children's coarse DOFs.  Q10: the top
    ("if the size of A is small enough") is the first level with
    <= top_clusters clusters.
"""
from __future__ import annotations

import dataclasses
import numpy as np


@dataclasses.dataclass
class Level:
    nclus: int
    H: list            # H_l adjacency, sorted lists (structural block pattern of A_l)
    nlist: list        # n(s) = H_l-adj(s), ascending
    wlist: list        # w(s) = F-adj(s) \ n(s) at the moment s is eliminated, ascending
    batches: list      # list of lists of cluster ids (ascending inside a batch)
    nphase1: int       # number of phase-I (interior) batches
    interior: np.ndarray   # bool per cluster: all of F_start-adj(s) in s's subdomain
    Ffinal: list       # fill graph after the level, sorted lists
    Fstart: list = None    # block pattern at the level start (= H under coarse_fill=1)


@dataclasses.dataclass
class Analysis:
    n: int
    D: int
    L_top: int
    nsub_log2: int
    perm: np.ndarray       # perm[new] = old  (int64)
    leaf_off: np.ndarray   # DOF offsets of the 2^D leaves in the permuted order (int64, 2^D + 1)
    levels: list           # Level for l = 0 .. L_top-1
    H_top: list            # block pattern of the top level (l = L_top)

    def subdomain(self, level: int, c: int) -> int:
        d = self.D - level
        sd = min(self.nsub_log2, self.D)
        return c >> (d - sd)


def _units(n, coords, column_id):
    """Units (O2.1): extruded columns (ascending column id) or single DOFs."""
    if column_id is None:
        dofs_of = None
        ucoord = np.asarray(coords, dtype=np.float64).reshape(n, -1)
        return ucoord, None
    column_id = np.asarray(column_id, dtype=np.int64)
    cids, first = np.unique(column_id, return_index=True)   # first = lowest DOF index per column
    c = np.asarray(coords, dtype=np.float64).reshape(n, -1)
    ucoord = c[first, : min(2, c.shape[1])]
    unit_of_dof = np.searchsorted(cids, column_id)
    return ucoord, unit_of_dof


def rcb(ucoord: np.ndarray, D: int):
    """O2.3: perfect binary RCB tree to depth D.  Returns the leaf of every unit.
    At a node: split on the axis of largest extent (lowest axis on ties), sort
    by (coordinate, unit id), left child = first ceil(|I|/2) units."""
    U = ucoord.shape[0]
    leaf = np.zeros(U, dtype=np.int64)
    nodes = [np.arange(U, dtype=np.int64)]
    for depth in range(D):
        nxt = []
        for I in nodes:
            if I.size == 0:
                nxt.append(I)
                nxt.append(I)
                continue
            cc = ucoord[I]
            ext = cc.max(axis=0) - cc.min(axis=0)
            ax = int(np.argmax(ext))                       # first maximum = lowest axis
            order = np.lexsort((I, cc[:, ax]))             # key: (coord_ax, unit id)
            S = I[order]
            h = (S.size + 1) // 2
            nxt.append(S[:h])
            nxt.append(S[h:])
        nodes = nxt
    for x, I in enumerate(nodes):
        leaf[I] = x
    return leaf


def _bfs_order(I_sorted, inset, rowptr, colind, start):
    """BFS over the subgraph induced by the unit set I (membership mask `inset`),
    neighbours in ascending id, restarting from the smallest unvisited unit of I when a
    component is exhausted."""
    from collections import deque
    seen = {start}
    order = [start]
    q = deque([start])
    nxt_start = 0
    while len(order) < len(I_sorted):
        if not q:
            while I_sorted[nxt_start] in seen:
                nxt_start += 1
            v = int(I_sorted[nxt_start])
            seen.add(v)
            order.append(v)
            q.append(v)
        u = q.popleft()
        for w in colind[rowptr[u]:rowptr[u + 1]]:      # CSR rows are sorted: ascending id
            w = int(w)
            if inset[w] and w not in seen:
                seen.add(w)
                order.append(w)
                q.append(w)
    return order


def gbisect(n, rowptr, colind, D):
    """O2.3 without coordinates (NEXT f4; "recursive BFS level-set bisection";
    the paper's clustering is "algebraic").  Perfect binary tree to depth D.
    At a node with unit set I (ascending):
      1. BFS on the subgraph induced by I from min(I) (restarting as in _bfs_order); its
         last unit g is a pseudo-peripheral start;
      2. order = the same BFS from g;
      3. left child = the first ceil(|I|/2) units of the order, right child = the rest.
    Returns the leaf of every unit (units are DOFs)."""
    leaf = np.zeros(n, dtype=np.int64)
    inset = np.zeros(n, dtype=bool)
    nodes = [np.arange(n, dtype=np.int64)]
    for depth in range(D):
        nxt = []
        for I in nodes:
            if I.size == 0:
                nxt += [I, I]
                continue
            inset[I] = True
            first = _bfs_order(I, inset, rowptr, colind, int(I[0]))
            order = _bfs_order(I, inset, rowptr, colind, first[-1])
            inset[I] = False
            order = np.asarray(order, dtype=np.int64)
            h = (order.size + 1) // 2
            nxt.append(np.sort(order[:h]))
            nxt.append(np.sort(order[h:]))
        nodes = nxt
    for x, I in enumerate(nodes):
        leaf[I] = x
    return leaf


def analyze(n, rowptr, colind, coords, column_id=None, leaf_size=64, leaf_columns=0,
            top_log2=3, nsub_log2=3, coarse_fill=0) -> Analysis:
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colind = np.asarray(colind, dtype=np.int64)
    if coords is None:
        if column_id is not None:
            raise ValueError("graph bisection works on DOF units (no column_id)")
        U = n
        leaf_units = leaf_size
        if leaf_units <= 0:
            raise ValueError("leaf size must be positive")
        D = 0
        while -(-U // (1 << D)) > leaf_units:
            D += 1
        return _schedule(n, rowptr, colind, gbisect(n, rowptr, colind, D), D, top_log2, nsub_log2, coarse_fill)
    ucoord, unit_of_dof = _units(n, coords, column_id)
    U = ucoord.shape[0]
    leaf_units = leaf_columns if column_id is not None else leaf_size
    if leaf_units <= 0:
        raise ValueError("leaf size must be positive")
    # O2.2 depth: smallest D with ceil(U / 2^D) <= leaf_units
    D = 0
    while -(-U // (1 << D)) > leaf_units:
        D += 1
    uleaf = rcb(ucoord, D)
    dof_leaf = uleaf if unit_of_dof is None else uleaf[unit_of_dof]
    return _schedule(n, rowptr, colind, dof_leaf, D, top_log2, nsub_log2, coarse_fill)


def _merge(adj, nclus):
    """Merge-quotient onto the parents (binary tree, reading Q9): P ~ Q iff some child of P
    is adjacent to some child of Q, P != Q."""
    out = [set() for _ in range(nclus // 2)]
    for c in range(nclus):
        P = c >> 1
        for q in adj[c]:
            if q >> 1 != P:
                out[P].add(q >> 1)
    return [sorted(h) for h in out]


def _schedule(n, rowptr, colind, dof_leaf, D, top_log2, nsub_log2, coarse_fill=0) -> Analysis:
    if coarse_fill not in (0, 1):
        raise ValueError("coarse_fill must be 0 (structural coarse neighbours) or 1 (fill-closed)")
    # O2.4 permutation: leaves left to right, DOFs ascending inside a leaf
    perm = np.lexsort((np.arange(n), dof_leaf)).astype(np.int64)
    nleaf = 1 << D
    counts = np.bincount(dof_leaf, minlength=nleaf)
    leaf_off = np.zeros(nleaf + 1, dtype=np.int64)
    np.cumsum(counts, out=leaf_off[1:])
    L_top = max(0, D - top_log2)
    sd = min(nsub_log2, D)
    # O2.7 H_0: leaves p != q adjacent iff the CSR stores an entry between them
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))
    lp = dof_leaf[rows]
    lq = dof_leaf[colind]
    off = lp != lq
    pairs = np.unique(lp[off] * nleaf + lq[off])
    H = [[] for _ in range(nleaf)]
    for pq in pairs.tolist():
        H[pq // nleaf].append(pq % nleaf)
    H = [sorted(set(h)) for h in H]
    F0 = H                  # block pattern of the level's input A_l (H_0 at level 0)
    levels = []
    for l in range(L_top):
        nclus = 1 << (D - l)
        d = D - l
        sub = [c >> (d - sd) for c in range(nclus)]
        F = [set(h) for h in F0]
        nlist = [list(h) for h in H]
        interior = np.array([all(sub[q] == sub[s] for q in F0[s]) for s in range(nclus)], dtype=bool)
        wlist = [None] * nclus
        processed = np.zeros(nclus, dtype=bool)
        batches = []
        nphase1 = 0
        for phase in (1, 2):
            while True:
                cand = [s for s in range(nclus) if not processed[s] and (phase == 2 or interior[s])]
                if not cand:
                    break
                B = []
                Bset = set()
                for s in cand:                                   # greedy, ascending id
                    if not (F[s] & Bset):
                        B.append(s)
                        Bset.add(s)
                for s in B:                                      # record w(s) before the fill
                    wlist[s] = sorted(F[s] - set(nlist[s]))
                for s in B:                                      # fill: clique on n(s)
                    ns = nlist[s]
                    for p in ns:
                        F[p].update(q for q in ns if q != p)
                for s in B:
                    processed[s] = True
                batches.append(B)
                if phase == 1:
                    nphase1 += 1
        Ffinal = [sorted(f) for f in F]
        levels.append(Level(nclus, H, nlist, wlist, batches, nphase1, interior, Ffinal, [list(f) for f in F0]))
        # the block pattern of A_c: parents adjacent iff some children are F_final-adjacent
        F0 = _merge(Ffinal, nclus)
        # H_{l+1}: R-coarse merges the structural neighbours; O2.9 takes the whole pattern
        H = F0 if coarse_fill else _merge(H, nclus)
    # the top's block pattern is the whole pattern of A_top under both readings
    return Analysis(n=n, D=D, L_top=L_top, nsub_log2=sd, perm=perm, leaf_off=leaf_off,
                    levels=levels, H_top=F0)


def analyze_problem(p, top_log2=3, nsub_log2=3, coarse_fill=0) -> Analysis:
    return analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id,
                   leaf_size=p.leaf_size, leaf_columns=p.leaf_columns,
                   top_log2=top_log2, nsub_log2=nsub_log2, coarse_fill=coarse_fill)
