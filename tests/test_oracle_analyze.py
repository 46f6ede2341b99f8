"""Pin P7: the oracle's analyze against closed forms and brute force.

* RCB on grid coordinates gives exact boxes: C1 -> 64 boxes of 4x4, C2 -> 4096
  cubes of 4^3, C3 -> 8192 leaves of 2x4 (or 4x2) whole columns, Q1 -> 1x2 columns
  (extruded partitioning keeps every vertical line in one cluster).
* every batch is an independent set of the fill graph at its time and is maximal
  (brute-force re-simulation of Alg. 1's loop), interior clusters first.
"""
import numpy as np
import pytest

from problems import gen_poisson2d, gen_laplace3d, gen_slab, gen_stokes_q1
from oracle.analyze import analyze_problem, analyze


def _boxes(p, an, dims):
    """For each leaf, return the set of per-axis extents of its unit coordinates."""
    out = set()
    inv = np.empty(p.n, dtype=np.int64)
    inv[an.perm] = np.arange(p.n)
    for c in range(an.leaf_off.shape[0] - 1):
        d = an.perm[an.leaf_off[c]:an.leaf_off[c + 1]]
        cc = p.coords[d][:, :dims]
        lo, hi = cc.min(0), cc.max(0)
        out.add(tuple((hi - lo).tolist()))
    return out


def test_C1_boxes():
    p = gen_poisson2d(32)
    an = analyze_problem(p)
    assert an.D == 6 and an.L_top == 3 and len(an.levels) == 3
    assert np.all(np.diff(an.leaf_off) == 16)
    assert _boxes(p, an, 2) == {(3.0, 3.0)}
    # leaves are aligned 4x4 boxes
    for c in range(64):
        d = an.perm[an.leaf_off[c]:an.leaf_off[c + 1]]
        cc = p.coords[d]
        assert np.all(cc.min(0) % 4 == 0)
    assert sorted(an.perm.tolist()) == list(range(p.n))


def test_C2_cubes():
    p = gen_laplace3d(64)
    an = analyze_problem(p)
    assert an.D == 12 and an.L_top == 9
    assert np.all(np.diff(an.leaf_off) == 64)
    assert _boxes(p, an, 3) == {(3.0, 3.0, 3.0)}


def test_C3_columns():
    p = gen_slab(256, 10)
    an = analyze_problem(p)
    assert an.D == 13
    assert np.all(np.diff(an.leaf_off) == 80)
    # column integrity: every column lies in exactly one leaf
    leaf_of = np.empty(p.n, dtype=np.int64)
    for c in range(1 << an.D):
        leaf_of[an.perm[an.leaf_off[c]:an.leaf_off[c + 1]]] = c
    for col in range(0, 256 * 256, 97):
        assert np.unique(leaf_of[p.column_id == col]).size == 1
    assert _boxes(p, an, 2) <= {(1000.0, 3000.0), (3000.0, 1000.0)}


def test_Q1_columns():
    p = gen_stokes_q1(16, 16, 4, leaf_columns=2)
    an = analyze_problem(p)
    assert an.D == 7
    assert np.all(np.diff(an.leaf_off) == 2 * 4 * 2)
    assert _boxes(p, an, 2) <= {(1.0, 0.0), (0.0, 1.0)}


def _resimulate(an):
    """Brute force: walk the batches with a fresh fill graph and check
    independence, maximality, phase order and the recorded w(s)."""
    for l, lev in enumerate(an.levels):
        nclus = lev.nclus
        F = [set(h) for h in lev.Fstart]
        assert all(set(h) <= set(f) for h, f in zip(lev.H, lev.Fstart))
        done = np.zeros(nclus, dtype=bool)
        for bi, B in enumerate(lev.batches):
            phase1 = bi < lev.nphase1
            Bs = set(B)
            for s in B:
                assert not done[s]
                assert not (F[s] & Bs), "batch not independent"
                if phase1:
                    assert lev.interior[s]
                assert lev.wlist[s] == sorted(F[s] - set(lev.H[s]))
                assert lev.nlist[s] == lev.H[s]
            # maximality: every skipped eligible cluster is adjacent to a member
            for t in range(nclus):
                if done[t] or t in Bs or (phase1 and not lev.interior[t]):
                    continue
                # greedy scan: t was skipped only because an earlier member is adjacent
                assert {b for b in F[t] & Bs if b < t}, "batch not maximal"
            for s in B:
                for p_ in lev.H[s]:
                    for q in lev.H[s]:
                        if p_ != q:
                            F[p_].add(q)
                done[s] = True
        assert done.all()
        assert [sorted(f) for f in F] == lev.Ffinal
        # subdomain locality of phase-I fill: an interior cluster's
        # whole starting pattern (its n and its inherited w) lies in its subdomain
        for s in range(nclus):
            if lev.interior[s]:
                assert all(an.subdomain(l, q) == an.subdomain(l, s) for q in lev.Fstart[s])
        # the next level starts from the block pattern of A_c: the merge of F_final
        nxt = an.levels[l + 1].Fstart if l + 1 < len(an.levels) else an.H_top
        merged = [set() for _ in range(nclus // 2)]
        for c in range(nclus):
            for q in F[c]:
                if q >> 1 != c >> 1:
                    merged[c >> 1].add(q >> 1)
        assert [sorted(m) for m in merged] == [list(x) for x in nxt]


@pytest.mark.parametrize("gen", [lambda: gen_poisson2d(32), lambda: gen_laplace3d(16, leaf_size=16),
                                 lambda: gen_slab(32, 4, leaf_columns=4),
                                 lambda: gen_stokes_q1(12, 12, 3, leaf_columns=2)])
@pytest.mark.parametrize("coarse_fill", [0, 1])
def test_batches_independent_maximal(gen, coarse_fill):
    p = gen()
    an = analyze_problem(p, coarse_fill=coarse_fill)
    assert len(an.levels) >= 1
    _resimulate(an)
    for l, lev in enumerate(an.levels):
        if coarse_fill:   # O2.9: the neighbours are the whole starting pattern
            assert [list(h) for h in lev.H] == [list(f) for f in lev.Fstart]


def _box_graph(p, an, l, dims):
    """Closed form of the structural coarse neighbours on a grid with a face-coupling
    stencil (5-point / 7-point): the level-l clusters are axis-aligned boxes of grid cells
    (RCB on grid coordinates), and two boxes are neighbours iff they share a face, i.e. their
    intervals touch (hi + 1 == lo) on one axis and overlap on all others."""
    nclus = an.levels[l].nclus
    lo = np.zeros((nclus, dims)); hi = np.zeros((nclus, dims))
    span = 1 << l
    for c in range(nclus):
        d = an.perm[an.leaf_off[c * span]:an.leaf_off[(c + 1) * span]]
        cc = p.coords[d][:, :dims]
        lo[c], hi[c] = cc.min(0), cc.max(0)
    G = [[] for _ in range(nclus)]
    for s in range(nclus):
        for q in range(nclus):
            if q == s:
                continue
            touch = overlap = 0
            for a in range(dims):
                if hi[s, a] + 1 == lo[q, a] or hi[q, a] + 1 == lo[s, a]:
                    touch += 1
                elif lo[s, a] <= hi[q, a] and lo[q, a] <= hi[s, a]:
                    overlap += 1
            if touch == 1 and overlap == dims - 1:
                G[s].append(q)
    return G


@pytest.mark.parametrize("gen,dims", [(lambda: gen_poisson2d(32), 2), (lambda: gen_laplace3d(16, leaf_size=8), 3)])
def test_rcoarse_neighbours_are_face_adjacent_boxes(gen, dims):
    """Pin of reading R-coarse: at every level n(s) = the clusters whose box
    shares a face with s's box (closed form from the coordinates, not from the merge), so the
    neighbour count stays <= 2*dims at every level (Thm 1 condition 1), while the
    starting pattern keeps the inherited fill as w."""
    p = gen()
    an = analyze_problem(p)
    for l, lev in enumerate(an.levels):
        assert [list(h) for h in lev.H] == _box_graph(p, an, l, dims), l
        assert max(len(h) for h in lev.H) <= 2 * dims
    # O2.9 instead grows the neighbour sets with the level (fill becomes n)
    an1 = analyze_problem(p, coarse_fill=1)
    assert max(len(h) for h in an1.levels[-1].H) > 2 * dims


def test_depth_rule_and_empty_children():
    # U = 10 units, leaf 3 -> D = 2 (ceil(10/4) = 3); children may be empty for tiny U
    p = gen_poisson2d(5, 2, leaf_size=3)
    an = analyze(p.n, p.rowptr, p.colind, p.coords, None, leaf_size=3)
    assert an.D == 2 and an.L_top == 0
    assert an.leaf_off[-1] == 10 and np.all(np.diff(an.leaf_off) <= 3)
    an1 = analyze(p.n, p.rowptr, p.colind, p.coords, None, leaf_size=1)
    assert an1.D == 4 and (np.diff(an1.leaf_off) == 0).sum() == 6


def test_graph_bisection_path_closed_form():
    """Pin of the coordinate-free tree (NEXT f4): on a path graph the BFS from min(I)
    ends at max(I), the BFS from there lists I in descending order, so every node splits
    into its upper and lower halves and every leaf is a contiguous index range."""
    import scipy.sparse as sp
    from oracle.analyze import gbisect
    n, D = 96, 4
    A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()
    leaf = gbisect(n, A.indptr.astype(np.int64), A.indices.astype(np.int64), D)
    # leaf 0 = the top of the index range (left child = first half of the descending BFS)
    expect = np.zeros(n, dtype=np.int64)
    lo, hi = [0], [n]
    nodes = [np.arange(n)]
    for _ in range(D):
        nxt = []
        for I in nodes:
            h = (I.size + 1) // 2
            desc = I[::-1]
            nxt += [np.sort(desc[:h]), np.sort(desc[h:])]
        nodes = nxt
    for x, I in enumerate(nodes):
        expect[I] = x
    assert np.array_equal(leaf, expect)
    for x in range(1 << D):   # contiguous leaves of 6 DOFs
        idx = np.nonzero(leaf == x)[0]
        assert idx.size == 6 and np.all(np.diff(idx) == 1)


def test_graph_bisection_disconnected_and_balanced():
    """Two disjoint grids: the BFS restarts on the unvisited component; every tree node
    splits into ceil/floor halves (perfect binary tree, O2.2)."""
    import scipy.sparse as sp
    from oracle.analyze import gbisect
    p = gen_poisson2d(6)
    A = p.to_scipy()
    B = sp.block_diag([A, A]).tocsr()
    n = B.shape[0]
    leaf = gbisect(n, B.indptr.astype(np.int64), B.indices.astype(np.int64), 3)
    counts = np.bincount(leaf, minlength=8)
    assert counts.sum() == n and counts.max() - counts.min() <= 1
