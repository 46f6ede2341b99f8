"""C4 at full size on one GPU (-m gpu): BASELINE.json configs[3], the bench's default workload
(Q1 first-order-Stokes-type operator, 512 x 512 x 20 hexahedra, 2 DOF/node, 10,485,760 DOF,
eps 1e-2, PCG to 1e-8), in the launch configuration bench.py times.  At this size the factor
runs with the record space active (completed levels' T_s / C_s spilled to pinned host memory
while the 131 GB level-2 store is resident) and with oversized batches split into sub-batches
by the workspace budget -- the two paths only C4 takes.

The whole oracle factor of C4 is out of reach (hours of Python), so this leg checks what the
oracle can compute one by one at this size, and what holds at any size (SURVEY §8(c) parity
protocol, full-size leg):
  * the analysis (partition, cluster tree, every level's batches) bit-exact with oracle/analyze;
  * the kept rank and pivot sequence of a seeded sample of 200 clusters of level 0's SECOND
    batch (the first with compression decisions: batch 0 has w(s) = ∅), each eliminated by the
    oracle (oracle.factor.eliminate) after exactly the batch-0 clusters that touch its blocks
    (its batch-0 neighbours, in batch order; a batch is an independent set and a phase-I batch
    stays inside its subdomain, so no other elimination reaches them), on level-0 blocks built
    from the permuted CSR on first access; a disagreement is allowed only where the oracle's
    margins flag the cluster;
  * operator properties of the factor apply (symmetry, positivity, linearity);
  * PCG to the config's tolerance with the true residual recomputed against A on the host;
  * bitwise determinism across two factors (every level's kept ranks, the apply), i.e. the
    sub-batch split and the spill / restore of the records change nothing between runs.
The C4 operator is compared with the oracle on every cluster at 1/16 scale (test_gpu_fullsize.py),
and the spill / restore path bitwise against resident records there.
"""
import numpy as np
import pytest

import scipy.sparse as sp

from problems import gen_config
from oracle.analyze import analyze
from oracle.factor import BlockStore, eliminate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch
    from paper_1811_11248_b200 import hsolve
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    hsolve.lib()
    return hsolve


class _LazyLevel0(BlockStore):
    """The oracle's block store on level 0 of the permuted A, each block built from the CSR on
    first access (an untouched block of an eliminated cluster is structurally zero)."""

    def __init__(self, p, an):
        super().__init__(np.diff(an.leaf_off).tolist())
        self.size0 = list(self.live)
        self.A = sp.csr_matrix((p.vals, p.colind, p.rowptr), shape=(p.n, p.n))
        self.off, self.perm = an.leaf_off, an.perm
        self.iperm = np.empty_like(an.perm)
        self.iperm[an.perm] = np.arange(an.perm.size)
        self.rows = {}

    def _row(self, q):
        if q not in self.rows:
            R = self.A[self.perm[self.off[q]:self.off[q + 1]]].tocoo()
            cn = self.iperm[R.col]
            self.rows[q] = (R.row, cn, R.data, np.searchsorted(self.off, cn, side="right") - 1)
        return self.rows[q]

    def get(self, p, q):
        key = (p, q) if p >= q else (q, p)
        if key not in self.blocks and all(self.live[c] == self.size0[c] for c in key):
            rr, cn, dv, lf = self._row(key[0])
            sel = lf == key[1]
            M = np.zeros((self.size0[key[0]], self.size0[key[1]]))
            np.add.at(M, (rr[sel], cn[sel] - self.off[key[1]]), dv[sel])
            self.blocks[key] = M
        return super().get(p, q)


def _level0_batch1_sample(p, an, ranks, pp, pv, nsample=200):
    lev = an.levels[0]
    assert lev.nphase1 >= 2
    b0 = set(lev.batches[0])
    S1 = sorted(np.random.default_rng(0).choice(lev.batches[1], nsample, replace=False).tolist())
    T = sorted({t for s in S1 for t in list(lev.nlist[s]) + list(lev.wlist[s]) if t in b0})
    st = _LazyLevel0(p, an)
    for t in T:   # batch 0 in batch order (ascending)
        eliminate(st, 0, t, lev.nlist[t], lev.wlist[t], p.eps, True)
    flagged_diff = ncpqr = 0
    for s in S1:
        e = eliminate(st, 0, s, lev.nlist[s], lev.wlist[s], p.eps, True)
        ncpqr += len(lev.wlist[s]) > 0
        g = pv[pp[s]:pp[s + 1]]
        if not (ranks[s] == e.r and np.array_equal(g, e.piv)):
            assert e.flagged, f"level-0 cluster {s}: gpu r={ranks[s]} oracle r={e.r} (unflagged)"
            flagged_diff += 1
    print(f"[C4] level-0 batch-1 sample: {len(S1)} clusters ({ncpqr} with compression) after {len(T)} "
          f"batch-0 eliminations, {flagged_diff} flagged differences")
    assert ncpqr > 0 and flagged_diff <= 2


def test_c4_full_size(H):
    import gc
    p = gen_config("C4")
    assert p.n == 10_485_760
    h = H.hs_create(0)
    try:
        _c4_checks(H, h, p)
    finally:   # the handle's ~170 GB of cached device memory must not outlive the test
        h.close()
        gc.collect()


def _c4_checks(H, h, p):
    a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    an = analyze(p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                 leaf_columns=p.leaf_columns)
    info = H.hs_analysis_get_info(a)
    assert info["L_top"] == an.L_top and info["depth"] == an.D
    assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_PERM), an.perm)
    for l, lev in enumerate(an.levels):
        flat = np.concatenate([np.asarray(b, dtype=np.int64) for b in lev.batches]) if lev.batches else np.zeros(0)
        assert np.array_equal(H.hs_analysis_export(a, H.HS_EXP_BATCH_IDX, l), flat), f"level {l} batches"

    L = H.hs_analysis_get_info(a)["L_top"]
    v = np.random.default_rng(5).standard_normal(p.n)
    runs = []
    for _ in range(2):
        f = H.hs_factor_create(h, a, p.vals, eps=p.eps)
        runs.append(([H.hs_factor_export(f, H.HS_FEXP_RANKS, l) for l in range(L)], H.hs_apply(f, v)))
        if len(runs) == 1:
            del f   # two C4 factors cannot coexist on one GPU
    _level0_batch1_sample(p, an, runs[1][0][0], H.hs_factor_export(f, H.HS_FEXP_PIV_PTR, 0),
                          H.hs_factor_export(f, H.HS_FEXP_PIV, 0))
    assert all(np.array_equal(x, y) for x, y in zip(runs[0][0], runs[1][0]))
    assert np.array_equal(runs[0][1], runs[1][1])

    n = p.n
    for sd in (11, 12):
        rng = np.random.default_rng(sd)
        u, v = rng.standard_normal(n), rng.standard_normal(n)
        Mu, Mv = H.hs_apply(f, u), H.hs_apply(f, v)
        scale = np.linalg.norm(Mu) * np.linalg.norm(v)
        assert abs(Mu @ v - u @ Mv) <= 1e-12 * scale
        assert u @ Mu > 0 and v @ Mv > 0
        Mw = H.hs_apply(f, 0.75 * u - 1.5 * v)
        assert np.linalg.norm(Mw - (0.75 * Mu - 1.5 * Mv)) <= 1e-12 * np.linalg.norm(Mw)

    x, rep = H.hs_pcg(f, p.b, tol=p.tol)
    A = p.to_scipy()
    res = np.linalg.norm(p.b - A @ x) / np.linalg.norm(p.b)
    print(f"[C4] PCG {rep['iters']} iterations, true relative residual {res:.2e}")
    assert rep["converged"] and res <= 10 * p.tol
    assert abs(res - rep["relres_true"]) <= 1e-3 * res + 1e-15
