"""Pin P8: the input generators against closed-form spectra.

* 5-point eps*u_xx + u_yy on n x n: eigenvalues 4(n+1)^2[eps sin^2(pi i/(2n+2)) +
  sin^2(pi j/(2n+2))] (§1), here with h^2 = 1/(n+1)^2 dropped.
* cell-centred 7-point with k = 1 and Dirichlet half-cell faces (boundary term 2k):
  the 1-D factor tridiag(-1, 2, -1) with end diagonals 3 has eigenvalues
  4 sin^2(k pi/(2n)), k = 1..n (ghost value u_{-1} = -u_0); 3-D = sums.
"""
import json
import os

import numpy as np
import pytest

from problems import gen_poisson2d, gen_laplace3d, gen_slab, gen_stokes_q1, grf

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("n,aniso", [(32, 1.0), (12, 1e-3), (9, 1e-6)])
def test_poisson2d_closed_form_spectrum(n, aniso):
    p = gen_poisson2d(n, aniso=aniso)
    A = p.to_scipy().toarray()
    ev = np.sort(np.linalg.eigvalsh(A))
    i = np.arange(1, n + 1)
    s2 = np.sin(np.pi * i / (2 * n + 2)) ** 2
    ref = np.sort((4 * (aniso * s2[:, None] + s2[None, :])).ravel())
    assert np.abs(ev - ref).max() <= 1e-12 * ref.max()


def test_aniso_golden_1x1():
    g = GOLD["aniso_eigs"]
    p = gen_poisson2d(g["n"], aniso=g["eps"])
    assert np.array_equal(p.to_scipy().toarray(), np.array(g["matrix"]))


def test_laplace3d_unit_k_closed_form():
    n = 6
    p = gen_laplace3d(n, sigma=0.0)
    A = p.to_scipy().toarray()
    k = np.arange(1, n + 1)
    l1 = 4 * np.sin(k * np.pi / (2 * n)) ** 2
    ref = np.sort((l1[:, None, None] + l1[None, :, None] + l1[None, None, :]).ravel())
    assert np.abs(np.sort(np.linalg.eigvalsh(A)) - ref).max() <= 1e-12 * ref.max()


def test_csr_format_and_symmetry():
    for p in [gen_laplace3d(10), gen_slab(12, 5), gen_stokes_q1(5, 4, 3)]:
        assert p.rowptr.dtype == np.int64 and p.colind.dtype == np.int32 and p.vals.dtype == np.float64
        for r in range(p.n):
            c = p.colind[p.rowptr[r]:p.rowptr[r + 1]]
            assert np.all(np.diff(c) > 0)
        A = p.to_scipy()
        assert abs(A - A.T).max() <= 1e-14 * abs(A).max()
        assert np.linalg.eigvalsh(A.toarray()).min() > 0


def test_stokes_q1_rigid_modes_only_killed_by_basal_friction():
    """Without basal friction the first-order-Stokes form annihilates constant
    horizontal velocity (u1 = const, u2 = 0): only the Robin term makes it SPD."""
    p = gen_stokes_q1(4, 5, 3, sigma_mu=0.0, sigma_beta=0.0)
    A = p.to_scipy()
    u = np.zeros(p.n)
    u[0::2] = 1.0
    Au = A @ u
    # only bottom-layer rows see the basal term
    nn = 4 * 5
    assert np.abs(Au[2 * nn:]).max() < 1e-12
    assert np.abs(Au[:2 * nn:2]).min() > 0


def test_grf_statistics():
    g = grf((64, 64), 8.0, 2.0, 1)
    assert abs(g.mean()) < 1e-12 and abs(g.std() - 2.0) < 1e-12
    g2 = grf((64, 64), 8.0, 2.0, 1)
    assert np.array_equal(g, g2)
    # correlation length: neighbours strongly correlated
    assert np.corrcoef(g[:, :-1].ravel(), g[:, 1:].ravel())[0, 1] > 0.9
