"""Pins of the oracle's operator and solves against the mathematics (not itself).

PAPER.md L133-139 (Eq. (2.1)) and L181-187 (Eq. (2.5)); readings R1-R6.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import (assemble, detector_matrix, frequency_matrix, make_grid, source_matrix)

D_TEST = 0.3
NU = 2.2e10


def _mu_smooth(g):
    return 0.05 + 0.1 * (g.X / g.L[0]) * (g.Z / g.L[2]) + 0.02 * np.sin(g.Y)


def test_operator_complex_symmetric():
    """A is complex symmetric (A^T = A, not Hermitian) -- needed by COCG and by
    reciprocity (BASELINE north_star)."""
    g = make_grid((5, 4, 6), (2.0, 1.5, 3.0))
    A = assemble(g, D_TEST, _mu_smooth(g), 2 * np.pi * 1e8, NU)
    assert abs(A - A.T).max() == 0.0
    assert abs(A - A.conj().T).max() > 0.0


def test_frequency_term_is_iomega_over_nu_E():
    """A(omega) - A(0) = i omega/nu E (Eq. (2.5) 'i omega_j/nu E + A(p)')."""
    g = make_grid((4, 5, 3), (1.0, 1.0, 1.0))
    mu = _mu_smooth(g)
    w = 2 * np.pi * 7e7
    dA = assemble(g, D_TEST, mu, w, NU) - assemble(g, D_TEST, mu, 0.0, NU)
    assert abs(dA - 1j * w / NU * frequency_matrix(g)).max() < 1e-18


def test_absorption_linearity():
    """assemble(mu1 + mu2) - assemble(mu1) = diag(theta mu2): mu enters the
    diagonal only, with the Robin-plane half weight."""
    g = make_grid((4, 3, 5), (1.0, 1.0, 1.0))
    mu1 = _mu_smooth(g)
    mu2 = np.random.default_rng(3).uniform(0, 1, g.N)
    dA = assemble(g, D_TEST, mu1 + mu2, 0.0, NU) - assemble(g, D_TEST, mu1, 0.0, NU)
    assert abs(dA - np.diag(g.theta * mu2)).max() < 1e-14


def test_constant_mu_interior_row_is_textbook_laplacian():
    """Interior row, mu = 0: diagonal 2D/hx^2 + 2D/hy^2 + 2D/hz^2, off-diagonals
    -D/h^2 (standard 7-point Laplacian)."""
    g = make_grid((5, 5, 5), (6.0, 6.0, 4.0))
    A = assemble(g, 1.0, np.zeros(g.N), 0.0, NU).toarray()
    n = (2 * 5 + 2) * 5 + 2
    assert A[n, n] == pytest.approx(2 / g.hx ** 2 + 2 / g.hy ** 2 + 2 / g.hz ** 2, rel=1e-14)
    assert A[n, n + 1] == pytest.approx(-1 / g.hx ** 2, rel=1e-14)
    assert A[n, n + 5] == pytest.approx(-1 / g.hy ** 2, rel=1e-14)
    assert A[n, n + 25] == pytest.approx(-1 / g.hz ** 2, rel=1e-14)
    assert np.count_nonzero(A[n]) == 7


def _mms_error(n, L, D, omega, mu_fn):
    """Manufactured solution phi* = sin(pi x/Lx) sin(pi y/Ly) g(z) with
    g(z) = 1 - 2z/Lz + a2 cos(pi z/Lz), a2 = -1 - 4D/Lz, which satisfies phi = 0
    on the lateral faces and 0.25 phi + (D/2) dphi/dxi = 0 on z = 0, Lz
    (PAPER.md L136-137).  Returns max nodal error of the discrete solve."""
    g = make_grid(n, L)
    Lx, Ly, Lz = L
    a2 = -1.0 - 4.0 * D / Lz
    gz = 1 - 2 * g.Z / Lz + a2 * np.cos(np.pi * g.Z / Lz)
    gzz = -a2 * (np.pi / Lz) ** 2 * np.cos(np.pi * g.Z / Lz)
    sxy = np.sin(np.pi * g.X / Lx) * np.sin(np.pi * g.Y / Ly)
    phi = sxy * gz
    mu = mu_fn(g)
    lap = sxy * (-((np.pi / Lx) ** 2 + (np.pi / Ly) ** 2) * gz + gzz)
    f = -D * lap + (mu + 1j * omega / NU) * phi
    A = assemble(g, D, mu, omega, NU)
    u = spla.spsolve(A.tocsc(), g.theta * f)
    return np.abs(u - phi).max()


@pytest.mark.parametrize("D,omega", [(0.3, 0.0), (1.0 / 30.15, 2 * np.pi * 1.4e8), (2.0, 2 * np.pi * 5e8)])
def test_manufactured_solution_second_order(D, omega):
    """Halving every spacing divides the error by ~4 (second order)."""
    L = (2.0, 2.5, 3.0)
    e1 = _mms_error((7, 7, 8), L, D, omega, _mu_smooth)
    e2 = _mms_error((15, 15, 15), L, D, omega, _mu_smooth)
    e3 = _mms_error((31, 31, 29), L, D, omega, _mu_smooth)
    r1, r2 = e1 / e2, e2 / e3
    assert 3.4 < r2 < 4.6, (e1, e2, e3)
    assert 3.0 < r1 < 5.0, (e1, e2, e3)


def test_wrong_robin_coefficient_breaks_convergence():
    """Sanity of the MMS pin itself: the same manufactured solution with a
    perturbed Robin factor (0.35 instead of 0.25) must NOT converge, i.e. the pin
    is sensitive to the boundary treatment."""
    L = (2.0, 2.5, 3.0)
    D = 0.3
    # phi* built for 0.35 phi + (D/2) dphi/dxi = 0 -> g'(0) = 0.7 g(0)/D ... use the
    # general construction: g = 1 + a1 z + a2 cos(pi z/L) with the 0.35 factor
    Lz = L[2]
    kappa = 0.35 * 2 / D
    # g'(0) = kappa g(0), g'(L) = -kappa g(L):  a1 = kappa (1 + a2);
    # a1 = -kappa (1 + a1 L - a2)  => solve 2x2
    M = np.array([[1.0, -kappa], [1.0 + kappa * Lz, -kappa]])
    a1, a2 = np.linalg.solve(M, [kappa, -kappa])

    def err(n):
        g = make_grid(n, L)
        gz = 1 + a1 * g.Z + a2 * np.cos(np.pi * g.Z / Lz)
        gzz = -a2 * (np.pi / Lz) ** 2 * np.cos(np.pi * g.Z / Lz)
        sxy = np.sin(np.pi * g.X / L[0]) * np.sin(np.pi * g.Y / L[1])
        phi = sxy * gz
        mu = _mu_smooth(g)
        f = -D * sxy * (-((np.pi / L[0]) ** 2 + (np.pi / L[1]) ** 2) * gz + gzz) + mu * phi
        u = spla.spsolve(assemble(g, D, mu, 0.0, NU).tocsc(), g.theta * f)
        return np.abs(u - phi).max() / np.abs(phi).max()

    e2, e3 = err((15, 15, 15)), err((31, 31, 29))
    assert e3 > 1e-2 and e2 / e3 < 2.0


def test_reciprocity_coinciding_sources_detectors():
    """C^T A^-1 B is symmetric when sources and detectors coincide (A complex
    symmetric; BASELINE north_star pin)."""
    g = make_grid((6, 5, 5), (3.0, 3.0, 2.0))
    A = assemble(g, D_TEST, _mu_smooth(g), 2 * np.pi * 1e8, NU).tocsc()
    nodes = np.array([1, 8, 13, 20, 27, 28])          # top face k = 0
    B, C = source_matrix(g, nodes), detector_matrix(g, nodes)
    M = C.T @ spla.spsolve(A, B.toarray())
    M = np.asarray(M)
    assert np.abs(M - M.T).max() < 1e-12 * np.abs(M).max()


def test_solve_matches_dense_inverse_and_transpose():
    """splu forward/transposed solves against a dense inverse on a tiny grid."""
    g = make_grid((3, 4, 4), (1.0, 1.0, 1.0))
    A = assemble(g, D_TEST, _mu_smooth(g), 2 * np.pi * 2e8, NU)
    lu = spla.splu(A.tocsc())
    rhs = np.random.default_rng(0).standard_normal((g.N, 3)) + 0j
    Ad = A.toarray()
    assert np.abs(lu.solve(rhs) - np.linalg.solve(Ad, rhs)).max() < 1e-12
    assert np.abs(lu.solve(rhs, trans="T") - np.linalg.solve(Ad.T, rhs)).max() < 1e-12
