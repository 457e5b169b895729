"""Pins of the oracle's misfit and Jacobian (Eqs. (2.5)-(2.8), (3.1)-(3.12),
(EsTResidual), (Jacobian kth column)) against independent routes."""
import numpy as np
import pytest

from oracle import (absorption, jacobian, jacobian_weights, measurements, misfit,
                    sketched_residual)
from tests._small import all_sign_vectors, small_config, small_problem


def _dense_measurements(prob, p):
    """Independent route: dense inverse of A(omega, p)."""
    mu = absorption(p, prob.grid, prob.cfg)
    out = []
    for f in range(len(prob.omegas)):
        Ainv = np.linalg.inv(prob.operator(mu, f).toarray())
        out.append(prob.C.T.toarray() @ Ainv @ prob.B.toarray())
    return np.stack(out)


def test_measurements_match_dense_inverse():
    prob, wl = small_problem(small_config(n=(5, 5, 4), src=(2, 2), det=(2, 2)))
    M = measurements(prob, wl.p)
    Md = _dense_measurements(prob, wl.p)
    assert np.abs(M - Md).max() <= 1e-11 * np.abs(Md).max()


def test_identity_sketch_reproduces_full_misfit():
    """W = I, V = I: sum_f ||V^T R_f W||_F^2 equals the full-data misfit
    sum_f ||C^T A^-1 B - D_f||_F^2 (Eq. (3.2)) computed by dense inverse."""
    prob, wl = small_problem(small_config(n=(5, 5, 4), src=(3, 1), det=(2, 2)))
    ns, nd = prob.B.shape[1], prob.C.shape[1]
    full = np.sum(np.abs(_dense_measurements(prob, wl.p) - prob.data) ** 2)
    got = misfit(prob, wl.p, np.eye(ns), np.eye(nd))
    assert got == pytest.approx(full, rel=1e-11)
    S = sketched_residual(prob, wl.p, np.eye(ns), np.eye(nd))
    assert np.abs(S - (_dense_measurements(prob, wl.p) - prob.data)).max() < 1e-11 * np.abs(S).max()


def test_rademacher_enumeration_is_unbiased():
    """Theorem 3.1 exactly: the mean of (v^T R w)^2 over ALL
    +-1 vectors w (n_s = 3) and v (n_d = 3) equals ||R||_F^2, here with the
    complex modulus, summed over frequencies."""
    prob, wl = small_problem(small_config(n=(5, 5, 4), src=(3, 1), det=(3, 1)))
    full = misfit(prob, wl.p, np.eye(3), np.eye(3))
    vals = [misfit(prob, wl.p, w[:, None], v[:, None])
            for w in all_sign_vectors(3) for v in all_sign_vectors(3)]
    assert np.mean(vals) == pytest.approx(full, rel=1e-11)
    assert np.std(vals) > 0.01 * full          # a single draw is not the answer


def test_sketched_residual_is_linear_in_sources():
    """V^T R (W1 + W2) = V^T R W1 + V^T R W2 (the simultaneous source B w is a
    linear combination)."""
    prob, wl = small_problem(small_config(n=(5, 5, 4)))
    rng = np.random.default_rng(0)
    W1, W2 = rng.standard_normal((4, 2)), rng.standard_normal((4, 2))
    V = rng.standard_normal((4, 3))
    a = sketched_residual(prob, wl.p, W1 + W2, V)
    b = sketched_residual(prob, wl.p, W1, V) + sketched_residual(prob, wl.p, W2, V)
    assert np.abs(a - b).max() < 1e-10 * np.abs(a).max()


@pytest.mark.parametrize("seed", [0, 1])
def test_jacobian_matches_central_differences(seed):
    """(W^T (x) V^T) J against central finite differences of the sketched
    residual: pins the co-state formula, the minus sign of Eq. (2.8), the
    theta-weighted dA/dp and the chain rule through PaLS."""
    cfg = small_config(n=(8, 8, 7), eps=0.4, seed=seed)
    prob, wl = small_problem(cfg)
    rng = np.random.default_rng(10 + seed)
    W = np.sign(rng.standard_normal((4, 2)))
    V = np.sign(rng.standard_normal((4, 2)))
    J = jacobian(prob, wl.p, W, V)
    assert (np.abs(jacobian_weights(wl.p, prob.grid, cfg)).sum(1) > 0).sum() > 20
    h = 1e-6
    num = np.zeros_like(J)
    for k in range(wl.p.size):
        e = np.zeros_like(wl.p)
        e[k] = h
        num[..., k] = (sketched_residual(prob, wl.p + e, W, V)
                       - sketched_residual(prob, wl.p - e, W, V)) / (2 * h)
    err = np.linalg.norm(J - num) / np.linalg.norm(num)
    assert err < 1e-6, err
    # every parameter column with a visible derivative matches individually
    for k in range(wl.p.size):
        nk = np.linalg.norm(num[..., k])
        if nk > 1e-3 * np.linalg.norm(num):
            assert np.linalg.norm(J[..., k] - num[..., k]) < 1e-5 * nk, k


def test_jacobian_kronecker_consistency():
    """(W^T (x) V^T) J equals V^T J_full W contracted from the full-data
    Jacobian (Eq. (3.12) and the star products of Eqs. (3.15)-(3.23))."""
    prob, wl = small_problem(small_config(n=(6, 6, 5), src=(2, 2), det=(3, 1)))
    rng = np.random.default_rng(2)
    W = np.sign(rng.standard_normal((4, 3)))
    V = np.sign(rng.standard_normal((3, 2)))
    Jf = jacobian(prob, wl.p, np.eye(4), np.eye(3))          # (nf, nd, ns, np)
    Js = jacobian(prob, wl.p, W, V)
    ref = np.einsum("dj,si,fdsk->fjik", V, W, Jf)
    assert np.abs(Js - ref).max() < 1e-11 * np.abs(ref).max()
