"""Pins of the oracle's simultaneous-optimized-direction machinery
(Lemma 3.2, Theorems 3.4-3.7 L648-951, Sec. 3.3.2)."""
import json
import os

import numpy as np
import pytest

from oracle import (add_detectors, add_sources, complement_basis, frob_objective,
                    jacobian, optimize_directions, remove_detectors, remove_sources)
from tests._small import small_config, small_problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1_svd_sizes.json")


def _rand_orth(rng, n, k):
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return Q[:, :k]


def _jfull(rng, nf, nd, ns, n_p):
    return rng.standard_normal((nf, nd, ns, n_p)) + 1j * rng.standard_normal((nf, nd, ns, n_p))


def _sk(Jf, W, V):
    return np.einsum("dj,si,fdsk->fjik", V, W, Jf)


@pytest.mark.parametrize("trial", range(10))
def test_remove_detectors_optimal_and_dominant(trial):
    """Lemma 3.2 certificate: ||(W^T (x) (V Gamma)^T) J||_F^2 = sum of the top
    l_d - s squared singular values, and no random orthonormal Gamma does better."""
    rng = np.random.default_rng(trial)
    nf, nd, ns, n_p, ls, ld, s = 2, 6, 6, 5, 3, 3, 1
    Jf = _jfull(rng, nf, nd, ns, n_p)
    W, V = _rand_orth(rng, ns, ls), _rand_orth(rng, nd, ld)
    Gam, om = remove_detectors(_sk(Jf, W, V), s)
    best = frob_objective(_sk(Jf, W, V @ Gam))
    assert best == pytest.approx(np.sum(om[:ld - s] ** 2), rel=1e-10)
    for _ in range(200):
        cand = frob_objective(_sk(Jf, W, V @ _rand_orth(rng, ld, ld - s)))
        assert cand <= best * (1 + 1e-12)


@pytest.mark.parametrize("trial", range(10))
def test_remove_sources_optimal_and_dominant(trial):
    rng = np.random.default_rng(100 + trial)
    nf, nd, ns, n_p, ls, ld, s = 2, 6, 6, 5, 3, 3, 1
    Jf = _jfull(rng, nf, nd, ns, n_p)
    W, V = _rand_orth(rng, ns, ls), _rand_orth(rng, nd, ld)
    Gam, om = remove_sources(_sk(Jf, W, V), s)
    best = frob_objective(_sk(Jf, W @ Gam, V))
    assert best == pytest.approx(np.sum(om[:ls - s] ** 2), rel=1e-10)
    for _ in range(200):
        assert frob_objective(_sk(Jf, W @ _rand_orth(rng, ls, ls - s), V)) <= best * (1 + 1e-12)


def test_remove_detector_angular_brute_force():
    """l_d = 2 -> 1: the optimum over unit vectors of span(V) found by a 0.01 degree
    sweep equals the theorem's value (independent route)."""
    rng = np.random.default_rng(7)
    Jf = _jfull(rng, 1, 3, 3, 2)
    W, V = _rand_orth(rng, 3, 2), _rand_orth(rng, 3, 2)
    Gam, _ = remove_detectors(_sk(Jf, W, V), 1)
    best = frob_objective(_sk(Jf, W, V @ Gam))
    th = np.deg2rad(np.arange(0, 180, 0.01))
    sweep = max(frob_objective(_sk(Jf, W, V @ np.array([[np.cos(t)], [np.sin(t)]]))) for t in th)
    assert sweep == pytest.approx(best, rel=1e-7)
    assert sweep <= best * (1 + 1e-12)


@pytest.mark.parametrize("trial", range(10))
def test_add_detectors_and_sources_optimal(trial):
    """Theorems 3.6 / 3.7: the added direction lies in the complement and the
    increase equals the top squared singular value of V_c^T [J^_1..J^_ls];
    random unit vectors of the complement never do better."""
    rng = np.random.default_rng(200 + trial)
    nf, nd, ns, n_p, ls, ld = 2, 6, 6, 5, 3, 3
    Jf = _jfull(rng, nf, nd, ns, n_p)
    W, V = _rand_orth(rng, ns, ls), _rand_orth(rng, nd, ld)
    base = frob_objective(_sk(Jf, W, V))
    q, om, _ = add_detectors(_sk(Jf, W, np.eye(nd)), V, 1)
    assert np.abs(V.T @ q).max() < 1e-12 and np.linalg.norm(q) == pytest.approx(1.0)
    gain = frob_objective(_sk(Jf, W, np.concatenate([V, q], 1))) - base
    assert gain == pytest.approx(om[0] ** 2, rel=1e-9)
    Vc = complement_basis(V)
    for _ in range(200):
        c = Vc @ _rand_orth(rng, nd - ld, 1)
        assert frob_objective(_sk(Jf, W, np.concatenate([V, c], 1))) - base <= gain * (1 + 1e-10)
    q, om, _ = add_sources(_sk(Jf, np.eye(ns), V), W, 1)
    assert np.abs(W.T @ q).max() < 1e-12
    gain = frob_objective(_sk(Jf, np.concatenate([W, q], 1), V)) - base
    assert gain == pytest.approx(om[0] ** 2, rel=1e-9)


def test_table1_svd_sizes_golden():
    g = json.load(open(GOLDEN))["rows"]
    rng = np.random.default_rng(0)
    nf, nd, ns, n_p, l, s = 2, 9, 8, 4, 4, 2
    env = dict(n_d=nd, n_s=ns, n_p=n_p, l_s=l, l_d=l, s=s)
    ev = lambda e: eval(e, {}, env)            # noqa: E731  (formulas of Table 1)
    Jf = _jfull(rng, nf, nd, ns, n_p)
    W, V = _rand_orth(rng, ns, l), _rand_orth(rng, nd, l)
    # removal: the SVD operand is the unfolded sketched Jacobian
    nsv = remove_detectors(_sk(Jf, W, V), s)[1].size
    assert nsv == min(ev(g["removing_detectors"][0]), 2 * nf * ev(g["removing_detectors"][1]))
    nsv = remove_sources(_sk(Jf, W, V), s)[1].size
    assert nsv == min(ev(g["removing_sources"][0]), 2 * nf * ev(g["removing_sources"][1]))
    # addition after removing s: l - s columns remain on both sides
    Wr, Vr = W[:, :l - s], V[:, :l - s]
    _, _, shape = add_detectors(_sk(Jf, Wr, np.eye(nd)), Vr, 1)
    assert shape == (ev(g["adding_detectors"][0]), 2 * nf * ev(g["adding_detectors"][1]))
    _, _, shape = add_sources(_sk(Jf, np.eye(ns), Vr), Wr, 1)
    assert shape == (ev(g["adding_sources"][0]), 2 * nf * ev(g["adding_sources"][1]))


def test_optimize_directions_end_to_end():
    """Two-phase replacement on a tiny DOT problem: sizes restored, new columns
    orthogonal to the kept ones with length sqrt(n), every add step increases the
    objective, and the full Jacobian costs n_s + n_d solves per frequency."""
    cfg = small_config(n=(7, 7, 6), src=(3, 2), det=(3, 2), eps=0.4)
    prob, wl = small_problem(cfg, with_data=False)
    rng = np.random.default_rng(3)
    W, V = np.sign(rng.standard_normal((6, 3))), np.sign(rng.standard_normal((6, 3)))
    trace = []
    prob.solves = 0
    Wn, Vn = optimize_directions(prob, wl.p, W, V, 1, trace=trace)
    assert prob.solves == len(cfg.freqs_hz) * (6 + 6)
    assert Wn.shape == W.shape and Vn.shape == V.shape
    assert np.linalg.norm(Wn[:, -1]) == pytest.approx(np.sqrt(6))
    assert np.linalg.norm(Vn[:, -1]) == pytest.approx(np.sqrt(6))
    assert np.abs(Wn[:, :-1].T @ Wn[:, -1]).max() < 1e-10
    assert np.abs(Vn[:, :-1].T @ Vn[:, -1]).max() < 1e-10
    removed = trace[0][3]
    final = frob_objective(jacobian(prob, wl.p, Wn, Vn))
    assert final > removed
    # the kept random subspace is inside the original span
    P = W @ np.linalg.pinv(W)
    assert np.abs(P @ Wn[:, :-1] - Wn[:, :-1]).max() < 1e-10


# ------------------------------------------------ subspace iteration (reading R16)
from oracle import optimize_directions_subspace, subspace_add_direction  # noqa: E402
from oracle.dot_oracle import _real_rows  # noqa: E402


def _xr_detectors(Jf, W):
    """Real unfolding [Re, Im] of (W^T (x) I) J as the n_d x (2 nf ls n_p) matrix of Theorem 3.6."""
    nf, nd = Jf.shape[0], Jf.shape[1]
    J_WI = _sk(Jf, W, np.eye(nd))
    return _real_rows(np.transpose(J_WI, (1, 0, 2, 3)).reshape(nd, -1))


@pytest.mark.parametrize("trial", range(5))
def test_subspace_iteration_converges_to_theorem_3_6(trial):
    rng = np.random.default_rng(100 + trial)
    nf, nd, ns, n_p, ls, ld = 2, 9, 7, 4, 3, 3
    Jf = _jfull(rng, nf, nd, ns, n_p)
    W, V = _rand_orth(rng, ns, ls), _rand_orth(rng, nd, ld)
    q_exact, _, _ = add_detectors(_sk(Jf, W, np.eye(nd)), V, 1)
    q = subspace_add_direction(_xr_detectors(Jf, W), V, rng.standard_normal((nd, 2)), 400)
    assert abs(float(q @ q_exact[:, 0])) > 1 - 1e-10
    assert np.linalg.norm(q) == pytest.approx(1.0)
    assert np.abs(V.T @ q).max() < 1e-12
    assert q[np.argmax(np.abs(q))] > 0


def test_subspace_single_step_is_best_direction_in_start_span():
    """iters = 1 is Rayleigh-Ritz on span(P X0): its direction maximises ||Xr^T q|| over
    that 2-D span -- checked against a brute-force angular sweep."""
    rng = np.random.default_rng(7)
    nf, nd, ns, n_p, ls, ld = 1, 8, 6, 3, 2, 3
    Jf = _jfull(rng, nf, nd, ns, n_p)
    W, V = _rand_orth(rng, ns, ls), _rand_orth(rng, nd, ld)
    Xr = _xr_detectors(Jf, W)
    X0 = rng.standard_normal((nd, 2))
    q = subspace_add_direction(Xr, V, X0, 1)
    Pm = np.eye(nd) - V @ V.T
    B, _ = np.linalg.qr(Pm @ X0)
    th = np.linspace(0, np.pi, 20001)
    cand = B @ np.stack([np.cos(th), np.sin(th)])
    vals = np.sum((Xr.T @ cand) ** 2, axis=0)
    best = float(np.sum((Xr.T @ q) ** 2))
    assert best >= vals.max() * (1 - 1e-12)
    assert best <= vals.max() * (1 + 1e-6)


def test_subspace_objective_grows_with_iterations():
    rng = np.random.default_rng(11)
    nf, nd, ns, n_p, ls, ld = 2, 12, 5, 3, 2, 4
    Jf = _jfull(rng, nf, nd, ns, n_p)
    W, V = _rand_orth(rng, ns, ls), _rand_orth(rng, nd, ld)
    Xr = _xr_detectors(Jf, W)
    X0 = rng.standard_normal((nd, 2))
    q_exact, _, _ = add_detectors(_sk(Jf, W, np.eye(nd)), V, 1)
    top = float(np.sum((Xr.T @ q_exact[:, 0]) ** 2))
    vals = [float(np.sum((Xr.T @ subspace_add_direction(Xr, V, X0, it)) ** 2)) for it in (1, 2, 5, 50)]
    assert all(v <= top * (1 + 1e-12) for v in vals)
    assert vals[-1] == pytest.approx(top, rel=1e-9)
    assert vals[0] <= vals[2] + 1e-12 * top


def test_optimize_directions_subspace_matches_exact_when_converged():
    cfg = small_config(n=(7, 7, 6), src=(3, 2), det=(3, 2), eps=0.4)
    prob, wl = small_problem(cfg, with_data=False)
    rng = np.random.default_rng(3)
    W, V = np.sign(rng.standard_normal((6, 3))), np.sign(rng.standard_normal((6, 3)))
    X0s, X0d = rng.standard_normal((6, 2)), rng.standard_normal((6, 2))   # s = 1: one block of 2
    We, Ve = optimize_directions(prob, wl.p, W, V, 1)
    Ws, Vs = optimize_directions_subspace(prob, wl.p, W, V, 1, 300, X0s, X0d)
    # kept columns identical (same remove steps); new columns equal up to sign
    assert np.abs(Ws[:, :-1] - We[:, :-1]).max() < 1e-9
    assert abs(float(Ws[:, -1] @ We[:, -1])) / 6 > 1 - 1e-8
    assert abs(float(Vs[:, -1] @ Ve[:, -1])) / 6 > 1 - 1e-8
    o5 = frob_objective(jacobian(prob, wl.p, *optimize_directions_subspace(prob, wl.p, W, V, 1, 5, X0s, X0d)))
    oe = frob_objective(jacobian(prob, wl.p, We, Ve))
    assert o5 <= oe * (1 + 1e-9)
