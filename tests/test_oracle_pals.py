"""Pins of the oracle's PaLS absorption model (Eqs. (2.3)-(2.4);
DESIGN.md readings R7-R9) against closed forms and finite differences."""
import numpy as np
import pytest

from oracle import (absorption, dmu_dp, heaviside, heaviside_d, jacobian_weights, make_grid,
                    pals_phi, wendland, wendland_d)
from synth import config_by_name, draw_params


def test_wendland_closed_forms():
    assert wendland(0.0) == 1.0 and wendland_d(0.0) == 0.0
    assert wendland(0.5) == pytest.approx(0.1875, abs=1e-15)      # (1/2)^4 * 3
    assert wendland_d(0.5) == pytest.approx(-1.25, abs=1e-15)     # -20 * 0.5 * (1/2)^3
    assert wendland(1.0) == 0.0 and wendland(2.0) == 0.0 and wendland_d(1.5) == 0.0
    # sqrt(0.37): (1 - r)^4 (4 r + 1) evaluated by hand to 12 digits
    assert wendland(np.sqrt(0.37)) == pytest.approx(0.0808363485798, rel=1e-11)


def test_wendland_derivative_and_c2_smoothness():
    r = np.linspace(0.01, 1.3, 500)
    h = 1e-6
    fd = (wendland(r + h) - wendland(r - h)) / (2 * h)
    assert np.abs(fd - wendland_d(r)).max() < 1e-8
    # C2 at the support edge: psi, psi', psi'' -> 0 as r -> 1-
    d2 = (wendland_d(1 - 1e-4) - wendland_d(1 - 2e-4)) / 1e-4
    assert abs(wendland(1 - 1e-4)) < 1e-14 and abs(wendland_d(1 - 1e-4)) < 1e-9 and abs(d2) < 1e-5


def test_heaviside_closed_forms():
    eps = 0.1
    assert heaviside(0.0, eps) == 0.5
    assert heaviside(eps, eps) == pytest.approx(1.0, abs=1e-15)
    assert heaviside(-eps, eps) == pytest.approx(0.0, abs=1e-15)
    assert heaviside(0.3, eps) == 1.0 and heaviside(-0.3, eps) == 0.0
    assert heaviside_d(0.0, eps) == pytest.approx(1.0 / eps)
    # H' integrates to one over its support (trapezoid, fine grid)
    t = np.linspace(-eps, eps, 200001)
    assert np.trapezoid(heaviside_d(t, eps), t) == pytest.approx(1.0, abs=1e-9)
    # derivative matches central differences, monotone
    t = np.linspace(-0.2, 0.2, 801)
    fd = (heaviside(t + 1e-7, eps) - heaviside(t - 1e-7, eps)) / 2e-7
    assert np.abs(fd - heaviside_d(t, eps)).max() < 1e-5
    assert np.all(np.diff(heaviside(t, eps)) >= -1e-15)


def test_pals_phi_special_cases():
    g = make_grid((5, 5, 5), (2.0, 2.0, 2.0))
    node = (2 * 5 + 2) * 5 + 2
    chi = (g.X[node], g.Y[node], g.Z[node])
    p = np.array([0.7, 1.3, *chi])
    phi = pals_phi(p, g, 0.01)
    assert phi[node] == pytest.approx(0.7 * wendland(0.01), rel=1e-15)   # norm reduces to gamma
    assert np.all(pals_phi(np.array([0.0, 1.3, *chi]), g, 0.01) == 0.0)  # alpha = 0
    # compact support: a basis far away changes nothing (exact)
    far = np.array([0.9, 2.0, 50.0, 50.0, 50.0])
    assert np.array_equal(pals_phi(np.concatenate([p, far]), g, 0.01), phi)


def test_absorption_range_and_midpoint():
    cfg = config_by_name("tiny16")
    g = make_grid(cfg.n, cfg.L)
    p = draw_params(np.random.default_rng(5), 6, cfg.L, 0.5, 1.0)
    mu = absorption(p, g, cfg)
    assert mu.min() >= cfg.mua_bg and mu.max() <= cfg.mua_anom
    assert (mu > cfg.mua_bg).any()


def test_absorption_orientation_and_midpoint():
    """Eq. (2.4) / PAPER.md L153-155: mu = mu_in where phi - c > eps (inside the anomaly),
    mu_out where phi - c < -eps, and (mu_in + mu_out)/2 where phi = c exactly (H_eps(0) = 1/2).
    One basis centred on a node with alpha chosen so that phi(node) = c: the node sits on the
    level set; nodes beyond the basis's support read mu_out."""
    cfg = config_by_name("tiny16")
    g = make_grid(cfg.n, cfg.L)
    node = 5 * 16 * 16 + 7 * 16 + 6
    chi = (g.X[node], g.Y[node], g.Z[node])
    beta = 1.0
    alpha_mid = cfg.cutoff / wendland(cfg.gamma)           # phi(node) = alpha psi(gamma) = c
    mu = absorption(np.array([alpha_mid, beta, *chi]), g, cfg)
    assert mu[node] == pytest.approx(0.5 * (cfg.mua_anom + cfg.mua_bg), rel=1e-12)
    far = np.sqrt((g.X - chi[0]) ** 2 + (g.Y - chi[1]) ** 2 + (g.Z - chi[2]) ** 2) > 1.0 / beta
    assert np.all(mu[far] == cfg.mua_bg)                     # outside: mu_out
    mu_in = absorption(np.array([1.0, beta, *chi]), g, cfg)  # phi(node) = psi(gamma) ~ 1 >> c + eps
    assert mu_in[node] == cfg.mua_anom                       # inside: mu_in (orientation)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_dmu_dp_matches_central_differences(seed):
    cfg = config_by_name("tiny16").with_(eps=0.4, n=(10, 10, 10))
    g = make_grid(cfg.n, cfg.L)
    p = draw_params(np.random.default_rng(seed), 3, cfg.L, 0.4, 1.0)
    G = dmu_dp(p, g, cfg)
    assert (np.abs(G) > 0).sum() > 50
    h = 1e-6
    for k in range(p.size):
        e = np.zeros_like(p)
        e[k] = h
        fd = (absorption(p + e, g, cfg) - absorption(p - e, g, cfg)) / (2 * h)
        scale = np.abs(G[:, k]).max() + 1e-300
        assert np.abs(fd - G[:, k]).max() <= 1e-5 * scale, k


def test_jacobian_weights_carry_theta():
    cfg = config_by_name("tiny16").with_(eps=0.4)
    g = make_grid(cfg.n, cfg.L)
    p = draw_params(np.random.default_rng(1), 3, cfg.L, 0.4, 1.0)
    Gw = jacobian_weights(p, g, cfg)
    assert np.array_equal(Gw, g.theta[:, None] * dmu_dp(p, g, cfg))
