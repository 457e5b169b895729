"""Oracle parity at full BASELINE.json sizes: configs[2] (`full64`: 64^3, 256 sources x 256
detectors, 3 frequencies, 80 parameters -- the configuration the bench metric is quoted on)
and configs[1] (`sketch32`: 32^3, 64 x 64, 3 frequencies, 40 parameters).

tests/golden/<config>_oracle.npz is written by tools/golden.py, which calls only
oracle/ (scipy splu in complex128, ~1 h of CPU at 64^3): the oracle's data D (hidden level set +
1% noise), measurements M_f = C^T A(omega_f, p)^-1 B at the iterate p (PAPER.md L181-185,
Eq. (2.5)), the full-data and sketched misfits (L365, Eq. (EsTResidual)) and the sketched
Jacobian (W^T (x) V^T) J (L966-972).  The GPU runs the bench's launch configuration
(all 1536 systems of a step as 512 real seeds in one batch) on the same seeded inputs.
Bar (north_star): measurements and misfit within 1e-8 relative, J within 1e-7 relative
Frobenius."""
import os

import numpy as np
import pytest

from synth import config_by_name, make_workload

CONFIGS = ["full64", "sketch32"]


def golden(name):
    return os.path.join(os.path.dirname(__file__), "golden", f"{name}_oracle.npz")


@pytest.mark.parametrize("name", CONFIGS)
def test_golden_is_self_consistent(name):
    """The stored misfits are those of the stored measurements and data (CPU; ties the
    golden arrays to each other: ||M_f - D_f||_F^2 and ||V^T (M_f - D_f) W||_F^2)."""
    z = np.load(golden(name))
    cfg = config_by_name(name)
    wl = make_workload(cfg)
    R = z["M"] - z["data"]
    mii = np.sum(np.abs(R) ** 2, axis=(1, 2))
    mwv = np.array([np.sum(np.abs(wl.V.T @ R[f] @ wl.W) ** 2) for f in range(R.shape[0])])
    assert np.allclose(mii, z["misfit_II"], rtol=1e-10)
    assert np.allclose(mwv, z["misfit_WV"], rtol=1e-10)
    assert z["M"].shape == (cfg.n_freq, cfg.n_d, cfg.n_s)
    assert z["J_WV"].shape == (cfg.n_freq, cfg.ld, cfg.ls, cfg.n_p)


@pytest.fixture(scope="module", params=CONFIGS)
def full64(request):
    from paper_1706_05586_b200 import build
    build.build()
    import paper_1706_05586_b200 as dot
    z = np.load(golden(request.param))
    cfg = config_by_name(request.param)
    wl = make_workload(cfg)
    g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
    g.set_data(z["data"])
    g.set_params(wl.p)
    J = g.jacobian(None, None)               # full64: the bench step's batch, 512 seeds -> 1536 systems
    return dict(g=g, z=z, wl=wl, cfg=cfg, J=J)


@pytest.mark.gpu
def test_measurements_match_oracle(full64):
    g, z, wl = full64["g"], full64["z"], full64["wl"]
    X = g.solve_sampled(0)                                   # cached forward fields [f][s][P]
    samp = g.samples()
    M = np.transpose(X[:, :, np.searchsorted(samp, wl.det_nodes)], (0, 2, 1))   # [f][d][s]
    Mo = z["M"]
    for f in range(Mo.shape[0]):
        err = np.abs(M[f] - Mo[f]).max() / np.abs(Mo[f]).max()
        fro = np.linalg.norm(M[f] - Mo[f]) / np.linalg.norm(Mo[f])
        assert err <= 1e-8 and fro <= 1e-8, (f, err, fro)


@pytest.mark.gpu
def test_adjoint_measurements_match_oracle(full64):
    """The adjoint (detector) fields of the same batch give M^T at the sources (A = A^T)."""
    g, z, wl, cfg = full64["g"], full64["z"], full64["wl"], full64["cfg"]
    Y = g.solve_sampled(1)                                   # [f][d][P]
    samp = g.samples()
    h = (cfg.L[0] / (cfg.n[0] + 1)) * (cfg.L[1] / (cfg.n[1] + 1)) * (cfg.L[2] / (cfg.n[2] - 1))
    Ma = Y[:, :, np.searchsorted(samp, wl.src_nodes)] * (0.5 / h)   # b_s = theta e_s / (hx hy hz), theta = 1/2
    fro = np.linalg.norm(Ma - z["M"]) / np.linalg.norm(z["M"])
    assert fro <= 1e-8, fro


@pytest.mark.gpu
def test_misfits_match_oracle(full64):
    g, z, wl = full64["g"], full64["z"], full64["wl"]
    m_ii = g.misfit(None, None)
    m_wv = g.misfit(wl.W, wl.V)
    assert abs(m_ii - z["misfit_II"].sum()) <= 1e-8 * z["misfit_II"].sum()
    assert abs(m_wv - z["misfit_WV"].sum()) <= 1e-8 * z["misfit_WV"].sum()


@pytest.mark.gpu
def test_sketched_jacobian_matches_oracle(full64):
    g, z, wl = full64["g"], full64["z"], full64["wl"]
    J = g.jacobian(wl.W, wl.V)
    Jo = z["J_WV"]
    assert np.linalg.norm(J - Jo) <= 1e-7 * np.linalg.norm(Jo)
    # and as the W, V combination of the full Jacobian of the bench step
    ref = np.einsum("sl,dm,fdsk->fmlk", wl.W, wl.V, full64["J"])
    assert np.linalg.norm(ref - Jo) <= 1e-7 * np.linalg.norm(Jo)
