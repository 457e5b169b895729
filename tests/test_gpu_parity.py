"""GPU parity of the sm_100a path (through the C-ABI) against the CPU oracle on
the same seeded inputs.  Tolerances (BASELINE north_star): measurements and
misfit 1e-8 relative, Jacobian 1e-7 relative Frobenius; mu, G, A u at rounding
level (1e-12)."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import (absorption, assemble, jacobian, jacobian_weights, make_grid, measurements, misfit,
                    sketched_residual)
from tests._small import small_config, small_problem

pytestmark = pytest.mark.gpu

# grids chosen to exercise one tile, several tiles and a ragged last tile
GRIDS = [
    dict(n=(8, 8, 7), L=(3.0, 3.0, 2.5)),
    dict(n=(16, 16, 16), L=(4.0, 4.0, 4.0)),
    dict(n=(64, 37, 6), L=(8.0, 5.0, 2.0), src=(4, 2), det=(3, 3)),
    dict(n=(33, 21, 9), L=(4.0, 3.0, 2.0), src=(3, 2), det=(2, 3)),
    # geometries of the compile-time specialised pass kernels (nx=64/TY=16, nx=32/TY=32)
    dict(n=(64, 64, 5), L=(8.0, 8.0, 1.0), src=(4, 4), det=(4, 4)),
    dict(n=(32, 32, 6), L=(4.0, 4.0, 1.5), src=(4, 2), det=(2, 4)),
]


@pytest.fixture(scope="module")
def dot():
    from paper_1706_05586_b200 import build
    build.build()
    import paper_1706_05586_b200 as d
    return d


def gpu_problem(dot, cfg, prob, wl, **kw):
    g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes, **kw)
    if prob.data is not None:
        g.set_data(prob.data)
    g.set_params(wl.p)
    return g


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_absorption_support_and_weights(dot, gi):
    cfg = small_config(**GRIDS[gi], eps=0.3)
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    mu_ref = absorption(wl.p, prob.grid, cfg)
    assert np.abs(g.absorption() - mu_ref).max() <= 1e-13 * mu_ref.max()
    Gref = jacobian_weights(wl.p, prob.grid, cfg)
    nodes, G = g.support()
    ref_nodes = np.nonzero(np.abs(Gref).sum(1) > 0)[0]
    # membership is decided by dH/dphi != 0 on both sides in fp64: nodes may only
    # differ where the weight is at rounding level (|phi - c| == eps)
    diff = np.setxor1d(nodes, ref_nodes)
    assert np.all(np.abs(Gref[diff]).max(initial=0.0) < 1e-12 * np.abs(Gref).max())
    common, ia, ib = np.intersect1d(nodes, ref_nodes, return_indices=True)
    assert len(common) > 0
    assert np.abs(G[ia] - Gref[common]).max() <= 1e-12 * np.abs(Gref).max()
    assert np.all(np.diff(nodes) > 0)
    samp = g.samples()
    assert set(wl.det_nodes) <= set(samp) and set(wl.src_nodes) <= set(samp) and set(nodes) <= set(samp)


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_apply_matches_oracle_operator(dot, gi):
    cfg = small_config(**GRIDS[gi])
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    rng = np.random.default_rng(gi)
    u = rng.standard_normal((3, prob.grid.N)) + 1j * rng.standard_normal((3, prob.grid.N))
    mu = absorption(wl.p, prob.grid, cfg)
    for f in range(len(prob.omegas)):
        A = prob.operator(mu, f)
        Au = g.apply(f, u)
        ref = (A @ u.T).T
        assert np.abs(Au - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_dense_solve_matches_sparse_lu(dot, gi):
    cfg = small_config(**GRIDS[gi])
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    N = prob.grid.N
    rng = np.random.default_rng(10 + gi)
    b = rng.standard_normal((2, N)) + 1j * rng.standard_normal((2, N))
    pt = np.zeros((1, N), complex)
    pt[0, wl.src_nodes[0]] = 1.0
    b = np.concatenate([b, pt])
    mu = absorption(wl.p, prob.grid, cfg)
    for f in range(len(prob.omegas)):
        x, iters = g.solve(b, f)
        lu = spla.splu(prob.operator(mu, f).tocsc())
        ref = lu.solve(b.T).T
        for r in range(b.shape[0]):
            assert rel(x[r], ref[r]) < 1e-11, (f, r)
        assert np.all(iters > 0)


def test_zero_rhs_gives_zero(dot):
    cfg = small_config(**GRIDS[0])
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    x, iters = g.solve(np.zeros((2, prob.grid.N), complex), 0)
    assert np.all(x == 0) and np.all(iters == 0)


@pytest.mark.parametrize("gi", range(len(GRIDS)))
@pytest.mark.parametrize("sketch", ["identity", "rademacher"])
def test_misfit_and_residual_parity(dot, gi, sketch):
    cfg = small_config(**GRIDS[gi])
    prob, wl = small_problem(cfg)
    g = gpu_problem(dot, cfg, prob, wl)
    ns, nd = len(wl.src_nodes), len(wl.det_nodes)
    if sketch == "identity":
        W = V = None
        Wm, Vm = np.eye(ns), np.eye(nd)
    else:
        rng = np.random.default_rng(gi)
        Wm = np.sign(rng.standard_normal((ns, 3)))
        Vm = np.sign(rng.standard_normal((nd, 2)))
        W, V = Wm, Vm
    m, S = g.misfit(W, V, return_resid=True)
    Sref = sketched_residual(prob, wl.p, Wm, Vm)
    mref = float(np.sum(np.abs(Sref) ** 2))
    assert abs(m - mref) <= 1e-8 * mref
    assert np.abs(S - Sref).max() <= 1e-8 * np.abs(Sref).max()


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_measurements_parity(dot, gi):
    """C^T A^-1 B (Eq. (2.5)) sampled at the detectors, all frequencies."""
    cfg = small_config(**GRIDS[gi])
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    X = g.solve_sampled(0)                 # [nf][ns][nP]
    samp = g.samples()
    det_slot = np.searchsorted(samp, wl.det_nodes)
    M = np.transpose(X[:, :, det_slot], (0, 2, 1))
    Mref = measurements(prob, wl.p)
    assert rel(M, Mref) < 1e-8


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_jacobian_parity(dot, gi):
    cfg = small_config(**GRIDS[gi], eps=0.4)
    prob, wl = small_problem(cfg)
    g = gpu_problem(dot, cfg, prob, wl)
    rng = np.random.default_rng(20 + gi)
    ns, nd = len(wl.src_nodes), len(wl.det_nodes)
    W = np.sign(rng.standard_normal((ns, 3)))
    V = np.sign(rng.standard_normal((nd, 2)))
    g.misfit(W, V)
    J = g.jacobian(W, V)
    Jref = jacobian(prob, wl.p, W, V)
    assert np.linalg.norm(Jref) > 0
    assert rel(J, Jref) < 1e-7
    Jf = g.jacobian(None, None)
    Jfref = jacobian(prob, wl.p, np.eye(ns), np.eye(nd))
    assert rel(Jf, Jfref) < 1e-7


def test_reciprocity_forward_vs_adjoint(dot):
    """c_d^T A^-1 b_s from forward solves equals (A^-T c_d)^T b_s from adjoint
    solves (property of the complex-symmetric operator, any size)."""
    cfg = small_config(**GRIDS[2])
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    samp = g.samples()
    Xs = g.solve_sampled(0)
    Xd = g.solve_sampled(1)
    M_fwd = Xs[:, :, np.searchsorted(samp, wl.det_nodes)]            # [f][s][d]
    scale = prob.grid.theta[wl.src_nodes] / prob.grid.cell_volume
    M_adj = Xd[:, :, np.searchsorted(samp, wl.src_nodes)] * scale     # [f][d][s]
    assert rel(M_fwd, np.transpose(M_adj, (0, 2, 1))) < 1e-9


def test_contract_kernel_against_direct_sums(dot):
    """Stateless DMMA contraction on seeded random panels, ragged sizes."""
    import torch
    rng = np.random.default_rng(5)
    for (nb, K, ld, ls, n_p) in [(1, 1, 1, 1, 1), (2, 37, 3, 5, 20), (3, 300, 12, 12, 80), (1, 17, 33, 7, 45)]:
        Lam = rng.standard_normal((nb, ld, K)) + 1j * rng.standard_normal((nb, ld, K))
        U = rng.standard_normal((nb, ls, K)) + 1j * rng.standard_normal((nb, ls, K))
        G = rng.standard_normal((K, n_p))
        J = dot.contract(torch.as_tensor(Lam, device="cuda"), torch.as_tensor(U, device="cuda"),
                         torch.as_tensor(G, device="cuda")).cpu().numpy()
        ref = -np.einsum("bjs,bis,sk->bjik", Lam, U, G)
        assert rel(J, ref) < 1e-13


def test_solve_accounting_reproduces_table4(dot):
    """PAPER.md Table 4 arithmetic (tests/golden/table1_svd_sizes.json "table4_pde_solves",
    cited there) with the library's solve counter: SAA with l = 10 for F = 10 function and
    J = 5 Jacobian evaluations costs F*l + J*l = 150 solves (forward fields are reused by the
    Jacobian); one optimized-direction replacement event adds n_s + n_d = 64 (32 sources,
    32 detectors, one frequency) -- the "Replacing" rows' full_jacobian_events term."""
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_svd_sizes.json")))
    saa = gold["table4_pde_solves"]["rows"][0]
    F, Jn, l = saa["F"], saa["J"], saa["l"]
    cfg = small_config(n=(32, 16, 6), L=(8.0, 4.0, 2.0), src=(8, 4), det=(8, 4), freqs=(0.0,), eps=0.4)
    prob, wl = small_problem(cfg)
    g = gpu_problem(dot, cfg, prob, wl)
    g.reset_stats()
    rng = np.random.default_rng(0)
    W = np.sign(rng.standard_normal((32, l)))
    V = np.sign(rng.standard_normal((32, l)))
    for it in range(F):
        g.set_params(wl.p * (1 + 1e-3 * it))
        g.misfit(W, V)
        if it % (F // Jn) == 0:
            g.jacobian(W, V)
    assert g.stats()["rhs_solved"] == F * l + Jn * l == saa["total"]
    g.optimize_directions(1, W, V)
    # each replacement event costs the full-data solves n_s + n_d (per frequency)
    for row in gold["table4_pde_solves"]["rows"][1:3]:
        assert row["total"] == (row["F"] + row["J"]) * row["l"] + row["full_jacobian_events"] * 64
    assert g.stats()["rhs_solved"] == saa["total"] + 64


def test_optimize_directions_parity(dot):
    from oracle import frob_objective, optimize_directions
    cfg = small_config(n=(12, 12, 8), L=(4.0, 4.0, 3.0), src=(3, 3), det=(3, 2), eps=0.5)
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    rng = np.random.default_rng(8)
    W = np.sign(rng.standard_normal((9, 4)))
    V = np.sign(rng.standard_normal((6, 3)))
    for k in (1, 2):
        Wg, Vg, obj = g.optimize_directions(k, W, V)
        Wr, Vr = optimize_directions(prob, wl.p, W, V, k)
        objr = frob_objective(jacobian(prob, wl.p, Wr, Vr))
        assert abs(obj - objr) <= 1e-7 * objr
        # same subspaces (columns are unique up to sign / rotation)
        for A, B in ((Wg, Wr), (Vg, Vr)):
            Qa, _ = np.linalg.qr(A)
            Qb, _ = np.linalg.qr(B)
            assert np.abs(Qa @ Qa.T - Qb @ Qb.T).max() < 1e-6
        assert np.allclose(np.linalg.norm(Wg[:, -1]), 3.0)


@pytest.mark.parametrize("iters,block", [(1, 2), (5, 2), (3, 1)])
def test_optimize_directions_subspace_parity(dot, iters, block):
    """Matrix-free subspace-iteration replacement (reading R16) against the oracle's
    explicit subspace iteration: same W, V, starting blocks and iteration count."""
    from oracle import frob_objective, optimize_directions_subspace
    cfg = small_config(n=(12, 12, 8), L=(4.0, 4.0, 3.0), src=(4, 3), det=(3, 3), eps=0.5)
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    rng = np.random.default_rng(21)
    ns, nd = 12, 9
    W = np.sign(rng.standard_normal((ns, 4)))
    V = np.sign(rng.standard_normal((nd, 3)))
    X0s_all, X0d_all = rng.standard_normal((ns, 2 * block)), rng.standard_normal((nd, 2 * block))
    for k in (1, 2):
        X0s, X0d = X0s_all[:, :k * block], X0d_all[:, :k * block]
        g.reset_stats()
        Wg, Vg, obj = g.optimize_directions_subspace(k, W, V, X0s, X0d, iters=iters)
        st = g.stats()
        Wr, Vr = optimize_directions_subspace(prob, wl.p, W, V, k, iters, X0s, X0d)
        objr = frob_objective(jacobian(prob, wl.p, Wr, Vr))
        assert abs(obj - objr) <= 1e-7 * objr
        # removed-and-kept columns span the same space; added columns match exactly (sign rule)
        for A, B in ((Wg, Wr), (Vg, Vr)):
            Qa, _ = np.linalg.qr(A[:, :-k])
            Qb, _ = np.linalg.qr(B[:, :-k])
            assert np.abs(Qa @ Qa.T - Qb @ Qb.T).max() < 1e-7
            assert np.abs(A[:, -k:] - B[:, -k:]).max() <= 1e-6 * np.abs(B[:, -k:]).max()
        # solve accounting: W and V fields once, then 2 solves per block vector per step per frequency
        nf = len(cfg.freqs_hz)
        assert st["rhs_solved"] == nf * (4 + 3) + 2 * k * iters * 2 * block * nf
        # the optimized W, V leave their fields (kept by combination, added from the last
        # block's solves) in the caches: J(W_hat, V_hat) needs no solves and matches the oracle
        g.reset_stats()
        J2 = g.jacobian(Wg, Vg)
        assert g.stats()["rhs_solved"] == 0
        assert rel(J2, jacobian(prob, wl.p, Wg, Vg)) < 1e-7
    # starting fields from the caches: after J(W, V) the subspace step solves only its blocks
    g.jacobian(W, V)
    g.reset_stats()
    g.optimize_directions_subspace(1, W, V, X0s_all[:, :block], X0d_all[:, :block], iters=iters)
    assert g.stats()["rhs_solved"] == 2 * iters * 2 * block * len(cfg.freqs_hz)


def test_optimize_directions_subspace_converges_to_exact(dot):
    cfg = small_config(n=(12, 12, 8), L=(4.0, 4.0, 3.0), src=(4, 3), det=(3, 3), eps=0.5)
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    rng = np.random.default_rng(5)
    W = np.sign(rng.standard_normal((12, 4)))
    V = np.sign(rng.standard_normal((9, 3)))
    We, Ve, oe = g.optimize_directions(1, W, V)
    Ws, Vs, os_ = g.optimize_directions_subspace(1, W, V, rng.standard_normal((12, 2)), rng.standard_normal((9, 2)),
                                                 iters=60)
    assert abs(os_ - oe) <= 1e-8 * oe
    assert abs(float(Ws[:, -1] @ We[:, -1])) / 12 > 1 - 1e-8


@pytest.mark.parametrize("knobs", [dict(DOT_CG_ZCHUNKS="1"), dict(DOT_CG_ZCHUNKS="2"),
                                   dict(DOT_CG_ZCHUNKS="3"), dict(DOT_CG_ZCHUNKS="4"),
                                   dict(DOT_CG_ZCHUNKS="3", DOT_CG_ROWS="1"),
                                   dict(DOT_CG_ZCHUNKS="4", DOT_CG_ROWS="2", DOT_CG_TY="5")])
def test_z_chunks_keep_parity(dot, knobs, monkeypatch):
    """z-chunked passes (each chunk recomputes 2 halo planes of p and 1 of r_{k+1},
    DESIGN.md "z chunks") solve the same systems: nz = 19 splits into 10+9, 7+7+5, 5+5+5+4."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    cfg = small_config(n=(24, 20, 19), L=(4.0, 3.5, 3.0), src=(3, 2), det=(2, 3), eps=0.4)
    prob, wl = small_problem(cfg, with_data=True)
    g = gpu_problem(dot, cfg, prob, wl)
    N = prob.grid.N
    rng = np.random.default_rng(4)
    b = rng.standard_normal((2, N)) + 1j * rng.standard_normal((2, N))
    mu = absorption(wl.p, prob.grid, cfg)
    x, _ = g.solve(b, 1)
    ref = spla.splu(prob.operator(mu, 1).tocsc()).solve(b.T).T
    assert rel(x, ref) < 1e-11
    X = g.solve_sampled(0)
    samp = g.samples()
    M = np.transpose(X[:, :, np.searchsorted(samp, wl.det_nodes)], (0, 2, 1))
    assert rel(M, measurements(prob, wl.p)) < 1e-8
    J = g.jacobian(None, None)
    assert rel(J, jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))) < 1e-7


KNOBS = [dict(DOT_CG_ROWS="1"), dict(DOT_CG_ROWS="2"),
         dict(DOT_CG_PREFETCH="1"), dict(DOT_CG_PREFETCH="3"), dict(DOT_CG_TY="3"), dict(DOT_CG_TY="5"),
         dict(DOT_CG_ROWS="1", DOT_CG_TY="4"), dict(DOT_CG_ROWS="2", DOT_CG_TY="3", DOT_CG_PREFETCH="1"),
         ]


@pytest.mark.parametrize("knobs", KNOBS)
def test_tiling_knobs_keep_parity(dot, knobs, monkeypatch):
    """Every tiling the run-time knobs can select solves the same systems
    (guards the generic kernel instance and the tiling constraints)."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    cfg = small_config(**GRIDS[4])
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    N = prob.grid.N
    rng = np.random.default_rng(3)
    b = rng.standard_normal((2, N)) + 1j * rng.standard_normal((2, N))
    mu = absorption(wl.p, prob.grid, cfg)
    x, _ = g.solve(b, 1)
    ref = spla.splu(prob.operator(mu, 1).tocsc()).solve(b.T).T
    assert rel(x, ref) < 1e-11
    X = g.solve_sampled(0)
    samp = g.samples()
    M = np.transpose(X[:, :, np.searchsorted(samp, wl.det_nodes)], (0, 2, 1))
    assert rel(M, measurements(prob, wl.p)) < 1e-8


def test_prefetch_fields_one_batch_then_cached(dot):
    """dot_prefetch_fields solves B W and C V together; misfit / jacobian /
    fields_on_support then run without solves and match the oracle."""
    from oracle import misfit as omisfit
    cfg = small_config(**GRIDS[3])
    prob, wl = small_problem(cfg)
    g = gpu_problem(dot, cfg, prob, wl)
    rng = np.random.default_rng(2)
    W = np.sign(rng.standard_normal((cfg.n_s, 3)))
    V = np.sign(rng.standard_normal((cfg.n_d, 2)))
    g.reset_stats()
    g.prefetch_fields(W, V)
    nf = len(cfg.freqs_hz)
    assert g.stats()["rhs_solved"] == nf * 5
    m = g.misfit(W, V)
    J = g.jacobian(W, V)
    g.fields_on_support(1, V)
    assert g.stats()["rhs_solved"] == nf * 5
    assert abs(m - omisfit(prob, wl.p, W, V)) <= 1e-8 * m
    assert rel(J, jacobian(prob, wl.p, W, V)) < 1e-7


@pytest.mark.parametrize("seed", range(16))
def test_random_geometries_and_tilings(dot, seed, monkeypatch):
    """Seeded random grids (odd / even / tiny extents, ragged tiles and chunks) under a
    random z-pass tiling option: dense solves and sampled measurements vs the oracle."""
    rng = np.random.default_rng(1000 + seed)
    nx, ny, nz = int(rng.integers(3, 40)), int(rng.integers(3, 40)), int(rng.integers(2, 30))
    opt = ["1", "2"][seed % 2]
    monkeypatch.setenv("DOT_CG_ROWS", opt)
    if seed % 3 == 0 and nz >= 8:
        monkeypatch.setenv("DOT_CG_ZCHUNKS", str(int(rng.integers(2, 5))))
    L = (float(rng.uniform(1.5, 4.0)), float(rng.uniform(1.5, 4.0)), float(rng.uniform(1.0, 3.0)))
    src = (min(2, nx), min(2, ny))
    det = (min(2, nx), min(3, ny))
    cfg = small_config(n=(nx, ny, nz), L=L, src=src, det=det, eps=0.5, seed=seed)
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    N = prob.grid.N
    b = rng.standard_normal((2, N)) + 1j * rng.standard_normal((2, N))
    mu = absorption(wl.p, prob.grid, cfg)
    for f in range(len(prob.omegas)):
        x, _ = g.solve(b, f)
        ref = spla.splu(prob.operator(mu, f).tocsc()).solve(b.T).T
        assert rel(x, ref) < 1e-11, (nx, ny, nz, opt, f)
    X = g.solve_sampled(0)
    samp = g.samples()
    M = np.transpose(X[:, :, np.searchsorted(samp, wl.det_nodes)], (0, 2, 1))
    assert rel(M, measurements(prob, wl.p)) < 1e-8, (nx, ny, nz, opt)


def test_block_sparse_contraction_equals_dense(dot, monkeypatch):
    """The block-sparse Jacobian contraction (per basis over its own support points,
    PAPER.md L972) equals the dense K x n_p contraction and the oracle."""
    cfg = small_config(n=(20, 18, 12), L=(4.0, 3.5, 3.0), src=(3, 2), det=(2, 3), n_rbf=5, eps=0.5)
    prob, wl = small_problem(cfg)
    rng = np.random.default_rng(6)
    W = np.sign(rng.standard_normal((cfg.n_s, 3)))
    V = np.sign(rng.standard_normal((cfg.n_d, 4)))
    g = gpu_problem(dot, cfg, prob, wl)
    g.reset_stats()
    Js = g.jacobian(W, V)
    st = g.stats()
    assert st["contract_flops"] < st["contract_flops_dense"]     # the sparse kernel ran
    monkeypatch.setenv("DOT_CONTRACT", "dense")
    gd = gpu_problem(dot, cfg, prob, wl)
    gd.reset_stats()
    Jd = gd.jacobian(W, V)
    std = gd.stats()
    assert std["contract_flops"] == std["contract_flops_dense"]
    assert rel(Js, Jd) < 1e-12
    assert rel(Js, jacobian(prob, wl.p, W, V)) < 1e-7


def test_block_sparse_gemm_contraction_equals_dense(dot, monkeypatch):
    """Large panels (ld >= 32, ls >= 8) take the per-(frequency, basis) complex GEMM
    form of the block-sparse contraction: equal to the dense kernel and the oracle."""
    cfg = small_config(n=(24, 20, 10), L=(4.0, 3.5, 2.5), src=(3, 3), det=(8, 5), n_rbf=5, eps=0.5)
    prob, wl = small_problem(cfg)
    g = gpu_problem(dot, cfg, prob, wl)
    g.reset_stats()
    Js = g.jacobian(None, None)                     # ld = 40, ls = 9
    st = g.stats()
    assert st["contract_flops"] < st["contract_flops_dense"]
    monkeypatch.setenv("DOT_CONTRACT", "dense")
    gd = gpu_problem(dot, cfg, prob, wl)
    Jd = gd.jacobian(None, None)
    assert rel(Js, Jd) < 1e-12
    Jo = jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    assert rel(Js, Jo) < 1e-7


@pytest.mark.parametrize("chunk", [None, "1"])
def test_segment_gemm_ragged_tiles_and_chunks(dot, monkeypatch, chunk):
    """The pre-formed-operand segment GEMM over several 64-row tiles on both sides with
    ragged tails (ld = 70 detectors, 5 ls = 65 (q, i) rows), bases whose point counts are
    not multiples of the 16-point k-tile, and (chunk = 1) the column tiles streamed one at a
    time through a workspace-sized chunk: equal to the dense kernel and the oracle."""
    if chunk:
        monkeypatch.setenv("DOT_SEG_CHUNK", chunk)
    cfg = small_config(n=(24, 20, 10), L=(4.0, 3.5, 2.5), src=(13, 1), det=(10, 7), n_rbf=4, eps=0.5)
    prob, wl = small_problem(cfg)
    g = gpu_problem(dot, cfg, prob, wl)
    g.reset_stats()
    Js = g.jacobian(None, None)                     # ld = 70, ls = 13
    st = g.stats()
    assert st["contract_flops"] < st["contract_flops_dense"]
    monkeypatch.setenv("DOT_CONTRACT", "dense")
    gd = gpu_problem(dot, cfg, prob, wl)
    Jd = gd.jacobian(None, None)
    assert rel(Js, Jd) < 1e-12
    Jo = jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    assert rel(Js, Jo) < 1e-7


@pytest.mark.parametrize("seed", range(8))
def test_x_split_tilings_keep_parity(dot, seed, monkeypatch):
    """Row tiles split into two x parts (DOT_CG_XS=2: 2 halo columns per side, slot tiles by
    tensor copies with zero fill outside the domain) on seeded grids with nx = 0 mod 4, ragged
    row tiles, z chunks and both thread mappings: dense solves and sampled measurements vs
    the oracle."""
    rng = np.random.default_rng(2000 + seed)
    nx = int(rng.choice([8, 12, 20, 28, 36]))
    ny, nz = int(rng.integers(3, 30)), int(rng.integers(2, 24))
    monkeypatch.setenv("DOT_CG_XS", "2")
    monkeypatch.setenv("DOT_CG_ROWS", ["1", "2"][seed % 2])
    if seed % 3 == 0 and nz >= 8:
        monkeypatch.setenv("DOT_CG_ZCHUNKS", str(int(rng.integers(2, 5))))
    L = (float(rng.uniform(1.5, 4.0)), float(rng.uniform(1.5, 4.0)), float(rng.uniform(1.0, 3.0)))
    cfg = small_config(n=(nx, ny, nz), L=L, src=(2, min(2, ny)), det=(3, min(2, ny)), eps=0.5, seed=seed)
    prob, wl = small_problem(cfg, with_data=False)
    g = gpu_problem(dot, cfg, prob, wl)
    N = prob.grid.N
    b = rng.standard_normal((2, N)) + 1j * rng.standard_normal((2, N))
    mu = absorption(wl.p, prob.grid, cfg)
    for f in range(len(prob.omegas)):
        x, _ = g.solve(b, f)
        ref = spla.splu(prob.operator(mu, f).tocsc()).solve(b.T).T
        assert rel(x, ref) < 1e-11, (nx, ny, nz, f)
    X = g.solve_sampled(0)
    samp = g.samples()
    M = np.transpose(X[:, :, np.searchsorted(samp, wl.det_nodes)], (0, 2, 1))
    assert rel(M, measurements(prob, wl.p)) < 1e-8, (nx, ny, nz)


def test_contraction_with_a_basis_without_support_points(dot):
    """A basis whose centre lies far outside the domain has dA/dp = 0 everywhere (no points
    in its segment): the segment GEMM's items of that basis and the small-panel chunks are
    empty and its five J columns are exactly zero; the other columns match the oracle."""
    cfg = small_config(n=(24, 20, 10), L=(4.0, 3.5, 2.5), src=(3, 3), det=(8, 5), n_rbf=4, eps=0.5)
    prob, wl = small_problem(cfg)
    wl.p[5 * 3 + 2: 5 * 3 + 5] = 100.0                    # basis 3: centre far outside
    g = gpu_problem(dot, cfg, prob, wl)
    J = g.jacobian(None, None)                            # ld = 40, ls = 9: the segment GEMM
    assert np.all(J[..., 15:20] == 0)
    Jo = jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    assert np.abs(Jo[..., 15:20]).max() == 0
    assert rel(J, Jo) < 1e-7
    rng = np.random.default_rng(8)
    W = np.sign(rng.standard_normal((cfg.n_s, 3)))
    V = np.sign(rng.standard_normal((cfg.n_d, 4)))
    Js = g.jacobian(W, V)                                 # 4 x 3 pairs: the small-panel form
    assert np.all(Js[..., 15:20] == 0)
    assert rel(Js, jacobian(prob, wl.p, W, V)) < 1e-7


def test_mid_size_sketched_panels_take_the_gathered_kernel(dot):
    """Sketched panels too wide for the small form (ld x ls = 400 > 256) and too narrow for
    the segment GEMM (ld < 32) run the S-ordered block-sparse kernel: oracle parity."""
    cfg = small_config(n=(24, 20, 10), L=(4.0, 3.5, 2.5), src=(3, 3), det=(8, 5), n_rbf=4, eps=0.5)
    prob, wl = small_problem(cfg)
    g = gpu_problem(dot, cfg, prob, wl)
    rng = np.random.default_rng(9)
    W = np.sign(rng.standard_normal((cfg.n_s, 20)))
    V = np.sign(rng.standard_normal((cfg.n_d, 20)))
    g.reset_stats()
    J = g.jacobian(W, V)
    st = g.stats()
    assert st["contract_flops"] < st["contract_flops_dense"]      # block-sparse
    assert st["contract_dmma_flops"] == 0                          # not the segment GEMM
    assert rel(J, jacobian(prob, wl.p, W, V)) < 1e-7


def test_dependent_launch_is_bitwise_neutral(dot, monkeypatch):
    """The passes are launched with programmatic stream serialization (DESIGN.md "Pass launch
    overlap"); DOT_CG_PDL=0 at problem creation launches them plainly.  The launch mode only
    moves the shared-memory set-up ahead of the previous pass's completion, so sampled solutions,
    iteration counts and the Jacobian must be bit-identical — a pass that read r, p or the active
    list before the previous pass had finished would differ.  Small batches (one wave, z chunks:
    the case in which the next pass is resident early) and a multi-wave batch; the default mode
    is also checked against the oracle.  The same holds for the fold of the shifted recurrences
    running on its side stream (two-period history ring) or in the pass stream."""
    for n, src, det in (((32, 32, 12), (3, 2), (2, 3)), ((64, 37, 9), (6, 5), (5, 5))):
        cfg = small_config(n=n, L=(4.0, 4.0, 2.0), src=src, det=det, eps=0.5, seed=5)
        prob, wl = small_problem(cfg)
        out = []
        for mode, fold in (("1", "1"), ("0", "0"), ("1", "0")):
            monkeypatch.setenv("DOT_CG_PDL", mode)
            monkeypatch.setenv("DOT_CG_FOLD_SIDE", fold)   # folds beside the next passes / in the pass stream
            g = gpu_problem(dot, cfg, prob, wl)
            X = g.solve_sampled(0)
            J = g.jacobian(None, None)
            out.append((X.copy(), J.copy(), g.stats()["rhs_iterations"]))
            del g
        for o in out[1:]:
            assert out[0][2] == o[2]
            assert np.array_equal(out[0][0], o[0])
            assert np.array_equal(out[0][1], o[1])
        assert rel(out[0][1], jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))) < 1e-7
