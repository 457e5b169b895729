"""Multi-rank host logic of paper_1706_05586_b200/sharded.py on CPU: world_size 2
over gloo, each rank backed by the CPU oracle (test infrastructure), must give
the same misfit, full Jacobian and sketched Jacobian as one unsharded oracle
evaluation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from tests._small import small_config, small_problem


class OracleBackend:
    """CPU stand-in exposing the DOTProblem methods sharded_step uses."""

    def __init__(self, prob):
        self.prob = prob
        self.n_freq = len(prob.omegas)

    def set_data(self, d):
        self.prob.data = np.asarray(d)

    def set_params(self, p):
        from oracle import jacobian_weights
        self.p = np.asarray(p.cpu() if isinstance(p, torch.Tensor) else p)
        G = jacobian_weights(self.p, self.prob.grid, self.prob.cfg)
        self.S = np.nonzero(np.abs(G).sum(1) > 0)[0]
        self.G = G[self.S]
        self.lus = [self.prob.factor(self.p, f) for f in range(len(self.prob.omegas))]

    @staticmethod
    def _np(x):
        return None if x is None else np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x)

    def misfit(self, W, V):
        from oracle import misfit
        W, V = self._np(W), self._np(V)
        W = np.eye(self.prob.B.shape[1]) if W is None else W
        V = np.eye(self.prob.C.shape[1]) if V is None else V
        return misfit(self.prob, self.p, W, V)

    def fields_on_support(self, side, coeff):
        coeff = self._np(coeff)
        M = (self.prob.B if side == 0 else self.prob.C) @ coeff
        out = []
        for lu in self.lus:
            X = self.prob.solve(lu, M, trans="N" if side == 0 else "T")
            out.append(X[self.S].T)
        return torch.as_tensor(np.stack(out))

    def support_weights(self):
        return torch.as_tensor(self.G)

    def contract(self, L, U, G):
        return -torch.einsum("fjs,fis,sk->fjik", L, U, G.to(L.dtype))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = {2: dict(n=(7, 7, 5), src=(3, 1), det=(2, 2), eps=0.4),
         # world 3 with 2 sources: one rank owns no source column (empty block)
         3: dict(n=(7, 7, 5), src=(2, 1), det=(2, 2), eps=0.4)}


def _worker(rank, world, port, out, sketch=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1706_05586_b200.sharded import ShardPlan, sharded_step
    cfg = small_config(**CASES[world])
    prob, wl = small_problem(cfg)
    rng = np.random.default_rng(0)
    W = np.sign(rng.standard_normal((cfg.n_s, 2)))
    V = np.sign(rng.standard_normal((cfg.n_d, 3)))
    plan = ShardPlan(rank, world, cfg.n_s, cfg.n_d)
    if not sketch:                       # the all-sources step of configs[4]: no sketch, full J only
        W = V = None
    try:
        r = sharded_step(OracleBackend(prob), plan, torch.as_tensor(wl.p),
                         None if W is None else torch.as_tensor(W), None if V is None else torch.as_tensor(V),
                         device=torch.device("cpu"))
    except Exception as e:  # report instead of hanging the parent
        out.put(("error", repr(e)))
        raise
    if rank == 0:
        out.put((r["misfit"], np.asarray(r["J_full"]), None if r["J_sketch"] is None else np.asarray(r["J_sketch"]),
                 prob.solves))
    else:
        out.put(("solves", prob.solves))
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_step_equals_unsharded(world):
    from oracle import jacobian, misfit
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    errors = [r for r in res if r[0] == "error"]
    assert not errors, errors
    main = [r for r in res if r[0] != "solves"][0]
    m, Jf, Js, solves0 = main
    cfg = small_config(**CASES[world])
    prob, wl = small_problem(cfg)
    rng = np.random.default_rng(0)
    W = np.sign(rng.standard_normal((cfg.n_s, 2)))
    V = np.sign(rng.standard_normal((cfg.n_d, 3)))
    assert m == pytest.approx(misfit(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d)), rel=1e-10)
    Jf_ref = jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    assert np.abs(Jf - Jf_ref).max() <= 1e-10 * np.abs(Jf_ref).max()
    Js_ref = jacobian(prob, wl.p, W, V)
    assert np.abs(Js - Js_ref).max() <= 1e-10 * np.abs(Js_ref).max()


def test_all_sources_step_shape_two_ranks():
    """The bench's configs[4] step (`--config all128 --gpus N`): no sketch, misfit and the full
    Jacobian gathered on rank 0, world 2 on gloo."""
    from oracle import jacobian, misfit
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, False)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert not [r for r in res if r[0] == "error"], res
    m, Jf, Js, _ = [r for r in res if r[0] != "solves"][0]
    assert Js is None
    cfg = small_config(**CASES[2])
    prob, wl = small_problem(cfg)
    assert m == pytest.approx(misfit(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d)), rel=1e-10)
    Jf_ref = jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    assert np.abs(Jf - Jf_ref).max() <= 1e-10 * np.abs(Jf_ref).max()


def test_shard_plan_blocks_cover_once():
    from paper_1706_05586_b200.sharded import ShardPlan
    for n, w in [(256, 8), (1024, 3), (7, 2), (5, 5), (12, 8), (2, 3)]:
        covered, sizes = [], []
        for r in range(w):
            lo, hi = ShardPlan(r, w, n, n).src_block()
            covered.extend(range(lo, hi))
            sizes.append(hi - lo)
        assert covered == list(range(n))
        assert max(sizes) - min(sizes) <= 1                  # balanced
        assert max(sizes) <= ShardPlan(0, w, n, n).per_src  # fits the all_gather padding
