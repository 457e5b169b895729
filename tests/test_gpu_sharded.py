"""The RHS-sharded step (paper_1706_05586_b200/sharded.py) with world_size 2 on ONE GPU:
two processes, each a rank with its own DOTProblem on cuda:0, collectives over gloo
(the ranks' kernels never wait on each other -- all exchange happens between calls).
Checked against the CPU oracle (misfit 1e-8, Jacobians 1e-7; north_star) and against
the unsharded GPU step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from tests._small import small_config, small_problem

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg():
    return small_config(n=(16, 14, 12), L=(4.0, 3.5, 3.0), src=(3, 2), det=(2, 3), eps=0.4)


def _worker(rank, world, port, q, data):
    # (the oracle data are computed in the parent: scipy in spawned CUDA workers is slow)
    try:
        import torch.distributed as tdist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1706_05586_b200 as dot
        from paper_1706_05586_b200.sharded import ShardPlan, sharded_step
        from synth import make_workload
        cfg = _cfg()
        wl = make_workload(cfg)
        wl.p[0] = max(wl.p[0], 0.8)        # as tests._small.small_problem
        rng = np.random.default_rng(0)
        W = np.sign(rng.standard_normal((cfg.n_s, 3)))
        V = np.sign(rng.standard_normal((cfg.n_d, 2)))
        g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
        plan = ShardPlan(rank, world, cfg.n_s, cfg.n_d)
        out = sharded_step(g, plan, wl.p, W, V, data=data, device=torch.device("cuda", 0),
                           comm_device=torch.device("cpu"))
        Js = out["J_sketch"]
        res = {"rank": rank, "misfit": out["misfit"],
               "J_sketch": np.asarray(Js.cpu() if isinstance(Js, torch.Tensor) else Js),
               "J_full": None if out["J_full"] is None else np.asarray(out["J_full"].cpu()
                                                                   if isinstance(out["J_full"], torch.Tensor)
                                                                   else out["J_full"]),
               "solves": g.stats()["rhs_solved"]}
        q.put(res)
        tdist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put({"rank": rank, "error": traceback.format_exc()})


def test_two_rank_sharded_step_on_one_gpu():
    import paper_1706_05586_b200 as dot
    from paper_1706_05586_b200.sharded import ShardPlan, sharded_step
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    prob0, _ = small_problem(_cfg())
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qu, prob0.data)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([qu.get(timeout=600) for _ in range(2)], key=lambda r: r["rank"])
    for p in procs:            # results are in; do not wait long for process teardown
        p.join(timeout=20)
        if p.is_alive():
            p.kill()
    assert all("error" not in r for r in res), [r.get("error") for r in res]
    cfg = _cfg()
    prob, wl = small_problem(cfg)
    rng = np.random.default_rng(0)
    W = np.sign(rng.standard_normal((cfg.n_s, 3)))
    V = np.sign(rng.standard_normal((cfg.n_d, 2)))
    from oracle import jacobian, misfit
    m_or = misfit(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    Jf_or = jacobian(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    Js_or = jacobian(prob, wl.p, W, V)
    for r in res:
        assert abs(r["misfit"] - m_or) <= 1e-8 * m_or
        assert np.linalg.norm(r["J_sketch"] - Js_or) <= 1e-7 * np.linalg.norm(Js_or)
    assert np.linalg.norm(res[0]["J_full"] - Jf_or) <= 1e-7 * np.linalg.norm(Jf_or)
    g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
    ref = sharded_step(g, ShardPlan(0, 1, cfg.n_s, cfg.n_d), wl.p, W, V, data=prob.data)
    for r in res:
        assert r["misfit"] == pytest.approx(ref["misfit"], rel=1e-10)
        assert np.abs(r["J_sketch"] - ref["J_sketch"]).max() <= 1e-10 * np.abs(ref["J_sketch"]).max()
        # each rank solved its own source block + detector block only
        nf = len(cfg.freqs_hz)
        assert r["solves"] == nf * (3 + 3)
    Jf = res[0]["J_full"]
    assert np.abs(Jf - ref["J_full"]).max() <= 1e-10 * np.abs(ref["J_full"]).max()
