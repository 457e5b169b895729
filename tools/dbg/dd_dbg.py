import os, sys, faulthandler, socket
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np

def worker(rank, world, port):
    faulthandler.enable()
    faulthandler.dump_traceback_later(90, exit=True)
    import torch, torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1706_05586_b200 as dot
    from paper_1706_05586_b200.dd import TransportDD
    from tests._small import small_config, small_problem
    cfg = small_config(n=(24, 20, 19), L=(4.0, 3.5, 3.0), src=(3, 2), det=(2, 3), eps=0.4)
    prob, wl = small_problem(cfg, with_data=True)
    rng = np.random.default_rng(world)
    W = np.sign(rng.standard_normal((cfg.n_s, 3))); V = np.sign(rng.standard_normal((cfg.n_d, 2)))
    g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
    g.set_data(prob.data); g.set_params(wl.p)
    print(rank, "created", flush=True)
    dd = TransportDD(g, rank, world)
    print(rank, "dd", flush=True)
    dd.fields(W, V)
    print(rank, "fields done", g.stats()["rhs_solved"], dd._transport.errors, flush=True)
    print(rank, "misfit", g.misfit(W, V), flush=True)

if __name__ == "__main__":
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ps = [mp.get_context("spawn").Process(target=worker, args=(r, 2, port)) for r in range(2)]
    [p.start() for p in ps]; [p.join(200) for p in ps]
    print("exit codes", [p.exitcode for p in ps])
