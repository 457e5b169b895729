"""Diagnostic: large sampled batches at 64^3 (bench sequence)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1706_05586_b200 as dot
from synth import config_by_name, make_workload
cfg = config_by_name('full64'); wl = make_workload(cfg)
g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
for pname, p in (("p", wl.p), ("p_true", wl.p_true)):
    if pname == "p_true":
        g2 = dot.DOTProblem.from_config(cfg.with_(n_rbf=cfg.n_rbf_true), wl.src_nodes, wl.det_nodes, max_rhs=2048)
    else:
        g2 = g
    g2.set_params(p)
    print(pname, 'K', g2.stats()['support_K'], 'nP', g2.stats()['n_samples'], flush=True)
    for ncols in (16, 64, 256):
        try:
            t = time.time(); X = g2.solve_sampled(0, np.eye(cfg.n_s)[:, :ncols])
            st = g2.stats()
            print(pname, ncols, 'ok', st['last_min_iters'], st['last_max_iters'], '%.3f s' % (time.time()-t), flush=True)
        except Exception as e:
            print(pname, ncols, 'ERROR', e, flush=True)
