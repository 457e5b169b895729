"""Diagnostic: solve point-source systems at increasing grid sizes on the GPU and
report iterations / true residuals (oracle matvec).  Not part of the product."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1706_05586_b200 as dot
from synth import config_by_name, make_workload
from oracle import make_problem, absorption

for name, n in [("sketch32", None), ("full64", (40, 40, 40)), ("full64", None)]:
    cfg = config_by_name(name)
    if n: cfg = cfg.with_(n=n)
    wl = make_workload(cfg)
    from synth import face_nodes
    src = face_nodes(cfg.n, cfg.src_grid, 0); det = face_nodes(cfg.n, cfg.det_grid, cfg.n[2]-1)
    prob = make_problem(cfg, src, det)
    g = dot.DOTProblem.from_config(cfg, src, det, max_rhs=64)
    g.set_params(wl.p)
    N = prob.grid.N
    b = np.zeros((2, N), complex); b[0, src[0]] = 1.0; b[1, src[5]] = 1.0
    for f in range(cfg.n_freq):
        try:
            x, it = g.solve(b, f)
            A = prob.operator(absorption(wl.p, prob.grid, cfg), f)
            res = [np.linalg.norm(b[r] - A @ x[r]) / np.linalg.norm(b[r]) for r in range(2)]
            print(name, cfg.n, 'f', f, 'iters', it, 'true res', res, flush=True)
        except Exception as e:
            print(name, cfg.n, 'f', f, 'ERROR', e, flush=True)
    for ncols in (1, 4):
        try:
            t = time.time(); X = g.solve_sampled(0, np.eye(cfg.n_s)[:, :ncols]); 
            print(name, 'sampled', ncols, 'ok', g.stats()['last_max_iters'], time.time()-t, flush=True)
        except Exception as e:
            print(name, 'sampled', ncols, 'ERROR', e, flush=True)
    g.close()
