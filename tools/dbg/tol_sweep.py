import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1706_05586_b200 as dot
from synth import config_by_name, make_workload
z = np.load("tests/golden/full64_oracle.npz")
cfg = config_by_name("full64"); wl = make_workload(cfg)
for tol in (1e-17, 3e-17, 1e-16, 3e-16):
    g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes, tol=tol)
    g.set_data(z["data"]); g.set_params(wl.p)
    X = g.solve_sampled(0); samp = g.samples()
    M = np.transpose(X[:, :, np.searchsorted(samp, wl.det_nodes)], (0, 2, 1))
    e = max(np.abs(M[f] - z["M"][f]).max() / np.abs(z["M"][f]).max() for f in range(3))
    fr = np.linalg.norm(M - z["M"]) / np.linalg.norm(z["M"])
    st = g.stats()
    J = g.jacobian(wl.W, wl.V)
    ej = np.linalg.norm(J - z["J_WV"]) / np.linalg.norm(z["J_WV"])
    m = g.misfit(None, None); em = abs(m - z["misfit_II"].sum()) / z["misfit_II"].sum()
    print(f"tol {tol:.0e}: iters {st['last_max_iters']}  M maxnorm {e:.2e} fro {fr:.2e}  J {ej:.2e}  misfit {em:.2e}", flush=True)
    g.close()
