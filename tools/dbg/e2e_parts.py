import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1706_05586_b200 as dot
from synth import config_by_name, make_workload
cfg = config_by_name("full64"); wl = make_workload(cfg)
g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
D = np.zeros((cfg.n_freq, cfg.n_d, cfg.n_s), complex)
pin = lambda a: torch.as_tensor(a).pin_memory().numpy()
p_h, D_h, W_h, V_h = pin(wl.p), pin(D), pin(wl.W), pin(wl.V)
def T(label, fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:30s} {1e3*(time.perf_counter()-t):8.2f} ms", flush=True); return r
for it in range(3):
    T("set_data", lambda: g.set_data(D_h))
    T("set_params", lambda: g.set_params(p_h))
    T("jacobian(I,I) host", lambda: g.jacobian(None, None, where=0))
    T("misfit", lambda: g.misfit(None, None))
    T("jacobian(W,V) host", lambda: g.jacobian(W_h, V_h))
    print("--")
pd = torch.as_tensor(wl.p, device="cuda")
T("set_params dev", lambda: g.set_params(pd))
T("jacobian(I,I) dev", lambda: g.jacobian(None, None, where=1))
