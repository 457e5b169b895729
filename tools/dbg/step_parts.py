"""Device-resident full64 bench step split by API call (wall time around a synchronize) next to the
library's pass-event time: where the step time outside the CG passes goes."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1706_05586_b200 as dot
from synth import config_by_name, make_workload
cfg = config_by_name("full64"); wl = make_workload(cfg)
g = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
g.set_data(np.zeros((cfg.n_freq, cfg.n_d, cfg.n_s), complex))
pd = torch.as_tensor(wl.p, device="cuda"); Wd = torch.as_tensor(wl.W, device="cuda"); Vd = torch.as_tensor(wl.V, device="cuda")
g.enable_timing(True)
def T(label, fn):
    torch.cuda.synchronize(); s0 = g.stats(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    dt = 1e3 * (time.perf_counter() - t); s1 = g.stats()
    print(f"{label:22s} {dt:8.2f} ms   passes {s1['pass_ms'] - s0['pass_ms']:8.2f}  contract {s1['contract_ms'] - s0['contract_ms']:6.2f}"
          f"  launches {s1['kernel_launches'] - s0['kernel_launches']}", flush=True); return r
for it in range(4):
    T("set_params", lambda: g.set_params(pd))
    T("prefetch_fields", lambda: g.prefetch_fields(None, None))
    T("jacobian(I,I)", lambda: g.jacobian(None, None, where=1))
    T("misfit(I,I)", lambda: g.misfit(None, None))
    T("jacobian(W,V)", lambda: g.jacobian(Wd, Vd, where=1))
    print("--")
