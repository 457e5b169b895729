"""Small seeded problems for the CPU pins and the GPU parity tests."""
import numpy as np

from synth import config_by_name, make_workload


def small_config(n=(8, 8, 7), L=(3.0, 3.0, 2.5), src=(2, 2), det=(2, 2), n_rbf=3,
                 freqs=(0.0, 1.4e8), eps=0.3, ls=None, ld=None, seed=0):
    base = config_by_name("tiny16")
    return base.with_(name="small", n=n, L=L, src_grid=src, det_grid=det, n_rbf=n_rbf,
                      freqs_hz=tuple(freqs), eps=eps, ls=ls, ld=ld, seed=seed)


def small_problem(cfg, with_data=True):
    from oracle import make_problem, simulate_data
    wl = make_workload(cfg)
    # make sure the current iterate has an interface: alpha of basis 0 pushed above the cut
    wl.p[0] = max(wl.p[0], 0.8)
    prob = make_problem(cfg, wl.src_nodes, wl.det_nodes)
    if with_data:
        prob.data = simulate_data(prob, wl.p_true, wl.xi, cfg.noise)
    return prob, wl


def all_sign_vectors(n):
    out = []
    for m in range(2 ** n):
        out.append(np.array([1.0 if (m >> b) & 1 else -1.0 for b in range(n)]))
    return out
