"""The block-sparse Jacobian contraction alone (values only; not a bench line).

  python tools/seg_bench.py [full64|all128|opt96 ...]

Per config: the problem at the synthetic iterate p (support S, basis segments), random
complex panels Lam [n_freq][n_d][K], U [n_freq][n_s][K] on S, `DOTProblem.contract` (basis
gather + contract_seg_kernel) timed by the library's events around the contraction kernel;
prints useful TFLOP/s (4 flop per (pair, point, parameter) with a nonzero weight block) and
the fraction of the measured FP64 peak, plus a spot check of a few J entries against a torch
complex matmul on the same panels."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05586_b200 as dot  # noqa: E402
from synth import config_by_name, make_workload  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["tflops"]


def run(name, reps=5):
    cfg = config_by_name(name)
    wl = make_workload(cfg)
    gp = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes, workspace_bytes=int(24e9))
    gp.set_params(wl.p)
    G = gp.support_weights()
    K = G.shape[0]
    nf, ld, ls = cfg.n_freq, cfg.n_d, cfg.n_s
    g = torch.Generator(device="cuda").manual_seed(0)
    Lam = torch.randn(nf, ld, K, dtype=torch.complex128, device="cuda", generator=g)
    U = torch.randn(nf, ls, K, dtype=torch.complex128, device="cuda", generator=g)
    J = gp.contract(Lam, U)
    torch.cuda.synchronize()
    gp.enable_timing(True)
    best = None
    for _ in range(reps):
        gp.reset_stats()
        J = gp.contract(Lam, U)
        st = gp.stats()
        r = (st["contract_ms"], st["contract_flops"])
        best = r if best is None or r[0] < best[0] else best
    ms, fl = best
    # spot check: J[f][d][i][:] for a few (f, d, i) against a torch matmul on the same panels
    err = 0.0
    for f, d, i in [(0, 0, 0), (nf - 1, ld - 1, ls - 1), (nf // 2, ld // 3, ls // 2)]:
        ref = -((Lam[f, d] * U[f, i])[None, :] @ G.to(torch.complex128))[0]
        err = max(err, ((J[f, d, i] - ref).abs().max() / ref.abs().max()).item())
    out = {"config": name, "K": K, "ms": ms, "useful_tflops": fl / ms / 1e9, "frac": fl / ms / 1e9 / PEAK,
           "spot_rel_err": err}
    print(json.dumps(out), flush=True)
    del Lam, U, J
    gp.close()
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for n in (sys.argv[1:] or ["full64", "all128"]):
        run(n)
