#!/usr/bin/env python
"""Writes tests/golden/<config>_oracle.npz: the oracle's measurements, data and misfits at a
BASELINE.json config at full size -- configs[2] (`full64`: 64^3, 256 sources x 256 detectors,
3 frequencies, 80 parameters; the configuration the bench metric is quoted on) by default,
or configs[1] (`--config sketch32`: 32^3, 64 x 64, 3 frequencies, 40 parameters).

Calls ONLY oracle/ (scipy splu in complex128) and synth/ (seeded inputs).  Each frequency
runs in its own process (one sparse LU of the 64^3 operator is ~400 s and ~6 GB):
  M_true_f, D_f  oracle.simulate_data at the hidden level set p_true with noise xi
                 (Eq. (2.5) + BASELINE "1% Gaussian noise"; reading R10)
  M_f            oracle.measurements at the iterate p: C^T A(omega_f, p)^-1 B (L181-185)
  misfit_II_f    oracle.misfit(W = I, V = I): ||C^T Z - D_f||_F^2 (L365, footnote L269)
  misfit_WV_f    oracle.misfit at the bench's Rademacher W, V 256 x 12 (Eq. (EsTResidual))
  J_WV_f         oracle.jacobian(W, V): (W^T (x) V^T) J (L966-972), 12 x 12 x 80 per freq

  python tools/golden.py [--config full64|sketch32] [--out PATH] [--procs 3]
"""
from __future__ import annotations

import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one_frequency(args):
    f, name = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import jacobian, make_problem, measurements, misfit, simulate_data
    from synth import config_by_name, make_workload
    cfg = config_by_name(name)
    wl = make_workload(cfg)
    t0 = time.time()
    prob = make_problem(cfg, wl.src_nodes, wl.det_nodes)
    prob.omegas = prob.omegas[f:f + 1]                   # this process: frequency f only
    D = simulate_data(prob, wl.p_true_padded, wl.xi[f:f + 1], cfg.noise)
    prob.data = D
    M = measurements(prob, wl.p)
    m_ii = misfit(prob, wl.p, np.eye(cfg.n_s), np.eye(cfg.n_d))
    m_wv = misfit(prob, wl.p, wl.W, wl.V)
    J = jacobian(prob, wl.p, wl.W, wl.V)
    print(f"freq {f}: {time.time() - t0:.0f} s", flush=True)
    return f, D[0], M[0], m_ii, m_wv, J[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="full64", choices=["full64", "sketch32"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--procs", type=int, default=3)
    a = ap.parse_args()
    out = a.out or os.path.join(ROOT, "tests", "golden", f"{a.config}_oracle.npz")
    from synth import config_by_name
    cfg = config_by_name(a.config)
    with mp.get_context("spawn").Pool(a.procs) as pool:
        res = sorted(pool.map(one_frequency, [(f, a.config) for f in range(cfg.n_freq)]))
    np.savez_compressed(
        out,
        data=np.stack([r[1] for r in res]),            # (n_freq, n_d, n_s) [f][d][s]
        M=np.stack([r[2] for r in res]),               # (n_freq, n_d, n_s) at p
        misfit_II=np.array([r[3] for r in res]),       # per frequency
        misfit_WV=np.array([r[4] for r in res]),
        J_WV=np.stack([r[5] for r in res]),            # (n_freq, ld, ls, n_p) [f][j][i][k]
        note=np.array("oracle/ only (scipy splu complex128); tools/golden.py"))
    print("wrote", out)


if __name__ == "__main__":
    main()
