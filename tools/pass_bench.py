"""Quick CG-pass throughput probe on one bench workload's grid (tiling A/B, not a bench line).

  python tools/pass_bench.py CONFIG NCOLS [REPS]
Solves NCOLS Rademacher source combinations at every frequency of CONFIG (sampled
solutions only) REPS times and prints the pass kernel HBM GB/s (library stats,
32 B/point/iteration per real seed) and its fraction of MEASURED_PEAKS.json.  The tiling knobs
(DOT_CG_TY, DOT_CG_ROWS, DOT_CG_ZCHUNKS, ...) are read from the environment."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1706_05586_b200 as dot  # noqa: E402
from synth import config_by_name, make_workload  # noqa: E402


def main():
    name, ncols = sys.argv[1], int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    cfg = config_by_name(name)
    wl = make_workload(cfg)
    gp = dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes)
    gp.set_params(wl.p)
    rng = np.random.default_rng(0)
    new_w = lambda: np.sign(rng.standard_normal((cfg.n_s, ncols)))     # noqa: E731 (fresh: no field-cache hit)
    gp.solve_sampled(0, new_w())                # warm-up (also sets kernel attributes)
    gp.enable_timing(True)
    gp.reset_stats()
    for _ in range(reps):
        gp.solve_sampled(0, new_w())
    st = gp.stats()
    gbs = st["pass_bytes"] / max(st["pass_ms"], 1e-9) / 1e6
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(f"{name} ncols {ncols}: pass {gbs:.0f} GB/s frac {gbs / peak:.4f} "
          f"({st['rhs_solved']} solves, {st['pass_ms']:.1f} ms in passes, "
          f"{st['rhs_iterations'] / max(st['rhs_solved'], 1):.1f} iterations/solve)")


if __name__ == "__main__":
    main()
