#!/usr/bin/env python
"""Throughput of the B200 DOT hot path (arXiv 1706.05586) on BASELINE.json configs[2].

One step at 64^3, 256 sources x 256 detectors x 3
frequencies, 16 RBFs (80 parameters):
  set_params(p)            PaLS mu(x,p), support S of dA/dp, G on S
  jacobian(I, I)           all 256 forward + 256 adjoint RHS per frequency (1536 systems,
                           solved as 512 real multi-shift CG seeds) and the full Jacobian
                           on FP64 DMMA
  misfit(I, I)             full-data misfit from the cached forward fields
  jacobian(W, V)           sketched Jacobian, W, V Rademacher 256 x 12
Metric: RHS solves/s (whole job; one solve = one (right-hand side, frequency) system), with
the CG pass kernel's HBM roofline and the Jacobian contraction's FP64 TFLOP/s beside it.
--config sketch32 | opt96 | all128 runs the other BASELINE rows (all128: configs[4], the
all-sources step with the full Jacobian).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]
Multi-GPU: launched by torch.distributed.run; RHS columns are sharded across ranks
(full64, all128; paper_1706_05586_b200/sharded.py), rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RHS solves/s at 64^3 complex fp64 (% HBM roofline); Jacobian FP64 TFLOP/s"
UNIT = "RHS solves/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 10 for full64 -- ~3 s, so that one host or NVML hiccup does not "
                         "move the line --, 30 for sketch32, 3 for opt96, 1 for all128)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="full64")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="one untimed step (for ncu launch lists)")
    ap.add_argument("--oracle-sample", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 3 if args.impl == "reference" else \
            {"full64": 10, "sketch32": 30, "opt96": 3, "all128": 1}.get(args.config, 3)
    return args


# ------------------------------------------------------------------ helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        if os.environ.get("DOT_BENCH_NO_CLOCKS") == "1":      # diagnostics only: no sampling
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's own start-up (NVML init) stalls the driver for ~100 ms: wait for its
            # first sample so that it lands before the timed region, not inside it
            t0 = time.perf_counter()
            while not self.rows and self.proc.poll() is None and time.perf_counter() - t0 < 10:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get("hbm_gbs", 6553.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak():
    """FP64 tensor (DMMA) peak: measured cuBLAS DGEMM figure if profiles/ holds one,
    else the nominal B200 40 TFLOP/s."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d["tflops"], d.get("how", "measured")
    return 40.0, "nominal B200 FP64 tensor 40 TFLOP/s"


def ncu_traffic(cfg_name):
    """DRAM traffic of one captured CG pass launch of this config's grid (tools/make_profiles.py),
    or None when no capture of that grid is committed."""
    path = os.path.join(ROOT, "profiles", f"cg_pass_traffic_{cfg_name}.json")
    if os.path.exists(path):
        return json.load(open(path))
    return None


CPU_SAMPLE_N = 32   # grid of the bounded oracle sample


def oracle_sample(cfg_name, n_rhs=8, freq=0):
    """Times the CPU oracle as it stands on a bounded sample of the bench workload:
    the same physics, sources/detectors and PaLS iterate on a CPU_SAMPLE_N^3 grid
    (the oracle's sparse LU of the 64^3 operator alone takes ~400 s and ~6 GB,
    DESIGN.md "CPU baseline"), one frequency: one factorisation + n_rhs solves.
    Returns (solves/s amortised over the n_s + n_d RHS of one frequency, detail)."""
    from oracle import make_problem
    from synth import config_by_name, make_workload
    n = CPU_SAMPLE_N
    cfg = config_by_name(cfg_name)
    cfg = cfg.with_(n=(n, n, n))
    wl = make_workload(cfg)
    prob = make_problem(cfg, wl.src_nodes, wl.det_nodes)
    t0 = time.perf_counter()
    lu = prob.factor(wl.p, freq)
    t1 = time.perf_counter()
    prob.solve(lu, prob.B[:, :n_rhs])
    t2 = time.perf_counter()
    t_factor, t_solve = t1 - t0, (t2 - t1) / n_rhs
    per_freq_rhs = cfg.n_s + cfg.n_d
    value = per_freq_rhs / (t_factor + per_freq_rhs * t_solve)
    sample = (f"{cfg_name} physics on a {n}^3 grid (64^3 LU alone ~400 s): oracle scipy splu factorisation "
              f"of A(omega_{freq}) {t_factor:.1f} s + {n_rhs} solves ({t_solve * 1e3:.1f} ms/RHS); "
              f"value = {per_freq_rhs} RHS / (factor + {per_freq_rhs} solves); an upper bound on the "
              f"oracle at 64^3")
    return value, sample, {"t_factor_s": t_factor, "t_solve_per_rhs_s": t_solve}


SINGLE_THREAD_ENV = {"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1",
                     "VECLIB_MAXIMUM_THREADS": "1", "NUMEXPR_NUM_THREADS": "1"}


def pinned_cmd(argv):
    """argv under `taskset -c <one core>` when taskset exists (the core the process may use)."""
    import shutil
    core = min(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 0
    if shutil.which("taskset"):
        return ["taskset", "-c", str(core)] + argv, 1
    return argv, 1


def run_cpu_baseline(cfg_name):
    """The CPU oracle on a bounded sample, alone (nothing else of this run is executing),
    in a child pinned to ONE core with single-threaded BLAS/OpenMP.  Returns the
    cpu_baseline object."""
    cmd, cores = pinned_cmd([sys.executable, os.path.abspath(__file__), "--oracle-sample", cfg_name])
    env = dict(os.environ, **SINGLE_THREAD_ENV)
    r = subprocess.run(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, timeout=1800)
    if r.returncode != 0:
        return {"unavailable": r.stderr.strip().splitlines()[-1] if r.stderr.strip() else "oracle sample failed"}
    out = json.loads(r.stdout.strip().splitlines()[-1])
    out.update({"unit": UNIT, "cores": cores, "kind": "oracle",
                "pinning": "taskset -c <1 core>, OMP/OPENBLAS/MKL_NUM_THREADS=1, run before the GPU warm-up"})
    return out


def oracle_sample_main(cfg_name):
    value, sample, detail = oracle_sample(cfg_name)
    print(json.dumps({"value": value, "sample": sample, **detail}), flush=True)


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands on a bounded sample of the same
    workload (PAPER.md has no code; the oracle is the reference arm).  Rank 0
    only; other ranks exit without work."""
    if rank != 0:
        return
    # same conditions as the main arm's cpu_baseline: one core, single-threaded BLAS / OpenMP
    os.environ.update(SINGLE_THREAD_ENV)
    if hasattr(os, "sched_setaffinity"):
        os.sched_setaffinity(0, {min(os.sched_getaffinity(0))})
    from synth import config_by_name
    cfg = config_by_name(args.config)
    times, vals, sample = [], [], ""
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        v, sample, _ = oracle_sample(args.config, n_rhs=8, freq=it % cfg.n_freq)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
            vals.append(v)
    value = statistics.mean(vals)
    t = statistics.mean(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": args.config, "grid": [CPU_SAMPLE_N] * 3,
                       "sample": "per step: oracle factorisation + 8 RHS at one frequency"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.oracle_sample:
        oracle_sample_main(args.oracle_sample)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch
    import torch.distributed as tdist

    import paper_1706_05586_b200 as dot
    from synth import config_by_name, make_workload

    # DOT_BENCH_BACKEND=gloo + DOT_BENCH_DEVICE=0: smoke-test the multi-rank path with all
    # ranks on one GPU (collectives through host memory; timings then mean nothing)
    backend_name = os.environ.get("DOT_BENCH_BACKEND", "nccl")
    if os.environ.get("DOT_BENCH_DEVICE") is not None:
        local = int(os.environ["DOT_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    if world > 1:
        if backend_name == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend_name)
    cfg = config_by_name(args.config)
    wl = make_workload(cfg)
    dev = torch.device("cuda", local)

    # cpu baseline: the oracle sample runs alone, BEFORE any GPU work (rank 0, N = 1), in a
    # child process pinned to one core with single-threaded BLAS / OpenMP
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        cpu = run_cpu_baseline(args.config)

    # synthetic data: forward model at the hidden level set + 1% noise (setup, untimed;
    # computed by the GPU path because the oracle's LU at 64^3 takes minutes -- the
    # data values only enter the misfit, which is not a parity claim here)
    from paper_1706_05586_b200.sharded import ShardPlan, make_problem_for_rank, sharded_step
    plan = ShardPlan(rank, world, cfg.n_s, cfg.n_d)
    gp = make_problem_for_rank(dot, cfg, wl, plan)
    gp.set_params(wl.p_true_padded)
    X = gp.solve_sampled(0)
    samp = gp.samples()
    M = np.transpose(X[:, :, np.searchsorted(samp, wl.det_nodes)], (0, 2, 1))
    data = M + cfg.noise * np.abs(M) * wl.xi
    gp.set_data(data)
    gp.reset_stats()

    p_d = torch.as_tensor(wl.p, device=dev)
    W_d = torch.as_tensor(wl.W, device=dev) if wl.W is not None else None
    V_d = torch.as_tensor(wl.V, device=dev) if wl.V is not None else None
    D_d = torch.as_tensor(data, device=dev)

    if cfg.name in ("full64", "all128"):
        def run_step(p, W, V, data=None):
            """configs[2] (full64) / configs[4] (all128): set_params, all n_s forward and n_d
            adjoint fields at every frequency (multi-shift seeds, RHS-sharded over the ranks),
            full-data misfit, the FULL Jacobian (gathered on
            rank 0) and, when the config has a sketch, (W^T (x) V^T) J."""
            return sharded_step(gp, plan, p, W, V, data=data,
                                comm_device=None if backend_name == "nccl" else torch.device("cpu"))
    else:
        if world > 1:
            raise SystemExit("bench: the full64 and all128 workloads shard over ranks; sketch32 / opt96 are "
                             "single-GPU rows")
        X0s = torch.as_tensor(wl.X0_src, device=dev) if wl.X0_src is not None else None
        X0d = torch.as_tensor(wl.X0_det, device=dev) if wl.X0_det is not None else None

        def run_step(p, W, V, data=None):
            """configs[1] (sketch32): set_params, jacobian(W,V), misfit(W,V).
            configs[3] (opt96): the same, then replace n_opt random directions by optimized
            ones (5 subspace iterations, block 2; reading R16) and evaluate the reduced
            problem (misfit, jacobian) with the new W, V."""
            host = not isinstance(p, torch.Tensor)
            if data is not None:
                gp.set_data(data)
            gp.set_params(p)
            J = gp.jacobian(W, V, where=0 if host else 1)     # forward W + adjoint V solves in one batch
            m = gp.misfit(W, V)                                 # cached forward fields
            d2h = J.nbytes + 8 if host else 0
            if cfg.n_opt:
                xs = wl.X0_src if host else X0s
                xd = wl.X0_det if host else X0d
                W2, V2, obj = gp.optimize_directions_subspace(cfg.n_opt, W, V, xs, xd,
                                                              iters=cfg.n_subspace_iters)
                J = gp.jacobian(W2, V2, where=0 if host else 1)
                m = gp.misfit(W2, V2)
                d2h += J.nbytes + 8 + 8 + W2.nbytes + V2.nbytes if host else 0
            return {"misfit": m, "J_sketch": J, "d2h_bytes": d2h}

    def step_device():
        return run_step(p_d, W_d, V_d, data=None)

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    if args.profile:
        step_device()
        torch.cuda.synchronize()
        return

    gp.enable_timing(True)
    for _ in range(args.warmup):
        step_device()
    barrier()
    gp.reset_stats()
    s0 = gp.stats()
    sampler = ClockSampler(local)
    sampler.start()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    # L2 hygiene: the full64 working set (~25 GB) dwarfs the 126 MB L2; smaller workloads
    # get a 256 MB write between timed steps (inside the timed region, ~0.05 ms)
    ws_bytes = min(cfg.n_freq * (cfg.n_s + cfg.n_d), 4096) * 4 * cfg.N * 16
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if ws_bytes < (1 << 30) else None
    ev0.record(stream)
    out = None
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        out = step_device()
    ev1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = gp.stats()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    solves_per_step = (st["rhs_solved"] - s0["rhs_solved"]) / args.steps     # counted by the library
    if cfg.name in ("full64", "all128"):
        solves_per_step = cfg.n_freq * (cfg.n_s + cfg.n_d)                     # per step, all ranks
    value = solves_per_step / (ms / 1e3)

    # ---- end to end through the public API with host buffers (pinned), N = 1 API
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.as_tensor(a).pin_memory().numpy()   # noqa: E731
        p_h, D_h = pin(wl.p), pin(data)
        W_h = pin(wl.W) if wl.W is not None else None
        V_h = pin(wl.V) if wl.V is not None else None
        h2d = p_h.nbytes + D_h.nbytes + (W_h.nbytes if W_h is not None else 0) + (V_h.nbytes if V_h is not None else 0)
        for _ in range(2):                                        # warm (pinned result buffers cached)
            run_step(p_h, W_h, V_h, data=D_h)
        barrier()
        t0 = time.perf_counter()
        e2e_ev0 = torch.cuda.Event(enable_timing=True)
        e2e_ev1 = torch.cuda.Event(enable_timing=True)
        e2e_ev0.record(stream)
        d2h = 0
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()                                     # same L2 hygiene as the device-timed loop
            r = run_step(p_h, W_h, V_h, data=D_h)
            d2h = r["d2h_bytes"]
            r = None                                              # results consumed: buffers reusable
        e2e_ev1.record(stream)
        barrier()
        e_ms = e2e_ev0.elapsed_time(e2e_ev1) / args.steps
        wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            t = torch.tensor([e_ms, wall_ms], device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            e_ms, wall_ms = float(t[0]), float(t[1])
        e2e = {"value": solves_per_step / (max(e_ms, wall_ms) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": max(e_ms, wall_ms)}

    if rank != 0:
        if world > 1:
            tdist.barrier()
            tdist.destroy_process_group()
        return
    # the dense DMMA GEMM (north_star's "GEMM over the Hadamard-formed panel against G") on
    # this step's own panels: all 256 adjoint x 256 forward fields on S, timed alone
    dense_gemm = None
    if cfg.name == "full64" and world == 1:
        Lsup = gp.fields_on_support(1, None, where=1)
        Usup = gp.fields_on_support(0, None, where=1)
        Gsup = gp.support_weights()
        for _ in range(2):
            dot.contract(Lsup, Usup, Gsup, stream=stream)          # stateless dense DMMA kernel
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps = 5
        for _ in range(reps):
            dot.contract(Lsup, Usup, Gsup, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        gms = e0.elapsed_time(e1) / reps
        gfl = 4.0 * Lsup.shape[0] * Lsup.shape[1] * Usup.shape[1] * Lsup.shape[2] * Gsup.shape[1]
        fpk0, _ = fp64_peak()
        dense_gemm = {"ms": gms, "tflops": gfl / gms / 1e9, "frac": gfl / gms / 1e9 / fpk0,
                      "shape": list(Lsup.shape) + [Gsup.shape[1]]}
    peak, peak_src = measured_peaks()
    gbs = (st["pass_bytes"] - s0["pass_bytes"]) / max(st["pass_ms"] - s0["pass_ms"], 1e-9) / 1e6
    traffic = ncu_traffic(cfg.name)
    roof = {"bound": "hbm", "kernel": "cg_pass_kernel", "achieved": gbs, "peak": peak, "unit": "GB/s",
            "frac": gbs / peak, "peak_source": peak_src,
            "algorithmic_bytes": ("32 B per grid point per CG iteration per real seed (read r_k, p_k-1; write "
                                  "r_k+1, p_k in fp64); one seed delivers every frequency (multi-shift CG)"),
            "traffic": traffic["dram_bytes"] if traffic else None,
            "traffic_algorithmic": traffic["algorithmic_bytes_if_all_active"] if traffic else None,
            "traffic_ratio": traffic["ratio"] if traffic else None,
            "traffic_note": traffic["note"] if traffic else "no ncu --set full capture committed yet"}
    jf = st["contract_flops"] / max(st["contract_ms"], 1e-9) / 1e9
    fpk, fsrc = fp64_peak()

    def gemm_line(st, s0, steps, fpk):
        gms = st["gemm_ms"] - s0["gemm_ms"]
        if gms <= 0:
            return None
        gfl = st["gemm_flops"] - s0["gemm_flops"]
        dmma = st["contract_dmma_flops"] - s0["contract_dmma_flops"]
        return {"what": "full-data Jacobian calls (prescale + segment GEMM, CUDA events on the library stream)",
                "achieved_tflops": gfl / gms / 1e9, "frac": gfl / gms / 1e9 / fpk,
                "ms_per_step": gms / steps, "flops_per_step": gfl / steps,
                "dmma_executed_tflops": dmma / gms / 1e9, "dmma_executed_frac": dmma / gms / 1e9 / fpk,
                "small_panel_ms_per_step": (st["contract_ms"] - s0["contract_ms"] - gms) / steps}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "dtype_note": "fp64 throughout: real seed CG in f64, complex (c128) shifted recurrences, fields and J",
        "data": "synthetic",
        "config": {"workload": cfg.name, "grid": list(cfg.n), "sources": cfg.n_s, "detectors": cfg.n_d,
                   "frequencies": cfg.n_freq, "n_params": cfg.n_p, "sketch": [cfg.ls, cfg.ld],
                   "solves_per_step": solves_per_step, "parallelism": f"rhs-shard x{world}",
                   "l2": (f"working set ~{ws_bytes / 1e9:.1f} GB >> 126 MB L2 (no flush needed)" if flush is None
                          else f"working set ~{ws_bytes / 1e6:.0f} MB: 256 MB L2 flush between timed steps"),
                   "cg_tol": gp.tol if hasattr(gp, "tol") else 1e-17},
        "krylov_iterations_per_s": (st["rhs_iterations"] - s0["rhs_iterations"]) / args.steps / (ms / 1e3),
        "seed_solves_per_step": (st["seeds_solved"] - s0["seeds_solved"]) / args.steps,
        "seed_iterations_per_s": (st["seed_iterations"] - s0["seed_iterations"]) / args.steps / (ms / 1e3),
        "mean_iters_per_solve": (st["rhs_iterations"] - s0["rhs_iterations"]) / max(st["rhs_solved"] - s0["rhs_solved"], 1),
        "roofline": roof,
        "jacobian": {"path": "block-sparse by basis (default)" if st["contract_flops"] < st["contract_flops_dense"]
                     else "dense DMMA GEMM",
                     "achieved_tflops": jf, "peak_tflops": fpk, "frac": jf / fpk, "peak_source": fsrc,
                     "dense_gemm": dense_gemm,
                     "support_K": st["support_K"], "flops_per_step": (st["contract_flops"] - s0["contract_flops"]) / args.steps,
                     "ms_per_step": (st["contract_ms"] - s0["contract_ms"]) / args.steps,
                     "dense_equivalent_tflops": st["contract_flops_dense"] / max(st["contract_ms"], 1e-9) / 1e9,
                     # executed DMMA flops of the segment GEMM (3 real products per complex one, padded
                     # tiles included) over the whole contraction time (prescale and small panels too):
                     # a lower bound of the FP64 tensor-pipe utilisation
                     "dmma_executed_tflops": (st["contract_dmma_flops"] - s0["contract_dmma_flops"])
                     / max(st["contract_ms"] - s0["contract_ms"], 1e-9) / 1e9,
                     "dmma_executed_frac": (st["contract_dmma_flops"] - s0["contract_dmma_flops"])
                     / max(st["contract_ms"] - s0["contract_ms"], 1e-9) / 1e9 / fpk,
                     # the segment-GEMM calls alone (large panels: the full-data Jacobian), apart from
                     # the small-panel sketched / optimized-direction contractions (few flops, latency-bound)
                     "gemm": gemm_line(st, s0, args.steps, fpk),
                     "note": ("block-sparse by basis (PAPER.md L972): useful flops = 4 per (pair, point, parameter) "
                              "with a nonzero dA/dp block (the 3-multiply complex GEMM executes 6, so frac <= 0.70); "
                              "dense_equivalent counts the K x n_p GEMM it replaces")},
        "cpu_baseline": cpu,
        "solver": "multi-shift CG: one real seed per (source|detector) column serves all n_freq frequencies",
        "e2e": e2e,
        "gpu_launches": int(st["kernel_launches"] - s0["kernel_launches"]),
        "clocks": clocks,
        "misfit": out["misfit"] if out else None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
