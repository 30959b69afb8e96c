"""Benchmark of the hot path: batched f(theta) evaluations (+ the numbers
that explain them) on the BASELINE workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--selinv]

Workload (BASELINE.json configs[1], the largest CPU-runnable config the
metric is quoted on): Poisson spatial GMRF, 200x200 SPDE lattice
(n = 40 003, m = 100 000, dim(theta) = 2), seeded synthetic data
(paper_2204_04678_b200/synth.py).  One STEP = one central finite-difference
gradient batch (2d+1 = 5 f(theta) evaluations, warm started from the
accepted iterate like fit.py) PER GPU; at N GPUs every rank evaluates its own
disjoint 5 theta points (theta sharding, weak scaling).  Each f(theta) runs
the full inner Newton loop: assembly, tile factorizations of Q_c, solves,
step halving, the prior factorization and the f assembly.

Reported:
  value      f-evals/s over all ranks, device-timed (engine stream events),
             model data resident in HBM (the per-GPU working set, 5 slots of
             tile factors ~1 GB, is larger than the 126 MB L2).
  e2e        same metric through the public API fd_gradient(...) with host
             theta / warm-start buffers, H2D and D2H inside the timed region.
  roofline   dominant kernel = the tile-DAG factorization (DMMA fp64):
             algorithmic flops of the tile algorithm x active slots per
             launch / average launch time, vs the measured fp64 DGEMM peak.
  cpu_baseline  the CPU oracle (C restatement of the reference numerics,
             reference ND ordering) on a bounded sample, host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "f(theta) evaluations/s (batched FD-gradient stencils, Poisson SPDE 200x200, n=40003)"
UNIT = "f-evals/s"


# ---------------------------------------------------------------------------
def clock_sampler(stop: threading.Event, out: list, device: int):
    cmd = ["nvidia-smi", f"--id={device}",
           "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
           "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
           "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
           "--format=csv,noheader,nounits"]
    while not stop.is_set():
        try:
            line = subprocess.run(cmd, capture_output=True, text=True, timeout=5).stdout.strip()
            if line:
                out.append([x.strip() for x in line.split(",")])
        except Exception:
            pass
        stop.wait(0.2)


def summarize_clocks(samples):
    if not samples:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
    sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
    mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = sorted({names[i] for s in samples for i in range(4)
                      if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": reasons, "samples": len(samples)}


def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["fp64_dgemm_tflops"]), "measured cuBLAS DGEMM 8192^3 (profiles/fp64_peak.json)"
    return 35.45, "fallback (round-1 measurement)"


def traffic_from_profile(avg_slots):
    """DRAM bytes of one factor launch from the committed ncu --set full
    capture (a 5-slot launch), scaled to the bench's average active slots
    per launch (each slot reads/writes its own tile factors)."""
    path = os.path.join(ROOT, "profiles", "factor_ncu_r01.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d["dram_bytes_per_launch"] * avg_slots / d.get("slots", 5)
    return None


def stencil(theta, eps=5e-3):
    d = theta.size
    pts = [theta.copy()]
    for i in range(d):
        e = np.zeros(d)
        e[i] = eps
        pts += [theta + e, theta - e]
    return pts


# ---------------------------------------------------------------------------
def reference_budget(d):
    """runtime.py:64-71 default_budget on this host: level 1 up to the FD batch
    width 2d+1, the remaining cores to level 2 (tree-parallel factorization)."""
    try:
        import psutil

        cores = psutil.cpu_count(logical=False) or os.cpu_count() or 1
    except Exception:
        cores = os.cpu_count() or 1
    l1 = max(1, min(2 * max(d, 1) + 1, cores))
    return l1, max(1, cores // l1)


def cpu_port_batch(inst, theta, warm, threads, l2=1):
    """Time the oracle (reference numerics, ND ordering, level-1 x level-2
    threads) on one FD batch."""
    from oracle.oracle import OracleEvaluator

    t0 = time.perf_counter()
    orc = OracleEvaluator(inst.spec, inst.y)
    t_an = time.perf_counter() - t0
    pts = stencil(theta)
    if warm is None:
        warm = orc.mode(theta)[0]
    t1 = time.perf_counter()
    vals = orc.eval_batch(pts, warm=warm, threads=threads, l2=l2)
    dt = time.perf_counter() - t1
    return len(pts), dt, t_an, vals, orc, warm


def run_reference(args, rank):
    """--impl reference: the reference's CPU implementation of the path
    (oracle port of its numerics; the Python reference cannot travel to the
    GPU box), all host threads, same metric/config."""
    if rank != 0:
        return
    from paper_2204_04678_b200.synth import make_instance

    inst = make_instance(args.config)
    theta = inst.theta_true
    threads, l2 = reference_budget(theta.size)
    # warm-up (analysis + cold mode for the warm start + W batches)
    n, dt, t_an, _, orc, warm = cpu_port_batch(inst, theta, None, threads, l2)
    for _ in range(max(0, args.warmup - 1)):
        orc.eval_batch(stencil(theta), warm=warm, threads=threads, l2=l2)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        orc.eval_batch(stencil(theta), warm=warm, threads=threads, l2=l2)
    T = time.perf_counter() - t0
    v = args.steps * n / T
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * T / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)",
        "config": {"workload": f"{args.config}: FD central batch of 2d+1=5 f(theta) per step",
                   "ordering": "reference nested dissection (restated)",
                   "budget": f"{threads}:{l2} (default_budget, runtime.py:64-71)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads * l2, "kind": "port",
                         "sample": f"{args.steps} FD batches x {n} f(theta), warm started; "
                                   f"ThreadBudget({threads}, {l2}): points x tree tasks"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch

    # PINLA_BENCH_SHARED_GPU=1: functional check of the multi-rank code path
    # with every rank on GPU 0 over gloo (numbers meaningless, never reported)
    shared = os.environ.get("PINLA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2204_04678_b200.fit import FitObjective
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.optimizer import FDConfig, fd_gradient
    from paper_2204_04678_b200.synth import make_instance

    inst = make_instance(args.config)
    d = inst.theta_true.size
    k = 2 * d + 1
    t_create = time.perf_counter()
    ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=k, device=local)
    create_s = time.perf_counter() - t_create
    eng = ev.engine
    # this rank's disjoint theta points: a shifted stencil per rank
    theta_r = inst.theta_true + 0.01 * rank
    pts = np.array(stencil(theta_r))
    warm, its, st, _, _ = eng.mode(theta_r)  # the accepted iterate's mode
    assert st == 0, "mode failed at the benchmark point"

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up
    for _ in range(args.warmup):
        eng.eval_batch(pts, warm)
    torch.cuda.synchronize()

    # ---- timed: device-resident path
    samples, stop = [], threading.Event()
    sampler = threading.Thread(target=clock_sampler, args=(stop, samples, local), daemon=True)
    eng.reset_stats()
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    dev_ms = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = eng.eval_batch(pts, warm)
        dev_ms += eng.stats()["last_call_ms"]
    e1.record()
    torch.cuda.synchronize()
    barrier()
    stop.set()
    sampler.join(timeout=5)
    st_stats = eng.stats()
    assert np.all(res["status"] == 0)
    T = max_over_ranks(dev_ms / 1000.0)
    value = world * k * args.steps / T

    # ---- roofline of the dominant kernel (tile-DAG factorization)
    peak_tf, peak_src = fp64_peak()
    # algorithmic flops = what the row/col-limited tile kernels execute per slot
    # (Sigma over update pairs of 2*m*n*k with tile heights rounded to 8/8/4,
    # + TRSM + diagonal POTRI), times the active slots of each launch
    fl_launch_avg = st_stats["factor_flops_limited"] * st_stats["factor_slot_runs"] / max(1, st_stats["factor_launches"])
    ms_launch_avg = st_stats["factor_ms"] / max(1, st_stats["factor_launches"])
    achieved = fl_launch_avg / (ms_launch_avg * 1e-3) / 1e12
    share = st_stats["factor_ms"] / max(1e-9, dev_ms)
    avg_slots = st_stats["factor_slot_runs"] / max(1, st_stats["factor_launches"])

    # ---- e2e through the public API (host buffers)
    obj = FitObjective(ev, extrapolate=False, reuse_accepted=False)  # the reference's objective semantics
    obj.warm = warm.copy()
    fd = FDConfig(scheme="central")
    for _ in range(2):
        fd_gradient(obj, theta_r, fd)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        g, f0 = fd_gradient(obj, theta_r.copy(), fd)
    torch.cuda.synchronize()
    barrier()
    T_e2e = max_over_ranks(time.perf_counter() - t0)
    e2e = world * k * args.steps / T_e2e
    h2d = k * d * 8 + inst.n * 8  # theta batch + warm start
    d2h = k * (8 + 5 * 8 + 4 + 8 + 4 + 2 * 8)  # f, comps, status, badcol, iters, logdets

    # ---- full optimisation wall time through the public fit() (rank 0,
    # N = 1): optimize (FD batches + parallel line search + final Hessian
    # stencil) -> explore -> latent marginals (selected inversion)
    # (N > 1: every theta batch sharded over the ranks, FitConfig.shard; the
    # ranks run the optimizer in lockstep; wall time = max over ranks)
    full_fit = None
    from paper_2204_04678_b200.fit import FitConfig, fit

    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fr = fit(inst.spec, inst.y, FitConfig(shard=world > 1), evaluator=ev)
    torch.cuda.synchronize()
    fit_wall = max_over_ranks(time.perf_counter() - t0)
    if rank == 0:
        sm = fr.summary()
        full_fit = {"wall_s": fit_wall, "n_fn_evals": sm["n_fn_evals"],
                    "iterations": sm["iterations"], "status": sm["status"],
                    "theta_mode": sm["theta_mode"], "f_mode": sm["f_mode"],
                    "note": "fit() from theta0 = 0 with the reference defaults (mixed FD, "
                            "5 line-search candidates); engine analysis done before (create_s); "
                            f"theta batches sharded over {world} rank(s); n_fn_evals = rank 0's",
                    "create_s": create_s}

    # ---- CPU baseline (rank 0, N = 1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads, l2 = reference_budget(theta_r.size)
        n, dt, t_an, vals, _, _ = cpu_port_batch(inst, theta_r, warm, threads, l2)
        ours = res["f"]
        cpu = {"value": n / dt, "unit": UNIT, "cores": threads * l2, "kind": "port",
               "sample": f"1 FD batch = {n} warm-started f(theta) on {args.config}, "
                         f"ThreadBudget({threads}, {l2}); "
                         f"analysis {t_an:.1f}s excluded; max |f_gpu - f_cpu|/|f| = "
                         f"{float(np.max(np.abs(np.array(vals) - ours) / np.abs(ours))):.2e}"}

    if full_fit is not None and cpu is not None:
        full_fit["cpu_port_estimate_s"] = full_fit["n_fn_evals"] / cpu["value"]
        full_fit["cpu_port_estimate_note"] = "n_fn_evals / cpu_baseline f-evals/s (warm-started rate)"
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * T / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, paper_2204_04678_b200/synth.py)",
            "config": {"workload": f"{args.config}: per GPU one central FD batch of 2d+1={k} "
                                   "warm-started f(theta) per step",
                       "n": inst.n, "m": inst.spec.m, "dim_theta": d,
                       "parallelism": f"theta-sharding x{world}",
                       "l2": "working set (5 slots of tile factors, ~1.3 GB) > 126 MB L2; no flush",
                       "newton_iterations": res["iters"].tolist()},
            "roofline": {"bound": "tensor", "kernel": "factor_kernel (tile-DAG Cholesky, DMMA fp64)",
                         "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "peak_source": peak_src,
                         "traffic": traffic_from_profile(avg_slots),
                         "traffic_source": "profiles/factor_ncu_r01.json (5-slot launch) x avg slots/5",
                         "flops_per_launch": fl_launch_avg, "ms_per_launch": ms_launch_avg,
                         "flops_per_slot_dense_tiles": st_stats["factor_flops"],
                         "flops_per_slot_executed": st_stats["factor_flops_limited"],
                         "share_of_step": share},
            "phases_ms_per_step": {kk: st_stats[kk] / args.steps for kk in
                                   ("factor_ms", "solve_ms", "assemble_ms")},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(st_stats["kernel_launches"]),
            "clocks": summarize_clocks(samples),
            "cpu_baseline": cpu,
            "full_fit": full_fit,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
