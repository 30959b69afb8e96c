"""Benchmark of the hot path: batched f(theta) evaluations and selected
inversion on the largest single-GPU BASELINE workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c4] [--no-cpu-baseline] [--no-c5-selinv] [--full-fit]

Workload (BASELINE.json configs[3], c4, the largest configuration whose
f(theta) fits one B200): AR(1) (x) SPDE on a 64x64 grid x 250 time points plus
8 fixed effects (n = 1 024 008, m = 2 000 000 Gaussian observations,
dim(theta) = 4), seeded synthetic data (paper_2204_04678_b200/synth.py).
One STEP = one central finite-difference gradient stencil of 2d+1 = 9
f(theta) evaluations around the accepted iterate, warm started from its
mode (fit.py).  At N GPUs the SAME stencil is sharded over the ranks with
``distributed.ThetaSharding`` (slot s on rank s mod N; NCCL broadcast of the
theta batch + all_gather of the slot results): strong scaling, a step is
done when every slot is.  The device holds as many slots as its memory
allows (c4: 3 slots of tile factors, 160 GB), so a rank runs its slots in
waves.  Each f(theta) = Q_c assembly + tile-DAG Cholesky (DMMA fp64) +
forward/backward solve + the f assembly (prior log det analytic).

Reported (one JSON line, rank 0):
  value       f-evals/s over the whole job, CUDA events around the K steps
              (model data resident in HBM; max over ranks).
  e2e         the same stencil through the public API fd_gradient(...) with
              host theta / warm-start buffers (H2D, D2H inside the timed region).
  roofline    dominant kernel = factor_ws_kernel (warp-specialised TMA factor kernel): executed tile flops per launch
              / average launch time (engine-stream CUDA events) vs the fp64
              DGEMM peak measured in this run; also on SURVEY s8d's dense-BTA
              count F_chol.
  hbm         solve_kernel and the assembly kernels: algorithmic bytes /
              their event time vs MEASURED_PEAKS.json hbm_gbs.
  selinv      selected inversion (block Takahashi, all n marginal variances)
              at theta_true on c4 and at the c5 fit's theta* (c5 in a second
              handle after the c4 one is freed).
  cpu_baseline  the CPU port of the reference numerics (reference ND
              ordering) on a reduced n_t instance of the same config, scaled
              linearly in n_t (an UPPER bound on the CPU's full-size rate: the
              ND factor cost grows super-linearly in n_t).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "f-evals/s"
# c5 theta* of the full quasi-Newton fit on one B200 (profiles/fit_c3_c5_r01.jsonl,
# last c5 record): the selected inversion of the c5 run happens at this point
C5_THETA_STAR = [2.074604122113563, -1.6099448536318428, 1.3928321064694096,
                 2.2804659918916594, 0.19954226210863032]
# reduced n_t of the CPU sample per config (full spatial grid, m scaled with n_t)
CPU_SAMPLE_NT = {"c3": 4, "c4": 4, "c5": 4}


def metric_name(cfg, inst):
    return (f"f(theta) evaluations/s (central FD stencils of 2d+1 points, {cfg}: "
            f"n={inst.n}, m={inst.spec.m}, d={inst.theta_true.size})")


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi -lms 200 running beside the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            line = line.strip()
            if line:
                self.lines.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread is not None:
                self.thread.join(timeout=5)
        return summarize_clocks(self.lines)


def _num(x):
    try:
        return float(x)
    except ValueError:
        return None


def summarize_clocks(samples):
    if not samples:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
    sm = [v for v in (_num(s[0]) for s in samples) if v is not None]
    mx = [v for v in (_num(s[1]) for s in samples) if v is not None]
    pw = [v for v in (_num(s[2]) for s in samples if len(s) > 2) if v is not None]
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = sorted({names[i] for s in samples for i in range(4)
                      if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "power_w_median": float(np.median(pw)) if pw else None,
            "reasons": reasons, "samples": len(samples)}


def measure_fp64_peak(device):
    """cuBLAS DGEMM 8192^3 (torch.matmul fp64), best of 10 after 3 warm-ups,
    with clocks sampled: the roofline denominator of the DMMA kernels,
    measured on this box in this run."""
    import torch

    n = 8192
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    clk = ClockSampler(device).start()
    best = math.inf
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    clocks = clk.stop()
    del a, b, c
    torch.cuda.empty_cache()
    return {"tflops": 2.0 * n ** 3 / (best * 1e-3) / 1e12, "how": "cuBLAS DGEMM 8192^3 "
            "(torch.matmul fp64), best of 10, this run", "clocks": clocks}


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return float(json.load(open(path))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def stencil(theta, eps=5e-3):
    """The central FD point list of fd_gradient (optimizer.py:119-130)."""
    d = theta.size
    pts = [theta.copy()]
    for i in range(d):
        e = np.zeros(d)
        e[i] = eps
        pts += [theta + e, theta - e]
    return pts


def f_chol_dense_bta(inst):
    """SURVEY s8d dense-BTA Cholesky count: (n_t - 1) 7/3 n_s^3 + n_s^3 / 3
    (+ the arrow, negligible)."""
    c = inst.spec.components[0]
    if c.kind != "ar1_spde2d":
        return None
    ns, nt = c.graph.n, c.nt
    return (nt - 1) * 7.0 / 3.0 * ns ** 3 + ns ** 3 / 3.0


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


def cpu_sample_instance(cfg):
    """A reduced-n_t instance of ``cfg`` with the full spatial grid and m
    scaled with n_t, and the factor that scales its rate to the full size."""
    from paper_2204_04678_b200.synth import CONFIGS, make_instance

    full = CONFIGS[cfg]
    if cfg in CPU_SAMPLE_NT and full["nt"] > CPU_SAMPLE_NT[cfg]:
        nt = CPU_SAMPLE_NT[cfg]
        inst = make_instance(cfg, nt=nt, m=full["m"] * nt // full["nt"])
        return inst, nt / full["nt"], f"{cfg} with n_t={nt} (n={inst.n}, m={inst.spec.m}), " \
                                      f"rate x {nt}/{full['nt']} (linear in n_t: an upper bound)"
    inst = make_instance(cfg)
    return inst, 1.0, f"{cfg} full size"


def cpu_stencil_rate(cfg, steps=1):
    """The CPU port of the reference numerics (oracle: reference ND ordering,
    reference Newton loop, C restatement of kernels.py) on central FD
    stencils of the sample instance, ThreadBudget = the reference default.
    Returns (full-size-scaled f-evals/s, cores, sample text, per-step rates)."""
    from oracle.oracle import OracleEvaluator

    inst, scale, what = cpu_sample_instance(cfg)
    theta = inst.theta_true
    l1, l2 = reference_budget(theta.size)
    t0 = time.perf_counter()
    orc = OracleEvaluator(inst.spec, inst.y)
    t_an = time.perf_counter() - t0
    warm = orc.mode(theta)[0]  # the accepted iterate's mode
    rates = []
    pts = stencil(theta)
    for _ in range(steps):
        t1 = time.perf_counter()
        orc.eval_batch(pts, warm=warm, threads=l1, l2=l2)
        rates.append(len(pts) / (time.perf_counter() - t1) * scale)
    rate = len(rates) / sum(1.0 / r for r in rates)
    sample = (f"{steps} central FD stencil(s) of {len(pts)} warm-started f(theta) on {what}; "
              f"ThreadBudget({l1}, {l2}) (points x tree tasks); analysis {t_an:.1f}s excluded")
    return rate, l1 * l2, sample, rates


def run_reference(args, rank):
    """--impl reference: the reference's CPU implementation of the path (the
    oracle port of its numerics; the Python reference cannot travel to the
    GPU box), all host threads, same metric / config / unit."""
    if rank != 0:
        return
    steps = args.steps
    # each step a bounded sample: warm-up then K stencils of the reduced instance
    rate, cores, sample, rates = cpu_stencil_rate(args.config, steps=max(1, steps))
    full = make_meta(args.config)
    line = {
        "impl": "reference", "metric": full["metric"], "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * full["k"] / rate, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
        "config": {"workload": full["workload"], "ordering": "reference nested dissection (restated)"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample, "per_step": rates},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_meta(cfg):
    from paper_2204_04678_b200.synth import CONFIGS

    c = CONFIGS[cfg]
    n = c["nx"] * c["ny"] * c["nt"] + c["p"] + (c["nt"] if c.get("temporal") else 0)
    d = (1 if c["family"] == "gaussian" else 0) + (3 if c["nt"] > 1 else 2) + (2 if c.get("temporal") else 0)
    k = 2 * d + 1
    return {"k": k, "metric": f"f(theta) evaluations/s (central FD stencils of 2d+1 points, {cfg}: "
                              f"n={n}, m={c['m']}, d={d})",
            "workload": f"{cfg}: one central FD stencil of 2d+1={k} warm-started f(theta) per "
                        f"step, sharded over the GPUs (strong scaling)"}


# ---------------------------------------------------------------------------
def spawn_ranks(args):
    """--gpus N without a torchrun environment: re-launch this script under
    torch.distributed.run with N ranks on 127.0.0.1."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class DeviceStencil:
    """Batch objective over the resident engine: warm-started f at every point
    (the `value` leg: no host-side bookkeeping beyond the C-ABI call)."""

    def __init__(self, engine, warm):
        self.engine = engine
        self.warm = warm
        self.last = None

    def eval_batch(self, points):
        res = self.engine.eval_batch(np.stack(points), self.warm)
        self.last = res
        if np.any(res["status"] != 0):
            raise RuntimeError(f"bench point failed: status {res['status'].tolist()}")
        return [float(v) for v in res["f"]]


def factor_traffic(config, slots):
    """DRAM bytes of one factor launch of the bench workload, from the committed ncu capture
    (`tools/gpu_round.sh factordram`: single-pass dram__bytes counters of one full-size launch;
    a --set full replay would have to save and restore the 105 GB the launch overwrites)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "factor_dram_c4_r02.csv")
    if config != "c4" or slots != 3 or not os.path.exists(path):
        return None, "no ncu DRAM capture for this configuration (profiles/factor_dram_c4_r02.csv is c4 x 3 slots)"
    rd = wr = None
    for line in open(path):
        f = [x.strip('"') for x in line.strip().split('","')]
        if len(f) > 2 and f[-3] == "dram__bytes_read.sum":
            rd = float(f[-1])
        if len(f) > 2 and f[-3] == "dram__bytes_write.sum":
            wr = float(f[-1])
    if rd is None or wr is None:
        return None, "profiles/factor_dram_c4_r02.csv unreadable"
    return rd + wr, ("ncu dram__bytes_read.sum + dram__bytes_write.sum of one full c4 3-slot factor_ws_kernel launch "
                     "(profiles/factor_dram_c4_r02.csv): the operand tiles of every pair product stream from DRAM "
                     "(L2 turnover ~40 us); compulsory traffic (Q in, L out) is 0.1 TB")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5-selinv", action="store_true")
    ap.add_argument("--full-fit", action="store_true",
                    help="also run fit() (optimize + explore + marginals) on the config")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":
            return run_reference(args, 0)
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")

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
    from paper_2204_04678_b200.distributed import ThetaSharding
    from paper_2204_04678_b200.fit import FitObjective
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.optimizer import FDConfig, fd_gradient
    from paper_2204_04678_b200.synth import make_instance

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    fp64 = measure_fp64_peak(local)
    hbm, hbm_src = hbm_peak()

    t0 = time.perf_counter()
    inst = make_instance(args.config)
    gen_s = time.perf_counter() - t0
    d = inst.theta_true.size
    k = 2 * d + 1
    t0 = time.perf_counter()
    ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=k, device=local)
    create_s = time.perf_counter() - t0
    eng = ev.engine
    theta = inst.theta_true.copy()
    pts = stencil(theta)
    warm, its, st, _, _ = eng.mode(theta)  # the accepted iterate's mode
    assert st == 0, "mode failed at the benchmark point"
    dev_obj = DeviceStencil(eng, warm)
    run = ThetaSharding(dev_obj) if world > 1 else dev_obj

    # ---- warm-up
    for _ in range(args.warmup):
        run.eval_batch(pts)
    barrier()

    # ---- timed: device-resident path (CUDA events on the current stream
    # bracket the K steps; the engine's own stream is synchronized by each
    # step's result read-back, so the interval covers all of its kernels)
    eng.reset_stats()
    clk = ClockSampler(local).start()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        fvals = run.eval_batch(pts)
    e1.record()
    barrier()
    clocks = clk.stop()
    my_ms = e0.elapsed_time(e1)
    ss = eng.stats()
    T = max_over_ranks(my_ms / 1000.0)
    value = k * args.steps / T

    # ---- the dominant kernel (tile-DAG factorization) and the HBM kernels
    launches = max(1, ss["factor_launches"])
    slots_per_launch = ss["factor_slot_runs"] / launches
    fl_exec = ss["factor_flops_limited"] * slots_per_launch
    ms_launch = ss["factor_ms"] / launches
    achieved = fl_exec / (ms_launch * 1e-3) / 1e12
    fchol = f_chol_dense_bta(inst)
    step_ms_dev = ss["factor_ms"] + ss["solve_ms"] + ss["assemble_ms"]
    solve_gbs = (ss["solve_bytes"] * ss["solve_slot_runs"] / (ss["solve_kernel_ms"] * 1e-3) / 1e9
                 if ss["solve_kernel_ms"] > 0 else None)
    asm_gbs = (ss["assemble_bytes_done"] / (ss["assemble_ms"] * 1e-3) / 1e9
               if ss["assemble_ms"] > 0 else None)
    traffic, traffic_note = factor_traffic(args.config, int(round(slots_per_launch)))
    roofline = {
        "bound": "tensor", "kernel": "factor_ws_kernel (tile-DAG Cholesky: producer warp + TMA box loads, 8 DMMA warps per SM, fp64)",
        "achieved": achieved, "peak": fp64["tflops"], "unit": "TFLOP/s",
        "frac": achieved / fp64["tflops"], "peak_source": fp64["how"],
        "traffic": traffic,
        "traffic_note": traffic_note,
        "flops_per_launch": fl_exec, "ms_per_launch": ms_launch,
        "flops_per_slot_executed": ss["factor_flops_limited"],
        "flops_per_slot_dense_tiles": ss["factor_flops"],
        "share_of_step": ss["factor_ms"] / max(1e-9, my_ms),
    }
    if fchol:
        roofline["f_chol_dense_bta"] = fchol
        roofline["achieved_on_f_chol"] = fchol * slots_per_launch / (ms_launch * 1e-3) / 1e12
        roofline["f_chol_note"] = ("SURVEY s8d dense-BTA count; the tile DAG skips the "
                                   "structurally zero tiles of the BTA blocks, so this rate can "
                                   "exceed the DGEMM peak")
    hbm_kernels = {
        "peak_gbs": hbm, "peak_source": hbm_src,
        "solve_kernel": {"achieved_gbs": solve_gbs, "frac": solve_gbs / hbm if solve_gbs else None,
                         "bytes_per_slot_solve": ss["solve_bytes"],
                         "ms_per_slot_solve": ss["solve_kernel_ms"] / max(1, ss["solve_slot_runs"])},
        "assembly": {"achieved_gbs": asm_gbs, "frac": asm_gbs / hbm if asm_gbs else None,
                     "bytes_per_slot": ss["assemble_bytes"],
                     "ms_per_step": ss["assemble_ms"] / args.steps},
    }

    # ---- e2e through the public API (host buffers): fd_gradient on the fit
    # objective with the reference's semantics (warm start = accepted mode)
    obj = FitObjective(ev, extrapolate=False, reuse_accepted=False)
    obj.warm = warm.copy()
    fobj = ThetaSharding(obj) if world > 1 else obj
    fd = FDConfig(scheme="central")
    fd_gradient(fobj, theta, fd)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        g, f0 = fd_gradient(fobj, theta.copy(), fd)
    barrier()
    T_e2e = max_over_ranks(time.perf_counter() - t0)
    e2e = k * e2e_steps / T_e2e
    mine = len(range(rank, k, world))
    h2d = mine * (d * 8 + inst.n * 8)  # theta rows + the warm start per device call
    d2h = mine * (8 + 5 * 8 + 4 + 8 + 4 + 2 * 8)  # f, comps, status, badcol, iters, logdets

    # ---- selected inversion (c4 at theta_true; every rank, timed on rank 0)
    sel = {}
    eng.reset_stats()
    t0 = time.perf_counter()
    var, _ = ev.marginal_variances(theta, warm)
    wall = time.perf_counter() - t0
    s2 = eng.stats()
    sel[args.config] = {"selinv_s": s2["selinv_ms"] / 1000.0, "call_s": wall,
                        "tflops": s2["selinv_flops"] / (s2["selinv_ms"] * 1e-3) / 1e12,
                        "frac": s2["selinv_flops"] / (s2["selinv_ms"] * 1e-3) / 1e12 / fp64["tflops"],
                        "flops": s2["selinv_flops"], "theta": "theta_true",
                        "var_min_max": [float(var.min()), float(var.max())]}

    full_fit = None
    if args.full_fit:
        from paper_2204_04678_b200.fit import FitConfig, fit

        barrier()
        t0 = time.perf_counter()
        fr = fit(inst.spec, inst.y, FitConfig(shard=world > 1, fd=FDConfig(scheme="central")),
                 evaluator=ev)
        fit_wall = max_over_ranks(time.perf_counter() - t0)
        sm = fr.summary()
        full_fit = {"wall_s": fit_wall, "n_fn_evals": sm["n_fn_evals"], "iterations": sm["iterations"],
                    "status": sm["status"], "theta_mode": sm["theta_mode"], "f_mode": sm["f_mode"],
                    "create_s": create_s}
    ev.close()
    del ev, eng
    torch.cuda.empty_cache()

    if not args.no_c5_selinv and args.config != "c5":
        inst5 = make_instance("c5")
        ev5 = ObjectiveEvaluator(inst5.spec, inst5.y, max_slots=1, device=local)
        th5 = np.array(C5_THETA_STAR)
        ev5.engine.reset_stats()
        t0 = time.perf_counter()
        var5, _ = ev5.marginal_variances(th5)
        wall = time.perf_counter() - t0
        s5 = ev5.engine.stats()
        sel["c5"] = {"selinv_s": s5["selinv_ms"] / 1000.0, "call_s": wall,
                     "tflops": s5["selinv_flops"] / (s5["selinv_ms"] * 1e-3) / 1e12,
                     "frac": s5["selinv_flops"] / (s5["selinv_ms"] * 1e-3) / 1e12 / fp64["tflops"],
                     "flops": s5["selinv_flops"], "theta": "c5 fit theta* (C5_THETA_STAR)",
                     "call_note": "call = cold Newton mode (Poisson) + selinv",
                     "var_min_max": [float(var5.min()), float(var5.max())]}
        ev5.close()
        del ev5

    # ---- CPU baseline (rank 0, N = 1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, sample, _ = cpu_stencil_rate(args.config, steps=1)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": metric_name(args.config, inst), "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * T / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, paper_2204_04678_b200/synth.py)",
            "config": {"workload": make_meta(args.config)["workload"],
                       "n": inst.n, "m": inst.spec.m, "dim_theta": d,
                       "parallelism": f"theta-sharding x{world} (slot s on rank s mod {world})",
                       "slots_per_gpu": int(ss["slots"]),
                       "l2": "inputs larger than L2 (one slot of tile factors ~35 GB >> 126 MB); no flush",
                       "newton_iterations": (dev_obj.last["iters"].tolist()
                                             if dev_obj.last is not None else None),
                       "gen_s": gen_s, "create_s": create_s},
            "roofline": roofline,
            "hbm_kernels": hbm_kernels,
            "phases_ms_per_step": {"factor_ms": ss["factor_ms"] / args.steps,
                                   "solve_ms": ss["solve_ms"] / args.steps,
                                   "solve_kernel_ms": ss["solve_kernel_ms"] / args.steps,
                                   "assemble_ms": ss["assemble_ms"] / args.steps,
                                   "device_sum_ms": step_ms_dev / args.steps},
            "selinv": sel,
            "selinv_s": sel[args.config]["selinv_s"],
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "api": "fd_gradient(FitObjective, theta, FDConfig('central'))"},
            "gpu_launches": int(ss["kernel_launches"]),
            "clocks": clocks,
            "fp64_peak": fp64,
            "cpu_baseline": cpu,
            "full_fit": full_fit,
            "f_at_theta": fvals[0],
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
