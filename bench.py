#!/usr/bin/env python
"""bench.py — throughput of the B200 EP N-particle hot path on BASELINE config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--path dense|cell|auto]

One "step" = one 100-step classical RK4 shooting solve (T = 1, 400 RHS evaluations) of
BASELINE.json configs[1]: N = 16384 particles uniform in [0,1]^2 (seed 0), momenta
N(0, 0.01^2) (seed 1), conical kernel with support radius sigma = 0.05 (KD-1: alpha =
sigma / (53 ln 2)).  The metric is particle-pair interactions per second in the RHS,
counting the reference's N^2 ordered pairs per RHS (particles.py:79-117 evaluates all of
them) for the dense path and the accepted pairs (d < sigma, plus the N self terms) for the
cell-list path.  Inputs are device resident for `value`; `e2e` times the public API on
host arrays (H2D + D2H inside the timed region).

Multi-GPU (torchrun, N > 1): target rows are sharded across ranks and the stage state is
all-gathered over NCCL per RK stage (paper_1510_03816_b200/sharded.py); the total work is
fixed ("strong" scaling), time is the max over ranks of CUDA-event device time.

`--impl reference` times the reference's CPU algorithm (the numpy restatement in
oracle/restate.py, which reproduces geoshoot.rhs bit for bit) on the host cores, rank 0
only, each step a bounded row sample of the same RHS workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

if "--impl" in sys.argv and "reference" in sys.argv:
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "particle-pair interactions/s in N-particle RHS (fp64)"
UNIT = "pairs/s"
W_ALG = 45  # DP-pipe issue slots per ordered pair, libm formulation = 90 flop-equivalents
# FP64-pipe instructions the implemented kernels issue per evaluated pair (SASS of the inner
# loops, profiles/r01_history.md): symmetric dense 31 per unordered pair = 15.5 per ordered pair;
# one-sided / cell-list ~28 per pair.  Used for the kernel's own FP64-pipe utilisation.
W_IMPL = {"sym": 15.5, "one_sided": 28.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="dense", choices=["dense", "cell", "auto"])
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--rk-steps", type=int, default=100)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the multi-GPU code path (ShardedSolver, NCCL) in a one-rank world (testing)")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi style clock / throttle-reason sampling during the timed region (pynvml)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def profile_traffic():
    """Per-launch DRAM bytes of the pair kernel from the committed ncu capture, if any."""
    path = os.path.join(REPO, "profiles", "ncu_pair_kernel.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


def arm_config(a, n):
    """The workload both arms report (BASELINE configs[1])."""
    return {"workload": f"C2: one {a.rk_steps}-step RK4 shooting solve (T=1, {4 * a.rk_steps} RHS) of N={n}, "
                        f"conical sigma=0.05 (KD-1), {a.path} path",
            "n": n, "rk_steps": a.rk_steps, "path": a.path}


# ---------------------------------------------------------------------------------------------
def reference_arm(a):
    """--impl reference: the reference's CPU algorithm (numpy restatement) on rank 0."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import restate
    from paper_1510_03816_b200 import configs

    w = configs.c2(a.n)
    k = restate.Kernel(0, w.alpha, True)
    rows = min(w.n, 1024)

    def step():
        restate.rhs_rows(k, 0.0, w.q, w.p, 0, rows)

    for _ in range(a.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    dt = time.perf_counter() - t0
    pairs = a.steps * rows * w.n
    value = pairs / dt
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE configs[1] recipe, seeds 0/1)",
        "config": dict(arm_config(a, w.n), parallelism="host cores",
                       sample=f"rows [0,{rows}) of one RHS per step (same pairs/s metric)"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"rows [0,{rows}) of one C2 RHS per step via oracle/restate.py (numpy, "
                                   "bitwise equal to geoshoot.rhs; elementwise on 1 core, BLAS on "
                                   f"{cores} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_port(w, spec_alpha, c1=None):
    """The C/OpenMP oracle port on all host cores, one RK4 step (4 RHS) of C2; with `c1`, also
    the reference's Algorithm 1 (numpy restatement, bitwise the reference) on config 1 — the
    CPU side of BASELINE's second metric, seconds per feedback iteration."""
    from oracle import native
    from oracle.restate import Kernel

    threads = native.max_threads()
    t0 = time.perf_counter()
    native.evolve(Kernel(0, spec_alpha, True), 0.0, w.q, w.p, 1.0, 1)
    dt = time.perf_counter() - t0
    out = {"value": 4.0 * w.n * w.n / dt, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"one RK4 step (4 dense RHS, N={w.n}) of C2 through oracle/gs_oracle.c (OpenMP, libm exp)",
           "seconds": dt, "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    if c1 is not None:
        from oracle import restate

        t0 = time.perf_counter()
        o = restate.match_momentum(Kernel(0, c1.alpha, True), 0.0, c1.q, c1.target, c1.h, c1.epsilon, c1.max_iter,
                                   "residual", "max", 1.0, c1.steps)
        out["c1_s_per_feedback_iteration"] = (time.perf_counter() - t0) / max(1, o["iterations"])
        out["c1_sample"] = "the whole C1 match (numpy restatement of geoshoot.match, momentum update, 1 core)"
    return out


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
        return
    import torch
    import torch.distributed as dist

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import configs, device, sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif a.force_sharded:
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(sk.getsockname()[1]))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    gs.set_path(a.path)

    w = configs.c2(a.n)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    ctx = N.Context.get(local)
    lib = ctx.lib
    q_d = torch.from_numpy(w.q).cuda()
    p_d = torch.from_numpy(w.p).cuda()
    solver = sharded.ShardedSolver(spec, force_split=a.force_sharded) if (world > 1 or a.force_sharded) else None

    def solve():
        if solver is not None:
            return solver.evolve(q_d, p_d, 1.0, a.rk_steps)
        return device.evolve(spec, q_d, p_d, 1.0, a.rk_steps)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2
    for _ in range(max(3, a.warmup)):
        solve()
    torch.cuda.synchronize()

    import ctypes

    lib.gs_profile_enable(ctx.handle, 1)
    pm, pl, ll, pp = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    lib.gs_profile_read(ctx.handle, ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(ll), ctypes.byref(pp), 1)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(a.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            starts[k].record()
            solve()
            ends[k].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib.gs_profile_read(ctx.handle, ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(ll), ctypes.byref(pp), 1)
    lib.gs_profile_enable(ctx.handle, 0)
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms, float(pp.value)], dtype=torch.float64, device="cuda")
    if world > 1:
        tp = t[1:].clone()
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tp, op=dist.ReduceOp.SUM)
        t[1] = tp[0]
    ms_max = float(t[0])
    total_pairs = float(t[1])          # evaluated ordered pairs, counted by the library (all ranks)
    pairs_per_rhs = total_pairs / (a.steps * 4 * a.rk_steps)
    value = total_pairs / (ms_max / 1e3)

    # roofline of the dominant kernel (pair kernel), measured live with CUDA events
    pair_ms_avg = pm.value / max(1, pl.value)
    pairs_per_launch = float(pp.value) / max(1, pl.value)
    ach_pairs = pairs_per_launch / (pair_ms_avg / 1e3)
    ach_tflops = ach_pairs * 2 * W_ALG / 1e12
    w_impl = W_IMPL["sym"] if (a.path == "dense" and w.n >= 1024) else W_IMPL["one_sided"]
    peak = None
    best = None
    for _ in range(3):
        pms, pfl = ctypes.c_double(), ctypes.c_double()
        lib.gs_fp64_peak_probe(ctx.handle, 20000, ctypes.byref(pms), ctypes.byref(pfl), None)
        r = pfl.value / (pms.value / 1e3) / 1e12
        best = r if best is None else max(best, r)
    peak = best
    traffic, _ = profile_traffic()

    # e2e: the public API on host arrays (H2D + D2H inside the timed region)
    e2e_reps = max(1, min(3, a.steps))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_reps):
        if solver is not None:
            qT, pT = solver.evolve(w.q, w.p, 1.0, a.rk_steps)
            qT.cpu(), pT.cpu()
        else:
            gs.evolve(spec, gs.ParticleState(w.q, w.p), gs.EvolveConfig(t_final=1.0, steps=a.rk_steps))
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = e2e_reps * 4 * a.rk_steps * pairs_per_rhs / float(te[0])

    extras = {}
    if rank == 0 and not a.no_extras:
        extras = run_extras(a, gs, device, configs, torch)
    if rank == 0:
        cpu = cpu_baseline_port(w, w.alpha, None if a.no_extras else configs.c1())
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (BASELINE configs[1] recipe: uniform [0,1]^2 seed 0, N(0,0.01^2) seed 1)",
            "config": dict(arm_config(a, w.n), parallelism=(
                f"rows{world}" if solver is None else
                f"{'pair-split' if a.path == 'dense' else 'rows'}{world}+{'p2p' if solver.p2p else 'nccl'}"),
                           l2="flushed between timed steps (256 MB write)"),
            "roofline": {"bound": "fp64", "achieved": ach_tflops, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach_tflops / peak if peak else None, "traffic": traffic,
                         "kernel": ("gsb::k_dense_sym (symmetric, 1 GPU) / gsb::k_dense_partial (row shards)"
                                    if a.path == "dense" else "gsb::k_cell_pair"),
                         "avg_launch_ms": pair_ms_avg, "pairs_per_launch": pairs_per_launch,
                         "work_per_pair": f"{W_ALG} DP-pipe slots = {2 * W_ALG} flop-equivalents (SURVEY.md §8(d))",
                         "peak_source": "measured live: gs_fp64_peak_probe (DFMA chains on all SMs, best of 3)",
                         # the implemented kernel's own FP64-pipe utilisation: issued FP64 slots
                         # per pair (SASS) x pairs/s against the peak slot rate (= peak / 2)
                         "fp64_pipe_frac": (ach_pairs * w_impl / (peak * 1e12 / 2)) if peak else None,
                         "fp64_slots_per_pair_implemented": w_impl},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * w.n * 2 * 8,
                    "d2h_bytes_per_step": 2 * w.n * 2 * 8,
                    "api": "gs.evolve(SystemSpec, ParticleState(numpy q, p), EvolveConfig(steps))"},
            "gpu_launches": int(ll.value),
            "clocks": clk.summary(),
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def run_extras(a, gs, device, configs, torch):
    """Secondary figures of BASELINE's metric pair: one C2 RHS, one C5 cell-list RHS, C1 seconds
    per feedback iteration."""
    out = {}
    w = configs.c2(a.n)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    q_d = torch.from_numpy(w.q).cuda()
    p_d = torch.from_numpy(w.p).cuda()
    for _ in range(3):
        device.rhs(spec, q_d, p_d)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    s.record()
    for _ in range(reps):
        device.rhs(spec, q_d, p_d)
    e.record()
    torch.cuda.synchronize()
    out["c2_rhs_ms"] = s.elapsed_time(e) / reps
    # the same C2 100-step solve through the cell list (pairs within the support radius only;
    # results equal the dense solve to ~1e-15)
    path0 = device.get_path()
    device.set_path("cell")
    try:
        for _ in range(2):
            device.evolve(spec, q_d, p_d, 1.0, a.rk_steps)
        s.record()
        for _ in range(3):
            device.evolve(spec, q_d, p_d, 1.0, a.rk_steps)
        e.record()
        torch.cuda.synchronize()
        out["c2_cell_solve_ms"] = s.elapsed_time(e) / 3
    finally:
        device.set_path(path0)
    # C5 cell-list RHS at the first feedback shoot's state (SURVEY §8(d) cell-list roofline:
    # accepted pairs/s x 45 slots against the FP64 peak)
    import ctypes

    from paper_1510_03816_b200 import _native as N

    w5 = configs.c5()
    spec5 = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w5.alpha), sigma2=w5.sigma2)
    q5 = torch.from_numpy(w5.q).cuda()
    p5 = torch.from_numpy(w5.h * (w5.target - w5.q)).cuda()
    path0 = device.get_path()
    device.set_path("cell")
    try:
        for _ in range(2):
            device.rhs(spec5, q5, p5)
        ctx = N.Context.get()
        pm, pl, ll, pp = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        ctx.lib.gs_profile_enable(ctx.handle, 1)
        ctx.lib.gs_profile_read(ctx.handle, ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(ll), ctypes.byref(pp), 1)
        s.record()
        for _ in range(3):
            device.rhs(spec5, q5, p5)
        e.record()
        torch.cuda.synchronize()
        ctx.lib.gs_profile_read(ctx.handle, ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(ll), ctypes.byref(pp), 1)
        ctx.lib.gs_profile_enable(ctx.handle, 0)
    finally:
        device.set_path(path0)
    rhs_ms = s.elapsed_time(e) / 3
    acc = pp.value / 3
    out["c5_cell_rhs_ms"] = rhs_ms
    out["c5_cell_pair_kernel_ms"] = pm.value / max(1, pl.value)
    out["c5_accepted_pairs_per_rhs"] = acc
    out["c5_cell_pairs_per_s"] = acc / (rhs_ms / 1e3)
    c1 = configs.c1()
    spec1 = gs.SystemSpec(kernel=gs.KernelSpec(alpha=c1.alpha))
    cfg = gs.ShootingConfig(h=c1.h, epsilon=c1.epsilon, max_iter=c1.max_iter, update_space="momentum",
                            evolve=gs.EvolveConfig(steps=c1.steps), system=spec1)
    ref, tgt = gs.LandmarkTemplate(c1.q, "X"), gs.LandmarkTemplate(c1.target, "Y")
    for _ in range(2):
        r = device.match(spec1, c1.q, c1.target, c1.h, c1.epsilon, c1.max_iter, "residual", "max", 1.0, c1.steps)
    out["c1_iterations"] = r["iterations"]
    out["c1_s_per_feedback_iteration"] = r["seconds_device"] / max(1, r["iterations"])
    t0 = time.perf_counter()
    res = gs.match(ref, tgt, cfg)
    out["c1_match_wall_s"] = time.perf_counter() - t0
    out["c1_converged"] = bool(res.converged)
    return out


if __name__ == "__main__":
    main()
