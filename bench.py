#!/usr/bin/env python
"""bench.py — throughput of the B200 EP N-particle hot path on BASELINE config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--path dense|cell|auto]

One "step" = one 100-step classical RK4 shooting solve (T = 1, 400 RHS evaluations) of
BASELINE.json configs[1]: N = 16384 particles uniform in [0,1]^2 (seed 0), momenta
N(0, 0.01^2) (seed 1), conical kernel with support radius sigma = 0.05 (KD-1: alpha =
sigma / (53 ln 2)).  The metric is particle-pair interactions per second in the RHS,
counting the reference's N^2 ordered pairs per RHS (particles.py:79-117 evaluates all of
them) for the dense path and the accepted pairs (d < sigma, plus the N self terms) for the
cell-list path.  Inputs are device resident for `value` (timed with the library's profiling
off); `e2e` times the public API on host arrays (H2D + D2H inside the timed region).  The
roofline comes from a separate profiled pass (CUDA events around every pair-kernel launch).

Multi-GPU: `--gpus N` re-launches itself under torch.distributed.run with N ranks (one per GPU,
NCCL, 127.0.0.1) unless WORLD_SIZE is already set.  The C2 solve is then split across ranks
(paper_1510_03816_b200/sharded.py: symmetric pair split + per-stage exchange); the total work is
fixed ("strong" scaling), time is the max over ranks of CUDA-event device time.  The BASELINE
scaling workloads (C3 dense, C5 cell list) are timed at the same N in `extras.scaling`.

`--impl reference` times the reference's CPU algorithm on the host cores, rank 0 only: the numpy
restatement oracle/restate.py (the reference's own formulas, bitwise equal to geoshoot.rhs on
the golden cases), one full C2 RHS per step in row blocks on a thread pool (numpy releases the
GIL), i.e. a 1/400 sample of our step with the same pairs/s metric.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

if "--impl" in sys.argv and "reference" in sys.argv:
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # threads come from the row-block pool

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "particle-pair interactions/s in N-particle RHS (fp64)"
UNIT = "pairs/s"
W_ALG = 45  # DP-pipe issue slots per ordered pair, libm formulation = 90 flop-equivalents


def parse(argv=None):
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
    ap.add_argument("--dry-run", action="store_true",
                    help="(testing) launch the ranks and print the JSON skeleton without touching a GPU")
    return ap.parse_args(argv)


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(a) -> int:
    """Re-exec this script under torch.distributed.run with one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    print(f"bench: launching {a.gpus} ranks: {' '.join(cmd[1:6])} ...", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


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


def profile_traffic(path_kind: str):
    """Per-launch DRAM bytes of the pair kernel from the committed ncu capture, if any."""
    name = {"dense": "ncu_pair_kernel.json", "cell": "ncu_cell_kernel.json"}.get(path_kind, "ncu_pair_kernel.json")
    try:
        with open(os.path.join(REPO, "profiles", name)) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


def arm_config(a, n):
    """The workload both arms report (BASELINE configs[1])."""
    return {"workload": f"C2: one {a.rk_steps}-step RK4 shooting solve (T=1, {4 * a.rk_steps} RHS) of N={n}, "
                        f"conical sigma=0.05 (KD-1), {a.path} path",
            "n": n, "rk_steps": a.rk_steps, "path": a.path}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------------------
def reference_rhs_pool(k, w, threads: int, block: int = 128):
    """One full RHS of the reference's algorithm (oracle/restate.rhs_rows: particles.py:79-117,
    kernels.py:121-178) in row blocks on `threads` host threads."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import restate

    blocks = [(r, min(r + block, w.n)) for r in range(0, w.n, block)]
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda b: restate.rhs_rows(k, 0.0, w.q, w.p, b[0], b[1]), blocks))


def reference_arm(a):
    """--impl reference: the reference's CPU algorithm on rank 0, one full C2 RHS per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import restate
    from paper_1510_03816_b200 import configs

    w = configs.c2(a.n)
    k = restate.Kernel(0, w.alpha, True)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)

    for _ in range(a.warmup):
        reference_rhs_pool(k, w, threads)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        reference_rhs_pool(k, w, threads)
    dt = time.perf_counter() - t0
    pairs = a.steps * w.n * w.n
    value = pairs / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE configs[1] recipe, seeds 0/1)",
        "config": dict(arm_config(a, w.n), parallelism=f"host cores ({threads} threads)",
                       sample="one full RHS (all N^2 ordered pairs) per step = 1/400 of the solve; same pairs/s metric"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"one full C2 RHS per step through oracle/restate.py rhs_rows (numpy restatement "
                                   f"of particles.py:79-117) in 128-row blocks on {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_port(w, spec_alpha, c1=None):
    """The C/OpenMP oracle port on all host cores, one RK4 step (4 RHS) of C2; with `c1`, also
    the reference's Algorithm 1 (numpy restatement) on config 1 — the CPU side of BASELINE's
    second metric, seconds per feedback iteration."""
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


def implemented_fp64_per_pair(path_kind: str):
    """(FP64-pipe instructions per ordered pair of the dominant kernel, the operand-read ceiling of
    its loop's FP64 instruction mix), both from the SASS of the library actually loaded
    (tools/sass_loops.py; cuobjdump ships with the CUDA toolkit)."""
    try:
        sys.path.insert(0, os.path.join(REPO, "tools"))
        import sass_loops

        from paper_1510_03816_b200 import _native as N

        if path_kind == "dense":
            w, loop = sass_loops.fp64_per_pair(N.LIB_PATH, r"k_dense_symILi0E", True)
        else:
            w, loop = sass_loops.fp64_per_pair(N.LIB_PATH, r"k_verlet_pairILi0ELi\d+ELb0E", False)
        return w, (sass_loops.operand_read_ceiling(loop) if loop else None)
    except Exception:
        return None, None


# ---------------------------------------------------------------------------------------------
def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        sys.exit(relaunch(a))
    if a.impl == "reference":
        reference_arm(a)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and not a.force_sharded:
        raise SystemExit(f"bench: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.dry_run:  # the launch and rank plumbing only (CPU test): ranks agree over gloo, rank 0 prints
        import torch.distributed as dist

        if world > 1:
            dist.init_process_group("gloo")
            t = __import__("torch").tensor([1.0])
            dist.all_reduce(t)
            world_seen = int(t.item())
            dist.destroy_process_group()
        else:
            world_seen = 1
        if rank == 0:
            print(json.dumps({"metric": METRIC, "n_gpus": world, "ranks_seen": world_seen, "dry_run": True}),
                  flush=True)
        return
    import torch
    import torch.distributed as dist

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import configs, device, sharded

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"bench: rank {rank}/{world} NCCL {'.'.join(map(str, torch.cuda.nccl.version()))} on cuda:{local} "
              f"({torch.cuda.get_device_name(local)})", file=sys.stderr, flush=True)
    elif a.force_sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(free_port()))
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

    import ctypes

    pm, pl, ll, pp = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()

    def prof_read(reset=1):
        lib.gs_profile_read(ctx.handle, ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(ll), ctypes.byref(pp), reset)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2
    for _ in range(max(3, a.warmup)):
        solve()
    torch.cuda.synchronize()

    # -- profiled pass (separate from the timed region): pair-kernel launch times, pairs per solve
    prof_reps = 2
    lib.gs_profile_enable(ctx.handle, 1)
    if solver is not None:  # the host-driven stage loop: a replayed graph has no profiling events
        solver.graphs = False
    prof_read()
    for _ in range(prof_reps):
        flush.zero_()
        solve()
    torch.cuda.synchronize()
    prof_read()
    lib.gs_profile_enable(ctx.handle, 0)
    if solver is not None:
        solver.graphs = True
    pair_ms_avg = pm.value / max(1, pl.value)
    pairs_per_launch = float(pp.value) / max(1, pl.value)
    pairs_per_solve = float(pp.value) / prof_reps        # evaluated ordered pairs (this rank)
    launches_per_solve = ll.value / prof_reps

    # -- timed region: profiling off, L2 flushed between steps, CUDA events, max over ranks
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    prof_read()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(a.steps):
            # ~1 ms device sleep ahead of the flush: the host enqueues the whole step (clones,
            # graph launch) while the GPU still sleeps, so the events time the GPU work only,
            # not the host's submission latency (the solve syncs at its end to read the status)
            torch.cuda._sleep(2_000_000)
            flush.zero_()  # outside the events
            starts[k].record()
            solve()
            ends[k].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    prof_read()
    launches_timed = int(ll.value)
    if solver is not None and getattr(solver, "_graph", None) is not None:
        # the sharded stage loop replays a torch-captured graph: the library's host-side launch
        # counter does not see its kernels; the profiled (host-driven) pass counted them per solve
        launches_timed = int(round(launches_per_solve * a.steps))
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms, pairs_per_solve * a.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        tp = t[1:].clone()
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tp, op=dist.ReduceOp.SUM)
        t[1] = tp[0]
    ms_max = float(t[0])
    total_pairs = float(t[1])          # evaluated ordered pairs, all ranks
    pairs_per_rhs = total_pairs / (a.steps * 4 * a.rk_steps)
    value = total_pairs / (ms_max / 1e3)

    # -- roofline of the dominant kernel (the pair kernel), from the profiled pass
    ach_pairs = pairs_per_launch / (pair_ms_avg / 1e3) if pair_ms_avg > 0 else 0.0
    path_kind = "dense" if a.path == "dense" else "cell"
    w_impl, op_ceiling = implemented_fp64_per_pair(path_kind)
    best = None
    for _ in range(3):
        pms, pfl = ctypes.c_double(), ctypes.c_double()
        lib.gs_fp64_peak_probe(ctx.handle, 20000, ctypes.byref(pms), ctypes.byref(pfl), None)
        r = pfl.value / (pms.value / 1e3) / 1e12
        best = r if best is None else max(best, r)
    peak = best
    traffic, _ = profile_traffic(path_kind)
    ach_tflops = ach_pairs * w_impl * 2 / 1e12 if w_impl else None  # FP64 slots issued x 2 flops (DFMA)

    # -- e2e: the public API on host arrays (H2D + D2H inside the timed region)
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
    if not a.no_extras:
        try:  # secondary figures must never cost the headline line
            extras = run_extras(a, gs, device, configs, torch, world, rank, dist, solver is not None)
        except Exception as exc:  # noqa: BLE001
            extras = {"error": f"{type(exc).__name__}: {exc}"}
            print(f"bench: extras failed on rank {rank}: {extras['error']}", file=sys.stderr, flush=True)
    if rank == 0:
        cpu = cpu_baseline_port(w, w.alpha, None if a.no_extras else configs.c1())
        kernel = ("gsb::k_dense_sym (symmetric, 1 GPU) / gsb::k_dense_partial (row shards)" if a.path == "dense"
                  else "gsb::k_verlet_pair (cluster Verlet lists)")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (BASELINE configs[1] recipe: uniform [0,1]^2 seed 0, N(0,0.01^2) seed 1)",
            "config": dict(arm_config(a, w.n), parallelism=(
                f"rows{world}" if solver is None else
                f"{'pair-split' if a.path == 'dense' else 'rows'}{world}+{'p2p' if solver.p2p else 'nccl'}"),
                           l2="flushed between timed steps (256 MB write)"),
            "roofline": {
                "bound": "fp64", "achieved": ach_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": ach_tflops / peak if (peak and ach_tflops) else None, "traffic": traffic,
                "kernel": kernel, "avg_launch_ms": pair_ms_avg, "pairs_per_launch": pairs_per_launch,
                "basis": "FP64-pipe utilisation: implemented FP64 instructions per ordered pair (counted in the "
                         "loaded library's SASS) x pairs/s x 2 flops, against the FP64 peak measured live",
                "fp64_slots_per_pair_implemented": w_impl,
                "operand_read_ceiling": op_ceiling,
                "operand_read_ceiling_basis": "a DFMA with three fresh 64-bit register operands holds the FP64 pipe's "
                                              "issue ~3.2 cycles instead of 2 (tools/issue_probe2.cu); share of the pipe "
                                              "this kernel's SASS mix can reach",
                "peak_source": "measured live: gs_fp64_peak_probe (DFMA chains on all SMs, best of 3)",
                "w45": {"work_per_pair": f"{W_ALG} DP-pipe slots = {2 * W_ALG} flop-equivalents (SURVEY.md §8(d) "
                                         "libm formulation)",
                        "achieved": ach_pairs * W_ALG * 2 / 1e12,
                        "frac": (ach_pairs * W_ALG * 2 / 1e12) / peak if peak else None}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * w.n * 2 * 8,
                    "d2h_bytes_per_step": 2 * w.n * 2 * 8,
                    "api": "gs.evolve(SystemSpec, ParticleState(numpy q, p), EvolveConfig(steps))"},
            "gpu_launches": launches_timed,
            "gpu_launches_per_step": launches_per_solve,
            "clocks": clk.summary(),
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def _timed(torch, fn, reps):
    """(last result, median ms per call): each call between its own pair of events on the stream
    (the median drops calls a host-side stall of the Python process stretched)."""
    ts = []
    out = None
    for _ in range(max(3, reps)):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return out, statistics.median(ts)


def _accepted_pairs(fn, torch):
    """(result, accepted ordered pairs) of one call with the library's pair counting on."""
    import ctypes

    from paper_1510_03816_b200 import _native as N

    ctx = N.Context.get()
    pm, pl, ll, pp = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    ctx.lib.gs_profile_enable(ctx.handle, 1)
    ctx.lib.gs_profile_read(ctx.handle, ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(ll), ctypes.byref(pp), 1)
    out = fn()
    torch.cuda.synchronize()
    ctx.lib.gs_profile_read(ctx.handle, ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(ll), ctypes.byref(pp), 1)
    ctx.lib.gs_profile_enable(ctx.handle, 0)
    return out, float(pp.value), pm.value / max(1, pl.value)


def run_extras(a, gs, device, configs, torch, world, rank, dist, sharded_run):
    """Secondary figures: BASELINE's second metric (seconds per feedback iteration) on C1, C4 and C5,
    the cell-list workloads (C2 cell solve, C4/C5 RHS), and at N > 1 the scaling workloads."""
    out = {}
    if world == 1:
        w = configs.c2(a.n)
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
        q_d, p_d = torch.from_numpy(w.q).cuda(), torch.from_numpy(w.p).cuda()
        path0 = device.get_path()
        try:
            device.set_path("dense")
            _, out["c2_dense_rhs_ms"] = _timed(torch, lambda: device.rhs(spec, q_d, p_d), 10)
            # the C2 solve through the cell list (pairs within the support radius only)
            device.set_path("cell")
            for _ in range(2):
                device.evolve(spec, q_d, p_d, 1.0, a.rk_steps)
            _, ms = _timed(torch, lambda: device.evolve(spec, q_d, p_d, 1.0, a.rk_steps), 3)
            _, acc, _ = _accepted_pairs(lambda: device.evolve(spec, q_d, p_d, 1.0, a.rk_steps), torch)
            out["c2_cell_solve"] = {"ms_per_solve": ms, "accepted_pairs_per_solve": acc,
                                    "accepted_pairs_per_s": acc / (ms / 1e3)}
            # C4 / C5 cell-list RHS inside an evolve (cluster Verlet lists) at the first shoot's state,
            # and seconds per feedback iteration of the full-size match (2 iterations)
            for name in ("C4", "C5"):
                wk = configs.CONFIGS[name]()
                sp = gs.SystemSpec(kernel=gs.KernelSpec(alpha=wk.alpha), sigma2=wk.sigma2)
                qk = torch.from_numpy(wk.q).cuda()
                pk = torch.from_numpy(np.ascontiguousarray(wk.h * (wk.target - wk.q))).cuda()
                device.set_path("auto")
                steps = 4
                tf = steps * wk.t_final / wk.steps
                # the first calls of a new size allocate the multi-GB list buffer and capture the graphs
                for _ in range(2):
                    device.evolve(sp, qk, pk, tf, steps)
                _, ms = _timed(torch, lambda: device.evolve(sp, qk, pk, tf, steps), 5)
                _, acc, pair_ms = _accepted_pairs(lambda: device.evolve(sp, qk, pk, tf, steps), torch)
                # the match loop's conditional graph is captured on its first call: warm it up
                device.match(sp, wk.q, wk.target, wk.h, wk.epsilon, 1, wk.stop_rule, "max", wk.t_final, wk.steps)
                r = device.match(sp, wk.q, wk.target, wk.h, wk.epsilon, 2, wk.stop_rule, "max", wk.t_final, wk.steps)
                out[name.lower()] = {"n": wk.n, "rhs_ms_in_evolve": ms / (4 * steps), "pair_kernel_ms": pair_ms,
                                     "accepted_pairs_per_rhs": acc / (4 * steps),
                                     "accepted_pairs_per_s": acc / (ms / 1e3),
                                     "s_per_feedback_iteration": r["seconds_device"] / max(1, r["iterations"]),
                                     "h": wk.h}
        finally:
            device.set_path(path0)
        # the multi-GPU cell path (slab decomposition) at W = 8 run on this one GPU: per-rank device
        # time per RHS, rows bitwise equal to W = 1 (tools/time_slab.py; exchange cost modelled)
        from tools import time_slab

        em = time_slab.measure("C5", 8, 4)
        w8 = em["W8"]
        out["c5_slab_w8_emulated"] = {
            "rank_ms_per_rhs": w8["rank_ms_per_rhs_measured"], "stage_ms_per_rhs": w8["stage_ms_per_rhs_max_rank"],
            "build_ms": w8["build_ms_per_build_max_rank"], "builds_per_16_rhs": w8["builds"],
            "halo_bytes_per_stage": w8["halo_bytes_per_stage_max_rank"],
            "modelled_rank_ms_per_rhs_with_exchange": w8["modelled_rank_ms_per_rhs"],
            "modelled_strong_scaling_eff": w8["modelled_strong_scaling_eff_vs_one_gpu"],
            "one_gpu_ms_per_rhs": em["one_gpu_verlet_ms_per_rhs"], "bitwise_equal_w1": em["bitwise_equal_w1_vs_w"]}
        c1 = configs.c1()
        spec1 = gs.SystemSpec(kernel=gs.KernelSpec(alpha=c1.alpha))
        for _ in range(2):
            r = device.match(spec1, c1.q, c1.target, c1.h, c1.epsilon, c1.max_iter, "residual", "max", 1.0, c1.steps)
        out["c1_iterations"] = r["iterations"]
        out["c1_s_per_feedback_iteration"] = r["seconds_device"] / max(1, r["iterations"])
        cfg = gs.ShootingConfig(h=c1.h, epsilon=c1.epsilon, max_iter=c1.max_iter, update_space="momentum",
                                evolve=gs.EvolveConfig(steps=c1.steps), system=spec1)
        t0 = time.perf_counter()
        res = gs.match(gs.LandmarkTemplate(c1.q, "X"), gs.LandmarkTemplate(c1.target, "Y"), cfg)
        out["c1_match_wall_s"] = time.perf_counter() - t0
        out["c1_converged"] = bool(res.converged)
        return out
    # N > 1: BASELINE's scaling workloads at this N (strong scaling: the same total work)
    from paper_1510_03816_b200 import sharded

    sc = {}
    for name, path, steps in (("C3", "dense", 2), ("C5", "cell", 4)):
        try:
            sc[name] = _scaling_workload(name, path, steps, gs, device, configs, sharded, torch, dist)
        except Exception as exc:  # noqa: BLE001  (every rank takes the same path: no collective is left waiting)
            sc[name] = {"error": f"{type(exc).__name__}: {exc}", "path": path}
    device.set_path(a.path)
    out["scaling"] = sc
    return out


def _scaling_workload(name, path, steps, gs, device, configs, sharded, torch, dist):
    """ms per RHS (max over ranks) of a short evolve of a BASELINE scaling workload at this N."""
    wk = configs.CONFIGS[name]()
    sp = gs.SystemSpec(kernel=gs.KernelSpec(alpha=wk.alpha), sigma2=wk.sigma2)
    pk = wk.p if wk.p is not None else wk.h * (wk.target - wk.q)
    device.set_path(path)
    solver = sharded.ShardedSolver(sp)
    qk, pkd = torch.from_numpy(wk.q).cuda(), torch.from_numpy(np.ascontiguousarray(pk)).cuda()
    tf = steps * wk.t_final / wk.steps
    solver.evolve(qk, pkd, tf, steps)
    dist.barrier()
    _, ms = _timed(torch, lambda: solver.evolve(qk, pkd, tf, steps), 1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"ms_per_rhs": float(t[0]) / (4 * steps), "path": path, "rk_steps": steps,
            "pairs_per_rhs": float(wk.n) ** 2 if path == "dense" else None}


if __name__ == "__main__":
    main()
