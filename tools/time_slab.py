"""One-GPU emulation of the W-rank slab decomposition of the cell path (paper_1510_03816_b200/slab.py).

    python tools/time_slab.py --config C5 --world 8 --steps 4 [--out profiles/r02_slab_c5.json]

Runs the same evolve with W = 1 and W = --world slab ranks in one process (LocalComm: one
library context per rank, collectives are copies) and times every rank's device work with CUDA
events on the launching stream: the stage (list sweep + RK4 epilogue of the rank's own rows)
and the list build (bbox, grid, row histogram, migration pack/unpack, layout sort, cell starts,
clusters, lists).  Ranks run one after the other on the one GPU, so each rank's time is its
time on a whole B200.  Also: the halo a rank receives per stage, the one-GPU cluster-list evolve
of the same state (device.evolve, the single-GPU product path) and whether W ranks reproduce
the W = 1 rows bitwise.  The exchange itself (halo slices over NVLink, flag all-reduce) is not
run across GPUs here; its cost is modelled from the measured halo bytes.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--gain", type=float, default=None, help="p = gain (Y - X); default the config's h")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default="")
    ap.add_argument("--only-world", action="store_true", help="skip W = 1 and the comparisons (launch lists)")
    a = ap.parse_args()
    out = measure(a.config, a.world, a.steps, a.gain, a.reps, only_world=a.only_world)
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


def measure(config="C5", world=8, steps=4, gain=None, reps=2, only_world=False) -> dict:
    """The emulation (see the module docstring) as a dict."""
    a = argparse.Namespace(config=config, world=world, steps=steps, gain=gain, reps=reps)
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import configs, device, slab

    w = configs.CONFIGS[a.config]()
    gain = a.gain if a.gain is not None else w.h
    p = w.p if w.p is not None else gain * (w.target - w.q)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    q_d, p_d = torch.from_numpy(w.q).cuda(), torch.from_numpy(np.ascontiguousarray(p)).cuda()
    tf = a.steps * w.t_final / w.steps
    rhs = 4 * a.steps

    # the single-GPU product path (cluster lists in one CUDA graph)
    device.set_path("cell")
    device.evolve(spec, q_d, p_d, tf, a.steps)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    q1, p1, _ = device.evolve(spec, q_d, p_d, tf, a.steps)
    e.record()
    torch.cuda.synchronize()
    one_gpu_ms = s.elapsed_time(e) / rhs
    device.set_path("auto")

    out = {"config": a.config, "n": w.n, "rk_steps": a.steps, "gain": gain, "one_gpu_verlet_ms_per_rhs": one_gpu_ms}
    results = {}
    for W in ((a.world,) if only_world else (1, a.world)):
        ctxs = [N.Context(0) for _ in range(W)]
        rec = []

        def timer(kind, rank, fn):
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            r = fn()
            e0.record()
            rec.append((kind, rank, s0, e0))
            return r

        solver = slab.SlabSolver(spec, [slab.DeviceSlabBackend(spec, ctx=c) for c in ctxs], slab.LocalComm(W),
                                 timer=timer)
        for _ in range(a.reps):
            rec.clear()
            qW, pW = solver.evolve(q_d, p_d, tf, a.steps)
            torch.cuda.synchronize()
        stage = np.zeros((rhs, W))
        k = 0
        build = {}
        phases = {}
        for kind, rank, s0, e0 in rec:
            t = s0.elapsed_time(e0)
            if kind == "stage":
                stage[k // W, rank] = t
                k += 1
            else:
                build.setdefault(rank, 0.0)
                build[rank] += t
                phases.setdefault(kind, np.zeros(W))[rank] += t
        plan = solver.plan
        halo = [plan.halo_particles(r) for r in range(W)]
        results[W] = (qW, pW)
        out[f"W{W}"] = {
            "stage_ms_per_rhs_max_rank": float(stage.max(axis=1).mean()),
            "stage_ms_per_rhs_by_rank": [float(x) for x in stage.mean(axis=0)],
            "builds": solver.builds,
            "build_ms_total_max_rank": float(max(build.values())),
            "build_ms_per_build_max_rank": float(max(build.values())) / max(1, solver.builds),
            "n_own": [r.n_own for r in plan.rows],
            "halo_particles": halo,
            "halo_bytes_per_stage_max_rank": 32 * max(halo),
            "slices": len(plan.slices),
            "build_phase_ms_max_rank": {k: float(v.max()) for k, v in phases.items()},
        }
        d = out[f"W{W}"]
        d["rank_ms_per_rhs_measured"] = d["stage_ms_per_rhs_max_rank"] + d["build_ms_total_max_rank"] / rhs
    if not only_world:
        q0, p0 = results[1]
        qW, pW = results[a.world]
        out["bitwise_equal_w1_vs_w"] = bool(torch.equal(q0, qW) and torch.equal(p0, pW))
        out["rel_diff_vs_one_gpu_verlet"] = [float((q0 - q1).abs().max() / q1.abs().max()),
                                             float((p0 - p1).abs().max() / p1.abs().max())]
    # modelled exchange per stage at W GPUs: halo slices over NVLink (~700 GB/s achieved by NCCL
    # P2P at these sizes) + ~15 us for the P2P launch and the flag all-reduce
    dW = out[f"W{a.world}"]
    xch = dW["halo_bytes_per_stage_max_rank"] / 700e9 * 1e3 + 0.015
    dW["modelled_exchange_ms_per_stage"] = xch
    dW["modelled_rank_ms_per_rhs"] = dW["rank_ms_per_rhs_measured"] + xch
    dW["modelled_strong_scaling_eff_vs_one_gpu"] = one_gpu_ms / (a.world * dW["modelled_rank_ms_per_rhs"])
    return out


if __name__ == "__main__":
    main()
