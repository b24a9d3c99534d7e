"""Run all five BASELINE configurations on the B200 with parity checks; write one JSON report.

    python tools/run_configs.py [--out gpurun_out/configs.json] [--only C1,C2,...] [--quick]

Per config (SURVEY.md §8(d) recipes, paper_1510_03816_b200/configs.py):
  C1  full match on the device vs the reference's golden record (tests/golden/match_cases.*)
  C2  one RHS (dense and cell) vs the reference's golden C2 RHS; 100-step solve timings;
      conserved quantities over the solve
  C3  one dense RHS, sampled rows vs the C oracle; one 50-step solve; conservation drift
  C4  full clustered match (cell list) — s per feedback iteration; the first shoot vs the
      C oracle's truncated evolve
  C5  20-iteration inexact match (cell list) — s per feedback iteration; first shoot vs the
      C oracle
Device times are CUDA events (gs_match's own event pair for matches).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def timed(torch, fn, reps=1, warm=0):
    for _ in range(warm):  # first calls pay one-time setup (workspaces, graphs, module loads)
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        out = fn()
    e.record()
    torch.cuda.synchronize()
    return out, s.elapsed_time(e) / 1e3 / reps


def conserved(gs, spec, q, p):
    c = gs.conserved_quantities(spec, gs.ParticleState(q, p))
    return float(c["H"]), np.asarray(c["P"], float), float(c["L"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "configs.json"))
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--quick", action="store_true", help="skip the slow CPU oracle comparisons")
    ap.add_argument("--n45", type=int, default=0, help="override N of C4/C5 (debugging)")
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    from oracle import native
    from oracle.restate import Kernel
    from paper_1510_03816_b200 import configs, device

    report = {"device": torch.cuda.get_device_name(0), "host_threads": native.max_threads()}
    only = set(a.only.split(","))

    def kern(alpha, fam=0):
        return Kernel(fam, alpha, True)

    if "C1" in only:
        w = configs.c1()
        with open(os.path.join(REPO, "tests", "golden", "match_cases.json")) as f:
            gold = json.load(f)["c1"]
        z = np.load(os.path.join(REPO, "tests", "golden", "match_cases.npz"))
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
        r = device.match(spec, w.q, w.target, w.h, w.epsilon, w.max_iter, "residual", "max", 1.0, w.steps)
        r = device.match(spec, w.q, w.target, w.h, w.epsilon, w.max_iter, "residual", "max", 1.0, w.steps)
        p0 = r["p0"].cpu().numpy()
        report["C1"] = {
            "iterations": r["iterations"], "converged": r["converged"], "hamiltonian": r["hamiltonian"],
            "reference_iterations": gold["iterations"], "reference_hamiltonian": gold["hamiltonian"],
            "p0_rel_err_vs_reference": rel(p0, z["c1__p0"]),
            "endpoint_err_vs_reference": float(np.abs(r["endpoint"].cpu().numpy() - z["c1__endpoint"]).max()),
            "s_per_feedback_iteration": r["seconds_device"] / max(1, r["iterations"]),
            "match_seconds_device": r["seconds_device"],
            "reference_match_seconds_cpu_in_golden_run": gold["seconds"],
        }
        print("C1", report["C1"], flush=True)

    if "C2" in only:
        w = configs.c2()
        z = np.load(os.path.join(REPO, "tests", "golden", "rhs_c2.npz"))
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
        out = {}
        qd, pd = torch.from_numpy(w.q).cuda(), torch.from_numpy(w.p).cuda()
        for path in ("dense", "cell"):
            gs.set_path(path)
            (dq, dp), t_rhs = timed(torch, lambda: device.rhs(spec, qd, pd), reps=5, warm=1)
            device.evolve(spec, qd, pd, 1.0, 100)
            (qT, pT, _), t_solve = timed(torch, lambda: device.evolve(spec, qd, pd, 1.0, 100), reps=2)
            H0, P0, L0 = conserved(gs, spec, w.q, w.p)
            H1, P1, L1 = conserved(gs, spec, qT.cpu().numpy(), pT.cpu().numpy())
            out[path] = {"rhs_ms": t_rhs * 1e3, "rhs_rel_err_dq": rel(dq.cpu().numpy(), z["dq"]),
                         "rhs_rel_err_dp": rel(dp.cpu().numpy(), z["dp"]), "solve_100_steps_s": t_solve,
                         "dH_rel": abs(H1 - H0) / abs(H0), "dP_abs": float(np.abs(P1 - P0).max()),
                         "dL_abs": abs(L1 - L0)}
        gs.set_path("auto")
        out["reference_rhs_s_cpu_in_golden_run"] = float(z["seconds"])
        report["C2"] = out
        print("C2", out, flush=True)

    if "C3" in only:
        w = configs.c3()
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
        qd, pd = torch.from_numpy(w.q).cuda(), torch.from_numpy(w.p).cuda()
        gs.set_path("dense")
        (dq, dp), t_rhs = timed(torch, lambda: device.rhs(spec, qd, pd), reps=2, warm=1)
        errs = []
        if not a.quick:
            for r0 in (0, 70001):
                oq, op = native.rhs(kern(w.alpha), 0.0, w.q, w.p, rows=(r0, r0 + 128))
                errs.append((rel(dq[r0:r0 + 128].cpu().numpy(), oq), rel(dp[r0:r0 + 128].cpu().numpy(), op)))
        (qT, pT, _), t_solve = timed(torch, lambda: device.evolve(spec, qd, pd, 1.0, w.steps))
        H0, P0, L0 = conserved(gs, spec, w.q, w.p)
        H1, P1, L1 = conserved(gs, spec, qT.cpu().numpy(), pT.cpu().numpy())
        gs.set_path("auto")
        pairs = 4 * w.steps * float(w.n) ** 2
        report["C3"] = {"rhs_s": t_rhs, "rhs_pairs_per_s": float(w.n) ** 2 / t_rhs, "solve_50_steps_s": t_solve,
                        "solve_pairs_per_s": pairs / t_solve, "sampled_rows_rel_err_vs_oracle": errs,
                        "dH_rel": abs(H1 - H0) / abs(H0), "dP_abs": float(np.abs(P1 - P0).max()),
                        "dL_abs": abs(L1 - L0)}
        print("C3", report["C3"], flush=True)

    for name, fn in (("C4", configs.c4), ("C5", configs.c5)):
        if name not in only:
            continue
        w = fn(a.n45) if a.n45 else fn()
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
        gs.set_path("auto")
        print(name, "match start n =", w.n, flush=True)
        t0 = time.perf_counter()
        r = device.match(spec, w.q, w.target, w.h, w.epsilon, w.max_iter, w.stop_rule, "max", 1.0, w.steps)
        wall = time.perf_counter() - t0
        out = {"n": w.n, "iterations": r["iterations"], "converged": r["converged"], "diagnosis": r["diagnosis"],
               "hamiltonian": r["hamiltonian"], "final_residual": r["final_residual"],
               "history_head": list(r["residual_history"][:5]), "history_tail": list(r["residual_history"][-3:]),
               "match_seconds_device": r["seconds_device"], "match_seconds_wall": wall,
               "s_per_feedback_iteration": r["seconds_device"] / max(1, r["iterations"])}
        # first shoot p = h (Y - X) through the device evolve vs the C oracle's truncated evolve:
        # the first 2 (C4) / 1 (C5) of the 20 RK4 steps with the same dt — the shoot diverges and
        # the flung-apart state defeats the oracle's plain grid (quadratic on the CPU)
        p1 = w.h * (w.target - w.q)
        (qT, pT, _), t_ev = timed(torch, lambda: device.evolve(spec, w.q, p1, 1.0, w.steps))
        out["first_shoot_s"] = t_ev
        out["first_shoot_max_abs_q"] = float(qT.abs().max())
        if not a.quick:
            # per-RHS parity at full size on the first shoot's initial state (before any blow-up)
            dq, dp = device.rhs(spec, w.q, p1)
            oq, op = native.rhs(kern(w.alpha), w.sigma2, w.q, p1, cutoff=w.sigma)
            out["rhs_rel_err_dq_vs_oracle"] = rel(dq.cpu().numpy(), oq)
            out["rhs_rel_err_dp_vs_oracle"] = rel(dp.cpu().numpy(), op)
            # the stiff flow amplifies rounding from the first step on: the 1-step shoot is info only
            ck = 1
            tf = 1.0 * ck / w.steps
            (qk, pk, _), _ = timed(torch, lambda: device.evolve(spec, w.q, p1, tf, ck))
            t0 = time.perf_counter()
            oq, op = native.evolve(kern(w.alpha), w.sigma2, w.q, p1, tf, ck, cutoff=w.sigma)
            out["oracle_check_steps"] = ck
            out["oracle_check_s_cpu"] = time.perf_counter() - t0
            out["check_rel_err_q"] = rel(qk.cpu().numpy(), oq)
            out["check_rel_err_p"] = rel(pk.cpu().numpy(), op)
        report[name] = out
        print(name, out, flush=True)

    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
