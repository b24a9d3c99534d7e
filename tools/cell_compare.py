"""Cell-path evolve: cluster Verlet lists vs the per-RHS cell sweep (and the C2 oracle fixture).

    python tools/cell_compare.py [--configs C2,C5,C4] [--steps 4] [--reps 3]

For each config: one evolve through the lists (GS_B200_VERLET=1, the default) and one through the
per-RHS sweep (a second context created with GS_B200_VERLET=0), device times by CUDA events, the
relative difference of the final states, and for C2 the 100-step solve against
tests/golden/oracle_c2_solve_cell.npz.  C4/C5 use the first shoot's momenta p = h (Y - X).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C5,C4")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import configs, device

    gs.set_path("cell")
    out = {}

    stats = {}

    def run(w, p, steps, tf, verlet):
        os.environ["GS_B200_VERLET"] = "1" if verlet else "0"
        N.Context.swap()  # fresh context: reads the env at gs_create
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
        qd = torch.from_numpy(w.q).cuda()
        pd = torch.from_numpy(p).cuda()
        device.evolve(spec, qd, pd, tf, steps)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(a.reps):
            qT, pT, _ = device.evolve(spec, qd, pd, tf, steps)
        e.record()
        torch.cuda.synchronize()
        ctx = N.Context.get()
        b, ent = ctypes.c_int64(), ctypes.c_int64()
        N.check(ctx.lib.gs_cell_stats(ctx.handle, ctypes.byref(b), ctypes.byref(ent), None), "gs_cell_stats")
        stats.update(builds=b.value, entries=ent.value)
        return qT.cpu().numpy(), pT.cpu().numpy(), s.elapsed_time(e) / a.reps

    for name in a.configs.split(","):
        w = configs.CONFIGS[name]()
        if name == "C2":
            p, steps, tf = w.p, 100, 1.0
        else:
            p, steps, tf = w.h * (w.target - w.q), a.steps, a.steps / w.steps
        qv, pv, tv = run(w, p, steps, tf, True)
        vstats = dict(stats)
        qo, po, to = run(w, p, steps, tf, False)
        rel = lambda x, y: float(np.abs(x - y).max() / np.abs(y).max())  # noqa: E731
        row = {"n": w.n, "steps": steps, "verlet_ms": tv, "sweep_ms": to, "ms_per_rhs_verlet": tv / (4 * steps),
               "ms_per_rhs_sweep": to / (4 * steps), "rel_q": rel(qv, qo), "rel_p": rel(pv, po),
               "list_builds_in_warmup_plus_reps": vstats.get("builds"), "list_entries": vstats.get("entries"),
               "evolves": 1 + a.reps}
        if name == "C2":
            z = np.load(os.path.join(REPO, "tests", "golden", "oracle_c2_solve_cell.npz"))
            rows = z["rows"]
            row["oracle_rel_q_verlet"] = rel(qv[rows], z["q"])
            row["oracle_rel_p_verlet"] = rel(pv[rows], z["p"])
            row["oracle_rel_q_sweep"] = rel(qo[rows], z["q"])
            row["oracle_rel_p_sweep"] = rel(po[rows], z["p"])
        out[name] = row
        print(name, json.dumps(row), flush=True)
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", "cell_compare.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
