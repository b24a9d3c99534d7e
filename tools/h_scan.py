"""Feedback-gain scan for the C4 / C5 matches at full size on the B200.

    python tools/h_scan.py [--only C4,C5] [--hs C4=0.1,0.05 ...] [--out gpurun_out/h_scan.json]

BASELINE.json leaves the feedback gain h of C4 and C5 open.  With
KD-1's narrow kernel the first shoots of the survey's proposals (h = 0.1 / 0.4) throw the clouds
apart and the reference's blow-up rule (shooting.py:287-291) ends both matches after 1-2
iterations.  This tool runs the full-size device match for a list of h values and records the
outcome, the iteration count, the residual history and the spread of the final endpoint, so the
configured h (paper_1510_03816_b200/configs.py) is a measured choice.
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

DEFAULT_HS = {"C4": [0.1, 0.05, 0.03, 0.02, 0.01, 0.005, 0.002],
              "C5": [0.4, 0.2, 0.1, 0.05, 0.03, 0.02, 0.01]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C4,C5")
    ap.add_argument("--hs", nargs="*", default=[])
    ap.add_argument("--n", type=int, default=0, help="override N (debugging)")
    ap.add_argument("--max-iter", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "h_scan.json"))
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    hs = dict(DEFAULT_HS)
    for item in a.hs:
        k, v = item.split("=")
        hs[k] = [float(x) for x in v.split(",")]
    report = {"device": torch.cuda.get_device_name(0)}
    for name in a.only.split(","):
        w = configs.CONFIGS[name](a.n) if a.n else configs.CONFIGS[name]()
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
        disp = float(np.hypot(*(w.target - w.q).T).max())
        rows = []
        for h in hs[name]:
            t0 = time.perf_counter()
            r = device.match(spec, w.q, w.target, h, w.epsilon, a.max_iter or w.max_iter, w.stop_rule, "max",
                             w.t_final, w.steps)
            wall = time.perf_counter() - t0
            ep = r["endpoint"].cpu().numpy()
            p0 = r["p0"].cpu().numpy()
            hist = list(r["residual_history"])
            row = {"h": h, "iterations": r["iterations"], "converged": r["converged"], "diagnosis": r["diagnosis"],
                   "history_head": hist[:4], "history_tail": hist[-4:], "history_min": min(hist) if hist else None,
                   "final_residual": r["final_residual"], "max_abs_endpoint": float(np.abs(ep).max()),
                   "max_abs_p0": float(np.abs(p0).max()), "hamiltonian": r["hamiltonian"],
                   "seconds_device": r["seconds_device"], "wall_s": wall,
                   "s_per_feedback_iteration": r["seconds_device"] / max(1, r["iterations"])}
            rows.append(row)
            print(name, json.dumps(row), flush=True)
        report[name] = {"n": w.n, "max_target_displacement": disp, "rows": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
