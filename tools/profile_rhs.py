"""One RHS of a BASELINE config on the device (target for ncu captures).

    python tools/profile_rhs.py --config C5 --path cell --reps 3
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--path", default="auto")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--save", default="", help="write dq, dp of the last RHS to this .npz")
    ap.add_argument("--evolve", type=int, default=0, help="time an evolve of this many RK4 steps instead")
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    w = configs.CONFIGS[a.config]()
    p = w.p if w.p is not None else w.h * (w.target - w.q)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    gs.set_path(a.path)
    q_d, p_d = torch.from_numpy(w.q).cuda(), torch.from_numpy(np.ascontiguousarray(p)).cuda()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(a.reps):
        s.record()
        if a.evolve:
            dq, dp, _ = device.evolve(spec, q_d, p_d, a.evolve * w.t_final / w.steps, a.evolve)
        else:
            dq, dp = device.rhs(spec, q_d, p_d)
        e.record()
        torch.cuda.synchronize()
        what = f"evolve {a.evolve} steps" if a.evolve else "rhs"
        print(f"{a.config} {a.path} {what} {s.elapsed_time(e):.3f} ms", flush=True)

    if a.save:
        np.savez(a.save, dq=dq.cpu().numpy(), dp=dp.cpu().numpy())


if __name__ == "__main__":
    main()
