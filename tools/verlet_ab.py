"""A/B of the cluster Verlet list knobs (read at gs_create) on the cell-path evolves.

    python tools/verlet_ab.py --knob GS_B200_SKIN=0.05,0.1,0.2 [--knob GS_B200_VERLET_DEPTH=128,1024]
                              [--configs C2,C4,C5] [--steps 4] [--reps 2]

C2: the 100-step solve; C4 / C5: `steps` RK4 steps from the first shoot's momenta.  Prints ms per
RHS, the list builds per evolve and the agreement with the first variant.
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import itertools
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--knob", action="append", default=[])
    ap.add_argument("--configs", default="C2,C4,C5")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import configs, device

    knobs = [(k.split("=")[0], k.split("=")[1].split(",")) for k in a.knob]
    gs.set_path("cell")
    for name in a.configs.split(","):
        w = configs.CONFIGS[name]()
        if name == "C2":
            p, steps, tf = w.p, 100, 1.0
        else:
            p, steps, tf = w.h * (w.target - w.q), a.steps, a.steps / w.steps
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
        qd, pd = torch.from_numpy(w.q).cuda(), torch.from_numpy(np.ascontiguousarray(p)).cuda()
        ref = None
        for combo in itertools.product(*[v for _, v in knobs]):
            env = {k: v for (k, _), v in zip(knobs, combo)}
            os.environ.update(env)
            N.Context.swap()
            gc.collect()  # free the previous variant's context now, not inside a timed region
            device.evolve(spec, qd, pd, tf, steps)
            ctx = N.Context.get()
            b0, e0 = ctypes.c_int64(), ctypes.c_int64()
            ctx.lib.gs_cell_stats(ctx.handle, ctypes.byref(b0), ctypes.byref(e0), None)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for _ in range(a.reps):
                qT, pT, _ = device.evolve(spec, qd, pd, tf, steps)
            e.record()
            torch.cuda.synchronize()
            b1, e1 = ctypes.c_int64(), ctypes.c_int64()
            ctx.lib.gs_cell_stats(ctx.handle, ctypes.byref(b1), ctypes.byref(e1), None)
            ms = s.elapsed_time(e) / a.reps
            out = qT.cpu().numpy()
            if ref is None:
                ref = out
            diff = float(np.abs(out - ref).max() / np.abs(ref).max())
            print(f"{name} {env}: {ms / (4 * steps):.4f} ms/RHS ({ms:.2f} ms/evolve), "
                  f"builds/evolve {(b1.value - b0.value) / a.reps:.1f}, list cap {e1.value}, vs first {diff:.1e}",
                  flush=True)


if __name__ == "__main__":
    main()
