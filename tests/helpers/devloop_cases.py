"""Large-N device matches (n > 512: the gs_match loop, not the small-N kernel) for
tests/test_gpu_devloop.py: run in this process, or as `python devloop_cases.py out.npz` in a
child whose environment selects the host-driven loop (GS_B200_DEVLOOP=0)."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def run_cases():
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import device

    n = 1024
    ref = gs.circle(1.0, n=n).points
    tgt = gs.ellipse_rot_shift(1.3, 0.7, 0.0, n=n).points
    narrow = gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.02 / gs.LAMBDA))
    wide = gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.3))
    cases = {
        # name: (spec, h, epsilon, max_iter, stop rule, norm, steps, path)
        "converge": (narrow, 0.3, 1e-6, 100, "residual", "max", 20, "dense"),
        "cap": (narrow, 0.3, 1e-6, 5, "residual", "l2", 20, "dense"),
        "mdelta": (narrow, 0.3, 1e-3, 100, "momentum-delta", "l2", 10, "dense"),
        "blowup": (wide, 50.0, 1e-6, 30, "residual", "max", 4, "dense"),
        "cell": (narrow, 0.3, 1e-6, 100, "residual", "max", 20, "cell"),
    }
    out = {}
    for name, (spec, h, eps, mi, rule, norm, steps, path) in cases.items():
        gs.set_path(path)
        try:
            r = device.match(spec, ref, tgt, h, eps, mi, rule, norm, 1.0, steps)
        finally:
            gs.set_path("auto")
        out[f"{name}__p0"] = r["p0"].cpu().numpy()
        out[f"{name}__endpoint"] = r["endpoint"].cpu().numpy()
        out[f"{name}__history"] = np.asarray(r["residual_history"], float)
        out[f"{name}__meta"] = np.array([r["iterations"], int(r["converged"]), r["hamiltonian"], r["final_residual"]])
        out[f"{name}__diagnosis"] = np.array(str(r["diagnosis"]))
    return out


if __name__ == "__main__":
    np.savez(sys.argv[1], **run_cases())
