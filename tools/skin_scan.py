"""Whole device matches of C4 / C5 per Verlet skin (one process per skin: GS_B200_SKIN is read
when the library context is created).

    python tools/skin_scan.py --config C5 --skins adaptive,default,0.04,0.05,0.075,0.1 [--iters 20]

Prints, per skin, the seconds per feedback iteration of the second whole match in the process
(the first allocates the list buffer and captures the graphs) and the list builds per iteration.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(config: str, iters: int) -> dict:
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import configs, device

    w = configs.CONFIGS[config]()
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    ctx = N.Context.get()

    def builds():
        b, e = ctypes.c_int64(), ctypes.c_int64()
        N.check(ctx.lib.gs_cell_stats(ctx.handle, ctypes.byref(b), ctypes.byref(e), None), "gs_cell_stats")
        return b.value

    out = {}
    for rep in range(2):
        b0 = builds()
        r = device.match(spec, w.q, w.target, w.h, w.epsilon, iters, w.stop_rule, "max", w.t_final, w.steps)
        it = max(1, r["iterations"])
        out = {"iterations": r["iterations"], "s_per_iteration": r["seconds_device"] / it,
               "builds_per_iteration": (builds() - b0) / it, "converged": bool(r["converged"])}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--skins", default="0.05,0.075,0.1")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(one(a.config, a.iters)))
        return
    for s in a.skins.split(","):
        # "adaptive": the library's adaptive skin; "default": its fixed default; else a fixed skin
        env = dict(os.environ)
        if s == "default":
            env["GS_B200_SKIN_ADAPT"] = "0"
        elif s != "adaptive":
            env["GS_B200_SKIN"] = s
        p = subprocess.run([sys.executable, __file__, "--child", "--config", a.config, "--iters", str(a.iters)],
                           env=env, capture_output=True, text=True)
        line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-400:]
        print(f"{a.config} skin {s}: {line}", flush=True)


if __name__ == "__main__":
    main()
