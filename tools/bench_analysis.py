"""Time the batched analysis entry points on the device.

    python tools/bench_analysis.py [--out gpurun_out/analysis_bench.json] [--reps 3]

Runs every case of tests/golden/analysis_cases.json (the inputs of the reference's own tests)
through this package — one batched launch per sweep / cluster test / exactness table, the
Newton Jacobian columns as one batched launch per iteration — and reports wall-clock seconds
(best of --reps, after one warm-up) beside the reference's serial CPU time recorded when the
fixture was generated (`seconds`, build container CPU; the reference cannot run on the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "analysis_bench.json"))
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    import test_gpu_analysis as T

    def run(name):
        m = T.META[name]
        if name.startswith("sweep_"):
            grid = gs.SweepGrid(m["alpha2"], m["h"], n_landmarks=m["n_landmarks"], kernel_family=m["family"],
                                tolerance=m["tolerance"], max_iter=m["max_iter"])
            return lambda: gs.convergence_sweep(T._tpl(gs, m["ref"]), T._tpl(gs, m["tgt"]), grid)
        if name.startswith("cluster_"):
            return lambda: gs.cluster_test(T._tpl(gs, m["a"]), T._tpl(gs, m["b"]),
                                           [T._tpl(gs, r) for r in m["refs"]], m["thresholds"], T._cfg(gs, m["cfg"]))
        if name.startswith("newton_"):
            return lambda: gs.newton_match(T._tpl(gs, m["ref"]), T._tpl(gs, m["tgt"]), T._cfg(gs, m["cfg"]))
        return None

    report = {"device": torch.cuda.get_device_name(0), "cases": {}}
    for name in sorted(T.META):
        fn = run(name)
        if fn is None:
            continue
        fn()
        best = float("inf")
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        ref_s = T.META[name].get("seconds")
        report["cases"][name] = {"seconds": best, "reference_seconds_cpu_serial": ref_s,
                                 "speedup": (ref_s / best) if ref_s else None}
        print(name, report["cases"][name], flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
