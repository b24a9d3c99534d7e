"""A/B of library builds (compile-time knobs) on the timed workloads, one process per build.

    python -c "from paper_1510_03816_b200 import _build; _build.build(defines=['GS_EXP_HISEL=1'], tag='zh')"
    python tools/ab_lib.py base zh base zh        # under gpurun; base = the product library

Per build: C2 dense RHS (symmetric kernel), the C2 dense 100-step solve, the C2 cell-path solve and
4 RK4 steps of C4 / C5 through the cluster Verlet lists (ms per RHS), plus the max relative
difference of every output against the first build listed.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def child(out: str, which: str):
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    def timed(fn, reps):
        """(last result, median ms per call; each call between its own events after 2 warm-ups)"""
        fn()
        fn()
        ts = []
        for _ in range(max(3, reps)):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            r = fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return r, float(np.median(ts))

    res, arrays = {}, {}
    w = configs.c2()
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    q, p = torch.from_numpy(w.q).cuda(), torch.from_numpy(w.p).cuda()
    if "dense" in which:
        device.set_path("dense")
        (dq, dp), res["c2_dense_rhs_ms"] = timed(lambda: device.rhs(spec, q, p), 20)
        arrays["c2_rhs_dq"], arrays["c2_rhs_dp"] = dq.cpu().numpy(), dp.cpu().numpy()
        (qT, pT, _), ms = timed(lambda: device.evolve(spec, q, p, 1.0, 100), 2)
        res["c2_dense_solve_ms"] = ms
        arrays["c2_solve_q"] = qT.cpu().numpy()
    if "cell" in which:
        device.set_path("cell")
        (qT, pT, _), res["c2_cell_solve_ms"] = timed(lambda: device.evolve(spec, q, p, 1.0, 100), 5)
        arrays["c2_cell_q"] = qT.cpu().numpy()
        for name in ("C4", "C5"):
            wk = configs.CONFIGS[name]()
            sp = gs.SystemSpec(kernel=gs.KernelSpec(alpha=wk.alpha), sigma2=wk.sigma2)
            qk = torch.from_numpy(wk.q).cuda()
            pk = torch.from_numpy(np.ascontiguousarray(wk.h * (wk.target - wk.q))).cuda()
            (qT, _, _), ms = timed(lambda: device.evolve(sp, qk, pk, 4 * wk.t_final / wk.steps, 4), 3)
            res[f"{name.lower()}_cell_rhs_ms"] = ms / 16
            arrays[f"{name.lower()}_q"] = qT.cpu().numpy()
    np.savez(out, **arrays)
    print("RESULT " + json.dumps(res), flush=True)


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        return
    which = os.environ.get("AB_WHICH", "dense,cell")
    tags = sys.argv[1:]
    first = None
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    for k, tag in enumerate(tags):
        lib = os.path.join(REPO, "paper_1510_03816_b200", "libgs_b200.so" if tag == "base" else f"libgs_b200_{tag}.so")
        out = os.path.join(REPO, "gpurun_out", f"ab_{k}_{tag}.npz")
        env = dict(os.environ, GS_B200_LIB=lib)
        r = subprocess.run([sys.executable, __file__, "--child", out, which], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if not line:
            print(tag, "FAILED", r.stdout[-2000:], r.stderr[-2000:], flush=True)
            continue
        res = json.loads(line[0][7:])
        a = np.load(out)
        if first is None:
            first = a
        diffs = {key: float(np.abs(a[key] - first[key]).max() / max(np.abs(first[key]).max(), 1e-300))
                 for key in a.files if key in first.files}
        worst = max(diffs.values()) if diffs else 0.0
        print(f"{tag:8s} " + " ".join(f"{key} {v:.4f}" for key, v in res.items()) + f"  maxrel vs {tags[0]} {worst:.1e}",
              flush=True)
        os.remove(out)


if __name__ == "__main__":
    main()
