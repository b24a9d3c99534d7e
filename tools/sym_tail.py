"""Wave / tail structure of the symmetric dense kernel: time gs_stage_pairs_sym over the first k
CTAs (k = whole waves of `resident` CTAs) and over all of them, at one config.

    python tools/sym_tail.py --config C2 [--resident 888]

If the CTAs run in lockstep waves, t(all) ~ t(ceil(waves)) and the partial last wave costs a whole
wave; if they desynchronise, t grows ~linearly in k.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--resident", type=int, default=888)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, sharded

    w = getattr(configs, a.config.lower())()
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    be = sharded.DeviceStageBackend(spec)
    q, p = torch.from_numpy(w.q).cuda(), torch.from_numpy(w.p).cuda()
    n = q.shape[0]
    be.begin(q, p, 0, n)
    total = be.sym_parts()
    R = be.new_partials(n)

    def t_of(k):
        be.pairs_sym(1, 0, 0, k, R)
        ts = []
        for _ in range(a.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            be.pairs_sym(1, 0, 0, k, R)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return float(np.median(ts))

    ks = sorted({min(total, a.resident * j) for j in range(1, math.ceil(total / a.resident) + 1)} | {total})
    rows = [{"ctas": k, "waves": k / a.resident, "ms": t_of(k)} for k in ks]
    for r in rows:
        r["ms_per_wave"] = r["ms"] / r["waves"]
    print(json.dumps({"config": a.config, "n": n, "ctas": total, "resident": a.resident, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
