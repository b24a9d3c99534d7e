"""Whole device matches of a BASELINE config (target for ncu captures of the small-N kernel).

    python tools/profile_match.py --config C1 --reps 3
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    w = configs.CONFIGS[a.config]()
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    for _ in range(a.reps):
        r = device.match(spec, w.q, w.target, w.h, w.epsilon, w.max_iter, "residual", "max", 1.0, w.steps)
        print(f"{a.config} match: {r['iterations']} iterations, {r['seconds_device'] / max(1, r['iterations']) * 1e3:.4f} "
              f"ms per feedback iteration", flush=True)


if __name__ == "__main__":
    main()
