"""Time the second feedback shoot of a matching config (the one after a blown-up first shoot).

    python tools/debug_shoot2.py --config C5 --n 262144
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--steps", type=int, default=0)
    a = ap.parse_args()
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    fn = configs.CONFIGS[a.config]
    w = fn(a.n) if a.n else fn()
    steps = a.steps or w.steps
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    p1 = w.h * (w.target - w.q)
    t0 = time.perf_counter()
    q1, _, _ = device.evolve(spec, w.q, p1, 1.0, steps)
    torch.cuda.synchronize()
    print(f"shoot 1: {time.perf_counter() - t0:.3f} s, max|q| {float(q1.abs().max()):.3e}", flush=True)
    p2 = p1 + w.h * (w.target - q1.cpu().numpy())
    big = np.abs(p2).max(axis=1)
    print(f"max|p2| {big.max():.3e}; |p2| > 1: {(big > 1).sum()} of {len(big)}; median {np.median(big):.3e}",
          flush=True)
    for k in (1, 2, 4):
        t0 = time.perf_counter()
        qk, _, _ = device.evolve(spec, w.q, p2, 1.0 * k / steps, k)
        torch.cuda.synchronize()
        qa = qk.abs().max(dim=1).values
        print(f"shoot 2, first {k} steps: {time.perf_counter() - t0:.3f} s, max|q| {float(qa.max()):.3e}, "
              f"#|q|>10: {int((qa > 10).sum())}", flush=True)
    t0 = time.perf_counter()
    try:
        q2, pp2, _ = device.evolve(spec, w.q, p2, 1.0, steps)
        torch.cuda.synchronize()
        print(f"shoot 2: {time.perf_counter() - t0:.3f} s, max|q| {float(q2.abs().max()):.3e}", flush=True)
    except Exception as exc:
        torch.cuda.synchronize()
        print(f"shoot 2: {time.perf_counter() - t0:.3f} s raised {type(exc).__name__}: {exc}", flush=True)


if __name__ == "__main__":
    main()
