"""Small workloads of each kernel family, run under compute-sanitizer by tools/sanitize.sh.

    python tools/sanitize_targets.py <target>

targets: small (C1 match: k_small on an 8-CTA cluster, DSMEM st.async + mbarrier exchange),
small1 (N = 40: one-CTA k_small), sym (dense RHS N = 4096: k_dense_sym, shared J accumulators),
partial (dense RHS N = 1024: k_dense_partial), cell (cell RHS N = 20000: k_cell_pair, CUB sort),
verlet (cell evolve N = 20000, 3 steps: cluster Verlet build + sweep + IF-node rebuilds),
match (dense match N = 600: the conditional-WHILE loop graph), batch (batched sweep items),
velocity (gs_gram + velocity-space match N = 96).
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    t = sys.argv[1]
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    rng = np.random.default_rng(1)
    if t in ("small", "small1"):
        w = configs.c1() if t == "small" else None
        if w is None:
            q = gs.circle(1.0, n=40).points
            y = gs.ellipse_rot_shift(1.3, 0.7, 0.0, n=40).points
            alpha = 0.5 / gs.LAMBDA
        else:
            q, y, alpha = w.q, w.target, w.alpha
        r = device.match(gs.SystemSpec(kernel=gs.KernelSpec(alpha=alpha)), q, y, 0.3, 1e-6, 5, "residual", "max", 1.0,
                         20)
        print(t, r["iterations"], r["diagnosis"])
    elif t in ("sym", "partial"):
        n = 4096 if t == "sym" else 1024
        q, p = rng.uniform(0, 1, (n, 2)), rng.normal(0, 0.01, (n, 2))
        gs.set_path("dense")
        dq, dp = gs.rhs(gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.05 / gs.LAMBDA)), gs.ParticleState(q, p))
        print(t, float(np.abs(dq).max()))
    elif t in ("cell", "verlet"):
        w = configs.c4(20000)
        p = rng.normal(0, 1e-3, w.q.shape)
        gs.set_path("cell")
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
        if t == "cell":
            dq, dp = gs.rhs(spec, gs.ParticleState(w.q, p))
        else:
            out = gs.evolve(spec, gs.ParticleState(w.q, p), gs.EvolveConfig(t_final=0.15, steps=3))
            dq = out.final.q
        print(t, float(np.abs(dq).max()))
    elif t == "match":
        q = gs.circle(1.0, n=600).points
        y = gs.ellipse_rot_shift(1.3, 0.7, 0.0, n=600).points
        gs.set_path("dense")
        r = device.match(gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.3 / gs.LAMBDA)), q, y, 0.3, 1e-6, 3, "residual",
                         "max", 1.0, 5)
        print(t, r["iterations"], r["diagnosis"])
    elif t == "batch":
        a, b = gs.circle(1.0, n=24), gs.ellipse_rot_shift(1.2, 0.8, 0.0, n=24)
        grid = gs.SweepGrid((0.3, 0.6), (0.2, 0.4), n_landmarks=24, max_iter=5)
        print(t, gs.convergence_sweep(a, b, grid).tolist())
    elif t == "velocity":
        a, b = gs.circle(1.0, n=96), gs.ellipse_rot_shift(1.2, 0.8, 0.0, n=96)
        cfg = gs.ShootingConfig(h=0.5, max_iter=4, update_space="velocity", evolve=gs.EvolveConfig(steps=5),
                                system=gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.4)))
        r = gs.match(a, b, cfg)
        print(t, r.iterations, r.diagnosis)
    else:
        raise SystemExit(f"unknown target {t}")


if __name__ == "__main__":
    main()
