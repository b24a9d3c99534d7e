"""Helper for tests/test_gpu_cluster.py: one match per update space and one evolve with frames
through the small-N kernel, in a process whose cluster size is fixed by GS_B200_CLUSTER."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main(out):
    import paper_1510_03816_b200 as gs

    n = 128
    ref = gs.circle(1.0, n=n)
    tgt = gs.ellipse_rot_shift(1.05, 0.97, 0.0, (0.01, 0.0), n=n)  # a gentle, well-conditioned match
    res = {}
    for space, h in (("momentum", 0.05), ("velocity", 0.4)):  # momentum steps need h < 2 / lambda_max(K)
        cfg = gs.ShootingConfig(h=h, epsilon=1e-8, max_iter=1000, update_space=space,
                                evolve=gs.EvolveConfig(steps=30), system=gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.3)))
        r = gs.match(ref, tgt, cfg)
        res[f"{space}_p0"] = r.p0
        res[f"{space}_it"] = np.array(r.iterations)
        res[f"{space}_H"] = np.array(r.hamiltonian)
    rng = np.random.default_rng(4)
    p = rng.normal(0, 0.2, (n, 2))
    ev = gs.evolve(gs.SystemSpec(sigma2=0.1), gs.ParticleState(ref.points, p), gs.EvolveConfig(steps=40, capture_every=7))
    res["evolve_q"] = ev.final.q
    res["frames_q"] = np.stack([s.q for _, s in ev.frames])
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
