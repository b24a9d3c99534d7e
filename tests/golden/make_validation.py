"""Input-validation fixtures: exception type and message of the UNMODIFIED reference for
malformed inputs (empty / ragged / wrong-shape / non-finite / mismatched arrays, bad configs,
duplicate landmarks).  Build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_validation.py

References: particles.py:36-64 (_as_points, ParticleState), :67-76 (SystemSpec),
kernels.py:72-81 (KernelSpec), shapes.py:38-67 (LandmarkTemplate), integrator.py:22-43
(EvolveConfig), shooting.py:218-240 (match's template check).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def cases(g):
    """name -> zero-argument callable that is expected to raise (or not) in `g`'s API."""
    Z = np.zeros
    return {
        "state_empty": lambda: g.ParticleState(Z((0, 2)), Z((0, 2))),
        "state_3col": lambda: g.ParticleState(Z((4, 3)), Z((4, 3))),
        "state_1d": lambda: g.ParticleState(Z(4), Z(4)),
        "state_mismatch": lambda: g.ParticleState(Z((4, 2)), Z((3, 2))),
        "state_nan_q": lambda: g.ParticleState(np.array([[0.0, np.nan]]), Z((1, 2))),
        "state_inf_p": lambda: g.ParticleState(Z((1, 2)), np.array([[np.inf, 0.0]])),
        "state_ragged": lambda: g.ParticleState([[0.0, 1.0], [2.0]], Z((2, 2))),
        "state_single": lambda: g.ParticleState(Z((1, 2)), Z((1, 2))),
        "spec_neg_sigma2": lambda: g.SystemSpec(kernel=g.KernelSpec(), sigma2=-1.0),
        "kernel_neg_alpha": lambda: g.KernelSpec(alpha=-1.0),
        "kernel_bad_family": lambda: g.KernelSpec(family="nope"),
        "tmpl_empty": lambda: g.LandmarkTemplate(Z((0, 2)), "e"),
        "tmpl_dup": lambda: g.LandmarkTemplate(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 0.0]]), "d"),
        "tmpl_nan": lambda: g.LandmarkTemplate(np.array([[0.0, np.nan]]), "n"),
        "evolve_steps0": lambda: g.EvolveConfig(t_final=1.0, steps=0),
        "evolve_tneg": lambda: g.EvolveConfig(t_final=-1.0, steps=3),
        "match_size_mismatch": lambda: g.match(g.circle(1.0, n=8), g.circle(1.0, n=9), g.ShootingConfig(h=0.3)),
    }


def outcomes(g):
    out = {}
    for name, f in cases(g).items():
        try:
            f()
            out[name] = None
        except Exception as e:  # noqa: BLE001 — the fixture records whatever the reference raises
            out[name] = [type(e).__name__, str(e)]
    return out


if __name__ == "__main__":
    sys.path.insert(0, "/root/reference/pkg/src")
    import geoshoot

    with open(os.path.join(HERE, "validation.json"), "w") as f:
        json.dump(outcomes(geoshoot), f, indent=1, sort_keys=True)
        f.write("\n")
