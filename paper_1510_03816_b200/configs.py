"""Seeded synthetic inputs for the five BASELINE configurations (C1..C5).

The reference publishes no datasets for this path; every BASELINE input is
synthetic.  The draw order below is frozen: tests, golden
fixtures and bench.py all build their inputs through these functions.

KD-1: "conical kernel with support radius sigma" is the
reference's ``KernelSpec(family="conical", alpha=sigma/LAMBDA)`` with
LAMBDA = 53 ln 2, so G(sigma) = 2**-53.  The kernel itself keeps the
reference's infinite support (``kernels.py:129-132``); the cell-list path
truncates at r = sigma, which changes results by <= ~1e-15 relative.

This module is numpy-only so that it can be imported by the golden-vector
generator (next to the reference) and by bench.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

LAMBDA = 53.0 * math.log(2.0)


def alpha_for_support(sigma: float) -> float:
    """KD-1: kernel length scale alpha whose conical kernel is 2**-53 at r = sigma."""
    return sigma / LAMBDA


@dataclass(frozen=True)
class Workload:
    name: str
    q: np.ndarray            # (N, 2) reference / initial positions
    p: np.ndarray | None     # (N, 2) initial momenta (RHS / evolve configs)
    target: np.ndarray | None  # (N, 2) target landmarks (matching configs)
    sigma: float             # support radius (KD-1)
    t_final: float
    steps: int
    h: float | None = None
    epsilon: float | None = None
    max_iter: int | None = None
    sigma2: float = 0.0
    stop_rule: str = "residual"

    @property
    def n(self) -> int:
        return self.q.shape[0]

    @property
    def alpha(self) -> float:
        return alpha_for_support(self.sigma)


def _circle(radius: float, n: int) -> np.ndarray:
    # shapes.py:79-87 (uniform angles, counterclockwise from angle 0)
    theta = 2.0 * np.pi * np.arange(n) / n
    return np.column_stack([0.0 + radius * np.cos(theta), 0.0 + radius * np.sin(theta)])


def _ellipse(a: float, b: float, n: int) -> np.ndarray:
    # shapes.py:90-118 at angle 0, shift (0, 0)
    theta = 2.0 * np.pi * np.arange(n) / n
    x = a * math.cos(0.0) * np.cos(theta) + b * math.sin(0.0) * np.sin(theta) + 0.0
    y = b * math.cos(0.0) * np.sin(theta) - a * math.sin(0.0) + 0.0
    return np.column_stack([x, y])


def c1() -> Workload:
    """Exact matching, N=64: unit circle -> ellipse (1.3, 0.7), sigma=0.5, h=0.3."""
    return Workload(
        name="C1", q=_circle(1.0, 64), p=None, target=_ellipse(1.3, 0.7, 64),
        sigma=0.5, t_final=1.0, steps=20, h=0.3, epsilon=1e-6, max_iter=200,
    )


def c2(n: int = 16384) -> Workload:
    """RHS microbenchmark: uniform [0,1]^2 (seed 0), p ~ N(0, 0.01^2) (seed 1), sigma=0.05."""
    q = np.random.default_rng(0).uniform(0.0, 1.0, (n, 2))
    p = np.random.default_rng(1).normal(0.0, 0.01, (n, 2))
    return Workload(name="C2", q=q, p=p, target=None, sigma=0.05, t_final=1.0, steps=100)


def c3(n: int = 131072) -> Workload:
    """Dense all-pairs stress: uniform (seed 2), p ~ N(0, 1e-4 variance) (seed 3), sigma=2."""
    q = np.random.default_rng(2).uniform(0.0, 1.0, (n, 2))
    p = np.random.default_rng(3).normal(0.0, 1e-2, (n, 2))
    return Workload(name="C3", q=q, p=p, target=None, sigma=2.0, t_final=1.0, steps=50)


def _displacement(x: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    a = rng.uniform(-1.0, 1.0, (4, 2))
    k = rng.integers(1, 4, (4, 2))
    phi = rng.uniform(0.0, 2.0 * np.pi, 4)
    out = np.zeros_like(x)
    for m in range(4):
        phase = 2.0 * np.pi * (x[:, 0] * k[m, 0] + x[:, 1] * k[m, 1]) + phi[m]
        out += a[m][None, :] * np.sin(phase)[:, None]
    return 0.05 * out


# Feedback gains of C4 / C5 (BASELINE.json leaves h open).  The survey's
# proposals (0.1 / 0.4) throw the first shoot's cloud apart: under KD-1 the momentum equation of
# these dense clouds is stiff, and a 20-step RK4 shoot blows up once max|p| reaches ~0.007 (C4) /
# ~0.015 (C5), whatever h is; h only sets how many iterations it takes to get there.  Measured on
# the B200 at full size (tools/h_scan.py, profiles/r02_h_scan.json): C4 blows up at iteration
# 1 / 4 / 36 / 71 / 91 for h = 0.1 / 0.02 / 0.002 / 0.001 / 0.0007 and completes its 100 iterations
# at 0.0005 and 0.0003; C5 blows up at iteration 2 / 6 / 10 / 19 for h = 0.4 / 0.02 / 0.01 / 0.005
# and completes its 20 at 0.004 (momentum delta already rising at the end), 0.003 and 0.002.
C4_H = 0.0005
C5_H = 0.003


def c4(n: int = 262144) -> Workload:
    """Clustered exact matching: 16 Gaussians (seed 4), smooth target (seed 5), sigma=0.02, h=C4_H."""
    r = np.random.default_rng(4)
    centres = r.uniform(0.1, 0.9, (16, 2))
    lab = r.integers(0, 16, n)
    x = centres[lab] + r.normal(0.0, 0.03, (n, 2))
    y = x + _displacement(x, np.random.default_rng(5))
    return Workload(
        name="C4", q=x, p=None, target=y, sigma=0.02, t_final=1.0, steps=20,
        h=C4_H, epsilon=1e-6, max_iter=100,
    )


def c5(n: int = 1048576) -> Workload:
    """Inexact matching: uniform (seed 6), smooth target + N(0, 0.002^2) noise (seed 7),
    sigma=0.01, sigma2=0.1, h=C5_H, exactly 20 iterations (eps=1e-300)."""
    x = np.random.default_rng(6).uniform(0.0, 1.0, (n, 2))
    r7 = np.random.default_rng(7)
    y = x + _displacement(x, r7)
    y = y + r7.normal(0.0, 0.002, (n, 2))
    return Workload(
        name="C5", q=x, p=None, target=y, sigma=0.01, t_final=1.0, steps=20,
        h=C5_H, epsilon=1e-300, max_iter=20, sigma2=0.1, stop_rule="momentum-delta",
    )


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}
