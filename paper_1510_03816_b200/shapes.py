"""Landmark templates (mirror of geoshoot/shapes.py:38-67) with an O(N log N) coincidence check.

The reference validates a template through an N x N distance matrix (shapes.py:52-58),
which caps it near N = 30k in host memory.  Here the same rule — reject
the first coincident pair (i, j), i != j, in row-major order, with the same message — is
decided by a lexicographic sort, so templates of N = 1M landmarks are cheap.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import errors as _errors
from . import types as _types

__all__ = ["LandmarkTemplate", "first_coincident_pair", "circle", "ellipse_rot_shift"]


def first_coincident_pair(pts: np.ndarray):
    """(i, j) of the row-major-first pair of identical points, or None."""
    n = pts.shape[0]
    if n < 2:
        return None
    order = np.lexsort((pts[:, 1], pts[:, 0]))
    s = pts[order]
    same = (s[1:, 0] == s[:-1, 0]) & (s[1:, 1] == s[:-1, 1])
    if not np.any(same):
        return None
    best = None
    k = 0
    idx = np.flatnonzero(same)
    # walk runs of equal points: run spans sorted positions [a, b]
    while k < idx.size:
        a = idx[k]
        b = a + 1
        while k + 1 < idx.size and idx[k + 1] == b:
            k += 1
            b += 1
        members = np.sort(order[a:b + 1])
        cand = (int(members[0]), int(members[1]))
        if best is None or cand < best:
            best = cand
        k += 1
    return best


@dataclass(frozen=True)
class LandmarkTemplate:
    """Ordered planar landmarks; index i of one template corresponds to index i of another."""

    points: np.ndarray
    label: str = ""

    def __post_init__(self):
        pts = np.asarray(self.points, dtype=float)
        if pts.ndim != 2 or pts.shape[1] != 2 or pts.shape[0] < 1:
            raise ValueError(f"points must have shape (N, 2), got {pts.shape}")
        if not np.all(np.isfinite(pts)):
            raise ValueError("points contain non-finite entries")
        pair = first_coincident_pair(pts)
        if pair is not None:
            raise _errors.DegenerateConfigurationError(
                f"landmarks {pair[0]} and {pair[1]} coincide in template {self.label!r}")
        object.__setattr__(self, "points", pts)

    @property
    def n(self) -> int:
        return self.points.shape[0]

    def stacked(self) -> np.ndarray:
        return self.points.ravel()


def _check_n(n: int, minimum: int = 3) -> None:
    if n < minimum:
        raise _errors.ConfigurationError(f"need at least {minimum} landmarks, got {n}")


def circle(radius: float, center=(0.0, 0.0), n: int = 64, label: str | None = None):
    """n points on a circle at uniform angles, counterclockwise from angle 0 (shapes.py:79-87)."""
    if radius <= 0:
        raise _errors.ConfigurationError(f"radius must be positive, got {radius}")
    _check_n(n)
    theta = 2.0 * np.pi * np.arange(n) / n
    cx, cy = float(center[0]), float(center[1])
    pts = np.column_stack([cx + radius * np.cos(theta), cy + radius * np.sin(theta)])
    return _types.get("LandmarkTemplate")(pts, label if label is not None else f"circle(r={radius:g})")


def ellipse_rot_shift(a: float, b: float, angle: float, shift=(0.0, 0.0), n: int = 64, label: str | None = None):
    """Sheared ellipse of shapes.py:90-118 (the axis-aligned ellipse at angle 0)."""
    if a <= 0 or b <= 0:
        raise _errors.ConfigurationError(f"semi-axes must be positive, got a={a}, b={b}")
    _check_n(n)
    theta = 2.0 * np.pi * np.arange(n) / n
    sx, sy = float(shift[0]), float(shift[1])
    x = a * math.cos(angle) * np.cos(theta) + b * math.sin(angle) * np.sin(theta) + sx
    y = b * math.cos(angle) * np.sin(theta) - a * math.sin(angle) + sy
    return _types.get("LandmarkTemplate")(np.column_stack([x, y]),
                                          label if label is not None else f"ellipse(a={a:g},b={b:g})")


_types.register_defaults(LandmarkTemplate=LandmarkTemplate)
