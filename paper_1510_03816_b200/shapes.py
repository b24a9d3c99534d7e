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


# Pairs can only have a zero computed distance if both coordinate differences are below ~2^-537
# (their squares underflow); grouping by this (larger) gap keeps every such pair in one group.
_GAP = 1e-150


def _chains(v: np.ndarray, gid: np.ndarray):
    """Sorted order of (gid, v) and the group id of each sorted element: groups of equal gid whose
    consecutive v differ by less than _GAP."""
    order = np.lexsort((v, gid))
    vs, gs_ = v[order], gid[order]
    brk = np.ones(v.size, dtype=bool)
    brk[1:] = (gs_[1:] != gs_[:-1]) | ~(np.abs(vs[1:] - vs[:-1]) < _GAP)
    return order, np.cumsum(brk) - 1


def first_coincident_pair(pts: np.ndarray):
    """(i, j) of the row-major-first pair whose distance the reference computes as 0.0
    (``sqrt(dx*dx + dy*dy) == 0``, kernels.py:174-178 via shapes.py:52-58), or None.

    The reference's test includes distinct points whose squared difference underflows; pairs
    are grouped by coordinate gaps below _GAP (x, then y within an x-group), and every pair
    inside a group is tested with the reference's own formula.  O(N log N) for any input
    whose groups are small (the common case: groups of one)."""
    n = pts.shape[0]
    if n < 2:
        return None
    x, y = np.ascontiguousarray(pts[:, 0]), np.ascontiguousarray(pts[:, 1])
    ox, gx = _chains(x, np.zeros(n, dtype=np.int64))
    gxi = np.empty(n, dtype=np.int64)
    gxi[ox] = gx
    oy, gy = _chains(y, gxi)
    sizes = np.bincount(gy)
    if sizes.max() < 2:
        return None
    best = None
    starts = np.concatenate([[0], np.cumsum(sizes)])
    for g in np.flatnonzero(sizes >= 2):
        members = np.sort(oy[starts[g]:starts[g + 1]])
        sub = pts[members]
        for k in range(0, members.size, 512):  # bounded memory even for one huge group
            d = sub[k:k + 512, None, :] - sub[None, :, :]
            dist = np.sqrt(np.sum(d * d, axis=-1))
            rows = np.arange(k, min(k + 512, members.size))
            dist[rows - k, rows] = np.inf
            hit = np.argwhere(dist == 0.0)
            if hit.size:
                a, b = hit[0]
                cand = (int(members[a + k]), int(members[b]))
                if best is None or cand < best:
                    best = cand
                break  # rows are in ascending member order: later chunks only give larger i
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
