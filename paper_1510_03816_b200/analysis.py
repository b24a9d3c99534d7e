"""Shape analysis over batches of independent matches (mirror of geoshoot/analysis.py).

SURVEY.md §8(f2): every function here that the reference runs as a serial loop of
independent matches — sweep cells (analysis.py:254-283), cluster-test pairs (:162-207),
exactness rows (:326-377), isometry pairs (:129-150) — runs them side by side as one
batched device launch (device.match_batch: one persistent CTA per match for N <= 512), with
the velocity-space Gram factors built on the device.  Names, arguments, results, validation
and error behaviour follow the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from . import device
from . import errors as _errors
from . import types as _types
from .kernels import KernelFamily, KernelSpec, family_name
from .particles import SystemSpec
from .shooting import (ShootingConfig, StopRule, _batchable, _enum_value, _factor_of, _make_result, _prepare,
                       match, match_config_dict)

__all__ = [
    "DIVERGED", "SweepGrid", "DistanceRecord", "ClusterVerdict", "ExactnessRow", "shape_distance",
    "iso_invariance_check", "cluster_test", "convergence_sweep", "predict",
    "exact_vs_inexact", "match_many",
]

DIVERGED = -1  # analysis.py:41


@dataclass(frozen=True)
class SweepGrid:
    """The alpha^2 x h plane of a sweep (analysis.py:44-76)."""

    alpha2_values: tuple
    h_values: tuple
    n_landmarks: int = 16
    kernel_family: KernelFamily = KernelFamily.CONICAL
    tolerance: float = 1e-6
    max_iter: int = 500

    def __post_init__(self):
        object.__setattr__(self, "alpha2_values", tuple(float(a) for a in self.alpha2_values))
        object.__setattr__(self, "h_values", tuple(float(h) for h in self.h_values))
        object.__setattr__(self, "kernel_family", KernelFamily(_enum_value(self.kernel_family)))
        if not self.alpha2_values or not self.h_values:
            raise _errors.ConfigurationError("sweep axes must be non-empty")
        for name, vals in (("alpha2", self.alpha2_values), ("h", self.h_values)):
            if any(not (v > 0 and math.isfinite(v)) for v in vals):
                raise _errors.ConfigurationError(f"{name} values must be positive, got {vals}")
        if self.n_landmarks < 3:
            raise _errors.ConfigurationError(f"n_landmarks must be >= 3, got {self.n_landmarks}")
        if not (self.tolerance > 0 and math.isfinite(self.tolerance)):
            raise _errors.ConfigurationError(f"tolerance must be positive, got {self.tolerance}")
        if self.max_iter < 1:
            raise _errors.ConfigurationError(f"max_iter must be >= 1, got {self.max_iter}")


@dataclass(frozen=True)
class DistanceRecord:
    reference_label: str
    target_label: str
    H: float
    iterations: int
    converged: bool


@dataclass(frozen=True)
class ClusterVerdict:
    same_cluster: bool | None
    evidence: tuple


@dataclass(frozen=True)
class ExactnessRow:
    sigma2: float
    h: float
    H: float
    final_residual: float
    iterations: int
    converged: bool


# --- the batched match ----------------------------------------------------------------------
def match_many(pairs, cfgs) -> list:
    """``[match(ref, tgt, cfg) for (ref, tgt), cfg in zip(pairs, cfgs)]`` as batched launches.

    Items with equal landmark count and kernel family run in one gs_match_batch launch (one
    CTA each); velocity-space items bring their Gram factor (built and factored on the
    device once per distinct (kernel, q0)).  An item whose setup raises (non-SPD Gram matrix,
    bad templates) yields that exception object in its slot instead of a result, so callers
    can reproduce the reference's per-item try/except.  Items that cannot batch (N > 512 or
    the cell path) run through shooting.match one by one.
    """
    torch = device._torch()
    out: list = [None] * len(pairs)
    groups: dict = {}
    for k, ((ref, tgt), cfg) in enumerate(zip(pairs, cfgs)):
        try:
            _prepare(ref, tgt)
            device.system_struct(cfg.system)  # family available on the device
        except _errors.GeoshootError as exc:
            out[k] = exc
            continue
        if not _batchable(ref.n):
            try:
                out[k] = match(ref, tgt, cfg)
            except _errors.GeoshootError as exc:
                out[k] = exc
            continue
        vel = _enum_value(cfg.update_space) == "velocity"
        key = (ref.n, _enum_value(cfg.system.kernel.family), vel)
        groups.setdefault(key, []).append(k)

    factors: dict = {}
    for (n, _, vel), idx in groups.items():
        live, Ls, warns = [], [], {}
        for k in idx:
            (ref, _), cfg = pairs[k], cfgs[k]
            if vel:
                fk = (cfg.system.kernel, ref.points.tobytes())
                if fk not in factors:
                    try:
                        K = device.gram(cfg.system, device.as_device(ref.points, torch))
                        factors[fk] = _factor_of(K, torch)
                    except _errors.GeoshootError as exc:
                        factors[fk] = exc
                f = factors[fk]
                if isinstance(f, Exception):
                    out[k] = f
                    continue
                Ls.append(f[0])
                warns[k] = f[2]
            live.append(k)
        if not live:
            continue
        q0 = torch.stack([device.as_device(pairs[k][0].points, torch) for k in live])
        tg = torch.stack([device.as_device(pairs[k][1].points, torch) for k in live])
        fac = torch.stack(Ls) if vel else None
        rs = device.match_batch([cfgs[k].system for k in live], [match_config_dict(cfgs[k]) for k in live], q0, tg,
                                factor=fac)
        p0 = torch.stack([r["p0"] for r in rs]).cpu().numpy()
        ep = torch.stack([r["endpoint"] for r in rs]).cpu().numpy()
        for i, (k, r) in enumerate(zip(live, rs)):
            ref, tgt = pairs[k]
            out[k] = _make_result(p0[i], r["iterations"], r["converged"], r["residual_history"], r["hamiltonian"],
                                  ep[i], ref, tgt, r["final_residual"], r["diagnosis"], warns.get(k, ()))
    return out


def _raise_or(res):
    if isinstance(res, Exception):
        raise res
    return res


def _record(reference, target, res) -> DistanceRecord:
    return _types.get("DistanceRecord")(reference_label=reference.label, target_label=target.label, H=res.hamiltonian,
                          iterations=res.iterations, converged=res.converged)


# --- analysis.py entry points ------------------------------------------------------------------
def shape_distance(reference, target, cfg) -> DistanceRecord:
    """analysis.py:109-126."""
    return _record(reference, target, match(reference, target, cfg))


def iso_invariance_check(a, b, g, cfg) -> float:
    """analysis.py:129-150: both matches in one batch."""
    plain, moved = (_raise_or(r) for r in match_many([(a, b), (g.apply(a), g.apply(b))], [cfg, cfg]))
    for name, res in (("original", plain), ("transformed", moved)):
        if not res.converged:
            raise _errors.DivergenceError(
                f"isometry check: the {name} pair did not converge ({res.diagnosis or 'iteration cap reached'})")
    return moved.hamiltonian - plain.hamiltonian


def _normalized(t):
    """analysis.py:153-159: centroid at the origin, unit RMS radius."""
    pts = t.points - t.points.mean(axis=0)
    scale = float(np.sqrt(np.mean(np.sum(pts * pts, axis=1))))
    if scale == 0.0:
        raise _errors.ConfigurationError(f"template {t.label!r} has zero extent")
    return _types.get("LandmarkTemplate")(pts / scale, t.label)


def cluster_test(a, b, refs: list, thresholds: dict, cfg, preprocess: bool = False) -> ClusterVerdict:
    """analysis.py:162-207: the 1 + 2 len(refs) distance matches in one batch."""
    if len(refs) < 2:
        raise _errors.ConfigurationError(f"need at least 2 reference shapes, got {len(refs)}")
    missing = {"pair", "ref_diff"} - set(thresholds)
    if missing:
        raise _errors.ConfigurationError(f"thresholds missing {sorted(missing)}")
    pair_thr = float(thresholds["pair"])
    ref_thr = float(thresholds["ref_diff"])
    if not (pair_thr > 0 and ref_thr > 0):
        raise _errors.ConfigurationError("thresholds must be positive")
    if preprocess:
        a, b = _normalized(a), _normalized(b)
        refs = [_normalized(r) for r in refs]
    pairs = [(a, b)]
    for ref in refs:
        pairs += [(ref, a), (ref, b)]
    results = [_raise_or(r) for r in match_many(pairs, [cfg] * len(pairs))]
    evidence = [_record(x, y, r) for (x, y), r in zip(pairs, results)]
    if not all(rec.converged for rec in evidence):
        return _types.get("ClusterVerdict")(same_cluster=None, evidence=tuple(evidence))
    verdict = evidence[0].H <= pair_thr and all(
        abs(evidence[i].H - evidence[i + 1].H) <= ref_thr for i in range(1, len(evidence), 2))
    return _types.get("ClusterVerdict")(same_cluster=verdict, evidence=tuple(evidence))


def convergence_sweep(reference, target, grid: SweepGrid) -> np.ndarray:
    """analysis.py:254-283: every (alpha^2, h) cell in ONE batched launch.

    A cell is DIVERGED when its run blows up, degenerates, or exhausts max_iter; a cell
    whose setup raises a GeoshootError is DIVERGED too, exactly as the reference's
    try/except around each match.
    """
    pairs, cfgs = [], []
    for alpha2 in grid.alpha2_values:
        kernel = KernelSpec(family=grid.kernel_family, alpha=math.sqrt(alpha2), normalized=True)
        for h in grid.h_values:
            cfgs.append(ShootingConfig(h=h, epsilon=grid.tolerance, max_iter=grid.max_iter,
                                       system=SystemSpec(kernel=kernel)))
            pairs.append((reference, target))
    if family_name(cfgs[0].system.kernel) not in ("conical", "gaussian"):
        device.system_struct(cfgs[0].system)  # raises: the family is not on the device path
    results = match_many(pairs, cfgs)
    out = np.empty((len(grid.alpha2_values), len(grid.h_values)), dtype=int)
    for k, res in enumerate(results):
        i, j = divmod(k, len(grid.h_values))
        if isinstance(res, _errors.GeoshootError):
            out[i, j] = DIVERGED
        elif isinstance(res, Exception):
            raise res
        else:
            out[i, j] = res.iterations if res.converged else DIVERGED
    return out


def predict(reference, target_partial, t_match: float, t_predict: float, cfg):
    """analysis.py:286-323: match over [0, t_match], then run the momenta on to t_predict."""
    if not (0.0 < t_match < 1.0):
        raise _errors.ConfigurationError(f"t_match must lie in (0, 1), got {t_match}")
    if not (t_predict >= t_match and math.isfinite(t_predict)):
        raise _errors.ConfigurationError(f"t_predict must be >= t_match ({t_match}), got {t_predict}")
    match_cfg = replace(cfg, evolve=replace(cfg.evolve, t_final=t_match))
    res = match(reference, target_partial, match_cfg)
    if not res.converged:
        raise _errors.DivergenceError(
            f"prediction match failed after {res.iterations} iterations "
            f"({res.diagnosis or 'iteration cap reached'})")
    steps = max(1, math.ceil(cfg.evolve.steps * t_predict / t_match))
    q, _, _ = device.evolve(cfg.system, reference.points, res.p0, t_predict, steps)
    label = f"{reference.label}>{target_partial.label}@t={t_predict:g}"
    return _types.get("LandmarkTemplate")(q.cpu().numpy(), label)


def exact_vs_inexact(reference, target, sigma2_values, cfg, h_by_sigma2: dict | None = None) -> tuple:
    """analysis.py:326-360: the exact row and every relaxation row in one batch."""
    exact_cfg = replace(cfg, stop_rule=StopRule.TARGET_RESIDUAL, system=replace(cfg.system, sigma2=0.0))
    rows_cfg = [(0.0, exact_cfg)]
    for sigma2 in sigma2_values:
        s2 = float(sigma2)
        if s2 < 0:
            raise _errors.ConfigurationError(f"sigma2 must be >= 0, got {s2}")
        h = cfg.h if h_by_sigma2 is None else float(h_by_sigma2.get(s2, cfg.h))
        rows_cfg.append((s2, replace(cfg, h=h, stop_rule=StopRule.MOMENTUM_DELTA,
                                     system=replace(cfg.system, sigma2=s2))))
    results = match_many([(reference, target)] * len(rows_cfg), [c for _, c in rows_cfg])
    rows = []
    for (s2, c), res in zip(rows_cfg, results):
        res = _raise_or(res)
        rows.append(_types.get("ExactnessRow")(sigma2=s2, h=c.h, H=res.hamiltonian, final_residual=res.final_residual,
                                 iterations=res.iterations, converged=res.converged))
    return tuple(rows)


_types.register_defaults(DistanceRecord=DistanceRecord, ClusterVerdict=ClusterVerdict, ExactnessRow=ExactnessRow)
