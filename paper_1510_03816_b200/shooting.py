"""Feedback-control geodesic shooting on the B200 (mirror of geoshoot/shooting.py:33-320).

``match`` with ``UpdateSpace.MOMENTUM`` — the update of BASELINE.json's north_star,
p0 <- p0 + h (Y - X(T)) (shooting.py:266-267) — runs entirely in libgs_b200.so: the
initial shoot, every RK4 stage, the residual, its norm, the update and both stop rules,
with one persistent kernel for N <= 512 and a device loop reading two scalars per
iteration above that.  ``UpdateSpace.VELOCITY`` (the reference default)
builds the Gram matrix on the device (gs_gram), factors it once with cuSOLVER (torch.linalg)
and runs each iteration as a triangular solve pair plus a device shoot.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import device
from . import errors as _errors
from . import types as _types
from .integrator import EvolveConfig
from .particles import SystemSpec

__all__ = ["UpdateSpace", "StopRule", "ResidualNorm", "ShootingConfig", "MatchResult", "match",
           "contraction_diagnostics", "momenta_from_velocity", "newton_match", "gram_factor"]

_BLOWUP_FACTOR = 1e6          # shooting.py:47
_ILL_CONDITIONED = 1e12       # shooting.py:48


class UpdateSpace(str, enum.Enum):
    VELOCITY = "velocity"
    MOMENTUM = "momentum"


class StopRule(str, enum.Enum):
    TARGET_RESIDUAL = "residual"
    MOMENTUM_DELTA = "momentum-delta"


class ResidualNorm(str, enum.Enum):
    MAX = "max"
    L2 = "l2"


@dataclass(frozen=True)
class ShootingConfig:
    """Knobs of the matching iteration (shooting.py:66-100)."""

    h: float
    epsilon: float = 1e-3
    max_iter: int = 500
    update_space: UpdateSpace = UpdateSpace.VELOCITY
    stop_rule: StopRule = StopRule.TARGET_RESIDUAL
    norm: ResidualNorm = ResidualNorm.MAX
    evolve: EvolveConfig = field(default_factory=EvolveConfig)
    system: SystemSpec = field(default_factory=SystemSpec)

    def __post_init__(self):
        object.__setattr__(self, "update_space", UpdateSpace(self.update_space))
        object.__setattr__(self, "stop_rule", StopRule(self.stop_rule))
        object.__setattr__(self, "norm", ResidualNorm(self.norm))
        if not (self.h > 0 and math.isfinite(self.h)):
            raise _errors.ConfigurationError(f"h must be positive, got {self.h}")
        if not (self.epsilon > 0 and math.isfinite(self.epsilon)):
            raise _errors.ConfigurationError(f"epsilon must be positive, got {self.epsilon}")
        if self.max_iter < 1:
            raise _errors.ConfigurationError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.system.sigma2 > 0 and self.stop_rule is not StopRule.MOMENTUM_DELTA:
            raise _errors.ConfigurationError(
                "inexact matching (sigma2 > 0) cannot stop on the endpoint "
                "residual; use stop_rule = MomentumDelta")


@dataclass(frozen=True)
class MatchResult:
    """Outcome of one matching run (shooting.py:103-121)."""

    p0: np.ndarray
    iterations: int
    converged: bool
    residual_history: tuple
    hamiltonian: float
    final_template: object
    final_residual: float
    diagnosis: str | None = None
    warnings: tuple = ()


def _enum_value(e) -> str:
    return str(getattr(e, "value", e))


def _norm(kind: str, vec: np.ndarray) -> float:
    """shooting.py:124-135."""
    arr = np.asarray(vec, dtype=float).reshape(-1, 2)
    if kind == "max":
        return float(np.max(np.hypot(arr[:, 0], arr[:, 1])))
    return float(np.linalg.norm(arr.ravel()))


def _make_result(p0, iterations, converged, history, hamiltonian, endpoint, reference, target, final_residual,
                 diagnosis, warnings):
    final = _types.get("LandmarkTemplate")(endpoint, f"{reference.label}>{target.label}")
    return _types.get("MatchResult")(
        p0=p0, iterations=iterations, converged=converged, residual_history=tuple(history),
        hamiltonian=hamiltonian, final_template=final, final_residual=final_residual, diagnosis=diagnosis,
        warnings=warnings)


def _prepare(reference, target) -> None:
    if reference.n != target.n:
        raise _errors.ConfigurationError(
            f"templates must have equal landmark counts: {reference.n} (reference) vs {target.n} (target)")


def match(reference, target, cfg):
    """Find initial momenta carrying ``reference`` onto ``target`` (shooting.py:218-301)."""
    _prepare(reference, target)
    if _enum_value(cfg.update_space) == "velocity":
        return _match_velocity(reference, target, cfg)
    r = device.match(cfg.system, reference.points, target.points, cfg.h, cfg.epsilon, cfg.max_iter,
                     _enum_value(cfg.stop_rule), _enum_value(cfg.norm), cfg.evolve.t_final, cfg.evolve.steps)
    return _make_result(r["p0"].cpu().numpy(), r["iterations"], r["converged"], r["residual_history"],
                        r["hamiltonian"], r["endpoint"].cpu().numpy(), reference, target, r["final_residual"],
                        r["diagnosis"], ())


# --- velocity-space update: Gram solve on the device -----------------------
SMALL_MAX = 512  # gs_small.cu kSmallMax: one persistent CTA per match


def gram_factor(spec, q0):
    """_GramSolver.__init__ (shooting.py:143-152) on the device.

    The Gram matrix over q0 comes from libgs_b200 (`gs_gram`, kernels.py:181-197); its
    Cholesky factor and 2-norm condition number (= np.linalg.cond for an SPD K, via the
    eigenvalues) from cuSOLVER through torch.linalg — a library factorisation, once per match.
    Returns (L, cond, warnings); raises DegenerateConfigurationError when K is not SPD.
    """
    torch = device._torch()
    K = device.gram(spec, device.as_device(q0, torch))
    return _factor_of(K, torch)


def _factor_of(K, torch):
    evals = torch.linalg.eigvalsh(K)
    amin, amax = float(evals.abs().min()), float(evals.abs().max())
    cond = amax / amin if amin > 0 else math.inf
    L, info = torch.linalg.cholesky_ex(K)
    if int(info) != 0:
        raise _errors.DegenerateConfigurationError(
            f"kernel Gram matrix is not positive definite: {int(info)}-th leading minor of the array is not "
            "positive definite")
    warnings = ()
    if not (cond < _ILL_CONDITIONED):
        warnings = (f"Gram matrix condition number {cond:.3e} exceeds {_ILL_CONDITIONED:.0e}; "
                    "momenta recovery may lose accuracy",)
    return L, cond, warnings


def _batchable(n: int) -> bool:
    return n <= SMALL_MAX and device.get_path() != "cell"


def match_config_dict(cfg) -> dict:
    """ShootingConfig -> the per-item dict of device.match_batch."""
    return dict(h=cfg.h, epsilon=cfg.epsilon, max_iter=cfg.max_iter, stop_rule=_enum_value(cfg.stop_rule),
                norm=_enum_value(cfg.norm), t_final=cfg.evolve.t_final, steps=cfg.evolve.steps)


CG_TOL = 1e-14          # relative residual of the matrix-free Gram solve
CG_MAX_IT = 2000
DENSE_FALLBACK_MAX = 16384  # CG stagnating (ill-conditioned K): dense Cholesky up to this N (K = 2 GB)


class CGGramSolver:
    """_GramSolver (shooting.py:138-159) for N above the persistent-kernel range, without forming K:
    p = K^-1 u by conjugate gradients on the device (gs_gram_cg: K v is the dq half of the RHS at
    (q0, v) through the pair kernels, dense or the cluster lists of q0), warm-started from the
    previous iteration's p (u changes by h r per iteration).  cond(K) for the reference's warning
    (shooting.py:145, 237-242) is estimated from the first solve's Lanczos coefficients.  When CG
    stagnates above 1e-10 (a near-singular K) and N <= DENSE_FALLBACK_MAX, the solver switches to the
    reference's own method: the dense Gram matrix (gs_gram) and its Cholesky factor (cuSOLVER)."""

    def __init__(self, spec, q0):
        self.spec, self.q0 = spec, q0
        self.p = None
        self.condition = None
        self.factor = None
        self.solves = self.cg_iterations = 0

    def solve(self, u):
        torch = device._torch()
        if self.factor is not None:
            return torch.cholesky_solve(u, self.factor)
        p, it, rel, coef = device.gram_cg(self.spec, self.q0, u, self.p, CG_TOL, CG_MAX_IT)
        self.solves += 1
        self.cg_iterations += it
        if self.condition is None and coef:
            self.condition = device.lanczos_condition(coef)
        if rel > 1e-10 and self.q0.shape[0] <= DENSE_FALLBACK_MAX:
            self.factor, self.condition, _ = gram_factor(self.spec, self.q0)
            return torch.cholesky_solve(u, self.factor)
        self.p = p
        return p

    def warnings(self, u_probe=None):
        if self.condition is None and u_probe is not None:
            self.solve(u_probe)
        cond = self.condition if self.condition is not None else 1.0
        if not (cond < _ILL_CONDITIONED):
            return (f"Gram matrix condition number {cond:.3e} exceeds {_ILL_CONDITIONED:.0e}; "
                    "momenta recovery may lose accuracy",)
        return ()


def _match_velocity(reference, target, cfg):
    """shooting.py:218-301 with UpdateSpace.VELOCITY: u <- u + h r, p = K^-1 u (:263-265).

    N <= 512: the whole loop — the triangular solve pair of every iteration included — runs in
    one persistent CTA (gs_match_batch with the Gram factor, cuSOLVER Cholesky once).  Above
    that K is never formed: each iteration solves K p = u by matrix-free conjugate gradients on
    the device (CGGramSolver), then shoots on the device; the host reads the residual norm.
    """
    torch = device._torch()
    q0 = device.as_device(reference.points, torch)
    if _batchable(reference.n):
        L, _, warnings = gram_factor(cfg.system, q0)
        r = device.match_batch([cfg.system], [match_config_dict(cfg)], q0, target.points, factor=L)[0]
        return _make_result(r["p0"].cpu().numpy(), r["iterations"], r["converged"], r["residual_history"],
                            r["hamiltonian"], r["endpoint"].cpu().numpy(), reference, target, r["final_residual"],
                            r["diagnosis"], warnings)
    solver = CGGramSolver(cfg.system, q0)
    tgt = device.as_device(target.points, torch)
    norm_kind = _enum_value(cfg.norm)
    mdelta = _enum_value(cfg.stop_rule) == "momentum-delta"
    ev = cfg.evolve

    def dnorm(r) -> float:
        if norm_kind == "max":
            return float(torch.hypot(r[:, 0], r[:, 1]).max())
        return float(torch.linalg.vector_norm(r.reshape(-1)))

    def result(p, history, converged, endpoint, diagnosis):
        return _make_result(p.cpu().numpy(), len(history), converged, history,
                            device.hamiltonian(cfg.system, q0, p), endpoint.cpu().numpy(), reference, target,
                            dnorm(tgt - endpoint), diagnosis, solver.warnings(tgt - q0))

    u = torch.zeros_like(q0)
    p = torch.zeros_like(q0)
    endpoint = q0.clone()  # evolve(q0, 0) leaves q0 unchanged
    residual = tgt - endpoint
    history: list = []
    initial = None
    if not mdelta:
        initial = dnorm(residual)
        if initial < cfg.epsilon:
            return result(p, history, True, endpoint, None)
    for _ in range(cfg.max_iter):
        delta = cfg.h * dnorm(residual)
        u = u + cfg.h * residual
        p = solver.solve(u)
        try:
            endpoint_new, _, _ = device.evolve(cfg.system, q0, p, ev.t_final, ev.steps, 0)
        except (_errors.DivergenceError, _errors.DegenerateConfigurationError) as exc:
            return result(p, history, False, endpoint, f"step too large ({exc})")
        endpoint = endpoint_new
        residual = tgt - endpoint
        value = delta if mdelta else dnorm(residual)
        if initial is None:
            initial = value
        history.append(value)
        if not math.isfinite(value) or (initial > 0 and value > _BLOWUP_FACTOR * initial):
            return result(p, history, False, endpoint, "step too large")
        if value < cfg.epsilon:
            return result(p, history, True, endpoint, None)
    return result(p, history, False, endpoint, "iteration cap reached before the stopping rule")


def momenta_from_velocity(kernel, q0, u0) -> np.ndarray:
    """shooting.py:162-175: solve (K (x) I2) p = u on the device (Gram kernel + Cholesky)."""
    q0 = np.asarray(q0, dtype=float)
    u0 = np.asarray(u0, dtype=float)
    if q0.shape != u0.shape or q0.ndim != 2 or q0.shape[1] != 2:
        raise ValueError(f"q0 and u0 must both have shape (N, 2), got {q0.shape} and {u0.shape}")
    torch = device._torch()
    spec = SystemSpec(kernel=kernel)
    if q0.shape[0] > SMALL_MAX:  # matrix-free: K is never formed
        return CGGramSolver(spec, device.as_device(q0, torch)).solve(device.as_device(u0, torch)).cpu().numpy()
    L, _, _ = gram_factor(spec, q0)
    return torch.cholesky_solve(device.as_device(u0, torch), L).cpu().numpy()


def newton_match(reference, target, cfg):
    """Finite-difference Newton baseline (shooting.py:327-411) with batched Jacobian columns.

    Every iteration needs 2N + 1 shoots; the reference runs the 2N Jacobian columns one after
    another.  Here the 2N probe momenta come from one multi-right-hand-side Cholesky solve and
    the 2N column shoots run side by side in ONE persistent launch (gs_evolve_batch, one CTA
    per column); the dense 2N x 2N Newton system is an LU solve on the device
    (torch.linalg, cuSOLVER).  Same probe step, same fallback to the feedback update on a
    singular or unevaluable Jacobian, same stop logic and diagnoses as the reference.
    """
    _prepare(reference, target)
    if _enum_value(cfg.stop_rule) != "residual":
        raise _errors.ConfigurationError("newton_match supports only the TargetResidual rule")
    torch = device._torch()
    n = reference.n
    q0 = device.as_device(reference.points, torch)
    tgt = device.as_device(target.points, torch).reshape(-1)
    L, _, warnings = gram_factor(cfg.system, q0)
    ev = cfg.evolve
    norm_kind = _enum_value(cfg.norm)

    def solve(u_flat):  # (..., 2n) -> p (..., n, 2)
        return torch.cholesky_solve(u_flat.reshape(n, 2), L)

    def shoot(u_flat):
        q, _, _ = device.evolve(cfg.system, q0, solve(u_flat), ev.t_final, ev.steps, 0)
        return q.reshape(-1)

    def dnorm(r) -> float:
        if norm_kind == "max":
            r2 = r.reshape(-1, 2)
            return float(torch.hypot(r2[:, 0], r2[:, 1]).max())
        return float(torch.linalg.vector_norm(r))

    def result(u, history, converged, endpoint, diagnosis):
        p = solve(u)
        return _make_result(p.cpu().numpy(), len(history), converged, history,
                            device.hamiltonian(cfg.system, q0, p), endpoint.reshape(n, 2).cpu().numpy(), reference,
                            target, dnorm(tgt - endpoint), diagnosis, warnings)

    u = torch.zeros(2 * n, dtype=torch.float64, device=q0.device)
    endpoint = shoot(u)
    residual = tgt - endpoint
    initial_norm = dnorm(residual)
    history: list = []
    if initial_norm < cfg.epsilon:
        return result(u, history, True, endpoint, None)
    eye = torch.eye(2 * n, dtype=torch.float64, device=q0.device)
    for _ in range(cfg.max_iter):
        step = 1e-5 * max(1.0, float(u.abs().max()))
        probes = u[None, :] + step * eye                      # row j = u + step e_j
        rhs_cols = probes.reshape(2 * n, n, 2).permute(1, 0, 2).reshape(n, 4 * n)
        P = torch.cholesky_solve(rhs_cols, L).reshape(n, 2 * n, 2).permute(1, 0, 2).contiguous()
        cols_q, _, errs = device.evolve_batch(cfg.system, q0, P, ev.t_final, ev.steps)
        newton_step = None
        if all(e is None for e in errs):
            jac = ((cols_q.reshape(2 * n, 2 * n) - endpoint[None, :]) / step).T.contiguous()
            sol, info = torch.linalg.solve_ex(jac, residual)
            if int(info) == 0 and bool(torch.isfinite(sol).all()):
                newton_step = sol
        elif any(e is not None and not isinstance(e, (_errors.DivergenceError,
                                                      _errors.DegenerateConfigurationError)) for e in errs):
            raise next(e for e in errs if e is not None)
        if newton_step is None:  # singular or unevaluable Jacobian: one feedback update
            newton_step = residual
        u = u + cfg.h * newton_step
        try:
            endpoint_new = shoot(u)
        except (_errors.DivergenceError, _errors.DegenerateConfigurationError) as exc:
            return result(u, history, False, endpoint, f"step too large ({exc})")
        endpoint = endpoint_new
        residual = tgt - endpoint
        value = dnorm(residual)
        history.append(value)
        if not math.isfinite(value) or (initial_norm > 0 and value > _BLOWUP_FACTOR * initial_norm):
            return result(u, history, False, endpoint, "step too large")
        if value < cfg.epsilon:
            return result(u, history, True, endpoint, None)
    return result(u, history, False, endpoint, "iteration cap reached before the stopping rule")


def contraction_diagnostics(result) -> list:
    """Consecutive stopping-norm ratios |r(k+1)| / |r(k)| (shooting.py:304-320)."""
    hist = result.residual_history
    if len(hist) < 2:
        return []
    return [hist[i + 1] / hist[i] if hist[i] > 0 else math.inf for i in range(len(hist) - 1)]


_types.register_defaults(MatchResult=MatchResult)
