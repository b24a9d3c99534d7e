"""numpy restatement of the reference hot path — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows, symbol by symbol:

* ``kernels.py:121-171``  kernel_value / kernel_derivative (conical, gaussian)
* ``kernels.py:174-178``  pairwise_distances (row-blocked here)
* ``particles.py:79-117`` _interaction_terms / rhs, including the coincidence
  error naming the first (i, j) in row-major order and the reference's own dp
  formula ``-(a.sum(1)[:, None] * q - a @ q)`` (``particles.py:116``)
* ``particles.py:120-131`` hamiltonian (full double sum, no 1/2)
* ``particles.py:140-150`` velocity_field (kernel-reconstructed velocity at sample points)
* ``integrator.py:66-121`` fixed-step RK4 with its error re-wrapping
* ``shooting.py:124-135, 178-179, 218-301`` _norm / _blown_up / match, both update spaces
  (momentum ``:266-267``; velocity ``:138-159, 263-265`` with scipy's Cholesky, as the reference),
  both stop rules, both norms.

Row blocking changes only the BLAS blocking of the row-block products, so the
results agree with the reference to rounding (pinned in tests/test_oracle.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CONICAL, GAUSSIAN = 0, 1
BLOWUP_FACTOR = 1e6          # shooting.py:47


class OracleDegenerate(ValueError):
    """Mirrors geoshoot.errors.DegenerateConfigurationError."""


class OracleDivergence(RuntimeError):
    """Mirrors geoshoot.errors.DivergenceError."""


@dataclass(frozen=True)
class Kernel:
    family: int = CONICAL
    alpha: float = 1.0
    normalized: bool = True

    def peak(self) -> float:                       # kernels.py:83-88
        return 1.0 / (2.0 * math.pi * self.alpha * self.alpha)

    @staticmethod
    def from_params(kp) -> "Kernel":
        return Kernel(int(kp[0]), float(kp[1]), bool(kp[2]))


def kernel_value(k: Kernel, r: np.ndarray) -> np.ndarray:
    """kernels.py:121-142 (conical/gaussian branches)."""
    if k.family == CONICAL:
        out = np.exp(-r / k.alpha)
    else:
        out = np.exp(-0.5 * (r / k.alpha) ** 2)
    if not k.normalized:
        out *= k.peak()
    return out


def kernel_derivative(k: Kernel, r: np.ndarray) -> np.ndarray:
    """kernels.py:145-171 (r > 0 only)."""
    if k.family == CONICAL:
        out = -np.exp(-r / k.alpha) / k.alpha
    else:
        out = -(r / k.alpha**2) * np.exp(-0.5 * (r / k.alpha) ** 2)
    if not k.normalized:
        out *= k.peak()
    return out


def _coincident_error(i: int, j: int) -> OracleDegenerate:
    # particles.py:92-98
    return OracleDegenerate(
        f"particles {i} and {j} coincide with interacting momenta; "
        "the momentum equation is singular there"
    )


def rhs_rows(k: Kernel, sigma2: float, q: np.ndarray, p: np.ndarray, r0: int, r1: int):
    """Rows [r0, r1) of particles.rhs (particles.py:79-117)."""
    qi, pi = q[r0:r1], p[r0:r1]
    diff = qi[:, None, :] - q[None, :, :]
    dist = np.sqrt(np.sum(diff * diff, axis=-1))
    with np.errstate(over="ignore", invalid="ignore"):
        kmat = kernel_value(k, dist)
        pdot = pi @ p.T
    rows = np.arange(r0, r1)
    off_diag = rows[:, None] != np.arange(q.shape[0])[None, :]
    coincident = (dist == 0.0) & off_diag
    bad = coincident & (pdot != 0.0)
    if np.any(bad):
        i, j = np.argwhere(bad)[0]
        raise _coincident_error(int(i) + r0, int(j))
    safe = dist.copy()
    safe[~off_diag] = 1.0
    safe[coincident] = 1.0
    with np.errstate(over="ignore", invalid="ignore"):
        a = pdot * kernel_derivative(k, safe) / safe
        a[~off_diag] = 0.0
        a[coincident] = 0.0
        dq = kmat @ p
        if sigma2 != 0.0:
            dq = dq + sigma2 * pi
        dp = -(a.sum(axis=1)[:, None] * qi - a @ q)
    return dq, dp


def rhs(k: Kernel, sigma2: float, q: np.ndarray, p: np.ndarray, block: int = 2048):
    """particles.rhs, evaluated in row blocks of ``block`` targets."""
    n = q.shape[0]
    if not (np.all(np.isfinite(q)) and np.all(np.isfinite(p))):
        raise ValueError("state contains non-finite entries")   # particles.py:57-58
    dq = np.empty_like(q)
    dp = np.empty_like(q)
    for r0 in range(0, n, block):
        r1 = min(n, r0 + block)
        dq[r0:r1], dp[r0:r1] = rhs_rows(k, sigma2, q, p, r0, r1)
    return dq, dp


def hamiltonian(k: Kernel, q: np.ndarray, p: np.ndarray, block: int = 2048) -> float:
    """particles.py:120-131: sum_ij (p_i . p_j) G(d_ij)."""
    n = q.shape[0]
    total = 0.0
    for r0 in range(0, n, block):
        r1 = min(n, r0 + block)
        diff = q[r0:r1, None, :] - q[None, :, :]
        kmat = kernel_value(k, np.sqrt(np.sum(diff * diff, axis=-1)))
        total += float(np.sum(p[r0:r1] * (kmat @ p)))
    return total


def velocity_field(k: Kernel, q: np.ndarray, p: np.ndarray, x: np.ndarray, block: int = 2048) -> np.ndarray:
    """particles.py:140-150: u(x_m) = sum_j G(|x_m - q_j|) p_j for an (M, 2) batch x."""
    x = np.atleast_2d(np.asarray(x, dtype=float))
    u = np.empty_like(x)
    for r0 in range(0, x.shape[0], block):
        r1 = min(x.shape[0], r0 + block)
        dist = np.sqrt(np.sum((x[r0:r1, None, :] - q[None, :, :]) ** 2, axis=-1))
        u[r0:r1] = kernel_value(k, dist) @ p
    return u


def evolve(k: Kernel, sigma2: float, q0: np.ndarray, p0: np.ndarray, t_final: float = 1.0,
           steps: int = 100, capture_every: int = 0, rhs_fn=None):
    """integrator.py:66-121.  Returns (q, p, frames)."""
    f = rhs_fn or (lambda qq, pp: rhs(k, sigma2, qq, pp))
    dt = t_final / steps
    t_at = lambda s: t_final * (s / steps)
    q = q0.copy()
    p = p0.copy()
    frames = []
    if capture_every > 0:
        frames.append((0.0, q.copy(), p.copy()))
    with np.errstate(over="ignore", invalid="ignore"):
        for step in range(steps):
            t = t_at(step)
            try:
                k1q, k1p = f(q, p)
                k2q, k2p = f(q + 0.5 * dt * k1q, p + 0.5 * dt * k1p)
                k3q, k3p = f(q + 0.5 * dt * k2q, p + 0.5 * dt * k2p)
                k4q, k4p = f(q + dt * k3q, p + dt * k3p)
            except OracleDegenerate as exc:
                raise OracleDegenerate(f"{exc} (during step {step + 1}, t in [{t:.6g}, {t + dt:.6g}])") from exc
            except ValueError as exc:
                raise OracleDivergence(
                    f"non-finite intermediate at step {step + 1} (t in [{t:.6g}, {t + dt:.6g}]); "
                    "the step size is too large for this configuration") from exc
            q = q + (dt / 6.0) * (k1q + 2.0 * k2q + 2.0 * k3q + k4q)
            p = p + (dt / 6.0) * (k1p + 2.0 * k2p + 2.0 * k3p + k4p)
            if not (np.all(np.isfinite(q)) and np.all(np.isfinite(p))):
                raise OracleDivergence(
                    f"non-finite state at step {step + 1} (t = {t_at(step + 1):.6g}); "
                    "the step size is too large for this configuration")
            if capture_every > 0 and ((step + 1) % capture_every == 0 or step + 1 == steps):
                frames.append((t_at(step + 1), q.copy(), p.copy()))
    return q, p, frames


def norm(kind: str, vec: np.ndarray) -> float:
    """shooting.py:124-135."""
    arr = np.asarray(vec, dtype=float).reshape(-1, 2)
    if kind == "max":
        return float(np.max(np.hypot(arr[:, 0], arr[:, 1])))
    return float(np.linalg.norm(arr.ravel()))


def gram_matrix(k: Kernel, q: np.ndarray) -> np.ndarray:
    """kernels.py:181-197: K_ij = G(|q_i - q_j|)."""
    return kernel_value(k, np.sqrt(np.sum((q[:, None, :] - q[None, :, :]) ** 2, axis=-1)))


def match_momentum(k: Kernel, sigma2: float, q0: np.ndarray, target: np.ndarray, h: float,
                   epsilon: float, max_iter: int, stop_rule: str = "residual", norm_kind: str = "max",
                   t_final: float = 1.0, steps: int = 100, evolve_fn=None, update_space: str = "momentum") -> dict:
    """shooting.py:218-301: update_space MOMENTUM (p <- p + h r, shooting.py:266-267) or VELOCITY
    (u <- u + h r, p = K^-1 u with the Cholesky factor of the Gram matrix over q0 computed once,
    shooting.py:138-159, 263-265).

    Returns the MatchResult fields (hamiltonian included, shooting.py:182-207).
    """
    ev = evolve_fn or (lambda qq, pp: evolve(k, sigma2, qq, pp, t_final, steps)[0])
    n = q0.shape[0]
    p = np.zeros((n, 2))
    u = np.zeros((n, 2))
    factor = None
    if update_space == "velocity":
        from scipy.linalg import cho_factor, cho_solve

        factor = cho_factor(gram_matrix(k, q0), lower=True)

    def result(history, converged, endpoint, diagnosis):
        return dict(p0=p, iterations=len(history), converged=converged, residual_history=tuple(history),
                    hamiltonian=hamiltonian(k, q0, p), endpoint=endpoint,
                    final_residual=norm(norm_kind, target - endpoint), diagnosis=diagnosis)

    endpoint = ev(q0, p)
    residual = target - endpoint
    history: list = []
    initial = None
    if stop_rule == "residual":
        initial = norm(norm_kind, residual)
        if initial < epsilon:
            return result(history, True, endpoint, None)
    for _ in range(max_iter):
        delta = h * norm(norm_kind, residual)
        if factor is not None:
            u = u + h * residual
            p = cho_solve(factor, u)
        else:
            p = p + h * residual
        try:
            endpoint_new = ev(q0, p)
        except (OracleDivergence, OracleDegenerate) as exc:
            return result(history, False, endpoint, f"step too large ({exc})")
        endpoint = endpoint_new
        residual = target - endpoint
        if stop_rule == "residual":
            value = norm(norm_kind, residual)
        else:
            value = delta
            if initial is None:
                initial = value
        history.append(value)
        if not math.isfinite(value) or (initial > 0 and value > BLOWUP_FACTOR * initial):
            return result(history, False, endpoint, "step too large")
        if value < epsilon:
            return result(history, True, endpoint, None)
    return result(history, False, endpoint, "iteration cap reached before the stopping rule")
