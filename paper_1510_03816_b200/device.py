"""Device-resident entry points on torch CUDA tensors (fp64, (N, 2) C-order).

This is the layer every public function goes through: it converts the reference's spec
objects into the C-ABI structs, calls libgs_b200.so on the current torch stream and turns
the library's status records back into the reference's exceptions and messages
(particles.py:92-98, integrator.py:58-63, 102-112).  torch supplies device memory and
streams only; all arithmetic of the hot path runs in the library's kernels.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _native as N
from . import errors as _errors
from .kernels import family_name, support_radius

_PATHS = {"auto": N.GS_PATH_AUTO, "dense": N.GS_PATH_DENSE, "cell": N.GS_PATH_CELL}
_path = os.environ.get("GS_B200_PATH", "auto")


def set_path(path: str) -> None:
    """Pair-sum strategy for all later calls: "auto" | "dense" | "cell"."""
    global _path
    if path not in _PATHS:
        raise ValueError(f"path must be one of {sorted(_PATHS)}, got {path!r}")
    _path = path


def get_path() -> str:
    return _path


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return torch


def system_struct(spec, path: str | None = None) -> N.System:
    """SystemSpec (particles.py:67-76) + KernelSpec (kernels.py:50-88) -> gs_system_t."""
    k = spec.kernel
    fam = family_name(k)
    if fam == "conical":
        code = N.GS_FAMILY_CONICAL
    elif fam == "gaussian":
        code = N.GS_FAMILY_GAUSSIAN
    else:
        raise _errors.ConfigurationError(
            f"kernel family {fam!r} is not available on the B200 device path (conical, gaussian)")
    return N.System(code, 1 if k.normalized else 0, float(k.alpha), float(spec.sigma2), support_radius(k),
                    _PATHS[path or _path], 0)


class _PlainSpec:
    """The same kernel with sigma2 = 0 (the Hamiltonian has no sigma2 term, particles.py:120-131)."""

    def __init__(self, spec):
        self.kernel = spec.kernel
        self.sigma2 = 0.0


def _plain_spec(spec):
    return _PlainSpec(spec)


def _stream_ptr(torch) -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t) -> int:
    return t.data_ptr()


def as_device(a, torch=None):
    """numpy / torch (N, 2) -> contiguous cuda float64 tensor (a copy for host inputs)."""
    torch = torch or _torch()
    if isinstance(a, torch.Tensor):
        t = a.to(device="cuda", dtype=torch.float64)
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to("cuda")


def coincident_message(i: int, j: int) -> str:
    return (f"particles {i} and {j} coincide with interacting momenta; "
            "the momentum equation is singular there")


def status_exception(st: N.Status, t_final: float | None = None, steps: int | None = None):
    """gs_status_t -> the reference's exception (or None)."""
    code = st.code
    if code == N.GS_OK:
        return None
    if code == N.GS_ERR_COINCIDENT and steps is None:
        return _errors.DegenerateConfigurationError(coincident_message(st.i, st.j))
    if code == N.GS_ERR_INVALID:
        return ValueError("state contains non-finite entries")
    if code in (N.GS_ERR_COINCIDENT, N.GS_ERR_NONFINITE_STAGE, N.GS_ERR_NONFINITE_STATE):
        step = int(st.step)
        dt = t_final / steps
        t = t_final * ((step - 1) / steps)
        if code == N.GS_ERR_COINCIDENT:
            return _errors.DegenerateConfigurationError(
                f"{coincident_message(st.i, st.j)} (during step {step}, t in [{t:.6g}, {t + dt:.6g}])")
        if code == N.GS_ERR_NONFINITE_STAGE:
            return _errors.DivergenceError(
                f"non-finite intermediate at step {step} (t in [{t:.6g}, {t + dt:.6g}]); "
                "the step size is too large for this configuration")
        return _errors.DivergenceError(
            f"non-finite state at step {step} (t = {t_final * (step / steps):.6g}); "
            "the step size is too large for this configuration")
    return N.NativeError(code, N.last_error())


def rhs(spec, q, p):
    """particles.rhs on device tensors -> (dq, dp) cuda float64 (N, 2)."""
    torch = _torch()
    ctx = N.Context.get()
    q = as_device(q, torch)
    p = as_device(p, torch)
    n = q.shape[0]
    dq = torch.empty_like(q)
    dp = torch.empty_like(q)
    st = N.Status()
    sysc = system_struct(spec)
    rc = ctx.lib.gs_rhs(ctx.handle, ctypes.byref(sysc), n, _ptr(q), _ptr(p), _ptr(dq), _ptr(dp), ctypes.byref(st),
                        _stream_ptr(torch))
    if rc not in (N.GS_OK, N.GS_ERR_COINCIDENT, N.GS_ERR_INVALID):
        N.check(rc, "gs_rhs")
    exc = status_exception(st)
    if exc is not None:
        raise exc
    return dq, dp


def hamiltonian(spec, q, p) -> float:
    torch = _torch()
    ctx = N.Context.get()
    q = as_device(q, torch)
    p = as_device(p, torch)
    out = ctypes.c_double()
    sysc = system_struct(spec)
    N.check(ctx.lib.gs_hamiltonian(ctx.handle, ctypes.byref(sysc), q.shape[0], _ptr(q), _ptr(p), ctypes.byref(out),
                                   _stream_ptr(torch)), "gs_hamiltonian")
    return float(out.value)


def gram(spec, q):
    """kernels.gram_matrix (kernels.py:181-197) on the device: (N, N) cuda float64."""
    torch = _torch()
    ctx = N.Context.get()
    q = as_device(q, torch)
    n = q.shape[0]
    K = torch.empty((n, n), dtype=torch.float64, device=q.device)
    bi, bj = ctypes.c_int64(), ctypes.c_int64()
    sysc = system_struct(spec)
    rc = ctx.lib.gs_gram(ctx.handle, ctypes.byref(sysc), n, _ptr(q), _ptr(K), ctypes.byref(bi), ctypes.byref(bj),
                         _stream_ptr(torch))
    if rc == N.GS_ERR_COINCIDENT:
        raise _errors.DegenerateConfigurationError(
            f"points {bi.value} and {bj.value} coincide; Gram matrix would be singular")
    N.check(rc, "gs_gram")
    return K


def gram_cg(spec, q0, u, p0=None, tol: float = 1e-14, max_it: int = 2000):
    """p = K^-1 u without forming K (gs_gram_cg): conjugate gradients whose K v is the dq half of
    the RHS at (q0, v) through the library's pair kernels.  p0: warm start (zeros if None).
    Returns (p, iterations, relative residual, [(alpha_k, beta_k)])."""
    torch = _torch()
    ctx = N.Context.get()
    q0 = as_device(q0, torch)
    u = as_device(u, torch)
    n = q0.shape[0]
    p = torch.zeros_like(q0) if p0 is None else as_device(p0, torch).clone()
    coef = (ctypes.c_double * (2 * max(1, max_it)))()
    iters, relres = ctypes.c_int32(), ctypes.c_double()
    sysc = system_struct(spec)
    rc = ctx.lib.gs_gram_cg(ctx.handle, ctypes.byref(sysc), n, _ptr(q0), _ptr(u), _ptr(p), float(tol), int(max_it),
                            ctypes.byref(iters), coef, ctypes.byref(relres), _stream_ptr(torch))
    if rc == N.GS_ERR_COINCIDENT:
        raise _errors.DegenerateConfigurationError("kernel Gram matrix is not positive definite: coincident points")
    N.check(rc, "gs_gram_cg")
    k = int(iters.value)
    return p, k, float(relres.value), [(coef[2 * i], coef[2 * i + 1]) for i in range(k)]


def lanczos_condition(coefs) -> float:
    """cond(K) estimate from the CG coefficients: the extreme eigenvalues of the Lanczos
    tridiagonal T (diag 1/a_k + b_(k-1)/a_(k-1), off-diagonal sqrt(b_k)/a_k).  A lower bound that
    tightens with the iteration count."""
    if not coefs:
        return 1.0
    a = np.array([c[0] for c in coefs])
    b = np.array([c[1] for c in coefs])
    diag = 1.0 / a
    diag[1:] += b[:-1] / a[:-1]
    off = np.sqrt(np.maximum(b[:-1], 0.0)) / a[:-1]
    T = np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)
    ev = np.linalg.eigvalsh(T)
    return float(ev[-1] / ev[0]) if ev[0] > 0 else math.inf


def velocity_field(spec, q, p, x):
    """particles.velocity_field (particles.py:140-150) on the device: u (M, 2) cuda float64 at the
    sample points x (M, 2) for the state (q, p)."""
    torch = _torch()
    ctx = N.Context.get()
    q = as_device(q, torch)
    p = as_device(p, torch)
    x = as_device(x, torch)
    m = x.shape[0]
    u = torch.empty((m, 2), dtype=torch.float64, device=q.device)
    sysc = system_struct(spec)
    N.check(ctx.lib.gs_velocity_field(ctx.handle, ctypes.byref(sysc), q.shape[0], _ptr(q), _ptr(p), m, _ptr(x),
                                      _ptr(u), _stream_ptr(torch)), "gs_velocity_field")
    return u


def n_frames(steps: int, capture_every: int) -> int:
    if capture_every <= 0:
        return 0
    return 1 + steps // capture_every + (1 if steps % capture_every else 0)


def evolve(spec, q, p, t_final: float, steps: int, capture_every: int = 0, inplace: bool = False):
    """integrator.evolve on device tensors -> (q, p, frames[F, N, 4] or None)."""
    torch = _torch()
    ctx = N.Context.get()
    q = as_device(q, torch)
    p = as_device(p, torch)
    if not inplace:
        q = q.clone()
        p = p.clone()
    n = q.shape[0]
    nf = n_frames(steps, capture_every)
    frames = torch.empty((nf, n, 4), dtype=torch.float64, device=q.device) if nf else None
    st = N.Status()
    sysc = system_struct(spec)
    rc = ctx.lib.gs_evolve(ctx.handle, ctypes.byref(sysc), n, float(t_final), int(steps), int(capture_every),
                           _ptr(q), _ptr(p), _ptr(frames) if frames is not None else None, ctypes.byref(st),
                           _stream_ptr(torch))
    if rc not in (N.GS_OK, N.GS_ERR_COINCIDENT, N.GS_ERR_NONFINITE_STAGE, N.GS_ERR_NONFINITE_STATE):
        N.check(rc, "gs_evolve")
    exc = status_exception(st, float(t_final), int(steps))
    if exc is not None:
        raise exc
    return q, p, frames


_STOP = {"residual": N.GS_STOP_TARGET_RESIDUAL, "momentum-delta": N.GS_STOP_MOMENTUM_DELTA}
_NORM = {"max": N.GS_NORM_MAX, "l2": N.GS_NORM_L2}


def match(spec, q0, target, h: float, epsilon: float, max_iter: int, stop_rule: str, norm: str, t_final: float,
          steps: int) -> dict:
    """shooting.match (momentum update) on the device.  Returns the MatchResult fields with
    p0/endpoint as cuda tensors and diagnosis text in the reference's wording."""
    torch = _torch()
    ctx = N.Context.get()
    q0 = as_device(q0, torch)
    target = as_device(target, torch)
    n = q0.shape[0]
    p0 = torch.empty_like(q0)
    endpoint = torch.empty_like(q0)
    hist = (ctypes.c_double * max(1, int(max_iter)))()
    res = N.MatchResultC()
    cfg = N.MatchConfig(float(h), float(epsilon), int(max_iter), _STOP[stop_rule], _NORM[norm], int(steps),
                        float(t_final))
    sysc = system_struct(spec)
    N.check(ctx.lib.gs_match(ctx.handle, ctypes.byref(sysc), ctypes.byref(cfg), n, _ptr(q0), _ptr(target), _ptr(p0),
                             _ptr(endpoint), hist, ctypes.byref(res), _stream_ptr(torch)), "gs_match")
    diagnosis = _diagnosis(res, t_final, steps)
    return dict(p0=p0, endpoint=endpoint, iterations=int(res.iterations),
                converged=res.outcome == N.GS_MATCH_CONVERGED,
                residual_history=tuple(float(hist[i]) for i in range(res.iterations)),
                hamiltonian=float(res.hamiltonian), final_residual=float(res.final_residual), diagnosis=diagnosis,
                seconds_device=float(res.seconds_device))


def _diagnosis(res: N.MatchResultC, t_final: float, steps: int):
    if res.outcome == N.GS_MATCH_CAP:
        return "iteration cap reached before the stopping rule"
    if res.outcome == N.GS_MATCH_BLOWUP:
        return "step too large"
    if res.outcome == N.GS_MATCH_EVOLVE_FAILED:
        return f"step too large ({status_exception(res.status, float(t_final), int(steps))})"
    return None


def _stack(a, torch, n: int | None = None):
    """(n, 2) -> shared (stride 0), (B, n, 2) -> per item; returns (tensor, stride in doubles)."""
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.float64)))
    t = t.to(device="cuda", dtype=torch.float64).contiguous()
    if t.dim() == 2:
        return t, 0
    return t, int(t[0].numel())


def match_batch(specs, cfgs, q0, target, factor=None) -> list:
    """Independent matches side by side (gs_match_batch).

    specs[b] / cfgs[b]: SystemSpec and a dict (h, epsilon, max_iter, stop_rule, norm, t_final,
    steps) per item; q0 / target: (n, 2) shared or (B, n, 2); factor: None (momentum update)
    or the lower Cholesky factor(s) of the Gram matrix, (n, n) shared or (B, n, n) (velocity
    update).  Returns one dict per item in device.match's format.
    """
    torch = _torch()
    ctx = N.Context.get()
    B = len(specs)
    if B != len(cfgs) or B < 1:
        raise ValueError("specs and cfgs must be non-empty and of equal length")
    q0, qs = _stack(q0, torch)
    target, ts = _stack(target, torch)
    n = q0.shape[-2]
    fac, fs = (None, 0)
    if factor is not None:
        fac = factor.to(device="cuda", dtype=torch.float64).contiguous()
        fs = 0 if fac.dim() == 2 else n * n
    items = (N.BatchItem * B)()
    hmax = 1
    for b, (spec, c) in enumerate(zip(specs, cfgs)):
        items[b].system = system_struct(spec)
        items[b].config = N.MatchConfig(float(c["h"]), float(c["epsilon"]), int(c["max_iter"]),
                                        _STOP[c["stop_rule"]], _NORM[c["norm"]], int(c["steps"]),
                                        float(c["t_final"]))
        hmax = max(hmax, int(c["max_iter"]))
    p0 = torch.empty((B, n, 2), dtype=torch.float64, device=q0.device)
    endpoint = torch.empty_like(p0)
    hist = torch.empty((B, hmax), dtype=torch.float64, device=q0.device)
    res = (N.MatchResultC * B)()
    N.check(ctx.lib.gs_match_batch(ctx.handle, items, B, n, _ptr(q0), qs, _ptr(target), ts,
                                   _ptr(fac) if fac is not None else None, fs, _ptr(p0), _ptr(endpoint), _ptr(hist),
                                   hmax, res, _stream_ptr(torch)), "gs_match_batch")
    hist_h = hist.cpu().numpy()
    out = []
    for b in range(B):
        r = res[b]
        c = cfgs[b]
        out.append(dict(p0=p0[b], endpoint=endpoint[b], iterations=int(r.iterations),
                        converged=r.outcome == N.GS_MATCH_CONVERGED,
                        residual_history=tuple(float(v) for v in hist_h[b, :r.iterations]),
                        hamiltonian=float(r.hamiltonian), final_residual=float(r.final_residual),
                        diagnosis=_diagnosis(r, c["t_final"], c["steps"]), seconds_device=float(r.seconds_device)))
    return out


def evolve_batch(spec, q0, p, t_final: float, steps: int):
    """B independent evolves of one system (gs_evolve_batch): q0 (n, 2) shared or (B, n, 2),
    p (B, n, 2).  Returns (q (B, n, 2), p (B, n, 2), [exception or None] * B)."""
    torch = _torch()
    ctx = N.Context.get()
    q0, qs = _stack(q0, torch)
    p = p.to(device="cuda", dtype=torch.float64).clone().contiguous() if isinstance(p, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(np.asarray(p, np.float64))).cuda()
    B, n = p.shape[0], p.shape[1]
    q = torch.empty_like(p)
    st = (N.Status * B)()
    sysc = system_struct(spec)
    N.check(ctx.lib.gs_evolve_batch(ctx.handle, ctypes.byref(sysc), B, n, float(t_final), int(steps), _ptr(q0), qs,
                                    _ptr(q), _ptr(p), st, _stream_ptr(torch)), "gs_evolve_batch")
    return q, p, [status_exception(st[b], float(t_final), int(steps)) for b in range(B)]
