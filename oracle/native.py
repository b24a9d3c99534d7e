"""ctypes wrapper of oracle/gs_oracle.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Raises the same exception kinds and messages as the reference
(``particles.py:92-98``, ``integrator.py:58-63, 102-112``), via the
``oracle.restate`` exception classes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import restate
from .restate import Kernel, OracleDegenerate, OracleDivergence

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libgs_oracle.so")


class _Params(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("normalized", ctypes.c_int), ("alpha", ctypes.c_double),
                ("sigma2", ctypes.c_double), ("cutoff", ctypes.c_double)]


def build() -> str:
    subprocess.run([os.path.join(_HERE, "build.sh")], check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        _lib.go_rhs.argtypes = [ctypes.POINTER(_Params), ctypes.c_long, dp, dp, dp, dp, ctypes.c_long,
                                ctypes.c_long, ctypes.POINTER(ctypes.c_longlong)]
        _lib.go_rhs.restype = ctypes.c_int
        _lib.go_evolve.argtypes = [ctypes.POINTER(_Params), ctypes.c_long, ctypes.c_double, ctypes.c_int,
                                   dp, dp, ctypes.POINTER(ctypes.c_longlong)]
        _lib.go_evolve.restype = ctypes.c_int
        _lib.go_hamiltonian.argtypes = [ctypes.POINTER(_Params), ctypes.c_long, dp, dp]
        _lib.go_hamiltonian.restype = ctypes.c_double
        _lib.go_max_threads.restype = ctypes.c_int
        _lib.go_set_threads.argtypes = [ctypes.c_int]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _params(k: Kernel, sigma2: float, cutoff: float) -> _Params:
    return _Params(k.family, 1 if k.normalized else 0, k.alpha, sigma2, cutoff)


def set_threads(t: int) -> None:
    lib().go_set_threads(int(t))


def max_threads() -> int:
    return int(lib().go_max_threads())


def rhs(k: Kernel, sigma2: float, q: np.ndarray, p: np.ndarray, cutoff: float = 0.0, rows=None):
    q = np.ascontiguousarray(q, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    n = q.shape[0]
    r0, r1 = (0, n) if rows is None else rows
    dq = np.empty((r1 - r0, 2))
    dp = np.empty((r1 - r0, 2))
    bad = ctypes.c_longlong(-1)
    prm = _params(k, sigma2, cutoff)
    code = lib().go_rhs(ctypes.byref(prm), n, _ptr(q), _ptr(p), _ptr(dq), _ptr(dp), r0, r1, ctypes.byref(bad))
    if code:
        raise restate._coincident_error(int(bad.value // n), int(bad.value % n))
    return dq, dp


def hamiltonian(k: Kernel, q: np.ndarray, p: np.ndarray) -> float:
    q = np.ascontiguousarray(q, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    prm = _params(k, 0.0, 0.0)
    return float(lib().go_hamiltonian(ctypes.byref(prm), q.shape[0], _ptr(q), _ptr(p)))


def evolve(k: Kernel, sigma2: float, q0: np.ndarray, p0: np.ndarray, t_final: float = 1.0, steps: int = 100,
           cutoff: float = 0.0):
    q = np.array(q0, dtype=np.float64, order="C", copy=True)
    p = np.array(p0, dtype=np.float64, order="C", copy=True)
    err = (ctypes.c_longlong * 3)()
    prm = _params(k, sigma2, cutoff)
    code = lib().go_evolve(ctypes.byref(prm), q.shape[0], t_final, steps, _ptr(q), _ptr(p), err)
    if code == 0:
        return q, p
    step = int(err[0])
    dt = t_final / steps
    t = t_final * ((step - 1) / steps)
    if code == 1:
        base = restate._coincident_error(int(err[1]), int(err[2]))
        raise OracleDegenerate(f"{base} (during step {step}, t in [{t:.6g}, {t + dt:.6g}])")
    if code == 2:
        raise OracleDivergence(f"non-finite intermediate at step {step} (t in [{t:.6g}, {t + dt:.6g}]); "
                               "the step size is too large for this configuration")
    raise OracleDivergence(f"non-finite state at step {step} (t = {t_final * (step / steps):.6g}); "
                           "the step size is too large for this configuration")


def match_momentum(k: Kernel, sigma2: float, q0, target, h, epsilon, max_iter, stop_rule="residual",
                   norm_kind="max", t_final=1.0, steps=100, cutoff: float = 0.0, update_space="momentum") -> dict:
    ev = lambda qq, pp: evolve(k, sigma2, qq, pp, t_final, steps, cutoff)[0]
    return restate.match_momentum(k, sigma2, q0, target, h, epsilon, max_iter, stop_rule, norm_kind,
                                  t_final, steps, evolve_fn=ev, update_space=update_space)
