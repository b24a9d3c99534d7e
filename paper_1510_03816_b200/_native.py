"""ctypes binding of libgs_b200.so (include/geoshoot_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is present, every
entry point raises :class:`NativeUnavailable` — the product path fails loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GS_B200_LIB") or os.path.join(_PKG, "libgs_b200.so")  # override: A/B variants

GS_OK = 0
GS_ERR_INVALID = 1
GS_ERR_COINCIDENT = 2
GS_ERR_NONFINITE_STAGE = 3
GS_ERR_NONFINITE_STATE = 4
GS_ERR_CUDA = 5
GS_ERR_UNSUPPORTED = 6

GS_FAMILY_CONICAL = 0
GS_FAMILY_GAUSSIAN = 1
GS_PATH_AUTO, GS_PATH_DENSE, GS_PATH_CELL = 0, 1, 2
GS_STOP_TARGET_RESIDUAL, GS_STOP_MOMENTUM_DELTA = 0, 1
GS_NORM_MAX, GS_NORM_L2 = 0, 1
GS_MATCH_CONVERGED, GS_MATCH_CAP, GS_MATCH_BLOWUP, GS_MATCH_EVOLVE_FAILED = 0, 1, 2, 3

# every symbol include/geoshoot_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "gs_version", "gs_abi_version", "gs_last_error", "gs_create", "gs_destroy", "gs_rhs", "gs_rhs_rows",
    "gs_status_fetch", "gs_status_reset", "gs_hamiltonian", "gs_evolve", "gs_match", "gs_stage_begin",
    "gs_stage_run", "gs_stage_state", "gs_stage_end", "gs_fp64_peak_probe", "gs_profile_enable",
    "gs_profile_read", "gs_stage_path", "gs_sym_parts", "gs_stage_pairs_sym", "gs_stage_finish", "gs_gram",
    "gs_match_batch", "gs_evolve_batch", "gs_velocity_field", "gs_p2p_local", "gs_p2p_export", "gs_p2p_import",
    "gs_p2p_set_peers", "gs_p2p_pairs", "gs_p2p_finish", "gs_p2p_sync", "gs_p2p_timeouts", "gs_p2p_close",
    "gs_cell_stats", "gs_gram_cg", "gs_slab_begin", "gs_slab_bbox", "gs_slab_grid", "gs_slab_rows", "gs_slab_pack",
    "gs_slab_unpack", "gs_slab_layout", "gs_slab_views", "gs_slab_lists", "gs_slab_stage", "gs_slab_status",
)


class NativeUnavailable(RuntimeError):
    """libgs_b200.so could not be loaded or has no CUDA device to run on."""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[gs code {code}] {msg}")
        self.code = code


class System(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("normalized", ctypes.c_int32), ("alpha", ctypes.c_double),
                ("sigma2", ctypes.c_double), ("cutoff", ctypes.c_double), ("path", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("step", ctypes.c_int32), ("i", ctypes.c_int64), ("j", ctypes.c_int64),
                ("iteration", ctypes.c_int32), ("event", ctypes.c_int32)]


class SlabGrid(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("y0", ctypes.c_double), ("h", ctypes.c_double), ("nx", ctypes.c_int32),
                ("ny", ctypes.c_int32), ("sub", ctypes.c_int32), ("hashed", ctypes.c_int32)]


class MatchConfig(ctypes.Structure):
    _fields_ = [("h", ctypes.c_double), ("epsilon", ctypes.c_double), ("max_iter", ctypes.c_int32),
                ("stop_rule", ctypes.c_int32), ("norm", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("t_final", ctypes.c_double)]


class MatchResultC(ctypes.Structure):
    _fields_ = [("outcome", ctypes.c_int32), ("iterations", ctypes.c_int32), ("hamiltonian", ctypes.c_double),
                ("final_residual", ctypes.c_double), ("status", Status), ("seconds_device", ctypes.c_double)]


class BatchItem(ctypes.Structure):
    _fields_ = [("system", System), ("config", MatchConfig)]


_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_dp = ctypes.c_void_p  # device pointers are passed as integers


def load(path: str = LIB_PATH):
    """Load and prototype the library (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -m paper_1510_03816_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        P = ctypes.POINTER
        proto = {
            "gs_version": ([], ctypes.c_char_p),
            "gs_abi_version": ([], ctypes.c_int),
            "gs_last_error": ([], ctypes.c_char_p),
            "gs_create": ([P(_vp), ctypes.c_int], ctypes.c_int),
            "gs_destroy": ([_vp], ctypes.c_int),
            "gs_rhs": ([_vp, P(System), _i64, _dp, _dp, _dp, _dp, P(Status), _vp], ctypes.c_int),
            "gs_rhs_rows": ([_vp, P(System), _i64, _dp, _dp, _i64, _i64, _dp, _dp, _vp], ctypes.c_int),
            "gs_status_fetch": ([_vp, P(Status), _vp], ctypes.c_int),
            "gs_status_reset": ([_vp, _vp], ctypes.c_int),
            "gs_hamiltonian": ([_vp, P(System), _i64, _dp, _dp, P(ctypes.c_double), _vp], ctypes.c_int),
            "gs_evolve": ([_vp, P(System), _i64, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, _dp, _dp, _dp,
                           P(Status), _vp], ctypes.c_int),
            "gs_match": ([_vp, P(System), P(MatchConfig), _i64, _dp, _dp, _dp, _dp, P(ctypes.c_double),
                          P(MatchResultC), _vp], ctypes.c_int),
            "gs_stage_begin": ([_vp, _i64, _dp, _dp, _i64, _i64, _vp], ctypes.c_int),
            "gs_stage_run": ([_vp, P(System), ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _vp], ctypes.c_int),
            "gs_stage_state": ([_vp], ctypes.c_void_p),
            "gs_stage_end": ([_vp, _dp, _dp, _vp], ctypes.c_int),
            "gs_fp64_peak_probe": ([_vp, ctypes.c_int32, P(ctypes.c_double), P(ctypes.c_double), _vp], ctypes.c_int),
            "gs_stage_path": ([_vp, P(System), _vp], ctypes.c_int),
            "gs_gram": ([_vp, P(System), _i64, _dp, _dp, P(_i64), P(_i64), _vp], ctypes.c_int),
            "gs_sym_parts": ([_i64], _i64),
            "gs_stage_pairs_sym": ([_vp, P(System), ctypes.c_int32, ctypes.c_int32, _i64, _i64, _dp, _vp],
                                   ctypes.c_int),
            "gs_stage_finish": ([_vp, P(System), ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _dp, _vp],
                                ctypes.c_int),
            "gs_match_batch": ([_vp, P(BatchItem), _i64, _i64, _dp, _i64, _dp, _i64, _dp, _i64, _dp, _dp, _dp, _i64,
                                P(MatchResultC), _vp], ctypes.c_int),
            "gs_evolve_batch": ([_vp, P(System), _i64, _i64, ctypes.c_double, ctypes.c_int32, _dp, _i64, _dp, _dp,
                                 P(Status), _vp], ctypes.c_int),
            "gs_velocity_field": ([_vp, P(System), _i64, _dp, _dp, _i64, _dp, _dp, _vp], ctypes.c_int),
            "gs_p2p_local": ([_vp, _i64, P(_vp), P(_vp), P(_vp)], ctypes.c_int),
            "gs_p2p_export": ([_vp, _i64, _vp], ctypes.c_int),
            "gs_p2p_import": ([_vp, ctypes.c_int, ctypes.c_int, _vp], ctypes.c_int),
            "gs_p2p_set_peers": ([_vp, ctypes.c_int, ctypes.c_int, P(_vp), P(_vp), P(_vp)], ctypes.c_int),
            "gs_p2p_pairs": ([_vp, P(System), ctypes.c_int32, ctypes.c_int32, _i64, _i64, _vp], ctypes.c_int),
            "gs_p2p_finish": ([_vp, P(System), ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _vp], ctypes.c_int),
            "gs_p2p_sync": ([_vp, _vp], ctypes.c_int),
            "gs_p2p_timeouts": ([_vp, P(_i64)], ctypes.c_int),
            "gs_p2p_close": ([_vp], ctypes.c_int),
            "gs_profile_enable": ([_vp, ctypes.c_int32], ctypes.c_int),
            "gs_cell_stats": ([_vp, P(_i64), P(_i64), _vp], ctypes.c_int),
            "gs_gram_cg": ([_vp, P(System), _i64, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int32,
                            P(ctypes.c_int32), P(ctypes.c_double), P(ctypes.c_double), _vp], ctypes.c_int),
            "gs_slab_begin": ([_vp, P(System), _i64, _i64, _dp, _dp, _dp, _vp], ctypes.c_int),
            "gs_slab_bbox": ([_vp, _dp, _vp], ctypes.c_int),
            "gs_slab_grid": ([_vp, _dp, P(SlabGrid), _vp], ctypes.c_int),
            "gs_slab_rows": ([_vp, _dp, _vp], ctypes.c_int),
            "gs_slab_pack": ([_vp, _dp, ctypes.c_int32, _dp, P(_i64), _vp], ctypes.c_int),
            "gs_slab_unpack": ([_vp, _i64, _dp, _vp], ctypes.c_int),
            "gs_slab_layout": ([_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _i64, _i64, _vp],
                               ctypes.c_int),
            "gs_slab_views": ([_vp, P(_vp), P(_vp), P(_vp), P(_vp)], ctypes.c_int),
            "gs_slab_lists": ([_vp, _i64, _vp], ctypes.c_int),
            "gs_slab_stage": ([_vp, P(System), ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _vp], ctypes.c_int),
            "gs_slab_status": ([_vp, P(Status), _vp], ctypes.c_int),
            "gs_profile_read": ([_vp, P(ctypes.c_double), P(ctypes.c_int64), P(ctypes.c_int64), P(ctypes.c_int64),
                                 ctypes.c_int32], ctypes.c_int),
        }
        for name, (args, res) in proto.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def last_error() -> str:
    return (load().gs_last_error() or b"").decode()


def check(rc: int, what: str) -> None:
    if rc != GS_OK:
        raise NativeError(rc, f"{what}: {last_error()}")


class Context:
    """One gs_context per (thread, device): the library's device workspaces and graph caches.

    The reference's calls are pure and may run concurrently; the C ABI asks
    for one context per concurrent caller (include/geoshoot_b200.h), so each Python thread gets
    its own context per device on first use."""

    _tls = threading.local()

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
        self.lib = load()
        self.device = device
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            check(self.lib.gs_create(ctypes.byref(h), device), "gs_create")
        self.handle = h

    @classmethod
    def _contexts(cls) -> dict:
        d = getattr(cls._tls, "by_device", None)
        if d is None:
            d = cls._tls.by_device = {}
        return d

    @classmethod
    def swap(cls, contexts: dict | None = None) -> dict:
        """Replace this thread's contexts (None: none yet, so the next call creates a fresh one —
        e.g. after changing a GS_B200_* environment knob read at gs_create); returns the old ones."""
        old = cls._contexts()
        cls._tls.by_device = {} if contexts is None else contexts
        return old

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        import torch

        if device is None:
            if not torch.cuda.is_available():
                raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
            device = torch.cuda.current_device()
        by_device = cls._contexts()
        ctx = by_device.get(device)
        if ctx is None:
            ctx = cls(device)
            by_device[device] = ctx
        return ctx

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.gs_destroy(self.handle)
        except Exception:
            pass
