"""Multi-GPU driver: target-row sharding with one all-gather of the stage state per RK stage.

SURVEY.md §8(e).  Each rank (one process per GPU, ``torch.distributed`` over NCCL) owns the
contiguous target rows [r0, r1) of an equal-size split (c = ceil(N / world) rows per rank,
the last rank's tail padded), evaluates their RHS against all N sources with
``gs_stage_run`` (the fused RHS + RK4 stage epilogue of csrc/gs_dense.cu), and the 32-byte
(x, y, px, py) records of its rows are all-gathered so that every rank holds the next stage
input in full.  The matching loop adds one scalar all-reduce per iteration (MAX for the
max-norm, SUM for the squared L2 norm) and one SUM for H.

Every row's sum runs over the same source chunks in the same order whatever the number of
ranks (the chunking depends on N only), so 1/2/4/8-GPU results are bitwise identical.

The orchestration is written against a small backend interface so that the same code runs
on CPU (``gloo``) with a numpy stage backend in tests/test_sharded_gloo.py; the product
backend is :class:`DeviceStageBackend` (libgs_b200.so).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as N
from . import device
from . import errors as _errors

STOP_RESIDUAL, STOP_MDELTA = "residual", "momentum-delta"


def row_split(n: int, world: int, rank: int):
    """Equal-size row blocks: rank owns [r0, r1) with c = ceil(n / world) rows (tail may be short)."""
    c = (n + world - 1) // world
    r0 = min(n, rank * c)
    r1 = min(n, r0 + c)
    return r0, r1, c


def rhs_rows(spec, q, p, r0: int, r1: int):
    """Rows [r0, r1) of particles.rhs on device tensors (gs_rhs_rows)."""
    import torch

    ctx = N.Context.get()
    q = device.as_device(q, torch)
    p = device.as_device(p, torch)
    dq = torch.empty((r1 - r0, 2), dtype=torch.float64, device=q.device)
    dp = torch.empty_like(dq)
    sysc = device.system_struct(spec)
    s = torch.cuda.current_stream().cuda_stream
    N.check(ctx.lib.gs_rhs_rows(ctx.handle, ctypes.byref(sysc), q.shape[0], q.data_ptr(), p.data_ptr(), r0, r1,
                                dq.data_ptr(), dp.data_ptr(), s), "gs_rhs_rows")
    st = N.Status()
    N.check(ctx.lib.gs_status_fetch(ctx.handle, ctypes.byref(st), s), "gs_status_fetch")
    exc = device.status_exception(st)
    if exc is not None:
        raise exc
    return dq, dp


class DeviceStageBackend:
    """gs_stage_* of libgs_b200.so on this rank's GPU (``ctx``: a library context, default the
    process's context for the current device)."""

    def __init__(self, spec, ctx=None):
        import torch

        self.torch = torch
        self.ctx = ctx or N.Context.get()
        self.spec = spec
        self.sysc = device.system_struct(spec)
        self.n = 0

    def _s(self):
        return self.torch.cuda.current_stream().cuda_stream

    def begin(self, q, p, r0: int, r1: int):
        torch = self.torch
        q = device.as_device(q, torch)
        p = device.as_device(p, torch)
        self.n, self.r0, self.r1 = q.shape[0], r0, r1
        N.check(self.ctx.lib.gs_stage_begin(self.ctx.handle, self.n, q.data_ptr(), p.data_ptr(), r0, r1, self._s()),
                "gs_stage_begin")

    def state(self, rows: int):
        """(rows, 4) float64 CUDA tensor aliasing the library's stage state S (rows <= n + 64)."""
        torch = self.torch
        ptr = self.ctx.lib.gs_stage_state(self.ctx.handle)
        n_pad = self.n + 64
        assert rows <= n_pad
        return _wrap_device_ptr(torch, ptr, (rows, 4))

    def run(self, step: int, stage: int, dt: float):
        N.check(self.ctx.lib.gs_stage_run(self.ctx.handle, ctypes.byref(self.sysc), step, stage, dt, self._s()),
                "gs_stage_run")

    # -- symmetric split (dense path, world > 1) -------------------------------------------
    supports_sym = True
    # -- slab decomposition (cell path, world > 1): slab.py over gs_slab_* ------------------
    supports_slab = True

    def slab_backend(self):
        from . import slab

        return slab.DeviceSlabBackend(self.spec, ctx=self.ctx)

    def path(self) -> str:
        rc = self.ctx.lib.gs_stage_path(self.ctx.handle, ctypes.byref(self.sysc), self._s())
        if rc < 0:
            N.check(-rc, "gs_stage_path")
        return "cell" if rc == N.GS_PATH_CELL else "dense"

    def sym_parts(self) -> int:
        return int(self.ctx.lib.gs_sym_parts(self.n))

    def new_partials(self, rows: int):
        return self.torch.zeros((rows, 4), dtype=self.torch.float64, device="cuda")

    def pairs_sym(self, step: int, stage: int, b: int, e: int, R):
        N.check(self.ctx.lib.gs_stage_pairs_sym(self.ctx.handle, ctypes.byref(self.sysc), step, stage, b, e,
                                                R.data_ptr(), self._s()), "gs_stage_pairs_sym")

    def finish(self, step: int, stage: int, dt: float, R_rows):
        N.check(self.ctx.lib.gs_stage_finish(self.ctx.handle, ctypes.byref(self.sysc), step, stage, dt,
                                             R_rows.data_ptr(), self._s()), "gs_stage_finish")

    def status(self) -> N.Status:
        st = N.Status()
        N.check(self.ctx.lib.gs_status_fetch(self.ctx.handle, ctypes.byref(st), self._s()), "gs_status_fetch")
        return st

    # -- fused stage exchange over peer memory (gs_p2p_*, opt-in) ---------------------------
    supports_p2p = True

    def state_ptr(self) -> int:
        return int(self.ctx.lib.gs_stage_state(self.ctx.handle) or 0)

    def p2p_local(self, rows_all: int):
        """(S, R, counters) device pointers of this rank (counters zeroed)."""
        ptr = [ctypes.c_void_p() for _ in range(3)]
        N.check(self.ctx.lib.gs_p2p_local(self.ctx.handle, rows_all, *(ctypes.byref(x) for x in ptr)), "gs_p2p_local")
        return tuple(int(x.value) for x in ptr)

    def p2p_export(self, rows_all: int) -> bytes:
        buf = ctypes.create_string_buffer(3 * 64)
        N.check(self.ctx.lib.gs_p2p_export(self.ctx.handle, rows_all, buf), "gs_p2p_export")
        return buf.raw

    def p2p_import(self, world: int, rank: int, handles: bytes):
        N.check(self.ctx.lib.gs_p2p_import(self.ctx.handle, world, rank, handles), "gs_p2p_import")

    def p2p_set_peers(self, world: int, rank: int, S, R, F):
        arr = ctypes.c_void_p * world
        N.check(self.ctx.lib.gs_p2p_set_peers(self.ctx.handle, world, rank, arr(*S), arr(*R), arr(*F)),
                "gs_p2p_set_peers")

    def p2p_pairs(self, step: int, stage: int, b: int, e: int):
        N.check(self.ctx.lib.gs_p2p_pairs(self.ctx.handle, ctypes.byref(self.sysc), step, stage, b, e, self._s()),
                "gs_p2p_pairs")

    def p2p_finish(self, step: int, stage: int, dt: float):
        N.check(self.ctx.lib.gs_p2p_finish(self.ctx.handle, ctypes.byref(self.sysc), step, stage, dt, self._s()),
                "gs_p2p_finish")

    def p2p_sync(self):
        N.check(self.ctx.lib.gs_p2p_sync(self.ctx.handle, self._s()), "gs_p2p_sync")

    def p2p_timeouts(self) -> int:
        v = ctypes.c_int64()
        N.check(self.ctx.lib.gs_p2p_timeouts(self.ctx.handle, ctypes.byref(v)), "gs_p2p_timeouts")
        return int(v.value)


def _wrap_device_ptr(torch, ptr: int, shape):
    """Zero-copy float64 CUDA tensor over a library-owned device pointer."""
    class _Holder:
        pass

    h = _Holder()
    numel = int(np.prod(shape))
    h.__cuda_array_interface__ = {"shape": (numel,), "typestr": "<f8", "data": (int(ptr), False), "version": 3}
    return torch.as_tensor(h, device="cuda").view(*shape)


def _event_key(st) -> tuple:
    if st.code == N.GS_OK:
        return (math.inf, 0, 0)
    return (st.step * 8 + st.event, st.i, st.j)


def _nvtx(name: str):
    """An NVTX range on the CUDA timeline (no-op without CUDA / a profiler)."""
    import contextlib

    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.nvtx.range(name)
    except Exception:
        pass
    return contextlib.nullcontext()


class ShardedSolver:
    """Row-sharded evolve / match across the ranks of ``group`` (default: the world)."""

    def __init__(self, spec, backend=None, group=None, force_split: bool = False, p2p: bool | None = None):
        """``force_split``: take the multi-rank code path (symmetric pair split, reduce-scatter,
        all-gather) even in a world of one — lets a single GPU exercise the NCCL plumbing.
        ``p2p`` (default: on when world > 1, see GS_B200_P2P): exchange the stage over peer memory
        (gs_p2p_*: the epilogue reads every rank's row sums and stores the new records into every
        rank's S over NVLink) instead of NCCL's reduce-scatter + all-gather; on any wait timeout
        the evolve is redone on the NCCL path and peer exchange is switched off."""
        import os

        import torch.distributed as dist

        self.spec = spec
        self.backend = backend or DeviceStageBackend(spec)
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.split = self.world > 1 or (force_split and dist.is_initialized())
        if p2p is None:  # default: on across GPUs; GS_B200_P2P=0 switches it off, =1 forces it on
            env = os.environ.get("GS_B200_P2P", "")
            p2p = env == "1" or (env != "0" and self.world > 1)
        self.p2p = bool(p2p) and getattr(self.backend, "supports_p2p", False)
        self._p2p_key = None
        # cell path across ranks: slab decomposition (GS_B200_SLAB=0: all-gather of every record)
        self.slab = os.environ.get("GS_B200_SLAB", "1") != "0"
        # dense split over NCCL: the whole evolve (pair share, reduce-scatter, finish, all-gather per
        # stage) captured once as a CUDA graph and replayed (GS_B200_SHARDED_GRAPHS=0: host loop)
        self.graphs = os.environ.get("GS_B200_SHARDED_GRAPHS", "1") != "0"
        self._graph = None
        self._graph_key = None
        self._bufs = {}

    # -- collectives (plumbing) -------------------------------------------------------------
    def _allgather_rows(self, S, r0: int, c: int):
        if self.split:
            self.dist.all_gather_into_tensor(S[: c * self.world], S[r0:r0 + c].clone(), group=self.group)

    def _reduce_scatter_rows(self, R_rows, R, c: int):
        """R_rows = (sum over ranks of R)[rank*c:(rank+1)*c]  (NCCL reduce-scatter; gloo, used by
        the CPU tests, has no reduce-scatter and takes an all-reduce)."""
        if self.dist.get_backend(self.group) == "gloo":
            self.dist.all_reduce(R, group=self.group)
            R_rows.copy_(R[self.rank * c:(self.rank + 1) * c])
        else:
            self.dist.reduce_scatter_tensor(R_rows, R, group=self.group)

    def _allreduce(self, t, op):
        if self.world > 1:
            self.dist.all_reduce(t, op=op, group=self.group)
        return t

    def _raise_first_failure(self, t_final, steps):
        torch = _torch_of(self.backend)
        st = self.backend.status()
        key = _event_key(st)
        if self.world > 1:
            enc = torch.tensor([key[0] if key[0] != math.inf else 2.0**62, float(st.i), float(st.j), float(st.code),
                                float(st.step), float(st.event)], dtype=torch.float64, device=_dev_of(self.backend))
            allk = [torch.empty_like(enc) for _ in range(self.world)]
            self.dist.all_gather(allk, enc, group=self.group)
            rows = sorted(tuple(x.tolist()) for x in allk)
            best = rows[0]
            if best[0] >= 2.0**62:
                return
            st = N.Status(int(best[3]), int(best[4]), int(best[1]), int(best[2]), 0, int(best[5]))
        exc = device.status_exception(st, t_final, steps)
        if exc is not None:
            raise exc

    # -- integrator.evolve ------------------------------------------------------------------
    def evolve(self, q, p, t_final: float, steps: int):
        """Full (q, p) at t_final on every rank (integrator.py:66-121).

        Dense path with world > 1: the symmetric split — rank r evaluates its share of the
        unordered pairs (each pair once, both rows fed), the raw row sums are reduce-scattered
        to the row owners (NCCL), the owners run the stage epilogue and the stage records are
        all-gathered.  Cell path with world > 1: the slab decomposition (slab.py: each rank
        owns a band of cell rows + a halo, exchanges only the halo per stage).  Otherwise (a
        cloud spread beyond a row-major grid) every rank evaluates its own rows one-sided and
        the stage records are all-gathered."""
        n = q.shape[0]
        W = self.world
        r0, r1, c = row_split(n, W, self.rank)
        self.backend.begin(q, p, r0, r1)
        if self.split and self.slab and getattr(self.backend, "supports_slab", False) and \
                self.backend.path() == "cell":
            from . import slab

            torch = _torch_of(self.backend)
            try:
                solver = slab.SlabSolver(self.spec, [self.backend.slab_backend()], slab.DistComm(self.group))
                return solver.evolve(device.as_device(q, torch), device.as_device(p, torch), t_final, steps)
            except slab.SlabUnavailable:
                self.slab = False  # hashed grid: the all-gather path below (the same on every rank)
                self.backend.begin(q, p, r0, r1)
        S = self.backend.state(c * W)
        dt = t_final / steps
        sym = False
        if self.split and getattr(self.backend, "supports_sym", False) and self.backend.path() == "dense":
            total = self.backend.sym_parts()
            sym = total > 0
        if sym:
            b, e = self.rank * total // W, (self.rank + 1) * total // W
            R, R_rows = self._partials(c)
            if self.p2p and self._p2p_ready(q, p, n, c, r0, r1, b, e, S, R, R_rows, dt):
                return self._evolve_p2p(q, p, t_final, steps, n, c, b, e, S, r0, r1)
        def stage(step, s):
            with _nvtx(f"stage {step}.{s}"):
                if sym:
                    self.backend.pairs_sym(step, s, b, e, R)
                    self._reduce_scatter_rows(R_rows, R, c)
                    self.backend.finish(step, s, dt, R_rows)
                else:
                    self.backend.run(step, s, dt)
                self._allgather_rows(S, r0, c)

        if sym and self._graphable():
            key = (n, c, steps, dt, b, e, int(S.data_ptr()), int(R.data_ptr()), int(R_rows.data_ptr()))
            if self._graph_key != key:
                torch = _torch_of(self.backend)
                # outside the capture: the first stage builds the slot lists and workspaces and
                # initialises the NCCL communicator; then the state is rewound
                stage(1, 0)
                torch.cuda.synchronize()
                self.backend.begin(q, p, r0, r1)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for step in range(1, steps + 1):
                        for s in range(4):
                            stage(step, s)
                self._graph, self._graph_key = g, key
            self._graph.replay()
        else:
            for step in range(1, steps + 1):
                for s in range(4):
                    stage(step, s)
        self._raise_first_failure(t_final, steps)
        return S[:n, 0:2].clone(), S[:n, 2:4].clone()

    def _partials(self, c: int):
        """The split's raw row sums (all rows) and this rank's reduced rows, kept across evolves
        (a captured graph bakes their addresses in)."""
        key = ("partials", c, self.world)
        if key not in self._bufs:
            self._bufs[key] = (self.backend.new_partials(c * self.world), self.backend.new_partials(c))
        return self._bufs[key]

    def _graphable(self) -> bool:
        """The dense split's stage loop can be captured: the device backend over NCCL (or a world of
        one), torch CUDA graphs available."""
        if not self.graphs or not isinstance(self.backend, DeviceStageBackend):
            return False
        if self.world > 1 or self.split:
            try:
                return self.dist.get_backend(self.group) == "nccl"
            except Exception:
                return False
        return True

    def _agree(self, ok: bool) -> bool:
        """All ranks' verdict (MIN over ranks)."""
        torch = _torch_of(self.backend)
        t = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device=_dev_of(self.backend))
        self._allreduce(t, self.dist.ReduceOp.MIN if self.world > 1 else None)
        return float(t[0]) > 0.5

    def _p2p_ready(self, q, p, n, c, r0, r1, b, e, S, R, R_rows, dt) -> bool:
        """Once per stage session (a collective): exchange the ranks' buffer handles, then run
        the first stage both ways — NCCL reduce-scatter + all-gather, and the peer-memory
        exchange — from the same state and keep the peer path only if every rank got the same
        records (1e-12) without a timeout.  Any failure switches peer exchange off everywhere."""
        torch = _torch_of(self.backend)
        key = (n, c, self.backend.state_ptr())
        if self._p2p_key == key:
            return True
        ok = True
        try:
            handles = self.backend.p2p_export(c * self.world)
        except Exception:
            ok, handles = False, b""
        allh = [None] * self.world
        self.dist.all_gather_object(allh, handles, group=self.group)
        ok = self._agree(ok and all(len(h) == len(handles) and h for h in allh))
        if ok:
            try:
                self.backend.p2p_import(self.world, self.rank, b"".join(allh))
            except Exception:
                ok = False
            ok = self._agree(ok)
        if ok:  # one stage both ways from (q, p)
            self.backend.pairs_sym(1, 0, b, e, R)
            self._reduce_scatter_rows(R_rows, R, c)
            self.backend.finish(1, 0, dt, R_rows)
            self._allgather_rows(S, r0, c)
            ref = S[:n].clone()
            self.backend.begin(q, p, r0, r1)
            before = self.backend.p2p_timeouts()
            self.backend.p2p_pairs(1, 0, b, e)
            self.backend.p2p_finish(1, 0, dt)
            self.backend.p2p_sync()
            got = S[:n]
            scale = float(ref.abs().max()) or 1.0
            same = bool(torch.isfinite(got).all()) and float((got - ref).abs().max()) <= 1e-12 * scale
            ok = self._agree(same and self.backend.p2p_timeouts() == before)
            self.backend.begin(q, p, r0, r1)
        if not ok:
            self.p2p = False
            return False
        self._p2p_key = key
        return True

    def _evolve_p2p(self, q, p, t_final, steps, n, c, b, e, S, r0, r1):
        torch = _torch_of(self.backend)
        before = self.backend.p2p_timeouts()
        dt = t_final / steps
        for step in range(1, steps + 1):
            for s in range(4):
                self.backend.p2p_pairs(step, s, b, e)
                self.backend.p2p_finish(step, s, dt)
        self.backend.p2p_sync()
        lost = torch.tensor([float(self.backend.p2p_timeouts() - before)], dtype=torch.float64,
                            device=_dev_of(self.backend))
        self._allreduce(lost, self.dist.ReduceOp.MAX if self.world > 1 else None)
        if float(lost[0]) > 0:  # a signal never arrived: redo this evolve on the NCCL path
            self.p2p = False
            return self.evolve(q, p, t_final, steps)
        self._raise_first_failure(t_final, steps)
        return S[:n, 0:2].clone(), S[:n, 2:4].clone()

    # -- shooting.match, momentum update ----------------------------------------------------
    def match(self, q0, target, h: float, epsilon: float, max_iter: int, stop_rule: str = STOP_RESIDUAL,
              norm: str = "max", t_final: float = 1.0, steps: int = 20) -> dict:
        torch = _torch_of(self.backend)
        dev = _dev_of(self.backend)
        q0 = torch.as_tensor(np.asarray(q0) if not isinstance(q0, torch.Tensor) else q0, dtype=torch.float64,
                             device=dev)
        target = torch.as_tensor(np.asarray(target) if not isinstance(target, torch.Tensor) else target,
                                 dtype=torch.float64, device=dev)
        n = q0.shape[0]
        r0, r1, _ = row_split(n, self.world, self.rank)
        p = torch.zeros_like(q0)
        endpoint = q0.clone()  # evolve(q0, 0) == q0 exactly
        residual = target - endpoint

        def norm_of(res):
            rows = res[r0:r1]
            if norm == "max":
                v = torch.hypot(rows[:, 0], rows[:, 1]).max() if r1 > r0 else torch.zeros((), dtype=torch.float64,
                                                                                          device=dev)
                return float(self._allreduce(v.reshape(1), self.dist.ReduceOp.MAX if self.world > 1 else None)[0])
            v = (rows * rows).sum().reshape(1)
            return math.sqrt(float(self._allreduce(v, self.dist.ReduceOp.SUM if self.world > 1 else None)[0]))

        history = []
        nrm = norm_of(residual)
        initial = nrm if stop_rule == STOP_RESIDUAL else None
        diagnosis, converged = None, False
        if stop_rule == STOP_RESIDUAL and nrm < epsilon:
            converged = True
        else:
            diagnosis = "iteration cap reached before the stopping rule"
            for it in range(max_iter):
                delta = h * nrm
                p = p + h * residual
                try:
                    with _nvtx(f"feedback iteration {it + 1}"):
                        qT, _ = self.evolve(q0, p, t_final, steps)
                except (_errors.DivergenceError, _errors.DegenerateConfigurationError) as exc:
                    diagnosis = f"step too large ({exc})"
                    break
                endpoint = qT
                residual = target - endpoint
                nrm = norm_of(residual)
                value = nrm if stop_rule == STOP_RESIDUAL else delta
                if initial is None:
                    initial = value
                history.append(value)
                if not math.isfinite(value) or (initial > 0 and value > 1e6 * initial):
                    diagnosis = "step too large"
                    break
                if value < epsilon:
                    diagnosis, converged = None, True
                    break
        H = self.hamiltonian(q0, p)
        return dict(p0=p, endpoint=endpoint, iterations=len(history), converged=converged,
                    residual_history=tuple(history), hamiltonian=H, final_residual=nrm, diagnosis=diagnosis)

    def hamiltonian(self, q, p) -> float:
        """particles.hamiltonian: this rank's rows of p_i . (K p)_i, SUM-reduced."""
        torch = _torch_of(self.backend)
        n = q.shape[0]
        r0, r1, _ = row_split(n, self.world, self.rank)
        part = self.backend.hamiltonian_rows(self.spec, q, p, r0, r1) if hasattr(self.backend, "hamiltonian_rows") \
            else _device_hamiltonian_rows(self.spec, q, p, r0, r1)
        t = torch.tensor([part], dtype=torch.float64, device=_dev_of(self.backend))
        return float(self._allreduce(t, self.dist.ReduceOp.SUM if self.world > 1 else None)[0])


def _device_hamiltonian_rows(spec, q, p, r0, r1) -> float:
    if r1 <= r0:
        return 0.0
    dq, _ = rhs_rows(device._plain_spec(spec), q, p, r0, r1)
    pr = device.as_device(p)[r0:r1]
    return float((pr * dq).sum())


def _torch_of(backend):
    import torch

    return torch


def _dev_of(backend):
    return getattr(backend, "device", "cuda")
