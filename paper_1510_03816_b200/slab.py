"""Slab-decomposed cell path across ranks: the multi-GPU driver of gs_slab_* (SURVEY.md §8(e)).

For the compactly supported kernel (KD-1) the RHS of row i (particles.py:109-117) only needs
the particles within the support radius.  Instead of all-gathering every stage record and
rebuilding the whole grid on every rank (sharded.py's cell path), each rank owns the particles
of a contiguous band of cell rows of the global grid and keeps ``sub`` halo rows on either side:

* per list build (when some particle moved half the skin, integrator.py:95-114 unchanged):
  MIN all-reduce of the ranks' bounding boxes -> the one-rank grid on every rank; SUM
  all-reduce of the per-row counts -> balanced slabs (:class:`SlabPlan`, identical on every
  rank); all-to-all migration of the particles whose row changed owner (state + RK4 base and
  accumulator); the halo slices (contiguous blocks of the neighbours' own particles, global
  sorted order); lists over slab + halo;
* per RK stage: sweep + epilogue of the own rows, the halo slices (32 B per halo particle),
  MAX all-reduce of the rebuild flag.

A row's sum is bitwise independent of the number of ranks (csrc/gs_slab.cu), so 1/2/4/8-GPU
evolves agree exactly.  The reference permits any deterministic summation order.

The driver is written against a communicator over "the ranks this process drives":
:class:`DistComm` (one rank per process, torch.distributed: NCCL on GPUs, gloo in the CPU tests)
or :class:`LocalComm` (several ranks in one process: the collectives are copies — used to run a
W-rank decomposition on one GPU, tests/test_gpu_slab.py, tools/time_slab.py).  Backends:
:class:`DeviceSlabBackend` (libgs_b200.so) or a numpy restatement in the CPU tests.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import device

PACK_W = 13  # doubles per migrating particle: record, RK4 base, RK4 accumulator, global index


class SlabUnavailable(RuntimeError):
    """The cloud no longer fits a row-major grid (hashed cells): the caller takes the all-gather path."""


# ---- ownership plan -----------------------------------------------------------------------------


@dataclass(frozen=True)
class RankRows:
    own0: int
    own1: int
    loc0: int
    loc1: int
    own_begin: int
    n_own: int
    n_loc: int


class SlabPlan:
    """Ownership of the cell rows for one list build, from the global per-row counts.

    Every rank computes the same plan from the same all-reduced histogram: rank r owns rows
    [Y_r, Y_r+1) with Y_r the first row whose prefix count reaches r N / W, and holds the
    ``sub`` rows on either side as halo (the stencil reach of a list build, gs_verlet.cu
    for_each_range).  ``slices`` lists every halo transfer (src rank, dst rank, offset in the
    source's local array, offset in the destination's local array, count): a source's rows
    inside a destination's halo are a contiguous run of its own block."""

    def __init__(self, hist, world: int, sub: int, rank_hists=None):
        """``hist``: particles per cell row (all ranks); ``rank_hists`` (W, ny): the same per
        current owner, which fixes every migration count (``send_counts`` / ``recv_counts``)."""
        hist = np.asarray(hist, dtype=np.int64)
        self.ny = ny = int(hist.shape[0])
        self.world = W = int(world)
        self.sub = int(sub)
        cum = np.zeros(ny + 1, dtype=np.int64)
        np.cumsum(hist, out=cum[1:])
        self.cum = cum
        self.n = n = int(cum[-1])
        Y = [int(np.searchsorted(cum * W, r * n, side="left")) for r in range(W)] + [ny]
        Y[0] = 0
        for r in range(1, W + 1):
            Y[r] = min(max(Y[r], Y[r - 1]), ny)
        self.Y = Y
        self.owner = np.zeros(ny, dtype=np.int32)
        for r in range(W):
            self.owner[Y[r]:Y[r + 1]] = r
        self.rows = []
        for r in range(W):
            own0, own1 = Y[r], Y[r + 1]
            n_own = int(cum[own1] - cum[own0])
            loc0, loc1 = (max(own0 - sub, 0), min(own1 + sub, ny)) if n_own else (own0, own1)
            self.rows.append(RankRows(own0, own1, loc0, loc1, int(cum[own0] - cum[loc0]), n_own,
                                      int(cum[loc1] - cum[loc0])))
        # own clusters per rank: pairs restart at every cell row (csrc/gs_slab.cu)
        self.ncl = [int(((hist[r.own0:r.own1] + 1) // 2).sum()) for r in self.rows]
        if rank_hists is not None:
            H = np.asarray(rank_hists, dtype=np.int64)
            csum = np.zeros((W, ny + 1), dtype=np.int64)
            np.cumsum(H, axis=1, out=csum[:, 1:])
            M = np.stack([csum[:, Y[d + 1]] - csum[:, Y[d]] for d in range(W)], axis=1)  # M[s, d]
            self.send_counts = [[int(x) for x in M[s]] for s in range(W)]
            self.recv_counts = [[int(x) for x in M[:, d]] for d in range(W)]
        self.slices = []
        for d in range(W):
            rd = self.rows[d]
            if not rd.n_own:
                continue
            for s in range(W):
                if s == d:
                    continue
                rs = self.rows[s]
                for a, b in ((rd.loc0, rd.own0), (rd.own1, rd.loc1)):
                    lo, hi = max(a, rs.own0), min(b, rs.own1)
                    cnt = int(cum[hi] - cum[lo]) if hi > lo else 0
                    if cnt:
                        self.slices.append((s, d, int(cum[lo] - cum[rs.loc0]), int(cum[lo] - cum[rd.loc0]), cnt))

    def halo_particles(self, rank: int) -> int:
        r = self.rows[rank]
        return r.n_loc - r.n_own


# ---- communicators ------------------------------------------------------------------------------


class LocalComm:
    """All W ranks driven by this process; collectives are in-process copies."""

    def __init__(self, world: int):
        self.world = int(world)
        self.ranks = list(range(self.world))

    def allreduce(self, ts, op: str) -> None:
        acc = ts[0].clone()
        for t in ts[1:]:
            acc = {"min": acc.minimum, "max": acc.maximum, "sum": acc.add}[op](t)
        for t in ts:
            t.copy_(acc)

    def allgather(self, ts):
        """Per local rank: the (W, ...) stack of every rank's tensor."""
        torch = _torch_mod()
        full = torch.stack(ts)
        return [full for _ in ts]

    def alltoallv(self, sends, counts, recv_counts=None):
        """sends[r]: rows grouped by destination, counts[r][d] rows for rank d -> recvs[d]."""
        torch = _torch_mod()
        offs = [np.concatenate([[0], np.cumsum(c)]) for c in counts]
        recvs = []
        for d in range(self.world):
            parts = [sends[s][int(offs[s][d]):int(offs[s][d + 1])] for s in range(self.world)]
            recvs.append(torch.cat(parts) if parts else sends[d][:0])
        return recvs

    def exchange(self, slices, bufs) -> None:
        for s, d, so, do, c in slices:
            bufs[d][do:do + c].copy_(bufs[s][so:so + c])

    def allgatherv(self, ts):
        torch = _torch_mod()
        full = torch.cat(ts)
        return [full for _ in ts]


class DistComm:
    """One rank per process over torch.distributed (NCCL between GPUs; gloo in the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranks = [self.rank]

    def allreduce(self, ts, op: str) -> None:
        R = self.dist.ReduceOp
        self.dist.all_reduce(ts[0], op={"min": R.MIN, "max": R.MAX, "sum": R.SUM}[op], group=self.group)

    def allgather(self, ts):
        torch = _torch_mod()
        parts = [torch.empty_like(ts[0]) for _ in range(self.world)]
        self.dist.all_gather(parts, ts[0].contiguous(), group=self.group)
        return [torch.stack(parts)]

    def alltoallv(self, sends, counts, recv_counts=None):
        torch = _torch_mod()
        send = sends[0]
        if recv_counts is None:
            cin = torch.tensor(list(counts[0]), dtype=torch.int64, device=send.device)
            cout = torch.empty_like(cin)
            self.dist.all_to_all_single(cout, cin, group=self.group)
            out_splits = [int(x) for x in cout.tolist()]
        else:
            out_splits = [int(x) for x in recv_counts[0]]
        recv = torch.empty((sum(out_splits),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, out_splits, [int(x) for x in counts[0]], group=self.group)
        return [recv]

    def exchange(self, slices, bufs) -> None:
        buf = bufs[0]
        ops = []
        for s, d, so, do, c in slices:
            if s == self.rank:
                ops.append(self.dist.P2POp(self.dist.isend, buf[so:so + c], d, self.group))
            elif d == self.rank:
                ops.append(self.dist.P2POp(self.dist.irecv, buf[do:do + c], s, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def allgatherv(self, ts):
        torch = _torch_mod()
        t = ts[0]
        cnt = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        cnts = [torch.empty_like(cnt) for _ in range(self.world)]
        self.dist.all_gather(cnts, cnt, group=self.group)
        sizes = [int(c.item()) for c in cnts]
        m = max(sizes) if sizes else 0
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        out = torch.empty((m * self.world,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, pad, group=self.group)
        return [torch.cat([out[r * m:r * m + sizes[r]] for r in range(self.world)])]


def _torch_mod():
    import torch

    return torch


# ---- device backend -----------------------------------------------------------------------------


class DeviceSlabBackend:
    """gs_slab_* of libgs_b200.so for one rank (its own library context; several backends may
    share a GPU when one process drives several ranks)."""

    def __init__(self, spec, ctx=None, stream=None):
        import torch

        self.torch = torch
        self.ctx = ctx or N.Context.get()
        self.sysc = device.system_struct(spec, "cell")
        self.stream = stream
        self.dev = torch.device("cuda", self.ctx.device)

    def _s(self):
        return (self.stream or self.torch.cuda.current_stream(self.dev)).cuda_stream

    def _chk(self, rc, what):
        N.check(rc, what)

    def begin(self, n_glob: int, q, p, g):
        t = self.torch
        q, p = q.contiguous(), p.contiguous()
        g = g.to(dtype=t.int32).contiguous()
        self._keep = (q, p, g)  # alive until the kernel that reads them has run
        self._n_own = int(q.shape[0])
        self._chk(self.ctx.lib.gs_slab_begin(self.ctx.handle, ctypes.byref(self.sysc), n_glob, q.shape[0],
                                             q.data_ptr(), p.data_ptr(), g.data_ptr(), self._s()), "gs_slab_begin")

    def bbox(self):
        b4 = self.torch.empty(4, dtype=self.torch.float64, device=self.dev)
        self._chk(self.ctx.lib.gs_slab_bbox(self.ctx.handle, b4.data_ptr(), self._s()), "gs_slab_bbox")
        return b4

    def grid(self, b4) -> N.SlabGrid:
        g = N.SlabGrid()
        self._chk(self.ctx.lib.gs_slab_grid(self.ctx.handle, b4.data_ptr(), ctypes.byref(g), self._s()), "gs_slab_grid")
        return g

    def rows(self, ny: int):
        h = self.torch.empty(ny, dtype=self.torch.int64, device=self.dev)
        rc = self.ctx.lib.gs_slab_rows(self.ctx.handle, h.data_ptr(), self._s())
        if rc == N.GS_ERR_UNSUPPORTED:
            raise SlabUnavailable(N.last_error())
        self._chk(rc, "gs_slab_rows")
        return h

    def pack(self, owner, world: int):
        """Own particles grouped by destination rank (the counts come from the plan)."""
        t = self.torch
        n_own = self._n_own
        send = t.empty((max(n_own, 0), PACK_W), dtype=t.float64, device=self.dev)
        self._chk(self.ctx.lib.gs_slab_pack(self.ctx.handle, owner.data_ptr(), world, send.data_ptr() if n_own else 0,
                                            None, self._s()), "gs_slab_pack")
        return send

    def unpack(self, recv):
        recv = recv.contiguous()
        self._recv = recv
        self._n_own = int(recv.shape[0])
        self._chk(self.ctx.lib.gs_slab_unpack(self.ctx.handle, recv.shape[0], recv.data_ptr() if recv.shape[0] else 0,
                                              self._s()), "gs_slab_unpack")

    def layout(self, r: RankRows):
        self._chk(self.ctx.lib.gs_slab_layout(self.ctx.handle, r.own0, r.own1, r.loc0, r.loc1, r.own_begin, r.n_loc,
                                              self._s()), "gs_slab_layout")
        S, S2, g, f = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        self._chk(self.ctx.lib.gs_slab_views(self.ctx.handle, ctypes.byref(S), ctypes.byref(S2), ctypes.byref(g),
                                             ctypes.byref(f)), "gs_slab_views")
        # the stage ping-pongs the local records: buffer 0 is current after the layout
        self._S = (_wrap(self.torch, S.value, (r.n_loc + 1, 4), "<f8", self.dev),
                   _wrap(self.torch, S2.value, (r.n_loc + 1, 4), "<f8", self.dev))
        self._par = 0
        self.g = _wrap(self.torch, g.value, (max(r.n_loc, 1),), "<i4", self.dev)[:r.n_loc]
        self.flag = _wrap(self.torch, f.value, (1,), "<i4", self.dev)
        self.rows_ = r

    def lists(self, ncl: int):
        self._chk(self.ctx.lib.gs_slab_lists(self.ctx.handle, ncl, self._s()), "gs_slab_lists")

    @property
    def S(self):
        """(n_loc + 1, 4) view of the current local records (the halo slices go here)."""
        return self._S[self._par]

    def stage(self, step: int, s: int, dt: float):
        self._chk(self.ctx.lib.gs_slab_stage(self.ctx.handle, ctypes.byref(self.sysc), step, s, dt, self._s()),
                  "gs_slab_stage")
        self._par ^= 1

    def own(self):
        """(records (n_own, 4), global indices) of the own particles (views)."""
        r = self.rows_
        return self.S[r.own_begin:r.own_begin + r.n_own], self.g[r.own_begin:r.own_begin + r.n_own]

    def status(self) -> N.Status:
        st = N.Status()
        self._chk(self.ctx.lib.gs_slab_status(self.ctx.handle, ctypes.byref(st), self._s()), "gs_slab_status")
        return st


def _wrap(torch, ptr, shape, typestr, dev):
    class _H:
        pass

    h = _H()
    numel = int(np.prod(shape))
    h.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (int(ptr or 0), False), "version": 3}
    with torch.cuda.device(dev):
        return torch.as_tensor(h, device=dev).view(*shape)


# ---- the driver ---------------------------------------------------------------------------------


class SlabSolver:
    """integrator.evolve (integrator.py:66-121) on the cell path, decomposed into slabs.

    ``backends``: one per rank this process drives (``comm.ranks``); ``timer`` (optional):
    called as timer(kind, rank, fn) around every per-rank device phase ("stage", "build"), so
    a one-GPU emulation can time each rank's work separately (tools/time_slab.py)."""

    def __init__(self, spec, backends, comm, timer=None):
        self.spec = spec
        self.backends = list(backends)
        self.comm = comm
        self.W = comm.world
        assert len(self.backends) == len(comm.ranks)
        self.timer = timer or (lambda kind, rank, fn: fn())
        self.builds = 0
        self.plan = None
        self.halo_rows_per_stage = 0

    def _each(self, kind, fn):
        return [self.timer(kind, r, lambda b=b, r=r: fn(b, r)) for b, r in zip(self.backends, self.comm.ranks)]

    def rebuild(self):
        comm, W = self.comm, self.W
        b4 = self._each("build:bbox", lambda b, r: b.bbox())
        comm.allreduce(b4, "min")
        grids = self._each("build:grid", lambda b, r: b.grid(b4[self.comm.ranks.index(r)]))
        g = grids[0]
        if g.hashed:
            raise SlabUnavailable("the cloud spread beyond a row-major grid (hashed cells)")
        hists = self._each("build:rows", lambda b, r: b.rows(g.ny))
        H = comm.allgather(hists)[0].cpu().numpy()  # (W, ny): particles per row and current owner
        plan = SlabPlan(H.sum(axis=0), W, g.sub, rank_hists=H)
        torch = _torch_mod()
        owner = [torch.as_tensor(plan.owner, device=h.device) for h in hists]
        sends = self._each("build:pack", lambda b, r: b.pack(owner[self.comm.ranks.index(r)], W))
        recvs = comm.alltoallv(sends, [plan.send_counts[r] for r in comm.ranks],
                               [plan.recv_counts[r] for r in comm.ranks])
        for b, r, rv in zip(self.backends, comm.ranks, recvs):
            assert rv.shape[0] == plan.rows[r].n_own, (rv.shape, plan.rows[r])
            self.timer("build:unpack", r, lambda b=b, rv=rv: b.unpack(rv))
        self._each("build:layout", lambda b, r: b.layout(plan.rows[r]))
        comm.exchange(plan.slices, [b.S for b in self.backends])
        comm.exchange(plan.slices, [b.g for b in self.backends])
        self._each("build:lists", lambda b, r: b.lists(plan.ncl[r]))
        self.plan = plan
        self.builds += 1

    def evolve(self, q, p, t_final: float, steps: int):
        """Full (q, p) at t_final on every rank (cuda / cpu tensors like the inputs)."""
        torch = _torch_mod()
        n = int(q.shape[0])
        W = self.W
        dt = t_final / steps
        self.builds = 0
        for b, r in zip(self.backends, self.comm.ranks):
            c = (n + W - 1) // W
            r0, r1 = min(n, r * c), min(n, (r + 1) * c)
            gi = torch.arange(r0, r1, dtype=torch.int32, device=q.device)
            b.begin(n, q[r0:r1], p[r0:r1], gi)
        self.rebuild()
        for step in range(1, steps + 1):
            for s in range(4):
                self._each("stage", lambda b, r: b.stage(step, s, dt))
                if step == steps and s == 3:
                    break
                self.comm.exchange(self.plan.slices, [b.S for b in self.backends])
                flags = [b.flag.clone() for b in self.backends]
                self.comm.allreduce(flags, "max")
                if int(flags[0].item()):
                    self.rebuild()
        self._raise_first_failure(t_final, steps)
        recs, gids = zip(*[b.own() for b in self.backends])
        allrec = self.comm.allgatherv([x.contiguous() for x in recs])
        allg = self.comm.allgatherv([x.contiguous() for x in gids])
        out = torch.empty((n, 4), dtype=allrec[0].dtype, device=allrec[0].device)
        out[allg[0].long()] = allrec[0]
        return out[:, 0:2].contiguous(), out[:, 2:4].contiguous()

    def _raise_first_failure(self, t_final, steps):
        sts = [b.status() for b in self.backends]
        keys = [(math.inf, 0, 0) if st.code == N.GS_OK else (st.step * 8 + st.event, st.i, st.j) for st in sts]
        torch = _torch_mod()
        dev = self.backends[0].S.device
        enc = [torch.tensor([k[0] if k[0] != math.inf else 2.0 ** 62, float(st.i), float(st.j), float(st.code),
                             float(st.step), float(st.event)], dtype=torch.float64, device=dev)
               for k, st in zip(keys, sts)]
        rows = [tuple(e.tolist()) for e in enc]
        if isinstance(self.comm, DistComm) and self.W > 1:
            allk = [torch.empty_like(enc[0]) for _ in range(self.W)]
            self.comm.dist.all_gather(allk, enc[0], group=self.comm.group)
            rows = [tuple(x.tolist()) for x in allk]
        best = sorted(rows)[0]
        if best[0] >= 2.0 ** 62:
            return
        st = N.Status(int(best[3]), int(best[4]), int(best[1]), int(best[2]), 0, int(best[5]))
        exc = device.status_exception(st, t_final, steps)
        if exc is not None:
            raise exc
