"""The multi-GPU building blocks on one GPU: stage API, symmetric pair split, ShardedSolver (world 1).

Nothing here runs ranks that wait on each other; the decomposition is checked by evaluating
the ranks' work items one after another on the single device.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _setup(n=6000, seed=7):
    import paper_1510_03816_b200 as gs

    rng = np.random.default_rng(seed)
    q = rng.uniform(0, 1, (n, 2))
    p = rng.normal(0, 0.01, (n, 2))
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.4 / gs.LAMBDA), sigma2=0.05)
    return gs, q, p, spec


def test_symmetric_split_sums_to_the_full_pair_sum(cuda):
    import torch

    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import device, sharded

    gs, q, p, spec = _setup()
    n = q.shape[0]
    be = sharded.DeviceStageBackend(spec)
    lib, h = be.ctx.lib, be.ctx.handle
    total = int(lib.gs_sym_parts(n))
    assert total > 0
    be.begin(q, p, 0, n)
    assert be.path() == "dense"
    full = be.new_partials(n)
    be.pairs_sym(1, 0, 0, total, full)
    parts = []
    for b, e in ((0, total // 3), (total // 3, 2 * total // 3), (2 * total // 3, total)):
        R = be.new_partials(n)
        be.pairs_sym(1, 0, b, e, R)
        parts.append(R)
    split = parts[0] + parts[1] + parts[2]
    torch.cuda.synchronize()
    assert rel(split.cpu().numpy(), full.cpu().numpy()) <= 1e-13
    # the raw sums reproduce particles.rhs after the kernel scales
    sysc = device.system_struct(spec)
    dq, dp = device.rhs(spec, q, p)
    alpha = spec.kernel.alpha
    want_dq = full[:, 0:2].cpu().numpy() + spec.sigma2 * p
    want_dp = full[:, 2:4].cpu().numpy() / alpha
    assert rel(want_dq, dq.cpu().numpy()) <= 1e-13 and rel(want_dp, dp.cpu().numpy()) <= 1e-12
    st = N.Status()
    N.check(lib.gs_status_fetch(h, ctypes.byref(st), None), "status")
    assert st.code == N.GS_OK


def test_stage_finish_matches_stage_run(cuda):
    """rows [r0, r1): (symmetric raw sums -> gs_stage_finish) == gs_stage_run on the same rows."""
    import torch

    from paper_1510_03816_b200 import sharded

    gs, q, p, spec = _setup(n=5000)
    n = q.shape[0]
    r0, r1 = 1200, 3700
    a = sharded.DeviceStageBackend(spec)
    a.begin(q, p, 0, n)
    R = a.new_partials(n)
    a.pairs_sym(1, 0, 0, a.sym_parts(), R)
    a.begin(q, p, r0, r1)
    a.finish(1, 0, 0.1, R[r0:r1].contiguous())
    Sa = a.state(n).clone()
    b = sharded.DeviceStageBackend(spec)
    b.ctx = sharded.N.Context(torch.cuda.current_device())  # separate workspaces
    b.begin(q, p, r0, r1)
    b.run(1, 0, 0.1)
    Sb = b.state(n).clone()
    torch.cuda.synchronize()
    assert rel(Sa[r0:r1].cpu().numpy(), Sb[r0:r1].cpu().numpy()) <= 1e-13
    np.testing.assert_array_equal(Sa[:r0].cpu().numpy(), Sb[:r0].cpu().numpy())  # other rows untouched


def test_sharded_solver_world1_equals_evolve(cuda):
    from paper_1510_03816_b200 import device, sharded

    gs, q, p, spec = _setup(n=3000)
    solver = sharded.ShardedSolver(spec)
    qT, pT = solver.evolve(q, p, 1.0, 4)
    q2, p2, _ = device.evolve(spec, q, p, 1.0, 4)
    np.testing.assert_array_equal(qT.cpu().numpy(), q2.cpu().numpy())
    np.testing.assert_array_equal(pT.cpu().numpy(), p2.cpu().numpy())


def test_sharded_match_world1_matches_device_match(cuda):
    from paper_1510_03816_b200 import configs, device, sharded

    import paper_1510_03816_b200 as gs

    w = configs.c1()
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    r = sharded.ShardedSolver(spec).match(w.q, w.target, w.h, w.epsilon, w.max_iter, "residual", "max", 1.0, w.steps)
    d = device.match(spec, w.q, w.target, w.h, w.epsilon, w.max_iter, "residual", "max", 1.0, w.steps)
    assert r["iterations"] == d["iterations"] == 36 and r["converged"]
    assert rel(r["p0"].cpu().numpy(), d["p0"].cpu().numpy()) <= 1e-10
    assert r["hamiltonian"] == pytest.approx(d["hamiltonian"], rel=1e-10)


def _nccl_world1():
    import os
    import socket

    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))


def test_sharded_solver_nccl_code_path_world1(cuda):
    """The exact multi-GPU code path (symmetric pair split, NCCL reduce-scatter of the raw row
    sums, stage finish, NCCL all-gather of the stage records, first-failure agreement) in a
    single-process NCCL world: one GPU, nothing waits on another rank."""
    import torch.distributed as dist

    from paper_1510_03816_b200 import device, sharded

    _nccl_world1()
    assert dist.get_backend() == "nccl"
    gs, q, p, spec = _setup(n=5000)
    solver = sharded.ShardedSolver(spec, force_split=True)
    qT, pT = solver.evolve(q, p, 1.0, 4)
    q2, p2, _ = device.evolve(spec, q, p, 1.0, 4)
    assert rel(qT.cpu().numpy(), q2.cpu().numpy()) <= 1e-13
    assert rel(pT.cpu().numpy(), p2.cpu().numpy()) <= 1e-13
    # failures are agreed and re-raised like the single-GPU path
    qc = q.copy()
    qc[7] = qc[3]
    pc = p.copy()
    with pytest.raises(gs.DegenerateConfigurationError, match="particles 3 and 7 coincide"):
        solver.evolve(qc, pc, 1.0, 2)
    # cell path through the same plumbing (rows + all-gather)
    gs.set_path("cell")
    try:
        qT, pT = sharded.ShardedSolver(spec, force_split=True).evolve(q, p, 1.0, 2)
        q2, p2, _ = device.evolve(spec, q, p, 1.0, 2)
        assert rel(qT.cpu().numpy(), q2.cpu().numpy()) <= 1e-13
    finally:
        gs.set_path("auto")
    from paper_1510_03816_b200 import configs

    w = configs.c1()
    spec1 = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    r = sharded.ShardedSolver(spec1, force_split=True).match(w.q, w.target, w.h, w.epsilon, w.max_iter, "residual",
                                                             "max", 1.0, w.steps)
    assert r["iterations"] == 36 and r["converged"]


def _two_rank_emulation(n=5000, steps=3, only_rank0=False, W=2):
    """W library contexts on one GPU play the ranks of the peer-memory exchange, driven in
    stream order (every wait is satisfied by work queued before it: nothing spins on a kernel
    that has not run)."""
    import torch

    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import sharded

    gs, q, p, spec = _setup(n=n)
    c = (n + W - 1) // W
    be = [sharded.DeviceStageBackend(spec, ctx=N.Context(0)) for _ in range(W)]
    for r, b in enumerate(be):
        r0, r1, _ = sharded.row_split(n, W, r)
        b.begin(q, p, r0, r1)
    ptrs = [b.p2p_local(c * W) for b in be]
    S, R, F = ([x[k] for x in ptrs] for k in range(3))
    for r, b in enumerate(be):
        b.p2p_set_peers(W, r, S, R, F)
    total = be[0].sym_parts()
    ranges = [(r * total // W, (r + 1) * total // W) for r in range(W)]
    dt = 1.0 / steps
    active = be[:1] if only_rank0 else be
    for step in range(1, steps + 1):
        for s in range(4):
            for r, b in enumerate(active):
                b.p2p_pairs(step, s, *ranges[r])
            for b in active:
                b.p2p_finish(step, s, dt)
    for b in active:
        b.p2p_sync()
    torch.cuda.synchronize()
    return gs, q, p, spec, be


@pytest.mark.parametrize("W,n", [(2, 5000), (3, 4999)])
def test_peer_exchange_two_ranks_emulated(cuda, W, n):
    """gs_p2p_*: the fused epilogue + peer stores of W ranks (uneven split for W = 3) reproduce
    the single-GPU evolve, and all ranks end with identical full states."""
    from paper_1510_03816_b200 import device

    gs, q, p, spec, be = _two_rank_emulation(n=n, W=W)
    SA = be[0].state(n).clone()
    for b in be:
        assert b.p2p_timeouts() == 0
        np.testing.assert_array_equal(b.state(n).cpu().numpy(), SA.cpu().numpy())
    q2, p2, _ = device.evolve(spec, q, p, 1.0, 3)
    # the ranks' row sums are added in rank order instead of the one-GPU slot order: rounding only
    assert rel(SA[:, 0:2].cpu().numpy(), q2.cpu().numpy()) <= 1e-13
    assert rel(SA[:, 2:4].cpu().numpy(), p2.cpu().numpy()) <= 1e-11


def test_peer_exchange_lost_signal_times_out(cuda, monkeypatch):
    """A rank whose peer never signals gives up after the timeout (no hang) and counts it."""
    monkeypatch.setenv("GS_B200_P2P_TIMEOUT_S", "0.02")
    gs, q, p, spec, be = _two_rank_emulation(n=3000, steps=1, only_rank0=True)
    assert be[0].p2p_timeouts() > 0


def test_sharded_solver_peer_exchange_world1(cuda):
    """ShardedSolver's peer-exchange path (handle export / import, pairs, fused finish, sync,
    timeout agreement) in a one-process NCCL world."""
    from paper_1510_03816_b200 import device, sharded

    _nccl_world1()
    gs, q, p, spec = _setup(n=5000)
    solver = sharded.ShardedSolver(spec, force_split=True, p2p=True)
    qT, pT = solver.evolve(q, p, 1.0, 4)
    assert solver.p2p  # no timeout, still on the peer path
    q2, p2, _ = device.evolve(spec, q, p, 1.0, 4)
    assert rel(qT.cpu().numpy(), q2.cpu().numpy()) <= 1e-13
    assert rel(pT.cpu().numpy(), p2.cpu().numpy()) <= 1e-13
    qc = q.copy()
    qc[7] = qc[3]
    with pytest.raises(gs.DegenerateConfigurationError, match="particles 3 and 7 coincide"):
        solver.evolve(qc, p, 1.0, 2)


def _ipc_worker(rank, world, port, out):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1510_03816_b200 import sharded

    gs, q, p, spec = _setup(n=2000)
    be = sharded.DeviceStageBackend(spec)
    r0, r1, c = sharded.row_split(2000, world, rank)
    be.begin(q, p, r0, r1)
    handles = be.p2p_export(c * world)
    allh = [None] * world
    dist.all_gather_object(allh, handles)
    be.p2p_import(world, rank, b"".join(allh))  # opens the other process's buffers (CUDA IPC)
    dist.barrier()
    be.ctx.lib.gs_p2p_close(be.ctx.handle)
    with open(f"{out}.{rank}", "w") as f:
        f.write("ok")
    dist.destroy_process_group()


def test_peer_handles_open_across_processes(cuda, tmp_path):
    """The IPC handle exchange of the peer-memory path between two processes (no kernel waits
    on the other process: only the mapping is exercised)."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "ipc")
    mp.spawn(_ipc_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        assert open(f"{out}.{r}").read() == "ok"


def test_cell_rows_of_a_rank_equal_the_full_cell_rhs(cuda):
    """The cell path of one rank (rows [r0, r1) of an uneven split) evaluates only its own
    targets, compacted in cell order (no warp carries another rank's rows), and every row keeps
    the summation order of the full-row launch: the slices are bitwise the full RHS."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import sharded

    rng = np.random.default_rng(31)
    n = 40000
    q = rng.uniform(0, 1, (n, 2))
    p = rng.normal(0, 0.01, (n, 2))
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.02 / gs.LAMBDA), sigma2=0.1)
    gs.set_path("cell")
    try:
        dq, dp = sharded.rhs_rows(spec, q, p, 0, n)
        cuts = [0, 7001, 7002, 23000, n]
        parts = [sharded.rhs_rows(spec, q, p, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    finally:
        gs.set_path("auto")
    np.testing.assert_array_equal(np.concatenate([a.cpu().numpy() for a, _ in parts]), dq.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate([b.cpu().numpy() for _, b in parts]), dp.cpu().numpy())


def test_sharded_dense_evolve_is_one_graph_replay(cuda, monkeypatch):
    """The dense split's stage loop (pair share, NCCL reduce-scatter, finish, NCCL all-gather) is
    captured once per configuration and replayed: bitwise the host-driven loop, the second evolve
    reuses the graph, and a coincidence inside the replayed stages is still raised."""
    import torch

    from paper_1510_03816_b200 import sharded

    _nccl_world1()
    gs, q, p, spec = _setup(n=5000)
    host = sharded.ShardedSolver(spec, force_split=True)
    host.graphs = False
    qh, ph = host.evolve(q, p, 1.0, 4)
    solver = sharded.ShardedSolver(spec, force_split=True)
    qg, pg = solver.evolve(q, p, 1.0, 4)
    assert solver._graph is not None
    assert torch.equal(qg, qh) and torch.equal(pg, ph)
    g0 = solver._graph
    q2, p2 = solver.evolve(q, p, 1.0, 4)
    assert solver._graph is g0 and torch.equal(q2, qh)
    qc = q.copy()
    qc[7] = qc[3]
    with pytest.raises(gs.DegenerateConfigurationError, match="particles 3 and 7 coincide"):
        solver.evolve(qc, p, 1.0, 4)
    q3, _ = solver.evolve(q, p, 1.0, 4)  # the status is reset by the next evolve
    assert torch.equal(q3, qh)
