"""Slab-decomposed cell path (csrc/gs_slab.cu + paper_1510_03816_b200/slab.py) on one GPU.

W ranks run in one process (LocalComm, one library context per rank, the collectives are
copies), so the exact per-rank device code of a W-GPU run executes here: each rank builds its
grid, clusters and lists over its own cell rows + halo only and sweeps its own rows.  Checks:
rows bitwise independent of W (1, 2, 3, 8), agreement with the one-GPU cluster-list evolve and
with the C oracle's truncated evolve, list rebuilds with migration mid-evolve, the reference's
coincidence error.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solver(torch, spec, W):
    from paper_1510_03816_b200 import _native as N
    from paper_1510_03816_b200 import slab

    backends = [slab.DeviceSlabBackend(spec, ctx=N.Context(0)) for _ in range(W)]
    return slab.SlabSolver(spec, backends, slab.LocalComm(W))


def _workload(n, gain):
    from paper_1510_03816_b200 import configs

    w = configs.c5(n)
    return w, np.ascontiguousarray(gain * (w.target - w.q))


def test_slab_rows_are_bitwise_independent_of_the_rank_count(cuda):
    torch = cuda
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import device

    w, p = _workload(65536, 0.01)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    q_d, p_d = torch.from_numpy(w.q).cuda(), torch.from_numpy(p).cuda()
    steps, tf = 4, 0.2
    ref = None
    for W in (1, 2, 3, 8):
        s = _solver(torch, spec, W)
        qT, pT = s.evolve(q_d, p_d, tf, steps)
        if ref is None:
            ref = (qT.clone(), pT.clone(), s.builds)
            assert s.builds >= 2, s.builds  # rebuilds (and migrations) happen mid-evolve
        else:
            assert torch.equal(qT, ref[0]) and torch.equal(pT, ref[1]), W
            assert s.builds == ref[2]
            assert len(s.plan.slices) >= 2 * (W - 1)
    # the one-GPU cluster-list evolve: the same truncation, another cluster pairing
    device.set_path("cell")
    try:
        q1, p1, _ = device.evolve(spec, q_d, p_d, tf, steps)
    finally:
        device.set_path("auto")
    eq = float((ref[0] - q1).abs().max() / q1.abs().max())
    ep = float((ref[1] - p1).abs().max() / p1.abs().max())
    assert eq <= 1e-13 and ep <= 1e-11, (eq, ep)


def test_slab_matches_the_truncated_oracle(cuda):
    torch = cuda
    import paper_1510_03816_b200 as gs
    from oracle import native
    from oracle.restate import Kernel

    w, p = _workload(12000, 0.01)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    s = _solver(torch, spec, 4)
    qT, pT = s.evolve(torch.from_numpy(w.q).cuda(), torch.from_numpy(p).cuda(), 0.1, 2)
    oq, op = native.evolve(Kernel(0, w.alpha, True), w.sigma2, w.q, p, 0.1, 2, cutoff=w.sigma)
    eq = np.abs(qT.cpu().numpy() - oq).max() / np.abs(oq).max()
    ep = np.abs(pT.cpu().numpy() - op).max() / np.abs(op).max()
    assert eq <= 1e-12 and ep <= 1e-10, (eq, ep)


def test_slab_raises_the_reference_coincidence_error(cuda):
    torch = cuda
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import device

    w, p = _workload(20000, 0.01)
    q = w.q.copy()
    q[15000] = q[300]
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    q_d, p_d = torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()
    msgs = []
    for W in (1, 3):
        with pytest.raises(gs.DegenerateConfigurationError) as ei:
            _solver(torch, spec, W).evolve(q_d, p_d, 0.1, 2)
        msgs.append(str(ei.value))
    device.set_path("cell")
    try:
        with pytest.raises(gs.DegenerateConfigurationError) as ei:
            device.evolve(spec, q_d, p_d, 0.1, 2)
    finally:
        device.set_path("auto")
    assert msgs[0] == msgs[1] == str(ei.value)
    assert msgs[0].startswith("particles 300 and 15000 coincide")


def test_sharded_solver_takes_the_slab_path_in_an_nccl_world(cuda):
    """ShardedSolver's multi-rank cell path (slab decomposition over DistComm: NCCL all-reduces,
    all-to-all, P2P halo slices, all-gather) in a one-process NCCL world equals the one-rank
    LocalComm run bitwise."""
    torch = cuda
    import os
    import socket

    import torch.distributed as dist

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import sharded, slab

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    w, p = _workload(30000, 0.01)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    q_d, p_d = torch.from_numpy(w.q).cuda(), torch.from_numpy(p).cuda()
    ref_q, ref_p = _solver(torch, spec, 1).evolve(q_d, p_d, 0.2, 4)
    gs.set_path("cell")
    calls = []
    orig = slab.SlabSolver.rebuild

    def spy(self):
        calls.append(1)
        return orig(self)

    slab.SlabSolver.rebuild = spy
    try:
        qT, pT = sharded.ShardedSolver(spec, force_split=True).evolve(w.q, p, 0.2, 4)
    finally:
        slab.SlabSolver.rebuild = orig
        gs.set_path("auto")
    assert calls, "the slab path was not taken"
    assert torch.equal(qT, ref_q) and torch.equal(pT, ref_p)


def test_full_size_c5_slab_ranks_match_the_one_gpu_lists(cuda):
    """C5 at full size (N = 2^20) on 8 slab ranks (one GPU, LocalComm) at the configured gain: one RK4
    step equals the one-GPU cluster-list evolve to rounding (the C oracle pins that one,
    tests/test_gpu_fullsize.py), and every rank holds a balanced share."""
    torch = cuda
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    w = configs.c5()
    p = np.ascontiguousarray(w.h * (w.target - w.q))
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    q_d, p_d = torch.from_numpy(w.q).cuda(), torch.from_numpy(p).cuda()
    s = _solver(torch, spec, 8)
    qT, pT = s.evolve(q_d, p_d, w.t_final / w.steps, 1)
    device.set_path("cell")
    try:
        q1, p1, _ = device.evolve(spec, q_d, p_d, w.t_final / w.steps, 1)
    finally:
        device.set_path("auto")
    assert float((qT - q1).abs().max() / q1.abs().max()) <= 1e-13
    assert float((pT - p1).abs().max() / p1.abs().max()) <= 1e-11
    own = [r.n_own for r in s.plan.rows]
    assert sum(own) == w.n and max(own) <= 1.05 * w.n / 8


def test_hashed_grid_falls_back_to_the_all_gather_path(cuda):
    """A cloud that needs the hashed grid (a far outlier: the row-major grid would exceed the cell
    cap) has no row slabs: ShardedSolver's cell path falls back to own rows + all-gather, and the
    result is the one-GPU cell path's."""
    torch = cuda
    import os
    import socket

    import torch.distributed as dist

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import device, sharded

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    w, p = _workload(20000, 0.01)
    q = w.q.copy()
    q[123] = (3.0e3, -2.0e3)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    gs.set_path("cell")
    try:
        solver = sharded.ShardedSolver(spec, force_split=True)
        qT, pT = solver.evolve(q, p, 0.1, 2)
        q1, p1, _ = device.evolve(spec, q, p, 0.1, 2)
    finally:
        gs.set_path("auto")
    assert solver.slab is False  # took the fallback
    assert float((qT - q1).abs().max() / q1.abs().max()) <= 1e-13


def test_slab_gaussian_family(cuda):
    """The gaussian family through the slab path (support radius alpha sqrt(2 Lambda)): W = 3 ranks
    bitwise W = 1, and the one-GPU cluster-list evolve to rounding."""
    torch = cuda
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import device

    rng = np.random.default_rng(12)
    n = 30000
    q = rng.uniform(0, 1, (n, 2))
    p = rng.normal(0, 1e-3, (n, 2))  # a gentle flow: particles move less than alpha (no chaotic amplification)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(family="gaussian", alpha=0.002), sigma2=0.05)
    q_d, p_d = torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()
    q1s, p1s = _solver(torch, spec, 1).evolve(q_d, p_d, 0.2, 3)
    q3s, p3s = _solver(torch, spec, 3).evolve(q_d, p_d, 0.2, 3)
    assert torch.equal(q1s, q3s) and torch.equal(p1s, p3s)
    device.set_path("cell")
    try:
        q1, p1, _ = device.evolve(spec, q_d, p_d, 0.2, 3)
    finally:
        device.set_path("auto")
    assert float((q1s - q1).abs().max() / q1.abs().max()) <= 1e-13
    assert float((p1s - p1).abs().max() / p1.abs().max()) <= 1e-11
