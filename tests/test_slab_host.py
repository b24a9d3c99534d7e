"""Host logic of the slab-decomposed cell path (paper_1510_03816_b200/slab.py) on CPU.

The product's SlabSolver (ownership plan from the all-reduced row histogram, migration
all-to-all, halo slices, rebuild flags, final gather) runs with a numpy stand-in for gs_slab_*
(tests/helpers/slab_numpy.py): over LocalComm for W = 1 .. 5 ranks in one process, and over
gloo with world_size 2 through DistComm.  Checks: the plan's invariants, results bitwise
independent of W, and agreement with a plain truncated RK4 of all particles.
"""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "helpers"))

from slab_numpy import NumpySlabBackend, direct_truncated_evolve  # noqa: E402

from paper_1510_03816_b200 import slab  # noqa: E402

LAMBDA = 53 * np.log(2.0)


def _cloud(n=900, seed=11):
    rng = np.random.default_rng(seed)
    q = rng.uniform(0, 1, (n, 2))
    q[: n // 3] = 0.3 + 0.05 * rng.normal(size=(n // 3, 2))  # a dense blob: unequal row counts
    p = rng.normal(0, 0.02, (n, 2))
    return q, p


def _backend(cutoff, skin=None):
    return NumpySlabBackend("conical", cutoff / LAMBDA, True, 0.1, cutoff, skin=skin)


def _run_local(W, q, p, cutoff, steps=6, t_final=1.0, skin=None):
    comm = slab.LocalComm(W)
    solver = slab.SlabSolver(None, [_backend(cutoff, skin) for _ in range(W)], comm)
    qT, pT = solver.evolve(torch.from_numpy(q), torch.from_numpy(p), t_final, steps)
    return qT.numpy(), pT.numpy(), solver


@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_plan_partitions_rows_and_covers_halos(W):
    rng = np.random.default_rng(W)
    hist = rng.integers(0, 40, 57)
    hist[10:14] = 0
    plan = slab.SlabPlan(hist, W, 2)
    assert plan.Y[0] == 0 and plan.Y[-1] == 57 and all(a <= b for a, b in zip(plan.Y, plan.Y[1:]))
    assert sum(r.n_own for r in plan.rows) == hist.sum()
    for r, rr in enumerate(plan.rows):
        assert (plan.owner[rr.own0:rr.own1] == r).all()
        assert rr.n_own == hist[rr.own0:rr.own1].sum()
        assert rr.n_loc == hist[rr.loc0:rr.loc1].sum()
        if rr.n_own:
            assert rr.loc0 == max(rr.own0 - 2, 0) and rr.loc1 == min(rr.own1 + 2, 57)
            # the slices into this rank fill exactly its halo, without overlap
            got = np.zeros(rr.n_loc, dtype=int)
            got[rr.own_begin:rr.own_begin + rr.n_own] += 1
            for s, d, so, do, c in plan.slices:
                if d == r:
                    got[do:do + c] += 1
                    rs = plan.rows[s]
                    assert rs.own_begin <= so and so + c <= rs.own_begin + rs.n_own  # from the sender's own block
            assert (got == 1).all()
    # migration counts from per-owner histograms: rows of d held by s
    H = np.stack([rng.multinomial(int(h), [1.0 / W] * W) for h in hist], axis=1)  # (W, ny), sums to hist
    plan2 = slab.SlabPlan(hist, W, 2, rank_hists=H)
    for s_ in range(W):
        for d in range(W):
            rd = plan2.rows[d]
            assert plan2.send_counts[s_][d] == H[s_, rd.own0:rd.own1].sum() == plan2.recv_counts[d][s_]
    assert [sum(c) for c in plan2.recv_counts] == [r.n_own for r in plan2.rows]
    assert plan2.ncl == [int(((hist[r.own0:r.own1] + 1) // 2).sum()) for r in plan2.rows]
    # balance: no rank owns more than its share plus one row
    for rr in plan.rows:
        assert rr.n_own <= hist.sum() / W + hist.max()


def test_local_ranks_are_bitwise_independent_of_w_and_match_direct_rk4():
    q, p = _cloud()
    cutoff = 0.12
    ref_q, ref_p, s1 = _run_local(1, q, p, cutoff)
    assert s1.builds >= 2  # the flow moves particles past half the skin: rebuilds mid-evolve
    for W in (2, 3, 5):
        qW, pW, sW = _run_local(W, q, p, cutoff)
        np.testing.assert_array_equal(qW, ref_q)
        np.testing.assert_array_equal(pW, ref_p)
        assert sW.builds == s1.builds
    dq, dp = direct_truncated_evolve("conical", cutoff / LAMBDA, True, 0.1, cutoff, q, p, 1.0, 6)
    assert np.abs(ref_q - dq).max() / np.abs(dq).max() <= 1e-13
    assert np.abs(ref_p - dp).max() / np.abs(dp).max() <= 1e-11


def test_empty_ranks_and_migration():
    # more ranks than occupied rows: some ranks own nothing; particles cross slab borders
    q, p = _cloud(200, seed=4)
    q[:, 1] = 0.5 + 0.02 * (q[:, 1] - 0.5)  # a thin horizontal band: few cell rows
    ref_q, ref_p, _ = _run_local(1, q, p, 0.08)
    qW, pW, sW = _run_local(8, q, p, 0.08)
    assert any(r.n_own == 0 for r in sW.plan.rows)
    np.testing.assert_array_equal(qW, ref_q)
    np.testing.assert_array_equal(pW, ref_p)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, p = _cloud()
        solver = slab.SlabSolver(None, [_backend(0.12)], slab.DistComm())
        qT, pT = solver.evolve(torch.from_numpy(q), torch.from_numpy(p), 1.0, 6)
        np.save(os.path.join(outdir, f"q_{rank}.npy"), qT.numpy())
        np.save(os.path.join(outdir, f"p_{rank}.npy"), pT.numpy())
        with open(os.path.join(outdir, f"b_{rank}.txt"), "w") as f:
            f.write(f"{solver.builds} {len(solver.plan.slices)}")
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_gloo_slab_solver_equals_one_rank():
    q, p = _cloud()
    ref_q, ref_p, s1 = _run_local(1, q, p, 0.12)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        for r in range(2):
            np.testing.assert_array_equal(np.load(os.path.join(d, f"q_{r}.npy")), ref_q)
            np.testing.assert_array_equal(np.load(os.path.join(d, f"p_{r}.npy")), ref_p)
            builds, nslices = map(int, open(os.path.join(d, f"b_{r}.txt")).read().split())
            assert builds == s1.builds and nslices == 2
