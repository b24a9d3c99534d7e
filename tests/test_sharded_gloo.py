"""Multi-rank host logic of the row-sharded driver (paper_1510_03816_b200/sharded.py) on CPU.

world_size = 2 over gloo.  The ranks run the product's ShardedSolver orchestration (row
split, per-stage all-gather of the 32-byte stage records, MAX/SUM all-reduces, first-failure
agreement) with a numpy stage backend standing in for gs_stage_* (test-only; the stage math
is the C oracle's row RHS plus the RK4 stage epilogue of csrc/gs_dense.cu k_finish).
"""

import os
import re
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1510_03816_b200 import _native as N


class NumpyStageBackend:
    """CPU stand-in for libgs_b200's gs_stage_* (same contract, see include/geoshoot_b200.h)."""

    device = "cpu"

    def __init__(self, spec, sym=False):
        from oracle.restate import Kernel

        self.k = Kernel(0 if spec.kernel.family.value == "conical" else 1, spec.kernel.alpha, spec.kernel.normalized)
        self.sigma2 = spec.sigma2
        self.supports_sym = sym

    def begin(self, q, p, r0, r1):
        q = np.asarray(q, dtype=np.float64)
        p = np.asarray(p, dtype=np.float64)
        self.n, self.r0, self.r1 = q.shape[0], r0, r1
        self.S = torch.zeros((self.n + 64, 4), dtype=torch.float64)
        self.S[: self.n, 0:2] = torch.from_numpy(q)
        self.S[: self.n, 2:4] = torch.from_numpy(p)
        self.B = self.S[r0:r1].clone().numpy()
        self.A = np.zeros_like(self.B)
        self.fail = None  # (event key, code, step, event, i, j)

    def state(self, rows):
        return self.S[:rows]

    def run(self, step, s, dt):
        from oracle import native
        from oracle.restate import OracleDegenerate

        if self.fail is not None or self.r1 <= self.r0:
            return
        S = self.S[: self.n].numpy()
        try:
            dq, dp = native.rhs(self.k, self.sigma2, S[:, 0:2], S[:, 2:4], rows=(self.r0, self.r1))
        except OracleDegenerate as exc:
            i, j = map(int, re.search(r"particles (\d+) and (\d+)", str(exc)).groups())
            self.fail = (step * 8 + 2 * s, N.GS_ERR_COINCIDENT, step, 2 * s, i, j)
            return
        k = np.concatenate([dq, dp], axis=1)
        if s == 0:
            self.A = k.copy()
        else:
            self.A = self.A + (1.0 if s == 3 else 2.0) * k
        if s < 3:
            nxt = self.B + ((dt if s == 2 else 0.5 * dt) * k)
        else:
            nxt = self.B + (dt / 6.0) * self.A
            self.B = nxt
        self.S[self.r0:self.r1] = torch.from_numpy(nxt)
        if not np.all(np.isfinite(nxt)):
            code = N.GS_ERR_NONFINITE_STATE if s == 3 else N.GS_ERR_NONFINITE_STAGE
            self.fail = (step * 8 + 2 * s + 1, code, step, 2 * s + 1, -1, -1)

    # -- symmetric split emulation: rank b..e owns source blocks of 32 columns ------------------
    def path(self):
        return "dense"

    def sym_parts(self):
        return (self.n + 31) // 32

    def new_partials(self, rows):
        return torch.zeros((rows, 4), dtype=torch.float64)

    def pairs_sym(self, step, s, b, e, R):
        """Raw sums (sum_j G p_j, sum_j c (q_i - q_j)) of all rows over sources [32b, 32e)."""
        R.zero_()
        if self.fail is not None:
            return
        S = self.S[: self.n].numpy()
        q, p = S[:, 0:2], S[:, 2:4]
        J = np.arange(32 * b, min(self.n, 32 * e))
        if J.size == 0:
            return
        d = q[:, None, :] - q[None, J, :]
        r = np.sqrt(np.sum(d * d, axis=-1))
        pdot = p @ p[J].T
        bad = (r == 0.0) & (np.arange(self.n)[:, None] != J[None, :]) & (pdot != 0.0)
        if np.any(bad):
            i, jj = np.argwhere(bad)[0]
            self.fail = (step * 8 + 2 * s, N.GS_ERR_COINCIDENT, step, 2 * s, int(i), int(J[jj]))
            return
        G = np.exp(-r / self.k.alpha) if self.k.family == 0 else np.exp(-0.5 * (r / self.k.alpha) ** 2)
        with np.errstate(divide="ignore", invalid="ignore"):
            c = np.where(r > 0, pdot * G / (r if self.k.family == 0 else 1.0), 0.0)
        R[: self.n, 0:2] = torch.from_numpy(G @ p[J])
        R[: self.n, 2:4] = torch.from_numpy(np.sum(c[..., None] * d, axis=1))

    def finish(self, step, s, dt, R_rows):
        if self.fail is not None or self.r1 <= self.r0:
            return
        raw = R_rows[: self.r1 - self.r0].numpy()
        sq = 1.0 if self.k.normalized else 1.0 / (2 * np.pi * self.k.alpha ** 2)
        sp = sq / (self.k.alpha if self.k.family == 0 else self.k.alpha ** 2)
        pin = self.S[self.r0:self.r1, 2:4].numpy()
        dq = raw[:, 0:2] * sq + (self.sigma2 * pin if self.sigma2 != 0.0 else 0.0)
        k = np.concatenate([dq, raw[:, 2:4] * sp], axis=1)
        self._epilogue(step, s, dt, k)

    def _epilogue(self, step, s, dt, k):
        if s == 0:
            self.A = k.copy()
        else:
            self.A = self.A + (1.0 if s == 3 else 2.0) * k
        if s < 3:
            nxt = self.B + ((dt if s == 2 else 0.5 * dt) * k)
        else:
            nxt = self.B + (dt / 6.0) * self.A
            self.B = nxt
        self.S[self.r0:self.r1] = torch.from_numpy(nxt)
        if not np.all(np.isfinite(nxt)):
            code = N.GS_ERR_NONFINITE_STATE if s == 3 else N.GS_ERR_NONFINITE_STAGE
            self.fail = (step * 8 + 2 * s + 1, code, step, 2 * s + 1, -1, -1)

    def status(self):
        if self.fail is None:
            return N.Status(N.GS_OK, 0, -1, -1, 0, 0)
        _, code, step, ev, i, j = self.fail
        return N.Status(code, step, i, j, 0, ev)

    def hamiltonian_rows(self, spec, q, p, r0, r1):
        from oracle import native

        q = np.asarray(q, dtype=np.float64)
        p = np.asarray(p, dtype=np.float64)
        if r1 <= r0:
            return 0.0
        dq, _ = native.rhs(self.k, 0.0, q, p, rows=(r0, r1))
        return float(np.sum(p[r0:r1] * dq))


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
        import paper_1510_03816_b200 as gs
        from paper_1510_03816_b200 import configs, sharded

        # 1) evolve, odd N (padded last slice)
        rng = np.random.default_rng(3)
        n = 301
        q = rng.uniform(0, 1, (n, 2))
        p = rng.normal(0, 0.05, (n, 2))
        spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.3 / gs.LAMBDA), sigma2=0.1)
        solver = sharded.ShardedSolver(spec, backend=NumpyStageBackend(spec))
        qT, pT = solver.evolve(q, p, 1.0, 5)
        np.save(os.path.join(outdir, f"evolve_q_{rank}.npy"), qT.numpy())
        np.save(os.path.join(outdir, f"evolve_p_{rank}.npy"), pT.numpy())
        # 1b) the symmetric split: pair subsets per rank + reduce-scatter of raw row sums
        sym = sharded.ShardedSolver(spec, backend=NumpyStageBackend(spec, sym=True))
        qS, pS = sym.evolve(q, p, 1.0, 5)
        np.save(os.path.join(outdir, f"sym_q_{rank}.npy"), qS.numpy())
        np.save(os.path.join(outdir, f"sym_p_{rank}.npy"), pS.numpy())

        # 2) the C1 match (momentum update) across ranks
        w = configs.c1()
        spec1 = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
        s1 = sharded.ShardedSolver(spec1, backend=NumpyStageBackend(spec1))
        r = s1.match(w.q, w.target, w.h, w.epsilon, w.max_iter, "residual", "max", 1.0, w.steps)
        np.save(os.path.join(outdir, f"match_p0_{rank}.npy"), r["p0"].numpy())
        with open(os.path.join(outdir, f"match_{rank}.txt"), "w") as f:
            f.write(f"{r['iterations']} {r['converged']} {r['hamiltonian']!r} {r['diagnosis']}")

        # 3) a coincidence inside rank 1's rows is raised identically on both ranks
        q2 = q.copy()
        q2[290] = q2[200]
        try:
            solver.evolve(q2, p, 1.0, 5)
            msg = "no error"
        except gs.DegenerateConfigurationError as exc:
            msg = str(exc)
        with open(os.path.join(outdir, f"err_{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_sharded_solver_matches_single_process_oracle():
    from oracle import native, restate
    from oracle.restate import Kernel
    from paper_1510_03816_b200 import configs, sharded
    import paper_1510_03816_b200 as gs

    assert sharded.row_split(301, 2, 0) == (0, 151, 151)
    assert sharded.row_split(301, 2, 1) == (151, 301, 151)
    assert sharded.row_split(5, 8, 7) == (5, 5, 1)

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        rng = np.random.default_rng(3)
        q = rng.uniform(0, 1, (301, 2))
        p = rng.normal(0, 0.05, (301, 2))
        k = Kernel(0, 0.3 / gs.LAMBDA, True)
        oq, op = native.evolve(k, 0.1, q, p, 1.0, 5)
        for r in range(2):
            np.testing.assert_array_equal(np.load(os.path.join(d, f"evolve_q_{r}.npy")), oq)
            np.testing.assert_array_equal(np.load(os.path.join(d, f"evolve_p_{r}.npy")), op)
            sq, sp = np.load(os.path.join(d, f"sym_q_{r}.npy")), np.load(os.path.join(d, f"sym_p_{r}.npy"))
            assert np.abs(sq - oq).max() / np.abs(oq).max() <= 1e-13
            assert np.abs(sp - op).max() / np.abs(op).max() <= 1e-11
        np.testing.assert_array_equal(np.load(os.path.join(d, "sym_q_0.npy")), np.load(os.path.join(d, "sym_q_1.npy")))

        w = configs.c1()
        o = restate.match_momentum(Kernel(0, w.alpha, True), 0.0, w.q, w.target, w.h, w.epsilon, w.max_iter,
                                   "residual", "max", 1.0, w.steps)
        for r in range(2):
            it, conv, H, diag = open(os.path.join(d, f"match_{r}.txt")).read().split(" ", 3)
            assert int(it) == o["iterations"] == 36 and conv == "True" and diag == "None"
            assert float(H) == pytest.approx(o["hamiltonian"], rel=1e-10)
            p0 = np.load(os.path.join(d, f"match_p0_{r}.npy"))
            assert np.abs(p0 - o["p0"]).max() / np.abs(o["p0"]).max() <= 1e-8

        msgs = [open(os.path.join(d, f"err_{r}.txt")).read() for r in range(2)]
        assert msgs[0] == msgs[1]
        assert msgs[0].startswith("particles 200 and 290 coincide with interacting momenta")
        assert "(during step 1, t in [0, 0.2])" in msgs[0]
