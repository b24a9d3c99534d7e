"""CPU stand-in for libgs_b200's gs_slab_* (test infrastructure, include/geoshoot_b200.h contract).

Same calls and tensors as paper_1510_03816_b200.slab.DeviceSlabBackend, on CPU torch tensors, so
the product's SlabSolver orchestration (ownership plan, migration all-to-all, halo slices,
rebuild flags, final gather) runs over gloo / LocalComm in the CPU suite.  The arithmetic is a
plain restatement: truncated RHS (pairs with d < cutoff, particles.py:109-117 under KD-1) summed
left to right in local order (np.cumsum: non-neighbours add an exact 0), the RK4 stage epilogue
of csrc/gs_dense.cu stage_update, and the grid / skin rules of csrc/gs_cell.cu / gs_api.cu.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from paper_1510_03816_b200 import _native as N


def cell_cap(n: int) -> int:
    cap = 16384
    while cap < n // 16:
        cap <<= 1
    return cap


class NumpySlabBackend:
    def __init__(self, fam: str, alpha: float, normalized: bool, sigma2: float, cutoff: float, skin=None):
        self.fam, self.alpha, self.sigma2, self.cutoff = fam, float(alpha), float(sigma2), float(cutoff)
        self.peak = 1.0 if normalized else 1.0 / (2.0 * math.pi * alpha * alpha)
        self.skin_opt = skin

    # -- per build ------------------------------------------------------------------------------
    def begin(self, n_glob, q, p, g):
        self.n_glob = int(n_glob)
        self.skin = self.skin_opt if self.skin_opt is not None else (0.1 if n_glob < 131072 else 0.05)
        self.rl = self.cutoff * (1.0 + self.skin)
        self.Su = torch.cat([q, p], dim=1).double().clone()
        self.Bu = self.Su.clone()
        self.Au = torch.zeros_like(self.Su)
        self.gu = g.to(torch.int32).clone()
        self.sorted = False
        self.fail = None

    def _own(self):
        if self.sorted:
            r = self.rows_
            return (self.S[r.own_begin:r.own_begin + r.n_own], self.B, self.A, self.g[r.own_begin:r.own_begin + r.n_own])
        return self.Su, self.Bu, self.Au, self.gu

    def bbox(self):
        S = self._own()[0]
        if S.shape[0] == 0:
            return torch.full((4,), math.inf, dtype=torch.float64)
        return torch.tensor([S[:, 0].min(), S[:, 1].min(), -S[:, 0].max(), -S[:, 1].max()], dtype=torch.float64)

    def grid(self, b4):
        mnx, mny, mxx, mxy = float(b4[0]), float(b4[1]), -float(b4[2]), -float(b4[3])
        cap = cell_cap(self.n_glob)
        sub = 2
        while sub > 1:
            h = self.rl / sub
            if (math.floor((mxx - mnx) / h) + 1) * (math.floor((mxy - mny) / h) + 1) <= cap:
                break
            sub -= 1
        h = self.rl / sub
        nx, ny = int(math.floor((mxx - mnx) / h) + 1), int(math.floor((mxy - mny) / h) + 1)
        self.g_ = N.SlabGrid(mnx, mny, h, nx, ny, sub, int(nx * ny > cap))
        self.inv_h = 1.0 / h
        return self.g_

    def _cells(self, S):
        g = self.g_
        cy = np.clip(np.floor((S[:, 1].numpy() - g.y0) * self.inv_h).astype(np.int64), 0, g.ny - 1)
        cx = np.clip(np.floor((S[:, 0].numpy() - g.x0) * self.inv_h).astype(np.int64), 0, g.nx - 1)
        return cy, cx

    def rows(self, ny):
        cy, _ = self._cells(self._own()[0])
        return torch.from_numpy(np.bincount(cy, minlength=ny).astype(np.int64))

    def pack(self, owner, world):
        S, B, A, g = self._own()
        cy, _ = self._cells(S)
        dest = owner.numpy()[cy]
        order = np.argsort(dest, kind="stable")
        send = torch.cat([S, B, A, g.double()[:, None]], dim=1)[torch.from_numpy(order)]
        return send.contiguous()

    def unpack(self, recv):
        self.Su, self.Bu, self.Au = recv[:, 0:4].clone(), recv[:, 4:8].clone(), recv[:, 8:12].clone()
        self.gu = recv[:, 12].to(torch.int32)
        self.sorted = False

    def layout(self, r):
        cy, cx = self._cells(self.Su)
        key = (cy - r.own0) * self.g_.nx + cx
        order = torch.from_numpy(np.lexsort((self.gu.numpy(), key)))
        self.S = torch.zeros((r.n_loc + 1, 4), dtype=torch.float64)
        self.S[r.n_loc] = torch.tensor([1e150, 1e150, 0.0, 0.0])
        self.g = torch.zeros(r.n_loc, dtype=torch.int32)
        self.S[r.own_begin:r.own_begin + r.n_own] = self.Su[order]
        self.g[r.own_begin:r.own_begin + r.n_own] = self.gu[order]
        self.B, self.A = self.Bu[order].clone(), self.Au[order].clone()
        self.flag = torch.zeros(1, dtype=torch.int32)
        self.rows_ = r
        self.sorted = True

    def lists(self, ncl):
        r = self.rows_
        self.Xb = self.S[r.own_begin:r.own_begin + r.n_own, 0:2].clone()

    # -- per stage ------------------------------------------------------------------------------
    def stage(self, step, s, dt):
        r = self.rows_
        if r.n_own == 0:
            self.flag.zero_()
            return
        L = self.S[:r.n_loc].numpy()
        own = L[r.own_begin:r.own_begin + r.n_own]
        dx = own[:, None, 0] - L[None, :, 0]
        dy = own[:, None, 1] - L[None, :, 1]
        d = np.sqrt(dx * dx + dy * dy)
        mask = d < self.cutoff
        if self.fam == "conical":
            G = self.peak * np.exp(-d / self.alpha)
            with np.errstate(divide="ignore", invalid="ignore"):
                c = np.where(d > 0, G / (self.alpha * d), 0.0)
        else:
            G = self.peak * np.exp(-d * d / (2.0 * self.alpha ** 2))
            c = G / self.alpha ** 2
        pdot = own[:, None, 2] * L[None, :, 2] + own[:, None, 3] * L[None, :, 3]
        c = np.where(mask, pdot * c, 0.0)
        G = np.where(mask, G, 0.0)

        def seq(x):  # left-to-right sum in local order
            return np.cumsum(x, axis=1)[:, -1]

        k = np.stack([seq(G * L[None, :, 2]), seq(G * L[None, :, 3]), seq(c * dx), seq(c * dy)], axis=1)
        k[:, 0] += self.sigma2 * own[:, 2]
        k[:, 1] += self.sigma2 * own[:, 3]
        B, A = self.B.numpy(), self.A.numpy()
        if s == 0:
            acc = k
        else:
            acc = A + (1.0 if s == 3 else 2.0) * k
        if s < 3:
            nxt = B + ((dt if s == 2 else 0.5 * dt) * k)
            A[:] = acc
        else:
            nxt = B + (dt / 6.0) * acc
            B[:] = nxt
        self.S[r.own_begin:r.own_begin + r.n_own] = torch.from_numpy(nxt)
        thr = 0.5 * self.skin * self.cutoff
        moved = ((nxt[:, 0:2] - self.Xb.numpy()) ** 2).sum(axis=1) > thr * thr * (1.0 - 1e-9)
        self.flag.fill_(int(moved.any()))

    def own(self):
        r = self.rows_
        return self.S[r.own_begin:r.own_begin + r.n_own], self.g[r.own_begin:r.own_begin + r.n_own]

    def status(self):
        return N.Status()


def direct_truncated_evolve(fam, alpha, normalized, sigma2, cutoff, q, p, t_final, steps):
    """Plain RK4 (integrator.py:95-114) of the truncated RHS over all particles (the check)."""
    peak = 1.0 if normalized else 1.0 / (2.0 * math.pi * alpha * alpha)

    def rhs(q, p):
        dx = q[:, None, 0] - q[None, :, 0]
        dy = q[:, None, 1] - q[None, :, 1]
        d = np.sqrt(dx * dx + dy * dy)
        m = d < cutoff
        if fam == "conical":
            G = peak * np.exp(-d / alpha)
            with np.errstate(divide="ignore", invalid="ignore"):
                c = np.where(d > 0, G / (alpha * d), 0.0)
        else:
            G = peak * np.exp(-d * d / (2 * alpha * alpha))
            c = G / alpha ** 2
        G = np.where(m, G, 0.0)
        c = np.where(m, c * (p @ p.T), 0.0)
        dq = G @ p + sigma2 * p
        dp = np.stack([(c * dx).sum(1), (c * dy).sum(1)], axis=1)
        return dq, dp

    dt = t_final / steps
    q, p = q.copy(), p.copy()
    for _ in range(steps):
        k1 = rhs(q, p)
        k2 = rhs(q + 0.5 * dt * k1[0], p + 0.5 * dt * k1[1])
        k3 = rhs(q + 0.5 * dt * k2[0], p + 0.5 * dt * k2[1])
        k4 = rhs(q + dt * k3[0], p + dt * k3[1])
        q = q + dt / 6 * (k1[0] + 2 * k2[0] + 2 * k3[0] + k4[0])
        p = p + dt / 6 * (k1[1] + 2 * k2[1] + 2 * k3[1] + k4[1])
    return q, p
