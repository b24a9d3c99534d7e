"""The cluster Verlet lists of the cell path (gs_verlet.cu) against the per-RHS cell sweep and the
C oracle: same pairs (d < cutoff), so the same sums up to summation order — for evolves that reuse
a list over many RHS, rebuild it when particles move, outgrow the list buffer, or hit a
coincident interacting pair (particles.py:92-98, integrator.py:102-105)."""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


class _Env:
    """A fresh library context created under the given environment (read at gs_create)."""

    def __init__(self, **env):
        self.env = env

    def __enter__(self):
        from paper_1510_03816_b200 import _native as N

        self.N = N
        self.saved = {k: os.environ.get(k) for k in self.env}
        os.environ.update({k: str(v) for k, v in self.env.items()})
        self.ctxs = N.Context.swap()
        return N

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        self.N.Context.swap(self.ctxs)


def _stats(N):
    ctx = N.Context.get()
    b, e = ctypes.c_int64(), ctypes.c_int64()
    N.check(ctx.lib.gs_cell_stats(ctx.handle, ctypes.byref(b), ctypes.byref(e), None), "gs_cell_stats")
    return b.value, e.value


def _evolve(gs, spec, q, p, steps, **env):
    from paper_1510_03816_b200 import device

    with _Env(**env) as N:
        gs.set_path("cell")
        try:
            out = gs.evolve(spec, gs.ParticleState(q, p), gs.EvolveConfig(t_final=steps / 20, steps=steps))
            st = _stats(N)
        finally:
            gs.set_path("auto")
    return out.final.q, out.final.p, st


def test_lists_equal_the_cell_sweep_and_rebuild_when_particles_move(cuda):
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    w = configs.c5(65536)
    p = 0.05 * (w.target - w.q)  # large enough that the 8-step shoot moves particles past half the skin
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    qv, pv, (builds, cap) = _evolve(gs, spec, w.q, p, 8)
    qs, ps, _ = _evolve(gs, spec, w.q, p, 8, GS_B200_VERLET=0)
    assert rel(qv, qs) <= TOL and rel(pv, ps) <= TOL
    assert builds >= 3  # sizing build + forced first build + at least one displacement rebuild
    assert cap > 0


def test_lists_match_the_oracle_on_the_clustered_cloud(cuda):
    import paper_1510_03816_b200 as gs
    from oracle import native
    from oracle.restate import Kernel
    from paper_1510_03816_b200 import configs

    w = configs.c4(20000)
    p = np.random.default_rng(9).normal(0, 1e-3, w.q.shape)
    for spec in (gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha)),
                 gs.SystemSpec(kernel=gs.KernelSpec(family="gaussian", alpha=0.004), sigma2=0.1)):
        qv, pv, _ = _evolve(gs, spec, w.q, p, 3)
        k = Kernel(0 if spec.kernel.family.value == "conical" else 1, spec.kernel.alpha, True)
        oq, op = native.evolve(k, spec.sigma2, w.q, p, 3 / 20, 3, cutoff=gs.support_radius(spec.kernel))
        assert rel(qv, oq) <= 1e-10 and rel(pv, op) <= 1e-10


def test_list_buffer_overflow_is_redone_with_a_larger_buffer(cuda):
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    w = configs.c5(32768)
    p = 0.05 * (w.target - w.q)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    qa, pa, (b_ok, _) = _evolve(gs, spec, w.q, p, 4)
    # a buffer sized at 30 % of the first build overflows on the first in-graph build
    qb, pb, (b_small, _) = _evolve(gs, spec, w.q, p, 4, GS_B200_VERLET_SLACK=-0.7)
    assert np.array_equal(qa, qb) and np.array_equal(pa, pb)  # the redo is the same computation
    assert b_small > b_ok


def test_coincident_interacting_pair_through_the_lists(cuda):
    import paper_1510_03816_b200 as gs

    rng = np.random.default_rng(4)
    n = 20000
    q = rng.uniform(0, 1, (n, 2))
    q[17001] = q[256]
    p = rng.normal(0, 0.01, (n, 2))
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.02 / gs.LAMBDA))
    with pytest.raises(gs.DegenerateConfigurationError,
                       match=r"particles 256 and 17001 coincide with interacting momenta.*during step 1"):
        _evolve(gs, spec, q, p, 2)
    p[17001] = 0.0  # an inert coincident pair is fine (particles.py:92-98: p_i . p_j == 0)
    qv, pv, _ = _evolve(gs, spec, q, p, 2)
    qs, ps, _ = _evolve(gs, spec, q, p, 2, GS_B200_VERLET=0)
    assert rel(qv, qs) <= TOL and rel(pv, ps) <= TOL


def test_fused_epilogue_equals_the_separate_epilogue(cuda):
    """Below GS_B200_VERLET_FUSE_MAX_N the list sweep carries the RK4 stage epilogue and the sorted
    records ping-pong between two buffers; the arithmetic is k_finish_verlet's, so the evolve is
    bitwise the one with the separate epilogue, rebuilds included — also after a larger cloud left
    a stale record in the second buffer (the lists' sentinel slot)."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    w = configs.c5(65536)
    p = 0.05 * (w.target - w.q)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    for n in (65536, 20000):
        q0, p0 = w.q[:n], p[:n]
        qf, pf, (bf, _) = _evolve(gs, spec, q0, p0, 6)
        qs, ps, (bs, _) = _evolve(gs, spec, q0, p0, 6, GS_B200_VERLET_FUSE_MAX_N=0, GS_B200_VERLET_REL=0)
        assert np.array_equal(qf, qs) and np.array_equal(pf, ps), n
        assert bf == bs and bf >= 3


def test_relative_displacement_trigger_rebuilds_less_and_keeps_the_sums(cuda):
    """Large clouds (the separate list epilogue) rebuild on the neighbours' relative displacement
    (coarse-cell displacement boxes, gs_verlet.cu k_verlet_trigger) instead of any particle moving
    half the skin: a smooth flow rebuilds less often, and the evolve agrees with the blanket rule and
    with the per-RHS cell sweep to rounding."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    w = configs.c4(20000)
    rng = np.random.default_rng(3)
    x = w.q
    p = 0.02 * np.column_stack([np.sin(2 * np.pi * x[:, 1]), np.cos(2 * np.pi * x[:, 0])])  # smooth
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    kw = dict(GS_B200_VERLET_FUSE_MAX_N=0)
    qr, pr, (br, _) = _evolve(gs, spec, x, p, 8, GS_B200_VERLET_REL=1, **kw)
    qb, pb, (bb, _) = _evolve(gs, spec, x, p, 8, GS_B200_VERLET_REL=0, **kw)
    qs, ps, _ = _evolve(gs, spec, x, p, 8, GS_B200_VERLET=0)
    assert bb >= 4 and br < bb, (br, bb)
    # a stiff clustered flow: three summation orders agree to the rounding its 8 steps amplify
    assert rel(qr, qs) <= 1e-10 and rel(pr, ps) <= 1e-10
    assert rel(qb, qs) <= 1e-10 and rel(pb, ps) <= 1e-10


def test_adaptive_skin_follows_the_rebuild_rate_and_keeps_the_sums(cuda):
    """The relative-trigger path adapts the list skin to the observed rebuild interval
    (gs_verlet.cu verlet_skin_adapt): the rebuild schedule departs from the fixed default's (here a
    rebuild every ~9 RHS: the skin narrows and lists are rebuilt more often, each one shorter), the
    sums agree with the per-RHS cell sweep to rounding, and every call starts from the default
    skin (two calls on one context are bitwise equal)."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    w = configs.c5(30000)
    rng = np.random.default_rng(11)
    p = 0.003 * (w.target - w.q) + 1e-3 * rng.standard_normal(w.q.shape)  # noisy
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)
    kw = dict(GS_B200_VERLET_FUSE_MAX_N=0, GS_B200_VERLET_REL=1)
    qa, pa, (ba, _) = _evolve(gs, spec, w.q, p, 20, **kw)
    qf, pf, (bf, _) = _evolve(gs, spec, w.q, p, 20, GS_B200_SKIN_ADAPT=0, **kw)
    qs, ps, _ = _evolve(gs, spec, w.q, p, 20, GS_B200_VERLET=0)
    assert bf >= 8 and ba > bf, (ba, bf)
    assert rel(qa, qs) <= 1e-10 and rel(pa, ps) <= 1e-10
    assert rel(qf, qs) <= 1e-10 and rel(pf, ps) <= 1e-10
    with _Env(**kw):
        device.set_path("cell")
        try:
            q_d = device.as_device(w.q, __import__("torch"))
            p_d = device.as_device(p, __import__("torch"))
            r1 = device.evolve(spec, q_d, p_d, 1.0, 20)
            r2 = device.evolve(spec, q_d, p_d, 1.0, 20)
        finally:
            device.set_path("auto")
    assert bool((r1[0] == r2[0]).all()) and bool((r1[1] == r2[1]).all())
