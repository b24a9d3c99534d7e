"""Seeded randomized parity sweep: many small configurations (size, family, normalisation,
sigma2, clustering, momentum scale, pair-sum path) through the C ABI against the numpy
C restatement (oracle/gs_oracle.c: the reference's formulas with the direct-difference dp, pinned
to the reference's golden vectors in tests/test_oracle.py).  Tolerance: BASELINE's per-RHS 1e-10
normwise for dq and dp."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RHS_TOL = 1e-10
SEEDS = list(range(64))


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 2, 3, 7, 31, 64, 65, 127, 255, 512, 513, 1000, 1024, 1500, 2048, 3001]))
    fam = int(rng.integers(0, 2))
    normalized = bool(rng.integers(0, 2))
    sigma2 = float(rng.choice([0.0, 0.0, 0.1, 1.3]))
    if rng.random() < 0.3:  # clustered
        c = rng.uniform(0, 1, (4, 2))
        q = c[rng.integers(0, 4, n)] + rng.normal(0, 0.02, (n, 2))
    else:
        q = rng.uniform(-1, 1, (n, 2)) * rng.choice([0.1, 1.0, 10.0])
    extent = float(np.ptp(q)) if n > 1 else 1.0
    alpha = float(extent * rng.choice([0.001, 0.01, 0.1, 1.0]) + 1e-3)
    p = rng.normal(0, float(rng.choice([1e-3, 1.0, 100.0])), (n, 2))
    path = str(rng.choice(["auto", "dense", "cell"]))
    return n, fam, normalized, sigma2, alpha, q, p, path


@pytest.mark.parametrize("seed", SEEDS)
def test_random_rhs_and_hamiltonian_match_restatement(cuda, seed):
    import paper_1510_03816_b200 as gs
    from oracle import native
    from oracle.restate import Kernel

    n, fam, normalized, sigma2, alpha, q, p, path = _case(seed)
    family = "conical" if fam == 0 else "gaussian"
    spec = gs.SystemSpec(kernel=gs.KernelSpec(family=family, alpha=alpha, normalized=normalized), sigma2=sigma2)
    k = Kernel(fam, alpha, normalized)
    gs.set_path(path)
    try:
        dq, dp = gs.rhs(spec, gs.ParticleState(q, p))
        H = gs.hamiltonian(spec, gs.ParticleState(q, p))
    finally:
        gs.set_path("auto")
    # dense semantics (all pairs) or the cell list's KD-1 truncation at the support radius (pairs
    # with G < 2^-53 dropped): "cell" is held to the truncated sum, "auto" to whichever it chose
    refs = []
    if path != "cell":
        refs.append(native.rhs(k, sigma2, q, p))
    if path != "dense":
        refs.append(native.rhs(k, sigma2, q, p, cutoff=gs.support_radius(spec.kernel)))

    def close(oq, op):
        # G below 2^-1020 (the subnormal range) is flushed to zero on the device: only a dp made
        # entirely of such terms (every pair > ~707 alpha apart) differs, by < 1e-290 absolute
        return rel(dq, oq) <= RHS_TOL and np.abs(dp - op).max() <= RHS_TOL * np.abs(op).max() + 1e-290

    assert any(close(oq, op) for oq, op in refs), (n, family, path)
    assert H == pytest.approx(native.hamiltonian(k, q, p), rel=1e-10)


@pytest.mark.parametrize("seed", SEEDS[:16])
def test_random_short_evolves_match_restatement(cuda, seed):
    import paper_1510_03816_b200 as gs
    from oracle import native
    from oracle.restate import Kernel

    n, fam, normalized, sigma2, alpha, q, p, path = _case(seed)
    p = p / max(1.0, np.abs(p).max()) * 0.05  # a gentle flow: the comparison measures rounding only
    family = "conical" if fam == 0 else "gaussian"
    spec = gs.SystemSpec(kernel=gs.KernelSpec(family=family, alpha=alpha, normalized=normalized), sigma2=sigma2)
    gs.set_path(path)
    try:
        r = gs.evolve(spec, gs.ParticleState(q, p), gs.EvolveConfig(t_final=0.5, steps=5))
    finally:
        gs.set_path("auto")
    oq, op = native.evolve(Kernel(fam, alpha, normalized), sigma2, q, p, 0.5, 5)
    assert rel(r.final.q, oq) <= 1e-10
    assert np.abs(r.final.p - op).max() <= 1e-9 * max(np.abs(op).max(), 1e-300) + 1e-14
