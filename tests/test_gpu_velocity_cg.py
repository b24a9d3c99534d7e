"""Velocity-space update above the persistent-kernel range: the reference solves
K p = u with a Cholesky factor of the dense Gram matrix (shooting.py:138-159, 263-265); the device
path never forms K (gs_gram_cg: conjugate gradients whose K v is the dq half of the RHS through the
pair kernels).  Pinned against the oracle's velocity matches (scipy Cholesky of the dense K,
tests/golden/make_oracle_fixtures.py vel_<n>): same iteration count and outcome, p0 / X(T) / H
within 1e-8."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = 1e-8


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("n", [600, 1024, 4096])
def test_velocity_match_matches_oracle_cholesky(cuda, n):
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, shooting

    z = np.load(os.path.join(GOLDEN, f"oracle_vel_{n}.npz"))
    m = json.loads(str(z["meta"]))
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=m["alpha"]))
    cfg = gs.ShootingConfig(h=m["h"], epsilon=m["epsilon"], max_iter=m["max_iter"], update_space="velocity",
                            evolve=gs.EvolveConfig(steps=m["steps"]), system=spec)
    a = gs.LandmarkTemplate(configs._circle(1.0, n), "circle")
    b = gs.LandmarkTemplate(configs._ellipse(*m["axes"], n), "ellipse")
    assert n > shooting.SMALL_MAX  # the matrix-free path
    res = gs.match(a, b, cfg)
    assert res.iterations == m["iterations"] and res.converged == m["converged"]
    assert (res.diagnosis or None) == m["diagnosis"]
    assert res.warnings == ()  # cond(K) ~ 1e2 << 1e12
    assert rel(res.p0, z["p0"]) <= TOL
    assert rel(res.final_template.points, z["endpoint"]) <= TOL
    assert res.hamiltonian == pytest.approx(m["hamiltonian"], rel=TOL)
    np.testing.assert_allclose(np.array(res.residual_history), z["history"], rtol=1e-6)


def test_cg_solution_reproduces_the_velocity_and_estimates_the_condition(cuda):
    """momenta_from_velocity at N = 4096 (shooting.py:162-175): K p = u to the CG tolerance (checked
    with the device velocity field, an independent dense kernel), cond(K) from the Lanczos
    coefficients close to the true one."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    n, sig = 1024, 1.0
    q0 = configs._circle(1.0, n)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=sig / gs.LAMBDA))
    u0 = np.random.default_rng(5).normal(0, 1, (n, 2))
    p = gs.momenta_from_velocity(spec.kernel, q0, u0)
    u = gs.velocity_field(spec, gs.ParticleState(q0, p), q0)
    assert rel(u, u0) <= 1e-12
    _, it, relres, coef = device.gram_cg(spec, q0, u0)
    assert relres <= 1e-14 and 0 < it < 2000
    K = device.gram(spec, q0).cpu().numpy()
    true = np.linalg.cond(K)
    est = device.lanczos_condition(coef)
    assert 0.5 * true <= est <= 1.0 + 1e-9 * true + true


def test_c4_size_velocity_solve_fits_in_memory(cuda):
    """At C4 size (N = 262144) the reference's Gram matrix would be 512 GB; the matrix-free solve
    runs through the cluster lists of q0 and converges."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    w = configs.c4()
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    u = w.h * (w.target - w.q)
    prev = gs.get_path()
    gs.set_path("auto")
    try:
        p, it, relres, coef = device.gram_cg(spec, w.q, u)
    finally:
        gs.set_path(prev)
    assert relres <= 1e-14 and it < 2000
    assert np.all(np.isfinite(p.cpu().numpy()))
    assert device.lanczos_condition(coef) < 1e12
