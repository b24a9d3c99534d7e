"""Full-size parity of the timed and headline workloads against the C oracle.

The unmodified reference cannot run these sizes (~49 B of RAM per pair), so the checker is the C
restatement oracle/gs_oracle.c — itself pinned to the reference's golden vectors by
tests/test_oracle.py.  The fixtures were generated once by tests/golden/make_oracle_fixtures.py
(sampled rows of every array + scalar outcomes); nothing here reads /root/reference.

Tolerances (BASELINE.json north_star): states and momenta of solves and matches within 1e-8
relative (normwise over the sampled rows; the C2 100-step solve: q 1e-10, p 1e-9 as in
tests/test_gpu_parity.py::test_evolve_matches_reference), residual histories to 1e-8, identical
iteration counts and outcomes.  Divergent runs (the survey's feedback gains, which blow up) are
compared step by step up to the onset of the blow-up, and by outcome and iteration count after it.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = 1e-8


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def fixture(name):
    path = os.path.join(GOLDEN, f"oracle_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"fixture {name} not generated (tests/golden/make_oracle_fixtures.py)")
    z = np.load(path)
    return z, json.loads(str(z["meta"]))


class _Path:
    def __init__(self, path):
        self.path = path

    def __enter__(self):
        import paper_1510_03816_b200 as gs

        self.prev = gs.get_path()
        gs.set_path(self.path)

    def __exit__(self, *exc):
        import paper_1510_03816_b200 as gs

        gs.set_path(self.prev)


def _spec(gs, w):
    return gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha), sigma2=w.sigma2)


@pytest.mark.parametrize("path", ["dense", "cell"])
def test_c2_100_step_solve_matches_oracle(cuda, path):
    """The bench workload (C2, N = 16384, 100 RK4 steps, integrator.py:66-121) on both pair paths."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    z, meta = fixture(f"c2_solve_{path}")
    w = configs.c2()
    with _Path(path):
        out = gs.evolve(_spec(gs, w), gs.ParticleState(w.q, w.p), gs.EvolveConfig(t_final=1.0, steps=100))
    rows = z["rows"]
    assert rel(out.final.q[rows], z["q"]) <= 1e-10
    assert rel(out.final.p[rows], z["p"]) <= 1e-9


def test_c3_one_step_matches_oracle(cuda):
    """C3 (N = 131072, every pair within the support): one dense RK4 step of the 50-step solve."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    z, meta = fixture("c3_step")
    w = configs.c3()
    with _Path("dense"):
        out = gs.evolve(_spec(gs, w), gs.ParticleState(w.q, w.p),
                        gs.EvolveConfig(t_final=meta["t_final"], steps=meta["steps"]))
    rows = z["rows"]
    assert rel(out.final.q[rows], z["q"]) <= 1e-12
    assert rel(out.final.p[rows], z["p"]) <= 1e-10


def _match(gs, w, h, max_iter):
    from paper_1510_03816_b200 import device

    return device.match(_spec(gs, w), w.q, w.target, h, w.epsilon, max_iter, w.stop_rule, "max", w.t_final,
                        w.steps)


def _check_match(r, z, meta):
    assert r["iterations"] == meta["iterations"]
    assert r["converged"] == meta["converged"]
    assert (r["diagnosis"] or None) == meta["diagnosis"]
    np.testing.assert_allclose(np.array(r["residual_history"]), z["history"], rtol=TOL, atol=0)
    rows = z["rows"]
    assert rel(r["p0"].cpu().numpy()[rows], z["p0"]) <= TOL
    assert rel(r["endpoint"].cpu().numpy()[rows], z["endpoint"]) <= TOL


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_first_feedback_iterations_match_oracle(cuda, name):
    """C4 (N = 262144) / C5 (N = 2^20) at the configured gain: the first two iterations of the
    feedback loop (shooting.py:259-296) on the cell path."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    z, meta = fixture(f"{name.lower()}_match2")
    w = configs.CONFIGS[name]()
    assert meta["h"] == w.h
    with _Path("auto"):
        r = _match(gs, w, w.h, meta["max_iter"])
    _check_match(r, z, meta)


@pytest.mark.parametrize("name,n", [("C4", 32768), ("C5", 65536)])
def test_mid_size_whole_match_matches_oracle(cuda, name, n):
    """The whole match (C4 recipe: 100 iterations to the cap; C5: exactly 20 inexact iterations) at
    mid size, where the oracle runs every iteration: identical outcome and history, p0 and X(T)."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    z, meta = fixture(f"{name.lower()}_mid")
    w = configs.CONFIGS[name](n)
    with _Path("auto"):
        r = _match(gs, w, w.h, w.max_iter)
    _check_match(r, z, meta)
    assert r["hamiltonian"] == pytest.approx(meta["hamiltonian_dense"], rel=TOL)


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_matches_run_all_iterations(cuda, name):
    """At the configured gains C4 runs its 100 and C5 its 20 feedback iterations without a blow-up
    (configs.py C4_H / C5_H; the survey's gains blow up, test_survey_gains_blow_up_like_the_oracle)."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs

    w = configs.CONFIGS[name]()
    with _Path("auto"):
        r = _match(gs, w, w.h, w.max_iter)
    assert r["iterations"] == w.max_iter
    assert r["diagnosis"] == "iteration cap reached before the stopping rule"
    assert float(r["endpoint"].abs().max()) < 2.0  # the cloud stays in place (no flung-apart state)
    hist = np.array(r["residual_history"])
    assert np.all(np.isfinite(hist)) and hist[-1] < hist[0]


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_survey_gains_blow_up_like_the_oracle(cuda, name):
    """The survey's gains (C4 h = 0.1, C5 h = 0.4): the first shoot, step by step, equals the oracle's
    up to the onset of the blow-up, and the match ends as "step too large" after the same number of
    iterations (shooting.py:287-291).

    Compared steps: those whose sampled rows all stay near the unit square in the oracle (the
    fixture stores exactly these).  Steps before the onset (every particle still in place) are held
    to 1e-8; the onset step itself — where some particle is already flung away and rounding starts
    to be amplified without bound (C4: step 2, C5: step 1) — to 1e-6."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device

    z, meta = fixture(f"{name.lower()}_onset")
    w = configs.CONFIGS[name]()
    spec = _spec(gs, w)
    rows = z["rows"]
    q, p = w.q.copy(), meta["h"] * (w.target - w.q)
    assert meta["stored_steps"] >= 1
    with _Path("auto"):
        for k in range(meta["stored_steps"]):
            qd, pd, _ = device.evolve(spec, q, p, meta["dt"], 1)
            q, p = qd.cpu().numpy(), pd.cpu().numpy()
            tol = TOL if z["q_absmax"][k] < meta["in_place_bound"] else 1e-6
            assert rel(q[rows], z["q"][k]) <= tol, f"step {k + 1}"
            assert rel(p[rows], z["p"][k]) <= tol, f"step {k + 1}"
        r = _match(gs, w, meta["h"], w.max_iter)
    out = meta["outcome"]
    assert r["diagnosis"] == "step too large" and out["blown_up"]
    assert r["iterations"] == out["iterations"]
    if w.stop_rule == "momentum-delta":  # delta = h |r| is taken before each shoot: iteration 1 is exact
        np.testing.assert_allclose(r["residual_history"][0], out["history"][0], rtol=TOL)
