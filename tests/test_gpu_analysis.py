"""Batched independent trajectories against the reference's golden outputs.

Fixtures: tests/golden/analysis_cases.* written by make_golden.py from the reference's
convergence_sweep / cluster_test / newton_match / exact_vs_inexact / predict /
iso_invariance_check on the inputs of its own tests.  Iteration counts and verdicts are
integers and must agree exactly; momenta and H within the match tolerance of
test_gpu_parity.py.  The batched launch must also be bitwise identical to the same matches
run one at a time (same kernel code per CTA).
"""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, cases

pytestmark = pytest.mark.gpu

MATCH_TOL = 1e-8

with open(os.path.join(GOLDEN, "analysis_cases.json")) as _f:
    META = json.load(_f)
ARR = cases("analysis_cases.npz")


def _arr(key):
    name, fld = key.split("__", 1)
    return ARR[name][fld]


def _tpl(gs, d):
    return gs.LandmarkTemplate(_arr(d["key"]), d["label"])


def _cfg(gs, m):
    spec = gs.SystemSpec(kernel=gs.KernelSpec(family=m["family"], alpha=m["alpha"], normalized=m["normalized"]),
                         sigma2=m["sigma2"])
    return gs.ShootingConfig(h=m["h"], epsilon=m["epsilon"], max_iter=m["max_iter"], update_space=m["update_space"],
                             stop_rule=m["stop_rule"], norm=m["norm"],
                             evolve=gs.EvolveConfig(t_final=m["t_final"], steps=m["steps"]), system=spec)


@pytest.mark.parametrize("name", sorted(k for k in META if k.startswith("sweep_")))
def test_convergence_sweep_matches_reference(cuda, name):
    import paper_1510_03816_b200 as gs

    m = META[name]
    grid = gs.SweepGrid(m["alpha2"], m["h"], n_landmarks=m["n_landmarks"], kernel_family=m["family"],
                        tolerance=m["tolerance"], max_iter=m["max_iter"])
    mat = gs.convergence_sweep(_tpl(gs, m["ref"]), _tpl(gs, m["tgt"]), grid)
    assert mat.dtype.kind == "i" and mat.shape == (len(m["alpha2"]), len(m["h"]))
    np.testing.assert_array_equal(mat, np.array(m["matrix"]))


@pytest.mark.parametrize("name", sorted(k for k in META if k.startswith("cluster_")))
def test_cluster_test_matches_reference(cuda, name):
    import paper_1510_03816_b200 as gs

    m = META[name]
    v = gs.cluster_test(_tpl(gs, m["a"]), _tpl(gs, m["b"]), [_tpl(gs, r) for r in m["refs"]], m["thresholds"],
                        _cfg(gs, m["cfg"]))
    assert v.same_cluster == m["same_cluster"]
    assert len(v.evidence) == len(m["evidence"])
    for got, want in zip(v.evidence, m["evidence"]):
        assert got.reference_label == want["reference_label"] and got.target_label == want["target_label"]
        assert got.iterations == want["iterations"] and got.converged == want["converged"]
        assert got.H == pytest.approx(want["H"], rel=MATCH_TOL, abs=1e-12)


@pytest.mark.parametrize("name", sorted(k for k in META if k.startswith("newton_")))
def test_newton_match_matches_reference(cuda, name):
    import paper_1510_03816_b200 as gs

    m = META[name]
    r = gs.newton_match(_tpl(gs, m["ref"]), _tpl(gs, m["tgt"]), _cfg(gs, m["cfg"]))
    assert r.iterations == m["iterations"] and r.converged == m["converged"]
    assert r.diagnosis == m["diagnosis"]
    assert bool(r.warnings) == bool(m["warnings"])
    p_ref = ARR[name]["p0"]
    # the finite-difference Jacobian carries ~sqrt(eps) relative error; the converged root does not
    tol = 1e-6 if m["converged"] else 1e-5
    assert np.abs(r.p0 - p_ref).max() / np.abs(p_ref).max() <= tol
    assert r.hamiltonian == pytest.approx(m["hamiltonian"], rel=tol)
    np.testing.assert_allclose(np.array(r.residual_history), ARR[name]["history"], rtol=1e-3, atol=1e-10)


def test_newton_rejects_momentum_delta_rule(cuda):
    import paper_1510_03816_b200 as gs

    m = META["newton_small"]
    cfg = _cfg(gs, dict(m["cfg"], stop_rule="momentum-delta"))
    with pytest.raises(gs.ConfigurationError, match="TargetResidual"):
        gs.newton_match(_tpl(gs, m["ref"]), _tpl(gs, m["tgt"]), cfg)


def test_exact_vs_inexact_matches_reference(cuda):
    import paper_1510_03816_b200 as gs

    m = META["exactness"]
    rows = gs.exact_vs_inexact(_tpl(gs, m["ref"]), _tpl(gs, m["tgt"]), m["sigma2_values"], _cfg(gs, m["cfg"]),
                               h_by_sigma2={float(k): v for k, v in m["h_by_sigma2"].items()})
    assert len(rows) == len(m["rows"])
    for got, want in zip(rows, m["rows"]):
        assert (got.sigma2, got.h, got.iterations, got.converged) == (want["sigma2"], want["h"], want["iterations"],
                                                                      want["converged"])
        assert got.H == pytest.approx(want["H"], rel=MATCH_TOL)
        assert got.final_residual == pytest.approx(want["final_residual"], rel=1e-6, abs=1e-12)
    with pytest.raises(gs.ConfigurationError, match="sigma2"):
        gs.exact_vs_inexact(_tpl(gs, m["ref"]), _tpl(gs, m["tgt"]), [-0.1], _cfg(gs, m["cfg"]))


def test_predict_matches_reference(cuda):
    import paper_1510_03816_b200 as gs

    m = META["predict"]
    pred = gs.predict(_tpl(gs, m["ref"]), _tpl(gs, m["partial"]), m["t_match"], m["t_predict"], _cfg(gs, m["cfg"]))
    assert pred.label == m["label"]
    np.testing.assert_allclose(pred.points, ARR["predict"]["pred"], rtol=0, atol=1e-8)
    with pytest.raises(gs.ConfigurationError, match="t_match"):
        gs.predict(_tpl(gs, m["ref"]), _tpl(gs, m["partial"]), 1.0, 1.0, _cfg(gs, m["cfg"]))


def test_iso_invariance_check_matches_reference(cuda):
    import paper_1510_03816_b200 as gs

    m = META["iso"]
    a, b = _tpl(gs, m["a"]), _tpl(gs, m["b"])
    ga, gb = _tpl(gs, m["ga"]), _tpl(gs, m["gb"])

    class Iso:  # the reference's PlanarIsometry, replayed from its recorded images
        def apply(self, t):
            return ga if t is a else gb

    val = gs.iso_invariance_check(a, b, Iso(), _cfg(gs, m["cfg"]))
    assert abs(val) <= 1e-12 and abs(m["value"]) <= 1e-12


def test_batch_is_bitwise_identical_to_single_matches(cuda):
    """One CTA per item runs the single-match kernel's code: a batch changes nothing."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import device, shooting

    m = META["cluster_small"]
    cfg = _cfg(gs, m["cfg"])
    pairs = [(_tpl(gs, m["a"]), _tpl(gs, m["b"]))] + [(_tpl(gs, r), _tpl(gs, m["a"])) for r in m["refs"]]
    for space in ("velocity", "momentum"):
        c = gs.ShootingConfig(h=cfg.h, epsilon=cfg.epsilon, max_iter=cfg.max_iter, update_space=space,
                              evolve=cfg.evolve, system=cfg.system)
        batched = gs.analysis.match_many(pairs, [c] * len(pairs))
        for (x, y), rb in zip(pairs, batched):
            rs = gs.match(x, y, c)
            assert rb.iterations == rs.iterations
            np.testing.assert_array_equal(rb.p0, rs.p0)
            np.testing.assert_array_equal(rb.final_template.points, rs.final_template.points)
            assert rb.residual_history == rs.residual_history
            assert rb.hamiltonian == rs.hamiltonian
    # momentum batch == device.match one by one
    q = np.stack([x.points for x, _ in pairs])
    t = np.stack([y.points for _, y in pairs])
    d = shooting.match_config_dict(cfg)
    rb = device.match_batch([cfg.system] * len(pairs), [dict(d, max_iter=40)] * len(pairs), q, t)
    for k in range(len(pairs)):
        rs = device.match(cfg.system, q[k], t[k], cfg.h, cfg.epsilon, 40, d["stop_rule"], d["norm"], d["t_final"],
                          d["steps"])
        assert rb[k]["iterations"] == rs["iterations"]
        assert bool((rb[k]["p0"] == rs["p0"]).all())


def test_evolve_batch_matches_single_evolves_and_reports_failures(cuda):
    import torch

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import device

    rng = np.random.default_rng(3)
    n, B = 24, 6
    q0 = gs.circle(1.0, n=n).points
    P = rng.normal(scale=0.3, size=(B, n, 2))
    P[4] *= 1e200  # this column diverges
    spec = gs.SystemSpec()
    q, p, errs = device.evolve_batch(spec, q0, torch.from_numpy(P), 1.0, 30)
    for b in range(B):
        if b == 4:
            assert isinstance(errs[b], gs.DivergenceError)
            continue
        assert errs[b] is None
        qs, ps, _ = device.evolve(spec, q0, P[b], 1.0, 30)
        assert bool((q[b] == qs).all()) and bool((p[b] == ps).all())


def test_velocity_match_on_device_solves_gram_system(cuda):
    """The in-kernel Cholesky solve reproduces K^-1 u: p0 of a velocity match satisfies K p0 = u
    with u = h * (sum of residuals) — checked through momenta_from_velocity's round trip."""
    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import shooting

    ref = gs.circle(2.0, n=16)
    rng = np.random.default_rng(7)
    u0 = rng.normal(size=(16, 2))
    p = shooting.momenta_from_velocity(gs.KernelSpec(), ref.points, u0)
    K = shooting.device.gram(gs.SystemSpec(), ref.points).cpu().numpy()
    assert np.abs(K @ p - u0).max() < 1e-10
    assert math.isfinite(float(np.abs(p).max()))
