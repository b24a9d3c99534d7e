"""Host-side logic of the drop-in (no GPU): validation, error messages, templates, configs, rebinding."""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1510_03816_b200 as gs
from paper_1510_03816_b200 import _native as N
from paper_1510_03816_b200 import configs, device, shapes
from paper_1510_03816_b200.integrator import frame_times

REF_SRC = "/root/reference/pkg/src"
have_reference = os.path.isdir(REF_SRC)


def _reference():
    import sys

    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import geoshoot

    return geoshoot


def test_status_messages_match_reference_wording():
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        msgs = json.load(f)
    e = device.status_exception(N.Status(N.GS_ERR_COINCIDENT, 0, 0, 1, 0, 2))
    assert isinstance(e, gs.DegenerateConfigurationError) and str(e) == msgs["rhs_coincident"]
    e = device.status_exception(N.Status(N.GS_ERR_COINCIDENT, 1, 0, 1, 0, 0), 1.0, 10)
    assert str(e) == msgs["evolve_coincident"]
    e = device.status_exception(N.Status(N.GS_ERR_NONFINITE_STAGE, 1, -1, -1, 0, 1), 1.0, 4)
    assert isinstance(e, gs.DivergenceError) and str(e) == msgs["evolve_divergence"]
    e = device.status_exception(N.Status(N.GS_ERR_NONFINITE_STATE, 3, -1, -1, 0, 7), 1.0, 60)
    assert str(e) == ("non-finite state at step 3 (t = 0.05); the step size is too large for this configuration")
    assert device.status_exception(N.Status(N.GS_OK, 0, -1, -1, 0, 0)) is None


def test_frame_times_follow_the_reference_grid():
    from conftest import cases

    c = cases("evolve_cases.npz")["capture_10_3"]
    tf, steps, cap = c["cfg"]
    np.testing.assert_array_equal(frame_times(tf, int(steps), int(cap)), c["times"])
    assert device.n_frames(100, 7) == 2 + 100 // 7
    assert device.n_frames(10, 1) == 11 and device.n_frames(10, 0) == 0


def test_first_coincident_pair_is_row_major_first():
    rng = np.random.default_rng(0)
    for trial in range(200):
        n = int(rng.integers(2, 40))
        pts = rng.integers(0, 6, (n, 2)).astype(float)  # many duplicates
        d = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
        np.fill_diagonal(d, np.inf)
        want = tuple(int(v) for v in np.argwhere(d == 0.0)[0]) if np.any(d == 0.0) else None
        assert shapes.first_coincident_pair(pts) == want
    pts = np.array([[0.0, 0.0], [1.0, 2.0], [3.0, 3.0], [1.0, 2.0]])
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        msgs = json.load(f)
    with pytest.raises(gs.DegenerateConfigurationError) as e:
        gs.LandmarkTemplate(pts, "dup")
    assert str(e.value) == msgs["template_dup"]
    pts = np.array([[0.0, 0.0], [-0.0, 0.0]])  # signed zeros coincide
    assert shapes.first_coincident_pair(pts) == (0, 1)


def test_first_coincident_pair_includes_underflowing_distances():
    """The reference rejects distinct points whose squared difference underflows (distance 0.0)."""
    rng = np.random.default_rng(1)
    for scale in (1e-170, 1e-161, 1e-200, 1e-300):
        for trial in range(60):
            n = int(rng.integers(2, 40))
            pts = rng.integers(0, 5, (n, 2)).astype(float) * scale + rng.integers(0, 3, (n, 1))
            d = np.sqrt(np.sum((pts[:, None, :] - pts[None, :, :]) ** 2, axis=-1))
            np.fill_diagonal(d, np.inf)
            want = tuple(int(v) for v in np.argwhere(d == 0.0)[0]) if np.any(d == 0.0) else None
            assert shapes.first_coincident_pair(pts) == want, scale
    pts = np.array([[0.5, 0.5], [0.5 + 2.0 ** -600 * 0.0, 0.5], [1e-170, 0.0], [0.0, 2e-170]])
    assert shapes.first_coincident_pair(pts) == (0, 1)
    assert shapes.first_coincident_pair(pts[2:]) == (0, 1)  # distinct, distance underflows to 0


def test_large_template_check_is_fast():
    import time

    w = configs.c5()
    t0 = time.perf_counter()
    gs.LandmarkTemplate(w.q, "X")
    assert time.perf_counter() - t0 < 10.0


def test_config_validation_matches_reference():
    with pytest.raises(gs.ConfigurationError, match="MomentumDelta"):
        gs.ShootingConfig(h=0.3, system=gs.SystemSpec(sigma2=0.1))
    for bad in (dict(h=0.0), dict(h=-1.0), dict(h=float("inf"))):
        with pytest.raises(gs.ConfigurationError):
            gs.ShootingConfig(**bad)
    with pytest.raises(gs.ConfigurationError):
        gs.ShootingConfig(h=0.5, epsilon=0.0)
    with pytest.raises(gs.ConfigurationError):
        gs.ShootingConfig(h=0.5, max_iter=0)
    cfg = gs.ShootingConfig(h=0.5, update_space="momentum", stop_rule="momentum-delta", norm="l2")
    assert cfg.update_space is gs.UpdateSpace.MOMENTUM and cfg.norm is gs.ResidualNorm.L2
    for bad in (dict(t_final=0.0), dict(steps=0), dict(capture_every=-1)):
        with pytest.raises(gs.ConfigurationError):
            gs.EvolveConfig(**bad)
    with pytest.raises(gs.ConfigurationError):
        gs.SystemSpec(sigma2=-0.1)
    with pytest.raises(ValueError):
        gs.ParticleState(np.zeros((3, 3)), np.zeros((3, 2)))
    bad = np.zeros((3, 2))
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        gs.ParticleState(bad, np.zeros((3, 2)))


def test_system_struct_and_kd1_support_radius():
    s = device.system_struct(gs.SystemSpec(kernel=gs.KernelSpec(alpha=0.05 / gs.LAMBDA), sigma2=0.1))
    assert s.family == N.GS_FAMILY_CONICAL and s.normalized == 1 and s.cutoff == pytest.approx(0.05)
    assert np.exp(-s.cutoff / s.alpha) == pytest.approx(2.0**-53, rel=1e-12)
    g = device.system_struct(gs.SystemSpec(kernel=gs.KernelSpec(family="gaussian", alpha=0.1, normalized=False)))
    assert g.family == N.GS_FAMILY_GAUSSIAN and g.normalized == 0
    assert np.exp(-0.5 * (g.cutoff / 0.1) ** 2) == pytest.approx(2.0**-53, rel=1e-12)
    with pytest.raises(gs.ConfigurationError, match="not available"):
        device.system_struct(gs.SystemSpec(kernel=gs.KernelSpec(family="bessel", nu=2.0)))


def test_configs_are_deterministic_and_follow_the_recipes():
    a, b = configs.c4(1000), configs.c4(1000)
    np.testing.assert_array_equal(a.q, b.q)
    np.testing.assert_array_equal(a.target, b.target)
    w = configs.c5(4096)
    assert w.sigma2 == 0.1 and w.h == configs.C5_H and w.max_iter == 20 and w.epsilon == 1e-300
    assert np.abs(w.target - w.q).max() < 0.5


@pytest.mark.skipif(not have_reference, reason="reference package not mounted")
def test_config1_templates_equal_the_reference_generators():
    ref = _reference()
    w = configs.c1()
    np.testing.assert_array_equal(w.q, ref.circle(1.0, n=64).points)
    np.testing.assert_array_equal(w.target, ref.ellipse_rot_shift(1.3, 0.7, 0.0, (0.0, 0.0), 64).points)
    np.testing.assert_array_equal(gs.circle(1.0, n=8).points, ref.circle(1.0, n=8).points)
    np.testing.assert_array_equal(gs.ellipse_rot_shift(1.3, 0.9, 0.4, (0.1, 0.0), n=8).points,
                                  ref.ellipse_rot_shift(1.3, 0.9, 0.4, (0.1, 0.0), n=8).points)


@pytest.mark.skipif(not have_reference, reason="reference package not mounted")
def test_dropin_rebinds_every_alias_and_restores():
    import torch

    from paper_1510_03816_b200 import dropin, integrator, particles, types

    import importlib

    ref = _reference()
    importlib.import_module("geoshoot.cli")
    originals = {(m, f): getattr(getattr(ref, m), f) for m, f in [
        ("particles", "rhs"), ("integrator", "rhs"), ("integrator", "evolve"), ("shooting", "evolve"),
        ("analysis", "evolve"), ("cli", "evolve"), ("shooting", "match"), ("analysis", "match"), ("cli", "match"),
        ("particles", "hamiltonian"), ("shooting", "hamiltonian"), ("shooting", "newton_match"),
        ("analysis", "convergence_sweep"), ("cli", "convergence_sweep"), ("analysis", "cluster_test"),
        ("cli", "cluster_test"), ("analysis", "exact_vs_inexact"), ("analysis", "predict")]}
    dropin.install(ref)

    def dev(f):  # the device function behind a rebound name (bessel calls go to the shadowed original)
        return getattr(f, "device", f)

    try:
        assert ref.integrator.rhs is ref.particles.rhs is ref.rhs and dev(ref.rhs) is particles.rhs
        assert ref.rhs.original is originals[("particles", "rhs")]
        for m in ("integrator", "shooting", "analysis", "cli"):
            assert dev(getattr(ref, m).evolve) is integrator.evolve
        assert ref.shooting.match is ref.analysis.match is ref.cli.match is ref.match
        assert dev(ref.shooting.hamiltonian) is particles.hamiltonian
        assert gs.errors.DivergenceError is ref.DivergenceError
        assert types.get("EvolveResult") is ref.EvolveResult
        assert types.get("DistanceRecord") is ref.DistanceRecord
        assert ref.shooting.newton_match is ref.newton_match and dev(ref.newton_match) is gs.newton_match
        assert ref.particles.velocity_field is ref.velocity_field and dev(ref.velocity_field) is gs.velocity_field
        for f in ("convergence_sweep", "cluster_test", "exact_vs_inexact", "predict", "shape_distance"):
            assert getattr(ref.analysis, f) is getattr(ref.cli, f) is getattr(ref, f)
            assert dev(getattr(ref, f)) is getattr(gs, f)
        # the reference's own template class, with the O(N log N) duplicate check
        big = np.random.default_rng(0).uniform(0, 1, (200000, 2))
        assert ref.LandmarkTemplate(big, "big").n == 200000
        dup = np.array([[0.0, 0.0], [1.0, 2.0], [3.0, 3.0], [1.0, 2.0], [0.0, 0.0]])
        with pytest.raises(ref.DegenerateConfigurationError, match=r"landmarks 0 and 4 coincide in template 'dup'"):
            ref.LandmarkTemplate(dup, "dup")
        grid = ref.SweepGrid((0.5,), (0.4,), n_landmarks=8)
        with pytest.raises(ref.ConfigurationError, match="thresholds"):  # reference error classes
            ref.cluster_test(ref.circle(1.0, n=8), ref.circle(1.2, n=8), [ref.circle(2.0, n=8)] * 2,
                             {"pair": -1, "ref_diff": 1}, ref.ShootingConfig(h=0.5))
        assert grid.n_landmarks == 8
        if not torch.cuda.is_available():
            st = ref.ParticleState(np.zeros((3, 2)), np.zeros((3, 2)))
            with pytest.raises(N.NativeUnavailable):
                ref.rhs(ref.SystemSpec(), st)  # no CPU fallback behind the drop-in
            with pytest.raises(N.NativeUnavailable):
                ref.integrator.evolve(ref.SystemSpec(), st)
        # a family the device does not provide stays on the reference's own function
        bes = ref.SystemSpec(kernel=ref.KernelSpec(family="bessel", nu=2.5, alpha=0.7))
        rng = np.random.default_rng(3)
        st2 = ref.ParticleState(rng.uniform(0, 1, (6, 2)), rng.normal(0, 0.1, (6, 2)))
        got = ref.rhs(bes, st2)
        want = originals[("particles", "rhs")](bes, st2)
        assert all(np.array_equal(a, b) for a, b in zip(got, want))
        cfg = ref.ShootingConfig(system=bes, h=0.5, max_iter=3, evolve=ref.EvolveConfig(steps=4))
        res = ref.match(ref.circle(1.0, n=6), ref.circle(1.1, n=6), cfg)  # bessel match, reference path
        assert res.iterations >= 1 and np.all(np.isfinite(res.p0))
    finally:
        dropin.uninstall()
    for (m, f), fn in originals.items():
        assert getattr(getattr(ref, m), f) is fn
    assert gs.errors.DivergenceError is not ref.DivergenceError
    assert types.get("EvolveResult") is integrator.EvolveResult


# --- analysis host logic; no device calls -------------------------------------
def test_sweep_grid_validation_mirrors_reference():
    import paper_1510_03816_b200 as gs

    g = gs.SweepGrid((0.5, 1), (0.1,), n_landmarks=8, kernel_family="gaussian")
    assert g.alpha2_values == (0.5, 1.0) and g.kernel_family is gs.KernelFamily.GAUSSIAN
    for bad in (dict(alpha2_values=(), h_values=(0.1,)), dict(alpha2_values=(0.5, -1.0), h_values=(0.1,)),
                dict(alpha2_values=(0.5,), h_values=(0.1,), tolerance=0.0),
                dict(alpha2_values=(0.5,), h_values=(0.1,), n_landmarks=2),
                dict(alpha2_values=(0.5,), h_values=(math.inf,)), dict(alpha2_values=(0.5,), h_values=(0.1,),
                                                                         max_iter=0)):
        with pytest.raises(gs.ConfigurationError):
            gs.SweepGrid(**bad)


def test_cluster_and_newton_validate_before_any_device_work():
    import paper_1510_03816_b200 as gs

    a, b = gs.circle(1.0, n=8), gs.circle(1.1, n=8)
    cfg = gs.ShootingConfig(h=0.5)
    with pytest.raises(gs.ConfigurationError, match="at least 2"):
        gs.cluster_test(a, b, [a], {"pair": 1, "ref_diff": 1}, cfg)
    with pytest.raises(gs.ConfigurationError, match="missing"):
        gs.cluster_test(a, b, [a, b], {"pair": 1}, cfg)
    with pytest.raises(gs.ConfigurationError, match="positive"):
        gs.cluster_test(a, b, [a, b], {"pair": 0, "ref_diff": 1}, cfg)
    with pytest.raises(gs.ConfigurationError, match="TargetResidual"):
        gs.newton_match(a, b, gs.ShootingConfig(h=0.5, stop_rule="momentum-delta"))
    with pytest.raises(gs.ConfigurationError, match="equal landmark counts"):
        gs.newton_match(a, gs.circle(1.0, n=9), cfg)
    with pytest.raises(gs.ConfigurationError, match="t_match"):
        gs.predict(a, b, 0.0, 0.5, cfg)
    with pytest.raises(gs.ConfigurationError, match="t_predict"):
        gs.predict(a, b, 0.5, 0.4, cfg)


@pytest.mark.skipif(not have_reference, reason="reference package not mounted")
def test_cli_front_end_runs_the_reference_cli_with_gpu_facts(tmp_path):
    """the reference's CLI through the drop-in; manifests gain "b200"."""
    from paper_1510_03816_b200 import cli, dropin

    _reference()
    out = tmp_path / "c.json"
    assert cli.main(["shapes", "circle", "--n", "8", "--out", str(out)]) == 0
    man = json.loads(out.with_suffix(".manifest.json").read_text())
    assert man["schema"] == "geoshoot.manifest/1"
    facts = man["extras"]["b200"]
    assert facts["abi"] == 2 and facts["library"].startswith("geoshoot-b200")
    assert not dropin.installed()
    import torch

    if not torch.cuda.is_available():  # the compute commands fail loudly without a device
        res = tmp_path / "r"
        with pytest.raises(N.NativeUnavailable):
            cli.main(["match", str(out), str(out), "--h", "0.3", "--out", str(res)])


def test_input_validation_matches_reference():
    """Malformed inputs (empty, ragged, wrong shape, non-finite, mismatched, bad configs,
    duplicate landmarks) raise the reference's exception types with its messages
    (tests/golden/validation.json, made by tests/golden/make_validation.py from the reference)."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_validation import outcomes

    want = json.load(open(os.path.join(GOLDEN, "validation.json")))
    got = outcomes(gs)
    assert got == want
