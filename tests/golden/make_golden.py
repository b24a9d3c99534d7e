"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-c2]

Every fixture records the reference's own outputs (``geoshoot.rhs``,
``geoshoot.evolve``, ``geoshoot.match``, ``geoshoot.hamiltonian``) on seeded
inputs, plus the independent sympy N=2 oracle of ``test_particles.py:22-71``.
The oracle restatement (oracle/) and the CUDA path are both checked against
these files; neither generated them.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import geoshoot as gs  # noqa: E402  (the reference package)

from paper_1510_03816_b200 import configs  # noqa: E402

LAM = configs.LAMBDA


def spec_of(family="conical", alpha=1.0, normalized=True, sigma2=0.0):
    return gs.SystemSpec(kernel=gs.KernelSpec(family=family, alpha=alpha, normalized=normalized),
                         sigma2=sigma2)


def kparams(spec):
    k = spec.kernel
    return np.array([0 if k.family.value == "conical" else 1, float(k.alpha),
                     1.0 if k.normalized else 0.0, float(spec.sigma2)])


def sympy_oracle():
    # same derivation as test_particles.py:22-49 (independent of the package)
    import sympy as sp
    qs = sp.symbols("q1x q1y q2x q2y", real=True)
    ps = sp.symbols("p1x p1y p2x p2y", real=True)
    s2, alpha = sp.symbols("s2 alpha", positive=True)
    q1x, q1y, q2x, q2y = qs
    p1x, p1y, p2x, p2y = ps
    d = sp.sqrt((q1x - q2x) ** 2 + (q1y - q2y) ** 2)
    kernel = sp.exp(-d / alpha)
    pp11 = p1x**2 + p1y**2
    pp22 = p2x**2 + p2y**2
    pp12 = p1x * p2x + p1y * p2y
    ham = sp.Rational(1, 2) * (pp11 + pp22 + 2 * pp12 * kernel) + s2 / 2 * (pp11 + pp22)
    dq = [sp.diff(ham, v) for v in ps]
    dp = [-sp.diff(ham, v) for v in qs]
    return sp.lambdify((qs, ps, s2, alpha), (dq, dp), "numpy")


def gen_sympy(out):
    oracle = sympy_oracle()
    rng = np.random.default_rng(2024)  # test_particles.py:54-61 recipe
    Q, P, S2, AL, DQ, DP, DQS, DPS = [], [], [], [], [], [], [], []
    for k in range(100):
        q = rng.uniform(-3.0, 3.0, size=(2, 2))
        while np.linalg.norm(q[0] - q[1]) < 1e-3:
            q = rng.uniform(-3.0, 3.0, size=(2, 2))
        p = rng.uniform(-2.0, 2.0, size=(2, 2))
        sigma2 = 0.0 if k % 2 == 0 else 0.3
        alpha = 1.0 if k % 3 else 0.7
        dq, dp = gs.rhs(spec_of(alpha=alpha, sigma2=sigma2), gs.ParticleState(q, p))
        wq, wp = oracle(tuple(q.ravel()), tuple(p.ravel()), sigma2, alpha)
        Q.append(q); P.append(p); S2.append(sigma2); AL.append(alpha)
        DQ.append(dq); DP.append(dp)
        DQS.append(np.asarray(wq, float).reshape(2, 2)); DPS.append(np.asarray(wp, float).reshape(2, 2))
    np.savez(os.path.join(out, "rhs_n2_sympy.npz"), q=np.array(Q), p=np.array(P),
             sigma2=np.array(S2), alpha=np.array(AL), dq=np.array(DQ), dp=np.array(DP),
             dq_sympy=np.array(DQS), dp_sympy=np.array(DPS))


def swirl(n=8, radius=2.0):
    # test_integrator.py:18-24
    pts = configs._circle(radius, n)
    t = np.arctan2(pts[:, 1], pts[:, 0])
    p = 0.8 * np.column_stack([-np.sin(t), np.cos(t)]) + 0.3 * np.column_stack([np.cos(2 * t), np.sin(2 * t)])
    return pts, p


def rhs_cases():
    cases = {}
    c1 = configs.c1()
    cases["c1_randp"] = (c1.q, np.random.default_rng(10).normal(size=(64, 2)), spec_of(alpha=c1.alpha))
    r = np.random.default_rng(11)
    q = r.normal(size=(9, 2)) * 2.0
    cases["n9_default"] = (q, r.normal(size=(9, 2)), spec_of())
    r = np.random.default_rng(20)
    q = r.uniform(0, 1, (1024, 2)); p = np.random.default_rng(21).normal(0, 0.1, (1024, 2))
    cases["u1024_cone_s005"] = (q, p, spec_of(alpha=0.05 / LAM))
    cases["u1024_cone_s05"] = (q, p, spec_of(alpha=0.5 / LAM))
    cases["u1024_cone_a1"] = (q, p, spec_of(alpha=1.0))
    cases["u1024_gauss"] = (q, p, spec_of(family="gaussian", alpha=0.1))
    cases["u1024_unnorm_s2"] = (q, p, spec_of(alpha=0.2, normalized=False, sigma2=0.3))
    cases["u1024_gauss_unnorm"] = (q, p, spec_of(family="gaussian", alpha=0.05, normalized=False, sigma2=0.1))
    q = np.random.default_rng(22).uniform(0, 1, (4096, 2)); p = np.random.default_rng(23).normal(0, 0.01, (4096, 2))
    cases["u4096_dense"] = (q, p, spec_of(alpha=2.0 / LAM))
    cases["coincident_inert"] = (np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 1.0]]),
                                 np.array([[1.0, 0.0], [0.0, 0.0], [0.0, 1.0]]), spec_of())
    sq, sp_ = swirl()
    cases["swirl8"] = (sq, sp_, spec_of())
    cases["n1"] = (np.array([[0.3, -0.2]]), np.array([[1.5, -2.0]]), spec_of(sigma2=0.25))
    return cases


def gen_rhs(out):
    arrays = {}
    for name, (q, p, spec) in rhs_cases().items():
        dq, dp = gs.rhs(spec, gs.ParticleState(q, p))
        h = gs.hamiltonian(spec, gs.ParticleState(q, p))
        arrays[f"{name}__q"] = q; arrays[f"{name}__p"] = p
        arrays[f"{name}__dq"] = dq; arrays[f"{name}__dp"] = dp
        arrays[f"{name}__kparams"] = kparams(spec)
        arrays[f"{name}__H"] = np.array(h)
    np.savez(os.path.join(out, "rhs_cases.npz"), **arrays)


def gen_c2(out):
    w = configs.c2()
    spec = spec_of(alpha=w.alpha)
    t0 = time.time()
    dq, dp = gs.rhs(spec, gs.ParticleState(w.q, w.p))
    dt = time.time() - t0
    np.savez_compressed(os.path.join(out, "rhs_c2.npz"), dq=dq, dp=dp, kparams=kparams(spec),
                        seconds=np.array(dt))
    print(f"C2 reference rhs: {dt:.1f} s")


def gen_evolve(out):
    arrays = {}
    cases = {}
    sq, sp_ = swirl()
    cases["swirl8_cone_100"] = (sq, sp_, spec_of(), 1.0, 100, 0)
    cases["swirl8_gauss_25"] = (sq, sp_, spec_of(family="gaussian"), 1.0, 25, 0)
    sq16, sp16 = swirl(16)
    cases["swirl16_cone_200"] = (sq16, sp16, spec_of(), 1.0, 200, 0)
    q10 = configs._circle(2.0, 10)
    p10 = 0.5 * np.random.default_rng(3).normal(size=(10, 2))
    cases["inexact10_200"] = (q10, p10, spec_of(sigma2=0.3), 1.0, 200, 0)
    c1 = configs.c1()
    cases["c1_p03_20"] = (c1.q, 0.3 * np.random.default_rng(30).normal(size=(64, 2)), spec_of(alpha=c1.alpha), 1.0, 20, 0)
    cases["capture_10_3"] = (sq, sp_, spec_of(), 0.5, 10, 3)
    q = np.random.default_rng(31).uniform(0, 1, (512, 2)); p = np.random.default_rng(32).normal(0, 0.05, (512, 2))
    cases["u512_cone_5"] = (q, p, spec_of(alpha=0.1 / LAM), 1.0, 5, 0)
    cases["u512_gauss_s2_5"] = (q, p, spec_of(family="gaussian", alpha=0.05, sigma2=0.2, normalized=False), 2.0, 5, 0)
    q = np.random.default_rng(33).uniform(0, 1, (4096, 2)); p = np.random.default_rng(34).normal(0, 0.01, (4096, 2))
    cases["u4096_1step"] = (q, p, spec_of(alpha=0.05 / LAM), 1.0, 1, 0)
    for name, (q, p, spec, tf, steps, cap) in cases.items():
        res = gs.evolve(spec, gs.ParticleState(q, p), gs.EvolveConfig(t_final=tf, steps=steps, capture_every=cap))
        arrays[f"{name}__q"] = q; arrays[f"{name}__p"] = p; arrays[f"{name}__kparams"] = kparams(spec)
        arrays[f"{name}__cfg"] = np.array([tf, steps, cap], dtype=float)
        arrays[f"{name}__qT"] = res.final.q; arrays[f"{name}__pT"] = res.final.p
        if cap:
            arrays[f"{name}__times"] = res.times
            arrays[f"{name}__frames_q"] = np.array([s.q for _, s in res.frames])
            arrays[f"{name}__frames_p"] = np.array([s.p for _, s in res.frames])
    np.savez(os.path.join(out, "evolve_cases.npz"), **arrays)


def match_cases():
    REF = gs.circle(1.0, n=8)
    TGT = gs.ellipse_rot_shift(1.3, 0.9, 0.0, (0.1, 0.0), n=8)

    def quick(**kw):  # test_shooting.py:37-41, momentum update (north_star)
        kw.setdefault("h", 0.5)
        kw.setdefault("epsilon", 1e-6)
        kw.setdefault("evolve", gs.EvolveConfig(steps=60))
        kw.setdefault("update_space", gs.UpdateSpace.MOMENTUM)
        return gs.ShootingConfig(**kw)

    c1 = configs.c1()
    c1cfg = gs.ShootingConfig(h=c1.h, epsilon=c1.epsilon, max_iter=c1.max_iter,
                              update_space="momentum", evolve=gs.EvolveConfig(t_final=1.0, steps=c1.steps),
                              system=spec_of(alpha=c1.alpha))
    cases = {
        "c1": (gs.LandmarkTemplate(c1.q, "X"), gs.LandmarkTemplate(c1.target, "Y"), c1cfg),
        "small_mom": (REF, TGT, quick(epsilon=1e-8)),
        "small_cap": (REF, TGT, quick(max_iter=2)),
        "small_mdelta": (REF, TGT, quick(stop_rule=gs.StopRule.MOMENTUM_DELTA)),
        "small_inexact": (REF, TGT, quick(h=0.4, stop_rule=gs.StopRule.MOMENTUM_DELTA, system=gs.SystemSpec(sigma2=0.3))),
        "small_l2": (REF, TGT, quick(norm=gs.ResidualNorm.L2)),
        "small_self": (REF, REF, quick()),
        "small_gauss": (REF, TGT, quick(h=0.3, system=spec_of(family="gaussian", alpha=0.5), evolve=gs.EvolveConfig(steps=30))),
        "blowup": (gs.circle(2.0, n=16), gs.heart4(n=16), quick(h=2.0, epsilon=1e-3)),
        "blowup_big": (gs.circle(2.0, n=16), gs.heart4(n=16), quick(h=60.0, epsilon=1e-3)),
        "blowup_inf": (gs.circle(2.0, n=16), gs.heart4(n=16), quick(h=1e160, epsilon=1e-3)),
        # velocity-space update (the reference default, shooting.py:80, 263-265)
        "vel_small": (REF, TGT, quick(epsilon=1e-8, update_space=gs.UpdateSpace.VELOCITY)),
        "vel_c1": (gs.LandmarkTemplate(c1.q, "X"), gs.LandmarkTemplate(c1.target, "Y"),
                   gs.ShootingConfig(h=c1.h, epsilon=c1.epsilon, max_iter=c1.max_iter, update_space="velocity",
                                     evolve=gs.EvolveConfig(t_final=1.0, steps=c1.steps),
                                     system=spec_of(alpha=c1.alpha))),
        "vel_inexact": (REF, TGT, quick(h=0.4, stop_rule=gs.StopRule.MOMENTUM_DELTA, system=gs.SystemSpec(sigma2=0.3),
                                        update_space=gs.UpdateSpace.VELOCITY)),
        "vel_heart": (gs.circle(2.0, n=16), gs.heart4(16), gs.ShootingConfig(h=0.4, max_iter=2000)),
        "vel_illcond": (gs.circle(1.0, n=8), gs.circle(1.1, n=8),
                        quick(epsilon=1e-2, max_iter=5, update_space=gs.UpdateSpace.VELOCITY,
                              system=spec_of(family="gaussian", alpha=20.0), evolve=gs.EvolveConfig(steps=20))),
        "circ256": (gs.circle(1.0, n=256), gs.ellipse_rot_shift(1.3, 0.7, 0.0, n=256),
                    gs.ShootingConfig(h=0.5, epsilon=1e-6, max_iter=300, update_space="momentum",
                                      evolve=gs.EvolveConfig(steps=20), system=spec_of(alpha=0.1 / LAM))),
    }
    return cases


def gen_match(out):
    arrays = {}
    meta = {}
    for name, (ref, tgt, cfg) in match_cases().items():
        t0 = time.time()
        res = gs.match(ref, tgt, cfg)
        dt = time.time() - t0
        arrays[f"{name}__ref"] = ref.points; arrays[f"{name}__tgt"] = tgt.points
        arrays[f"{name}__p0"] = res.p0; arrays[f"{name}__endpoint"] = res.final_template.points
        arrays[f"{name}__history"] = np.array(res.residual_history, dtype=float)
        k = cfg.system.kernel
        meta[name] = dict(
            ref_label=ref.label, tgt_label=tgt.label,
            family=k.family.value, alpha=k.alpha, normalized=k.normalized, sigma2=cfg.system.sigma2,
            h=cfg.h, epsilon=cfg.epsilon, max_iter=cfg.max_iter, update_space=cfg.update_space.value,
            stop_rule=cfg.stop_rule.value, norm=cfg.norm.value,
            t_final=cfg.evolve.t_final, steps=cfg.evolve.steps,
            iterations=res.iterations, converged=res.converged, hamiltonian=res.hamiltonian,
            final_residual=res.final_residual, diagnosis=res.diagnosis,
            final_label=res.final_template.label, seconds=dt, warnings=list(res.warnings),
        )
        print(f"match {name}: it={res.iterations} conv={res.converged} H={res.hamiltonian:.10g} "
              f"diag={res.diagnosis!r} ({dt:.2f}s)")
    np.savez(os.path.join(out, "match_cases.npz"), **arrays)
    with open(os.path.join(out, "match_cases.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def _cfg_meta(cfg):
    k = cfg.system.kernel
    return dict(family=k.family.value, alpha=k.alpha, normalized=k.normalized, sigma2=cfg.system.sigma2, h=cfg.h,
                epsilon=cfg.epsilon, max_iter=cfg.max_iter, update_space=cfg.update_space.value,
                stop_rule=cfg.stop_rule.value, norm=cfg.norm.value, t_final=cfg.evolve.t_final,
                steps=cfg.evolve.steps)


def _tpl(arrays, key, t):
    arrays[key] = t.points
    return dict(key=key, label=t.label)


def gen_analysis(out):
    """SURVEY.md §8(f2) callers: the reference's analysis.py / newton_match on the inputs of its
    own tests (test_analysis.py:31-33, 66-77, 139-153, 160-213; test_shooting.py:87-93;
    test_acceptance.py:196-240, 259-285, 327-340)."""
    arrays, meta = {}, {}
    REF = gs.circle(1.0, n=8)
    TGT = gs.ellipse_rot_shift(1.3, 0.9, 0.0, (0.1, 0.0), n=8)
    CFG = gs.ShootingConfig(h=0.5, epsilon=1e-6, evolve=gs.EvolveConfig(steps=60))
    axes = (0.2, 0.4, 0.6, 0.8, 1.0)
    sweeps = {
        "sweep_small": (REF, TGT, gs.SweepGrid(alpha2_values=(0.5, 1.0), h_values=(0.4, 0.8, 2.5), n_landmarks=8,
                                               tolerance=1e-3, max_iter=200)),
        "sweep_c16": (gs.circle(2.0, n=16), gs.heart4(16), gs.SweepGrid(axes, axes, n_landmarks=16, tolerance=1e-3)),
        "sweep_g32": (gs.circle(2.0, n=32), gs.heart4(32), gs.SweepGrid(axes, axes, n_landmarks=32,
                                                                        kernel_family="gaussian")),
        "sweep_c32": (gs.circle(2.0, n=32), gs.heart4(32), gs.SweepGrid(axes, axes, n_landmarks=32)),
    }
    for name, (a, b, grid) in sweeps.items():
        t0 = time.time()
        mat = gs.convergence_sweep(a, b, grid)
        dt = time.time() - t0
        meta[name] = dict(ref=_tpl(arrays, f"{name}__ref", a), tgt=_tpl(arrays, f"{name}__tgt", b),
                          alpha2=list(grid.alpha2_values), h=list(grid.h_values), n_landmarks=grid.n_landmarks,
                          family=grid.kernel_family.value, tolerance=grid.tolerance, max_iter=grid.max_iter,
                          matrix=mat.tolist(), seconds=dt)
        print(f"{name}: {mat.tolist()} ({dt:.1f}s)", flush=True)

    clusters = {
        "cluster_small": (REF, gs.circle(1.0, n=8, label="copy"),
                          [gs.circle(3.0, n=8, label="big"), gs.heart4(n=8, label="h")],
                          {"pair": 0.05, "ref_diff": 1.5}, CFG),
        "cluster_64": (gs.ellipse_rot_shift(4.0, 1.0, 0.0, (0.0, 0.0), 64, label="A"),
                       gs.ellipse_rot_shift(4.0, 1.05, 0.0, (0.0, 0.0), 64, label="B"),
                       [gs.circle(2.0, n=64, label="C"), gs.circle(3.0, n=64, label="D")],
                       {"pair": 0.05, "ref_diff": 1.0},
                       gs.ShootingConfig(h=0.3, epsilon=1e-3, max_iter=2000)),
    }
    for name, (a, b, refs, thr, cfg) in clusters.items():
        t0 = time.time()
        v = gs.cluster_test(a, b, refs, thr, cfg)
        dt = time.time() - t0
        meta[name] = dict(a=_tpl(arrays, f"{name}__a", a), b=_tpl(arrays, f"{name}__b", b),
                          refs=[_tpl(arrays, f"{name}__r{i}", r) for i, r in enumerate(refs)], thresholds=thr,
                          cfg=_cfg_meta(cfg), same_cluster=v.same_cluster,
                          evidence=[dict(reference_label=e.reference_label, target_label=e.target_label, H=e.H,
                                         iterations=e.iterations, converged=e.converged) for e in v.evidence],
                          seconds=dt)
        print(f"{name}: {v.same_cluster} {[round(e.H, 6) for e in v.evidence]} ({dt:.1f}s)", flush=True)

    newtons = {
        "newton_small": (REF, TGT, gs.ShootingConfig(h=1.0, epsilon=1e-8, evolve=gs.EvolveConfig(steps=60))),
        "newton_l2_30": (gs.circle(2.0, n=30), gs.standard_rotated_ellipse(4.0, 1.0, -math.pi / 4, (1.0, 0.0), 30),
                         gs.ShootingConfig(h=1.0, epsilon=1e-3, max_iter=2000, norm=gs.ResidualNorm.L2)),
        "newton_cap": (REF, TGT, gs.ShootingConfig(h=1.0, epsilon=1e-12, max_iter=2, evolve=gs.EvolveConfig(steps=60))),
    }
    for name, (a, b, cfg) in newtons.items():
        t0 = time.time()
        r = gs.newton_match(a, b, cfg)
        dt = time.time() - t0
        arrays[f"{name}__p0"] = r.p0
        arrays[f"{name}__endpoint"] = r.final_template.points
        arrays[f"{name}__history"] = np.array(r.residual_history, dtype=float)
        meta[name] = dict(ref=_tpl(arrays, f"{name}__ref", a), tgt=_tpl(arrays, f"{name}__tgt", b),
                          cfg=_cfg_meta(cfg), iterations=r.iterations, converged=r.converged,
                          hamiltonian=r.hamiltonian, final_residual=r.final_residual, diagnosis=r.diagnosis,
                          warnings=list(r.warnings), seconds=dt)
        print(f"{name}: it={r.iterations} conv={r.converged} H={r.hamiltonian:.12g} ({dt:.1f}s)", flush=True)

    t0 = time.time()
    rows = gs.exact_vs_inexact(REF, TGT, [0.0, 0.3], CFG, h_by_sigma2={0.3: 0.4})
    meta["exactness"] = dict(ref=_tpl(arrays, "exactness__ref", REF), tgt=_tpl(arrays, "exactness__tgt", TGT),
                             cfg=_cfg_meta(CFG), sigma2_values=[0.0, 0.3], h_by_sigma2={"0.3": 0.4},
                             rows=[dict(sigma2=r.sigma2, h=r.h, H=r.H, final_residual=r.final_residual,
                                        iterations=r.iterations, converged=r.converged) for r in rows],
                             seconds=time.time() - t0)

    full = gs.match(REF, TGT, CFG)
    half = gs.evolve(CFG.system, gs.ParticleState(REF.points, full.p0), gs.EvolveConfig(t_final=0.5, steps=50))
    partial = gs.LandmarkTemplate(half.final.q, "partial")
    pcfg = gs.ShootingConfig(h=0.5, epsilon=1e-6, evolve=gs.EvolveConfig(steps=50))
    pred = gs.predict(REF, partial, 0.5, 1.0, pcfg)
    arrays["predict__pred"] = pred.points
    meta["predict"] = dict(ref=_tpl(arrays, "predict__ref", REF), partial=_tpl(arrays, "predict__partial", partial),
                           t_match=0.5, t_predict=1.0, cfg=_cfg_meta(pcfg), label=pred.label)

    g = gs.PlanarIsometry(angle=math.pi / 3, translation=(0.5, 0.5), reflect_x=True)
    val = gs.iso_invariance_check(REF, TGT, g, CFG)
    meta["iso"] = dict(a=_tpl(arrays, "iso__a", REF), b=_tpl(arrays, "iso__b", TGT),
                       ga=_tpl(arrays, "iso__ga", g.apply(REF)), gb=_tpl(arrays, "iso__gb", g.apply(TGT)),
                       cfg=_cfg_meta(CFG), value=val)
    np.savez(os.path.join(out, "analysis_cases.npz"), **arrays)
    with open(os.path.join(out, "analysis_cases.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def gen_vfield(out):
    """particles.velocity_field (particles.py:140-150) on seeded states: at the landmarks,
    at random sample points, at a single point; conical and gaussian, normalized or not."""
    arrays, meta = {}, {}
    rng = np.random.default_rng(11)
    cases = {
        "landmarks10": (gs.circle(1.5, n=10).points, rng.normal(size=(10, 2)), None, spec_of()),
        "cloud_conical": (rng.uniform(0, 1, (1000, 2)), rng.normal(0, 0.1, (1000, 2)),
                          rng.uniform(-0.2, 1.2, (777, 2)), spec_of(alpha=0.05 / LAM)),
        "cloud_gauss": (rng.uniform(0, 1, (600, 2)), rng.normal(0, 0.1, (600, 2)),
                        rng.uniform(-0.2, 1.2, (300, 2)), spec_of(family="gaussian", alpha=0.07, normalized=False)),
        "single": (np.array([[0.0, 0.0], [1.0, 0.0]]), np.array([[0.0, 1.0], [1.0, 0.0]]),
                   np.array([[0.25, -0.5]]), spec_of()),
    }
    for name, (q, p, x, spec) in cases.items():
        x = q if x is None else x
        u = gs.velocity_field(spec, gs.ParticleState(q, p), x)
        arrays.update({f"{name}__q": q, f"{name}__p": p, f"{name}__x": x, f"{name}__u": u,
                       f"{name}__kparams": kparams(spec)})
    np.savez(os.path.join(out, "vfield_cases.npz"), **arrays)


def gen_errors(out):
    msgs = {}
    q = np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 1.0]])
    p = np.array([[1.0, 0.0], [1.0, 0.0], [0.0, 0.0]])
    try:
        gs.rhs(gs.SystemSpec(), gs.ParticleState(q, p))
    except gs.DegenerateConfigurationError as e:
        msgs["rhs_coincident"] = str(e)
    q = np.array([[0.0, 0.0], [0.0, 0.0], [2.0, 0.0]])
    p = np.array([[0.0, 1.0], [0.0, 1.0], [0.0, 0.0]])
    try:
        gs.evolve(gs.SystemSpec(), gs.ParticleState(q, p), gs.EvolveConfig(steps=10))
    except gs.DegenerateConfigurationError as e:
        msgs["evolve_coincident"] = str(e)
    q = np.array([[-0.5, 0.0], [0.5, 0.0]])
    p = np.array([[1e200, 0.0], [-1e200, 0.0]])
    try:
        gs.evolve(gs.SystemSpec(), gs.ParticleState(q, p), gs.EvolveConfig(steps=4))
    except gs.DivergenceError as e:
        msgs["evolve_divergence"] = str(e)
    # a later-step coincidence: two particles converge head-on
    q = np.array([[0.0, 0.0], [1.0, 0.0], [5.0, 5.0], [1.0, 0.0]])
    p = np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 0.0], [0.0, 0.0]])
    try:
        gs.rhs(gs.SystemSpec(), gs.ParticleState(q, p))
        msgs["rhs_coincident_zero_p"] = "ok"
    except gs.DegenerateConfigurationError as e:
        msgs["rhs_coincident_zero_p"] = str(e)
    q = np.array([[0.0, 0.0], [1.0, 0.0], [5.0, 5.0], [1.0, 0.0], [0.0, 0.0]])
    p = np.array([[1.0, 0.0], [0.0, 2.0], [1.0, 0.0], [0.0, 1.0], [3.0, 0.0]])
    try:
        gs.rhs(gs.SystemSpec(), gs.ParticleState(q, p))
    except gs.DegenerateConfigurationError as e:
        msgs["rhs_coincident_two_groups"] = str(e)
    try:
        gs.LandmarkTemplate(np.array([[0.0, 0.0], [1.0, 2.0], [3.0, 3.0], [1.0, 2.0]]), "dup")
    except gs.DegenerateConfigurationError as e:
        msgs["template_dup"] = str(e)
    with open(os.path.join(out, "errors.json"), "w") as f:
        json.dump(msgs, f, indent=1, sort_keys=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c2", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    out = HERE
    steps = {"sympy": gen_sympy, "rhs": gen_rhs, "evolve": gen_evolve, "match": gen_match,
             "errors": gen_errors, "c2": gen_c2, "analysis": gen_analysis, "vfield": gen_vfield}
    for name, fn in steps.items():
        if a.only and name not in a.only.split(","):
            continue
        if name == "c2" and a.skip_c2:
            continue
        t0 = time.time()
        fn(out)
        print(f"[{name}] {time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(out, "PROVENANCE.json"), "w") as f:
        json.dump({"reference": "/root/reference/pkg/src/geoshoot", "version": gs.__version__,
                   "numpy": np.__version__, "generator": "tests/golden/make_golden.py"}, f, indent=1)


if __name__ == "__main__":
    main()
