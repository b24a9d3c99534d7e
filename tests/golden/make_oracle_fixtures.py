"""Full-size parity fixtures from the C oracle (oracle/gs_oracle.c) — run once in the build container.

    python tests/golden/make_oracle_fixtures.py [--only NAME,...] [--threads T]

The unmodified reference cannot run these sizes (it needs ~49 B of RAM per pair: SURVEY.md §0.6),
so the checker here is the C restatement, itself pinned to the reference's golden vectors by
tests/test_oracle.py.  Each fixture stores sampled rows (every `stride`-th particle) plus scalar
outcomes; the `-m gpu` tests in tests/test_gpu_fullsize.py compare the device path with them.

Fixtures (tests/golden/oracle_<name>.npz):
  c2_solve_dense  C2 (N = 16384) 100-step RK4 solve, all pairs          (integrator.py:66-121)
  c2_solve_cell   the same solve, pairs within the support radius (KD-1 truncation)
  c3_step         C3 (N = 131072) one RK4 step (4 dense RHS), dt = 1/50
  c4_onset        C4 first shoot at the survey's h = 0.1, step by step (all 20 steps), and the
                  match outcome it implies (iteration 1 blows up: shooting.py:287-291)
  c5_onset        C5 first shoot at the survey's h = 0.4 (sigma2 = 0.1), step by step, plus the
                  second shoot of the match (iteration 2 blows up)
  c4_match2       C4 at the configured h: the first 2 feedback iterations (max_iter = 2)
  c5_match2       C5 at the configured h: the first 2 feedback iterations
  c4_mid          C4 recipe at N = 32768: the whole 100-iteration match at the configured h
  c5_mid          C5 recipe at N = 65536: the whole 20-iteration match at the configured h
  vel_<n>         velocity-space matches (UpdateSpace.VELOCITY, shooting.py:138-159, 263-265) above the
                  persistent-kernel range, N = 600 / 1024 / 4096, circle -> ellipse (converging cases), dense oracle
                  evolve and scipy's Cholesky of the Gram matrix (the reference's own method)
The feedback loop below restates shooting.py:218-301 (momentum branch, :266-267) exactly as
oracle/restate.py does, with the oracle's truncated evolve and the exact zero-momentum shoot
(p = 0 gives dq = dp = 0, so the endpoint is q0 bitwise).
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
sys.path.insert(0, REPO)

from oracle import native  # noqa: E402
from oracle.restate import BLOWUP_FACTOR, Kernel, OracleDegenerate, OracleDivergence, norm  # noqa: E402
from paper_1510_03816_b200 import configs  # noqa: E402

ONSET_H = {"C4": 0.1, "C5": 0.4}  # the survey's proposals, which blow up


def kern(w):
    return Kernel(0, w.alpha, True)


def oracle_match(w, h, max_iter, cutoff, log=None):
    """shooting.py:218-301, momentum update, truncated oracle evolve.  Returns the MatchResult fields
    (without H) plus the per-iteration wall time."""
    k = kern(w)
    q0, target = w.q, w.target

    def ev(p):
        if not np.any(p):
            return q0.copy()  # exact: zero momenta leave q unchanged
        return native.evolve(k, w.sigma2, q0, p, w.t_final, w.steps, cutoff=cutoff)[0]

    p = np.zeros_like(q0)
    endpoint = ev(p)
    residual = target - endpoint
    history = []
    initial = None
    diagnosis = "iteration cap reached before the stopping rule"
    converged = False
    if w.stop_rule == "residual":
        initial = norm("max", residual)
    for it in range(max_iter):
        delta = h * norm("max", residual)
        p = p + h * residual
        t0 = time.perf_counter()
        try:
            endpoint_new = ev(p)
        except (OracleDivergence, OracleDegenerate) as exc:
            diagnosis = f"step too large ({exc})"
            break
        endpoint = endpoint_new
        residual = target - endpoint
        value = norm("max", residual) if w.stop_rule == "residual" else delta
        if initial is None:
            initial = value
        history.append(value)
        if log:
            log(f"  iteration {it + 1}: value {value:.6e} ({time.perf_counter() - t0:.1f} s)")
        if not math.isfinite(value) or (initial > 0 and value > BLOWUP_FACTOR * initial):
            diagnosis = "step too large"
            break
        if value < w.epsilon:
            diagnosis, converged = None, True
            break
    return dict(p0=p, endpoint=endpoint, history=np.array(history), iterations=len(history), converged=converged,
                diagnosis=diagnosis, final_residual=norm("max", target - endpoint))


def save(name, meta, **arrays):
    path = os.path.join(HERE, f"oracle_{name}.npz")
    np.savez_compressed(path, meta=json.dumps(meta), **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)", flush=True)


def solve_fixture(name, w, steps, t_final, cutoff, stride):
    t0 = time.perf_counter()
    q, p = native.evolve(kern(w), w.sigma2, w.q, w.p, t_final, steps, cutoff=cutoff)
    rows = np.arange(0, w.n, stride)
    save(name, dict(config=w.name, n=w.n, steps=steps, t_final=t_final, cutoff=cutoff, stride=stride,
                    seconds=time.perf_counter() - t0, threads=native.max_threads()),
         rows=rows, q=q[rows], p=p[rows], q_absmax=np.abs(q).max(), p_absmax=np.abs(p).max())


def onset_fixture(name, w, h, stride):
    """The first shoot p = h (Y - X), one RK4 step at a time (autonomous RHS: chaining 1-step evolves
    of dt = T/steps is the same arithmetic as the steps-step evolve), then the match outcome of the
    survey's h (shooting.py:259-301): for the residual rule iteration 1's value is |Y - X(T)|; for
    the momentum-delta rule iteration 2 shoots p + h (Y - X(T)) and its value is h |Y - X(T)|."""
    k = kern(w)
    dt = w.t_final / w.steps
    q, p = w.q.copy(), h * (w.target - w.q)
    rows = np.arange(0, w.n, stride)
    qs, ps, qmax, pmax, secs = [], [], [], [], []
    failed = None
    for step in range(1, w.steps + 1):
        t0 = time.perf_counter()
        try:
            q, p = native.evolve(k, w.sigma2, q, p, dt, 1, cutoff=w.sigma)
        except (OracleDivergence, OracleDegenerate) as exc:
            failed = f"step {step}: {exc}"
            break
        secs.append(time.perf_counter() - t0)
        qmax.append(float(np.abs(q).max()))
        pmax.append(float(np.abs(p).max()))
        qs.append(q[rows])
        ps.append(p[rows])
        print(f"  {name} step {step}: max|q| {qmax[-1]:.3e} max|p| {pmax[-1]:.3e} ({secs[-1]:.1f} s)", flush=True)
    r0 = norm("max", w.target - w.q)
    outcome = {}
    if failed is None:
        r1 = norm("max", w.target - q)
        if w.stop_rule == "residual":
            hist = [r1]
        else:
            hist = [h * r0]
            p2 = h * (w.target - w.q) + h * (w.target - q)
            try:
                native.evolve(k, w.sigma2, w.q, p2, w.t_final, w.steps, cutoff=w.sigma)
                hist.append(h * r1)
            except (OracleDivergence, OracleDegenerate) as exc:
                outcome["second_shoot_failed"] = str(exc)
        blown = len(hist) > 0 and (not math.isfinite(hist[-1]) or hist[-1] > BLOWUP_FACTOR * hist[0]) \
            if w.stop_rule != "residual" else not (hist[0] <= BLOWUP_FACTOR * r0)
        outcome.update(iterations=len(hist), history=hist, blown_up=bool(blown))
    # rows are stored for the steps whose sampled rows all stay near the unit square (the test compares
    # those); q_absmax / p_absmax (over all particles) are kept for every step
    bound = 1.5 * float(np.abs(w.q).max())
    keep = 0
    while keep < len(qs) and np.abs(qs[keep]).max() < bound:
        keep += 1
    save(name, dict(config=w.name, n=w.n, h=h, dt=dt, stride=stride, failed=failed, seconds=float(sum(secs)),
                    threads=native.max_threads(), outcome=outcome, stored_steps=keep, in_place_bound=bound),
         rows=rows, q=np.array(qs[:keep]), p=np.array(ps[:keep]), q_absmax=np.array(qmax), p_absmax=np.array(pmax))


def match_fixture(name, w, h, max_iter, stride, with_h=False):
    t0 = time.perf_counter()
    r = oracle_match(w, h, max_iter, w.sigma, log=print)
    rows = np.arange(0, w.n, stride)
    meta = dict(config=w.name, n=w.n, h=h, max_iter=max_iter, stop_rule=w.stop_rule, epsilon=w.epsilon,
                sigma2=w.sigma2, stride=stride, iterations=r["iterations"], converged=r["converged"],
                diagnosis=r["diagnosis"], final_residual=r["final_residual"], seconds=time.perf_counter() - t0,
                threads=native.max_threads())
    if with_h:
        meta["hamiltonian_dense"] = native.hamiltonian(kern(w), w.q, r["p0"])
    save(name, meta, rows=rows, p0=r["p0"][rows], endpoint=r["endpoint"][rows], history=r["history"])


# (N, support radius, ellipse axes): converging velocity-space matches (larger deformations or the
# narrowest kernels blow up, which would only pin an amplified rounding race)
VEL_CASES = ((600, 2.0, 1.1, 0.9), (1024, 1.0, 1.1, 0.9), (4096, 0.2, 1.05, 0.95))


def vel_fixture(n, sig, ax, ay):
    from oracle import restate

    q0 = configs._circle(1.0, n)
    y = configs._ellipse(ax, ay, n)
    k = Kernel(0, sig / configs.LAMBDA, True)
    t0 = time.perf_counter()
    ev = lambda qq, pp: q0.copy() if not np.any(pp) else native.evolve(k, 0.0, qq, pp, 1.0, 20)[0]  # noqa: E731
    r = restate.match_momentum(k, 0.0, q0, y, 0.5, 1e-6, 100, "residual", "max", 1.0, 20, evolve_fn=ev,
                               update_space="velocity")
    meta = dict(n=n, sigma=sig, alpha=k.alpha, axes=[ax, ay], h=0.5, epsilon=1e-6, max_iter=100, steps=20,
                iterations=r["iterations"], converged=r["converged"], diagnosis=r["diagnosis"],
                hamiltonian=r["hamiltonian"], final_residual=r["final_residual"], seconds=time.perf_counter() - t0,
                cond=float(np.linalg.cond(restate.gram_matrix(k, q0))))
    save(f"vel_{n}", meta, p0=r["p0"], endpoint=r["endpoint"], history=np.array(r["residual_history"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    if a.threads:
        native.set_threads(a.threads)
    only = set(a.only.split(",")) if a.only else None

    def want(n):
        return only is None or n in only

    t_all = time.perf_counter()
    if want("c2_solve_cell"):
        w = configs.c2()
        solve_fixture("c2_solve_cell", w, 100, 1.0, w.sigma, stride=4)
    if want("c4_mid"):
        w = configs.c4(32768)
        match_fixture("c4_mid", w, w.h, w.max_iter, stride=8, with_h=True)
    if want("c5_mid"):
        w = configs.c5(65536)
        match_fixture("c5_mid", w, w.h, w.max_iter, stride=16, with_h=True)
    for n, sig, ax, ay in VEL_CASES:
        if want(f"vel_{n}"):
            vel_fixture(n, sig, ax, ay)
    if want("c4_onset"):
        w = configs.c4()
        onset_fixture("c4_onset", w, ONSET_H["C4"], stride=64)
    if want("c5_onset"):
        w = configs.c5()
        onset_fixture("c5_onset", w, ONSET_H["C5"], stride=256)
    if want("c4_match2"):
        w = configs.c4()
        match_fixture("c4_match2", w, w.h, 2, stride=64)
    if want("c5_match2"):
        w = configs.c5()
        match_fixture("c5_match2", w, w.h, 2, stride=256)
    if want("c3_step"):
        w = configs.c3()
        solve_fixture("c3_step", w, 1, w.t_final / w.steps, 0.0, stride=64)
    if want("c2_solve_dense"):
        w = configs.c2()
        solve_fixture("c2_solve_dense", w, 100, 1.0, 0.0, stride=4)
    print(f"total {time.perf_counter() - t_all:.0f} s")


if __name__ == "__main__":
    main()
