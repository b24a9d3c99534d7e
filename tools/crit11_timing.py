"""Wall-clock of the reference's acceptance criterion 11 (feedback vs Newton) through the drop-in.

    tools/run_reference_suite.sh prepare   # once, here
    PYTHONPATH=baseline/_ref:. python tools/crit11_timing.py   # on a GPU box

Times match() (momentum feedback, h = 0.3) and newton_match() (h = 1.0) for N = 60 and 30 as the
reference's test_criterion_11_feedback_beats_newton_walltime does, three times each (cold, warm)."""

import math
import time

from paper_1510_03816_b200 import dropin

dropin.install()
from geoshoot import KernelSpec, ResidualNorm, ShootingConfig, SystemSpec, match, newton_match  # noqa: E402
from geoshoot.shapes import circle, standard_rotated_ellipse  # noqa: E402

SYS = SystemSpec(kernel=KernelSpec())


def cfg(h, **kw):
    kw.setdefault("max_iter", 2000)
    kw.setdefault("system", SYS)
    return ShootingConfig(h=h, epsilon=1e-3, **kw)


for rep in range(3):
    for n in (60, 30):
        ref = circle(2.0, n=n)
        tgt = standard_rotated_ellipse(4.0, 1.0, -math.pi / 4, (1.0, 0.0), n)
        t0 = time.perf_counter()
        fb = match(ref, tgt, cfg(0.3, norm=ResidualNorm.L2))
        t1 = time.perf_counter()
        nw = newton_match(ref, tgt, cfg(1.0, norm=ResidualNorm.L2))
        t2 = time.perf_counter()
        print(f"rep {rep} N={n}: feedback {t1 - t0:.4f} s ({fb.iterations} it), newton {t2 - t1:.4f} s "
              f"({nw.iterations} it)")
