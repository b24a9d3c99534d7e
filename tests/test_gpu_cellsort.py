"""The one-CTA cell sort (k_sort_small, n <= 16384, gs_cell.cu) against the device-wide CUB
radix sort it replaces: the cell-list RHS must be bitwise identical — both are stable sorts of
(cell key, index), so the sorted order, every target's candidate order and its sums are the same.
The sort choice is read once per process (GS_B200_SORT_SMALL_MAX), so the CUB run is a child."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1510_03816_b200 as gs
from paper_1510_03816_b200 import configs
gs.set_path("cell")
out = {}
for name, n in (("c2", 16384), ("c4_5000", 5000), ("c4_16385", 16385), ("dup", 3000)):
    if name == "c2":
        w = configs.c2(n); q, p, alpha = w.q, w.p, w.alpha
    elif name == "dup":
        # many particles per cell and equal keys in long runs: a coarse lattice with jitter-free rows
        r = np.random.default_rng(11)
        q = np.stack(np.meshgrid(np.arange(60) * 0.01, np.arange(50) * 0.013), -1).reshape(-1, 2)
        q = q[r.permutation(len(q))]
        p = r.normal(0, 0.1, q.shape); alpha = 0.05 / (53 * np.log(2))
    else:
        w = configs.c4(n); q, p, alpha = w.q, w.h * (w.target - w.q), w.alpha
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=float(alpha)))
    dq, dp = gs.rhs(spec, gs.ParticleState(q, p))
    out[name + "_dq"], out[name + "_dp"] = dq, dp
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, tag, env_extra):
    out = tmp_path / f"{tag}.npz"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, REPO, str(out)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def test_small_sort_is_bitwise_the_device_sort(cuda, tmp_path):
    a = _run(tmp_path, "small", {})
    b = _run(tmp_path, "cub", {"GS_B200_SORT_SMALL_MAX": "0"})
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
        assert np.isfinite(a[k]).all(), k
