"""The small-N kernel on a thread-block cluster (8 CTAs, DSMEM stage exchange) against the same
kernel on one CTA: same iterations, momenta and frames (summation order differs only in the
split of each row's source sweep)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(cluster, out):
    env = dict(os.environ, GS_B200_CLUSTER=str(cluster))
    subprocess.run([sys.executable, os.path.join(HERE, "helpers", "cluster_run.py"), out], env=env, check=True,
                   timeout=600)
    return np.load(out)


def test_cluster_kernel_matches_single_cta(cuda, tmp_path):
    a = _run(1, str(tmp_path / "c1.npz"))
    b = _run(8, str(tmp_path / "c8.npz"))
    for space in ("momentum", "velocity"):
        assert int(a[f"{space}_it"]) == int(b[f"{space}_it"]) > 0
        p_a, p_b = a[f"{space}_p0"], b[f"{space}_p0"]
        assert np.abs(p_a - p_b).max() <= 1e-8 * np.abs(p_a).max()
        assert float(a[f"{space}_H"]) == pytest.approx(float(b[f"{space}_H"]), rel=1e-10)
    assert np.abs(a["evolve_q"] - b["evolve_q"]).max() <= 1e-12
    assert a["frames_q"].shape == b["frames_q"].shape
    assert np.abs(a["frames_q"] - b["frames_q"]).max() <= 1e-12
