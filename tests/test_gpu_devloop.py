"""The large-N feedback loop as one conditional-WHILE graph (gs_match, n > 512) against the
host-driven loop it replaced: same kernels in the same order, so every field must be bitwise
equal — converging, capped, momentum-delta, blown-up and cell-list runs."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_device_loop_equals_host_loop(cuda, tmp_path):
    sys.path.insert(0, os.path.join(HERE, "helpers"))
    import devloop_cases

    dev = devloop_cases.run_cases()
    out = tmp_path / "host.npz"
    env = dict(os.environ, GS_B200_DEVLOOP="0")
    subprocess.run([sys.executable, os.path.join(HERE, "helpers", "devloop_cases.py"), str(out)], check=True, env=env,
                   timeout=600)
    host = np.load(out)
    assert sorted(dev) == sorted(host.files)
    for k in host.files:
        np.testing.assert_array_equal(dev[k], host[k], err_msg=k)
    # the cases cover every outcome
    diag = {k.split("__")[0]: str(host[k]) for k in host.files if k.endswith("__diagnosis")}
    assert diag["converge"] == "None" and diag["cell"] == "None"
    assert diag["cap"] == "iteration cap reached before the stopping rule"
    assert diag["blowup"].startswith("step too large")
    assert host["mdelta__meta"][1] == 1.0
