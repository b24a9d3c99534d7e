"""bench.py plumbing on CPU: `--gpus N` launches N ranks (torch.distributed.run, gloo in the dry
run), and the reference arm's row-block pool computes the reference's RHS."""

import json
import os
import subprocess
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_2_launches_two_ranks():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2


def test_bench_rejects_a_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=3" in (out.stderr + out.stdout)


def test_reference_arm_pool_is_the_reference_rhs():
    sys.path.insert(0, REPO)
    import bench
    from oracle import restate
    from paper_1510_03816_b200 import configs

    w = configs.c2(700)
    k = restate.Kernel(0, w.alpha, True)
    got = {}

    def rows(kk, s2, q, p, r0, r1):  # capture what the pool computes
        got[(r0, r1)] = restate_rhs_rows(kk, s2, q, p, r0, r1)
        return got[(r0, r1)]

    restate_rhs_rows = restate.rhs_rows
    restate.rhs_rows = rows
    try:
        bench.reference_rhs_pool(k, w, threads=3, block=128)
    finally:
        restate.rhs_rows = restate_rhs_rows
    dq = np.concatenate([got[b][0] for b in sorted(got)])
    dp = np.concatenate([got[b][1] for b in sorted(got)])
    wq, wp = restate.rhs(k, 0.0, w.q, w.p)
    assert np.array_equal(dq, wq) and np.allclose(dp, wp, rtol=0, atol=1e-15 * np.abs(wp).max())


def test_roofline_counts_come_from_the_built_library():
    """bench.py's FP64 instructions per ordered pair and operand-read ceiling are read from the SASS
    of the library actually built (tools/sass_loops.py, cuobjdump; no GPU needed)."""
    import shutil

    import pytest

    if not (shutil.which("cuobjdump") or os.path.exists("/usr/local/cuda/bin/cuobjdump")):
        pytest.skip("cuobjdump not installed")
    sys.path.insert(0, REPO)
    import bench

    for kind, lo, hi in (("dense", 12.0, 20.0), ("cell", 20.0, 32.0)):
        w, ceiling = bench.implemented_fp64_per_pair(kind)
        assert w is not None and lo <= w <= hi, (kind, w)
        # a mix of 2-cycle and ~3.2-cycle FP64 instructions: between 2 / 3.2 and 1
        assert ceiling is not None and 0.625 <= ceiling <= 1.0, (kind, ceiling)
