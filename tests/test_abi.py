"""The C-ABI library loads and exports every entry point include/geoshoot_b200.h declares.

CPU-only: nothing here launches device work.
"""

import ctypes
import os
import re

from conftest import REPO

HEADER = os.path.join(REPO, "include", "geoshoot_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(gs_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("gs_rhs", "gs_evolve", "gs_match", "gs_hamiltonian", "gs_rhs_rows", "gs_stage_run"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1510_03816_b200 import _native

    lib = _native.load()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
    assert sorted(_native.EXPORTS) == declared_symbols()
    assert lib.gs_abi_version() == 2
    assert b"sm_100a" in lib.gs_version()


def test_library_is_built_for_sm100a_only():
    import subprocess

    from paper_1510_03816_b200 import _native

    out = subprocess.run(["cuobjdump", "-lelf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_struct_layouts_match_header():
    from paper_1510_03816_b200 import _native as N

    assert ctypes.sizeof(N.System) == 40
    assert ctypes.sizeof(N.Status) == 32
    assert ctypes.sizeof(N.MatchConfig) == 40
    assert ctypes.sizeof(N.MatchResultC) == 64
    assert ctypes.sizeof(N.BatchItem) == 80
    assert ctypes.sizeof(N.SlabGrid) == 40


def test_no_device_means_loud_failure():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200._native import NativeUnavailable

    st = gs.ParticleState(np.zeros((3, 2)), np.zeros((3, 2)))
    with pytest.raises(NativeUnavailable):
        gs.rhs(gs.SystemSpec(), st)
