"""The reference's command line on the B200 path.

    python -m paper_1510_03816_b200.cli match ref.json tgt.json --h 0.3 --out run/
    python -m paper_1510_03816_b200.cli predict ref.json partial.json --t-match 0.6 --t-predict 1 --h 0.3

Runs ``geoshoot.cli.main`` (cli.py:436-452) unchanged — same sub-commands, flags, files and
exit codes — with the drop-in installed, so ``match`` / ``predict`` / ``distance`` /
``cluster`` / ``sweep`` compute on the device (sweeps and cluster tests as batched launches).
Every manifest the reference writes (io.py:201-223, cli.py:110-121) gains one ``extras``
entry, ``"b200"``, with the GPU facts of the run: device name, library version and ABI,
pair-sum path, and the kernel launches / device pair evaluations the run issued.
The reference package must be importable (it owns the CLI, the file formats and the shape
generators); there is no CPU fallback for the compute.
"""

from __future__ import annotations

import sys

from . import _native as N
from . import device, dropin


def gpu_facts() -> dict:
    """The "b200" manifest entry (launch / pair counters are this process's totals)."""
    facts = {"library": None, "abi": None, "device": None, "path": device.get_path()}
    try:
        lib = N.load()
        facts["library"] = lib.gs_version().decode()
        facts["abi"] = int(lib.gs_abi_version())
    except N.NativeUnavailable as exc:
        facts["library"] = f"unavailable: {exc}"
        return facts
    try:
        import torch

        if torch.cuda.is_available():
            facts["device"] = torch.cuda.get_device_name(torch.cuda.current_device())
            if N.Context._contexts():
                import ctypes

                ctx = N.Context.get()
                ms, pl, la, pa = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
                if ctx.lib.gs_profile_read(ctx.handle, ctypes.byref(ms), ctypes.byref(pl), ctypes.byref(la),
                                           ctypes.byref(pa), 0) == N.GS_OK:
                    facts["kernel_launches"] = int(la.value)
                    facts["pair_evaluations"] = int(pa.value)
    except Exception as exc:  # facts are best effort; the run's own outcome is what matters
        facts["device_error"] = str(exc)
    return facts


def main(argv=None) -> int:
    try:
        import geoshoot
        import geoshoot.cli as ref_cli
    except ImportError as exc:
        print(f"error: the reference package geoshoot is required for the command line ({exc})", file=sys.stderr)
        return 2
    dropin.install(geoshoot)
    original = ref_cli._manifest

    def manifest(args, t0, outcome, config=None, inputs=(), extras=None):
        extras = dict(extras or {})
        extras["b200"] = gpu_facts()
        return original(args, t0, outcome, config, inputs, extras)

    ref_cli._manifest = manifest
    try:
        return ref_cli.main(argv)
    finally:
        ref_cli._manifest = original
        dropin.uninstall()


if __name__ == "__main__":
    sys.exit(main())
