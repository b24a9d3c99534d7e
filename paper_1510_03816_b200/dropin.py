"""Drop-in registration: rebind the reference package ``geoshoot`` onto the B200 path.

The reference has no plugin registry: its modules import their
callees by name, so every alias must be rebound (SURVEY.md §8(b) "Rebinding points"):

    rhs          geoshoot.particles.rhs, geoshoot.integrator.rhs (integrator.py:17, used :89), geoshoot.rhs
    evolve       geoshoot.integrator.evolve, geoshoot.shooting.evolve (shooting.py:28), geoshoot.analysis.evolve
                 (analysis.py:19), geoshoot.cli.evolve (cli.py:34), geoshoot.evolve
    match        geoshoot.shooting.match, geoshoot.analysis.match (analysis.py:23), geoshoot.cli.match
                 (cli.py:58), geoshoot.match
    hamiltonian  geoshoot.particles.hamiltonian, geoshoot.shooting.hamiltonian (shooting.py:30), geoshoot.hamiltonian
    template     geoshoot.shapes.LandmarkTemplate.__post_init__ (shapes.py:45-58: the duplicate check via an
                 N x N distance matrix, SURVEY §8(b) "template duplicate check") -> an O(N log N) sort-based
                 check with the same first pair and message, so templates of C4/C5 size can be built
    newton_match geoshoot.shooting.newton_match, geoshoot.newton_match  (batched Jacobian columns)
    analysis     shape_distance, iso_invariance_check, cluster_test, convergence_sweep, predict,
                 exact_vs_inexact in geoshoot.analysis, geoshoot.cli (cli.py:24-32), geoshoot
                 (independent matches batched into one launch)

After ``install()`` the reference's own callers (analysis, cli, newton_match) run their shoots
on the device, with the reference's exception classes and result types.  ``match`` runs on the
device in both update spaces (momentum: one device loop; velocity: device Gram matrix, cuSOLVER
Cholesky via torch.linalg, device shoots), as does ``momenta_from_velocity``.  The device
provides the conical and gaussian families (the north_star's path); a call whose kernel is of
another family (bessel, ``kernels.py:91-118``) is not replaced: the rebound name hands it to the
reference's own function it shadowed, so the drop-in never narrows what the reference accepts.
The package's own API (``paper_1510_03816_b200.rhs`` etc.) still raises ConfigurationError for
bessel — there is no CPU fallback inside this package.  Use ``pytest -p paper_1510_03816_b200.pytest_dropin`` to run a geoshoot-based
test suite against the device path.
"""

from __future__ import annotations

import importlib

from . import analysis as _analysis
from . import errors as _errors
from . import integrator as _integrator
from . import particles as _particles
from . import shapes as _shapes
from . import shooting as _shooting
from . import types as _types

_saved: list = []
_ALIASES = {
    "rhs": ("particles", "integrator", ""),
    "evolve": ("integrator", "shooting", "analysis", "cli", ""),
    "match": ("shooting", "analysis", "cli", ""),
    "hamiltonian": ("particles", "shooting", ""),
    "momenta_from_velocity": ("shooting", ""),
    "velocity_field": ("particles", ""),
    # batched analysis: independent matches / shoots side by side
    "newton_match": ("shooting", ""),
    "shape_distance": ("analysis", "cli", ""),
    "iso_invariance_check": ("analysis", ""),
    "cluster_test": ("analysis", "cli", ""),
    "convergence_sweep": ("analysis", "cli", ""),
    "predict": ("analysis", "cli", ""),
    "exact_vs_inexact": ("analysis", "cli", ""),
}


def _module(pkg, sub: str):
    if not sub:
        return pkg
    try:
        return importlib.import_module(f"{pkg.__name__}.{sub}")
    except ImportError:
        return None


_DEVICE_FAMILIES = ("conical", "gaussian")


def _kernel_specs(obj, depth: int = 0):
    """KernelSpec-like objects reachable from a call argument: a KernelSpec, a SystemSpec
    (.kernel), a ShootingConfig (.system.kernel), a SweepGrid (.kernel_family) or a list of them."""
    if depth > 2 or obj is None:
        return
    if isinstance(obj, (list, tuple)):
        for o in obj:
            yield from _kernel_specs(o, depth + 1)
        return
    fam = getattr(obj, "kernel_family", None)
    if fam is not None:
        yield str(getattr(fam, "value", fam))
    if hasattr(obj, "family") and hasattr(obj, "alpha"):
        yield str(getattr(obj.family, "value", obj.family))
    for attr in ("kernel", "system"):
        sub = getattr(obj, attr, None)
        if sub is not None and sub is not obj:
            yield from _kernel_specs(sub, depth + 1)


def _on_device(args, kwargs) -> bool:
    return all(f in _DEVICE_FAMILIES for a in (*args, *kwargs.values()) for f in _kernel_specs(a))


def _dispatch(device_fn, reference_fn):
    """The device function for the device's kernel families, the shadowed reference function otherwise."""

    def fn(*args, **kwargs):
        if _on_device(args, kwargs):
            return device_fn(*args, **kwargs)
        return reference_fn(*args, **kwargs)

    fn.__name__ = getattr(device_fn, "__name__", "fn")
    fn.__doc__ = getattr(device_fn, "__doc__", None)
    fn.device = device_fn
    fn.original = reference_fn
    return fn


def install(pkg=None):
    """Rebind ``geoshoot`` (or the given package object) onto this package.  Idempotent."""
    if _saved:
        return pkg or importlib.import_module("geoshoot")
    pkg = pkg or importlib.import_module("geoshoot")
    ref_shooting = _module(pkg, "shooting")
    original_match = ref_shooting.match

    for name in ("GeoshootError", "ConfigurationError", "DegenerateConfigurationError", "DivergenceError"):
        _saved.append((_errors, name, getattr(_errors, name)))
        setattr(_errors, name, getattr(pkg, name))
    _types.use(ParticleState=pkg.ParticleState, EvolveResult=pkg.EvolveResult, EvolveConfig=pkg.EvolveConfig,
               MatchResult=pkg.MatchResult, LandmarkTemplate=pkg.LandmarkTemplate,
               DistanceRecord=pkg.DistanceRecord, ClusterVerdict=pkg.ClusterVerdict, ExactnessRow=pkg.ExactnessRow)

    def match(reference, target, cfg):
        """shooting.match on the device, both update spaces (momentum: one device loop;
        velocity: device Gram + cuSOLVER factor + device shoots)."""
        return _shooting.match(reference, target, cfg)

    match.original = original_match
    tpl = getattr(_module(pkg, "shapes"), "LandmarkTemplate", None)
    if tpl is not None:
        _saved.append((tpl, "__post_init__", tpl.__post_init__))
        tpl.__post_init__ = _shapes.LandmarkTemplate.__post_init__
    impl = {"rhs": _particles.rhs, "evolve": _integrator.evolve, "match": match,
            "hamiltonian": _particles.hamiltonian, "momenta_from_velocity": _shooting.momenta_from_velocity,
            "newton_match": _shooting.newton_match, "velocity_field": _particles.velocity_field}
    for fname in ("shape_distance", "iso_invariance_check", "cluster_test", "convergence_sweep", "predict",
                  "exact_vs_inexact"):
        impl[fname] = getattr(_analysis, fname)
    wrappers = {}
    for fname, subs in _ALIASES.items():
        for sub in subs:
            mod = _module(pkg, sub)
            if mod is not None and hasattr(mod, fname):
                orig = getattr(mod, fname)
                _saved.append((mod, fname, orig))
                key = (fname, id(orig))
                if key not in wrappers:  # one wrapper per shadowed function: aliases stay identical
                    wrappers[key] = _dispatch(impl[fname], orig)
                setattr(mod, fname, wrappers[key])
    return pkg


def uninstall() -> None:
    """Restore every attribute ``install`` rebound."""
    while _saved:
        mod, name, val = _saved.pop()
        setattr(mod, name, val)
    from . import integrator, particles, shapes, shooting  # noqa: F401  (re-register own types)

    _types.use(ParticleState=particles.ParticleState, EvolveResult=integrator.EvolveResult,
               EvolveConfig=integrator.EvolveConfig, MatchResult=shooting.MatchResult,
               LandmarkTemplate=shapes.LandmarkTemplate, DistanceRecord=_analysis.DistanceRecord,
               ClusterVerdict=_analysis.ClusterVerdict, ExactnessRow=_analysis.ExactnessRow)


def installed() -> bool:
    return bool(_saved)
