"""B200-native Euler–Poincaré N-particle hot path of arXiv 1510.03816 (reference: ``geoshoot``).

Drop-in for the reference's hot-path entry points (``geoshoot/__init__.py:4-74``):
``rhs``, ``hamiltonian``, ``evolve``, ``match`` and their spec/result types, with the same
names, argument meaning and error behaviour, computed by the fp64 sm_100a kernels of
``libgs_b200.so`` (C ABI: include/geoshoot_b200.h).  ``dropin.install()`` rebinds the
reference package itself onto these implementations.  There is no CPU fallback.
"""

from .errors import ConfigurationError, DegenerateConfigurationError, DivergenceError, GeoshootError
from .kernels import LAMBDA, KernelFamily, KernelSpec, support_radius
from .particles import (ParticleState, SystemSpec, conserved_quantities, hamiltonian, inexactness_energy, rhs,
                        velocity_field)
from .integrator import EvolveConfig, EvolveResult, evolve
from .shapes import LandmarkTemplate, circle, ellipse_rot_shift
from .shooting import (MatchResult, ResidualNorm, ShootingConfig, StopRule, UpdateSpace, contraction_diagnostics,
                       match, momenta_from_velocity, newton_match)
from .analysis import (DIVERGED, ClusterVerdict, DistanceRecord, ExactnessRow, SweepGrid, cluster_test,
                       convergence_sweep, exact_vs_inexact, iso_invariance_check, predict, shape_distance)
from .device import get_path, set_path
from . import dropin  # noqa: E402  (dropin.install() rebinds the reference package)

__version__ = "0.1.0"

__all__ = [
    "ConfigurationError", "DegenerateConfigurationError", "DivergenceError", "GeoshootError", "LAMBDA",
    "KernelFamily", "KernelSpec", "support_radius", "ParticleState", "SystemSpec", "conserved_quantities",
    "hamiltonian", "inexactness_energy", "rhs", "velocity_field", "EvolveConfig", "EvolveResult", "evolve", "LandmarkTemplate",
    "circle", "ellipse_rot_shift", "MatchResult", "ResidualNorm", "ShootingConfig", "StopRule", "UpdateSpace",
    "contraction_diagnostics", "match", "momenta_from_velocity", "newton_match", "get_path", "set_path",
    "DIVERGED", "ClusterVerdict", "DistanceRecord", "ExactnessRow", "SweepGrid", "cluster_test", "convergence_sweep",
    "exact_vs_inexact", "iso_invariance_check", "predict", "shape_distance",
]
