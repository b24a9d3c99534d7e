"""Result-type registry.

Functions of this package build their results (ParticleState, EvolveResult, MatchResult,
LandmarkTemplate) through this registry.  By default the classes are this package's
mirrors; ``dropin.install`` points them at the reference's own classes so that code
written against ``geoshoot`` receives exactly the types it expects.
"""

from __future__ import annotations

_classes: dict = {}


def register_defaults(**classes) -> None:
    for k, v in classes.items():
        _classes.setdefault(k, v)


def use(**classes) -> None:
    _classes.update(classes)


def get(name: str):
    return _classes[name]
