"""Fixed-step RK4 integration on the B200 (mirror of geoshoot/integrator.py:19-121).

``evolve`` runs the whole integration in libgs_b200.so: every stage's RHS, the stage
inputs q + (dt/2) k, the combine q + (dt/6)(k1 + 2k2 + 2k3 + k4) and the finite-state
checks stay on the device; one launch per stage pair (or one persistent kernel for
N <= 512).  Errors carry the reference's step/time-window messages.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device
from . import errors as _errors
from . import types as _types

__all__ = ["EvolveConfig", "EvolveResult", "evolve"]


@dataclass(frozen=True)
class EvolveConfig:
    """Time horizon and grid for one evolution (integrator.py:22-43)."""

    t_final: float = 1.0
    steps: int = 100
    capture_every: int = 0

    def __post_init__(self):
        if not (self.t_final > 0 and np.isfinite(self.t_final)):
            raise _errors.ConfigurationError(f"t_final must be positive, got {self.t_final}")
        if self.steps < 1:
            raise _errors.ConfigurationError(f"steps must be >= 1, got {self.steps}")
        if self.capture_every < 0:
            raise _errors.ConfigurationError(f"capture_every must be >= 0, got {self.capture_every}")


@dataclass(frozen=True)
class EvolveResult:
    """Final state plus optionally captured (time, state) frames (integrator.py:46-55)."""

    final: object
    frames: tuple

    @property
    def times(self) -> np.ndarray:
        return np.array([t for t, _ in self.frames])


def frame_times(t_final: float, steps: int, capture_every: int) -> list:
    # integrator.py:79-80, 84-86, 116-119: t_at(k) = t_final * (k / steps)
    out = [0.0]
    for step in range(1, steps + 1):
        if step % capture_every == 0 or step == steps:
            out.append(t_final * (step / steps))
    return out


def evolve(spec, state, config=None):
    """Integrate the system from ``state`` over [0, t_final] (integrator.py:66-121)."""
    if config is None:
        config = _types.get("EvolveConfig")()
    q, p, frames = device.evolve(spec, state.q, state.p, config.t_final, config.steps, config.capture_every)
    PS = _types.get("ParticleState")
    out_frames = ()
    if frames is not None:
        fr = frames.cpu().numpy()
        times = frame_times(config.t_final, config.steps, config.capture_every)
        out_frames = tuple((t, PS(fr[k, :, 0:2].copy(), fr[k, :, 2:4].copy())) for k, t in enumerate(times))
    return _types.get("EvolveResult")(final=PS(q.cpu().numpy(), p.cpu().numpy()), frames=out_frames)


_types.register_defaults(EvolveConfig=EvolveConfig, EvolveResult=EvolveResult)
