"""Kernel selection (mirror of geoshoot/kernels.py:44-88) and device-side parameters.

Only the spec types live here; the kernel itself is evaluated inside the fp64 pair kernels
(csrc/gs_device.cuh).  The bessel family (kernels.py:91-118) needs a device K_nu and is not
provided: selecting it for a device call raises ConfigurationError.
"""

from __future__ import annotations

import enum
import math
import warnings
from dataclasses import dataclass

from . import errors as _errors

__all__ = ["KernelFamily", "KernelSpec", "support_radius", "LAMBDA"]

# KD-1: the conical kernel exp(-r/alpha) is 2^-53 at r = LAMBDA * alpha.
LAMBDA = 53.0 * math.log(2.0)


class KernelFamily(str, enum.Enum):
    CONICAL = "conical"
    GAUSSIAN = "gaussian"
    BESSEL = "bessel"


@dataclass(frozen=True)
class KernelSpec:
    """kernels.py:50-88: family, order nu (bessel only), length scale alpha, normalization."""

    family: KernelFamily = KernelFamily.CONICAL
    nu: float = 1.5
    alpha: float = 1.0
    normalized: bool = True

    def __post_init__(self):
        object.__setattr__(self, "family", KernelFamily(self.family))
        if not (self.alpha > 0 and math.isfinite(self.alpha)):
            raise _errors.ConfigurationError(f"alpha must be positive, got {self.alpha}")
        if not (self.nu > 0 and math.isfinite(self.nu)):
            raise _errors.ConfigurationError(f"nu must be positive, got {self.nu}")
        if self.family is KernelFamily.BESSEL:
            if self.nu <= 1:
                raise _errors.ConfigurationError(
                    f"bessel kernels require nu > 1 (kernel unbounded otherwise), got nu={self.nu}")
            if self.nu < 1.5:
                warnings.warn(f"nu={self.nu} in (1, 1.5): kernel has a cusp at r=0 and is used unmollified",
                              stacklevel=2)

    def peak(self) -> float:
        """Unnormalized kernel value at r = 0 (kernels.py:83-88)."""
        a2 = self.alpha * self.alpha
        if self.family is KernelFamily.BESSEL:
            return 1.0 / (4.0 * math.pi * a2 * (self.nu - 1.0))
        return 1.0 / (2.0 * math.pi * a2)


def family_name(kernel) -> str:
    """Family of a KernelSpec of this package or of the reference (duck-typed)."""
    fam = kernel.family
    return str(getattr(fam, "value", fam))


def support_radius(kernel) -> float:
    """Radius beyond which the normalized kernel is below 2^-53 of its peak.

    conical exp(-r/alpha): LAMBDA * alpha (KD-1); gaussian exp(-r^2 / 2 alpha^2):
    alpha * sqrt(2 LAMBDA).  The cell-list path drops pairs at or beyond this radius.
    """
    fam = family_name(kernel)
    if fam == "conical":
        return LAMBDA * float(kernel.alpha)
    if fam == "gaussian":
        return math.sqrt(2.0 * LAMBDA) * float(kernel.alpha)
    raise _errors.ConfigurationError(f"kernel family {fam!r} is not available on the device")
