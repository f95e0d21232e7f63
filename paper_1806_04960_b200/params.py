"""Model constants (drop-in for ``wbflow.params.ModelParams``,
pkg/src/wbflow/params.py:6-33): Tait closure k0 / rho0 / gamma, gravity g and
the gas volume-fraction floor epsilon, with the reference's validation and
``ValueError`` messages."""

import math
from dataclasses import dataclass

__all__ = ["ModelParams"]


@dataclass(frozen=True)
class ModelParams:
    k0: float
    rho0: float = 1000.0
    gamma: float = 1.0
    g: float = 9.81
    epsilon: float = 1.0e-3

    def __post_init__(self):
        checks = (
            (self.k0 > 0.0, f"k0 must be positive, got {self.k0}"),
            (self.rho0 > 0.0, f"rho0 must be positive, got {self.rho0}"),
            (self.gamma >= 1.0, f"gamma must be >= 1, got {self.gamma}"),
            (self.g >= 0.0, f"g must be non-negative, got {self.g}"),
            (0.0 < self.epsilon < 0.5,
             f"epsilon must lie in (0, 0.5), got {self.epsilon}"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def sound_speed_ref(self):
        """c(rho0) = sqrt(gamma k0 / rho0) (params.py:35-39)."""
        return math.sqrt(self.gamma * self.k0 / self.rho0) if self.gamma != 1.0 \
            else math.sqrt(self.k0 / self.rho0)
