"""B200-native solver for the time-stepping hot path of the well-balanced
Osher-Romberg scheme (arXiv 1806.04960), drop-in for ``wbflow``'s driver API.
"""
from .errors import (ConfigError, UnsupportedConfigurationError, SimulationError,
                     NearSonicWarning, DeviceError)
from .params import ModelParams
from .grid import (CartesianGrid, build_grid, BoundaryCondition, BoundarySpec,
                   ghost_state, EdgeSet, enumerate_edges)
from .state import prim_to_cons, cons_to_prim, EquilibriumProfile

__all__ = ["ConfigError", "UnsupportedConfigurationError", "SimulationError",
           "NearSonicWarning", "DeviceError", "ModelParams", "CartesianGrid",
           "build_grid", "BoundaryCondition", "BoundarySpec", "ghost_state",
           "EdgeSet", "enumerate_edges", "prim_to_cons", "cons_to_prim",
           "EquilibriumProfile", "Simulation", "set_workers", "compute_dt",
           "advance_step", "total_mass"]


def __getattr__(name):
    # the time stepper loads the CUDA library; import it lazily so that the
    # host-only pieces (grid, params, scenarios) work on machines without it
    if name in ("Simulation", "set_workers", "compute_dt", "advance_step", "total_mass"):
        from . import timestepper
        return getattr(timestepper, name)
    raise AttributeError(name)
