"""B200-native stencil hot path of arXiv 1201.2118 (CaCUDA; reference "stencilforge").

The product is the CUDA library ``_lib/libsfb200.so`` (sm_100a kernels + C++
host driver) behind the C ABI of ``include/sforge_b200.h``.  This package is
its Python face: ``Simulation`` mirrors ``sforge::cfd::simulation`` and the
executor operations, ``decompose`` mirrors ``grid::decompose``.
"""
from ._lib import CfdError, ConfigError, ExecError, GridError, SfError, lib  # noqa: F401
from .sim import (  # noqa: F401
    FIELDS,
    Decomposition,
    ExecutionPlan,
    FluidParams,
    ScheduleStep,
    Simulation,
    SolverConfig,
    StepStats,
    cavity_fluid,
    decompose,
    nccl_unique_id,
)

__all__ = [
    "Simulation", "SolverConfig", "FluidParams", "StepStats", "cavity_fluid", "decompose",
    "Decomposition", "ExecutionPlan", "ScheduleStep", "nccl_unique_id", "FIELDS", "SfError", "ConfigError", "GridError", "ExecError", "CfdError", "lib",
]
