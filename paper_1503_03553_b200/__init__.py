"""B200-native DEM step (arXiv 1503.03553) behind the reference demforge::Simulation API.

The compute path is libdem_b200.so (hand-written sm_100a CUDA, see csrc/); this package is the
host-side mirror of the reference C++ interface. Importing it loads the library and fails
loudly if it has not been built.
"""
from . import _capi
from .simulation import (BASELINE, TWO_PHASE, CapacityError, ConfigError, ContactEntry,
                         DegenerateContactError, DeviceError, ForceAccumulator, Grid, KernelError,
                         LineWall, MaterialParams, MaterialTable, ParticleSet, RectWall, SimConfig,
                         Simulation, StepMetrics, device_kernel_names, gen_packing, gen_periodic_packing,
                         packing_config, periodic_config,
                         total_kinetic_energy, total_momentum, wall_id)

PHASE_INTEGRATE = _capi.PHASE_INTEGRATE
PHASE_GRAVITY = _capi.PHASE_GRAVITY
PHASE_PP = _capi.PHASE_PP
PHASE_RECT = _capi.PHASE_RECT
PHASE_LINE = _capi.PHASE_LINE
PHASE_STEP = _capi.PHASE_STEP

_capi.lib()  # load now: no silent fallback

__all__ = [n for n in dir() if not n.startswith("_")]
