"""Host-side mirror of the reference Simulation / SimConfig API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/core/include/demforge/: pipeline.hpp:62-136, sim_config.hpp:42-63,
materials.hpp:23-58, particle_set.hpp:13-51, error.hpp:10-49) so the parity tests read like the
reference's own tests. All compute runs in libdem_b200.so on the GPU; this module only marshals
arrays. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi

# ---------------------------------------------------------------------------------------------
# Exceptions (error.hpp:10-49)


class ConfigError(RuntimeError):
    """error.hpp:10-13 — configuration / validation failure (CLI exit 2)."""


class KernelError(RuntimeError):
    """error.hpp:17-26 — runtime failure inside a kernel; carries the kernel name."""

    def __init__(self, kernel: str, what: str, particle: Optional[int] = None,
                 particle_id: Optional[int] = None, step: Optional[int] = None):
        super().__init__(what)
        self.kernel = kernel
        self._particle = particle
        self.particle_id = particle_id
        self.step = step


class CapacityError(KernelError):
    """error.hpp:30-42 — a particle's contact row is full."""

    def particle(self) -> Optional[int]:
        return self._particle


class DegenerateContactError(KernelError):
    """error.hpp:46-49 — coincident centres."""


class DeviceError(RuntimeError):
    """CUDA / driver failure (no reference counterpart)."""


# ---------------------------------------------------------------------------------------------
# Value types


@dataclass
class MaterialParams:  # materials.hpp:10-21
    poisson_ratio: float = 0.3
    shear_modulus: float = 4e5
    youngs_modulus: float = 1e6
    restitution: float = 0.9
    sliding_friction: float = 0.3


class MaterialTable:  # materials.hpp:23-58
    def __init__(self):
        self._names: List[str] = []
        self._mats: List[MaterialParams] = []
        self._overrides = {}

    def add(self, name: str, params: MaterialParams) -> int:
        if name in self._names:
            raise ConfigError(f"material '{name}' defined twice")
        self._names.append(name)
        self._mats.append(params)
        return len(self._mats) - 1

    def index_of(self, name: str) -> int:
        if name not in self._names:
            raise ConfigError(f"unknown material '{name}'")
        return self._names.index(name)

    def contains(self, name: str) -> bool:
        return name in self._names

    def params(self, i: int) -> MaterialParams:
        return self._mats[i]

    def name(self, i: int) -> str:
        return self._names[i]

    def size(self) -> int:
        return len(self._mats)

    def __len__(self):
        return len(self._mats)

    def set_pair_restitution(self, a: int, b: int, eps: float):
        self._overrides[(min(a, b), max(a, b))] = eps

    def pair_overridden(self, a: int, b: int) -> bool:
        return (min(a, b), max(a, b)) in self._overrides

    def pair_restitution(self, a: int, b: int) -> float:  # materials.cpp:58-64
        lo, hi = min(a, b), max(a, b)
        if (lo, hi) in self._overrides:
            return self._overrides[(lo, hi)]
        return math.sqrt(self._mats[lo].restitution * self._mats[hi].restitution)

    def pair_sliding_friction(self, a: int, b: int) -> float:  # materials.cpp:66-68
        return math.sqrt(self._mats[a].sliding_friction * self._mats[b].sliding_friction)


@dataclass
class RectWall:  # geometry.hpp:55-61
    corner: Sequence[float]
    edge_u: Sequence[float]
    edge_v: Sequence[float]
    material_id: int = 0


@dataclass
class LineWall:  # geometry.hpp:63-67
    a: Sequence[float]
    b: Sequence[float]
    material_id: int = 0


BASELINE = 0
TWO_PHASE = 1


@dataclass
class SimConfig:  # sim_config.hpp:42-63 (fields the step reads)
    dt: float = 0.0
    gravity: Sequence[float] = (0.0, 0.0, -9.81)
    domain_min: Sequence[float] = (0.0, 0.0, 0.0)
    domain_max: Sequence[float] = (0.0, 0.0, 0.0)
    materials: MaterialTable = field(default_factory=MaterialTable)
    rect_walls: List[RectWall] = field(default_factory=list)
    line_walls: List[LineWall] = field(default_factory=list)
    grid_cell_size: float = 0.0
    contact_capacity: int = 16
    collide_variant: int = TWO_PHASE
    # beyond the reference: periodic axes bit 0 x, 1 y, 2 z; Lees-Edwards rate
    periodic: int = 0
    shear_rate: float = 0.0
    # 0 fp64 parity mode (bitwise with the reference), 1 fp32 throughput mode (1e-5)
    precision: int = 0


class ParticleSet:  # particle_set.hpp:13-37, numpy SoA
    def __init__(self, n: int = 0):
        self.ids = np.zeros(n, np.uint32)
        self.positions = np.zeros((n, 3), np.float64)
        self.velocities = np.zeros((n, 3), np.float64)
        self.angular_velocities = np.zeros((n, 3), np.float64)
        self.radii = np.zeros(n, np.float64)
        self.masses = np.zeros(n, np.float64)
        self.material_ids = np.zeros(n, np.uint32)

    @classmethod
    def from_lists(cls, rows):
        """rows: iterable of (id, pos, vel, angvel, radius, mass, material) like push_back."""
        rows = list(rows)
        s = cls(len(rows))
        for i, (pid, p, v, w, r, m, mat) in enumerate(rows):
            s.ids[i] = pid
            s.positions[i] = p
            s.velocities[i] = v
            s.angular_velocities[i] = w
            s.radii[i] = r
            s.masses[i] = m
            s.material_ids[i] = mat
        return s

    def size(self) -> int:
        return len(self.ids)

    def __len__(self):
        return len(self.ids)

    def max_radius(self) -> float:
        return float(self.radii.max()) if len(self.radii) else 0.0

    def copy(self) -> "ParticleSet":
        s = ParticleSet(0)
        for k in ("ids", "positions", "velocities", "angular_velocities", "radii", "masses",
                  "material_ids"):
            setattr(s, k, getattr(self, k).copy())
        return s

    def contiguous(self) -> "ParticleSet":
        s = ParticleSet(0)
        s.ids = np.ascontiguousarray(self.ids, np.uint32)
        s.positions = np.ascontiguousarray(self.positions, np.float64).reshape(-1, 3)
        s.velocities = np.ascontiguousarray(self.velocities, np.float64).reshape(-1, 3)
        s.angular_velocities = np.ascontiguousarray(self.angular_velocities, np.float64).reshape(-1, 3)
        s.radii = np.ascontiguousarray(self.radii, np.float64)
        s.masses = np.ascontiguousarray(self.masses, np.float64)
        s.material_ids = np.ascontiguousarray(self.material_ids, np.uint32)
        return s

    _FIELDS = (("ids", np.uint32), ("positions", np.float64), ("velocities", np.float64),
               ("angular_velocities", np.float64), ("radii", np.float64), ("masses", np.float64),
               ("material_ids", np.uint32))

    def is_contiguous(self) -> bool:
        """Every present array C-contiguous with the ABI dtype (then c_struct can view it as is)."""
        for k, dt in self._FIELDS:
            a = getattr(self, k)
            if a is not None and (a.dtype != dt or not a.flags.c_contiguous):
                return False
        return True

    def c_struct(self) -> _capi.dem_particles:
        # cached per set of array buffers (host-coupled loops pass the same pinned arrays every step)
        key = tuple(None if getattr(self, k) is None else (getattr(self, k).ctypes.data, getattr(self, k).size)
                    for k, _ in self._FIELDS)
        cached = getattr(self, "_c_cache", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        p = self._c_struct_build()
        self._c_cache = (key, p)
        return p

    def _c_struct_build(self) -> _capi.dem_particles:
        p = _capi.dem_particles()
        p.count = len(self.positions)

        def ptr(a, t):  # None -> NULL (dem_get_particles skips it, dem_set_particles keeps it)
            return None if a is None else a.ctypes.data_as(C.POINTER(t))
        p.ids = ptr(self.ids, C.c_uint32)
        p.positions = ptr(self.positions, C.c_double)
        p.velocities = ptr(self.velocities, C.c_double)
        p.angular_velocities = ptr(self.angular_velocities, C.c_double)
        p.radii = ptr(self.radii, C.c_double)
        p.masses = ptr(self.masses, C.c_double)
        p.material_ids = ptr(self.material_ids, C.c_uint32)
        return p


def total_momentum(s: ParticleSet) -> np.ndarray:  # particle_set.cpp:65-69 (sequential order)
    p = np.zeros(3)
    for i in range(len(s.ids)):
        p = p + s.velocities[i] * s.masses[i]
    return p


def total_kinetic_energy(s: ParticleSet) -> float:  # particle_set.cpp:71-79
    inertia = 0.4 * s.masses * s.radii * s.radii
    v2 = (s.velocities ** 2).sum(axis=1)
    w2 = (s.angular_velocities ** 2).sum(axis=1)
    return float((0.5 * s.masses * v2 + 0.5 * inertia * w2).sum())


@dataclass
class ForceAccumulator:  # particle_set.hpp:40-51
    force: np.ndarray
    torque: np.ndarray


@dataclass
class StepMetrics:  # pipeline.hpp:35-48
    step: int = 0
    contacts: int = 0
    pp_contact_events: int = 0
    max_contacts_per_particle: int = 0
    clamps: int = 0
    friction_max_ratio: float = 0.0
    capped_contacts: int = 0
    cells: int = 0
    device_kernel_ms: tuple = ()

    @classmethod
    def from_c(cls, m: _capi.dem_step_metrics) -> "StepMetrics":
        return cls(m.step, m.contacts, m.pp_contact_events, m.max_contacts_per_particle,
                   m.clamps, m.friction_max_ratio, m.capped_contacts, m.cells,
                   tuple(m.device_kernel_ms))


@dataclass
class Grid:  # grid.hpp:14-31
    origin: tuple
    cell_size: float
    nx: int
    ny: int
    nz: int

    def cell_count(self) -> int:
        return self.nx * self.ny * self.nz


@dataclass
class ContactEntry:
    owner: int        # slot
    partner: int      # slot, or wall id -(w+1)
    delta_t: np.ndarray


def wall_id(w: int) -> int:  # contact_table.hpp:35
    return -(w + 1)


class _Config:
    """Keeps the ctypes arrays behind a dem_config alive."""

    def __init__(self, cfg: SimConfig):
        m = cfg.materials.size()
        self.mats = (_capi.dem_material * max(m, 1))()
        for k in range(m):
            p = cfg.materials.params(k)
            self.mats[k] = _capi.dem_material(p.poisson_ratio, p.shear_modulus, p.youngs_modulus,
                                              p.restitution, p.sliding_friction)
        self.pair = (C.c_double * max(m * m, 1))()
        for a in range(m):
            for b in range(m):
                self.pair[a * m + b] = cfg.materials.pair_restitution(a, b)
        nr, nl = len(cfg.rect_walls), len(cfg.line_walls)
        self.rects = (_capi.dem_rect_wall * max(nr, 1))()
        for k, w in enumerate(cfg.rect_walls):
            self.rects[k] = _capi.dem_rect_wall(_capi.D3(*w.corner), _capi.D3(*w.edge_u),
                                                _capi.D3(*w.edge_v), w.material_id)
        self.lines = (_capi.dem_line_wall * max(nl, 1))()
        for k, w in enumerate(cfg.line_walls):
            self.lines[k] = _capi.dem_line_wall(_capi.D3(*w.a), _capi.D3(*w.b), w.material_id)
        c = _capi.dem_config()
        c.dt = cfg.dt
        c.gravity = _capi.D3(*cfg.gravity)
        c.domain_min = _capi.D3(*cfg.domain_min)
        c.domain_max = _capi.D3(*cfg.domain_max)
        c.material_count = m
        c.materials = self.mats
        c.pair_restitution = self.pair
        c.rect_wall_count = nr
        c.rect_walls = self.rects
        c.line_wall_count = nl
        c.line_walls = self.lines
        c.grid_cell_size = cfg.grid_cell_size
        c.contact_capacity = cfg.contact_capacity
        c.collide_variant = cfg.collide_variant
        c.periodic = getattr(cfg, "periodic", 0)
        c.shear_rate = getattr(cfg, "shear_rate", 0.0)
        c.precision = getattr(cfg, "precision", 0)
        self.c = c


def _raise(lib, ctx, code: int):
    err = _capi.dem_error()
    lib.dem_last_error(ctx, C.byref(err))
    msg = err.message.decode(errors="replace")
    kernel = _capi.KERNEL_NAMES[err.kernel] if 0 <= err.kernel < len(_capi.KERNEL_NAMES) else "?"
    if code == 1:
        raise ConfigError(msg)
    if code == 3:
        raise CapacityError(kernel, msg, err.particle_slot, err.particle_id, err.step)
    if code == 4:
        raise DegenerateContactError("Collide", msg, err.particle_slot, err.particle_id, err.step)
    if code == 2:
        raise KernelError(kernel, msg, err.particle_slot, err.particle_id, err.step)
    if code == 5:
        raise ValueError(msg or "bad argument at the C ABI")
    raise DeviceError(msg or f"dem error {code}")


class Simulation:
    """pipeline.hpp:62-136 over libdem_b200.so. Construction runs the priming force pass."""

    def __init__(self, initial: ParticleSet, config: SimConfig, device: int = 0, _ctx=None):
        self._lib = _capi.lib()
        self._cfg = config
        if _ctx is not None:
            self._ctx = _ctx
            return
        self._ccfg = _Config(config)
        ps = initial.contiguous()
        ctx = C.c_void_p()
        rc = self._lib.dem_create(C.byref(self._ccfg.c), C.byref(ps.c_struct()), device, C.byref(ctx))
        if rc != 0:
            _raise(self._lib, None, rc)
        self._ctx = ctx
        self._record_traces = False

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx:
            self._lib.dem_destroy(ctx)
            self._ctx = None

    def _check(self, rc):
        if rc != 0:
            _raise(self._lib, self._ctx, rc)

    # --- the reference's per-kernel methods, pipeline.hpp:77-86 ---
    # The B200 step fuses kernels: calls compose into one force phase in pipeline order that runs
    # when a result is observed or a kernel earlier in that order is called again (the C++
    # drop-in, include/demb200/simulation.hpp, does the same). Every composed phase bins and
    # starts from zeroed accumulators; errors surface when the phase runs.
    _ORDER = {"integrate": (0, _capi.PHASE_INTEGRATE), "calc_hash": (1, 0), "bitonic_sort": (2, 0),
              "find_cell_bounds_and_reorder": (3, 0), "zero_forces": (4, 0),
              "force_gravity": (5, _capi.PHASE_GRAVITY), "initialize_contact_ids": (6, 0),
              "collide": (7, _capi.PHASE_PP), "collide_rectangle": (8, _capi.PHASE_RECT),
              "collide_line": (9, _capi.PHASE_LINE)}

    def _compose(self, name, variant=None):
        k, flag = self._ORDER[name]
        pend = self.__dict__.setdefault("_pending", [-1, 0, None])
        if k <= pend[0]:
            self._run_pending()
            pend = self._pending
        pend[0], pend[1] = k, pend[1] | flag
        if variant is not None:
            pend[2] = variant

    def _run_pending(self):
        pend = self.__dict__.get("_pending")
        if not pend or pend[0] < 0:
            return None
        self._pending = [-1, 0, None]
        flags, variant = pend[1], pend[2]
        cur = getattr(self._cfg, "collide_variant", TWO_PHASE)
        if variant is not None and variant != cur:
            self._check(self._lib.dem_set_collide_variant(self._ctx, int(variant)))
        m = _capi.dem_step_metrics()
        try:
            self._check(self._lib.dem_force_phase(self._ctx, flags, C.byref(m)))
        finally:
            if variant is not None and variant != cur:
                self._lib.dem_set_collide_variant(self._ctx, int(cur))
        self._last_composed = StepMetrics.from_c(m)
        return self._last_composed

    def kernel_integrate(self): self._compose("integrate")
    def kernel_calc_hash(self): self._compose("calc_hash")
    def kernel_bitonic_sort(self): self._compose("bitonic_sort")
    def kernel_find_cell_bounds_and_reorder(self): self._compose("find_cell_bounds_and_reorder")
    def zero_forces(self): self._compose("zero_forces")
    def kernel_force_gravity(self): self._compose("force_gravity")
    def kernel_initialize_contact_ids(self): self._compose("initialize_contact_ids")
    def kernel_collide(self, variant: int = TWO_PHASE, record_traces: bool = False):
        self._compose("collide", variant)
    def kernel_collide_rectangle(self): self._compose("collide_rectangle")
    def kernel_collide_line(self): self._compose("collide_line")

    # --- pipeline.hpp:64-86 ---
    def step(self) -> StepMetrics:
        self._run_pending()
        m = _capi.dem_step_metrics()
        self._check(self._lib.dem_step(self._ctx, 1, C.byref(m)))
        return StepMetrics.from_c(m)

    def steps(self, n: int) -> StepMetrics:
        self._run_pending()
        m = _capi.dem_step_metrics()
        self._check(self._lib.dem_step(self._ctx, n, C.byref(m)))
        return StepMetrics.from_c(m)

    def step_async(self, n: int = 1) -> None:
        """Enqueue n steps and return at once (dem_step_async). The next call that reads or
        replaces the state reports their errors; particles() / particles_into() right after it
        overlap the readback with the last step's detection and forces."""
        self._run_pending()
        self._check(self._lib.dem_step_async(self._ctx, n))

    def sync(self) -> StepMetrics:
        """Wait for asynchronous steps; the last one's metrics (dem_sync)."""
        m = _capi.dem_step_metrics()
        self._check(self._lib.dem_sync(self._ctx, C.byref(m)))
        return StepMetrics.from_c(m)

    def force_phase(self, flags: int) -> StepMetrics:
        self._run_pending()
        m = _capi.dem_step_metrics()
        self._check(self._lib.dem_force_phase(self._ctx, flags, C.byref(m)))
        return StepMetrics.from_c(m)

    def advance_and_collide(self) -> StepMetrics:
        """advance_to_collide + kernel_collide (tests/test_pipeline.cpp:69-76): integrate, bin,
        sweep, pp contacts only, no gravity, no walls."""
        self._run_pending()
        return self.force_phase(_capi.PHASE_INTEGRATE | _capi.PHASE_PP)

    def set_record_traces(self, on: bool):
        self._record_traces = bool(on)  # traces are a §8f 'next' row; metrics are always on

    def set_collide_variant(self, v: int):
        self._run_pending()
        self._check(self._lib.dem_set_collide_variant(self._ctx, int(v)))

    def clone(self) -> "Simulation":
        self._run_pending()
        out = C.c_void_p()
        self._check(self._lib.dem_clone(self._ctx, C.byref(out)))
        s = Simulation(None, self._cfg, _ctx=out)
        s._ccfg = getattr(self, "_ccfg", None)
        return s

    __copy__ = clone

    # --- accessors, pipeline.hpp:88-107 ---
    def config(self) -> SimConfig:
        return self._cfg

    def size(self) -> int:
        return int(self._lib.dem_size(self._ctx))

    def step_index(self) -> int:
        return int(self._lib.dem_step_index(self._ctx))

    def particles(self) -> ParticleSet:
        self._run_pending()
        s = ParticleSet(self.size())
        self._check(self._lib.dem_get_particles(self._ctx, C.byref(s.c_struct())))
        return s

    def particles_into(self, s: ParticleSet) -> ParticleSet:
        """particles() into caller-owned (e.g. pinned) contiguous arrays of the right size.
        The arrays are written through raw pointers, so their dtype, contiguity and size are
        checked first (ValueError), never trusted."""
        self._run_pending()
        n = self.size()
        if not s.is_contiguous():
            raise ValueError("particles_into: every array must be C-contiguous with the ABI dtype")
        for k, _ in ParticleSet._FIELDS:
            a = getattr(s, k)
            if a is None:
                continue
            per = 3 if k in ("positions", "velocities", "angular_velocities") else 1
            if a.size != per * n:
                raise ValueError(f"particles_into: {k} has {a.size} elements, expected {per * n}")
        self._check(self._lib.dem_get_particles(self._ctx, C.byref(s.c_struct())))
        return s

    def set_particles(self, s: ParticleSet):
        self._run_pending()
        if not s.is_contiguous():
            s = s.contiguous()
        self._check(self._lib.dem_set_particles(self._ctx, C.byref(s.c_struct())))

    def set_motion(self, positions, velocities, angular_velocities):
        """Replace only the kinematic state (current slot order, as particles() returns it); ids,
        radii, masses and materials stay (dem_set_particles with those arrays NULL)."""
        self._run_pending()
        s = getattr(self, "_motion", None)
        if s is None:
            s = self._motion = ParticleSet(0)
            s.ids = s.radii = s.masses = s.material_ids = None
        s.positions = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
        s.velocities = np.ascontiguousarray(velocities, np.float64).reshape(-1, 3)
        s.angular_velocities = np.ascontiguousarray(angular_velocities, np.float64).reshape(-1, 3)
        if len(s.positions) != self.size():
            raise ValueError("set_motion: arrays must have one row per particle")
        self._check(self._lib.dem_set_particles(self._ctx, C.byref(s.c_struct())))

    def forces(self) -> ForceAccumulator:
        self._run_pending()
        n = self.size()
        f = np.zeros((n, 3))
        t = np.zeros((n, 3))
        self._check(self._lib.dem_get_forces(self._ctx, f.ctypes.data_as(C.POINTER(C.c_double)),
                                             t.ctypes.data_as(C.POINTER(C.c_double))))
        return ForceAccumulator(f, t)

    def set_forces(self, fa: ForceAccumulator):
        self._run_pending()
        f = np.ascontiguousarray(fa.force, np.float64)
        t = np.ascontiguousarray(fa.torque, np.float64)
        self._check(self._lib.dem_set_forces(self._ctx, f.ctypes.data_as(C.POINTER(C.c_double)),
                                             t.ctypes.data_as(C.POINTER(C.c_double))))

    def periodic_box(self):
        """(cell extent per axis, Lees-Edwards image offset) — DESIGN.md §6."""
        self._run_pending()
        ext = (C.c_double * 3)()
        off = C.c_double()
        self._check(self._lib.dem_get_periodic_box(self._ctx, ext, C.byref(off)))
        return tuple(ext), off.value

    def grid(self) -> Grid:
        self._run_pending()
        g = _capi.dem_grid()
        self._check(self._lib.dem_get_grid(self._ctx, C.byref(g)))
        return Grid(tuple(g.origin), g.cell_size, g.nx, g.ny, g.nz)

    def order(self):
        self._run_pending()
        n = self.size()
        k = np.zeros(n, np.uint32)
        p = np.zeros(n, np.uint32)
        self._check(self._lib.dem_get_order(self._ctx, k.ctypes.data_as(C.POINTER(C.c_uint32)),
                                            p.ctypes.data_as(C.POINTER(C.c_uint32))))
        return k, p

    def set_contacts(self, owner_slot, partner, delta_t):
        """Replace the live contact history (current slot order; partners as slots or -(w+1)), as
        the reference's bench restores its ContactTable (runner.cpp:131-132)."""
        self._run_pending()
        o = np.ascontiguousarray(owner_slot, np.uint32)
        p = np.ascontiguousarray(partner, np.int32)
        d = np.ascontiguousarray(delta_t, np.float64).reshape(-1, 3)
        if not (len(o) == len(p) == len(d)):
            raise ValueError("set_contacts: arrays of different lengths")
        self._check(self._lib.dem_set_contacts(self._ctx, o.ctypes.data_as(C.POINTER(C.c_uint32)),
                                               p.ctypes.data_as(C.POINTER(C.c_int32)),
                                               d.ctypes.data_as(C.POINTER(C.c_double)), len(o)))

    def contacts(self):
        """Touched contact-table entries: (owner slot[], partner[] (slot or -(w+1)), delta_t[,3])."""
        cnt = self._lib.dem_get_contacts(self._ctx, None, None, None, 0)
        if cnt < 0:
            self._check(-cnt)
        o = np.zeros(cnt, np.uint32)
        p = np.zeros(cnt, np.int32)
        d = np.zeros((cnt, 3))
        got = self._lib.dem_get_contacts(self._ctx, o.ctypes.data_as(C.POINTER(C.c_uint32)),
                                         p.ctypes.data_as(C.POINTER(C.c_int32)),
                                         d.ctypes.data_as(C.POINTER(C.c_double)), cnt)
        if got < 0:
            self._check(-got)
        return o, p, d

    def traces(self):
        """Traversal traces of the last force phase (pipeline.hpp:97): (offsets[n+1] uint64,
        candidate slot int32[], contact bool[]); slot i's events are [offsets[i], offsets[i+1])."""
        self._run_pending()
        n = self.size()
        off = np.zeros(n + 1, np.uint64)
        total = self._lib.dem_get_traces(self._ctx, off.ctypes.data_as(C.POINTER(C.c_uint64)), None, 0)
        if total < 0:
            self._check(-total)
        ev = np.zeros((max(total, 1), 2), np.int32)
        if total:
            got = self._lib.dem_get_traces(self._ctx, None, ev.ctypes.data_as(C.c_void_p), total)
            if got < 0:
                self._check(-got)
        return off, ev[:total, 0].copy(), ev[:total, 1].astype(bool)

    def contact_table(self):
        o, p, d = self.contacts()
        return [ContactEntry(int(a), int(b), c) for a, b, c in zip(o, p, d)]

    def mean_coordination(self, metrics: StepMetrics) -> float:  # pipeline.cpp:310-315
        n = self.size()
        return metrics.pp_contact_events / n if n else 0.0

    # --- measurement helpers (bench.py) ---
    def time_steps(self, nsteps: int, flush_bytes: int = 0):
        self._run_pending()
        ms = (C.c_float * max(nsteps, 1))()
        m = _capi.dem_step_metrics()
        self._check(self._lib.dem_time_steps(self._ctx, nsteps, flush_bytes, ms, C.byref(m)))
        return [float(ms[k]) for k in range(nsteps)], StepMetrics.from_c(m)

    def profile_step(self, flush_bytes: int = 0) -> StepMetrics:
        self._run_pending()
        m = _capi.dem_step_metrics()
        self._check(self._lib.dem_profile_step(self._ctx, flush_bytes, C.byref(m)))
        return StepMetrics.from_c(m)

    def kernels_per_step(self) -> int:
        return int(self._lib.dem_kernels_per_step(self._ctx))

    def device_bytes(self) -> int:
        return int(self._lib.dem_device_bytes(self._ctx))


def device_kernel_names():
    lib = _capi.lib()
    return [lib.dem_device_kernel_name(k).decode() for k in range(_capi.DEM_DEVICE_KERNEL_COUNT)]


def gen_packing(n: int, s: float = 1.8, jit: float = 0.2, poly: bool = False, seed: int = 1,
                omega_half: float = 0.5):
    """SURVEY §8d generator G (include/dem_b200_gen.h). Returns (ParticleSet, domain_max)."""
    ps = ParticleSet(n)
    dm = (C.c_double * 3)()
    rc = _capi.lib().dem_gen_packing(n, s, jit, 1 if poly else 0, seed, omega_half,
                                     C.byref(ps.c_struct()), dm)
    if rc != 0:
        raise ValueError("dem_gen_packing failed")
    return ps, tuple(dm)


def gen_periodic_packing(n: int, s: float = 1.8, jit: float = 0.2, poly: bool = False, seed: int = 1,
                         omega_half: float = 0.5):
    """G(N, s, jit, poly, seed) laid out for a periodic box: the same
    draws as gen_packing, the lattice starting at the origin, positions wrapped into
    [0, side*s*r0). Returns (ParticleSet, box length L)."""
    ps, dm = gen_packing(n, s=s, jit=jit, poly=poly, seed=seed, omega_half=omega_half)
    r0 = 0.005
    side = int(round((dm[0] - 4.0 * r0) / (s * r0)))  # the generator's lattice side
    L = side * s * r0
    ps.positions = np.mod(ps.positions - 2.0 * r0, L)
    return ps, L


def packing_config(domain_max, poly: bool = False, dt: float = 1e-5, capacity: Optional[int] = None,
                   gravity=(0.0, 0.0, 0.0)) -> SimConfig:
    """The §8d benchmark configuration: MaterialParams defaults, g = 0, no walls, K = 16 (32 poly)."""
    cfg = SimConfig()
    cfg.dt = dt
    cfg.gravity = gravity
    cfg.domain_min = (0.0, 0.0, 0.0)
    cfg.domain_max = tuple(domain_max)
    cfg.materials.add("bead", MaterialParams())
    cfg.contact_capacity = capacity if capacity is not None else (32 if poly else 16)
    return cfg


def periodic_config(L: float, shear_rate: float = 0.0, poly: bool = False, dt: float = 1e-5,
                    capacity: Optional[int] = None) -> SimConfig:
    """the §8d benchmark configuration in a fully periodic box [0, L)^3,
    with Lees-Edwards shear (flow x, gradient y) at `shear_rate`."""
    cfg = packing_config((L, L, L), poly=poly, dt=dt, capacity=capacity)
    cfg.periodic = 7
    cfg.shear_rate = shear_rate
    return cfg
