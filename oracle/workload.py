"""TEST INFRASTRUCTURE ONLY — the bench workload built without the product library.

bench.py's reference arm (and its cpu_baseline leg) must run the reference alone: it builds the
configs[1] input here, with the oracle's copy of the §8d generator (orc_gen_packing in
dem_oracle.c, bitwise the product's dem_gen_packing; tests/test_oracle_golden.py checks it) and
duck-typed SimConfig / ParticleSet objects that oracle.CConfig / RefSim accept. Nothing here
imports paper_1503_03553_b200.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .oracle import ORACLE_SO


@dataclass
class Material:  # materials.hpp:10-21 defaults
    poisson_ratio: float = 0.3
    shear_modulus: float = 4e5
    youngs_modulus: float = 1e6
    restitution: float = 0.9
    sliding_friction: float = 0.3


class Materials:
    def __init__(self, mats):
        self._m = list(mats)

    def size(self):
        return len(self._m)

    def params(self, k):
        return self._m[k]

    def pair_restitution(self, a, b):  # materials.cpp:58-64 (no overrides)
        return float(np.sqrt(self._m[a].restitution * self._m[b].restitution))


@dataclass
class Config:  # sim_config.hpp:42-63, the fields the reference step reads
    dt: float = 1e-5
    gravity: tuple = (0.0, 0.0, 0.0)
    domain_min: tuple = (0.0, 0.0, 0.0)
    domain_max: tuple = (0.0, 0.0, 0.0)
    materials: Materials = field(default_factory=lambda: Materials([Material()]))
    rect_walls: List = field(default_factory=list)
    line_walls: List = field(default_factory=list)
    grid_cell_size: float = 0.0
    contact_capacity: int = 16
    periodic: int = 0
    shear_rate: float = 0.0


class Particles:
    def __init__(self, n):
        self.ids = np.zeros(n, np.uint32)
        self.positions = np.zeros((n, 3))
        self.velocities = np.zeros((n, 3))
        self.angular_velocities = np.zeros((n, 3))
        self.radii = np.zeros(n)
        self.masses = np.zeros(n)
        self.material_ids = np.zeros(n, np.uint32)


def gen_packing(n, s=1.8, jit=0.2, poly=False, seed=1, omega_half=0.5):
    """G(n, s, jit, poly, seed) of SURVEY §8d -> (Particles, domain_max)."""
    L = C.CDLL(ORACLE_SO)
    PD, PU = C.POINTER(C.c_double), C.POINTER(C.c_uint32)
    L.orc_gen_packing.restype = C.c_int
    L.orc_gen_packing.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_double,
                                  PU, PD, PD, PD, PD, PD, PU, PD]
    p = Particles(n)
    dmax = (C.c_double * 3)()
    L.orc_gen_packing(n, s, jit, int(poly), seed, omega_half, p.ids.ctypes.data_as(PU),
                      p.positions.ctypes.data_as(PD), p.velocities.ctypes.data_as(PD),
                      p.angular_velocities.ctypes.data_as(PD), p.radii.ctypes.data_as(PD),
                      p.masses.ctypes.data_as(PD), p.material_ids.ctypes.data_as(PU), dmax)
    return p, tuple(dmax)


def packing_config(domain_max, poly=False, dt=1e-5):
    """§8d benchmark configuration: MaterialParams defaults, g = 0, no walls, K = 16 (32 poly)."""
    return Config(dt=dt, domain_max=tuple(domain_max), contact_capacity=32 if poly else 16)
