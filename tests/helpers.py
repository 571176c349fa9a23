"""Shared test fixtures: the reference tests' state generators (tests/test_pipeline.cpp:17-76)
restated with numpy RNGs (inputs only; both implementations receive the same arrays)."""
from __future__ import annotations

import math

import numpy as np

from paper_1503_03553_b200.simulation import (LineWall, MaterialParams, ParticleSet, RectWall,
                                              SimConfig)


def basic_config(box: float = 1.0) -> SimConfig:  # test_pipeline.cpp:17-35
    cfg = SimConfig()
    cfg.dt = 1e-5
    cfg.gravity = (0.0, 0.0, 0.0)
    cfg.domain_min = (0.0, 0.0, 0.0)
    cfg.domain_max = (box, box, box)
    cfg.materials.add("bead", MaterialParams(0.3, 3.85e5, 1e6, 0.9, 0.3))
    return cfg


def random_dense_state(n: int, seed: int) -> ParticleSet:  # test_pipeline.cpp:39-60
    rng = np.random.default_rng(seed)
    r0 = 0.005
    sp = 1.7 * r0
    side = int(math.ceil(round(n ** (1.0 / 3.0), 9)))
    s = ParticleSet(n)
    i = np.arange(n)
    ix, iy, iz = i % side, (i // side) % side, i // (side * side)
    s.ids[:] = i
    base = np.stack([0.02 + ix * sp, 0.02 + iy * sp, 0.02 + iz * sp], axis=1)
    s.positions[:] = base + 0.1 * sp * rng.uniform(-1, 1, (n, 3))
    s.radii[:] = r0 * (0.8 + 0.2 * np.abs(rng.uniform(-1, 1, n)))
    s.velocities[:] = 0.5 * rng.uniform(-1, 1, (n, 3))
    s.angular_velocities[:] = 5.0 * rng.uniform(-1, 1, (n, 3))
    s.masses[:] = 1.3e-3
    return s


def box_for(n: int) -> float:  # test_pipeline.cpp:62-65
    side = int(math.ceil(round(n ** (1.0 / 3.0), 9)))
    return 0.05 + side * 1.7 * 0.005


def walled_config(n_side: int = 8) -> SimConfig:
    """A settle-type box: floor + 4 sides (SURVEY App. B shape) and one line wall."""
    cfg = basic_config(0.2)
    cfg.domain_max = (0.2, 0.2, 0.4)
    cfg.gravity = (0.0, 0.0, -9.81)
    cfg.dt = 1e-4
    cfg.materials.add("wall", MaterialParams(0.3, 3.85e5, 1e6, 0.9, 0.3))
    cfg.rect_walls = [
        RectWall((0, 0, 0), (0.2, 0, 0), (0, 0.2, 0), 1),
        RectWall((0, 0, 0), (0, 0.2, 0), (0, 0, 0.4), 1),
        RectWall((0.2, 0, 0), (0, 0.2, 0), (0, 0, 0.4), 1),
        RectWall((0, 0, 0), (0.2, 0, 0), (0, 0, 0.4), 1),
        RectWall((0, 0.2, 0), (0.2, 0, 0), (0, 0, 0.4), 1),
    ]
    cfg.line_walls = [LineWall((0, 0.1, 0.004), (0.2, 0.1, 0.004), 1)]
    return cfg


def settling_state(n: int, seed: int) -> ParticleSet:
    """Particles near the floor of walled_config with downward velocities: wall contacts form."""
    rng = np.random.default_rng(seed)
    r0 = 0.005
    side = int(math.ceil(math.sqrt(n / 2)))
    s = ParticleSet(n)
    for i in range(n):
        ix, iy, iz = i % side, (i // side) % side, i // (side * side)
        s.ids[i] = i
        s.positions[i] = (0.006 + ix * 0.0105 + 0.0004 * rng.uniform(-1, 1),
                          0.006 + iy * 0.0105 + 0.0004 * rng.uniform(-1, 1),
                          0.0052 + iz * 0.0105 + 0.0004 * rng.uniform(-1, 1))
        s.velocities[i] = (0.3 * rng.uniform(-1, 1), 0.3 * rng.uniform(-1, 1), -0.5)
        s.angular_velocities[i] = 3.0 * rng.uniform(-1, 1, 3)
        s.radii[i] = r0
        s.masses[i] = 1.309e-3
    return s


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def bitwise_equal(a, b) -> bool:
    return np.array_equal(bits(a), bits(b))
