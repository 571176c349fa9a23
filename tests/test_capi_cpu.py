"""CPU: the drop-in boundary. The C-ABI library loads without a GPU, exports every symbol the
headers in include/ declare, validates configurations like the reference
(sim_config.cpp:10-60, particle_set.cpp:40-58) before touching a device, and the input
generator is deterministic."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in ("dem_b200.h", "dem_b200_gen.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s+\*?(dem_[a-z_0-9]+)\s*\(", txt, flags=re.M):
            names.add(m.group(1))
    return names


def test_headers_declare_the_abi():
    names = declared_functions()
    for must in ("dem_create", "dem_step", "dem_destroy", "dem_get_particles", "dem_get_contacts",
                 "dem_clone", "dem_force_phase", "dem_last_error", "dem_gen_packing"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1503_03553_b200 import _capi
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    bound = {n for n, _, _ in _capi.SIGNATURES}
    assert declared_functions() <= bound
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_sm100a():
    from paper_1503_03553_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version():
    from paper_1503_03553_b200 import _capi
    assert _capi.lib().dem_abi_version() == 2


def test_generator_deterministic_and_shaped():
    import paper_1503_03553_b200 as dem
    a, dmax = dem.gen_packing(1000, s=1.8, jit=0.2, seed=3)
    b, _ = dem.gen_packing(1000, s=1.8, jit=0.2, seed=3)
    c, _ = dem.gen_packing(1000, s=1.8, jit=0.2, seed=4)
    assert np.array_equal(a.positions, b.positions) and not np.array_equal(a.positions, c.positions)
    side = 10
    assert abs(dmax[0] - (side * 1.8 * 0.005 + 4 * 0.005)) < 1e-15
    assert np.all(np.abs(a.velocities) <= 0.5) and np.all(a.radii == 0.005)
    p, _ = dem.gen_packing(1000, s=1.4, jit=0.2, poly=True, seed=3, omega_half=50.0)
    assert p.radii.min() >= 0.0025 and p.radii.max() < 0.005
    assert np.allclose(p.masses, 1e-3 * (p.radii / 0.005) ** 3, rtol=1e-15)
    assert np.abs(p.angular_velocities).max() > 10.0


def _expect_config_error(cfg, ps):
    import paper_1503_03553_b200 as dem
    with pytest.raises(dem.ConfigError) as e:
        dem.Simulation(ps, cfg)
    return str(e.value)


def test_config_validation_before_device():
    """sim_config.cpp:10-60 — rejected on the host, no GPU needed."""
    import paper_1503_03553_b200 as dem
    from helpers import basic_config, random_dense_state
    ps = random_dense_state(8, 1)
    cfg = basic_config(1.0)
    cfg.dt = 0.0
    assert "dt" in _expect_config_error(cfg, ps)
    cfg = basic_config(1.0)
    cfg.domain_max = (1.0, 0.0, 1.0)
    assert "domain" in _expect_config_error(cfg, ps)
    cfg = basic_config(1.0)
    cfg.contact_capacity = 0
    assert "capacity" in _expect_config_error(cfg, ps)
    cfg = basic_config(1.0)
    cfg.rect_walls = [dem.RectWall((0, 0, 0), (1, 0, 0), (1, 1, 0), 0)]
    assert "orthogonal" in _expect_config_error(cfg, ps)
    cfg = basic_config(1.0)
    cfg.line_walls = [dem.LineWall((0, 0, 0), (0, 0, 0), 0)]
    assert "zero-length" in _expect_config_error(cfg, ps)
    cfg = basic_config(1.0)
    cfg.materials = dem.MaterialTable()
    cfg.materials.add("x", dem.MaterialParams(poisson_ratio=0.6))
    assert "poisson" in _expect_config_error(cfg, ps)
    bad = random_dense_state(8, 1)
    bad.radii[3] = 0.0
    assert "radius" in _expect_config_error(basic_config(1.0), bad)
    bad = random_dense_state(8, 1)
    bad.positions[2, 1] = np.nan
    assert "non-finite" in _expect_config_error(basic_config(1.0), bad)


def test_id_and_capacity_validation_before_device():
    """The B200 history is keyed by stable id: duplicate ids and ids in the wall-key
    range are rejected (the reference keys its table by slot and accepts them); contact capacity is
    bounded by k_detect's shared-memory rows (K <= 80)."""
    from helpers import basic_config, random_dense_state
    ps = random_dense_state(8, 1)
    ps.ids[5] = ps.ids[2]
    assert "duplicate stable id" in _expect_config_error(basic_config(1.0), ps)
    ps = random_dense_state(8, 1)
    ps.ids[7] = 0xFFFFFFC0
    assert "wall-key range" in _expect_config_error(basic_config(1.0), ps)
    ps = random_dense_state(8, 1)
    ps.material_ids[1] = 3
    assert "bad material" in _expect_config_error(basic_config(1.0), ps)
    cfg = basic_config(1.0)
    cfg.contact_capacity = 81
    assert "at most 80" in _expect_config_error(cfg, random_dense_state(8, 1))


def test_material_table_rules():
    """materials.cpp:58-68: pair restitution default sqrt(ea eb), overrides symmetric; mu."""
    import paper_1503_03553_b200 as dem
    t = dem.MaterialTable()
    t.add("a", dem.MaterialParams(restitution=0.81, sliding_friction=0.4))
    t.add("b", dem.MaterialParams(restitution=0.64, sliding_friction=0.1))
    assert t.pair_restitution(0, 1) == t.pair_restitution(1, 0) == np.sqrt(0.81 * 0.64)
    t.set_pair_restitution(1, 0, 0.5)
    assert t.pair_restitution(0, 1) == 0.5 and t.pair_overridden(0, 1)
    assert t.pair_sliding_friction(0, 1) == np.sqrt(0.4 * 0.1)
    with pytest.raises(dem.ConfigError):
        t.add("a", dem.MaterialParams())
