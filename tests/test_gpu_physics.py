"""GPU: full-size parity and the reference's physical property tests
(tests/test_pipeline.cpp:222-413, runner.cpp:274-417) on the B200 path."""
import math
import os

import numpy as np
import pytest

from helpers import basic_config, bitwise_equal, box_for, random_dense_state

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gpu_history(sim, ps=None):
    ps = ps if ps is not None else sim.particles()
    o, p, d = sim.contacts()
    keys = np.where(p >= 0, ps.ids[np.maximum(p, 0)], p.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
    return ps.ids[o].astype(np.uint32), keys, d, (o, p)


def grid_of(sim):
    from oracle.oracle import orc_grid
    g = sim.grid()
    return orc_grid((g.origin[0], g.origin[1], g.origin[2]), g.cell_size, g.nx, g.ny, g.nz)


def check_step_against_oracle(dem, orc, ps0, cfg, steps=1):
    """After each step(): pair set bit-exact vs brute force; forces/torques/history bitwise vs
    the oracle replaying the GPU's own slot order with the GPU's previous history."""
    from oracle.oracle import collide_arrays
    sim = dem.Simulation(ps0, cfg)
    for _ in range(steps):
        ho, hk, hd, _ = gpu_history(sim)
        m = sim.step()
        ps = sim.particles()
        f, t, (to, tk, td), ev = collide_arrays(orc, ps, cfg, grid_of(sim), ho, hk, hd)
        fa = sim.forces()
        assert bitwise_equal(fa.force, f) and bitwise_equal(fa.torque, t)
        go, gk, gd, (o, p) = gpu_history(sim, ps)
        assert np.array_equal(o, ev[0]) and np.array_equal(p.astype(np.uint32), ev[1])
        assert np.array_equal(gk, tk) and bitwise_equal(gd, td)
        # contact completeness (runner.cpp:301-311): unordered pp pairs == brute force
        bi, bj = orc.contact_pairs(ps.positions, ps.radii, binned=True)
        pp = p >= 0
        a, b = np.minimum(o[pp], p[pp]), np.maximum(o[pp], p[pp])
        key = np.unique(a.astype(np.int64) * len(ps.ids) + b)
        assert np.array_equal(key, bi.astype(np.int64) * len(ps.ids) + bj)
        assert m.contacts == len(o) and m.pp_contact_events == int(pp.sum())
    return sim, m


def test_fullsize_262k_dense_bitwise(cuda, orc):
    """BASELINE configs[1] at full size: 262,144 dense spheres, two steps."""
    dem = cuda
    ps, dmax = dem.gen_packing(262144, s=1.8, jit=0.2, seed=1)
    sim, m = check_step_against_oracle(dem, orc, ps, dem.packing_config(dmax), steps=2)
    assert m.contacts / 262144 > 4.5  # dense: ~5.06 contacts per particle


def test_polydisperse_friction_bitwise(cuda, orc):
    """configs[2] shape (radius ratio 1:2, s = 1.4, omega ~ U(-50, 50): friction cap engages),
    K = 32, at 110,592 particles."""
    dem = cuda
    ps, dmax = dem.gen_packing(110592, s=1.4, jit=0.2, poly=True, seed=3, omega_half=50.0)
    sim, m = check_step_against_oracle(dem, orc, ps, dem.packing_config(dmax, poly=True), steps=2)
    assert m.capped_contacts > 0 and m.friction_max_ratio <= 1.0 + 1e-9


def test_fullsize_config3_polydisperse_friction_bitwise(cuda, orc):
    """BASELINE configs[2] at full size: 1,048,576 polydisperse spheres (radius ratio 1:2), sliding
    friction active (omega ~ U(-50, 50)), K = 32; forces, torques, histories and pair sets
    bitwise after two steps."""
    dem = cuda
    ps, dmax = dem.gen_packing(1048576, s=1.4, jit=0.2, poly=True, seed=3, omega_half=50.0)
    sim, m = check_step_against_oracle(dem, orc, ps, dem.packing_config(dmax, poly=True), steps=2)
    assert m.capped_contacts > 0.1 * m.contacts and m.friction_max_ratio <= 1.0 + 1e-9


def test_config4_periodic_lees_edwards_1m_bitwise(cuda, orc):
    """BASELINE configs[3] physics (fully periodic box, Lees-Edwards shear) at 1,048,576 spheres:
    whole steps bitwise against the CPU restatement."""
    from oracle.oracle import OracleSim
    dem = cuda
    ps, L = dem.gen_periodic_packing(1048576, s=1.8, jit=0.2, seed=4)
    cfg = dem.periodic_config(L, shear_rate=1.0)
    sim = dem.Simulation(ps, cfg)
    osim = OracleSim(orc, ps, cfg)
    for _ in range(2):
        m = sim.step()
        om = osim.step()
        assert (m.contacts, m.pp_contact_events) == (om.contacts, om.pp_contact_events)
    a, b = sim.particles(), osim.state()
    assert np.array_equal(a.ids, b.ids)
    assert bitwise_equal(a.positions, b.positions) and bitwise_equal(a.velocities, b.velocities)
    fa = sim.forces()
    fb, tb = osim.forces()
    assert bitwise_equal(fa.force, fb) and bitwise_equal(fa.torque, tb)


@pytest.mark.parametrize("s", [2.35, 2.2, 2.0, 1.6])
def test_density_sweep_pair_sets(cuda, orc, s):
    """configs[4] packing-fraction sweep shape at 32,768 particles: exact pair sets at each s."""
    dem = cuda
    ps, dmax = dem.gen_packing(32768, s=s, jit=0.2, seed=5)
    check_step_against_oracle(dem, orc, ps, dem.packing_config(dmax), steps=1)


def test_restitution_head_on(cuda):
    """test_pipeline.cpp:389-413: eps = 0.9 head-on pair, outgoing speed in (0.855, 0.945)."""
    dem = cuda
    cfg = basic_config(0.1)
    cfg.materials = dem.MaterialTable()
    cfg.materials.add("bead", dem.MaterialParams(0.3, 3.85e5, 1e6, 0.9, 0.0))
    ps = dem.ParticleSet.from_lists([
        (0, (0.045, 0.05, 0.05), (0.5, 0, 0), (0, 0, 0), 0.005, 1.309e-3, 0),
        (1, (0.056, 0.05, 0.05), (-0.5, 0, 0), (0, 0, 0), 0.005, 1.309e-3, 0)])
    sim = dem.Simulation(ps, cfg)
    contact_steps = 0
    for _ in range(1500):
        if sim.step().contacts > 0:
            contact_steps += 1
    assert contact_steps >= 200
    v = sim.particles()
    order = np.argsort(v.ids)
    vv = v.velocities[order]
    v_out = abs(vv[1, 0] - vv[0, 0])
    assert 0.855 < v_out < 0.945


def test_momentum_conservation(cuda):
    """test_pipeline.cpp:309-319: no gravity, no walls, 400 steps, drift <= 1e-9 |p0|."""
    dem = cuda
    cfg = basic_config(box_for(125))
    sim = dem.Simulation(random_dense_state(125, 31), cfg)
    p0 = dem.total_momentum(sim.particles())
    events = 0
    for _ in range(400):
        events += sim.step().contacts
    drift = np.linalg.norm(dem.total_momentum(sim.particles()) - p0)
    assert events > 0 and drift <= 1e-9 * np.linalg.norm(p0)


def test_free_fall_first_step_sees_gravity(cuda):
    """test_pipeline.cpp:285-296."""
    dem = cuda
    cfg = basic_config(1.0)
    cfg.gravity = (0, 0, -9.8)
    cfg.dt = 1e-3
    sim = dem.Simulation(dem.ParticleSet.from_lists([(0, (0.5, 0.5, 0.5), (0, 0, 0), (0, 0, 0), 0.005, 2.0, 0)]), cfg)
    sim.step()
    p = sim.particles()
    assert math.isclose(p.velocities[0, 2], -9.8e-3, rel_tol=1e-12)
    assert math.isclose(p.positions[0, 2], 0.5 - 9.8e-3 * 1e-3, rel_tol=1e-12)


def test_determinism_and_clone(cuda):
    """test_pipeline.cpp:298-307 + the copy constructor (runner.cpp:261-270)."""
    dem = cuda
    cfg = basic_config(box_for(1000))
    a = dem.Simulation(random_dense_state(1000, 21), cfg)
    b = dem.Simulation(random_dense_state(1000, 21), cfg)
    a.steps(10)
    b.steps(10)
    c = a.clone()
    a.steps(7)
    c.steps(7)
    for x, y in ((a.particles(), c.particles()), (a.particles(), a.particles())):
        assert np.array_equal(x.ids, y.ids) and bitwise_equal(x.positions, y.positions)
        assert bitwise_equal(x.angular_velocities, y.angular_velocities)
    b.steps(7)
    assert bitwise_equal(a.particles().positions, b.particles().positions)
    assert bitwise_equal(a.forces().force, c.forces().force)


def test_resting_wall_contact_is_pure_normal(cuda):
    """test_pipeline.cpp:226-244 (the collide half; line 240 is a known reference-test defect,
    SURVEY §4): a particle pressed into the floor gets only a +z wall force, stored under the
    wall's id."""
    dem = cuda
    cfg = basic_config(0.2)
    cfg.rect_walls = [dem.RectWall((0, 0, 0), (0.2, 0, 0), (0, 0.2, 0), 0)]
    r = 0.005
    sim = dem.Simulation(dem.ParticleSet.from_lists([(0, (0.1, 0.1, r - 0.0002), (0, 0, 0), (0, 0, 0), r, 1.3e-3, 0)]), cfg)
    f = sim.forces().force[0]
    assert f[2] > 0.0 and abs(f[0]) < 1e-18 and abs(f[1]) < 1e-18
    o, p, d = sim.contacts()
    assert list(p) == [dem.wall_id(0)]


def test_sliding_on_floor_caps_friction(cuda):
    """test_pipeline.cpp:246-259."""
    dem = cuda
    cfg = basic_config(0.2)
    cfg.rect_walls = [dem.RectWall((0, 0, 0), (0.2, 0, 0), (0, 0.2, 0), 0)]
    r = 0.005
    sim = dem.Simulation(dem.ParticleSet.from_lists([(0, (0.08, 0.1, r - 0.0003), (0.5, 0, 0), (0, 0, 0), r, 1.3e-3, 0)]), cfg)
    mx = max(sim.step().friction_max_ratio for _ in range(40))
    assert 0.5 < mx <= 1.0 + 1e-9


def test_line_wall_pushes_away(cuda):
    """test_pipeline.cpp:271-281."""
    dem = cuda
    cfg = basic_config(0.2)
    cfg.line_walls = [dem.LineWall((0, 0.1, 0.05), (0.2, 0.1, 0.05), 0)]
    sim = dem.Simulation(dem.ParticleSet.from_lists([(0, (0.1, 0.1, 0.05 + 0.0048), (0, 0, 0), (0, 0, 0), 0.005, 1.3e-3, 0)]), cfg)
    f = sim.forces().force[0]
    assert f[2] > 0.0 and abs(f[0]) < 1e-18


def test_clamp_metric(cuda):
    """test_pipeline.cpp:346-354."""
    dem = cuda
    cfg = basic_config(0.05)
    sim = dem.Simulation(dem.ParticleSet.from_lists([(0, (0.2, 0.2, 0.2), (0, 0, 0), (0, 0, 0), 0.005, 1.3e-3, 0)]), cfg)
    m = sim.step()
    assert m.clamps == 1 and m.contacts == 0


def test_config1_statistics_vs_reference(cuda):
    """configs[0] (4,096 settling spheres, 5 walls) built by the reference's own config/lattice
    path (tests/golden/config1.npz): 20 steps on the B200 vs the reference Simulation. Positions
    agree to 1e-12 m and the kinetic-energy / coordination series to 1e-9 relative."""
    dem = cuda
    d = np.load(os.path.join(GOLD, "config1.npz"))
    cfg = dem.SimConfig()
    cfg.dt = float(d["dt"])
    cfg.gravity = tuple(d["gravity"])
    cfg.domain_min = tuple(d["domain_min"])
    cfg.domain_max = tuple(d["domain_max"])
    for k, m in enumerate(d["materials"]):
        cfg.materials.add(f"m{k}", dem.MaterialParams(*m))
    cfg.rect_walls = [dem.RectWall(tuple(w[0:3]), tuple(w[3:6]), tuple(w[6:9]), int(w[9])) for w in d["walls"]]
    ps = dem.ParticleSet(len(d["ids"]))
    ps.ids[:], ps.positions[:], ps.velocities[:] = d["ids"], d["pos"], d["vel"]
    ps.angular_velocities[:], ps.radii[:], ps.masses[:], ps.material_ids[:] = d["omg"], d["rad"], d["mass"], d["mat"]
    sim = dem.Simulation(ps, cfg)
    ke, coord = [], []
    for _ in range(int(d["steps"])):
        m = sim.step()
        ke.append(dem.total_kinetic_energy(sim.particles()))
        coord.append(m.pp_contact_events / len(ps.ids))
    end = sim.particles()
    ia, ib = np.argsort(end.ids), np.argsort(d["end_ids"])
    assert np.abs(end.positions[ia] - d["end_pos"][ib]).max() <= 1e-12
    assert np.allclose(ke, d["ke"], rtol=1e-9, atol=0)
    assert np.allclose(coord, d["coord"], rtol=0, atol=0)
