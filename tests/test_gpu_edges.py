"""GPU edge cases of the hot path against the CPU restatement (oracle/): an empty set, a single
particle, pairs placed ulps around the contact boundary (the exact classification's ambiguous
band), coincident centres (DegenerateContactError, geometry.cpp:32), a contact row filled to
exactly K and one past it (CapacityError, contact_table.cpp:15-35), and particle counts that do not
fill the last 32-slot tile."""
import numpy as np
import pytest

from helpers import basic_config, box_for, random_dense_state
from test_periodic import _compare

import paper_1503_03553_b200 as dem

pytestmark = pytest.mark.gpu


def _pair_state(n_pairs, seed):
    """n_pairs two-particle clusters; in each the centre distance is reach * (1 + k 2^-52),
    k in -4..4, along a random direction (distance rounding puts some exactly on reach)."""
    rng = np.random.default_rng(seed)
    rows = []
    r = 0.005
    pid = 0
    for c in range(n_pairs):
        k = (c % 9) - 4
        centre = np.array([0.05 + 0.04 * (c % 10), 0.05 + 0.04 * ((c // 10) % 10), 0.05 + 0.04 * (c // 100)])
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        d = 2 * r * (1.0 + k * 2.0 ** -52)
        a, b = centre - 0.5 * d * u, centre + 0.5 * d * u
        v = rng.uniform(-0.1, 0.1, 3)
        rows.append((pid, tuple(a), tuple(v), (0.0, 0.0, 0.0), r, 1e-3, 0))
        rows.append((pid + 1, tuple(b), tuple(-v), (0.0, 0.0, 0.0), r, 1e-3, 0))
        pid += 2
    return dem.ParticleSet.from_lists(rows)


def test_empty_set(cuda, orc):
    from oracle.oracle import OracleSim, OracleError
    cfg = basic_config(0.1)
    # no radius to size the cells from (grid.cpp:10-28): a ConfigError in both implementations
    with pytest.raises(dem.ConfigError):
        dem.Simulation(dem.ParticleSet(0), cfg)
    with pytest.raises(OracleError) as eo:
        OracleSim(orc, dem.ParticleSet(0), cfg)
    assert eo.value.code == 1
    cfg.grid_cell_size = 0.01
    sim = dem.Simulation(dem.ParticleSet(0), cfg)
    m = sim.step()
    assert (m.step, m.contacts, m.pp_contact_events) == (1, 0, 0)
    sim.step_async(2)
    assert sim.sync().contacts == 0
    assert sim.step_index() == 3
    assert len(sim.particles().ids) == 0
    assert sim.forces().force.shape == (0, 3)


@pytest.mark.parametrize("n", [1, 33, 129, 160, 1000, 4097])
def test_ragged_counts_bitwise(cuda, orc, n):
    """1 particle (free fall), and counts that leave the last 32-slot tile partly empty or the last
    4-tile detection block with one tile (129, 160, 4097)."""
    from oracle.oracle import OracleSim
    cfg = basic_config(box_for(n))
    cfg.gravity = (0.0, 0.0, -9.81)
    ps = random_dense_state(n, 70 + n)
    sim = dem.Simulation(ps, cfg)
    osim = OracleSim(orc, ps, cfg)
    for _ in range(5):
        m, om = sim.step(), osim.step()
        assert (m.contacts, m.pp_contact_events) == (om.contacts, om.pp_contact_events)
    _compare(sim, osim)


def test_contact_boundary_ulps(cuda, orc):
    """Pairs at reach (1 + k 2^-52): contact iff RN(sqrt(d.d)) < reach, decided as the reference
    does, with forces and histories bitwise."""
    from oracle.oracle import OracleSim
    ps = _pair_state(450, 3)
    cfg = basic_config(0.5)
    sim = dem.Simulation(ps, cfg)
    osim = OracleSim(orc, ps, cfg)
    hits = 0
    for _ in range(3):
        m, om = sim.step(), osim.step()
        assert (m.contacts, m.pp_contact_events) == (om.contacts, om.pp_contact_events)
        hits += m.pp_contact_events
    assert 0 < hits < 3 * 450 * 2  # some pairs touch, some do not
    _compare(sim, osim)


def test_coincident_centres_raise_degenerate(cuda, orc):
    from oracle.oracle import OracleSim, OracleError
    rows = [(0, (0.05, 0.05, 0.05), (0, 0, 0), (0, 0, 0), 0.005, 1e-3, 0),
            (1, (0.05, 0.05, 0.05), (0, 0, 0), (0, 0, 0), 0.005, 1e-3, 0),
            (2, (0.02, 0.02, 0.02), (0, 0, 0), (0, 0, 0), 0.005, 1e-3, 0)]
    ps = dem.ParticleSet.from_lists(rows)
    cfg = basic_config(0.1)
    with pytest.raises(dem.DegenerateContactError) as e:
        dem.Simulation(ps, cfg)  # the constructor's priming pass detects it
    assert e.value.kernel == "Collide"
    with pytest.raises(OracleError) as eo:
        OracleSim(orc, ps, cfg)
    assert eo.value.code == 4


@pytest.mark.parametrize("k_neighbours,ok", [(4, True), (5, False)])
def test_capacity_exactly_full_and_one_over(cuda, orc, k_neighbours, ok):
    """A centre particle touching k neighbours with contact_capacity 4."""
    from oracle.oracle import OracleSim, OracleError
    r = 0.005
    c = np.array([0.05, 0.05, 0.05])
    dirs = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    rows = [(0, tuple(c), (0, 0, 0), (0, 0, 0), r, 1e-3, 0)]
    for q in range(k_neighbours):
        rows.append((q + 1, tuple(c + 1.9 * r * np.array(dirs[q], float)), (0, 0, 0), (0, 0, 0), r, 1e-3, 0))
    ps = dem.ParticleSet.from_lists(rows)
    cfg = basic_config(0.1)
    cfg.contact_capacity = 4
    if ok:
        sim = dem.Simulation(ps, cfg)
        osim = OracleSim(orc, ps, cfg)
        m, om = sim.step(), osim.step()
        assert m.max_contacts_per_particle == om.max_contacts_per_particle == 4
        _compare(sim, osim)
    else:
        with pytest.raises(dem.CapacityError) as e:
            dem.Simulation(ps, cfg)
        assert e.value.kernel == "Collide"
        with pytest.raises(OracleError) as eo:
            OracleSim(orc, ps, cfg)
        assert eo.value.code == 3


def _icosahedron_cluster(rel, centre=(0.05, 0.05, 0.05), box=None):
    """A centre sphere and 12 neighbours at the icosahedron's vertices, neighbour q at distance
    reach (1 + rel[q]) from the centre, the neighbours 1.05 reach apart from each other
    (positions wrapped into [0, box) for a periodic box)."""
    r = 0.005
    c = np.array(centre, float)
    g = (1 + 5 ** 0.5) / 2
    verts = [(0, 1, g), (0, -1, g), (0, 1, -g), (0, -1, -g), (1, g, 0), (-1, g, 0), (1, -g, 0), (-1, -g, 0),
             (g, 0, 1), (-g, 0, 1), (g, 0, -1), (-g, 0, -1)]
    rows = [(0, tuple(c), (0.0, 0.0, 0.0), (0.0, 0.0, 0.0), r, 1e-3, 0)]
    for q, (v, e) in enumerate(zip(verts, rel)):
        u = np.array(v, float) / np.linalg.norm(v)
        x = c + 2 * r * (1.0 + e) * u
        if box is not None:
            x = np.mod(x, box)
        rows.append((q + 1, tuple(x), (0.0, 0.0, 0.0), (0.0, 0.0, 0.0), r, 1e-3, 0))
    return dem.ParticleSet.from_lists(rows)


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("n_touch,ok", [(3, True), (5, False)])
def test_prefilter_overflow_takes_exact_walk(cuda, orc, n_touch, ok, periodic):
    """The centre has 12 fp32-prefilter survivors against a kept-list capacity of K = 4: n_touch
    neighbours overlap it and the other 12 - n_touch sit at reach (1 + 1e-7 .. 1e-6), inside the
    prefilter's conservative bound but outside the reference's d2 screen (reach2 (1 + 1e-9),
    pipeline.cpp:144-149). The detection lane falls back to the exact one-stage walk, which finds
    the reference's contacts (forces bitwise) or raises its CapacityError (5 screen passers > 4).
    Periodic: the cluster straddles the corner of a periodic box, so the centre's warp takes the
    wrapped (minimum-image) walk and its fallback."""
    from oracle.oracle import OracleSim, OracleError
    rel = [-(6 - q) * 2.0 ** -44 for q in range(n_touch)] + [(q + 1) * 1e-7 for q in range(12 - n_touch)]
    if periodic:
        ps = _icosahedron_cluster(rel, centre=(0.001, 0.002, 0.003), box=0.1)
        cfg = dem.periodic_config(0.1)
    else:
        ps = _icosahedron_cluster(rel)
        cfg = basic_config(0.1)
    cfg.contact_capacity = 4
    if ok:
        sim = dem.Simulation(ps, cfg)
        osim = OracleSim(orc, ps, cfg)
        for _ in range(3):
            m, om = sim.step(), osim.step()
            assert (m.contacts, m.max_contacts_per_particle) == (om.contacts, om.max_contacts_per_particle)
        assert m.max_contacts_per_particle == n_touch
        _compare(sim, osim)
    else:
        with pytest.raises(dem.CapacityError) as e:
            dem.Simulation(ps, cfg)
        assert e.value.kernel == "Collide"
        with pytest.raises(OracleError) as eo:
            OracleSim(orc, ps, cfg)
        assert eo.value.code == 3


def test_set_particles_validates_on_device(cuda):
    """dem_set_particles validates every uploaded particle (ParticleSet::validate,
    particle_set.cpp:40-58, plus unique ids below the wall keys): a rejected upload raises
    ConfigError and the context refuses to step until a valid state is uploaded."""
    cfg = basic_config(box_for(64))
    ps = random_dense_state(64, 5)
    sim = dem.Simulation(ps, cfg)
    sim.step()
    good = sim.particles()
    for field, value, msg in (("material_ids", 7, "bad material"), ("radii", -1.0, "radius"),
                              ("masses", 0.0, "mass"), ("velocities", np.inf, "non-finite"),
                              ("ids", 0xFFFFFFF0, "wall-key")):
        bad = good.copy()
        getattr(bad, field)[11] = value
        with pytest.raises(dem.ConfigError, match=msg):
            sim.set_particles(bad)
        with pytest.raises(dem.ConfigError):
            sim.step()
        sim.set_particles(good)
        sim.step()
    # duplicates: screened on the device by an id bitmap, confirmed exactly on the host
    dup = good.copy()
    dup.ids[3] = dup.ids[4]
    with pytest.raises(dem.ConfigError, match="duplicate"):
        sim.set_particles(dup)
    with pytest.raises(dem.ConfigError):
        sim.step()
    # a hash collision that is no duplicate (ids equal modulo the bitmap size) is accepted
    far = good.copy()
    far.ids[5] = far.ids[6] + (1 << 20)
    sim.set_particles(far)
    sim.step()
    sim.set_particles(good)
    sim.step()
    # particles_into checks the caller's arrays before writing through their pointers
    out = dem.ParticleSet(64)
    out.positions = np.zeros((64, 3), np.float32)
    with pytest.raises(ValueError):
        sim.particles_into(out)
    out = dem.ParticleSet(63)
    with pytest.raises(ValueError):
        sim.particles_into(out)
    assert sim.particles_into(dem.ParticleSet(64)).size() == 64


@pytest.mark.parametrize("periodic", [0, 7])
def test_largest_contact_capacity(cuda, orc, periodic):
    """The largest accepted row capacity (K = 80, k_detect's shared-memory bound) runs."""
    n = 512
    cfg = basic_config(box_for(n))
    cfg.contact_capacity = 80
    cfg.periodic = periodic
    if periodic:
        cfg.gravity = (0.0, 0.0, 0.0)
    ps = random_dense_state(n, 9)
    sim = dem.Simulation(ps, cfg)
    m = sim.step()
    assert m.contacts > 0


def _poly_pair_state(n_pairs, seed):
    """Polydisperse two-particle clusters (radius ratio up to 1:2, masses ~ r^3) at centre distance
    (r_a + r_b)(1 + e) with e = k 2^-52 (k = -4..4) and e = +-2^-41, +-2^-39 (the edges of the
    sqrt-free classification's 2^-40 band): k_detect's non-monodisperse bounds (MONO = false)."""
    rng = np.random.default_rng(seed)
    eps = [k * 2.0 ** -52 for k in range(-4, 5)] + [2.0 ** -41, -(2.0 ** -41), 2.0 ** -39, -(2.0 ** -39)]
    rows, pid = [], 0
    for c in range(n_pairs):
        e = eps[c % len(eps)]
        ra, rb = 0.005 * rng.uniform(0.5, 1.0), 0.005 * rng.uniform(0.5, 1.0)
        centre = np.array([0.05 + 0.04 * (c % 10), 0.05 + 0.04 * ((c // 10) % 10), 0.05 + 0.04 * (c // 100)])
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        d = (ra + rb) * (1.0 + e)
        a, b = centre - 0.5 * d * u, centre + 0.5 * d * u
        rows.append((pid, tuple(a), (0.0, 0.0, 0.0), (0.0, 0.0, 0.0), ra, 1e-3 * (ra / 0.005) ** 3, 0))
        rows.append((pid + 1, tuple(b), (0.0, 0.0, 0.0), (0.0, 0.0, 0.0), rb, 1e-3 * (rb / 0.005) ** 3, 0))
        pid += 2
    return dem.ParticleSet.from_lists(rows)


def test_contact_boundary_ulps_polydisperse(cuda, orc):
    """The polydisperse classification path (per-candidate reach and bounds) decides pairs around
    the contact boundary exactly as the reference: the priming pass (positions exactly as built)
    and two steps bitwise against the CPU restatement."""
    from oracle.oracle import OracleSim
    ps = _poly_pair_state(520, 11)
    cfg = basic_config(0.5)
    sim = dem.Simulation(ps, cfg)
    osim = OracleSim(orc, ps, cfg)
    o, _, _ = sim.contacts()
    n_prime = len(o)
    assert n_prime == len(osim.history())
    assert 0 < n_prime < 2 * 520  # some pairs touch, some do not
    _compare(sim, osim)
    for _ in range(2):
        m, om = sim.step(), osim.step()
        assert (m.contacts, m.pp_contact_events) == (om.contacts, om.pp_contact_events)
        _compare(sim, osim)
