"""Periodic boxes and Lees-Edwards shear (beyond the reference, whose box is
walled: SPEC.md:383, grid.cpp:60-82). The specification is DESIGN.md §6; the CPU restatement is
oracle/dem_oracle.c (pb_*), checked here against an independent numpy brute force and physical
invariants, and the B200 path is checked bitwise against it.
"""
import numpy as np
import pytest

from helpers import bits, bitwise_equal

import paper_1503_03553_b200 as dem


def min_image(d, L, delta, periodic=7, sheared=True):
    """numpy restatement of the minimum-image rule, vectorised over rows of d."""
    d = d.copy()
    dvx = np.zeros(len(d))
    if periodic & 2:
        up, dn = d[:, 1] > 0.5 * L, d[:, 1] < -0.5 * L
        d[up, 1] -= L
        d[dn, 1] += L
        if sheared:
            d[up, 0] -= delta
            d[dn, 0] += delta
    for k, bit in ((0, 1), (2, 4)):
        if periodic & bit:
            far = np.abs(d[:, k]) > 0.5 * L
            d[far, k] = d[far, k] - L * np.rint(d[far, k] / L)
    return d, dvx


def brute_pairs(pos, rad, L, delta, sheared):
    n = len(pos)
    out = set()
    for i in range(n):
        d, _ = min_image(pos - pos[i], L, delta, sheared=sheared)
        dist = np.sqrt((d * d).sum(axis=1))
        hit = np.nonzero(dist < rad + rad[i])[0]
        for j in hit:
            if j != i:
                out.add((min(i, int(j)), max(i, int(j))))
    return out


def oracle_pairs(osim):
    st = osim.state()
    slot = {int(i): s for s, i in enumerate(st.ids)}
    out = set()
    for h in osim.history():
        if h.partner_key < 0x80000000:
            a, b = slot[h.owner_id], slot[h.partner_key]
            out.add((min(a, b), max(a, b)))
    return out, st


@pytest.mark.parametrize("rate", [0.0, 40.0])
def test_oracle_periodic_pairs_match_brute_force(orc, rate):
    """Every min-image contact is found, including those across the (sheared) faces."""
    from oracle.oracle import OracleSim
    ps, L = dem.gen_periodic_packing(1000, s=1.8, jit=0.2, seed=11)
    cfg = dem.periodic_config(L, shear_rate=rate)
    osim = OracleSim(orc, ps, cfg)
    osim.step(3)
    got, st = oracle_pairs(osim)
    _, delta, steps = osim.pbox()
    assert steps == 3
    want = brute_pairs(st.positions, st.radii, L, delta, sheared=rate != 0.0)
    assert got == want
    # pairs that only exist through a periodic face
    d = st.positions[[a for a, _ in got]] - st.positions[[b for _, b in got]]
    assert (np.abs(d) > 0.5 * L).any()


def test_oracle_periodic_conserves_momentum(orc):
    """No walls, no gravity, no shear: pair forces cancel (Newton's third law holds for the
    reference force law), so total momentum is conserved to rounding in a periodic box."""
    from oracle.oracle import OracleSim
    ps, L = dem.gen_periodic_packing(1000, seed=12)
    cfg = dem.periodic_config(L)
    osim = OracleSim(orc, ps, cfg)
    p0 = (ps.velocities * ps.masses[:, None]).sum(axis=0)
    osim.step(50)
    st = osim.state()
    p1 = (st.velocities * st.masses[:, None]).sum(axis=0)
    scale = (np.abs(ps.velocities) * ps.masses[:, None]).sum()
    assert np.abs(p1 - p0).max() <= 1e-12 * scale
    assert (st.positions >= 0.0).all() and (st.positions < L).all()


def test_oracle_lees_edwards_crossing(orc):
    """A free particle leaving through the top face re-enters at the bottom shifted by -Delta in
    x with its x velocity reduced by the image velocity rate * L_y (and vice versa)."""
    from oracle.oracle import OracleSim
    L, rate, dt = 0.1, 3.0, 1e-3
    ps = dem.ParticleSet.from_lists([
        (0, (0.05, L - 1e-5, 0.05), (0.0, 0.5, 0.0), (0, 0, 0), 0.004, 1e-3, 0),
        (1, (0.02, 2e-5, 0.02), (0.0, -0.5, 0.0), (0, 0, 0), 0.004, 1e-3, 0),
    ])
    cfg = dem.periodic_config(L, shear_rate=rate, dt=dt)
    osim = OracleSim(orc, ps, cfg)
    osim.step(1)
    st = osim.state()
    _, delta, _ = osim.pbox()
    U = rate * L
    assert np.isclose(delta, U * dt)
    by_id = {int(i): s for s, i in enumerate(st.ids)}
    a, b = by_id[0], by_id[1]
    assert st.positions[a, 1] < 0.01 and np.isclose(st.velocities[a, 0], -U)
    assert np.isclose(st.positions[a, 0], 0.05 - delta)
    assert st.positions[b, 1] > L - 0.01 and np.isclose(st.velocities[b, 0], U)
    assert np.isclose(st.positions[b, 0], 0.02 + delta)


def test_periodic_config_validation(cuda=None):
    """Bad periodic configurations are ConfigErrors at the boundary (no GPU needed)."""
    ps, L = dem.gen_periodic_packing(64, seed=1)
    cfg = dem.periodic_config(L, shear_rate=1.0)
    cfg.periodic = 4  # shear without periodic x, y
    with pytest.raises(dem.ConfigError):
        dem.Simulation(ps, cfg)
    cfg = dem.periodic_config(0.02)  # fewer than 3 cells
    with pytest.raises(dem.ConfigError):
        dem.Simulation(ps, cfg)
    cfg = dem.periodic_config(L)
    cfg.collide_variant = dem.BASELINE
    with pytest.raises(dem.ConfigError):
        dem.Simulation(ps, cfg)


def _compare(sim, osim):
    from test_gpu_parity import hist_from_gpu
    a, b = sim.particles(), osim.state()
    assert np.array_equal(a.ids, b.ids)
    for fld in ("positions", "velocities", "angular_velocities"):
        assert bitwise_equal(getattr(a, fld), getattr(b, fld)), fld
    fa = sim.forces()
    fb, tb = osim.forces()
    assert bitwise_equal(fa.force, fb) and bitwise_equal(fa.torque, tb)
    got, _ = hist_from_gpu(sim)
    want = {(h.owner_id, h.partner_key): tuple(bits(np.array(h.delta_t))) for h in osim.history()}
    assert got == want
    k_gpu, _ = sim.order()
    assert np.array_equal(k_gpu, osim.keys())


@pytest.mark.gpu
@pytest.mark.parametrize("n,rate,seed", [(4096, 0.0, 31), (4096, 60.0, 32), (32768, 25.0, 33)])
def test_gpu_periodic_bitwise_vs_oracle(cuda, orc, n, rate, seed):
    """Periodic and Lees-Edwards steps on the B200 equal the CPU restatement bit for bit."""
    from oracle.oracle import OracleSim
    ps, L = dem.gen_periodic_packing(n, s=1.8, jit=0.2, seed=seed)
    cfg = dem.periodic_config(L, shear_rate=rate)
    sim = dem.Simulation(ps, cfg)
    osim = OracleSim(orc, ps, cfg)
    for _ in range(8):
        m = sim.step()
        om = osim.step()
        assert (m.contacts, m.pp_contact_events, m.max_contacts_per_particle) == \
            (om.contacts, om.pp_contact_events, om.max_contacts_per_particle)
        assert m.clamps == om.clamps == 0
        assert m.friction_max_ratio == om.friction_max_ratio
    _compare(sim, osim)
    ext, delta = sim.periodic_box()
    oext, odelta, _ = osim.pbox()
    assert ext == oext and delta == odelta


@pytest.mark.gpu
def test_gpu_periodic_with_walls_and_gravity(cuda, orc):
    """Periodic x, y over a floor (z walled): the periodic and wall paths together."""
    from oracle.oracle import OracleSim
    ps, L = dem.gen_periodic_packing(2197, s=1.9, jit=0.2, seed=34)
    ps.positions[:, 2] += 0.006
    cfg = dem.periodic_config(L, shear_rate=10.0)
    cfg.periodic = 3
    cfg.domain_max = (L, L, L + 0.02)
    cfg.gravity = (0.0, 0.0, -9.81)
    cfg.rect_walls.append(dem.RectWall((0.0, 0.0, 0.0), (L, 0.0, 0.0), (0.0, L, 0.0), 0))
    sim = dem.Simulation(ps, cfg)
    osim = OracleSim(orc, ps, cfg)
    for _ in range(10):
        m = sim.step()
        om = osim.step()
        assert (m.contacts, m.pp_contact_events, m.clamps) == (om.contacts, om.pp_contact_events, om.clamps)
    _compare(sim, osim)
