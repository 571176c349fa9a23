"""GPU parity: the B200 path (through the C ABI) against the CPU oracles on identical inputs.

Bar (BASELINE.json north_star): contact-pair sets bit-exact; forces, torques and
tangential histories bitwise in fp64 when the accumulation order is the same (the oracle
replays the GPU's own slot order, oracle.cpp:47-105); full steps bitwise against the C
restatement that uses the same canonical (cell, stable id) order; and within 1e-9 relative
(scale = sum of |contributions|) against the reference's own Simulation, whose bitonic tie
order differs.
"""
import numpy as np
import pytest

from helpers import (basic_config, bits, bitwise_equal, box_for, random_dense_state,
                     settling_state, walled_config)

pytestmark = pytest.mark.gpu


def hist_from_gpu(sim):
    """GPU history as {(owner id, partner key): delta_t} plus event list in slot terms."""
    ps = sim.particles()
    o, p, d = sim.contacts()
    ids = ps.ids
    out = {}
    for ow, pa, dt in zip(o, p, d):
        key = int(ids[pa]) if pa >= 0 else (int(pa) & 0xFFFFFFFF)
        out[(int(ids[ow]), key)] = tuple(bits(dt))
    return out, (o, p)


def to_orc_hist(hmap):
    from oracle.oracle import orc_hist
    out = []
    for (ow, key), dtb in hmap.items():
        out.append(orc_hist(ow, key, tuple(np.array(dtb, np.uint64).view(np.float64))))
    return out


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_collide_matches_oracle_bitwise(cuda, orc, seed):
    """tests/test_pipeline.cpp:163-189 on the GPU: two rounds so delta_t history is non-zero."""
    dem = cuda
    cfg = basic_config(box_for(64))
    sim = dem.Simulation(random_dense_state(64, seed), cfg)
    for rnd in range(2):
        before, _ = hist_from_gpu(sim)
        sim.advance_and_collide()
        ps = sim.particles()
        g = sim.grid()
        from oracle.oracle import orc_grid
        og = orc_grid((g.origin[0], g.origin[1], g.origin[2]), g.cell_size, g.nx, g.ny, g.nz)
        f, t, hout, ev = orc.collide(ps, cfg, og, to_orc_hist(before))
        fa = sim.forces()
        assert bitwise_equal(fa.force, f)
        assert bitwise_equal(fa.torque, t)
        after, (o, p) = hist_from_gpu(sim)
        want = {(h.owner_id, h.partner_key): tuple(bits(np.array(h.delta_t))) for h in hout}
        assert after == want
        assert np.array_equal(o, ev[0]) and np.array_equal(p.astype(np.uint32), ev[1])
        assert len(o) > 0


@pytest.mark.parametrize("seed", [1, 2])
def test_collide_matches_reference_oracle_bitwise(cuda, ref, seed):
    """Same check against the reference's own oracle_collide (oracle/_ref)."""
    dem = cuda
    cfg = basic_config(box_for(125))
    sim = dem.Simulation(random_dense_state(125, seed), cfg)
    for rnd in range(2):
        pre = sim.particles()
        o0, p0, d0 = sim.contacts()
        sim.advance_and_collide()
        ps = sim.particles()
        slot_of = {int(i): s for s, i in enumerate(ps.ids)}
        own = np.array([slot_of[int(pre.ids[a])] for a in o0], np.uint32)
        par = np.array([slot_of[int(pre.ids[b])] if b >= 0 else b for b in p0], np.int32)
        g = sim.grid()
        from oracle.oracle import orc_grid
        og = orc_grid((g.origin[0], g.origin[1], g.origin[2]), g.cell_size, g.nx, g.ny, g.nz)
        f, t, tab, ev = ref.oracle_collide(ps, cfg, og, (own, par, d0))
        fa = sim.forces()
        assert bitwise_equal(fa.force, f)
        assert bitwise_equal(fa.torque, t)
        o, p, d = sim.contacts()
        got = {(int(a), int(b)): tuple(bits(x)) for a, b, x in zip(o, p, d)}
        want = {(int(a), int(b)): tuple(bits(x)) for a, b, x in zip(*tab)}
        assert got == want
        assert np.array_equal(o, ev[0]) and np.array_equal(p.astype(np.uint32), ev[1])


@pytest.mark.parametrize("n,seed", [(64, 21), (1331, 61)])
def test_full_steps_bitwise_vs_oracle_sim(cuda, orc, n, seed):
    """Whole step() (integrate, bin, detect, force, reduce) vs the C restatement using the same
    canonical order: state, forces and history bitwise for several steps."""
    from oracle.oracle import OracleSim
    dem = cuda
    cfg = basic_config(box_for(n))
    st = random_dense_state(n, seed)
    sim = dem.Simulation(st, cfg)
    osim = OracleSim(orc, st, cfg)
    for k in range(5):
        m = sim.step()
        om = osim.step()
        assert m.contacts == om.contacts and m.pp_contact_events == om.pp_contact_events
        assert m.max_contacts_per_particle == om.max_contacts_per_particle
        assert m.clamps == om.clamps
        assert m.friction_max_ratio == om.friction_max_ratio
    a, b = sim.particles(), osim.state()
    assert np.array_equal(a.ids, b.ids)
    for fld in ("positions", "velocities", "angular_velocities", "radii", "masses"):
        assert bitwise_equal(getattr(a, fld), getattr(b, fld)), fld
    fa = sim.forces()
    fb, tb = osim.forces()
    assert bitwise_equal(fa.force, fb) and bitwise_equal(fa.torque, tb)
    got, _ = hist_from_gpu(sim)
    want = {(h.owner_id, h.partner_key): tuple(bits(np.array(h.delta_t))) for h in osim.history()}
    assert got == want
    k_gpu, _ = sim.order()
    assert np.array_equal(k_gpu, osim.keys())


def test_walls_bitwise_vs_oracle_sim(cuda, orc):
    """Rectangle + line wall contacts with gravity (pipeline.cpp:244-308) over 30 steps."""
    from oracle.oracle import OracleSim
    dem = cuda
    cfg = walled_config()
    st = settling_state(200, 5)
    sim = dem.Simulation(st, cfg)
    osim = OracleSim(orc, st, cfg)
    wall_events = 0
    for k in range(30):
        m = sim.step()
        om = osim.step()
        assert (m.contacts, m.pp_contact_events) == (om.contacts, om.pp_contact_events)
        wall_events += m.contacts - m.pp_contact_events
    assert wall_events > 0
    a, b = sim.particles(), osim.state()
    assert bitwise_equal(a.positions, b.positions) and bitwise_equal(a.angular_velocities, b.angular_velocities)
    fa = sim.forces()
    fb, tb = osim.forces()
    assert bitwise_equal(fa.force, fb) and bitwise_equal(fa.torque, tb)


def test_pair_set_bit_exact_vs_brute_force(cuda, orc):
    """Contact completeness (runner.cpp:301-311, oracle.cpp:11-24)."""
    dem = cuda
    cfg = basic_config(box_for(512))
    sim = dem.Simulation(random_dense_state(512, 9), cfg)
    sim.step()
    ps = sim.particles()
    o, p, _ = sim.contacts()
    pp = p >= 0
    got = sorted({(min(a, b), max(a, b)) for a, b in zip(o[pp].tolist(), p[pp].tolist())})
    bi, bj = orc.contact_pairs(ps.positions, ps.radii, binned=False)
    assert got == list(zip(bi.tolist(), bj.tolist()))
    assert len(got) > 0


def test_capacity_error_names_collide(cuda):
    """test_pipeline.cpp:356-369: contact_capacity = 1 overflows in the priming pass."""
    dem = cuda
    cfg = basic_config(box_for(27))
    cfg.contact_capacity = 1
    with pytest.raises(dem.CapacityError) as e:
        sim = dem.Simulation(random_dense_state(27, 51), cfg)
        sim.step()
    assert "Collide" in str(e.value)


def test_nonfinite_force_raises_integrate(cuda):
    """test_pipeline.cpp:114-119 through the step: a NaN force aborts in Integrate."""
    dem = cuda
    cfg = basic_config(box_for(64))
    sim = dem.Simulation(random_dense_state(64, 3), cfg)
    fa = sim.forces()
    fa.force[5, 0] = np.nan
    sim.set_forces(fa)
    with pytest.raises(dem.KernelError) as e:
        sim.step()
    assert e.value.kernel == "Integrate"
    assert "non-finite force" in str(e.value)


def test_nonfinite_force_from_the_force_phase_raises_next_integrate(cuda):
    """A force phase that itself produces non-finite forces (two touching particles at +-1e308 m/s:
    the relative velocity overflows) completes; the NEXT step's Integrate raises KernelError
    (pipeline.cpp:35-38), as the reference would. On the B200 path the force kernel pre-integrates
    the next Integrate and defers the error to it; a clone, whose first step
    integrates from its state, must report the same error (kernel, particle)."""
    dem = cuda
    cfg = basic_config(box_for(64))
    ps = random_dense_state(64, 3)
    ps.velocities[:] = 0.0
    a, b = 10, 11  # neighbours in the lattice: make them overlap, then give them opposite huge speeds
    ps.positions[b] = ps.positions[a] + np.array([ps.radii[a] + ps.radii[b] - 1e-4, 0.0, 0.0])
    ps.velocities[a, 0], ps.velocities[b, 0] = 1e308, -1e308
    sim = dem.Simulation(ps, cfg)  # the priming pass computes the non-finite forces without error
    f = sim.forces().force
    assert not np.all(np.isfinite(f))
    twin = sim.clone()
    with pytest.raises(dem.KernelError) as e1:
        sim.step()
    with pytest.raises(dem.KernelError) as e2:
        twin.step()
    assert e1.value.kernel == e2.value.kernel == "Integrate"
    assert str(e1.value) == str(e2.value) and "non-finite force" in str(e1.value)


@pytest.mark.parametrize("seed", [7, 8])
def test_single_loop_variant_bitwise_equals_two_phase(cuda, seed):
    """test_pipeline.cpp:191-220 on the GPU: Alg. 1 (single loop, set_collide_variant(baseline))
    and the two-phase kernels give bitwise identical states, forces and histories; switching
    variants mid-run keeps the history compatible."""
    dem = cuda
    cfg = basic_config(box_for(1000))
    a = dem.Simulation(random_dense_state(1000, seed), cfg)
    cfg_b = basic_config(box_for(1000))
    cfg_b.collide_variant = dem.BASELINE
    b = dem.Simulation(random_dense_state(1000, seed), cfg_b)
    for k in range(6):
        ma, mb = a.step(), b.step()
        assert (ma.contacts, ma.pp_contact_events, ma.max_contacts_per_particle) == \
            (mb.contacts, mb.pp_contact_events, mb.max_contacts_per_particle)
        assert ma.friction_max_ratio == mb.friction_max_ratio and ma.capped_contacts == mb.capped_contacts
        if k == 3:
            b.set_collide_variant(dem.TWO_PHASE)
            a.set_collide_variant(dem.BASELINE)
    pa, pb = a.particles(), b.particles()
    assert bitwise_equal(pa.positions, pb.positions) and bitwise_equal(pa.angular_velocities, pb.angular_velocities)
    assert bitwise_equal(a.forces().force, b.forces().force) and bitwise_equal(a.forces().torque, b.forces().torque)
    ha, _ = hist_from_gpu(a)
    hb, _ = hist_from_gpu(b)
    assert ha == hb


def test_per_kernel_composition_equals_force_phase(cuda, orc):
    """The reference's per-kernel API (pipeline.hpp:77-86) composed as tests/test_pipeline.cpp
    advance_to_collide + kernel_collide / kernel_collide_rectangle / kernel_collide_line does:
    bitwise equal to the fused phase, and to the C restatement's phase with the same flags."""
    from oracle.oracle import OracleSim
    dem = cuda
    cfg = walled_config()
    st = settling_state(300, 17)
    a = dem.Simulation(st, cfg)
    b = dem.Simulation(st, cfg)
    o = OracleSim(orc, st, cfg)
    for rnd in range(4):
        a.kernel_integrate()
        a.kernel_calc_hash()
        a.kernel_bitonic_sort()
        a.kernel_find_cell_bounds_and_reorder()
        a.zero_forces()
        a.kernel_force_gravity()
        a.kernel_initialize_contact_ids()
        a.kernel_collide(dem.BASELINE if rnd % 2 else dem.TWO_PHASE, False)
        a.kernel_collide_rectangle()
        a.kernel_collide_line()
        b.force_phase(dem.PHASE_STEP)
        o.force_phase(31)
    pa, pb, po = a.particles(), b.particles(), o.state()
    for fld in ("positions", "velocities", "angular_velocities"):
        assert bitwise_equal(getattr(pa, fld), getattr(pb, fld)) and bitwise_equal(getattr(pa, fld), getattr(po, fld))
    fa, fb = a.forces(), b.forces()
    fo, to = o.forces()
    assert bitwise_equal(fa.force, fb.force) and bitwise_equal(fa.force, fo) and bitwise_equal(fa.torque, to)
    # a kernel earlier in pipeline order starts a new phase: integrate, then integrate again
    a.kernel_integrate()
    a.kernel_integrate()
    b.force_phase(dem.PHASE_INTEGRATE)
    b.force_phase(dem.PHASE_INTEGRATE)
    assert bitwise_equal(a.particles().positions, b.particles().positions)
