"""GPU: asynchronous stepping (dem_step_async / dem_sync) and the readback that overlaps the last
step's detection and forces (dem_get_particles after dem_step_async). Same results, bit for bit,
as synchronous steps; errors surface at the next synchronizing call, attributed to the step that
failed, exactly as dem_step reports them."""
import numpy as np
import pytest

from helpers import basic_config, bitwise_equal, box_for, random_dense_state

import paper_1503_03553_b200 as dem

pytestmark = pytest.mark.gpu


def _pair(n=32768, seed=3):
    ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, seed=seed)
    cfg = dem.packing_config(dmax)
    return dem.Simulation(ps, cfg), dem.Simulation(ps, cfg)


def _same_state(a, b):
    pa, pb = a.particles(), b.particles()
    assert np.array_equal(pa.ids, pb.ids)
    for f in ("positions", "velocities", "angular_velocities"):
        assert bitwise_equal(getattr(pa, f), getattr(pb, f)), f
    fa, fb = a.forces(), b.forces()
    assert bitwise_equal(fa.force, fb.force) and bitwise_equal(fa.torque, fb.torque)


def test_async_steps_equal_sync_steps(cuda):
    a, b = _pair()
    for k in range(4):
        ma = a.step()
        b.step_async(1)
        mb = b.sync()
        assert (ma.step, ma.contacts, ma.pp_contact_events, ma.friction_max_ratio) == \
            (mb.step, mb.contacts, mb.pp_contact_events, mb.friction_max_ratio)
    a.steps(3)
    b.step_async(3)
    assert b.step_index() == a.step_index()
    _same_state(a, b)


def test_overlapped_readback(cuda):
    """set -> step_async -> particles_into, the e2e loop: the state read while the step's
    detection and forces run is the step's final state."""
    a, b = _pair(65536, 4)
    host = b.particles()
    for _ in range(3):
        a.set_particles(host)
        a.step()
        want = a.particles()
        b.set_particles(host)
        b.step_async()
        got = b.particles_into(host.contiguous())
        m = b.sync()
        assert m.contacts > 0
        for f in ("positions", "velocities", "angular_velocities", "radii", "masses"):
            assert bitwise_equal(getattr(got, f), getattr(want, f)), f
        assert np.array_equal(got.ids, want.ids)
        host = got
    _same_state(a, b)


def test_async_error_surfaces_at_next_call(cuda):
    """A NaN force fails the first asynchronous step in Integrate; the error comes from the next
    synchronizing call with the same step attribution as dem_step, and later steps did not run."""
    def make():
        sim = dem.Simulation(random_dense_state(64, 3), basic_config(box_for(64)))
        sim.step()
        fa = sim.forces()
        fa.force[5, 0] = np.nan
        sim.set_forces(fa)
        return sim
    a, b = make(), make()
    with pytest.raises(dem.KernelError) as ea:
        a.steps(3)
    b.step_async(3)
    with pytest.raises(dem.KernelError) as eb:
        b.particles()
    assert ea.value.kernel == eb.value.kernel == "Integrate"
    assert ea.value.step == eb.value.step
    assert a.step_index() == b.step_index()
    b.particles()  # the context stays usable


def test_motion_only_set_and_partial_get(cuda):
    """dem_set_particles with ids / radii / masses / materials NULL keeps them per slot; the step
    after it equals the step after a full set, bit for bit. dem_get_particles fills only the
    arrays it is given."""
    a, b = _pair(32768, 5)
    a.steps(2)
    b.steps(2)
    full = a.particles()
    full.positions = full.positions + 1e-7
    a.set_particles(full)
    b.set_motion(full.positions, full.velocities, full.angular_velocities)
    a.step()
    b.step()
    _same_state(a, b)
    part = b.particles()
    part.radii = part.masses = part.material_ids = None
    part.positions[:] = 0.0
    b.particles_into(part)
    assert bitwise_equal(part.positions, a.particles().positions)
    with pytest.raises(ValueError):
        b.set_motion(full.positions[:10], full.velocities[:10], full.angular_velocities[:10])


def test_async_periodic_and_fp32(cuda):
    """The asynchronous graphs of a periodic Lees-Edwards box and of the fp32 mode."""
    ps, L = dem.gen_periodic_packing(27000, s=1.8, jit=0.2, seed=8)
    a, b = dem.Simulation(ps, dem.periodic_config(L, shear_rate=5.0)), dem.Simulation(ps, dem.periodic_config(L, shear_rate=5.0))
    a.steps(3)
    b.step_async(3)
    got = b.particles()
    assert b.sync().step == a.step_index()
    want = a.particles()
    for f in ("positions", "velocities", "angular_velocities"):
        assert bitwise_equal(getattr(got, f), getattr(want, f)), f
    assert a.periodic_box() == b.periodic_box()
    ps2, dmax = dem.gen_packing(27000, s=1.8, jit=0.2, seed=9)
    cfg = dem.packing_config(dmax)
    cfg.precision = 1
    c, d = dem.Simulation(ps2, cfg), dem.Simulation(ps2, cfg)
    c.steps(2)
    d.step_async(2)
    _same_state(c, d)
