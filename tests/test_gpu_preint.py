"""GPU: the force kernel's pre-integration — the next step's Integrate done where the
forces are computed — is the reference's Integrate bit for bit, and every host-side change of the
state or the forces between steps is honoured (pipeline.cpp:31-44: a step integrates the CURRENT
particles with the CURRENT forces).

* a clone (whose first step integrates from its state, not from the pre-integrated buffer) steps
  bitwise like the original, in the walled box, the periodic Lees-Edwards box (where the wrap is
  applied by the next phase) and the fp32 mode;
* after dem_set_particles / dem_set_forces the step's new positions and velocities are exactly
  those of the reference's Integrate expressions (evaluated here in numpy, fp64, left to right)
  applied to the uploaded state / forces."""
import numpy as np
import pytest

from helpers import bitwise_equal

import paper_1503_03553_b200 as dem

pytestmark = pytest.mark.gpu


def _walled(n=32768, seed=11):
    ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, seed=seed)
    return ps, dem.packing_config(dmax)


def _same(a, b):
    pa, pb = a.particles(), b.particles()
    assert np.array_equal(pa.ids, pb.ids)
    for f in ("positions", "velocities", "angular_velocities"):
        assert bitwise_equal(getattr(pa, f), getattr(pb, f)), f
    fa, fb = a.forces(), b.forces()
    assert bitwise_equal(fa.force, fb.force) and bitwise_equal(fa.torque, fb.torque)


@pytest.mark.parametrize("mode", ["walled", "periodic_le", "fp32"])
def test_clone_integrates_like_the_pre_integrated_original(cuda, mode):
    if mode == "periodic_le":
        ps, L = dem.gen_periodic_packing(32768, s=1.8, jit=0.2, seed=12)
        cfg = dem.periodic_config(L, shear_rate=50.0)
    else:
        ps, cfg = _walled()
        cfg.precision = 1 if mode == "fp32" else 0
    a = dem.Simulation(ps, cfg)
    a.steps(2)
    for _ in range(3):
        b = a.clone()  # its next Integrate reads the state, not the pre-integrated buffer
        a.step()
        b.step()
        _same(a, b)


def _integrate(s, f, t, dt):
    """pipeline.cpp:31-44 in the reference's order (numpy fp64, no contraction)."""
    m, r = s.masses[:, None], s.radii[:, None]
    v = s.velocities + f * (dt / m)
    x = s.positions + v * dt
    inertia = 0.4 * s.masses * s.radii * s.radii
    w = s.angular_velocities + t * (dt / inertia)[:, None]
    return x, v, w


def _by_id(s):
    o = np.argsort(s.ids)
    return o


def test_set_particles_between_steps_is_integrated(cuda):
    ps, cfg = _walled()
    sim = dem.Simulation(ps, cfg)
    sim.steps(2)
    s = sim.particles()
    rng = np.random.default_rng(5)
    s.velocities[:] = s.velocities + rng.uniform(-1e-3, 1e-3, s.velocities.shape)
    s.angular_velocities[:] = -s.angular_velocities
    sim.set_particles(s)
    fa = sim.forces()
    x, v, w = _integrate(s, fa.force, fa.torque, cfg.dt)
    sim.step()
    after = sim.particles()
    oa, ob = _by_id(after), _by_id(s)
    assert np.array_equal(after.ids[oa], s.ids[ob])
    assert bitwise_equal(after.positions[oa], x[ob])
    assert bitwise_equal(after.velocities[oa], v[ob])
    assert bitwise_equal(after.angular_velocities[oa], w[ob])


def test_set_forces_between_steps_is_integrated(cuda):
    ps, cfg = _walled()
    sim = dem.Simulation(ps, cfg)
    sim.steps(2)
    s = sim.particles()
    fa = sim.forces()
    fa.force[:] = 0.5 * fa.force + 1e-6
    fa.torque[:] = -fa.torque
    sim.set_forces(fa)
    x, v, w = _integrate(s, fa.force, fa.torque, cfg.dt)
    sim.step()
    after = sim.particles()
    oa, ob = _by_id(after), _by_id(s)
    assert bitwise_equal(after.positions[oa], x[ob])
    assert bitwise_equal(after.velocities[oa], v[ob])
    assert bitwise_equal(after.angular_velocities[oa], w[ob])
