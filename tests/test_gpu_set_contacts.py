"""GPU: dem_set_contacts — the mutable ContactTable the reference's bench restores
(runner.cpp:131-132). Restoring a saved table reproduces the step bit for bit, and an arbitrary
table (scaled delta_t, dropped entries) is merged exactly as oracle_collide merges it
(tests/test_pipeline.cpp:163-189 replay on the GPU's slot order)."""
import numpy as np
import pytest

from helpers import basic_config, bits, bitwise_equal, box_for, random_dense_state
from test_gpu_parity import hist_from_gpu, to_orc_hist

import paper_1503_03553_b200 as dem

pytestmark = pytest.mark.gpu


def test_restored_table_reproduces_the_step(cuda):
    ps, dmax = dem.gen_packing(32768, s=1.8, jit=0.2, seed=9, omega_half=20.0)
    a = dem.Simulation(ps, dem.packing_config(dmax))
    a.steps(3)
    b = a.clone()
    o, p, d = a.contacts()
    assert len(o) > 0 and np.abs(d).max() > 0
    a.step()
    b.set_contacts([], [], np.zeros((0, 3)))  # wipe, then restore
    b.set_contacts(o, p, d)
    b.step()
    pa, pb = a.particles(), b.particles()
    for f in ("positions", "velocities", "angular_velocities"):
        assert bitwise_equal(getattr(pa, f), getattr(pb, f)), f
    fa, fb = a.forces(), b.forces()
    assert bitwise_equal(fa.force, fb.force) and bitwise_equal(fa.torque, fb.torque)
    assert hist_from_gpu(a)[0] == hist_from_gpu(b)[0]


def test_modified_table_matches_oracle_collide(cuda, orc):
    cfg = basic_config(box_for(343))
    sim = dem.Simulation(random_dense_state(343, 17), cfg)
    sim.steps(2)
    o, p, d = sim.contacts()
    keep = np.arange(len(o)) % 3 != 0  # drop a third, scale the rest
    sim.set_contacts(o[keep], p[keep], 1.5 * d[keep])
    before, _ = hist_from_gpu(sim)
    assert len(before) == int(keep.sum())
    sim.advance_and_collide()
    ps = sim.particles()
    g = sim.grid()
    from oracle.oracle import orc_grid
    og = orc_grid((g.origin[0], g.origin[1], g.origin[2]), g.cell_size, g.nx, g.ny, g.nz)
    f, t, hout, ev = orc.collide(ps, cfg, og, to_orc_hist(before))
    fa = sim.forces()
    assert bitwise_equal(fa.force, f) and bitwise_equal(fa.torque, t)
    after, _ = hist_from_gpu(sim)
    assert after == {(h.owner_id, h.partner_key): tuple(bits(np.array(h.delta_t))) for h in hout}


def test_bad_tables_rejected(cuda):
    cfg = basic_config(box_for(64))
    sim = dem.Simulation(random_dense_state(64, 3), cfg)
    o, p, d = sim.contacts()
    assert len(o) > 1
    with pytest.raises(Exception):
        sim.set_contacts([0, 0], [1, 1], np.zeros((2, 3)))  # repeated partner
    with pytest.raises(Exception):
        sim.set_contacts([10 ** 6], [1], np.zeros((1, 3)))  # owner out of range
    k = cfg.contact_capacity
    with pytest.raises(Exception):
        sim.set_contacts([0] * (k + 1), list(range(1, k + 2)), np.zeros((k + 1, 3)))  # over capacity
    sim.set_contacts(o, p, d)  # still usable
    sim.step()
