"""GPU: the slab decomposition on one B200 through the loopback transport — 2, 3 and
4 slab contexts on the same device — is bitwise identical to the single-context run: positions,
velocities, forces, torques and tangential histories of every particle, by stable id."""
import numpy as np
import pytest

from helpers import bits, bitwise_equal

pytestmark = pytest.mark.gpu


def by_id(ids, *arrays):
    o = np.argsort(ids)
    return [a[o] for a in arrays]


def single_run(dem, ps, cfg, steps):
    sim = dem.Simulation(ps, cfg)
    for _ in range(steps):
        sim.step()
    s = sim.particles()
    fa = sim.forces()
    o, p, d = sim.contacts()
    keys = np.where(p >= 0, s.ids[np.maximum(p, 0)], p.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
    hist = {(int(a), int(b)): tuple(bits(x)) for a, b, x in zip(s.ids[o], keys, d)}
    return s, fa.force, fa.torque, hist


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_slab_loopback_bitwise_equals_single_gpu(cuda, nranks):
    dem = cuda
    from paper_1503_03553_b200.slab import LoopbackTransport, SlabDriver, build_local_slabs
    ps, dmax = dem.gen_packing(32768, s=1.8, jit=0.2, seed=11)
    cfg = dem.packing_config(dmax)
    steps = 6
    s1, f1, t1, h1 = single_run(dem, ps, cfg, steps)
    ranks, bounds, g = build_local_slabs(ps, cfg, nranks, range(nranks))
    drv = SlabDriver(ranks, LoopbackTransport(ranks))
    drv.prime()
    contacts = 0
    for _ in range(steps):
        ms = drv.step()
        contacts = sum(m.contacts for m in ms)
    parts = [rk.owned() for rk in ranks]
    ids = np.concatenate([p[0].ids for p in parts])
    assert len(ids) == len(s1.ids) and len(np.unique(ids)) == len(ids)
    pos = np.concatenate([p[0].positions for p in parts])
    vel = np.concatenate([p[0].velocities for p in parts])
    f = np.concatenate([p[1] for p in parts])
    t = np.concatenate([p[2] for p in parts])
    a = by_id(ids, ids, pos, vel, f, t)
    b = by_id(s1.ids, s1.ids, s1.positions, s1.velocities, f1, t1)
    assert np.array_equal(a[0], b[0])
    for x, y in zip(a[1:], b[1:]):
        assert bitwise_equal(x, y)
    hist = {}
    for p in parts:
        for ow, k, d in zip(*p[3]):
            hist[(int(ow), int(k))] = tuple(bits(d))
    assert hist == h1
    assert contacts == len(h1)
    # particles actually crossed slab boundaries at least as ghosts
    assert all(rk.send_count["ghost"][0] + rk.send_count["ghost"][1] > 0 for rk in ranks)


def test_slab_migration_and_walls_with_gravity(cuda):
    """Settling pack under gravity with walls, 3 slabs, 40 steps: particles migrate between
    slabs (history rows move with them) and the result still equals one context bitwise."""
    dem = cuda
    from helpers import walled_config, settling_state
    from paper_1503_03553_b200.slab import LoopbackTransport, SlabDriver, build_local_slabs
    cfg = walled_config()
    ps = settling_state(600, 8)
    ps.velocities[:, 2] = -2.0  # fast fall: plane crossings within the run
    steps = 40
    s1, f1, t1, h1 = single_run(dem, ps, cfg, steps)
    ranks, bounds, g = build_local_slabs(ps, cfg, 3, range(3))
    drv = SlabDriver(ranks, LoopbackTransport(ranks))
    drv.prime()
    migrated = 0
    for _ in range(steps):
        drv.step()
        migrated += sum(rk.send_count["migrant"][0] + rk.send_count["migrant"][1] for rk in ranks)
    parts = [rk.owned() for rk in ranks]
    ids = np.concatenate([p[0].ids for p in parts])
    pos = np.concatenate([p[0].positions for p in parts])
    f = np.concatenate([p[1] for p in parts])
    a = by_id(ids, ids, pos, f)
    b = by_id(s1.ids, s1.ids, s1.positions, f1)
    assert np.array_equal(a[0], b[0]) and bitwise_equal(a[1], b[1]) and bitwise_equal(a[2], b[2])
    hist = {}
    for p in parts:
        for ow, k, d in zip(*p[3]):
            hist[(int(ow), int(k))] = tuple(bits(d))
    assert hist == h1
    assert migrated > 0


@pytest.mark.parametrize("nranks,rate", [(1, 30.0), (2, 30.0), (3, 0.0), (4, 30.0)])
def test_slab_periodic_ring_bitwise_equals_single_gpu(cuda, nranks, rate):
    """Config 4's decomposition: a fully periodic (Lees-Edwards sheared) box cut into slabs along
    z, the slabs forming a ring. Fast z motion makes particles cross the periodic
    z face between the last and the first slab; the result equals one context bitwise."""
    dem = cuda
    from paper_1503_03553_b200.slab import LoopbackTransport, SlabDriver, build_local_slabs
    ps, L = dem.gen_periodic_packing(27000, s=1.8, jit=0.2, seed=51)
    ps.velocities[:, 2] += np.where(ps.ids % 2 == 0, 40.0, -40.0)  # cross z planes quickly
    cfg = dem.periodic_config(L, shear_rate=rate)
    steps = 25
    s1, f1, t1, h1 = single_run(dem, ps, cfg, steps)
    ranks, bounds, g = build_local_slabs(ps, cfg, nranks, range(nranks))
    assert g.ring
    drv = SlabDriver(ranks, LoopbackTransport(ranks, ring=True))
    drv.prime()
    migrated = 0
    for _ in range(steps):
        drv.step()
        migrated += sum(rk.send_count["migrant"][0] + rk.send_count["migrant"][1] for rk in ranks)
    parts = [rk.owned() for rk in ranks]
    ids = np.concatenate([p[0].ids for p in parts])
    assert len(ids) == len(s1.ids) and len(np.unique(ids)) == len(ids)
    pos = np.concatenate([p[0].positions for p in parts])
    vel = np.concatenate([p[0].velocities for p in parts])
    f = np.concatenate([p[1] for p in parts])
    t = np.concatenate([p[2] for p in parts])
    a = by_id(ids, ids, pos, vel, f, t)
    b = by_id(s1.ids, s1.ids, s1.positions, s1.velocities, f1, t1)
    assert np.array_equal(a[0], b[0])
    for x, y in zip(a[1:], b[1:]):
        assert bitwise_equal(x, y)
    hist = {}
    for p in parts:
        for ow, k, d in zip(*p[3]):
            hist[(int(ow), int(k))] = tuple(bits(d))
    assert hist == h1
    assert migrated > 0
