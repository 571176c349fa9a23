"""GPU: the host-free sharded step (dem_create_sharded) — record
counts on the device, peer stores into the neighbours' inboxes, flag waits in the stream, one CUDA
graph per step — is bitwise identical to one context: positions, velocities, forces, torques and
tangential histories of every particle, by stable id. Ranks of one process (connect_local) and one
process per rank (CUDA-IPC inboxes, handles all-gathered over gloo); walled boxes with migrations
and a periodic Lees-Edwards ring."""
import os
import socket
import tempfile

import numpy as np
import pytest

from helpers import bits, bitwise_equal
from test_gpu_slab import by_id, single_run

pytestmark = pytest.mark.gpu


def _gather(parts):
    ids = np.concatenate([p[0].ids for p in parts])
    pos = np.concatenate([p[0].positions for p in parts])
    vel = np.concatenate([p[0].velocities for p in parts])
    f = np.concatenate([p[1] for p in parts])
    t = np.concatenate([p[2] for p in parts])
    hist = {}
    for p in parts:
        for ow, k, d in zip(*p[3]):
            hist[(int(ow), int(k))] = tuple(bits(d))
    return ids, pos, vel, f, t, hist


def _assert_same(parts, s1, f1, t1, h1):
    ids, pos, vel, f, t, hist = _gather(parts)
    assert len(ids) == len(s1.ids) and len(np.unique(ids)) == len(ids)
    a = by_id(ids, ids, pos, vel, f, t)
    b = by_id(s1.ids, s1.ids, s1.positions, s1.velocities, f1, t1)
    assert np.array_equal(a[0], b[0])
    for x, y in zip(a[1:], b[1:]):
        assert bitwise_equal(x, y)
    assert hist == h1


def _case(dem, kind):
    if kind == "walled":
        ps, dmax = dem.gen_packing(32768, s=1.8, jit=0.2, seed=21)
        ps.velocities[:, 2] += np.where(ps.ids % 2 == 0, 30.0, -30.0)  # plane crossings every few steps
        return ps, dem.packing_config(dmax)
    if kind == "periodic":
        ps, L = dem.gen_periodic_packing(27000, s=1.8, jit=0.2, seed=22)
        ps.velocities[:, 2] += np.where(ps.ids % 2 == 0, 40.0, -40.0)
        return ps, dem.periodic_config(L, shear_rate=30.0)
    from helpers import settling_state, walled_config
    ps = settling_state(600, 8)
    ps.velocities[:, 2] = -2.0
    return ps, walled_config()


@pytest.mark.parametrize("kind,nranks", [("walled", 1), ("walled", 2), ("walled", 3), ("walled", 4),
                                         ("periodic", 1), ("periodic", 2), ("periodic", 3),
                                         ("settle", 3)])
def test_shard_local_bitwise_equals_single_gpu(cuda, kind, nranks):
    dem = cuda
    from paper_1503_03553_b200.slab import local_shards, step_local
    ps, cfg = _case(dem, kind)
    steps = 40 if kind == "settle" else 8
    s1, f1, t1, h1 = single_run(dem, ps, cfg, steps)
    shards = local_shards(ps, cfg, nranks)
    step_local(shards, 3)  # graph launches; the first launch also runs the priming pass
    ms = step_local(shards, steps - 3)
    assert sum(m.contacts for m in ms) == len(h1)
    _assert_same([sh.owned() for sh in shards], s1, f1, t1, h1)
    for sh in shards:
        sh.close()


def test_shard_step_metrics_and_timing(cuda):
    """dem_time_steps on sharded ranks (the bench path): per-rank device times, counts refreshed."""
    dem = cuda
    from paper_1503_03553_b200.slab import local_shards, step_local
    ps, cfg = _case(dem, "walled")
    shards = local_shards(ps, cfg, 2)
    step_local(shards, 1)
    for sh in shards:
        sh.launch(0)
    for sh in shards:
        sh.wait()
    owned = sum(sh.info()[2] for sh in shards)
    assert owned == len(ps.ids)
    # one rank's timed steps need its neighbour stepping too: time rank 0 while rank 1 launches
    shards[1].launch(4)
    ms, m = shards[0].time_steps(4)
    shards[1].wait()
    assert len(ms) == 4 and all(x > 0 for x in ms) and m.contacts > 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, kind, steps):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist
    import paper_1503_03553_b200 as dem
    from paper_1503_03553_b200.slab import ShardedSimulation, connect_torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps, cfg = _case(dem, kind)
    sim = ShardedSimulation(ps, cfg, rank, world, device=0)
    connect_torch(sim)
    for _ in range(steps):
        sim.step()
    p, f, t, (ho, hk, hd) = sim.owned()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), ids=p.ids, pos=p.positions, vel=p.velocities, f=f, t=t,
             ho=ho, hk=hk, hd=hd)
    dist.barrier()  # no rank frees its inbox while a neighbour may still store into it
    sim.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "walled"), (3, "walled"), (2, "periodic"), (3, "periodic")])
def test_shard_ipc_processes_bitwise(cuda, world, kind):
    import torch.multiprocessing as mp
    dem = cuda
    steps = 10
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, kind, steps), nprocs=world, join=True)
        parts = []
        for r in range(world):
            q = np.load(os.path.join(d, f"rank{r}.npz"))
            s = dem.ParticleSet(len(q["ids"]))
            s.ids[:], s.positions[:], s.velocities[:] = q["ids"], q["pos"], q["vel"]
            parts.append((s, q["f"], q["t"], (q["ho"], q["hk"], q["hd"])))
    ps, cfg = _case(dem, kind)
    s1, f1, t1, h1 = single_run(dem, ps, cfg, steps)
    _assert_same(parts, s1, f1, t1, h1)


def _hist_sorted(owner, key, d):
    k = (owner.astype(np.uint64) << np.uint64(32)) | key.astype(np.uint64)
    o = np.argsort(k, kind="stable")
    return k[o], bits(d[o])


def test_shard_configs3_full_size_bitwise(cuda):
    """configs[3] at its full size — 8,388,608 spheres in the periodic Lees-Edwards box — over 4
    sharded ranks (one process, peer pointers) against one context, 4 steps: positions, velocities,
    forces, torques and every tangential history bitwise equal by stable id."""
    dem = cuda
    from paper_1503_03553_b200.slab import local_shards, step_local
    ps, L = dem.gen_periodic_packing(1 << 23, s=1.8, jit=0.2, seed=4)
    cfg = dem.periodic_config(L, shear_rate=1.0)
    steps = 4
    sim = dem.Simulation(ps, cfg)
    sim.steps(steps)
    s1 = sim.particles()
    fa = sim.forces()
    o, p, d = sim.contacts()
    k1 = np.where(p >= 0, s1.ids[np.maximum(p, 0)], p.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
    h1 = _hist_sorted(s1.ids[o], k1, d)
    a1 = by_id(s1.ids, s1.ids, s1.positions, s1.velocities, fa.force, fa.torque)
    del sim, o, p, d, k1
    shards = local_shards(ps, cfg, 4)
    del ps
    step_local(shards, 3)
    step_local(shards, steps - 3)
    parts = [sh.owned() for sh in shards]
    for sh in shards:
        sh.close()
    ids = np.concatenate([q[0].ids for q in parts])
    a2 = by_id(ids, ids, np.concatenate([q[0].positions for q in parts]),
               np.concatenate([q[0].velocities for q in parts]), np.concatenate([q[1] for q in parts]),
               np.concatenate([q[2] for q in parts]))
    assert np.array_equal(a1[0], a2[0])
    for x, y in zip(a1[1:], a2[1:]):
        assert bitwise_equal(x, y)
    h2 = _hist_sorted(np.concatenate([q[3][0] for q in parts]), np.concatenate([q[3][1] for q in parts]),
                      np.concatenate([q[3][2] for q in parts]))
    assert np.array_equal(h1[0], h2[0]) and np.array_equal(h1[1], h2[1])
