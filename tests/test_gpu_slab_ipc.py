"""GPU: the slab decomposition with records moved through CUDA-IPC peer memory (PeerTransport;
DESIGN.md §5): one process per slab, the migrate / halo pack kernels storing straight into the
neighbours' receive buffers, only the counts exchanged over gloo. On this one-GPU pool every
process opens the same device, so the peer stores stay on one B200 (on an HGX box they cross
NVLink); the protocol, the IPC plumbing and the results are the same. Results are bitwise equal to
one context."""
import os
import socket
import tempfile

import numpy as np
import pytest

from helpers import bits, bitwise_equal

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, periodic, steps):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch
    import torch.distributed as dist
    import paper_1503_03553_b200 as dem
    from paper_1503_03553_b200.slab import PeerTransport, SlabDriver, build_local_slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps, cfg = _case(dem, periodic)
    ranks, bounds, g = build_local_slabs(ps, cfg, world, [rank], device=0)
    tr = PeerTransport(rank, world, ring=g.ring)
    tr.bind(ranks[0])
    drv = SlabDriver(ranks, tr)
    drv.prime()
    migrated = 0
    for _ in range(steps):
        drv.step()
        migrated += sum(ranks[0].send_count["migrant"])
    p, f, t, (ho, hk, hd) = ranks[0].owned()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), ids=p.ids, pos=p.positions, vel=p.velocities, f=f, t=t,
             ho=ho, hk=hk, hd=hd, migrated=migrated)
    dist.barrier()
    tr.close()
    del drv, ranks
    dist.destroy_process_group()


def _case(dem, periodic):
    if periodic:
        ps, L = dem.gen_periodic_packing(27000, s=1.8, jit=0.2, seed=61)
        ps.velocities[:, 2] += np.where(ps.ids % 2 == 0, 40.0, -40.0)
        return ps, dem.periodic_config(L, shear_rate=30.0)
    ps, dmax = dem.gen_packing(32768, s=1.8, jit=0.2, seed=62)
    ps.velocities[:, 2] += np.where(ps.ids % 2 == 0, 40.0, -40.0)
    return ps, dem.packing_config(dmax)


@pytest.mark.parametrize("world,periodic", [(2, False), (3, False), (2, True), (3, True)])
def test_slab_peer_memory_bitwise(cuda, world, periodic):
    import torch.multiprocessing as mp
    dem = cuda
    steps = 20
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, periodic, steps), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    ps, cfg = _case(dem, periodic)
    sim = dem.Simulation(ps, cfg)
    for _ in range(steps):
        sim.step()
    s1 = sim.particles()
    fa = sim.forces()
    o, p, dd = sim.contacts()
    keys = np.where(p >= 0, s1.ids[np.maximum(p, 0)], p.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
    h1 = {(int(a), int(b)): tuple(bits(x)) for a, b, x in zip(s1.ids[o], keys, dd)}
    ids = np.concatenate([q["ids"] for q in parts])
    assert len(ids) == len(s1.ids) and len(np.unique(ids)) == len(ids)
    order = np.argsort(ids)
    ref = np.argsort(s1.ids)
    for fld, ref_arr in (("pos", s1.positions), ("vel", s1.velocities), ("f", fa.force), ("t", fa.torque)):
        got = np.concatenate([q[fld] for q in parts])[order]
        assert bitwise_equal(got, ref_arr[ref]), fld
    hist = {}
    for q in parts:
        for ow, k, x in zip(q["ho"], q["hk"], q["hd"]):
            hist[(int(ow), int(k))] = tuple(bits(x))
    assert hist == h1
    assert sum(int(q["migrated"]) for q in parts) > 0
