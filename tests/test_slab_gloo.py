"""CPU, world_size > 1 over gloo: the slab-decomposition protocol of
paper_1503_03553_b200.slab (partitioning, neighbour exchange of counts then records through
torch.distributed, migrant hand-over with tangential history, one-plane halos, phase order)
driving oracle-backed ranks reproduces the single-process oracle step bitwise."""
import os
import socket
import tempfile

import numpy as np
import pytest

from helpers import bits, bitwise_equal


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, n, seed, steps):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist
    import paper_1503_03553_b200 as dem
    from paper_1503_03553_b200.slab import SlabDriver, TorchTransport, build_local_slabs
    from slab_oracle_backend import SlabRankOracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, seed=seed)
    cfg = dem.packing_config(dmax)
    ranks, bounds, g = build_local_slabs(ps, cfg, world, [rank], backend=SlabRankOracle)
    tr = TorchTransport(rank, world)
    tr.bind(ranks[0])
    drv = SlabDriver(ranks, tr)
    drv.prime()
    migrated = 0
    for _ in range(steps):
        drv.step()
        migrated += sum(ranks[0].send_count["migrant"])
    p, f, t, (ho, hk, hd) = ranks[0].owned()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), ids=p.ids, pos=p.positions, vel=p.velocities, f=f, t=t,
             ho=ho, hk=hk, hd=hd, migrated=migrated, ghosts=sum(ranks[0].send_count["ghost"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_gloo_bitwise(orc, world):
    import torch.multiprocessing as mp
    import paper_1503_03553_b200 as dem
    from oracle.oracle import OracleSim
    n, seed, steps = 4096, 13, 4
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, n, seed, steps), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, seed=seed)
        cfg = dem.packing_config(dmax)
        sim = OracleSim(orc, ps, cfg)
        sim.step(steps)
        s = sim.state()
        f1, t1 = sim.forces()
        ids = np.concatenate([p["ids"] for p in parts])
        assert len(ids) == n and len(np.unique(ids)) == n
        o = np.argsort(ids)
        ob = np.argsort(s.ids)
        for key, ref in (("pos", s.positions), ("vel", s.velocities), ("f", f1), ("t", t1)):
            got = np.concatenate([p[key] for p in parts])[o]
            assert bitwise_equal(got, ref[ob]), key
        hist = {}
        for p in parts:
            for a, b, x in zip(p["ho"], p["hk"], p["hd"]):
                hist[(int(a), int(b))] = tuple(bits(x))
        want = {(h.owner_id, h.partner_key): tuple(bits(np.array(h.delta_t))) for h in sim.history()}
        assert hist == want and len(want) > 0
        assert all(int(p["ghosts"]) > 0 for p in parts)


def test_slab_bounds_balance():
    from paper_1503_03553_b200.slab import slab_bounds
    planes = np.repeat(np.arange(10), [5, 5, 5, 5, 100, 100, 5, 5, 5, 5])
    b = slab_bounds(planes, 10, 4)
    assert b[0][0] == 0 and b[-1][1] == 10
    assert all(lo < hi for lo, hi in b)
    assert all(b[k][1] == b[k + 1][0] for k in range(3))
    with pytest.raises(ValueError):
        slab_bounds(planes, 10, 11)


class _FakeRank:
    """Record buffers only: what TorchTransport moves (CPU tensors over gloo)."""

    def __init__(self, rank):
        import torch
        self.rec = 8
        self.send = {"ghost": [torch.full((64,), 10 * rank + s, dtype=torch.uint8) for s in (0, 1)]}
        self.recv = {"ghost": [torch.zeros(64, dtype=torch.uint8) for _ in (0, 1)]}
        self.send_count = {"ghost": [rank + 1, rank + 2]}
        self.recv_count = {"ghost": [0, 0]}

    def buffer_device(self):
        return self.send["ghost"][0].device

    def send_view(self, kind, side, n):
        return self.send[kind][side][: n * self.rec]

    def recv_view(self, kind, side, n):
        return self.recv[kind][side][: n * self.rec]


def _ring_worker(rank, world, port, outdir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist
    from paper_1503_03553_b200.slab import TorchTransport
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rk = _FakeRank(rank)
    tr = TorchTransport(rank, world, ring=True)
    tr.bind(rk)
    tr.exchange("ghost")
    np.savez(os.path.join(outdir, f"ring{rank}.npz"), cnt=np.array(rk.recv_count["ghost"]),
             lo=rk.recv["ghost"][0].numpy(), hi=rk.recv["ghost"][1].numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ring_transport_gloo(world):
    """Periodic z: slab neighbours form a ring. Each rank receives, from below, the
    hi buffer of rank r-1 mod R and, from above, the lo buffer of rank r+1 mod R — including on a
    ring of 2, where both neighbours are the same process."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_ring_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for r in range(world):
            z = np.load(os.path.join(d, f"ring{r}.npz"))
            lo, hi = (r - 1) % world, (r + 1) % world
            assert list(z["cnt"]) == [lo + 2, hi + 1]
            assert (z["lo"][: (lo + 2) * 8] == 10 * lo + 1).all()
            assert (z["hi"][: (hi + 1) * 8] == 10 * hi + 0).all()
