"""Workloads for the compute-sanitizer gate (tools/sanitize.sh): small, complete DEM steps on ONE
GPU. Modes:
  walled    4,096 spheres settling in the 5-rectangle + 1-line walled box (gravity, walls, history),
            priming pass + 3 steps, plus the Alg. 1 single-loop variant for one step
  periodic  4,096 spheres in a periodic Lees-Edwards box (shear 30/s), priming + 3 steps
  fp32      the walled case in the fp32 throughput mode
  slab      2 processes, one z-slab each: the host-free sharded step (CUDA-IPC inboxes, flags,
            stream waits), priming + 3 steps
  shard_local  3 sharded ranks of one process, periodic Lees-Edwards ring, 3 steps
Prints one line per mode; exit status 0 when the steps ran (the sanitizer decides the gate)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def walled(precision=0):
    import paper_1503_03553_b200 as dem
    from helpers import settling_state, walled_config
    cfg = walled_config()
    cfg.precision = precision
    sim = dem.Simulation(settling_state(4096, 7), cfg)
    for _ in range(3):
        m = sim.step()
    if precision == 0:
        sim.set_collide_variant(dem.BASELINE)
        m = sim.step()
    sim.particles(), sim.forces(), sim.contacts()
    del sim  # dem_destroy before exit, so memcheck's leak check sees every allocation freed
    return m


def periodic():
    import paper_1503_03553_b200 as dem
    ps, L = dem.gen_periodic_packing(4096, s=1.8, jit=0.2, seed=5)
    sim = dem.Simulation(ps, dem.periodic_config(L, shear_rate=30.0))
    for _ in range(3):
        m = sim.step()
    sim.particles(), sim.forces()
    del sim
    return m


def _slab_worker(rank, world, port):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch.distributed as dist
    import paper_1503_03553_b200 as dem
    from paper_1503_03553_b200.slab import ShardedSimulation, connect_torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps, dmax = dem.gen_packing(8000, s=1.8, jit=0.2, seed=9)
    ps.velocities[:, 2] += np.where(ps.ids % 2 == 0, 40.0, -40.0)  # migrations every few steps
    sim = ShardedSimulation(ps, dem.packing_config(dmax), rank, world, device=0)
    connect_torch(sim)
    for _ in range(3):
        sim.step()
    sim.owned()
    dist.barrier()  # no rank frees its inbox while a neighbour may still store into it
    sim.close()
    dist.destroy_process_group()


def slab():
    """2 processes, one z-slab each: the host-free sharded step with CUDA-IPC inboxes."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_slab_worker, args=(2, port), nprocs=2, join=True)
    return None


def shard_local():
    """3 ranks of one process (direct peer pointers), periodic Lees-Edwards ring."""
    import paper_1503_03553_b200 as dem
    from paper_1503_03553_b200.slab import local_shards, step_local
    ps, L = dem.gen_periodic_packing(8000, s=1.8, jit=0.2, seed=10)
    shards = local_shards(ps, dem.periodic_config(L, shear_rate=30.0), 3)
    ms = step_local(shards, 3)
    for sh in shards:
        sh.close()
    return ms[0]


if __name__ == "__main__":
    mode = sys.argv[1]
    m = {"walled": walled, "periodic": periodic, "fp32": lambda: walled(1), "slab": slab,
         "shard_local": shard_local}[mode]()
    print(f"sanitize_driver {mode}: ok" + (f" (contacts {m.contacts})" if m is not None else ""), flush=True)
