"""Single-GPU check of the slab path: S slab contexts on one device joined by the loopback
transport, vs the single-context graph path, on the same packing. Prints ms/step of both."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1503_03553_b200 as dem
from paper_1503_03553_b200.slab import LoopbackTransport, SlabDriver, build_local_slabs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
for S in [int(x) for x in (sys.argv[2:] or ["1", "2", "4"])]:
    ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, seed=1)
    cfg = dem.packing_config(dmax)
    ranks, bounds, g = build_local_slabs(ps, cfg, S, range(S))
    drv = SlabDriver(ranks, LoopbackTransport(ranks))
    drv.prime()
    for _ in range(3):
        drv.step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K = 10
    for _ in range(K):
        drv.step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    print(f"slabs={S} n={n}: {dt*1e3:.3f} ms/step (all slabs serialised on one GPU), bounds={bounds}")
sim = dem.Simulation(ps, cfg)
ms, m = sim.time_steps(10, 0)
print(f"single context graph path: {sum(ms)/len(ms):.3f} ms/step")
