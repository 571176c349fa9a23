"""The host-free sharded step's own cost on one GPU: configs[1] (262,144 dense) as one context and
as a 1-rank shard (dem_create_sharded, no neighbours: migrate / post / import / halo / post /
ghosts + the force phase over device-resident counts), and the periodic configs[3] physics at 1M
as one context and as a 1-rank ring (the rank is its own neighbour on both sides: records and
flags go through its own inbox). Device time per step (CUDA events, L2 flushed), median of 10."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem  # noqa: E402
from paper_1503_03553_b200.slab import ShardedSimulation  # noqa: E402

FLUSH = 512 << 20


def single(ps, cfg):
    sim = dem.Simulation(ps, cfg)
    sim.steps(5)
    ms, _ = sim.time_steps(10, FLUSH)
    return statistics.median(ms)


def shard(ps, cfg):
    sh = ShardedSimulation(ps, cfg, 0, 1)
    ring = bool(cfg.periodic & 4)
    sh.connect_local(sh if ring else None, sh if ring else None)
    sh.step(5)
    ms, _ = sh.time_steps(10, FLUSH)
    sh.close()
    return statistics.median(ms)


ps, dmax = dem.gen_packing(262144, s=1.8, jit=0.2, seed=1)
cfg = dem.packing_config(dmax)
a, b = single(ps, cfg), shard(ps, cfg)
print(f"configs[1] 262,144: one context {a * 1e3:.1f} us/step, 1-rank shard {b * 1e3:.1f} us/step ({100 * (b / a - 1):+.1f}%)")
ps, L = dem.gen_periodic_packing(1 << 20, s=1.8, jit=0.2, seed=4)
cfg = dem.periodic_config(L, shear_rate=1.0)
a, b = single(ps, cfg), shard(ps, cfg)
print(f"periodic LE 1,048,576: one context {a * 1e3:.1f} us/step, 1-rank ring {b * 1e3:.1f} us/step ({100 * (b / a - 1):+.1f}%)")
