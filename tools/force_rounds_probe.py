"""Force-kernel round quantisation (profiles/r01_action_reaction.md): k_force_reduce time against N
around whole rounds of the persistent grid (2,368 warps = 16 per SM x 148). One GPU; prints one line per N."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem
for n in (227328, 240000, 250000, 262144, 280000, 303104):
    ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, seed=1)
    sim = dem.Simulation(ps, dem.packing_config(dmax))
    sim.steps(3)
    prof = [sim.profile_step(512 << 20) for _ in range(5)]
    fr = statistics.median(p.device_kernel_ms[6] for p in prof)
    det = statistics.median(p.device_kernel_ms[5] for p in prof)
    print(n, "tiles/warp %.2f" % (n / 32 / (16 * 148)), "force us %.1f" % (fr * 1e3), "per 1k particles %.3f" % (fr * 1e6 / n), "detect %.1f" % (det * 1e3), flush=True)
