"""Profiling driver for the non-headline modes (run under ncu on ONE GPU; numbers printed here are
never bench values): --mode fp32 (262,144 dense, fp32 throughput mode) or --mode periodic
(1,048,576 spheres, periodic box with Lees-Edwards shear, configs[3] physics)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", choices=["fp32", "periodic"], required=True)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
if a.mode == "fp32":
    ps, dmax = dem.gen_packing(262144, s=1.8, jit=0.2, seed=1)
    cfg = dem.packing_config(dmax)
    cfg.precision = 1
else:
    ps, L = dem.gen_periodic_packing(1048576, s=1.8, jit=0.2, seed=4)
    cfg = dem.periodic_config(L, shear_rate=1.0)
sim = dem.Simulation(ps, cfg)
sim.steps(a.warmup)
for _ in range(a.steps):
    m = sim.profile_step(512 << 20)
print(a.mode, "contacts", m.contacts, "kernel ms", [round(x, 4) for x in m.device_kernel_ms])
