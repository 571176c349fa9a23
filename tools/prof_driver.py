"""Profiling driver: the bench workload (262,144 dense, seed 1), W warm-up steps then S steps.
Run under ncu on ONE GPU; numbers printed here are never bench values."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=262144)
ap.add_argument("--s", type=float, default=1.8)
ap.add_argument("--poly", action="store_true")
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
ps, dmax = dem.gen_packing(a.n, s=a.s, jit=0.2, poly=a.poly, seed=1, omega_half=50.0 if a.poly else 0.5)
sim = dem.Simulation(ps, dem.packing_config(dmax, poly=a.poly))
sim.steps(a.warmup)
for _ in range(a.steps):
    m = sim.profile_step(512 << 20)
print("contacts", m.contacts, "kernel ms", [round(x, 4) for x in m.device_kernel_ms])
