"""Per-kernel device ms (events between kernels, L2 flushed, median of 3 profile steps after 5
warm-up steps) of k_force_reduce / k_detect / the step for several workloads on one GPU:
  mono     configs[1], 262,144 dense, fp64
  fp32     the same in the fp32 throughput mode
  poly     configs[2], 1,048,576 polydisperse 1:2, friction, K = 32
Used to compare compile-time variants (tools/gpu_variants_modes.sh)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem  # noqa: E402


def case(name):
    if name == "poly":
        ps, dmax = dem.gen_packing(1 << 20, s=1.4, jit=0.2, poly=True, seed=3, omega_half=50.0)
        return ps, dem.packing_config(dmax, poly=True)
    ps, dmax = dem.gen_packing(262144, s=1.8, jit=0.2, seed=1)
    cfg = dem.packing_config(dmax)
    cfg.precision = 1 if name == "fp32" else 0
    return ps, cfg


out = []
names = dem.device_kernel_names()
for name in (sys.argv[1:] or ["mono", "fp32", "poly"]):
    ps, cfg = case(name)
    sim = dem.Simulation(ps, cfg)
    sim.steps(5)
    prof = [sim.profile_step(512 << 20) for _ in range(3)]
    k = {nm: statistics.median(p.device_kernel_ms[i] for p in prof) for i, nm in enumerate(names)}
    step_ms, _ = sim.time_steps(5, 512 << 20)
    out.append(f"{name}: force {1e3 * k['k_force_reduce']:.1f} detect {1e3 * k['k_detect']:.1f} "
               f"step {1e3 * statistics.median(step_ms):.1f} us")
    del sim
print(" | ".join(out))
