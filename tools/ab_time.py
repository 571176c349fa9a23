"""A/B timing of compile-time variants with enough samples to resolve ~1 µs: the device timer
ticks in ~1-2 µs steps, so a median of a few steps cannot separate close variants. Prints the mean
of 40 graph-captured steps (L2 flushed before each) and the mean per-kernel event times of 10
profiled steps, per workload:
  mono  configs[1], 262,144 dense, fp64      fp32  the same in the fp32 mode
  poly  configs[2], 1,048,576 polydisperse   le    1,048,576 periodic Lees-Edwards box
  sX    8,388,608 walled dense pack at spacing X (e.g. s2.0)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem  # noqa: E402


def case(name):
    if name == "poly":
        ps, dmax = dem.gen_packing(1 << 20, s=1.4, jit=0.2, poly=True, seed=3, omega_half=50.0)
        return ps, dem.packing_config(dmax, poly=True)
    if name.startswith("s") and name[1:].replace(".", "").isdigit():  # e.g. s2.0: 8M walled pack at that spacing
        ps, dmax = dem.gen_packing(1 << 23, s=float(name[1:]), jit=0.2, seed=5)
        return ps, dem.packing_config(dmax)
    if name == "le":
        ps, L = dem.gen_periodic_packing(1 << 20, s=1.8, jit=0.2, seed=4)
        return ps, dem.periodic_config(L, shear_rate=1.0)
    ps, dmax = dem.gen_packing(262144, s=1.8, jit=0.2, seed=1)
    cfg = dem.packing_config(dmax)
    cfg.precision = 1 if name == "fp32" else 0
    return ps, cfg


out = []
names = dem.device_kernel_names()
for name in (sys.argv[1:] or ["mono", "poly"]):
    ps, cfg = case(name)
    sim = dem.Simulation(ps, cfg)
    sim.steps(5)
    prof = [sim.profile_step(512 << 20) for _ in range(10)]
    k = {nm: statistics.mean(p.device_kernel_ms[i] for p in prof) for i, nm in enumerate(names)}
    step_ms, _ = sim.time_steps(40, 512 << 20)
    bin_ = " ".join(f"{nm[2:]} {1e3 * k[nm]:.2f}" for nm in names if nm not in ("k_force_reduce", "k_detect"))
    out.append(f"{name}: force {1e3 * k['k_force_reduce']:.2f} detect {1e3 * k['k_detect']:.2f} "
               f"step {1e3 * statistics.mean(step_ms):.2f} us" + (f" [{bin_}]" if os.environ.get("AB_ALL") else ""))
    del sim
print(" | ".join(out))
