"""configs[4]: divergence impact across the packing-fraction sweep. For each lattice
spacing s, the same packing is stepped with the paper's Alg. 1 single loop (collide_variant =
baseline, k_collide_single_loop) and with the two-phase kernels (k_detect + k_force_reduce); the two
are bitwise identical (tests/test_gpu_parity.py). Prints one JSON line per (N, s): contact density
(fraction of particles with >= 1 contact), contacts per particle, device µs per Collide variant
(median of profiled steps, CUDA events between kernels, L2 flushed) and the speed-up.

usage: python tools/divergence_sweep.py [N ...]        (default 1048576)
Run under ncu with -k regex:"k_collide_single_loop|k_detect|k_force_reduce" for warp efficiency.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1503_03553_b200 as dem  # noqa: E402

SPACINGS = [float(x) for x in os.environ.get("DS_SPACINGS", "2.35,2.3,2.2,2.1,2.0,1.9,1.8,1.7,1.6").split(",")]
STEPS = int(os.environ.get("DS_STEPS", "3"))

for n in [int(x) for x in (sys.argv[1:] or ["1048576"])]:
    for s in SPACINGS:
        ps, dmax = dem.gen_packing(n, s=s, jit=0.2, seed=5)
        rec = {"n": n, "s": s}
        for name, variant in (("single_loop", dem.BASELINE), ("two_phase", dem.TWO_PHASE)):
            cfg = dem.packing_config(dmax)
            cfg.collide_variant = variant
            sim = dem.Simulation(ps, cfg)
            sim.steps(2)
            prof = [sim.profile_step(512 << 20) for _ in range(STEPS)]
            k = [statistics.median(p.device_kernel_ms[i] for p in prof) for i in range(len(prof[0].device_kernel_ms))]
            collide_us = 1e3 * (k[5] + k[6])  # single loop: the kernel sits in the detect slot
            rec[name + "_us"] = round(collide_us, 2)
            if name == "two_phase":
                rec["detect_us"] = round(1e3 * k[5], 2)
                rec["force_reduce_us"] = round(1e3 * k[6], 2)
                o, p_, _ = sim.contacts()
                rec["contacts_per_particle"] = round(len(o) / n, 4)
                rec["contact_density"] = round(len(np.unique(o)) / n, 4)
            del sim
        rec["speedup"] = round(rec["single_loop_us"] / rec["two_phase_us"], 3)
        print(json.dumps(rec), flush=True)
