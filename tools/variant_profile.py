"""Paper claim check (arXiv 1503.03553): Collide time of the single-loop
Alg. 1 vs the two-phase split, on B200, dense packs. Prints device ms per kernel (events between
kernels, L2 flushed). Run under ncu with -k regex:"k_collide_single_loop|k_detect|k_force_reduce"
to read warp execution efficiency."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import statistics
import paper_1503_03553_b200 as dem

steps = int(os.environ.get("VP_STEPS", "5"))
for n in [int(x) for x in (sys.argv[1:] or ["131072", "262144"])]:
    for s in (1.8, 2.2):
        ps, dmax = dem.gen_packing(n, s=s, jit=0.2, seed=1)
        out = {}
        for variant in (dem.BASELINE, dem.TWO_PHASE):
            cfg = dem.packing_config(dmax)
            cfg.collide_variant = variant
            sim = dem.Simulation(ps, cfg)
            sim.steps(3)
            prof = [sim.profile_step(512 << 20) for _ in range(steps)]
            det = statistics.median(p.device_kernel_ms[5] for p in prof)
            frc = statistics.median(p.device_kernel_ms[6] for p in prof)
            out[variant] = (det, frc, prof[-1].contacts)
        b, t = out[dem.BASELINE], out[dem.TWO_PHASE]
        print(f"n={n} s={s} contacts/particle={t[2]/n:.2f}: single-loop Collide {b[0]*1e3:.1f} us | "
              f"two-phase detect {t[0]*1e3:.1f} + force_reduce {t[1]*1e3:.1f} = {(t[0]+t[1])*1e3:.1f} us | "
              f"speedup {b[0]/(t[0]+t[1]):.2f}x")
