"""Detection cost in periodic / Lees-Edwards boxes against a walled box of the same size (DESIGN.md §3,
periodic two-stage detection). One GPU; prints detect / force ms per case."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem
for n in (1048576, 8388608):
    ps, L = dem.gen_periodic_packing(n, s=1.8, jit=0.2, seed=4)
    for name, cfg in (("periodic_le", dem.periodic_config(L, shear_rate=1.0)), ("periodic", dem.periodic_config(L)),
                      ("walled_same_box", None)):
        if cfg is None:
            cfg = dem.periodic_config(L); cfg.periodic = 0
        sim = dem.Simulation(ps, cfg)
        sim.steps(2)
        prof = [sim.profile_step(512 << 20) for _ in range(3)]
        k = [statistics.median(p.device_kernel_ms[i] for p in prof) for i in range(7)]
        print(n, name, "detect %.3f force %.3f ms" % (k[5], k[6]), "contacts", prof[-1].contacts, flush=True)
        del sim
