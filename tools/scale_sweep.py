"""One-GPU throughput across BASELINE.json's configs (sizes / densities). Writes JSON lines to
gpurun_out/sweep.jsonl: N, s, poly, contacts/particle, ms/step (events, L2 flushed), PU/s, and the
per-kernel breakdown of one profiled step."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_03553_b200 as dem

CASES = {
    "c2_262k": dict(n=262144, s=1.8, poly=False, seed=1),
    "c2_262k_fp32": dict(n=262144, s=1.8, poly=False, seed=1, precision=1),
    "c5_32m_s1.8_fp32": dict(n=33554432, s=1.8, poly=False, seed=5, precision=1),
    "c3_1m_poly": dict(n=1048576, s=1.4, poly=True, seed=3, omega=50.0),
    "c4_8m": dict(n=8388608, s=1.8, poly=False, seed=4),
    "c4_8m_periodic_le": dict(n=8388608, s=1.8, poly=False, seed=4, periodic=True, shear=1.0),
    "c5_32m_s2.35": dict(n=33554432, s=2.35, poly=False, seed=5),
    "c5_32m_s2.2": dict(n=33554432, s=2.2, poly=False, seed=5),
    "c5_32m_s2.0": dict(n=33554432, s=2.0, poly=False, seed=5),
    "c5_32m_s1.8": dict(n=33554432, s=1.8, poly=False, seed=5),
    "c5_32m_s1.6": dict(n=33554432, s=1.6, poly=False, seed=5),
}
names = sys.argv[1:] or list(CASES)
os.makedirs("gpurun_out", exist_ok=True)
out = open("gpurun_out/sweep.jsonl", "a")
for name in names:
    c = CASES[name]
    t0 = time.time()
    if c.get("periodic"):  # config 4 proper: periodic box, Lees-Edwards shear
        ps, L = dem.gen_periodic_packing(c["n"], s=c["s"], jit=0.2, poly=c["poly"], seed=c["seed"])
        cfg = dem.periodic_config(L, shear_rate=c["shear"], poly=c["poly"])
    else:
        ps, dmax = dem.gen_packing(c["n"], s=c["s"], jit=0.2, poly=c["poly"], seed=c["seed"], omega_half=c.get("omega", 0.5))
        cfg = dem.packing_config(dmax, poly=c["poly"])
    cfg.precision = c.get("precision", 0)
    sim = dem.Simulation(ps, cfg)
    del ps
    sim.steps(2)
    ms, m = sim.time_steps(5, 512 << 20)
    p = sim.profile_step(512 << 20)
    names_k = dem.device_kernel_names()
    rec = {"case": name, **c, "contacts_per_particle": m.contacts / c["n"], "capped_frac": m.capped_contacts / max(m.contacts, 1),
           "ms_per_step": statistics.mean(ms), "pu_s": c["n"] / (statistics.mean(ms) * 1e-3),
           "kernel_ms": {k: round(v, 4) for k, v in zip(names_k, p.device_kernel_ms)},
           "device_gb": sim.device_bytes() / 1e9, "setup_s": time.time() - t0}
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    out.flush()
    del sim
