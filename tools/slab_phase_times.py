"""Where a slab step's wall time goes (one slab on one GPU, loopback): host wall ms per phase call
of SlabDriver.step, averaged over K steps. Diagnostic for the per-phase host synchronisations."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1503_03553_b200 as dem
from paper_1503_03553_b200.slab import LoopbackTransport, SlabDriver, build_local_slabs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, seed=1)
cfg = dem.packing_config(dmax)
ranks, bounds, g = build_local_slabs(ps, cfg, S, range(S))
tr = LoopbackTransport(ranks)
drv = SlabDriver(ranks, tr)
drv.prime()
for _ in range(3):
    drv.step()
torch.cuda.synchronize()
acc = collections.defaultdict(float)
K = 20
def t(name, f):
    t0 = time.perf_counter(); r = f(); acc[name] += time.perf_counter() - t0; return r
T0 = time.perf_counter()
for _ in range(K):
    for rk in ranks: t("migrate", lambda: rk.migrate(True))
    t("xchg_migrant", lambda: tr.exchange("migrant"))
    for rk in ranks: t("import", rk.import_)
    for rk in ranks: t("halo", rk.halo)
    t("xchg_ghost", lambda: tr.exchange("ghost"))
    for rk in ranks: t("ghosts", rk.ghosts)
    for rk in ranks: t("force", lambda: rk.force(dem.PHASE_STEP))
torch.cuda.synchronize()
tot = (time.perf_counter() - T0) / K
print(f"slabs={S} n={n}: {tot*1e3:.3f} ms/step;", {k: round(v / K * 1e3, 3) for k, v in acc.items()})
sim = dem.Simulation(ps, cfg)
ms, m = sim.time_steps(10, 0)
print(f"single context graph path: {sum(ms)/len(ms):.3f} ms/step")
