"""Per-phase wall times of the slab step with PeerTransport and the bare gloo count
exchange latency. Run under torchrun (ranks may share a GPU: then the times include the other rank's work):
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/slab_peer_phase_times.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
import paper_1503_03553_b200 as dem
from paper_1503_03553_b200.slab import PeerTransport, SlabDriver, build_local_slabs
ps, dmax = dem.gen_packing(262144 * world, s=1.8, jit=0.2, seed=1)
cfg = dem.packing_config(dmax)
ranks, bounds, g = build_local_slabs(ps, cfg, world, [rank], device=local)
tr = PeerTransport(rank, world); tr.bind(ranks[0])
drv = SlabDriver(ranks, tr); drv.prime()
for _ in range(3): drv.step()
rk = ranks[0]
acc = {}
def t(name, f):
    t0 = time.perf_counter(); r = f(); acc.setdefault(name, []).append(time.perf_counter() - t0); return r
for _ in range(10):
    t("migrate", lambda: rk.migrate(True))
    t("xchg_m", lambda: tr.exchange("migrant"))
    t("import", lambda: rk.import_())
    t("halo", lambda: rk.halo())
    t("xchg_g", lambda: tr.exchange("ghost"))
    t("ghosts", lambda: rk.ghosts())
    t("force", lambda: rk.force(SlabDriver.STEP))
import statistics
print(rank, {k: round(1e6 * statistics.median(v), 1) for k, v in acc.items()}, flush=True)
# bare gloo all_gather latency
x = torch.zeros(2, dtype=torch.int64); ys = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
ts = []
for _ in range(50):
    t0 = time.perf_counter(); dist.all_gather(ys, x, group=tr.ctrl); ts.append(time.perf_counter() - t0)
print(rank, "gloo all_gather us", round(1e6 * statistics.median(ts), 1), flush=True)
dist.barrier(); tr.close(); dist.destroy_process_group()
