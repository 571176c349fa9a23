#!/usr/bin/env python3
"""DEM step benchmark (BASELINE.json metric: particle-updates/s; force-kernel HBM % of peak).

Workload at N=1: BASELINE.json configs[1] — 262,144 monodisperse spheres, dense random packing
(SURVEY §8d generator G(262144, s=1.8, jit=0.2, mono, seed=1), dt=1e-5, g=0, no walls, K=16),
fp64 (the reference's arithmetic). One "step" = one Simulation::step() (pipeline.cpp:366-378):
integrate, bin, detect, force, history merge, reduce.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Timing: W untimed warm-up steps, then K steps each timed with CUDA events on the launching
stream; before every timed step a 512 MiB buffer is overwritten to flush L2 (126 MB), outside
the events. value = N_particles * K * world / max-over-ranks(sum of step times).
e2e: the same metric through the C ABI with host buffers: per step the full particle state is
uploaded from host memory (dem_set_particles), one step runs, and the state is read back
(dem_get_particles); wall-clock per step.
--impl reference: the reference's own CPU Simulation::step() (oracle/_ref, compiled from the
reference sources) on this host with all cores, on the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PARTICLES = 262144
FLUSH_BYTES = 512 << 20
METRIC = "particle-updates/sec"
UNIT = "particle-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(n, c, m):
    """Compulsory bytes per launch of each kernel (d64) in the steady stepping state, where the
    previous force kernel pre-integrated the state: k_integrate_hash only
    hashes (reads 32 B of position, writes key + arrival rank), k_force_reduce also writes the
    96 B/particle pre-integrated state."""
    return {
        "k_phase_begin": 0,
        "k_integrate_hash": 40 * n,
        "k_scan_cells": 12 * m,
        "k_scatter": 24 * n,
        "k_reorder": 252 * n,
        "k_detect": 60 * n + 4 * m + 8 * c,
        "k_force_reduce": 268 * n + 64 * c,
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def pinned_particles(n):
    """A ParticleSet whose arrays live in page-locked host memory (cudaHostAlloc via torch)."""
    import torch
    import paper_1503_03553_b200 as dem
    ps = dem.ParticleSet(0)

    def pin(shape, dt):
        return torch.empty(shape, dtype=dt, pin_memory=True).numpy()
    ps.ids = pin((n,), torch.int32).view(np.uint32)
    ps.positions = pin((n, 3), torch.float64)
    ps.velocities = pin((n, 3), torch.float64)
    ps.angular_velocities = pin((n, 3), torch.float64)
    ps.radii = pin((n,), torch.float64)
    ps.masses = pin((n,), torch.float64)
    ps.material_ids = pin((n,), torch.int32).view(np.uint32)
    return ps


# The N=1 workload, identical in both arms (the driver compares the two `config` dicts).
CONFIG_N1 = {"workload": "262,144 monodisperse spheres, dense random packing (configs[1])",
             "generator": "G(262144, s=1.8, jit=0.2, mono, seed=1)", "dt": 1e-5,
             "contact_capacity": 16, "parallelism": "single-gpu",
             "l2": "flushed before every timed step (512 MiB write), outside the events"}


def workload(seed=1):
    import paper_1503_03553_b200 as dem
    ps, dmax = dem.gen_packing(N_PARTICLES, s=1.8, jit=0.2, poly=False, seed=seed)
    cfg = dem.packing_config(dmax)
    return ps, cfg


def reference_workload(seed=1):
    """The same arrays built by the oracle's copy of the generator: the reference legs never load
    the product library (oracle/workload.py; bitwise equal, tests/test_oracle_golden.py)."""
    from oracle.workload import gen_packing, packing_config
    ps, dmax = gen_packing(N_PARTICLES, s=1.8, jit=0.2, poly=False, seed=seed)
    return ps, packing_config(dmax)


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "nproc": usable, "logical_cpus": os.cpu_count()}


def cpu_reference_run(ps, cfg, steps, warmup, budget_s, threads=None):
    """Reference Simulation::step() on host cores (oracle/_ref). Returns dict. `threads` sets the
    reference's pool size (DEMFORGE_THREADS semantics, parallel.cpp:14-33); None = all cores."""
    from oracle.oracle import RefLib, RefSim
    ref = RefLib()
    ref.set_threads(threads if threads else host_info()["nproc"])
    cores = ref.thread_count()
    t0 = time.perf_counter()
    sim = RefSim(ref, ps, cfg)  # priming pass untimed, pipeline.cpp:83
    t_ctor = time.perf_counter() - t0
    for _ in range(warmup):
        sim.step()
    done, t_total = 0, 0.0
    while done < steps:
        t1 = time.perf_counter()
        sim.step()
        t_total += time.perf_counter() - t1
        done += 1
        if t_total > budget_s:
            break
    value = len(ps.ids) * done / t_total
    return {"value": value, "steps": done, "seconds": t_total, "cores": cores, "ctor_s": t_ctor}


def cpu_baseline_block(ps, cfg, steps, warmup, budget_s, sample="262,144-particle"):
    """All host threads, then one thread (both, with the CPU model and core count)."""
    info = host_info()
    r = cpu_reference_run(ps, cfg, steps, warmup, budget_s)
    r1 = cpu_reference_run(ps, cfg, 3 if len(ps.ids) <= 1 << 20 else 1, 0,
                           float(os.environ.get("DEM_CPU1_BUDGET_S", "10")), threads=1)
    block = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
             "sample": f"{r['steps']} full steps of the same {sample} workload "
                       f"({r['seconds']:.1f} s) through the reference Simulation::step() compiled from "
                       f"its sources (oracle/_ref), DEMFORGE threads={r['cores']}",
             "threads1": {"value": r1["value"], "unit": UNIT, "cores": 1,
                          "sample": f"{r1['steps']} steps ({r1['seconds']:.1f} s), DEMFORGE threads=1"},
             **info}
    return r, block


def run_reference(args):
    """--impl reference: the reference's own CPU Simulation::step() on this host's cores, on the
    b200 arm's workload/config/metric, exactly --steps timed after --warmup untimed steps. Inputs
    come from the oracle's generator copy; nothing from paper_1503_03553_b200 is loaded."""
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    if world == 1:
        ps, cfg = reference_workload()
        sample = "262,144-particle"
    else:
        # configs[3]'s 8M packing; the reference has no periodic box or shear, so it
        # runs the walled proxy of the same packing
        from oracle.workload import gen_packing, packing_config
        ps, dmax = gen_packing(N_CONFIG3, s=1.8, jit=0.2, poly=False, seed=4)
        cfg = packing_config(dmax)
        sample = "8,388,608-particle (walled proxy of configs[3])"
    r, block = cpu_baseline_block(ps, cfg, args.steps, args.warmup,
                                  float(os.environ.get("DEM_REF_BUDGET_S", "900")), sample)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup,
        "ms_per_step": 1e3 * r["seconds"] / r["steps"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY §8d generator, xorshift64*)",
        "config": dict(CONFIG_N1) if world == 1 else slab_config(world),
        "cpu_baseline": block,
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


N_CONFIG3 = 8388608


def slab_config(world):
    """The N > 1 workload (identical in both arms): BASELINE configs[3], 8M spheres in a periodic
    Lees-Edwards shear box, z-slabs over the N GPUs (strong scaling: the total is fixed)."""
    return {"workload": "8,388,608 monodisperse spheres in a periodic Lees-Edwards shear box (configs[3])",
            "generator": "G(8388608, s=1.8, jit=0.2, mono, seed=4), periodic x/y/z, shear rate 1/s (flow x, gradient y)",
            "dt": 1e-5, "contact_capacity": 16, "parallelism": f"z-slabs x{world}, host-free sharded step",
            "l2": "inputs larger than L2 (>= 0.4 GB of particle state per GPU), no flush"}


def run_sharded(args, world, rank, local):
    """N > 1: BASELINE configs[3] over N GPUs with the host-free sharded step (dem_create_sharded):
    one process per GPU, the neighbours' inboxes opened through CUDA IPC (NVLink peer memory),
    counts on the device, each step one CUDA graph. value = 8,388,608 x K / max over ranks of the
    summed per-step device times (CUDA events on each rank's stream)."""
    import torch
    import torch.distributed as dist
    import paper_1503_03553_b200 as dem
    from paper_1503_03553_b200.slab import ShardedSimulation, connect_torch
    ps, L = dem.gen_periodic_packing(N_CONFIG3, s=1.8, jit=0.2, seed=4)
    cfg = dem.periodic_config(L, shear_rate=1.0)
    sim = ShardedSimulation(ps, cfg, rank, world, device=local)
    del ps
    connect_torch(sim)
    for _ in range(max(1, args.warmup)):
        sim.step()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        step_ms, m = sim.time_steps(args.steps, 0)
    barrier(world)
    total_s = max_over_ranks(sum(step_ms) / 1e3, world)
    value = N_CONFIG3 * args.steps / total_s
    contacts = max_over_ranks(float(m.contacts), world)  # per-rank; reported for the slowest rank
    z_lo, z_hi, owned = sim.info()
    # e2e: the same steps through the public API (dem_step) with every rank reading its slab's
    # state back into pinned host memory after each step, wall clock, max over ranks
    host = pinned_particles(int(sim.size()) + 4096)
    import ctypes as C
    t_e2e, d2h = [], 0
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(e2e_steps):
        barrier(world)
        t0 = time.perf_counter()
        sim.step()
        n_loc = sim.size()
        view = dem.ParticleSet(0)
        for f in ("ids", "positions", "velocities", "angular_velocities", "radii", "masses", "material_ids"):
            setattr(view, f, getattr(host, f)[:n_loc])
        rc = sim.lib.dem_get_particles(sim.ctx, C.byref(view.c_struct()))
        assert rc == 0, rc
        t_e2e.append(time.perf_counter() - t0)
        d2h += n_loc * 96
    e2e_s = max_over_ranks(sum(t_e2e), world)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY §8d generator, xorshift64*)",
        "config": slab_config(world),
        "workload_stats": {"particles": N_CONFIG3, "box_length": L, "rank0_slab_planes": [z_lo, z_hi],
                           "rank0_owned": owned, "contacts_per_step_max_rank": contacts},
        "gpu_launches": 16 * args.steps,
        "e2e": {"value": N_CONFIG3 * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(d2h / e2e_steps),
                "how": "dem_step (host-free sharded step) + per-rank dem_get_particles of the slab into pinned host memory, wall clock, max over ranks"},
        "clocks": clk.summary(),
    }
    del sim
    if world > 1 and not args.no_north_star:
        barrier(world)
        line["north_star_32m"] = north_star_sharded(args, world, rank, local)
    barrier(world)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def north_star_sharded(args, world, rank, local):
    """north_star's target on N GPUs: 32M dense frictional spheres, walled box, z-slabs."""
    import torch
    import paper_1503_03553_b200 as dem
    from paper_1503_03553_b200.slab import ShardedSimulation, connect_torch
    n = 1 << 25
    ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, poly=False, seed=5)
    sim = ShardedSimulation(ps, dem.packing_config(dmax), rank, world, device=local)
    del ps
    connect_torch(sim)
    for _ in range(3):
        sim.step()
    steps = max(3, min(args.steps, 10))
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        step_ms, m = sim.time_steps(steps, 0)
    total_s = max_over_ranks(sum(step_ms) / 1e3, world)
    del sim
    return {"workload": "33,554,432 monodisperse spheres, dense frictional packing (north_star target)",
            "generator": "G(33554432, s=1.8, jit=0.2, mono, seed=5)", "dtype": "f64", "contact_capacity": 16,
            "value": n * steps / total_s, "unit": UNIT, "steps": steps, "warmup": 3,
            "ms_per_step": 1e3 * total_s / steps, "scaling": "strong", "clocks": clk.summary(),
            "l2": "inputs larger than L2, no flush"}


def config3_block(args):
    """BASELINE configs[3] on this one GPU — 8,388,608 spheres in the periodic Lees-Edwards shear
    box, the workload of the N > 1 lines — so the scaling curve has its own N = 1 point (the
    headline `value` stays configs[1]). Single context (the sharded step is bitwise the same)."""
    import paper_1503_03553_b200 as dem
    ps, L = dem.gen_periodic_packing(N_CONFIG3, s=1.8, jit=0.2, seed=4)
    sim = dem.Simulation(ps, dem.periodic_config(L, shear_rate=1.0), device=0)
    del ps
    steps = max(3, min(args.steps, 10))
    for _ in range(3):
        sim.step()
    with ClockSampler(0) as clk:
        step_ms, m = sim.time_steps(steps, 0)
    total_s = sum(step_ms) / 1e3
    del sim
    return {"workload": "8,388,608 spheres, periodic box with Lees-Edwards shear (configs[3]), one GPU",
            "generator": "G_periodic(8388608, s=1.8, jit=0.2, mono, seed=4), shear rate 1/s", "dtype": "f64",
            "value": N_CONFIG3 * steps / total_s, "unit": UNIT, "steps": steps, "warmup": 3,
            "ms_per_step": 1e3 * total_s / steps, "contacts_per_step": int(m.contacts), "clocks": clk.summary(),
            "l2": "inputs larger than L2, no flush (as the N > 1 lines)"}


def north_star_block(args):
    """north_star's target workload on this one GPU: 32M dense frictional spheres (G(33554432,
    s=1.8, jit=0.2, mono, seed=5), mu = 0.3, K = 16), fp64, its own warm-up / timed steps (CUDA
    events, L2 flushed), clocks and force-kernel roofline. A second measured block; the headline
    `value` stays configs[1]."""
    import paper_1503_03553_b200 as dem
    n = 1 << 25
    ps, dmax = dem.gen_packing(n, s=1.8, jit=0.2, poly=False, seed=5)
    sim = dem.Simulation(ps, dem.packing_config(dmax), device=0)
    del ps
    steps = max(3, min(args.steps, 10))
    for _ in range(3):
        sim.step()
    with ClockSampler(0) as clk:
        step_ms, m = sim.time_steps(steps, FLUSH_BYTES)
    prof = [sim.profile_step(FLUSH_BYTES) for _ in range(2)]
    names = dem.device_kernel_names()
    kms = {nm: statistics.median(p.device_kernel_ms[k] for p in prof) for k, nm in enumerate(names)}
    c = prof[-1].contacts
    nbytes = algorithmic_bytes(n, c, prof[-1].cells)
    peak, peak_kind = peaks()
    fa = nbytes["k_force_reduce"] / (kms["k_force_reduce"] * 1e-3) / 1e9
    total_s = sum(step_ms) / 1e3
    del sim
    return {"workload": "33,554,432 monodisperse spheres, dense frictional packing (north_star target, configs[4] s=1.8)",
            "generator": "G(33554432, s=1.8, jit=0.2, mono, seed=5)", "dtype": "f64", "contact_capacity": 16,
            "value": n * steps / total_s, "unit": UNIT, "steps": steps, "warmup": 3,
            "ms_per_step": 1e3 * total_s / steps, "contacts_per_step": c, "cells": prof[-1].cells,
            "capped_contacts": int(prof[-1].capped_contacts), "friction_max_ratio": prof[-1].friction_max_ratio,
            "roofline": {"bound": "hbm", "kernel": "k_force_reduce", "achieved": fa, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": fa / peak,
                         "algorithmic_bytes": nbytes["k_force_reduce"], "ms": kms["k_force_reduce"]},
            "kernel_ms": kms, "clocks": clk.summary(),
            "l2": "flushed before every timed step (512 MiB write), outside the events"}


def run_b200(args):
    world, rank, local = dist_env()
    import torch
    if world > 1:
        import torch.distributed as dist
        ngpu = torch.cuda.device_count()
        if world <= ngpu:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # more ranks than GPUs (a functional check of the N > 1 path on a small box): ranks
            # share devices, the control plane runs on gloo; not a scaling measurement
            local = local % ngpu
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        return run_sharded(args, world, rank, local)
    torch.cuda.set_device(0)
    import paper_1503_03553_b200 as dem

    ps, cfg = workload(seed=1)
    n = len(ps.ids)
    sim = dem.Simulation(ps, cfg, device=local)
    for _ in range(args.warmup):
        sim.step()

    # --- timed region: K steps, CUDA events per step on the launching stream ---
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        step_ms, m_last = sim.time_steps(args.steps, FLUSH_BYTES)
    torch.cuda.synchronize()
    barrier(world)
    total_s = sum(step_ms) / 1e3
    total_s_max = max_over_ranks(total_s, world)
    value = n * args.steps * world / total_s_max
    ms_per_step = 1e3 * total_s_max / args.steps

    # --- per-kernel device times (events between kernels, same stream, L2 flushed) ---
    prof = []
    for _ in range(3):
        prof.append(sim.profile_step(FLUSH_BYTES))
    names = dem.device_kernel_names()
    kms = {nm: statistics.median(p.device_kernel_ms[k] for p in prof) for k, nm in enumerate(names)}
    c = prof[-1].contacts
    nbytes = algorithmic_bytes(n, c, prof[-1].cells)
    dom = max((k for k in kms if k != "k_phase_begin"), key=lambda k: kms[k])
    peak, peak_kind = peaks()
    force_ach = nbytes["k_force_reduce"] / (kms["k_force_reduce"] * 1e-3) / 1e9
    dom_ach = nbytes[dom] / (kms[dom] * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom)
        except Exception:
            traffic = None
    # what actually bounds the dominant kernel (FP64 pipe / latency, not HBM): the ncu capture
    # of the same workload committed under profiles/ (tools/profile_round.sh)
    util = None
    upath = os.path.join(ROOT, "profiles", "r02_kernel_util.json")
    if os.path.exists(upath):
        try:
            util = json.load(open(upath)).get(dom)
        except Exception:
            util = None

    # --- e2e through the C ABI with host buffers ---
    # (pinned host arrays, as a production caller keeps them; the state goes up and comes back
    # every step: dem_set_particles + dem_step_async + dem_get_particles + dem_sync. The readback
    # of the step's final state overlaps its detection and forces; dem_get_particles waits for
    # the step and checks its errors, dem_sync returns its metrics)
    e2e_steps = max(3, min(args.steps, 10))
    host = pinned_particles(n)
    sim.particles_into(host)
    t_e2e = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        sim.set_particles(host)
        sim.step_async()
        sim.particles_into(host)
        m_e2e = sim.sync()
        t_e2e.append(time.perf_counter() - t0)
    assert m_e2e.contacts > 0
    e2e_s = max_over_ranks(sum(t_e2e), world)
    e2e_value = n * e2e_steps * world / e2e_s
    state_bytes = n * (4 + 24 * 3 + 8 + 8 + 4)
    # the host-coupled variant: only the motion goes up (positions, velocities, angular velocities;
    # ids / radii / masses / materials stay on the device), the motion and ids come back
    motion = pinned_particles(n)
    motion.radii = motion.masses = motion.material_ids = None
    sim.particles_into(motion)
    t_mo = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        sim.set_motion(motion.positions, motion.velocities, motion.angular_velocities)
        sim.step_async()
        sim.particles_into(motion)
        m_e2e = sim.sync()
        t_mo.append(time.perf_counter() - t0)
    mo_s = max_over_ranks(sum(t_mo), world)
    e2e_motion = {"value": n * e2e_steps * world / mo_s, "unit": UNIT, "h2d_bytes_per_step": n * 72,
                  "d2h_bytes_per_step": n * 76,
                  "how": "dem_set_particles(motion only; ids/radii/masses/materials NULL = kept) + "
                         "dem_step_async + dem_get_particles(motion + ids) + dem_sync, wall clock"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY §8d generator, xorshift64*)",
        "config": dict(CONFIG_N1),
        "workload_stats": {"particles": n, "contacts_per_step": c, "cells": prof[-1].cells, "radix_passes": 1},
        "gpu_launches": sim.kernels_per_step() * args.steps,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes,
                "how": "dem_set_particles(pinned host) + dem_step_async(1) + dem_get_particles(pinned host, overlapping the step's detection and forces) + dem_sync (metrics), wall clock"},
        "e2e_motion": e2e_motion,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_ach, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": dom_ach / peak,
                     "traffic": traffic, "algorithmic_bytes": nbytes[dom], "ms": kms[dom],
                     "ncu": dict(util, source="profiles/r02_kernel_util.json (ncu --set full)") if util else None},
        "force_kernel": {"name": "k_force_reduce", "achieved": force_ach, "frac": force_ach / peak, "ms": kms["k_force_reduce"],
                         "algorithmic_bytes": nbytes["k_force_reduce"]},
        "kernel_ms": kms,
        "clocks": clk.summary(),
    }
    del sim
    if world == 1 and not args.no_north_star:
        line["configs3_1gpu"] = config3_block(args)
        line["north_star_32m"] = north_star_block(args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rps, rcfg = reference_workload()
            _, line["cpu_baseline"] = cpu_baseline_block(rps, rcfg, 1000, 0,
                                                         float(os.environ.get("DEM_CPU_BUDGET_S", "20")))
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-north-star", action="store_true", help="skip the 32M north-star block (N=1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
