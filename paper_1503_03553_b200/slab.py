"""Slab domain decomposition of the DEM step over several GPUs.

The reference is single-process; this is the B200 build's multi-GPU path. Space is
cut into slabs of whole cell planes along z, balanced by particle count. Each rank owns the
particles whose cell plane lies in its slab, and each step it:

  1. integrates its owned particles and hands the ones whose plane left the slab, with their
     tangential-history rows (keyed by stable id), to the z-neighbour          (migrate/import)
  2. sends its boundary-plane particles to the neighbours as ghosts             (halo/ghosts)
  3. bins owned + ghosts, detects and computes forces for owned particles only  (force)

Exchanges are neighbour point-to-point transfers: NCCL over NVLink when the transport is
torch.distributed with backend "nccl" (device tensors), gloo in CPU tests, or an in-process
loopback (several ranks on one GPU, for single-GPU validation). The canonical in-cell order
(cell, stable id) makes the result bitwise identical to a single-GPU run for any rank count.

This module holds the protocol (partitioning, the exchange pattern, the phase order) and the
CUDA-backed rank. The test suite drives the same protocol with a CPU oracle-backed rank
(tests/slab_oracle_backend.py) over gloo.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from .simulation import ParticleSet, SimConfig, StepMetrics, _Config, _raise

GHOST_BIT = 0x80000000


# ---------------------------------------------------------------------------------------------
# Partitioning (pure host arithmetic, identical on every rank)

@dataclass
class GlobalGrid:
    oz: float
    h: float
    inv_h: float      # 1 / cell extent along z
    nz: int
    ring: bool = False  # periodic z: slab neighbours form a ring


def global_grid(cfg: SimConfig, r_max: float) -> GlobalGrid:
    """make_grid (grid.cpp:10-28) for the z axis, with the cell size every rank must share; a
    periodic z gets floor(L/h) cells of extent L/n."""
    h = cfg.grid_cell_size if cfg.grid_cell_size > 0.0 else 2.0 * r_max * (1.0 + 1e-6)
    ez = cfg.domain_max[2] - cfg.domain_min[2]
    if getattr(cfg, "periodic", 0) & 4:
        nz = int(math.floor(ez / h))
        return GlobalGrid(cfg.domain_min[2], h, 1.0 / (ez / nz), nz, True)
    nz = max(1, int(math.ceil(ez / h)))
    return GlobalGrid(cfg.domain_min[2], h, 1.0 / h, nz)


def cell_planes(z: np.ndarray, g: GlobalGrid) -> np.ndarray:
    """z part of calc_hash (grid.cpp:30-52): floor((z - origin) * (1/h)), clamped."""
    f = np.floor((np.asarray(z, np.float64) - g.oz) * g.inv_h)
    f = np.where(np.isfinite(f), f, -1.0)
    return np.clip(f, 0, g.nz - 1).astype(np.int64)


def slab_bounds(planes: np.ndarray, nz: int, nranks: int) -> List[tuple]:
    """Contiguous plane ranges [z_lo, z_hi) with balanced particle counts, >= 1 plane each."""
    if nranks > nz:
        raise ValueError(f"{nranks} slabs need at least {nranks} cell planes (grid has {nz})")
    hist = np.bincount(planes, minlength=nz).astype(np.float64)
    cum = np.cumsum(hist)
    total = cum[-1] if len(cum) else 0.0
    cuts = [0]
    for k in range(1, nranks):
        target = total * k / nranks
        z = int(np.searchsorted(cum, target, side="left")) + 1
        z = max(z, cuts[-1] + 1)
        z = min(z, nz - (nranks - k))
        cuts.append(z)
    cuts.append(nz)
    return [(cuts[k], cuts[k + 1]) for k in range(nranks)]


def select(ps: ParticleSet, mask: np.ndarray) -> ParticleSet:
    out = ParticleSet(0)
    for k in ("ids", "positions", "velocities", "angular_velocities", "radii", "masses", "material_ids"):
        setattr(out, k, np.ascontiguousarray(getattr(ps, k)[mask]))
    return out


# ---------------------------------------------------------------------------------------------
# Transports

class LoopbackTransport:
    """Several ranks in one process (e.g. on one GPU): records are copied between the ranks'
    buffers directly. Used to validate the decomposition on a single device."""

    def __init__(self, ranks, ring: bool = False):
        self.ranks = ranks
        self.ring = ring  # periodic z: rank 0 and rank R-1 are neighbours

    def exchange(self, kind: str):
        R = len(self.ranks)
        for r, rk in enumerate(self.ranks):
            rk.recv_count[kind] = [0, 0]
        for r, rk in enumerate(self.ranks):
            n_lo, n_hi = rk.send_count[kind]
            lo, hi = r - 1, r + 1
            if self.ring:
                lo, hi = lo % R, hi % R
            if 0 <= lo and n_lo:  # to the rank below, which receives it from above
                self.ranks[lo].receive(kind, 1, rk.send_view(kind, 0, n_lo), n_lo)
            if hi < R and n_hi:
                self.ranks[hi].receive(kind, 0, rk.send_view(kind, 1, n_hi), n_hi)


class TorchTransport:
    """One rank per process over torch.distributed: counts, then payloads, to the z-neighbours
    with batched isend/irecv (NCCL P2P over NVLink for device buffers; gloo for CPU buffers).
    Each exchange is two half-exchanges — every rank sends up (its hi buffer) and receives from
    below, then sends down and receives from above — so that on a ring of 2 ranks, where the
    neighbour below and above are the same process, the two messages cannot be confused."""

    def __init__(self, rank: int, world: int, ring: bool = False):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = rank, world
        self.ring = ring
        self.ranks = None

    def bind(self, rk):
        self.ranks = [rk]

    def _half(self, rk, kind, dev, send_side, to, frm):
        """send buffer `send_side` to rank `to` (None: nobody), receive into the opposite side
        from rank `frm` (None: nobody); returns the received count."""
        torch, dist = self.torch, self.dist
        recv_side = 1 - send_side
        n_send = rk.send_count[kind][send_side]
        c_send = torch.tensor([n_send], dtype=torch.int64, device=dev)
        c_recv = torch.zeros(1, dtype=torch.int64, device=dev)
        ops = []
        if to is not None:
            ops.append(dist.P2POp(dist.isend, c_send, to))
        if frm is not None:
            ops.append(dist.P2POp(dist.irecv, c_recv, frm))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        m = int(c_recv[0].item()) if frm is not None else 0
        ops = []
        if to is not None and n_send:
            ops.append(dist.P2POp(dist.isend, rk.send_view(kind, send_side, n_send), to))
        if frm is not None and m:
            ops.append(dist.P2POp(dist.irecv, rk.recv_view(kind, recv_side, m), frm))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return m

    def exchange(self, kind: str):
        rk = self.ranks[0]
        dev = rk.buffer_device()
        R, r = self.world, self.rank
        lo = (r - 1) % R if (self.ring or r > 0) else None
        hi = (r + 1) % R if (self.ring or r < R - 1) else None
        if R == 1 and self.ring:  # a ring of one: both halves come back to this rank
            for side in (0, 1):
                n = rk.send_count[kind][side]
                rk.recv_view(kind, 1 - side, n).copy_(rk.send_view(kind, side, n))
            rk.recv_count[kind] = [rk.send_count[kind][1], rk.send_count[kind][0]]
            return
        m_lo = self._half(rk, kind, dev, 1, hi, lo)   # up: my hi buffer -> above; from below
        m_hi = self._half(rk, kind, dev, 0, lo, hi)   # down: my lo buffer -> below; from above
        if dev.type == "cuda":
            self.torch.cuda.current_stream(dev).synchronize()
        rk.recv_count[kind] = [m_lo, m_hi]


class PeerTransport:
    """One rank per process, records moved over NVLink peer memory instead of NCCL messages: each
    rank's receive buffers are CUDA-IPC-shared with its z-neighbours, whose migrate / halo pack
    kernels store the records straight into them (the pack and the transfer are one kernel).
    Only the record counts travel, as one all-gather on a gloo group, which also orders the
    neighbours' completed stores before this rank's unpack kernels. ring: periodic z."""

    def __init__(self, rank: int, world: int, ring: bool = False):
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.world, self.ring = rank, world, ring
        self.ctrl = dist.new_group(backend="gloo")
        self.ranks = None
        self.opened = []

    def _nbr(self):
        R, r = self.world, self.rank
        lo = (r - 1) % R if (self.ring or r > 0) else None
        hi = (r + 1) % R if (self.ring or r < R - 1) else None
        return lo, hi

    def bind(self, rk):
        lib = _capi.lib()
        self.ranks, self.lib, self.dev = [rk], lib, rk.device
        rk.peer_recv, handles = {}, {}
        for kind in ("migrant", "ghost"):
            rk.peer_recv[kind], handles[kind] = [], []
            for side in (0, 1):
                ptr = C.c_void_p()
                rc = lib.dem_ipc_alloc(self.dev, rk.cap[kind] * rk.rec_bytes[kind], C.byref(ptr))
                if rc != 0:
                    raise RuntimeError("dem_ipc_alloc failed")
                h = (C.c_char * 64)()
                if lib.dem_ipc_handle(self.dev, ptr, h) != 0:
                    raise RuntimeError("dem_ipc_handle failed")
                rk.peer_recv[kind].append(ptr.value)
                handles[kind].append(bytes(h))
        allh = [None] * self.world
        self.dist.all_gather_object(allh, handles, group=self.ctrl)
        lo, hi = self._nbr()
        rk.peer_send = {}
        for kind in ("migrant", "ghost"):
            rk.peer_send[kind] = [None, None]
            # my lo-side records land in the lower neighbour's "from above" buffer, and vice versa
            for side, nbr, their_side in ((0, lo, 1), (1, hi, 0)):
                if nbr is None:
                    continue
                if nbr == self.rank:
                    rk.peer_send[kind][side] = rk.peer_recv[kind][their_side]
                    continue
                ptr = C.c_void_p()
                if lib.dem_ipc_open(self.dev, (C.c_char * 64).from_buffer_copy(allh[nbr][kind][their_side]), C.byref(ptr)) != 0:
                    raise RuntimeError("dem_ipc_open failed (no peer access to rank %d?)" % nbr)
                rk.peer_send[kind][side] = ptr.value
                self.opened.append(ptr.value)

    def exchange(self, kind: str):
        import torch
        rk = self.ranks[0]
        mine = torch.tensor(rk.send_count[kind], dtype=torch.int64)
        allc = [torch.zeros(2, dtype=torch.int64) for _ in range(self.world)]
        self.dist.all_gather(allc, mine, group=self.ctrl)
        lo, hi = self._nbr()
        rk.recv_count[kind] = [int(allc[lo][1]) if lo is not None else 0,
                               int(allc[hi][0]) if hi is not None else 0]

    def close(self):
        for p in self.opened:
            self.lib.dem_ipc_close(self.dev, C.c_void_p(p))
        self.opened = []
        rk = self.ranks[0] if self.ranks else None
        if rk is not None and getattr(rk, "peer_recv", None):
            for kind in rk.peer_recv:
                for p in rk.peer_recv[kind]:
                    self.lib.dem_ipc_free(self.dev, C.c_void_p(p))
            rk.peer_recv, rk.peer_send = None, None


# ---------------------------------------------------------------------------------------------
# The CUDA-backed rank

class SlabRankCuda:
    """One slab on one GPU: a dem_create_slab context plus its record buffers (torch tensors,
    so NCCL can move them)."""

    def __init__(self, cfg: SimConfig, owned: ParticleSet, z_lo: int, z_hi: int, capacity: int,
                 device: int = 0, record_capacity: Optional[int] = None):
        import torch
        self.torch = torch
        self.lib = _capi.lib()
        self.cfg = cfg
        self.device = device
        self._ccfg = _Config(cfg)
        ps = owned.contiguous()
        ctx = C.c_void_p()
        rc = self.lib.dem_create_slab(C.byref(self._ccfg.c), C.byref(ps.c_struct()), device, z_lo, z_hi,
                                      capacity, C.byref(ctx))
        if rc != 0:
            _raise(self.lib, None, rc)
        self.ctx = ctx
        mb, gb = C.c_uint64(), C.c_uint64()
        self.lib.dem_slab_record_bytes(ctx, C.byref(mb), C.byref(gb))
        self.rec_bytes = {"migrant": mb.value, "ghost": gb.value}
        cap = record_capacity or max(4096, capacity // 4)
        self.cap = {"migrant": cap, "ghost": cap}
        dev = torch.device("cuda", device)
        self.send = {k: [torch.empty(self.cap[k] * self.rec_bytes[k], dtype=torch.uint8, device=dev) for _ in range(2)]
                     for k in self.cap}
        self.recv = {k: [torch.empty(self.cap[k] * self.rec_bytes[k], dtype=torch.uint8, device=dev) for _ in range(2)]
                     for k in self.cap}
        self.send_count = {"migrant": [0, 0], "ghost": [0, 0]}
        self.recv_count = {"migrant": [0, 0], "ghost": [0, 0]}

    def __del__(self):
        if getattr(self, "ctx", None):
            self.lib.dem_destroy(self.ctx)
            self.ctx = None

    def _check(self, rc):
        if rc != 0:
            _raise(self.lib, self.ctx, rc)

    def buffer_device(self):
        return self.send["migrant"][0].device

    # device pointers the pack / unpack kernels use: this rank's torch buffers, or — under
    # PeerTransport — the neighbours' receive buffers (send) and IPC-shareable ones (receive)
    def send_ptr(self, kind, side):
        o = getattr(self, "peer_send", None)
        return o[kind][side] if o and o[kind][side] else self.send[kind][side].data_ptr()

    def recv_ptr(self, kind, side):
        o = getattr(self, "peer_recv", None)
        return o[kind][side] if o else self.recv[kind][side].data_ptr()

    def send_view(self, kind, side, n):
        return self.send[kind][side][: n * self.rec_bytes[kind]]

    def recv_view(self, kind, side, n):
        return self.recv[kind][side][: n * self.rec_bytes[kind]]

    def receive(self, kind, side, data, n):  # loopback delivery
        self.recv_view(kind, side, n).copy_(data)
        self.recv_count[kind][side] = n

    # --- phases ---
    def migrate(self, integrate: bool):
        lo, hi = C.c_uint64(), C.c_uint64()
        self._check(self.lib.dem_slab_migrate(self.ctx, 1 if integrate else 0, self.send_ptr("migrant", 0),
                                              self.send_ptr("migrant", 1), self.cap["migrant"],
                                              C.byref(lo), C.byref(hi)))
        self.send_count["migrant"] = [lo.value, hi.value]

    def import_(self):
        self.torch.cuda.synchronize(self.device)
        n_lo, n_hi = self.recv_count["migrant"]
        self._check(self.lib.dem_slab_import(self.ctx, self.recv_ptr("migrant", 0), n_lo,
                                             self.recv_ptr("migrant", 1), n_hi))

    def halo(self):
        lo, hi = C.c_uint64(), C.c_uint64()
        self._check(self.lib.dem_slab_halo(self.ctx, self.send_ptr("ghost", 0), self.send_ptr("ghost", 1),
                                           self.cap["ghost"], C.byref(lo), C.byref(hi)))
        self.send_count["ghost"] = [lo.value, hi.value]

    def ghosts(self):
        self.torch.cuda.synchronize(self.device)
        n_lo, n_hi = self.recv_count["ghost"]
        self._check(self.lib.dem_slab_ghosts(self.ctx, self.recv_ptr("ghost", 0), n_lo,
                                             self.recv_ptr("ghost", 1), n_hi))

    def force(self, flags: int) -> StepMetrics:
        m = _capi.dem_step_metrics()
        self._check(self.lib.dem_slab_force(self.ctx, flags, C.byref(m)))
        return StepMetrics.from_c(m)

    # --- results (owned particles only) ---
    def owned(self):
        n = int(self.lib.dem_size(self.ctx))
        s = ParticleSet(n)
        self._check(self.lib.dem_get_particles(self.ctx, C.byref(s.c_struct())))
        f = np.zeros((n, 3))
        t = np.zeros((n, 3))
        self._check(self.lib.dem_get_forces(self.ctx, f.ctypes.data_as(C.POINTER(C.c_double)),
                                            t.ctypes.data_as(C.POINTER(C.c_double))))
        cnt = self.lib.dem_get_contacts(self.ctx, None, None, None, 0)
        o = np.zeros(cnt, np.uint32)
        p = np.zeros(cnt, np.int32)
        d = np.zeros((cnt, 3))
        self.lib.dem_get_contacts(self.ctx, o.ctypes.data_as(C.POINTER(C.c_uint32)),
                                  p.ctypes.data_as(C.POINTER(C.c_int32)), d.ctypes.data_as(C.POINTER(C.c_double)), cnt)
        own = (s.material_ids & GHOST_BIT) == 0
        ids = s.ids
        hist_owner = ids[o]
        hist_key = np.where(p >= 0, ids[np.maximum(p, 0)], p.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
        mine = own[o] if cnt else np.zeros(0, bool)
        return select(s, own), f[own], t[own], (hist_owner[mine], hist_key[mine], d[mine])


# ---------------------------------------------------------------------------------------------
# The driver: the per-step phase order for a set of local ranks and a transport

class SlabDriver:
    STEP = _capi.PHASE_STEP
    PRIME = _capi.PHASE_GRAVITY | _capi.PHASE_PP | _capi.PHASE_RECT | _capi.PHASE_LINE

    def __init__(self, ranks: Sequence, transport):
        self.ranks = list(ranks)
        self.transport = transport

    def _phase(self, integrate: bool, flags: int):
        for rk in self.ranks:
            rk.migrate(integrate)
        self.transport.exchange("migrant")
        for rk in self.ranks:
            rk.import_()
        for rk in self.ranks:
            rk.halo()
        self.transport.exchange("ghost")
        for rk in self.ranks:
            rk.ghosts()
        return [rk.force(flags) for rk in self.ranks]

    def prime(self):
        """The constructor's force-only pass (pipeline.cpp:83)."""
        return self._phase(False, self.PRIME)

    def step(self):
        """Simulation::step() (pipeline.cpp:366-378) on every local rank."""
        return self._phase(True, self.STEP)


def build_local_slabs(ps: ParticleSet, cfg: SimConfig, nranks: int, rank_ids: Sequence[int], device: int = 0,
                      headroom: float = 1.5, backend=SlabRankCuda):
    """Partition `ps` into `nranks` slabs and construct the ranks in `rank_ids` (all of them for a
    loopback run on one device, or just this process's rank under torch.distributed)."""
    g = global_grid(cfg, float(ps.radii.max()))
    scfg = replace(cfg, grid_cell_size=g.h)
    planes = cell_planes(ps.positions[:, 2], g)
    bounds = slab_bounds(planes, g.nz, nranks)
    per_plane = np.bincount(planes, minlength=g.nz)
    ranks = []
    for r in rank_ids:
        z_lo, z_hi = bounds[r]
        mask = (planes >= z_lo) & (planes < z_hi)
        owned = select(ps, mask)
        if g.ring:
            ghosts = per_plane[(z_lo - 1) % g.nz] + per_plane[z_hi % g.nz]
        else:
            ghosts = (per_plane[z_lo - 1] if z_lo > 0 else 0) + (per_plane[z_hi] if z_hi < g.nz else 0)
        capacity = int(1024 + headroom * (len(owned.ids) + ghosts))
        ranks.append(backend(scfg, owned, z_lo, z_hi, capacity, device=device))
    return ranks, bounds, g


# ---------------------------------------------------------------------------------------------
# Host-free sharded stepping (dem_create_sharded): the whole step is one CUDA graph
# per rank, counts stay on the device, neighbours store records into each other's inboxes.

def _owned_of(lib, ctx, check):
    """The slab's owned particles, their forces and history rows (halo copies dropped)."""
    n = int(lib.dem_size(ctx))
    s = ParticleSet(n)
    check(lib.dem_get_particles(ctx, C.byref(s.c_struct())))
    f = np.zeros((n, 3))
    t = np.zeros((n, 3))
    check(lib.dem_get_forces(ctx, f.ctypes.data_as(C.POINTER(C.c_double)), t.ctypes.data_as(C.POINTER(C.c_double))))
    cnt = lib.dem_get_contacts(ctx, None, None, None, 0)
    o = np.zeros(cnt, np.uint32)
    p = np.zeros(cnt, np.int32)
    d = np.zeros((cnt, 3))
    lib.dem_get_contacts(ctx, o.ctypes.data_as(C.POINTER(C.c_uint32)), p.ctypes.data_as(C.POINTER(C.c_int32)),
                         d.ctypes.data_as(C.POINTER(C.c_double)), cnt)
    own = (s.material_ids & GHOST_BIT) == 0
    ids = s.ids
    hist_owner = ids[o]
    hist_key = np.where(p >= 0, ids[np.maximum(p, 0)], p.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
    mine = own[o] if cnt else np.zeros(0, bool)
    return select(s, own), f[own], t[own], (hist_owner[mine], hist_key[mine], d[mine])


class ShardedSimulation:
    """Rank `rank` of `nranks` of the host-free sharded step. Every rank passes the same GLOBAL
    initial set; the library keeps this rank's z-slab. Connect with connect_torch (one process per
    rank, CUDA-IPC inboxes over NVLink) or connect_local (ranks of one process)."""

    def __init__(self, all_particles: ParticleSet, cfg: SimConfig, rank: int, nranks: int, device: int = 0):
        self.lib = _capi.lib()
        self.cfg, self.rank, self.nranks, self.device = cfg, rank, nranks, device
        self._ccfg = _Config(cfg)
        ps = all_particles.contiguous()
        ctx = C.c_void_p()
        rc = self.lib.dem_create_sharded(C.byref(self._ccfg.c), C.byref(ps.c_struct()), device, rank, nranks,
                                         C.byref(ctx))
        if rc != 0:
            _raise(self.lib, None, rc)
        self.ctx = ctx

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.dem_destroy(self.ctx)
            self.ctx = None

    def _check(self, rc):
        if rc != 0:
            _raise(self.lib, self.ctx, rc)

    def info(self):
        lo, hi, n = C.c_int32(), C.c_int32(), C.c_uint64()
        self._check(self.lib.dem_shard_info(self.ctx, C.byref(lo), C.byref(hi), C.byref(n)))
        return lo.value, hi.value, n.value

    def handle(self) -> bytes:
        h = (C.c_char * 64)()
        self._check(self.lib.dem_shard_handle(self.ctx, h))
        return bytes(h)

    def connect(self, handles: Sequence[bytes]):
        buf = (C.c_char * (64 * len(handles))).from_buffer_copy(b"".join(handles))
        self._check(self.lib.dem_shard_connect(self.ctx, buf))

    def connect_local(self, lo: Optional["ShardedSimulation"], hi: Optional["ShardedSimulation"]):
        self._check(self.lib.dem_shard_connect_local(self.ctx, lo.ctx if lo else None, hi.ctx if hi else None))

    def launch(self, n: int = 1):
        self._check(self.lib.dem_shard_launch(self.ctx, n))

    def wait(self) -> StepMetrics:
        m = _capi.dem_step_metrics()
        self._check(self.lib.dem_shard_wait(self.ctx, C.byref(m)))
        return StepMetrics.from_c(m)

    def step(self, n: int = 1) -> StepMetrics:
        """n graph-launched steps (one rank per process: dem_step = launch + wait)."""
        m = _capi.dem_step_metrics()
        self._check(self.lib.dem_step(self.ctx, n, C.byref(m)))
        return StepMetrics.from_c(m)

    def time_steps(self, nsteps: int, flush_bytes: int = 0):
        ms = (C.c_float * max(nsteps, 1))()
        m = _capi.dem_step_metrics()
        self._check(self.lib.dem_time_steps(self.ctx, nsteps, flush_bytes, ms, C.byref(m)))
        return [float(ms[k]) for k in range(nsteps)], StepMetrics.from_c(m)

    def size(self) -> int:
        return int(self.lib.dem_size(self.ctx))

    def owned(self):
        return _owned_of(self.lib, self.ctx, self._check)


def connect_torch(sim: ShardedSimulation, group=None):
    """All-gather the 64-byte inbox handles over torch.distributed (any backend) and connect."""
    import torch.distributed as dist
    allh = [None] * sim.nranks
    dist.all_gather_object(allh, sim.handle(), group=group)
    sim.connect(allh)


def local_shards(ps: ParticleSet, cfg: SimConfig, nranks: int, device: int = 0) -> List[ShardedSimulation]:
    """All ranks of one process (one GPU or several with peer access), wired directly."""
    shards = [ShardedSimulation(ps, cfg, r, nranks, device) for r in range(nranks)]
    ring = bool(getattr(cfg, "periodic", 0) & 4)
    for r, sh in enumerate(shards):
        lo = shards[(r - 1) % nranks] if (ring or r > 0) else None
        hi = shards[(r + 1) % nranks] if (ring or r < nranks - 1) else None
        sh.connect_local(lo, hi)
    return shards


def step_local(shards: Sequence[ShardedSimulation], n: int = 1) -> List[StepMetrics]:
    """n steps of every rank of one process: launch all, then wait for all."""
    for sh in shards:
        sh.launch(n)
    return [sh.wait() for sh in shards]
