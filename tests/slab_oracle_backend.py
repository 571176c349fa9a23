"""TEST INFRASTRUCTURE: a CPU slab rank backed by the C oracle, with the same interface as
paper_1503_03553_b200.slab.SlabRankCuda, so the decomposition protocol (partitioning, exchange
pattern, phase order, migrant/ghost record semantics, history hand-over) can be exercised with
world_size > 1 over gloo on a machine without a GPU.

Records are numpy structured arrays carried in uint8 torch CPU tensors. Supported subset: the
pp-only step without walls (gravity 0), which is the benchmark configuration.
"""
import math

import numpy as np

from oracle.oracle import Oracle, collide_arrays, orc_grid


def record_dtype(K):
    return np.dtype([("pos", "<f8", (3,)), ("vel", "<f8", (3,)), ("omg", "<f8", (3,)), ("rad", "<f8"),
                     ("mass", "<f8"), ("id", "<u4"), ("mat", "<u4"), ("hcnt", "<u4"), ("pad", "<u4"),
                     ("hkey", "<u4", (K,)), ("hdt", "<f8", (K, 3))])


class SlabRankOracle:
    def __init__(self, cfg, owned, z_lo, z_hi, capacity, device=0, record_capacity=None):
        import torch
        self.torch = torch
        self.cfg = cfg
        self.K = cfg.contact_capacity
        self.z_lo, self.z_hi = z_lo, z_hi
        self.orc = Oracle()
        h = cfg.grid_cell_size
        ext = [cfg.domain_max[a] - cfg.domain_min[a] for a in range(3)]
        self.h, self.inv_h = h, 1.0 / h
        self.dims = [max(1, int(math.ceil(e / h))) for e in ext]
        self.grid = orc_grid(tuple(cfg.domain_min), h, *self.dims)
        self.dtype = record_dtype(self.K)
        self.rb = self.dtype.itemsize
        self.cap = record_capacity or max(4096, capacity)
        self.own = {k: np.array(getattr(owned, k)).copy() for k in
                    ("ids", "positions", "velocities", "angular_velocities", "radii", "masses", "material_ids")}
        n = len(self.own["ids"])
        self.F = np.zeros((n, 3))
        self.T = np.zeros((n, 3))
        self.hist = {}  # owner id -> list of (partner key, dt) of the previous phase
        self.ghost = None
        self.send = {"migrant": [None, None], "ghost": [None, None]}
        self.recv = {"migrant": [None, None], "ghost": [None, None]}
        self.send_count = {"migrant": [0, 0], "ghost": [0, 0]}
        self.recv_count = {"migrant": [0, 0], "ghost": [0, 0]}
        self.metrics = None

    def _tensor(self, recs):
        b = recs.tobytes()
        return self.torch.frombuffer(bytearray(b), dtype=self.torch.uint8) if b else self.torch.zeros(0, dtype=self.torch.uint8)

    # --- transport hooks ---
    def buffer_device(self):
        return self.torch.device("cpu")

    def send_view(self, kind, side, n):
        return self.send[kind][side]

    def recv_view(self, kind, side, n):
        t = self.torch.zeros(n * self.rb, dtype=self.torch.uint8)
        self.recv[kind][side] = t
        return t

    def receive(self, kind, side, data, n):
        self.recv[kind][side] = data.clone()
        self.recv_count[kind][side] = n

    def _records(self, kind, side):
        n = self.recv_count[kind][side]
        if not n:
            return np.zeros(0, self.dtype)
        return np.frombuffer(self.recv[kind][side].numpy().tobytes(), dtype=self.dtype, count=n)

    def _planes(self, z):
        f = np.floor((z - self.cfg.domain_min[2]) * self.inv_h)
        return np.clip(np.where(np.isfinite(f), f, -1.0), 0, self.dims[2] - 1).astype(np.int64)

    def _pack(self, sel, with_hist):
        o = self.own
        r = np.zeros(int(sel.sum()), self.dtype)
        r["pos"], r["vel"], r["omg"] = o["positions"][sel], o["velocities"][sel], o["angular_velocities"][sel]
        r["rad"], r["mass"], r["id"], r["mat"] = o["radii"][sel], o["masses"][sel], o["ids"][sel], o["material_ids"][sel]
        if with_hist:
            for k, pid in enumerate(o["ids"][sel]):
                rows = self.hist.get(int(pid), [])
                r["hcnt"][k] = len(rows)
                for q, (key, dt) in enumerate(rows):
                    r["hkey"][k, q] = key
                    r["hdt"][k, q] = dt
        return r

    def _keep(self, sel):
        for k in self.own:
            self.own[k] = self.own[k][sel]

    # --- phases (same semantics as dem_slab_*) ---
    def migrate(self, integrate):
        o = self.own
        if integrate:  # pipeline.cpp:31-44, element-wise IEEE ops in the reference order
            m, r = o["masses"], o["radii"]
            s = self.cfg.dt / m
            o["velocities"] = o["velocities"] + self.F * s[:, None]
            o["positions"] = o["positions"] + o["velocities"] * self.cfg.dt
            inertia = 0.4 * m * r * r
            s2 = self.cfg.dt / inertia
            o["angular_velocities"] = o["angular_velocities"] + self.T * s2[:, None]
        cz = self._planes(o["positions"][:, 2])
        lo, hi = cz < self.z_lo, cz >= self.z_hi
        recs = [self._pack(lo, True), self._pack(hi, True)]
        for pid in o["ids"][lo | hi]:
            self.hist.pop(int(pid), None)
        self._keep(~(lo | hi))
        for side in (0, 1):
            self.send["migrant"][side] = self._tensor(recs[side])
        self.send_count["migrant"] = [len(recs[0]), len(recs[1])]

    def _append(self, recs, ghost):
        if ghost:
            g = self.ghost
            for k, f in (("ids", "id"), ("positions", "pos"), ("velocities", "vel"), ("angular_velocities", "omg"),
                         ("radii", "rad"), ("masses", "mass"), ("material_ids", "mat")):
                g[k] = np.concatenate([g[k], recs[f]])
            return
        o = self.own
        for k, f in (("ids", "id"), ("positions", "pos"), ("velocities", "vel"), ("angular_velocities", "omg"),
                     ("radii", "rad"), ("masses", "mass"), ("material_ids", "mat")):
            o[k] = np.concatenate([o[k], recs[f]])
        for r in recs:
            self.hist[int(r["id"])] = [(int(r["hkey"][q]), r["hdt"][q].copy()) for q in range(int(r["hcnt"]))]

    def import_(self):
        for side in (0, 1):
            self._append(self._records("migrant", side), ghost=False)

    def halo(self):
        cz = self._planes(self.own["positions"][:, 2])
        recs = [self._pack(cz == self.z_lo, False), self._pack(cz == self.z_hi - 1, False)]
        for side in (0, 1):
            self.send["ghost"][side] = self._tensor(recs[side])
        self.send_count["ghost"] = [len(recs[0]), len(recs[1])]

    def ghosts(self):
        self.ghost = {k: v[:0].copy() for k, v in self.own.items()}
        for side in (0, 1):
            self._append(self._records("ghost", side), ghost=True)

    def force(self, flags):
        o, g = self.own, self.ghost
        n_own = len(o["ids"])
        u = {k: np.concatenate([o[k], g[k]]) for k in o}
        nx, ny, nz = self.dims
        ox, oy, oz = self.cfg.domain_min

        def axis(v, org, dim):
            f = np.floor((v - org) * self.inv_h)
            return np.clip(np.where(np.isfinite(f), f, -1.0), 0, dim - 1).astype(np.int64)

        key = axis(u["positions"][:, 0], ox, nx) + nx * (axis(u["positions"][:, 1], oy, ny) + ny * axis(u["positions"][:, 2], oz, nz))
        order = np.lexsort((u["ids"], key))  # canonical (cell, stable id)

        class S:
            pass
        st = S()
        st.ids = u["ids"][order]
        st.positions = u["positions"][order]
        st.velocities = u["velocities"][order]
        st.angular_velocities = u["angular_velocities"][order]
        st.radii = u["radii"][order]
        st.masses = u["masses"][order]
        st.material_ids = u["material_ids"][order]
        ho, hk, hd = [], [], []
        for pid, rows in self.hist.items():
            for key_, dt in rows:
                ho.append(pid)
                hk.append(key_)
                hd.append(dt)
        f, t, (to, tk, td), ev = collide_arrays(self.orc, st, self.cfg, self.grid,
                                                np.array(ho, np.uint32), np.array(hk, np.uint32),
                                                np.array(hd).reshape(-1, 3))
        is_own = order < n_own
        slot_of = np.empty(len(order), np.int64)
        slot_of[order] = np.arange(len(order))
        own_slots = slot_of[:n_own]
        self.F, self.T = f[own_slots], t[own_slots]
        own_ids = set(int(x) for x in o["ids"])
        self.hist = {}
        contacts = 0
        for a, b, d in zip(to, tk, td):
            if int(a) in own_ids:
                self.hist.setdefault(int(a), []).append((int(b), d.copy()))
                contacts += 1
        self.metrics = contacts
        return contacts

    def owned(self):
        o = self.own
        ho, hk, hd = [], [], []
        for pid, rows in self.hist.items():
            for key_, dt in rows:
                ho.append(pid)
                hk.append(key_)
                hd.append(dt)

        class P:
            pass
        p = P()
        for k in o:
            setattr(p, k, o[k])
        return p, self.F, self.T, (np.array(ho, np.uint32), np.array(hk, np.uint32), np.array(hd).reshape(-1, 3))
