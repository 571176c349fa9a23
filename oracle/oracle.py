"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracles.

* ``Oracle``  : oracle/liboracle.so, the plain-C restatement of the reference path
                (dem_oracle.c; every function cites the reference file:line it restates).
* ``RefLib``  : oracle/_ref/libdemforge_ref.so, the UNMODIFIED reference core compiled from its
                own sources plus our extern "C" shim (ref_shim.cpp). Used to pin the
                restatement and as the CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdemforge_ref.so")

D3 = C.c_double * 3
PD = C.POINTER(C.c_double)
PU = C.POINTER(C.c_uint32)
PI = C.POINTER(C.c_int32)


class orc_material(C.Structure):
    _fields_ = [("poisson_ratio", C.c_double), ("shear_modulus", C.c_double),
                ("youngs_modulus", C.c_double), ("restitution", C.c_double),
                ("sliding_friction", C.c_double)]


class orc_rect(C.Structure):
    _fields_ = [("corner", D3), ("edge_u", D3), ("edge_v", D3), ("material_id", C.c_uint32)]


class orc_line(C.Structure):
    _fields_ = [("a", D3), ("b", D3), ("material_id", C.c_uint32)]


class orc_config(C.Structure):
    _fields_ = [("dt", C.c_double), ("gravity", D3), ("domain_min", D3), ("domain_max", D3),
                ("material_count", C.c_uint32), ("materials", C.POINTER(orc_material)),
                ("pair_restitution", PD), ("rect_count", C.c_uint32),
                ("rects", C.POINTER(orc_rect)), ("line_count", C.c_uint32),
                ("lines", C.POINTER(orc_line)), ("grid_cell_size", C.c_double),
                ("contact_capacity", C.c_int32), ("periodic", C.c_uint32), ("shear_rate", C.c_double)]


class orc_grid(C.Structure):
    _fields_ = [("origin", D3), ("cell_size", C.c_double), ("nx", C.c_int32), ("ny", C.c_int32),
                ("nz", C.c_int32)]


class orc_hist(C.Structure):
    _fields_ = [("owner_id", C.c_uint32), ("partner_key", C.c_uint32), ("delta_t", D3)]


class orc_metrics(C.Structure):
    _fields_ = [("step", C.c_int64), ("contacts", C.c_int64), ("pp_contact_events", C.c_int64),
                ("max_contacts_per_particle", C.c_int32), ("clamps", C.c_int64),
                ("friction_max_ratio", C.c_double)]


class orc_error(C.Structure):
    _fields_ = [("code", C.c_int32), ("kernel", C.c_int32), ("particle_slot", C.c_uint32),
                ("particle_id", C.c_uint32), ("step", C.c_int64)]


class CConfig:
    """orc_config built from a paper_1503_03553_b200.SimConfig-like object (duck-typed)."""

    def __init__(self, cfg):
        m = cfg.materials.size()
        self.mats = (orc_material * max(m, 1))()
        for k in range(m):
            p = cfg.materials.params(k)
            self.mats[k] = orc_material(p.poisson_ratio, p.shear_modulus, p.youngs_modulus,
                                        p.restitution, p.sliding_friction)
        self.pair = (C.c_double * max(m * m, 1))()
        for a in range(m):
            for b in range(m):
                self.pair[a * m + b] = cfg.materials.pair_restitution(a, b)
        self.rects = (orc_rect * max(len(cfg.rect_walls), 1))()
        for k, w in enumerate(cfg.rect_walls):
            self.rects[k] = orc_rect(D3(*w.corner), D3(*w.edge_u), D3(*w.edge_v), w.material_id)
        self.lines = (orc_line * max(len(cfg.line_walls), 1))()
        for k, w in enumerate(cfg.line_walls):
            self.lines[k] = orc_line(D3(*w.a), D3(*w.b), w.material_id)
        c = orc_config()
        c.dt = cfg.dt
        c.gravity = D3(*cfg.gravity)
        c.domain_min = D3(*cfg.domain_min)
        c.domain_max = D3(*cfg.domain_max)
        c.material_count = m
        c.materials = self.mats
        c.pair_restitution = self.pair
        c.rect_count = len(cfg.rect_walls)
        c.rects = self.rects
        c.line_count = len(cfg.line_walls)
        c.lines = self.lines
        c.grid_cell_size = cfg.grid_cell_size
        c.contact_capacity = cfg.contact_capacity
        c.periodic = getattr(cfg, "periodic", 0)
        c.shear_rate = getattr(cfg, "shear_rate", 0.0)
        self.c = c


def _arr(ps):
    """(n, ids, pos, vel, omg, rad, mass, mat) ctypes pointers for a ParticleSet-like object."""
    ids = np.ascontiguousarray(ps.ids, np.uint32)
    pos = np.ascontiguousarray(ps.positions, np.float64)
    vel = np.ascontiguousarray(ps.velocities, np.float64)
    omg = np.ascontiguousarray(ps.angular_velocities, np.float64)
    rad = np.ascontiguousarray(ps.radii, np.float64)
    mass = np.ascontiguousarray(ps.masses, np.float64)
    mat = np.ascontiguousarray(ps.material_ids, np.uint32)
    keep = (ids, pos, vel, omg, rad, mass, mat)
    ptrs = (ids.ctypes.data_as(PU), pos.ctypes.data_as(PD), vel.ctypes.data_as(PD),
            omg.ctypes.data_as(PD), rad.ctypes.data_as(PD), mass.ctypes.data_as(PD),
            mat.ctypes.data_as(PU))
    return len(ids), keep, ptrs


class State:
    """Plain numpy particle state (same field names as ParticleSet)."""

    def __init__(self, n):
        self.ids = np.zeros(n, np.uint32)
        self.positions = np.zeros((n, 3))
        self.velocities = np.zeros((n, 3))
        self.angular_velocities = np.zeros((n, 3))
        self.radii = np.zeros(n)
        self.masses = np.zeros(n)
        self.material_ids = np.zeros(n, np.uint32)

    def ptrs(self):
        return (self.ids.ctypes.data_as(PU), self.positions.ctypes.data_as(PD),
                self.velocities.ctypes.data_as(PD), self.angular_velocities.ctypes.data_as(PD),
                self.radii.ctypes.data_as(PD), self.masses.ctypes.data_as(PD),
                self.material_ids.ctypes.data_as(PU))


class OracleError(RuntimeError):
    def __init__(self, code, kernel=-1, slot=0, pid=0, step=0, msg=""):
        super().__init__(msg or f"oracle error code={code} kernel={kernel} slot={slot} id={pid} step={step}")
        self.code, self.kernel, self.slot, self.pid, self.step = code, kernel, slot, pid, step


# ---------------------------------------------------------------------------------------------
class Oracle:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: make -C oracle")
        L = self.L = C.CDLL(path)
        L.orc_restitution_alpha.restype = C.c_double
        L.orc_restitution_alpha.argtypes = [C.c_double]
        L.orc_contact_coefficients.argtypes = [C.c_double, C.POINTER(orc_material), C.POINTER(orc_material),
                                               C.c_double, C.c_double, C.c_double, C.c_double,
                                               C.c_double, C.c_int, PD]
        L.orc_contact_geometry.restype = C.c_int
        L.orc_contact_geometry.argtypes = [PD, C.c_double, PD, PD, PD, C.c_int, C.c_double, PD, PD, PD]
        L.orc_contact_force.argtypes = [PD, PD, PD, C.c_double, C.c_double, PD]
        L.orc_update_tangential.argtypes = [PD, PD, PD, C.c_double, PD]
        L.orc_make_grid.restype = C.c_int
        L.orc_make_grid.argtypes = [PD, PD, C.c_double, C.c_double, C.POINTER(orc_grid)]
        L.orc_calc_hash.restype = C.c_uint32
        L.orc_calc_hash.argtypes = [PD, C.POINTER(orc_grid), C.POINTER(C.c_int)]
        L.orc_neighbor_cells.restype = C.c_int
        L.orc_neighbor_cells.argtypes = [C.c_uint32, C.POINTER(orc_grid), PU]
        L.orc_closest_point_rect.argtypes = [PD, C.POINTER(orc_rect), PD]
        L.orc_closest_point_line.argtypes = [PD, C.POINTER(orc_line), PD]
        L.orc_contact_pairs.restype = C.c_int64
        L.orc_contact_pairs.argtypes = [C.c_size_t, PD, PD, C.c_int, PU, PU, C.c_int64]
        L.orc_collide.restype = C.c_int64
        L.orc_collide.argtypes = [C.c_size_t, PU, PD, PD, PD, PD, PD, PU, C.POINTER(orc_config),
                                  C.POINTER(orc_grid), C.POINTER(orc_hist), C.c_int64, PD, PD,
                                  C.POINTER(orc_hist), PU, PU, C.c_int64]
        L.orc_sim_create.restype = C.c_void_p
        L.orc_sim_create.argtypes = [C.POINTER(orc_config), C.c_size_t, PU, PD, PD, PD, PD, PD, PU,
                                     C.POINTER(orc_error)]
        L.orc_sim_destroy.argtypes = [C.c_void_p]
        L.orc_sim_step.restype = C.c_int
        L.orc_sim_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(orc_metrics), C.POINTER(orc_error)]
        L.orc_sim_force_phase.restype = C.c_int
        L.orc_sim_force_phase.argtypes = [C.c_void_p, C.c_int, C.POINTER(orc_metrics), C.POINTER(orc_error)]
        L.orc_sim_size.restype = C.c_size_t
        L.orc_sim_size.argtypes = [C.c_void_p]
        L.orc_sim_get_state.argtypes = [C.c_void_p, PU, PD, PD, PD, PD, PD, PU]
        L.orc_sim_get_forces.argtypes = [C.c_void_p, PD, PD]
        L.orc_sim_get_keys.argtypes = [C.c_void_p, PU]
        L.orc_sim_get_force_scale.argtypes = [C.c_void_p, PD, PD]
        L.orc_sim_history_count.restype = C.c_int64
        L.orc_sim_history_count.argtypes = [C.c_void_p]
        L.orc_sim_get_history.argtypes = [C.c_void_p, C.POINTER(orc_hist)]
        L.orc_sim_get_grid.argtypes = [C.c_void_p, C.POINTER(orc_grid)]
        L.orc_sim_get_pbox.argtypes = [C.c_void_p, PD, PD, C.POINTER(C.c_int64)]

    # -- pure functions --
    def restitution_alpha(self, e):
        return self.L.orc_restitution_alpha(e)

    def contact_coefficients(self, dn, m1, m2, r1, r2, ma, mb, alpha, wall):
        out = (C.c_double * 4)()
        a = orc_material(*m1)
        b = orc_material(*m2)
        self.L.orc_contact_coefficients(dn, C.byref(a), C.byref(b), r1, r2, ma, mb, alpha, int(wall), out)
        return list(out)

    def contact_geometry(self, p1, r1, v1, w1, pp, wall, r2=0.0, v2=(0, 0, 0), w2=(0, 0, 0)):
        out = (C.c_double * 10)()
        rc = self.L.orc_contact_geometry(D3(*p1), r1, D3(*v1), D3(*w1), D3(*pp), int(wall), r2,
                                         D3(*v2), D3(*w2), out)
        return rc, list(out)

    def contact_force(self, geom, coeffs, delta, mu, r1):
        out = (C.c_double * 12)()
        self.L.orc_contact_force((C.c_double * 10)(*geom), (C.c_double * 4)(*coeffs), D3(*delta), mu, r1, out)
        return list(out)

    def update_tangential(self, old, n, vt, dt):
        out = D3()
        self.L.orc_update_tangential(D3(*old), D3(*n), D3(*vt), dt, out)
        return list(out)

    def make_grid(self, bmin, bmax, rmax, h=0.0):
        g = orc_grid()
        rc = self.L.orc_make_grid(D3(*bmin), D3(*bmax), rmax, h, C.byref(g))
        return rc, g

    def calc_hash(self, p, g):
        cl = C.c_int(0)
        k = self.L.orc_calc_hash(D3(*p), C.byref(g), C.byref(cl))
        return k, bool(cl.value)

    def neighbor_cells(self, cell, g):
        out = (C.c_uint32 * 27)()
        n = self.L.orc_neighbor_cells(cell, C.byref(g), out)
        return list(out)[:n]

    def closest_point_rect(self, p, corner, u, v):
        out = (C.c_double * 4)()
        w = orc_rect(D3(*corner), D3(*u), D3(*v), 0)
        self.L.orc_closest_point_rect(D3(*p), C.byref(w), out)
        return list(out)

    def closest_point_line(self, p, a, b):
        out = (C.c_double * 4)()
        w = orc_line(D3(*a), D3(*b), 0)
        self.L.orc_closest_point_line(D3(*p), C.byref(w), out)
        return list(out)

    def contact_pairs(self, positions, radii, binned=True):
        pos = np.ascontiguousarray(positions, np.float64)
        rad = np.ascontiguousarray(radii, np.float64)
        n = len(rad)
        cap = max(16, 8 * n)
        while True:
            oi = np.zeros(cap, np.uint32)
            oj = np.zeros(cap, np.uint32)
            c = self.L.orc_contact_pairs(n, pos.ctypes.data_as(PD), rad.ctypes.data_as(PD),
                                         1 if binned else 0, oi.ctypes.data_as(PU), oj.ctypes.data_as(PU), cap)
            if c >= 0:
                return oi[:c].copy(), oj[:c].copy()
            cap = -c + 16

    def collide(self, state, cfg, grid, hist_in):
        """oracle_collide restatement: returns (forces, torques, hist_out array of orc_hist, events)."""
        n, keep, ptrs = _arr(state)
        cc = CConfig(cfg)
        hin = (orc_hist * max(len(hist_in), 1))(*hist_in)
        cap = max(16, n * cfg.contact_capacity)
        f = np.zeros((n, 3))
        t = np.zeros((n, 3))
        hout = (orc_hist * cap)()
        eo = np.zeros(cap, np.uint32)
        ep = np.zeros(cap, np.uint32)
        c = self.L.orc_collide(n, *ptrs, C.byref(cc.c), C.byref(grid), hin, len(hist_in),
                               f.ctypes.data_as(PD), t.ctypes.data_as(PD), hout,
                               eo.ctypes.data_as(PU), ep.ctypes.data_as(PU), cap)
        if c < 0:
            raise OracleError(-c)
        return f, t, list(hout[:c]), (eo[:c].copy(), ep[:c].copy())


HIST_DTYPE = np.dtype([("owner_id", "<u4"), ("partner_key", "<u4"), ("delta_t", "<f8", (3,))])
assert HIST_DTYPE.itemsize == C.sizeof(orc_hist)


def collide_arrays(orc: "Oracle", state, cfg, grid, owner_ids, partner_keys, delta_t):
    """Vectorised Oracle.collide for large N: history in/out as numpy arrays.
    Returns forces, torques, (owner_id, partner_key, delta_t) touched, (ev_owner, ev_partner)."""
    n, keep, ptrs = _arr(state)
    cc = CConfig(cfg)
    hin = np.zeros(max(len(owner_ids), 1), HIST_DTYPE)
    hin["owner_id"][:len(owner_ids)] = owner_ids
    hin["partner_key"][:len(owner_ids)] = partner_keys
    hin["delta_t"][:len(owner_ids)] = delta_t
    cap = max(16, n * cfg.contact_capacity)
    f = np.zeros((n, 3))
    t = np.zeros((n, 3))
    hout = np.zeros(cap, HIST_DTYPE)
    eo = np.zeros(cap, np.uint32)
    ep = np.zeros(cap, np.uint32)
    c = orc.L.orc_collide(n, *ptrs, C.byref(cc.c), C.byref(grid),
                          hin.ctypes.data_as(C.POINTER(orc_hist)), len(owner_ids),
                          f.ctypes.data_as(PD), t.ctypes.data_as(PD),
                          hout.ctypes.data_as(C.POINTER(orc_hist)), eo.ctypes.data_as(PU),
                          ep.ctypes.data_as(PU), cap)
    if c < 0:
        raise OracleError(-c)
    h = hout[:c]
    return f, t, (h["owner_id"].copy(), h["partner_key"].copy(), h["delta_t"].copy()), (eo[:c].copy(), ep[:c].copy())


class OracleSim:
    """Full-step restatement with canonical (cell, stable id) order (pipeline.cpp:31-378)."""

    def __init__(self, orc: Oracle, state, cfg):
        self.o = orc
        self.cc = CConfig(cfg)
        n, keep, ptrs = _arr(state)
        err = orc_error()
        self.h = orc.L.orc_sim_create(C.byref(self.cc.c), n, *ptrs, C.byref(err))
        if not self.h:
            raise OracleError(err.code, err.kernel, err.particle_slot, err.particle_id, err.step)
        self.n = n

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.orc_sim_destroy(self.h)
            self.h = None

    def step(self, k=1):
        m, err = orc_metrics(), orc_error()
        rc = self.o.L.orc_sim_step(self.h, k, C.byref(m), C.byref(err))
        if rc:
            raise OracleError(rc, err.kernel, err.particle_slot, err.particle_id, err.step)
        return m

    def force_phase(self, flags):
        m, err = orc_metrics(), orc_error()
        rc = self.o.L.orc_sim_force_phase(self.h, flags, C.byref(m), C.byref(err))
        if rc:
            raise OracleError(rc, err.kernel, err.particle_slot, err.particle_id, err.step)
        return m

    def state(self):
        s = State(self.n)
        self.o.L.orc_sim_get_state(self.h, *s.ptrs())
        return s

    def forces(self):
        f = np.zeros((self.n, 3))
        t = np.zeros((self.n, 3))
        self.o.L.orc_sim_get_forces(self.h, f.ctypes.data_as(PD), t.ctypes.data_as(PD))
        return f, t

    def force_scale(self):
        """Per slot: sum of |F| and of |T| contributions of the last phase (SURVEY §8a's 1e-9 scale)."""
        f = np.zeros(self.n)
        t = np.zeros(self.n)
        self.o.L.orc_sim_get_force_scale(self.h, f.ctypes.data_as(PD), t.ctypes.data_as(PD))
        return f, t

    def keys(self):
        k = np.zeros(self.n, np.uint32)
        self.o.L.orc_sim_get_keys(self.h, k.ctypes.data_as(PU))
        return k

    def history(self):
        c = self.o.L.orc_sim_history_count(self.h)
        h = (orc_hist * max(c, 1))()
        self.o.L.orc_sim_get_history(self.h, h)
        return list(h[:c])

    def grid(self):
        g = orc_grid()
        self.o.L.orc_sim_get_grid(self.h, C.byref(g))
        return g

    def pbox(self):
        """(cell extent per axis, Lees-Edwards offset, integrates so far)"""
        ext, off, st = D3(), C.c_double(), C.c_int64()
        self.o.L.orc_sim_get_pbox(self.h, ext, C.byref(off), C.byref(st))
        return tuple(ext), off.value, st.value


# ---------------------------------------------------------------------------------------------
class RefLib:
    """The reference core itself (oracle/_ref/libdemforge_ref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: make -C oracle (needs /root/reference)")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_thread_count.restype = C.c_int
        L.ref_sim_create.restype = C.c_void_p
        L.ref_sim_create.argtypes = [C.POINTER(orc_config), C.c_size_t, PU, PD, PD, PD, PD, PD, PU,
                                     C.POINTER(C.c_int)]
        L.ref_sim_clone.restype = C.c_void_p
        L.ref_sim_clone.argtypes = [C.c_void_p]
        L.ref_sim_destroy.argtypes = [C.c_void_p]
        L.ref_sim_set_record_traces.argtypes = [C.c_void_p, C.c_int]
        L.ref_sim_step.restype = C.c_int
        L.ref_sim_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(orc_metrics)]
        L.ref_sim_run_kernel.restype = C.c_int
        L.ref_sim_run_kernel.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_sim_size.restype = C.c_size_t
        L.ref_sim_size.argtypes = [C.c_void_p]
        L.ref_sim_get_state.argtypes = [C.c_void_p, PU, PD, PD, PD, PD, PD, PU]
        L.ref_sim_get_forces.argtypes = [C.c_void_p, PD, PD]
        L.ref_sim_get_grid.argtypes = [C.c_void_p, C.POINTER(orc_grid)]
        L.ref_sim_mean_coordination.restype = C.c_double
        L.ref_sim_mean_coordination.argtypes = [C.c_void_p]
        L.ref_sim_traces.restype = C.c_int64
        L.ref_sim_traces.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), PI, C.POINTER(C.c_uint8), C.c_int64]
        L.ref_model_report.argtypes = [C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_uint8), C.c_int,
                                       C.c_double, C.c_double, C.c_double, C.c_double, PD]
        L.ref_sim_table.restype = C.c_int64
        L.ref_sim_table.argtypes = [C.c_void_p, PU, PI, C.POINTER(C.c_uint8), PD, C.c_int64]
        L.ref_oracle_collide.restype = C.c_int64
        L.ref_oracle_collide.argtypes = [C.POINTER(orc_config), C.c_size_t, PU, PD, PD, PD, PD, PD, PU,
                                         C.POINTER(orc_grid), C.c_int64, PU, PI, PD, PD, PD, PU, PI, PD,
                                         PU, PU, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_brute_force_pairs.restype = C.c_int64
        L.ref_brute_force_pairs.argtypes = [C.c_size_t, PD, PD, PU, PU, C.c_int64]
        L.ref_restitution_alpha.restype = C.c_double
        L.ref_restitution_alpha.argtypes = [C.c_double]
        L.ref_contact_coefficients.argtypes = [C.c_double, C.POINTER(orc_material), C.POINTER(orc_material),
                                               C.c_double, C.c_double, C.c_double, C.c_double,
                                               C.c_double, C.c_int, PD]
        L.ref_contact_geometry.restype = C.c_int
        L.ref_contact_geometry.argtypes = [PD, C.c_double, PD, PD, PD, C.c_int, C.c_double, PD, PD, PD]
        L.ref_contact_force.argtypes = [PD, PD, PD, C.c_double, C.c_double, PD]
        L.ref_update_tangential.argtypes = [PD, PD, PD, C.c_double, PD]
        L.ref_make_grid.restype = C.c_int
        L.ref_make_grid.argtypes = [PD, PD, C.c_double, C.c_double, C.POINTER(orc_grid)]
        L.ref_calc_hash.restype = C.c_uint32
        L.ref_calc_hash.argtypes = [PD, C.POINTER(orc_grid), C.POINTER(C.c_int)]
        L.ref_neighbor_cells.restype = C.c_int
        L.ref_neighbor_cells.argtypes = [C.c_uint32, C.POINTER(orc_grid), PU]
        L.ref_closest_point_rect.argtypes = [PD, C.POINTER(orc_rect), PD]
        L.ref_closest_point_line.argtypes = [PD, C.POINTER(orc_line), PD]
        L.ref_parse_and_build.restype = C.c_int64
        L.ref_parse_and_build.argtypes = [C.c_char_p, C.POINTER(orc_config), C.POINTER(orc_material),
                                          C.POINTER(orc_rect), C.POINTER(orc_line), PU, PD, PD, PD, PD,
                                          PD, PU, C.POINTER(C.c_int64)]

    def set_threads(self, n):
        self.L.ref_set_threads(int(n))

    def model_report(self, offsets, contact, warp_size=32, c_check=1.0, c_force=20.0, c_store=1.0, c_load=1.0):
        """warp_model.cpp:118-136 over flattened traces -> dict."""
        offsets = np.ascontiguousarray(offsets, np.uint64)
        contact = np.ascontiguousarray(contact, np.uint8)
        out = np.zeros(5)
        self.L.ref_model_report(len(offsets) - 1, offsets.ctypes.data_as(C.POINTER(C.c_uint64)),
                                contact.ctypes.data_as(C.POINTER(C.c_uint8)), warp_size, c_check, c_force,
                                c_store, c_load, out.ctypes.data_as(PD))
        return {"cycles_baseline": out[0], "cycles_two_phase": out[1], "utilization_baseline": out[2],
                "utilization_two_phase": out[3], "warp_count": int(out[4])}

    def thread_count(self):
        return self.L.ref_thread_count()

    def last_error(self):
        return self.L.ref_last_error().decode(errors="replace")

    # pure functions, same signatures as Oracle
    def restitution_alpha(self, e):
        return self.L.ref_restitution_alpha(e)

    def contact_coefficients(self, dn, m1, m2, r1, r2, ma, mb, alpha, wall):
        out = (C.c_double * 4)()
        a = orc_material(*m1)
        b = orc_material(*m2)
        self.L.ref_contact_coefficients(dn, C.byref(a), C.byref(b), r1, r2, ma, mb, alpha, int(wall), out)
        return list(out)

    def contact_geometry(self, p1, r1, v1, w1, pp, wall, r2=0.0, v2=(0, 0, 0), w2=(0, 0, 0)):
        out = (C.c_double * 10)()
        rc = self.L.ref_contact_geometry(D3(*p1), r1, D3(*v1), D3(*w1), D3(*pp), int(wall), r2,
                                         D3(*v2), D3(*w2), out)
        return rc, list(out)

    def contact_force(self, geom, coeffs, delta, mu, r1):
        out = (C.c_double * 12)()
        self.L.ref_contact_force((C.c_double * 10)(*geom), (C.c_double * 4)(*coeffs), D3(*delta), mu, r1, out)
        return list(out)

    def update_tangential(self, old, n, vt, dt):
        out = D3()
        self.L.ref_update_tangential(D3(*old), D3(*n), D3(*vt), dt, out)
        return list(out)

    def make_grid(self, bmin, bmax, rmax, h=0.0):
        g = orc_grid()
        rc = self.L.ref_make_grid(D3(*bmin), D3(*bmax), rmax, h, C.byref(g))
        return rc, g

    def calc_hash(self, p, g):
        cl = C.c_int(0)
        k = self.L.ref_calc_hash(D3(*p), C.byref(g), C.byref(cl))
        return k, bool(cl.value)

    def neighbor_cells(self, cell, g):
        out = (C.c_uint32 * 27)()
        n = self.L.ref_neighbor_cells(cell, C.byref(g), out)
        return list(out)[:n]

    def closest_point_rect(self, p, corner, u, v):
        out = (C.c_double * 4)()
        w = orc_rect(D3(*corner), D3(*u), D3(*v), 0)
        self.L.ref_closest_point_rect(D3(*p), C.byref(w), out)
        return list(out)

    def closest_point_line(self, p, a, b):
        out = (C.c_double * 4)()
        w = orc_line(D3(*a), D3(*b), 0)
        self.L.ref_closest_point_line(D3(*p), C.byref(w), out)
        return list(out)

    def brute_force_pairs(self, positions, radii):
        pos = np.ascontiguousarray(positions, np.float64)
        rad = np.ascontiguousarray(radii, np.float64)
        n = len(rad)
        cap = max(16, 8 * n)
        oi = np.zeros(cap, np.uint32)
        oj = np.zeros(cap, np.uint32)
        c = self.L.ref_brute_force_pairs(n, pos.ctypes.data_as(PD), rad.ctypes.data_as(PD),
                                         oi.ctypes.data_as(PU), oj.ctypes.data_as(PU), cap)
        assert c <= cap
        return oi[:c].copy(), oj[:c].copy()

    def oracle_collide(self, state, cfg, grid, table):
        """Reference oracle_collide (oracle.cpp:47-105). table: (owner_slot[], partner[], dt[,3])
        live after the sweep. Returns forces, torques, (owner, partner, dt) touched rows, events."""
        n, keep, ptrs = _arr(state)
        cc = CConfig(cfg)
        io, ip, idt = table
        io = np.ascontiguousarray(io, np.uint32)
        ip = np.ascontiguousarray(ip, np.int32)
        idt = np.ascontiguousarray(idt, np.float64).reshape(-1, 3)
        cap = max(16, n * cfg.contact_capacity)
        f = np.zeros((n, 3))
        t = np.zeros((n, 3))
        oo = np.zeros(cap, np.uint32)
        op = np.zeros(cap, np.int32)
        od = np.zeros((cap, 3))
        eo = np.zeros(cap, np.uint32)
        ep = np.zeros(cap, np.uint32)
        nev = C.c_int64(0)
        c = self.L.ref_oracle_collide(C.byref(cc.c), n, *ptrs, C.byref(grid), len(io),
                                      io.ctypes.data_as(PU), ip.ctypes.data_as(PI), idt.ctypes.data_as(PD),
                                      f.ctypes.data_as(PD), t.ctypes.data_as(PD), oo.ctypes.data_as(PU),
                                      op.ctypes.data_as(PI), od.ctypes.data_as(PD), eo.ctypes.data_as(PU),
                                      ep.ctypes.data_as(PU), cap, C.byref(nev))
        if c < 0:
            raise OracleError(-c, msg=self.last_error())
        e = nev.value
        return f, t, (oo[:c].copy(), op[:c].copy(), od[:c].copy()), (eo[:e].copy(), ep[:e].copy())

    def parse_and_build(self, text: str):
        """Reference parse_config_text + build_initial_state (config_io.cpp, lattice.cpp:46-129)."""
        cfg = orc_config()
        steps = C.c_int64(0)
        n = self.L.ref_parse_and_build(text.encode(), C.byref(cfg), None, None, None, None, None, None,
                                       None, None, None, None, C.byref(steps))
        if n < 0:
            raise OracleError(-n, msg=self.last_error())
        mats = (orc_material * max(cfg.material_count, 1))()
        rects = (orc_rect * max(cfg.rect_count, 1))()
        lines = (orc_line * max(cfg.line_count, 1))()
        s = State(n)
        self.L.ref_parse_and_build(text.encode(), C.byref(cfg), mats, rects, lines, *s.ptrs(), C.byref(steps))
        return cfg, list(mats[:cfg.material_count]), list(rects[:cfg.rect_count]), \
            list(lines[:cfg.line_count]), s, steps.value


class RefSim:
    """demforge::Simulation (pipeline.hpp:62-136) through the shim."""

    def __init__(self, ref: RefLib, state, cfg, _h=None):
        self.r = ref
        self.cfg = cfg
        if _h is not None:
            self.h = _h
        else:
            self.cc = CConfig(cfg)
            n, keep, ptrs = _arr(state)
            code = C.c_int(0)
            self.h = ref.L.ref_sim_create(C.byref(self.cc.c), n, *ptrs, C.byref(code))
            if not self.h:
                raise OracleError(code.value, msg=ref.last_error())
        self.n = ref.L.ref_sim_size(self.h)
        ref.L.ref_sim_set_record_traces(self.h, 0)

    def __del__(self):
        if getattr(self, "h", None):
            self.r.L.ref_sim_destroy(self.h)
            self.h = None

    def clone(self):
        return RefSim(self.r, None, self.cfg, _h=self.r.L.ref_sim_clone(self.h))

    def step(self, k=1):
        m = orc_metrics()
        rc = self.r.L.ref_sim_step(self.h, k, C.byref(m))
        if rc:
            raise OracleError(rc, msg=self.r.last_error())
        return m

    def run_kernel(self, which, variant=1):
        rc = self.r.L.ref_sim_run_kernel(self.h, which, variant)
        if rc:
            raise OracleError(rc, msg=self.r.last_error())

    def advance_to_collide(self):  # tests/test_pipeline.cpp:69-76
        for k in (0, 1, 2, 3, 4, 6):
            self.run_kernel(k)

    def state(self):
        s = State(self.n)
        self.r.L.ref_sim_get_state(self.h, *s.ptrs())
        return s

    def forces(self):
        f = np.zeros((self.n, 3))
        t = np.zeros((self.n, 3))
        self.r.L.ref_sim_get_forces(self.h, f.ctypes.data_as(PD), t.ctypes.data_as(PD))
        return f, t

    def grid(self):
        g = orc_grid()
        self.r.L.ref_sim_get_grid(self.h, C.byref(g))
        return g

    def traces(self):
        """(offsets[n+1], candidate slots, contact flags) of the last traced kernel_collide."""
        total = self.r.L.ref_sim_traces(self.h, None, None, None, 0)
        off = np.zeros(self.n + 1, np.uint64)
        cand = np.zeros(max(total, 1), np.int32)
        hit = np.zeros(max(total, 1), np.uint8)
        self.r.L.ref_sim_traces(self.h, off.ctypes.data_as(C.POINTER(C.c_uint64)), cand.ctypes.data_as(PI),
                                hit.ctypes.data_as(C.POINTER(C.c_uint8)), total)
        return off, cand[:total], hit[:total].astype(bool)

    def table(self):
        cap = int(self.n) * self.cfg.contact_capacity + 16
        o = np.zeros(cap, np.uint32)
        p = np.zeros(cap, np.int32)
        tch = np.zeros(cap, np.uint8)
        d = np.zeros((cap, 3))
        c = self.r.L.ref_sim_table(self.h, o.ctypes.data_as(PU), p.ctypes.data_as(PI),
                                   tch.ctypes.data_as(C.POINTER(C.c_uint8)), d.ctypes.data_as(PD), cap)
        return o[:c].copy(), p[:c].copy(), tch[:c].astype(bool), d[:c].copy()


def have_ref() -> bool:
    return os.path.exists(REF_SO)
