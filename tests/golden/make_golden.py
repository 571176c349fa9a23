#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libdemforge_ref.so, compiled from
/root/reference/proj/core/src by oracle/Makefile). The committed .npz/.json files let the CPU
oracle be pinned on machines without the reference sources (the GPU box).

  python tests/golden/make_golden.py

Fixtures:
  physics_vectors.npz   random inputs + reference outputs of contact_geometry,
                        contact_coefficients_with_alpha, contact_force, update_tangential
                        (contact_mechanics.cpp, geometry.cpp), bitwise
  collide_n{64,125}_s*.npz  a reference Simulation advanced to the pre-collide point
                        (tests/test_pipeline.cpp:69-76), its post-sweep table, and the reference
                        oracle_collide output (forces, torques, touched table, events)
  config1.npz           reference parse_config_text + build_initial_state of the SURVEY App. B
                        settle config (4,096 particles, 5 walls) + 20-step reference end state
  step_n125_s31.npz     initial state + reference state/forces after 10 step() calls
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import RefLib, RefSim  # noqa: E402
from helpers import basic_config, box_for, random_dense_state  # noqa: E402

CONFIG1 = """dt = 1e-4
gravity.x = 0
gravity.y = 0
gravity.z = -9.81
domain.min.x = 0
domain.min.y = 0
domain.min.z = 0
domain.max.x = 0.2
domain.max.y = 0.2
domain.max.z = 0.4
seed = 42
particles.count = 4096
particles.radius = 0.005
particles.mass = 1.309e-3
particles.material = bead
particles.init = lattice
particles.lattice_spacing = 0.011
material.bead.poisson = 0.3
material.bead.shear_modulus = 3.85e5
material.bead.youngs_modulus = 1e6
material.bead.restitution = 0.9
material.bead.mu_d = 0.3
material.wall.poisson = 0.3
material.wall.shear_modulus = 3.85e5
material.wall.youngs_modulus = 1e6
material.wall.restitution = 0.9
material.wall.mu_d = 0.3
wall.rect.0.corner = 0 0 0
wall.rect.0.edge_u = 0.2 0 0
wall.rect.0.edge_v = 0 0.2 0
wall.rect.0.material = wall
wall.rect.1.corner = 0 0 0
wall.rect.1.edge_u = 0 0.2 0
wall.rect.1.edge_v = 0 0 0.4
wall.rect.1.material = wall
wall.rect.2.corner = 0.2 0 0
wall.rect.2.edge_u = 0 0.2 0
wall.rect.2.edge_v = 0 0 0.4
wall.rect.2.material = wall
wall.rect.3.corner = 0 0 0
wall.rect.3.edge_u = 0.2 0 0
wall.rect.3.edge_v = 0 0 0.4
wall.rect.3.material = wall
wall.rect.4.corner = 0 0.2 0
wall.rect.4.edge_u = 0.2 0 0
wall.rect.4.edge_v = 0 0 0.4
wall.rect.4.material = wall
run.steps = 1000
run.collide_variant = two_phase
"""

MAT = (0.3, 4e4, 1e5, 0.9, 0.3)


def physics_vectors(ref, n=400, seed=123):
    rng = np.random.default_rng(seed)
    rows_in, rows_geom, rows_coef, rows_force, rows_ut = [], [], [], [], []
    for it in range(n):
        p1 = rng.uniform(-1, 1, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        r1, r2 = 0.8 + 0.4 * rng.random(), 0.8 + 0.4 * rng.random()
        wall = it % 7 == 0
        p2 = p1 + d * (rng.uniform(0.5, 0.99) * (r1 if wall else r1 + r2))
        v1, v2, w1, w2 = (rng.uniform(-1, 1, 3) for _ in range(4))
        m1, m2 = 1 + rng.random(), 1 + rng.random()
        rc, g = ref.contact_geometry(p1, r1, v1, w1, p2, wall, r2, v2, w2)
        assert rc == 1
        alpha = ref.restitution_alpha(0.5 + 0.5 * rng.random())
        mat2 = (0.2 + 0.2 * rng.random(), 3e4 + 2e4 * rng.random(), 1e5, 0.9, 0.3)
        co = ref.contact_coefficients(g[3], MAT, mat2, r1, r2, m1, m2, alpha, wall)
        delta = rng.uniform(-0.05, 0.05, 3)
        mu = [0.3, 1e-4, 0.0][it % 3]
        ut = ref.update_tangential(delta, g[:3], g[7:10], 1e-3)
        f = ref.contact_force(g, co, ut, mu, r1)
        rows_in.append(np.concatenate([p1, [r1], v1, w1, p2, [r2], v2, w2, [m1, m2, float(wall), alpha],
                                       mat2, delta, [mu]]))
        rows_geom.append(g)
        rows_coef.append(co)
        rows_ut.append(ut)
        rows_force.append(f)
    np.savez_compressed(os.path.join(HERE, "physics_vectors.npz"), inputs=np.array(rows_in),
                        geom=np.array(rows_geom), coef=np.array(rows_coef),
                        ut=np.array(rows_ut), force=np.array(rows_force))


def collide_fixture(ref, n, seed, rounds=2):
    cfg = basic_config(box_for(n))
    sim = RefSim(ref, random_dense_state(n, seed), cfg)
    for _ in range(rounds):
        sim.advance_to_collide()
    st = sim.state()
    o, p, tch, d = sim.table()
    g = sim.grid()
    f, t, tab, ev = ref.oracle_collide(st, cfg, g, (o, p, d))
    np.savez_compressed(
        os.path.join(HERE, f"collide_n{n}_s{seed}.npz"),
        box=box_for(n), ids=st.ids, pos=st.positions, vel=st.velocities, omg=st.angular_velocities,
        rad=st.radii, mass=st.masses, mat=st.material_ids,
        grid=np.array([g.origin[0], g.origin[1], g.origin[2], g.cell_size, g.nx, g.ny, g.nz]),
        tin_owner=o, tin_partner=p, tin_dt=d, forces=f, torques=t, tout_owner=tab[0],
        tout_partner=tab[1], tout_dt=tab[2], ev_owner=ev[0], ev_partner=ev[1])


def config1_fixture(ref, steps=20):
    cfg, mats, rects, lines, st, nsteps = ref.parse_and_build(CONFIG1)
    from paper_1503_03553_b200.simulation import MaterialParams, RectWall, SimConfig
    sc = SimConfig()
    sc.dt = cfg.dt
    sc.gravity = tuple(cfg.gravity)
    sc.domain_min = tuple(cfg.domain_min)
    sc.domain_max = tuple(cfg.domain_max)
    for k, m in enumerate(mats):
        sc.materials.add(f"m{k}", MaterialParams(m.poisson_ratio, m.shear_modulus, m.youngs_modulus,
                                                 m.restitution, m.sliding_friction))
    sc.rect_walls = [RectWall(tuple(w.corner), tuple(w.edge_u), tuple(w.edge_v), w.material_id) for w in rects]
    sc.contact_capacity = cfg.contact_capacity
    sim = RefSim(ref, st, sc)
    ke, coord = [], []
    for _ in range(steps):
        m = sim.step()
        s2 = sim.state()
        ke.append(float((0.5 * s2.masses * (s2.velocities ** 2).sum(1)).sum()
                        + (0.5 * 0.4 * s2.masses * s2.radii ** 2 * (s2.angular_velocities ** 2).sum(1)).sum()))
        coord.append(m.pp_contact_events / len(s2.ids))
    end = sim.state()
    f, t = sim.forces()
    walls = np.array([list(w.corner) + list(w.edge_u) + list(w.edge_v) + [w.material_id] for w in rects])
    matarr = np.array([[m.poisson_ratio, m.shear_modulus, m.youngs_modulus, m.restitution, m.sliding_friction]
                       for m in mats])
    np.savez_compressed(
        os.path.join(HERE, "config1.npz"), dt=cfg.dt, gravity=np.array(cfg.gravity),
        domain_min=np.array(cfg.domain_min), domain_max=np.array(cfg.domain_max), walls=walls,
        materials=matarr, capacity=cfg.contact_capacity, run_steps=nsteps,
        ids=st.ids, pos=st.positions, vel=st.velocities, omg=st.angular_velocities, rad=st.radii,
        mass=st.masses, mat=st.material_ids, steps=steps, end_ids=end.ids, end_pos=end.positions,
        end_vel=end.velocities, end_omg=end.angular_velocities, end_f=f, end_t=t,
        ke=np.array(ke), coord=np.array(coord))


def step_fixture(ref, n=125, seed=31, steps=10):
    cfg = basic_config(box_for(n))
    st0 = random_dense_state(n, seed)
    sim = RefSim(ref, st0, cfg)
    sim.step(steps)
    st = sim.state()
    f, t = sim.forces()
    np.savez_compressed(
        os.path.join(HERE, f"step_n{n}_s{seed}.npz"), box=box_for(n), steps=steps,
        ids=st0.ids, pos=st0.positions, vel=st0.velocities, omg=st0.angular_velocities,
        rad=st0.radii, mass=st0.masses, end_ids=st.ids, end_pos=st.positions,
        end_vel=st.velocities, end_omg=st.angular_velocities, end_f=f, end_t=t)


def main():
    ref = RefLib()
    ref.set_threads(1)
    physics_vectors(ref)
    for n, seeds in ((64, (1, 2, 3)), (125, (7,))):
        for s in seeds:
            collide_fixture(ref, n, s)
    config1_fixture(ref)
    step_fixture(ref)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
